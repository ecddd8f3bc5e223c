# A/B of two library builds on one box: gpu_ab_lib.sh "nameA nameB" [tests-k-expr]  (libadop_<name>.so)
cd ${GRAFT_REPO_ROOT:-.}
T=gpurun_out/ablib; mkdir -p $T
if [ -n "$2" ]; then timeout 1500 python -m pytest tests -m gpu -q -k "$2" > $T/tests.log 2>&1; echo "tests rc=$?" >> $T/summary.txt; tail -2 $T/tests.log >> $T/summary.txt; fi
for rep in 1 2; do for v in $1; do
  L=paper_2110_06635_b200/libadop_$v.so
  ADOP_LIB=$L python bench.py --steps 40 --no-e2e --no-cpu-baseline --no-secondary > $T/bench_$v.log 2>&1
  python -c "
import json
for l in open('$T/bench_$v.log'):
    if l.startswith('{'):
        d=json.loads(l); print('$v', round(d['ms_per_step'],4), 'depth', round(d['phases_ms']['depth'],4), 'frac', round(d['roofline']['frac'],3), 'culled', round(d['tile_culled']['depth_ms'],4))" >> $T/summary.txt
  for c in "2 6" "4 3" "1 8"; do ADOP_LIB=$L python scripts/run_config.py $c 2>&1 | tail -2 | head -1 | sed "s/^/$v /" >> $T/summary.txt; done
done; done
