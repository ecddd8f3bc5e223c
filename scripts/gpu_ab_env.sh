# A/B of a runtime knob on one box: gpu_ab_env.sh VAR "v1 v2 ..." [tests-k-expr]
cd ${GRAFT_REPO_ROOT:-.}
VAR=$1; VALS=$2; T=gpurun_out/ab_${VAR}; mkdir -p $T
if [ -n "$3" ]; then for v in $VALS; do env $VAR=$v timeout 900 python -m pytest tests -m gpu -q -x -k "$3" > $T/tests_$v.log 2>&1; echo "$VAR=$v tests rc=$?" >> $T/summary.txt; done; fi
for rep in 1 2; do for v in $VALS; do
  env $VAR=$v python bench.py --steps 40 --no-e2e --no-cpu-baseline --no-secondary > $T/bench_$v.log 2>&1
  python -c "
import json
for l in open('$T/bench_$v.log'):
    if l.startswith('{'):
        d=json.loads(l); print('$VAR=$v', round(d['ms_per_step'],4), 'depth', round(d['phases_ms']['depth'],4), 'frac', round(d['roofline']['frac'],3), 'culled', round(d['tile_culled']['depth_ms'],4))" >> $T/summary.txt
  env $VAR=$v python scripts/run_config.py 2 6 2>&1 | tail -2 | head -1 | sed "s/^/$VAR=$v /" >> $T/summary.txt
  env $VAR=$v python scripts/run_config.py 4 3 2>&1 | tail -2 | head -1 | sed "s/^/$VAR=$v /" >> $T/summary.txt
  env $VAR=$v python scripts/run_config.py 1 8 2>&1 | tail -2 | head -1 | sed "s/^/$VAR=$v /" >> $T/summary.txt
done; done
