# headline-only A/B (bench.py, 60 steps) of the listed variants in both orders, twice.  usage: gpu_ab_head.sh name...
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out; : > gpurun_out/ab_head.txt
REV=$(printf '%s\n' "$@" | tac | tr '\n' ' ')
for order in "$*" "$REV" "$*"; do
  for v in $order; do
    ADOP_LIB=paper_2110_06635_b200/libadop_$v.so python bench.py --steps 60 --no-e2e --no-cpu-baseline --no-secondary > gpurun_out/head_$v.log 2>&1
    python -c "
import json
for l in open('gpurun_out/head_$v.log'):
    if l.startswith('{'):
        d=json.loads(l); p=d['phases_ms']; print('$v', round(d['ms_per_step'],4), 'median', round(d['ms_per_step_stats']['median'],4), 'depth', round(p['depth'],4), 'blend', round(p['blend'],4), 'frac', round(d['roofline']['frac'],4))" >> gpurun_out/ab_head.txt
  done
done
echo done >> gpurun_out/ab_head.txt
