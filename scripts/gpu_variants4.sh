# per variant: headline, configs[1] / [4] / [2] (fwd, bwd).  usage: gpu_variants4.sh name...
for v in "$@"; do
  ADOP_LIB=paper_2110_06635_b200/libadop_$v.so python bench.py --steps 40 --no-e2e --no-cpu-baseline --no-secondary > gpurun_out/var_$v.log 2>&1
  python -c "
import json
for l in open('gpurun_out/var_$v.log'):
    if l.startswith('{'):
        d=json.loads(l); p=d['phases_ms']; print('$v', round(d['ms_per_step'],4), 'depth', round(p['depth'],4))"
  for c in 1 4 2; do ADOP_LIB=paper_2110_06635_b200/libadop_$v.so python scripts/run_config.py $c 6 2>&1 | tail -2 | head -1; done
done
