# per tuning variant: headline frame / depth / blend phase, configs[4] and configs[2] fwd/bwd.  usage: gpu_variants3.sh name...
for v in "$@"; do
  ADOP_LIB=paper_2110_06635_b200/libadop_$v.so python bench.py --steps 40 --no-e2e --no-cpu-baseline --no-secondary > gpurun_out/var_$v.log 2>&1
  python -c "
import json
for l in open('gpurun_out/var_$v.log'):
    if l.startswith('{'):
        d=json.loads(l); p=d['phases_ms']; print('$v', round(d['ms_per_step'],4), 'depth', round(p['depth'],4), 'blend', round(p['blend'],4), 'resolve', round(p['resolve'],4))"
  ADOP_LIB=paper_2110_06635_b200/libadop_$v.so python scripts/run_config.py 4 3 2>&1 | tail -2 | head -1
  ADOP_LIB=paper_2110_06635_b200/libadop_$v.so python scripts/run_config.py 2 4 2>&1 | tail -2 | head -1
done
