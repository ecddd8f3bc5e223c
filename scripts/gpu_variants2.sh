# headline + configs[4] forward per tuning variant: gpu_variants2.sh name...
for v in "$@"; do
  ADOP_LIB=paper_2110_06635_b200/libadop_$v.so python bench.py --steps 40 --no-e2e --no-cpu-baseline --no-secondary > gpurun_out/var_$v.log 2>&1
  python -c "
import json
for l in open('gpurun_out/var_$v.log'):
    if l.startswith('{'):
        d=json.loads(l); print('$v', round(d['ms_per_step'],4), 'depth', round(d['phases_ms']['depth'],4), 'culled', round(d['tile_culled']['depth_ms'],4))"
  ADOP_LIB=paper_2110_06635_b200/libadop_$v.so python scripts/run_config.py 4 3 2>&1 | tail -2 | head -1
  ADOP_LIB=paper_2110_06635_b200/libadop_$v.so python scripts/run_config.py 2 4 2>&1 | tail -2 | head -1
done
