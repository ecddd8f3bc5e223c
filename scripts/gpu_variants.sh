# quick headline bench for each tuning variant: gpu_variants.sh name...
for v in "$@"; do
  ADOP_LIB=paper_2110_06635_b200/libadop_$v.so python bench.py --steps 40 --no-e2e --no-cpu-baseline --no-secondary > gpurun_out/var_$v.log 2>&1
  python -c "
import json,sys
for l in open('gpurun_out/var_$v.log'):
    if l.startswith('{'):
        d=json.loads(l); print('$v', round(d['ms_per_step'],4), {k: round(x,4) for k,x in d['phases_ms'].items() if k in ('depth','blend','resolve')}, 'frac', round(d['roofline']['frac'],3))"
done
