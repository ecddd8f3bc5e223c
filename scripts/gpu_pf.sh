timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/gputests.log
bash scripts/gpu_variants.sh nopf > gpurun_out/variants.txt 2>&1
python bench.py --steps 40 --no-e2e --no-cpu-baseline --no-secondary > gpurun_out/bench_quick.log 2>&1
python -c "
import json
for l in open('gpurun_out/bench_quick.log'):
    if l.startswith('{'):
        d=json.loads(l); print('prefilter', round(d['ms_per_step'],4), {k: round(x,4) for k,x in d['phases_ms'].items() if k in ('depth','blend','resolve')}, 'frac', round(d['roofline']['frac'],3), 'culled', round(d['tile_culled']['depth_ms'],4), round(d['tile_culled']['ms_per_step'],4))" >> gpurun_out/variants.txt
python scripts/run_config.py 2 4 >> gpurun_out/variants.txt 2>&1
python scripts/run_config.py 4 2 >> gpurun_out/variants.txt 2>&1
