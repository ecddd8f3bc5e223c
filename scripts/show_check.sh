grep -E "FAILED|passed|failed" gpurun_out/gputests.log
cat gpurun_out/cfg2.log gpurun_out/cfg4.log | grep -v "^record"
python -c "
import json
for l in open('gpurun_out/bench_quick.log'):
    if l.startswith('{'):
        d=json.loads(l); print('bench', round(d['ms_per_step'],4), 'ms', {k: round(v,4) for k,v in d['phases_ms'].items()}, 'frac', round(d['roofline']['frac'],3))"
for c in 3 2 4; do echo "== cfg$c"; python scripts/launch_table.py gpurun_out/launches_cfg$c.csv; done
