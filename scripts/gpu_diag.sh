# depth-pass timing diagnostics: the stream micro-benchmark and ADOP_DIAG variants (wrong results, timing only)
# usage: gpu_diag.sh variant...
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
./scripts/micro/stream_read > gpurun_out/diag_micro.txt 2>&1
for v in "$@"; do
  ADOP_LIB=paper_2110_06635_b200/libadop_$v.so python bench.py --steps 40 --no-e2e --no-cpu-baseline --no-secondary > gpurun_out/diag_$v.log 2>&1
  python -c "
import json
for l in open('gpurun_out/diag_$v.log'):
    if l.startswith('{'):
        d=json.loads(l); p=d['phases_ms']; print('$v', round(d['ms_per_step'],4), 'depth', round(p['depth'],4), 'blend', round(p['blend'],4))" >> gpurun_out/diag.txt
done
