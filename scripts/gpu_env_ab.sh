# GPU suite, then configs[2] / configs[4] fwd+bwd and the headline with an environment switch off and on:
# gpu_env_ab.sh VAR   (runs VAR=0 and VAR=1, twice, alternating)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
V=$1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/envab_tests.log 2>&1
echo tests=$? > gpurun_out/envab_status.txt
for rep in 1 2; do
  for val in 0 1; do
    echo "== $V=$val" >> gpurun_out/envab.txt
    env $V=$val python scripts/run_config.py 4 3 2>&1 | tail -2 | head -1 >> gpurun_out/envab.txt
    env $V=$val python scripts/run_config.py 2 4 2>&1 | tail -2 | head -1 >> gpurun_out/envab.txt
  done
done
echo done >> gpurun_out/envab_status.txt
# headline: this build vs the listed variants
for v in ${@:2}; do
  ADOP_LIB=paper_2110_06635_b200/libadop_$v.so python bench.py --steps 40 --no-e2e --no-cpu-baseline --no-secondary > gpurun_out/envab_$v.log 2>&1
  python -c "
import json
for l in open('gpurun_out/envab_$v.log'):
    if l.startswith('{'):
        d=json.loads(l); p=d['phases_ms']; print('$v', round(d['ms_per_step'],4), 'depth', round(p['depth'],4), 'blend', round(p['blend'],4))" >> gpurun_out/envab.txt
done
