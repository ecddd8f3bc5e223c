# quick iteration: parity subset, bench headline, profile of the top kernel
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${1:-it}
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -k "${2:-not full}" > gpurun_out/${T}_tests.log 2>&1; echo tests=$? >> gpurun_out/${T}_status.txt
timeout 600 python bench.py --steps 50 --warmup 5 --no-e2e --no-cpu-baseline ${3:-} > gpurun_out/${T}_bench.log 2>&1; echo bench=$? >> gpurun_out/${T}_status.txt
bash scripts/gpu_prof.sh ${T} ${4:-k_depth}
