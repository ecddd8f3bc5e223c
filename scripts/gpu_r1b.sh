cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 -x > gpurun_out/gpu_tests.log 2>&1; echo tests=$? >> gpurun_out/status.txt
bash scripts/gpu_prof.sh r1a
