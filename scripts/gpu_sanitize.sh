# compute-sanitizer (memcheck, racecheck, synccheck, initcheck) over the small GPU tests that cover every
# kernel family: tiny config fwd+bwd, reduced room configs (1 / 4 / 16 views), record overflow -> re-stream,
# backward work-list overflow -> inline, forward lists reused or re-swept by the backward, the backward side
# stream under CUDA-graph capture, and the two-process IPC (peer-memory) reduction.
# usage: gpu_sanitize.sh [TAG]   -> gpurun_out/sanitizer_TAG/<tool>.log
cd ${GRAFT_REPO_ROOT:-.}
T=gpurun_out/sanitizer_${1:-r02}; mkdir -p $T
SEL="tiny_config or room_configs_reduced or record_overflow or work_lists_overflow or consumes_forward_lists or captured_in_a_cuda_graph or empty_cloud or channels_scalar or fisheye_fwd_bwd"
CS="compute-sanitizer --error-exitcode 99 --print-limit 50 --target-processes all"
run() {  # tool extra-args test-selection file
  local tool=$1 extra=$2 sel=$3 f=$4
  timeout 1500 $CS --tool $tool $extra python -m pytest -q -m gpu -x -p no:cacheprovider "$f" -k "$sel" \
    > $T/$tool.log 2>&1
  echo "$tool rc=$?" >> $T/status.txt
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed" $T/$tool.log | tail -4 >> $T/status.txt
}
nvidia-smi --query-gpu=name,driver_version --format=csv,noheader > $T/status.txt
compute-sanitizer --version | tail -1 >> $T/status.txt
run memcheck "--leak-check full" "$SEL" tests/test_gpu_parity.py
run racecheck "--racecheck-report hazard" "tiny_config or room_configs_reduced or consumes_forward_lists or record_overflow" tests/test_gpu_parity.py
run synccheck "" "tiny_config or room_configs_reduced or consumes_forward_lists" tests/test_gpu_parity.py
run initcheck "" "tiny_config or room_configs_reduced" tests/test_gpu_parity.py
timeout 900 $CS --tool memcheck python -m pytest -q -m gpu -x -p no:cacheprovider tests/test_gpu_p2p.py > $T/memcheck_ipc.log 2>&1
echo "memcheck_ipc rc=$?" >> $T/status.txt
grep -E "ERROR SUMMARY|passed|failed" $T/memcheck_ipc.log | tail -4 >> $T/status.txt
echo done >> $T/status.txt
