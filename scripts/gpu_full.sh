# full round check: all gpu tests, smoke, default bench (with e2e, cpu baseline, secondary), launch list
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${1:-full}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${T}_nvsmi.txt 2>&1
timeout 300 python __graft_entry__.py --smoke > gpurun_out/${T}_smoke.log 2>&1; echo smoke=$? >> gpurun_out/${T}_status.txt
timeout 2400 python -m pytest tests -m gpu -q --timeout 1200 > gpurun_out/${T}_tests.log 2>&1; echo tests=$? >> gpurun_out/${T}_status.txt
timeout 900 python bench.py > gpurun_out/${T}_bench.log 2>&1; echo bench=$? >> gpurun_out/${T}_status.txt
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary"
$CMD > gpurun_out/${T}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:'k_|nccl' --csv --log-file gpurun_out/${T}_launches.csv $CMD > gpurun_out/${T}_ncu_launches.log 2>&1
echo done >> gpurun_out/${T}_status.txt
