# GPU parity tests, then per-config timings and launch lists of our kernels.  usage: gpu_check.sh [notests]
if [ "$1" != "notests" ]; then
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo tests=$? >> gpurun_out/gputests.log
tail -3 gpurun_out/gputests.log
fi
python scripts/run_config.py 2 5 > gpurun_out/cfg2.log 2>&1
python scripts/run_config.py 4 3 > gpurun_out/cfg4.log 2>&1
python bench.py --steps 30 --no-e2e --no-cpu-baseline --no-secondary > gpurun_out/bench_quick.log 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
ncu --metrics $M --clock-control none -k regex:'^k_' -c 60 --csv --log-file gpurun_out/launches_cfg2.csv \
  python scripts/run_config.py 2 3 > gpurun_out/ncu2.log 2>&1
ncu --metrics $M --clock-control none -k regex:'^k_' -c 60 --csv --log-file gpurun_out/launches_cfg4.csv \
  python scripts/run_config.py 4 2 > gpurun_out/ncu4.log 2>&1
ncu --metrics $M --clock-control none -k regex:'^k_' -c 40 --csv --log-file gpurun_out/launches_cfg3.csv \
  python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary > gpurun_out/ncu3.log 2>&1
