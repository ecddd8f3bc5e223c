# per-kernel launch lists (cold-cache, serialised) of the headline bench and the fwd+bwd configs
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
python scripts/run_config.py 2 5 > gpurun_out/cfg2.log 2>&1
python scripts/run_config.py 4 3 > gpurun_out/cfg4.log 2>&1
ncu --metrics $M --clock-control none -k regex:'^k_' -c 40 --csv --log-file gpurun_out/launches_cfg3.csv \
  python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary > gpurun_out/ncu3.log 2>&1
ncu --metrics $M --clock-control none -k regex:'^k_' -c 60 --csv --log-file gpurun_out/launches_cfg2.csv \
  python scripts/run_config.py 2 3 > gpurun_out/ncu2.log 2>&1
ncu --metrics $M --clock-control none -k regex:'^k_' -c 60 --csv --log-file gpurun_out/launches_cfg4.csv \
  python scripts/run_config.py 4 2 > gpurun_out/ncu4.log 2>&1
