# launch lists (ncu, cold, serialised) of configs[1] and configs[0] forwards.  usage: gpu_small_launches.sh TAG
cd ${GRAFT_REPO_ROOT:-.}
T=gpurun_out/small_$1; mkdir -p $T
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
python scripts/phase_probe.py 1 > $T/phase1.txt 2>&1
python scripts/phase_probe.py 0 > $T/phase0.txt 2>&1
ncu --metrics $M --clock-control none -k regex:'^k_' -c 40 --csv --log-file $T/launches_cfg1.csv python scripts/run_config.py 1 3 > $T/ncu1.log 2>&1
ncu --metrics $M --clock-control none -k regex:'^k_' -c 40 --csv --log-file $T/launches_cfg0.csv python scripts/run_config.py 0 3 > $T/ncu0.log 2>&1
