# Round profile: bench line, per-kernel launch lists (configs 3, 2, 4) and ncu --set full of the top kernels.
# usage: gpu_profile.sh TAG   (outputs under gpurun_out/prof_TAG/)
T=gpurun_out/prof_$1; mkdir -p $T
python bench.py > $T/bench.log 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
ncu --metrics $M --clock-control none -k regex:'^k_' -c 40 --csv --log-file $T/launches_cfg3.csv \
  python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary > $T/ncu3.log 2>&1
ncu --metrics $M --clock-control none -k regex:'^k_' -c 60 --csv --log-file $T/launches_cfg2.csv \
  python scripts/run_config.py 2 3 > $T/ncu2.log 2>&1
ncu --metrics $M --clock-control none -k regex:'^k_' -c 60 --csv --log-file $T/launches_cfg4.csv \
  python scripts/run_config.py 4 2 > $T/ncu4.log 2>&1
full() {  # name kernel-regex skip command...
  local name=$1 kre=$2 skip=$3; shift 3
  ncu --set full --clock-control none --import-source on -k regex:"$kre" -s $skip -c 1 -o /tmp/$name "$@" > $T/ncu_$name.log 2>&1
  python scripts/ncu_summary.py /tmp/$name.ncu-rep 30 > $T/${name}_summary.txt 2>&1
  bash scripts/ncu_stalls.sh /tmp/$name.ncu-rep > $T/${name}_stalls.txt 2>&1
  python scripts/ncu_lines_cuda.py /tmp/$name.ncu-rep 40 > $T/${name}_lines.txt 2>&1
}
full cfg3_depth '^k_depth_(pool|async)' 3 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary
full cfg3_blend '^k_blend' 3 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary
full cfg2_ghost '^k_bwd_ghost' 3 python scripts/run_config.py 2 5
full cfg4_ghost '^k_bwd_ghost' 1 python scripts/run_config.py 4 2
full cfg2_tex '^k_bwd_tex' 3 python scripts/run_config.py 2 5
full cfg4_depth '^k_depth_(pool|async)' 0 python scripts/run_config.py 4 1
