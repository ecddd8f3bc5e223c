# Round-2 profile: ncu --set full of the hot kernels (configs[3] depth / blend, configs[4] depth / blend / ghost)
# and an L2-atomics metric list of every kernel of configs[3] and configs[4].  usage: gpu_prof2.sh TAG
cd ${GRAFT_REPO_ROOT:-.}
T=gpurun_out/prof2_$1; mkdir -p $T
B3="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary"
$B3 > $T/bench3.log 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_op_red.sum,lts__t_sectors_op_atom.sum,lts__t_requests_op_red.sum,lts__t_sector_hit_rate.pct,lts__t_sector_op_red_hit_rate.pct,smsp__inst_executed.sum
ncu --metrics $M --clock-control none -k regex:'^k_' -c 40 --csv --log-file $T/atom_cfg3.csv $B3 > $T/ncu_a3.log 2>&1
ncu --metrics $M --clock-control none -k regex:'^k_' -c 60 --csv --log-file $T/atom_cfg4.csv python scripts/run_config.py 4 2 > $T/ncu_a4.log 2>&1
full() {  # name kernel-regex skip command...
  local name=$1 kre=$2 skip=$3; shift 3
  mkdir -p /tmp/prof; ncu --set full --clock-control none --import-source on -k regex:"$kre" -s $skip -c 1 -f -o /tmp/prof/$name "$@" > $T/ncu_$name.log 2>&1
  python scripts/ncu_summary.py /tmp/prof/$name.ncu-rep 30 > $T/${name}_summary.txt 2>&1
  bash scripts/ncu_stalls.sh /tmp/prof/$name.ncu-rep > $T/${name}_stalls.txt 2>&1
  python scripts/ncu_lines_cuda.py /tmp/prof/$name.ncu-rep 45 > $T/${name}_lines.txt 2>&1
}
full cfg3_depth '^k_depth_async' 3 $B3
full cfg3_blend '^k_blend' 3 $B3
full cfg4_depth '^k_depth_async' 1 python scripts/run_config.py 4 2
full cfg4_blend '^k_blend' 1 python scripts/run_config.py 4 2
full cfg4_ghost '^k_bwd_ghost' 1 python scripts/run_config.py 4 2
rm -f $T/*.ncu-rep.tmp
echo done > $T/status.txt
