# ncu --set full of the configs[4] depth sweep with the forward ghost listing off / on
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for g in 0 1; do
  ADOP_GHOST_FWD=$g ncu --set full --clock-control none --import-source on -k regex:'^k_depth_pool' -s 1 -c 1 \
    -o /tmp/c4d_$g python scripts/run_config.py 4 2 > gpurun_out/ncu_c4d_$g.log 2>&1
  bash scripts/ncu_stalls.sh /tmp/c4d_$g.ncu-rep > gpurun_out/c4d_${g}_stalls.txt 2>&1
  python scripts/ncu_lines_cuda.py /tmp/c4d_$g.ncu-rep 50 > gpurun_out/c4d_${g}_lines.txt 2>&1
  python scripts/ncu_lines.py /tmp/c4d_$g.ncu-rep 40 > gpurun_out/c4d_${g}_sass.txt 2>&1
done
