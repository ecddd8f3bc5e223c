# ncu --set full reports (with source) of the configs[4] kernels, brought back gzipped.  usage: gpu_cfg4_reps.sh TAG
cd ${GRAFT_REPO_ROOT:-.}
T=gpurun_out/c4reps_$1; mkdir -p $T
for k in k_blend k_bwd_tex k_bwd_ghost k_depth_pool; do
  s=1; [ $k = k_depth_pool ] && s=0
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^$k" -s $s -c 1 -o /tmp/$k \
    python scripts/run_config.py 4 2 > $T/ncu_$k.log 2>&1
  python scripts/ncu_summary.py /tmp/$k.ncu-rep 25 > $T/${k}_summary.txt 2>&1
  bash scripts/ncu_stalls.sh /tmp/$k.ncu-rep > $T/${k}_stalls.txt 2>&1
  python scripts/ncu_lines_cuda.py /tmp/$k.ncu-rep 60 > $T/${k}_lines.txt 2>&1
  gzip -c /tmp/$k.ncu-rep > $T/$k.ncu-rep.gz
done
ls -la $T > $T/ls.txt
