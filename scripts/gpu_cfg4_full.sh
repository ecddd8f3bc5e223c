# ncu --set full of the configs[4] record/ghost consumers (blend, tex, ghost).  usage: gpu_cfg4_full.sh TAG
T=gpurun_out/c4full_$1; mkdir -p $T
for k in k_blend k_bwd_tex k_bwd_ghost; do
  ncu --set full --clock-control none --import-source on -k regex:"^$k" -s 1 -c 1 -o /tmp/$k \
    python scripts/run_config.py 4 2 > $T/ncu_$k.log 2>&1
  python scripts/ncu_summary.py /tmp/$k.ncu-rep 25 > $T/${k}_summary.txt 2>&1
  bash scripts/ncu_stalls.sh /tmp/$k.ncu-rep > $T/${k}_stalls.txt 2>&1
  python scripts/ncu_lines_cuda.py /tmp/$k.ncu-rep 30 > $T/${k}_lines.txt 2>&1
done
