# ncu --set full captures of configs[4] kernels (one launch each), summarised on the box
# usage: gpu_ncu_cfg4.sh tag kernel...
TAG=$1; shift
for K in "$@"; do
ncu --set full --clock-control none --import-source on -k regex:"^$K" -c 1 -o /tmp/${TAG}_$K \
  python scripts/run_config.py 4 1 > gpurun_out/ncu_${TAG}_$K.log 2>&1
python scripts/ncu_summary.py /tmp/${TAG}_$K.ncu-rep 30 > gpurun_out/${TAG}_${K}_summary.txt 2>&1
bash scripts/ncu_stalls.sh /tmp/${TAG}_$K.ncu-rep > gpurun_out/${TAG}_${K}_stalls.txt 2>&1
python scripts/ncu_lines_cuda.py /tmp/${TAG}_$K.ncu-rep 40 > gpurun_out/${TAG}_${K}_lines.txt 2>&1
done
