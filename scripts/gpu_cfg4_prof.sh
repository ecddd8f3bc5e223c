ncu --set full --clock-control none --import-source on -k regex:'^k_depth_async' -s 0 -c 1 -o /tmp/c4 \
  python scripts/run_config.py 4 1 > gpurun_out/ncu_c4.log 2>&1
bash scripts/ncu_stalls.sh /tmp/c4.ncu-rep > gpurun_out/c4_stalls.txt 2>&1
python scripts/ncu_lines_cuda.py /tmp/c4.ncu-rep 50 > gpurun_out/c4_lines.txt 2>&1
cp /tmp/c4.ncu-rep gpurun_out/
