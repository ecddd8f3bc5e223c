ncu --set full --clock-control none --import-source on -k regex:'^k_depth_async' -s 2 -c 1 -o /tmp/culled \
  python scripts/run_headline.py 3 cull > gpurun_out/ncu_culled.log 2>&1
python scripts/ncu_summary.py /tmp/culled.ncu-rep 30 > gpurun_out/culled_summary.txt 2>&1
bash scripts/ncu_stalls.sh /tmp/culled.ncu-rep > gpurun_out/culled_stalls.txt 2>&1
python scripts/ncu_lines_cuda.py /tmp/culled.ncu-rep 40 > gpurun_out/culled_lines.txt 2>&1
cp /tmp/culled.ncu-rep gpurun_out/
