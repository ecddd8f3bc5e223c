ncu --set full --clock-control none --import-source on -k regex:'^k_depth_async' -s 2 -c 1 -o /tmp/dep \
  python scripts/run_headline.py 3 > gpurun_out/ncu_dep.log 2>&1
bash scripts/ncu_stalls.sh /tmp/dep.ncu-rep > gpurun_out/dep_stalls.txt 2>&1
python scripts/ncu_lines_cuda.py /tmp/dep.ncu-rep 50 > gpurun_out/dep_lines.txt 2>&1
cp /tmp/dep.ncu-rep gpurun_out/
