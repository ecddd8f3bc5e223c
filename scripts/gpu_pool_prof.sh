# ncu --set full of the headline pooled depth sweep per variant: gpu_pool_prof.sh variant...
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in "$@"; do
  ADOP_LIB=paper_2110_06635_b200/libadop_$v.so ncu --set full --clock-control none --import-source on \
    -k regex:'^k_depth_pool' -s 2 -c 1 -o /tmp/pool_$v python scripts/run_headline.py 3 > gpurun_out/ncu_pool_$v.log 2>&1
  bash scripts/ncu_stalls.sh /tmp/pool_$v.ncu-rep > gpurun_out/pool_${v}_stalls.txt 2>&1
  python scripts/ncu_lines_cuda.py /tmp/pool_$v.ncu-rep 60 > gpurun_out/pool_${v}_lines.txt 2>&1
  python scripts/ncu_lines.py /tmp/pool_$v.ncu-rep 60 > gpurun_out/pool_${v}_sass.txt 2>&1
  ls -la /tmp/pool_$v.ncu-rep >> gpurun_out/pool_sizes.txt
done
