# run_config.py CFG timings of the listed variants in both orders, twice.  usage: gpu_ab_cfg.sh CFG name...
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out; : > gpurun_out/ab_cfg.txt
C=$1; shift
REV=$(printf '%s\n' "$@" | tac | tr '\n' ' ')
for order in "$*" "$REV"; do
  for v in $order; do
    echo "$v $(ADOP_LIB=paper_2110_06635_b200/libadop_$v.so python scripts/run_config.py $C 6 2>&1 | tail -4 | head -3 | tr '\n' ' ')" >> gpurun_out/ab_cfg.txt
  done
done
echo done >> gpurun_out/ab_cfg.txt
