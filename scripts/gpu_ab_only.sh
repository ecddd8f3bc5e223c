# gpu_variants3.sh timings of the listed variants in both orders (no tests).  usage: gpu_ab_only.sh name...
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
bash scripts/gpu_variants3.sh "$@" > gpurun_out/ab_var.txt 2>&1
REV=$(printf '%s\n' "$@" | tac | tr '\n' ' ')
bash scripts/gpu_variants3.sh $REV >> gpurun_out/ab_var.txt 2>&1
echo done >> gpurun_out/ab_var.txt
