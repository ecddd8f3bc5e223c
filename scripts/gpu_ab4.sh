# GPU suite against one variant, then gpu_variants4.sh timings of the listed variants in both orders.
# usage: gpu_ab4.sh TESTVARIANT name...
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
TV=$1; shift
ADOP_LIB=paper_2110_06635_b200/libadop_$TV.so timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ab_tests_$TV.log 2>&1
echo tests=$? > gpurun_out/ab_status.txt
bash scripts/gpu_variants4.sh "$@" > gpurun_out/ab_var.txt 2>&1
REV=$(printf '%s\n' "$@" | tac | tr '\n' ' ')
bash scripts/gpu_variants4.sh $REV >> gpurun_out/ab_var.txt 2>&1
echo done >> gpurun_out/ab_status.txt
