# usage: bash scripts/gpu_prof.sh <tag> [kernel-regex]   (run on the GPU box via gpurun)
cd $GRAFT_REPO_ROOT
T=${1:-prof}
K=${2:-k_depth}
mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary"
$CMD > gpurun_out/${T}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_|nccl' --csv --log-file gpurun_out/${T}_launches.csv $CMD > gpurun_out/${T}_ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 -o gpurun_out/${T}_top $CMD > gpurun_out/${T}_ncu_full.log 2>&1
echo done >> gpurun_out/${T}_status.txt
