# usage: bash scripts/gpu_prof_cfg.sh <tag> <config idx> <kernel regex>
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=$1; I=$2; K=$3
CMD="python scripts/run_config.py $I 3"
$CMD > gpurun_out/${T}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:'k_' --csv --log-file gpurun_out/${T}_launches.csv $CMD > gpurun_out/${T}_ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 -o gpurun_out/${T}_top $CMD > gpurun_out/${T}_ncu_full.log 2>&1
echo done >> gpurun_out/${T}_status.txt
