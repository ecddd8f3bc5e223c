# warp pre-reduction of the depth keys: parity with the variant, timings, L2 reduction counters
cd ${GRAFT_REPO_ROOT:-.}
T=gpurun_out/pre; mkdir -p $T
ADOP_LIB=paper_2110_06635_b200/libadop_pre.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "tiny or full_config3 or room_configs_reduced or full_config4 or precull" > $T/tests.log 2>&1; echo "pre tests rc=$?" >> $T/summary.txt
bash scripts/gpu_ab_lib.sh "cur pre"
cat gpurun_out/ablib/summary.txt >> $T/summary.txt
M=gpu__time_duration.sum,lts__t_requests_op_red.sum,lts__t_sectors_op_red.sum,smsp__inst_executed.sum
for v in cur pre; do
  ADOP_LIB=paper_2110_06635_b200/libadop_$v.so ncu --metrics $M --clock-control none -k regex:'^k_depth' -c 3 --csv --log-file $T/depth3_$v.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary --no-graph > /dev/null 2>&1
  ADOP_LIB=paper_2110_06635_b200/libadop_$v.so ncu --metrics $M --clock-control none -k regex:'^k_depth' -c 2 --csv --log-file $T/depth4_$v.csv python scripts/run_config.py 4 2 > /dev/null 2>&1
done
