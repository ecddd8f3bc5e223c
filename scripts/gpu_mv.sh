# multi-view lists: parity of the multi-view tests, then configs[4] / configs[1] timings with and without them,
# and a launch list of configs[4] (usage: gpu_mv.sh TAG)
cd ${GRAFT_REPO_ROOT:-.}
T=gpurun_out/mv_${1:-x}; mkdir -p $T
timeout 1200 python -m pytest tests -m gpu -q -k "room_configs_reduced or full_config4 or tile_culling or consumes_forward or fisheye_fwd_bwd or view_id_base or captured or overflow or list_orders" > $T/tests.log 2>&1; echo tests=$? >> $T/status.txt
for mv in 5 0 7 1 5 0; do
  echo "MV=$mv" >> $T/cfg4.log; ADOP_MV_LISTS=$mv python scripts/run_config.py 4 5 >> $T/cfg4.log 2>&1
  echo "MV=$mv" >> $T/cfg1.log; ADOP_MV_LISTS=$mv python scripts/run_config.py 1 10 >> $T/cfg1.log 2>&1
done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_op_red.sum,lts__t_sectors_op_atom.sum,lts__t_sector_hit_rate.pct
ncu --metrics $M --clock-control none -k regex:'^k_' -c 60 --csv --log-file $T/launches_cfg4.csv \
  python scripts/run_config.py 4 2 > $T/ncu4.log 2>&1
ADOP_MV_LISTS=0 ncu --metrics $M --clock-control none -k regex:'^k_' -c 60 --csv --log-file $T/launches_cfg4_flat.csv \
  python scripts/run_config.py 4 2 > $T/ncu4f.log 2>&1
echo done >> $T/status.txt
