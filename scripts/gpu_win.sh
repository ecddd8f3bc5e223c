# OpenCV8 window test: GPU tests, work counters, configs[4] / configs[2] timings with and without it (usage: gpu_win.sh TAG)
cd ${GRAFT_REPO_ROOT:-.}
T=gpurun_out/win_${1:-x}; mkdir -p $T
timeout 2400 python -m pytest tests -m gpu -q --timeout 1500 > $T/tests.log 2>&1; echo tests=$? >> $T/status.txt
cp gpurun_out/parity_report.json $T/ 2>/dev/null
for c in 4 2; do for wv in 1 0; do echo "cfg$c WINDOW=$wv" >> $T/counters.txt; ADOP_WINDOW=$wv ADOP_LIB=paper_2110_06635_b200/libadop_cnt.so python scripts/depth_counters.py $c >> $T/counters.txt 2>&1; done; done
for wv in 1 0 1 0; do
  echo "WINDOW=$wv" >> $T/cfg4.log; ADOP_WINDOW=$wv python scripts/run_config.py 4 5 >> $T/cfg4.log 2>&1
  echo "WINDOW=$wv" >> $T/cfg2.log; ADOP_WINDOW=$wv python scripts/run_config.py 2 10 >> $T/cfg2.log 2>&1
done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
ncu --metrics $M --clock-control none -k regex:'^k_' -c 60 --csv --log-file $T/launches_cfg4.csv python scripts/run_config.py 4 2 > $T/ncu4.log 2>&1
echo done >> $T/status.txt
