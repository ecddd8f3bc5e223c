# tests + smoke + default bench + launch list, with per-step status (usage: gpu_round.sh TAG)
cd ${GRAFT_REPO_ROOT:-.}
T=gpurun_out/round_${1:-x}; mkdir -p $T
nproc > $T/nproc.txt; free -g >> $T/nproc.txt
timeout 300 python __graft_entry__.py --smoke > $T/smoke.log 2>&1; echo smoke=$? >> $T/status.txt
timeout 3000 python -m pytest tests -m gpu -q --timeout 1500 > $T/tests.log 2>&1; echo tests=$? >> $T/status.txt
cp gpurun_out/parity_report.json $T/ 2>/dev/null
timeout 900 python bench.py > $T/bench.log 2>&1; echo bench=$? >> $T/status.txt
echo done >> $T/status.txt
