"""Summarise an ncu report: key SOL metrics + hottest SASS lines.  usage: ncu_summary.py rep [topN]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
keys = ["Duration", "DRAM Throughput", "Achieved Occupancy", "Theoretical Occupancy", "Registers Per Thread",
        "Executed Ipc Active", "Issue Slots Busy", "Compute (SM) Throughput", "L2 Hit Rate", "Executed Instructions",
        "No Eligible", "Active Warps Per Scheduler", "Eligible Warps Per Scheduler", "Grid Size", "Block Size",
        "Dynamic Shared Memory Per Block", "Memory Throughput"]
for row in csv.reader(io.StringIO(det)):
    if len(row) > 10 and row[-6 if False else 8] in keys:
        print(f"  {row[8]:32s} {row[10]:>14s} {row[9]}  [{row[0][:40]}]")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
for k, row in enumerate(r[2:]):
    for i, n in enumerate(r[0]):
        if n in ("dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sectors_op_red.sum", "lts__t_sectors_op_atom.sum",
                 "smsp__inst_executed.sum", "gpu__time_duration.sum"):
            print(f"  {n:40s} {row[i]:>16s} {r[1][i]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = rows[1]; data = rows[2:]
ia = hdr.index("Instructions Executed"); isrc = hdr.index("Source"); ist = hdr.index("Warp Stall Sampling (All Samples)")
num = lambda x: int(x) if x.isdigit() else 0
tot = sum(num(d[ia]) for d in data); tots = sum(num(d[ist]) for d in data) or 1
print(f"  total warp inst {tot:,}  stall samples {tots:,}")
hot = sorted(data, key=lambda d: -num(d[ist]))[:top]
hot_set = set(id(d) for d in hot)
for d in data:
    if id(d) in hot_set:
        print(f"  {d[0][-5:]} {num(d[ia])/1e6:8.2f}M {100*num(d[ist])/tots:5.1f}%  {d[isrc].strip()[:80]}")
