"""Per CUDA source line: warp instructions and stall samples from an ncu report (cuda,sass view).
usage: ncu_lines_cuda.py report.ncu-rep [topN]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname = "?"
rows = []
num = lambda x: int(x) if x.isdigit() else 0
for r in csv.reader(io.StringIO(out)):
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    elif len(r) > 8 and r[0].isdigit():
        rows.append((fname, int(r[0]), r[1].strip()[:70], num(r[7]), num(r[4])))
ti = sum(x[3] for x in rows) or 1
ts = sum(x[4] for x in rows) or 1
print(f"total warp inst {ti:,}  stall samples {ts:,}")
for f, ln, s, i, st in sorted(rows, key=lambda x: -x[3])[:top]:
    print(f"{f[:16]:16s}:{ln:<5d} inst {100*i/ti:5.1f}%  stall {100*st/ts:5.1f}%  {s}")
