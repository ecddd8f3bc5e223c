"""Aggregate an ncu report's per-SASS metrics by CUDA source line.
usage: python scripts/ncu_lines.py report.ncu-rep [top]"""
import csv, io, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
agg = {}; src = {}; fname = None; hdr = None
for row in csv.reader(io.StringIO(out)):
    if not row: continue
    if row[0] == "File Path": fname = row[1].split("/")[-1]; continue
    if row[0] == "Line No": hdr = row; continue
    if hdr is None or not row[0].isdigit(): continue
    d = dict(zip(hdr[2:], row[2:]))
    line = (fname, int(row[0])); src.setdefault(line, row[1].strip()[:70])
    def f(k):
        try: return float(d.get(k, 0) or 0)
        except ValueError: return 0.0
    a = agg.setdefault(line, [0.0, 0.0])
    a[0] += f("Instructions Executed"); a[1] += f("Warp Stall Sampling (All Samples)")
ti = sum(v[0] for v in agg.values()) or 1; ts = sum(v[1] for v in agg.values()) or 1
print(f"total warp inst {ti:,.0f}  stall samples {ts:,.0f}")
for line, (i, s) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"{line[0][:16]:16s}:{line[1]:<5d} inst {100*i/ti:5.1f}%  stall {100*s/ts:5.1f}%  {src[line]}")
