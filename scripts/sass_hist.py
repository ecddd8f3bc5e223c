"""Opcode histogram of a kernel from an ncu source-page SASS dump (ncu -i rep --page source --csv --print-source sass):
static count of each opcode and its executed warp instructions; the Blackwell-specific ones are flagged.
usage: sass_hist.py dump.csv [top]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
kernel = rows[0][1] if rows and len(rows[0]) > 1 else "?"
hdr = rows[1]
isrc, iex = hdr.index("Source"), hdr.index("Instructions Executed")
static, executed = collections.Counter(), collections.Counter()
for r in rows[2:]:
    if len(r) <= iex:
        continue
    ins = r[isrc].strip()
    if ins.startswith("@"):
        ins = ins.split(None, 1)[1] if " " in ins else ins
    op = ins.split()[0] if ins else "?"
    static[op] += 1
    executed[op] += int(r[iex]) if r[iex].isdigit() else 0
tot_s, tot_e = sum(static.values()), sum(executed.values()) or 1
marks = ("UTMALDG", "UBLKCP", "SYNCS", "REDG", "REDUX", "MATCH", "FMNMX3", "ELECT", "UTMA", "LDGSTS")
print(f"{kernel}\n{tot_s} SASS instructions, {tot_e:,} warp instructions executed")
print(f"{'opcode':28s} {'static':>7s} {'executed':>14s} {'share':>6s}")
for op, e in executed.most_common(top):
    print(f"{op:28s} {static[op]:7d} {e:14,d} {100 * e / tot_e:5.1f}%{'  <-' if op.startswith(marks) else ''}")
print("Blackwell / async-copy / reduction opcodes present:")
for op in sorted(static):
    if op.startswith(marks):
        print(f"  {op:28s} static {static[op]:5d}  executed {executed[op]:,}")
