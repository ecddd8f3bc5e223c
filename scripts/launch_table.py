"""Per-kernel mean time / DRAM bytes from an ncu --csv launch list.  usage: launch_table.py file.csv"""
import csv, statistics, sys
from collections import defaultdict
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
h = rows[0]; ik = h.index('Kernel Name'); im = h.index('Metric Name'); iv = h.index('Metric Value'); iid = h.index('ID')
d = defaultdict(dict); names = {}
for r in rows[1:]:
    try:
        d[int(r[iid])][r[im]] = float(r[iv]); names[int(r[iid])] = r[ik][:48]
    except ValueError:
        pass
per = defaultdict(list)
for k in sorted(d): per[names[k]].append(d[k])
tot = 0
for n, l in per.items():
    t = statistics.mean(x.get('gpu__time_duration.sum', 0) for x in l) / 1e3
    tot += t
    print(f"  {n:48s} x{len(l)} {t:9.1f} us  rd {statistics.mean(x.get('dram__bytes_read.sum', 0) for x in l)/1e6:8.1f} MB"
          f"  wr {statistics.mean(x.get('dram__bytes_write.sum', 0) for x in l)/1e6:8.1f} MB")
print(f"  total {tot:.1f} us")
