#!/bin/bash
# usage: ncu_stalls.sh report  -> occupancy/issue/stall summary
ncu -i $1 --page details --csv 2>/dev/null | python -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]
im=h.index('Metric Name'); iv=h.index('Metric Value'); iu=h.index('Metric Unit')
want={'Duration','DRAM Throughput','Executed Ipc Active','Issue Slots Busy','No Eligible','Active Warps Per Scheduler','Eligible Warps Per Scheduler','Achieved Occupancy','Registers Per Thread','Dynamic Shared Memory Per Block','Warp Cycles Per Issued Instruction','L2 Hit Rate','Mem Busy','Max Bandwidth'}
for row in r[1:]:
  if row[im] in want: print(f'  {row[im]:40s} {row[iv]:>12s} {row[iu]}')
"
ncu -i $1 --page raw --csv 2>/dev/null | python -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]
tot=0; vals={}
for i,n in enumerate(h):
  if 'pcsamp_warps_issue_stalled' in n and not n.endswith('not_issued'):
    try: vals[n.replace('smsp__pcsamp_warps_issue_stalled_','')]=float(r[2][i])
    except: pass
s=sum(vals.values()) or 1
print('  stalls:', ', '.join(f'{k} {100*v/s:.0f}%' for k,v in sorted(vals.items(), key=lambda x:-x[1]) if v/s>0.02))
"
