import csv,sys,subprocess
rep=sys.argv[1]
src=subprocess.run(["ncu","-i",rep,"--page","source","--csv","--print-source","sass"],capture_output=True,text=True).stdout
rows=list(csv.reader(src.splitlines())); h=rows[1]; d=rows[2:]
ix={n:h.index(n) for n in h}
num=lambda x: float(x) if x.replace('.','',1).isdigit() else 0.0
tot=sum(num(r[ix['Warp Stall Sampling (All Samples)']]) for r in d) or 1
for r in d:
    sec=num(r[ix['L2 Theoretical Sectors Global']])
    if sec>0 or num(r[ix['Warp Stall Sampling (All Samples)']])/tot>0.02:
        print(f"{r[0][-5:]} {r[1][:60]:60s} inst {num(r[ix['Instructions Executed']])/1e6:7.2f}M thr {num(r[ix['Avg. Threads Executed']]):5.1f} sect {sec/1e6:7.2f}M ideal {num(r[ix['L2 Theoretical Sectors Global Ideal']])/1e6:7.2f}M stall {100*num(r[ix['Warp Stall Sampling (All Samples)']])/tot:5.1f}%")
