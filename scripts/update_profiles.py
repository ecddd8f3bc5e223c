"""Copy a gpu_profile.sh run (gpurun_out/prof_TAG) into profiles/rNN: launch lists, per-kernel tables,
ncu --set full summaries, and profiles/traffic.json (ncu DRAM bytes of the depth phase, read by bench.py).
usage: python scripts/update_profiles.py TAG rNN"""
import csv, json, os, shutil, statistics, sys
from collections import defaultdict

tag, rnd = sys.argv[1], sys.argv[2]
src = f"gpurun_out/prof_{tag}"
dst = f"profiles/{rnd}"
os.makedirs(dst, exist_ok=True)


def table(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    h = rows[0]
    ik, im, iv, iid = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    d, names = defaultdict(dict), {}
    for r in rows[1:]:
        try:
            d[int(r[iid])][r[im]] = float(r[iv].replace(",", ""))
            names[int(r[iid])] = r[ik].split("(")[0]
        except ValueError:
            pass
    per = defaultdict(list)
    for k in sorted(d):
        per[names[k]].append(d[k])
    out = []
    for n, l in per.items():
        m = lambda key: statistics.mean(x.get(key, 0.0) for x in l)
        out.append((n, len(l), m("gpu__time_duration.sum") / 1e3, m("dram__bytes_read.sum"), m("dram__bytes_write.sum")))
    return out


md = [f"# {rnd} launch lists (ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
      "--clock-control none -k regex:'^k_')", "",
      "ncu times are cold-cache and serialised: compare SHARES with bench.py's phases_ms, not absolutes.", ""]
cmds = {"cfg3": "python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary  (configs[3], 100M, fwd)",
        "cfg2": "python scripts/run_config.py 2 3  (configs[2], 10M C=8 OpenCV, fwd+bwd)",
        "cfg4": "python scripts/run_config.py 4 2  (configs[4], 50M x 16 views 1024^2, fwd+bwd)"}
traffic = {}
for c in ("cfg3", "cfg2", "cfg4"):
    p = f"{src}/launches_{c}.csv"
    if not os.path.exists(p):
        continue
    shutil.copy(p, f"{dst}/launches_{c}.csv")
    t = table(p)
    setup = [x for x in t if x[0] == "k_tile_bounds"]  # one-time setup of the tile-culled variant, not a frame
    t = [x for x in t if x[0] != "k_tile_bounds"]
    tot = sum(x[2] for x in t)
    md += [f"## {c}: `{cmds[c]}`", "", "| kernel | launches | mean us | share | DRAM read MB | DRAM write MB |",
           "|---|---|---|---|---|---|"]
    for n, k, us, rd, wr in t:
        md.append(f"| `{n}` | {k} | {us:.1f} | {100 * us / tot:.1f}% | {rd / 1e6:.1f} | {wr / 1e6:.1f} |")
    md += ["", f"Sum of kernel means: {tot:.1f} us", ""]
    for n, k, us, rd, wr in setup:
        md += [f"(not in the shares: `{n}`, the tile-culled variant's one-time per-tile bounds, {us:.1f} us)", ""]
    if c == "cfg3":
        isdep = lambda name: "k_depth_pool" in name or "k_depth_async" in name
        dep = [x for x in t if isdep(x[0]) or x[0].endswith("k_clear<0>")]
        traffic = {"depth_phase_bytes": int(sum(x[3] + x[4] for x in dep)),
                   "depth_kernel_bytes": int(sum(x[3] + x[4] for x in t if isdep(x[0]))),
                   "source": f"profiles/{rnd}/launches_summary.md (ncu dram__bytes_read.sum + dram__bytes_write.sum per launch)"}
open(f"{dst}/launches_summary.md", "w").write("\n".join(md) + "\n")
for f in sorted(os.listdir(src)):
    if f.endswith(("_summary.txt", "_stalls.txt", "_lines.txt")) and os.path.getsize(f"{src}/{f}") > 200:
        shutil.copy(f"{src}/{f}", f"{dst}/ncu_{f}")
if os.path.exists(f"{src}/bench.log"):
    for l in open(f"{src}/bench.log"):
        if l.startswith("{"):
            json.dump(json.loads(l), open(f"{dst}/bench_line.json", "w"), indent=1)
if traffic:
    json.dump(traffic, open("profiles/traffic.json", "w"), indent=1)
print(open(f"{dst}/launches_summary.md").read())
