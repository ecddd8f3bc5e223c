"""Per-phase GPU time (depth / blend / resolve / backward) of one BASELINE config.  usage: phase_probe.py IDX"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2110_06635_b200 import adop as A  # noqa: E402
from paper_2110_06635_b200 import scene as S  # noqa: E402

idx = int(sys.argv[1]) if len(sys.argv) > 1 else 2
w = S.workload(idx, device="cuda")
r = A.Renderer(w.cloud, w.cameras, w.poses, w.params)
args = (r.points, r.cams, r.poses, r.params, r.pyrs, r.ws)
for _ in range(3):
    A.forward_depth(*args); A.forward_blend(*args); A.forward_resolve(*args)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
t = [0.0, 0.0, 0.0]
for _ in range(10):
    ev[0].record(); A.forward_depth(*args); ev[1].record(); A.forward_blend(*args); ev[2].record()
    A.forward_resolve(*args); ev[3].record(); torch.cuda.synchronize()
    for i in range(3):
        t[i] += ev[i].elapsed_time(ev[i + 1]) / 10
print(f"configs[{idx}] depth {t[0]:.4f} blend {t[1]:.4f} resolve {t[2]:.4f} ms; records {r.ws.stats()}")
