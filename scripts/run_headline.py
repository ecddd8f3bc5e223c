"""configs[3] frames (100M points) as a profiling target.  usage: run_headline.py STEPS [cull] [points]"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2110_06635_b200 import adop as A  # noqa: E402
from paper_2110_06635_b200 import scene as S  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
cull = len(sys.argv) > 2 and sys.argv[2] == "cull"
n = int(sys.argv[3]) if len(sys.argv) > 3 else 100_000_000
w = S.workload(3, device="cuda", n=n)
r = A.Renderer(w.cloud, w.cameras, w.poses, w.params)
if cull:
    r.points.enable_tile_culling()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for k in range(steps):
    ev[0].record()
    r.forward()
    ev[1].record()
    torch.cuda.synchronize()
    print(f"frame {k}: {ev[0].elapsed_time(ev[1]):.3f} ms", flush=True)
