"""Run one BASELINE config's forward (+ backward) a few times -- target for ncu captures.
usage: python scripts/run_config.py IDX [steps] [n_points]"""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2110_06635_b200 import adop as A  # noqa: E402
from paper_2110_06635_b200 import scene as S  # noqa: E402

idx = int(sys.argv[1])
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
n = int(sys.argv[3]) if len(sys.argv) > 3 else None
w = S.workload(idx, device="cuda", n=n)
r = A.Renderer(w.cloud, w.cameras, w.poses, w.params)
G = None
if w.backward:
    P = A.pyramid_pixels(w.cameras[0].width, w.cameras[0].height, w.params.layers)
    Gt = S.grad_pyramid(len(w.cameras), w.cloud.channels, P, device="cuda")
    G = [Gt[v] for v in range(len(w.cameras))]
ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
for k in range(steps):
    ev[0].record()
    r.forward()
    ev[1].record()
    if G is not None:
        r.backward(G)
    ev[2].record()
    torch.cuda.synchronize()
    print(f"{w.name}: fwd {ev[0].elapsed_time(ev[1]):.3f} ms bwd {ev[1].elapsed_time(ev[2]):.3f} ms", flush=True)
rec, of = r.ws.stats()
print("record slots", rec, "overflow", of)
