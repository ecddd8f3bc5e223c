"""Eager vs CUDA-graph frame time for configs[3] (launch overhead probe)."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2110_06635_b200 import adop as A  # noqa: E402
from paper_2110_06635_b200 import scene as S  # noqa: E402

w = S.workload(3, device="cuda")
pts = A.Points.from_cloud(w.cloud)
ap = A.Params(w.params, 4)
pyrs = A.alloc_pyramids(w.cameras, 5, 4, "cuda")
ws = A.Workspace(pts, w.cameras, ap, "cuda", A.default_record_capacity(pts.n, 1, 5, True))


def step(s):
    A.forward_depth(pts, w.cameras, w.poses, ap, pyrs, ws, s)
    A.forward_blend(pts, w.cameras, w.poses, ap, pyrs, ws, s)
    A.forward_resolve(pts, w.cameras, w.poses, ap, pyrs, ws, s)


s = torch.cuda.current_stream()
for _ in range(5):
    step(s)
torch.cuda.synchronize()
K = 100
for rep in range(2):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(K):
        step(s)
    e1.record()
    torch.cuda.synchronize()
    print("eager ms/frame", e0.elapsed_time(e1) / K)
gs = torch.cuda.Stream()
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(gs):
    step(gs)  # warm on the side stream
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=gs):
        step(gs)
torch.cuda.synchronize()
for rep in range(2):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(K):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    print("graph ms/frame", e0.elapsed_time(e1) / K)
# the graph's result equals the eager one
k1 = pyrs[0].keys.clone()
step(s)
torch.cuda.synchronize()
print("keys equal after graph replay:", bool(torch.equal(k1, pyrs[0].keys)))
