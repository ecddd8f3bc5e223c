"""configs[3] blend with the descriptors in pinned HOST memory (zero-copy reads over PCIe) vs in HBM.
usage: python scripts/zero_copy_probe.py"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2110_06635_b200 import adop as A  # noqa: E402
from paper_2110_06635_b200 import scene as S  # noqa: E402

w = S.workload(3, device="cuda")
cloud = w.cloud
C = cloud.channels
ap = A.Params(w.params, C)
pyrs = A.alloc_pyramids(w.cameras, w.params.layers, C, "cuda")
pts = A.Points.from_cloud(cloud)
h_feat = cloud.feat.cpu().pin_memory()
pts_h = A.Points(cloud.pos, cloud.radius, h_feat, 0)
ws = A.Workspace(pts, w.cameras, ap, "cuda", A.default_record_capacity(cloud.n, 1, w.params.layers, True))
args = (w.cameras, w.poses, ap, pyrs, ws)
for name, p in (("hbm", pts), ("host", pts_h), ("hbm", pts), ("host", pts_h)):
    A.forward_depth(p, *args)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    ev[0].record()
    A.forward_blend(p, *args)
    ev[1].record()
    A.forward_resolve(p, *args)
    ev[2].record()
    torch.cuda.synchronize()
    img = pyrs[0].image.clone()
    print(f"{name}: blend {ev[0].elapsed_time(ev[1]):.3f} ms resolve {ev[1].elapsed_time(ev[2]):.3f} ms "
          f"img sum {float(img.double().sum()):.6f}", flush=True)
h_pos, h_rad = cloud.pos.cpu().pin_memory(), cloud.radius.cpu().pin_memory()
h_img = torch.empty_like(pyrs[0].image, device="cpu").pin_memory()
for mode in ("copy_all", "zero_copy_feat", "copy_all", "zero_copy_feat"):
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(3):
        cloud.pos.copy_(h_pos, non_blocking=True)
        cloud.radius.copy_(h_rad, non_blocking=True)
        p = pts_h
        if mode == "copy_all":
            cloud.feat.copy_(h_feat, non_blocking=True)
            p = pts
        A.forward_depth(p, *args)
        A.forward_blend(p, *args)
        A.forward_resolve(p, *args)
        h_img.copy_(pyrs[0].image, non_blocking=True)
    e.record()
    torch.cuda.synchronize()
    print(f"e2e {mode}: {s.elapsed_time(e) / 3:.2f} ms/frame", flush=True)
