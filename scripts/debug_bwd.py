"""Diagnose d_pos differences between the CUDA backward and the oracle (run on the GPU box)."""
import dataclasses
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import oracle as O  # noqa: E402
from paper_2110_06635_b200 import adop as A  # noqa: E402
from paper_2110_06635_b200 import scene as S  # noqa: E402
from tests.parity import grads_for, run_oracle  # noqa: E402


def report(tag, r, bwd):
    g = r.d_pos.cpu().numpy().astype(np.float64)
    err = np.abs(g - bwd.dx)
    rel = err / (bwd.dx_abs + 1e-30)
    ghosts = bwd.dx_abs.sum(0) > 0
    print(f"[{tag}] ghosts {ghosts.sum()} max err/S {rel.max():.3e} p99.9 {np.quantile(rel[:, ghosts], 0.999):.3e} "
          f"median {np.median(rel[:, ghosts]):.3e} n(>1e-5) {(rel > 1e-5).sum()}")
    idx = np.argsort(rel.max(0))[-5:]
    for i in idx:
        print("   pt", i, "gpu", g[:, i], "orc", bwd.dx[:, i], "S", bwd.dx_abs[:, i])
    gp = r.d_pose.cpu().numpy()
    print("   pose err", np.abs(gp - bwd.dpose).max(), "scale", bwd.dpose_abs.max())
    return idx


for model in (S.OPENCV8, S.PINHOLE):
    w = S.workload(2, n=200_013)
    if model == S.PINHOLE:
        w.cameras[:] = [S.pinhole(1920, 1080)]
    G = grads_for(w.cameras, w.params.layers, w.cloud.channels)
    dev = torch.device("cuda")
    r = A.Renderer(w.cloud.to(dev), w.cameras, w.poses, w.params)
    r.forward()
    r.backward([g.to(dev) for g in G])
    torch.cuda.synchronize()
    pts, fwd, bwd = run_oracle(w.cloud, w.cameras, w.poses, w.params, grads=G)
    report(f"model{model} gpu-image", r, bwd)
    # same backward with the oracle's image (rounded to fp32) in the GPU pyramid
    r.pyrs[0].image.copy_(torch.from_numpy(fwd.image[0].astype(np.float32)))
    r.backward([g.to(dev) for g in G])
    torch.cuda.synchronize()
    report(f"model{model} oracle-image", r, bwd)
