"""The oracle's OpenMP loops do not change any result: per-point work runs in parallel into
per-point slots, every reduction over points (keys, blend sums, pose / intrinsics sums) runs serially in point
order, so 1 thread and several threads agree bit for bit -- CPU only."""
import dataclasses

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2110_06635_b200 import scene as S


def _run(threads, w, prm, G):
    O.set_threads(threads)
    pts = O.Points.from_cloud(w.cloud)
    f = O.forward(pts, w.cameras, w.poses, prm)
    b = O.backward(pts, w.cameras, w.poses, prm, f, G)
    m = O.point_masks(pts, w.cameras, w.poses, prm)
    return f, b, m


@pytest.mark.parametrize("idx,n,views,extra", [
    (2, 300_000, 1, {}),                       # > one 2^18 chunk, OpenCV8, C = 8
    (4, 80_000, 3, {"log_descriptors": True}),
    (0, None, 1, {"env": True}),               # env map: the parallel resolve and the serial dE scatter
])
def test_thread_count_does_not_change_results(idx, n, views, extra):
    w = S.workload(idx, n=n, n_views=views) if n else S.workload(idx)
    prm = dataclasses.replace(w.params, ghost_rate=0.25, log_descriptors=extra.get("log_descriptors", False))
    if extra.get("env"):
        g = torch.Generator().manual_seed(3)
        prm = dataclasses.replace(prm, env_map=torch.rand(16, 32, w.cloud.channels, generator=g))
    P = O.pyramid_pixels(w.cameras[0].width, w.cameras[0].height, prm.layers)
    G = S.grad_pyramid(len(w.cameras), w.cloud.channels, P).numpy()
    try:
        f1, b1, m1 = _run(1, w, prm, G)
        f3, b3, m3 = _run(3, w, prm, G)
    finally:
        O.set_threads(1)
    assert np.array_equal(m1, m3)
    for a in ("keys", "accum", "count", "image"):
        assert np.array_equal(getattr(f1, a), getattr(f3, a)), a
    for a in ("dtau", "dx", "dpose", "dintr", "dtau_abs", "dx_abs", "dpose_abs", "dintr_abs", "denv"):
        x1, x3 = getattr(b1, a), getattr(b3, a)
        assert (x1 is None and x3 is None) or np.array_equal(x1, x3), a
    assert np.abs(b1.dx).sum() > 0 and np.abs(b1.dtau).sum() > 0
