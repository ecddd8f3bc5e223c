"""Shared helpers of the GPU parity tests: run the CUDA path (through the C-ABI binding) and the CPU
oracle on the same seeded inputs and compare element by element.

Tolerances:
  keys, counts, masks: bit-exact (integer results, R8/R26).
  image: |gpu - oracle| <= 1e-6 + 1e-5 |oracle|  (north_star: 1e-5 rel / 1e-6 abs; fp32 atomic sums of
         k <= ~150 positive terms err by <= k * 2^-24 relative).
  d_feat, d_pos: |gpu - oracle| <= 1e-6 + 1e-5 * S, S = the oracle's per-element sum of term magnitudes
         (fp32 sums of <= L*V terms with cancellation: the error scales with S, not with the result).
  d_pose: |gpu - oracle| <= 1e-6 + 1e-5 * max(|oracle|, 1e-2 * S)  (R20).
"""
from __future__ import annotations

import numpy as np
import torch

from oracle import oracle as O
from paper_2110_06635_b200 import adop as A
from paper_2110_06635_b200 import scene as S

# Every floating-point comparison is also recorded here (conftest writes it to gpurun_out/parity_report.json):
# the largest |gpu - oracle|, the largest relative error |gpu - oracle| / |oracle| over elements with
# |oracle| >= 1e-3 * max |oracle|, the largest err / tol of the test's own tolerance, and the fraction of
# elements that would also pass north_star's literal 1e-5 relative / 1e-6 absolute.
REPORT = []


def _record(ctx, what, g, o, err, tol):
    o = np.asarray(o, dtype=np.float64)
    if err.size == 0:
        return
    ao = np.abs(o)
    big = ao >= 1e-3 * ao.max() if ao.max() > 0 else np.zeros_like(ao, dtype=bool)
    REPORT.append({"ctx": ctx, "what": what, "n": int(err.size), "max_abs_err": float(err.max()),
                   "max_rel_err": float((err[big] / ao[big]).max()) if big.any() else 0.0,
                   "max_err_over_tol": float((err / tol).max()),
                   "literal_1e-5_rel_1e-6_abs_pass": float(np.mean(err <= 1e-6 + 1e-5 * ao))})


def run_gpu(cloud, cams, poses, params, record_capacity=None, grads=None, global_offset=0, intrinsics=True):
    dev = torch.device("cuda")
    r = A.Renderer(cloud.to(dev), cams, poses, params, global_offset=global_offset,
                   record_capacity=record_capacity, intrinsics=intrinsics)
    r.forward()
    if grads is not None:
        r.backward([g.to(dev) for g in grads])
    torch.cuda.synchronize()
    return r


def run_oracle(cloud, cams, poses, params, grads=None, global_offset=0):
    O.set_threads(0)  # all host cores; results do not depend on the thread count (tests/test_oracle_threads.py)
    pts = O.Points.from_cloud(cloud.to("cpu"), global_offset)
    fwd = O.forward(pts, cams, poses, params)
    bwd = None
    if grads is not None:
        G = np.stack([g.cpu().numpy() for g in grads])
        bwd = O.backward(pts, cams, poses, params, fwd, G)
    return pts, fwd, bwd


def keys_u64(t: torch.Tensor) -> np.ndarray:
    return t.cpu().numpy().view(np.uint64)


def compare_forward(r, fwd, views=None, ctx=""):
    views = range(len(r.pyrs)) if views is None else views
    for j, v in enumerate(views):
        p = r.pyrs[v]
        k = keys_u64(p.keys)
        bad = np.nonzero(k != fwd.keys[j])[0]
        assert len(bad) == 0, f"{ctx} view {v}: {len(bad)} keys differ, first at {bad[:5]}: " \
                              f"gpu {k[bad[:3]]} oracle {fwd.keys[j][bad[:3]]}"
        c = p.count.cpu().numpy()
        assert np.array_equal(c, fwd.count[j]), f"{ctx} view {v}: counts differ at " \
                                                f"{np.nonzero(c != fwd.count[j])[0][:5]}"
        img = p.image.cpu().numpy().astype(np.float64)
        err = np.abs(img - fwd.image[j])
        tol = 1e-6 + 1e-5 * np.abs(fwd.image[j])
        _record(ctx, f"image[{v}]", img, fwd.image[j], err, tol)
        assert np.all(err <= tol), f"{ctx} view {v}: image max err {err.max()} (excess {(err - tol).max()})"


def compare_backward(r, bwd, ctx="", check_feat=True, check_pos=True, views=None):
    if check_feat:
        g = r.d_feat.cpu().numpy().astype(np.float64)
        err = np.abs(g - bwd.dtau)
        tol = 1e-6 + 1e-5 * bwd.dtau_abs
        _record(ctx, "d_feat", g, bwd.dtau, err, tol)
        assert np.all(err <= tol), f"{ctx} d_feat max excess {(err - tol).max()} at {np.unravel_index((err - tol).argmax(), err.shape)}"
    if check_pos:
        g = r.d_pos.cpu().numpy().astype(np.float64)
        err = np.abs(g - bwd.dx)
        tol = 1e-6 + 1e-5 * bwd.dx_abs
        _record(ctx, "d_pos", g, bwd.dx, err, tol)
        i = np.unravel_index((err - tol).argmax(), err.shape)
        assert np.all(err <= tol), f"{ctx} d_pos max excess {(err - tol).max()} at {i}: gpu {g[i]} oracle {bwd.dx[i]} S {bwd.dx_abs[i]}"
    g = r.d_pose.cpu().numpy()
    if views is not None:
        g = g[list(views)]
    err = np.abs(g - bwd.dpose)
    tol = 1e-6 + 1e-5 * np.maximum(np.abs(bwd.dpose), 1e-2 * bwd.dpose_abs)
    _record(ctx, "d_pose", g, bwd.dpose, err, tol)
    assert np.all(err <= tol), f"{ctx} d_pose err {err} tol {tol}\ngpu {g}\noracle {bwd.dpose}"
    if getattr(r, "d_env", None) is not None and bwd.denv is not None:
        # NEXT-2 environment-map gradient: fp32 sums of w G terms plus the bilinear weights' error -- the
        # fp32 lookup coordinates err by a few ulp of the angles, i.e. ~(W + H) 2^-22 texels -- both scaled
        # by S = sum over the texel's taps of |G|
        g = r.d_env.cpu().numpy().astype(np.float64)
        H_, W_ = g.shape[0], g.shape[1]
        err = np.abs(g - bwd.denv)
        tol = 1e-6 + (1e-5 + (W_ + H_) * 2.0 ** -22) * bwd.denv_abs
        _record(ctx, "d_env", g, bwd.denv, err, tol)
        assert np.all(err <= tol), f"{ctx} d_env max excess {(err - tol).max()}"
    if getattr(r, "d_intr", None) is not None and bwd.dintr is not None:
        # NEXT-1 intrinsics gradient: same tolerance form as d_pose (R20)
        g = r.d_intr.cpu().numpy()
        if views is not None:
            g = g[list(views)]
        err = np.abs(g - bwd.dintr)
        tol = 1e-6 + 1e-5 * np.maximum(np.abs(bwd.dintr), 1e-2 * bwd.dintr_abs)
        _record(ctx, "d_intr", g, bwd.dintr, err, tol)
        assert np.all(err <= tol), f"{ctx} d_intr err {err} tol {tol}\ngpu {g}\noracle {bwd.dintr}"


def grads_for(cams, layers, C, seed=S.SEED_GRADS):
    P = [A.pyramid_pixels(c.width, c.height, layers) for c in cams]
    assert len(set(P)) == 1
    G = S.grad_pyramid(len(cams), C, P[0], seed=seed)
    return [G[v] for v in range(len(cams))]
