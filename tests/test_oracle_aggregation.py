"""Pins for R17: how the oracle aggregates the structural (ghost) gradients over pyramid LAYERS and over
VIEWS -- CPU only.

Eq. 2 renders layer l at P_l = 2^-l C(Rx + t), so a layer-l image-space gradient g_l (per
layer-l pixel, Eqs. 9-10) reaches the layer-0 projection u0 through du_l/du0 = 2^-l, and the
loss of a batch is the sum of its views' losses.  The chain rule therefore gives

    dL/du0 = sum_v sum_l 2^-l g_{v,l},     dx = sum_v R_v^T J_v^T (dL/du0, dL/dv0)_v      (Eq. 8)

-- a sum, where SPEC averages over layers (a documented deviation: DESIGN.md R17).  The pins:

1. closed form by hand on linear ramps at two layers with different adjoints per layer and per view (every
   other reading -- no factor, 2^+l, a layer average, a view average -- gives a different number);
2. an independent re-render check: the ghost is RENDERED (oracle forward, no backward code involved) as a
   front point displaced by +-s layer-0 pixels, s = 2^(L-1), and the central difference of L = sum G.I over
   all views and layers must equal dL/dx from the backward.  On linear ramps this difference is exact;
3. SPEC's descent-direction check (Eq. 17): on 100 random synthetic scenes a small step
   along -d_pose (camera) and along -d_x (ghost points) lowers the loss in >= 95% of them.
"""
import math

import numpy as np
import pytest

from oracle import oracle as O
from paper_2110_06635_b200 import scene as S
from tests.test_oracle_backward import _at_pixel, _cam, arrange, _rodrigues

F = np.float32
IDENT = S.Pose(np.eye(3, dtype=F), np.zeros(3, dtype=F))
PRM2 = S.Params(layers=2, discard=False, alpha=0.01, ghost_rate=0.5, seed=4242)

# scene of pins 1-2: a 32x8 pinhole (f = 8, c = (16, 4)), 2 layers (32x8, 16x4).  Rendered points on
# layer-0 row 4 at depth 2 with tau = c*u: layer 0 row 4 is the ramp I_0(u) = c*u; layer-1 pixel k of row 2
# receives u in {2k-1, 2k} (R3: round half away from zero), so I_1(k) = c*(2k - 1/2): slope 2c.  The ghost
# sits in front (depth 1) at layer-0 pixel (16, 4) = layer-1 pixel (8, 2) with tau = 16c; its neighbours:
#   layer 0: (17,4) I = 17c, (15,4) I = 15c        -> Delta = -c, +c  (Eq. 11 case 3: in front)
#   layer 1: ( 9,2) I = 17.5c, (7,2) I = 13.5c     -> Delta = -1.5c, +2.5c
# adjoints G_l only on the ramp rows (G on every other pixel is 0, so g_v = 0):
#   g_0 = 1/2 (G_0 (-c) - G_0 c) = -G_0 c,   g_1 = 1/2 (G_1 (-1.5c) - G_1 2.5c) = -2 G_1 c
#   dL/du0 = g_0 + 2^-1 g_1 = -c (G_0 + G_1)
CAM = _cam(32, 8, 8.0, 16.0, 4.0)
C_RAMP = 1.0 / 64
W, H = 32, 8
P_PYR = W * H + 16 * 4


def _ramp_scene(ghost_u, as_ghost=True):
    render = [_at_pixel(CAM, u, 4, 2.0) for u in range(32)]
    feats = [[C_RAMP * u] for u in range(32)]
    probe = _at_pixel(CAM, ghost_u, 4, 1.0)
    if as_ghost:
        return arrange(render, [probe], PRM2, feats, [[C_RAMP * 16]])
    return arrange(render + [probe], [], PRM2, feats + [[C_RAMP * 16]], [])


def _grad(G0, G1):
    """Adjoint pyramid of one view: G0 on layer-0 row 4, G1 on layer-1 row 2, 0 elsewhere (C = 1)."""
    g = np.zeros(P_PYR, F)
    g[4 * W:5 * W] = G0
    g[W * H + 2 * 16: W * H + 3 * 16] = G1
    return g


ADJ = [(0.5, 3.0), (1.0, -0.25)]   # (G_0, G_1) of view 0 and view 1


def _views(nv):
    return [CAM] * nv, [IDENT] * nv, np.stack([_grad(*ADJ[v]) for v in range(nv)])


@pytest.mark.parametrize("nv", [1, 2])
def test_layer_and_view_sum_closed_form(nv):
    cams, poses, G = _views(nv)
    pts, gids = _ramp_scene(16)
    fwd = O.forward(pts, cams, poses, PRM2)
    # the scene is what the docstring says
    np.testing.assert_allclose(fwd.image[0, 4 * W + 15: 4 * W + 18], [15 * C_RAMP, 16 * C_RAMP, 17 * C_RAMP])
    np.testing.assert_allclose(fwd.image[0, W * H + 2 * 16 + 7: W * H + 2 * 16 + 10],
                               [13.5 * C_RAMP, 15.5 * C_RAMP, 17.5 * C_RAMP])
    bwd = O.backward(pts, cams, poses, PRM2, fwd, G)
    g = gids[0]
    du = [-C_RAMP * (G0 + G1) for G0, G1 in ADJ[:nv]]  # per view: -c (G_0 + 2^-1 * 2 G_1)
    # J at Xc = (0, 0, 1): u-row [fx/Z, 0, -fx X/Z^2] = [8, 0, 0]
    np.testing.assert_allclose(bwd.dx[:, g], [8.0 * sum(du), 0.0, 0.0], rtol=1e-12, atol=1e-15)
    for v in range(nv):  # per-view pose rows (w, Xc x w), Xc = (0, 0, 1): (8 du, 0, 0, 0, 8 du, 0)
        np.testing.assert_allclose(bwd.dpose[v], [8.0 * du[v], 0, 0, 0, 8.0 * du[v], 0], rtol=1e-12, atol=1e-15)
    # the readings R17 rejects give other numbers on this scene
    G0, G1 = ADJ[0]
    if nv == 1:
        for name, val in {"no layer factor": -C_RAMP * (G0 + 2 * G1), "2^+l": -C_RAMP * (G0 + 4 * G1),
                          "layer average (S:L381)": -C_RAMP * (G0 + G1) / 2}.items():
            assert abs(bwd.dx[0, g] - 8.0 * val) > 1e-3, name
    else:  # a view average would halve the sum
        assert abs(bwd.dx[0, g] - 8.0 * sum(du) / 2) > 1e-3


@pytest.mark.parametrize("nv", [1, 2])
def test_ghost_gradient_equals_rerender_central_difference(nv):
    """The ghost, rendered as a front point at u0 +- 2 (= +-1 pixel at layer 1), through the oracle FORWARD
    only: (L(+2) - L(-2)) / (2 * 2 * dx_world/du0) equals the backward's dL/dx along x."""
    cams, poses, G = _views(nv)
    pts, gids = _ramp_scene(16)
    bwd = O.backward(pts, cams, poses, PRM2, O.forward(pts, cams, poses, PRM2), G)
    Gd = G.astype(np.float64)

    def loss(u):
        q, _ = _ramp_scene(u, as_ghost=False)
        return float((O.forward(q, cams, poses, PRM2).image * Gd).sum())

    s = 2.0                                    # layer-0 pixels; u0 = fx X / Z + cx, Z = 1 -> dX = s / 8
    slope_u0 = (loss(16 + s) - loss(16 - s)) / (2 * s)
    assert slope_u0 != 0.0
    assert abs(bwd.dx[0, gids[0]] - 8.0 * slope_u0) < 1e-12


# --------------------------------------------------------------------------- #
# 3. descent direction: pose and ghost points
# --------------------------------------------------------------------------- #
def _wall_scene(rng, n=60000):
    """A textured wall 3 m in front of an identity camera (pinhole 64x48, f = 32) with a smooth random
    texture (two channels of low-frequency sinusoids).  Dense enough (~13 points per layer-0 pixel) that the
    one-pixel render has no holes: holes would make the loss a function of where the sampling gaps fall
    rather than of the pose.  (With front occluder patches the ghost approximation of Eq. 11 is one-sided at
    occlusion edges -- P:L307-309 calls the plain spatial gradients "not accurate" -- and the descent rate
    drops to 75-93%: DESIGN.md section 3.)"""
    x = rng.uniform(-3.6, 3.6, n)
    y = rng.uniform(-2.8, 2.8, n)
    z = np.full(n, 3.0)
    k = rng.uniform(0.6, 1.6, (2, 2)) * rng.choice([-1, 1], (2, 2))
    ph = rng.uniform(0, 2 * math.pi, (2, 2))
    tex = np.stack([0.5 + 0.35 * np.sin(k[c, 0] * x + ph[c, 0]) * np.cos(k[c, 1] * y + ph[c, 1]) for c in range(2)], 1)
    pos = np.stack([x, y, z]).astype(F)
    return pos, tex.astype(F)


def _perturb(pose, xi):
    """exp(xi) applied on the left (Eq. 17): Xc' = Rot(w) Xc + rho (first-order retraction)."""
    Rw = _rodrigues(np.asarray(xi[3:], np.float64))
    R = Rw @ pose.R.astype(np.float64)
    t = Rw @ pose.t.astype(np.float64) + np.asarray(xi[:3], np.float64)
    return S.Pose(R.astype(F), t.astype(F))


def _motion(cam, pose, xi):
    """Largest layer-0 image motion (pixels) of points on the wall's visible part under the twist xi."""
    grid = [(u, v) for u in (0, 32, 63) for v in (0, 24, 47)]
    X = np.array([[(u - cam.cx) * 3.0 / cam.fx, (v - cam.cy) * 3.0 / cam.fy, 3.0] for u, v in grid])
    Rp, tp = pose.R.astype(np.float64), pose.t.astype(np.float64)
    q = _perturb(pose, xi)
    a = X @ Rp.T + tp
    b = X @ q.R.astype(np.float64).T + q.t.astype(np.float64)
    return float(np.max(np.hypot(cam.fx * (a[:, 0] / a[:, 2] - b[:, 0] / b[:, 2]),
                                 cam.fy * (a[:, 1] / a[:, 2] - b[:, 1] / b[:, 2]))))


def test_descent_direction_pose_and_ghosts():
    """SPEC S:L369 (and its ghost-point analogue): the target T is the render at the true pose; the camera is
    moved off by a random twist of 4 layer-0 pixels (largest image motion); L = 1/2 |I - T|^2 over all layers, adjoint G = I - T.
    A step of ~1 layer-0 pixel along -d_pose lowers L and the opposite step raises it; moving every ghost ~1
    pixel along its -d_x lowers L of the render in which the ghosts take part, the opposite move raises it.
    Required: >= 95 of 100 scenes for each of the four."""
    cam = S.pinhole(64, 48)
    prm = S.Params(layers=3, discard=False, ghost_rate=0.25, seed=99)
    prm_all = S.Params(layers=3, discard=False, ghost_rate=0.0, seed=99)
    ok = {"pose down": 0, "pose up": 0, "ghosts down": 0, "ghosts up": 0}
    for trial in range(100):
        rng = np.random.default_rng(1000 + trial)
        pos, tex = _wall_scene(rng)
        pts = O.Points(pos, np.full(pos.shape[1], 0.005, F), tex)
        target = O.forward(pts, [cam], [IDENT], prm).image
        target_all = O.forward(pts, [cam], [IDENT], prm_all).image

        def L(points, pose, p=prm, T=target):
            return 0.5 * float(((O.forward(points, [cam], [pose], p).image - T) ** 2).sum())

        # a random twist moving the image by 4 pixels at most (1 px = 1/32 rad, or 3/32 m at 3 m)
        d = rng.normal(size=6) * np.repeat([3.0 / 32, 1.0 / 32], 3)
        pose = _perturb(IDENT, d * 4.0 / _motion(cam, IDENT, d))
        fwd = O.forward(pts, [cam], [pose], prm)
        G = (fwd.image - target).astype(F)
        bwd = O.backward(pts, [cam], [pose], prm, fwd, G)
        L0 = 0.5 * float(((fwd.image - target) ** 2).sum())
        # pose step: the preconditioned -d_pose (pixel scales as above), 1 px of largest image motion
        g = bwd.dpose[0].copy()
        step = -g
        step[:3] *= (3.0 / 32) ** 2
        step[3:] *= (1.0 / 32) ** 2
        step /= _motion(cam, pose, step)
        ok["pose down"] += L(pts, _perturb(pose, step)) < L0
        ok["pose up"] += L(pts, _perturb(pose, -step)) > L0
        # ghost step: every ghost with a gradient moves ~1 layer-0 pixel along -dx (image-plane motion J R dx)
        gh = np.nonzero(np.abs(bwd.dx).sum(0))[0]
        R = pose.R.astype(np.float64)
        move = np.zeros_like(pos, dtype=np.float64)
        for i in gh:
            _, Xc, *_ = O.project(cam, pose, *pos[:, i])
            move[:, i] = -bwd.dx[:, i] / np.linalg.norm(O.jacobian(cam, Xc) @ (R @ bwd.dx[:, i]))
        A0 = L(pts, pose, prm_all, target_all)
        ok["ghosts down"] += L(O.Points((pos + move).astype(F), pts.radius, tex), pose, prm_all, target_all) < A0
        ok["ghosts up"] += L(O.Points((pos - move).astype(F), pts.radius, tex), pose, prm_all, target_all) > A0
    print("descent:", ok)
    for k, v in ok.items():
        assert v >= 95, (k, ok)
