"""Pins for the oracle's backward pass (texture gradient, Eqs. 9-11, ghosts, chain rule) -- CPU only."""
import dataclasses
import json
import math
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2110_06635_b200 import scene as S

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_values.json")))
F = np.float32
IDENT = S.Pose(np.eye(3, dtype=F), np.zeros(3, dtype=F))


def _cam(w, h, f, cx, cy):
    return S.Camera(w, h, S.PINHOLE, float(F(f)), float(F(f)), float(F(cx)), float(F(cy)))


def _at_pixel(cam, u, v, z):
    """World point (identity pose) whose layer-0 projection rounds to pixel (u, v) at depth z."""
    return [(u - cam.cx) * z / cam.fx, (v - cam.cy) * z / cam.fy, z]


def arrange(render, ghost, params, feat_r, feat_g):
    """Build a cloud whose global indices put `render` points on non-ghost ids and `ghost` points on ghost
    ids (R13 hash), padding unused ids with points behind the camera.  -> (Points, ghost ids)."""
    render, ghost = list(render), list(ghost)
    feat_r, feat_g = list(feat_r), list(feat_g)
    xyz, feat, gids = [], [], []
    C = len((feat_r + feat_g)[0])
    gi = 0
    while render or ghost:
        is_g = O.is_ghost(params, gi)
        if is_g and ghost:
            xyz.append(ghost.pop(0)); feat.append(feat_g.pop(0)); gids.append(gi)
        elif not is_g and render:
            xyz.append(render.pop(0)); feat.append(feat_r.pop(0))
        else:
            xyz.append([0.0, 0.0, -1.0]); feat.append([0.0] * C)
        gi += 1
    pos = np.asarray(xyz, dtype=F).T.copy()
    return O.Points(pos, np.full(pos.shape[1], 0.005, F), np.asarray(feat, F)), gids


def _grad_image(cam, L, C, fill):
    P = O.pyramid_pixels(cam.width, cam.height, L)
    return np.full((1, C * P), fill, dtype=F)


# --------------------------------------------------------------------------- #
# texture gradient (§4.2 "straightforward", R24)
# --------------------------------------------------------------------------- #
@pytest.mark.parametrize("case", GOLDEN["texture_grad"])
def test_texture_grad_worked(case):
    cam = _cam(16, 16, 8.0, 8.0, 8.0)
    k = case["points_in_pixel"]
    pts = O.Points(np.asarray([[0.0, 0.0, 2.0 + 0.001 * i] for i in range(k)], F).T.copy(),
                   np.full(k, 0.005, F), np.full((k, 1), 0.5, F))
    prm = S.Params(layers=1, discard=False)
    fwd = O.forward(pts, [cam], [IDENT], prm)
    G = _grad_image(cam, 1, 1, 0.0)
    G[0, 8 * 16 + 8] = case["adjoint"]
    bwd = O.backward(pts, [cam], [IDENT], prm, fwd, G)
    assert np.allclose(bwd.dtau[:, 0], case["d_tau_each"])


def _loss(pts, cams, poses, prm, G):
    fwd = O.forward(pts, cams, poses, prm)
    return float((fwd.image * G.astype(np.float64)).sum()), fwd


def test_texture_grad_equals_finite_differences():
    """I is linear in tau with geometry fixed, so a central FD on tau is exact up to rounding."""
    rng = np.random.default_rng(0)
    room = S.make_room(4.0)
    cloud = S.room_cloud(3000, room, channels=3, seed=11)
    cams = [S.pinhole(96, 64), S.opencv_camera(96, 64, seed=5)]
    poses = S.room_poses(2, room, seed=3)
    pts = O.Points.from_cloud(cloud)
    pts = O.Points(pts.pos, np.full(pts.n, 0.03, F), pts.feat)
    prm = S.Params(layers=3, discard=True, ghost_rate=0.2, seed=77)
    P = O.pyramid_pixels(96, 64, 3)
    G = (rng.random((2, 3 * P)) * 2 - 1).astype(F)
    L0, fwd = _loss(pts, cams, poses, prm, G)
    bwd = O.backward(pts, cams, poses, prm, fwd, G)
    nz = np.argwhere(bwd.dtau != 0)
    assert len(nz) > 50
    picks = list(nz[rng.choice(len(nz), 25, replace=False)]) + [np.argwhere(bwd.dtau == 0)[0]]
    for i, c in picks:
        h = F(1.0 / 1024)
        fp, fm = pts.feat.copy(), pts.feat.copy()
        fp[i, c] = F(fp[i, c] + h)
        fm[i, c] = F(fm[i, c] - h)
        Lp, _ = _loss(O.Points(pts.pos, pts.radius, fp), cams, poses, prm, G)
        Lm, _ = _loss(O.Points(pts.pos, pts.radius, fm), cams, poses, prm, G)
        fd = (Lp - Lm) / (float(fp[i, c]) - float(fm[i, c]))
        assert abs(fd - bwd.dtau[i, c]) < 1e-9 * max(1.0, abs(fd)), (i, c, fd, bwd.dtau[i, c])


# --------------------------------------------------------------------------- #
# Eq. 11 (R14)
# --------------------------------------------------------------------------- #
def _key(m, idx=0):
    if m is None:
        return O.SENTINEL
    return (int(np.array([m], F).view(np.uint32)[0]) << 32) | idx


@pytest.mark.parametrize("case", GOLDEN["eq11"])
def test_eq11_worked_values(case):
    kase, d = O.induced_change([case["tau"]], case["z"], 0.01, case["n"], _key(case["m"]), [case["I"]])
    assert kase == case["case"]
    assert abs(d[0] - case["delta"]) < 1e-7


def test_eq11_equals_rerender_with_ghost_inserted():
    """For cases 1-3 and case 4 with z >= min_z, Delta of Eq. 11 is exactly the change of Eq. 7 at the
    neighbour when the shifted point is rendered there (S:L351 cross-check, generalised)."""
    rng = np.random.default_rng(1)
    cam = _cam(8, 4, 4.0, 4.0, 2.0)
    prm = S.Params(layers=1, discard=False, alpha=0.01)
    seen = set()
    for trial in range(400):
        n = int(rng.integers(0, 4))
        base_z = rng.uniform(1.0, 2.0)
        depths = base_z * (1 + rng.uniform(0, 0.012, n))
        xyz = [_at_pixel(cam, 5, 2, z) for z in depths]
        tau = rng.random((n, 2)).astype(F)
        zg = F(base_z * rng.choice([0.9, 0.995, 1.0, 1.004, 1.02, 1.2]))
        tg = rng.random(2).astype(F)
        pts = O.Points(np.asarray(xyz, F).reshape(-1, 3).T.copy(), np.full(n, 0.005, F), tau.reshape(n, 2))
        fwd = O.forward(pts, [cam], [IDENT], prm)
        q = 2 * 8 + 5
        Iq = [fwd.image[0, c * 32 + q] for c in range(2)]
        kase, delta = O.induced_change(tg, zg, prm.alpha, fwd.count[0, q], int(fwd.keys[0, q]), Iq)
        m_q = np.array([int(fwd.keys[0, q]) >> 32], np.uint32).view(F)[0]
        if kase == 4 and zg < m_q:
            continue
        seen.add(kase)
        xyz2 = np.asarray(xyz + [_at_pixel(cam, 5, 2, float(zg))], F).reshape(-1, 3).T.copy()
        assert O.project(cam, IDENT, *xyz2[:, -1])[1][2] == zg
        pts2 = O.Points(xyz2, np.full(n + 1, 0.005, F), np.vstack([tau.reshape(n, 2), tg[None]]))
        fwd2 = O.forward(pts2, [cam], [IDENT], prm)
        for c in range(2):
            assert abs((fwd2.image[0, c * 32 + q] - Iq[c]) - delta[c]) < 1e-12, (trial, kase)
    assert seen == {1, 2, 3, 4}


# --------------------------------------------------------------------------- #
# Eqs. 9-10 spatial gradient, ghosts (§4.3), chain rule (Eq. 8, Eq. 17)
# --------------------------------------------------------------------------- #
GPRM = S.Params(layers=1, discard=False, alpha=0.01, ghost_rate=0.5, seed=4242)


def test_linear_ramp_recovers_gradient():
    """Rendered row I(u) = c*u at depth 2, ghost in front carrying tau = I(u_g): the signed central
    difference (R15) gives g_u = -G*c exactly (S:L359 ramp; magnitude G*c, sign from moving right onto a
    brighter pixel lowering L = sum G*I).  dx = J^T g with J = [fx/Z, 0, -fx X/Z^2] (R21)."""
    cam = _cam(32, 8, 8.0, 16.0, 4.0)
    c = 1.0 / 64  # exact in fp32
    render = [_at_pixel(cam, u, 4, 2.0) for u in range(32)]
    feats = [[c * u] for u in range(32)]
    pts, gids = arrange(render, [_at_pixel(cam, 16, 4, 1.0)], GPRM, feats, [[c * 16]])
    fwd = O.forward(pts, [cam], [IDENT], GPRM)
    G = _grad_image(cam, 1, 1, 0.0)
    G[0, 4 * 32: 5 * 32] = 1.0
    bwd = O.backward(pts, [cam], [IDENT], GPRM, fwd, G)
    g = gids[0]
    gu = -1.0 * c
    np.testing.assert_allclose(bwd.dx[:, g], [8.0 / 1.0 * gu, 0.0, 0.0], atol=1e-9)
    np.testing.assert_allclose(bwd.dpose[0], [8.0 * gu, 0, 0, 0, 8.0 * gu, 0], atol=1e-9)  # (w, Xc x w), Xc = (0,0,1)
    # only the ghost gets a spatial gradient, only rendered points get texture gradients (Fig. 4, R22)
    assert np.count_nonzero(bwd.dx) == 1 and bwd.dtau[g, 0] == 0.0
    assert np.count_nonzero(bwd.dtau) > 0


def test_border_drops_outside_neighbour():
    """at u = 0 the left term is dropped, g_u = 1/2 <G(1,v), Delta+>."""
    cam = _cam(8, 4, 4.0, 4.0, 2.0)
    pts, gids = arrange([], [_at_pixel(cam, 0, 2, 1.0)], GPRM, [], [[0.75]])
    fwd = O.forward(pts, [cam], [IDENT], GPRM)
    G = _grad_image(cam, 1, 1, 0.0)
    G[0, 2 * 8 + 1] = 2.0   # right neighbour: background (case 1), Delta = 0.75 - 0
    bwd = O.backward(pts, [cam], [IDENT], GPRM, fwd, G)
    gu = 0.5 * 2.0 * 0.75
    np.testing.assert_allclose(bwd.dx[:, gids[0]], [4.0 * gu, 0.0, 4.0 * gu], atol=1e-9)  # J_u = [fx/Z, 0, -fx X/Z^2], X=-1


def test_uniform_covisible_field_gives_zero():
    """uniform image, uniform depth, tau = I -> every Delta vanishes (case 4) -> g = 0."""
    cam = _cam(12, 10, 6.0, 6.0, 5.0)
    render = [_at_pixel(cam, u, v, 2.0) for v in range(10) for u in range(12)]
    ghosts = [_at_pixel(cam, u, v, 2.0) for u, v in ((3, 3), (6, 5), (0, 0), (11, 9))]
    pts, gids = arrange(render, ghosts, GPRM, [[0.5, 0.25]] * len(render), [[0.5, 0.25]] * 4)
    fwd = O.forward(pts, [cam], [IDENT], GPRM)
    G = np.random.default_rng(2).uniform(-1, 1, (1, 2 * 120)).astype(F)
    bwd = O.backward(pts, [cam], [IDENT], GPRM, fwd, G)
    assert np.abs(bwd.dx).max() < 1e-12 and np.abs(bwd.dpose).max() < 1e-12


def test_empty_ghost_set_gives_zero_structural_gradients():
    room = S.make_room(4.0)
    pts = O.Points.from_cloud(S.room_cloud(2000, room, 3, seed=5))
    cams, poses = [S.pinhole(64, 48)], S.room_poses(1, room)
    prm = S.Params(layers=3, discard=True, ghost_rate=0.0)
    fwd = O.forward(pts, cams, poses, prm)
    G = S.grad_pyramid(1, 3, fwd.count.shape[1]).numpy()
    bwd = O.backward(pts, cams, poses, prm, fwd, G)
    assert not bwd.dx.any() and not bwd.dpose.any()


def _rodrigues(w):
    th = np.linalg.norm(w)
    K = np.array([[0, -w[2], w[1]], [w[2], 0, -w[0]], [-w[1], w[0], 0]])
    if th < 1e-300:
        return np.eye(3)
    return np.eye(3) + math.sin(th) / th * K + (1 - math.cos(th)) / th ** 2 * K @ K


def test_pose_gradient_is_left_tangent_chain_rule():
    """Eq. 17: d/dxi of w . (exp(xi) Xc) at 0 equals (w, Xc x w) (R19); translation part = R dx (Xc = R x + t)."""
    room = S.make_room(4.0)
    cloud = S.room_cloud(4000, room, 2, seed=8)
    pts = O.Points.from_cloud(cloud)
    pts = O.Points(pts.pos, np.full(pts.n, 0.02, F), pts.feat)
    cams, poses = [S.pinhole(80, 60)], S.room_poses(1, room, seed=9)
    prm = S.Params(layers=3, discard=True, ghost_rate=0.3, seed=3)
    fwd = O.forward(pts, cams, poses, prm)
    G = S.grad_pyramid(1, 2, fwd.count.shape[1], seed=12).numpy()
    bwd = O.backward(pts, cams, poses, prm, fwd, G)
    R = poses[0].R.astype(np.float64)
    ghosts = np.nonzero(np.abs(bwd.dx).sum(0))[0]
    assert len(ghosts) > 20
    w = R @ bwd.dx[:, ghosts]                       # dL/dXc per ghost
    np.testing.assert_allclose(bwd.dpose[0, :3], w.sum(1), rtol=1e-6, atol=1e-9)  # fp32 R is orthonormal to ~1e-7
    rot = np.zeros(3)
    for j, i in enumerate(ghosts):
        Xc = O.project(cams[0], poses[0], *pts.pos[:, i])[1].astype(np.float64)
        for k in range(3):                          # FD through the exponential map (rotation part)
            e = np.zeros(3); e[k] = 1e-6
            rot[k] += w[:, j] @ (_rodrigues(e) @ Xc - _rodrigues(-e) @ Xc) / 2e-6
    np.testing.assert_allclose(bwd.dpose[0, 3:], rot, rtol=1e-6, atol=1e-9)


# --------------------------------------------------------------------------- #
# NEXT-1: camera-intrinsics gradient from the same ghost (g_u, g_v) (Eq. 8 into the camera model C of
# Eq. 2; the paper optimizes the camera model, Fig. 4)
# --------------------------------------------------------------------------- #
THETA = ["fx", "fy", "cx", "cy", "k1", "k2", "k3", "k4", "k5", "k6", "p1", "p2"]


def _perturbed(cam, j, h):
    """(camera with parameter j moved by ~h, the actual fp32 value of that parameter)."""
    if j < 4:
        v = float(F(getattr(cam, THETA[j]) + h))
        return dataclasses.replace(cam, **{THETA[j]: v}), v
    if j < 10:
        k = list(cam.k); k[j - 4] = float(F(k[j - 4] + h))
        return dataclasses.replace(cam, k=tuple(k)), k[j - 4]
    p = list(cam.p); p[j - 10] = float(F(p[j - 10] + h))
    return dataclasses.replace(cam, p=tuple(p)), p[j - 10]


@pytest.mark.parametrize("model", [S.PINHOLE, S.OPENCV8])
def test_intrinsics_jacobian_matches_finite_differences(model):
    """d(u0, v0)/d theta against central differences of the continuous fp64 projection with perturbed
    camera parameters (a pin independent of the closed form's algebra)."""
    cam = S.pinhole(640, 480) if model == S.PINHOLE else S.opencv_camera(640, 480, seed=5)
    rng = np.random.default_rng(7)
    for _ in range(20):
        X = np.array([rng.uniform(-0.6, 0.6), rng.uniform(-0.45, 0.45), 1.0], F) * F(rng.uniform(0.5, 4.0))
        Jt = O.intrinsics_jacobian(cam, X)
        for j in range(12):
            h = 2.0 ** -4 if j < 4 else 2.0 ** -12  # camera parameters are fp32: divide by the actual step
            cp, vp = _perturbed(cam, j, h)
            cm, vm = _perturbed(cam, j, -h)
            d = (O.project_f64(cp, X.astype(np.float64)) - O.project_f64(cm, X.astype(np.float64))) / (vp - vm)
            if model == S.PINHOLE and j >= 4:
                assert not Jt[:, j].any() and not d.any()  # the pinhole has no distortion parameters
            np.testing.assert_allclose(Jt[:, j], d, rtol=1e-5, atol=1e-6 * max(1.0, np.abs(d).max()))


def test_intrinsics_gradient_ramp_closed_form():
    """Linear ramp (g_u = -G c exactly, R15): ghosts at layer-0 columns 16 (xn = 0) and 20 (xn = 1/2) give
    dL/dcx = sum g_u, dL/dfx = sum g_u xn, dL/dfy = dL/dcy = 0."""
    cam = _cam(32, 8, 8.0, 16.0, 4.0)
    c = 1.0 / 64
    render = [_at_pixel(cam, u, 4, 2.0) for u in range(32)]
    feats = [[c * u] for u in range(32)]
    for col, xn in ((16, 0.0), (20, 0.5)):
        pts, gids = arrange(render, [_at_pixel(cam, col, 4, 1.0)], GPRM, feats, [[c * col]])
        fwd = O.forward(pts, [cam], [IDENT], GPRM)
        G = _grad_image(cam, 1, 1, 0.0)
        G[0, 4 * 32: 5 * 32] = 1.0
        bwd = O.backward(pts, [cam], [IDENT], GPRM, fwd, G)
        gu = -1.0 * c
        np.testing.assert_allclose(bwd.dintr[0, :4], [gu * xn, 0.0, gu, 0.0], atol=1e-12)
        assert not bwd.dintr[0, 4:].any()


def test_intrinsics_gradient_sums_pinhole_chain_rule_per_ghost():
    """Pinhole: per ghost, w = J^T g with J = [[fx/z, 0, -fx x/z^2], [0, fy/z, -fy y/z^2]] (R21) is
    invertible for (g_u, g_v) from w = R dx (pinned above); then d theta = sum (g_u xn, g_v yn, g_u, g_v)."""
    room = S.make_room(4.0)
    cloud = S.room_cloud(4000, room, 2, seed=8)
    pts = O.Points.from_cloud(cloud)
    pts = O.Points(pts.pos, np.full(pts.n, 0.02, F), pts.feat)
    cams, poses = [S.pinhole(80, 60)], S.room_poses(1, room, seed=9)
    prm = S.Params(layers=3, discard=True, ghost_rate=0.3, seed=3)
    fwd = O.forward(pts, cams, poses, prm)
    G = S.grad_pyramid(1, 2, fwd.count.shape[1], seed=12).numpy()
    bwd = O.backward(pts, cams, poses, prm, fwd, G)
    R = poses[0].R.astype(np.float64)
    ghosts = np.nonzero(np.abs(bwd.dx).sum(0))[0]
    assert len(ghosts) > 20
    ref = np.zeros(4)
    for i in ghosts:
        Xc = O.project(cams[0], poses[0], *pts.pos[:, i])[1].astype(np.float64)
        w = R @ bwd.dx[:, i]
        gu, gv = w[0] * Xc[2] / cams[0].fx, w[1] * Xc[2] / cams[0].fy
        ref += [gu * Xc[0] / Xc[2], gv * Xc[1] / Xc[2], gu, gv]
    np.testing.assert_allclose(bwd.dintr[0, :4], ref, rtol=1e-6, atol=1e-9)
    assert not bwd.dintr[0, 4:].any()


# --------------------------------------------------------------------------- #
# NEXT-3 (R31): ghost gradients disabled -- the §6.2 baseline: Eqs. 9-11 for rendered points
# --------------------------------------------------------------------------- #
def test_spatial_rendered_equals_ghost_gradient_of_the_same_point():
    """Eq. 11 only reads the NEIGHBOUR pixels' state (R14), which a point never changes (it lands on its own
    pixel), so the rendered-point spatial gradient of point i equals the ghost gradient i gets when it is
    made a ghost instead -- exactly; the texture gradients of the other points are unchanged."""
    cam = _cam(32, 8, 8.0, 16.0, 4.0)
    c = 1.0 / 64
    render = [_at_pixel(cam, u, 4, 2.0) for u in range(32)] + [_at_pixel(cam, u, 3, 2.5) for u in range(0, 32, 3)]
    feats = [[c * u] for u in range(32)] + [[0.3]] * 11
    probe = _at_pixel(cam, 16.2, 4.1, 1.0)
    prm_t = dataclasses.replace(GPRM, spatial_rendered=True)
    G = _grad_image(cam, 1, 1, 0.0)
    G[0, :] = np.linspace(-1, 1, G.shape[1], dtype=F)
    # (a) probe rendered, ghost gradients disabled
    pts_a, _ = arrange(render + [probe], [], GPRM, feats + [[c * 16]], [])
    fwd_a = O.forward(pts_a, [cam], [IDENT], prm_t)
    b_a = O.backward(pts_a, [cam], [IDENT], prm_t, fwd_a, G)
    ia = pts_a.n - 1
    while pts_a.pos[2, ia] < 0:
        ia -= 1
    # (b) probe as a ghost, ghost gradients on
    pts_b, gids = arrange(render, [probe], GPRM, feats, [[c * 16]])
    fwd_b = O.forward(pts_b, [cam], [IDENT], GPRM)
    b_b = O.backward(pts_b, [cam], [IDENT], GPRM, fwd_b, G)
    assert np.abs(b_b.dx[:, gids[0]]).sum() > 0
    np.testing.assert_array_equal(b_a.dx[:, ia], b_b.dx[:, gids[0]])
    # every rendered point now has a spatial gradient (incl. the ramp points), the pose sums them all
    assert np.count_nonzero(np.abs(b_a.dx).sum(0)) > 20
    assert b_a.dtau[ia, 0] != 0.0  # and keeps its texture gradient


def test_spatial_rendered_mode_gives_ghosts_nothing():
    room = S.make_room(4.0)
    cloud = S.room_cloud(4000, room, 2, seed=8)
    pts = O.Points.from_cloud(cloud)
    pts = O.Points(pts.pos, np.full(pts.n, 0.02, F), pts.feat)
    cams, poses = [S.pinhole(80, 60)], S.room_poses(1, room, seed=9)
    prm = S.Params(layers=3, discard=True, ghost_rate=0.3, seed=3)
    prm_t = dataclasses.replace(prm, spatial_rendered=True)
    fwd = O.forward(pts, cams, poses, prm)
    G = S.grad_pyramid(1, 2, fwd.count.shape[1], seed=12).numpy()
    b = O.backward(pts, cams, poses, prm, fwd, G)
    bt = O.backward(pts, cams, poses, prm_t, fwd, G)
    np.testing.assert_array_equal(bt.dtau, b.dtau)  # texture gradients do not depend on the mode
    ghost = np.array([O.is_ghost(prm, i) for i in range(pts.n)])
    assert not bt.dx[:, ghost].any() and np.abs(bt.dx[:, ~ghost]).sum() > 0
    assert not b.dx[:, ~ghost].any()
