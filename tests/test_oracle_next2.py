"""Pins for NEXT-2 in the oracle -- CPU only:
  * the spherical environment map E of Eq. 7 ("background color sampled from a spherical environment
    map", P:L224-229 E(R^T C^{-1}(u, v))) with the parameterization of reading R29, and its gradient
    ("straightforward");
  * logarithmic descriptors (stored as log, converted to linear space during rasterization).
"""
import dataclasses
import math

import numpy as np
import pytest

from oracle import oracle as O
from paper_2110_06635_b200 import scene as S

F = np.float32
IDENT = S.Pose(np.eye(3, dtype=F), np.zeros(3, dtype=F))


def _roty(deg):
    a = math.radians(deg)
    return np.array([[math.cos(a), 0, math.sin(a)], [0, 1, 0], [-math.sin(a), 0, math.cos(a)]], dtype=F)


# --------------------------------------------------------------------------- #
# C^{-1} and the equirectangular lookup (R29)
# --------------------------------------------------------------------------- #
def test_unproject_pinhole_closed_form_and_opencv_round_trip():
    cam = S.pinhole(640, 480)
    xn, yn = O.unproject(cam, 400.0, 100.0)
    assert xn == pytest.approx((400.0 - cam.cx) / cam.fx, abs=1e-15)
    assert yn == pytest.approx((100.0 - cam.cy) / cam.fy, abs=1e-15)
    oc = S.opencv_camera(640, 480, seed=5)
    rng = np.random.default_rng(1)
    for _ in range(50):
        u0, v0 = rng.uniform(0, 640), rng.uniform(0, 480)
        xn, yn = O.unproject(oc, u0, v0)
        uv = O.project_f64(oc, np.array([xn, yn, 1.0]))  # independent forward map (Eq. 2 + R6)
        assert uv == pytest.approx([u0, v0], abs=1e-8)


def test_env_direction_closed_forms():
    cam = S.pinhole(64, 48, f=32.0, cx=32.0, cy=24.0)
    np.testing.assert_allclose(O.env_dir(cam, IDENT, 0, 32, 24), [0, 0, 1], atol=1e-15)
    # layer 2 pixel (12, 3) is layer-0 (48, 12): xn = 0.5, yn = -0.375
    np.testing.assert_allclose(O.env_dir(cam, IDENT, 2, 12, 3), [0.5, -0.375, 1.0], atol=1e-15)
    # d = R^T dc: a camera turned 90 degrees about y looks along world -x or +x
    pose = S.Pose(_roty(90.0), np.zeros(3, F))
    np.testing.assert_allclose(O.env_dir(cam, pose, 0, 32, 24), _roty(90.0).T.astype(np.float64) @ [0, 0, 1],
                               atol=1e-7)


def test_env_taps_closed_forms_wrap_and_clamp():
    E = np.zeros((8, 16, 1), F)
    idx, w = O.env_taps(E, [0.0, 0.0, 1.0])    # lon = lat = 0 -> s = 7.5, t = 3.5: the 4 centre texels
    assert sorted(idx.tolist()) == [3 * 16 + 7, 3 * 16 + 8, 4 * 16 + 7, 4 * 16 + 8]
    np.testing.assert_allclose(w, 0.25)
    idx, w = O.env_taps(E, [1.0, 0.0, 0.0])    # lon = pi/2 -> s = 11.5
    assert sorted(set((idx % 16).tolist())) == [11, 12]
    idx, w = O.env_taps(E, [0.0, 0.0, -1.0])   # lon = pi -> s = 15.5: columns 15 and 0 (wrap)
    assert sorted(set((idx % 16).tolist())) == [0, 15] and np.isclose(w.sum(), 1.0)
    idx, w = O.env_taps(E, [0.0, 1.0, 0.0])    # lat = pi/2 -> t = 7.5: rows 7 and 8 -> both clamped to 7
    assert set((idx // 16).tolist()) == {7} and np.isclose(w.sum(), 1.0)


def test_bilinear_reproduces_a_linear_texture():
    H, W = 16, 32
    r, c = np.meshgrid(np.arange(H), np.arange(W), indexing="ij")
    E = (0.25 * c + 0.5 * r).astype(F)[..., None]
    rng = np.random.default_rng(2)
    for _ in range(40):
        lon, lat = rng.uniform(-2.5, 2.5), rng.uniform(-1.2, 1.2)   # away from the wrap seam and the poles
        d = [math.cos(lat) * math.sin(lon), math.sin(lat), math.cos(lat) * math.cos(lon)]
        s = (lon / (2 * math.pi) + 0.5) * W - 0.5
        t = (lat / math.pi + 0.5) * H - 0.5
        idx, w = O.env_taps(E, d)
        val = float((w * E.reshape(-1)[idx]).sum())
        assert val == pytest.approx(0.25 * s + 0.5 * t, abs=1e-12)


# --------------------------------------------------------------------------- #
# forward / backward with an environment map
# --------------------------------------------------------------------------- #
def _scene(C=3, ghost=0.2, log=False, env=None, opencv=False, seed=11):
    room = S.make_room(4.0)
    cloud = S.room_cloud(3000, room, channels=C, seed=seed)
    cams = [S.opencv_camera(96, 64, seed=5) if opencv else S.pinhole(96, 64), S.pinhole(96, 64)]
    poses = S.room_poses(2, room, seed=3)
    pts = O.Points.from_cloud(cloud)
    pts = O.Points(pts.pos, np.full(pts.n, 0.03, F), pts.feat)
    prm = S.Params(layers=3, discard=True, ghost_rate=ghost, seed=77, log_descriptors=log, env_map=env)
    return pts, cams, poses, prm


def test_env_forward_empty_pixels_sample_E_and_constant_map_equals_background():
    rng = np.random.default_rng(3)
    E = rng.random((12, 24, 3)).astype(F)
    pts, cams, poses, prm = _scene(env=E)
    fwd = O.forward(pts, cams, poses, prm)
    P = fwd.count.shape[1]
    base = O.forward(pts, cams, poses, dataclasses.replace(prm, env_map=None))
    np.testing.assert_array_equal(fwd.keys, base.keys)          # E affects only the empty pixels
    np.testing.assert_array_equal(fwd.count, base.count)
    for v in range(2):
        img = fwd.image[v].reshape(-1)
        for l in range(3):
            wl, hl = -(-96 // (1 << l)), -(-64 // (1 << l))
            off = O.pyramid_pixels(96, 64, l) if l else 0
            for j in rng.choice(wl * hl, 40, replace=False):
                if fwd.count[v, off + j] != 0:
                    assert img[3 * off + j] == base.image[v].reshape(-1)[3 * off + j]
                    continue
                idx, w = O.env_taps(E, O.env_dir(cams[v], poses[v], l, j % wl, j // wl))
                for c in range(3):
                    assert img[3 * off + c * wl * hl + j] == pytest.approx((w * E[..., c].reshape(-1)[idx]).sum(),
                                                                           abs=1e-12)
    const = np.broadcast_to(np.array([0.3, -0.2, 0.7], F), (5, 7, 3)).copy()
    a = O.forward(pts, cams, poses, dataclasses.replace(prm, env_map=const))
    b = O.forward(pts, cams, poses, dataclasses.replace(prm, env_map=None, background=[0.3, -0.2, 0.7]))
    np.testing.assert_allclose(a.image, b.image, atol=1e-7)   # R18 is E constant
    assert P > 0


@pytest.mark.parametrize("opencv", [False, True])
def test_env_gradient_is_exact_derivative(opencv):
    """I is linear in E (geometry fixed), so for any E' the identity sum(dL/dE * E') = L(E') - L(0) is
    exact; also spot central differences."""
    rng = np.random.default_rng(4)
    E = rng.random((10, 20, 3)).astype(F)
    pts, cams, poses, prm = _scene(env=E, opencv=opencv)
    fwd = O.forward(pts, cams, poses, prm)
    G = (rng.random(fwd.image.shape) * 2 - 1).astype(F)
    bwd = O.backward(pts, cams, poses, prm, fwd, G)
    assert np.count_nonzero(bwd.denv) > 100

    def L(Em):
        f = O.forward(pts, cams, poses, dataclasses.replace(prm, env_map=Em))
        return float((f.image * G.astype(np.float64)).sum())
    E2 = (rng.random(E.shape) * 2 - 1).astype(F)
    lhs = float((bwd.denv * E2.astype(np.float64)).sum())
    assert lhs == pytest.approx(L(E2) - L(np.zeros_like(E)), rel=1e-9, abs=1e-9)
    for _ in range(5):
        k = tuple(rng.integers(0, s) for s in E.shape)
        Ep, Em = E.copy(), E.copy()
        Ep[k] += F(0.25)
        Em[k] -= F(0.25)
        step = float(Ep[k]) - float(Em[k])  # E is fp32: divide by the actual step
        assert (L(Ep) - L(Em)) / step == pytest.approx(bwd.denv[k], rel=1e-9, abs=1e-9)


# --------------------------------------------------------------------------- #
# logarithmic descriptors
# --------------------------------------------------------------------------- #
def test_log_descriptors_forward_equals_linear_forward_of_exp():
    pts, cams, poses, prm = _scene(log=True)
    a = O.forward(pts, cams, poses, prm)
    lin = O.Points(pts.pos, pts.radius, np.exp(pts.feat.astype(np.float64)).astype(F))
    b = O.forward(lin, cams, poses, dataclasses.replace(prm, log_descriptors=False))
    np.testing.assert_array_equal(a.keys, b.keys)
    np.testing.assert_array_equal(a.count, b.count)
    np.testing.assert_allclose(a.image, b.image, rtol=2e-7)    # b's descriptors went through fp32


def test_log_descriptor_gradients():
    """Texture gradient = exp(tau) x the linear-space gradient (chain rule) and matches central FD; the
    ghosts' structural gradients only see the linear descriptor exp(tau)."""
    rng = np.random.default_rng(5)
    pts, cams, poses, prm = _scene(log=True, ghost=0.25)
    fwd = O.forward(pts, cams, poses, prm)
    G = (rng.random(fwd.image.shape) * 2 - 1).astype(F)
    bwd = O.backward(pts, cams, poses, prm, fwd, G)
    lin = O.Points(pts.pos, pts.radius, np.exp(pts.feat.astype(np.float64)).astype(F))
    prm_l = dataclasses.replace(prm, log_descriptors=False)
    fl = O.forward(lin, cams, poses, prm_l)
    bl = O.backward(lin, cams, poses, prm_l, fl, G)
    np.testing.assert_allclose(bwd.dtau, np.exp(pts.feat.astype(np.float64)) * bl.dtau, rtol=1e-6, atol=1e-12)
    np.testing.assert_allclose(bwd.dx, bl.dx, rtol=1e-5, atol=1e-9 * np.abs(bl.dx).max())
    np.testing.assert_allclose(bwd.dpose, bl.dpose, rtol=1e-5, atol=1e-9 * np.abs(bl.dpose).max())
    nz = np.argwhere(bwd.dtau != 0)
    assert len(nz) > 50

    def L(feat):
        f = O.forward(O.Points(pts.pos, pts.radius, feat), cams, poses, prm)
        return float((f.image * G.astype(np.float64)).sum())
    for i, c in nz[rng.choice(len(nz), 10, replace=False)]:
        fp, fm = pts.feat.copy(), pts.feat.copy()
        fp[i, c] = F(fp[i, c] + F(2.0 ** -10))
        fm[i, c] = F(fm[i, c] - F(2.0 ** -10))
        fd = (L(fp) - L(fm)) / (float(fp[i, c]) - float(fm[i, c]))
        assert fd == pytest.approx(bwd.dtau[i, c], rel=1e-6, abs=1e-9)
