"""Pins for the CPU oracle (oracle/adop_oracle.c) -- CPU only (-m "not gpu").

Each test ties the oracle to something other than itself: hand-evaluated
closed forms of the paper's equations, worked values (tests/golden), a
per-pixel brute force written separately (oracle/bruteforce.py), finite
differences, invariants, and special cases that reduce to textbook results.
"""
import dataclasses
import json
import math
import os

import numpy as np
import pytest

from oracle import bruteforce as BF
from oracle import oracle as O
from paper_2110_06635_b200 import scene as S

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_values.json")))
F = np.float32


def _cam(w=64, h=48, f=40.0, cx=None, cy=None, model=S.PINHOLE, k=(0.0,) * 6, p=(0.0, 0.0), r2_max=math.inf):
    return S.Camera(w, h, model, float(F(f)), float(F(f)), float(F(w / 2 if cx is None else cx)),
                    float(F(h / 2 if cy is None else cy)), tuple(k), tuple(p), r2_max)


IDENT = S.Pose(np.eye(3, dtype=F), np.zeros(3, dtype=F))


def _points(xyz, feat=None, radius=None, goff=0):
    xyz = np.asarray(xyz, dtype=F).reshape(-1, 3).T.copy()
    n = xyz.shape[1]
    feat = np.full((n, 1), 0.5, dtype=F) if feat is None else np.asarray(feat, dtype=F).reshape(n, -1)
    radius = np.full(n, 0.005, dtype=F) if radius is None else np.asarray(radius, dtype=F)
    return O.Points(xyz, radius, feat, goff)


def _layer_hits(keys, cam, layers):
    """-> list per layer of (u, v) pixels with a non-sentinel key."""
    dims, _ = S.layer_dims(cam.width, cam.height, layers)
    out = []
    for wl, hl, off in dims:
        idx = np.nonzero(keys[off:off + wl * hl] != np.uint64(O.SENTINEL))[0]
        out.append([(int(j % wl), int(j // wl)) for j in idx])
    return out


# --------------------------------------------------------------------------- #
# Eq. 2-4: projection, rounding, bounds
# --------------------------------------------------------------------------- #
@pytest.mark.parametrize("case", GOLDEN["projection"])
def test_projection_closed_forms(case):
    c = case["cam"]
    cam = _cam(c["w"], c["h"], c["f"], c["cx"], c["cy"])
    if "Xc" in case:
        ok, Xc, u0, v0, iz = O.project(cam, IDENT, *case["Xc"])
        assert ok
        assert abs(u0 - case["uv"][0]) < 1e-4 and abs(v0 - case["uv"][1]) < 1e-4
        assert Xc[2] == F(case["z"])
        return
    pose = S.tiny_pose()
    ok, Xc, u0, v0, iz = O.project(cam, pose, *case["world"])
    assert ok
    if "uv" in case:
        assert (u0, v0) == tuple(case["uv"]) and Xc[2] == F(case["z"])
    if "u_pixels" in case:
        pts = _points([case["world"]])
        prm = S.Params(layers=4, discard=False)
        keys = O.forward_depth(pts, [cam], [pose], prm)[0]
        hits = _layer_hits(keys, cam, 4)
        assert [h[0] for h in hits] == list(zip(case["u_pixels"], case["v_pixels"]))


@pytest.mark.parametrize("case", GOLDEN["rounding"])
def test_rounding_rule(case):
    cam = _cam(64, 64, 1.0, case["uv0"][0], case["uv0"][1])
    pts = _points([[0.0, 0.0, 1.0]])
    L = case["layer"] + 1
    keys = O.forward_depth(pts, [cam], [IDENT], S.Params(layers=L, discard=False))[0]
    assert _layer_hits(keys, cam, L)[case["layer"]] == [tuple(case["pixel"])]


@pytest.mark.parametrize("case", GOLDEN["layer_sizes"])
def test_layer_sizes(case):
    assert O.pyramid_pixels(case["w"], case["h"], case["layers"]) == case["pixels"]
    if "dims" in case:
        dims, _ = S.layer_dims(case["w"], case["h"], case["layers"])
        assert [[a, b] for a, b, _ in dims] == case["dims"]


def test_bounds_and_validity():
    cam = _cam(8, 8, 1.0, 0.0, 0.0)
    # u0 = -0.5 rounds away from zero to -1 -> outside at layer 0; -0.49 -> 0 inside (Eq. 4, R3)
    for cx, inside in [(-0.5, False), (-0.49, True), (7.49, True), (7.5, False)]:
        c = dataclasses.replace(cam, cx=cx, cy=3.0)
        keys = O.forward_depth(_points([[0, 0, 1]]), [c], [IDENT], S.Params(layers=1, discard=False))[0]
        assert (keys != np.uint64(O.SENTINEL)).any() == inside, cx
    # behind the camera, on the principal plane, non-finite: culled silently (R7)
    for xyz in ([0, 0, -1], [0, 0, 0], [0, 0, np.inf], [np.nan, 0, 1], [0, 0, np.nan]):
        ok = O.project(cam, IDENT, *[F(v) for v in xyz])[0]
        keys = O.forward_depth(_points([xyz]), [dataclasses.replace(cam, cx=4.0, cy=4.0)], [IDENT],
                               S.Params(layers=1, discard=False))[0]
        assert not (keys != np.uint64(O.SENTINEL)).any(), xyz
        if xyz[2] in (-1, 0, np.inf):
            assert not ok
    # a point left of layer 0 can still land in layer 1 (every layer is tested on its own)
    c = dataclasses.replace(cam, cx=-0.9, cy=3.0)
    keys = O.forward_depth(_points([[0, 0, 1]]), [c], [IDENT], S.Params(layers=2, discard=False))[0]
    hits = _layer_hits(keys, c, 2)
    assert hits[0] == [] and hits[1] == [(0, 2)]


def test_layer_scale_equivariance():
    """Eq. 2: P_l = P_0 / 2^l exactly in fp32 -> layer-l pixel = round(u0 / 2^l)."""
    rng = np.random.default_rng(0)
    cam = _cam(640, 480, 300.0)
    xyz = np.c_[rng.uniform(-1, 1, (500, 2)), rng.uniform(1, 3, 500)]
    pts = _points(xyz)
    L = 5
    keys = O.forward_depth(pts, [cam], [IDENT], S.Params(layers=L, discard=False))[0]
    dims, _ = S.layer_dims(cam.width, cam.height, L)
    for i in range(0, 500, 37):
        ok, Xc, u0, v0, _ = O.project(cam, IDENT, *[F(v) for v in xyz[i]])
        for l, (wl, hl, off) in enumerate(dims):
            u = BF.round_half_away(F(u0) / F(2 ** l))
            v = BF.round_half_away(F(v0) / F(2 ** l))
            if 0 <= u < wl and 0 <= v < hl:
                assert keys[off + int(v) * wl + int(u)] != np.uint64(O.SENTINEL)


# --------------------------------------------------------------------------- #
# Camera model (R6) and Jacobian (R21)
# --------------------------------------------------------------------------- #
def test_opencv_zero_distortion_is_pinhole_bitexact():
    rng = np.random.default_rng(1)
    pin = _cam(640, 480, 320.0)
    dist = dataclasses.replace(pin, model=S.OPENCV8, r2_max=math.inf)
    for _ in range(2000):
        xyz = [F(v) for v in (*rng.uniform(-2, 2, 2), rng.uniform(0.1, 5))]
        a = O.project(pin, IDENT, *xyz)
        b = O.project(dist, IDENT, *xyz)
        assert a[0] == b[0] and a[2] == b[2] and a[3] == b[3]


def test_opencv_single_k1_closed_form():
    cam = _cam(640, 480, 320.0, model=S.OPENCV8, k=(0.05, 0, 0, 0, 0, 0), r2_max=10.0)
    rng = np.random.default_rng(2)
    for _ in range(500):
        X = rng.uniform(-1, 1, 2)
        Z = rng.uniform(1, 3)
        xyz = [F(X[0]), F(X[1]), F(Z)]
        ok, Xc, u0, v0, _ = O.project(cam, IDENT, *xyz)
        xn, yn = float(xyz[0]) / float(xyz[2]), float(xyz[1]) / float(xyz[2])
        r2 = xn * xn + yn * yn
        assert ok
        assert abs(u0 - (cam.fx * xn * (1 + 0.05 * r2) + cam.cx)) < 2e-3
        assert abs(v0 - (cam.fy * yn * (1 + 0.05 * r2) + cam.cy)) < 2e-3


def test_opencv_guard_culls_outside_r2max():
    cam = S.opencv_camera(1024, 1024, seed=9)
    assert 0 < cam.r2_max < math.inf
    r = math.sqrt(cam.r2_max)
    ok_in = O.project(cam, IDENT, F(0.99 * r), F(0.0), F(1.0))[0]
    ok_out = O.project(cam, IDENT, F(1.01 * r), F(0.0), F(1.0))[0]
    assert ok_in and not ok_out


@pytest.mark.parametrize("model", [S.PINHOLE, S.OPENCV8])
def test_jacobian_matches_finite_differences(model):
    rng = np.random.default_rng(3)
    cam = S.opencv_camera(1920, 1080, seed=4) if model == S.OPENCV8 else _cam(1920, 1080, 960.0)
    for _ in range(200):
        X = np.array([rng.uniform(-0.5, 0.5), rng.uniform(-0.3, 0.3), rng.uniform(1, 4)], dtype=F)
        J = O.jacobian(cam, X)
        Xd = X.astype(np.float64)
        Jfd = np.zeros((2, 3))
        for k in range(3):
            h = 1e-6 * max(1.0, abs(Xd[k]))
            e = np.zeros(3); e[k] = h
            Jfd[:, k] = (O.project_f64(cam, Xd + e) - O.project_f64(cam, Xd - e)) / (2 * h)
        assert np.allclose(J, Jfd, rtol=1e-5, atol=1e-4 * np.abs(Jfd).max())
        # the fp32 pinned projection agrees with the continuous one to fp32 rounding
        ok, _, u0, v0, _ = O.project(cam, IDENT, *X)
        uv = O.project_f64(cam, Xd)
        assert ok and abs(u0 - uv[0]) < 1e-3 and abs(v0 - uv[1]) < 1e-3


def test_project_matches_independent_numpy_fp32():
    """The C oracle (built -ffp-contract=off) and numpy per-op fp32 agree bit for bit."""
    rng = np.random.default_rng(5)
    cams = [S.opencv_camera(1920, 1080, seed=s) for s in range(3)] + [_cam(1920, 1080, 960.0)]
    poses = S.room_poses(3, S.make_room(10.0))
    for cam in cams:
        for pose in poses:
            for _ in range(300):
                xyz = [F(v) for v in rng.uniform(-5, 5, 3)]
                a = O.project(cam, pose, *xyz)
                b = BF.project(cam, pose, *xyz, F(0.0))
                assert a[0] == (b is not None)
                if b is not None:
                    assert (a[2], a[3], a[1][2]) == (float(b[3]), float(b[4]), float(b[2]))


# --------------------------------------------------------------------------- #
# Eq. 6-7: depth test, fuzzy test, blend
# --------------------------------------------------------------------------- #
def _axis_points(depths, feats, cam):
    return _points([[0.0, 0.0, d] for d in depths], feat=np.asarray(feats, dtype=F).reshape(len(depths), -1))


@pytest.mark.parametrize("case", GOLDEN["fuzzy"])
def test_fuzzy_boundary(case):
    cam = _cam(16, 16, 8.0)
    pts = _axis_points([case["min_z"], case["z"]], [[1.0], [3.0]], cam)
    prm = S.Params(layers=1, discard=False, alpha=case["alpha"])
    fwd = O.forward(pts, [cam], [IDENT], prm)
    p = 8 * 16 + 8
    assert fwd.count[0, p] == (2 if case["pass"] else 1)
    # alpha = 0 reduces Eq. 6 to z <= min_z
    fwd0 = O.forward(pts, [cam], [IDENT], dataclasses.replace(prm, alpha=0.0))
    assert fwd0.count[0, p] == 1


@pytest.mark.parametrize("case", GOLDEN["blend"])
def test_blend_mean(case):
    cam = _cam(16, 16, 8.0)
    n = len(case["tau"])
    pts = _axis_points([2.0 + 0.001 * i for i in range(n)], [[t] for t in case["tau"]], cam)
    fwd = O.forward(pts, [cam], [IDENT], S.Params(layers=1, discard=False))
    assert abs(fwd.image[0, 8 * 16 + 8] - case["mean"]) < 1e-7


def test_depth_key_tie_goes_to_lower_index_and_winner_is_min():
    cam = _cam(16, 16, 8.0)
    pts = _axis_points([3.0, 2.0, 2.0, 2.5], [[0.1], [0.2], [0.3], [0.4]], cam)
    keys = O.forward_depth(pts, [cam], [IDENT], S.Params(layers=1, discard=False))[0]
    k = int(keys[8 * 16 + 8])
    assert k & 0xFFFFFFFF == 1 and np.array([k >> 32], dtype=np.uint32).view(F)[0] == F(2.0)


def _random_scene(seed, n=1200, model=S.PINHOLE, discard=True, rho=0.0, layers=3):
    rng = np.random.default_rng(seed)
    w, h = 64, 48
    if model == S.OPENCV8:
        cam = dataclasses.replace(S.opencv_camera(w, h, seed=seed), fx=float(F(40.0)), fy=float(F(40.0)))
        cam = dataclasses.replace(cam, r2_max=S.distortion_r2_max(cam))
    else:
        cam = _cam(w, h, 40.0)
    # two slanted walls at nearby depths + clutter -> many collisions and fuzzy blends
    xy = rng.uniform(-0.9, 0.9, (n, 2))
    z = np.where(rng.random(n) < 0.5, 1.5 + 0.01 * xy[:, 0], 1.51) + rng.normal(0, 0.004, n)
    z[: n // 10] = rng.uniform(-0.5, 3.0, n // 10)
    xyz = np.c_[xy * z[:, None], z].astype(F)
    feat = rng.random((n, 3)).astype(F)
    radius = rng.uniform(0.0, 0.05, n).astype(F)
    pts = _points(xyz, feat, radius, goff=int(rng.integers(0, 1000)))
    prm = S.Params(layers=layers, discard=discard, gamma=1.5, ghost_rate=rho, seed=int(seed) * 7 + 1,
                   view_id_base=int(seed) % 5, background=[0.25, -1.0, 2.0])
    return pts, cam, prm


@pytest.mark.parametrize("seed,model,discard,rho", [
    (10, S.PINHOLE, False, 0.0), (11, S.PINHOLE, True, 0.0), (12, S.PINHOLE, True, 0.3),
    (13, S.OPENCV8, True, 0.25), (14, S.OPENCV8, False, 0.0)])
def test_three_pass_equals_per_pixel_bruteforce(seed, model, discard, rho):
    pts, cam, prm = _random_scene(seed, model=model, discard=discard, rho=rho)
    fwd = O.forward(pts, [cam], [IDENT], prm)
    keys, count, image = BF.forward(pts.pos, pts.radius, pts.feat, cam, IDENT, prm, view=0,
                                    global_offset=int(pts.s.global_offset))
    assert np.array_equal(fwd.keys[0], keys)
    assert np.array_equal(fwd.count[0], count)
    np.testing.assert_allclose(fwd.image[0], image, rtol=0, atol=1e-12)
    assert count.sum() > 100  # the scene is not trivially empty


def test_point_masks_match_bruteforce_hash_and_discard():
    pts, cam, prm = _random_scene(21, discard=True, rho=0.3)
    m = O.point_masks(pts, [cam], [IDENT], prm)[0]
    goff = int(pts.s.global_offset)
    thr = int(np.floor(float(F(prm.ghost_rate)) * 2 ** 24))
    for i in range(pts.n):
        assert bool(m[i] & 0x80) == (BF.h24(prm.seed, 1, 0, goff + i) < thr)
    for i in range(0, 1 << 20, 4099):
        for stream, view in ((1, 0), (2, 3)):
            assert O.h24(prm.seed, stream, view, i) == BF.h24(prm.seed, stream, view, i)


def test_order_invariance_and_count_background_equivalence():
    pts, cam, prm = _random_scene(30, discard=False)
    prm = dataclasses.replace(prm, background=[0.125, 0.5, 0.75])
    fwd = O.forward(pts, [cam], [IDENT], prm)
    perm = np.random.default_rng(0).permutation(pts.n)
    pts2 = O.Points(pts.pos[:, perm], pts.radius[perm], pts.feat[perm], int(pts.s.global_offset))
    fwd2 = O.forward(pts2, [cam], [IDENT], prm)
    # winners are the same points; the index halves of the keys are permuted ids
    assert np.array_equal(fwd.keys[0] >> np.uint64(32), fwd2.keys[0] >> np.uint64(32))
    assert np.array_equal(fwd.count, fwd2.count)
    np.testing.assert_allclose(fwd.image, fwd2.image, atol=1e-12)
    empty = fwd.count[0] == 0
    assert np.array_equal(empty, fwd.keys[0] == np.uint64(O.SENTINEL))
    P = fwd.count.shape[1]
    dims, _ = S.layer_dims(cam.width, cam.height, prm.layers)
    for wl, hl, off in dims:
        for c, b in enumerate(prm.background):
            plane = fwd.image[0, 3 * off + c * wl * hl: 3 * off + (c + 1) * wl * hl]
            assert np.all(plane[empty[off:off + wl * hl]] == b)


def test_monotone_alpha():
    pts, cam, prm = _random_scene(31, discard=False)
    counts = [O.forward(pts, [cam], [IDENT], dataclasses.replace(prm, alpha=a)).count[0]
              for a in (0.0, 0.001, 0.01, 0.05)]
    for a, b in zip(counts, counts[1:]):
        assert np.all(a <= b)
    assert counts[-1].sum() > counts[0].sum()


# --------------------------------------------------------------------------- #
# Eq. 12: stochastic discarding; §4.3 ghost split
# --------------------------------------------------------------------------- #
def _disc_points(n, r_screen, f=100.0, z=1.0):
    # all points on the optical axis at depth z; radius so that r_w * f / z = r_screen
    xyz = np.tile([0.0, 0.0, z], (n, 1))
    return _points(xyz, radius=np.full(n, r_screen * z / f, dtype=F))


@pytest.mark.parametrize("r", [0.1, 0.25, 0.5, 1.0, 2.0])
def test_discard_keep_probability_closed_form(r):
    cam = _cam(64, 64, 100.0)
    n = 100_000
    gamma = 1.5
    prm = S.Params(layers=1, discard=True, gamma=gamma, seed=12345)
    m = O.point_masks(_disc_points(n, r), [cam], [IDENT], prm)[0]
    p = min(1.0, gamma * gamma * r * r)
    freq = float((m & 1).mean())
    sigma = math.sqrt(max(p * (1 - p), 1e-12) / n)
    assert abs(freq - p) <= 3 * sigma + 1e-9, (freq, p)


@pytest.mark.parametrize("case", GOLDEN["discard"])
def test_discard_worked_values(case):
    if "r_screen" in case and "r_world" in case:
        # r_screen = r_world * f / z at layer 0: gamma chosen so that keep <=> r_screen >= threshold
        cam = _cam(64, 64, case["f"])
        ok, Xc, u0, v0, iz = O.project(cam, IDENT, 0.0, 0.0, case["z"])
        assert abs(F(F(case["r_world"]) * F(case["f"])) * iz - case["r_screen"]) < 1e-6
        return
    cam = _cam(64, 64, 100.0)
    n = 50_000
    prm = S.Params(layers=1, discard=True, gamma=case["gamma"], seed=99)
    m = O.point_masks(_disc_points(n, case["r_screen"]), [cam], [IDENT], prm)[0]
    freq = float((m & 1).mean())
    p = case["p_keep"]
    assert abs(freq - p) <= 3 * math.sqrt(max(p * (1 - p), 1e-12) / n) + 1e-9


def test_discard_edge_cases_and_nesting():
    cam = _cam(64, 64, 100.0)
    n = 20_000
    L = 4
    off = O.point_masks(_disc_points(n, 0.01), [cam], [IDENT], S.Params(layers=L, discard=False))[0]
    assert np.all(off == (1 << L) - 1)                        # off -> all kept
    zero = O.point_masks(_disc_points(n, 0.0), [cam], [IDENT], S.Params(layers=L, discard=True))[0]
    assert np.all(zero == 0)                                  # r_w = 0 -> none kept
    big = O.point_masks(_disc_points(n, 100.0), [cam], [IDENT], S.Params(layers=L, discard=True))[0]
    assert np.all(big == (1 << L) - 1)                        # gamma r >= 1 at every layer -> all
    mid = O.point_masks(_disc_points(n, 0.9), [cam], [IDENT], S.Params(layers=L, discard=True))[0]
    for l in range(L - 1):                                    # nested: kept at l+1 => kept at l (R11)
        assert np.all(((mid >> (l + 1)) & 1) <= ((mid >> l) & 1))
    fr = [float(((mid >> l) & 1).mean()) for l in range(L)]
    for l in range(L):                                        # per-layer closed form with r/2^l
        p = min(1.0, (1.5 * 0.9 / 2 ** l) ** 2)
        assert abs(fr[l] - p) <= 3 * math.sqrt(max(p * (1 - p), 1e-12) / n) + 1e-9


def test_ghost_split_fraction_and_invisibility():
    n = 100_000
    rho = 0.25
    pts = _points(np.tile([0.0, 0.0, -1.0], (n, 1)))
    cam = _cam(8, 8, 1.0)
    m = O.point_masks(pts, [cam], [IDENT], S.Params(layers=1, discard=False, ghost_rate=rho, seed=7))[0]
    frac = float(((m & 0x80) != 0).mean())
    assert abs(frac - rho) <= 3 * math.sqrt(rho * (1 - rho) / n)
    m0 = O.point_masks(pts, [cam], [IDENT], S.Params(layers=1, discard=False, ghost_rate=0.0, seed=7))[0]
    assert not np.any(m0 & 0x80)
    # ghosts never alter the forward: same image as the cloud with the ghosts moved behind the camera
    pts2, cam2, prm = _random_scene(40, discard=True, rho=0.3)
    fwd = O.forward(pts2, [cam2], [IDENT], prm)
    g = (O.point_masks(pts2, [cam2], [IDENT], prm)[0] & 0x80) != 0
    pos = pts2.pos.copy()
    pos[2, g] = -1.0
    pts3 = O.Points(pos, pts2.radius, pts2.feat, int(pts2.s.global_offset))
    fwd3 = O.forward(pts3, [cam2], [IDENT], dataclasses.replace(prm, ghost_rate=0.0))
    assert g.sum() > 100
    assert np.array_equal(fwd.keys, fwd3.keys) and np.array_equal(fwd.image, fwd3.image)


# --------------------------------------------------------------------------- #
# NEXT-3: normal culling, Eq. 5 with reading R32
# --------------------------------------------------------------------------- #
def _with_normals(pts, normal):
    return O.Points(pts.pos, pts.radius, pts.feat, int(pts.s.global_offset), normal=normal)


def test_normal_culling_closed_form():
    """A point on the optical axis at z = 2 (Xc = (0,0,2)) with normal (0,0,-1) (facing the camera):
    (R n).Xc = -2 < 0 -> culled by Eq. 5 as printed (+1), kept by the flipped test (-1); (0,0,+1) the reverse."""
    cam = _cam(16, 16, 8.0)
    for nz, keep_printed in ((-1.0, False), (1.0, True)):
        pts = _with_normals(_points(np.array([[0.0, 0.0, 2.0]], F), np.ones((1, 1), F), None),
                            np.array([[0.0], [0.0], [nz]], F))
        for mode, kept in ((0, True), (1, keep_printed), (-1, not keep_printed)):
            m = O.point_masks(pts, [cam], [IDENT], S.Params(layers=2, discard=False, normal_culling=mode))[0]
            assert bool(m[0] & 1) == kept, (nz, mode)


@pytest.mark.parametrize("seed,model,mode", [(30, S.PINHOLE, 1), (31, S.PINHOLE, -1), (32, S.OPENCV8, -1)])
def test_normal_culling_equals_bruteforce_and_removal(seed, model, mode):
    pts, cam, prm = _random_scene(seed, model=model, discard=True, rho=0.2)
    rng = np.random.default_rng(seed)
    nrm = rng.normal(size=(3, pts.n)).astype(F)
    nrm /= np.linalg.norm(nrm, axis=0, keepdims=True)
    pts = _with_normals(pts, nrm)
    prm = dataclasses.replace(prm, normal_culling=mode)
    fwd = O.forward(pts, [cam], [IDENT], prm)
    keys, count, image = BF.forward(pts.pos, pts.radius, pts.feat, cam, IDENT, prm, view=0,
                                    global_offset=int(pts.s.global_offset), normal=nrm)
    assert np.array_equal(fwd.keys[0], keys) and np.array_equal(fwd.count[0], count)
    np.testing.assert_allclose(fwd.image[0], image, rtol=0, atol=1e-12)
    # culled points take no part: same result as moving them behind the camera
    culled = [i for i in range(pts.n)
              if (r := BF.project(cam, IDENT, *pts.pos[:, i], F(0.0))) is not None
              and not BF.normal_kept(IDENT, nrm[:, i], r[0], r[1], r[2], mode)]
    assert len(culled) > 100
    pos2 = pts.pos.copy()
    pos2[2, culled] = -1.0
    off = O.forward(O.Points(pos2, pts.radius, pts.feat, int(pts.s.global_offset)), [cam], [IDENT],
                    dataclasses.replace(prm, normal_culling=0))
    assert np.array_equal(fwd.keys, off.keys) and np.array_equal(fwd.count, off.count)
