"""Pins for the equidistant fisheye camera with distance depth (NEXT-3; "If the camera model does not
provide a valid z-value, we instead use the distance", §6.3 fisheye cameras; reading R35) -- CPU only."""
import dataclasses
import math

import numpy as np
import pytest

from oracle import bruteforce as BF
from oracle import oracle as O
from paper_2110_06635_b200 import scene as S

F = np.float32
IDENT = S.Pose(np.eye(3, dtype=F), np.zeros(3, dtype=F))


def test_atan2p_accuracy_and_quadrants():
    rng = np.random.default_rng(0)
    for _ in range(20000):
        y, x = F(abs(rng.normal())), F(rng.normal())
        b = BF.atan2p(y, x)
        assert abs(float(b) - math.atan2(float(y), float(x))) < 4e-7
    assert BF.atan2p(F(0.0), F(1.0)) == 0.0 and BF.atan2p(F(1.0), F(0.0)) == F(1.57079632679490)
    assert BF.atan2p(F(0.0), F(-1.0)) == F(3.14159265358979)


def test_fisheye_closed_forms():
    cam = S.Camera(64, 64, S.FISHEYE, 20.0, 20.0, 32.0, 32.0, r2_max=float(F(math.pi * 0.75)))
    ok, Xc, u0, v0, iz = O.project(cam, IDENT, 0.0, 0.0, 2.0)        # on axis: principal point, depth 2
    assert ok and (u0, v0) == (32.0, 32.0) and iz == F(0.5)
    ok, _, u0, v0, iz = O.project(cam, IDENT, 1.0, 0.0, 1.0)         # 45 degrees: r_d = f pi / 4
    assert ok and u0 == pytest.approx(32.0 + 20.0 * math.pi / 4, abs=2e-5) and v0 == 32.0
    assert iz == pytest.approx(1 / math.sqrt(2), rel=1e-6)
    ok, _, u0, _, _ = O.project(cam, IDENT, 1.0, 0.0, -1.0)          # 135 degrees: behind the image plane
    assert ok and u0 == pytest.approx(32.0 + 20.0 * 3 * math.pi / 4, abs=5e-5)
    ok, *_ = O.project(cam, IDENT, 0.1, 0.0, -1.0)                    # ~174 degrees > theta_max: culled
    assert not ok


def test_fisheye_projection_matches_bruteforce_bitwise():
    rng = np.random.default_rng(1)
    cam = S.fisheye_camera(96, 80, 200.0)
    poses = S.room_poses(2, S.make_room(10.0))
    for pose in poses:
        for _ in range(2000):
            xyz = [F(v) for v in rng.uniform(-5, 5, 3)]
            a = O.project(cam, pose, *xyz)
            b = BF.project(cam, pose, *xyz, F(0.0))
            assert a[0] == (b is not None)
            if b is not None:
                assert (a[2], a[3], a[4]) == (float(b[3]), float(b[4]), float(b[5]))


def test_fisheye_jacobian_and_intrinsics_match_finite_differences():
    cam = S.fisheye_camera(640, 480, 190.0)
    rng = np.random.default_rng(2)
    for _ in range(30):
        X = rng.normal(size=3).astype(F)
        if X[2] < -0.5 * np.linalg.norm(X):
            X[2] = -X[2]
        J = O.jacobian(cam, X)
        for k in range(3):
            e = np.zeros(3); e[k] = 1e-6
            d = (O.project_f64(cam, X.astype(np.float64) + e) - O.project_f64(cam, X.astype(np.float64) - e)) / 2e-6
            np.testing.assert_allclose(J[:, k], d, rtol=1e-5, atol=1e-5)
        Jt = O.intrinsics_jacobian(cam, X)
        assert not Jt[:, 4:].any()
        for j, name in enumerate(["fx", "fy", "cx", "cy"]):
            cp = dataclasses.replace(cam, **{name: getattr(cam, name) + 0.0625})
            cm = dataclasses.replace(cam, **{name: getattr(cam, name) - 0.0625})
            d = (O.project_f64(cp, X.astype(np.float64)) - O.project_f64(cm, X.astype(np.float64))) / 0.125
            np.testing.assert_allclose(Jt[:, j], d, rtol=1e-9, atol=1e-9)


@pytest.mark.parametrize("seed,fov,rho", [(40, 120.0, 0.0), (41, 200.0, 0.3)])
def test_fisheye_three_pass_equals_bruteforce(seed, fov, rho):
    rng = np.random.default_rng(seed)
    n = 1500
    d = rng.normal(size=(3, n))
    d /= np.linalg.norm(d, axis=0)
    pos = (d * rng.uniform(1.0, 1.02, n)).astype(F)   # a thin shell around the camera: many collisions
    pts = O.Points(pos, rng.uniform(0.0, 0.05, n).astype(F), rng.random((n, 3)).astype(F), 17)
    cam = S.fisheye_camera(64, 48, fov)
    prm = S.Params(layers=3, discard=True, ghost_rate=rho, seed=seed, background=[0.125, 0.25, -0.5])
    fwd = O.forward(pts, [cam], [IDENT], prm)
    keys, count, image = BF.forward(pts.pos, pts.radius, pts.feat, cam, IDENT, prm, view=0, global_offset=17)
    assert np.array_equal(fwd.keys[0], keys) and np.array_equal(fwd.count[0], count)
    np.testing.assert_allclose(fwd.image[0], image, rtol=0, atol=1e-12)
    assert count.sum() > 100
    if fov > 180:  # points behind the image plane are rendered, their key depth is the distance
        assert any(O.project(cam, IDENT, *pos[:, i])[1][2] < 0 and fwd.count[0].sum() > 0 for i in range(n)
                   if O.project(cam, IDENT, *pos[:, i])[0])
