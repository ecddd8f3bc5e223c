"""The OpenCV8 candidate window (adop_camera_window, host code of the library; no GPU): every point of the
camera's valid disk whose distorted pixel (R6, evaluated here independently in numpy fp64) lies in the
all-layer window must lie inside the returned box -- the depth and backward sweeps cull points outside it
before the distortion model, so a point the box misses would be a lost render-set point.  The box should
also be tight (much smaller than the valid cone) for the configs' cameras."""
import math

import numpy as np
import pytest

from paper_2110_06635_b200 import adop as A
from paper_2110_06635_b200 import scene as S


def _distort(cam, xn, yn):
    k, p = cam.k, cam.p
    r2 = xn * xn + yn * yn
    rad = (1 + k[0] * r2 + k[1] * r2 ** 2 + k[2] * r2 ** 3) / (1 + k[3] * r2 + k[4] * r2 ** 2 + k[5] * r2 ** 3)
    xd = xn * rad + 2 * p[0] * xn * yn + p[1] * (r2 + 2 * xn * xn)
    yd = yn * rad + p[0] * (r2 + 2 * yn * yn) + 2 * p[1] * xn * yn
    return cam.fx * xd + cam.cx, cam.fy * yd + cam.cy


def _cameras():
    cams = [S.opencv_camera(1024, 1024, seed=S.SEED_CAMERAS + v) for v in range(16)]   # configs[4]
    cams += [S.opencv_camera(1920, 1080, seed=S.SEED_CAMERAS)]                         # configs[2]
    cams += [S.opencv_camera(320, 240, seed=s) for s in range(100, 140)]
    return cams


@pytest.mark.parametrize("layers", [1, 5])
def test_window_contains_every_point_landing_in_the_image(layers):
    rng = np.random.default_rng(7)
    lmax = 2.0 ** (layers - 1)
    tight = []
    for cam in _cameras():
        win = A.camera_window(cam, layers)
        assert win is not None, cam
        xlo, xhi, ylo, yhi = win
        R = math.sqrt(cam.r2_max)
        # dense random samples of the valid disk, plus its boundary circle
        n = 400_000
        rr = R * np.sqrt(rng.random(n))
        th = rng.random(n) * 2 * np.pi
        xn = np.concatenate([rr * np.cos(th), R * np.cos(np.linspace(0, 2 * np.pi, 20_000))])
        yn = np.concatenate([rr * np.sin(th), R * np.sin(np.linspace(0, 2 * np.pi, 20_000))])
        u, v = _distort(cam, xn, yn)
        inimg = (u > -lmax - 2) & (u < cam.width + lmax + 2) & (v > -lmax - 2) & (v < cam.height + lmax + 2)
        assert inimg.any()
        assert xn[inimg].min() >= xlo and xn[inimg].max() <= xhi, (cam, win, xn[inimg].min(), xn[inimg].max())
        assert yn[inimg].min() >= ylo and yn[inimg].max() <= yhi, (cam, win, yn[inimg].min(), yn[inimg].max())
        # tight: the box exceeds the sampled extent by little
        tight.append(max(xn[inimg].min() - xlo, xhi - xn[inimg].max(), yn[inimg].min() - ylo, yhi - yn[inimg].max()))
    assert np.median(tight) < 0.02


def test_no_window_for_pinhole_and_fisheye():
    assert A.camera_window(S.pinhole(640, 480), 5) is None
    assert A.camera_window(S.fisheye_camera(640, 480, 180.0), 5) is None
