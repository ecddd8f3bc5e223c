"""Tiny, independent per-pixel brute-force checker for the C oracle.

TEST INFRASTRUCTURE ONLY.  It does not call adop_oracle.c: it recomputes the
per-point projection in numpy float32 (per-op IEEE, same pinned operation
order R1/R2/R6), the rounding rule R3, the discard rule R10 and the hash of
R11/R13, and then evaluates Eqs. 4-7 literally PER PIXEL: for every pixel p
of every layer it collects the render-set points that land on p, takes the
minimum key, keeps those within the fuzzy threshold and averages their
descriptors.  That is the plain definition the oracle's three-pass structure
(§4.5) must reproduce.  Sizes: N <= a few thousand, images <=
128x128.
"""
from __future__ import annotations

import numpy as np

F = np.float32
SENTINEL = 0x7FFFFFFFFFFFFFFF


def _mix32(x: int) -> int:
    x &= 0xFFFFFFFF
    x ^= x >> 16
    x = (x * 0x7FEB352D) & 0xFFFFFFFF
    x ^= x >> 15
    x = (x * 0x846CA68B) & 0xFFFFFFFF
    x ^= x >> 16
    return x


def h24(seed: int, stream: int, view: int, i: int) -> int:
    s = _mix32((seed & 0xFFFFFFFF) + ((0x9E3779B9 * (stream + 1)) & 0xFFFFFFFF))
    s = _mix32(s ^ (seed >> 32))
    salt = _mix32(s + ((0x85EBCA6B * (view + 1)) & 0xFFFFFFFF))
    return _mix32(i ^ salt) >> 8


def round_half_away(x: F) -> F:
    t = np.trunc(x)
    d = x - t  # exact
    if abs(d) >= F(0.5):
        t = t + np.copysign(F(1.0), x)
    return F(t)


ATAN_C = [F(v) for v in (-0.0015244261594489217, 0.009669913910329342, -0.028764614835381508, 0.05541255697607994,
                          -0.08245089650154114, 0.10893233865499496, -0.14251546561717987, 0.1999710500240326,
                          -0.33333227038383484, 1.0)]


def atan2p(y: F, x: F) -> F:
    """R35: angle in [0, pi] of (x, y), y >= 0, from the fixed degree-9 polynomial (fp32, one rounding per op)."""
    def a01(t):
        u, p = F(t * t), ATAN_C[0]
        for c in ATAN_C[1:]:
            p = F(F(p * u) + c)
        return F(t * p)
    ax = F(abs(x))
    if y <= ax:
        a = a01(F(y / ax)) if ax > 0 else F(0.0)
    else:
        a = F(F(1.57079632679490) - a01(F(ax / y)))
    return a if x >= 0 else F(F(3.14159265358979) - a)


def project(cam, pose, x: F, y: F, z: F, z_near: F):
    """-> (X, Y, Z, u0, v0, 1/depth, depth) or None (pinned fp32)."""
    R = np.asarray(pose.R, dtype=F).reshape(9)
    t = np.asarray(pose.t, dtype=F)
    X = F(F(F(R[0] * x) + F(R[1] * y)) + F(R[2] * z)) + t[0]
    Y = F(F(F(R[3] * x) + F(R[4] * y)) + F(R[5] * z)) + t[1]
    Z = F(F(F(R[6] * x) + F(R[7] * y)) + F(R[8] * z)) + t[2]
    if cam.model == 2:  # equidistant fisheye, distance depth (R35)
        rho2 = F(F(X * X) + F(Y * Y))
        d = F(np.sqrt(F(rho2 + F(Z * Z))))
        if not (d > z_near and d <= np.finfo(F).max):
            return None
        rho = F(np.sqrt(rho2))
        th = atan2p(rho, Z)
        if not (th <= F(cam.r2_max)):
            return None
        s = F(th / rho) if rho > 0 else F(0.0)
        u0 = F(F(F(cam.fx) * F(X * s)) + F(cam.cx))
        v0 = F(F(F(cam.fy) * F(Y * s)) + F(cam.cy))
        return X, Y, Z, u0, v0, F(F(1.0) / d), d
    if not (Z > z_near and Z <= np.finfo(F).max):
        return None
    iz = F(F(1.0) / Z)
    xn, yn = F(X * iz), F(Y * iz)
    xd, yd = xn, yn
    if cam.model == 1:
        k = [F(v) for v in cam.k]
        p = [F(v) for v in cam.p]
        xx, yy, xy = F(xn * xn), F(yn * yn), F(xn * yn)
        r2 = F(xx + yy)
        if not (r2 <= F(cam.r2_max)):
            return None
        r4 = F(r2 * r2)
        r6 = F(r4 * r2)
        num = F(F(F(F(1.0) + F(k[0] * r2)) + F(k[1] * r4)) + F(k[2] * r6))
        den = F(F(F(F(1.0) + F(k[3] * r2)) + F(k[4] * r4)) + F(k[5] * r6))
        if not (den > 0):
            return None
        rad = F(num / den)
        a1 = F(F(2.0) * xy)
        a2 = F(r2 + F(F(2.0) * xx))
        a3 = F(r2 + F(F(2.0) * yy))
        xd = F(F(F(xn * rad) + F(p[0] * a1)) + F(p[1] * a2))
        yd = F(F(F(yn * rad) + F(p[0] * a3)) + F(p[1] * a1))
    u0 = F(F(F(cam.fx) * xd) + F(cam.cx))
    v0 = F(F(F(cam.fy) * yd) + F(cam.cy))
    return X, Y, Z, u0, v0, iz, Z


def forward(pos, radius, feat, cam, pose, params, view: int = 0, global_offset: int = 0, normal=None):
    """Per-pixel definition of Eqs. 2-7 for one view -> (keys, count, image[C*P])."""
    with np.errstate(all="ignore"):
        return _forward(pos, radius, feat, cam, pose, params, view, global_offset, normal)


def normal_kept(pose, n, X: F, Y: F, Z: F, mode: int) -> bool:
    """Eq. 5 with reading R32: sign of (R n) . Xc, pinned fp32 order; mode +1 as printed, -1 flipped."""
    R = np.asarray(pose.R, dtype=F).reshape(9)
    nx, ny, nz = F(n[0]), F(n[1]), F(n[2])
    ncx = F(F(F(R[0] * nx) + F(R[1] * ny)) + F(R[2] * nz))
    ncy = F(F(F(R[3] * nx) + F(R[4] * ny)) + F(R[5] * nz))
    ncz = F(F(F(R[6] * nx) + F(R[7] * ny)) + F(R[8] * nz))
    dot = F(F(F(ncx * X) + F(ncy * Y)) + F(ncz * Z))
    return bool(dot > 0) if mode > 0 else bool(dot < 0)


def _forward(pos, radius, feat, cam, pose, params, view, global_offset, normal):
    L = params.layers
    n = pos.shape[1]
    C = feat.shape[1]
    dims = []
    off = 0
    for l in range(L):
        wl = -(-cam.width // (1 << l))
        hl = -(-cam.height // (1 << l))
        dims.append((wl, hl, off))
        off += wl * hl
    P = off
    ghost_thr = int(np.floor(float(F(params.ghost_rate)) * 16777216.0))
    onepa = F(F(1.0) + F(params.alpha))
    # per point: list of (layer, local pixel, z, key)
    hits = {}  # (l, local) -> list of (key, z, i)
    for i in range(n):
        gi = global_offset + i
        if ghost_thr and h24(params.seed, 1, 0, gi) < ghost_thr:
            continue
        pr = project(cam, pose, F(pos[0, i]), F(pos[1, i]), F(pos[2, i]), F(params.z_near))
        if pr is None:
            continue
        X, Y, Z, u0, v0, iz, D = pr
        mode = int(getattr(params, "normal_culling", 0))
        if mode and normal is not None and not normal_kept(pose, normal[:, i], X, Y, Z, mode):
            continue
        nkeep = L
        if params.discard:
            feff = F(F(F(cam.fx) + F(cam.fy)) * F(0.5))
            rs0 = F(F(F(radius[i]) * feff) * iz)
            om = F(F(16777216 - h24(params.seed, 2, params.view_id_base + view, gi)) * F(1.0 / 16777216.0))
            nkeep = 0
            for l in range(L):
                a = F(F(params.gamma) * F(rs0 * F(2.0 ** -l)))
                if not (F(a * a) > om):
                    break
                nkeep += 1
        zb = int(np.array([D], dtype=F).view(np.uint32)[0])
        key = (zb << 32) | (gi & 0xFFFFFFFF)
        for l in range(nkeep):
            wl, hl, o = dims[l]
            s = F(2.0 ** -l)
            ru, rv = round_half_away(F(u0 * s)), round_half_away(F(v0 * s))
            if ru >= 0 and ru < F(wl) and rv >= 0 and rv < F(hl):
                hits.setdefault((l, int(rv) * wl + int(ru)), []).append((key, D, i))
    keys = np.full(P, SENTINEL, dtype=np.uint64)
    count = np.zeros(P, dtype=np.float64)
    image = np.zeros(C * P, dtype=np.float64)
    bg = np.zeros(C) if params.background is None else np.asarray(params.background, dtype=np.float64)
    for l in range(L):
        wl, hl, o = dims[l]
        hw = wl * hl
        for j in range(hw):  # every pixel: Eq. 7 by definition
            lst = hits.get((l, j), [])
            if lst:
                kmin = min(k for k, _, _ in lst)
                m = np.array([kmin >> 32], dtype=np.uint32).view(F)[0]
                lam = [i for k, z, i in lst if z <= F(onepa * m)]
                keys[o + j] = kmin
                count[o + j] = len(lam)
                for c in range(C):
                    image[C * o + c * hw + j] = sum(float(feat[i, c]) for i in lam) / len(lam)
            else:
                for c in range(C):
                    image[C * o + c * hw + j] = bg[c]
    return keys, count, image
