"""ctypes wrapper around oracle/adop_oracle.c (the CPU oracle).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs; never by the product package
(paper_2110_06635_b200).  It declares its own ctypes structs from
adop_oracle.c; nothing here is shared with the CUDA path's binding.
"""
from __future__ import annotations

import ctypes as C
import math
import os
import subprocess
from typing import List, Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "adop_oracle.c")
LIB = os.path.join(HERE, "liborc.so")
CFLAGS = ["-O2", "-std=c99", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC", "-shared"]

SENTINEL = 0x7FFFFFFFFFFFFFFF
STREAM_GHOST, STREAM_DISCARD = 1, 2


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        tmp = LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, SRC, "-lm"])
        os.replace(tmp, LIB)
    return LIB


class _Camera(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("model", C.c_int32),
                ("fx", C.c_float), ("fy", C.c_float), ("cx", C.c_float), ("cy", C.c_float),
                ("k", C.c_float * 6), ("p", C.c_float * 2), ("r2_max", C.c_float)]


class _Pose(C.Structure):
    _fields_ = [("R", C.c_float * 9), ("t", C.c_float * 3)]


class _Params(C.Structure):
    _fields_ = [("layers", C.c_int32), ("alpha", C.c_float), ("discard", C.c_int32), ("gamma", C.c_float),
                ("ghost_rate", C.c_float), ("z_near", C.c_float), ("seed", C.c_uint64),
                ("view_id_base", C.c_int32), ("log_descriptors", C.c_int32), ("spatial_rendered", C.c_int32),
                ("normal_culling", C.c_int32)]


class _Env(C.Structure):
    _fields_ = [("data", C.c_void_p), ("width", C.c_int32), ("height", C.c_int32)]


class _Points(C.Structure):
    _fields_ = [("n", C.c_int64), ("global_offset", C.c_int64), ("pos_stride", C.c_int64),
                ("pos", C.c_void_p), ("radius", C.c_void_p), ("radius_uniform", C.c_float),
                ("feat", C.c_void_p), ("channels", C.c_int32), ("normal", C.c_void_p)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        P = C.POINTER
        _lib.orc_pyramid_pixels.restype = C.c_int64
        _lib.orc_pyramid_pixels.argtypes = [C.c_int32, C.c_int32, C.c_int32]
        _lib.orc_h24.restype = C.c_uint32
        _lib.orc_h24.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32]
        _lib.orc_is_ghost.restype = C.c_int
        _lib.orc_is_ghost.argtypes = [P(_Params), C.c_uint32]
        _lib.orc_project.restype = C.c_int
        _lib.orc_project.argtypes = [P(_Camera), P(_Pose), C.c_float, C.c_float, C.c_float, C.c_float,
                                     C.c_void_p]
        _lib.orc_point_masks.argtypes = [P(_Points), C.c_int32, P(_Camera), P(_Pose), P(_Params), C.c_void_p]
        _lib.orc_forward_depth.argtypes = [P(_Points), C.c_int32, P(_Camera), P(_Pose), P(_Params), C.c_void_p]
        _lib.orc_forward_blend.argtypes = [P(_Points), C.c_int32, P(_Camera), P(_Pose), P(_Params), C.c_void_p,
                                           C.c_void_p, C.c_void_p]
        _lib.orc_forward_resolve.argtypes = [C.c_int32, P(_Camera), P(_Pose), P(_Params), C.c_int32, C.c_void_p,
                                             C.c_void_p, C.c_void_p, P(_Env), C.c_void_p]
        _lib.orc_unproject.argtypes = [P(_Camera), C.c_double, C.c_double, P(C.c_double), P(C.c_double)]
        _lib.orc_env_taps.argtypes = [P(_Env), C.c_void_p, C.c_void_p, C.c_void_p]
        _lib.orc_env_dir.argtypes = [P(_Camera), P(_Pose), C.c_int, C.c_int64, C.c_int64, C.c_void_p]
        _lib.orc_induced_change.restype = C.c_int
        _lib.orc_induced_change.argtypes = [C.c_int32, C.c_void_p, C.c_float, C.c_float, C.c_double,
                                            C.c_uint64, C.c_void_p, C.c_void_p]
        _lib.orc_jacobian.argtypes = [P(_Camera), C.c_void_p, C.c_void_p]
        _lib.orc_project_f64.argtypes = [P(_Camera), C.c_void_p, C.c_void_p]
        _lib.orc_intrinsics_jacobian.argtypes = [P(_Camera), C.c_void_p, C.c_void_p]
        _lib.orc_set_threads.restype = C.c_int
        _lib.orc_set_threads.argtypes = [C.c_int]
        _lib.orc_get_threads.restype = C.c_int
        _lib.orc_backward.argtypes = [P(_Points), C.c_int32, P(_Camera), P(_Pose), P(_Params), P(_Env),
                                      C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                      C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                      C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    return _lib


# --------------------------------------------------------------------------- #
# marshalling helpers
# --------------------------------------------------------------------------- #
def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data


def camera_struct(cam) -> _Camera:
    s = _Camera()
    s.width, s.height, s.model = int(cam.width), int(cam.height), int(cam.model)
    s.fx, s.fy, s.cx, s.cy = cam.fx, cam.fy, cam.cx, cam.cy
    for i in range(6):
        s.k[i] = cam.k[i]
    for i in range(2):
        s.p[i] = cam.p[i]
    s.r2_max = cam.r2_max
    return s


def pose_struct(pose) -> _Pose:
    s = _Pose()
    R = np.asarray(pose.R, dtype=np.float32).reshape(9)
    t = np.asarray(pose.t, dtype=np.float32).reshape(3)
    for i in range(9):
        s.R[i] = float(R[i])
    for i in range(3):
        s.t[i] = float(t[i])
    return s


def params_struct(p) -> _Params:
    s = _Params()
    s.layers, s.alpha, s.discard, s.gamma = int(p.layers), p.alpha, int(bool(p.discard)), p.gamma
    s.ghost_rate, s.z_near, s.seed, s.view_id_base = p.ghost_rate, p.z_near, int(p.seed), int(p.view_id_base)
    s.log_descriptors = int(bool(getattr(p, "log_descriptors", False)))
    s.spatial_rendered = int(bool(getattr(p, "spatial_rendered", False)))
    s.normal_culling = int(getattr(p, "normal_culling", 0))
    return s


class Env:
    """Host copy of params.env_map ([H][W][C] float32) as the oracle's orc_env (NULL data if none)."""

    def __init__(self, params):
        e = getattr(params, "env_map", None)
        self.arr = None if e is None else np.ascontiguousarray(
            e.cpu().numpy() if hasattr(e, "cpu") else e, dtype=np.float32)
        self.s = _Env()
        if self.arr is not None:
            self.s.data, self.s.height, self.s.width = self.arr.ctypes.data, self.arr.shape[0], self.arr.shape[1]


class Points:
    """Host-side point shard: keeps the numpy arrays alive while the struct points at them."""

    def __init__(self, pos: np.ndarray, radius: Optional[np.ndarray], feat: np.ndarray,
                 global_offset: int = 0, radius_uniform: float = 0.0, normal: Optional[np.ndarray] = None):
        self.pos = np.ascontiguousarray(pos, dtype=np.float32)
        self.normal = None if normal is None else np.ascontiguousarray(normal, dtype=np.float32)
        assert self.normal is None or self.normal.shape == self.pos.shape
        self.radius = None if radius is None else np.ascontiguousarray(radius, dtype=np.float32)
        self.feat = np.ascontiguousarray(feat, dtype=np.float32)
        self.n = self.pos.shape[1]
        self.C = self.feat.shape[1]
        s = _Points()
        s.n, s.global_offset, s.pos_stride = self.n, int(global_offset), self.n
        s.pos, s.radius, s.radius_uniform = _ptr(self.pos), _ptr(self.radius), radius_uniform
        s.feat, s.channels = _ptr(self.feat), self.C
        s.normal = _ptr(self.normal)
        self.s = s

    @staticmethod
    def from_cloud(cloud, global_offset: int = 0) -> "Points":
        nrm = getattr(cloud, "normal", None)
        return Points(cloud.pos.cpu().numpy(), cloud.radius.cpu().numpy(), cloud.feat.cpu().numpy(), global_offset,
                      normal=None if nrm is None else nrm.cpu().numpy())


def _arrays(cams, poses):
    V = len(cams)
    ca = (_Camera * V)(*[camera_struct(c) for c in cams])
    pa = (_Pose * V)(*[pose_struct(p) for p in poses])
    return ca, pa


def set_threads(n: int) -> int:
    """OpenMP threads of the oracle's parallel loops (n <= 0: all processors); returns the count in effect.
    Results do not depend on it (per-point map in parallel, reductions serial in point order)."""
    return int(lib().orc_set_threads(int(n)))


def get_threads() -> int:
    return int(lib().orc_get_threads())


def pyramid_pixels(w: int, h: int, layers: int) -> int:
    return int(lib().orc_pyramid_pixels(w, h, layers))


def h24(seed: int, stream: int, view: int, i: int) -> int:
    return int(lib().orc_h24(seed, stream, view, i))


def is_ghost(params, gi: int) -> bool:
    ps = params_struct(params)
    return bool(lib().orc_is_ghost(C.byref(ps), gi))


def project(cam, pose, x, y, z, z_near=0.0):
    """-> (valid, Xc[3], u0, v0, 1/depth) for one point, pinned fp32 (Eq. 2, R1/R2/R6/R35)."""
    out = np.zeros(7, dtype=np.float32)
    cs, ps = camera_struct(cam), pose_struct(pose)
    ok = lib().orc_project(C.byref(cs), C.byref(ps), x, y, z, z_near, out.ctypes.data)
    return bool(ok), out[:3].copy(), float(out[3]), float(out[4]), float(out[5])


def point_masks(pts: Points, cams, poses, params) -> np.ndarray:
    V = len(cams)
    ca, pa = _arrays(cams, poses)
    ps = params_struct(params)
    out = np.zeros((V, pts.n), dtype=np.uint8)
    lib().orc_point_masks(C.byref(pts.s), V, ca, pa, C.byref(ps), out.ctypes.data)
    return out


class Forward:
    def __init__(self, keys, accum, count, image):
        self.keys, self.accum, self.count, self.image = keys, accum, count, image


def forward_depth(pts: Points, cams, poses, params) -> np.ndarray:
    V = len(cams)
    P = pyramid_pixels(cams[0].width, cams[0].height, params.layers)
    ca, pa = _arrays(cams, poses)
    ps = params_struct(params)
    keys = np.empty((V, P), dtype=np.uint64)
    lib().orc_forward_depth(C.byref(pts.s), V, ca, pa, C.byref(ps), keys.ctypes.data)
    return keys


def forward_blend(pts: Points, cams, poses, params, keys: np.ndarray):
    V = len(cams)
    P = keys.shape[1]
    ca, pa = _arrays(cams, poses)
    ps = params_struct(params)
    accum = np.empty((V, P, pts.C), dtype=np.float64)
    count = np.empty((V, P), dtype=np.float64)
    keys = np.ascontiguousarray(keys, dtype=np.uint64)
    lib().orc_forward_blend(C.byref(pts.s), V, ca, pa, C.byref(ps), keys.ctypes.data, accum.ctypes.data,
                            count.ctypes.data)
    return accum, count


def forward_resolve(cams, params, channels: int, accum: np.ndarray, count: np.ndarray, bg=None,
                    poses=None) -> np.ndarray:
    V, P = count.shape
    if poses is None:
        poses = [None] * V
    ca = (_Camera * V)(*[camera_struct(c) for c in cams])
    pa = (_Pose * V)(*[pose_struct(p) if p is not None else _Pose() for p in poses])
    ps = params_struct(params)
    env = Env(params)
    assert env.arr is None or all(p is not None for p in poses), "an environment map needs the poses"
    image = np.empty((V, channels * P), dtype=np.float64)
    bga = None if bg is None else np.ascontiguousarray(bg, dtype=np.float32)
    accum = np.ascontiguousarray(accum, dtype=np.float64)
    count = np.ascontiguousarray(count, dtype=np.float64)
    lib().orc_forward_resolve(V, ca, pa, C.byref(ps), channels, accum.ctypes.data, count.ctypes.data, _ptr(bga),
                              C.byref(env.s), image.ctypes.data)
    return image


def unproject(cam, u0: float, v0: float):
    """C^{-1} of R29: layer-0 continuous pixel -> normalized camera coordinates (xn, yn)."""
    x, y = C.c_double(), C.c_double()
    cs = camera_struct(cam)
    lib().orc_unproject(C.byref(cs), float(u0), float(v0), C.byref(x), C.byref(y))
    return x.value, y.value


def env_dir(cam, pose, l: int, u: int, v: int) -> np.ndarray:
    d = np.zeros(3)
    cs, ps = camera_struct(cam), pose_struct(pose)
    lib().orc_env_dir(C.byref(cs), C.byref(ps), l, u, v, d.ctypes.data)
    return d


def env_taps(env_map, d):
    """(texel indices row * W + col, bilinear weights) of direction d in env_map [H][W][C] (R29)."""
    e = Env(type("P", (), {"env_map": env_map})())
    dd = np.ascontiguousarray(d, dtype=np.float64)
    idx, w = np.zeros(4, dtype=np.int64), np.zeros(4)
    lib().orc_env_taps(C.byref(e.s), dd.ctypes.data, idx.ctypes.data, w.ctypes.data)
    return idx, w


def forward(pts: Points, cams, poses, params) -> Forward:
    """Eq. 1 for every view and layer: keys [V][P] u64, accum [V][P][C], count [V][P], image [V][C*P]."""
    keys = forward_depth(pts, cams, poses, params)
    accum, count = forward_blend(pts, cams, poses, params, keys)
    image = forward_resolve(cams, params, pts.C, accum, count, params.background, poses)
    return Forward(keys, accum, count, image)


def induced_change(tau, z, alpha, n_q, key_q, I_q):
    tau = np.ascontiguousarray(tau, dtype=np.float32)
    I_q = np.ascontiguousarray(I_q, dtype=np.float64)
    out = np.zeros(len(tau), dtype=np.float64)
    kase = lib().orc_induced_change(len(tau), tau.ctypes.data, z, alpha, float(n_q), int(key_q),
                                    I_q.ctypes.data, out.ctypes.data)
    return int(kase), out


def jacobian(cam, Xc) -> np.ndarray:
    X = np.ascontiguousarray(Xc, dtype=np.float32)
    J = np.zeros(6, dtype=np.float64)
    cs = camera_struct(cam)
    lib().orc_jacobian(C.byref(cs), X.ctypes.data, J.ctypes.data)
    return J.reshape(2, 3)


def project_f64(cam, Xc) -> np.ndarray:
    X = np.ascontiguousarray(Xc, dtype=np.float64)
    uv = np.zeros(2, dtype=np.float64)
    cs = camera_struct(cam)
    lib().orc_project_f64(C.byref(cs), X.ctypes.data, uv.ctypes.data)
    return uv


def intrinsics_jacobian(cam, Xc) -> np.ndarray:
    """d(u0, v0)/d(fx, fy, cx, cy, k1..k6, p1, p2) at camera point Xc (NEXT-1), shape (2, 12)."""
    X = np.ascontiguousarray(Xc, dtype=np.float32)
    J = np.zeros(24, dtype=np.float64)
    cs = camera_struct(cam)
    lib().orc_intrinsics_jacobian(C.byref(cs), X.ctypes.data, J.ctypes.data)
    return J.reshape(2, 12)


class Backward:
    def __init__(self, dtau, dx, dpose, dtau_abs, dx_abs, dpose_abs, dintr=None, dintr_abs=None, denv=None,
                 denv_abs=None):
        self.dtau, self.dx, self.dpose = dtau, dx, dpose
        self.dtau_abs, self.dx_abs, self.dpose_abs = dtau_abs, dx_abs, dpose_abs
        self.dintr, self.dintr_abs = dintr, dintr_abs
        self.denv, self.denv_abs = denv, denv_abs


def backward(pts: Points, cams, poses, params, fwd: Forward, G: np.ndarray) -> Backward:
    V = len(cams)
    ca, pa = _arrays(cams, poses)
    ps = params_struct(params)
    n, Cc = pts.n, pts.C
    dtau = np.empty((n, Cc)); dtau_abs = np.empty((n, Cc))
    dx = np.empty((3, n)); dx_abs = np.empty((3, n))
    dpose = np.empty((V, 6)); dpose_abs = np.empty((V, 6))
    dintr = np.empty((V, 12)); dintr_abs = np.empty((V, 12))
    env = Env(params)
    denv = denv_abs = None
    if env.arr is not None:
        denv, denv_abs = np.empty(env.arr.shape), np.empty(env.arr.shape)
    G = np.ascontiguousarray(G, dtype=np.float32)
    keys = np.ascontiguousarray(fwd.keys, dtype=np.uint64)
    lib().orc_backward(C.byref(pts.s), V, ca, pa, C.byref(ps), C.byref(env.s), keys.ctypes.data,
                       np.ascontiguousarray(fwd.count).ctypes.data, np.ascontiguousarray(fwd.image).ctypes.data,
                       G.ctypes.data, dtau.ctypes.data, dx.ctypes.data, dpose.ctypes.data, dintr.ctypes.data,
                       _ptr(denv), dtau_abs.ctypes.data, dx_abs.ctypes.data, dpose_abs.ctypes.data,
                       dintr_abs.ctypes.data, _ptr(denv_abs))
    return Backward(dtau, dx, dpose, dtau_abs, dx_abs, dpose_abs, dintr, dintr_abs, denv, denv_abs)
