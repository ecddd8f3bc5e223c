"""The C-ABI library loads and exports every symbol include/adop.h declares; host-side argument
validation rejects bad input before touching the GPU.  CPU only: no compute calls."""
import ctypes as C
import math
import os
import re

import pytest

from paper_2110_06635_b200 import adop as A
from paper_2110_06635_b200 import scene as S

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "adop.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(adop_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = A.lib()
    syms = declared_symbols()
    assert len(syms) >= 11
    for s in syms:
        assert hasattr(lib, s), s
    assert "sm_100a" in A.version()


def test_pyramid_pixels_and_workspace_size():
    assert A.pyramid_pixels(1920, 1080, 5) == 2762160
    assert A.pyramid_pixels(256, 256, 4) == 87040
    assert A.pyramid_pixels(0, 10, 1) == 0 and A.pyramid_pixels(10, 10, 9) == 0
    pts = A.adop_points()
    pts.n, pts.channels = 1000, 4
    prm = A.adop_params()
    prm.layers = 5
    sz = C.c_size_t()
    cam = A.adop_camera()
    cam.width, cam.height = 64, 32
    cams = (A.adop_camera * 2)(cam, cam)
    assert A.lib().adop_workspace_size(C.byref(pts), 2, cams, C.byref(prm), -1, C.byref(sz)) == 0
    P = A.pyramid_pixels(64, 32, 5)
    tables = -(-2 * P * (16 + 4 * 4) // 256) * 256  # rows of 16 + 4 roundup4(C) bytes
    rec = lambda cap: -(-cap // 64) * (64 * 16 + 1 + 8) + 1024  # 64-slot chunks + chunk tables (include/adop.h)
    assert sz.value == 4096 + 2048 * 16 * 18 * 8 + tables + rec(1000 * 2 * 5 + (1 << 20))
    assert A.lib().adop_workspace_size(C.byref(pts), 2, cams, C.byref(prm), 100, C.byref(sz)) == 0
    assert sz.value == 4096 + 2048 * 16 * 18 * 8 + tables + rec(100)
    prm.layers = 1  # a ghost entry takes 2 slots: worst case n * V * max(L, 2)
    assert A.lib().adop_workspace_size(C.byref(pts), 2, cams, C.byref(prm), -1, C.byref(sz)) == 0
    tables1 = -(-2 * A.pyramid_pixels(64, 32, 1) * 32 // 256) * 256
    assert sz.value == 4096 + 2048 * 16 * 18 * 8 + tables1 + rec(1000 * 2 * 2 + (1 << 20))
    prm.layers = 5
    assert A.lib().adop_workspace_size(C.byref(pts), 0, cams, C.byref(prm), -1, C.byref(sz)) == 1
    assert A.lib().adop_workspace_size(C.byref(pts), 2, None, C.byref(prm), -1, C.byref(sz)) == 1


def _call(points, cams, poses, params, pyrs, ws_ptr=256 * 1024, ws_bytes=1 << 30):
    V = len(cams)
    ca = (A.adop_camera * V)(*[A.camera_struct(c) for c in cams])
    pa = (A.adop_pose * V)(*[A.pose_struct(p) for p in poses])
    py = (A.adop_pyramid * V)(*pyrs) if pyrs is not None else None
    st = A.lib().adop_rasterize_forward(C.byref(points), V, ca, pa, C.byref(params), py, C.c_void_p(ws_ptr),
                                        ws_bytes, None, None)
    return st, A.lib().adop_last_error().decode()


def _valid():
    pts = A.adop_points()
    pts.n, pts.pos_stride, pts.pos, pts.feat, pts.channels = 8, 8, 4096, 8192, 4
    pts.radius_uniform = 0.005
    prm = A.Params(S.Params(layers=4, discard=True), 4).s
    pyr = A.adop_pyramid()
    pyr.image, pyr.count, pyr.keys, pyr.accum = 1 << 20, 2 << 20, 3 << 20, 4 << 20
    cam = S.pinhole(256, 256, f=200.0)
    return pts, [cam], [S.tiny_pose()], prm, [pyr]


@pytest.mark.parametrize("mutate,expect", [
    (lambda p, c, q, r, y: setattr(p, "n", -1), "n = -1"),
    (lambda p, c, q, r, y: setattr(p, "channels", 0), "channels"),
    (lambda p, c, q, r, y: setattr(p, "channels", 33), "channels"),
    (lambda p, c, q, r, y: setattr(p, "pos", 0), "pos is NULL"),
    (lambda p, c, q, r, y: setattr(p, "pos", 4098), "aligned"),
    (lambda p, c, q, r, y: setattr(p, "pos_stride", 4), "pos_stride"),
    (lambda p, c, q, r, y: setattr(p, "global_offset", (1 << 32) - 4), "global_offset"),
    (lambda p, c, q, r, y: setattr(r, "layers", 0), "layers"),
    (lambda p, c, q, r, y: setattr(r, "layers", 9), "layers"),
    (lambda p, c, q, r, y: setattr(r, "alpha", -0.1), "alpha"),
    (lambda p, c, q, r, y: setattr(r, "gamma", 0.0), "gamma"),
    (lambda p, c, q, r, y: setattr(r, "ghost_rate", 1.0), "ghost_rate"),
    (lambda p, c, q, r, y: setattr(r, "z_near", -1.0), "z_near"),
    (lambda p, c, q, r, y: setattr(c[0], "width", 0), "width"),
    (lambda p, c, q, r, y: setattr(c[0], "model", 7), "model"),
    (lambda p, c, q, r, y: setattr(c[0], "fx", math.nan), "intrinsics"),
    (lambda p, c, q, r, y: setattr(y[0], "keys", 0), "NULL pyramid"),
    (lambda p, c, q, r, y: setattr(y[0], "keys", (3 << 20) + 4), "misaligned"),
])
def test_invalid_arguments_rejected_before_launch(mutate, expect):
    pts, cams, poses, prm, pyrs = _valid()
    cams = [A.camera_struct(c) for c in cams]
    mutate(pts, cams, poses, prm, pyrs)
    V = 1
    ca = (A.adop_camera * V)(*cams)
    pa = (A.adop_pose * V)(*[A.pose_struct(p) for p in poses])
    py = (A.adop_pyramid * V)(*pyrs)
    st = A.lib().adop_rasterize_forward(C.byref(pts), V, ca, pa, C.byref(prm), py, C.c_void_p(256 * 1024),
                                        1 << 30, None, None)
    assert st == 1, st
    assert expect in A.lib().adop_last_error().decode()


def test_workspace_checks():
    pts, cams, poses, prm, pyrs = _valid()
    st, msg = _call(pts, cams, poses, prm, pyrs, ws_ptr=256 * 1024 + 8)
    assert st == 1 and "256-byte" in msg
    st, msg = _call(pts, cams, poses, prm, pyrs, ws_bytes=1024)
    assert st == 4 and "workspace" in msg
    st, msg = _call(pts, cams, poses, prm, pyrs, ws_ptr=0)
    assert st == 1


def test_view_count_limits():
    pts, cams, poses, prm, pyrs = _valid()
    st, msg = _call(pts, cams * 17, poses * 17, prm, pyrs * 17)
    assert st == 1 and "n_views" in msg


def test_shared_pyramid_and_ipc_arguments_rejected():
    """adop_clear_pyramid / adop_ipc_* validate their arguments before any CUDA call."""
    L = A.lib()
    _, cams, _, _, pyrs = _valid()
    ca = (A.adop_camera * 1)(A.camera_struct(cams[0]))
    py = (A.adop_pyramid * 1)(*pyrs)
    assert L.adop_clear_pyramid(1, None, 4, 4, py, None) == 1
    assert L.adop_clear_pyramid(0, ca, 4, 4, py, None) == 1 and "n_views" in L.adop_last_error().decode()
    assert L.adop_clear_pyramid(1, ca, 0, 4, py, None) == 1 and "layers" in L.adop_last_error().decode()
    assert L.adop_clear_pyramid(1, ca, 4, 0, py, None) == 1 and "channels" in L.adop_last_error().decode()
    bad = A.adop_pyramid()
    bad.image, bad.count, bad.keys, bad.accum = 1 << 20, 0, 3 << 20, 4 << 20
    assert L.adop_clear_pyramid(1, ca, 4, 4, (A.adop_pyramid * 1)(bad), None) == 1
    assert "NULL pyramid" in L.adop_last_error().decode()
    h = C.create_string_buffer(64)
    off = C.c_uint64(0)
    assert L.adop_ipc_export(None, h, C.byref(off)) == 1
    assert L.adop_ipc_export(C.c_void_p(4096), None, C.byref(off)) == 1
    b, p = C.c_void_p(0), C.c_void_p(0)
    assert L.adop_ipc_open(None, 0, C.byref(b), C.byref(p)) == 1
    assert L.adop_ipc_open(h.raw, 0, None, C.byref(p)) == 1
    assert L.adop_ipc_close(None) == 1


def test_comm_arguments_rejected_without_a_gpu():
    """adop_comm_init validates its arguments before touching NCCL or the GPU."""
    p = C.c_void_p()
    uid = C.create_string_buffer(128)
    assert A.lib().adop_comm_init(2, 2, uid, 0, 0, C.byref(p)) == 1 and not p.value
    assert A.lib().adop_comm_init(0, 0, uid, 0, 0, C.byref(p)) == 1
    assert A.lib().adop_comm_init(1, 0, uid, 7, 0, C.byref(p)) == 1
    assert A.lib().adop_comm_init(1, 0, uid, 0, 4, C.byref(p)) == 1
    assert A.lib().adop_comm_destroy(None) == 0


def test_resolve_range_rejects_bad_ranges_before_launch():
    """adop_forward_resolve_range: p0 < 0 or p1 < p0 is an invalid argument (checked before any device work)."""
    pts, cams, poses, prm, pyrs = _valid()
    V = 1
    ca = (A.adop_camera * V)(*[A.camera_struct(c) for c in cams])
    pa = (A.adop_pose * V)(*[A.pose_struct(p) for p in poses])
    py = (A.adop_pyramid * V)(*pyrs)
    for p0, p1 in ((-4, 8), (16, 8)):
        st = A.lib().adop_forward_resolve_range(C.byref(pts), V, ca, pa, C.byref(prm), py, p0, p1,
                                                C.c_void_p(256 * 1024), 1 << 30, None)
        assert st == 1, st
        assert "resolve range" in A.lib().adop_last_error().decode()
