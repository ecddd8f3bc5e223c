"""Thin ctypes binding of libadop.so (include/adop.h) -- argument marshalling only.

Every step of the rasterizer runs in the library's sm_100a kernels; torch is used
for device memory and streams.  There is no CPU fallback: if libadop.so is
missing or no CUDA device is present, the calls raise.

Names follow the C-ABI without the `adop_` prefix:
    pyramid_pixels, workspace_size, forward_depth, forward_blend, forward_resolve, forward_resolve_range,
    rasterize_forward, rasterize_backward, point_masks, workspace_stats.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import math
import os
from typing import List, Optional, Sequence, Tuple

import numpy as np
import torch

from . import build as _build

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ADOP_LIB", os.path.join(PKG, "libadop.so"))  # ADOP_LIB: a tuning variant
MAX_VIEWS = 16
SENTINEL = 0x7FFFFFFFFFFFFFFF

STATUS = {0: "OK", 1: "INVALID_ARGUMENT", 2: "SHAPE_MISMATCH", 3: "UNSUPPORTED", 4: "WORKSPACE_TOO_SMALL",
          5: "CUDA"}


class AdopError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"adop status {status} ({STATUS.get(status, '?')}): {msg}")
        self.status = status


class adop_points(C.Structure):
    _fields_ = [("n", C.c_int64), ("global_offset", C.c_int64), ("pos_stride", C.c_int64),
                ("pos", C.c_void_p), ("radius", C.c_void_p), ("radius_uniform", C.c_float),
                ("feat", C.c_void_p), ("channels", C.c_int32), ("normal", C.c_void_p), ("tile_bounds", C.c_void_p)]


class adop_camera(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("model", C.c_int32),
                ("fx", C.c_float), ("fy", C.c_float), ("cx", C.c_float), ("cy", C.c_float),
                ("k", C.c_float * 6), ("p", C.c_float * 2), ("r2_max", C.c_float)]


class adop_pose(C.Structure):
    _fields_ = [("R", C.c_float * 9), ("t", C.c_float * 3)]


class adop_params(C.Structure):
    _fields_ = [("layers", C.c_int32), ("alpha", C.c_float), ("discard", C.c_int32), ("gamma", C.c_float),
                ("ghost_rate", C.c_float), ("z_near", C.c_float), ("seed", C.c_uint64),
                ("view_id_base", C.c_int32), ("background", C.c_void_p), ("grad_accumulate", C.c_int32),
                ("log_descriptors", C.c_int32), ("env_map", C.c_void_p), ("env_width", C.c_int32),
                ("env_height", C.c_int32), ("spatial_rendered", C.c_int32), ("normal_culling", C.c_int32),
                ("shared_pyramid", C.c_int32)]


class adop_pyramid(C.Structure):
    _fields_ = [("image", C.c_void_p), ("count", C.c_void_p), ("keys", C.c_void_p), ("accum", C.c_void_p)]


_lib = None


def lib():
    """Load libadop.so (building it first if the sources are newer).  Raises if it cannot be loaded."""
    global _lib
    if _lib is None:
        if LIB_PATH == _build.LIB and _build.needs_build():
            _build.build()
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"libadop.so not found at {LIB_PATH}; run python -m paper_2110_06635_b200.build")
        L = C.CDLL(LIB_PATH)
        P = C.POINTER
        common = [P(adop_points), C.c_int32, P(adop_camera), P(adop_pose), P(adop_params), P(adop_pyramid),
                  C.c_void_p, C.c_size_t, C.c_void_p]
        for name in ("adop_forward_depth", "adop_forward_blend", "adop_forward_resolve"):
            f = getattr(L, name)
            f.restype, f.argtypes = C.c_int, common
        L.adop_forward_resolve_range.restype = C.c_int
        L.adop_forward_resolve_range.argtypes = common[:6] + [C.c_int64, C.c_int64] + common[6:]
        L.adop_rasterize_forward.restype = C.c_int
        L.adop_rasterize_forward.argtypes = common[:-1] + [C.c_void_p, C.c_void_p]  # ..., comm, stream
        L.adop_rasterize_backward.restype = C.c_int
        L.adop_rasterize_backward.argtypes = [P(adop_points), C.c_int32, P(adop_camera), P(adop_pose),
                                              P(adop_params), P(adop_pyramid), P(C.c_void_p), C.c_void_p,
                                              C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                              C.c_size_t, C.c_void_p, C.c_void_p]
        L.adop_comm_unique_id.restype = C.c_int
        L.adop_comm_unique_id.argtypes = [C.c_char_p]
        L.adop_comm_init.restype = C.c_int
        L.adop_comm_init.argtypes = [C.c_int32, C.c_int32, C.c_char_p, C.c_int32, C.c_int32, P(C.c_void_p)]
        L.adop_comm_destroy.restype = C.c_int
        L.adop_comm_destroy.argtypes = [C.c_void_p]
        L.adop_point_masks.restype = C.c_int
        L.adop_point_masks.argtypes = [P(adop_points), C.c_int32, P(adop_camera), P(adop_pose), P(adop_params),
                                       C.c_void_p, C.c_void_p]
        L.adop_pyramid_pixels.restype = C.c_int64
        L.adop_pyramid_pixels.argtypes = [C.c_int32, C.c_int32, C.c_int32]
        L.adop_workspace_size.restype = C.c_int
        L.adop_workspace_size.argtypes = [P(adop_points), C.c_int32, P(adop_camera), P(adop_params), C.c_int64,
                                          P(C.c_size_t)]
        L.adop_workspace_stats.restype = C.c_int
        L.adop_workspace_stats.argtypes = [C.c_void_p, C.c_size_t, C.c_void_p, P(C.c_int64), P(C.c_int64),
                                           P(C.c_int32), P(C.c_int64)]
        L.adop_clear_pyramid.restype = C.c_int
        L.adop_clear_pyramid.argtypes = [C.c_int32, P(adop_camera), C.c_int32, C.c_int32, P(adop_pyramid), C.c_void_p]
        L.adop_ipc_export.restype = C.c_int
        L.adop_ipc_export.argtypes = [C.c_void_p, C.c_char_p, P(C.c_uint64)]
        L.adop_ipc_open.restype = C.c_int
        L.adop_ipc_open.argtypes = [C.c_char_p, C.c_uint64, P(C.c_void_p), P(C.c_void_p)]
        L.adop_ipc_close.restype = C.c_int
        L.adop_ipc_close.argtypes = [C.c_void_p]
        L.adop_tile_bounds.restype = C.c_int
        L.adop_tile_bounds.argtypes = [P(adop_points), C.c_void_p, C.c_void_p]
        L.adop_camera_window.restype = C.c_int
        L.adop_camera_window.argtypes = [P(adop_camera), C.c_int32, P(C.c_float), P(C.c_int32)]
        L.adop_prep_workspace_size.restype = C.c_int
        L.adop_prep_workspace_size.argtypes = [C.c_int64, C.c_int32, P(C.c_size_t)]
        L.adop_blocked_morton_order.restype = C.c_int
        L.adop_blocked_morton_order.argtypes = [P(adop_points), C.c_int32, C.c_uint64, C.c_void_p, C.c_void_p,
                                                C.c_size_t, C.c_void_p]
        L.adop_apply_order.restype = C.c_int
        L.adop_apply_order.argtypes = [P(adop_points), C.c_void_p, P(adop_points), C.c_void_p]
        L.adop_knn_radius.restype = C.c_int
        L.adop_knn_radius.argtypes = [P(adop_points), C.c_int32, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]
        L.adop_last_error.restype = C.c_char_p
        L.adop_version.restype = C.c_char_p
        _lib = L
    return _lib


def _check(status: int):
    if status != 0:
        raise AdopError(status, lib().adop_last_error().decode())


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else t.data_ptr()


# --------------------------------------------------------------------------- #
# descriptors
# --------------------------------------------------------------------------- #
class Points:
    """adop_points over torch CUDA tensors (keeps them alive).  pos: (3, N) or (3, stride) float32."""

    def __init__(self, pos: torch.Tensor, radius: Optional[torch.Tensor], feat: torch.Tensor,
                 global_offset: int = 0, radius_uniform: float = 0.0, n: Optional[int] = None,
                 normal: Optional[torch.Tensor] = None):
        assert pos.dtype == torch.float32 and pos.dim() == 2 and pos.shape[0] == 3 and pos.stride(1) == 1
        assert feat.dtype == torch.float32 and feat.dim() == 2 and feat.is_contiguous()
        # normals (Eq. 5 culling) share the positions' SoA stride
        assert normal is None or (normal.dtype == torch.float32 and normal.shape[0] == 3 and normal.stride() == pos.stride())
        self.pos, self.radius, self.feat, self.normal = pos, radius, feat, normal
        self.n = int(feat.shape[0]) if n is None else int(n)
        self.channels = int(feat.shape[1])
        s = adop_points()
        s.n, s.global_offset, s.pos_stride = self.n, int(global_offset), int(pos.stride(0))
        s.pos, s.radius, s.radius_uniform = _ptr(pos), _ptr(radius), float(radius_uniform)
        s.feat, s.channels = _ptr(feat), self.channels
        s.normal = _ptr(normal)
        self.bounds = None
        self.s = s

    def enable_tile_culling(self, stream=None) -> "Points":
        """Compute per-tile bounds (adop_tile_bounds) so the depth pass skips tiles outside every view.
        Call again after the positions change."""
        if self.bounds is None:
            self.bounds = torch.empty((self.n + 255) // 256 * 8 + 4, dtype=torch.float32, device=self.pos.device)
        ptr = (self.bounds.data_ptr() + 15) // 16 * 16
        self.s.tile_bounds = None
        _check(lib().adop_tile_bounds(C.byref(self.s), ptr, _stream(stream)))
        self.s.tile_bounds = ptr
        return self

    @staticmethod
    def from_cloud(cloud, global_offset: int = 0) -> "Points":
        return Points(cloud.pos, cloud.radius, cloud.feat, global_offset, normal=getattr(cloud, "normal", None))


def camera_struct(cam) -> adop_camera:
    s = adop_camera()
    s.width, s.height, s.model = int(cam.width), int(cam.height), int(cam.model)
    s.fx, s.fy, s.cx, s.cy = cam.fx, cam.fy, cam.cx, cam.cy
    for i in range(6):
        s.k[i] = cam.k[i]
    s.p[0], s.p[1] = cam.p
    s.r2_max = cam.r2_max
    return s


def pose_struct(pose) -> adop_pose:
    s = adop_pose()
    R = [float(v) for v in torch.as_tensor(pose.R, dtype=torch.float32).reshape(9)]
    t = [float(v) for v in torch.as_tensor(pose.t, dtype=torch.float32).reshape(3)]
    for i in range(9):
        s.R[i] = R[i]
    for i in range(3):
        s.t[i] = t[i]
    return s


class Params:
    def __init__(self, p, channels: int):
        s = adop_params()
        s.layers, s.alpha, s.discard, s.gamma = int(p.layers), p.alpha, int(bool(p.discard)), p.gamma
        s.ghost_rate, s.z_near, s.seed, s.view_id_base = p.ghost_rate, p.z_near, int(p.seed), int(p.view_id_base)
        bg = p.background if p.background is not None else None
        self._bg = (C.c_float * channels)(*bg) if bg is not None else None
        s.background = C.cast(self._bg, C.c_void_p) if self._bg is not None else None
        s.grad_accumulate = int(getattr(p, "grad_accumulate", 0))
        s.log_descriptors = int(bool(getattr(p, "log_descriptors", False)))
        s.spatial_rendered = int(bool(getattr(p, "spatial_rendered", False)))
        s.normal_culling = int(getattr(p, "normal_culling", 0))
        s.shared_pyramid = int(bool(getattr(p, "shared_pyramid", False)))
        env = getattr(p, "env_map", None)
        self.env = None
        if env is not None:  # device [H][W][C] float32 (NEXT-2)
            env = torch.as_tensor(env, dtype=torch.float32)
            if not env.is_cuda:
                env = env.cuda()
            self.env = env.contiguous()
            assert self.env.dim() == 3 and self.env.shape[2] == channels
            s.env_map, s.env_height, s.env_width = self.env.data_ptr(), self.env.shape[0], self.env.shape[1]
        self.s = s
        self.layers = int(p.layers)


def pyramid_pixels(width: int, height: int, layers: int) -> int:
    return int(lib().adop_pyramid_pixels(width, height, layers))


@dataclasses.dataclass
class Pyramid:
    """Buffers of one view.  accum and count are views of one tensor `ac` so a point-sharded
    caller can sum-reduce both in a single collective."""
    image: torch.Tensor   # [C*P] float32
    count: torch.Tensor   # [P] float32
    keys: torch.Tensor    # [P] int64 (uint64 bit pattern)
    accum: torch.Tensor   # [P*C] float32
    ac: torch.Tensor      # [P*(C+1)] float32 backing accum ++ count
    width: int
    height: int
    layers: int

    def struct(self) -> adop_pyramid:
        s = adop_pyramid()
        s.image, s.count, s.keys, s.accum = (self.image.data_ptr(), self.count.data_ptr(), self.keys.data_ptr(),
                                             self.accum.data_ptr())
        return s

    def layer_image(self, l: int, channels: int) -> torch.Tensor:
        """Layer l as a (C, h_l, w_l) view of the planar image (Eq. 1's I_l)."""
        off = 0
        for k in range(l):
            off += -(-self.width // (1 << k)) * -(-self.height // (1 << k))
        wl, hl = -(-self.width // (1 << l)), -(-self.height // (1 << l))
        return self.image[channels * off: channels * (off + wl * hl)].view(channels, hl, wl)


class PeerPyramid:
    """A view's pyramid whose keys / accum / count live in another process's memory (CUDA IPC, peer
    access over NVLink; point sharding).  The image pointer is this process's own
    (only the owner resolves)."""

    def __init__(self, keys: int, accum: int, count: int, image: int, width: int, height: int, layers: int):
        self.keys_ptr, self.accum_ptr, self.count_ptr, self.image_ptr = keys, accum, count, image
        self.width, self.height, self.layers = width, height, layers

    def struct(self) -> adop_pyramid:
        s = adop_pyramid()
        s.image, s.count, s.keys, s.accum = self.image_ptr, self.count_ptr, self.keys_ptr, self.accum_ptr
        return s


def clear_pyramid(cams, layers: int, channels: int, pyrs, stream=None):
    """keys <- sentinel, accum, count <- 0 (the owner's reset of a shared pyramid)."""
    ca = (adop_camera * len(cams))(*[camera_struct(c) for c in cams])
    pa = (adop_pyramid * len(pyrs))(*[p.struct() for p in pyrs])
    _check(lib().adop_clear_pyramid(len(cams), ca, int(layers), int(channels), pa, _stream(stream)))


def ipc_export(t: torch.Tensor) -> Tuple[bytes, int]:
    """(64-byte handle of the allocation holding t, byte offset of t in it)."""
    h = C.create_string_buffer(64)
    off = C.c_uint64(0)
    _check(lib().adop_ipc_export(t.data_ptr(), h, C.byref(off)))
    return h.raw, int(off.value)


_ipc_maps = {}


def ipc_open(handle: bytes, offset: int) -> int:
    """Device pointer of an exported tensor in this process (one mapping per allocation, cached)."""
    base = _ipc_maps.get(handle)
    if base is None:
        b, p = C.c_void_p(0), C.c_void_p(0)
        _check(lib().adop_ipc_open(handle, 0, C.byref(b), C.byref(p)))
        base = _ipc_maps[handle] = int(b.value)
    return base + int(offset)


def ipc_close_all():
    for base in _ipc_maps.values():
        _check(lib().adop_ipc_close(base))
    _ipc_maps.clear()


def alloc_pyramids(cams, layers: int, channels: int, device) -> List[Pyramid]:
    out = []
    for cam in cams:
        P = pyramid_pixels(cam.width, cam.height, layers)
        ac = torch.empty(P * (channels + 1), dtype=torch.float32, device=device)
        out.append(Pyramid(torch.empty(channels * P, dtype=torch.float32, device=device),
                           ac[P * channels:], torch.empty(P, dtype=torch.int64, device=device),
                           ac[:P * channels], ac, cam.width, cam.height, layers))
    return out


class Workspace:
    """Caller-owned scratch of adop_workspace_size bytes (256-B aligned): header, pose partials, the
    backward's pixel tables and the record region (survivor records + ghost list).  The backward consumes
    the depth pass's lists when it is given the same workspace and the same inputs."""

    def __init__(self, points: Points, cams, params: Params, device, record_capacity: int = -1):
        V = len(cams)
        ca = (adop_camera * V)(*[camera_struct(c) for c in cams])
        size = C.c_size_t(0)
        _check(lib().adop_workspace_size(C.byref(points.s), V, ca, C.byref(params.s), int(record_capacity),
                                         C.byref(size)))
        self.nbytes = int(size.value)
        self.buf = torch.empty((self.nbytes + 255) // 256 * 256 + 256, dtype=torch.uint8, device=device)
        base = self.buf.data_ptr()
        self.ptr = (base + 255) // 256 * 256

    def stats(self, stream=None):
        """(survivor record slots, overflowed) of the last depth pass (synchronizes the stream)."""
        rec, _, of = self.stats3(stream)
        return rec, of

    def stats3(self, stream=None):
        """(survivor record slots, ghost-list entries of the last backward, overflowed)."""
        rec, gh, of, tr = C.c_int64(0), C.c_int64(0), C.c_int32(0), C.c_int64(0)
        _check(lib().adop_workspace_stats(self.ptr, self.nbytes, _stream(stream), C.byref(rec), C.byref(gh),
                                          C.byref(of), C.byref(tr)))
        self.tiles_read = int(tr.value)
        return int(rec.value), int(gh.value), bool(of.value)


def default_record_capacity(n: int, n_views: int, layers: int, discard: bool) -> int:
    """Worst case n*V*L (+ chunk slack) when affordable (< 4 GiB), else a generous bound: with stochastic discarding
    the kept points per pixel are bounded (Eq. 12), so the records are far below the worst case;
    exceeding the capacity is still correct (the blend pass re-streams the points)."""
    slack = 1 << 20  # partially filled per-warp record chunks (dead slots)
    worst = n * n_views * max(layers, 2)  # a ghost entry takes 2 slots
    if worst * 16 <= (4 << 30) or not discard:
        return worst + slack
    return max(1 << 22, worst // 4) + slack


def _stream(stream):
    if stream is None:
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))


class _Call:
    """Marshalled arguments of one call (keeps ctypes arrays alive)."""

    def __init__(self, points: Points, cams, poses, params: Params, pyrs: Optional[Sequence[Pyramid]]):
        V = len(cams)
        if V < 1 or V > MAX_VIEWS:
            raise ValueError(f"1..{MAX_VIEWS} views per call, got {V}")
        self.V = V
        self.cams = (adop_camera * V)(*[camera_struct(c) for c in cams])
        self.poses = (adop_pose * V)(*[pose_struct(p) for p in poses])
        self.pyrs = (adop_pyramid * V)(*[p.struct() for p in pyrs]) if pyrs is not None else None
        self.points, self.params = points, params


def _phase(fn_name, points, cams, poses, params, pyrs, ws: Workspace, stream=None, call=None):
    c = _Call(points, cams, poses, params, pyrs) if call is None else call
    fn = getattr(lib(), fn_name)
    _check(fn(C.byref(points.s), c.V, c.cams, c.poses, C.byref(params.s), c.pyrs, ws.ptr, ws.nbytes,
              _stream(stream)))


def forward_depth(points, cams, poses, params, pyrs, ws, stream=None, call=None):
    """Phase 1.  `call`: a cached _Call of the same arguments (skips the per-call marshalling)."""
    _phase("adop_forward_depth", points, cams, poses, params, pyrs, ws, stream, call)


def forward_blend(points, cams, poses, params, pyrs, ws, stream=None, call=None):
    _phase("adop_forward_blend", points, cams, poses, params, pyrs, ws, stream, call)


def forward_resolve(points, cams, poses, params, pyrs, ws, stream=None, call=None):
    _phase("adop_forward_resolve", points, cams, poses, params, pyrs, ws, stream, call)


def forward_resolve_range(points, cams, poses, params, pyrs, ws, p0: int, p1: int, stream=None, call=None):
    """Phase 3 over pyramid pixels [p0, p1) of every view (adop_forward_resolve_range)."""
    c = _Call(points, cams, poses, params, pyrs) if call is None else call
    _check(lib().adop_forward_resolve_range(C.byref(points.s), c.V, c.cams, c.poses, C.byref(params.s), c.pyrs,
                                            int(p0), int(p1), ws.ptr, ws.nbytes, _stream(stream)))


def rasterize_forward(points, cams, poses, params, pyrs, ws, stream=None, call=None, comm=None):
    """Fused forward; comm: a Comm (multi-GPU collectives between the phases) or None."""
    c = _Call(points, cams, poses, params, pyrs) if call is None else call
    _check(lib().adop_rasterize_forward(C.byref(points.s), c.V, c.cams, c.poses, C.byref(params.s), c.pyrs, ws.ptr,
                                        ws.nbytes, None if comm is None else comm.ptr, _stream(stream)))


SHARD_POINTS, SHARD_VIEWS, COMM_KEYS32 = 0, 1, 1


class Comm:
    """The library's NCCL communicator (adop_comm_init): ADOP_SHARD_POINTS or ADOP_SHARD_VIEWS collectives run
    inside adop_rasterize_forward / _backward.  Rank 0 creates the id (unique_id()), every rank passes it."""

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        _check(lib().adop_comm_unique_id(buf))
        return buf.raw

    def __init__(self, nranks: int, rank: int, uid: bytes, mode: int, flags: int = 0):
        p = C.c_void_p()
        _check(lib().adop_comm_init(int(nranks), int(rank), C.create_string_buffer(uid, 128), int(mode), int(flags),
                                    C.byref(p)))
        self.ptr = p

    def close(self):
        if self.ptr:
            _check(lib().adop_comm_destroy(self.ptr))
            self.ptr = None


def rasterize_backward(points, cams, poses, params, pyrs, grads: Sequence[torch.Tensor], ws,
                       d_feat: Optional[torch.Tensor], d_pos: Optional[torch.Tensor],
                       d_pose: Optional[torch.Tensor], d_intr: Optional[torch.Tensor] = None,
                       d_env: Optional[torch.Tensor] = None, stream=None, call=None, comm=None):
    """d_intr: optional [V][12] float64 camera-intrinsics gradient (fx, fy, cx, cy, k1..k6, p1, p2);
    d_env: optional [H][W][C] float32 environment-map gradient (needs params.env_map)."""
    c = _Call(points, cams, poses, params, pyrs) if call is None else call
    g = (C.c_void_p * c.V)(*[t.data_ptr() for t in grads])
    _check(lib().adop_rasterize_backward(C.byref(points.s), c.V, c.cams, c.poses, C.byref(params.s), c.pyrs, g,
                                         _ptr(d_feat), _ptr(d_pos), _ptr(d_pose), _ptr(d_intr), _ptr(d_env), ws.ptr,
                                         ws.nbytes, None if comm is None else comm.ptr, _stream(stream)))


def point_masks(points, cams, poses, params, mask: torch.Tensor, stream=None):
    c = _Call(points, cams, poses, params, None)
    _check(lib().adop_point_masks(C.byref(points.s), c.V, c.cams, c.poses, C.byref(params.s), mask.data_ptr(),
                                  _stream(stream)))


# --------------------------------------------------------------------------- #
# preprocessing (NEXT-4): blocked Morton shuffle, kNN world radius
# --------------------------------------------------------------------------- #
def _prep_ws(n: int, block: int, device):
    size = C.c_size_t(0)
    _check(lib().adop_prep_workspace_size(int(n), int(block), C.byref(size)))
    buf = torch.empty(int(size.value) + 256, dtype=torch.uint8, device=device)
    return buf, (buf.data_ptr() + 255) // 256 * 256, int(size.value)


def blocked_morton_order(points: Points, block: int = 1024, seed: int = 0, stream=None) -> torch.Tensor:
    """int64 permutation of the blocked Morton shuffle (R34): perm[j] = old index."""
    dev = points.pos.device
    buf, ptr, size = _prep_ws(points.n, block, dev)
    perm = torch.empty(points.n, dtype=torch.int64, device=dev)
    _check(lib().adop_blocked_morton_order(C.byref(points.s), int(block), int(seed), perm.data_ptr(), ptr, size,
                                           _stream(stream)))
    del buf  # torch's caching allocator only reuses the block for work ordered after this stream's
    return perm


def apply_order(points: Points, perm: torch.Tensor, stream=None) -> Points:
    """A new Points whose arrays are points' arrays gathered by perm (positions, radii, descriptors, normals)."""
    pos = torch.empty_like(points.pos)
    rad = None if points.radius is None else torch.empty_like(points.radius)
    feat = torch.empty_like(points.feat)
    nrm = None if points.normal is None else torch.empty_like(points.normal)
    dst = Points(pos, rad, feat, int(points.s.global_offset), float(points.s.radius_uniform), points.n, normal=nrm)
    _check(lib().adop_apply_order(C.byref(points.s), perm.data_ptr(), C.byref(dst.s), _stream(stream)))
    return dst


def knn_radius(points: Points, k: int = 8, stream=None) -> torch.Tensor:
    """r_world (R33): median distance to the k nearest neighbours, float32 [n]."""
    dev = points.pos.device
    buf, ptr, size = _prep_ws(points.n, 1, dev)
    r = torch.empty(points.n, dtype=torch.float32, device=dev)
    _check(lib().adop_knn_radius(C.byref(points.s), int(k), r.data_ptr(), ptr, size, _stream(stream)))
    del buf  # (as above)
    return r


def camera_window(cam, layers: int):
    """(xlo, xhi, ylo, yhi) of the OpenCV8 candidate window in undistorted normalized coordinates, or None
    (adop_camera_window; host only)."""
    out, valid = (C.c_float * 4)(), C.c_int32(0)
    cs = camera_struct(cam)
    _check(lib().adop_camera_window(C.byref(cs), int(layers), out, C.byref(valid)))
    return tuple(out) if valid.value else None


def version() -> str:
    return lib().adop_version().decode()


class Renderer:
    """Convenience owner of the device buffers of one (cloud, views) configuration.

    forward()  -> adop_rasterize_forward into self.pyrs
    backward(grads) -> adop_rasterize_backward into self.d_feat / self.d_pos / self.d_pose
    """

    def __init__(self, cloud, cams, poses, params, global_offset: int = 0, record_capacity: Optional[int] = None,
                 device=None, intrinsics: bool = False, comm: Optional["Comm"] = None):
        device = cloud.pos.device if device is None else device
        self.comm = comm  # multi-GPU collectives inside the fused calls (Comm) or None
        self.cams, self.poses, self.sparams = list(cams), list(poses), params
        self.points = Points.from_cloud(cloud, global_offset)
        self.C = self.points.channels
        self.params = Params(params, self.C)
        self.pyrs = alloc_pyramids(self.cams, params.layers, self.C, device)
        if record_capacity is None:
            record_capacity = default_record_capacity(self.points.n, len(self.cams), params.layers, params.discard)
        self.ws = Workspace(self.points, self.cams, self.params, device, record_capacity)
        self.device = device
        self.d_feat = self.d_pos = self.d_pose = self.d_intr = self.d_env = None
        self.intrinsics = intrinsics  # backward also produces d_intr [V][12] (NEXT-1)

    def set_poses(self, poses):
        """Replace the views' poses (e.g. after a pose-refinement step with d_pose)."""
        assert len(poses) == len(self.cams)
        self.poses = list(poses)

    def set_cameras(self, cams):
        """Replace the views' cameras (e.g. after an intrinsics step with d_intr); same image sizes."""
        assert len(cams) == len(self.cams) and all(
            (a.width, a.height) == (b.width, b.height) for a, b in zip(cams, self.cams))
        self.cams = list(cams)

    def _key(self):
        # the values the marshalled descriptors are built from: poses and cameras may be replaced or edited in
        # place between calls (refinement with d_pose / d_intr), so the cache is keyed on their values
        k = []
        for c, p in zip(self.cams, self.poses):
            k.append((c.width, c.height, c.model, c.fx, c.fy, c.cx, c.cy, tuple(c.k), tuple(c.p), c.r2_max,
                      np.asarray(p.R, dtype=np.float32).tobytes(), np.asarray(p.t, dtype=np.float32).tobytes()))
        return tuple(k)

    def _call(self):
        # marshalled descriptors, rebuilt only when a pose or camera value changed
        key = self._key()
        if getattr(self, "_c", None) is None or self._ckey != key:
            self._c = _Call(self.points, self.cams, self.poses, self.params, self.pyrs)
            self._ckey = key
        return self._c

    def forward(self, stream=None):
        rasterize_forward(self.points, self.cams, self.poses, self.params, self.pyrs, self.ws, stream, self._call(),
                          self.comm)
        return self.pyrs

    def alloc_grads(self):
        n = self.points.n
        self.d_feat = torch.empty(n, self.C, dtype=torch.float32, device=self.device)
        self.d_pos = torch.empty(3, n, dtype=torch.float32, device=self.device)
        self.d_pose = torch.empty(len(self.cams), 6, dtype=torch.float64, device=self.device)
        if self.intrinsics:
            self.d_intr = torch.empty(len(self.cams), 12, dtype=torch.float64, device=self.device)
        if self.params.env is not None:
            self.d_env = torch.empty_like(self.params.env)

    def backward(self, grads: Sequence[torch.Tensor], stream=None):
        if getattr(self, "peer_non_owner", False):
            raise RuntimeError("backward on a non-owner of a shared (peer-memory) pyramid: its image is never "
                               "resolved; run the backward on the owner (the p2p point sharding is forward-only)")
        if self.d_feat is None:
            self.alloc_grads()
        rasterize_backward(self.points, self.cams, self.poses, self.params, self.pyrs, grads, self.ws,
                           self.d_feat, self.d_pos, self.d_pose, self.d_intr, self.d_env, stream, self._call(),
                           self.comm)
        return self.d_feat, self.d_pos, self.d_pose

    def masks(self, stream=None) -> torch.Tensor:
        m = torch.empty(len(self.cams), self.points.n, dtype=torch.uint8, device=self.device)
        point_masks(self.points, self.cams, self.poses, self.params, m, stream)
        return m
