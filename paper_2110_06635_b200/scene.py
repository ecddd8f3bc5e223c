"""Seeded synthetic inputs for the ADOP rasterizer hot path (arXiv 2110.06635).

This module is the ONE place both the CUDA path and the CPU oracle get their
inputs from.  It holds none of the method's arithmetic: no projection, no
rounding, no discard test, no depth test, no blending.  It only draws point
clouds, features, camera intrinsics, poses and upstream image gradients, and
orders the cloud (blocked Morton shuffle, an untimed preprocessing step).

Recipe (SURVEY.md §8(d) "Concrete synthetic inputs"):

* The paper's clouds are unnamed scans of 1.35M-10.3M points at 1080p
  (Table 1) and 8-73M point scenes (L665, L683, L804).  None
  are in the container; a synthetic room stands in for them: the 6 walls of an
  axis-aligned box of side S plus 20 spheres (radius U[0.2,1]*S/10), points
  sampled uniformly by area, isotropic N(0, 5 mm) noise, world radius 5 mm.
* Features tau ~ U(0,1) fp32 (the neural descriptor of Eq. 1).
* Poses: camera centre uniform in [-0.4S, 0.4S]^3 away from the spheres,
  uniformly random orientation; world->camera (R, t), Xc = R x + t (Eq. 2).
* Pinhole f = w/2, c = (w/2, h/2); OpenCV 8-coefficient distortion with
  k1..k6 ~ U(-0.1, 0.1), p1, p2 ~ U(-0.01, 0.01) (BASELINE.json configs[2]).
  The camera descriptor carries r2_max, the radius (in normalized r^2) up to
  which the distortion map is monotone and its denominator safely positive; it
  is a property of the chosen camera, computed here once per camera in fp64
  (reading R6) and read by both sides.
* Upstream gradients G ~ U(-1, 1) for every pyramid element.
* Blocked Morton shuffle (§4.5): quantize to 2^21 cells per
  axis, sort by 63-bit Morton code, cut into blocks of B points, permute the
  blocks with a seeded permutation.
"""
from __future__ import annotations

import dataclasses
import math
from typing import List, Optional

import numpy as np
import torch

PINHOLE = 0
OPENCV8 = 1
FISHEYE = 2  # equidistant fisheye, distance depth (R35); Camera.r2_max holds theta_max (radians)

# Seeds (proposed and fixed here).
SEED_SCENE, SEED_POSES, SEED_CAMERAS, SEED_FEATURES, SEED_GRADS, SEED_STEP = 2110, 6635, 3, 4, 5, 6


@dataclasses.dataclass
class Camera:
    width: int
    height: int
    model: int
    fx: float
    fy: float
    cx: float
    cy: float
    k: tuple = (0.0,) * 6
    p: tuple = (0.0, 0.0)
    r2_max: float = math.inf


@dataclasses.dataclass
class Pose:
    R: np.ndarray  # (3,3) float32, world->camera, row-major
    t: np.ndarray  # (3,) float32


@dataclasses.dataclass
class Cloud:
    pos: torch.Tensor      # (3, N) float32 SoA: rows x, y, z
    radius: torch.Tensor   # (N,) float32 world radius
    feat: torch.Tensor     # (N, C) float32 neural descriptor tau
    normal: Optional[torch.Tensor] = None  # (3, N) float32 SoA unit normals n of Eq. 1 (Eq. 5 culling), optional

    @property
    def n(self) -> int:
        return int(self.pos.shape[1])

    @property
    def channels(self) -> int:
        return int(self.feat.shape[1])

    def to(self, device) -> "Cloud":
        return Cloud(self.pos.to(device), self.radius.to(device), self.feat.to(device),
                     None if self.normal is None else self.normal.to(device))

    def slice(self, a: int, b: int) -> "Cloud":
        return Cloud(self.pos[:, a:b].contiguous(), self.radius[a:b].contiguous(), self.feat[a:b].contiguous(),
                     None if self.normal is None else self.normal[:, a:b].contiguous())


@dataclasses.dataclass
class Params:
    layers: int = 5
    alpha: float = 0.01      # fuzzy depth threshold
    discard: bool = True     # stochastic point discarding, §4.4
    gamma: float = 1.5
    ghost_rate: float = 0.0  # dropout rate rho of the ghost split, §4.3
    z_near: float = 0.0
    seed: int = SEED_STEP
    view_id_base: int = 0
    background: Optional[List[float]] = None  # constant E; None -> zeros
    log_descriptors: bool = False  # NEXT-2: tau stored as log, exp() when rasterized
    env_map: Optional[object] = None  # NEXT-2: [H][W][C] float32 equirectangular E of Eq. 7 (R29); None -> background
    spatial_rendered: bool = False  # NEXT-3: ghost gradients disabled, Eqs. 9-11 for rendered points (R31)
    normal_culling: int = 0  # NEXT-3: Eq. 5 (R32): 0 off, +1 keep (Rn).Xc > 0 as printed, -1 flipped


# --------------------------------------------------------------------------- #
# Point clouds
# --------------------------------------------------------------------------- #
def _gen(seed: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    return g


def uniform_cube_cloud(n: int, channels: int = 4, seed: int = SEED_SCENE, device="cpu") -> Cloud:
    """Tiny config (BASELINE.json configs[0]): points U[-1,1]^3, features U(0,1)."""
    g = _gen(seed, device)
    pos = (torch.rand(3, n, generator=g, device=device, dtype=torch.float32) * 2.0 - 1.0).contiguous()
    feat = torch.rand(n, channels, generator=g, device=device, dtype=torch.float32)
    radius = torch.full((n,), 0.005, dtype=torch.float32, device=device)
    return Cloud(pos, radius, feat)


@dataclasses.dataclass
class Room:
    size: float
    centers: np.ndarray  # (20, 3) float64
    radii: np.ndarray    # (20,) float64


def make_room(size: float, n_spheres: int = 20, seed: int = SEED_SCENE) -> Room:
    rng = np.random.default_rng(seed)
    radii = rng.uniform(0.2, 1.0, n_spheres) * size / 10.0
    half = size / 2.0
    centers = np.stack([rng.uniform(-half + r, half - r, 3) for r in radii])
    return Room(size, centers, radii)


def room_cloud(n: int, room: Room, channels: int = 4, noise: float = 0.005, radius: float = 0.005,
               seed: int = SEED_SCENE, device="cpu", chunk: int = 1 << 24) -> Cloud:
    """Synthetic room: walls + spheres sampled by area, N(0, noise) jitter."""
    S = room.size
    half = S / 2.0
    areas = np.concatenate([np.full(6, S * S), 4.0 * np.pi * room.radii ** 2])
    cdf = torch.tensor(np.cumsum(areas) / areas.sum(), dtype=torch.float64, device=device)
    centers = torch.tensor(room.centers, dtype=torch.float32, device=device)
    radii = torch.tensor(room.radii, dtype=torch.float32, device=device)
    g = _gen(seed, device)
    pos = torch.empty(3, n, dtype=torch.float32, device=device)
    nrm = torch.empty(3, n, dtype=torch.float32, device=device)
    for a in range(0, n, chunk):
        b = min(n, a + chunk)
        m = b - a
        surf = torch.searchsorted(cdf, torch.rand(m, generator=g, device=device, dtype=torch.float64), right=True)
        surf.clamp_(max=len(areas) - 1)
        uv = (torch.rand(2, m, generator=g, device=device) * 2.0 - 1.0) * half
        p = torch.zeros(3, m, dtype=torch.float32, device=device)
        axis = torch.div(surf.clamp(max=5), 2, rounding_mode="floor")  # faces 0..5: axis = f//2, sign by parity
        sign = torch.where(surf % 2 == 0, -1.0, 1.0).to(torch.float32)
        # wall points: fixed coordinate on the chosen axis, the two others uniform
        for ax, (o1, o2) in enumerate(((1, 2), (0, 2), (0, 1))):
            sel = (axis == ax) & (surf < 6)
            p[ax] = torch.where(sel, sign * half, p[ax])
            p[o1] = torch.where(sel, uv[0], p[o1])
            p[o2] = torch.where(sel, uv[1], p[o2])
        # sphere points: centre + r * uniform direction
        d = torch.randn(3, m, generator=g, device=device)
        d = d / d.norm(dim=0, keepdim=True).clamp_min(1e-12)
        sid = (surf - 6).clamp(min=0)
        sph = centers[sid].T + radii[sid] * d
        p = torch.where((surf >= 6).unsqueeze(0), sph, p)
        # normals (no random draws): walls face the room's inside, spheres outward
        nw = torch.zeros(3, m, dtype=torch.float32, device=device)
        for ax in range(3):
            nw[ax] = torch.where((axis == ax) & (surf < 6), -sign, nw[ax])
        nrm[:, a:b] = torch.where((surf >= 6).unsqueeze(0), d, nw)
        p += torch.randn(3, m, generator=g, device=device) * noise
        pos[:, a:b] = p
    gf = _gen(seed + SEED_FEATURES, device)
    feat = torch.rand(n, channels, generator=gf, device=device, dtype=torch.float32)
    rad = torch.full((n,), radius, dtype=torch.float32, device=device)
    return Cloud(pos, rad, feat, nrm)


def _split_bits(x: torch.Tensor) -> torch.Tensor:
    x = x & 0x1FFFFF
    x = (x | (x << 32)) & 0x1F00000000FFFF
    x = (x | (x << 16)) & 0x1F0000FF0000FF
    x = (x | (x << 8)) & 0x100F00F00F00F00F
    x = (x | (x << 4)) & 0x10C30C30C30C30C3
    x = (x | (x << 2)) & 0x1249249249249249
    return x


def morton_codes(pos: torch.Tensor) -> torch.Tensor:
    lo = pos.amin(dim=1, keepdim=True)
    hi = pos.amax(dim=1, keepdim=True)
    q = ((pos - lo) / (hi - lo).clamp_min(1e-30) * float((1 << 21) - 1)).to(torch.int64)
    return _split_bits(q[0]) | (_split_bits(q[1]) << 1) | (_split_bits(q[2]) << 2)


def blocked_morton_order(pos: torch.Tensor, block: int = 1024, seed: int = SEED_SCENE) -> torch.Tensor:
    """Permutation for the blocked Morton shuffle: Morton sort, then shuffle blocks."""
    n = pos.shape[1]
    order = torch.sort(morton_codes(pos), stable=True).indices
    nb = (n + block - 1) // block
    g = _gen(seed + 17, "cpu")
    bperm = torch.randperm(nb, generator=g).to(pos.device)
    starts = bperm * block
    lens = torch.clamp(n - starts, max=block)
    idx = torch.repeat_interleave(starts, lens) + _ragged_arange(lens)
    return order[idx]


def _ragged_arange(lens: torch.Tensor) -> torch.Tensor:
    total = int(lens.sum())
    offs = torch.cumsum(lens, 0) - lens
    return torch.arange(total, device=lens.device) - torch.repeat_interleave(offs, lens)


def apply_order(cloud: Cloud, perm: torch.Tensor) -> Cloud:
    return Cloud(cloud.pos[:, perm].contiguous(), cloud.radius[perm].contiguous(), cloud.feat[perm].contiguous(),
                 None if cloud.normal is None else cloud.normal[:, perm].contiguous())


# --------------------------------------------------------------------------- #
# Cameras and poses
# --------------------------------------------------------------------------- #
def pinhole(width: int, height: int, f: Optional[float] = None, cx: Optional[float] = None,
            cy: Optional[float] = None) -> Camera:
    f = width / 2.0 if f is None else f
    return Camera(width, height, PINHOLE, float(np.float32(f)), float(np.float32(f)),
                  float(np.float32(width / 2.0 if cx is None else cx)),
                  float(np.float32(height / 2.0 if cy is None else cy)))


def _radial64(k, r2):
    num = 1.0 + k[0] * r2 + k[1] * r2 ** 2 + k[2] * r2 ** 3
    den = 1.0 + k[3] * r2 + k[4] * r2 ** 2 + k[5] * r2 ** 3
    return num, den


def distortion_r2_max(cam: Camera, steps: int = 1 << 16) -> float:
    """Validity radius of the OpenCV rational model for this camera (R6).

    Scans r^2 in [0, 4 * corner r^2] in fp64 and stops where the denominator
    drops to 0.05 or the radial map rho * radial(rho^2) stops increasing.
    """
    corner = ((cam.width / 2.0) / cam.fx) ** 2 + ((cam.height / 2.0) / cam.fy) ** 2
    r2 = np.linspace(0.0, 4.0 * corner, steps + 1)
    num, den = _radial64(cam.k, r2)
    rho = np.sqrt(r2) * num / np.where(den == 0, 1e-300, den)
    bad = (den <= 0.05) | np.concatenate([[False], np.diff(rho) <= 0])
    last = int(np.argmax(bad)) - 1 if bad.any() else steps
    return float(np.float32(r2[max(last, 0)]))


def fisheye_camera(width: int, height: int, fov_deg: float = 180.0) -> Camera:
    """Equidistant fisheye (R35) whose image circle theta_max = fov/2 touches the shorter image side."""
    th = math.radians(fov_deg) / 2.0
    f = float(np.float32(min(width, height) / 2.0 / th))
    return Camera(width, height, FISHEYE, f, f, float(np.float32(width / 2.0)), float(np.float32(height / 2.0)),
                  r2_max=float(np.float32(th)))


def opencv_camera(width: int, height: int, seed: int = SEED_CAMERAS) -> Camera:
    rng = np.random.default_rng(seed)
    k = tuple(float(np.float32(v)) for v in rng.uniform(-0.1, 0.1, 6))
    p = tuple(float(np.float32(v)) for v in rng.uniform(-0.01, 0.01, 2))
    cam = pinhole(width, height)
    cam = dataclasses.replace(cam, model=OPENCV8, k=k, p=p)
    return dataclasses.replace(cam, r2_max=distortion_r2_max(cam))


def look_pose(center, R_cw) -> Pose:
    """world->camera pose from a camera centre and camera->world rotation."""
    R_cw = np.asarray(R_cw, dtype=np.float64)
    c = np.asarray(center, dtype=np.float64)
    R = R_cw.T
    t = -R @ c
    return Pose(R.astype(np.float32), t.astype(np.float32))


def tiny_pose() -> Pose:
    """BASELINE configs[0]: camera at z=-3 looking at the origin (+z), R = I, t = (0,0,3)."""
    return Pose(np.eye(3, dtype=np.float32), np.array([0.0, 0.0, 3.0], dtype=np.float32))


def _random_rotation(rng) -> np.ndarray:
    q = rng.normal(size=4)
    q /= np.linalg.norm(q)
    w, x, y, z = q
    return np.array([
        [1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w)],
        [2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w)],
        [2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)],
    ])


def room_poses(n_views: int, room: Room, seed: int = SEED_POSES) -> List[Pose]:
    rng = np.random.default_rng(seed)
    out = []
    S = room.size
    while len(out) < n_views:
        c = rng.uniform(-0.4 * S, 0.4 * S, 3)
        if np.any(np.linalg.norm(room.centers - c, axis=1) < room.radii + 0.025 * S):
            continue
        out.append(look_pose(c, _random_rotation(rng)))
    return out


# --------------------------------------------------------------------------- #
# Pyramid geometry helpers (sizes only; no method arithmetic)
# --------------------------------------------------------------------------- #
def layer_dims(width: int, height: int, layers: int):
    """(w_l, h_l, off_l) with w_l = ceil(w/2^l)."""
    dims, off = [], 0
    for l in range(layers):
        wl = (width + (1 << l) - 1) >> l
        hl = (height + (1 << l) - 1) >> l
        dims.append((wl, hl, off))
        off += wl * hl
    return dims, off


def grad_pyramid(n_views: int, channels: int, pixels: int, seed: int = SEED_GRADS, device="cpu") -> torch.Tensor:
    g = _gen(seed, device)
    return torch.rand(n_views, channels * pixels, generator=g, device=device, dtype=torch.float32) * 2.0 - 1.0


# --------------------------------------------------------------------------- #
# Workload presets (BASELINE.json configs[0..4])
# --------------------------------------------------------------------------- #
@dataclasses.dataclass
class Workload:
    name: str
    cloud: Cloud
    cameras: List[Camera]
    poses: List[Pose]
    params: Params
    backward: bool


def workload(idx: int, device="cpu", n: Optional[int] = None, n_views: Optional[int] = None,
             morton_block: int = 1024, shard: int = 0) -> Workload:
    """BASELINE.json configs[idx] with optional reduced n / views (for parity-size cases).

    shard > 0 draws a different cloud of the same room (the shard of rank `shard` in a point-sharded run)."""
    if idx == 0:
        n = 10_000 if n is None else n
        cloud = uniform_cube_cloud(n, 4, device=device)
        cam = pinhole(256, 256, f=200.0, cx=128.0, cy=128.0)
        return Workload("tiny", cloud, [cam], [tiny_pose()],
                        Params(layers=4, discard=False, ghost_rate=0.0), False)
    spec = {
        1: dict(n=1_000_000, C=4, S=10.0, w=1920, h=1080, model=PINHOLE, views=4, rho=0.0, bwd=False),
        2: dict(n=10_000_000, C=8, S=10.0, w=1920, h=1080, model=OPENCV8, views=1, rho=0.25, bwd=True),
        3: dict(n=100_000_000, C=4, S=50.0, w=1920, h=1080, model=PINHOLE, views=1, rho=0.0, bwd=False),
        4: dict(n=50_000_000, C=4, S=10.0, w=1024, h=1024, model=OPENCV8, views=16, rho=0.25, bwd=True),
    }[idx]
    n = spec["n"] if n is None else n
    V = spec["views"] if n_views is None else n_views
    room = make_room(spec["S"])
    cloud = room_cloud(n, room, spec["C"], seed=SEED_SCENE + 1000 * shard, device=device)
    if morton_block:
        cloud = apply_order(cloud, blocked_morton_order(cloud.pos, morton_block, seed=SEED_SCENE + shard))
    poses = room_poses(V, room)
    if spec["model"] == PINHOLE:
        cams = [pinhole(spec["w"], spec["h"]) for _ in range(V)]
    else:
        cams = [opencv_camera(spec["w"], spec["h"], seed=SEED_CAMERAS + v) for v in range(V)]
    params = Params(layers=5, discard=True, ghost_rate=spec["rho"])
    names = {1: "room1M_4view_fwd", 2: "room10M_C8_opencv_fwdbwd", 3: "room100M_fwd", 4: "room50M_16view_fwdbwd"}
    return Workload(names[idx], cloud, cams, poses, params, spec["bwd"])
