"""Multi-GPU orchestration of the rasterizer over torch.distributed (NCCL on the B200 box, gloo in CPU tests).

The paper is single-GPU.  The north star adds two partitionings:

* Point sharding (huge clouds; BASELINE configs[3]): rank r owns a contiguous chunk of the blocked-Morton
  ordered cloud with global indices [offset_r, offset_r + n_r).  Forward = phase 1 into a full local key
  pyramid -> MIN all-reduce of the 64-bit keys (exact global depth winners, R8 makes the int64 order equal
  the uint64 order) -> phase 2 against the global keys -> SUM all-reduce of accum++count (one buffer) ->
  phase 3.  Backward (if used) runs per shard against the reduced pyramid; d_pose partials are summed.
* View sharding (training batches; BASELINE configs[4]): rank r owns a contiguous range of views of the
  batch (view_id_base keeps the per-(view, point) discard draws identical to the unsharded batch) and the
  whole cloud; after the backward the point gradients d_feat ++ d_pos are SUM all-reduced in one buffer,
  d_pose rows are all-gathered.

Both functions only sequence collectives between phase calls: the phases themselves are the C-ABI
entry points (CudaPhases) -- or any object with the same methods (the CPU tests plug the oracle's
phase functions in to check this host logic with world_size 2 on gloo).
"""
from __future__ import annotations

from typing import List, Sequence, Tuple

import torch
import torch.distributed as dist


def shard_range(n: int, world: int, rank: int, align: int = 1024) -> Tuple[int, int]:
    """Contiguous chunk [a, b) of n points for `rank`, cut at multiples of `align` (Morton blocks)."""
    blocks = (n + align - 1) // align
    per = blocks // world
    extra = blocks % world
    a_blk = rank * per + min(rank, extra)
    b_blk = a_blk + per + (1 if rank < extra else 0)
    return min(n, a_blk * align), min(n, b_blk * align)


def view_range(n_views: int, world: int, rank: int) -> Tuple[int, int]:
    per = n_views // world
    extra = n_views % world
    a = rank * per + min(rank, extra)
    return a, a + per + (1 if rank < extra else 0)


def point_sharded_forward(phases, pyramids: Sequence, group=None):
    """phases.depth(); MIN(keys); phases.blend(); SUM(accum++count); phases.resolve().

    pyramids: objects with `.keys` (int64 tensor) and `.ac` (accum ++ count tensor) per view."""
    phases.depth()
    for p in pyramids:
        dist.all_reduce(p.keys, op=dist.ReduceOp.MIN, group=group)
    phases.blend()
    for p in pyramids:
        dist.all_reduce(p.ac, op=dist.ReduceOp.SUM, group=group)
    phases.resolve()


def point_sharded_backward(phases, d_pose: torch.Tensor, group=None):
    """Per-shard backward against the reduced pyramid; point gradients stay with their shard, the
    per-view pose gradient is the sum over shards."""
    phases.backward()
    dist.all_reduce(d_pose, op=dist.ReduceOp.SUM, group=group)


def view_sharded_step(phases, grad_points: torch.Tensor, d_pose_local: torch.Tensor, n_views_total: int,
                      group=None) -> torch.Tensor:
    """Forward + backward of this rank's views, then SUM of the point gradients (grad_points is one
    buffer holding d_feat ++ d_pos) and an all-gather of the per-view pose gradients.
    Returns d_pose for all views [n_views_total, 6]."""
    phases.forward()
    phases.backward()
    dist.all_reduce(grad_points, op=dist.ReduceOp.SUM, group=group)
    world = dist.get_world_size(group)
    counts = [view_range(n_views_total, world, r) for r in range(world)]
    width = max(b - a for a, b in counts)
    buf = torch.zeros(width, 6, dtype=d_pose_local.dtype, device=d_pose_local.device)
    buf[: d_pose_local.shape[0]] = d_pose_local
    gathered = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(gathered, buf, group=group)
    return torch.cat([g[: b - a] for g, (a, b) in zip(gathered, counts)], dim=0)


class CudaPhases:
    """The C-ABI phases of one rank (paper_2110_06635_b200.adop) bound to its buffers."""

    def __init__(self, renderer, grads: Sequence[torch.Tensor] = ()):
        self.r = renderer
        self.grads = list(grads)

    def depth(self):
        from . import adop as A
        r = self.r
        A.forward_depth(r.points, r.cams, r.poses, r.params, r.pyrs, r.ws)

    def blend(self):
        from . import adop as A
        r = self.r
        A.forward_blend(r.points, r.cams, r.poses, r.params, r.pyrs, r.ws)

    def resolve(self):
        from . import adop as A
        r = self.r
        A.forward_resolve(r.points, r.cams, r.poses, r.params, r.pyrs, r.ws)

    def forward(self):
        self.r.forward()

    def backward(self):
        self.r.backward(self.grads)


def grad_buffer(n: int, channels: int, device) -> Tuple[torch.Tensor, torch.Tensor, torch.Tensor]:
    """One buffer for the SUM all-reduce of view sharding: returns (buf, d_feat [n][C], d_pos [3][n])."""
    buf = torch.zeros(n * channels + 3 * n, dtype=torch.float32, device=device)
    return buf, buf[: n * channels].view(n, channels), buf[n * channels:].view(3, n)
