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

* Point sharding over peer memory (`PeerPointSharding`, `point_sharded_forward_p2p`): instead of two
  all-reduces of full private pyramids, every shard's depth pass min-reduces its keys and every blend
  sum-reduces its descriptors straight into ONE pyramid owned by one rank (CUDA IPC mapping; red.min /
  red.add over NVLink from inside the kernels), so each frame moves only the touched pixels and the
  exchange overlaps the kernels' own work; host barriers order the phases across ranks.

The functions only sequence collectives between phase calls: the phases themselves are the C-ABI
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


def min_depth_words(keys: torch.Tensor, group=None, scratch: torch.Tensor = None):
    """MIN all-reduce of only the 32-bit depth word (bits(z), the high word of every key, R8) -- half the bytes
    of the 64-bit key exchange (SURVEY §8(e) mitigation 3).  The blend and resolve read only the depth word
    (Eq. 6's min_z), so counts, sums and images equal the 64-bit exchange's; the low words (winner indices)
    stay each shard's local winners, i.e. the global winner index is not exchanged (verification-only)."""
    hi = keys.view(torch.int32)[1::2]  # little endian: word 1 of each key is bits(z)
    buf = torch.empty_like(hi) if scratch is None else scratch
    buf.copy_(hi)
    dist.all_reduce(buf, op=dist.ReduceOp.MIN, group=group)
    hi.copy_(buf)
    return buf


def point_sharded_forward(phases, pyramids: Sequence, group=None, keys32: bool = False):
    """phases.depth(); MIN(keys); phases.blend(); SUM(accum++count); phases.resolve().

    pyramids: objects with `.keys` (int64 tensor) and `.ac` (accum ++ count tensor) per view.
    keys32: exchange only the depth words (min_depth_words)."""
    phases.depth()
    for p in pyramids:
        if keys32:
            min_depth_words(p.keys, group)
        else:
            dist.all_reduce(p.keys, op=dist.ReduceOp.MIN, group=group)
    phases.blend()
    for p in pyramids:
        dist.all_reduce(p.ac, op=dist.ReduceOp.SUM, group=group)
    phases.resolve()


def pixel_chunk(P: int, world: int, align: int = 4) -> int:
    """Pixels per rank of the reduce-scatter: ceil(P / world) rounded up to `align` (the resolve's vector width)."""
    return max(align, -(-(-(-P // world)) // align) * align)


def pixel_range(P: int, world: int, rank: int, align: int = 4) -> Tuple[int, int]:
    """Slice [a, b) of a view's P pyramid pixels that `rank` receives and resolves (equal chunks of
    pixel_chunk pixels; the last is shorter or empty)."""
    c = pixel_chunk(P, world, align)
    return min(P, rank * c), min(P, (rank + 1) * c)


def reduce_scatter_accum(pyramids: Sequence, group=None, scratch=None) -> Tuple[int, int]:
    """The SUM exchange of point_sharded_forward_rs: accum and count of every view packed rank-major
    ([rank][accum slice | count slice]) and reduce-scattered in one collective per view; this rank's slice of
    its own accum / count then holds the global sums.  Returns the rank's (a, b) pixel slice."""
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    P = pyramids[0].count.numel()
    C = pyramids[0].accum.numel() // P
    ch = pixel_chunk(P, world)
    full = P // ch  # ranks whose slice is a whole chunk
    a, b = pixel_range(P, world, rank)
    for p in pyramids:
        acc, cnt = p.accum, p.count
        n = world * ch * (C + 1)
        buf = torch.zeros(n, dtype=acc.dtype, device=acc.device) if scratch is None else scratch[:n]
        if scratch is not None:
            buf.zero_()
        rows = buf.view(world, ch * (C + 1))
        if full:
            rows[:full, : ch * C].copy_(acc[: full * ch * C].view(full, ch * C))
            rows[:full, ch * C:].copy_(cnt[: full * ch].view(full, ch))
        if full < world and full * ch < P:  # the short last slice
            t = P - full * ch
            rows[full, : t * C].copy_(acc[full * ch * C:])
            rows[full, ch * C: ch * C + t].copy_(cnt[full * ch:])
        out = torch.empty(ch * (C + 1), dtype=acc.dtype, device=acc.device)
        dist.reduce_scatter_tensor(out, buf, op=dist.ReduceOp.SUM, group=group)
        if a < b:
            acc[a * C: b * C].copy_(out[: (b - a) * C])
            cnt[a:b].copy_(out[ch * C: ch * C + (b - a)])
    return a, b


def point_sharded_forward_rs(phases, pyramids: Sequence, group=None, keys32: bool = False, scratch=None):
    """Point sharding with a reduce-scatter instead of the SUM all-reduce: phases.depth();
    MIN(keys); phases.blend(); accum and count are packed rank-major ([rank][accum slice | count slice], one
    copy per part) and reduce-scattered in ONE collective -- (G-1)/G of the all-reduce's bus traffic -- so rank
    r holds the sums of its pixel slice (pixel_range); phases.resolve_range(a_r, b_r) writes that slice of the
    image, which stays distributed by pixel slice.  Forward only: outside its slice a rank's accum / count
    are its shard's partial sums (like the peer-memory mode's non-owners, it must not run a backward).

    pyramids: objects with `.keys`, `.accum` ([P * C] view) and `.count` ([P] view) per view.
    scratch: optional flat buffer of >= world * pixel_chunk(P, world) * (C + 1) elements (allocated if None).
    Returns this rank's (a, b) pixel slice."""
    phases.depth()
    for p in pyramids:
        if keys32:
            min_depth_words(p.keys, group)
        else:
            dist.all_reduce(p.keys, op=dist.ReduceOp.MIN, group=group)
    phases.blend()
    a, b = reduce_scatter_accum(pyramids, group, scratch)
    phases.resolve_range(a, b)
    return a, b


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


def point_sharded_forward_p2p(phases, owner: int, group=None):
    """One frame of point sharding over a shared (peer-memory) pyramid: the owner resets it; every shard's
    depth pass min-reduces into it; after all of them, every shard's blend sum-reduces into it; after all
    of those the owner resolves.  Each step ends with the rank's stream synchronized and a barrier."""
    rank = dist.get_rank()
    if rank == owner:
        phases.clear()
    phases.sync()
    dist.barrier(group=group)
    phases.depth()
    phases.sync()
    dist.barrier(group=group)
    phases.blend()
    phases.sync()
    dist.barrier(group=group)
    if rank == owner:
        phases.resolve()


class PeerPointSharding:
    """Points the renderer of this rank (its shard, with its global_offset) at the owner's pyramid: the
    owner exports the keys / accum / count allocations (adop_ipc_export), the others map them
    (adop_ipc_open; peer access over NVLink between GPUs) and render into them with
    adop_params.shared_pyramid = 1.  Non-owners keep their own image buffer (only the owner resolves), so the
    p2p path is forward-only on them: a backward there raises (the owner's backward is a normal one)."""

    def __init__(self, renderer, owner: int = 0, group=None):
        from . import adop as A
        self.r = renderer
        self.owner = owner
        rank = dist.get_rank()
        renderer.params.s.shared_pyramid = 1
        obj = [None]
        if rank == owner:
            obj = [[(A.ipc_export(p.keys), A.ipc_export(p.accum), A.ipc_export(p.count)) for p in renderer.pyrs]]
        dist.broadcast_object_list(obj, src=owner, group=group)
        if rank != owner:
            self.own = renderer.pyrs  # keeps this rank's (unused) buffers alive for the image pointer
            renderer.pyrs = [A.PeerPyramid(A.ipc_open(*k), A.ipc_open(*a), A.ipc_open(*c), p.image.data_ptr(),
                                           p.width, p.height, p.layers)
                             for (k, a, c), p in zip(obj[0], self.own)]
            renderer._c = None  # the cached marshalled call holds the old pyramid pointers
            # forward-only on non-owners: their image buffer is never resolved (only the owner resolves), and
            # the backward reads the image (pixel tables, Eq. 11's I_q): Renderer.backward refuses
            renderer.peer_non_owner = True

    def close(self):
        from . import adop as A
        if dist.get_rank() != self.owner:
            A.ipc_close_all()


class CudaPhases:
    """The C-ABI phases of one rank (paper_2110_06635_b200.adop) bound to its buffers."""

    def __init__(self, renderer, grads: Sequence[torch.Tensor] = ()):
        self.r = renderer
        self.grads = list(grads)

    def depth(self):
        from . import adop as A
        r = self.r
        A.forward_depth(r.points, r.cams, r.poses, r.params, r.pyrs, r.ws, call=r._call())

    def blend(self):
        from . import adop as A
        r = self.r
        A.forward_blend(r.points, r.cams, r.poses, r.params, r.pyrs, r.ws, call=r._call())

    def resolve(self):
        from . import adop as A
        r = self.r
        A.forward_resolve(r.points, r.cams, r.poses, r.params, r.pyrs, r.ws, call=r._call())

    def resolve_range(self, p0: int, p1: int):
        from . import adop as A
        r = self.r
        A.forward_resolve_range(r.points, r.cams, r.poses, r.params, r.pyrs, r.ws, p0, p1, call=r._call())

    def clear(self):
        from . import adop as A
        r = self.r
        A.clear_pyramid(r.cams, r.params.layers, r.C, r.pyrs)

    def sync(self):
        torch.cuda.current_stream().synchronize()

    def forward(self):
        self.r.forward()

    def backward(self):
        self.r.backward(self.grads)


def grad_buffer(n: int, channels: int, device) -> Tuple[torch.Tensor, torch.Tensor, torch.Tensor]:
    """One buffer for the SUM all-reduce of view sharding: returns (buf, d_feat [n][C], d_pos [3][n])."""
    buf = torch.zeros(n * channels + 3 * n, dtype=torch.float32, device=device)
    return buf, buf[: n * channels].view(n, channels), buf[n * channels:].view(3, n)
