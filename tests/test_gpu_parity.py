"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle, element by element.

Marked gpu: run on the B200 box (pytest -m gpu).  Keys, counts and masks must be bit-exact; floating
outputs within the tolerances documented in tests/parity.py.
"""
import dataclasses
import math

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2110_06635_b200 import adop as A
from paper_2110_06635_b200 import scene as S

from .parity import compare_backward, compare_forward, grads_for, keys_u64, run_gpu, run_oracle

pytestmark = pytest.mark.gpu


def test_tiny_config_forward():
    w = S.workload(0)
    r = run_gpu(w.cloud, w.cameras, w.poses, w.params)
    _, fwd, _ = run_oracle(w.cloud, w.cameras, w.poses, w.params)
    compare_forward(r, fwd, ctx="tiny")
    assert (fwd.count > 0).sum() > 1000


def test_tiny_config_with_discard_ghosts_background_and_backward():
    w = S.workload(0)
    prm = dataclasses.replace(w.params, discard=True, ghost_rate=0.3, background=[0.1, 0.2, 0.3, 0.4])
    cloud = dataclasses.replace(w.cloud, radius=torch.full_like(w.cloud.radius, 0.02))
    G = grads_for(w.cameras, prm.layers, 4)
    r = run_gpu(cloud, w.cameras, w.poses, prm, grads=G)
    _, fwd, bwd = run_oracle(cloud, w.cameras, w.poses, prm, grads=G)
    compare_forward(r, fwd, ctx="tiny+")
    compare_backward(r, bwd, ctx="tiny+")
    assert np.abs(bwd.dx).sum() > 0 and np.abs(bwd.dtau).sum() > 0


@pytest.mark.parametrize("idx,n,views", [(1, 200_000, 4), (2, 200_000, 1), (4, 60_000, 16)])
def test_room_configs_reduced(idx, n, views):
    """configs[1], [2], [4] at reduced N (full camera, layers, C, views): several tiles + ragged tails."""
    w = S.workload(idx, n=n + 13, n_views=views)
    G = grads_for(w.cameras, w.params.layers, w.cloud.channels) if w.backward else None
    r = run_gpu(w.cloud, w.cameras, w.poses, w.params, grads=G)
    _, fwd, bwd = run_oracle(w.cloud, w.cameras, w.poses, w.params, grads=G)
    compare_forward(r, fwd, ctx=w.name)
    if G is not None:
        compare_backward(r, bwd, ctx=w.name)
    assert (fwd.count > 0).sum() > 10_000


@pytest.mark.parametrize("C,ghost", [(1, 0.0), (3, 0.25), (8, 0.5), (5, 0.1)])
def test_channels_scalar_path_uniform_radius(C, ghost):
    """generic C, the unaligned (scalar-load) path via an odd row stride, radius=NULL."""
    room = S.make_room(6.0)
    base = S.room_cloud(40_003, room, C, seed=31)
    stride = base.n + 3
    pos = torch.zeros(3, stride)
    pos[:, :base.n] = base.pos
    cams = [S.opencv_camera(320, 200, seed=7), S.opencv_camera(320, 200, seed=8)]
    cams = [dataclasses.replace(c, fx=160.0, fy=160.0) for c in cams]
    cams = [dataclasses.replace(c, r2_max=S.distortion_r2_max(c)) for c in cams]
    poses = S.room_poses(2, room, seed=2)
    prm = S.Params(layers=4, discard=True, ghost_rate=ghost, seed=99, view_id_base=3)
    dev = torch.device("cuda")
    pts = A.Points(pos.to(dev), None, base.feat.to(dev), global_offset=1234, radius_uniform=0.02, n=base.n)
    ap = A.Params(prm, C)
    pyrs = A.alloc_pyramids(cams, prm.layers, C, dev)
    ws = A.Workspace(pts, cams, ap, dev)
    A.rasterize_forward(pts, cams, poses, ap, pyrs, ws)
    G = grads_for(cams, prm.layers, C)
    d_feat = torch.empty(base.n, C, device=dev)
    d_pos = torch.empty(3, base.n, device=dev)
    d_pose = torch.empty(2, 6, dtype=torch.float64, device=dev)
    A.rasterize_backward(pts, cams, poses, ap, pyrs, [g.to(dev) for g in G], ws, d_feat, d_pos, d_pose)
    torch.cuda.synchronize()
    opts = O.Points(pos.numpy(), None, base.feat.numpy(), 1234, radius_uniform=0.02)
    opts.n = base.n
    opts.s.n, opts.s.pos_stride = base.n, stride
    fwd = O.forward(opts, cams, poses, prm)
    bwd = O.backward(opts, cams, poses, prm, fwd, np.stack([g.numpy() for g in G]))

    class R:
        pass
    r = R()
    r.pyrs, r.d_feat, r.d_pos, r.d_pose = pyrs, d_feat, d_pos, d_pose
    compare_forward(r, fwd, ctx=f"C={C}")
    compare_backward(r, bwd, ctx=f"C={C}")


def test_point_masks_bitexact():
    w = S.workload(2, n=150_001)
    prm = dataclasses.replace(w.params, ghost_rate=0.25)
    dev = torch.device("cuda")
    r = A.Renderer(w.cloud.to(dev), w.cameras, w.poses, prm)
    m = r.masks().cpu().numpy()
    mo = O.point_masks(O.Points.from_cloud(w.cloud), w.cameras, w.poses, prm)
    assert np.array_equal(m, mo), np.nonzero(m != mo)
    assert (mo & 0x1F).any() and (mo & 0x80).any()


def test_empty_cloud():
    cam = S.pinhole(64, 48)
    cloud = S.Cloud(torch.zeros(3, 0), torch.zeros(0), torch.zeros(0, 4))
    prm = S.Params(layers=3, background=[1.0, 2.0, 3.0, 4.0])
    G = grads_for([cam], 3, 4)
    r = run_gpu(cloud, [cam], [S.tiny_pose()], prm, grads=G)
    _, fwd, bwd = run_oracle(cloud, [cam], [S.tiny_pose()], prm, grads=G)
    compare_forward(r, fwd, ctx="empty")
    assert (keys_u64(r.pyrs[0].keys) == np.uint64(A.SENTINEL)).all()
    assert not r.d_pose.cpu().numpy().any()


def test_record_overflow_falls_back_to_restreaming():
    w = S.workload(1, n=100_000, n_views=2)
    r = run_gpu(w.cloud, w.cameras, w.poses, w.params, record_capacity=1000)
    rec, of = r.ws.stats()
    assert of and rec <= 1024  # only the successful (prefix) reservations count (capacity: whole 64-slot chunks)
    _, fwd, _ = run_oracle(w.cloud, w.cameras, w.poses, w.params)
    compare_forward(r, fwd, ctx="overflow")
    r2 = run_gpu(w.cloud, w.cameras, w.poses, w.params)
    rec2, of2 = r2.ws.stats()
    assert not of2 and rec2 > 1000  # slot counts vary with the dynamic tile schedule (dead chunk tails)


def test_backward_null_outputs():
    """Any of d_feat / d_pos / d_pose / d_intrinsics may be NULL (include/adop.h); the others are unchanged."""
    w = S.workload(2, n=60_000)
    dev = torch.device("cuda")
    G = [g.to(dev) for g in grads_for(w.cameras, w.params.layers, w.cloud.channels)]
    r = A.Renderer(w.cloud.to(dev), w.cameras, w.poses, w.params, intrinsics=True)
    r.forward()
    f1, p1, q1 = [t.clone() for t in r.backward(G)]
    i1 = r.d_intr.clone()
    assert i1[:, 4:].abs().sum() > 0  # OpenCV8 camera: distortion terms present
    for drop in range(4):
        outs = [torch.full_like(t, 7.0) for t in (f1, p1, q1, i1)]
        args = [None if k == drop else outs[k] for k in range(4)]
        A.rasterize_backward(r.points, r.cams, r.poses, r.params, r.pyrs, G, r.ws, *args)
        torch.cuda.synchronize()
        for k, ref in enumerate((f1, p1, q1, i1)):
            if k == drop:
                assert (outs[k] == 7.0).all()
            else:
                torch.testing.assert_close(outs[k], ref, rtol=1e-5, atol=1e-6)


def test_grad_accumulate_adds():
    w = S.workload(2, n=50_000)
    dev = torch.device("cuda")
    G = [g.to(dev) for g in grads_for(w.cameras, w.params.layers, w.cloud.channels)]
    r = A.Renderer(w.cloud.to(dev), w.cameras, w.poses, w.params)
    r.forward()
    f1, p1, q1 = [t.clone() for t in r.backward(G)]
    r.params.s.grad_accumulate = 1
    r.backward(G)
    torch.cuda.synchronize()
    torch.testing.assert_close(r.d_feat, 2 * f1)
    torch.testing.assert_close(r.d_pos, 2 * p1)
    torch.testing.assert_close(r.d_pose, 2 * q1)


def test_intrinsics_gradient_pinhole_zero_distortion_terms():
    """NEXT-1 on a pinhole camera: the 8 distortion entries are exactly 0, the rest match the oracle."""
    w = S.workload(1, n=120_000, n_views=2)
    prm = dataclasses.replace(w.params, ghost_rate=0.25)
    G = grads_for(w.cameras, prm.layers, w.cloud.channels)
    r = run_gpu(w.cloud, w.cameras, w.poses, prm, grads=G)
    _, fwd, bwd = run_oracle(w.cloud, w.cameras, w.poses, prm, grads=G)
    assert (r.d_intr[:, 4:] == 0).all() and r.d_intr[:, :4].abs().sum() > 0
    compare_backward(r, bwd, ctx="pinhole intrinsics")


def test_phase_split_point_sharding_on_one_gpu():
    """The point-sharded forward (§8e): each shard runs phase 1 into its own keys, keys are min-reduced,
    each shard runs phase 2 against the global keys, accum/count are sum-reduced, then phase 3.  Done here
    with 3 shards on one GPU and torch.minimum / + in place of the collectives: keys must equal the
    unsharded run bit for bit."""
    w = S.workload(1, n=120_000, n_views=2)
    dev = torch.device("cuda")
    cloud = w.cloud.to(dev)
    C = cloud.channels
    ap = A.Params(w.params, C)
    full = A.Renderer(cloud, w.cameras, w.poses, w.params)
    full.forward()
    bounds = [0, 37_001, 80_000, cloud.n]
    shards = []
    for a, b in zip(bounds, bounds[1:]):
        pts = A.Points.from_cloud(cloud.slice(a, b), global_offset=a)
        pyrs = A.alloc_pyramids(w.cameras, w.params.layers, C, dev)
        ws = A.Workspace(pts, w.cameras, ap, dev)
        A.forward_depth(pts, w.cameras, w.poses, ap, pyrs, ws)
        shards.append((pts, pyrs, ws))
    for v in range(2):
        kmin = torch.stack([s[1][v].keys for s in shards]).amin(0)
        for s in shards:
            s[1][v].keys.copy_(kmin)
    for pts, pyrs, ws in shards:
        A.forward_blend(pts, w.cameras, w.poses, ap, pyrs, ws)
    for v in range(2):
        tot = torch.stack([s[1][v].ac for s in shards]).sum(0)
        for s in shards:
            s[1][v].ac.copy_(tot)
    pts0, pyrs0, ws0 = shards[0]
    A.forward_resolve(pts0, w.cameras, w.poses, ap, pyrs0, ws0)
    torch.cuda.synchronize()
    for v in range(2):
        assert torch.equal(pyrs0[v].keys, full.pyrs[v].keys)
        assert torch.equal(pyrs0[v].count, full.pyrs[v].count)
        torch.testing.assert_close(pyrs0[v].image, full.pyrs[v].image, rtol=1e-5, atol=1e-6)


def _image_idx(width, height, layers, C, p0, p1, device):
    """Indices into the planar layer-concatenated image of pyramid pixels [p0, p1) (include/adop.h layout)."""
    out, off = [], 0
    for l in range(layers):
        wl, hl = -(-width // (1 << l)), -(-height // (1 << l))
        hw = wl * hl
        a, b = max(p0, off), min(p1, off + hw)
        if a < b:
            for c in range(C):
                out.append(torch.arange(C * off + c * hw + (a - off), C * off + c * hw + (b - off), device=device))
        off += hw
    return torch.cat(out) if out else torch.empty(0, dtype=torch.int64, device=device)


def test_resolve_range_matches_full_resolve():
    """adop_forward_resolve_range: the vector path (ends at multiples of 4), the scalar path (odd ends) and the
    empty range write exactly the full resolve's values on their pixels and leave the rest untouched."""
    w = S.workload(1, n=120_000, n_views=2)
    r = run_gpu(w.cloud, w.cameras, w.poses, w.params)
    cam, L, C = w.cameras[0], w.params.layers, w.cloud.channels
    P = r.pyrs[0].count.numel()
    full = [p.image.clone() for p in r.pyrs]
    for p0, p1 in ((0, P), (4, 2_000_004), (7, 1_234_567), (P - 5, P + 100), (11, 11)):
        for p in r.pyrs:
            p.image.fill_(-7.0)
        A.forward_resolve_range(r.points, r.cams, r.poses, r.params, r.pyrs, r.ws, p0, p1)
        torch.cuda.synchronize()
        idx = _image_idx(cam.width, cam.height, L, C, p0, min(p1, P), r.pyrs[0].image.device)
        for v in range(2):
            img = r.pyrs[v].image
            assert torch.equal(img[idx], full[v][idx]), (p0, p1)
            mask = torch.ones_like(img, dtype=torch.bool)
            mask[idx] = False
            assert bool((img[mask] == -7.0).all()), (p0, p1)
    with pytest.raises(RuntimeError):
        A.forward_resolve_range(r.points, r.cams, r.poses, r.params, r.pyrs, r.ws, 10, 5)


def test_reduce_scatter_point_sharding_on_one_gpu():
    """Point sharding with a reduce-scatter (parallel.point_sharded_forward_rs, §8e) on one GPU: 3 shards,
    keys min-combined, each shard r receives the sums of ITS pixel slice only and resolves it with
    adop_forward_resolve_range; the slices together equal the unsharded forward (counts exact, image within
    the fp32 summation tolerance)."""
    from paper_2110_06635_b200 import parallel as PL
    w = S.workload(1, n=120_000, n_views=2)
    dev = torch.device("cuda")
    cloud = w.cloud.to(dev)
    C = cloud.channels
    ap = A.Params(w.params, C)
    full = A.Renderer(cloud, w.cameras, w.poses, w.params)
    full.forward()
    bounds = [0, 37_001, 80_000, cloud.n]
    G = len(bounds) - 1
    shards = []
    for a, b in zip(bounds, bounds[1:]):
        pts = A.Points.from_cloud(cloud.slice(a, b), global_offset=a)
        pyrs = A.alloc_pyramids(w.cameras, w.params.layers, C, dev)
        ws = A.Workspace(pts, w.cameras, ap, dev)
        A.forward_depth(pts, w.cameras, w.poses, ap, pyrs, ws)
        shards.append((pts, pyrs, ws))
    for v in range(2):
        kmin = torch.stack([s[1][v].keys for s in shards]).amin(0)
        for s in shards:
            s[1][v].keys.copy_(kmin)
    for pts, pyrs, ws in shards:
        A.forward_blend(pts, w.cameras, w.poses, ap, pyrs, ws)
    P = shards[0][1][0].count.numel()
    ranges = [PL.pixel_range(P, G, r) for r in range(G)]
    for v in range(2):  # the reduce to rank r of slice r (accum and count), as the NCCL reduces do
        for r, (a, b) in enumerate(ranges):
            shards[r][1][v].accum[a * C:b * C] = torch.stack([s[1][v].accum[a * C:b * C] for s in shards]).sum(0)
            shards[r][1][v].count[a:b] = torch.stack([s[1][v].count[a:b] for s in shards]).sum(0)
    for r, (a, b) in enumerate(ranges):
        pts, pyrs, ws = shards[r]
        A.forward_resolve_range(pts, w.cameras, w.poses, ap, pyrs, ws, a, b)
    torch.cuda.synchronize()
    cam = w.cameras[0]
    assert ranges[0][0] == 0 and ranges[-1][1] == P and all(a % 4 == 0 for a, _ in ranges)
    for r, (a, b) in enumerate(ranges):
        idx = _image_idx(cam.width, cam.height, w.params.layers, C, a, b, dev)
        for v in range(2):
            assert torch.equal(shards[r][1][v].count[a:b], full.pyrs[v].count[a:b])
            torch.testing.assert_close(shards[r][1][v].image[idx], full.pyrs[v].image[idx], rtol=1e-5, atol=1e-6)


def test_view_id_base_matches_per_view_calls():
    """beta is keyed by the global view id: rendering views 2..3 of a batch alone (view_id_base=2)
    gives the same pyramids as the 4-view call (view sharding)."""
    w = S.workload(1, n=80_000, n_views=4)
    allv = run_gpu(w.cloud, w.cameras, w.poses, w.params)
    part = run_gpu(w.cloud, w.cameras[2:], w.poses[2:], dataclasses.replace(w.params, view_id_base=2))
    for j in range(2):
        assert torch.equal(part.pyrs[j].keys, allv.pyrs[2 + j].keys)
        assert torch.equal(part.pyrs[j].image, allv.pyrs[2 + j].image) or torch.allclose(
            part.pyrs[j].image, allv.pyrs[2 + j].image, rtol=1e-5, atol=1e-6)


# --------------------------------------------------------------------------- #
# full BASELINE sizes, in the launch configuration bench.py times
# --------------------------------------------------------------------------- #
def _cloud_on_gpu(idx, **kw):
    return S.workload(idx, device="cuda", **kw)


def test_full_config3_100M_forward_vs_oracle():
    """configs[3] (the bench workload): 100M points, 5 layers, 1080p, discard on: full oracle compare."""
    w = _cloud_on_gpu(3)
    r = A.Renderer(w.cloud, w.cameras, w.poses, w.params)
    r.forward()
    torch.cuda.synchronize()
    rec, of = r.ws.stats()
    assert not of and rec > 0
    _, fwd, _ = run_oracle(w.cloud.to("cpu"), w.cameras, w.poses, w.params)
    compare_forward(r, fwd, ctx="config3-full")


def test_full_config2_10M_fwd_bwd_vs_oracle():
    w = _cloud_on_gpu(2)
    G = grads_for(w.cameras, w.params.layers, w.cloud.channels)
    r = A.Renderer(w.cloud, w.cameras, w.poses, w.params, intrinsics=True)
    r.forward()
    r.backward([g.cuda() for g in G])
    torch.cuda.synchronize()
    _, fwd, bwd = run_oracle(w.cloud.to("cpu"), w.cameras, w.poses, w.params, grads=G)
    compare_forward(r, fwd, ctx="config2-full")
    compare_backward(r, bwd, ctx="config2-full")


def test_full_config4_50M_16views_fwd_bwd_vs_oracle():
    """configs[4]: 50M points x 16 views 1024^2 OpenCV8 in ONE fused forward + backward (as bench times it)
    against the (OpenMP) oracle on the same inputs: keys and counts of all 16 views bit-exact, images, and the
    full backward -- d_feat, d_pos of all 50M points, d_pose and d_intrinsics of all 16 views."""
    w = _cloud_on_gpu(4)
    C = w.cloud.channels
    G = grads_for(w.cameras, w.params.layers, C)
    r = A.Renderer(w.cloud, w.cameras, w.poses, w.params, intrinsics=True)
    r.forward()
    r.backward([g.cuda() for g in G])
    torch.cuda.synchronize()
    _, fwd, bwd = run_oracle(w.cloud.to("cpu"), w.cameras, w.poses, w.params, grads=G)
    compare_forward(r, fwd, ctx="config4-full")
    compare_backward(r, bwd, ctx="config4-full")
    assert np.count_nonzero(np.abs(bwd.dx).sum(0)) > 1_000_000


@pytest.mark.parametrize("model,tight", [(S.PINHOLE, False), (S.OPENCV8, False), (S.PINHOLE, True),
                                         (S.OPENCV8, True)])
def test_precull_is_conservative_at_frustum_borders(model, tight):
    """Adversarial points around every layer's bounds (u0 near -2^(l-1) and w_l*2^l) and at tiny /
    huge depths: the GPU's division-free pre-culls (per point, and per 128-point warp box) must never
    reject a point the exact test keeps.  tight=True makes every warp tile a cluster of 128 jittered
    copies of one border point, so the warp-box test sits exactly on the border."""
    rng = np.random.default_rng(17)
    w, h, f = 64, 48, 40.0
    cam = S.Camera(w, h, S.PINHOLE, f, f, 32.0, 24.0)
    if model == S.OPENCV8:
        cam = dataclasses.replace(cam, model=S.OPENCV8, k=(0.01, -0.02, 0.0, 0.005, 0.0, 0.0), p=(0.001, -0.001))
        cam = dataclasses.replace(cam, r2_max=S.distortion_r2_max(cam))
    us = np.concatenate([np.arange(-20, w + 20, 0.25), -0.5 * 2.0 ** np.arange(5), w - 0.5 + np.zeros(5)])
    vs = np.concatenate([np.arange(-20, h + 20, 0.5), -0.5 * 2.0 ** np.arange(5)])
    zs = np.array([1e-4, 1e-2, 0.5, 3.0, 1e3, 1e6])
    U, Vv, Z = [a.ravel() for a in np.meshgrid(us, vs[::3], zs)]
    U = U + rng.choice([-1e-4, 0, 1e-4], U.shape)
    X = (U - cam.cx) / f * Z
    Y = (Vv - cam.cy) / f * Z
    xyz = np.stack([X, Y, Z]).astype(np.float32)
    if tight:
        sel = rng.choice(xyz.shape[1], 400, replace=False)
        base = np.repeat(xyz[:, sel], 128, axis=1).astype(np.float64)
        jit = 1.0 + rng.uniform(-2e-7, 2e-7, base.shape)
        xyz = (base * jit).astype(np.float32)
    n = xyz.shape[1]
    cloud = S.Cloud(torch.from_numpy(xyz), torch.full((n,), 0.01), torch.rand(n, 4, generator=torch.Generator().manual_seed(1)))
    prm = S.Params(layers=5, discard=False)
    r = run_gpu(cloud, [cam], [S.Pose(np.eye(3, dtype=np.float32), np.zeros(3, dtype=np.float32))], prm)
    _, fwd, _ = run_oracle(cloud, [cam], [S.Pose(np.eye(3, dtype=np.float32), np.zeros(3, dtype=np.float32))], prm)
    compare_forward(r, fwd, ctx="precull")
    assert (fwd.count > 0).sum() > (50 if tight else 500)


def _hdr(ws):
    """WsHeader fields (adop_internal.h): resv u64 @0, overflow i32 @8, mode i32 @12, tag u64 @16,
    front_ok u64 @24, back_ok u64 @32, tiles_read / tiles_fwd / tiles_bwd u64 @40..64, ghosts_fwd i32 @64."""
    off = ws.ptr - ws.buf.data_ptr()
    h = ws.buf[off:off + 72].cpu().numpy()
    u = lambda a, b: int(h[a:b].view(np.uint64)[0])
    return {"resv": u(0, 8), "overflow": int(h[8:12].view(np.int32)[0]), "mode": int(h[12:16].view(np.int32)[0]),
            "tag": u(16, 24), "front_ok": u(24, 32), "back_ok": u(32, 40),
            "ghosts_fwd": int(h[64:68].view(np.int32)[0])}


def _set_hdr_i32(ws, byte_off, value):
    off = ws.ptr - ws.buf.data_ptr() + byte_off
    ws.buf[off:off + 4] = torch.from_numpy(np.array([value], dtype=np.int32).view(np.uint8)).to(ws.buf.device)


@pytest.mark.parametrize("idx,n,views,cap", [(2, 120_000, None, 3000), (4, 60_000, 16, 8192)])
def test_backward_work_lists_overflow_to_inline(idx, n, views, cap):
    """A record region far too small for the survivors: the forward overflows (blend re-streams), the
    backward re-renders and its texture/ghost work lists overflow almost at once, so the sweep
    processes the rest inline -- same results.  The 16-view case runs the per-view chunk lists (their
    warp pools of reserved chunks run dry mid-drain)."""
    w = S.workload(idx, n=n, n_views=views)
    G = grads_for(w.cameras, w.params.layers, w.cloud.channels)
    small = run_gpu(w.cloud, w.cameras, w.poses, w.params, grads=G, record_capacity=cap)
    assert _hdr(small.ws)["mode"] == 0
    _, fwd, bwd = run_oracle(w.cloud, w.cameras, w.poses, w.params, grads=G)
    compare_forward(small, fwd, ctx="overflow")
    compare_backward(small, bwd, ctx="inline")


def test_backward_consumes_forward_lists_or_resweeps():
    """With ghosts (rho > 0) the depth pass lists them too (back of the record region), and the backward
    consumes both of its lists when the workspace holds them for the same inputs (mode 2: no sweep); with the
    header's ghost flag cleared (a ghost that did not fit the forward's list) the sweep re-finds the ghosts and
    keeps the survivor records (mode 1); with the fingerprint cleared it re-renders every point (mode 0).  All
    three agree with the oracle; a second backward after a re-render re-sweeps again."""
    w = S.workload(2, n=150_000)
    dev = torch.device("cuda")
    G = [g.to(dev) for g in grads_for(w.cameras, w.params.layers, w.cloud.channels)]
    r = A.Renderer(w.cloud.to(dev), w.cameras, w.poses, w.params)
    r.forward()
    h = _hdr(r.ws)
    front = h["resv"] & ((1 << 40) - 1)
    assert h["tag"] != 0 and h["overflow"] == 0 and h["ghosts_fwd"] == 1 and h["front_ok"] == front > 0
    assert h["back_ok"] == (h["resv"] >> 40) * 256 > 0  # the depth pass wrote the ghost list
    listed = [t.clone() for t in r.backward(G)]
    h0 = _hdr(r.ws)
    assert h0["mode"] == 2 and h0["back_ok"] == h["back_ok"] and h0["front_ok"] == h["front_ok"]
    r.backward(G)  # the lists stay consumable
    assert _hdr(r.ws)["mode"] == 2
    _set_hdr_i32(r.ws, 64, 0)  # as if a ghost had not fitted the forward's list
    reuse = [t.clone() for t in r.backward(G)]
    h1 = _hdr(r.ws)
    assert h1["mode"] == 1 and h1["back_ok"] == (h1["resv"] >> 40) * 256 > 0  # the sweep wrote the ghost list
    assert h1["front_ok"] == h["front_ok"]  # ... and left the survivor records alone
    off = r.ws.ptr - r.ws.buf.data_ptr()
    r.ws.buf[off + 16:off + 24] = 0  # clear the fingerprint: the lists no longer count as the forward's
    sweep = [t.clone() for t in r.backward(G)]
    assert _hdr(r.ws)["mode"] == 0 and _hdr(r.ws)["tag"] == 0
    r.backward(G)
    assert _hdr(r.ws)["mode"] == 0
    torch.cuda.synchronize()
    _, fwd, bwd = run_oracle(w.cloud, w.cameras, w.poses, w.params, grads=[g.cpu() for g in G])
    for name, res in (("listed", listed), ("reuse", reuse), ("sweep", sweep)):
        r.d_feat.copy_(res[0]); r.d_pos.copy_(res[1]); r.d_pose.copy_(res[2])
        compare_backward(r, bwd, ctx=name)
    r.forward()  # a fresh forward makes the lists consumable again
    r.backward(G)
    assert _hdr(r.ws)["mode"] == 2


@pytest.mark.parametrize("idx,n,views", [(2, 150_000, None), (4, 60_000, 16)])
def test_forward_ghost_list_overflow(idx, n, views):
    """A record region with room for the survivor records but not for every ghost: the depth pass clears its
    ghost flag and the backward re-finds the ghosts with its sweep (mode 1; mode 0 if the survivors did not fit
    either) -- same results.  The 16-view case runs the per-view ghost chunks."""
    w = S.workload(idx, n=n, n_views=views)
    G = grads_for(w.cameras, w.params.layers, w.cloud.channels)
    full = run_gpu(w.cloud, w.cameras, w.poses, w.params, grads=None)
    hf = _hdr(full.ws)
    assert hf["ghosts_fwd"] == 1 and hf["back_ok"] > 0
    cap = int(hf["front_ok"] + hf["back_ok"] // 3)
    small = run_gpu(w.cloud, w.cameras, w.poses, w.params, grads=G, record_capacity=cap)
    hs = _hdr(small.ws)
    assert hs["mode"] in (0, 1) and hs["ghosts_fwd"] == 0
    _, fwd, bwd = run_oracle(w.cloud, w.cameras, w.poses, w.params, grads=G)
    compare_forward(small, fwd, ctx="ghost overflow")
    compare_backward(small, bwd, ctx="ghost overflow")


# --------------------------------------------------------------------------- #
# NEXT-2: environment map (R29) and logarithmic descriptors
# --------------------------------------------------------------------------- #
def smooth_env(H, W, C, seed=0):
    """Low-frequency equirectangular map (so fp32-vs-fp64 direction differences stay far below tolerance)."""
    rng = np.random.default_rng(seed)
    lon = (np.arange(W) + 0.5) / W * 2 * np.pi - np.pi
    lat = (np.arange(H) + 0.5) / H * np.pi - np.pi / 2
    LA, LO = np.meshgrid(lat, lon, indexing="ij")
    chans = [0.5 + 0.3 * np.sin(LO + rng.uniform(0, 6)) * np.cos(LA) + 0.1 * np.sin(2 * LA + rng.uniform(0, 6))
             for _ in range(C)]
    return np.stack(chans, -1).astype(np.float32)


@pytest.mark.parametrize("cfg,log", [(0, False), (0, True), (2, False), (2, True)])
def test_env_map_and_log_descriptors_fwd_bwd(cfg, log):
    w = S.workload(cfg, n=60_000 if cfg else None)
    C = w.cloud.channels
    prm = dataclasses.replace(w.params, discard=True, ghost_rate=0.3, log_descriptors=log,
                              env_map=smooth_env(32, 64, C, seed=cfg))
    cloud = w.cloud
    if cfg == 0:
        cloud = dataclasses.replace(w.cloud, radius=torch.full_like(w.cloud.radius, 0.02))
    if log:  # descriptors in log space (U(0,1) -> [-1.5, 0.5])
        cloud = dataclasses.replace(cloud, feat=cloud.feat * 2 - 1.5)
    G = grads_for(w.cameras, prm.layers, C)
    r = run_gpu(cloud, w.cameras, w.poses, prm, grads=G)
    _, fwd, bwd = run_oracle(cloud, w.cameras, w.poses, prm, grads=G)
    compare_forward(r, fwd, ctx=f"env cfg{cfg} log={log}")
    compare_backward(r, bwd, ctx=f"env cfg{cfg} log={log}")
    assert r.d_env is not None and r.d_env.abs().sum() > 0
    assert np.abs(bwd.dx).sum() > 0 and np.abs(bwd.dtau).sum() > 0


def test_env_map_gradient_with_empty_cloud():
    cam = S.pinhole(64, 48)
    cloud = S.Cloud(torch.zeros(3, 0), torch.zeros(0), torch.zeros(0, 4))
    prm = S.Params(layers=3, env_map=smooth_env(16, 32, 4, seed=3))
    G = grads_for([cam], 3, 4)
    r = run_gpu(cloud, [cam], [S.tiny_pose()], prm, grads=G)
    _, fwd, bwd = run_oracle(cloud, [cam], [S.tiny_pose()], prm, grads=G)
    compare_forward(r, fwd, ctx="env empty")
    compare_backward(r, bwd, ctx="env empty", check_feat=False, check_pos=False)
    assert r.d_env.abs().sum() > 0


@pytest.mark.parametrize("ghost,cfg", [(0.0, 2), (0.25, 2), (0.0, 1)])
def test_spatial_gradients_for_rendered_points(ghost, cfg):
    """NEXT-3 (R31): ghost gradients disabled (the §6.2 baseline): Eqs. 9-11 for the rendered points."""
    w = S.workload(cfg, n=80_000, n_views=2 if cfg == 1 else None)
    prm = dataclasses.replace(w.params, ghost_rate=ghost, spatial_rendered=True)
    G = grads_for(w.cameras, prm.layers, w.cloud.channels)
    r = run_gpu(w.cloud, w.cameras, w.poses, prm, grads=G)
    _, fwd, bwd = run_oracle(w.cloud, w.cameras, w.poses, prm, grads=G)
    compare_backward(r, bwd, ctx=f"spatial_rendered rho={ghost}")
    assert np.count_nonzero(np.abs(bwd.dx).sum(0)) > 1000


@pytest.mark.parametrize("mode,cfg", [(1, 2), (-1, 2), (-1, 1), (-1, 0)])
def test_normal_culling_fwd_bwd(mode, cfg):
    """NEXT-3: Eq. 5 normal culling (R32) -- keys/counts/masks bit-exact, gradients within tolerance."""
    w = S.workload(cfg, n=80_000 if cfg else None, n_views=2 if cfg == 1 else None)
    cloud = w.cloud
    if cloud.normal is None:  # configs[0] (uniform cube): random unit normals
        g = torch.Generator().manual_seed(9)
        nrm = torch.randn(3, cloud.n, generator=g)
        cloud = dataclasses.replace(cloud, normal=nrm / nrm.norm(dim=0, keepdim=True))
    prm = dataclasses.replace(w.params, ghost_rate=0.25, normal_culling=mode)
    G = grads_for(w.cameras, prm.layers, cloud.channels)
    r = run_gpu(cloud, w.cameras, w.poses, prm, grads=G)
    _, fwd, bwd = run_oracle(cloud, w.cameras, w.poses, prm, grads=G)
    compare_forward(r, fwd, ctx=f"normal culling {mode}")
    compare_backward(r, bwd, ctx=f"normal culling {mode}")
    m = r.masks().cpu().numpy()
    om = O.point_masks(O.Points.from_cloud(cloud.to("cpu")), w.cameras, w.poses, prm)
    assert np.array_equal(m, om)
    base = run_gpu(cloud, w.cameras, w.poses, dataclasses.replace(prm, normal_culling=0))
    assert (r.pyrs[0].count.sum() < base.pyrs[0].count.sum()).item()  # something was culled


# --------------------------------------------------------------------------- #
# NEXT-3: equidistant fisheye with distance depth (R35)
# --------------------------------------------------------------------------- #
@pytest.mark.parametrize("fov,ghost,views", [(120.0, 0.25, 1), (200.0, 0.25, 1), (179.0, 0.0, 3)])
def test_fisheye_fwd_bwd(fov, ghost, views):
    room = S.make_room(10.0)
    cloud = S.room_cloud(150_000, room, channels=4, seed=21)
    cloud = dataclasses.replace(cloud, radius=torch.full_like(cloud.radius, 0.05))  # ~1 px splats: most kept
    cams = [S.fisheye_camera(160, 120, fov) for _ in range(views)]
    poses = S.room_poses(views, room, seed=8)
    prm = S.Params(layers=4, discard=True, ghost_rate=ghost, seed=5, background=[0.5, 0.25, -0.5, 1.0])
    G = grads_for(cams, prm.layers, 4)
    r = run_gpu(cloud, cams, poses, prm, grads=G if ghost else None)
    _, fwd, bwd = run_oracle(cloud, cams, poses, prm, grads=G if ghost else None)
    compare_forward(r, fwd, ctx=f"fisheye {fov}")
    if ghost:
        compare_backward(r, bwd, ctx=f"fisheye {fov}")
        assert np.abs(bwd.dx).sum() > 0 and (r.d_intr[:, 4:] == 0).all()
    m = r.masks().cpu().numpy()
    assert np.array_equal(m, O.point_masks(O.Points.from_cloud(cloud), cams, poses, prm))
    assert (fwd.count > 0).sum() > 5000


@pytest.mark.parametrize("fov", [120.0, 200.0])
def test_fisheye_precull_is_conservative(fov):
    """Points on rings just inside / outside theta_max at tiny to huge distances: never dropped by the
    pre-culls (cone + warp box for the narrow lens, none for the wide one)."""
    cam = S.fisheye_camera(64, 64, fov)
    th_max = cam.r2_max
    rng = np.random.default_rng(3)
    th = np.concatenate([th_max + np.array([-1e-3, -1e-5, -1e-7, 0.0, 1e-7, 1e-5]), rng.uniform(0, th_max, 50)])
    ph = np.linspace(0, 2 * np.pi, 64, endpoint=False)
    ds = np.array([1e-3, 0.5, 3.0, 1e3, 1e5])
    T, Ph, D = [a.ravel() for a in np.meshgrid(th, ph, ds)]
    xyz = np.stack([D * np.sin(T) * np.cos(Ph), D * np.sin(T) * np.sin(Ph), D * np.cos(T)]).astype(np.float32)
    n = xyz.shape[1]
    cloud = S.Cloud(torch.from_numpy(xyz), torch.full((n,), 0.01), torch.rand(n, 4, generator=torch.Generator().manual_seed(2)))
    prm = S.Params(layers=5, discard=False)
    pose = S.Pose(np.eye(3, dtype=np.float32), np.zeros(3, dtype=np.float32))
    r = run_gpu(cloud, [cam], [pose], prm)
    _, fwd, _ = run_oracle(cloud, [cam], [pose], prm)
    compare_forward(r, fwd, ctx=f"fisheye precull {fov}")
    assert (fwd.count > 0).sum() > 300


# --------------------------------------------------------------------------- #
# tile culling with precomputed tile bounds (adop_tile_bounds): identical results
# --------------------------------------------------------------------------- #
@pytest.mark.parametrize("idx,n,views,bwd", [(3, 2_000_000, 1, False), (1, 400_000, 4, False), (4, 300_000, 16, True),
                                             (2, 300_000, 1, True)])
def test_tile_culling_is_exact(idx, n, views, bwd):
    w = S.workload(idx, n=n, n_views=views if idx != 4 else None)
    dev = torch.device("cuda")
    cloud = w.cloud.to(dev)
    G = [g.to(dev) for g in grads_for(w.cameras, w.params.layers, cloud.channels)] if bwd else None
    plain = A.Renderer(cloud, w.cameras, w.poses, w.params)
    plain.forward()
    culled = A.Renderer(cloud, w.cameras, w.poses, w.params)
    culled.points.enable_tile_culling()
    culled.forward()
    if bwd:
        plain.backward(G)
        culled.backward(G)
    torch.cuda.synchronize()
    culled.ws.stats3()
    ntiles = (cloud.n + 255) // 256
    assert 0 < culled.ws.tiles_read <= ntiles
    if views == 1:
        assert culled.ws.tiles_read < ntiles  # one view sees only part of the cloud
    for p, q in zip(plain.pyrs, culled.pyrs):
        assert torch.equal(p.keys, q.keys) and torch.equal(p.count, q.count)
        torch.testing.assert_close(p.image, q.image, rtol=1e-5, atol=1e-6)
    if bwd:
        # fp32 atomic sums in another order (cancellation in d_pos): tolerance scaled by the field's magnitude
        torch.testing.assert_close(plain.d_feat, culled.d_feat, rtol=1e-5, atol=1e-6)
        torch.testing.assert_close(plain.d_pos, culled.d_pos, rtol=1e-4, atol=1e-5 * float(plain.d_pos.abs().max()))
    if idx == 2:  # and against the oracle
        _, fwd, ob = run_oracle(w.cloud, w.cameras, w.poses, w.params, grads=[g.cpu() for g in G])
        compare_forward(culled, fwd, ctx="tile culling")
        compare_backward(culled, ob, ctx="tile culling")


@pytest.mark.parametrize("model", [S.PINHOLE, S.OPENCV8, S.FISHEYE])
def test_discard_prefilter_is_conservative(model):
    """One point per layer-0 pixel (so every kept point owns its key) with radii putting gamma r_screen in
    [0.2, 1.3]: thousands of keep / discard decisions near 1 - beta; the depth pass's hash-first discard
    prefilter (a lane bound on r_screen) must never drop a point the exact test keeps -- keys bit-exact."""
    rng = np.random.default_rng(23)
    w, h = 256, 192
    if model == S.FISHEYE:
        cam = S.fisheye_camera(w, h, 120.0)
    else:
        cam = S.Camera(w, h, S.PINHOLE, 128.0, 128.0, 128.0, 96.0)
        if model == S.OPENCV8:
            cam = dataclasses.replace(cam, model=S.OPENCV8, k=(0.01, -0.02, 0.0, 0.005, 0.0, 0.0), p=(0.001, -0.001))
            cam = dataclasses.replace(cam, r2_max=S.distortion_r2_max(cam))
    us, vs = np.meshgrid(np.arange(w), np.arange(h))
    z = rng.uniform(0.5, 40.0, us.size)
    if model == S.FISHEYE:
        xd, yd = (us.ravel() - cam.cx) / cam.fx, (vs.ravel() - cam.cy) / cam.fy
        th = np.hypot(xd, yd)
        keep = th < cam.r2_max * 0.98
        s = np.where(th > 0, np.sin(th) / np.maximum(th, 1e-12), 1.0)
        xyz = np.stack([s * xd * z, s * yd * z, np.cos(th) * z])[:, keep]
        z = z[keep]
    else:
        xyz = np.stack([(us.ravel() - cam.cx) / cam.fx * z, (vs.ravel() - cam.cy) / cam.fy * z, z])
    f = (cam.fx + cam.fy) / 2
    rad = rng.uniform(0.2, 1.3, z.size) / 1.5 * z / f   # gamma r_screen in [0.2, 1.3]
    perm = rng.permutation(z.size)
    cloud = S.Cloud(torch.from_numpy(np.ascontiguousarray(xyz[:, perm], dtype=np.float32)),
                    torch.from_numpy(np.ascontiguousarray(rad[perm], dtype=np.float32)),
                    torch.rand(z.size, 4, generator=torch.Generator().manual_seed(4)))
    prm = S.Params(layers=4, discard=True, seed=77)
    pose = S.Pose(np.eye(3, dtype=np.float32), np.zeros(3, dtype=np.float32))
    r = run_gpu(cloud, [cam], [pose], prm)
    _, fwd, _ = run_oracle(cloud, [cam], [pose], prm)
    compare_forward(r, fwd, ctx=f"prefilter {model}")
    assert 0.2 < (fwd.count[0][: w * h] > 0).mean() < 0.95


@pytest.mark.parametrize("fov", [120.0, 200.0])
def test_fisheye_with_env_map_log_descriptors_and_tile_culling(fov):
    """The NEXT items together on the fisheye: environment map (fisheye C^-1), log descriptors, ghosts,
    intrinsics, and the same frame with tile culling -- against the oracle."""
    room = S.make_room(10.0)
    cloud = S.room_cloud(120_000, room, channels=4, seed=31)
    cloud = dataclasses.replace(cloud, radius=torch.full_like(cloud.radius, 0.05), feat=cloud.feat * 2 - 1.5)
    cams = [S.fisheye_camera(128, 96, fov)]
    poses = S.room_poses(1, room, seed=12)
    prm = S.Params(layers=4, discard=True, ghost_rate=0.25, seed=9, log_descriptors=True,
                   env_map=smooth_env(32, 64, 4, seed=5))
    G = grads_for(cams, prm.layers, 4)
    dev = torch.device("cuda")
    r = A.Renderer(cloud.to(dev), cams, poses, prm, intrinsics=True)
    r.points.enable_tile_culling()
    r.forward()
    r.backward([g.to(dev) for g in G])
    torch.cuda.synchronize()
    _, fwd, bwd = run_oracle(cloud, cams, poses, prm, grads=G)
    compare_forward(r, fwd, ctx=f"fisheye+env {fov}")
    compare_backward(r, bwd, ctx=f"fisheye+env {fov}")
    assert r.d_env.abs().sum() > 0 and (fwd.count > 0).sum() > 1000


def test_largest_index_range_2_31_points_ending_at_index_2_32():
    """Maximum sizes: 2^31 + 4196 points (tile and point indices past int32, a ragged last tile, no TMA tensor
    map past 2^31 points) whose global indices end at 2^32 - 1, the largest the packed key holds.  All but the
    last 5000 points lie behind the camera; those 5000 are checked against the oracle (run on them alone with
    the same global indices): keys bit-exact (index half included), counts exact, image, d_feat, d_pos, d_pose
    and d_intr within tolerance, every other point's gradient exactly zero."""
    n = (1 << 31) + 4196
    tail = 5000
    dev = torch.device("cuda")
    goff = (1 << 32) - n
    pos = torch.zeros(3, n, dtype=torch.float32, device=dev)
    pos[2].fill_(-1.0)  # behind the camera: culled
    g = torch.Generator(device="cpu").manual_seed(7)
    vis = torch.empty(3, tail)
    vis[0].uniform_(-1.0, 1.0, generator=g)
    vis[1].uniform_(-0.75, 0.75, generator=g)
    vis[2].uniform_(2.0, 4.0, generator=g)
    pos[:, n - tail:] = vis.to(dev)
    radius = torch.full((n,), 0.02, dtype=torch.float32, device=dev)
    feat = torch.zeros(n, 1, dtype=torch.float32, device=dev)
    feat[n - tail:, 0] = torch.rand(tail, generator=g).to(dev)
    cloud = S.Cloud(pos, radius, feat)
    cams = [S.pinhole(320, 240)]
    poses = [S.Pose(np.eye(3, dtype=np.float32), np.zeros(3, dtype=np.float32))]
    prm = S.Params(layers=3, discard=True, ghost_rate=0.2, seed=5, background=[0.25])
    G = grads_for(cams, prm.layers, 1)
    r = run_gpu(cloud, cams, poses, prm, record_capacity=1 << 20, global_offset=goff, grads=G)
    assert not r.ws.stats()[1]
    sub = S.Cloud(vis.clone(), torch.full((tail,), 0.02), feat[n - tail:].cpu())
    del cloud, pos, radius, feat
    _, fwd, bwd = run_oracle(sub, cams, poses, prm, global_offset=goff + n - tail, grads=G)
    compare_forward(r, fwd, ctx="2^31 points")
    # backward: the tail's gradients against the oracle, every other point's exactly zero
    tail_view = type("Tail", (), {})()
    tail_view.d_feat, tail_view.d_pos = r.d_feat[n - tail:], r.d_pos[:, n - tail:]
    tail_view.d_pose, tail_view.d_intr = r.d_pose, r.d_intr
    compare_backward(tail_view, bwd, ctx="2^31 points")
    assert float(r.d_feat[: n - tail].abs().max()) == 0.0 and float(r.d_pos[:, : n - tail].abs().max()) == 0.0
    assert np.abs(bwd.dx).sum() > 0 and np.abs(bwd.dtau).sum() > 0
    assert (fwd.count > 0).sum() > 1000
    keys = keys_u64(r.pyrs[0].keys)
    hit = keys != np.uint64(0x7FFFFFFFFFFFFFFF)
    assert (keys[hit] & np.uint64(0xFFFFFFFF)).max() > (1 << 31)  # winners carry indices past 2^31


def test_descriptors_in_pinned_host_memory():
    """adop_points.feat in pinned host memory (zero-copy, UVA): the blend reads the survivors' descriptors in
    place; same result as with the descriptors in HBM, and against the oracle."""
    w = S.workload(1, n=200_004, n_views=4)
    dev = torch.device("cuda")
    cloud = w.cloud.to(dev)
    ref = A.Renderer(cloud, w.cameras, w.poses, w.params)
    ref.forward()
    h_feat = w.cloud.feat.cpu().pin_memory()
    r = A.Renderer(S.Cloud(cloud.pos, cloud.radius, h_feat), w.cameras, w.poses, w.params)
    assert r.points.s.feat == h_feat.data_ptr()
    r.forward()
    torch.cuda.synchronize()
    for v in range(4):
        assert torch.equal(r.pyrs[v].keys, ref.pyrs[v].keys) and torch.equal(r.pyrs[v].count, ref.pyrs[v].count)
        torch.testing.assert_close(r.pyrs[v].image, ref.pyrs[v].image, rtol=1e-5, atol=1e-6)
    _, fwd, _ = run_oracle(w.cloud, w.cameras, w.poses, w.params)
    compare_forward(r, fwd, ctx="host descriptors")


def test_backward_captured_in_a_cuda_graph():
    """The backward's side-stream fork / join (texture consumer beside the ghost consumer) inside CUDA-graph
    capture: replaying the captured backward reproduces the eager one."""
    w = S.workload(2, n=200_004)
    dev = torch.device("cuda")
    G = [g.to(dev) for g in grads_for(w.cameras, w.params.layers, w.cloud.channels)]
    r = A.Renderer(w.cloud.to(dev), w.cameras, w.poses, w.params)
    r.forward()
    r.backward(G)
    torch.cuda.synchronize()
    eager = [t.clone() for t in (r.d_feat, r.d_pos, r.d_pose)]
    s = torch.cuda.Stream(dev)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        r.backward(G, stream=s)
        torch.cuda.synchronize()
        with torch.cuda.graph(graph, stream=s):
            r.backward(G, stream=s)
    for t in (r.d_feat, r.d_pos, r.d_pose):
        t.zero_()
    graph.replay()
    torch.cuda.synchronize()
    for got, ref in zip((r.d_feat, r.d_pos, r.d_pose), eager):
        torch.testing.assert_close(got, ref, rtol=1e-5, atol=1e-6 * float(ref.abs().max()))
    assert float(eager[0].abs().sum()) > 0 and float(eager[1].abs().sum()) > 0


def test_pose_and_camera_updates_between_forwards():
    """Renderer keys its marshalled descriptors on the pose / camera values: a pose replaced with set_poses(),
    a pose edited in place and a camera replaced with set_cameras() all reach the next forward and backward."""
    w = S.workload(2, n=150_000, n_views=2)
    prm = w.params
    G = grads_for(w.cameras, prm.layers, w.cloud.channels)
    r = A.Renderer(w.cloud.to("cuda"), w.cameras, w.poses, prm, intrinsics=True)
    r.forward()
    room = S.make_room(10.0)
    new_poses = S.room_poses(2, room, seed=77)
    r.set_poses(new_poses)
    r.forward()
    r.backward([g.cuda() for g in G])
    torch.cuda.synchronize()
    _, fwd, bwd = run_oracle(w.cloud, w.cameras, new_poses, prm, grads=G)
    compare_forward(r, fwd, ctx="set_poses")
    compare_backward(r, bwd, ctx="set_poses")
    # in-place edit of a translation and a new camera for view 1
    r.poses[0].t[:] = r.poses[0].t + np.array([0.05, -0.02, 0.01], np.float32)
    cams = [w.cameras[0], S.opencv_camera(w.cameras[1].width, w.cameras[1].height, seed=99)]
    r.set_cameras(cams)
    r.forward()
    r.backward([g.cuda() for g in G])
    torch.cuda.synchronize()
    _, fwd, bwd = run_oracle(w.cloud, cams, r.poses, prm, grads=G)
    compare_forward(r, fwd, ctx="in-place pose + set_cameras")
    compare_backward(r, bwd, ctx="in-place pose + set_cameras")


@pytest.mark.parametrize("mv", ["0", "5", "9", "15"])
def test_multi_view_list_orders(mv):
    """ADOP_MV_LISTS (read once per process, so each setting runs in a subprocess): 0 flat mixed-view lists,
    5 the default (this small launch: flat), 9 per-view chunks with only the blend view-major, 15 every consumer
    view-major.  All match the oracle."""
    import os
    import subprocess
    import sys
    code = (
        "import sys; sys.path.insert(0, '.')\n"
        "from paper_2110_06635_b200 import scene as S\n"
        "from tests.parity import compare_backward, compare_forward, grads_for, run_gpu, run_oracle\n"
        "w = S.workload(4, n=80_013, n_views=6)\n"
        "G = grads_for(w.cameras, w.params.layers, w.cloud.channels)\n"
        "r = run_gpu(w.cloud, w.cameras, w.poses, w.params, grads=G)\n"
        "_, fwd, bwd = run_oracle(w.cloud, w.cameras, w.poses, w.params, grads=G)\n"
        "compare_forward(r, fwd, ctx='mv')\n"
        "compare_backward(r, bwd, ctx='mv')\n"
        "print('ok')\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True, timeout=600,
                         env={**os.environ, "ADOP_MV_LISTS": mv})
    assert res.returncode == 0 and "ok" in res.stdout, res.stderr[-3000:]
