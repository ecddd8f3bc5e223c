"""Multi-process (world_size 2, gloo, CPU) tests of the sharding host logic in
paper_2110_06635_b200/parallel.py.  The phases are the CPU oracle's phase functions plugged into the
same orchestration the CUDA path uses, so what is checked here is the partitioning, global indexing,
view-id bookkeeping and the collectives (MIN on int64 keys, SUM on accum++count, SUM on point grads,
all-gather of pose rows): sharded == unsharded, keys bit-exact."""
import dataclasses
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O
from paper_2110_06635_b200 import parallel as PL
from paper_2110_06635_b200 import scene as S


class _Pyr:
    def __init__(self, P, C):
        self.P, self.C = P, C
        self.keys = torch.empty(P, dtype=torch.int64)
        self.ac = torch.zeros(P * (C + 1), dtype=torch.float64)
        self.image = torch.zeros(C * P, dtype=torch.float64)

    @property
    def accum(self):
        return self.ac[: self.P * self.C]

    @property
    def count(self):
        return self.ac[self.P * self.C:]


class OraclePhases:
    """Oracle phase functions behind the CudaPhases interface (test stand-in for the GPU)."""

    def __init__(self, pts, cams, poses, prm, pyrs, grads=None, d_feat=None, d_pos=None, d_pose=None):
        self.pts, self.cams, self.poses, self.prm, self.pyrs = pts, cams, poses, prm, pyrs
        self.grads, self.d_feat, self.d_pos, self.d_pose = grads, d_feat, d_pos, d_pose
        self.C = pts.C

    def depth(self):
        keys = O.forward_depth(self.pts, self.cams, self.poses, self.prm)
        for v, p in enumerate(self.pyrs):
            p.keys.copy_(torch.from_numpy(keys[v].view(np.int64)))

    def _keys(self):
        return np.stack([p.keys.numpy().view(np.uint64) for p in self.pyrs])

    def blend(self):
        accum, count = O.forward_blend(self.pts, self.cams, self.poses, self.prm, self._keys())
        for v, p in enumerate(self.pyrs):
            p.ac.copy_(torch.from_numpy(np.concatenate([accum[v].ravel(), count[v]])))

    def _ac(self):
        P, C = self.pyrs[0].P, self.C
        acc = np.stack([p.ac.numpy()[: P * C].reshape(P, C) for p in self.pyrs])
        cnt = np.stack([p.ac.numpy()[P * C:] for p in self.pyrs])
        return acc, cnt

    def resolve(self):
        acc, cnt = self._ac()
        img = O.forward_resolve(self.cams, self.prm, self.C, acc, cnt, self.prm.background)
        for v, p in enumerate(self.pyrs):
            p.image.copy_(torch.from_numpy(img[v]))

    def resolve_range(self, p0, p1):
        """The oracle resolves every pixel; only the image entries of pyramid pixels [p0, p1) are written (what
        adop_forward_resolve_range leaves touched)."""
        acc, cnt = self._ac()
        img = O.forward_resolve(self.cams, self.prm, self.C, acc, cnt, self.prm.background)
        idx = _image_indices(self.cams[0], self.prm.layers, self.C, p0, p1)
        for v, p in enumerate(self.pyrs):
            p.image[idx] = torch.from_numpy(img[v][idx.numpy()])

    def forward(self):
        self.depth()
        self.blend()
        self.resolve()

    def backward(self):
        acc, cnt = self._ac()
        fwd = O.Forward(self._keys(), acc, cnt, np.stack([p.image.numpy() for p in self.pyrs]))
        b = O.backward(self.pts, self.cams, self.poses, self.prm, fwd, self.grads)
        self.d_feat.copy_(torch.from_numpy(b.dtau))
        self.d_pos.copy_(torch.from_numpy(b.dx))
        self.d_pose.copy_(torch.from_numpy(b.dpose))


def _image_indices(cam, layers, C, p0, p1):
    """Indices into the planar layer-concatenated image of pyramid pixels [p0, p1) (layout of include/adop.h)."""
    out, off = [], 0
    for l in range(layers):
        w, h = -(-cam.width // 2 ** l), -(-cam.height // 2 ** l)  # ceil (oracle layer_w)
        hw = w * h
        a, b = max(p0, off), min(p1, off + hw)
        for c in range(C):
            out.append(np.arange(C * off + c * hw + (a - off), C * off + c * hw + (b - off)) if a < b else [])
        off += hw
    return torch.from_numpy(np.concatenate([np.asarray(x, dtype=np.int64) for x in out]))


def _scene():
    room = S.make_room(5.0)
    cloud = S.room_cloud(20_011, room, 3, seed=77)
    cloud = S.apply_order(cloud, S.blocked_morton_order(cloud.pos, 256))
    cloud = dataclasses.replace(cloud, radius=torch.full_like(cloud.radius, 0.03))
    cams = [S.pinhole(96, 64), S.pinhole(96, 64), S.pinhole(96, 64)]
    poses = S.room_poses(3, room, seed=5)
    prm = S.Params(layers=3, discard=True, ghost_rate=0.25, seed=11, background=[0.5, 0.25, 0.125])
    return cloud, cams, poses, prm


def _point_sharded(rank, world, port, q, keys32=False):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    cloud, cams, poses, prm = _scene()
    a, b = PL.shard_range(cloud.n, world, rank, align=256)
    pts = O.Points.from_cloud(cloud.slice(a, b), global_offset=a)
    P = O.pyramid_pixels(96, 64, prm.layers)
    pyrs = [_Pyr(P, 3) for _ in cams]
    PL.point_sharded_forward(OraclePhases(pts, cams, poses, prm, pyrs), pyrs, keys32=keys32)
    if rank == 0:
        q.put(([p.keys.numpy().copy() for p in pyrs], [p.ac.numpy().copy() for p in pyrs],
               [p.image.numpy().copy() for p in pyrs]))
    dist.barrier()
    dist.destroy_process_group()


def _point_sharded_rs(rank, world, port, q):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    cloud, cams, poses, prm = _scene()
    a, b = PL.shard_range(cloud.n, world, rank, align=256)
    pts = O.Points.from_cloud(cloud.slice(a, b), global_offset=a)
    P = O.pyramid_pixels(96, 64, prm.layers)
    pyrs = [_Pyr(P, 3) for _ in cams]
    p0, p1 = PL.point_sharded_forward_rs(OraclePhases(pts, cams, poses, prm, pyrs), pyrs)
    q.put((rank, p0, p1, [p.count[p0:p1].numpy().copy() for p in pyrs], [p.image.numpy().copy() for p in pyrs]))
    dist.barrier()
    dist.destroy_process_group()


def _point_sharded32(rank, world, port, q):
    _point_sharded(rank, world, port, q, keys32=True)


def _view_sharded(rank, world, port, q):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    cloud, cams, poses, prm = _scene()
    V = len(cams)
    a, b = PL.view_range(V, world, rank)
    pts = O.Points.from_cloud(cloud)
    P = O.pyramid_pixels(96, 64, prm.layers)
    G = S.grad_pyramid(V, 3, P, seed=9).numpy()
    pyrs = [_Pyr(P, 3) for _ in range(a, b)]
    n = cloud.n
    buf = torch.zeros(n * 3 + 3 * n, dtype=torch.float64)
    d_feat, d_pos = buf[: 3 * n].view(n, 3), buf[3 * n:].view(3, n)
    d_pose = torch.zeros(b - a, 6, dtype=torch.float64)
    ph = OraclePhases(pts, cams[a:b], poses[a:b], dataclasses.replace(prm, view_id_base=a), pyrs, G[a:b],
                      d_feat, d_pos, d_pose)
    all_pose = PL.view_sharded_step(ph, buf, d_pose, V)
    if rank == 0:
        q.put((d_feat.numpy().copy(), d_pos.numpy().copy(), all_pose.numpy().copy()))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _spawn(fn, world=2, nres=1):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=fn, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=300) if nres == 1 else [q.get(timeout=300) for _ in range(nres)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return res


def test_shard_ranges_partition():
    for n in (0, 1, 1023, 1024, 10_000, 20_011):
        for world in (1, 2, 3, 8):
            rs = [PL.shard_range(n, world, r, align=256) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(rs[i][1] == rs[i + 1][0] for i in range(world - 1))
            assert all(a % 256 == 0 for a, _ in rs if a < n)
    for V in (1, 3, 16):
        for world in (1, 2, 4, 8):
            rs = [PL.view_range(V, world, r) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == V and all(rs[i][1] == rs[i + 1][0] for i in range(world - 1))


def test_point_sharded_forward_gloo_ws2_equals_unsharded():
    keys, ac, image = _spawn(_point_sharded)
    cloud, cams, poses, prm = _scene()
    fwd = O.forward(O.Points.from_cloud(cloud), cams, poses, prm)
    P = fwd.count.shape[1]
    for v in range(len(cams)):
        assert np.array_equal(keys[v].view(np.uint64), fwd.keys[v])
        assert np.array_equal(ac[v][P * 3:], fwd.count[v])
        np.testing.assert_allclose(image[v], fwd.image[v], rtol=1e-12, atol=1e-12)
    assert fwd.count.sum() > 500


def test_point_sharded_forward_reduce_scatter_gloo_ws2():
    """Reduce-scatter variant: each rank's pixel slice of counts and image equals the unsharded
    forward's; the slices partition the pyramid."""
    res = sorted(_spawn(_point_sharded_rs, nres=2), key=lambda r: r[0])
    cloud, cams, poses, prm = _scene()
    fwd = O.forward(O.Points.from_cloud(cloud), cams, poses, prm)
    P = fwd.count.shape[1]
    assert res[0][1] == 0 and res[0][2] == res[1][1] and res[1][2] == P and res[0][1] < res[0][2] < P
    for rank, p0, p1, counts, images in res:
        idx = _image_indices(cams[0], prm.layers, 3, p0, p1).numpy()
        for v in range(len(cams)):
            assert np.array_equal(counts[v], fwd.count[v][p0:p1])
            np.testing.assert_allclose(images[v][idx], fwd.image[v][idx], rtol=1e-12, atol=1e-12)
    assert fwd.count.sum() > 500


def test_point_sharded_forward_depth_words_only_gloo_ws2():
    """32-bit depth-word MIN exchange: depth words, counts and images equal the unsharded forward; the
    low words are the shard-local winners (not exchanged)."""
    keys, ac, image = _spawn(_point_sharded32)
    cloud, cams, poses, prm = _scene()
    fwd = O.forward(O.Points.from_cloud(cloud), cams, poses, prm)
    P = fwd.count.shape[1]
    for v in range(len(cams)):
        assert np.array_equal(keys[v].view(np.uint64) >> np.uint64(32), fwd.keys[v] >> np.uint64(32))
        assert np.array_equal(ac[v][P * 3:], fwd.count[v])
        np.testing.assert_allclose(image[v], fwd.image[v], rtol=1e-12, atol=1e-12)


def test_view_sharded_training_gloo_ws2_equals_unsharded():
    d_feat, d_pos, d_pose = _spawn(_view_sharded)
    cloud, cams, poses, prm = _scene()
    pts = O.Points.from_cloud(cloud)
    fwd = O.forward(pts, cams, poses, prm)
    G = S.grad_pyramid(len(cams), 3, fwd.count.shape[1], seed=9).numpy()
    b = O.backward(pts, cams, poses, prm, fwd, G)
    np.testing.assert_allclose(d_feat, b.dtau, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(d_pos, b.dx, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(d_pose, b.dpose, rtol=1e-12, atol=1e-12)
    assert np.abs(b.dx).sum() > 0


# --------------------------------------------------------------------------- #
# point sharding over a shared (peer-memory) pyramid: the orchestration of point_sharded_forward_p2p
# --------------------------------------------------------------------------- #
class _SharedPyr:
    """The owner's pyramid as every rank sees it: file-backed shared tensors stand in for the IPC-mapped
    device memory; a file lock stands in for the atomicity of the kernels' red.min / red.add."""

    def __init__(self, path, P, C):
        self.P, self.C = P, C
        self.keys = torch.from_file(path + ".k", shared=True, size=P, dtype=torch.int64)
        self.ac = torch.from_file(path + ".ac", shared=True, size=P * (C + 1), dtype=torch.float64)
        self.image = torch.zeros(C * P, dtype=torch.float64)


class SharedOraclePhases(OraclePhases):
    def __init__(self, lock_path, *args):
        super().__init__(*args)
        self.lock_path = lock_path

    def _locked(self, fn):
        import fcntl
        with open(self.lock_path, "a") as f:
            fcntl.flock(f, fcntl.LOCK_EX)
            try:
                fn()
            finally:
                fcntl.flock(f, fcntl.LOCK_UN)

    def clear(self):
        for p in self.pyrs:
            p.keys.fill_(np.iinfo(np.int64).max)
            p.ac.zero_()

    def sync(self):
        pass

    def depth(self):  # this shard's keys min-reduced into the shared pyramid
        keys = O.forward_depth(self.pts, self.cams, self.poses, self.prm)

        def upd():
            for v, p in enumerate(self.pyrs):
                p.keys.copy_(torch.minimum(p.keys, torch.from_numpy(keys[v].view(np.int64))))
        self._locked(upd)

    def blend(self):  # this shard's sums added into the shared pyramid
        accum, count = O.forward_blend(self.pts, self.cams, self.poses, self.prm, self._keys())

        def upd():
            for v, p in enumerate(self.pyrs):
                p.ac.add_(torch.from_numpy(np.concatenate([accum[v].ravel(), count[v]])))
        self._locked(upd)


def _point_sharded_p2p(rank, world, port, q, tmp):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    cloud, cams, poses, prm = _scene()
    a, b = PL.shard_range(cloud.n, world, rank, align=256)
    pts = O.Points.from_cloud(cloud.slice(a, b), global_offset=a)
    P = O.pyramid_pixels(96, 64, prm.layers)
    pyrs = [_SharedPyr(os.path.join(tmp, f"pyr{v}"), P, 3) for v in range(len(cams))]
    ph = SharedOraclePhases(os.path.join(tmp, "lock"), pts, cams, poses, prm, pyrs)
    for _ in range(2):  # the second frame checks the owner's per-frame reset
        PL.point_sharded_forward_p2p(ph, owner=1)
    if rank == 1:
        q.put(([p.keys.numpy().copy() for p in pyrs], [p.ac.numpy().copy() for p in pyrs],
               [p.image.numpy().copy() for p in pyrs]))
    dist.barrier()
    dist.destroy_process_group()


def test_point_sharded_forward_over_a_shared_pyramid_gloo_ws2(tmp_path):
    cloud, cams, poses, prm = _scene()
    P = O.pyramid_pixels(96, 64, prm.layers)
    for v in range(len(cams)):  # the owner's buffers (pre-sized backing files)
        (tmp_path / f"pyr{v}.k").write_bytes(b"\0" * (8 * P))
        (tmp_path / f"pyr{v}.ac").write_bytes(b"\0" * (8 * P * 4))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_point_sharded_p2p, args=(r, 2, port, q, str(tmp_path))) for r in range(2)]
    for p in procs:
        p.start()
    keys, ac, image = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    fwd = O.forward(O.Points.from_cloud(cloud), cams, poses, prm)
    for v in range(len(cams)):
        assert np.array_equal(keys[v].view(np.uint64), fwd.keys[v])
        assert np.array_equal(ac[v][P * 3:], fwd.count[v])
        np.testing.assert_allclose(image[v], fwd.image[v], rtol=1e-12, atol=1e-12)
    assert fwd.count.sum() > 500


def test_peer_non_owner_backward_is_refused():
    """The peer-memory point sharding is forward-only on non-owners (their image is never resolved)."""
    import types
    from paper_2110_06635_b200 import adop as A
    fake = types.SimpleNamespace(peer_non_owner=True, d_feat=None)
    with pytest.raises(RuntimeError, match="non-owner"):
        A.Renderer.backward(fake, [])
