"""GPU parity of the preprocessing calls against oracle/preprocess.py."""
import numpy as np
import pytest
import torch

from oracle import preprocess as PP
from paper_2110_06635_b200 import adop as A
from paper_2110_06635_b200 import scene as S

pytestmark = pytest.mark.gpu


def _pts(pos, feat=None, normal=None, radius=None):
    dev = torch.device("cuda")
    n = pos.shape[1]
    feat = torch.rand(n, 3) if feat is None else feat
    return A.Points(pos.to(dev).contiguous(), None if radius is None else radius.to(dev), feat.to(dev).contiguous(),
                    radius_uniform=0.01, normal=None if normal is None else normal.to(dev).contiguous())


@pytest.mark.parametrize("n,block,seed", [(1, 4, 0), (8, 8, 3), (5000, 64, 9), (20_011, 256, 5)])
def test_blocked_morton_order_bitexact(n, block, seed):
    room = S.make_room(10.0)
    cloud = S.room_cloud(n, room, channels=3, seed=seed + 1)
    perm = A.blocked_morton_order(_pts(cloud.pos), block=block, seed=seed).cpu().numpy()
    ref = PP.blocked_morton_order(cloud.pos.numpy(), block, seed)
    assert np.array_equal(perm, ref)


def test_morton_codes_degenerate_axis_and_duplicates():
    pos = torch.zeros(3, 3000)
    pos[0] = torch.rand(3000)
    pos[1, ::3] = 0.5            # y takes 2 values, z is constant: a degenerate axis
    pos[:, 1000:1010] = pos[:, 1000:1001]  # duplicates: ties broken by index
    perm = A.blocked_morton_order(_pts(pos), block=100, seed=1).cpu().numpy()
    assert np.array_equal(perm, PP.blocked_morton_order(pos.numpy(), 100, 1))


def test_apply_order_gathers_every_array():
    cloud = S.room_cloud(10_000, S.make_room(10.0), channels=5, seed=4)
    p = _pts(cloud.pos, cloud.feat, cloud.normal, cloud.radius)
    perm = A.blocked_morton_order(p, 128, 7)
    q = A.apply_order(p, perm)
    pc = perm.cpu()
    assert torch.equal(q.pos.cpu(), cloud.pos[:, pc]) and torch.equal(q.feat.cpu(), cloud.feat[pc])
    assert torch.equal(q.normal.cpu(), cloud.normal[:, pc]) and torch.equal(q.radius.cpu(), cloud.radius[pc])


@pytest.mark.parametrize("k,n", [(2, 12), (8, 3000), (7, 2500), (16, 1500)])
def test_knn_radius_matches_bruteforce(k, n):
    if n == 12:
        pos = torch.zeros(3, 12)
        pos[0] = torch.arange(12.0)  # unit lattice
    else:
        pos = S.room_cloud(n, S.make_room(4.0), channels=1, seed=n).pos
    r = A.knn_radius(_pts(pos), k).cpu().numpy().astype(np.float64)
    ref = PP.knn_radius(pos.numpy(), k)
    np.testing.assert_allclose(r, ref, rtol=2e-6, atol=1e-12)


def test_knn_radius_clusters_and_duplicates():
    g = torch.Generator().manual_seed(0)
    a = torch.rand(3, 400, generator=g)
    pos = torch.cat([a, 0.1 * a + 100.0], 1)
    pos[:, 10:13] = pos[:, 10:11]  # exact duplicates
    r = A.knn_radius(_pts(pos), 6).cpu().numpy().astype(np.float64)
    np.testing.assert_allclose(r, PP.knn_radius(pos.numpy(), 6), rtol=2e-5, atol=1e-9)
