"""Pins for the preprocessing oracle: kNN world radius (reading R33) and
the blocked Morton shuffle (reading R34) -- CPU only."""
import numpy as np
import pytest

from oracle import preprocess as PP

F = np.float32


def test_knn_radius_unit_lattice():
    """Unit-spaced 1-D lattice, k = 2: interior points have neighbours at distance 1, 1 -> 1; the ends at 1, 2
    -> median 1.5."""
    pos = np.zeros((3, 12), F)
    pos[0] = np.arange(12)
    r = PP.knn_radius(pos, 2)
    np.testing.assert_array_equal(r[1:-1], 1.0)
    assert r[0] == r[-1] == 1.5


def test_knn_radius_scales_with_the_cloud():
    """The same point set scaled by 0.1 (far away from the first copy) has radii exactly 0.1x."""
    rng = np.random.default_rng(0)
    a = rng.random((3, 200))
    pos = np.concatenate([a, 0.1 * a + 100.0], 1).astype(np.float64)
    r = PP.knn_radius(pos, 6)
    np.testing.assert_allclose(r[200:], 0.1 * r[:200], rtol=1e-9)


def test_knn_radius_duplicates_are_floored():
    pos = np.zeros((3, 6), F)
    pos[0, 3:] = 1.0  # two triples of duplicates at distance 1
    r = PP.knn_radius(pos, 2)
    assert (r == 1e-9 * 1.0).all()  # both neighbours at distance 0 -> floor = 1e-9 x bbox diagonal


def test_morton_cube_corners_in_z_order():
    corners = np.array([[x, y, z] for z in (0, 1) for y in (0, 1) for x in (0, 1)], F).T  # index = x + 2y + 4z
    rng = np.random.default_rng(1)
    shuffled = rng.permutation(8)
    perm = PP.blocked_morton_order(corners[:, shuffled], block=8, seed=3)
    assert [int(shuffled[j]) for j in perm] == list(range(8))
    assert PP.morton_codes(corners)[7] == (1 << 63) - 1  # all 21 bits set on all three axes


def test_single_point_and_bijection_and_whole_blocks():
    assert PP.blocked_morton_order(np.zeros((3, 1), F), 4, 0).tolist() == [0]
    rng = np.random.default_rng(2)
    pos = rng.random((3, 1000)).astype(F)
    perm = PP.blocked_morton_order(pos, 64, seed=9)
    assert sorted(perm.tolist()) == list(range(1000))
    codes = PP.morton_codes(pos)
    order = sorted(range(1000), key=lambda i: (int(codes[i]), i))
    where = {p: k for k, p in enumerate(order)}
    pos_, runs = 0, []
    while pos_ < 1000:  # the output is a concatenation of whole Morton blocks (runs of `order`)
        k = where[int(perm[pos_])]
        assert k % 64 == 0
        L = min(64, 1000 - k)
        assert perm[pos_:pos_ + L].tolist() == order[k:k + L]
        runs.append(k // 64)
        pos_ += L
    assert sorted(runs) == list(range(16)) and runs != list(range(16))  # every block once, shuffled
