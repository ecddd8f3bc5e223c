"""Plain CPU oracle of the preprocessing steps before the hot path.

TEST INFRASTRUCTURE ONLY: imported by tests/ alone; it shares no code with paper_2110_06635_b200/csrc/.

  * world-space radius r_world of every point "inside its local neighborhood" (§4.4): the
    median distance to its k nearest neighbours (reading R33), by brute force over all pairs in fp64;
  * the blocked Morton shuffle (§4.5 "adopted the proposed blocked-morton-shuffle"), reading
    R34: quantize every position to 21 bits per axis over the cloud's bounding box (fp32, pinned order),
    interleave into a 63-bit Morton code, sort stably by code (ties by index), cut the sorted sequence into
    blocks of B points and order the blocks by (h(seed, block), block), h = the R11 hash finalizer.
"""
from __future__ import annotations

import numpy as np

F = np.float32


def knn_radius(pos: np.ndarray, k: int) -> np.ndarray:
    """Median distance to the k nearest other points (fp64, all pairs), floored at 1e-9 x bbox diagonal."""
    p = np.asarray(pos, dtype=np.float64)
    n = p.shape[1]
    assert n >= k + 1
    diag = float(np.linalg.norm(p.max(1) - p.min(1)))
    out = np.empty(n)
    for i in range(n):
        d = np.sqrt(((p - p[:, i:i + 1]) ** 2).sum(0))
        d[i] = np.inf
        out[i] = np.median(np.sort(d)[:k])
    return np.maximum(out, 1e-9 * diag)


def _split3(v: int) -> int:
    r = 0
    for b in range(21):
        r |= ((v >> b) & 1) << (3 * b)
    return r


def morton_codes(pos: np.ndarray) -> np.ndarray:
    """63-bit codes: q_a = trunc(fl(fl(fl(x_a - lo_a) / fl(hi_a - lo_a)) * (2^21 - 1))) per axis (fp32), bits
    interleaved x (bit 0), y (bit 1), z (bit 2) from the least significant end."""
    p = np.asarray(pos, dtype=F)
    lo, hi = p.min(1), p.max(1)
    codes = np.zeros(p.shape[1], dtype=np.uint64)
    for i in range(p.shape[1]):
        c = 0
        for a in range(3):
            ext = F(hi[a] - lo[a])
            t = F(F(p[a, i] - lo[a]) / ext) if ext > 0 else F(0.0)
            q = int(F(t * F(2097151.0)))
            q = min(max(q, 0), 2097151)
            c |= _split3(q) << a
        codes[i] = c
    return codes


def _mix32(x: int) -> int:
    x &= 0xFFFFFFFF
    x ^= x >> 16
    x = (x * 0x7FEB352D) & 0xFFFFFFFF
    x ^= x >> 15
    x = (x * 0x846CA68B) & 0xFFFFFFFF
    x ^= x >> 16
    return x


def block_key(seed: int, b: int) -> int:
    """Hash of block b: mix32(b ^ mix32(lo32(seed) + 0x9E3779B9 * 4)) (R34; the 4th hash stream)."""
    salt = _mix32((seed & 0xFFFFFFFF) + ((0x9E3779B9 * 4) & 0xFFFFFFFF))
    return _mix32((b & 0xFFFFFFFF) ^ salt)


def blocked_morton_order(pos: np.ndarray, block: int, seed: int) -> np.ndarray:
    """Permutation perm (new position j holds old point perm[j]) of the blocked Morton shuffle (R34)."""
    codes = morton_codes(pos)
    n = len(codes)
    order = sorted(range(n), key=lambda i: (int(codes[i]), i))
    nb = (n + block - 1) // block
    blocks = sorted(range(nb), key=lambda b: (block_key(seed, b), b))
    perm = []
    for b in blocks:
        perm.extend(order[b * block: min(n, (b + 1) * block)])
    return np.asarray(perm, dtype=np.int64)
