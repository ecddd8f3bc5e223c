"""The library's NCCL communicator (adop_comm_*, include/adop.h) inside the fused calls.  This run has one GPU, so
the communicators have one rank: every collective is then an identity, and the results must equal the calls
without a communicator bit for bit (keys, counts) / exactly (floats: a one-rank SUM copies).  The multi-rank
orchestration of the same exchanges is covered with gloo (tests/test_parallel_gloo.py)."""
import dataclasses

import numpy as np
import pytest
import torch

from paper_2110_06635_b200 import adop as A
from paper_2110_06635_b200 import scene as S

from .parity import grads_for, keys_u64

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("mode,flags", [(A.SHARD_POINTS, 0), (A.SHARD_POINTS, A.COMM_KEYS32), (A.SHARD_VIEWS, 0)])
def test_one_rank_communicator_is_an_identity(mode, flags):
    w = S.workload(2, n=150_013, n_views=3)
    G = [g.cuda() for g in grads_for(w.cameras, w.params.layers, w.cloud.channels)]
    cloud = w.cloud.to("cuda")
    ref = A.Renderer(cloud, w.cameras, w.poses, w.params, intrinsics=True)
    ref.forward()
    ref.backward(G)
    comm = A.Comm(1, 0, A.Comm.unique_id(), mode, flags)
    try:
        r = A.Renderer(cloud, w.cameras, w.poses, w.params, intrinsics=True, comm=comm)
        r.forward()
        r.backward(G)
        torch.cuda.synchronize()
    finally:
        comm.close()
    for p, q in zip(r.pyrs, ref.pyrs):
        assert np.array_equal(keys_u64(p.keys), keys_u64(q.keys))
        assert torch.equal(p.count, q.count)  # the images' fp32 sums follow the atomics' order
        assert torch.allclose(p.image, q.image, rtol=1e-6, atol=1e-7)
    assert torch.allclose(r.d_feat, ref.d_feat, rtol=0, atol=1e-6) and torch.allclose(r.d_pos, ref.d_pos, rtol=1e-5, atol=1e-5)
    assert torch.allclose(r.d_pose, ref.d_pose, rtol=1e-9, atol=1e-9)
