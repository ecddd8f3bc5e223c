"""Point sharding over a shared (peer-memory) pyramid on the GPU: two processes, each rendering its shard
of the cloud through the C-ABI straight into the owner's keys / accum / count (CUDA IPC mapping,
adop_params.shared_pyramid = 1).  On the B200 box both processes share the one GPU -- the IPC mapping
and the kernels' reductions into another process's allocation are the same code as across NVLink; no
kernel waits on another (host barriers order the phases).  Sharded == unsharded: keys and counts
bit-exact, image within the fp32 tolerance."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q, owner, n, views):
    from paper_2110_06635_b200 import adop as A
    from paper_2110_06635_b200 import parallel as PL
    from paper_2110_06635_b200 import scene as S
    try:
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        dev = torch.device("cuda")
        w = S.workload(1, n=n, n_views=views)
        cloud = w.cloud.to(dev)
        a, b = PL.shard_range(cloud.n, world, rank, align=1024)
        r = A.Renderer(cloud.slice(a, b), w.cameras, w.poses, w.params, global_offset=a)
        sh = PL.PeerPointSharding(r, owner=owner)
        ph = PL.CudaPhases(r)
        for _ in range(2):  # the second frame checks the owner's per-frame reset
            PL.point_sharded_forward_p2p(ph, owner)
        torch.cuda.synchronize()
        if rank == owner:
            full = A.Renderer(cloud, w.cameras, w.poses, w.params)
            full.forward()
            torch.cuda.synchronize()
            res = []
            for v in range(views):
                p, f = r.pyrs[v], full.pyrs[v]
                res.append((torch.equal(p.keys, f.keys), torch.equal(p.count, f.count),
                            float((p.image - f.image).abs().max()), float(f.image.abs().max()),
                            int((f.count > 0).sum())))
            q.put(("ok", res))
        dist.barrier()
        sh.close()
        dist.destroy_process_group()
    except Exception as e:  # report instead of hanging the parent on q.get
        q.put(("error", f"rank {rank}: {type(e).__name__}: {e}"))
        raise


@pytest.mark.parametrize("owner,views", [(0, 1), (1, 4)])
def test_point_sharding_into_a_shared_pyramid_two_processes(owner, views):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, owner, 300_000, views)) for r in range(2)]
    for p in procs:
        p.start()
    status, res = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
    assert status == "ok", res
    assert all(p.exitcode == 0 for p in procs)
    for keys_eq, count_eq, err, mx, covered in res:
        assert keys_eq and count_eq
        assert err <= 1e-6 + 1e-5 * mx
        assert covered > 10_000
