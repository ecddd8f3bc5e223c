"""Work-list sizes of one config with the forward ghost listing on / off (ADOP_GHOST_FWD read once per process).
usage: ADOP_GHOST_FWD=0|1 python scripts/ghost_probe.py IDX"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2110_06635_b200 import adop as A  # noqa: E402
from paper_2110_06635_b200 import scene as S  # noqa: E402

idx = int(sys.argv[1])
w = S.workload(idx, device="cuda")
r = A.Renderer(w.cloud, w.cameras, w.poses, w.params)
P = A.pyramid_pixels(w.cameras[0].width, w.cameras[0].height, w.params.layers)
Gt = S.grad_pyramid(len(w.cameras), w.cloud.channels, P, device="cuda")
G = [Gt[v] for v in range(len(w.cameras))]


def hdr():
    off = r.ws.ptr - r.ws.buf.data_ptr()
    h = r.ws.buf[off:off + 72].cpu().numpy()
    u = lambda a, b: int(h[a:b].view(np.uint64)[0])
    return dict(resv_front=u(0, 8) & ((1 << 40) - 1), resv_back_chunks=u(0, 8) >> 40, mode=int(h[12:16].view(np.int32)[0]),
                front_ok=u(24, 32), back_ok=u(32, 40), ghosts_fwd=int(h[64:68].view(np.int32)[0]))


for k in range(3):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    ev[0].record()
    r.forward()
    ev[1].record()
    torch.cuda.synchronize()
    hf = hdr()
    ev[1].record()
    r.backward(G)
    ev[2].record()
    torch.cuda.synchronize()
    print(w.name, f"fwd {ev[0].elapsed_time(ev[1]):.3f} bwd {ev[1].elapsed_time(ev[2]):.3f}", "after fwd", hf, "after bwd", hdr(), flush=True)
