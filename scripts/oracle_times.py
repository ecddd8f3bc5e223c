"""Oracle (oracle/adop_oracle.c, OpenMP) wall time per BASELINE config on the host cores, all threads and one thread,
plus the GPU time of the same call (CUDA events) -- the reporting table of BASELINE.md.
usage: python scripts/oracle_times.py [--skip4]"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import oracle as O  # noqa: E402
from paper_2110_06635_b200 import adop as A  # noqa: E402
from paper_2110_06635_b200 import scene as S  # noqa: E402

out = {"os_cpu_count": os.cpu_count()}
for idx in (0, 1, 2, 3, 4):
    if idx == 4 and "--skip4" in sys.argv:
        continue
    w = S.workload(idx)
    V, C = len(w.cameras), w.cloud.channels
    P = A.pyramid_pixels(w.cameras[0].width, w.cameras[0].height, w.params.layers)
    G = S.grad_pyramid(V, C, P).numpy() if w.backward else None
    pts = O.Points.from_cloud(w.cloud)
    rec = {"points": w.cloud.n, "views": V, "backward": bool(w.backward)}
    for threads in ((0, 1) if idx in (0, 1, 2) else (0,)):
        used = O.set_threads(threads)
        t0 = time.perf_counter()
        f = O.forward(pts, w.cameras, w.poses, w.params)
        t1 = time.perf_counter()
        if G is not None:
            O.backward(pts, w.cameras, w.poses, w.params, f, G)
        t2 = time.perf_counter()
        rec[f"oracle_{'all' if threads == 0 else '1'}"] = {"threads": used, "fwd_ms": (t1 - t0) * 1e3,
                                                          "bwd_ms": (t2 - t1) * 1e3 if G is not None else None}
    # the GPU: fwd (+ bwd), median of 20 back-to-back iterations (CUDA events)
    wd = S.workload(idx, device="cuda")
    r = A.Renderer(wd.cloud, wd.cameras, wd.poses, wd.params)
    Gd = [torch.from_numpy(G[v]).cuda() for v in range(V)] if G is not None else None
    for _ in range(3):
        r.forward()
        if Gd is not None:
            r.backward(Gd)
    torch.cuda.synchronize()
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(20)]
    for e in ev:
        e[0].record()
        r.forward()
        e[1].record()
        if Gd is not None:
            r.backward(Gd)
        e[2].record()
    torch.cuda.synchronize()
    rec["gpu_fwd_ms"] = float(np.median([e[0].elapsed_time(e[1]) for e in ev]))
    rec["gpu_bwd_ms"] = float(np.median([e[1].elapsed_time(e[2]) for e in ev])) if Gd is not None else None
    out[f"configs[{idx}]"] = rec
    print(json.dumps({f"configs[{idx}]": rec}), flush=True)
    del r, wd, Gd
    torch.cuda.empty_cache()
json.dump(out, open("gpurun_out/oracle_times.json", "w"), indent=1)
