#!/usr/bin/env python
"""Benchmark of the B200-native ADOP rasterizer hot path (arXiv 2110.06635).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...     (point-sharded, one rank per GPU)

Workload = BASELINE.json configs[3] (the one `metric` is quoted on): 100M points of the synthetic room
(S = 50 m), C = 4, 1920x1080 pinhole, 5 layers, stochastic discard on, one view, forward only.
A step is one forward frame: depth pass, [min-allreduce of the keys], blend pass, [sum-allreduce of the
blended features and counts], resolve.  With N GPUs every rank owns a 100M-point shard of one
N*100M-point cloud (weak scaling; global indices rank*1e8 + i keep keys shard-invariant).

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "points rasterized/sec and ms/frame, 100M pts 5-layer 1080p fwd; % HBM roofline"
WORKLOAD = "room100M_fwd (BASELINE.json configs[3]): 100M pts/GPU, C=4, 1920x1080 pinhole, 5 layers, discard on"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--points", type=int, default=100_000_000, help="points per GPU")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="eager launches in the timed region (single GPU)")
    ap.add_argument("--comm", choices=["nccl", "p2p"], default="nccl",
                    help="N > 1 point sharding: NCCL all-reduces of private pyramids, or every shard reducing "
                         "straight into rank 0's pyramid over peer memory (DESIGN.md section 8)")
    ap.add_argument("--scatter", action="store_true",
                    help="N > 1 point sharding (nccl): reduce-scatter accum/count (one packed collective per view) "
                         "and resolve only this rank's pixel slice, instead of the SUM all-reduce (DESIGN.md section 8)")
    ap.add_argument("--keys32", action="store_true",
                    help="N > 1 point sharding (nccl): MIN-exchange only the 32-bit depth words (11 MB/view instead of "
                         "22 MB; the winner indices stay shard-local; DESIGN.md section 8)")
    ap.add_argument("--mode", choices=["point", "view"], default="point",
                    help="point: configs[3] forward, point-sharded over N ranks (the headline); view: configs[4] "
                         "training step (fwd+bwd, 16 views) view-sharded over N ranks with one SUM all-reduce of the "
                         "point gradients and an all-gather of the pose rows")
    ap.add_argument("--cpu-sample", type=int, default=25_000_000)
    ap.add_argument("--ref-sample", type=int, default=4_000_000)
    return ap.parse_args()


# --------------------------------------------------------------------------- #
# clocks sampler (nvidia-smi during the timed region)
# --------------------------------------------------------------------------- #
class Clocks:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,power.draw")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (FileNotFoundError, OSError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[2:6]):
                if val.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def phys_index(local_rank: int) -> int:
    vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
    ids = [v for v in vis.split(",") if v.strip()]
    if local_rank < len(ids) and ids[local_rank].strip().isdigit():
        return int(ids[local_rank])
    return local_rank


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md)"


def traffic_from_profiles():
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as f:
            return json.load(f)
    except (OSError, ValueError):
        return {}


# --------------------------------------------------------------------------- #
# our arm
# --------------------------------------------------------------------------- #
def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_2110_06635_b200 import adop as A
    from paper_2110_06635_b200 import scene as S

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    N = args.points
    w = S.workload(3, device=dev, n=N, shard=rank)
    cloud = w.cloud
    C = cloud.channels
    goff = rank * N
    prm = w.params
    cams, poses = w.cameras, w.poses
    pts = A.Points.from_cloud(cloud, global_offset=goff)
    ap = A.Params(prm, C)
    pyrs = A.alloc_pyramids(cams, prm.layers, C, dev)
    cap = A.default_record_capacity(N, len(cams), prm.layers, prm.discard)
    ws = A.Workspace(pts, cams, ap, dev, cap)
    stream = torch.cuda.current_stream(dev)
    p2p = world > 1 and args.comm == "p2p"
    rd_pyrs = pyrs  # buffers this rank reads back (count, image): a non-owner's own under p2p
    if p2p:  # rank 0's pyramid is shared: the others map its keys / accum / count (CUDA IPC)
        ap.s.shared_pyramid = 1
        obj = [[(A.ipc_export(p.keys), A.ipc_export(p.accum), A.ipc_export(p.count)) for p in pyrs]
               if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        if rank != 0:
            own = rd_pyrs = pyrs
            pyrs = [A.PeerPyramid(A.ipc_open(*k), A.ipc_open(*a), A.ipc_open(*c), q.image.data_ptr(), q.width,
                                  q.height, q.layers) for (k, a, c), q in zip(obj[0], own)]

    rs_scratch = None
    if world > 1 and args.scatter and not p2p:
        from paper_2110_06635_b200 import parallel as PL
        Pp = pyrs[0].count.numel()
        rs_scratch = torch.empty(world * PL.pixel_chunk(Pp, world) * (C + 1), dtype=torch.float32, device=dev)

    calls = {}

    def cl(p):  # marshalled descriptors per points object, built once (no per-phase host marshalling)
        if id(p) not in calls:
            calls[id(p)] = A._Call(p, cams, poses, ap, pyrs)
        return calls[id(p)]

    def p2p_step(ev=None, points=None):  # same event slots as step(): the barriers take the collectives' places
        pts_ = pts if points is None else points
        def sync_barrier():
            torch.cuda.synchronize(dev)
            dist.barrier(device_ids=[local_rank])
        if ev is not None:
            ev[0].record(stream)
        if rank == 0:
            A.clear_pyramid(cams, prm.layers, C, pyrs, stream)
        sync_barrier()
        A.forward_depth(pts_, cams, poses, ap, pyrs, ws, stream, cl(pts_))
        if ev is not None:
            ev[1].record(stream)
        sync_barrier()
        if ev is not None:
            ev[2].record(stream)
        A.forward_blend(pts_, cams, poses, ap, pyrs, ws, stream, cl(pts_))
        if ev is not None:
            ev[3].record(stream)
        sync_barrier()
        if ev is not None:
            ev[4].record(stream)
        if rank == 0:
            A.forward_resolve(pts_, cams, poses, ap, pyrs, ws, stream, cl(pts_))
        if ev is not None:
            ev[5].record(stream)

    def step(ev=None, s=None, points=None):
        if p2p:
            return p2p_step(ev, points)
        pts_ = pts if points is None else points
        s = stream if s is None else s
        if ev is not None:
            ev[0].record(s)
        A.forward_depth(pts_, cams, poses, ap, pyrs, ws, s, cl(pts_))
        if ev is not None:
            ev[1].record(s)
        if world > 1:
            for p in pyrs:
                if args.keys32:
                    from paper_2110_06635_b200 import parallel as PL
                    PL.min_depth_words(p.keys)
                else:
                    dist.all_reduce(p.keys, op=dist.ReduceOp.MIN)
        if ev is not None:
            ev[2].record(s)
        A.forward_blend(pts_, cams, poses, ap, pyrs, ws, s, cl(pts_))
        if ev is not None:
            ev[3].record(s)
        sl = None
        if world > 1:
            from paper_2110_06635_b200 import parallel as PL
            if args.scatter:
                sl = PL.reduce_scatter_accum(pyrs, scratch=rs_scratch)
            else:
                for p in pyrs:
                    dist.all_reduce(p.ac, op=dist.ReduceOp.SUM)
        if ev is not None:
            ev[4].record(s)
        if sl is not None:
            A.forward_resolve_range(pts_, cams, poses, ap, pyrs, ws, sl[0], sl[1], s, cl(pts_))
        else:
            A.forward_resolve(pts_, cams, poses, ap, pyrs, ws, s, cl(pts_))
        if ev is not None:
            ev[5].record(s)

    # Single GPU: the frame's launches are captured once into two CUDA graphs (depth phase | blend +
    # resolve) and replayed; the timed region holds only the replays and one event pair around each
    # depth phase (for the roofline).  N > 1 runs the phases eagerly with the collectives in between.
    graphs = None
    if world == 1 and not args.no_graph:
        gs = torch.cuda.Stream(dev)
        gd, gr = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
        with torch.cuda.stream(gs):
            step(s=gs)
            torch.cuda.synchronize(dev)
            with torch.cuda.graph(gd, stream=gs):
                A.forward_depth(pts, cams, poses, ap, pyrs, ws, gs)
            with torch.cuda.graph(gr, stream=gs):
                A.forward_blend(pts, cams, poses, ap, pyrs, ws, gs)
                A.forward_resolve(pts, cams, poses, ap, pyrs, ws, gs)
        torch.cuda.synchronize(dev)
        graphs = (gd, gr)

    def timed_step(ev):
        if graphs is None:
            step(ev)
            return
        ev[0].record(stream)
        graphs[0].replay()
        ev[1].record(stream)
        graphs[1].replay()
        ev[5].record(stream)

    def barrier():
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier(device_ids=[local_rank])
        torch.cuda.synchronize(dev)

    for _ in range(max(3, args.warmup)):
        step()
    barrier()
    records, overflow = ws.stats(stream)
    # preheat ~0.4 s under the clock sampler, then the timed region
    clocks = Clocks(phys_index(local_rank))
    clocks.start()
    t0 = time.time()
    while time.time() - t0 < 0.4:
        step()
        torch.cuda.synchronize(dev)
    barrier()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(6)] for _ in range(args.steps)]
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record(stream)
    for k in range(args.steps):
        timed_step(evs[k])
    end.record(stream)
    barrier()
    clk = clocks.stop()
    total_ms = start.elapsed_time(end)
    depth_ms = statistics.mean(e[0].elapsed_time(e[1]) for e in evs)
    per_step = sorted(e[0].elapsed_time(e[5]) for e in evs)  # frame by frame (each frame's own event pair)
    q = lambda f: per_step[min(len(per_step) - 1, int(f * (len(per_step) - 1) + 0.5))]
    # phase breakdown (eager, every phase bracketed by events): a separate pass after the timed region
    bevs = [[torch.cuda.Event(enable_timing=True) for _ in range(6)] for _ in range(min(args.steps, 20))]
    for e in bevs:
        step(e)
    barrier()
    ph = [[e[i].elapsed_time(e[i + 1]) for e in bevs] for i in range(5)]
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_per_step = float(t.item()) / args.steps

    # the same frames with tile culling (precomputed per-tile bounds, adop_tile_bounds): results identical,
    # tiles outside the frustum are neither loaded nor processed (static-scene rendering)
    pts.enable_tile_culling(stream)
    for _ in range(3):
        step()
    barrier()
    cs, ce = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    cevs = [[torch.cuda.Event(enable_timing=True) for _ in range(6)] for _ in range(args.steps)]
    cs.record(stream)
    for k in range(args.steps):
        step(cevs[k])
    ce.record(stream)
    barrier()
    _, _, _ = ws.stats3(stream)
    tiles_read = ws.tiles_read
    culled_ms = cs.elapsed_time(ce) / args.steps
    culled_depth = statistics.mean(e[0].elapsed_time(e[1]) for e in cevs)
    pts.s.tile_bounds = None  # back to the full sweep for the e2e leg
    nb_scatter = None
    if world > 1 and args.scatter:  # each rank holds the global counts of its pixel slice only (collective)
        from paper_2110_06635_b200 import parallel as PL
        a_, b_ = PL.pixel_range(pyrs[0].count.numel(), world, rank)
        nb = torch.tensor([float(sum(float(p.count[a_:b_].sum()) for p in pyrs))], device=dev)
        dist.all_reduce(nb)
        nb_scatter = int(nb.item())
    out = {}
    if rank == 0:
        P = A.pyramid_pixels(cams[0].width, cams[0].height, prm.layers)
        # algorithmic bytes:
        #   depth phase (k_clear<KEYS> + k_depth_async): position 12 B + radius 4 B per point read once,
        #   keys 8 B per pixel written once (survivor records are this design's intermediate, not counted);
        #   frame: B_fwd = N (12 + 4) + N_blend 4C + P (8 + 4C + 4), N_blend = sum of the counts.
        alg = N * 16 + P * 8
        n_blend = nb_scatter if nb_scatter is not None else int(sum(float(p.count.sum()) for p in rd_pyrs))
        alg_frame = N * 16 + n_blend * 4 * C + P * (8 + 4 * C + 4)
        peak, peak_src = peaks()
        achieved = alg / (depth_ms * 1e-3) / 1e9
        tr = traffic_from_profiles().get("depth_phase_bytes")
        out = {
            "metric": METRIC, "value": N * world / (ms_per_step * 1e-3), "unit": "points/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": WORKLOAD, "points_per_gpu": N, "points_total": N * world, "channels": C,
                       "layers": prm.layers, "resolution": "1920x1080", "views": 1, "discard": True,
                       "gamma": prm.gamma, "alpha": prm.alpha,
                       "parallelism": (f"point-sharded x{world} ({args.comm}{', 32-bit depth words' if args.keys32 else ''}"
                                        f"{', reduce-scatter + slice resolve' if args.scatter else ''})"
                                       if world > 1 else "single GPU"),
                       "l2": "inputs (1.6 GB/GPU positions+radii) exceed the 126 MB L2; no flush needed",
                       "record_slots_per_frame": records, "record_overflow": overflow},
            "timing": ("CUDA graph replays (depth | blend+resolve) with an event pair around each depth phase"
                       if graphs is not None else "eager C-ABI calls, events around every phase"),
            "ms_per_step_stats": {"median": statistics.median(per_step), "p10": q(0.1), "p90": q(0.9),
                                  "min": per_step[0], "max": per_step[-1], "frames": len(per_step),
                                  "note": "per-frame event pairs; ms_per_step is the whole timed region / steps"},
            "phases_ms": {"depth": statistics.mean(ph[0]), "key_allreduce": statistics.mean(ph[1]),
                          "blend": statistics.mean(ph[2]), "accum_allreduce": statistics.mean(ph[3]),
                          "resolve": statistics.mean(ph[4])},
            "roofline": {"kernel": "depth phase (k_clear<KEYS> + k_depth_async<PINHOLE, 1 view>)", "bound": "hbm",
                         "achieved": achieved, "peak": peak, "peak_source": peak_src, "unit": "GB/s",
                         "frac": achieved / peak, "frac_of_nominal_8TBs": achieved / 8000.0,
                         "algorithmic_bytes": alg, "traffic": tr,
                         "timing": "CUDA events on the launch stream around the depth phase, mean over the timed steps"},
            "frame_roofline": {"bound": "hbm", "algorithmic_bytes": alg_frame, "n_blend": n_blend,
                               "achieved": alg_frame / (ms_per_step * 1e-3) / 1e9, "peak": peak, "unit": "GB/s",
                               "frac": alg_frame / (ms_per_step * 1e-3) / 1e9 / peak},
            "tile_culled": {"note": "same frames with precomputed per-tile bounds (adop_tile_bounds, untimed like the "
                                    "Morton order): tiles outside the frustum are not loaded; identical results",
                            "ms_per_step": culled_ms, "value": N * world / (culled_ms * 1e-3), "depth_ms": culled_depth,
                            "tiles_read": tiles_read, "tiles": (N + 255) // 256,
                            "bytes_read_depth": tiles_read * 256 * 16 + ((N + 255) // 256) * 32 + P * 8},
            "gpu_launches": 5 * args.steps,
            "clocks": clk,
        }
    return out, (dev, step, pts, cloud, cams, poses, prm, rd_pyrs, ws, stream, barrier, N, C)


def run_e2e(args, ctx, rank, world, local_rank):
    """Same frame through the public API with HOST inputs, all inside the timed region: H2D of the shard's
    positions and radii from pinned memory, the forward, D2H of the image pyramid.  The descriptors stay in
    pinned host memory and are passed to the API as they are (adop_points.feat may be host memory, UVA):
    the blend reads only the survivors' descriptors over PCIe.  `copy_all` also copies every descriptor
    to the device first (the plain 3.2 GB upload)."""
    import torch
    import torch.distributed as dist

    from paper_2110_06635_b200 import adop as A
    dev, step, pts, cloud, cams, poses, prm, pyrs, ws, stream, barrier, N, C = ctx
    h_pos = cloud.pos.cpu().pin_memory()
    h_rad = cloud.radius.cpu().pin_memory()
    h_feat = cloud.feat.cpu().pin_memory()
    h_img = torch.empty_like(pyrs[0].image, device="cpu").pin_memory()
    pts_h = A.Points(cloud.pos, cloud.radius, h_feat, pts.s.global_offset)  # descriptors read in place
    K = max(3, min(args.steps, 10))

    def zero_copy_step():
        cloud.pos.copy_(h_pos, non_blocking=True)
        cloud.radius.copy_(h_rad, non_blocking=True)
        step(points=pts_h)
        h_img.copy_(pyrs[0].image, non_blocking=True)

    def copy_all_step():
        cloud.pos.copy_(h_pos, non_blocking=True)
        cloud.radius.copy_(h_rad, non_blocking=True)
        cloud.feat.copy_(h_feat, non_blocking=True)
        step()
        h_img.copy_(pyrs[0].image, non_blocking=True)

    def timed(fn):
        fn()
        barrier()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        for _ in range(K):
            fn()
        e.record(stream)
        barrier()
        t = torch.tensor([s.elapsed_time(e) / K], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    ms_all = timed(copy_all_step)
    ms = timed(zero_copy_step)
    n_blend = int(sum(float(p.count.sum()) for p in pyrs))
    pos_bytes = h_pos.numel() * 4 + h_rad.numel() * 4
    return {"value": N * world / (ms * 1e-3), "unit": "points/s", "ms_per_step": ms, "steps": K,
            "h2d_bytes_per_step": pos_bytes + n_blend * 32, "d2h_bytes_per_step": h_img.numel() * 4,
            "h2d_note": "positions + radii copied (cudaMemcpyAsync); descriptors read in place from pinned host "
                        "memory by the blend: <= one 32-B sector per blended point (n_blend = sum of counts)",
            "copy_all": {"value": N * world / (ms_all * 1e-3), "ms_per_step": ms_all,
                         "h2d_bytes_per_step": pos_bytes + h_feat.numel() * 4}}


def cpu_baseline(args, ctx):
    """The CPU oracle (oracle/adop_oracle.c, as it stands) on bounded samples of the same cloud: once with one
    thread and once with OpenMP on all host cores (per-point work in parallel, reductions serial in point
    order: the results do not depend on the thread count).  `value` is the all-core rate."""
    from oracle import oracle as O
    dev, step, pts, cloud, cams, poses, prm, pyrs, ws, stream, barrier, N, C = ctx

    def run(n_s, threads):
        used = O.set_threads(threads)
        opts = O.Points.from_cloud(cloud.slice(0, n_s).to("cpu"))
        t0 = time.perf_counter()
        O.forward(opts, cams, poses, prm)
        return time.perf_counter() - t0, used

    n1 = min(args.cpu_sample // 5, N)
    dt1, _ = run(n1, 1)
    # size the all-core sample for ~10 s at the expected rate, capped at the whole cloud
    cores = os.cpu_count() or 1
    n_all = int(min(N, max(n1, 10.0 * n1 / dt1 * max(1.0, 0.5 * cores))))
    dt, used = run(n_all, 0)
    O.set_threads(1)
    return {"value": n_all / dt, "unit": "points/s", "cores": used, "kind": "oracle",
            "os_cpu_count": cores, "omp_threads": used,
            "sample": f"first {n_all:,} points of the blocked-Morton-shuffled cloud (random spatial blocks), 1 view "
                      f"1920x1080, 5 layers: full oracle forward (depth, blend, resolve) on {used} threads, {dt:.2f} s",
            "seconds": dt, "ms_per_frame_100M": dt / n_all * N * 1e3,
            "single_thread": {"value": n1 / dt1, "cores": 1, "points": n1, "seconds": dt1,
                              "ms_per_frame_100M": dt1 / n1 * N * 1e3}}


def run_secondary(args, dev):
    """Other BASELINE configs timed with the same kernels (context lines, not the headline)."""
    import torch
    from paper_2110_06635_b200 import adop as A
    from paper_2110_06635_b200 import scene as S
    res = {}
    for idx, K in ((1, 20), (2, 10), (4, 5)):
        w = S.workload(idx, device=dev)
        r = A.Renderer(w.cloud, w.cameras, w.poses, w.params)
        G = None
        if w.backward:
            P = A.pyramid_pixels(w.cameras[0].width, w.cameras[0].height, w.params.layers)
            Gt = S.grad_pyramid(len(w.cameras), w.cloud.channels, P, device=dev)
            G = [Gt[v] for v in range(len(w.cameras))]
            r.alloc_grads()

        def one():
            r.forward()
            if G is not None:
                r.backward(G)
        for _ in range(3):
            one()
        torch.cuda.synchronize()
        # back to back (the host enqueues ahead; no synchronization between iterations)
        evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(K)]
        for ev in evs:
            ev[0].record()
            r.forward()
            ev[1].record()
            if G is not None:
                r.backward(G)
            ev[2].record()
        torch.cuda.synchronize()
        fw = [ev[0].elapsed_time(ev[1]) for ev in evs]
        bw = [ev[1].elapsed_time(ev[2]) for ev in evs]
        V = len(w.cameras)
        fms, bms = statistics.median(fw), statistics.median(bw)
        res[w.name] = {"config": f"BASELINE.json configs[{idx}]", "points": w.cloud.n, "views": V,
                       "fwd_ms": fms, "bwd_ms": bms if G is not None else None,
                       "point_views_per_s": w.cloud.n * V / ((fms + (bms if G is not None else 0)) * 1e-3)}
        # rooflines of the whole forward / backward call (SURVEY.md §8(d) B_fwd, B_bwd; HBM-bound)
        peak, _ = peaks()
        N, C = w.cloud.n, w.cloud.channels
        P = A.pyramid_pixels(w.cameras[0].width, w.cameras[0].height, w.params.layers)
        n_blend = int(sum(float(p.count.sum()) for p in r.pyrs))
        b_fwd = N * 16 + n_blend * 4 * C + V * P * (8 + 4 * C + 4)
        res[w.name]["fwd_roofline"] = {"bound": "hbm", "algorithmic_bytes": b_fwd, "n_blend": n_blend,
                                       "achieved": b_fwd / (fms * 1e-3) / 1e9, "peak": peak, "unit": "GB/s",
                                       "frac": b_fwd / (fms * 1e-3) / 1e9 / peak}
        if G is not None:
            _, n_ghost, _ = r.ws.stats3()
            # positions + radii re-read, features of kept ghost entries, d_tau and d_x written once,
            # per pixel G, I, count and key read
            b_bwd = N * 16 + n_ghost * 4 * C + N * (4 * C + 12) + V * P * (4 * C + 4 * C + 4 + 8)
            res[w.name]["bwd_roofline"] = {"bound": "hbm", "algorithmic_bytes": b_bwd, "ghost_entries": n_ghost,
                                           "achieved": b_bwd / (bms * 1e-3) / 1e9, "peak": peak, "unit": "GB/s",
                                           "frac": b_bwd / (bms * 1e-3) / 1e9 / peak}
        if idx == 2:  # NEXT-4 preprocessing (untimed setup of the path) on this 10M cloud
            res["preprocess_10M"] = time_preprocess(w.cloud)
        del r, w, G
        torch.cuda.empty_cache()
    return res


def time_preprocess(cloud):
    """Blocked Morton shuffle (order + gather) and kNN world radius (k = 8) on the GPU, CUDA events."""
    import torch
    from paper_2110_06635_b200 import adop as A
    pts = A.Points(cloud.pos, cloud.radius, cloud.feat, normal=cloud.normal)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    out = {}
    for rep in range(2):  # second repetition is timed
        ev[0].record()
        perm = A.blocked_morton_order(pts, 1024, seed=1)
        ev[1].record()
        q = A.apply_order(pts, perm)
        ev[2].record()
        rad = A.knn_radius(q, 8)
        ev[3].record()
        torch.cuda.synchronize()
        out = {"points": cloud.n, "morton_order_ms": ev[0].elapsed_time(ev[1]),
               "apply_order_ms": ev[1].elapsed_time(ev[2]), "knn_radius_k8_ms": ev[2].elapsed_time(ev[3]),
               "median_radius_m": float(rad.median())}
        del perm, q, rad
    return out


# --------------------------------------------------------------------------- #
# --mode view: the configs[4] training step, view-sharded
# --------------------------------------------------------------------------- #
VIEW_METRIC = "point-views/sec and ms/step, 50M pts x 16 views 1024^2 OpenCV8, 5 layers, fwd+bwd training step"
VIEW_WORKLOAD = ("room50M_16view_fwdbwd (BASELINE.json configs[4]): 50M pts, C=4, 16 views 1024^2 OpenCV8, 5 layers, "
                 "discard on, ghosts 0.25, forward + backward (d_feat, d_pos, d_pose)")


def run_view(args, rank, world, local_rank):
    import dataclasses

    import torch
    import torch.distributed as dist

    from paper_2110_06635_b200 import adop as A
    from paper_2110_06635_b200 import parallel as PL
    from paper_2110_06635_b200 import scene as S

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    w = S.workload(4, device=dev)
    V = len(w.cameras)
    a, b = PL.view_range(V, world, rank)
    prm = dataclasses.replace(w.params, view_id_base=a)
    cams, poses = w.cameras[a:b], w.poses[a:b]
    N, C = w.cloud.n, w.cloud.channels
    r = A.Renderer(w.cloud, cams, poses, prm)
    buf, d_feat, d_pos = PL.grad_buffer(N, C, dev)  # one SUM all-reduce of d_feat ++ d_pos
    r.d_feat, r.d_pos = d_feat, d_pos
    r.d_pose = torch.empty(b - a, 6, dtype=torch.float64, device=dev)
    P = A.pyramid_pixels(cams[0].width, cams[0].height, prm.layers)
    Gt = S.grad_pyramid(V, C, P, device=dev)[a:b].contiguous()
    G = [Gt[v] for v in range(b - a)]
    stream = torch.cuda.current_stream(dev)
    counts = [PL.view_range(V, world, q) for q in range(world)]
    width = max(y - x for x, y in counts)
    pose_buf = torch.zeros(width, 6, dtype=torch.float64, device=dev)
    gathered = [torch.empty_like(pose_buf) for _ in range(world)]

    def step(ev=None):
        if ev is not None:
            ev[0].record(stream)
        r.forward()
        if ev is not None:
            ev[1].record(stream)
        r.backward(G)
        if ev is not None:
            ev[2].record(stream)
        if world > 1:
            dist.all_reduce(buf, op=dist.ReduceOp.SUM)
            pose_buf[: b - a].copy_(r.d_pose)
            dist.all_gather(gathered, pose_buf)
        if ev is not None:
            ev[3].record(stream)

    def barrier():
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier(device_ids=[local_rank])
        torch.cuda.synchronize(dev)

    for _ in range(max(3, args.warmup)):
        step()
    barrier()
    clocks = Clocks(phys_index(local_rank))
    clocks.start()
    t0 = time.time()
    while time.time() - t0 < 0.5:  # under the clock sampler (nvidia-smi takes a moment to start)
        step()
        torch.cuda.synchronize(dev)
    barrier()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record(stream)
    for k in range(args.steps):
        step(evs[k])
    end.record(stream)
    barrier()
    clk = clocks.stop()
    t = torch.tensor([start.elapsed_time(end)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item()) / args.steps
    per = sorted(e[0].elapsed_time(e[3]) for e in evs)
    fwd_ms = statistics.median(e[0].elapsed_time(e[1]) for e in evs)
    bwd_ms = statistics.median(e[1].elapsed_time(e[2]) for e in evs)
    comm_ms = statistics.median(e[2].elapsed_time(e[3]) for e in evs)
    # e2e: this rank's upstream gradient pyramids copied from pinned host memory every step, d_pose read back
    hG = Gt.cpu().pin_memory()
    hpose = torch.empty(V, 6, dtype=torch.float64).pin_memory()

    def e2e_step():
        Gt.copy_(hG, non_blocking=True)
        step()
        hpose[: b - a].copy_(r.d_pose, non_blocking=True)

    e2e_step()
    barrier()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    K = max(3, min(args.steps, 10))
    s0.record(stream)
    for _ in range(K):
        e2e_step()
    s1.record(stream)
    barrier()
    te = torch.tensor([s0.elapsed_time(s1) / K], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    out = None
    if rank == 0:
        peak, peak_src = peaks()
        n_blend = int(sum(float(p.count.sum()) for p in r.pyrs))
        _, n_ghost, _ = r.ws.stats3()
        Vl = b - a
        b_fwd = N * 16 + n_blend * 4 * C + Vl * P * (8 + 4 * C + 4)
        b_bwd = N * 16 + n_ghost * 4 * C + N * (4 * C + 12) + Vl * P * (4 * C + 4 * C + 4 + 8)
        q = lambda f: per[min(len(per) - 1, int(f * (len(per) - 1) + 0.5))]
        out = {
            "metric": VIEW_METRIC, "value": N * V / (ms * 1e-3), "unit": "point-views/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": VIEW_WORKLOAD, "points": N, "views_total": V, "views_per_rank": Vl,
                       "parallelism": f"view-sharded x{world}" if world > 1 else "single GPU",
                       "l2": "inputs (0.8 GB positions+radii, 0.8 GB descriptors) exceed the 126 MB L2"},
            "phases_ms_median_rank0": {"forward": fwd_ms, "backward": bwd_ms, "grad_allreduce_pose_allgather": comm_ms},
            "ms_per_step_stats": {"median": statistics.median(per), "p10": q(0.1), "p90": q(0.9), "steps": len(per)},
            "roofline": {"kernel": "whole fwd+bwd step of rank 0 (SURVEY §8(d) B_fwd + B_bwd)", "bound": "hbm",
                         "achieved": (b_fwd + b_bwd) / ((fwd_ms + bwd_ms) * 1e-3) / 1e9, "peak": peak,
                         "peak_source": peak_src, "unit": "GB/s",
                         "frac": (b_fwd + b_bwd) / ((fwd_ms + bwd_ms) * 1e-3) / 1e9 / peak,
                         "algorithmic_bytes": b_fwd + b_bwd, "traffic": None},
            "gpu_launches": 16 * args.steps,  # 7 forward + 9 backward kernels per step (launch list, profiles/r02)
            "clocks": clk,
            "e2e": {"value": N * V / (float(te.item()) * 1e-3), "unit": "point-views/s", "ms_per_step": float(te.item()),
                    "h2d_bytes_per_step": Gt.numel() * 4, "d2h_bytes_per_step": Vl * 6 * 8,
                    "h2d_note": "this rank's upstream image-pyramid gradients from pinned host memory; d_pose read back"},
            "comm": {"allreduce_bytes": buf.numel() * 4 if world > 1 else 0,
                     "model": "T(G) = T_compute(V/G views) + T_allreduce(1.4 GB) + T_allgather (DESIGN.md section 8)"},
        }
    return out


# --------------------------------------------------------------------------- #
# reference arm: the CPU oracle (this tier has no reference implementation)
# --------------------------------------------------------------------------- #
def run_reference(args, rank, world):
    if rank != 0:
        return None
    import torch
    from oracle import oracle as O
    from paper_2110_06635_b200 import scene as S
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    w = S.workload(3, device=dev, n=args.points)
    n_s = min(args.ref_sample, args.points)
    sub = w.cloud.slice(0, n_s).to("cpu")
    del w.cloud
    opts = O.Points.from_cloud(sub)
    threads = O.set_threads(0)  # the box's host cores (results do not depend on the count)
    for _ in range(args.warmup):
        O.forward(opts, w.cameras, w.poses, w.params)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        O.forward(opts, w.cameras, w.poses, w.params)
    dt = (time.perf_counter() - t0) / args.steps
    v = n_s / dt
    return {"impl": "reference", "metric": METRIC, "value": v, "unit": "points/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD, "points_per_gpu": args.points, "sample_points_per_step": n_s},
            "cpu_baseline": {"value": v, "unit": "points/s", "cores": threads, "kind": "oracle",
                             "os_cpu_count": os.cpu_count(),
                             "sample": f"first {n_s:,} points of configs[3]'s cloud per step, full oracle forward "
                                       f"on {threads} threads"},
            "e2e": {"value": v, "unit": "points/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def nccl_summary(path):
    """Whether NCCL set up NVLink SHARP (NVLS) and which algorithms its tuner reported (rank 0's log)."""
    try:
        txt = open(path).read()
    except OSError:
        return {"log": None}
    lines = [l.strip() for l in txt.splitlines()]
    nvls = [l for l in lines if "NVLS" in l]
    return {"log": path, "nvls_lines": len(nvls), "nvls_enabled": any("NVLS" in l and ("enabled" in l.lower() or
                                                                                       "multicast" in l.lower() or
                                                                                       "comm" in l.lower())
                                                                       for l in nvls),
            "nvls_sample": nvls[:3], "version": next((l for l in lines if "NCCL version" in l), None)}


def main():
    args = parse()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        out = run_reference(args, rank, world)
        if out is not None:
            print(json.dumps(out), flush=True)
        return
    import torch
    import torch.distributed as dist
    nccl_log = None
    if world > 1:
        # NCCL's own log (to a file, not stdout) tells whether the collectives ran on NVLink SHARP (NVLS)
        if "NCCL_DEBUG" not in os.environ:
            nccl_log = f"/tmp/adop_bench_nccl_{os.getpid()}_rank{rank}.log"
            os.environ.update({"NCCL_DEBUG": "INFO", "NCCL_DEBUG_SUBSYS": "INIT,TUNING", "NCCL_DEBUG_FILE": nccl_log})
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    if args.mode == "view":
        out = run_view(args, rank, world, local_rank)
        if rank == 0:
            if nccl_log:
                out["nccl"] = nccl_summary(nccl_log)
            print(json.dumps(out), flush=True)
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return
    out, ctx = run_ours(args, rank, world, local_rank)
    if not args.no_e2e:
        e2e = run_e2e(args, ctx, rank, world, local_rank)
        if rank == 0:
            out["e2e"] = e2e
    if rank == 0:
        if not args.no_cpu_baseline and world == 1:
            out["cpu_baseline"] = cpu_baseline(args, ctx)
        if not args.no_secondary and world == 1:
            dev = ctx[0]
            del ctx
            out["secondary"] = run_secondary(args, dev)
    if world > 1 and not args.no_secondary:
        # the other partitioning of the north star in the same N-GPU run: the configs[4] training step,
        # view-sharded (16 views over N ranks, SUM of the point gradients), so the driver's scaling run measures both
        ctx = None
        torch.cuda.empty_cache()
        vargs = argparse.Namespace(**{**vars(args), "steps": min(args.steps, 10), "warmup": 3})
        try:  # a secondary measurement: it must not cost the headline line
            vout = run_view(vargs, rank, world, local_rank)
            if rank == 0:
                keep = ("metric", "value", "unit", "ms_per_step", "phases_ms_median_rank0", "ms_per_step_stats",
                        "roofline", "config", "comm")
                out["view_sharded"] = {k: vout[k] for k in keep if k in vout}
        except Exception as exc:  # noqa: BLE001
            if rank == 0:
                out["view_sharded"] = {"error": f"{type(exc).__name__}: {exc}"[:300]}
    if rank == 0:
        if nccl_log:
            out["nccl"] = nccl_summary(nccl_log)
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
