"""Host cost of the public API per frame (configs[1], 4 views): synchronized frames, back-to-back frames,
and the host time of one forward() call."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2110_06635_b200 import adop as A  # noqa: E402
from paper_2110_06635_b200 import scene as S  # noqa: E402

idx = int(sys.argv[1]) if len(sys.argv) > 1 else 1
w = S.workload(idx, device="cuda")
r = A.Renderer(w.cloud, w.cameras, w.poses, w.params)
for _ in range(5):
    r.forward()
torch.cuda.synchronize()
K = 50
t0 = time.perf_counter()
for _ in range(K):
    r.forward()
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"host per forward() {1e3 * (t1 - t0) / K:.3f} ms; back-to-back frames {1e3 * (t2 - t0) / K:.3f} ms")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(K):
    r.forward()
e1.record()
torch.cuda.synchronize()
print(f"GPU time per frame back-to-back {e0.elapsed_time(e1) / K:.3f} ms")
