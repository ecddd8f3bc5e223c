"""Per-stage work counts of the depth sweep on configs[3] (needs a build with -DADOP_COUNTERS=1):
    python scripts/build_variants.py cnt=ADOP_COUNTERS=1
    ADOP_LIB=paper_2110_06635_b200/libadop_cnt.so python scripts/depth_counters.py [cfg] [cull]"""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
from paper_2110_06635_b200 import adop as A  # noqa: E402
from paper_2110_06635_b200 import scene as S  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
w = S.workload(cfg, device="cuda")
r = A.Renderer(w.cloud, w.cameras, w.poses, w.params)
if len(sys.argv) > 2 and sys.argv[2] == "cull":
    r.points.enable_tile_culling()
L = A.lib()
out = (C.c_ulonglong * 8)()
r.forward()
torch.cuda.synchronize()
L.adop_debug_depth_counts(out, 1)
r.forward()
torch.cuda.synchronize()
L.adop_debug_depth_counts(out, 1)
tiles, vt, cand, kept, hits, valid, disc, proj = list(out)[:8]
print(f"configs[{cfg}]: {len(w.cameras)} views")
print(f"tiles {tiles:,}  box-visible view-tiles {vt:,} ({100 * vt / max(tiles, 1):.1f}%)")
print(f"candidates {cand:,} ({cand / max(vt, 1):.1f} per visible tile)  kept {kept:,} ({100 * kept / max(cand, 1):.1f}% "
      f"of candidates)  layer hits {hits:,} ({hits / max(kept, 1):.2f} per kept)")
print(f"of the candidates: valid depth {valid:,} ({100 * valid / max(cand, 1):.1f}%), kept by the exact discard {disc:,} "
      f"({100 * disc / max(cand, 1):.1f}%), inside the camera's valid radius {proj:,} ({100 * proj / max(cand, 1):.1f}%), "
      f"in the image at some kept layer {kept:,} ({100 * kept / max(cand, 1):.1f}%)")
