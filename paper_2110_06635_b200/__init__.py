"""B200-native ADOP one-pixel point rasterizer (arXiv 2110.06635): the data-parallel hot path.

Submodules:
  adop      -- ctypes binding of the C-ABI library libadop.so (include/adop.h)
  scene     -- seeded synthetic inputs (no method arithmetic)
  parallel  -- point-sharded / view-sharded orchestration over torch.distributed
The CUDA library is loaded lazily by `adop`; importing the package does not touch the GPU.
"""
