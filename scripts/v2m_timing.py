"""Host vs device voxel_to_mesh on large grids (8f.4)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_08715_b200 import b3d  # noqa: E402

ctx = b3d.GpuContext(0)
for side in (20, 60, 100):
    r = np.arange(side)
    g = np.stack(np.meshgrid(r, r, r, indexing="ij"), -1).reshape(-1, 3).astype(np.int32)
    rng = np.random.Generator(np.random.PCG64(side))
    g = g[rng.random(g.shape[0]) < 0.7]  # porous cube: many exterior faces
    t0 = time.perf_counter()
    hv, ht = b3d.voxel_to_mesh(g, 0.005, (0, 0, 0))
    t1 = time.perf_counter()
    ctx.voxel_to_mesh(g, 0.005, (0, 0, 0))
    t2 = time.perf_counter()
    dv, dt = ctx.voxel_to_mesh(g, 0.005, (0, 0, 0))
    t3 = time.perf_counter()
    same = np.array_equal(dt, ht) and np.array_equal(dv, hv)
    print(f"{g.shape[0]:>8} voxels {ht.shape[0]:>9} triangles  host {1e3*(t1-t0):8.1f} ms  "
          f"device {1e3*(t3-t2):7.1f} ms (incl. copies)  equal={same}")
