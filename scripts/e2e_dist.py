"""Distribution of the bench's end-to-end cfg1 step (wall clock, L2 flushed
before each step as bench.py does): mean, percentiles, max over 300 steps."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_08715_b200 import b3d, configs  # noqa: E402

ctx = b3d.GpuContext(0)


def render_fn(k, v, t, p):
    ctx.set_camera(b3d.Intrinsics(*k.as_tuple()))
    m = ctx.upload_mesh(v, t)
    return ctx.render_poses(m, np.asarray(p, dtype=np.float64)[None], with_ids=False)[0][0]


w = configs.cfg1(render_fn, b3d.voxel_to_mesh, seed=0)
ctx.set_camera(b3d.Intrinsics(*w.k.as_tuple()))
mid = ctx.upload_mesh(w.vertices, w.triangles)
ctx.set_likelihood(w.noise, w.sigma_max, w.window)
h_obs = torch.from_numpy(w.observed).pin_memory().numpy()
h_poses = torch.from_numpy(w.grid_poses()).pin_memory().numpy()
h_scores = torch.zeros((1024, 1), dtype=torch.float64).pin_memory().numpy()
h_rng = b3d.rng_seed(7)
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
for flushing in (True, False):
    for _ in range(10):
        ctx.enumerate_observed(mid, h_obs, h_poses, rng_state=h_rng, scores=h_scores)
    ts = []
    for i in range(300):
        if flushing:
            flush.fill_(float(i))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ctx.enumerate_observed(mid, h_obs, h_poses, rng_state=h_rng, scores=h_scores)
        ts.append((time.perf_counter() - t0) * 1e6)
    ts = np.array(ts)
    print(f"flush={flushing}: mean {ts.mean():.1f} us  p50 {np.median(ts):.1f}  p90 "
          f"{np.percentile(ts, 90):.1f}  p99 {np.percentile(ts, 99):.1f}  max {ts.max():.1f}  "
          f"-> {1024 / ts.mean():.2f} M hyp/s (mean)")
