"""Where the end-to-end (host buffers) step spends its time (cfg1)."""
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
for _ in range(20):
    ctx.set_observation(h_obs)
    ctx.enumerate_poses(mid, h_poses, rng_state=h_rng, scores=h_scores)
ta, tb = [], []
for _ in range(200):
    t0 = time.perf_counter()
    ctx.set_observation(h_obs)
    t1 = time.perf_counter()
    ctx.enumerate_poses(mid, h_poses, rng_state=h_rng, scores=h_scores)
    t2 = time.perf_counter()
    ta.append(t1 - t0)
    tb.append(t2 - t1)
print(f"set_observation {np.median(ta)*1e6:.1f} us   enumerate_poses {np.median(tb)*1e6:.1f} us "
      f"total {np.median(np.array(ta)+np.array(tb))*1e6:.1f} us")
# device-only reference: same calls with device buffers
d_obs = torch.from_numpy(w.observed).cuda()
d_poses = torch.from_numpy(w.grid_poses()).cuda()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(200):
    ctx.set_observation(d_obs)
    ctx.enumerate_poses(mid, h_poses, rng_state=h_rng, scores=h_scores)
print(f"device obs + host poses {1e6*(time.perf_counter()-t0)/200:.1f} us")
