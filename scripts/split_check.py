"""Split-tail A/B: cfg1 scores with and without the 2-CTA tail launch must be
bitwise equal (run twice with B3D_SPLIT_TAIL=0/1, compare the saved arrays)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_08715_b200 import b3d, configs  # noqa: E402

ctx = b3d.GpuContext(0)


def render_fn(k, v, t, p):
    ctx.set_camera(b3d.Intrinsics(*k.as_tuple()))
    m = ctx.upload_mesh(v, t)
    return ctx.render_poses(m, np.asarray(p, dtype=np.float64)[None], with_ids=False)[0][0]


out = []
for seed in (0, 1):
    w = configs.cfg1(render_fn, b3d.voxel_to_mesh, seed=seed)
    ctx.set_camera(b3d.Intrinsics(*w.k.as_tuple()))
    mid = ctx.upload_mesh(w.vertices, w.triangles)
    ctx.set_likelihood(w.noise, w.sigma_max, w.window)
    ctx.set_observation(w.observed)
    for n in (1024, 1000, 700, 296 * 2 + 10):
        s, st = ctx.score_poses(mid, w.grid_poses()[:n])
        out.append(s.copy())
    d_rot = torch.from_numpy(w.rotations).cuda()
    grid = ctx.make_grid(w.center, w.extent, w.count, d_rot, w.grid_mode)
    sc = torch.zeros((1024, 1), dtype=torch.float64, device="cuda")
    stt = torch.zeros(1024, dtype=torch.uint8, device="cuda")
    ctx.score_grid(mid, grid, sc, stt)
    out.append(sc.cpu().numpy())
np.save(sys.argv[1], np.concatenate([o.ravel() for o in out]))
