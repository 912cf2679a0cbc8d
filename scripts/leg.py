"""Run one extra bench leg and print its JSON: python scripts/leg.py bench_tracking|scene_graph|coarse_to_fine|sharded"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2312_08715_b200 import b3d, configs  # noqa: E402

ctx = b3d.GpuContext(0)
bench.LEG_CPU["enabled"] = False  # device legs only (ncu captures)


def render_fn(k, v, t, p):
    ctx.set_camera(b3d.Intrinsics(*k.as_tuple()))
    mid = ctx.upload_mesh(v, t)
    d, _ = ctx.render_poses(mid, np.asarray(p, dtype=np.float64)[None], with_ids=False)
    return d[0]


leg = sys.argv[1]
if leg == "bench_tracking":
    res = [int(x) for x in sys.argv[2:]] or [25, 50, 100, 200]
    out = bench.run_bench_tracking(ctx, b3d, configs, resolutions=res)
elif leg == "scene_graph":
    out = bench.run_scene_graph(ctx, b3d, configs)
elif leg == "coarse_to_fine":
    out = bench.run_coarse_to_fine(ctx, b3d, configs, render_fn)
elif leg == "smc":
    out = bench.run_smc_leg(ctx, b3d, configs)
elif leg == "cfg1":  # the headline batch: five score launches of configs[0]
    w = configs.cfg1(render_fn, b3d.voxel_to_mesh, seed=0)
    ctx.set_camera(b3d.Intrinsics(*w.k.as_tuple()))
    mid = ctx.upload_mesh(w.vertices, w.triangles)
    ctx.set_likelihood(w.noise, w.sigma_max, w.window)
    ctx.set_observation(torch.from_numpy(w.observed).cuda())
    grid = ctx.make_grid(w.center, w.extent, w.count, torch.from_numpy(w.rotations).cuda(),
                         w.grid_mode)
    sc = torch.zeros((1024, 1), dtype=torch.float64, device="cuda")
    st = torch.zeros(1024, dtype=torch.uint8, device="cuda")
    for _ in range(5):
        ctx.score_grid(mid, grid, sc, st)
    torch.cuda.synchronize()
    out = {"scores_sum": float(sc.sum())}
elif leg == "tracking":
    out = bench.run_tracking(ctx, b3d, configs, 40, render_fn)
else:
    out = bench.run_sharded(ctx, b3d, configs, 1, 0)
print(json.dumps(out))
