"""run_smc with the harness defaults but two objects placed (smc_extend:
a device stage 0 per distinct partial scene after resampling): wall time
and the device evaluation count, 1,000 and 200 particles."""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2312_08715_b200 import b3d, configs  # noqa: E402

ctx = b3d.GpuContext(0)
ctx.set_stream(torch.cuda.current_stream().cuda_stream)
rng = np.random.Generator(np.random.PCG64(8000))
k = configs.Intr(400.0, 400.0, 160.0, 120.0, 320, 240, 0.01, 10.0)
camera = np.array([0.0, 1.0, 0.0, 0.0, 0.0, 0.0, 0.7])
tw = th = 0.5
tv, tt, _, _ = configs.table_mesh(b3d.box_mesh, tw, th)
lib = []
for i, n in enumerate((500, 1000, 2000, 3000, 4000)):
    v, t = configs.make_mesh(configs.synth.eden_blob(n, 300 + i), b3d.voxel_to_mesh)
    lib.append((v, t, v.min(axis=0), v.max(axis=0)))
p1 = b3d.contact_to_pose(tw, th, lib[2][2], lib[2][3], 1, 0.21, 0.17, 2.2)
p2 = b3d.contact_to_pose(tw, th, lib[0][2], lib[0][3], 1, 0.05, 0.3, 0.5)
render = bench._scene_renderer(ctx, b3d)
ident = np.array([1.0, 0, 0, 0, 0, 0, 0])
depth = render(k, camera, [(tv, tt, ident), (lib[2][0], lib[2][1], p1), (lib[0][0], lib[0][1], p2)])
obs = configs.synth.noisy_observation(depth, k.far, 0.003, 0.05, 0.2, 1.5, rng, k.near)
ctx.set_camera(b3d.Intrinsics(*k.as_tuple()), camera)
table = ctx.upload_mesh(tv, tt)
mids = [ctx.upload_mesh(v, t) for v, t, _, _ in lib]
ctx.set_observation(obs)
noise = [(p, f * 0.1) for p in (0.05, 0.3, 0.8) for f in (0.25, 0.5, 1.0)]
libs = [(mids[i], lib[i][2], lib[i][3]) for i in range(len(lib))]
sched = ((10, 10, 8), [(5, 5, 5), (5, 5, 5)])
for particles in (200, 1000):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ps, le = ctx.run_smc(libs, table, tw, th, sched, noise, 0.1, 2, n_objects=2,
                         n_particles=particles, resample_threshold=0.5, seed=0)
    dt = time.perf_counter() - t0
    best = max(ps, key=lambda p: p[3])
    print(json.dumps({"particles": particles, "seconds": dt, "renders_device": ctx.last_smc_renders,
                      "log_evidence": le, "map_children": best[0]}))
