"""Kernel time vs hypothesis count on the cfg1 workload (tail-effect probe).
python scripts/hyp_scaling.py  -> one line per N: us, us/hyp, Mhyp/s"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_08715_b200 import b3d, configs  # noqa: E402

ctx = b3d.GpuContext(0)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
ctx.set_stream(stream.cuda_stream)


def render_fn(k, v, t, p):
    ctx.set_camera(b3d.Intrinsics(*k.as_tuple()))
    m = ctx.upload_mesh(v, t)
    d, _ = ctx.render_poses(m, np.asarray(p, dtype=np.float64)[None], with_ids=False)
    return d[0]


w = configs.cfg1(render_fn, b3d.voxel_to_mesh, seed=0)
ctx.set_camera(b3d.Intrinsics(*w.k.as_tuple()))
mid = ctx.upload_mesh(w.vertices, w.triangles)
ctx.set_likelihood(w.noise, w.sigma_max, w.window)
ctx.set_observation(torch.from_numpy(w.observed).cuda())
base = w.grid_poses()
for n in [int(a) for a in (sys.argv[1:] or [148, 296, 592, 888, 1024, 1184, 2048, 4096, 8192])]:
    poses = torch.from_numpy(np.tile(base, (n // 1024 + 1, 1))[:n].copy()).cuda()
    sc = torch.zeros((n, 1), dtype=torch.float64, device="cuda")
    stt = torch.zeros(n, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        ctx.score_poses(mid, poses, sc, stt)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    e0.record(stream)
    for _ in range(reps):
        ctx.score_poses(mid, poses, sc, stt)
    e1.record(stream)
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / reps
    print(f"N={n:6d} {us:9.1f} us  {us / n * 1e3:7.1f} ns/hyp  {n / us:6.2f} Mhyp/s", flush=True)
