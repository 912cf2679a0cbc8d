"""Device time of the cfg1 bench step's parts (CUDA events, L2 flushed
before each sample, median of 50): the score kernel alone, the stage
reduction alone over the same 1,024 scores, and the fused
b3d_gpu_enumerate_grid step (score + reduction, PDL)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_08715_b200 import b3d, configs  # noqa: E402

ctx = b3d.GpuContext(0)
stream = torch.cuda.current_stream()
ctx.set_stream(stream.cuda_stream)


def render_fn(k, v, t, p):
    ctx.set_camera(b3d.Intrinsics(*k.as_tuple()))
    m = ctx.upload_mesh(v, t)
    return ctx.render_poses(m, np.asarray(p, dtype=np.float64)[None], with_ids=False)[0][0]


w = configs.cfg1(render_fn, b3d.voxel_to_mesh, seed=0)
ctx.set_camera(b3d.Intrinsics(*w.k.as_tuple()))
mid = ctx.upload_mesh(w.vertices, w.triangles)
ctx.set_likelihood(w.noise, w.sigma_max, w.window)
dev = torch.device("cuda", 0)
ctx.set_observation(torch.from_numpy(w.observed).to(dev))
d_rot = torch.from_numpy(w.rotations).to(dev)
grid = ctx.make_grid(w.center, w.extent, w.count, d_rot, w.grid_mode)
d_scores = torch.zeros((1024, 1), dtype=torch.float64, device=dev)
d_status = torch.zeros(1024, dtype=torch.uint8, device=dev)
d_rng = torch.from_numpy(b3d.rng_seed(7).view(np.int64)).to(dev)
d_res = torch.zeros(64, dtype=torch.uint8, device=dev)
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)


def timed(fn, n=50):
    for _ in range(5):
        fn()
    ts = []
    for i in range(n):
        flush.fill_(float(i))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn()
        b.record(stream)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return np.median(ts), np.percentile(ts, 10), np.percentile(ts, 90)


parts = [
    ("score kernel", lambda: ctx.score_grid(mid, grid, d_scores, d_status)),
    ("stage reduce", lambda: ctx.stage_reduce(d_scores, n=1024, rng_state=d_rng, out=d_res)),
    ("enumerate_grid", lambda: ctx.enumerate_grid(mid, grid, d_rng, d_res, d_scores)),
    ("score + reduce (2 calls)", lambda: (ctx.score_grid(mid, grid, d_scores, d_status),
                                          ctx.stage_reduce(d_scores, n=1024, rng_state=d_rng,
                                                           out=d_res))),
]
for name, fn in parts:
    med, p10, p90 = timed(fn)
    print(f"{name:26s} median {med:7.1f} us  p10 {p10:7.1f}  p90 {p90:7.1f}")
