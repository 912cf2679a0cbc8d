"""GPU time (events) of score/enumerate with device vs host buffers; results equal?"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_08715_b200 import b3d, configs  # noqa: E402

ctx = b3d.GpuContext(0)
ctx.set_stream(torch.cuda.current_stream().cuda_stream)


def render_fn(k, v, t, p):
    ctx.set_camera(b3d.Intrinsics(*k.as_tuple()))
    m = ctx.upload_mesh(v, t)
    return ctx.render_poses(m, np.asarray(p, dtype=np.float64)[None], with_ids=False)[0][0]


w = configs.cfg1(render_fn, b3d.voxel_to_mesh, seed=0)
ctx.set_camera(b3d.Intrinsics(*w.k.as_tuple()))
mid = ctx.upload_mesh(w.vertices, w.triangles)
ctx.set_likelihood(w.noise, w.sigma_max, w.window)
L = ctx._L
P = w.grid_poses()
print("poses", P.shape, P.dtype, P.flags["C_CONTIGUOUS"])
d_obs = torch.from_numpy(w.observed).cuda()
d_poses = torch.from_numpy(P).cuda()
d_scores = torch.zeros((1024, 1), dtype=torch.float64, device="cuda")
d_status = torch.zeros(1024, dtype=torch.uint8, device="cuda")
h_scores = np.zeros((1024, 1))
h_status = np.zeros(1024, dtype=np.uint8)
ctx.set_observation(d_obs)


def gtime(fn, n=50):
    for _ in range(5):
        fn()
    ts = []
    for _ in range(n):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return np.median(ts)


t_dev = gtime(lambda: b3d._check(L.b3d_gpu_score_poses(ctx.h, mid, d_poses.data_ptr(), 1024,
                                                       d_scores.data_ptr(), d_status.data_ptr())))
t_host = gtime(lambda: b3d._check(L.b3d_gpu_score_poses(ctx.h, mid, P.ctypes.data, 1024,
                                                        h_scores.ctypes.data,
                                                        h_status.ctypes.data)))
print(f"score_poses device {t_dev:.1f} us   host {t_host:.1f} us")
print("scores equal:", np.array_equal(d_scores.cpu().numpy(), h_scores),
      "status sums", int(d_status.sum()), int(h_status.sum()), "score range", h_scores.min(), h_scores.max())
