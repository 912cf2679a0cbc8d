"""CPU enqueue cost vs GPU time of the cfg1 enumerate call (host vs device buffers)."""
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
d_obs = torch.from_numpy(w.observed).cuda()
d_poses = torch.from_numpy(w.grid_poses()).cuda()
d_scores = torch.zeros((1024, 1), dtype=torch.float64, device="cuda")
d_rng = torch.from_numpy(b3d.rng_seed(7).view(np.int64)).cuda()
d_out = torch.zeros(8, dtype=torch.float64, device="cuda")
h_obs = torch.from_numpy(w.observed).pin_memory().numpy()
h_poses = torch.from_numpy(w.grid_poses()).pin_memory().numpy()
h_scores = torch.zeros((1024, 1), dtype=torch.float64).pin_memory().numpy()
h_rng = b3d.rng_seed(7)

L = ctx._L


def dev_call():
    ctx.set_observation(d_obs)
    b3d._check(L.b3d_gpu_enumerate_poses(ctx.h, mid, d_poses.data_ptr(), 1024, d_rng.data_ptr(),
                                         d_out.data_ptr(), d_scores.data_ptr()))


for _ in range(20):
    dev_call()
torch.cuda.synchronize()
cpu, gpu = [], []
for _ in range(100):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0.record()
    dev_call()
    e1.record()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    cpu.append(t1 - t0)
    gpu.append(e0.elapsed_time(e1) * 1e-3)
print(f"device buffers: enqueue {np.median(cpu)*1e6:.1f} us  gpu {np.median(gpu)*1e6:.1f} us")

hh = []
for _ in range(100):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ctx.set_observation(h_obs)
    ctx.enumerate_poses(mid, h_poses, rng_state=h_rng, scores=h_scores)
    hh.append(time.perf_counter() - t0)
print(f"host buffers: wall {np.median(hh)*1e6:.1f} us")
# pieces
d_status = torch.zeros(1024, dtype=torch.uint8, device="cuda")
pieces = [("set_observation(host pinned)", lambda: ctx.set_observation(h_obs)),
          ("set_observation(device)", lambda: ctx.set_observation(d_obs)),
          ("score_poses(device)", lambda: b3d._check(L.b3d_gpu_score_poses(
              ctx.h, mid, d_poses.data_ptr(), 1024, d_scores.data_ptr(), d_status.data_ptr()))),
          ("stage_reduce(device)", lambda: b3d._check(L.b3d_gpu_stage_reduce(
              ctx.h, d_scores.data_ptr(), 1024, 1, 0, d_rng.data_ptr(), d_out.data_ptr(), None))),
          ("synchronize only", lambda: torch.cuda.synchronize()),
          ("torch event record", lambda: torch.cuda.Event().record())]
for name, fn in pieces:
    ts = []
    for _ in range(100):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    print(f"{name}: enqueue {np.median(ts)*1e6:.1f} us")
