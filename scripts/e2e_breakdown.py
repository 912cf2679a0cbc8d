"""Where the end-to-end cfg1 step's time goes (host wall clock, median of 200):
the full boundary call with host buffers, the same with device-resident
inputs, the bare ctypes round trip, the observation upload alone, and the
device-only step (CUDA events)."""
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
L = ctx._L
h_obs = torch.from_numpy(w.observed).pin_memory().numpy()
h_poses = torch.from_numpy(w.grid_poses()).pin_memory().numpy()
h_scores = torch.zeros((1024, 1), dtype=torch.float64).pin_memory().numpy()
h_rng = b3d.rng_seed(7)
d_obs = torch.from_numpy(w.observed).cuda()
d_poses = torch.from_numpy(w.grid_poses()).cuda()
res = b3d.StageResult()


def wall(fn, n=200):
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        fn()
        ts.append((time.perf_counter() - t0) * 1e6)
    return float(np.median(ts)), float(np.percentile(ts, 90))


def full():
    ctx.enumerate_observed(mid, h_obs, h_poses, rng_state=h_rng, scores=h_scores)


def raw_full():
    b3d._check(L.b3d_gpu_enumerate_observed(ctx.h, mid, h_obs.ctypes.data, h_poses.ctypes.data,
                                            1024, h_rng.ctypes.data, b3d.C.addressof(res),
                                            h_scores.ctypes.data))


def raw_no_scores():
    b3d._check(L.b3d_gpu_enumerate_observed(ctx.h, mid, h_obs.ctypes.data, h_poses.ctypes.data,
                                            1024, h_rng.ctypes.data, b3d.C.addressof(res), None))


def dev_inputs():
    b3d._check(L.b3d_gpu_enumerate_observed(ctx.h, mid, d_obs.data_ptr(), d_poses.data_ptr(),
                                            1024, h_rng.ctypes.data, b3d.C.addressof(res), None))


def obs_only():
    b3d._check(L.b3d_gpu_set_observation(ctx.h, h_obs.ctypes.data))
    b3d._check(L.b3d_gpu_synchronize(ctx.h))


def sync_only():
    b3d._check(L.b3d_gpu_synchronize(ctx.h))


for name, fn in [("full (python wrapper)", full), ("full raw ctypes", raw_full),
                 ("raw, no score read-back", raw_no_scores), ("device obs+poses", dev_inputs),
                 ("set_observation + sync", obs_only), ("synchronize only", sync_only)]:
    med, p90 = wall(fn)
    print(f"{name:28s} median {med:7.1f} us   p90 {p90:7.1f} us")

# device time of the full call
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ctx.set_stream(torch.cuda.current_stream().cuda_stream)
ts = []
for _ in range(50):
    torch.cuda.synchronize()
    e0.record()
    raw_full()
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) * 1e3)
print(f"{'device span of the call':28s} median {np.median(ts):7.1f} us")
