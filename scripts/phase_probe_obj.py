"""Per-phase time inside the object-mode score kernel (B3D_PHASE_CLOCK build):
cfg1 (1,024 hyps, window 1) and cfg4 (8,192 hyps, window 2).
B3D_LIB=_ab/lib_pclk.so python scripts/phase_probe_obj.py"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_08715_b200 import b3d, configs  # noqa: E402

ctx = b3d.GpuContext(0)
L = ctx._L
names = ["prologue+A", "B vertices", "zinit", "raster (warps)", "huge (CTA)", "D1 count",
         "D2+D3 score"]


def render_fn(k, v, t, p):
    ctx.set_camera(b3d.Intrinsics(*k.as_tuple()))
    m = ctx.upload_mesh(v, t)
    return ctx.render_poses(m, np.asarray(p, dtype=np.float64)[None], with_ids=False)[0][0]


def report(tag, reader, n_cta):
    buf = np.zeros((256, 8), dtype=np.int64)
    assert getattr(L, reader)(buf.ctypes.data_as(C.POINTER(C.c_longlong))) == 0
    b = buf[:min(n_cta, 256)].astype(np.float64)
    d = np.diff(b, axis=1) / 1e3
    print(f"{tag}: per-hypothesis phase times (last hypothesis of CTAs 0..{b.shape[0]-1})")
    tot = np.median(d.sum(axis=1))
    for i, n in enumerate(names):
        print(f"   {n:15s} median {np.median(d[:, i]):7.2f} us  ({100*np.median(d[:, i])/tot:4.1f} %)")


w = configs.cfg1(render_fn, b3d.voxel_to_mesh, seed=0)
ctx.set_camera(b3d.Intrinsics(*w.k.as_tuple()))
mid = ctx.upload_mesh(w.vertices, w.triangles)
ctx.set_observation(w.observed)
ctx.set_likelihood(w.noise, w.sigma_max, w.window)
P = w.grid_poses()
for _ in range(3):
    ctx.score_poses(mid, P)
report("cfg1", "b3d_debug_phase_clock_w1", 296)

tr = configs.cfg4(render_fn, b3d.voxel_to_mesh, seed=0, n_frames=2)
ctx.set_camera(b3d.Intrinsics(*tr["k"].as_tuple()))
mid = ctx.upload_mesh(tr["vertices"], tr["triangles"])
st0 = tr["stages"][0]
ctx.set_likelihood([st0["noise"]], 0.1, st0["window"])
ctx.set_observation(tr["frames"][1])
rng = np.random.Generator(np.random.PCG64(3))
gt = tr["gt"][1]
P = np.repeat(gt[None], 8192, axis=0)
P[:, 4:] += rng.uniform(-0.015, 0.015, size=(8192, 3))
for _ in range(3):
    ctx.score_poses(mid, P)
report("cfg4", "b3d_debug_phase_clock_w2", 296)

# cfg2: 3,000-voxel blob at 200x200, stage windows 3 and 1
w2 = configs.cfg2(render_fn, b3d.voxel_to_mesh, seed=0)
ctx.set_camera(b3d.Intrinsics(*w2.k.as_tuple()))
mid = ctx.upload_mesh(w2.vertices, w2.triangles)
ctx.set_observation(w2.observed)
P = np.repeat(w2.gt_pose[None], 32768, axis=0)
P[:, 4:] += rng.uniform(-0.02, 0.02, size=(32768, 3))
for win, reader in ((3, "b3d_debug_phase_clock_w3"), (1, "b3d_debug_phase_clock_w1")):
    ctx.set_likelihood([(0.01, 0.01)], 0.1, win)
    for _ in range(2):
        ctx.score_poses(mid, P)
    report(f"cfg2 window {win}", reader, 296)
