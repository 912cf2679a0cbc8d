"""Per-stage cost of camera tracking at each bench-tracking resolution:
GPU time of one 125-camera score launch (device buffers, events) vs the
per-frame wall time of track_camera."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_08715_b200 import b3d, configs  # noqa: E402

ctx = b3d.GpuContext(0)
L = ctx._L


def rc(k, inst, cams):
    ctx.set_camera(b3d.Intrinsics(*k.as_tuple()))
    mids = [ctx.upload_mesh(v, t) for v, t, _ in inst]
    ctx.set_camera_scene(mids, [p for _, _, p in inst])
    return ctx.render_cameras(np.asarray(cams), with_ids=False)[0]


for res in [int(a) for a in sys.argv[1:]] or (25, 50, 100, 200):
    seq = configs.orbit_sequence(rc, b3d.voxel_to_mesh, b3d.box_mesh, b3d.contact_to_pose,
                                 res=res, n_frames=40)
    cams = np.array([b3d.camera_pose_from_spherical(seq["distance"], a, seq["altitude"])
                     for a in seq["azimuths"]])
    frames = configs.orbit_frames(seq, cams)
    ctx.set_likelihood([seq["noise"]], seq["sigma_max"], seq["window"])
    ctx.set_observation(frames[0])
    rng = np.random.Generator(np.random.PCG64(1))
    hyp = np.array([b3d.camera_pose_from_spherical(0.9 + rng.uniform(-0.05, 0.05),
                                                   rng.uniform(0, 6), 0.7 + rng.uniform(-0.1, 0.1))
                    for _ in range(125)])
    d_h = torch.from_numpy(hyp).cuda()
    d_s = torch.zeros((125, 1), dtype=torch.float64, device="cuda")
    d_st = torch.zeros(125, dtype=torch.uint8, device="cuda")
    f = lambda: b3d._check(L.b3d_gpu_score_cameras(ctx.h, d_h.data_ptr(), 125, d_s.data_ptr(),
                                                   d_st.data_ptr()))
    for _ in range(5):
        f()
    ts = []
    for _ in range(30):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        f()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    est, ms = ctx.track_camera(frames, cams[0])
    print(f"{res:4d} px: score_cameras(125) gpu {np.median(ts):6.1f} us;  track frame "
          f"{np.median(ms[1:])*1e3:6.1f} us (3 stages)")
