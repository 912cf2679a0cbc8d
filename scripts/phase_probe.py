"""Per-phase wall time inside the camera-mode score kernel (B3D_PHASE_CLOCK
build: B3D_LIB=_ab/lib_pclk.so python scripts/phase_probe.py [res ...])."""
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


def rc(k, inst, cams):
    ctx.set_camera(b3d.Intrinsics(*k.as_tuple()))
    mids = [ctx.upload_mesh(v, t) for v, t, _ in inst]
    ctx.set_camera_scene(mids, [p for _, _, p in inst])
    return ctx.render_cameras(np.asarray(cams), with_ids=False)[0]


for res in [int(a) for a in sys.argv[1:]] or (25, 100, 200):
    seq = configs.orbit_sequence(rc, b3d.voxel_to_mesh, b3d.box_mesh, b3d.contact_to_pose,
                                 res=res, n_frames=4)
    cams = np.array([b3d.camera_pose_from_spherical(seq["distance"], a, seq["altitude"])
                     for a in seq["azimuths"]])
    frames = configs.orbit_frames(seq, cams)
    ctx.set_likelihood([seq["noise"]], seq["sigma_max"], seq["window"])
    ctx.set_observation(frames[0])
    rng = np.random.Generator(np.random.PCG64(1))
    hyp = np.array([b3d.camera_pose_from_spherical(0.9 + rng.uniform(-0.05, 0.05),
                                                   rng.uniform(0, 6), 0.7 + rng.uniform(-0.1, 0.1))
                    for _ in range(125)])
    for _ in range(3):
        ctx.score_cameras(hyp)
    buf = np.zeros((256, 8), dtype=np.int64)
    assert L.b3d_debug_phase_clock(buf.ctypes.data_as(C.POINTER(C.c_longlong))) == 0
    b = buf[:125].astype(np.float64)
    t0 = b[:, 0].min()
    d = np.diff(b, axis=1) / 1e3
    print(f"{res} px: kernel span {(b[:, 7].max() - t0)/1e3:.1f} us; CTA start spread "
          f"{(b[:, 0].max() - t0)/1e3:.1f} us")
    for i, n in enumerate(names):
        print(f"   {n:12s} median {np.median(d[:, i]):7.2f} us  max {d[:, i].max():7.2f} us")
