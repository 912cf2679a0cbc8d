import sys, numpy as np
sys.path.insert(0, '.')
from paper_2312_08715_b200 import b3d, configs
ctx = b3d.GpuContext(0)
def rf(k, v, t, p):
    ctx.set_camera(b3d.Intrinsics(*k.as_tuple())); mid = ctx.upload_mesh(v, t)
    d, _ = ctx.render_poses(mid, np.asarray(p, dtype=np.float64)[None], with_ids=False); return d[0]
tr = configs.cfg4(rf, b3d.voxel_to_mesh, seed=0, n_frames=12)
ctx.set_camera(b3d.Intrinsics(*tr["k"].as_tuple())); mid = ctx.upload_mesh(tr["vertices"], tr["triangles"])
st0 = tr["stages"][0]; ctx.set_likelihood([st0["noise"]], 0.1, st0["window"])
est = tr["gt"][0].copy()
def ang(a, b):
    d = min(1.0, abs(float(np.dot(a[:4], b[:4])))); return float(np.degrees(2*np.arccos(d)))
for f in range(1, 12):
    ctx.set_observation(tr["frames"][f])
    res, centers = ctx.coarse_to_fine(mid, est, tr["stages"])
    prev = est; est = centers[-1]; gt = tr["gt"][f]
    # score of gt pose vs est pose
    s_gt, _ = ctx.score_poses(mid, np.array([gt, est, prev]))
    print(f, 'cm %.3f deg %.2f | gt-vs-prev %.2f | scores gt %.1f est %.1f prev %.1f | argmax %s' % (100*np.linalg.norm(est[4:]-gt[4:]), ang(est, gt), ang(prev, gt), s_gt[0,0], s_gt[1,0], s_gt[2,0], [r.argmax for r in res]))
