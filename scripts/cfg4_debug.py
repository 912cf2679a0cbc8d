"""Where does the device cfg4 chain first differ from the reference fixture?"""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import pyoracle as O
from paper_2312_08715_b200 import b3d, configs
g = np.load("tests/golden/ref_cfg4.npz")
tr = configs.cfg4(lambda k, v, t, p: O.render(k, [(v, t, p)]), O.voxel_to_mesh, seed=0)
ctx = b3d.GpuContext(0)
ctx.set_camera(b3d.Intrinsics(*tr["k"].as_tuple()))
mid = ctx.upload_mesh(tr["vertices"], tr["triangles"])
st0 = tr["stages"][0]
ctx.set_likelihood([st0["noise"]], 0.1, st0["window"])
est = tr["gt"][0].copy()
i = 0
for f in range(1, 100):
    ctx.set_observation(tr["frames"][f])
    res, centers = ctx.coarse_to_fine(mid, est, tr["stages"])
    for s, stg in enumerate(tr["stages"]):
        host = configs.grid_poses(centers[s], stg["extent"], stg["count"], stg["rotations"], 0)
        ok_c = np.array_equal(centers[s], g["centers"][i])
        ok_next = np.array_equal(centers[s + 1], host[res[s].argmax])
        if not ok_c or not ok_next or res[s].argmax != g["argmax"][i]:
            print(f"frame {f} stage {s} i {i}: centre_eq {ok_c} next_eq_host {ok_next} "
                  f"argmax dev {res[s].argmax} ref {g['argmax'][i]} max dev {res[s].max_score!r} "
                  f"ref top2 {g['top2'][i]}")
            print("  dev centre", centers[s].tolist())
            print("  ref centre", g["centers"][i].tolist())
        i += 1
    est = centers[-1]
print("done", i)
