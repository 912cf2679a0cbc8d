"""The oracle's run_smc restatement (inference.cpp:398-520) on a small case:
it runs, keeps every child inside its contact support, and its weights and
log-evidence are finite (the GPU test pins the device SMC to it)."""
import numpy as np

from oracle import pyoracle as O
from smc_case import (CAMERA, K, NOISE_GRID, SCHEDULE, TABLE_H, TABLE_W, build)


def _render(k, cam, inst):
    return O.render(k, inst, camera=cam)


def test_oracle_run_smc_small_case():
    lib, (tv, tt), obs, placed = build(O.voxel_to_mesh, O.box_mesh, O.contact_to_pose, _render)
    ps, le = O.run_smc(K, CAMERA, obs, lib, (tv, tt, TABLE_W, TABLE_H), SCHEDULE, NOISE_GRID,
                       0.1, 1, n_objects=1, n_particles=4, resample_threshold=0.5, seed=9)
    assert len(ps) == 4 and np.isfinite(le)
    for children, e, lt, lw in ps:
        assert len(children) == 1 and 0 <= e < 9 and np.isfinite(lt) and np.isfinite(lw)
        obj, face, dx, dy, dt = children[0]
        lo, hi = O.rotated_bounds(lib[obj][2], lib[obj][3], face)
        assert 0 <= dx <= TABLE_W - (hi[0] - lo[0]) and 0 <= dt < 2 * np.pi
