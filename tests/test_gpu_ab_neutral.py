"""GPU: the bulk-copy observation staging switch (B3D_OBS_STAGE: window sums
read shared memory instead of L2) changes where data lives, never the
scores: cfg1 scored in two processes, staging on and off, bitwise equal."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
from helpers import b3d_intr, cfg1_oracle
from paper_2312_08715_b200 import b3d
w = cfg1_oracle()
ctx = b3d.GpuContext(0)
ctx.set_camera(b3d_intr(w.k))
mid = ctx.upload_mesh(w.vertices, w.triangles)
ctx.set_observation(w.observed)
out = []
if {big}:  # a 3,000-voxel blob: the vertex cache lives in global scratch
    from paper_2312_08715_b200 import configs
    from oracle import pyoracle as O
    w = configs.cfg2(lambda k, v, t, p: O.render(k, [(v, t, p)]), O.voxel_to_mesh, seed=0)
    ctx.set_camera(b3d_intr(w.k))
    mid = ctx.upload_mesh(w.vertices, w.triangles)
    ctx.set_observation(w.observed)
    g = w.stages[0]
    from paper_2312_08715_b200 import configs as C
    w.grid_poses = lambda: C.grid_poses(w.center, g["extent"], g["count"], g["rotations"], 0)[::7]
for noise, win in (([(0.01, 0.005)], 1), ([(0.01, 0.005), (0.2, 0.02)], 3), ([(0.05, 0.01)], 0)):
    ctx.set_likelihood(noise, 0.1, win)
    s, st = ctx.score_poses(mid, w.grid_poses())
    out.append(s.ravel())
np.save(sys.argv[1], np.concatenate(out))
"""


def _run(var, flag, path, big=False):
    env = dict(os.environ, **{var: flag})
    code = SCRIPT.format(root=ROOT, tests=os.path.join(ROOT, "tests"), big=big)
    r = subprocess.run([sys.executable, "-c", code, str(path)], env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return np.load(path)


def test_obs_staging_is_bitwise_neutral(tmp_path):
    a = _run("B3D_OBS_STAGE", "1", tmp_path / "on.npy")
    b = _run("B3D_OBS_STAGE", "0", tmp_path / "off.npy")
    np.testing.assert_array_equal(a.view(np.uint64), b.view(np.uint64))

