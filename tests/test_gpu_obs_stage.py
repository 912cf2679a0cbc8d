"""GPU: the bulk-copy observation staging (B3D_OBS_STAGE) changes where the
window sums read the observation from, never the scores: cfg1 and a
base-scene case scored in two processes, staging on and off, are bitwise
equal."""
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
for noise, win in (([(0.01, 0.005)], 1), ([(0.01, 0.005), (0.2, 0.02)], 3), ([(0.05, 0.01)], 0)):
    ctx.set_likelihood(noise, 0.1, win)
    s, st = ctx.score_poses(mid, w.grid_poses())
    out.append(s.ravel())
np.save(sys.argv[1], np.concatenate(out))
"""


def _run(flag, path):
    env = dict(os.environ, B3D_OBS_STAGE=flag)
    code = SCRIPT.format(root=ROOT, tests=os.path.join(ROOT, "tests"))
    r = subprocess.run([sys.executable, "-c", code, str(path)], env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return np.load(path)


def test_obs_staging_is_bitwise_neutral(tmp_path):
    a = _run("1", tmp_path / "on.npy")
    b = _run("0", tmp_path / "off.npy")
    np.testing.assert_array_equal(a.view(np.uint64), b.view(np.uint64))
