"""Seeded synthetic workloads (BASELINE configs) are deterministic and have
the advertised structure."""
import numpy as np

from helpers import cfg1_oracle
from paper_2312_08715_b200 import synth


def _connected(vox):
    occ = set(map(tuple, vox))
    start = next(iter(occ))
    seen, stack = {start}, [start]
    while stack:
        x, y, z = stack.pop()
        for d in ((1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0), (0, 0, 1), (0, 0, -1)):
            n = (x + d[0], y + d[1], z + d[2])
            if n in occ and n not in seen:
                seen.add(n)
                stack.append(n)
    return len(seen) == len(occ)


def test_blobs_are_seeded_6_connected_and_sorted():
    for gen in (synth.eden_blob, synth.random_walk_blob):
        a, b = gen(1000, 0), gen(1000, 0)
        assert np.array_equal(a, b) and a.shape == (1000, 3)
        assert _connected(a)
        assert np.array_equal(a, np.unique(a, axis=0))  # sorted + unique


def test_vmf_concentration():
    rng = np.random.Generator(np.random.PCG64(0))
    q = synth.vmf_quaternions(4000, 1000.0, rng)
    assert np.allclose(np.linalg.norm(q, axis=1), 1.0)
    # E[1 - w] ~ 3 / (2 kappa) for large kappa on S^3
    assert abs((1 - q[:, 0]).mean() - 1.5e-3) < 2e-4


def test_cfg1_workload_shape_and_determinism():
    w1, w2 = cfg1_oracle(), cfg1_oracle()
    assert np.array_equal(w1.observed, w2.observed)
    assert w1.n_hyp == 1024 and w1.grid_poses().shape == (1024, 7)
    assert w1.observed.shape == (120, 160)
    valid = (w1.observed < np.float32(10.0)).mean()
    assert 0.10 < valid < 0.20  # ~10% outliers + the object
    p = w1.grid_poses()
    assert np.allclose(np.linalg.norm(p[:, :4], axis=1), 1.0)
    assert abs(p[:, 4].min() + 0.02) < 1e-12 and abs(p[:, 6].max() - 0.62) < 1e-12
