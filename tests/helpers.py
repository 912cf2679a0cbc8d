"""Shared test helpers: intrinsics factories and the CUDA <-> oracle glue."""
import math

import numpy as np

from paper_2312_08715_b200 import b3d, configs


def square_k(res, fov_deg=60.0, near=0.1, far=5.0):
    """test_renderer.cpp:18-27"""
    f = res / (2.0 * math.tan(fov_deg * math.pi / 360.0))
    return configs.Intr(f, f, (res - 1) / 2.0, (res - 1) / 2.0, res, res, near, far)


def make_k(w, h, f, near, far):
    """test_likelihood.cpp:19-30"""
    return configs.Intr(f, f, (w - 1) / 2.0, (h - 1) / 2.0, w, h, near, far)


def b3d_intr(k):
    return b3d.Intrinsics(*k.as_tuple())


def cfg1_oracle(seed=0, blob="eden"):
    from oracle import pyoracle as O
    rf = lambda k, v, t, p: O.render(k, [(v, t, p)])
    return configs.cfg1(rf, O.voxel_to_mesh, seed=seed, blob=blob)


def rel_err(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return np.abs(a - b) / np.maximum(np.abs(b), 1e-300)
