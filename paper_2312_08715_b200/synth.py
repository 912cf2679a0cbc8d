"""Seeded synthetic inputs for the BASELINE configs (no dataset exists here).

BASELINE.json describes seeded voxel blobs, 6-DoF pose grids with von
Mises-Fisher rotation perturbations and noisy observed depth images; the
reference has no generator for any of these, so they are
defined here, deterministically from one integer seed (numpy PCG64).  They
are input generation only -- neither product nor oracle.
"""
from __future__ import annotations

import math

import numpy as np

_NBR = np.array([[-1, 0, 0], [1, 0, 0], [0, -1, 0], [0, 1, 0], [0, 0, -1], [0, 0, 1]],
                dtype=np.int64)


def _sorted_unique(v: np.ndarray) -> np.ndarray:
    # lexicographic (x, y, z) order = VoxelGrid's sorted+unique invariant
    # (geometry.hpp:71-72, geometry.cpp:100-105), which fixes triangle ids
    v = np.unique(v.astype(np.int32), axis=0)
    return np.ascontiguousarray(v, dtype=np.int32)


def eden_blob(n_voxels: int, seed: int) -> np.ndarray:
    """Compact 6-connected blob by Eden growth: start at the origin voxel and
    repeatedly occupy a uniformly chosen face-neighbour of the occupied set."""
    rng = np.random.Generator(np.random.PCG64(seed))
    occ = {(0, 0, 0)}
    frontier = []
    fset = set()

    def push_nbrs(c):
        for d in _NBR:
            nb = (c[0] + int(d[0]), c[1] + int(d[1]), c[2] + int(d[2]))
            if nb not in occ and nb not in fset:
                fset.add(nb)
                frontier.append(nb)

    push_nbrs((0, 0, 0))
    while len(occ) < n_voxels:
        i = int(rng.integers(len(frontier)))
        c = frontier[i]
        frontier[i] = frontier[-1]
        frontier.pop()
        fset.discard(c)
        occ.add(c)
        push_nbrs(c)
    return _sorted_unique(np.array(sorted(occ), dtype=np.int64))


def random_walk_blob(n_voxels: int, seed: int) -> np.ndarray:
    """Stringy 6-connected blob: a lattice random walk until n distinct voxels."""
    rng = np.random.Generator(np.random.PCG64(seed))
    occ = {(0, 0, 0)}
    c = (0, 0, 0)
    while len(occ) < n_voxels:
        d = _NBR[int(rng.integers(6))]
        c = (c[0] + int(d[0]), c[1] + int(d[1]), c[2] + int(d[2]))
        occ.add(c)
    return _sorted_unique(np.array(sorted(occ), dtype=np.int64))


def centered_origin(voxels: np.ndarray, resolution: float) -> np.ndarray:
    """Grid origin placing the blob's bounding-box centre at the model origin
    (all three axes, cf. centered_cube_grid, tests/support/shapes.cpp:41-45)."""
    lo = voxels.min(axis=0).astype(np.float64)
    hi = voxels.max(axis=0).astype(np.float64)
    return -resolution * (lo + (hi - lo + 1.0) / 2.0)


# The generators below use Python's math (the image's libm) and explicit
# sums, never numpy's SIMD transcendental / BLAS kernels: those dispatch on
# the CPU's vector extensions, so the build container and a GPU box would
# otherwise draw ulp-different rotations from the same seed, and the
# committed reference fixtures (tests/golden) would not match bit for bit.
def norm(v) -> float:
    """Euclidean norm, summed in index order."""
    s = 0.0
    for x in v:
        s += float(x) * float(x)
    return math.sqrt(s)


def uniform_quaternion(rng: np.random.Generator) -> np.ndarray:
    """Uniform random rotation: normalised 4-D Gaussian, (w, x, y, z), w >= 0."""
    q = rng.standard_normal(4)
    q /= norm(q)
    return q if q[0] >= 0 else -q


def vmf_quaternions(n: int, kappa: float, rng: np.random.Generator) -> np.ndarray:
    """n unit quaternions from a von Mises-Fisher distribution on S^3 with mean
    (1,0,0,0) and concentration kappa (Wood 1994 rejection sampler, p = 4).
    Used as rotation perturbations dq: q_hyp = q_center * dq."""
    m = 4
    b = (-2.0 * kappa + math.sqrt(4.0 * kappa * kappa + (m - 1) ** 2)) / (m - 1)
    x0 = (1.0 - b) / (1.0 + b)
    c = kappa * x0 + (m - 1) * math.log(1.0 - x0 * x0)
    out = np.zeros((n, 4), dtype=np.float64)
    for i in range(n):
        while True:
            z = float(rng.beta((m - 1) / 2.0, (m - 1) / 2.0))
            w = (1.0 - (1.0 + b) * z) / (1.0 - (1.0 - b) * z)
            u = float(rng.random())
            if kappa * w + (m - 1) * math.log(1.0 - x0 * w) - c >= math.log(u):
                break
        v = rng.standard_normal(3)
        v /= norm(v)
        out[i, 0] = w
        out[i, 1:] = math.sqrt(max(0.0, 1.0 - w * w)) * v
        out[i] /= norm(out[i])
    return out


def noisy_observation(depth: np.ndarray, far: float, sigma: float, outlier_frac: float,
                      outlier_lo: float, outlier_hi: float, rng: np.random.Generator,
                      near: float = 0.0) -> np.ndarray:
    """Observed depth: Gaussian depth noise on valid pixels, then a fraction
    of ALL pixels replaced by uniform [lo, hi] outliers (BASELINE configs)."""
    far_f = np.float32(far)
    obs = depth.astype(np.float64).copy()
    valid = depth < far_f
    obs[valid] += rng.normal(0.0, sigma, size=int(valid.sum()))
    n = obs.size
    k = int(round(outlier_frac * n))
    idx = rng.choice(n, size=k, replace=False)
    flat = obs.reshape(-1)
    flat[idx] = rng.uniform(outlier_lo, outlier_hi, size=k)
    obs = np.clip(obs, max(near, 1e-6), far).astype(np.float32)
    obs[obs >= far_f] = far_f
    return obs


def rotation_lattice(step_rad: float, extra: int = 0, kappa: float = 0.0,
                     rng: np.random.Generator = None) -> np.ndarray:
    """Rotation perturbations on a 3 x 3 x 3 lattice of rotation vectors
    step * (i, j, k), i, j, k in {-1, 0, 1} (27 quaternions, identity first),
    optionally followed by `extra` vMF(kappa) draws."""
    qs = [np.array([1.0, 0.0, 0.0, 0.0])]
    for i in (-1, 0, 1):
        for j in (-1, 0, 1):
            for k in (-1, 0, 1):
                if i == j == k == 0:
                    continue
                r = step_rad * np.array([i, j, k], dtype=np.float64)
                a = norm(r)
                qs.append(np.concatenate([[math.cos(a / 2)], math.sin(a / 2) * r / a]))
    out = np.array(qs)
    if extra:
        out = np.vstack([out, vmf_quaternions(extra, kappa, rng)])
    return out
