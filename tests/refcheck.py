"""Numpy restatements of the reference's TEST oracles
(proj/tests/support/oracles.cpp) and fixtures (support/shapes.cpp), plus the
scene sampler the reference tests draw scenes with (scene_graph.cpp:144-168).

These are independent of the CPU oracle they check (oracles.hpp:3-4: "nothing
here may call into the implementation paths it is used to check"): the ray
caster and the naive likelihood loops share no code with oracle/b3d_oracle.c.
"""
from __future__ import annotations

import math

import numpy as np

TWO_PI = 6.283185307179586476925287


# --------------------------------------------------------- oracles.cpp:12-54
def raycast_depth(instances, camera, k, pose_mats):
    """Brute-force Moller-Trumbore ray casting: nearest camera-frame hit in
    [near, far), sentinel (float)far otherwise.  `pose_mats(pose) -> (R, t)`
    maps a model-to-camera pose to a rotation matrix and translation."""
    tris = []
    for verts, faces, m2c in instances:
        R, t = pose_mats(m2c)
        cam = np.asarray(verts) @ R.T + t
        tris.append(cam[np.asarray(faces, dtype=np.int64)])
    W, H = k.width, k.height
    img = np.full((H, W), np.float32(k.far), dtype=np.float32)
    if not tris:
        return img
    T = np.concatenate(tris)  # (n, 3, 3)
    v0, v1, v2 = T[:, 0], T[:, 1], T[:, 2]
    e1, e2 = v1 - v0, v2 - v0
    for v in range(H):
        for u in range(W):
            d = np.array([(u - k.cx) / k.fx, (v - k.cy) / k.fy, 1.0])
            pvec = np.cross(d, e2)
            det = np.einsum("ij,ij->i", e1, pvec)
            ok = np.abs(det) >= 1e-14
            inv = np.where(ok, 1.0 / np.where(ok, det, 1.0), 0.0)
            tvec = -v0
            bu = np.einsum("ij,ij->i", tvec, pvec) * inv
            qvec = np.cross(tvec, e1)
            bv = (qvec @ d) * inv
            tt = np.einsum("ij,ij->i", e2, qvec) * inv
            hit = ok & (bu >= 0) & (bu <= 1) & (bv >= 0) & (bu + bv <= 1) & (tt >= k.near)
            best = k.far
            if hit.any():
                best = min(best, float(tt[hit].min()))
            img[v, u] = np.float32(best)
    return img


# --------------------------------------------------------- oracles.cpp:56-78
def edge_mask(img, k, threshold=1e-3):
    H, W = img.shape
    sentinel = np.float32(k.far)
    mask = np.zeros((H, W), dtype=bool)
    for v in range(H):
        for u in range(W):
            c = img[v, u]
            edge = u == 0 or v == 0 or u == W - 1 or v == H - 1
            for dv in (-1, 0, 1):
                for du in (-1, 0, 1):
                    if edge:
                        break
                    nu, nv = u + du, v + dv
                    if nu < 0 or nv < 0 or nu >= W or nv >= H:
                        continue
                    n = img[nv, nu]
                    if (c < sentinel) != (n < sentinel) or abs(float(n) - float(c)) > threshold:
                        edge = True
            mask[v, u] = edge
    return mask


# -------------------------------------------------------- oracles.cpp:80-137
def naive_full_loglik(obs, rend, p_outlier, sigma, volume, sigma_max, printed=True):
    s2 = sigma * sigma
    total = math.log(sigma / sigma_max) if printed else math.log(1.0 / sigma_max)
    for o in obs:
        g = 0.0
        for r in rend:
            d2 = float(np.sum((np.asarray(o) - np.asarray(r)) ** 2))
            g += (2.0 * math.pi * s2) ** -1.5 * math.exp(-d2 / (2.0 * s2))
        total += math.log(p_outlier / volume + (1.0 - p_outlier) / len(rend) * g)
    return total


def naive_windowed_loglik(obs, rend, k, p_outlier, sigma, volume, sigma_max, window,
                          printed=True):
    H, W = obs.shape
    sentinel = np.float32(k.far)
    s2 = sigma * sigma

    def bp(u, v, z):
        return np.array([(u - k.cx) * z / k.fx, (v - k.cy) * z / k.fy, z])

    rend_count = int((rend < sentinel).sum())
    total = math.log(sigma / sigma_max) if printed else math.log(1.0 / sigma_max)
    for v in range(H):
        for u in range(W):
            oz = obs[v, u]
            if oz >= sentinel:
                continue
            o = bp(u, v, float(oz))
            g = 0.0
            for rv in range(max(0, v - window), min(H - 1, v + window) + 1):
                for ru in range(max(0, u - window), min(W - 1, u + window) + 1):
                    rz = rend[rv, ru]
                    if rz >= sentinel:
                        continue
                    d2 = float(np.sum((o - bp(ru, rv, float(rz))) ** 2))
                    g += (2.0 * math.pi * s2) ** -1.5 * math.exp(-d2 / (2.0 * s2))
            total += math.log(p_outlier / volume + (1.0 - p_outlier) / rend_count * g)
    return total


# ------------------------------------------------------ oracles.cpp:139-152
def quat_to_matrix(w, x, y, z):
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                     [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                     [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])


# ----------------------------------------------------- shapes.cpp (fixtures)
def grid_from_voxels(voxels, resolution):
    """x/y-centred model frame, z = 0 at the lowest layer; sorted + unique."""
    v = np.unique(np.asarray(voxels, dtype=np.int32), axis=0)
    lo, hi = v.min(axis=0), v.max(axis=0)
    origin = np.array([-resolution * (lo[0] + (hi[0] - lo[0] + 1) / 2.0),
                       -resolution * (lo[1] + (hi[1] - lo[1] + 1) / 2.0),
                       -resolution * lo[2]])
    return v, resolution, origin


def box_grid(nx, ny, nz, res):
    return grid_from_voxels([(x, y, z) for x in range(nx) for y in range(ny)
                             for z in range(nz)], res)


def centered_cube_grid(n, res):
    v, r, o = box_grid(n, n, n, res)
    o = o.copy()
    o[2] = -res * n / 2.0
    return v, r, o


def lblock_grid(res):
    vox = [(x, y, z) for x in range(6) for y in range(4) for z in range(2)]
    vox += [(x, y, z) for x in range(2) for y in range(4) for z in range(2, 5)]
    return grid_from_voxels(vox, res)


def mug_grid(res, with_handle=True):
    vox = []
    for x in range(8):
        for y in range(8):
            d = math.hypot(x - 3.5, y - 3.5)
            if d > 4.0:
                continue
            vox.append((x, y, 0))
            if d >= 2.9:
                vox += [(x, y, z) for z in range(1, 8)]
    if with_handle:
        vox += [(x, y, z) for x in range(8, 11) for y in range(3, 5) for z in range(2, 6)]
    return grid_from_voxels(vox, res)


class Model:
    """ObjectModel (scene_graph.hpp:15-27): mesh + model-frame AABB."""

    def __init__(self, verts, tris):
        self.verts = np.asarray(verts, dtype=np.float64)
        self.tris = np.asarray(tris, dtype=np.uint32)
        self.aabb_min = self.verts.min(axis=0)
        self.aabb_max = self.verts.max(axis=0)

    @property
    def extents(self):
        return self.aabb_max - self.aabb_min


def make_model(O, grid):
    v, res, origin = grid
    verts, tris = O.voxel_to_mesh(v, res, origin)
    return Model(verts, tris)


def make_table(O, w, h, thickness=0.01):
    """ObjectModel::table (scene_graph.cpp:26-35)."""
    lo = np.array([-w / 2, -h / 2, -thickness])
    hi = np.array([w / 2, h / 2, 0.0])
    verts, tris = O.box_mesh(lo, hi)
    m = Model(verts, tris)
    m.aabb_min, m.aabb_max = lo, hi
    return m


# ------------------------------------------ scene_graph.cpp:91-95,144-168
def footprint(O, obj, face):
    lo, hi = O.rotated_bounds(obj.aabb_min, obj.aabb_max, face)
    return hi[0] - lo[0], hi[1] - lo[1]


def rng_uniform_range(O, st, lo, hi):
    """Rng::uniform(lo, hi) (rng.cpp:46)."""
    return lo + (hi - lo) * O.rng_uniform(st)


def sample_scene_prior(O, st, n, library, table):
    tw, th = table.extents[0], table.extents[1]
    children = []
    for _ in range(n):
        obj = library[O.rng_uniform_int(st, len(library))]
        face = O.rng_uniform_int(st, 6) + 1
        fx, fy = footprint(O, obj, face)
        dxr, dyr = tw - fx, th - fy
        assert dxr > 0 and dyr > 0
        dx = rng_uniform_range(O, st, 0.0, dxr)
        dy = rng_uniform_range(O, st, 0.0, dyr)
        dtheta = rng_uniform_range(O, st, 0.0, TWO_PI)
        children.append((obj, face, dx, dy, dtheta))
    return children


def scene_instances(O, table, children):
    """renderer.cpp:153-162: table at identity, then children in order."""
    inst = [(table.verts, table.tris, np.array([1, 0, 0, 0, 0, 0, 0.0]))]
    tw, th = table.extents[0], table.extents[1]
    for obj, face, dx, dy, dt in children:
        pose = O.contact_to_pose(tw, th, obj.aabb_min, obj.aabb_max, face, dx, dy, dt)
        inst.append((obj.verts, obj.tris, pose))
    return inst
