"""Pins the oracle's pose math, meshes and scene-graph poses to the
reference tests test_geometry.cpp and test_scene_graph.cpp."""
import math

import numpy as np
import pytest

import refcheck as RC

PI = 3.141592653589793238462643


def rot_angle(a, b):
    """Geodesic angle between two rotations (rotation_angle_between,
    geometry.cpp:33-36, computes 2 acos|a.b|, which loses ~1e-8 to rounding
    next to 0; the numerically stable form 4 atan2(|a-b|, |a+b|) (sign of
    the quaternion folded in) keeps the reference tests' 1e-12 bars
    meaningful)."""
    qa, qb = np.asarray(a[:4]), np.asarray(b[:4])
    if np.dot(qa, qb) < 0:
        qb = -qb
    return 4.0 * math.atan2(np.linalg.norm(qa - qb), np.linalg.norm(qa + qb))


def test_compose_identity_and_inverse(oracle):
    """test_geometry.cpp:33-49"""
    st = oracle.rng_seed(7)
    ident = np.array([1, 0, 0, 0, 0, 0, 0.0])
    for _ in range(20):
        ax = [oracle.rng_normal(st), oracle.rng_normal(st), oracle.rng_normal(st)]
        ang = RC.rng_uniform_range(oracle, st, -PI, PI)
        t = [oracle.rng_normal(st), oracle.rng_normal(st), oracle.rng_normal(st)]
        p = oracle.from_axis_angle(ax, ang, t)
        left = oracle.compose(ident, p)
        assert rot_angle(left, p) < 1e-12
        assert np.linalg.norm(left[4:] - p[4:]) < 1e-12
        rnd = oracle.compose(p, oracle.inverse(p))
        assert rot_angle(rnd, ident) < 1e-9
        assert np.linalg.norm(rnd[4:]) < 1e-9
        assert abs(np.linalg.norm(rnd[:4]) - 1.0) < 1e-9


def test_compose_matches_matrix_oracle(oracle):
    """test_geometry.cpp:51-88"""
    a = oracle.from_axis_angle([0, 0, 1], PI / 2)
    ab = oracle.compose(a, a)
    mab = RC.quat_to_matrix(*a[:4]) @ RC.quat_to_matrix(*a[:4])
    np.testing.assert_allclose(oracle.rotation_matrix(ab), mab, rtol=1e-12, atol=1e-15)
    assert rot_angle(ab, oracle.from_axis_angle([0, 0, 1], PI)) < 1e-12
    st = oracle.rng_seed(13)
    for _ in range(25):
        p = oracle.from_axis_angle([oracle.rng_normal(st) for _ in range(3)],
                                   RC.rng_uniform_range(oracle, st, -PI, PI))
        q = oracle.from_axis_angle([oracle.rng_normal(st) for _ in range(3)],
                                   RC.rng_uniform_range(oracle, st, -PI, PI))
        mpq = RC.quat_to_matrix(*p[:4]) @ RC.quat_to_matrix(*q[:4])
        np.testing.assert_allclose(oracle.rotation_matrix(oracle.compose(p, q)), mpq,
                                   rtol=1e-10, atol=1e-10)


def test_depth_to_cloud_hand_computed(oracle):
    """test_geometry.cpp:90-145 (2x2 hand-computed case, reprojection)."""
    from paper_2312_08715_b200.configs import Intr
    k = Intr(10.0, 20.0, 0.5, 1.0, 2, 2, 0.01, 10.0)
    img = np.array([[1.0, 2.0], [3.0, 4.0]], dtype=np.float32)
    c = oracle.depth_to_cloud(img, k)
    want = [[-0.5 * 1 / 10, -1.0 * 1 / 20, 1], [0.5 * 2 / 10, -1.0 * 2 / 20, 2],
            [-0.5 * 3 / 10, 0.0, 3], [0.5 * 4 / 10, 0.0, 4]]
    np.testing.assert_allclose(c, want, atol=1e-12)
    k = Intr(20.0, 25.0, 7.5, 5.5, 16, 12, 0.01, 10.0)
    st = oracle.rng_seed(3)
    img = np.zeros((12, 16), dtype=np.float32)
    for v in range(12):
        for u in range(16):
            img[v, u] = np.float32(RC.rng_uniform_range(oracle, st, 0.5, 5.0))
    c = oracle.depth_to_cloud(img, k)
    uu = k.fx * c[:, 0] / c[:, 2] + k.cx
    vv = k.fy * c[:, 1] / c[:, 2] + k.cy
    gu, gv = np.meshgrid(np.arange(16), np.arange(12))
    assert np.abs(uu - gu.ravel()).max() < 1e-6 and np.abs(vv - gv.ravel()).max() < 1e-6


def _expected_faces(vox):
    occ = set(map(tuple, vox))
    offs = [(-1, 0, 0), (1, 0, 0), (0, -1, 0), (0, 1, 0), (0, 0, -1), (0, 0, 1)]
    return sum(1 for v in occ for o in offs if (v[0] + o[0], v[1] + o[1], v[2] + o[2]) not in occ)


def _watertight(tris):
    from collections import Counter
    c = Counter()
    for t in tris:
        for e in range(3):
            a, b = int(t[e]), int(t[(e + 1) % 3])
            c[(min(a, b), max(a, b))] += 1
    return all(v == 2 for v in c.values())


def test_voxel_to_mesh(oracle):
    """test_geometry.cpp:263-340"""
    v, t = oracle.voxel_to_mesh(np.array([[0, 0, 0]]), 0.1, [0, 0, 0])
    assert t.shape[0] == 12 and v.shape[0] == 8
    area = sum(0.5 * np.linalg.norm(np.cross(v[b] - v[a], v[c] - v[a])) for a, b, c in t)
    assert area == pytest.approx(0.06, rel=1e-12)
    v, t = oracle.voxel_to_mesh(np.array([[0, 0, 0], [1, 0, 0]]), 0.1, [0, 0, 0])
    assert t.shape[0] == 20
    st = oracle.rng_seed(9)
    for _ in range(5):
        seen, vox = set(), []
        for _ in range(30):
            p = tuple(oracle.rng_uniform_int(st, 5) for _ in range(3))
            if p not in seen:
                seen.add(p)
                vox.append(p)
        vox = np.array(vox)
        v, t = oracle.voxel_to_mesh(vox, 0.02, [0, 0, 0])
        assert t.shape[0] == 2 * _expected_faces(vox)
        for a, b, c in t:
            assert np.linalg.norm(np.cross(v[b] - v[a], v[c] - v[a])) > 1e-12
    box = np.array([(x, y, z) for x in range(3) for y in range(2) for z in range(2)])
    ell = np.array([(0, 0, 0), (1, 0, 0), (1, 1, 0), (1, 1, 1)])
    ball = np.array([(x, y, z) for x in range(-3, 4) for y in range(-3, 4) for z in range(-3, 4)
                     if x * x + y * y + z * z <= 9])
    for g in (box, ell, ball):
        _, t = oracle.voxel_to_mesh(g, 0.01, [0, 0, 0])
        assert _watertight(t)


def test_product_voxel_to_mesh_matches_oracle(oracle):
    """The product's host voxel_to_mesh (b3d_voxel_to_mesh) defines the same
    vertex and triangle order (= triangle ids) as the oracle."""
    from paper_2312_08715_b200 import b3d, synth
    for vox in (synth.eden_blob(500, 1), synth.random_walk_blob(300, 2)):
        o = synth.centered_origin(vox, 0.005)
        v1, t1 = b3d.voxel_to_mesh(vox, 0.005, o)
        v2, t2 = oracle.voxel_to_mesh(vox, 0.005, o)
        assert np.array_equal(t1, t2) and np.array_equal(v1.view(np.uint64), v2.view(np.uint64))


def test_contact_to_pose_flush(oracle):
    """test_scene_graph.cpp:30-46"""
    table = RC.make_table(oracle, 0.5, 0.5)
    cube = RC.make_model(oracle, RC.centered_cube_grid(4, 0.02))
    for face in range(1, 7):
        pose = oracle.contact_to_pose(0.5, 0.5, cube.aabb_min, cube.aabb_max, face, 0, 0, 0)
        assert pose[6] == pytest.approx(0.04, rel=1e-9)
        lo, hi = oracle.rotated_bounds(cube.aabb_min, cube.aabb_max, face)
        assert pose[4] - (hi[0] - lo[0]) / 2 == pytest.approx(-0.25, rel=1e-9)
    assert table.extents[0] == pytest.approx(0.5)


def test_face_heights(oracle):
    """test_scene_graph.cpp:71-94"""
    box = RC.make_model(oracle, RC.box_grid(6, 4, 2, 0.01))

    def top(face):
        lo, hi = oracle.rotated_bounds(box.aabb_min, box.aabb_max, face)
        return hi[2] - lo[2]
    assert top(3) == pytest.approx(0.06, rel=1e-12)
    assert top(5) == pytest.approx(0.04, rel=1e-12)
    assert top(1) == pytest.approx(0.02, rel=1e-12)
    for face in (1, 3, 5):
        pose = oracle.contact_to_pose(0.5, 0.5, box.aabb_min, box.aabb_max, face, 0.01, 0.02, 0.3)
        R = oracle.rotation_matrix(pose)
        max_z = (box.verts @ R.T + pose[4:])[:, 2].max()
        assert max_z == pytest.approx(top(face), rel=1e-9)


def test_dtheta_pi_symmetric_cube(oracle):
    """test_scene_graph.cpp:48-69"""
    from helpers import square_k
    k = square_k(48, near=0.1, far=5.0)
    cube = RC.make_model(oracle, RC.centered_cube_grid(4, 0.02))
    table = RC.make_table(oracle, 0.5, 0.5)
    cam = oracle.from_axis_angle([1, 0, 0], PI, [0, 0, 1.0])
    fx, fy = RC.footprint(oracle, cube, 1)
    dx, dy = (0.5 - fx) / 2, (0.5 - fy) / 2
    ia = oracle.render(k, RC.scene_instances(oracle, table, [(cube, 1, dx, dy, 0.0)]), camera=cam)
    ib = oracle.render(k, RC.scene_instances(oracle, table, [(cube, 1, dx, dy, PI)]), camera=cam)
    assert (np.abs(ia - ib) > 1e-5).sum() <= ia.size // 100


def test_product_contact_grid_poses_match_oracle(oracle):
    """b3d_contact_grid_poses (host side of the device contact grid) ==
    contact_to_pose at the stage-0 cell centres (inference.cpp:208-238,
    Interval::center), bitwise, for every face."""
    from paper_2312_08715_b200 import b3d
    cube = RC.make_model(oracle, RC.lblock_grid(0.015))
    TWO_PI = 6.283185307179586476925287
    for face in range(1, 7):
        cnt = (3, 2, 5)
        g = b3d.ContactGrid.make(0.5, 0.4, cube.aabb_min, cube.aabb_max, face, cnt)
        P = b3d.contact_grid_poses(g)
        lo, hi = oracle.rotated_bounds(cube.aabb_min, cube.aabb_max, face)
        dxr, dyr = 0.5 - (hi[0] - lo[0]), 0.4 - (hi[1] - lo[1])
        Q = []
        for ix in range(cnt[0]):
            for iy in range(cnt[1]):
                for it in range(cnt[2]):
                    dx = 0.5 * (dxr * ix / cnt[0] + dxr * (ix + 1) / cnt[0])
                    dy = 0.5 * (dyr * iy / cnt[1] + dyr * (iy + 1) / cnt[1])
                    dt = 0.5 * (TWO_PI * it / cnt[2] + TWO_PI * (it + 1) / cnt[2])
                    Q.append(oracle.contact_to_pose(0.5, 0.4, cube.aabb_min, cube.aabb_max, face,
                                                    dx, dy, dt))
        assert np.array_equal(P.view(np.uint64), np.array(Q).view(np.uint64)), face
