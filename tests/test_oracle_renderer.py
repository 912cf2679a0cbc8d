"""Pins the CPU oracle's renderer to the reference's renderer tests
(proj/tests/test_renderer.cpp), same parameters and tolerances, with the
reference's own test oracles (ray caster, edge mask) restated in refcheck.py."""
import math

import numpy as np

import refcheck as RC
from helpers import square_k

PI = 3.141592653589793238462643


def pose_mats(O, camera):
    w2c = O.inverse(camera)

    def f(m2w):
        m2c = O.compose(w2c, m2w)
        return O.rotation_matrix(m2c), m2c[4:]
    return f


def test_empty_scene_renders_all_sentinel(oracle):
    """test_renderer.cpp:36-40"""
    k = square_k(16)
    img = oracle.render(k, [])
    assert (img == np.float32(k.far)).all()


def test_unit_cube_face_on(oracle):
    """test_renderer.cpp:42-54: centre pixel hits the front face at 1.5 m."""
    v, t = oracle.box_mesh([-0.5, -0.5, 1.5], [0.5, 0.5, 2.5])
    k = square_k(33)
    ident = [1, 0, 0, 0, 0, 0, 0.0]
    img = oracle.render(k, [(v, t, ident)])
    assert abs(img[16, 16] - 1.5) <= 1e-6 * 1.5
    ray = RC.raycast_depth([(v, t, ident)], ident, k, pose_mats(oracle, ident))
    assert abs(ray[16, 16] - 1.5) <= 1e-6 * 1.5


def _library(oracle, *grids):
    return [RC.make_model(oracle, g) for g in grids]


def test_raster_matches_raycast_away_from_edges(oracle):
    """test_renderer.cpp:56-82: >= 99% of non-edge pixels within 1e-5 m."""
    st = oracle.rng_seed(42)
    table = RC.make_table(oracle, 0.5, 0.5)
    lib = _library(oracle, RC.lblock_grid(0.015), RC.mug_grid(0.012))
    k = square_k(32)
    for trial in range(5):
        s = oracle.rng_split(st, trial)
        children = RC.sample_scene_prior(oracle, s, 1, lib, table)
        cam = oracle.camera_pose_from_spherical(RC.rng_uniform_range(oracle, s, 0.7, 1.1),
                                                RC.rng_uniform_range(oracle, s, 0.0, 2 * PI),
                                                RC.rng_uniform_range(oracle, s, 0.5, 1.0))
        inst = RC.scene_instances(oracle, table, children)
        img = oracle.render(k, inst, camera=cam)
        ray = RC.raycast_depth(inst, cam, k, pose_mats(oracle, cam))
        edges = RC.edge_mask(ray, k)
        checked = (~edges).sum()
        matched = ((np.abs(img - ray) < 1e-5) & ~edges).sum()
        assert checked > 0
        assert matched / checked >= 0.99


def test_near_plane_clipping_matches_oracle(oracle):
    """test_renderer.cpp:84-103: a triangle piercing z = near."""
    v = np.array([[-2.0, 0.5, -1.0], [2.0, 0.5, 3.0], [0.0, -1.5, 1.5]])
    t = np.array([[0, 1, 2]], dtype=np.uint32)
    k = square_k(48)
    ident = [1, 0, 0, 0, 0, 0, 0.0]
    img = oracle.render(k, [(v, t, ident)])
    ray = RC.raycast_depth([(v, t, ident)], ident, k, pose_mats(oracle, ident))
    edges = RC.edge_mask(ray, k)
    checked = (~edges).sum()
    bad = ((np.abs(img - ray) > 1e-5) & ~edges).sum()
    assert checked > 100 and bad == 0


def test_repeat_renders_bitwise(oracle):
    """test_renderer.cpp:105-148: determinism (batched == sequential == repeat)."""
    st = oracle.rng_seed(3)
    table = RC.make_table(oracle, 0.5, 0.5)
    lib = _library(oracle, RC.mug_grid(0.012))
    children = RC.sample_scene_prior(oracle, st, 1, lib, table)
    cam = oracle.camera_pose_from_spherical(0.9, 1.1, 0.8)
    k = square_k(40)
    inst = RC.scene_instances(oracle, table, children)
    a = oracle.render(k, inst, camera=cam)
    b = oracle.render(k, inst, camera=cam)
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


def test_occlusion_monotonicity(oracle):
    """test_renderer.cpp:150-170: adding an object never increases depth."""
    st = oracle.rng_seed(19)
    table = RC.make_table(oracle, 0.5, 0.5)
    lib = _library(oracle, RC.box_grid(5, 5, 5, 0.02), RC.lblock_grid(0.02))
    k = square_k(32)
    for trial in range(20):
        s = oracle.rng_split(st, trial)
        two = RC.sample_scene_prior(oracle, s, 2, lib, table)
        cam = oracle.camera_pose_from_spherical(RC.rng_uniform_range(oracle, s, 0.7, 1.2),
                                                RC.rng_uniform_range(oracle, s, 0.0, 2 * PI),
                                                RC.rng_uniform_range(oracle, s, 0.5, 1.0))
        base = oracle.render(k, RC.scene_instances(oracle, table, two[:1]), camera=cam)
        more = oracle.render(k, RC.scene_instances(oracle, table, two), camera=cam)
        assert (more <= base).all()


def test_camera_equivariance(oracle):
    """test_renderer.cpp:172-197: <= 1% of pixels off by > 1e-5 m."""
    st = oracle.rng_seed(23)
    v, t = oracle.box_mesh([-0.05, -0.04, 0.0], [0.05, 0.04, 0.09])
    k = square_k(32)
    for trial in range(5):
        s = oracle.rng_split(st, trial)
        cam = oracle.camera_pose_from_spherical(RC.rng_uniform_range(oracle, s, 0.5, 1.0),
                                                RC.rng_uniform_range(oracle, s, 0.0, 2 * PI),
                                                RC.rng_uniform_range(oracle, s, 0.4, 1.0))
        ax = [oracle.rng_normal(s), oracle.rng_normal(s), oracle.rng_normal(s)]
        obj = oracle.from_axis_angle(ax, RC.rng_uniform_range(oracle, s, 0, PI),
                                     [RC.rng_uniform_range(oracle, s, -0.1, 0.1),
                                      RC.rng_uniform_range(oracle, s, -0.1, 0.1), 0])
        ax2 = [oracle.rng_normal(s), oracle.rng_normal(s), oracle.rng_normal(s)]
        wt = oracle.from_axis_angle(ax2, RC.rng_uniform_range(oracle, s, 0, PI), [0.4, -0.2, 0.7])
        a = oracle.render(k, [(v, t, obj)], camera=cam)
        b = oracle.render(k, [(v, t, oracle.compose(wt, obj))], camera=oracle.compose(wt, cam))
        assert (np.abs(a - b) > 1e-5).sum() <= a.size // 100


def test_shared_edges_covered_once(oracle):
    """test_renderer.cpp:199-228: top-left fill rule on a split convex quad."""
    st = oracle.rng_seed(31)
    k = square_k(24)
    ident = [1, 0, 0, 0, 0, 0, 0.0]
    for trial in range(50):
        s = oracle.rng_split(st, trial)
        z = RC.rng_uniform_range(oracle, s, 0.5, 2.0)
        cx = RC.rng_uniform_range(oracle, s, -0.2, 0.2)
        cy = RC.rng_uniform_range(oracle, s, -0.2, 0.2)
        rad = RC.rng_uniform_range(oracle, s, 0.05, 0.4)
        verts = []
        for i in range(4):
            ang = PI / 2 * i + RC.rng_uniform_range(oracle, s, 0.05, PI / 2 - 0.05)
            verts.append([cx + rad * math.cos(ang), cy + rad * math.sin(ang), z])
        verts = np.array(verts)
        t1 = (verts[[0, 1, 2]], np.array([[0, 1, 2]], dtype=np.uint32), ident)
        t2 = (verts[[0, 2, 3]], np.array([[0, 1, 2]], dtype=np.uint32), ident)
        a = oracle.render(k, [t1])
        b = oracle.render(k, [t2])
        sent = np.float32(k.far)
        assert not ((a < sent) & (b < sent)).any()


def test_draw_index_extension_follows_tie_rule(oracle):
    """Oracle extension: the per-pixel draw index is the
    earliest-drawn triangle among the equal-depth winners (strict less,
    renderer.cpp:100).  A quad drawn twice: the first copy owns every pixel."""
    v, t = oracle.box_mesh([-0.2, -0.2, 1.0], [0.2, 0.2, 1.2])
    k = square_k(32)
    ident = [1, 0, 0, 0, 0, 0, 0.0]
    d1, i1 = oracle.render(k, [(v, t, ident), (v, t, ident)], with_ids=True)
    d0, i0 = oracle.render(k, [(v, t, ident)], with_ids=True)
    assert np.array_equal(d1, d0) and np.array_equal(i1, i0)
    assert (i0 >= 0).sum() > 100 and i0.max() < 12
