"""Pins the CPU oracle's likelihood to the reference's likelihood tests
(proj/tests/test_likelihood.cpp), same parameters and tolerances, against the
reference's naive double-loop oracles (restated in refcheck.py)."""
import math

import numpy as np
import pytest

import refcheck as RC
from helpers import make_k

PI = 3.141592653589793238462643


def random_surface(O, st, k, sparsity=0.0):
    """test_likelihood.cpp:32-39"""
    img = np.full((k.height, k.width), np.float32(k.far), dtype=np.float32)
    for v in range(k.height):
        for u in range(k.width):
            if O.rng_uniform(st) >= sparsity:
                img[v, u] = np.float32(RC.rng_uniform_range(O, st, 0.5, 0.9 * k.far))
    return img


def test_visible_volume(oracle):
    """test_likelihood.cpp:43-79"""
    k = make_k(1, 1, 1.0, 1e-9, 1.0)
    k.cx = k.cy = 0.0
    assert oracle.visible_volume(k) == pytest.approx(1.0 / 3.0, rel=1e-6)
    k = make_k(4, 4, 10.0, 1e-9, 1.0)
    v1 = oracle.visible_volume(k)
    k.far = 2.0
    assert oracle.visible_volume(k) == pytest.approx(8.0 * v1, rel=1e-6)
    # Monte Carlo rejection oracle within 1%
    k = make_k(640, 480, 500.0, 0.1, 5.0)
    v = oracle.visible_volume(k)
    rng = np.random.Generator(np.random.PCG64(99))
    x_lo, x_hi = (0.0 - k.cx) * k.far / k.fx, (k.width - k.cx) * k.far / k.fx
    y_lo, y_hi = (0.0 - k.cy) * k.far / k.fy, (k.height - k.cy) * k.far / k.fy
    box = (x_hi - x_lo) * (y_hi - y_lo) * (k.far - k.near)
    n = 2_000_000
    z = rng.uniform(k.near, k.far, n)
    x = rng.uniform(x_lo, x_hi, n)
    y = rng.uniform(y_lo, y_hi, n)
    u = k.fx * x / z + k.cx
    vv = k.fy * y / z + k.cy
    hits = ((u >= 0) & (u <= k.width) & (vv >= 0) & (vv <= k.height)).sum()
    assert abs(box * hits / n - v) / v < 0.01


def test_full_closed_forms(oracle):
    """test_likelihood.cpp:88-132"""
    vol = 2.5
    rend = [[0, 0, 1], [0.1, 0, 1], [0, 0.1, 1.2]]
    got = oracle.full_loglik_points([[3, 2, 1], [0, 0, 1]], rend, (1.0, 0.02), vol, 0.1)
    assert got == pytest.approx(math.log(0.02 / 0.1) + 2.0 * math.log(1.0 / vol), rel=1e-12)
    sigma = 0.015
    got = oracle.full_loglik_points([[0.3, -0.2, 0.9]], [[0.3, -0.2, 0.9]], (0.0, sigma), vol, 0.1)
    want = math.log(sigma / 0.1) - 1.5 * math.log(2 * PI * sigma * sigma)
    assert got == pytest.approx(want, rel=1e-12)
    printed = oracle.full_loglik_points([[0, 0, 1]], rend, (0.5, 0.03), vol, 0.1, prefactor=0)
    uniform = oracle.full_loglik_points([[0, 0, 1]], rend, (0.5, 0.03), vol, 0.1, prefactor=1)
    assert printed - uniform == pytest.approx(math.log(0.03), rel=1e-12)
    with pytest.raises(ValueError):
        oracle.full_loglik_points([[0, 0, 1]], np.zeros((0, 3)), (0.5, 0.01), vol, 0.1)
    with pytest.raises(ValueError):
        oracle.full_loglik_points([[0, 0, 1]], rend, (0.5, 0.0), vol, 0.1)


def test_full_matches_naive_double_loop(oracle):
    """test_likelihood.cpp:134-150 (1e-10 relative)"""
    st = oracle.rng_seed(5)
    for _ in range(10):
        obs = [[RC.rng_uniform_range(oracle, st, -0.5, 0.5), RC.rng_uniform_range(oracle, st, -0.5, 0.5),
                RC.rng_uniform_range(oracle, st, 0.5, 2.0)] for _ in range(5)]
        rend = [[RC.rng_uniform_range(oracle, st, -0.5, 0.5), RC.rng_uniform_range(oracle, st, -0.5, 0.5),
                 RC.rng_uniform_range(oracle, st, 0.5, 2.0)] for _ in range(7)]
        p = RC.rng_uniform_range(oracle, st, 0.05, 0.95)
        s = RC.rng_uniform_range(oracle, st, 0.005, 0.1)
        vol = RC.rng_uniform_range(oracle, st, 1.0, 10.0)
        got = oracle.full_loglik_points(obs, rend, (p, s), vol, 0.1)
        want = RC.naive_full_loglik(obs, rend, p, s, vol, 0.1)
        assert abs(got - want) <= 1e-10 * abs(want)


def test_full_permutation_invariant(oracle):
    """test_likelihood.cpp:152-168"""
    st = oracle.rng_seed(6)
    obs, rend = [], []
    for _ in range(20):
        obs.append([oracle.rng_normal(st), oracle.rng_normal(st),
                    RC.rng_uniform_range(oracle, st, 0.5, 2.0)])
        rend.append([oracle.rng_normal(st), oracle.rng_normal(st),
                     RC.rng_uniform_range(oracle, st, 0.5, 2.0)])
    base = oracle.full_loglik_points(obs, rend, (0.2, 0.05), 4.0, 0.1)
    obs_s = obs[::-1]
    rend_s = rend[7:] + rend[:7]
    shuffled = oracle.full_loglik_points(obs_s, rend_s, (0.2, 0.05), 4.0, 0.1)
    assert abs(base - shuffled) <= 1e-9 * abs(base)


K16 = make_k(16, 16, 20.0, 0.1, 5.0)


def test_windowed_full_window_equals_full(oracle):
    """test_likelihood.cpp:175-189 (1e-9)"""
    k = K16
    vol = oracle.visible_volume(k)
    st = oracle.rng_seed(7)
    for trial in range(50):
        s = oracle.rng_split(st, trial)
        obs = random_surface(oracle, s, k, 0.3)
        rend = random_surface(oracle, s, k, 0.3)
        p = RC.rng_uniform_range(oracle, s, 0.05, 0.95)
        sg = RC.rng_uniform_range(oracle, s, 0.01, 0.1)
        oc = oracle.depth_to_cloud(obs, k)
        rc = oracle.depth_to_cloud(rend, k)
        if len(oc) == 0 or len(rc) == 0:
            continue
        full = oracle.full_loglik_points(oc, rc, (p, sg), vol, 0.1)
        win = oracle.windowed_loglik_multi(obs, rend, k, [(p, sg)], 0.1, 16)[0]
        assert abs(full - win) <= 1e-9 * abs(full)


def test_windowed_matches_masked_double_loop(oracle):
    """test_likelihood.cpp:191-203: w=2, 1e-10 relative -- the score kernel's
    parity anchor."""
    k = K16
    vol = oracle.visible_volume(k)
    st = oracle.rng_seed(7)
    for trial in range(50):
        s = oracle.rng_split(st, 1000 + trial)
        obs = random_surface(oracle, s, k, 0.4)
        rend = random_surface(oracle, s, k, 0.4)
        p = RC.rng_uniform_range(oracle, s, 0.05, 0.95)
        sg = RC.rng_uniform_range(oracle, s, 0.01, 0.1)
        if len(oracle.depth_to_cloud(rend, k)) == 0 or len(oracle.depth_to_cloud(obs, k)) == 0:
            continue
        got = oracle.windowed_loglik_multi(obs, rend, k, [(p, sg)], 0.1, 2)[0]
        want = RC.naive_windowed_loglik(obs, rend, k, p, sg, vol, 0.1, 2)
        assert abs(got - want) <= 1e-10 * abs(want)


def test_windowed_w0_outlier_floor(oracle):
    """test_likelihood.cpp:205-214"""
    k = K16
    vol = oracle.visible_volume(k)
    obs = np.full((16, 16), np.float32(k.far), dtype=np.float32)
    rend = obs.copy()
    obs[8, 8] = 1.0
    rend[8, 8] = 3.0
    got = oracle.windowed_loglik_multi(obs, rend, k, [(0.3, 0.01)], 0.1, 0)[0]
    assert got == pytest.approx(math.log(0.01 / 0.1) + math.log(0.3 / vol), rel=1e-9)


def test_windowed_monotone_in_window(oracle):
    """test_likelihood.cpp:216-229"""
    k = K16
    st = oracle.rng_split(oracle.rng_seed(7), 77)
    obs = random_surface(oracle, st, k, 0.2)
    rend = random_surface(oracle, st, k, 0.2)
    prev = -math.inf
    for w in (0, 1, 2, 4, 8, 16):
        ll = oracle.windowed_loglik_multi(obs, rend, k, [(0.2, 0.05)], 0.1, w)[0]
        assert ll >= prev - 1e-12
        prev = ll
    assert prev == pytest.approx(
        oracle.windowed_loglik_multi(obs, rend, k, [(0.2, 0.05)], 0.1, 32)[0], rel=1e-12)


def test_windowed_floor_lower_bound(oracle):
    """test_likelihood.cpp:231-243"""
    k = K16
    vol = oracle.visible_volume(k)
    st = oracle.rng_split(oracle.rng_seed(7), 88)
    obs = random_surface(oracle, st, k, 0.3)
    rend = random_surface(oracle, st, k, 0.3)
    m = int((obs < np.float32(k.far)).sum())
    ll = oracle.windowed_loglik_multi(obs, rend, k, [(0.25, 0.02)], 0.1, 2)[0]
    assert ll >= math.log(0.02 / 0.1) + m * math.log(0.25 / vol) - 1e-9


def test_multi_noise_equals_one_at_a_time_bitwise(oracle):
    """test_likelihood.cpp:245-257"""
    k = K16
    st = oracle.rng_split(oracle.rng_seed(7), 99)
    obs = random_surface(oracle, st, k, 0.3)
    rend = random_surface(oracle, st, k, 0.3)
    grid = [(0.05, 0.025), (0.3, 0.025), (0.8, 0.05)]
    multi = oracle.windowed_loglik_multi(obs, rend, k, grid, 0.1, 2)
    for i, g in enumerate(grid):
        one = oracle.windowed_loglik_multi(obs, rend, k, [g], 0.1, 2)[0]
        assert multi[i] == one


def test_windowed_errors(oracle):
    """test_likelihood.cpp:259-267: empty render is an error."""
    k = K16
    obs = np.full((16, 16), np.float32(1.0), dtype=np.float32)
    empty = np.full((16, 16), np.float32(k.far), dtype=np.float32)
    with pytest.raises(ValueError):
        oracle.windowed_loglik_multi(obs, empty, k, [(0.5, 0.01)], 0.1, 2)


def test_default_window(oracle):
    """test_likelihood.cpp:371-376"""
    L = oracle.lib()
    assert L.orc_default_window(100) == 2
    assert L.orc_default_window(200) == 4
    assert L.orc_default_window(50) == 1
    assert L.orc_default_window(25) == 1
