"""sample_observation (likelihood.cpp:44-80) and orbit frames
(tracking.cpp:174-206): the product's host routine vs the oracle restatement
(bitwise, same Rng stream) and the reference's own test properties
(test_likelihood.cpp:270-368)."""
import numpy as np
import pytest

from oracle import pyoracle as orc
from paper_2312_08715_b200 import b3d


def make_k(w, h, f, near, far):  # test_likelihood.cpp:19-30
    return b3d.Intrinsics(f, f, (w - 1) / 2.0, (h - 1) / 2.0, w, h, near, far)


def kt(k):  # the oracle takes intrinsics as a tuple
    return (k.fx, k.fy, k.cx, k.cy, k.width, k.height, k.near_m, k.far_m)


def random_surface(st, k, sparsity=0.0):  # test_likelihood.cpp:32-39, with the oracle's Rng
    img = np.full((k.height, k.width), np.float32(k.far_m), dtype=np.float32)
    for v in range(k.height):
        for u in range(k.width):
            if orc.rng_uniform(st) >= sparsity:
                img[v, u] = np.float32(0.5 + (0.9 * k.far_m - 0.5) * orc.rng_uniform(st))
    return img


@pytest.mark.parametrize("w,h,p,sigma,sparsity,seed", [
    (24, 24, 0.0, 1e-12, 0.5, 11),
    (24, 24, 0.1, 0.01, 0.0, 3),
    (40, 30, 0.5, 0.05, 0.3, 5),
    (17, 9, 1.0, 0.01, 0.7, 8),
    (33, 21, 0.02, 0.002, 0.9, 9),
])
def test_product_equals_oracle(w, h, p, sigma, sparsity, seed):
    k = make_k(w, h, 30.0, 0.1, 5.0)
    rend = random_surface(orc.rng_seed(seed), k, sparsity)
    if not (rend < np.float32(k.far_m)).any():
        rend[0, 0] = 1.0
    st_o = orc.rng_seed(seed + 100)
    st_p = st_o.copy()
    want = orc.sample_observation(rend, kt(k), p, sigma, st_o)
    got = b3d.sample_observation(k, rend, p, sigma, st_p)
    assert got.tobytes() == want.tobytes()
    assert np.array_equal(st_p, st_o)  # the stream advanced by the same draws


def test_noiseless_inliers_reproduce_rendered():  # test_likelihood.cpp:271-295
    k = make_k(24, 24, 30.0, 0.1, 5.0)
    rend = random_surface(orc.rng_seed(11), k, 0.5)
    obs = b3d.sample_observation(k, rend, 0.0, 1e-12, b3d.rng_seed(3))
    sent = np.float32(k.far_m)
    filled = obs < sent
    assert filled.sum() > 0
    assert np.allclose(obs[filled], rend[filled], rtol=1e-6, atol=0)
    assert filled.sum() <= (rend < sent).sum()


def test_pure_outliers_follow_frustum_law():  # test_likelihood.cpp:297-320
    k = make_k(128, 128, 64.0, 0.2, 4.0)
    rend = np.full((128, 128), np.float32(k.far_m), dtype=np.float32)
    rend[60:65, 60:65] = 1.0
    sampler = b3d.rng_seed(5)
    n3, f3 = k.near_m ** 3, k.far_m ** 3
    vals = []
    for run in range(400):
        st = b3d.rng_split(sampler, run)
        obs = b3d.sample_observation(k, rend, 1.0, 0.01, st)
        z = obs[obs < np.float32(k.far_m)].astype(np.float64)
        vals.append((z ** 3 - n3) / (f3 - n3))
    c = np.sort(np.concatenate(vals))
    assert c.size > 9000
    n = c.size
    d = max(np.max(np.arange(1, n + 1) / n - c), np.max(c - np.arange(0, n) / n))
    assert d < 1.63 / np.sqrt(n)


def test_inlier_residual_spread_matches_sigma():  # test_likelihood.cpp:322-360
    k = make_k(120, 120, 40.0, 0.2, 6.0)
    rend = np.full((120, 120), 2.0, dtype=np.float32)
    sigma = 0.01
    obs = b3d.sample_observation(k, rend, 0.0, sigma, b3d.rng_seed(9))
    v, u = np.nonzero(obs < np.float32(k.far_m))
    assert u.size > 8000
    z = obs[v, u].astype(np.float64)
    # every rendered point has z = 2, so the nearest one's z residual is z - 2
    res = z - 2.0
    assert np.std(res, ddof=1) == pytest.approx(sigma, rel=0.05)


def test_errors():  # test_likelihood.cpp:362-367 + validate_noise
    k = make_k(8, 8, 10.0, 0.1, 5.0)
    empty = np.full((8, 8), np.float32(k.far_m), dtype=np.float32)
    with pytest.raises(b3d.B3DError):
        b3d.sample_observation(k, empty, 0.5, 0.01, b3d.rng_seed(1))
    assert orc.sample_observation(empty, kt(k), 0.5, 0.01, orc.rng_seed(1)) is None
    rend = empty.copy()
    rend[3, 3] = 1.0
    for p, s in ((0.5, 0.0), (-0.1, 0.01), (1.5, 0.01)):
        with pytest.raises(b3d.B3DError):
            b3d.sample_observation(k, rend, p, s, b3d.rng_seed(1))
    with pytest.raises(b3d.B3DError):
        b3d.sample_observations(k, np.stack([rend, empty]), 0.5, 0.01, b3d.rng_seed(1))


def test_orbit_frames_use_split_streams():  # tracking.cpp:199-202
    k = make_k(32, 24, 28.0, 0.1, 5.0)
    st = orc.rng_seed(77)
    frames = np.stack([random_surface(st, k, 0.4) for _ in range(5)])
    base = b3d.rng_split(b3d.rng_seed(0), 0, 32)  # root.split(obj, res)
    before = base.copy()
    got = b3d.sample_observations(k, frames, 0.02, 0.002, base)
    assert np.array_equal(base, before)
    for i in range(5):
        want = orc.sample_observation(frames[i], kt(k), 0.02, 0.002, orc.rng_split(base, 0x0F, i))
        assert got[i].tobytes() == want.tobytes()
