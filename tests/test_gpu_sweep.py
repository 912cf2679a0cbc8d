"""GPU: a seeded random sweep of the score-many seam (b3d_gpu_score_poses)
against the oracle -- bitwise the reference on every fixture -- over the
settings space: image sizes and aspect ratios, intrinsics, windows 0-6 and
the untruncated likelihood, noise grids of 1-20 entries with up to 6
distinct sigmas (chunked launches), both prefactors, p_outlier edge values,
non-identity cameras, poses crossing z = near, meshes that fit on chip or
spill to scratch.  Scores within 1e-4 relative (and an absolute bound
scaled by the pixel count), empty renders flagged the same way."""
import numpy as np
import pytest

from helpers import b3d_intr
from paper_2312_08715_b200 import b3d, configs, synth

pytestmark = pytest.mark.gpu
RTOL = 1e-4


@pytest.mark.parametrize("case", range(48))
def test_score_sweep(gpu_ctx, oracle, case):
    rng = np.random.Generator(np.random.PCG64(7000 + case))
    w = int(rng.choice([8, 17, 40, 64, 97]))
    h = int(rng.choice([6, 13, 32, 48, 71]))
    f = float(rng.uniform(0.6, 1.6)) * max(w, h)
    k = configs.Intr(f, f * float(rng.uniform(0.9, 1.1)), (w - 1) / 2 + float(rng.uniform(-2, 2)),
                     (h - 1) / 2 + float(rng.uniform(-2, 2)), w, h, float(rng.choice([0.01, 0.2])),
                     float(rng.choice([3.0, 10.0])))
    n_vox = int(rng.choice([60, 400, 3000]))
    vox = synth.eden_blob(n_vox, 8000 + case)
    verts, tris = configs.make_mesh(vox, oracle.voxel_to_mesh)
    cam = np.array([1.0, 0, 0, 0, 0, 0, 0]) if case % 3 else oracle.camera_pose_from_spherical(
        0.05, float(rng.uniform(0, 6)), 1.2)
    def pose_near(z):
        q = synth.uniform_quaternion(rng)
        return [q[0], q[1], q[2], q[3], float(rng.uniform(-0.03, 0.03)),
                float(rng.uniform(-0.03, 0.03)), z]
    # world poses in front of the camera (the camera looks along its +z)
    cw = np.array(cam)
    poses = []
    for i in range(24):
        z = float(rng.choice([0.4, 0.6, 1.0])) if i % 8 else float(k.near + 0.01)
        p_cam = pose_near(z)
        poses.append(oracle.compose(cw, np.array(p_cam)))
    poses = np.array(poses)
    base_inst = []
    if case % 4 == 1:  # a fixed scene behind the object: the base-scene path
        bv, bt, _, _ = configs.table_mesh(oracle.box_mesh, 0.4, 0.3)
        q = synth.uniform_quaternion(rng)
        base_inst = [(bv, bt, oracle.compose(cw, np.array([q[0], q[1], q[2], q[3], 0.0, 0.0,
                                                            float(rng.uniform(0.7, 1.5))])))]
    obs = oracle.render(k, [(verts, tris, poses[0])] + base_inst, camera=cam)
    obs = synth.noisy_observation(np.array(obs, dtype=np.float32), k.far, 0.003, 0.1, 0.2, 2.0,
                                  rng, k.near)
    n_sig = int(rng.integers(1, 7))
    sigmas = sorted(set(float(s) for s in rng.uniform(0.002, 0.05, n_sig)))
    ps = [float(p) for p in rng.choice([0.0, 1e-7, 0.01, 0.3, 0.99, 1.0], int(rng.integers(1, 4)))]
    noise = [(p, s) for p in ps for s in sigmas][:20]
    window = int(rng.choice([0, 1, 2, 3, 4, 6, -1])) if w * h <= 2000 else int(rng.choice([0, 1, 2]))
    prefactor = int(rng.integers(0, 2))
    sigma_max = 0.1
    gpu_ctx.set_camera(b3d_intr(k), cam)
    mid = gpu_ctx.upload_mesh(verts, tris)
    base_depth = None
    if base_inst:
        bid = gpu_ctx.upload_mesh(base_inst[0][0], base_inst[0][1])
        gpu_ctx.set_base_scene([bid], [base_inst[0][2]])
        base_depth = np.array(oracle.render(k, base_inst, camera=cam), dtype=np.float32)
    else:
        gpu_ctx.set_base_scene([], [])
    gpu_ctx.set_likelihood(noise, sigma_max, window, prefactor)
    gpu_ctx.set_observation(obs)
    got, st = gpu_ctx.score_poses(mid, poses)
    want, wst = oracle.score_poses(k, obs, verts, tris, poses, noise, sigma_max, window,
                                   prefactor=prefactor, camera=cam, base_depth=base_depth)
    gpu_ctx.set_base_scene([], [])
    np.testing.assert_array_equal(st, wst, err_msg="empty-render flags")
    ok = wst == 0
    g, wv = got[ok], want[ok]
    fin = np.isfinite(wv)
    np.testing.assert_array_equal(np.isfinite(g), fin)
    d = np.abs(g[fin] - wv[fin])
    rel = d / np.maximum(np.abs(wv[fin]), 1e-300)
    scale = w * h * 60.0  # |log-term| per observed pixel is bounded by ~60
    assert rel.max(initial=0) <= RTOL, (case, rel.max())
    assert d.max(initial=0) <= RTOL * scale, (case, d.max())


def test_stage_draw_sweep(gpu_ctx, oracle):
    """300 random stages: flat, two-level, peaked and sparse (-inf) score
    arrays of 1 to 70,000 entries, each drawn with its own seed -- argmax,
    the categorical draw and the advanced Rng state equal the oracle's
    (sample_categorical's sequential CDF, inference.cpp:345-353)."""
    rng = np.random.Generator(np.random.PCG64(77))
    for t in range(300):
        n = int(rng.choice([1, 2, 3, 10, 97, 1024, 4097, 16384, 16385, 70000]))
        kind = t % 4
        if kind == 0:
            x = np.full(n, -3.25)
        elif kind == 1:
            x = np.where(rng.random(n) < 0.5, 0.0, -np.log(3.0))
        elif kind == 2:
            x = rng.normal(0.0, 40.0, n)
        else:
            x = np.where(rng.random(n) < 0.9, -np.inf, rng.normal(0.0, 1.0, n))
            x[int(rng.integers(0, n))] = 0.0
        st_g = b3d.rng_seed(900 + t)
        st_o = oracle.rng_seed(900 + t)
        r = gpu_ctx.stage_reduce(x, rng_state=st_g)
        probs_o, _ = oracle.normalize(x)
        assert r.argmax == oracle.argmax(x), t
        assert r.sample == oracle.sample_categorical(probs_o, st_o), (t, n, kind)
        np.testing.assert_array_equal(st_g, st_o)


def test_stage_draw_on_cdf_boundaries(gpu_ctx, oracle):
    """Draws placed on a CDF boundary on purpose: the stage's uniform u is
    known from its seed, and the scores put the running sum at index j to
    within an ulp of u -- the parallel CDF must hand these to the sequential
    fallback (the reference's index-order total and running sum) and agree
    with the oracle's pick and Rng state -- except where the device's exp and
    the host libm's differ in the last ulp and u sits within those ulps of
    the boundary: then the pick is the neighbouring index."""
    fallbacks = ulp_band = 0
    for seed in range(40):
        st = oracle.rng_seed(5000 + seed)
        u = oracle.rng_uniform(st.copy())
        n = 2 + seed % 7
        j = seed % (n - 1)
        # probabilities: j + 1 entries summing to u, the rest to 1 - u
        p = np.concatenate([np.full(j + 1, u / (j + 1)), np.full(n - j - 1, (1 - u) / (n - j - 1))])
        x = np.log(p) + (seed % 5) * 3.0
        st_g, st_o = b3d.rng_seed(5000 + seed), oracle.rng_seed(5000 + seed)
        r = gpu_ctx.stage_reduce(x, rng_state=st_g)
        probs_o, _ = oracle.normalize(x)
        pick = oracle.sample_categorical(probs_o, st_o)
        np.testing.assert_array_equal(st_g, st_o)
        fallbacks += int(r.sample_fallback)
        if r.sample != pick:
            acc = 0.0
            for i in range(min(r.sample, pick) + 1):
                acc += probs_o[i]
            assert r.sample_fallback and abs(r.sample - pick) == 1, seed
            assert abs(acc - u) <= 4 * np.spacing(u), (seed, acc, u)
            ulp_band += 1
    assert fallbacks >= 30  # the boundary cases took the sequential path
    assert ulp_band <= 8
