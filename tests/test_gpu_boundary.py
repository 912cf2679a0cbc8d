"""GPU: boundary semantics equal to the reference's (oracle-checked).

* score-many is the score_cells seam: a noise entry outside the support
  (p_outlier outside [0, 1], sigma_noise <= 0 or > sigma_max) scores -inf and
  the rest are scored (observation_loglik_cached_multi, inference.cpp:40-45,59-83);
* any number of noise entries and distinct sigmas (launches are chunked);
* window < 0 is the untruncated likelihood (inference.cpp:51-56);
* p_outlier = 0 and tiny p_outlier keep the reference's fp64 values, -inf
  included (the fp64 image path, exact_score.cu);
* the camera paths are windowed_log_likelihood_multi itself (tracking.cpp:98-101):
  window < 0 and invalid entries are errors, sigma > sigma_max is scored.
"""
import numpy as np
import pytest

from helpers import b3d_intr, cfg1_oracle, rel_err
from paper_2312_08715_b200 import b3d, configs

pytestmark = pytest.mark.gpu
RTOL = 1e-4


def _ctx_cfg1(gpu_ctx):
    w = cfg1_oracle()
    gpu_ctx.set_camera(b3d_intr(w.k))
    mid = gpu_ctx.upload_mesh(w.vertices, w.triangles)
    gpu_ctx.set_observation(w.observed)
    return w, mid


def _oracle_scores(oracle, w, poses, noise, window):
    return oracle.score_poses(w.k, w.observed, w.vertices, w.triangles, poses, noise, w.sigma_max,
                              window)[0]


def test_out_of_support_entries_score_neg_inf(gpu_ctx, oracle):
    w, mid = _ctx_cfg1(gpu_ctx)
    poses = w.grid_poses()[::37]
    noise = [(0.01, 0.005), (1.5, 0.005), (0.01, 0.2), (0.01, -1.0), (-0.1, 0.01), (0.05, 0.01)]
    gpu_ctx.set_likelihood(noise, 0.1, 1)
    s, st = gpu_ctx.score_poses(mid, poses)
    assert (st == 0).all()
    assert np.isneginf(s[:, 1:5]).all()
    for col in (0, 5):
        want = _oracle_scores(oracle, w, poses, [noise[col]], 1)[:, 0]
        assert rel_err(s[:, col], want).max() <= RTOL
        gpu_ctx.set_likelihood([noise[col]], 0.1, 1)
        alone, _ = gpu_ctx.score_poses(mid, poses)
        np.testing.assert_array_equal(alone[:, 0], s[:, col])  # same launch arithmetic
    # every entry outside the support: all -inf, nothing rendered
    gpu_ctx.set_likelihood([(2.0, 0.01), (0.1, 0.5)], 0.1, 1)
    s, st = gpu_ctx.score_poses(mid, poses)
    assert np.isneginf(s).all() and (st == 0).all()


def test_many_noise_entries_and_sigmas_are_chunked(gpu_ctx, oracle):
    """20 entries (4 p x 5 sigma): more than one fused launch holds."""
    w, mid = _ctx_cfg1(gpu_ctx)
    poses = w.grid_poses()[::53]
    noise = [(p, s) for p in (0.01, 0.05, 0.2, 0.5) for s in (0.003, 0.005, 0.01, 0.02, 0.04)]
    assert len(noise) > b3d_max_noise() and len({s for _, s in noise}) > 4
    gpu_ctx.set_likelihood(noise, 0.1, 2)
    s, _ = gpu_ctx.score_poses(mid, poses)
    want = _oracle_scores(oracle, w, poses, noise, 2)
    assert rel_err(s, want).max() <= RTOL
    # the device pose grid path and a 13-entry list with one sigma
    grid = gpu_ctx.make_grid(w.center, w.extent, w.count, w.rotations, w.grid_mode)
    noise13 = [(0.01 + 0.02 * i, 0.005) for i in range(13)]
    gpu_ctx.set_likelihood(noise13, 0.1, 1)
    sg, _ = gpu_ctx.score_grid(mid, grid)
    idx = np.arange(0, 1024, 97)
    want = _oracle_scores(oracle, w, w.grid_poses()[idx], noise13, 1)
    assert rel_err(sg[idx], want).max() <= RTOL


def b3d_max_noise():
    return 12


def test_window_negative_is_the_full_likelihood(gpu_ctx, oracle):
    w, mid = _ctx_cfg1(gpu_ctx)
    poses = w.grid_poses()[::101]
    noise = [(0.01, 0.005), (0.3, 0.02)]
    gpu_ctx.set_likelihood(noise, 0.1, -1)
    s, st = gpu_ctx.score_poses(mid, poses)
    assert (st == 0).all()
    for i, p in enumerate(poses):
        rend = oracle.render(w.k, [(w.vertices, w.triangles, p)])
        for e, nz in enumerate(noise):
            want = oracle.full_loglik(w.observed, rend, w.k, nz, 0.1)
            assert abs(s[i, e] - want) <= 1e-9 * abs(want)
    # empty render under the full form: -inf (inference.cpp:54)
    far = poses[:1].copy()
    far[0, 4:] = [0.0, 0.0, -1.0]  # behind the camera
    s, st = gpu_ctx.score_poses(mid, far)
    assert np.isneginf(s).all() and st[0] == 1


@pytest.mark.parametrize("p_out", [0.0, 1e-9])
def test_zero_and_tiny_outlier_probability_match_fp64(gpu_ctx, oracle, p_out):
    """p_outlier = 0: a pixel with no rendered point in its window gives
    log(0) = -inf (likelihood.cpp:216); with p tiny, windows whose points are
    far enough that an fp32 exp underflows still give finite fp64 terms."""
    w, mid = _ctx_cfg1(gpu_ctx)
    clean = oracle.render(w.k, [(w.vertices, w.triangles, w.gt_pose)])
    gpu_ctx.set_observation(clean)
    poses = np.concatenate([w.gt_pose[None], w.grid_poses()[::29]])
    noise = [(p_out, 0.0005), (p_out, 0.005)]  # a narrow sigma: exp(-d2/2s2) underflows fp32
    for win in (0, 2):
        gpu_ctx.set_likelihood(noise, 0.1, win)
        s, _ = gpu_ctx.score_poses(mid, poses)
        want = oracle.score_poses(w.k, clean, w.vertices, w.triangles, poses, noise, 0.1, win)[0]
        np.testing.assert_array_equal(np.isfinite(s), np.isfinite(want))
        fin = np.isfinite(want)
        assert fin.any()
        assert rel_err(s[fin], want[fin]).max() <= 1e-9
    gpu_ctx.set_observation(w.observed)


def test_coarse_to_fine_stage_on_the_fp64_path(gpu_ctx, oracle):
    """A stage with p_outlier = 0 inside the device chain equals score_grid +
    stage_reduce under the same settings."""
    w, mid = _ctx_cfg1(gpu_ctx)
    stages = [{"extent": w.extent, "count": (4, 4, 4), "rotations": w.rotations[:8], "mode": 0,
               "noise": (0.0, 0.01), "window": 2, "select": 1}]
    res, centers = gpu_ctx.coarse_to_fine(mid, w.gt_pose, stages)
    gpu_ctx.set_likelihood([(0.0, 0.01)], 0.1, 2)
    grid = gpu_ctx.make_grid(w.gt_pose, w.extent, (4, 4, 4), w.rotations[:8], 0)
    s, _ = gpu_ctx.score_grid(mid, grid)
    r = gpu_ctx.stage_reduce(s[:, 0])
    assert r.argmax == res[0].argmax and r.max_score == res[0].max_score


def _camera_world(gpu_ctx, oracle):
    seq = configs.orbit_sequence(None, oracle.voxel_to_mesh, oracle.box_mesh,
                                 oracle.contact_to_pose, 40)
    gpu_ctx.set_camera(b3d_intr(seq["k"]))
    mids = [gpu_ctx.upload_mesh(v, t) for v, t, _ in seq["instances"]]
    gpu_ctx.set_camera_scene(mids, [p for _, _, p in seq["instances"]])
    cams = np.array([oracle.camera_pose_from_spherical(0.9, a, seq["altitude"])
                     for a in (0.0, 0.3, 0.6)])
    obs = oracle.render(seq["k"], seq["instances"], camera=cams[1])
    gpu_ctx.set_observation(obs)
    return seq, cams, obs


def test_camera_paths_follow_the_windowed_seam(gpu_ctx, oracle):
    seq, cams, obs = _camera_world(gpu_ctx, oracle)
    gpu_ctx.set_likelihood([(0.1, 0.005)], 0.1, -1)
    with pytest.raises(b3d.B3DError, match="window radius must be >= 0"):
        gpu_ctx.score_cameras(cams)
    gpu_ctx.set_likelihood([(0.1, -0.005)], 0.1, 1)
    with pytest.raises(b3d.B3DError, match="sigma_noise must be positive"):
        gpu_ctx.score_cameras(cams)
    # sigma > sigma_max is scored by windowed_log_likelihood_multi
    noise = [(0.1, 0.2), (0.0, 0.003)] + [(0.05 * i, 0.001 * i) for i in range(1, 14)]
    gpu_ctx.set_likelihood(noise, 0.1, 1)
    s, _ = gpu_ctx.score_cameras(cams)
    for i, c in enumerate(cams):
        rend = oracle.render(seq["k"], seq["instances"], camera=c)
        want = oracle.windowed_loglik_multi(obs, rend, seq["k"], noise, 0.1, 1)
        np.testing.assert_array_equal(np.isfinite(s[i]), np.isfinite(want))
        fin = np.isfinite(want)
        assert rel_err(s[i][fin], want[fin]).max() <= RTOL
