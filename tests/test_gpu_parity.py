"""GPU parity: the sm_100a product path (through the C ABI) against the CPU
oracle on the same seeded inputs.

Bars (BASELINE.json north_star): per-pixel depth and triangle ids
bit-exact (the kernels follow the oracle's fp64 operation order with no FMA;
the north_star allows 1e-5 relative on depth, we require equality), log
scores within 1e-4 relative (fp32 likelihood terms, fp64 accumulation), argmax
identical unless the two top scores tie within that tolerance.
"""
import numpy as np
import pytest

from helpers import b3d_intr, cfg1_oracle, rel_err, square_k
from paper_2312_08715_b200 import b3d, configs, synth

pytestmark = pytest.mark.gpu

SCORE_RTOL = 1e-4


def _setup(ctx, w):
    ctx.set_camera(b3d_intr(w.k))
    mid = ctx.upload_mesh(w.vertices, w.triangles)
    ctx.set_observation(w.observed)
    ctx.set_likelihood(w.noise, w.sigma_max, w.window)
    return mid


def _render_parity(ctx, oracle, k, verts, tris, poses):
    ctx.set_camera(b3d_intr(k))
    mid = ctx.upload_mesh(verts, tris)
    depth, ids = ctx.render_poses(mid, poses, with_ids=True)
    for i in range(poses.shape[0]):
        od, oi = oracle.render(k, [(verts, tris, poses[i])], with_ids=True)
        np.testing.assert_array_equal(depth[i].view(np.uint32), od.view(np.uint32),
                                      err_msg=f"depth bits differ, hypothesis {i}")
        np.testing.assert_array_equal(ids[i], oi, err_msg=f"triangle ids differ, hypothesis {i}")
    # depth-only render mode agrees with the id mode
    d2, _ = ctx.render_poses(mid, poses, with_ids=False)
    np.testing.assert_array_equal(d2.view(np.uint32), depth.view(np.uint32))
    return depth, ids


def test_render_parity_cfg1(gpu_ctx, oracle):
    w = cfg1_oracle()
    poses = w.grid_poses()[::16]
    depth, ids = _render_parity(gpu_ctx, oracle, w.k, w.vertices, w.triangles, poses)
    assert (ids >= 0).sum() > 1000


def test_render_parity_random_walk_blob(gpu_ctx, oracle):
    w = cfg1_oracle(seed=3, blob="random_walk")
    _render_parity(gpu_ctx, oracle, w.k, w.vertices, w.triangles, w.grid_poses()[::64])


def test_render_parity_near_clipping_and_overflow(gpu_ctx, oracle):
    """Objects crossing z = near (renderer.cpp:127-141): the clipped fan path
    and the full-image region that spills to global scratch."""
    w = cfg1_oracle()
    rng = np.random.Generator(np.random.PCG64(5))
    poses = []
    for i in range(12):
        q = synth.uniform_quaternion(rng)
        poses.append([q[0], q[1], q[2], q[3], rng.uniform(-0.01, 0.01),
                      rng.uniform(-0.01, 0.01), rng.uniform(0.005, 0.05)])
    poses = np.array(poses)
    depth, ids = _render_parity(gpu_ctx, oracle, w.k, w.vertices, w.triangles, poses)
    assert (ids >= 0).mean() > 0.2  # big on screen


def test_render_parity_large_mesh_vertex_spill(gpu_ctx, oracle):
    """A 4,000-voxel random-walk blob (>64 KB of projected vertices) uses the
    global vertex scratch instead of shared memory."""
    vox = synth.random_walk_blob(4000, 11)
    verts, tris = configs.make_mesh(vox, oracle.voxel_to_mesh)
    assert verts.shape[0] * 24 > 64 * 1024
    k = configs.Intr(250.0, 250.0, 100.0, 100.0, 200, 200, 0.01, 10.0)
    rng = np.random.Generator(np.random.PCG64(2))
    poses = np.array([[*synth.uniform_quaternion(rng), 0.0, 0.0, 0.9] for _ in range(4)])
    _render_parity(gpu_ctx, oracle, k, verts, tris, poses)


def test_render_parity_table_box_scene(gpu_ctx, oracle):
    """A box mesh (make_box_mesh) seen from a spherical camera, as in the
    reference renderer tests (test_renderer.cpp:172-197)."""
    k = square_k(32)
    verts, tris = oracle.box_mesh([-0.05, -0.04, 0.0], [0.05, 0.04, 0.09])
    cams = [oracle.camera_pose_from_spherical(0.5 + 0.1 * i, 0.7 * i, 0.5 + 0.05 * i)
            for i in range(6)]
    gpu_ctx.set_camera(b3d_intr(k))
    mid = gpu_ctx.upload_mesh(verts, tris)
    ident = np.array([[1, 0, 0, 0, 0, 0, 0.0]])
    for cam in cams:
        gpu_ctx.set_camera(b3d_intr(k), cam)
        d, ids = gpu_ctx.render_poses(mid, ident)
        od, oi = oracle.render(k, [(verts, tris, ident[0])], camera=cam, with_ids=True)
        np.testing.assert_array_equal(d[0].view(np.uint32), od.view(np.uint32))
        np.testing.assert_array_equal(ids[0], oi)


def test_score_parity_cfg1(gpu_ctx, oracle):
    w = cfg1_oracle()
    mid = _setup(gpu_ctx, w)
    grid = gpu_ctx.make_grid(w.center, w.extent, w.count, w.rotations, w.grid_mode)
    s_gpu, st_gpu = gpu_ctx.score_grid(mid, grid)
    poses = w.grid_poses()
    s_orc, st_orc = oracle.score_poses(w.k, w.observed, w.vertices, w.triangles, poses, w.noise,
                                       w.sigma_max, w.window)
    np.testing.assert_array_equal(st_gpu, st_orc)
    assert rel_err(s_gpu, s_orc).max() <= SCORE_RTOL
    # the fp32 likelihood terms are far tighter than the bar in practice
    assert np.abs(s_gpu - s_orc).max() < 0.05
    a_gpu, a_orc = int(np.argmax(s_gpu[:, 0])), oracle.argmax(s_orc[:, 0])
    if a_gpu != a_orc:
        assert abs(s_orc[a_gpu, 0] - s_orc[a_orc, 0]) <= SCORE_RTOL * abs(s_orc[a_orc, 0])
    # explicit poses == device grid, bitwise
    s_p, _ = gpu_ctx.score_poses(mid, poses)
    np.testing.assert_array_equal(s_p, s_gpu)


def test_score_parity_multi_noise(gpu_ctx, oracle):
    w = cfg1_oracle(seed=1)
    noise = [(0.01, 0.005), (0.3, 0.005), (0.05, 0.02), (0.8, 0.01)]
    gpu_ctx.set_camera(b3d_intr(w.k))
    mid = gpu_ctx.upload_mesh(w.vertices, w.triangles)
    gpu_ctx.set_observation(w.observed)
    gpu_ctx.set_likelihood(noise, 0.1, 2)
    poses = w.grid_poses()[::8]
    s_gpu, _ = gpu_ctx.score_poses(mid, poses)
    s_orc, _ = oracle.score_poses(w.k, w.observed, w.vertices, w.triangles, poses, noise, 0.1, 2)
    assert rel_err(s_gpu, s_orc).max() <= SCORE_RTOL


def test_score_uniform_prefactor_and_windows(gpu_ctx, oracle):
    w = cfg1_oracle(seed=2)
    poses = w.grid_poses()[::32]
    gpu_ctx.set_camera(b3d_intr(w.k))
    mid = gpu_ctx.upload_mesh(w.vertices, w.triangles)
    gpu_ctx.set_observation(w.observed)
    for window in (0, 1, 3, 5):
        gpu_ctx.set_likelihood(w.noise, 0.1, window, b3d.PREFACTOR_UNIFORM)
        s_gpu, _ = gpu_ctx.score_poses(mid, poses)
        s_orc, _ = oracle.score_poses(w.k, w.observed, w.vertices, w.triangles, poses, w.noise,
                                      0.1, window, prefactor=1)
        assert rel_err(s_gpu, s_orc).max() <= SCORE_RTOL, window


def test_empty_render_status(gpu_ctx, oracle):
    """Hypotheses entirely behind the camera render nothing: the reference
    throws (likelihood.cpp:159-160); batched scoring flags them and returns
    -inf so the rest of the batch survives."""
    w = cfg1_oracle()
    mid = _setup(gpu_ctx, w)
    poses = w.grid_poses()[:4].copy()
    poses[1, 6] = -0.5
    poses[3, 4] = 50.0
    s, st = gpu_ctx.score_poses(mid, poses)
    assert list(st) == [0, 1, 0, 1]
    assert np.isneginf(s[1, 0]) and np.isneginf(s[3, 0])
    assert np.isfinite(s[0, 0]) and np.isfinite(s[2, 0])


def test_stage_reduce_matches_oracle(gpu_ctx, oracle):
    rng = np.random.Generator(np.random.PCG64(9))
    # sizes above 16,384 take the grid-wide reduction (stage.cu)
    for n in (1, 7, 1024, 16384, 16385, 32768, 100003, 1 << 20):
        x = rng.normal(-2.0e4, 30.0, size=n)
        if n > 10:
            x[n // 3] = x.max() + 5.0
            x[n // 2] = x[n // 3]  # tie: lowest index must win
            x[5] = -np.inf
        st_g = b3d.rng_seed(1234 + n)
        st_o = oracle.rng_seed(1234 + n)
        probs_g = np.zeros(n)
        r = gpu_ctx.stage_reduce(x, rng_state=st_g, probs=probs_g)
        probs_o, all_zero = oracle.normalize(x)
        assert r.argmax == oracle.argmax(x)
        assert not r.all_zero and not all_zero
        assert abs(r.logsumexp - oracle.logsumexp(x)) <= 1e-12 * abs(oracle.logsumexp(x))
        np.testing.assert_allclose(probs_g, probs_o, rtol=1e-12, atol=1e-300)
        assert r.sample == oracle.sample_categorical(probs_o, st_o)
        np.testing.assert_array_equal(st_g, st_o)  # stream advanced identically


def test_stage_reduce_all_neg_inf(gpu_ctx, oracle):
    for n in (1000, 50000):  # single-CTA and grid-wide paths
        x = np.full(n, -np.inf)
        st_g, st_o = b3d.rng_seed(5), oracle.rng_seed(5)
        r = gpu_ctx.stage_reduce(x, rng_state=st_g)
        probs_o, all_zero = oracle.normalize(x)
        assert r.all_zero and all_zero and r.argmax == 0
        assert r.sample == oracle.sample_categorical(probs_o, st_o)


def test_stage_reduce_nonfinite_entries(gpu_ctx, oracle):
    """NaN never wins the argmax and is counted (with +-inf) as non-finite,
    on both reduction paths."""
    rng = np.random.Generator(np.random.PCG64(4))
    for n in (3000, 70000):
        x = rng.normal(0.0, 1.0, size=n)
        x[[3, n // 2, n - 1]] = np.nan
        x[[7, n // 3]] = -np.inf
        r = gpu_ctx.stage_reduce(x)
        finite = np.where(np.isfinite(x), x, -np.inf)
        assert r.argmax == int(np.argmax(finite)) and r.n_nonfinite == 5


def test_log_likelihood_c_abi(oracle):
    """b3d_log_likelihood keeps the reference signature and semantics."""
    from helpers import make_k
    k = make_k(16, 16, 20.0, 0.1, 5.0)
    rng = np.random.Generator(np.random.PCG64(4))

    def surf(sp):
        img = np.full((16, 16), np.float32(5.0), dtype=np.float32)
        m = rng.random((16, 16)) >= sp
        img[m] = rng.uniform(0.5, 4.5, size=int(m.sum())).astype(np.float32)
        return img

    for trial in range(10):
        obs, ren = surf(0.3), surf(0.3)
        p, s = rng.uniform(0.05, 0.95), rng.uniform(0.01, 0.1)
        for window in (0, 2, 16):
            got = b3d.log_likelihood(obs, ren, b3d_intr(k), p, s, 0.1, window)
            want = oracle.windowed_loglik_multi(obs, ren, k, [(p, s)], 0.1, window)[0]
            assert abs(got - want) <= 1e-10 * abs(want)
        got = b3d.log_likelihood(obs, ren, b3d_intr(k), p, s, 0.1, -1)
        want = oracle.full_loglik(obs, ren, k, (p, s), 0.1)
        assert abs(got - want) <= 1e-10 * abs(want)
    empty = np.full((16, 16), np.float32(5.0), dtype=np.float32)
    with pytest.raises(b3d.B3DError, match="empty rendered cloud"):
        b3d.log_likelihood(surf(0.3), empty, b3d_intr(k), 0.5, 0.01, 0.1, 2)


def test_device_pointers_async_path(gpu_ctx, oracle):
    """Device-resident inputs/outputs (torch CUDA tensors) give the same bits
    as the host-buffer path."""
    import torch
    w = cfg1_oracle()
    mid = _setup(gpu_ctx, w)
    poses = w.grid_poses()
    s_host, _ = gpu_ctx.score_poses(mid, poses)
    dp = torch.from_numpy(poses).cuda()
    ds = torch.zeros((poses.shape[0], 1), dtype=torch.float64, device="cuda")
    dst = torch.zeros(poses.shape[0], dtype=torch.uint8, device="cuda")
    gpu_ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    gpu_ctx.set_observation(torch.from_numpy(w.observed).cuda())
    gpu_ctx.score_poses(mid, dp, ds, dst)
    torch.cuda.synchronize()
    gpu_ctx.set_stream(None)
    np.testing.assert_array_equal(ds.cpu().numpy(), s_host)


def _oracle_stage(oracle, w, center, g):
    poses = configs.grid_poses(center, g["extent"], g["count"], g["rotations"], g.get("mode", 0))
    s, _ = oracle.score_poses(w.k, w.observed, w.vertices, w.triangles, poses, [g["noise"]],
                              w.sigma_max, g["window"])
    return poses, s[:, 0]


def test_coarse_to_fine_chain_matches_oracle(gpu_ctx, oracle):
    """Device-resident stage chain (b3d_gpu_coarse_to_fine): every stage's
    selection equals the oracle's reduce/sample semantics applied to that
    stage's scores, each next centre is bitwise the selected grid pose, the
    device Rng stream advances exactly like the reference Rng, and the stage
    scores match the oracle's within the score tolerance."""
    from helpers import b3d_intr
    rf = lambda k, v, t, p: oracle.render(k, [(v, t, p)])
    w = configs.cfg2(rf, oracle.voxel_to_mesh, seed=1, counts=(4, 4, 4), n_rot=4)
    gpu_ctx.set_camera(b3d_intr(w.k))
    mid = gpu_ctx.upload_mesh(w.vertices, w.triangles)
    gpu_ctx.set_observation(w.observed)
    gpu_ctx.set_likelihood([w.stages[0]["noise"]], w.sigma_max, 1)
    st = b3d.rng_seed(2024)
    res, centers = gpu_ctx.coarse_to_fine(mid, w.center, w.stages, rng_state=st)
    st_o = oracle.rng_seed(2024)
    np.testing.assert_array_equal(centers[0], w.center)
    for s, g in enumerate(w.stages):
        # GPU scores of this stage (same centre) via score-many
        gpu_ctx.set_likelihood([g["noise"]], w.sigma_max, g["window"])
        grid = gpu_ctx.make_grid(centers[s], g["extent"], g["count"], g["rotations"], 0)
        s_gpu, _ = gpu_ctx.score_grid(mid, grid)
        poses, s_orc = _oracle_stage(oracle, w, centers[s], g)
        assert rel_err(s_gpu[:, 0], s_orc).max() <= SCORE_RTOL
        probs, _ = oracle.normalize(s_gpu[:, 0])
        pick = oracle.sample_categorical(probs, st_o)
        assert res[s].sample == pick and res[s].argmax == oracle.argmax(s_gpu[:, 0])
        np.testing.assert_array_equal(centers[s + 1], poses[pick])
    np.testing.assert_array_equal(st, st_o)


def test_coarse_to_fine_argmax_selection(gpu_ctx, oracle):
    from helpers import b3d_intr
    rf = lambda k, v, t, p: oracle.render(k, [(v, t, p)])
    w = configs.cfg2(rf, oracle.voxel_to_mesh, seed=2, counts=(4, 4, 2), n_rot=2, n_stages=2)
    for g in w.stages:
        g["select"] = b3d.SELECT_ARGMAX
    gpu_ctx.set_camera(b3d_intr(w.k))
    mid = gpu_ctx.upload_mesh(w.vertices, w.triangles)
    gpu_ctx.set_observation(w.observed)
    gpu_ctx.set_likelihood([w.stages[0]["noise"]], w.sigma_max, 1)
    res, centers = gpu_ctx.coarse_to_fine(mid, w.center, w.stages)
    for s, g in enumerate(w.stages):
        gpu_ctx.set_likelihood([g["noise"]], w.sigma_max, g["window"])
        grid = gpu_ctx.make_grid(centers[s], g["extent"], g["count"], g["rotations"], 0)
        s_gpu, _ = gpu_ctx.score_grid(mid, grid)
        a = int(np.argmax(s_gpu[:, 0]))
        assert res[s].argmax == a
        poses = configs.grid_poses(centers[s], g["extent"], g["count"], g["rotations"], 0)
        np.testing.assert_array_equal(centers[s + 1], poses[a])


def _cfg3(oracle, counts=(4, 4, 8)):
    rs = lambda k, cam, inst: oracle.render(k, inst, camera=cam)
    return configs.cfg3(rs, oracle.voxel_to_mesh, oracle.box_mesh, oracle.contact_to_pose,
                        counts=counts)


def _setup_cfg3(ctx, oracle, w):
    from helpers import b3d_intr
    ctx.set_camera(b3d_intr(w["k"]), w["camera"])
    tv, tt = w["table"][0], w["table"][1]
    mids = [ctx.upload_mesh(tv, tt)] + [ctx.upload_mesh(o[0], o[1]) for o in w["objects"]]
    ident = np.array([1.0, 0, 0, 0, 0, 0, 0])
    ctx.set_base_scene([mids[0]] + [mids[1 + i] for i in w["base"]],
                       [ident] + [w["poses"][i] for i in w["base"]])
    base_inst = [(tv, tt, ident)] + [(w["objects"][i][0], w["objects"][i][1], w["poses"][i])
                                     for i in w["base"]]
    return mids, base_inst


def test_base_scene_render_parity(gpu_ctx, oracle):
    """compose_render (inference.cpp:102-109): a fixed table + 3 objects
    rendered once, the enumerated object composited per hypothesis; depth and
    global draw indices bit-identical to rendering the whole scene."""
    w = _cfg3(oracle)
    mids, base_inst = _setup_cfg3(gpu_ctx, oracle, w)
    o = w["objects"][w["target"]]
    g = b3d.ContactGrid.make(0.5, 0.5, o[2], o[3], 1, (4, 4, 8))
    poses = b3d.contact_grid_poses(g)[::9]
    depth, ids = gpu_ctx.render_poses(mids[1 + w["target"]], poses)
    for i in range(poses.shape[0]):
        od, oi = oracle.render(w["k"], base_inst + [(o[0], o[1], poses[i])], camera=w["camera"],
                               with_ids=True)
        np.testing.assert_array_equal(depth[i].view(np.uint32), od.view(np.uint32))
        np.testing.assert_array_equal(ids[i], oi)
    gpu_ctx.set_base_scene([], [])


def test_base_scene_contact_grid_score_parity(gpu_ctx, oracle):
    """cfg3-shaped scoring: contact grid on the device, base scene composited,
    likelihood including the base-only term G(|y|) (Chebyshev interpolant)."""
    w = _cfg3(oracle)
    mids, base_inst = _setup_cfg3(gpu_ctx, oracle, w)
    gpu_ctx.set_observation(w["observed"])
    gpu_ctx.set_likelihood(w["noise"], w["sigma_max"], w["window"])
    o = w["objects"][w["target"]]
    g = b3d.ContactGrid.make(0.5, 0.5, o[2], o[3], 1, (4, 4, 8))
    s_gpu, st_gpu = gpu_ctx.score_contact_grid(mids[1 + w["target"]], g)
    poses = b3d.contact_grid_poses(g)
    base = oracle.render(w["k"], base_inst, camera=w["camera"])
    s_orc, st_orc = oracle.score_poses(w["k"], w["observed"], o[0], o[1], poses, w["noise"],
                                       w["sigma_max"], w["window"], base_depth=base,
                                       camera=w["camera"])
    assert (st_gpu == 0).all() and (st_orc == 0).all()
    assert rel_err(s_gpu, s_orc).max() <= SCORE_RTOL
    assert np.abs(s_gpu - s_orc).max() < 0.5
    # explicit poses through the same base scene
    s_p, _ = gpu_ctx.score_poses(mids[1 + w["target"]], poses)
    assert rel_err(s_p, s_orc).max() <= SCORE_RTOL
    gpu_ctx.set_base_scene([], [])


def test_sample_many_matches_sequential_draws(gpu_ctx, oracle):
    """1,000 posterior draws (cfg5's final step): each equals
    sample_categorical with the next uniform() of the same Rng stream."""
    rng = np.random.Generator(np.random.PCG64(21))
    for n in (5, 4096, 200003, 1 << 20):
        x = rng.normal(0.0, 3.0, size=n)
        st_g = b3d.rng_seed(77 + n)
        samples, r = gpu_ctx.sample_many(x, 1000, st_g)
        st_o = oracle.rng_seed(77 + n)
        probs, _ = oracle.normalize(x)
        want = [oracle.sample_categorical(probs, st_o) for _ in range(1000)]
        assert list(samples.astype(np.int64)) == want
        np.testing.assert_array_equal(st_g, st_o)
        assert r.argmax == oracle.argmax(x) and r.sample == want[0]


def test_score_grid_range_is_a_shard_of_the_grid(gpu_ctx, oracle):
    w = cfg1_oracle()
    mid = _setup(gpu_ctx, w)
    grid = gpu_ctx.make_grid(w.center, w.extent, w.count, w.rotations, w.grid_mode)
    full, _ = gpu_ctx.score_grid(mid, grid)
    for lo, hi in ((0, 100), (100, 611), (611, 1024)):
        part, _ = gpu_ctx.score_grid_range(mid, grid, lo, hi - lo)
        np.testing.assert_array_equal(part, full[lo:hi])


def test_tracking_frames_match_oracle(gpu_ctx, oracle):
    """cfg4 tracking: for the first frames, every stage's MAP hypothesis from
    the device chain equals the oracle's argmax over oracle scores (or ties it
    within the score tolerance), and the scores agree within 1e-4."""
    from helpers import b3d_intr
    rf = lambda k, v, t, p: oracle.render(k, [(v, t, p)])
    tr = configs.cfg4(rf, oracle.voxel_to_mesh, seed=0, n_frames=3)
    gpu_ctx.set_camera(b3d_intr(tr["k"]))
    mid = gpu_ctx.upload_mesh(tr["vertices"], tr["triangles"])
    st0 = tr["stages"][0]
    gpu_ctx.set_likelihood([st0["noise"]], 0.1, st0["window"])
    est = tr["gt"][0].copy()
    for f in (1, 2):
        gpu_ctx.set_observation(tr["frames"][f])
        res, centers = gpu_ctx.coarse_to_fine(mid, est, tr["stages"])
        for s, g in enumerate(tr["stages"]):
            poses = configs.grid_poses(centers[s], g["extent"], g["count"], g["rotations"], 0)
            s_orc, _ = oracle.score_poses(tr["k"], tr["frames"][f], tr["vertices"],
                                          tr["triangles"], poses, [g["noise"]], 0.1, g["window"])
            a_orc = oracle.argmax(s_orc[:, 0])
            a_gpu = res[s].argmax
            assert abs(res[s].max_score - s_orc[a_orc, 0]) <= SCORE_RTOL * abs(s_orc[a_orc, 0])
            if a_gpu != a_orc:
                assert abs(s_orc[a_gpu, 0] - s_orc[a_orc, 0]) <= SCORE_RTOL * abs(s_orc[a_orc, 0])
            np.testing.assert_array_equal(centers[s + 1], poses[a_gpu])
        est = centers[-1]


def test_enumerate_poses_one_call(gpu_ctx, oracle):
    """b3d_gpu_enumerate_poses == score_poses + stage_reduce."""
    import torch
    w = cfg1_oracle()
    mid = _setup(gpu_ctx, w)
    poses = torch.from_numpy(w.grid_poses()).pin_memory().numpy()
    st1, st2 = b3d.rng_seed(3), b3d.rng_seed(3)
    scores = np.zeros((poses.shape[0], 1))
    r1 = gpu_ctx.enumerate_poses(mid, poses, rng_state=st1, scores=scores)
    s2, _ = gpu_ctx.score_poses(mid, poses)
    r2 = gpu_ctx.stage_reduce(s2[:, 0], rng_state=st2)
    np.testing.assert_array_equal(scores, s2)
    assert (r1.argmax, r1.sample, r1.logsumexp) == (r2.argmax, r2.sample, r2.logsumexp)
    np.testing.assert_array_equal(st1, st2)
    # observation + enumeration in one boundary call (the bench's e2e step)
    st3 = b3d.rng_seed(3)
    obs = torch.from_numpy(np.ascontiguousarray(w.observed)).pin_memory().numpy()
    scores3 = np.zeros_like(scores)
    r3 = gpu_ctx.enumerate_observed(mid, obs, poses, rng_state=st3, scores=scores3)
    np.testing.assert_array_equal(scores3, s2)
    assert (r3.argmax, r3.sample) == (r2.argmax, r2.sample)


def test_base_scene_with_near_clipping_and_scratch(gpu_ctx, oracle):
    """Base scene + hypotheses crossing z = near: full-image regions that
    spill to the global z-buffer scratch, composited over the base keys."""
    w = _cfg3(oracle)
    mids, base_inst = _setup_cfg3(gpu_ctx, oracle, w)
    o = w["objects"][w["target"]]
    rng = np.random.Generator(np.random.PCG64(8))
    poses = []
    for _ in range(6):  # world poses close to the camera (camera at z = 0.7 looking down)
        q = synth.uniform_quaternion(rng)
        poses.append([q[0], q[1], q[2], q[3], rng.uniform(-0.02, 0.02), rng.uniform(-0.02, 0.02),
                      rng.uniform(0.66, 0.69)])
    poses = np.array(poses)
    depth, ids = gpu_ctx.render_poses(mids[1 + w["target"]], poses)
    for i in range(poses.shape[0]):
        od, oi = oracle.render(w["k"], base_inst + [(o[0], o[1], poses[i])], camera=w["camera"],
                               with_ids=True)
        np.testing.assert_array_equal(depth[i].view(np.uint32), od.view(np.uint32))
        np.testing.assert_array_equal(ids[i], oi)
    gpu_ctx.set_observation(w["observed"])
    gpu_ctx.set_likelihood(w["noise"], w["sigma_max"], w["window"])
    s_gpu, _ = gpu_ctx.score_poses(mids[1 + w["target"]], poses)
    base = oracle.render(w["k"], base_inst, camera=w["camera"])
    s_orc, _ = oracle.score_poses(w["k"], w["observed"], o[0], o[1], poses, w["noise"],
                                  w["sigma_max"], w["window"], base_depth=base, camera=w["camera"])
    assert rel_err(s_gpu, s_orc).max() <= SCORE_RTOL
    gpu_ctx.set_base_scene([], [])


def _scores_with_and_without_culling(ctx, fn):
    ctx.set_culling(True)
    a = fn()
    ctx.set_culling(False)
    b = fn()
    ctx.set_culling(True)
    return a, b


def test_back_face_culling_leaves_scores_bitwise_unchanged(gpu_ctx, oracle):
    """Score-many culls back faces of closed meshes: the
    region z-buffer and hence every score are bit-identical to the unculled
    render, for the cfg1 grid, another blob, a wide window and multi-noise."""
    w = cfg1_oracle()
    mid = _setup(gpu_ctx, w)
    assert gpu_ctx.mesh_cull_sign(mid) == 1
    grid = gpu_ctx.make_grid(w.center, w.extent, w.count, w.rotations, w.grid_mode)
    a, b = _scores_with_and_without_culling(gpu_ctx, lambda: gpu_ctx.score_grid(mid, grid)[0])
    np.testing.assert_array_equal(a, b)
    w2 = cfg1_oracle(seed=3, blob="random_walk")
    mid2 = gpu_ctx.upload_mesh(w2.vertices, w2.triangles)
    gpu_ctx.set_observation(w2.observed)
    gpu_ctx.set_likelihood([(0.01, 0.005), (0.2, 0.02)], 0.1, 3)
    rng = np.random.Generator(np.random.PCG64(9))
    poses = []
    for _ in range(256):
        q = synth.uniform_quaternion(rng)
        poses.append([*q, rng.uniform(-0.05, 0.05), rng.uniform(-0.05, 0.05),
                      rng.uniform(0.2, 1.2)])
    poses = np.array(poses)
    a, b = _scores_with_and_without_culling(gpu_ctx, lambda: gpu_ctx.score_poses(mid2, poses)[0])
    np.testing.assert_array_equal(a, b)
    # an inward-wound copy culls the other sign and still agrees
    mid3 = gpu_ctx.upload_mesh(w2.vertices, w2.triangles[:, ::-1])
    assert gpu_ctx.mesh_cull_sign(mid3) == -1
    c, _ = gpu_ctx.score_poses(mid3, poses)
    np.testing.assert_array_equal(c, a)


def test_back_face_culling_with_base_scene_and_near_clip(gpu_ctx, oracle):
    """Culling composes with the base scene; hypotheses with a vertex in
    front of z = near are never culled."""
    w = _cfg3(oracle)
    mids, base_inst = _setup_cfg3(gpu_ctx, oracle, w)
    gpu_ctx.set_observation(w["observed"])
    gpu_ctx.set_likelihood(w["noise"], w["sigma_max"], w["window"])
    o = w["objects"][w["target"]]
    g = b3d.ContactGrid.make(0.5, 0.5, o[2], o[3], 1, (4, 4, 8))
    m = mids[1 + w["target"]]
    a, b = _scores_with_and_without_culling(gpu_ctx, lambda: gpu_ctx.score_contact_grid(m, g)[0])
    np.testing.assert_array_equal(a, b)
    rng = np.random.Generator(np.random.PCG64(8))
    poses = np.array([[*synth.uniform_quaternion(rng), rng.uniform(-0.02, 0.02),
                       rng.uniform(-0.02, 0.02), rng.uniform(0.66, 0.69)] for _ in range(6)])
    a, b = _scores_with_and_without_culling(gpu_ctx, lambda: gpu_ctx.score_poses(m, poses)[0])
    np.testing.assert_array_equal(a, b)
    gpu_ctx.set_base_scene([], [])


def _orbit(oracle, res, n_frames=40, n_voxels=600, ref_frames=False):
    """ref_frames: the reference's sample_observation frames (oracle restatement,
    Rng(0).split(0, res).split(0x0f, i))."""
    rc = lambda k, inst, cams: np.stack([oracle.render(k, inst, camera=c) for c in cams])
    kw = {}
    if ref_frames:
        kw = dict(sample_fn=lambda k, d, p, s, st: np.stack([
            oracle.sample_observation(d[i], k, p, s, oracle.rng_split(st, 0x0F, i))
            for i in range(d.shape[0])]),
                  rng_state=oracle.rng_split(oracle.rng_seed(0), 0, res))
    return configs.orbit_sequence(rc, oracle.voxel_to_mesh, oracle.box_mesh,
                                  oracle.contact_to_pose, res=res, n_frames=n_frames,
                                  n_voxels=n_voxels, **kw)


def _camera_scene(ctx, seq):
    from helpers import b3d_intr
    ctx.set_camera(b3d_intr(seq["k"]))
    mids = [ctx.upload_mesh(v, t) for v, t, _ in seq["instances"]]
    ctx.set_camera_scene(mids, [p for _, _, p in seq["instances"]])


def test_render_cameras_multi_instance_parity(gpu_ctx, oracle):
    """render_instances (renderer.cpp:153-189) of table + object under camera
    hypotheses: depth and global draw indices bit-identical to the oracle,
    including cameras close enough to clip the table at z = near."""
    for res in (50, 100):
        seq = _orbit(oracle, res)
        _camera_scene(gpu_ctx, seq)
        rng = np.random.Generator(np.random.PCG64(res))
        cams = [oracle.camera_pose_from_spherical(rng.uniform(0.3, 1.5), rng.uniform(0, 6.28),
                                                  rng.uniform(0.2, 1.4)) for _ in range(8)]
        cams.append(oracle.camera_pose_from_spherical(0.12, 0.5, 0.3))  # near-plane clipping
        d, ids = gpu_ctx.render_cameras(np.array(cams))
        for i, c in enumerate(cams):
            od, oi = oracle.render(seq["k"], seq["instances"], camera=c, with_ids=True)
            np.testing.assert_array_equal(d[i].view(np.uint32), od.view(np.uint32))
            np.testing.assert_array_equal(ids[i], oi)
        assert (ids[:-1] >= seq["instances"][0][1].shape[0]).any()  # object pixels present


def test_score_cameras_parity(gpu_ctx, oracle):
    seq = _orbit(oracle, 100)
    _camera_scene(gpu_ctx, seq)
    cam0 = oracle.camera_pose_from_spherical(seq["distance"], 0.4, seq["altitude"])
    obs = configs.orbit_frames(seq, [cam0])[0]
    gpu_ctx.set_observation(obs)
    gpu_ctx.set_likelihood([seq["noise"]], seq["sigma_max"], seq["window"])
    rng = np.random.Generator(np.random.PCG64(12))
    cams = np.array([oracle.camera_pose_from_spherical(0.9 + rng.uniform(-0.05, 0.05),
                                                       0.4 + rng.uniform(-0.2, 0.2),
                                                       seq["altitude"] + rng.uniform(-0.2, 0.2))
                     for _ in range(64)])
    s_gpu, st = gpu_ctx.score_cameras(cams)
    s_orc = np.array([oracle.windowed_loglik_multi(
        obs, oracle.render(seq["k"], seq["instances"], camera=c), seq["k"], [seq["noise"]],
        seq["sigma_max"], seq["window"])[0] for c in cams])
    assert (st == 0).all()
    assert rel_err(s_gpu[:, 0], s_orc).max() <= SCORE_RTOL


def test_track_camera_matches_oracle(gpu_ctx, oracle):
    """bench-tracking's orbit (harness.cpp:743-770) at 50 x 50: the device
    track_camera picks the oracle's lattice point at every frame (poses
    bitwise equal; a differing pick must tie within the score tolerance)."""
    seq = _orbit(oracle, 50, ref_frames=True)
    _camera_scene(gpu_ctx, seq)
    gpu_ctx.set_likelihood([seq["noise"]], seq["sigma_max"], seq["window"])
    cams = [oracle.camera_pose_from_spherical(seq["distance"], a, seq["altitude"])
            for a in seq["azimuths"][:4]]
    frames = configs.orbit_frames(seq, cams)
    est, ms = gpu_ctx.track_camera(frames, cams[0])
    log = []
    ref = oracle.track_camera(frames, seq["k"], seq["instances"], cams[0], seq["noise"],
                              seq["sigma_max"], seq["window"], stage_log=log)
    assert (ms > 0).all()
    for f in range(4):
        if not np.array_equal(est[f], ref[f]):
            # only a score tie inside the tolerance may flip the pick
            _, _, grid, scores = [e for e in log if e[0] == f][-1]
            s = np.array(scores)
            assert np.sort(s)[-1] - np.sort(s)[-2] <= SCORE_RTOL * abs(np.max(s))
        assert np.linalg.norm(est[f][4:] - cams[f][4:]) < 0.03


@pytest.mark.parametrize("ppd,stages,beam", [(4, 1, 1), (3, 3, 1), (5, 2, 2)])
def test_track_camera_search_variants_match_oracle(gpu_ctx, oracle, ppd, stages, beam):
    """Other TrackSearch settings: the device stage chain (beam 1; even
    lattices, deeper refinement) and the host beam path (beam 2) pick the
    oracle's lattice points (a differing pick must tie within the tolerance)."""
    seq = _orbit(oracle, 25, ref_frames=True)
    _camera_scene(gpu_ctx, seq)
    gpu_ctx.set_likelihood([seq["noise"]], seq["sigma_max"], seq["window"])
    cams = [oracle.camera_pose_from_spherical(seq["distance"], a, seq["altitude"])
            for a in seq["azimuths"][:4]]
    frames = configs.orbit_frames(seq, cams)
    search = b3d.TrackSearch.default(points_per_dim=ppd, refine_stages=stages, beam_width=beam)
    est, _ = gpu_ctx.track_camera(frames, cams[0], search)
    log = []
    ref = oracle.track_camera(frames, seq["k"], seq["instances"], cams[0], seq["noise"],
                              seq["sigma_max"], seq["window"], points_per_dim=ppd,
                              refine_stages=stages, beam_width=beam, stage_log=log)
    for f in range(4):
        if not np.array_equal(est[f], ref[f]):
            _, _, grid, scores = [e for e in log if e[0] == f][-1]
            s = np.sort(np.array(scores))
            assert s[-1] - s[-2] <= SCORE_RTOL * abs(s[-1])


def test_track_camera_device_frames_equal_host_frames(gpu_ctx, oracle):
    """Frames already on the device (no per-frame upload) track identically."""
    import torch
    seq = _orbit(oracle, 50, ref_frames=True)
    _camera_scene(gpu_ctx, seq)
    gpu_ctx.set_likelihood([seq["noise"]], seq["sigma_max"], seq["window"])
    cams = [oracle.camera_pose_from_spherical(seq["distance"], a, seq["altitude"])
            for a in seq["azimuths"][:6]]
    frames = configs.orbit_frames(seq, cams)
    est_h, _ = gpu_ctx.track_camera(frames, cams[0])
    est_d, _ = gpu_ctx.track_camera(torch.from_numpy(frames).cuda(), cams[0])
    np.testing.assert_array_equal(est_h, est_d)


def test_orbit_frames_equal_the_reference(gpu_ctx, oracle):
    """generate_orbit_sequence (tracking.cpp:174-206) as the bench builds it:
    device camera renders + the product's sample_observation on split streams
    give frames bitwise equal to the oracle's render + sample_observation."""
    for res in (25, 100):
        seq = _orbit(oracle, res, ref_frames=True)
        _camera_scene(gpu_ctx, seq)
        cams = np.array([oracle.camera_pose_from_spherical(seq["distance"], a, seq["altitude"])
                         for a in seq["azimuths"][:6]])
        want = configs.orbit_frames(seq, cams)
        d = gpu_ctx.render_cameras(cams, with_ids=False)[0]
        got = b3d.sample_observations(b3d_intr(seq["k"]), d, *seq["noise"],
                                      b3d.rng_split(b3d.rng_seed(0), 0, res))
        assert got.tobytes() == want.tobytes()


def test_enumerate_grid_matches_score_then_reduce(gpu_ctx, oracle):
    """b3d_gpu_enumerate_grid (one call, device buffers): same scores,
    argmax, logsumexp, draw and Rng state as score_grid followed by
    stage_reduce, over repeated calls."""
    import torch
    w = cfg1_oracle()
    mid = _setup(gpu_ctx, w)
    rot = torch.from_numpy(w.rotations).cuda()
    grid = gpu_ctx.make_grid(w.center, w.extent, w.count, rot, w.grid_mode)
    n = w.n_hyp
    for rep in range(3):
        st_f = torch.from_numpy(b3d.rng_seed(11 + rep).view(np.int64)).cuda()
        out = torch.zeros(64, dtype=torch.uint8, device="cuda")
        sc = torch.zeros((n, 1), dtype=torch.float64, device="cuda")
        gpu_ctx.enumerate_grid(mid, grid, st_f, out, sc)
        torch.cuda.synchronize()
        s2, _ = gpu_ctx.score_grid(mid, grid)
        np.testing.assert_array_equal(sc.cpu().numpy(), s2)
        st_s = b3d.rng_seed(11 + rep)
        r2 = gpu_ctx.stage_reduce(s2[:, 0], rng_state=st_s)
        r1 = b3d.StageResult.from_buffer_copy(out.cpu().numpy().tobytes()[:C_SIZEOF_RESULT()])
        assert (r1.argmax, r1.sample, r1.logsumexp, r1.total) == (r2.argmax, r2.sample,
                                                                   r2.logsumexp, r2.total)
        np.testing.assert_array_equal(st_f.cpu().numpy().view(np.uint64), st_s)


def C_SIZEOF_RESULT():
    import ctypes
    return ctypes.sizeof(b3d.StageResult)


def test_score_parity_default_noise_grid(gpu_ctx, oracle):
    """default_noise_grid (inference.cpp:127-133): 9 noise entries over 3
    distinct sigmas in one call, against the oracle."""
    w = cfg1_oracle(seed=4)
    smax = 0.1
    noise = [(p, f * smax) for p in (0.05, 0.3, 0.8) for f in (0.25, 0.5, 1.0)]
    gpu_ctx.set_camera(b3d_intr(w.k))
    mid = gpu_ctx.upload_mesh(w.vertices, w.triangles)
    gpu_ctx.set_observation(w.observed)
    gpu_ctx.set_likelihood(noise, smax, 1)
    poses = w.grid_poses()[::16]
    s_gpu, _ = gpu_ctx.score_poses(mid, poses)
    s_orc, _ = oracle.score_poses(w.k, w.observed, w.vertices, w.triangles, poses, noise, smax, 1)
    assert s_gpu.shape == (poses.shape[0], 9)
    assert rel_err(s_gpu, s_orc).max() <= SCORE_RTOL


def _smc_setup(gpu_ctx, oracle, n_placed):
    import smc_case as S
    from helpers import b3d_intr

    def render_scene(k, cam, inst):
        return oracle.render(k, inst, camera=cam)
    lib, (tv, tt), obs, placed = S.build(oracle.voxel_to_mesh, oracle.box_mesh,
                                         oracle.contact_to_pose, render_scene, n_placed)
    gpu_ctx.set_camera(b3d_intr(S.K), S.CAMERA)
    table = gpu_ctx.upload_mesh(tv, tt)
    mids = [gpu_ctx.upload_mesh(v, t) for v, t, _, _ in lib]
    gpu_ctx.set_observation(obs)
    return S, lib, (tv, tt), obs, table, mids


def _compare_smc(ps_g, le_g, ps_o, le_o):
    assert len(ps_g) == len(ps_o)
    for (cg, eg, ltg, lwg), (co, eo, lto, lwo) in zip(ps_g, ps_o):
        assert eg == eo and len(cg) == len(co)
        for a, b in zip(cg, co):
            assert a[:2] == b[:2]                      # object, face
            assert np.allclose(a[2:], b[2:], rtol=0, atol=1e-12)  # same leaf draws
        assert abs(ltg - lto) <= SCORE_RTOL * abs(lto)
        assert abs(lwg - lwo) <= SCORE_RTOL * max(1.0, abs(lwo))
    assert abs(le_g - le_o) <= SCORE_RTOL * max(1.0, abs(le_o))


def test_run_smc_matches_oracle(gpu_ctx, oracle):
    """run_smc (inference.cpp:398-520) with every render+score on the device:
    stage-0 cells (2 objects x 6 faces x 36 cells x 9 noise entries), one
    refine stage, 4 particles; the same cells, leaf draws and noise choices
    as the oracle's restatement, weights within the score tolerance."""
    S, lib, (tv, tt), obs, table, mids = _smc_setup(gpu_ctx, oracle, 1)
    ps_g, le_g = gpu_ctx.run_smc([(mids[i], lib[i][2], lib[i][3]) for i in range(2)], table,
                                 S.TABLE_W, S.TABLE_H, S.SCHEDULE, S.NOISE_GRID, 0.1, 1,
                                 n_objects=1, n_particles=4, resample_threshold=0.5, seed=9)
    ps_o, le_o = oracle.run_smc(S.K, S.CAMERA, obs, lib, (tv, tt, S.TABLE_W, S.TABLE_H),
                                S.SCHEDULE, S.NOISE_GRID, 0.1, 1, n_objects=1, n_particles=4,
                                resample_threshold=0.5, seed=9)
    _compare_smc(ps_g, le_g, ps_o, le_o)
    gpu_ctx.set_base_scene([], [])


def test_run_smc_two_objects_with_extend_and_resampling(gpu_ctx, oracle):
    """smc_extend (per-particle partial scenes as the base image) and the
    ESS-triggered systematic resampling, against the oracle."""
    S, lib, (tv, tt), obs, table, mids = _smc_setup(gpu_ctx, oracle, 2)
    ps_g, le_g = gpu_ctx.run_smc([(mids[i], lib[i][2], lib[i][3]) for i in range(2)], table,
                                 S.TABLE_W, S.TABLE_H, S.SCHEDULE, S.NOISE_GRID, 0.1, 1,
                                 n_objects=2, n_particles=3, resample_threshold=0.9, seed=4)
    ps_o, le_o = oracle.run_smc(S.K, S.CAMERA, obs, lib, (tv, tt, S.TABLE_W, S.TABLE_H),
                                S.SCHEDULE, S.NOISE_GRID, 0.1, 1, n_objects=2, n_particles=3,
                                resample_threshold=0.9, seed=4)
    _compare_smc(ps_g, le_g, ps_o, le_o)
    gpu_ctx.set_base_scene([], [])


def test_b3d_render_scene_handle_matches_oracle(oracle):
    """b3d_render (b3d.h:107-108): render_depth of a scene JSON over an
    in-memory library (table + 2 children), bitwise equal to the oracle."""
    import json
    vox0, vox1 = synth.eden_blob(300, 1), synth.eden_blob(500, 2)
    m0 = b3d.Model.from_voxels(vox0, 0.005, np.zeros(3), 0)
    m1 = b3d.Model.from_voxels(vox1, 0.005, np.zeros(3), 1)
    lib = b3d.Library.create([m0, m1])
    children = [(1, 3, 0.1, 0.2, 0.7), (0, 1, 0.25, 0.05, 5.5)]
    sc = b3d.Scene.from_json(json.dumps({"table": {"width": 0.5, "height": 0.4},
                                         "children": [dict(object_id=o, face=f, dx=x, dy=y,
                                                           dtheta=t)
                                                      for o, f, x, y, t in children]}), lib)
    k = configs.Intr(200.0, 200.0, 79.5, 59.5, 160, 120, 0.05, 5.0)
    intr = b3d_intr(k)
    inst = [(*configs.table_mesh(oracle.box_mesh, 0.5, 0.4)[:2], np.array([1.0, 0, 0, 0, 0, 0, 0]))]
    for o, f, x, y, t in children:
        v, tt = (m0 if o == 0 else m1).mesh()
        pose = oracle.contact_to_pose(0.5, 0.4, v.min(axis=0), v.max(axis=0), f, x, y, t)
        inst.append((v, tt, pose))
    for d, az, alt in ((0.9, 0.3, 0.7), (0.6, 2.0, 1.1), (1.2, 4.0, 0.4)):
        cam = oracle.camera_pose_from_spherical(d, az, alt)
        got = b3d.render(sc, cam, intr)
        want = oracle.render(k, inst, camera=cam)
        np.testing.assert_array_equal(got.view(np.uint32), want.view(np.uint32))


def test_b3d_infer_matches_oracle_run_smc(oracle):
    """b3d_infer (b3d.h:121-124) with the `infer` JSON schema: particles,
    log-evidence and MAP pose agree with the oracle's run_smc on the same
    seed (same draws, weights within the score tolerance)."""
    import json
    import smc_case as S
    lib_o, (tv, tt), obs, placed = S.build(oracle.voxel_to_mesh, oracle.box_mesh,
                                           oracle.contact_to_pose,
                                           lambda k, c, i: oracle.render(k, i, camera=c))
    models = [b3d.Model.from_voxels(synth.eden_blob(n, 40 + i), configs.RESOLUTION,
                                    configs.synth.centered_origin(synth.eden_blob(n, 40 + i),
                                                                  configs.RESOLUTION), i)
              for i, n in enumerate((150, 260))]
    for m, lo in zip(models, lib_o):
        np.testing.assert_array_equal(m.mesh()[0], lo[0])
    lib = b3d.Library.create(models)
    cfg = {"intrinsics": {"fx": S.K.fx, "fy": S.K.fy, "cx": S.K.cx, "cy": S.K.cy,
                          "width": S.K.width, "height": S.K.height, "near": S.K.near,
                          "far": S.K.far},
           "table": {"width": S.TABLE_W, "height": S.TABLE_H}, "sigma_max": 0.1, "window": 1,
           "schedule": {"stage0": list(S.SCHEDULE[0]), "refine": [list(s) for s in S.SCHEDULE[1]]},
           "particles": 4, "resample_threshold": 0.5, "n_objects": 1}
    lines, le, marg, map_pose = b3d.infer(obs, S.CAMERA, lib, json.dumps(cfg), 9)
    ps_o, le_o = oracle.run_smc(S.K, S.CAMERA, obs, lib_o, (tv, tt, S.TABLE_W, S.TABLE_H),
                                S.SCHEDULE, S.NOISE_GRID, 0.1, 1, n_objects=1, n_particles=4,
                                resample_threshold=0.5, seed=9)
    assert len(lines) == 4 and abs(le - le_o) <= SCORE_RTOL * abs(le_o)
    for line, (co, eo, lto, lwo) in zip(lines, ps_o):
        j = json.loads(line)
        c = j["children"][0]
        assert (c["object_id"], c["face"]) == co[0][:2]
        assert np.allclose([c["dx"], c["dy"], c["dtheta"]], co[0][2:], rtol=0, atol=1e-12)
        assert (j["noise"]["p_outlier"], j["noise"]["sigma_noise"]) == S.NOISE_GRID[eo]
        assert abs(j["log_weight"] - lwo) <= SCORE_RTOL * max(1.0, abs(lwo))
    assert marg is not None and abs(marg.sum() - 1.0) < 1e-12
    best = max(ps_o, key=lambda p: p[2])
    o, f, x, y, t = best[0][0]
    want = oracle.contact_to_pose(S.TABLE_W, S.TABLE_H, lib_o[o][2], lib_o[o][3], f, x, y, t)
    np.testing.assert_allclose(map_pose, want, rtol=0, atol=1e-15)


def test_ragged_batches_and_image_borders(gpu_ctx, oracle):
    """Batch sizes that are not multiples of the persistent grid (1, 295,
    297), objects straddling the image borders (regions clipped to the
    image), and an empty batch (the reference's "score_cells: no cells")."""
    w = cfg1_oracle(seed=5)
    mid = _setup(gpu_ctx, w)
    rng = np.random.Generator(np.random.PCG64(31))
    base = w.grid_poses()
    for n in (1, 295, 297):
        poses = base[rng.choice(base.shape[0], n)].copy()
        # push about a third across the left / right / top / bottom borders
        shift = rng.integers(0, 6, n)
        poses[shift == 1, 4] -= 0.45
        poses[shift == 2, 4] += 0.45
        poses[shift == 3, 5] -= 0.34
        poses[shift == 4, 5] += 0.34
        s_gpu, st_gpu = gpu_ctx.score_poses(mid, poses)
        s_orc, st_orc = oracle.score_poses(w.k, w.observed, w.vertices, w.triangles, poses,
                                           w.noise, w.sigma_max, w.window)
        np.testing.assert_array_equal(st_gpu, st_orc)
        ok = st_orc == 0
        assert rel_err(s_gpu[ok], s_orc[ok]).max() <= SCORE_RTOL
    d, ids = gpu_ctx.render_poses(mid, base[:3] + np.array([0, 0, 0, 0, 0.42, 0.3, 0]))
    for i in range(3):
        od, oi = oracle.render(w.k, [(w.vertices, w.triangles, base[i] +
                                      np.array([0, 0, 0, 0, 0.42, 0.3, 0]))], with_ids=True)
        np.testing.assert_array_equal(d[i].view(np.uint32), od.view(np.uint32))
        np.testing.assert_array_equal(ids[i], oi)
    with pytest.raises(b3d.B3DError) as e:
        gpu_ctx.score_poses(mid, base[:0])
    assert "score_cells: no cells" in str(e.value)


def test_large_image_regions_in_global_scratch(gpu_ctx, oracle):
    """A 1,024 x 768 image with the object close enough that its region
    exceeds shared memory: the global-scratch instantiation, against the
    oracle (depth/ids bitwise, scores within the tolerance)."""
    w = cfg1_oracle(seed=6)
    k = configs.Intr(700.0, 700.0, 511.5, 383.5, 1024, 768, 0.01, 10.0)
    rf = lambda kk, v, t, p: oracle.render(kk, [(v, t, p)])
    obs = rf(k, w.vertices, w.triangles, np.array([*w.gt_pose[:4], 0.0, 0.0, 0.25]))
    gpu_ctx.set_camera(b3d_intr(k))
    mid = gpu_ctx.upload_mesh(w.vertices, w.triangles)
    gpu_ctx.set_observation(obs)
    gpu_ctx.set_likelihood([(0.05, 0.004)], 0.1, 2)
    rng = np.random.Generator(np.random.PCG64(3))
    poses = np.array([[*w.gt_pose[:4], rng.uniform(-0.01, 0.01), rng.uniform(-0.01, 0.01),
                       rng.uniform(0.2, 0.3)] for _ in range(6)])
    s_gpu, _ = gpu_ctx.score_poses(mid, poses)
    s_orc, _ = oracle.score_poses(k, obs, w.vertices, w.triangles, poses, [(0.05, 0.004)], 0.1, 2)
    assert rel_err(s_gpu, s_orc).max() <= SCORE_RTOL
    d, ids = gpu_ctx.render_poses(mid, poses[:2])
    for i in range(2):
        od, oi = oracle.render(k, [(w.vertices, w.triangles, poses[i])], with_ids=True)
        np.testing.assert_array_equal(d[i].view(np.uint32), od.view(np.uint32))
        np.testing.assert_array_equal(ids[i], oi)


def test_fused_score_gather_to_peer_buffers(gpu_ctx, oracle):
    """b3d_gpu_set_score_peers: the score kernel stores every score into each
    peer copy of the global array at its rank offset (the all-gather fused
    into the kernel); here two local buffers stand in for two ranks' copies."""
    import torch
    w = cfg1_oracle()
    mid = _setup(gpu_ctx, w)
    grid = gpu_ctx.make_grid(w.center, w.extent, w.count, torch.from_numpy(w.rotations).cuda(),
                             w.grid_mode)
    n = w.n_hyp
    a = torch.full((3 * n, 1), -1.0, dtype=torch.float64, device="cuda")
    b = torch.full((3 * n, 1), -1.0, dtype=torch.float64, device="cuda")
    sc = torch.zeros((n, 1), dtype=torch.float64, device="cuda")
    gpu_ctx.set_score_peers([a.data_ptr(), b.data_ptr()], n, 3 * n)  # this "rank" owns [n, 2n)
    try:
        gpu_ctx.score_grid(mid, grid, sc, None)
        torch.cuda.synchronize()
    finally:
        gpu_ctx.set_score_peers([], 0)
    for buf in (a, b):
        assert torch.equal(buf[n:2 * n], sc)
        assert (buf[:n] == -1).all() and (buf[2 * n:] == -1).all()
    s2, _ = gpu_ctx.score_grid(mid, grid)  # peers off again: plain scores
    np.testing.assert_array_equal(s2, sc.cpu().numpy())


def test_fused_score_gather_symmetric_memory_single_rank(gpu_ctx, oracle):
    """The bench's N > 1 plumbing on one rank: a 1-rank NCCL group,
    symmetric-memory rendezvous, the peer pointer from the handle, the
    symmetric-memory barrier."""
    import os
    import socket
    import torch
    import torch.distributed as dist
    try:
        import torch.distributed._symmetric_memory as symm_mem
    except Exception:
        pytest.skip("symmetric memory unavailable")
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        w = cfg1_oracle()
        mid = _setup(gpu_ctx, w)
        poses = torch.from_numpy(w.grid_poses()[:300]).cuda()
        try:
            sym = symm_mem.empty(300, 1, dtype=torch.float64, device="cuda")
            hdl = symm_mem.rendezvous(sym, dist.group.WORLD)
        except Exception as e:
            pytest.skip(f"symmetric memory rendezvous unavailable: {e}")
        sym.fill_(0.0)
        sc = torch.zeros((300, 1), dtype=torch.float64, device="cuda")
        gpu_ctx.set_score_peers([int(x) for x in hdl.buffer_ptrs], 0, 300)
        try:
            gpu_ctx.score_poses(mid, poses, sc, None)
            hdl.barrier(channel=0)
            torch.cuda.synchronize()
        finally:
            gpu_ctx.set_score_peers([], 0)
        assert torch.equal(sym, sc)
    finally:
        dist.destroy_process_group()


def test_device_voxel_to_mesh_matches_host_walk(gpu_ctx, oracle):
    """voxel_to_mesh on the device (hash sets + prefix scans) gives the
    reference walk's vertices, numbering and triangle order (geometry.cpp:142-177):
    blobs, a sparse random grid, duplicate voxels, negative coordinates, and
    device-resident input/output."""
    import torch
    rng = np.random.Generator(np.random.PCG64(5))
    grids = [synth.eden_blob(1000, 1), synth.random_walk_blob(3000, 2), synth.eden_blob(20000, 3),
             rng.integers(-40, 40, size=(5000, 3)).astype(np.int32),
             np.array([[0, 0, 0], [1, 0, 0], [0, 0, 0], [-7, 3, 1 << 19]], dtype=np.int32)]
    for g in grids:
        origin = (-0.0123, 0.5, 0.25)
        hv, ht = b3d.voxel_to_mesh(g, 0.005, origin)
        dv, dt = gpu_ctx.voxel_to_mesh(g, 0.005, origin)
        np.testing.assert_array_equal(dt, ht)
        np.testing.assert_array_equal(dv.view(np.uint64), hv.view(np.uint64))
        if g.shape[0] <= 1000:
            ov, ot = oracle.voxel_to_mesh(g, 0.005, origin)
            np.testing.assert_array_equal(ot, ht)
    tv, tt = gpu_ctx.voxel_to_mesh(torch.from_numpy(grids[1]).cuda(), 0.005, (0, 0, 0))
    hv, ht = b3d.voxel_to_mesh(grids[1], 0.005, (0, 0, 0))
    np.testing.assert_array_equal(tt.cpu().numpy().astype(np.uint32), ht)
    np.testing.assert_array_equal(tv.cpu().numpy(), hv)
    with pytest.raises(b3d.B3DError):
        gpu_ctx.voxel_to_mesh(np.array([[1 << 21, 0, 0]], dtype=np.int32), 0.005, (0, 0, 0))


def test_cfg5_full_size_shards_and_spot_parity(gpu_ctx, oracle):
    """BASELINE configs[4] at full size (1,048,576 hypotheses, 480x640, a
    10-object base scene): scoring the grid in four shards gives the single
    call's scores bitwise (the multi-GPU partition), and the global argmax plus
    15 random hypotheses score within 1e-4 of the oracle's composed render."""
    import torch
    from helpers import b3d_intr
    rs = lambda k, cam, inst: oracle.render(k, inst, camera=cam)
    w = configs.cfg5(rs, oracle.voxel_to_mesh, oracle.box_mesh, oracle.contact_to_pose)
    gpu_ctx.set_camera(b3d_intr(w["k"]), w["camera"])
    tv, tt = w["table"]
    mids = [gpu_ctx.upload_mesh(tv, tt)] + [gpu_ctx.upload_mesh(l[0], l[1]) for l in w["library"]]
    n_placed = len(w["base_poses"]) - 1
    gpu_ctx.set_base_scene([mids[0]] + [mids[1 + i] for i in range(n_placed)], w["base_poses"])
    gpu_ctx.set_observation(w["observed"])
    gpu_ctx.set_likelihood(w["noise"], w["sigma_max"], w["window"])
    d_rot = torch.from_numpy(w["rotations"]).cuda()
    grid = gpu_ctx.make_grid(w["gt"], w["extent"], w["count"], d_rot, b3d.GRID_PRODUCT)
    n = w["n_hyp"]
    mid = mids[1 + w["target"]]
    full = torch.zeros((n, 1), dtype=torch.float64, device="cuda")
    gpu_ctx.score_grid_range(mid, grid, 0, n, full, None)
    parts = torch.zeros_like(full)
    bounds = [0, n // 4, n // 2, 3 * n // 4 + 17, n]
    for lo, hi in zip(bounds[:-1], bounds[1:]):
        gpu_ctx.score_grid_range(mid, grid, lo, hi - lo, parts[lo:hi], None)
    torch.cuda.synchronize()
    assert torch.equal(full, parts)
    s = full[:, 0].cpu().numpy()
    rng = np.random.Generator(np.random.PCG64(55))
    pick = np.concatenate([[int(np.argmax(s))], rng.integers(0, n, size=15)])
    poses = configs.grid_poses(w["gt"], w["extent"], w["count"], w["rotations"], 0)[pick]
    base = [(tv, tt, w["base_poses"][0])] + [
        (w["library"][i][0], w["library"][i][1], w["base_poses"][1 + i]) for i in range(n_placed)]
    base_depth = oracle.render(w["k"], base, camera=w["camera"])
    lib_t = w["library"][w["target"]]
    s_orc, st = oracle.score_poses(w["k"], w["observed"], lib_t[0], lib_t[1], poses, w["noise"],
                                   w["sigma_max"], w["window"], base_depth=base_depth,
                                   camera=w["camera"])
    assert (st == 0).all()
    assert rel_err(s[pick], s_orc[:, 0]).max() <= SCORE_RTOL
    gpu_ctx.set_base_scene([], [])


def test_cfg3_full_size_contact_grid_spot_parity(gpu_ctx, oracle):
    """BASELINE configs[2] at full size (16 x 16 x 512 = 131,072 contact
    hypotheses over the base scene): the argmax and 31 random cells score
    within 1e-4 of the oracle, and the argmax lies at the true contact."""
    w = _cfg3(oracle, counts=(16, 16, 512))
    mids, base_inst = _setup_cfg3(gpu_ctx, oracle, w)
    gpu_ctx.set_observation(w["observed"])
    gpu_ctx.set_likelihood(w["noise"], w["sigma_max"], w["window"])
    o = w["objects"][w["target"]]
    g = b3d.ContactGrid.make(0.5, 0.5, o[2], o[3], 1, (16, 16, 512))
    s_gpu, st_gpu = gpu_ctx.score_contact_grid(mids[1 + w["target"]], g)
    assert s_gpu.shape[0] == 131072
    rng = np.random.Generator(np.random.PCG64(33))
    best = int(np.argmax(s_gpu[:, 0]))
    pick = np.concatenate([[best], rng.integers(0, s_gpu.shape[0], size=31)])
    poses = b3d.contact_grid_poses(g)[pick]
    base = oracle.render(w["k"], base_inst, camera=w["camera"])
    s_orc, st_orc = oracle.score_poses(w["k"], w["observed"], o[0], o[1], poses, w["noise"],
                                       w["sigma_max"], w["window"], base_depth=base,
                                       camera=w["camera"])
    assert (st_orc == st_gpu[pick]).all()
    ok = st_orc == 0
    assert rel_err(s_gpu[pick][ok, 0], s_orc[ok, 0]).max() <= SCORE_RTOL
    truth = w["poses"][w["target"]]
    assert np.linalg.norm(poses[0][4:6] - truth[4:6]) < 0.03  # within about one grid cell
    gpu_ctx.set_base_scene([], [])


def test_cfg2_full_size_chain_spot_parity_and_determinism(gpu_ctx, oracle):
    """BASELINE configs[1] at full size (5 stages x 32,768 hypotheses, 200x200,
    3,000 voxels): the device chain is deterministic (two runs bitwise
    equal), each stage's sample / argmax are the reference semantics over that
    stage's device scores, each next centre is the drawn grid pose, and the
    drawn pose plus 7 random ones per stage score within 1e-4 of the oracle."""
    from helpers import b3d_intr
    rf = lambda k, v, t, p: oracle.render(k, [(v, t, p)])
    w = configs.cfg2(rf, oracle.voxel_to_mesh, seed=0)
    assert w.stages[0]["count"] == (16, 16, 16) and len(w.stages) == 5
    gpu_ctx.set_camera(b3d_intr(w.k))
    mid = gpu_ctx.upload_mesh(w.vertices, w.triangles)
    gpu_ctx.set_observation(w.observed)
    gpu_ctx.set_likelihood([w.stages[0]["noise"]], w.sigma_max, 1)
    st = b3d.rng_seed(99)
    res, centers = gpu_ctx.coarse_to_fine(mid, w.center, w.stages, rng_state=st)
    st2 = b3d.rng_seed(99)
    res2, centers2 = gpu_ctx.coarse_to_fine(mid, w.center, w.stages, rng_state=st2)
    np.testing.assert_array_equal(np.array(centers), np.array(centers2))
    assert [r.sample for r in res] == [r.sample for r in res2]
    st_o = oracle.rng_seed(99)
    rng = np.random.Generator(np.random.PCG64(8))
    for s, g in enumerate(w.stages):
        gpu_ctx.set_likelihood([g["noise"]], w.sigma_max, g["window"])
        grid = gpu_ctx.make_grid(centers[s], g["extent"], g["count"], g["rotations"], 0)
        s_gpu, _ = gpu_ctx.score_grid(mid, grid)
        probs, _ = oracle.normalize(s_gpu[:, 0])
        pick = oracle.sample_categorical(probs, st_o)
        assert res[s].sample == pick and res[s].argmax == oracle.argmax(s_gpu[:, 0])
        poses = configs.grid_poses(centers[s], g["extent"], g["count"], g["rotations"], 0)
        np.testing.assert_array_equal(centers[s + 1], poses[pick])
        idx = np.concatenate([[pick], rng.integers(0, poses.shape[0], size=7)])
        s_orc, _ = oracle.score_poses(w.k, w.observed, w.vertices, w.triangles, poses[idx],
                                      [g["noise"]], w.sigma_max, g["window"])
        assert rel_err(s_gpu[idx, 0], s_orc[:, 0]).max() <= SCORE_RTOL
    np.testing.assert_array_equal(st, st_o)


def test_c_abi_is_thread_safe_like_the_reference():
    """The reference's C ABI is pure host code, callable from many threads at
    once (thread-local error, no shared state).  Here every thread gets its
    own device context: b3d_render and b3d_log_likelihood called from 8
    threads at once (ctypes releases the GIL) give exactly the serial results."""
    import json
    import threading
    vox = synth.eden_blob(400, 5)
    m0 = b3d.Model.from_voxels(vox, 0.005, np.zeros(3), 0)
    lib = b3d.Library.create([m0])
    k = configs.Intr(200.0, 200.0, 79.5, 59.5, 160, 120, 0.05, 5.0)
    intr = b3d_intr(k)
    cams = [np.array([0.0, 1.0, 0.0, 0.0, 0.02 * i, 0.01 * i, 0.8]) for i in range(8)]
    scenes = [b3d.Scene.from_json(json.dumps({"table": {"width": 0.5, "height": 0.4},
                                              "children": [dict(object_id=0, face=1 + i % 6,
                                                                dx=0.05 + 0.03 * i, dy=0.1,
                                                                dtheta=0.4 * i)]}), lib)
              for i in range(8)]
    serial = [b3d.render(scenes[i], cams[i], intr) for i in range(8)]
    serial_ll = [b3d.log_likelihood(serial[i], serial[(i + 1) % 8], intr, 0.1, 0.01, 0.1, 2)
                 for i in range(8)]
    got, got_ll, errs = [None] * 8, [None] * 8, []

    def work(i):
        try:
            for _ in range(5):
                got[i] = b3d.render(scenes[i], cams[i], intr)
                got_ll[i] = b3d.log_likelihood(got[i], serial[(i + 1) % 8], intr, 0.1, 0.01,
                                               0.1, 2)
        except Exception as e:  # pragma: no cover - reported below
            errs.append(repr(e))

    ts = [threading.Thread(target=work, args=(i,)) for i in range(8)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs
    for i in range(8):
        np.testing.assert_array_equal(got[i].view(np.uint32), serial[i].view(np.uint32))
        assert got_ll[i] == serial_ll[i]


@pytest.mark.parametrize("wh", [(1, 1), (3, 2), (2, 3), (1920, 1080)])
def test_extreme_image_sizes(gpu_ctx, oracle, wh):
    """1x1, 3x2, 2x3 and 1920x1080 images: depth / ids bitwise, scores within
    1e-4 of the oracle (= the reference, bitwise on every fixture)."""
    w_px, h_px = wh
    f = 0.9 * max(w_px, h_px)
    k = configs.Intr(f, f, (w_px - 1) / 2, (h_px - 1) / 2, w_px, h_px, 0.01, 10.0)
    vox = synth.eden_blob(500, 21)
    verts, tris = configs.make_mesh(vox, oracle.voxel_to_mesh)
    rng = np.random.Generator(np.random.PCG64(9))
    poses = np.array([[*synth.uniform_quaternion(rng), rng.uniform(-0.02, 0.02),
                       rng.uniform(-0.02, 0.02), rng.uniform(0.3, 0.6)] for _ in range(4)])
    _render_parity(gpu_ctx, oracle, k, verts, tris, poses)
    obs = np.array(oracle.render(k, [(verts, tris, poses[0])]), dtype=np.float32)
    if (obs < k.far).sum() == 0:
        return  # nothing visible at this size: the renders above are the check
    gpu_ctx.set_camera(b3d_intr(k))
    mid = gpu_ctx.upload_mesh(verts, tris)
    gpu_ctx.set_likelihood([(0.1, 0.01)], 0.1, 1)
    gpu_ctx.set_observation(obs)
    s, st = gpu_ctx.score_poses(mid, poses)
    for i in range(poses.shape[0]):
        d = oracle.render(k, [(verts, tris, poses[i])])
        if (d < k.far).sum() == 0:
            assert st[i] == 1
            continue
        want = oracle.windowed_loglik_multi(obs, d, k, [(0.1, 0.01)], 0.1, 1)[0]
        assert rel_err(s[i, 0], want) <= 1e-4, (wh, i, s[i, 0], want)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_adversarial_triangle_soup(gpu_ctx, oracle, seed):
    """Triangle soups built to hit the rasterizer's corner cases: vertices
    placed on pixel centres and half-pixels (edges through centres, the
    top-left tie rule), shared edges, zero-area and sliver triangles, equal
    depths (the draw-index tie), vertices behind / on / just in front of
    z = near (the clipped fan), and triangles far outside the image --
    depth and ids bitwise equal to the oracle."""
    rng = np.random.Generator(np.random.PCG64(100 + seed))
    k = configs.Intr(40.0, 40.0, 15.5, 11.5, 32, 24, 0.1, 5.0)
    pts = []
    for _ in range(300):
        u = rng.integers(-8, 40) + rng.choice([0.0, 0.5, 0.25])
        v = rng.integers(-8, 32) + rng.choice([0.0, 0.5])
        z = rng.choice([0.1, 0.1 * (1 - 1e-13), 0.09, 0.05, 0.5, 1.0, 1.0, 2.0, 4.99, 6.0])
        pts.append([(u - k.cx) * z / k.fx, (v - k.cy) * z / k.fy, z])
    pts = np.array(pts)
    tris = []
    for _ in range(400):
        a, b, c = rng.integers(0, len(pts), 3)
        tris.append([a, b, c])
        if rng.random() < 0.2:  # a neighbour sharing the edge (a, b)
            tris.append([b, a, rng.integers(0, len(pts))])
        if rng.random() < 0.05:
            tris.append([a, a, b])  # zero area
    tris = np.array(tris, dtype=np.uint32)
    poses = np.array([[1.0, 0, 0, 0, 0, 0, 0], [1.0, 0, 0, 0, 0.01, -0.02, 0.3]])
    _render_parity(gpu_ctx, oracle, k, pts, tris, poses)


def _crowded_scene(oracle, n_objects=23):
    """Table + n_objects blobs on a grid: more instances than one camera-mode
    launch holds (B3D_MAX_INSTANCES = 16)."""
    seq = _orbit(oracle, 64, n_frames=3)
    (tv, tt, tp) = seq["instances"][0]
    inst = [(tv, tt, tp)]
    for i in range(n_objects):
        vox = synth.eden_blob(60 + 7 * i, 500 + i)
        v, t = configs.make_mesh(vox, oracle.voxel_to_mesh)
        lo, hi = v.min(axis=0), v.max(axis=0)
        pose = oracle.contact_to_pose(0.5, 0.5, lo, hi, 1 + i % 6, 0.02 + 0.06 * (i % 6),
                                      0.02 + 0.07 * (i // 6), (0.3 * i) % 6.0)
        inst.append((v, t, pose))
    return dict(seq, instances=inst)


def test_camera_scene_beyond_one_launch(gpu_ctx, oracle):
    """24 instances (table + 23 objects): per-group renders merged per pixel
    -- depth and global draw indices bitwise equal to the oracle's
    render_instances -- and scores through the fp64 image likelihood within
    the tolerance; the same scene split below the limit gives the same renders."""
    seq = _crowded_scene(oracle)
    _camera_scene(gpu_ctx, seq)
    rng = np.random.Generator(np.random.PCG64(31))
    cams = [oracle.camera_pose_from_spherical(rng.uniform(0.4, 1.2), rng.uniform(0, 6.28),
                                              rng.uniform(0.3, 1.3)) for _ in range(6)]
    cams.append(oracle.camera_pose_from_spherical(0.1, 0.5, 0.3))  # near-plane clipping
    cams = np.array(cams)
    d, ids = gpu_ctx.render_cameras(cams)
    d_only = gpu_ctx.render_cameras(cams, with_ids=False)[0]
    for i, c in enumerate(cams):
        od, oi = oracle.render(seq["k"], seq["instances"], camera=c, with_ids=True)
        np.testing.assert_array_equal(d[i].view(np.uint32), od.view(np.uint32))
        np.testing.assert_array_equal(d_only[i].view(np.uint32), od.view(np.uint32))
        np.testing.assert_array_equal(ids[i], oi)
    n_table = seq["instances"][0][1].shape[0]
    assert (ids[:-1] > n_table + 16 * 40).any()  # pixels of the later groups' objects
    obs = d[0].copy()
    gpu_ctx.set_observation(obs)
    gpu_ctx.set_likelihood([seq["noise"]], seq["sigma_max"], seq["window"])
    s_gpu, st = gpu_ctx.score_cameras(cams)
    s_orc = np.array([oracle.windowed_loglik_multi(
        obs, oracle.render(seq["k"], seq["instances"], camera=c), seq["k"], [seq["noise"]],
        seq["sigma_max"], seq["window"])[0] for c in cams])
    assert (st == 0).all()
    assert rel_err(s_gpu[:, 0], s_orc).max() <= SCORE_RTOL


def test_track_camera_crowded_scene(gpu_ctx, oracle):
    """track_camera over the 24-instance scene (merged group renders, fp64
    image likelihood) picks the oracle's lattice points (a differing pick
    must tie within the score tolerance)."""
    seq = _crowded_scene(oracle)
    _camera_scene(gpu_ctx, seq)
    gpu_ctx.set_likelihood([seq["noise"]], seq["sigma_max"], seq["window"])
    cams = [oracle.camera_pose_from_spherical(seq["distance"], a, seq["altitude"])
            for a in seq["azimuths"][:3]]
    frames = np.stack([oracle.render(seq["k"], seq["instances"], camera=c) for c in cams])
    est, ms = gpu_ctx.track_camera(frames, cams[0])
    log = []
    ref = oracle.track_camera(frames, seq["k"], seq["instances"], cams[0], seq["noise"],
                              seq["sigma_max"], seq["window"], stage_log=log)
    assert len(cams) == 3
    for f in range(len(cams)):
        if not np.array_equal(est[f], ref[f]):
            _, _, grid, scores = [e for e in log if e[0] == f][-1]
            s = np.array(scores)
            assert np.sort(s)[-1] - np.sort(s)[-2] <= SCORE_RTOL * abs(np.max(s))
