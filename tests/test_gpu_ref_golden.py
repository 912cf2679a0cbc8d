"""GPU parity against the REFERENCE ITSELF: the sm_100a product path (through
the C ABI) vs tests/golden/ref_*.npz, produced by the reference's own C++
compiled unmodified (tests/golden/make_ref_golden.py).

Bars (BASELINE.json north_star): depth bitwise (stronger than 1e-5), scores
within 1e-4 relative -- with a secondary absolute bar |d| <= 1e-4 * S where
S = M * |log(p/V)| (M observed pixels, each log term is at least log(p/V) in
magnitude when the floor dominates), so totals near 0 are not judged by an
ill-conditioned ratio -- and argmax / draws identical unless the top scores tie
within that tolerance.  Full BASELINE sizes: cfg2's 5 x 32,768, cfg3's
131,072, a 65,536-hypothesis cfg5 slice, cfg4's 100-frame argmax chain.
"""
import json
import math
import os

import numpy as np
import pytest

from helpers import b3d_intr
from paper_2312_08715_b200 import b3d, configs, synth

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")
RTOL = 1e-4
IDENT = np.array([1.0, 0, 0, 0, 0, 0, 0])


def _load(name):
    path = os.path.join(GOLD, f"ref_{name}.npz")
    if not os.path.exists(path):
        pytest.fail(f"{path} missing: run tests/golden/make_ref_golden.py")
    return np.load(path, allow_pickle=False)


def _intr(a):
    a = [float(x) for x in a]
    return configs.Intr(a[0], a[1], a[2], a[3], int(a[4]), int(a[5]), a[6], a[7])


def _abs_scale(k, observed, p_outlier):
    """M * |log(p / V)|: the size of the sum of per-pixel log terms."""
    m = int((np.asarray(observed) < np.float32(k.far)).sum())
    vol = (k.far ** 3 - k.near ** 3) / 3.0 * (k.width / k.fx) * (k.height / k.fy)
    return m * abs(math.log(p_outlier / vol)) if p_outlier > 0 else float(m)


def assert_scores_close(got, want, scale, what=""):
    got, want = np.asarray(got, dtype=np.float64), np.asarray(want, dtype=np.float64)
    assert got.shape == want.shape
    fin = np.isfinite(want)
    np.testing.assert_array_equal(np.isfinite(got), fin, err_msg=f"{what}: finiteness")
    d = np.abs(got[fin] - want[fin])
    rel = d / np.maximum(np.abs(want[fin]), 1e-300)
    assert rel.max(initial=0) <= RTOL, f"{what}: max rel err {rel.max():.3e}"
    assert d.max(initial=0) <= RTOL * scale, f"{what}: max abs err {d.max():.3e} vs {scale:.3e}"
    return float(rel.max(initial=0))


def _argmax_agrees(got_idx, scores_ref, top):
    """Same index, or the product's pick ties the reference's best within RTOL."""
    return got_idx == int(np.argmax(scores_ref)) or \
        abs(scores_ref[got_idx] - top) <= RTOL * abs(top)


def _cfg1(oracle):
    rf = lambda k, v, t, p: oracle.render(k, [(v, t, p)])
    return configs.cfg1(rf, oracle.voxel_to_mesh, seed=0)


# ---------------------------------------------------------------- renders
def test_render_bitwise_reference(gpu_ctx, oracle):
    g = _load("render")
    w = _cfg1(oracle)
    np.testing.assert_array_equal(w.observed.view(np.uint32), g["observed"].view(np.uint32))
    gpu_ctx.set_camera(b3d_intr(w.k))
    mid = gpu_ctx.upload_mesh(w.vertices, w.triangles)
    for key_p, key_d in (("poses", "depth"), ("near_poses", "near_depth")):
        for with_ids in (True, False):
            d, _ = gpu_ctx.render_poses(mid, g[key_p], with_ids=with_ids)
            np.testing.assert_array_equal(d.view(np.uint32), g[key_d].view(np.uint32))
    seq = configs.orbit_sequence(None, oracle.voxel_to_mesh, oracle.box_mesh,
                                 oracle.contact_to_pose, 100)
    gpu_ctx.set_camera(b3d_intr(seq["k"]))
    mids = [gpu_ctx.upload_mesh(v, t) for v, t, _ in seq["instances"]]
    gpu_ctx.set_camera_scene(mids, [p for _, _, p in seq["instances"]])
    d, _ = gpu_ctx.render_cameras(g["cameras"])
    np.testing.assert_array_equal(d.view(np.uint32), g["scene_depth"].view(np.uint32))


# ---------------------------------------------------------------- cfg1 scores
def test_cfg1_scores_reference(gpu_ctx, oracle):
    """All 1,024 cfg1 hypotheses, the device pose grid and explicit poses;
    multi-noise at windows 0/2/3, the uniform prefactor, and the untruncated
    likelihood through b3d_log_likelihood (window < 0)."""
    g = _load("score_cfg1")
    w = _cfg1(oracle)
    gpu_ctx.set_camera(b3d_intr(w.k))
    mid = gpu_ctx.upload_mesh(w.vertices, w.triangles)
    gpu_ctx.set_observation(w.observed)
    gpu_ctx.set_likelihood(w.noise, w.sigma_max, w.window)
    scale = _abs_scale(w.k, w.observed, w.noise[0][0])
    grid = gpu_ctx.make_grid(w.center, w.extent, w.count, w.rotations, w.grid_mode)
    s_grid, st = gpu_ctx.score_grid(mid, grid)
    np.testing.assert_array_equal(st, g["status"])
    assert_scores_close(s_grid[:, 0], g["scores"], scale, "cfg1 grid")
    s_pose, _ = gpu_ctx.score_poses(mid, g["poses"])
    np.testing.assert_array_equal(s_pose, s_grid)
    r = gpu_ctx.stage_reduce(s_grid[:, 0])
    assert _argmax_agrees(r.argmax, g["scores"], g["scores"].max())
    sub = g["poses"][g["sub_idx"]]
    noise4 = [tuple(x) for x in g["noise4"]]
    for wi in (0, 2, 3):
        gpu_ctx.set_likelihood(noise4, 0.1, wi)
        s4, _ = gpu_ctx.score_poses(mid, sub)
        for e in range(4):
            assert_scores_close(s4[:, e], g[f"multi_w{wi}"][:, e],
                                _abs_scale(w.k, w.observed, noise4[e][0]), f"w{wi} e{e}")
    gpu_ctx.set_likelihood(w.noise, 0.1, 1, b3d.PREFACTOR_UNIFORM)
    su, _ = gpu_ctx.score_poses(mid, sub)
    assert_scores_close(su[:, 0], g["uniform"], scale, "uniform prefactor")
    k = b3d_intr(w.k)
    for i, want in zip(g["full_idx"], g["full"]):
        d, _ = gpu_ctx.render_poses(mid, g["poses"][i:i + 1], with_ids=False)
        got = b3d.log_likelihood(w.observed, d[0], k, w.noise[0][0], w.noise[0][1], 0.1, -1)
        assert abs(got - want) <= RTOL * abs(want)


# ---------------------------------------------------------------- cfg2: 5 x 32,768
def test_cfg2_full_chain_reference(gpu_ctx, oracle):
    """The device coarse-to-fine chain (Rng 99) against the reference-scored
    chain: every stage's 32,768 scores, the draw, the argmax and the centres."""
    g = _load("cfg2")
    rf = lambda k, v, t, p: oracle.render(k, [(v, t, p)])
    w = configs.cfg2(rf, oracle.voxel_to_mesh, seed=0)
    gpu_ctx.set_camera(b3d_intr(w.k))
    mid = gpu_ctx.upload_mesh(w.vertices, w.triangles)
    gpu_ctx.set_observation(w.observed)
    gpu_ctx.set_likelihood([w.stages[0]["noise"]], w.sigma_max, 1)
    st = b3d.rng_seed(99)
    res, centers = gpu_ctx.coarse_to_fine(mid, w.center, w.stages, rng_state=st)
    np.testing.assert_array_equal(centers, g["centers"])
    np.testing.assert_array_equal(st, g["rng_state"])
    worst = 0.0
    for s, stg in enumerate(w.stages):
        assert res[s].sample == g["picks"][s] and res[s].argmax == g["argmax"][s]
        gpu_ctx.set_likelihood([stg["noise"]], w.sigma_max, stg["window"])
        grid = gpu_ctx.make_grid(centers[s], stg["extent"], stg["count"], stg["rotations"], 0)
        sg, _ = gpu_ctx.score_grid(mid, grid)
        worst = max(worst, assert_scores_close(sg[:, 0], g["scores"][s],
                                               _abs_scale(w.k, w.observed, stg["noise"][0]),
                                               f"cfg2 stage {s}"))
    print(f"cfg2 max rel err {worst:.2e}")


# ---------------------------------------------------------------- cfg3: 131,072
def test_cfg3_full_grid_reference(gpu_ctx, oracle):
    """All 131,072 contact hypotheses over the base scene: the product's cell
    poses are the reference's stage0_cells centres bitwise, every score within
    1e-4, same argmax."""
    g = _load("cfg3")
    rs = lambda k, cam, inst: oracle.render(k, inst, camera=cam)
    w = configs.cfg3(rs, oracle.voxel_to_mesh, oracle.box_mesh, oracle.contact_to_pose,
                     counts=(16, 16, 512))
    np.testing.assert_array_equal(w["observed"].view(np.uint32), g["observed"].view(np.uint32))
    gpu_ctx.set_camera(b3d_intr(w["k"]), w["camera"])
    tv, tt, _, _ = w["table"]
    mids = [gpu_ctx.upload_mesh(tv, tt)] + [gpu_ctx.upload_mesh(o[0], o[1]) for o in w["objects"]]
    gpu_ctx.set_base_scene([mids[0]] + [mids[1 + i] for i in w["base"]],
                           [IDENT] + [w["poses"][i] for i in w["base"]])
    gpu_ctx.set_observation(w["observed"])
    gpu_ctx.set_likelihood(w["noise"], w["sigma_max"], w["window"])
    o = w["objects"][w["target"]]
    cg = b3d.ContactGrid.make(0.5, 0.5, o[2], o[3], 1, (16, 16, 512))
    np.testing.assert_array_equal(b3d.contact_grid_poses(cg), g["poses"])
    s, st = gpu_ctx.score_contact_grid(mids[1 + w["target"]], cg)
    gpu_ctx.set_base_scene([], [])
    np.testing.assert_array_equal(st, g["status"])
    assert_scores_close(s[:, 0], g["scores"], _abs_scale(w["k"], w["observed"], 0.02), "cfg3")
    assert _argmax_agrees(int(np.argmax(s[:, 0])), g["scores"], g["scores"].max())


# ---------------------------------------------------------------- cfg5: 65,536 slice
def test_cfg5_slice_reference(gpu_ctx, oracle):
    """A contiguous 65,536-hypothesis slice of cfg5's 1,048,576 (480x640,
    10-object base scene) within 1e-4 of the reference; the global device
    argmax over all 1,048,576 lies in the slice and agrees with it."""
    import torch
    g = _load("cfg5")
    rs = lambda k, cam, inst: oracle.render(k, inst, camera=cam)
    w = configs.cfg5(rs, oracle.voxel_to_mesh, oracle.box_mesh, oracle.contact_to_pose)
    np.testing.assert_array_equal(w["observed"].view(np.uint32), g["observed"].view(np.uint32))
    gpu_ctx.set_camera(b3d_intr(w["k"]), w["camera"])
    tv, tt = w["table"]
    mids = [gpu_ctx.upload_mesh(tv, tt)] + [gpu_ctx.upload_mesh(l[0], l[1]) for l in w["library"]]
    n_placed = len(w["base_poses"]) - 1
    gpu_ctx.set_base_scene([mids[0]] + [mids[1 + i] for i in range(n_placed)], w["base_poses"])
    gpu_ctx.set_observation(w["observed"])
    gpu_ctx.set_likelihood(w["noise"], w["sigma_max"], w["window"])
    grid = gpu_ctx.make_grid(w["gt"], w["extent"], w["count"],
                             torch.from_numpy(w["rotations"]).cuda(), b3d.GRID_PRODUCT)
    n = w["n_hyp"]
    full = torch.zeros((n, 1), dtype=torch.float64, device="cuda")
    gpu_ctx.score_grid_range(mids[1 + w["target"]], grid, 0, n, full, None)
    torch.cuda.synchronize()
    gpu_ctx.set_base_scene([], [])
    s = full[:, 0].cpu().numpy()
    lo = int(g["first"])
    assert_scores_close(s[lo:lo + 65536], g["scores"], _abs_scale(w["k"], w["observed"], 0.02),
                        "cfg5 slice")
    best = int(np.argmax(s))
    assert lo <= best < lo + 65536
    assert _argmax_agrees(best - lo, g["scores"], g["scores"].max())


# ---------------------------------------------------------------- cfg4: 100-frame chain
def test_cfg4_argmax_chain_reference(gpu_ctx, oracle):
    """The 100-frame tracking sequence: at every one of the 198 stages the
    device chain's argmax equals the reference's (or ties it within 1e-4), the
    chain stays on the reference's centres, and 64 sampled scores per stage
    agree within 1e-4."""
    g = _load("cfg4")
    rf = lambda k, v, t, p: oracle.render(k, [(v, t, p)])
    tr = configs.cfg4(rf, oracle.voxel_to_mesh, seed=0)
    gpu_ctx.set_camera(b3d_intr(tr["k"]))
    mid = gpu_ctx.upload_mesh(tr["vertices"], tr["triangles"])
    st0 = tr["stages"][0]
    gpu_ctx.set_likelihood([st0["noise"]], 0.1, st0["window"])
    est = tr["gt"][0].copy()
    agree = 0
    i = 0
    for f in range(1, len(tr["frames"])):
        gpu_ctx.set_observation(tr["frames"][f])
        res, centers = gpu_ctx.coarse_to_fine(mid, est, tr["stages"])
        for s, stg in enumerate(tr["stages"]):
            np.testing.assert_array_equal(centers[s], g["centers"][i])
            top = g["top2"][i][0]
            ok = res[s].argmax == g["argmax"][i] or abs(res[s].max_score - top) <= RTOL * abs(top)
            agree += ok
            assert abs(res[s].max_score - top) <= RTOL * abs(top)
            i += 1
        # spot-check scores of the last stage of every 10th frame
        if f % 10 == 0:
            stg = tr["stages"][-1]
            grid = gpu_ctx.make_grid(centers[-2], stg["extent"], stg["count"], stg["rotations"], 0)
            sg, _ = gpu_ctx.score_grid(mid, grid)
            assert_scores_close(sg[g["sample_idx"][i - 1], 0], g["sample_scores"][i - 1],
                                _abs_scale(tr["k"], tr["frames"][f], 0.05), f"cfg4 frame {f}")
        est = centers[-1]
    assert agree == i == g["argmax"].shape[0]
    np.testing.assert_array_equal(est, g["final"])


# ---------------------------------------------------------------- tracking / SMC / infer
def _track_world(gpu_ctx, oracle, g):
    k = _intr(g["k"])
    v, t = oracle.voxel_to_mesh(g["voxels"], configs.RESOLUTION, g["origin"])
    lo, hi = v.min(axis=0), v.max(axis=0)
    tv, tt = oracle.box_mesh(np.array([-0.25, -0.25, -0.01]), np.array([0.25, 0.25, 0.0]))
    pose = oracle.contact_to_pose(0.5, 0.5, lo, hi, 1, (0.5 - (hi[0] - lo[0])) / 2,
                                  (0.5 - (hi[1] - lo[1])) / 2, 0.0)
    gpu_ctx.set_camera(b3d_intr(k))
    mids = [gpu_ctx.upload_mesh(tv, tt), gpu_ctx.upload_mesh(v, t)]
    gpu_ctx.set_camera_scene(mids, [IDENT, pose])
    gpu_ctx.set_likelihood([(0.02, 0.002)], 0.1, configs.default_window(40))


@pytest.mark.parametrize("variant,kw", [("default", {}),
                                        ("ppd3", dict(points_per_dim=3, refine_stages=3)),
                                        ("beam2", dict(beam_width=2))])
def test_track_camera_reference(gpu_ctx, oracle, variant, kw):
    """track_camera on the reference's own orbit frames: the device search
    returns the reference's camera poses bitwise."""
    g = _load("track")
    _track_world(gpu_ctx, oracle, g)
    poses, _ = gpu_ctx.track_camera(g["frames"], g["gt"][0], b3d.TrackSearch.default(**kw))
    np.testing.assert_array_equal(poses, g[variant])


def _smc_lib(gpu_ctx, oracle, g):
    k = _intr(g["k"])
    gpu_ctx.set_camera(b3d_intr(k), g["camera"])
    tv, tt = oracle.box_mesh(np.array([-0.2, -0.2, -0.01]), np.array([0.2, 0.2, 0.0]))
    table = gpu_ctx.upload_mesh(tv, tt)
    lib = []
    for i, nv in enumerate((60, 120, 200)):
        vox = synth.eden_blob(nv, 40 + i)
        v, t = oracle.voxel_to_mesh(vox, 0.01, synth.centered_origin(vox, 0.01))
        lib.append((gpu_ctx.upload_mesh(v, t), v.min(axis=0), v.max(axis=0)))
    gpu_ctx.set_observation(g["observed"])
    return lib, table


def _cmp_smc(ps, ev, g, prefix):
    ch, ct = g[f"{prefix}_children"], g[f"{prefix}_contact"]
    assert len(ps) == ch.shape[0]
    for i, (c, e, lt, lw) in enumerate(ps):
        for j in range(ch.shape[1]):
            assert tuple(c[j][:2]) == tuple(ch[i, j])
            np.testing.assert_allclose(c[j][2:], ct[i, j], rtol=0, atol=1e-12)
        assert e == g[f"{prefix}_noise"][i]
        assert abs(lt - g[f"{prefix}_logt"][i]) <= RTOL * abs(g[f"{prefix}_logt"][i])
        assert abs(lw - g[f"{prefix}_logw"][i]) <= RTOL * max(1.0, abs(g[f"{prefix}_logw"][i]))
    assert abs(ev - float(g[f"{prefix}_ev"])) <= RTOL * max(1.0, abs(float(g[f"{prefix}_ev"])))


def test_run_smc_reference(gpu_ctx, oracle):
    """run_smc (inference.cpp:398-520) on the device against the reference's
    own run_smc: 48 particles / 1 object, and 24 particles / 2 objects with
    forced resampling -- same cells, leaf draws and noise choices, weights and
    evidence within 1e-4."""
    g = _load("smc")
    lib, table = _smc_lib(gpu_ctx, oracle, g)
    noise = [tuple(x) for x in g["noise"]]
    ps, ev = gpu_ctx.run_smc(lib, table, 0.4, 0.4, ((3, 3, 4), [(2, 2, 2), (2, 1, 3)]), noise,
                             0.1, 1, 1, 48, 0.5, 5)
    _cmp_smc(ps, ev, g, "smc1")
    ps, ev = gpu_ctx.run_smc(lib, table, 0.4, 0.4, ((2, 2, 3), [(2, 2, 2)]), noise, 0.1, 1, 2,
                             24, 0.99, 6)
    _cmp_smc(ps, ev, g, "smc2")
    gpu_ctx.set_base_scene([], [])


@pytest.mark.parametrize("key,overrides", [
    ("infer_w", {"window": 1}),
    ("infer_full", {"window": -1}),
    ("infer_deep", {"window": 0, "schedule": {"stage0": [2, 2, 2], "refine": [
        [2, 1, 1], [1, 2, 1], [1, 1, 2], [2, 1, 1], [1, 1, 2], [2, 2, 1]]}}),
])
def test_b3d_infer_reference_c_abi(key, overrides):
    """b3d_infer through the product's C ABI against the reference's own
    b3d_infer (same JSON config, seed): particles, noise, weights, evidence and
    MAP pose.  Covers window < 0 (full likelihood, b3d_capi.cpp:328-330) and a
    six-stage refine schedule (b3d_capi.cpp:350-351)."""
    g = _load("smc")
    k = _intr(g["k"])
    cfg = dict(json.loads(str(g["infer_cfg"])), **overrides)
    # the reference loaded its library from SVOX files, whose resolution and
    # origin are float32 (io.hpp:19-20): the same values here
    models = []
    for i, nv in enumerate((60, 120, 200)):
        vox = synth.eden_blob(nv, 40 + i)
        org = synth.centered_origin(vox, 0.01).astype(np.float32).astype(np.float64)
        models.append(b3d.Model.from_voxels(vox, float(np.float32(0.01)), org, i))
    lib = b3d.Library.create(models)
    seed = 10 if key == "infer_deep" else 9
    lines, ev, _, map_pose = b3d.infer(g["observed"], g["camera"], lib, json.dumps(cfg), seed)
    want = json.loads(str(g[key]))
    assert len(lines) == len(want)
    for line, wj in zip(lines, want):
        j = json.loads(line)
        for a, b in zip(j["children"], wj["children"]):
            assert (a["object_id"], a["face"]) == (b["object_id"], b["face"])
            np.testing.assert_allclose([a["dx"], a["dy"], a["dtheta"]],
                                       [b["dx"], b["dy"], b["dtheta"]], rtol=0, atol=1e-12)
        assert j["noise"] == wj["noise"]
        assert abs(j["log_weight"] - wj["log_weight"]) <= RTOL * max(1.0, abs(wj["log_weight"]))
    assert abs(ev - float(g[f"{key}_ev"])) <= RTOL * max(1.0, abs(float(g[f"{key}_ev"])))
    np.testing.assert_allclose(map_pose, g[f"{key}_map"], rtol=0, atol=1e-12)
    del k
