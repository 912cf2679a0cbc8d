"""Parity anchored on the REFERENCE ITSELF (CPU, no GPU needed).

tests/golden/ref_*.npz were produced by the reference's own C++ sources
compiled unmodified into oracle/_ref/libb3d_ref.so
(tests/golden/make_ref_golden.py).  These tests pin

  * the C restatement (oracle/), which every GPU parity test uses as checker,
  * the product's host-side C++ (pose helpers, voxel_to_mesh, sample_observation),

to that output: pose math, meshes, renders, scores, score_cells probabilities,
proposals, run_smc, track_camera and the observation sampler are BITWISE the
reference's.  When oracle/_ref/libb3d_ref.so is present (the build container)
they also cross-check the oracle against the reference on fresh random cases.
"""
import json
import os

import numpy as np
import pytest

from paper_2312_08715_b200 import b3d, configs, synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")
IDENT = np.array([1.0, 0, 0, 0, 0, 0, 0])


def _load(name):
    path = os.path.join(GOLD, f"ref_{name}.npz")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated yet")
    return np.load(path, allow_pickle=False)


def _intr(a):
    a = [float(x) for x in a]
    return configs.Intr(a[0], a[1], a[2], a[3], int(a[4]), int(a[5]), a[6], a[7])


def _bits(a):
    a = np.ascontiguousarray(a)
    return a.view(np.uint64 if a.dtype == np.float64 else np.uint32)


def _eq(a, b, msg=""):
    np.testing.assert_array_equal(_bits(np.asarray(a)), _bits(np.asarray(b)), err_msg=msg)


# ---------------------------------------------------------------- pose math / meshes
def test_pose_math_bitwise_reference(oracle):
    g = _load("pose")
    for i in range(g["a"].shape[0]):
        _eq(oracle.compose(g["a"][i], g["b"][i]), g["compose"][i])
        _eq(oracle.inverse(g["a"][i]), g["inverse"][i])
        _eq(np.asarray(oracle.rotation_matrix(g["a"][i])).reshape(3, 3), g["rotation"][i])
    for s, c in zip(g["spherical"], g["camera"]):
        _eq(oracle.camera_pose_from_spherical(*s), c)
        _eq(b3d.camera_pose_from_spherical(*s), c)  # product host path


def test_contact_to_pose_bitwise_reference(oracle):
    g = _load("pose")
    v, _ = oracle.voxel_to_mesh(g["contact_voxels"], 0.005, g["contact_origin"])
    lo, hi = v.min(axis=0), v.max(axis=0)
    for c, want in zip(g["contact_in"], g["contact"]):
        args = (0.5, 0.5, lo, hi, int(c[0]), c[1], c[2], c[3])
        _eq(oracle.contact_to_pose(*args), want)
        _eq(b3d.contact_to_pose(*args), want)


def test_voxel_to_mesh_bitwise_reference(oracle):
    g = _load("mesh")
    for i in (1, 2):
        res = 0.005 if i == 1 else 0.01
        for fn in (oracle.voxel_to_mesh, b3d.voxel_to_mesh):
            v, t = fn(g[f"vox{i}"], res, g[f"origin{i}"])
            _eq(v, g[f"verts{i}"])
            np.testing.assert_array_equal(t, g[f"tris{i}"])


# ---------------------------------------------------------------- renderer / likelihood
def _cfg1_oracle():
    from oracle import pyoracle as O
    return configs.cfg1(lambda k, v, t, p: O.render(k, [(v, t, p)]), O.voxel_to_mesh, seed=0)


def test_render_bitwise_reference(oracle):
    g = _load("render")
    w = _cfg1_oracle()
    _eq(oracle.render(w.k, [(w.vertices, w.triangles, w.gt_pose)]), g["gt_depth"])
    _eq(w.observed, g["observed"])
    for p, d in zip(g["poses"], g["depth"]):
        _eq(oracle.render(w.k, [(w.vertices, w.triangles, p)]), d)
    for p, d in zip(g["near_poses"], g["near_depth"]):
        _eq(oracle.render(w.k, [(w.vertices, w.triangles, p)]), d)
    seq = configs.orbit_sequence(None, oracle.voxel_to_mesh, oracle.box_mesh,
                                 oracle.contact_to_pose, 100)
    for c, d in zip(g["cameras"], g["scene_depth"]):
        _eq(oracle.render(seq["k"], seq["instances"], camera=c), d)


def test_scores_bitwise_reference(oracle):
    g = _load("score_cfg1")
    w = _cfg1_oracle()
    s, st = oracle.score_poses(w.k, w.observed, w.vertices, w.triangles, g["poses"], w.noise,
                               w.sigma_max, w.window)
    np.testing.assert_array_equal(st, g["status"])
    _eq(s[:, 0], g["scores"])
    sub = g["poses"][g["sub_idx"]]
    noise4 = [tuple(x) for x in g["noise4"]]
    for wi in (0, 2, 3):
        s4, _ = oracle.score_poses(w.k, w.observed, w.vertices, w.triangles, sub, noise4, 0.1, wi)
        _eq(s4, g[f"multi_w{wi}"])
    su, _ = oracle.score_poses(w.k, w.observed, w.vertices, w.triangles, sub, w.noise, 0.1, 1,
                               prefactor=1)
    _eq(su[:, 0], g["uniform"])
    for i, want in zip(g["full_idx"], g["full"]):
        rend = oracle.render(w.k, [(w.vertices, w.triangles, g["poses"][i])])
        _eq(oracle.full_loglik(w.observed, rend, w.k, w.noise[0], 0.1), want)


# ---------------------------------------------------------------- sampler / tracking
def _track_inputs(oracle, g):
    k = _intr(g["k"])
    v, t = oracle.voxel_to_mesh(g["voxels"], configs.RESOLUTION, g["origin"])
    lo, hi = v.min(axis=0), v.max(axis=0)
    tv, tt = oracle.box_mesh(np.array([-0.25, -0.25, -0.01]), np.array([0.25, 0.25, 0.0]))
    pose = oracle.contact_to_pose(0.5, 0.5, lo, hi, 1, (0.5 - (hi[0] - lo[0])) / 2,
                                  (0.5 - (hi[1] - lo[1])) / 2, 0.0)
    return k, [(tv, tt, IDENT), (v, t, pose)]


def test_orbit_frames_and_sampler_bitwise_reference(oracle):
    """generate_orbit_sequence (tracking.cpp:174-206) = render + sample_observation
    with rng.split(0x0f, i): the oracle and the product's host sampler."""
    g = _load("track")
    k, inst = _track_inputs(oracle, g)
    root = oracle.rng_seed(21)
    for i in range(g["frames"].shape[0]):
        rend = oracle.render(k, inst, camera=g["gt"][i])
        _eq(oracle.camera_pose_from_spherical(0.9, 0.5 * i / g["frames"].shape[0],
                                              0.6981317007977318), g["gt"][i])
        st = oracle.rng_split(root, 0x0F, i)
        _eq(oracle.sample_observation(rend, k, 0.02, 0.002, st.copy()), g["frames"][i])
        _eq(b3d.sample_observation(b3d.Intrinsics(*k.as_tuple()), rend, 0.02, 0.002, st.copy()),
            g["frames"][i])
    v, t = oracle.voxel_to_mesh(g["voxels"], configs.RESOLUTION, g["origin"])
    rend = oracle.render(k, [(v, t, IDENT)], camera=np.array([0, 1.0, 0, 0, 0, 0, 0.3]))
    st = oracle.rng_split(oracle.rng_seed(8), 1, 2, 3)
    _eq(oracle.sample_observation(rend, k, 0.3, 0.004, st), g["sampled"])


@pytest.mark.parametrize("variant,kw", [("default", {}),
                                        ("ppd3", dict(points_per_dim=3, refine_stages=3)),
                                        ("beam2", dict(beam_width=2))])
def test_track_camera_bitwise_reference(oracle, variant, kw):
    g = _load("track")
    k, inst = _track_inputs(oracle, g)
    poses = oracle.track_camera(list(g["frames"]), k, inst, g["gt"][0], (0.02, 0.002), 0.1,
                                configs.default_window(40), **kw)
    _eq(poses, g[variant])


# ---------------------------------------------------------------- scene-graph inference
def _smc_world(oracle, g):
    k = _intr(g["k"])
    lib = []
    for i, nv in enumerate((60, 120, 200)):
        vox = synth.eden_blob(nv, 40 + i)
        v, t = oracle.voxel_to_mesh(vox, 0.01, synth.centered_origin(vox, 0.01))
        lib.append((v, t, v.min(axis=0), v.max(axis=0)))
    tv, tt = oracle.box_mesh(np.array([-0.2, -0.2, -0.01]), np.array([0.2, 0.2, 0.0]))
    return k, lib, (tv, tt, 0.4, 0.4)


def _cmp_particles(ps, ev, g, prefix):
    children = g[f"{prefix}_children"]
    contact = g[f"{prefix}_contact"]
    assert len(ps) == children.shape[0]
    for i, (ch, e, lt, lw) in enumerate(ps):
        for c in range(children.shape[1]):
            assert (ch[c][0], ch[c][1]) == tuple(children[i, c]), (i, c)
            _eq(np.array(ch[c][2:]), contact[i, c])
        assert e == g[f"{prefix}_noise"][i]
        _eq(lt, g[f"{prefix}_logt"][i])
        _eq(lw, g[f"{prefix}_logw"][i])
    _eq(ev, g[f"{prefix}_ev"])


def test_run_smc_bitwise_reference(oracle):
    """run_smc (inference.cpp:398-520): particles, noise indices, log targets,
    log weights and evidence, 1 object and 2 objects with forced resampling."""
    g = _load("smc")
    k, lib, table = _smc_world(oracle, g)
    noise = [tuple(x) for x in g["noise"]]
    ps, ev = oracle.run_smc(k, g["camera"], g["observed"], lib, table,
                            ((3, 3, 4), [(2, 2, 2), (2, 1, 3)]), noise, 0.1, 1, 1, 48, 0.5, 5)
    _cmp_particles(ps, ev, g, "smc1")
    ps, ev = oracle.run_smc(k, g["camera"], g["observed"], lib, table, ((2, 2, 3), [(2, 2, 2)]),
                            noise, 0.1, 1, 2, 24, 0.99, 6)
    _cmp_particles(ps, ev, g, "smc2")


def test_infer_fixture_is_self_consistent():
    """The b3d_infer fixtures (reference C ABI): windowed, window < 0 (full
    likelihood) and a 6-stage refine schedule all produced particles."""
    g = _load("smc")
    for key in ("infer_w", "infer_full", "infer_deep"):
        parts = json.loads(str(g[key]))
        assert len(parts) == 16 and all(np.isfinite(p["log_weight"]) for p in parts)
        assert np.isfinite(float(g[f"{key}_ev"]))


# ---------------------------------------------------------------- BASELINE full-size sets
def test_cfg2_stage_scores_reference_spot(oracle):
    """cfg2 (5 x 32,768 reference scores): the oracle reproduces 64 random
    hypotheses per stage bitwise, and the chain's picks follow the reference's
    normalisation + sample_categorical from Rng(99)."""
    g = _load("cfg2")
    from oracle import pyoracle as O
    w = configs.cfg2(lambda k, v, t, p: O.render(k, [(v, t, p)]), O.voxel_to_mesh, seed=0)
    _eq(w.observed, g["observed"])
    st = oracle.rng_seed(99)
    rng = np.random.Generator(np.random.PCG64(2))
    for s, stg in enumerate(w.stages):
        poses = configs.grid_poses(g["centers"][s], stg["extent"], stg["count"],
                                   stg["rotations"], 0)
        probs, _ = oracle.normalize(g["scores"][s])
        assert oracle.sample_categorical(probs, st) == g["picks"][s]
        _eq(poses[g["picks"][s]], g["centers"][s + 1])
        idx = rng.integers(0, poses.shape[0], 64)
        so, _ = oracle.score_poses(w.k, w.observed, w.vertices, w.triangles, poses[idx],
                                   [stg["noise"]], w.sigma_max, stg["window"])
        _eq(so[:, 0], g["scores"][s][idx])
    _eq(st, g["rng_state"])


# ---------------------------------------------------------------- live cross-check (build box)
needs_ref = pytest.mark.skipif(
    not os.path.exists(os.path.join(os.path.dirname(os.path.dirname(__file__)), "oracle", "_ref",
                                    "libb3d_ref.so")),
    reason="oracle/_ref/libb3d_ref.so not built (needs /root/reference)")


@needs_ref
def test_oracle_equals_reference_random_cases(oracle):
    """Fresh random cases, oracle vs the reference library, bitwise: poses
    straddling the near plane, random meshes, windows 0..4 and the
    untruncated likelihood (window < 0), multi-noise."""
    from oracle import pyref as R
    rng = np.random.Generator(np.random.PCG64(2024))
    k = configs.Intr(120.0, 110.0, 40.5, 30.25, 80, 60, 0.05, 3.0)
    for trial in range(7):
        vox = synth.random_walk_blob(int(rng.integers(20, 200)), int(rng.integers(0, 1000)))
        org = synth.centered_origin(vox, 0.01)
        v, t = oracle.voxel_to_mesh(vox, 0.01, org)
        poses = []
        for _ in range(12):
            q = rng.standard_normal(4)
            q /= np.linalg.norm(q)
            poses.append(np.concatenate([q, rng.uniform(-0.1, 0.1, 2), rng.uniform(0.0, 0.6, 1)]))
        poses = np.array(poses)
        obs = R.render(k, [(v, t, poses[0])])
        obs = synth.noisy_observation(obs, k.far, 0.004, 0.2, 0.1, 2.0, rng, k.near)
        for p in poses:
            _eq(oracle.render(k, [(v, t, p)]), R.render(k, [(v, t, p)]))
        noise = [(0.01, 0.01), (0.3, 0.01), (0.1, 0.04)]
        wi = trial % 5 if trial < 6 else -1
        so, sto = oracle.score_poses(k, obs, v, t, poses, noise, 0.1, wi)
        sr, str_ = R.score_poses(k, obs, v, t, poses, noise, 0.1, wi)
        np.testing.assert_array_equal(sto, str_)
        _eq(so, sr)


def test_cfg3_cfg4_cfg5_reference_spot(oracle):
    """The full-size fixtures (cfg3's 131,072 contact cells, cfg4's 100-frame
    chain, cfg5's 65,536-hypothesis slice): the oracle reproduces sampled
    entries bitwise, so the GPU tests against these files and against the
    oracle judge the same numbers."""
    from oracle import pyoracle as O
    rng = np.random.Generator(np.random.PCG64(9))
    ident = np.array([1.0, 0, 0, 0, 0, 0, 0])
    rs = lambda k, cam, inst: O.render(k, inst, camera=cam)
    # cfg3
    g = _load("cfg3")
    w = configs.cfg3(rs, O.voxel_to_mesh, O.box_mesh, O.contact_to_pose, counts=(16, 16, 512))
    _eq(w["observed"], g["observed"])
    tv, tt, _, _ = w["table"]
    base = [(tv, tt, ident)] + [(w["objects"][i][0], w["objects"][i][1], w["poses"][i])
                               for i in w["base"]]
    o = w["objects"][w["target"]]
    cg = b3d.ContactGrid.make(0.5, 0.5, o[2], o[3], 1, (16, 16, 512))
    _eq(b3d.contact_grid_poses(cg), g["poses"])  # product host cells = reference stage0_cells
    idx = np.concatenate([[int(np.argmax(g["scores"]))], rng.integers(0, 131072, 11)])
    bd = O.render(w["k"], base, camera=w["camera"])
    s, _ = O.score_poses(w["k"], w["observed"], o[0], o[1], g["poses"][idx], w["noise"],
                         w["sigma_max"], w["window"], base_depth=bd, camera=w["camera"])
    _eq(s[:, 0], g["scores"][idx])
    # cfg4: frame 1, both stages' sampled scores
    g = _load("cfg4")
    # (all 100 frames: the stage rotation tables are drawn after the frames)
    tr = configs.cfg4(lambda k, v, t, p: O.render(k, [(v, t, p)]), O.voxel_to_mesh, seed=0)
    for st in range(2):
        stg = tr["stages"][st]
        poses = configs.grid_poses(g["centers"][st], stg["extent"], stg["count"],
                                   stg["rotations"], 0)
        ii = g["sample_idx"][st][:16]
        s, _ = O.score_poses(tr["k"], tr["frames"][1], tr["vertices"], tr["triangles"], poses[ii],
                             [stg["noise"]], 0.1, stg["window"])
        _eq(s[:, 0], g["sample_scores"][st][:16])
    # cfg5: a few slice entries incl. the slice argmax
    g = _load("cfg5")
    w = configs.cfg5(rs, O.voxel_to_mesh, O.box_mesh, O.contact_to_pose)
    _eq(w["observed"], g["observed"])
    lo = int(g["first"])
    idx = np.concatenate([[int(np.argmax(g["scores"]))], rng.integers(0, 65536, 3)])
    allp = configs.grid_poses(w["gt"], w["extent"], w["count"], w["rotations"], 0)
    tv, tt = w["table"]
    n_placed = len(w["base_poses"]) - 1
    base = [(tv, tt, w["base_poses"][0])] + [
        (w["library"][i][0], w["library"][i][1], w["base_poses"][1 + i]) for i in range(n_placed)]
    bd = O.render(w["k"], base, camera=w["camera"])
    lt = w["library"][w["target"]]
    s, _ = O.score_poses(w["k"], w["observed"], lt[0], lt[1], allp[lo + idx], w["noise"],
                         w["sigma_max"], w["window"], base_depth=bd, camera=w["camera"])
    _eq(s[:, 0], g["scores"][idx])
