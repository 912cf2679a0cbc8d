#!/usr/bin/env python
"""Golden fixtures produced by the REFERENCE'S OWN implementation.

Run in the build container (needs /root/reference):

    make -C oracle ref            # oracle/_ref/libb3d_ref.so: the reference library
    python tests/golden/make_ref_golden.py [section ...]

oracle/_ref/libb3d_ref.so is every /root/reference/proj/src/core/*.cpp plus
src/capi/b3d_capi.cpp compiled unmodified (oracle/Makefile `ref`, Eigen-subset
shim in oracle/ref_shim/).  Each section writes tests/golden/ref_<section>.npz;
the CPU tests pin the C restatement (oracle/) to these files and the GPU tests
pin the product to them, so parity is anchored on the reference's own output,
not only on the restatement.  Inputs are the BASELINE workloads
(paper_2312_08715_b200/configs.py) with every render done by the reference.

Where the reference has no function for a step (the BASELINE 6-DoF grids'
stage chaining), the chain uses the oracle's restatement of score_cells'
normalisation and sample_categorical (inference.cpp:315-353, pinned by
tests/test_oracle_stage.py) on reference-computed scores, and says so.
"""
from __future__ import annotations

import math
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import pyoracle as O  # noqa: E402
from oracle import pyref as R  # noqa: E402
from paper_2312_08715_b200 import configs, synth  # noqa: E402

IDENT = np.array([1.0, 0, 0, 0, 0, 0, 0])


def _save(name, **arrays):
    path = os.path.join(HERE, f"ref_{name}.npz")
    np.savez_compressed(path, **arrays)
    print(f"  wrote {os.path.relpath(path, ROOT)} ({os.path.getsize(path) / 1e3:.0f} kB)")


def _rf(k, v, t, p):
    return R.render(k, [(v, t, p)])


def _rs(k, cam, inst):
    return R.render(k, inst, camera=cam)


def _unit_q(rng):
    q = rng.standard_normal(4)
    return q / np.linalg.norm(q)


def sec_pose():
    """geometry.cpp:11-31, generative.cpp:35-59, scene_graph.cpp:60-121."""
    rng = np.random.Generator(np.random.PCG64(101))
    n = 256
    a = np.concatenate([np.array([_unit_q(rng) for _ in range(n)]), rng.normal(size=(n, 3))], 1)
    b = np.concatenate([np.array([_unit_q(rng) for _ in range(n)]), rng.normal(size=(n, 3))], 1)
    comp = np.array([R.compose(a[i], b[i]) for i in range(n)])
    inv = np.array([R.inverse(a[i]) for i in range(n)])
    rot = np.array([R.rotation_matrix(a[i]) for i in range(n)])
    sph = np.stack([rng.uniform(0.3, 2.0, 128), rng.uniform(-7, 7, 128),
                    rng.uniform(0.02, 1.55, 128)], 1)
    cam = np.array([R.camera_pose_from_spherical(*s) for s in sph])
    vox = synth.eden_blob(300, 11)
    org = synth.centered_origin(vox, 0.005)
    cin = np.stack([rng.integers(1, 7, 96).astype(np.float64), rng.uniform(0, 0.4, 96),
                    rng.uniform(0, 0.4, 96), rng.uniform(0, 2 * np.pi, 96)], 1)
    contact = np.array([R.contact_to_pose(0.5, 0.5, vox, 0.005, org, int(c[0]), c[1], c[2], c[3])
                        for c in cin])
    _save("pose", a=a, b=b, compose=comp, inverse=inv, rotation=rot, spherical=sph, camera=cam,
          contact_voxels=vox, contact_origin=org, contact_in=cin, contact=contact)


def sec_mesh():
    """geometry.cpp:142-177: vertex numbering and triangle order (= ids)."""
    v1 = synth.eden_blob(1000, 0)
    o1 = synth.centered_origin(v1, 0.005)
    m1v, m1t = R.voxel_to_mesh(v1, 0.005, o1)
    v2 = synth.random_walk_blob(400, 7) - 3  # negative coordinates
    o2 = np.array([-0.013, 0.02, 0.5])
    m2v, m2t = R.voxel_to_mesh(v2, 0.01, o2)
    _save("mesh", vox1=v1, origin1=o1, verts1=m1v, tris1=m1t, vox2=v2, origin2=o2, verts2=m2v,
          tris2=m2t)


def sec_render():
    """renderer.cpp:61-189: cfg1 poses, near-plane clipping, a camera-mode scene."""
    w = configs.cfg1(_rf, R.voxel_to_mesh, seed=0)
    poses = w.grid_poses()[::32]
    depth = np.array([_rf(w.k, w.vertices, w.triangles, p) for p in poses])
    rng = np.random.Generator(np.random.PCG64(5))
    near = []
    for _ in range(8):  # object straddling z = near (0.01 m)
        q = _unit_q(rng)
        near.append(np.concatenate([q, [rng.uniform(-0.01, 0.01), rng.uniform(-0.01, 0.01),
                                        rng.uniform(0.0, 0.02)]]))
    near = np.array(near)
    near_depth = np.array([_rf(w.k, w.vertices, w.triangles, p) for p in near])
    # bench-tracking style scene: table + blob at 100 px, orbit cameras
    seq = configs.orbit_sequence(None, O.voxel_to_mesh, O.box_mesh, O.contact_to_pose, 100)
    cams = np.array([R.camera_pose_from_spherical(0.9, az, seq["altitude"])
                     for az in np.linspace(0, 2 * np.pi, 6, endpoint=False)])
    scene_depth = np.array([_rs(seq["k"], c, seq["instances"]) for c in cams])
    _save("render", poses=poses, depth=depth, gt_depth=_rf(w.k, w.vertices, w.triangles, w.gt_pose),
          observed=w.observed, near_poses=near, near_depth=near_depth, cameras=cams,
          scene_depth=scene_depth)


def sec_score_cfg1():
    """likelihood.cpp:106-233 over the whole cfg1 batch + variants."""
    w = configs.cfg1(_rf, R.voxel_to_mesh, seed=0)
    poses = w.grid_poses()
    t = time.time()
    s, st = R.score_poses(w.k, w.observed, w.vertices, w.triangles, poses, w.noise, w.sigma_max,
                          w.window)
    print(f"  cfg1 1,024 scores in {time.time() - t:.1f} s")
    sub = poses[::16]
    noise4 = [(0.01, 0.005), (0.2, 0.005), (0.05, 0.02), (0.5, 0.02)]
    multi = {wi: R.score_poses(w.k, w.observed, w.vertices, w.triangles, sub, noise4, 0.1, wi)[0]
             for wi in (0, 2, 3)}
    uniform = R.score_poses(w.k, w.observed, w.vertices, w.triangles, sub, w.noise, 0.1, 1,
                            prefactor=1)[0]
    full = R.score_poses(w.k, w.observed, w.vertices, w.triangles, poses[::64], w.noise, 0.1,
                         -1)[0]
    _save("score_cfg1", observed=w.observed, poses=poses, scores=s[:, 0], status=st,
          sub_idx=np.arange(0, 1024, 16), noise4=np.array(noise4), multi_w0=multi[0],
          multi_w2=multi[2], multi_w3=multi[3], uniform=uniform[:, 0],
          full_idx=np.arange(0, 1024, 64), full=full[:, 0])


def _stage_chain(w, stages, center, seed, score_fn):
    """Coarse-to-fine chain: per stage the grid around `center`, reference
    scores, then score_cells normalisation + sample_categorical (oracle
    restatement of inference.cpp:315-353) with Rng(seed)."""
    st = O.rng_seed(seed)
    out = {"centers": [np.asarray(center, dtype=np.float64)], "scores": [], "picks": [],
           "argmax": []}
    for g in stages:
        poses = configs.grid_poses(center, g["extent"], g["count"], g["rotations"], g["mode"])
        t = time.time()
        s = score_fn(poses, g)
        probs, _ = O.normalize(s)
        pick = O.sample_categorical(probs, st) if g.get("select", 0) == 0 else O.argmax(s)
        print(f"  stage: {poses.shape[0]} hypotheses in {time.time() - t:.1f} s, pick {pick}")
        out["scores"].append(s)
        out["picks"].append(pick)
        out["argmax"].append(O.argmax(s))
        center = poses[pick]
        out["centers"].append(center)
    out["rng_state"] = st
    return out


def sec_cfg2():
    """BASELINE configs[1] at full size: 5 x 32,768 reference scores along the
    sampled chain (seed 99)."""
    w = configs.cfg2(_rf, R.voxel_to_mesh, seed=0)

    def score(poses, g):
        return R.score_poses(w.k, w.observed, w.vertices, w.triangles, poses, [g["noise"]],
                             w.sigma_max, g["window"])[0][:, 0]

    ch = _stage_chain(w, w.stages, w.center, 99, score)
    _save("cfg2", observed=w.observed, centers=np.array(ch["centers"]),
          scores=np.array(ch["scores"]), picks=np.array(ch["picks"]),
          argmax=np.array(ch["argmax"]), rng_state=ch["rng_state"])


def _cfg3_world(w, counts):
    objs = w["objects"]
    tgt = w["target"]
    vox = synth.eden_blob([500, 1000, 2000, 3000, 4000][tgt], tgt)  # configs.cfg3, seed 0
    org = synth.centered_origin(vox, configs.RESOLUTION)
    world = R.World([(vox, configs.RESOLUTION, org)], 0.5, 0.5, w["sigma_max"], w["window"],
                    counts, [], w["noise"])
    assert np.array_equal(R.voxel_to_mesh(vox, configs.RESOLUTION, org)[0], objs[tgt][0])
    return world


def sec_cfg3():
    """BASELINE configs[2] at full size: all 131,072 contact hypotheses (the
    reference's own stage-0 cell centres of (object 4, face 1)) composited over
    the base scene and scored by the reference."""
    counts = (16, 16, 512)
    w = configs.cfg3(_rs, R.voxel_to_mesh, O.box_mesh, O.contact_to_pose, counts=counts)
    world = _cfg3_world(w, counts)
    poses = R.stage0_cell_poses(w["k"], world, 0, 1)
    assert poses.shape[0] == 131072
    tv, tt, _, _ = w["table"]
    base = [(tv, tt, IDENT)] + [(w["objects"][i][0], w["objects"][i][1], w["poses"][i])
                               for i in w["base"]]
    o = w["objects"][w["target"]]
    t = time.time()
    s, st = R.score_poses(w["k"], w["observed"], o[0], o[1], poses, w["noise"], w["sigma_max"],
                          w["window"], camera=w["camera"], base=base)
    print(f"  cfg3 131,072 scores in {time.time() - t:.1f} s, argmax {int(np.argmax(s[:, 0]))}")
    _save("cfg3", observed=w["observed"], poses=poses, scores=s[:, 0], status=st)


def sec_cfg5():
    """BASELINE configs[4]: a contiguous 65,536-hypothesis slice of the
    1,048,576 grid, around the ground truth, scored by the reference over the
    10-object base scene at 480x640."""
    w = configs.cfg5(_rs, R.voxel_to_mesh, O.box_mesh, O.contact_to_pose)
    n = w["n_hyp"]
    poses_all = configs.grid_poses(w["gt"], w["extent"], w["count"], w["rotations"], 0)
    centre = n // 2 + (w["count"][1] * w["count"][2] * 8) // 2  # the lattice point at the truth
    lo = centre - 32768
    idx = np.arange(lo, lo + 65536)
    tv, tt = w["table"]
    n_placed = len(w["base_poses"]) - 1
    base = [(tv, tt, w["base_poses"][0])] + [
        (w["library"][i][0], w["library"][i][1], w["base_poses"][1 + i]) for i in range(n_placed)]
    lib_t = w["library"][w["target"]]
    t = time.time()
    s, st = R.score_poses(w["k"], w["observed"], lib_t[0], lib_t[1], poses_all[idx], w["noise"],
                          w["sigma_max"], w["window"], camera=w["camera"], base=base)
    print(f"  cfg5 65,536 scores in {time.time() - t:.1f} s, slice argmax {lo + int(np.argmax(s))}")
    _save("cfg5", observed=w["observed"], first=np.int64(lo), scores=s[:, 0], status=st)


def _from_c(p):
    """The reference C ABI's from_c (b3d_capi.cpp:68-75): q / ||q|| with
    Eigen's scalar norm, (x^2 + y^2) + (z^2 + w^2)."""
    p = np.array(p, dtype=np.float64)
    w, x, y, z = (float(v) for v in p[:4])
    n = math.sqrt((x * x + y * y) + (z * z + w * w))
    p[:4] = [w / n, x / n, y / n, z / n]
    return p


def sec_cfg4():
    """BASELINE configs[3]: the 100-frame tracking sequence.  Per frame two
    argmax stages (strict >, lowest index: tracking.cpp:132-134) of 8,192
    reference-scored hypotheses each, centred on the previous estimate.
    Stored per stage: centre, argmax, the two best scores and 64 sampled
    scores (the whole 1.6 M scores would be 13 MB)."""
    tr = configs.cfg4(_rf, R.voxel_to_mesh, seed=0)
    k, verts, tris = tr["k"], tr["vertices"], tr["triangles"]
    est = tr["gt"][0].copy()
    rng = np.random.Generator(np.random.PCG64(44))
    centers, amax, top2, samp_idx, samp = [], [], [], [], []
    t0 = time.time()
    for f in range(1, len(tr["frames"])):
        obs = tr["frames"][f]
        c = est
        for g in tr["stages"]:
            poses = configs.grid_poses(c, g["extent"], g["count"], g["rotations"], 0)
            s = R.score_poses(k, obs, verts, tris, poses, [g["noise"]], 0.1, g["window"])[0][:, 0]
            a = O.argmax(s)
            order = np.argsort(-s, kind="stable")
            centers.append(c)
            amax.append(a)
            top2.append([s[order[0]], s[order[1]]])
            ii = rng.integers(0, s.shape[0], 64)
            samp_idx.append(ii)
            samp.append(s[ii])
            c = poses[a]
        # the next frame's centre crosses the C ABI as a b3d_pose, which the
        # boundary renormalises (from_c, b3d_capi.cpp:68-75)
        est = _from_c(c)
        if f % 10 == 0:
            print(f"  cfg4 frame {f}: {time.time() - t0:.0f} s")
    _save("cfg4", centers=np.array(centers), argmax=np.array(amax), top2=np.array(top2),
          sample_idx=np.array(samp_idx), sample_scores=np.array(samp), final=est)


def _smc_inputs():
    """A small scene-graph world: 3 library objects, a 0.4 m table, a camera
    looking down at 45 degrees, an observation from the reference's own
    renderer + sample_observation."""
    objs = []
    for i, nv in enumerate((60, 120, 200)):
        vox = synth.eden_blob(nv, 40 + i)
        objs.append((vox, 0.01, synth.centered_origin(vox, 0.01)))
    k = configs.Intr(60.0, 60.0, 31.5, 23.5, 64, 48, 0.05, 4.0)
    camera = R.camera_pose_from_spherical(0.8, 0.7, 0.9)
    # the true object on face 2 at a known contact
    v, t = R.voxel_to_mesh(*objs[1])
    pose = R.contact_to_pose(0.4, 0.4, objs[1][0], objs[1][1], objs[1][2], 2, 0.13, 0.21, 1.1)
    tv, tt = O.box_mesh(np.array([-0.2, -0.2, -0.01]), np.array([0.2, 0.2, 0.0]))
    rend = R.render(k, [(tv, tt, IDENT), (v, t, pose)], camera=camera)
    obs = R.sample_observation(rend, k, 0.1, 0.005, 1234, 3)
    return objs, k, camera, obs


def sec_smc():
    """inference.cpp:208-520 and b3d_infer (b3d_capi.cpp:297-379) on a small
    world: stage-0 cells and probabilities, 32 coarse-to-fine proposals,
    run_smc with 1 and 2 objects (resampling forced), and b3d_infer through
    the reference's own C ABI (windowed and window < 0)."""
    objs, k, camera, obs = _smc_inputs()
    noise = [(0.05, 0.0125), (0.3, 0.025), (0.05, 0.05)]
    world = R.World(objs, 0.4, 0.4, 0.1, 1, (3, 3, 4), [(2, 2, 2), (2, 1, 3)], noise)
    ints, iv, sc, az = R.stage0(k, obs, camera, world)
    paths, leaf, contact, log_q = R.propose(k, obs, camera, world, 77, 32)
    smc1 = R.run_smc(k, obs, camera, world, 1, 48, 0.5, 5)
    world2 = R.World(objs, 0.4, 0.4, 0.1, 1, (2, 2, 3), [(2, 2, 2)], noise)
    smc2 = R.run_smc(k, obs, camera, world2, 2, 24, 0.99, 6)
    kk = {"fx": k.fx, "fy": k.fy, "cx": k.cx, "cy": k.cy, "width": k.width, "height": k.height,
          "near": k.near, "far": k.far}
    base_cfg = {"intrinsics": kk, "table": {"width": 0.4, "height": 0.4},
                "schedule": {"stage0": [3, 3, 2], "refine": [[2, 2, 2]]},
                "noise_grid": {"p_outlier": [0.1, 0.4], "sigma": [0.01, 0.04]},
                "particles": 16, "n_objects": 1}
    inf_w = R.capi_infer(obs, k, camera, objs, dict(base_cfg, window=1), 9)
    inf_full = R.capi_infer(obs, k, camera, objs, dict(base_cfg, window=-1), 9)
    inf_deep = R.capi_infer(obs, k, camera, objs, dict(base_cfg, window=0, schedule={
        "stage0": [2, 2, 2], "refine": [[2, 1, 1], [1, 2, 1], [1, 1, 2], [2, 1, 1], [1, 1, 2],
                                        [2, 2, 1]]}), 10)
    import json
    _save("smc", observed=obs, camera=camera, k=np.array(k.as_tuple()), noise=np.array(noise),
          cells=ints, cell_iv=iv, stage0_scores=sc, all_zero=np.int32(az), paths=paths,
          leaf=leaf, contact=contact, log_q=log_q,
          smc1_children=smc1["children"], smc1_contact=smc1["contact"],
          smc1_noise=smc1["noise_index"], smc1_logw=smc1["log_weight"],
          smc1_logt=smc1["log_target"], smc1_ev=smc1["log_evidence"],
          smc2_children=smc2["children"], smc2_contact=smc2["contact"],
          smc2_noise=smc2["noise_index"], smc2_logw=smc2["log_weight"],
          smc2_logt=smc2["log_target"], smc2_ev=smc2["log_evidence"],
          infer_cfg=json.dumps(base_cfg),
          infer_w=json.dumps(inf_w["particles"]), infer_w_ev=inf_w["log_evidence"],
          infer_w_map=inf_w["map_pose"],
          infer_full=json.dumps(inf_full["particles"]), infer_full_ev=inf_full["log_evidence"],
          infer_full_map=inf_full["map_pose"],
          infer_deep=json.dumps(inf_deep["particles"]), infer_deep_ev=inf_deep["log_evidence"],
          infer_deep_map=inf_deep["map_pose"])


def sec_track():
    """tracking.cpp:59-206: the reference's own orbit frames
    (generate_orbit_sequence) and track_camera poses, default search and two
    variants (3 points x 3 stages; beam 2)."""
    vox = synth.eden_blob(600, 500)
    org = synth.centered_origin(vox, configs.RESOLUTION)
    k = configs.square_intrinsics(40)
    frames, gt = R.orbit_sequence(k, vox, configs.RESOLUTION, org, 10, sweep=0.5, p_outlier=0.02,
                                  sigma=0.002, seed=21)
    common = dict(window=configs.default_window(40), p_outlier=0.02, sigma=0.002)
    default = R.track_camera(k, vox, configs.RESOLUTION, org, frames, gt[0], **common)
    var3 = R.track_camera(k, vox, configs.RESOLUTION, org, frames, gt[0], points_per_dim=3,
                          refine_stages=3, **common)
    beam2 = R.track_camera(k, vox, configs.RESOLUTION, org, frames, gt[0], beam_width=2,
                           **common)
    obs1 = R.sample_observation(
        R.render(k, [(*R.voxel_to_mesh(vox, configs.RESOLUTION, org), IDENT)],
                 camera=np.array([0, 1.0, 0, 0, 0, 0, 0.3])), k, 0.3, 0.004, 8, 1, 2, 3)
    _save("track", voxels=vox, origin=org, k=np.array(k.as_tuple()), frames=frames, gt=gt,
          default=default, ppd3=var3, beam2=beam2, sampled=obs1)


def sec_capi():
    """The reference C ABI's status codes and error texts for boundary misuse
    (tests/capi_cases.py, the same calls the product is checked with)."""
    import json
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import capi_cases
    out = capi_cases.run_cases(R.lib(), gpu=True)
    path = os.path.join(HERE, "ref_capi.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    print(f"  wrote {os.path.relpath(path, ROOT)} ({len(out)} cases)")



def sec_fuzz():
    """The reference's b3d_infer on 240 seeded random configurations (and 200
    character-level edits of one, for the JSON parser's verdicts) and its
    b3d_scene_from_json / b3d_scene_to_json on 200 random scene documents
    (tests/infer_fuzz.py): status + message, or the result."""
    import json
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import infer_fuzz
    texts = infer_fuzz.configs() + infer_fuzz.syntax_texts()
    res = infer_fuzz.run(R.lib(), texts, True)
    path = os.path.join(HERE, "ref_infer_fuzz.json")
    with open(path, "w") as f:
        json.dump([{"config": t, "result": r} for t, r in zip(texts, res)], f, indent=0)
    ok = sum(1 for r in res if r[0] == 0)
    print(f"  wrote {os.path.relpath(path, ROOT)} ({len(res)} cases, {ok} valid)")
    scenes = infer_fuzz.scene_texts()
    res = infer_fuzz.run_scenes(R.lib(), scenes)
    path = os.path.join(HERE, "ref_scene_fuzz.json")
    with open(path, "w") as f:
        json.dump([{"scene": t, "result": r} for t, r in zip(scenes, res)], f, indent=0)
    print(f"  wrote {os.path.relpath(path, ROOT)} ({len(res)} cases)")
    import base64
    files = infer_fuzz.file_cases()
    res = infer_fuzz.run_files(R.lib(), files)
    path = os.path.join(HERE, "ref_file_fuzz.json")
    with open(path, "w") as f:
        json.dump([{"kind": k, "bytes": base64.b64encode(b).decode(), "result": r}
                   for (k, b), r in zip(files, res)], f, indent=0)
    print(f"  wrote {os.path.relpath(path, ROOT)} ({len(res)} cases)")
    for name, gen, run in (("loglik", infer_fuzz.loglik_cases, infer_fuzz.run_loglik),
                           ("render", infer_fuzz.render_cases, infer_fuzz.run_render)):
        cases = gen()
        res = run(R.lib(), cases)
        path = os.path.join(HERE, f"ref_{name}_fuzz.json")
        with open(path, "w") as f:
            json.dump([{"case": c, "result": r} for c, r in zip(cases, res)], f, indent=0)
        print(f"  wrote {os.path.relpath(path, ROOT)} ({len(res)} cases)")
    mans = infer_fuzz.manifest_texts()
    res = infer_fuzz.run_manifests(R.lib(), mans)
    path = os.path.join(HERE, "ref_manifest_fuzz.json")
    with open(path, "w") as f:
        json.dump([{"manifest": t, "result": r} for t, r in zip(mans, res)], f, indent=0)
    print(f"  wrote {os.path.relpath(path, ROOT)} ({len(res)} cases)")


SECTIONS = {"pose": sec_pose, "mesh": sec_mesh, "render": sec_render, "score_cfg1": sec_score_cfg1,
            "smc": sec_smc, "track": sec_track, "cfg2": sec_cfg2, "cfg3": sec_cfg3,
            "cfg5": sec_cfg5, "cfg4": sec_cfg4, "capi": sec_capi,
            "fuzz": sec_fuzz}


def main(argv):
    names = argv or list(SECTIONS)
    for n in names:
        t = time.time()
        print(f"[{n}]")
        SECTIONS[n]()
        print(f"  {time.time() - t:.1f} s")


if __name__ == "__main__":
    main(sys.argv[1:])

