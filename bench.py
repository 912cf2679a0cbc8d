#!/usr/bin/env python
"""Benchmark: pose hypotheses rendered+scored per second (BASELINE.json).

Workload (N=1): configs[0], the configuration the metric is quoted on
(120x160 = H x W): a 1,000-voxel blob, 1,024 6-DoF hypotheses per step
(8x8x16 lattice zipped with vMF(kappa=1000) rotations), windowed likelihood
r=5 mm, 3x3 window.  One step = score the batch on the GPU (pose grid
generated on the device, fused raster + likelihood, rendered images never
leave the SM) + the stage reduction (argmax, logsumexp, one categorical
draw).  Weak scaling: at N GPUs each rank scores its own 1,024-hypothesis
batch against the shared observation, scores are all-gathered over NCCL and
every rank reduces the global array in one fixed order.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

--impl reference times the reference's algorithm on the host cores (the CPU
oracle port; the reference itself cannot be compiled here).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "pose hypotheses rendered+scored/sec at 120x160 @1/2/4/8 B200; tracking FPS"
UNIT = "hypotheses/s"
BATCH = 1024


def _ncu_traffic():
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the score
    kernel from the newest committed `ncu --set full` summary
    (profiles/r*_render_score_details.txt), or None."""
    import glob
    import re
    # the most recent capture: round tags sort by length then name (r1z < r1z4)
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_render_score_details.txt")),
                   key=lambda f: (len(os.path.basename(f)), os.path.basename(f)))
    # round 2 on: one capture per leg, the cfg1 one is the headline kernel's
    files += sorted(glob.glob(os.path.join(ROOT, "profiles", "r[0-9]*_cfg1_score_details.txt")),
                    key=lambda f: (len(os.path.basename(f)), os.path.basename(f)))
    # profiles/CURRENT names the tag of the build's own capture when set
    cur = os.path.join(ROOT, "profiles", "CURRENT")
    if os.path.exists(cur):
        tag = open(cur).read().strip()
        f = os.path.join(ROOT, "profiles", f"{tag}_cfg1_score_details.txt")
        if tag and os.path.exists(f):
            files.append(f)
    if not files:
        return None
    text = open(files[-1]).read()
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    total = 0.0
    for key in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        m = re.search(key + r"\s+([0-9.]+)\s+(\w+)", text)
        if not m:
            return None
        total += float(m.group(1)) * scale.get(m.group(2), 1.0)
    return {"bytes_per_launch": total, "source": os.path.relpath(files[-1], ROOT)}


def _golden(name):
    """A committed reference fixture (tests/golden/ref_<name>.npz, produced by
    the reference's own C++: tests/golden/make_ref_golden.py), or None."""
    path = os.path.join(ROOT, "tests", "golden", f"ref_{name}.npz")
    return np.load(path, allow_pickle=False) if os.path.exists(path) else None


def _max_rel(got, want) -> float:
    got = np.asarray(got, dtype=np.float64).ravel()
    want = np.asarray(want, dtype=np.float64).ravel()
    fin = np.isfinite(want)
    if not np.array_equal(np.isfinite(got), fin):
        return float("inf")
    if not fin.any():
        return 0.0
    return float((np.abs(got[fin] - want[fin]) / np.abs(want[fin])).max())


LEG_CPU = {"enabled": True, "seconds": 4.0, "fp64_peak": None}


def cpu_scorer(threads):
    """The CPU implementation the baselines time: the reference's own code --
    oracle/_ref/libb3d_ref.so, the reference's sources compiled unmodified
    (render_instances / raster_mesh / ObservationCache / windowed likelihood
    under its own parallel_for) -- when it is present (kind "reference"),
    else the oracle port of the same algorithm (kind "port").  Both give the
    same scores bit for bit (tests/test_ref_golden.py)."""
    try:
        from oracle import pyref as R
        have_ref = os.path.exists(R.LIB)
    except Exception:  # pragma: no cover
        have_ref = False
    if have_ref:
        def ref(k, obs, v, t, poses, noise, smax, window, base=None, camera=None):
            return R.score_poses(k, obs, v, t, poses, noise, smax, window, threads=threads,
                                 camera=camera, base=base or ())[0]
        return "reference", ref
    from oracle import pyoracle as O
    rendered = {}

    def port(k, obs, v, t, poses, noise, smax, window, base=None, camera=None):
        bd = None
        if base:
            if id(base) not in rendered:
                rendered[id(base)] = O.render(k, base, camera=camera)
            bd = rendered[id(base)]
        return O.score_poses(k, obs, v, t, poses, noise, smax, window, base_depth=bd,
                             camera=camera, threads=threads)[0]
    return "port", port


def leg_cpu_and_roofline(k, observed, verts, tris, poses, noise, sigma_max, window, gpu_value,
                         base=None, camera=None, what=""):
    """A leg's CPU baseline -- the reference's own code (or the oracle port,
    cpu_scorer) on all host threads, timed on a bounded sample of the leg's
    own hypotheses (about LEG_CPU seconds) -- and its roofline: the oracle's exact
    algorithmic op count per hypothesis times the leg's
    measured device rate, against the in-run non-FMA FP64 peak."""
    if not LEG_CPU["enabled"]:
        return None, None
    from oracle import pyoracle as O
    threads = cpu_threads()
    base_depth = None
    if base:
        base_depth = O.render(k, base, camera=camera)
    kw = dict(base_depth=base_depth, camera=camera, threads=threads)
    m = min(64, poses.shape[0])
    n_sigma = len({s for _, s in noise})
    if base:
        # the base-scene path's own work: the object's raster
        # and its windowed pairs; the base scene's per-pixel terms are a
        # per-observation table, so neither the base's pairs nor the
        # whole-image log terms are per-hypothesis work
        _, _, cnt = O.score_poses(k, observed, verts, tris, poses[:m], noise, sigma_max, window,
                                  counters=True, camera=camera, threads=threads)
        cnt = dict(cnt, obs_valid=0)
    else:
        _, _, cnt = O.score_poses(k, observed, verts, tris, poses[:m], noise, sigma_max, window,
                                  counters=True, **kw)
    ops = _ops_per_hyp(cnt, n_sigma, len(noise), m)
    kind, score = cpu_scorer(threads)
    done, t0, chunk = 0, time.perf_counter(), 16 * threads
    while True:
        i0 = done % poses.shape[0]
        sel = poses[i0:i0 + chunk]
        score(k, observed, verts, tris, sel, noise, sigma_max, window, base=base, camera=camera)
        done += sel.shape[0]
        el = time.perf_counter() - t0
        if el >= LEG_CPU["seconds"]:
            break
        chunk = min(4 * chunk, max(threads, int(done / el * (LEG_CPU["seconds"] - el)) + 1))
    cpu = {"value": done / el, "unit": UNIT, "cores": threads, "kind": kind,
           "sample": f"{done} of the leg's hypotheses{what}, {el:.1f} s"}
    roof = None
    if LEG_CPU["fp64_peak"]:
        ach = ops * gpu_value
        roof = {"bound": "sm_fp64", "achieved": ach / 1e12, "peak": LEG_CPU["fp64_peak"] / 1e12,
                "unit": "Tops/s", "frac": ach / LEG_CPU["fp64_peak"], "ops_per_hypothesis": ops,
                "note": "leg rate over its whole device time (all kernels of the leg)"
                        + ("; ops = the object's raster + windowed pairs (base-scene terms are "
                           "tabulated once per observation)" if base else "")}
    return cpu, roof


def _ops_per_hyp(c: dict, n_sigma: int, n_noise: int, n: int) -> float:
    """Algorithmic op count per hypothesis (BASELINE.md §3 / SURVEY.md 8d),
    from the oracle's exact counters."""
    return (18 * c["vertices"] + 45 * c["triangles"] + 18 * c["bbox_px"] + 10 * c["fragments"]
            + 6 * c["rend_valid"] + (8 + 3 * n_sigma) * c["pairs"]
            + 3 * n_noise * c["obs_valid"]) / n


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def cpu_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def build_workload_oracle(seed=0, shard=0):
    from oracle import pyoracle as O
    from paper_2312_08715_b200 import configs
    rf = lambda k, v, t, p: O.render(k, [(v, t, p)])
    return configs.cfg1(rf, O.voxel_to_mesh, seed=seed, shard=shard)


def cpu_baseline(w, seconds=12.0, threads=None, counters=True):
    """The reference's own code (cpu_scorer: oracle/_ref, else the oracle
    port) timed on this host's cores over repeated passes of the
    1,024-hypothesis batch; the oracle's op counters from one untimed pass."""
    from oracle import pyoracle as O
    threads = threads or cpu_threads()
    poses = w.grid_poses()
    cnt = None
    if counters:
        _, _, cnt = O.score_poses(w.k, w.observed, w.vertices, w.triangles, poses, w.noise,
                                  w.sigma_max, w.window, threads=threads, counters=True)
    kind, score = cpu_scorer(threads)
    done, t0 = 0, time.perf_counter()
    scores = None
    while True:
        scores = score(w.k, w.observed, w.vertices, w.triangles, poses, w.noise, w.sigma_max,
                       w.window)
        done += poses.shape[0]
        el = time.perf_counter() - t0
        if el >= seconds or done >= 64 * poses.shape[0]:
            break
    return {"value": done / el, "unit": UNIT, "cores": threads, "kind": kind,
            "sample": f"{done} hypotheses ({done // poses.shape[0]} passes of the cfg1 batch), "
                      f"{el:.1f} s"}, cnt, scores


def bench_config(world: int, w) -> dict:
    """The workload both arms report (identical dicts: same_config)."""
    return {"workload": "configs[0]: single-object scoring 160x120 (WxH), 1,024 "
                        "hypotheses/step/GPU (weak scaling: rank r scores rotation batch r)",
            "hypotheses_per_step": BATCH * world, "image": "120x160", "window": "3x3",
            "triangles": int(w.triangles.shape[0]), "vertices": int(w.vertices.shape[0]),
            "parallelism": f"dp{world} (hypothesis shards, score all-gather)"}


DTYPE = "f64/f32"
DTYPE_NOTE = ("pose math and raster in fp64 without FMA (bitwise the reference's depth); "
              "likelihood terms in fp32, accumulated in fp64 (SURVEY.md A.4)")


def run_reference(args, rank, world):
    """--impl reference: the reference's own code (cpu_scorer: oracle/_ref,
    compiled unmodified from the reference sources; the oracle port if it is
    absent) on host cores, all threads, over the same workload as our arm at
    this rank count (one 1,024-hypothesis batch per GPU-rank per step); the
    stage's normalisation / argmax / draw by the oracle.  Rank 0 alone runs."""
    if rank != 0:
        return
    from oracle import pyoracle as O
    threads = cpu_threads()
    kind, score = cpu_scorer(threads)
    batches = [build_workload_oracle(shard=r) for r in range(world)]
    w = batches[0]

    def step():
        for b in batches:
            s = score(b.k, b.observed, b.vertices, b.triangles, b.grid_poses(), b.noise,
                      b.sigma_max, b.window)
        probs, _ = O.normalize(s[:, 0])
        O.argmax(s[:, 0])
        O.sample_categorical(probs, O.rng_seed(7))

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    el = time.perf_counter() - t0
    v = args.steps * BATCH * world / el
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * el / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "dtype_note": ("the reference's own code" if kind == "reference" else
                           "the oracle port") + " computes everything in fp64",
            "data": "synthetic (seeded 1,000-voxel Eden blob, noisy rendered observation)",
            "impl": "reference", "config": bench_config(world, w),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": kind,
                             "sample": f"{args.steps} steps x {world} x {BATCH} hypotheses "
                                       "(the full per-step workload)"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_tracking(ctx, b3d, configs, frames_n, render_fn):
    """configs[3]: per frame, upload the observation (pinned host buffer) and
    run the two-stage argmax chain (b3d_gpu_coarse_to_fine) centred on the
    previous estimate; wall-clock per frame as in track_camera
    (tracking.cpp:73-82), host result read back every frame."""
    import torch
    # the context's work and the CUDA events / NCCL calls below on one stream
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    tr = configs.cfg4(render_fn, b3d.voxel_to_mesh, seed=0, n_frames=frames_n)
    ctx.set_camera(b3d.Intrinsics(*tr["k"].as_tuple()))
    mid = ctx.upload_mesh(tr["vertices"], tr["triangles"])
    st0 = tr["stages"][0]
    ctx.set_likelihood([st0["noise"]], 0.1, st0["window"])
    frames = [torch.from_numpy(f).pin_memory().numpy() for f in tr["frames"]]
    est = tr["gt"][0].copy()
    ctx.set_observation(frames[0])  # warm-up
    ctx.coarse_to_fine(mid, est, tr["stages"])
    ms, errs_cm, errs_deg, picks = [], [], [], []
    for f in range(1, frames_n):
        t0 = time.perf_counter()
        ctx.set_observation(frames[f])
        res, centers = ctx.coarse_to_fine(mid, est, tr["stages"])
        est = centers[-1]
        ms.append(1e3 * (time.perf_counter() - t0))
        picks += [(r.argmax, r.max_score, centers[s]) for s, r in enumerate(res)]
        gt = tr["gt"][f]
        errs_cm.append(100.0 * float(np.linalg.norm(est[4:] - gt[4:])))
        d = min(1.0, abs(float(np.dot(est[:4], gt[:4]))))
        errs_deg.append(float(np.degrees(2.0 * np.arccos(d))))
    total = sum(ms) * 1e-3
    # per-stage argmax agreement with the reference's chain over the same
    # frames (tracking.cpp:132-139 semantics; a tie within 1e-4 of the
    # reference's best counts as agreement)
    agree = None
    g = _golden("cfg4")
    if g is not None and len(picks) == g["argmax"].shape[0]:
        ok, same_idx, centres_ok, worst = 0, 0, 0, 0.0
        for i, (a, m, c) in enumerate(picks):
            top = float(g["top2"][i][0])
            same_idx += int(a == g["argmax"][i])
            ok += int(a == g["argmax"][i] or abs(m - top) <= 1e-4 * abs(top))
            centres_ok += int(np.array_equal(c, g["centers"][i]))
            worst = max(worst, abs(m - top) / abs(top))
        agree = {"stages": len(picks), "argmax_agreement": ok / len(picks),
                 "same_index": same_idx, "same_centre_bitwise": centres_ok,
                 "max_rel_err_best_score": worst,
                 "reference": "tests/golden/ref_cfg4.npz (the reference's own render + "
                              "windowed likelihood over the 100-frame sequence)"}
    g0 = tr["stages"][0]
    cpu, roof = leg_cpu_and_roofline(
        tr["k"], tr["frames"][1], tr["vertices"], tr["triangles"],
        configs.grid_poses(tr["gt"][0], g0["extent"], g0["count"], g0["rotations"], 0),
        [g0["noise"]], 0.1, g0["window"], 16384 * (frames_n - 1) / total,
        what=" (frame 1, stage 0)")
    if cpu is not None:
        cpu["fps"] = cpu["value"] / 16384.0
    return {"cpu_baseline": cpu, "roofline": roof,
            "workload": "configs[3]: 2,000-voxel blob, 240x320, 2 stages x 8,192 hypotheses "
                        "per frame (argmax chain on device), observation uploaded per frame",
            "fps": (frames_n - 1) / total, "frames": frames_n - 1,
            "ms_per_frame_mean": statistics.mean(ms), "ms_per_frame_p50": statistics.median(ms),
            "ms_per_frame_max": max(ms), "hypotheses_per_frame": 16384,
            "pose_error_cm_mean": statistics.mean(errs_cm),
            "pose_error_deg_mean": statistics.mean(errs_deg),
            "triangles": int(tr["triangles"].shape[0]), "reference_agreement": agree}


def run_bench_tracking(ctx, b3d, configs, resolutions=(25, 50, 100, 200), n_frames=120):
    """bench-tracking (harness.cpp:704-770, the paper's Table 1 analog): per
    resolution, an orbit sequence (table + one 1,000-voxel blob, camera at
    0.9 m / 40 deg sweeping 360 deg) tracked by b3d_gpu_track_camera with the
    reference's default search (5^3 spherical lattice, 3 stages, argmax);
    frames uploaded per frame from pinned host memory; FPS = frames / sum of
    the per-frame wall times (the reference's close_frame)."""
    import torch
    # the context's work and the CUDA events / NCCL calls below on one stream
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)

    def rc(k, inst, cams):
        ctx.set_camera(b3d.Intrinsics(*k.as_tuple()))
        mids = [ctx.upload_mesh(v, t) for v, t, _ in inst]
        ctx.set_camera_scene(mids, [p for _, _, p in inst])
        return ctx.render_cameras(np.asarray(cams), with_ids=False)[0]

    out = []
    for res in resolutions:
        # the reference's frames: sample_observation with Rng(0).split(obj, res).split(0x0f, i)
        seq = configs.orbit_sequence(
            rc, b3d.voxel_to_mesh, b3d.box_mesh, b3d.contact_to_pose, res=res, n_frames=n_frames,
            sample_fn=lambda k, d, p, s, st: b3d.sample_observations(
                b3d.Intrinsics(*k.as_tuple()), d, p, s, st),
            rng_state=b3d.rng_split(b3d.rng_seed(0), 0, res))
        cams = np.array([b3d.camera_pose_from_spherical(seq["distance"], a, seq["altitude"])
                         for a in seq["azimuths"]])
        frames = torch.from_numpy(configs.orbit_frames(seq, cams)).pin_memory().numpy()
        ctx.set_likelihood([seq["noise"]], seq["sigma_max"], seq["window"])
        ctx.track_camera(frames[:3], cams[0])  # warm-up
        est, ms = ctx.track_camera(frames, cams[0])
        pos = [100.0 * float(np.linalg.norm(est[i][4:] - cams[i][4:])) for i in range(n_frames)]
        rot = [float(np.degrees(2.0 * np.arccos(min(1.0, abs(float(np.dot(est[i][:4],
                                                                          cams[i][:4])))))))
               for i in range(n_frames)]
        # the paper's Table 1 budget: 2,048 hypotheses per frame
        # as an 8^3 lattice x 4 stages of the same search
        wide = b3d.TrackSearch.default(points_per_dim=8, refine_stages=3)
        ctx.track_camera(frames[:3], cams[0], wide)
        est2, ms2 = ctx.track_camera(frames, cams[0], wide)
        pos2 = [100.0 * float(np.linalg.norm(est2[i][4:] - cams[i][4:])) for i in range(n_frames)]
        out.append({"resolution": res, "fps": n_frames / (float(ms.sum()) * 1e-3),
                    "ms_per_frame_mean": float(ms[1:].mean()),
                    "mean_position_error_cm": statistics.mean(pos),
                    "mean_orientation_error_deg": statistics.mean(rot),
                    "window": seq["window"],
                    "fps_2048_hypotheses_per_frame": n_frames / (float(ms2.sum()) * 1e-3),
                    "mean_position_error_cm_2048": statistics.mean(pos2)})
    return {"workload": "bench-tracking orbit (Table 1 analog): table + 1,000-voxel blob, "
                        f"{n_frames} frames (the reference's sample_observation noise model, "
                        "p_outlier 0.02, sigma 2 mm), 125-point spherical lattice x 3 stages "
                        "(the reference harness's search; fps_2048_hypotheses_per_frame: 512 x 4, "
                        "the paper's Table 1 budget) "
                        "per frame, "
                        "camera-mode multi-instance render+score on device",
            "frames": n_frames, "per_resolution": out}


def run_smc_leg(ctx, b3d, configs, n_particles=1000, seed=0):
    """Scene-graph SMC (cmd_infer / cmd_pose_benchmark: run_smc with the
    harness defaults, harness.cpp:463-475): 0.5 x 0.5 m table seen from 0.7 m,
    a 5-blob library (500-4,000 voxels), one object placed in the observation
    (240x320, N(0, 3 mm), 5 % outliers), stage 0 10x10x8 x 6 faces x 9 noise
    entries, two 5x5x5 refine stages, 1,000 particles.  Every render+score runs
    on the device (b3d_gpu_run_smc); wall time of the whole inference."""
    import torch
    # the context's work and the CUDA events / NCCL calls below on one stream
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    rng = np.random.Generator(np.random.PCG64(8000 + seed))
    k = configs.Intr(400.0, 400.0, 160.0, 120.0, 320, 240, 0.01, 10.0)
    camera = np.array([0.0, 1.0, 0.0, 0.0, 0.0, 0.0, 0.7])
    tw = th = 0.5
    tv, tt, _, _ = configs.table_mesh(b3d.box_mesh, tw, th)
    lib = []
    for i, n in enumerate((500, 1000, 2000, 3000, 4000)):
        v, t = configs.make_mesh(configs.synth.eden_blob(n, 300 + i), b3d.voxel_to_mesh)
        lib.append((v, t, v.min(axis=0), v.max(axis=0)))
    truth = (2, 1, 0.21, 0.17, 2.2)
    pose = b3d.contact_to_pose(tw, th, lib[2][2], lib[2][3], 1, *truth[2:])
    render = _scene_renderer(ctx, b3d)
    depth = render(k, camera, [(tv, tt, np.array([1.0, 0, 0, 0, 0, 0, 0])),
                               (lib[2][0], lib[2][1], pose)])
    obs = configs.synth.noisy_observation(depth, k.far, 0.003, 0.05, 0.2, 1.5, rng, k.near)
    ctx.set_camera(b3d.Intrinsics(*k.as_tuple()), camera)
    table = ctx.upload_mesh(tv, tt)
    mids = [ctx.upload_mesh(v, t) for v, t, _, _ in lib]
    ctx.set_observation(obs)
    noise = [(p, f * 0.1) for p in (0.05, 0.3, 0.8) for f in (0.25, 0.5, 1.0)]
    sched = ((10, 10, 8), [(5, 5, 5), (5, 5, 5)])
    libs = [(mids[i], lib[i][2], lib[i][3]) for i in range(len(lib))]
    # one full-size warm-up run (buffer growth, host pool), then the median of
    # three timed runs (a single run is exposed to host-side stalls: one
    # box's bench saw 0.12 s against 0.024 s in every other run)
    ctx.run_smc(libs, table, tw, th, sched, noise, 0.1, 2, n_objects=1,
                n_particles=n_particles, resample_threshold=0.5, seed=seed)
    torch.cuda.synchronize()
    runs = []
    for _ in range(3):
        t0 = time.perf_counter()
        ps, le = ctx.run_smc(libs, table, tw, th, sched, noise, 0.1, 2, n_objects=1,
                             n_particles=n_particles, resample_threshold=0.5, seed=seed)
        runs.append(time.perf_counter() - t0)
    dt = float(np.median(runs))
    ctx.set_base_scene([], [])
    n_stage0 = 0
    for o in lib:
        for face in range(1, 7):
            lo, hi = b3d.rotated_bounds(o[2], o[3], face)
            if tw - (hi[0] - lo[0]) > 0 and th - (hi[1] - lo[1]) > 0:
                n_stage0 += 800
    renders = n_stage0 + n_particles * (2 * 125 + 1)
    best = max(ps, key=lambda p: p[3])
    c = best[0][0]
    cpu = None
    if LEG_CPU["enabled"]:
        # the reference's own render+score (cpu_scorer) on a bounded sample of
        # the inference's stage-0 hypotheses (object 2 = the true one, face 1,
        # all 9 noise entries, over the table): its render+score rate and the
        # run_smc time it implies for the workload's 275,000 renders
        threads = cpu_threads()
        kind, score = cpu_scorer(threads)
        cg = b3d.ContactGrid.make(tw, th, lib[2][2], lib[2][3], 1, (10, 10, 8))
        cells = b3d.contact_grid_poses(cg)
        table_inst = [(tv, tt, np.array([1.0, 0, 0, 0, 0, 0, 0]))]
        done, t0, chunk = 0, time.perf_counter(), threads
        while True:
            sel = cells[done % cells.shape[0]:done % cells.shape[0] + chunk]
            score(k, obs, lib[2][0], lib[2][1], sel, noise, 0.1, 2, base=table_inst,
                  camera=camera)
            done += sel.shape[0]
            el = time.perf_counter() - t0
            if el >= LEG_CPU["seconds"]:
                break
            chunk = min(4 * chunk, max(threads, int(done / el * (LEG_CPU["seconds"] - el)) + 1))
        rate = done / el
        cpu = {"value": rate, "unit": "renders/s", "cores": threads, "kind": kind,
               "sample": f"{done} stage-0 hypotheses (true object, face 1, 9 noise entries, "
                         f"table base), {el:.1f} s",
               "seconds_for_the_workload_est": renders / rate}
    return {"workload": "run_smc harness defaults: 5-object library, 240x320, stage 0 "
                        "10x10x8 x faces x 9 noise, 2 x 5x5x5 refine, 1,000 particles, "
                        "1 object; all render+score on device",
            "particles": n_particles, "seconds": dt, "seconds_runs": runs, "renders": renders,
            "renders_per_s": renders / dt,
            "renders_device": ctx.last_smc_renders,
            "renders_note": "renders = the reference's render+score evaluations for this "
                            "workload; renders_device = distinct ones launched (particles on "
                            "the same base scene, object, noise entry and cell share them: "
                            "identical values)",
            "log_evidence": le,
            "map_child": list(c), "truth": list(truth),
            "map_position_error_cm": 100.0 * float(np.hypot(c[2] - truth[2], c[3] - truth[3])),
            "map_object_correct": bool(c[0] == truth[0]), "cpu_baseline": cpu}


def run_coarse_to_fine(ctx, b3d, configs, render_fn, reps=5):
    """configs[1]: five 32,768-hypothesis stages chained on the device
    (sample selection); device time per schedule with CUDA events."""
    import torch
    # the context's work and the CUDA events / NCCL calls below on one stream
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    w = configs.cfg2(render_fn, b3d.voxel_to_mesh, seed=0)
    ctx.set_camera(b3d.Intrinsics(*w.k.as_tuple()))
    mid = ctx.upload_mesh(w.vertices, w.triangles)
    ctx.set_likelihood([w.stages[0]["noise"]], w.sigma_max, w.stages[0]["window"])
    d_obs = torch.from_numpy(w.observed).cuda()
    ctx.set_observation(d_obs)
    st = b3d.rng_seed(99)
    res0, centers0 = ctx.coarse_to_fine(mid, w.center, w.stages, rng_state=st)  # warm-up
    parity = None
    g = _golden("cfg2")
    if g is not None:  # the first chain from Rng(99) against the reference-scored chain
        parity = {"same_draws": [int(r.sample) for r in res0] == [int(x) for x in g["picks"]],
                  "same_argmax": [int(r.argmax) for r in res0] == [int(x) for x in g["argmax"]],
                  "same_centres_bitwise": bool(np.array_equal(centers0, g["centers"])),
                  "max_rel_err_stage_max": _max_rel([r.max_score for r in res0],
                                                    [s.max() for s in g["scores"]])}
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        res, centers = ctx.coarse_to_fine(mid, w.center, w.stages, rng_state=st)
        times.append(time.perf_counter() - t0)
    n = sum(int(np.prod(g["count"])) * g["rotations"].shape[0] for g in w.stages)
    gt = w.gt_pose
    g0 = w.stages[0]
    cpu, roof = leg_cpu_and_roofline(
        w.k, w.observed, w.vertices, w.triangles,
        configs.grid_poses(w.center, g0["extent"], g0["count"], g0["rotations"], 0),
        [g0["noise"]], w.sigma_max, g0["window"], n / statistics.median(times),
        what=" (stage 0's 32,768)")
    return {"workload": "configs[1]: 3,000-voxel blob, 200x200, 5 stages x 32,768 hypotheses, "
                        "sampled centres, chained on device",
            "hypotheses": n, "ms_per_schedule": 1e3 * statistics.median(times),
            "value": n / statistics.median(times), "unit": UNIT, "cpu_baseline": cpu,
            "roofline": roof,
            "final_error_cm": 100.0 * float(np.linalg.norm(centers[-1][4:] - gt[4:])),
            "triangles": int(w.triangles.shape[0]), "reference_parity": parity}


def _scene_renderer(ctx, b3d):
    """render_instances of a whole scene through the product (camera mode,
    one camera hypothesis): builds the configs' observations on the GPU."""
    def render(k, cam, inst):
        ctx.set_camera(b3d.Intrinsics(*k.as_tuple()))
        mids = [ctx.upload_mesh(v, t) for v, t, _ in inst]
        ctx.set_camera_scene(mids, [p for _, _, p in inst])
        return ctx.render_cameras(np.asarray(cam, dtype=np.float64)[None], with_ids=False)[0][0]
    return render


def run_scene_graph(ctx, b3d, configs, reps=3):
    """configs[2]: 131,072 table-contact hypotheses of the 4th object over a
    fixed table + 3 objects (base scene rendered once, composited per
    hypothesis), 240x320, device time per pass (CUDA events)."""
    import torch
    # the context's work and the CUDA events / NCCL calls below on one stream
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    w = configs.cfg3(_scene_renderer(ctx, b3d), b3d.voxel_to_mesh, b3d.box_mesh,
                     b3d.contact_to_pose)
    ctx.set_camera(b3d.Intrinsics(*w["k"].as_tuple()), w["camera"])
    tv, tt = w["table"][0], w["table"][1]
    mids = [ctx.upload_mesh(tv, tt)] + [ctx.upload_mesh(o[0], o[1]) for o in w["objects"]]
    ident = np.array([1.0, 0, 0, 0, 0, 0, 0])
    ctx.set_base_scene([mids[0]] + [mids[1 + i] for i in w["base"]],
                       [ident] + [w["poses"][i] for i in w["base"]])
    ctx.set_observation(torch.from_numpy(w["observed"]).cuda())
    ctx.set_likelihood(w["noise"], w["sigma_max"], w["window"])
    o = w["objects"][w["target"]]
    g = b3d.ContactGrid.make(0.5, 0.5, o[2], o[3], 1, w["contact"]["count"])
    n = g.n
    d_scores = torch.zeros((n, 1), dtype=torch.float64, device="cuda")
    d_status = torch.zeros(n, dtype=torch.uint8, device="cuda")
    ctx.score_contact_grid(mids[1 + w["target"]], g, d_scores, d_status)  # warm-up + terms
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    times = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        ctx.score_contact_grid(mids[1 + w["target"]], g, d_scores, d_status)
        e1.record(stream)
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) * 1e-3)
    best = int(torch.argmax(d_scores[:, 0]).item())
    gold = _golden("cfg3")
    parity = None
    if gold is not None:
        s = d_scores[:, 0].cpu().numpy()
        parity = {"hypotheses_compared": int(s.shape[0]),
                  "max_rel_err": _max_rel(s, gold["scores"]),
                  "same_argmax": best == int(np.argmax(gold["scores"]))}
    placements = w["placements"][w["target"]]
    ctx.set_base_scene([], [])
    base = [(tv, tt, ident)] + [(w["objects"][i][0], w["objects"][i][1], w["poses"][i])
                                for i in w["base"]]
    cpu, roof = leg_cpu_and_roofline(
        w["k"], w["observed"], o[0], o[1], b3d.contact_grid_poses(g)[best // 64 * 64:][:4096],
        w["noise"], w["sigma_max"], w["window"], n / statistics.median(times), base=base,
        camera=w["camera"], what=" (contact cells around the argmax)")
    return {"workload": "configs[2]: table + 3 fixed objects (base scene), 4th object over "
                        "16x16 (x,y) x 512 yaw contact cells, 240x320",
            "hypotheses": n, "ms": 1e3 * statistics.median(times),
            "value": n / statistics.median(times), "unit": UNIT,
            "triangles": int(o[1].shape[0]), "argmax": best,
            "true_contact": [round(v, 4) for v in placements], "reference_parity": parity,
            "cpu_baseline": cpu, "roofline": roof}


def run_sharded(ctx, b3d, configs, world, rank, reps=1):
    """configs[4]: 1,048,576 6-DoF hypotheses of one object over a 10-object
    base scene at 480x640, sharded evenly over the ranks; NCCL all-gather of
    the scores (8 MiB), global argmax / logsumexp and 1,000 posterior samples
    on every rank.  Device time, max over ranks."""
    import torch
    # the context's work and the CUDA events / NCCL calls below on one stream
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    import torch.distributed as dist
    from paper_2312_08715_b200.shard import gather_scores, shard_range
    w = configs.cfg5(_scene_renderer(ctx, b3d), b3d.voxel_to_mesh, b3d.box_mesh,
                     b3d.contact_to_pose)
    ctx.set_camera(b3d.Intrinsics(*w["k"].as_tuple()), w["camera"])
    tv, tt = w["table"]
    mids = [ctx.upload_mesh(tv, tt)] + [ctx.upload_mesh(l[0], l[1]) for l in w["library"]]
    n_placed = len(w["base_poses"]) - 1
    ctx.set_base_scene([mids[0]] + [mids[1 + i] for i in range(n_placed)], w["base_poses"])
    ctx.set_observation(torch.from_numpy(w["observed"]).cuda())
    ctx.set_likelihood(w["noise"], w["sigma_max"], w["window"])
    d_rot = torch.from_numpy(w["rotations"]).cuda()
    grid = ctx.make_grid(w["gt"], w["extent"], w["count"], d_rot, b3d.GRID_PRODUCT)
    n = w["n_hyp"]
    lo, hi = shard_range(n, rank, world)
    d_local = torch.zeros((hi - lo, 1), dtype=torch.float64, device="cuda")
    d_samples = torch.zeros(1000, dtype=torch.int64, device="cuda")
    st = torch.from_numpy(b3d.rng_seed(5).view(np.int64)).cuda()
    stream = torch.cuda.current_stream()
    mid = mids[1 + w["target"]]

    # N > 1: scores stored straight into every rank's symmetric-memory copy
    # of the 1M-entry array by the score kernel (the all-gather fused into the
    # scoring over NVLink), the ranks meet on a device signal-pad barrier,
    # every rank reduces / samples its complete copy; the two halves of each
    # copy alternate per exchange so no rank overwrites a half a peer may
    # still be reading.  Checked once against the NCCL gather; NCCL otherwise.
    xch = None
    gather = "single rank" if world == 1 else "nccl all_gather_into_tensor"
    if world > 1:
        try:
            from paper_2312_08715_b200.shard import SymmetricExchange
            xch = SymmetricExchange(n, 1, torch.device("cuda", torch.cuda.current_device()))
        except Exception as e:  # pragma: no cover - depends on the box
            gather = f"nccl all_gather_into_tensor (symmetric memory unavailable: {e})"

    def once(use_x=True):
        if xch is not None and use_x:
            e = xch.epoch + 1
            own = xch.half(e)
            ctx.set_score_peers(xch.peer_ptrs(e), lo, n)
            ctx.score_grid_range(mid, grid, lo, hi - lo, own[lo:hi], None)
            ctx.set_score_peers([], 0)
            xch.epoch = e
            ctx.shard_barrier(xch.signal_ptrs, rank, e)
            allv = own
        else:
            ctx.score_grid_range(mid, grid, lo, hi - lo, d_local, None)
            allv = gather_scores(d_local, n, world)
        return allv, ctx.sample_many(allv, 1000, st, n=n, samples=d_samples)

    once(use_x=False)  # warm-up (builds the base-scene likelihood terms)
    if xch is not None:
        ref_all = gather_scores(d_local, n, world).clone()
        allv, _ = once()
        torch.cuda.synchronize()
        same = torch.tensor([1 if torch.equal(allv, ref_all) else 0], device="cuda")
        dist.all_reduce(same, op=dist.ReduceOp.MIN)
        if int(same.item()) == 1:
            gather = ("fused into the score kernel (NVLink remote stores to symmetric memory, "
                      "signal-pad barrier, double-buffered)")
        else:
            xch = None
            gather = "nccl all_gather_into_tensor (fused path disagreed; fell back)"
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    times = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        allv, (_, r) = once()
        e1.record(stream)
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) * 1e-3)
    t = max(times)
    if world > 1:
        tt_ = torch.tensor([t], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt_, op=dist.ReduceOp.MAX)
        t = float(tt_.item())
    cpu = roof = None
    if rank == 0:
        base = [(tv, tt, w["base_poses"][0])] + [
            (w["library"][i][0], w["library"][i][1], w["base_poses"][1 + i])
            for i in range(n_placed)]
        lt = w["library"][w["target"]]
        best = int(r.argmax)
        allp = configs.grid_poses(w["gt"], w["extent"], w["count"], w["rotations"], 0)
        cpu, roof = leg_cpu_and_roofline(
            w["k"], w["observed"], lt[0], lt[1], allp[best // 64 * 64:][:4096], w["noise"],
            w["sigma_max"], w["window"], n / t, base=base, camera=w["camera"],
            what=" (a slice at the argmax)")
    parity = None
    g = _golden("cfg5")
    if g is not None:
        lo5 = int(g["first"])
        s5 = allv[lo5:lo5 + g["scores"].shape[0], 0].cpu().numpy()
        parity = {"hypotheses_compared": int(s5.shape[0]), "first": lo5,
                  "max_rel_err": _max_rel(s5, g["scores"]),
                  "global_argmax_in_slice_and_equal": int(r.argmax) == lo5 + int(
                      np.argmax(g["scores"]))}
    ctx.set_base_scene([], [])
    return {"workload": "configs[4]: 10-object base scene, 1,048,576 6-DoF hypotheses of a "
                        "new object, 480x640, sharded over ranks, NCCL score all-gather, global "
                        "argmax/logsumexp + 1,000 samples",
            "hypotheses": n, "n_gpus": world, "scaling": "strong", "s": t, "value": n / t,
            "unit": UNIT, "triangles": int(w["library"][w["target"]][1].shape[0]),
            "argmax": int(r.argmax), "logsumexp": r.logsumexp, "score_gather": gather,
            "reference_parity": parity, "cpu_baseline": cpu, "roofline": roof}


def spawn_ranks(args):
    """`bench.py --gpus N` run directly: re-launch as N ranks under
    torch.distributed.run on 127.0.0.1 (the driver's own launch), so the
    line reports the N-rank measurement, never a silent single rank."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1", "--master-port",
           str(port), os.path.abspath(__file__)] + sys.argv[1:]
    sys.stdout.flush()
    os.execv(sys.executable, cmd)


def dry_run(args, rank, world):
    """--dry-run: the ranks rendezvous (gloo, no GPU work) and all-reduce their
    ranks; rank 0 prints one line.  Checks the N-rank launch on CPU."""
    import torch
    import torch.distributed as dist
    total = rank
    if world > 1:
        dist.init_process_group("gloo")
        t = torch.tensor([rank], dtype=torch.int64)
        dist.all_reduce(t)
        total = int(t.item())
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "rank_sum": total,
                          "impl": args.impl}), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--tracking-frames", type=int, default=100)
    ap.add_argument("--no-extra", action="store_true", help="skip the cfg2/cfg4 legs")
    ap.add_argument("--dry-run", action="store_true",
                    help="launch / rendezvous check only: ranks meet over gloo, rank 0 prints")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        return spawn_ranks(args)  # one process per GPU, as the driver's torchrun would
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "ours" and world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.dry_run:
        return dry_run(args, rank, world)
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist
    from paper_2312_08715_b200 import b3d, configs

    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    # a dedicated (non-default) stream shared by torch and the C ABI context,
    # so the CUDA events below bracket exactly the work they time
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    ctx = b3d.GpuContext(local)
    ctx.set_stream(stream.cuda_stream)

    def render_fn(k, v, t, p):
        ctx.set_camera(b3d.Intrinsics(*k.as_tuple()))
        mid = ctx.upload_mesh(v, t)
        d, _ = ctx.render_poses(mid, np.asarray(p, dtype=np.float64)[None], with_ids=False)
        return d[0]

    w = configs.cfg1(render_fn, b3d.voxel_to_mesh, seed=0, shard=rank)
    ctx.set_camera(b3d.Intrinsics(*w.k.as_tuple()))
    mid = ctx.upload_mesh(w.vertices, w.triangles)
    ctx.set_likelihood(w.noise, w.sigma_max, w.window)
    n_all = BATCH * world

    # ---- device-resident arm (value)
    d_obs = torch.from_numpy(w.observed).to(dev)
    ctx.set_observation(d_obs)
    d_rot = torch.from_numpy(w.rotations).to(dev)
    grid = ctx.make_grid(w.center, w.extent, w.count, d_rot, w.grid_mode)
    d_scores = torch.zeros((BATCH, 1), dtype=torch.float64, device=dev)
    d_status = torch.zeros(BATCH, dtype=torch.uint8, device=dev)
    d_all = torch.zeros((n_all, 1), dtype=torch.float64, device=dev) if world > 1 else d_scores
    d_rng = torch.from_numpy(b3d.rng_seed(7).view(np.int64)).to(dev)
    d_res = torch.zeros(64, dtype=torch.uint8, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # > 126 MB L2

    # N > 1: one b3d_gpu_enumerate_shard call per step -- the score kernel
    # stores every score straight into all ranks' symmetric-memory copies of
    # the global array over NVLink (the all-gather fused into the scoring), a
    # device signal-pad barrier, then every rank reduces its complete copy
    # (the copies' two halves alternate per step: no write-after-read race).
    # NCCL all_gather_into_tensor is the fallback and the check: both must
    # give the same global array, else NCCL is used.
    xch = None
    gather = "single rank"
    if world > 1:
        gather = "nccl all_gather_into_tensor"
        try:
            from paper_2312_08715_b200.shard import SymmetricExchange
            xch = SymmetricExchange(n_all, 1, dev)
        except Exception as e:  # pragma: no cover - depends on the box
            gather = f"nccl all_gather_into_tensor (symmetric memory unavailable: {e})"

    def step(ev_k=None, use_x=True):
        if world == 1:  # score-many + stage reduction through one API call
            ctx.enumerate_grid(mid, grid, d_rng, d_res, d_scores)
            if ev_k is not None:
                ev_k.record(stream)
            return
        if xch is not None and use_x:
            ctx.enumerate_shard(mid, xch.exchange(rank * BATCH), grid=grid, n_local=BATCH,
                                rng_state=d_rng, out=d_res)
            if ev_k is not None:
                ev_k.record(stream)
            return
        ctx.score_grid(mid, grid, d_scores, d_status)
        if ev_k is not None:
            ev_k.record(stream)
        dist.all_gather_into_tensor(d_all, d_scores)
        ctx.stage_reduce(d_all, n=n_all, rng_state=d_rng, out=d_res)

    if xch is not None:
        step(use_x=False)  # reference gather into d_all
        step()
        torch.cuda.synchronize()
        same = torch.tensor([1 if torch.equal(xch.half(), d_all) else 0], device=dev)
        dist.all_reduce(same, op=dist.ReduceOp.MIN)
        if int(same.item()) == 1:
            gather = ("fused into the score kernel (b3d_gpu_enumerate_shard: NVLink remote "
                      "stores to symmetric memory, signal-pad barrier, double-buffered)")
        else:
            xch = None
            gather = "nccl all_gather_into_tensor (fused path disagreed; fell back)"
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
            torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    clocks = ClockSampler(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    time.sleep(0.3)
    # the device idles ~20 ms first (outside every event) while the host
    # queues all the timed steps, so a host-side stall (an nvidia-smi sample
    # holding the driver, a context switch) cannot open a gap between a
    # step's start event and its kernels: the events time device work only
    torch.cuda._sleep(40_000_000)
    for i in range(args.steps):
        flush.fill_(float(i))  # L2 flush between timed steps (outside the events)
        e0, ek, e1 = evs[i]
        e0.record(stream)
        step(ek)
        e1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    step_ms = [e0.elapsed_time(e1) for e0, _, e1 in evs]
    # the score kernel alone (roofline): same batch, L2 flushed before each
    # launch, CUDA events on the launching stream, outside the timed steps
    kern_ms = []
    for i in range(10):
        flush.fill_(float(i))
        torch.cuda._sleep(2_000_000)  # the launch is queued before the device gets to it
        ka, kb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ka.record(stream)
        ctx.score_grid(mid, grid, d_scores, d_status)
        kb.record(stream)
        torch.cuda.synchronize()
        kern_ms.append(ka.elapsed_time(kb))
    total_ms = sum(step_ms)
    parity_cfg1 = None
    g1 = _golden("score_cfg1")
    if g1 is not None and rank == 0:  # rank 0 scores configs[0]'s own batch (shard 0)
        s1 = d_scores[:, 0].cpu().numpy()
        parity_cfg1 = {"hypotheses_compared": int(s1.shape[0]),
                       "max_rel_err": _max_rel(s1, g1["scores"]),
                       "same_argmax": int(np.argmax(s1)) == int(np.argmax(g1["scores"]))}

    # ---- end-to-end arm: public C ABI with pinned host buffers
    ctx.set_stream(None)
    h_obs = torch.from_numpy(w.observed).pin_memory().numpy()
    h_poses = torch.from_numpy(w.grid_poses()).pin_memory().numpy()
    h_scores = torch.zeros((BATCH, 1), dtype=torch.float64).pin_memory().numpy()
    h_status = torch.zeros(BATCH, dtype=torch.uint8).pin_memory().numpy()
    h_all = torch.zeros((n_all, 1), dtype=torch.float64).pin_memory().numpy()
    h_rng = b3d.rng_seed(7)

    def e2e_step():
        if world == 1:  # one boundary call: upload observation + poses, score, reduce, read back
            return ctx.enumerate_observed(mid, h_obs, h_poses, rng_state=h_rng, scores=h_scores)
        if xch is not None:  # one boundary call: observation + shard in, fused gather, result out
            return ctx.enumerate_shard(mid, xch.exchange(rank * BATCH), poses=h_poses,
                                       depth=h_obs, rng_state=h_rng)
        ctx.set_observation(h_obs)  # pinned: stream-ordered upload
        ctx.score_poses(mid, h_poses, h_scores, h_status)
        t = torch.from_numpy(h_scores).to(dev)
        g = torch.empty((n_all, 1), dtype=torch.float64, device=dev)
        dist.all_gather_into_tensor(g, t)
        h_all[:] = g.cpu().numpy()
        return ctx.stage_reduce(h_all, n=n_all, rng_state=h_rng)

    for _ in range(args.warmup):
        e2e_step()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e2e_ms = []
    for i in range(args.steps):
        flush.fill_(float(i))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e2e_step()
        e2e_ms.append(1e3 * (time.perf_counter() - t0))
    e2e_total = sum(e2e_ms)
    clk = clocks.stop()

    if world > 1:
        t = torch.tensor([total_ms, e2e_total], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms, e2e_total = t.tolist()
    peaks = {}
    try:  # the roofline denominator, measured in-run (non-FMA DMUL/DADD probe)
        import ctypes
        L = ctypes.CDLL(os.path.join(ROOT, "paper_2312_08715_b200", "_lib", "libb3d_peaks.so"))
        r = ctypes.c_double()
        L.b3d_bench_fp64_rate.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_double)]
        if L.b3d_bench_fp64_rate(local, ctypes.byref(r)) == 0:
            peaks["fp64_nofma_ops"] = r.value
    except Exception as e:  # pragma: no cover
        peaks["error"] = str(e)
    LEG_CPU["enabled"] = not args.no_cpu_baseline
    LEG_CPU["fp64_peak"] = peaks.get("fp64_nofma_ops")
    sharded = None
    if not args.no_extra:
        sharded = run_sharded(ctx, b3d, configs, world, rank)

    if rank == 0:
        value = args.steps * n_all / (total_ms * 1e-3)
        e2e_value = args.steps * n_all / (e2e_total * 1e-3)
        kern_avg = statistics.mean(kern_ms) * 1e-3
        cpu = None
        cnt = None
        if not args.no_cpu_baseline:
            cpu, cnt, cpu_scores = cpu_baseline(w, seconds=args.cpu_seconds)
        extra = {}
        if not args.no_extra:
            extra["coarse_to_fine"] = run_coarse_to_fine(ctx, b3d, configs, render_fn)
            extra["tracking"] = run_tracking(ctx, b3d, configs, args.tracking_frames, render_fn)
            extra["scene_graph"] = run_scene_graph(ctx, b3d, configs)
            extra["bench_tracking"] = run_bench_tracking(ctx, b3d, configs)
            extra["smc"] = run_smc_leg(ctx, b3d, configs)
        roof = None
        if cnt is not None and "fp64_nofma_ops" in peaks:
            ops = _ops_per_hyp(cnt, 1, 1, BATCH)
            achieved = ops * BATCH / kern_avg
            roof = {"bound": "sm_fp64", "achieved": achieved / 1e12,
                    "peak": peaks["fp64_nofma_ops"] / 1e12, "unit": "Tops/s",
                    "frac": achieved / peaks["fp64_nofma_ops"],
                    "traffic": (_ncu_traffic() or {}).get("bytes_per_launch"),
                    "traffic_unit": "DRAM bytes per launch (ncu --set full)",
                    "traffic_source": (_ncu_traffic() or {}).get("source"),
                    "ops_per_hypothesis": ops,
                    # transcendentals reported separately
                    "transcendentals_per_hypothesis": {
                        "exp": cnt["pairs"] * 1 / BATCH, "log": cnt["obs_valid"] * 1 / BATCH},
                    "counts_per_hypothesis": {k: cnt[k] / BATCH for k in (
                        "vertices", "triangles", "bbox_px", "fragments", "rend_valid", "pairs",
                        "obs_valid") if k in cnt},
                    "kernel_ms": kern_avg * 1e3,
                    "peak_source": "measured in-run (non-FMA DMUL/DADD microbenchmark)"}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": DTYPE,
            "dtype_note": DTYPE_NOTE, "kernel_ms": kern_avg * 1e3,
            "data": "synthetic (seeded 1,000-voxel Eden blob, noisy rendered observation)",
            "config": bench_config(world, w),
            "l2": "flushed between timed steps (256 MB write)", "score_gather": gather,
            "gpu_launches": 2 * args.steps,  # render_score + stage_reduce per step
            "e2e": {"value": e2e_value, "unit": UNIT,
                    # N = 1: observation + poses + Rng state in; scores + stage result +
                    # Rng state out (b3d_gpu_enumerate_observed).  N > 1
                    # (b3d_gpu_enumerate_shard): observation + shard poses + Rng in,
                    # stage result + Rng out; the gather stays on the devices.
                    "h2d_bytes_per_step": int(h_obs.nbytes + h_poses.nbytes + 40
                                              + (0 if world == 1 or xch is not None
                                                 else h_scores.nbytes + h_all.nbytes)),
                    "d2h_bytes_per_step": int(h_scores.nbytes + 64 + 40 if world == 1
                                              else 64 + 40 if xch is not None
                                              else h_scores.nbytes + h_status.nbytes
                                              + h_all.nbytes + 64 + 40),
                    "ms_per_step": e2e_total / args.steps,
                    "ms_per_step_p50": float(np.median(e2e_ms)),
                    "ms_per_step_max": float(max(e2e_ms))},
            "clocks": clk,
            "roofline": roof,
            "cpu_baseline": cpu,
        }
        line.update(extra)
        if sharded is not None:
            line["sharded_enumeration"] = sharded
        # parity against the reference's own output on the same inputs
        # (tests/golden/ref_*.npz from the reference C++ compiled unmodified)
        line["parity"] = {
            "reference": "tests/golden/ref_*.npz (make_ref_golden.py: the reference's own "
                         "renderer, likelihood, inference and tracking code)",
            "bar": "scores <= 1e-4 relative; argmax equal or tied within 1e-4; depth/ids "
                   "bitwise (GPU tests)",
            "cfg1": parity_cfg1,
            "cfg2": extra.get("coarse_to_fine", {}).get("reference_parity"),
            "cfg3": extra.get("scene_graph", {}).get("reference_parity"),
            "cfg4": extra.get("tracking", {}).get("reference_agreement"),
            "cfg5": (sharded or {}).get("reference_parity")}
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
