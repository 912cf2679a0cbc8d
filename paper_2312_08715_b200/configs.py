"""BASELINE.json configs restated as concrete seeded workloads.

Each builder returns a Workload holding the mesh, intrinsics, observation,
hypothesis grid and likelihood settings.  The observation is rendered at the
ground-truth pose by `render_fn(k, vertices, triangles, pose) -> depth`
(the product renderer on a GPU box, or the CPU oracle in CPU-only tests; the
two are bit-identical, which the parity suite checks) and then corrupted.
Mapping of BASELINE terms onto the reference:
r -> sigma_noise, f x f window -> window = (f-1)/2, sigma_max = 0.1,
prefactor "printed".
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Callable, List, Optional

import numpy as np

from . import synth

RESOLUTION = 0.005  # 5 mm voxels


@dataclass
class Intr:
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int
    near: float
    far: float

    def as_tuple(self):
        return (self.fx, self.fy, self.cx, self.cy, self.width, self.height, self.near, self.far)


@dataclass
class Workload:
    name: str
    k: Intr
    voxels: np.ndarray
    vertices: np.ndarray
    triangles: np.ndarray
    gt_pose: np.ndarray            # (7,) model-to-camera ground truth
    observed: np.ndarray           # (H, W) float32
    center: np.ndarray             # (7,) grid centre
    extent: tuple
    count: tuple
    rotations: np.ndarray          # (n_rot, 4) perturbations dq
    grid_mode: int
    noise: List[tuple]             # [(p_outlier, sigma)]
    window: int
    sigma_max: float = 0.1
    stages: Optional[list] = None  # coarse-to-fine schedule (cfg2/cfg4)
    extra: dict = field(default_factory=dict)

    @property
    def n_hyp(self) -> int:
        nt = self.count[0] * self.count[1] * self.count[2]
        return nt * self.rotations.shape[0] if self.grid_mode == 0 else nt

    def grid_poses(self) -> np.ndarray:
        """All hypothesis poses on the host (same formulas as the device grid;
        used for the explicit-pose API and the CPU oracle)."""
        return _grid_poses_host(self.center, self.extent, self.count, self.rotations,
                                self.grid_mode)


def _grid_poses_host(center, extent, count, rotations, mode) -> np.ndarray:
    """Host restatement of the device pose grid (posemath.cuh grid_pose):
    tracking.cpp:34-35 lattice and q = normalized(center.q * dq), scalar
    Eigen evaluation order, no FMA (numpy float64 ops are single-rounded)."""
    nx, ny, nz = count
    nt = nx * ny * nz
    n_rot = rotations.shape[0]
    n = nt * n_rot if mode == 0 else nt
    idx = np.arange(n, dtype=np.int64)
    ti = idx // n_rot if mode == 0 else idx
    ri = idx % n_rot if mode == 0 else idx
    iz = ti % nz
    iy = (ti // nz) % ny
    ix = ti // (nz * ny)

    def lat(c, e, cnt, i):
        if cnt == 1:
            return np.full(i.shape, c, dtype=np.float64)
        return (c - e) + ((2.0 * e) * i.astype(np.float64)) / float(cnt - 1)

    aw, ax, ay, az = center[0], center[1], center[2], center[3]
    d = rotations[ri]
    bw, bx, by, bz = d[:, 0], d[:, 1], d[:, 2], d[:, 3]
    w = ((aw * bw - ax * bx) - ay * by) - az * bz
    x = ((aw * bx + ax * bw) + ay * bz) - az * by
    y = ((aw * by + ay * bw) + az * bx) - ax * bz
    z = ((aw * bz + az * bw) + ax * by) - ay * bx
    n2 = (x * x + y * y) + (z * z + w * w)
    nrm = np.sqrt(n2)
    out = np.zeros((n, 7), dtype=np.float64)
    out[:, 0] = w / nrm
    out[:, 1] = x / nrm
    out[:, 2] = y / nrm
    out[:, 3] = z / nrm
    out[:, 4] = lat(center[4], extent[0], nx, ix)
    out[:, 5] = lat(center[5], extent[1], ny, iy)
    out[:, 6] = lat(center[6], extent[2], nz, iz)
    return out


RenderFn = Callable[[Intr, np.ndarray, np.ndarray, np.ndarray], np.ndarray]


def make_mesh(voxels: np.ndarray, mesh_fn) -> tuple:
    origin = synth.centered_origin(voxels, RESOLUTION)
    return mesh_fn(voxels, RESOLUTION, origin)


def cfg1(render_fn: RenderFn, mesh_fn, seed: int = 0, blob: str = "eden",
         shard: int = 0) -> Workload:
    """configs[0]: single-object scoring at 160x120 (W x H).

    1,000-voxel blob (5 mm), pinhole fx=fy=200, cx=80, cy=60, near 0.01,
    far 10.  Observation: render at t=(0,0,0.6) with a uniform random
    rotation, N(0, 2 mm) depth noise, 10% of pixels -> U[0.2, 1.5] m.
    Hypotheses: 8x8x16 translation lattice over +-2 cm (16 along z) zipped
    with 1,024 independent vMF(kappa=1000) rotation perturbations.
    Likelihood r=5 mm, 3x3 window (w=1), outlier_prob 0.01.
    `shard` selects an independent batch of rotation perturbations (weak
    scaling: rank r scores batch r against the same observation).
    """
    rng = np.random.Generator(np.random.PCG64(1000 + seed))
    rng_rot = np.random.Generator(np.random.PCG64([2000 + seed, shard]))
    vox = synth.eden_blob(1000, seed) if blob == "eden" else synth.random_walk_blob(1000, seed)
    verts, tris = make_mesh(vox, mesh_fn)
    k = Intr(200.0, 200.0, 80.0, 60.0, 160, 120, 0.01, 10.0)
    q = synth.uniform_quaternion(rng)
    gt = np.array([q[0], q[1], q[2], q[3], 0.0, 0.0, 0.6])
    depth = render_fn(k, verts, tris, gt)
    obs = synth.noisy_observation(depth, k.far, 0.002, 0.10, 0.2, 1.5, rng, k.near)
    count = (8, 8, 16)
    rots = synth.vmf_quaternions(8 * 8 * 16, 1000.0, rng_rot)
    return Workload("cfg1_single_object_160x120", k, vox, verts, tris, gt, obs, gt.copy(),
                    (0.02, 0.02, 0.02), count, rots, 1, [(0.01, 0.005)], 1)


def grid_poses(center, extent, count, rotations, mode) -> np.ndarray:
    """Host poses of a device pose grid (same arithmetic as posemath.cuh)."""
    return _grid_poses_host(np.asarray(center, dtype=np.float64), extent, count,
                            np.asarray(rotations, dtype=np.float64), mode)


def _geom(a, b, n):
    return [a * (b / a) ** (i / (n - 1)) for i in range(n)]


def cfg2(render_fn: RenderFn, mesh_fn, seed: int = 0, n_stages: int = 5,
         counts=(16, 16, 16), n_rot: int = 8) -> Workload:
    """configs[1]: coarse-to-fine schedule, one object, 200x200, fx=fy=250.

    3,000-voxel blob; observation as cfg1 (N(0, 2 mm), 10% outliers).  Five
    stages of a 16x16x16 translation grid times 8 vMF rotations (PRODUCT,
    32,768 hypotheses); translation width 4 -> 2 -> 1 -> 0.5 -> 0.2 cm
    (extent = width / 2), kappa 50 -> 2000 and sigma 20 -> 2 mm geometric,
    window 7,7,5,5,3 (w = 3,3,2,2,1).  Each stage's centre is drawn from the
    previous stage's categorical posterior (seeded).  Stage 0 is centred on
    the ground truth displaced by 1.5 cm and ~10 degrees.
    """
    rng = np.random.Generator(np.random.PCG64(3000 + seed))
    vox = synth.eden_blob(3000, seed)
    verts, tris = make_mesh(vox, mesh_fn)
    k = Intr(250.0, 250.0, 100.0, 100.0, 200, 200, 0.01, 10.0)
    q = synth.uniform_quaternion(rng)
    gt = np.array([q[0], q[1], q[2], q[3], 0.0, 0.0, 0.6])
    depth = render_fn(k, verts, tris, gt)
    obs = synth.noisy_observation(depth, k.far, 0.002, 0.10, 0.2, 1.5, rng, k.near)
    d = rng.standard_normal(3)
    start = gt.copy()
    start[4:] += 0.015 * d / synth.norm(d)
    dq = synth.vmf_quaternions(1, 300.0, rng)[0]
    start[:4] = _qmul(gt[:4], dq)
    widths = [0.04, 0.02, 0.01, 0.005, 0.002]
    kappas = _geom(50.0, 2000.0, 5)
    sigmas = _geom(0.02, 0.002, 5)
    windows = [3, 3, 2, 2, 1]
    stages = []
    for s in range(n_stages):
        stages.append({"extent": (widths[s] / 2,) * 3, "count": counts,
                       "rotations": synth.vmf_quaternions(n_rot, kappas[s], rng), "mode": 0,
                       "noise": (0.01, sigmas[s]), "window": windows[s], "select": 0})
    w = Workload("cfg2_coarse_to_fine_200x200", k, vox, verts, tris, gt, obs, start,
                 stages[0]["extent"], counts, stages[0]["rotations"], 0, [stages[0]["noise"]],
                 windows[0], stages=stages)
    return w


def _qmul(a, b):
    aw, ax, ay, az = a
    bw, bx, by, bz = b
    q = np.array([aw * bw - ax * bx - ay * by - az * bz, aw * bx + ax * bw + ay * bz - az * by,
                  aw * by + ay * bw + az * bx - ax * bz, aw * bz + az * bw + ax * by - ay * bx])
    return q / synth.norm(q)


def _axis_angle_q(axis, angle):
    axis = np.asarray(axis, dtype=np.float64)
    axis = axis / synth.norm(axis)
    return np.concatenate([[math.cos(angle / 2)], math.sin(angle / 2) * axis])


def cfg4(render_fn: RenderFn, mesh_fn, seed: int = 0, n_frames: int = 100):
    """configs[3]: real-time tracking, 2,000-voxel blob, 240x320 (H x W),
    fx=fy=400 (cfg1's field of view), cx=160, cy=120.  Ground truth: seeded
    random walk, 1 cm translation and 5 degrees rotation per frame from
    (0, 0, 0.6); observations with N(0, 2 mm) noise and 5% outliers.  Per
    frame two stages of 8,192 hypotheses centred on the previous estimate,
    MAP (argmax) selection; likelihood
    r = 5 mm, 5x5 window, outlier_prob 0.05.  Per stage 8 x 8 x 4
    translations x 32 rotations (3x3x3 rotation-vector lattice + 5 vMF)."""
    rng = np.random.Generator(np.random.PCG64(4000 + seed))
    vox = synth.eden_blob(2000, seed)
    verts, tris = make_mesh(vox, mesh_fn)
    k = Intr(400.0, 400.0, 160.0, 120.0, 320, 240, 0.01, 10.0)
    q = synth.uniform_quaternion(rng)
    pose = np.array([q[0], q[1], q[2], q[3], 0.0, 0.0, 0.6])
    gts, frames = [], []
    for f in range(n_frames):
        if f:
            d = rng.standard_normal(3)
            pose = pose.copy()
            pose[4:] += 0.01 * d / synth.norm(d)
            pose[:4] = _qmul(_axis_angle_q(rng.standard_normal(3), math.radians(5.0)), pose[:4])
        gts.append(pose)
        depth = render_fn(k, verts, tris, pose)
        frames.append(synth.noisy_observation(depth, k.far, 0.002, 0.05, 0.2, 1.5, rng, k.near))
    # 8 x 8 x 4 translations x 32 rotations (a 3x3x3 rotation-vector lattice
    # plus 5 vMF draws) per stage: coarse (+-1.5 cm, 6 deg) then fine
    # (+-3 mm, 2 deg)
    stages = [
        {"extent": (0.015, 0.015, 0.01), "count": (8, 8, 4),
         "rotations": synth.rotation_lattice(math.radians(6.0), 5, 300.0, rng),
         "mode": 0, "noise": (0.05, 0.005), "window": 2, "select": 1},
        {"extent": (0.003, 0.003, 0.003), "count": (8, 8, 4),
         "rotations": synth.rotation_lattice(math.radians(2.0), 5, 5000.0, rng),
         "mode": 0, "noise": (0.05, 0.005), "window": 2, "select": 1},
    ]
    return {"k": k, "vertices": verts, "triangles": tris, "voxels": vox, "gt": np.array(gts),
            "frames": frames, "stages": stages, "name": "cfg4_tracking_240x320"}


TABLE_THICKNESS = 0.01


def table_mesh(mesh_box, w: float, h: float):
    """ObjectModel::table (scene_graph.cpp:26-35): thin box, top at z = 0."""
    lo = np.array([-w / 2, -h / 2, -TABLE_THICKNESS])
    hi = np.array([w / 2, h / 2, 0.0])
    v, t = mesh_box(lo, hi)
    return v, t, lo, hi


def cfg3(render_scene, mesh_fn, box_fn, contact_fn, seed: int = 0, counts=(16, 16, 512)):
    """configs[2]: multi-object scene graph with occlusion, 240x320 (H x W).

    A 0.5 x 0.5 m table (top plane at camera depth 0.7 m; the camera looks
    straight down at it) carries five seeded blobs of 500-4,000 voxels: three
    fixed ones (the base scene, rendered once), the enumerated fourth, and a
    fifth present only in the observation (a distractor).  The fourth object
    is enumerated over table-contact cells (face 1): a 16 x 16 (x, y) grid of
    cell centres times 512 yaw cells = 131,072 hypotheses.  Observation:
    ground-truth scene, N(0, 3 mm) depth noise, 5 % outliers.  Likelihood
    r = 5 mm, 5 x 5 window, outlier_prob 0.02.  fx = fy = 400, cx = 160, cy = 120.

    render_scene(k, camera, instances) -> depth; contact_fn(table_w, table_h,
    aabb_min, aabb_max, face, dx, dy, dtheta) -> pose; box_fn(lo, hi) -> mesh.
    """
    rng = np.random.Generator(np.random.PCG64(5000 + seed))
    k = Intr(400.0, 400.0, 160.0, 120.0, 320, 240, 0.01, 10.0)
    tw = th = 0.5
    tv, tt, tlo, thi = table_mesh(box_fn, tw, th)
    sizes = [500, 1000, 2000, 3000, 4000]
    objs = []
    for i, n in enumerate(sizes):
        vox = synth.eden_blob(n, 100 * seed + i)
        v, t = make_mesh(vox, mesh_fn)
        objs.append((v, t, v.min(axis=0), v.max(axis=0)))
    # camera: 0.7 m above the table centre looking down -z (camera +z forward)
    camera = np.array([0.0, 1.0, 0.0, 0.0, 0.0, 0.0, 0.7])  # 180 deg about x
    placements = []
    for i in range(5):
        v, t, lo, hi = objs[i]
        for _ in range(100):
            dx, dy = rng.uniform(0.05, 0.35), rng.uniform(0.05, 0.35)
            ok = all((dx - px) ** 2 + (dy - py) ** 2 > 0.12 ** 2 for px, py, _ in placements)
            if ok:
                break
        placements.append((dx, dy, rng.uniform(0.0, 2 * np.pi)))
    poses = [contact_fn(tw, th, objs[i][2], objs[i][3], 1, *placements[i]) for i in range(5)]
    ident = np.array([1.0, 0, 0, 0, 0, 0, 0])
    inst = [(tv, tt, ident)] + [(objs[i][0], objs[i][1], poses[i]) for i in range(5)]
    depth = render_scene(k, camera, inst)
    obs = synth.noisy_observation(depth, k.far, 0.003, 0.05, 0.2, 1.5, rng, k.near)
    return {"name": "cfg3_scene_graph_240x320", "k": k, "camera": camera, "table": (tv, tt, tlo, thi),
            "objects": objs, "poses": poses, "placements": placements, "observed": obs,
            "base": [0, 1, 2], "target": 3, "contact": dict(table_w=tw, table_h=th, face=1,
                                                          count=counts),
            "noise": [(0.02, 0.005)], "window": 2, "sigma_max": 0.1}


def cfg5(render_scene, mesh_fn, box_fn, contact_fn, seed: int = 0, counts=(64, 64, 32),
         n_rot: int = 8, n_library: int = 20, n_placed: int = 10):
    """configs[4]: large-scale sharded enumeration at 480x640 (H x W),
    fx = fy = 600, cx = 320, cy = 240.  A library of 20 seeded ~4,000-voxel
    blobs; 10 of them placed on a 0.6 x 0.6 m table (base scene, camera 0.8 m
    above it looking down); one more library object is enumerated over a
    64 x 64 x 32 translation lattice (+-4 cm x/y, +-2 cm z around its true
    position) times 8 vMF(kappa = 500) rotations = 1,048,576 6-DoF
    hypotheses.  Observation: ground truth with N(0, 2 mm) noise and 5 %
    outliers.  Likelihood r = 3 mm, 5 x 5 window, outlier_prob 0.02."""
    rng = np.random.Generator(np.random.PCG64(6000 + seed))
    k = Intr(600.0, 600.0, 320.0, 240.0, 640, 480, 0.01, 10.0)
    tw = th = 0.6
    tv, tt, tlo, thi = table_mesh(box_fn, tw, th)
    lib = []
    for i in range(n_library):
        vox = synth.eden_blob(4000, 1000 * seed + i)
        v, t = make_mesh(vox, mesh_fn)
        lib.append((v, t, v.min(axis=0), v.max(axis=0)))
    camera = np.array([0.0, 1.0, 0.0, 0.0, 0.0, 0.0, 0.8])
    placements = []
    for i in range(n_placed + 1):
        for _ in range(200):
            dx, dy = rng.uniform(0.02, 0.48), rng.uniform(0.02, 0.48)
            if all((dx - px) ** 2 + (dy - py) ** 2 > 0.11 ** 2 for px, py, _ in placements):
                break
        placements.append((dx, dy, rng.uniform(0.0, 2 * np.pi)))
    poses = [contact_fn(tw, th, lib[i][2], lib[i][3], 1, *placements[i])
             for i in range(n_placed + 1)]
    ident = np.array([1.0, 0, 0, 0, 0, 0, 0])
    base = [(tv, tt, ident)] + [(lib[i][0], lib[i][1], poses[i]) for i in range(n_placed)]
    target = n_placed  # library object n_placed is the enumerated one
    depth = render_scene(k, camera, base + [(lib[target][0], lib[target][1], poses[target])])
    obs = synth.noisy_observation(depth, k.far, 0.002, 0.05, 0.2, 1.5, rng, k.near)
    rots = synth.vmf_quaternions(n_rot, 500.0, rng)
    return {"name": "cfg5_sharded_480x640", "k": k, "camera": camera, "table": (tv, tt),
            "library": lib, "base_poses": [ident] + poses[:n_placed], "target": target,
            "gt": poses[target], "observed": obs, "extent": (0.04, 0.04, 0.02),
            "count": counts, "rotations": rots, "noise": [(0.02, 0.003)], "window": 2,
            "sigma_max": 0.1, "n_hyp": counts[0] * counts[1] * counts[2] * n_rot}


def square_intrinsics(res: int, fov_deg: float = 60.0, near: float = 0.1, far: float = 5.0):
    """harness.cpp:731-740 square_intrinsics (bench-tracking)."""
    f = res / (2.0 * math.tan(fov_deg * math.pi / 360.0))
    return Intr(f, f, (res - 1) / 2.0, (res - 1) / 2.0, res, res, near, far)


def default_window(width: int) -> int:
    """likelihood.cpp:231-233"""
    return max(1, int(np.floor(2.0 * width / 100.0 + 0.5)))


def orbit_sequence(render_cameras, mesh_fn, box_fn, contact_fn, res: int, n_frames: int = 120,
                   seed: int = 0, n_voxels: int = 1000, distance: float = 0.9,
                   altitude_deg: float = 40.0, sweep_deg: float = 360.0, sample_fn=None,
                   rng_state=None):
    """bench-tracking's orbit sequence (generate_orbit_sequence,
    tracking.cpp:174-215; harness.cpp:743-770 defaults): a 0.5 x 0.5 m table
    with one seeded voxel blob (stands in for the library object) standing on
    face 1 at the table centre, a camera orbiting at 0.9 m / 40 deg altitude
    sweeping 360 deg over the frames, square intrinsics (60 deg FOV, near 0.1,
    far 5).  Frames: render + N(0, 2 mm) depth noise, 2 % outliers (noise
    p_outlier 0.02, sigma 2 mm, the bench default).  render_cameras(k,
    instances, cameras) -> depth images.

    With sample_fn(k, depth_stack, p_outlier, sigma, rng_state) -> frames
    (b3d.sample_observations) and rng_state = Rng(seed).split(obj, res), the
    frames are the reference's own: sample_observation with
    rng.split(0x0f, i) per frame (tracking.cpp:196-203, harness.cpp:744-746);
    without, a numpy depth-noise model stands in."""
    rng = np.random.Generator(np.random.PCG64(7000 + 13 * seed + res))
    k = square_intrinsics(res)
    tw = th = 0.5
    tv, tt, tlo, thi = table_mesh(box_fn, tw, th)
    vox = synth.eden_blob(n_voxels, 500 + seed)
    v, t = make_mesh(vox, mesh_fn)
    lo, hi = v.min(axis=0), v.max(axis=0)
    fp = hi[:2] - lo[:2]  # face 1 footprint (x, y extents)
    pose = contact_fn(tw, th, lo, hi, 1, (tw - fp[0]) / 2, (th - fp[1]) / 2, 0.0)
    ident = np.array([1.0, 0, 0, 0, 0, 0, 0])
    inst = [(tv, tt, ident), (v, t, pose)]
    alt = altitude_deg * np.pi / 180.0
    sweep = sweep_deg * np.pi / 180.0
    az = [sweep * i / n_frames for i in range(n_frames)]
    return {"k": k, "instances": inst, "azimuths": az, "distance": distance, "altitude": alt,
            "noise": (0.02, 0.002), "window": default_window(res), "sigma_max": 0.1,
            "rng": rng, "render_cameras": render_cameras, "sample_fn": sample_fn,
            "rng_state": rng_state}


def orbit_frames(seq, cameras):
    """Rendered frames of an orbit sequence at the given camera poses, with
    the sequence's seeded depth noise and outliers."""
    k = seq["k"]
    depth = seq["render_cameras"](k, seq["instances"], cameras)
    if seq.get("sample_fn") is not None:  # frames 0..n-1 of the sequence
        p_out, sigma = seq["noise"]
        return seq["sample_fn"](k, depth, p_out, sigma, seq["rng_state"])
    out = np.empty_like(depth)
    for i in range(depth.shape[0]):
        out[i] = synth.noisy_observation(depth[i], k.far, 0.002, 0.02, k.near, k.far, seq["rng"],
                                         k.near)
    return out
