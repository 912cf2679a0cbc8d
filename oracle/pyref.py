"""ctypes binding of the REFERENCE'S OWN implementation (oracle/_ref/libb3d_ref.so).

TEST INFRASTRUCTURE ONLY.  `make -C oracle ref` compiles every
/root/reference/proj/src/core/*.cpp plus src/capi/b3d_capi.cpp unmodified
against oracle/ref_shim/ (Eigen-subset stand-in, nlohmann forwarder) together
with oracle/ref_bridge.cpp (extern "C" entry points into the internals).  The
library exists only where /root/reference was present at build time; it is
used to generate the committed golden fixtures (tests/golden/make_ref_golden.py)
and, when present, by CPU tests that check the C restatement against it
directly.  Nothing in the product imports this module.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import tempfile

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(_HERE, "_ref", "libb3d_ref.so")

vp = C.c_void_p


class Intr(C.Structure):
    _fields_ = [("fx", C.c_double), ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("width", C.c_uint32), ("height", C.c_uint32),
                ("near_m", C.c_double), ("far_m", C.c_double)]


class Pose(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("qw", "qx", "qy", "qz", "tx", "ty", "tz")]


class SmcSpec(C.Structure):
    _fields_ = [("n_objects", C.c_int), ("voxels", vp), ("counts", vp), ("resolutions", vp),
                ("origins", vp), ("table_w", C.c_double), ("table_h", C.c_double),
                ("sigma_max", C.c_double), ("window", C.c_int), ("stage0", C.c_int * 3),
                ("n_refine", C.c_int), ("refine", vp), ("n_noise", C.c_int),
                ("noise_p", vp), ("noise_sigma", vp), ("threads", C.c_int)]


class TrackSpec(C.Structure):
    _fields_ = [("table_w", C.c_double), ("table_h", C.c_double), ("sigma_max", C.c_double),
                ("window", C.c_int), ("p_outlier", C.c_double), ("sigma", C.c_double),
                ("pos_extent", C.c_double), ("angle_extent", C.c_double),
                ("points_per_dim", C.c_int), ("refine_stages", C.c_int),
                ("refine_factor", C.c_double), ("beam_width", C.c_int), ("threads", C.c_int)]


class RefError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"reference status {status}: {msg}")
        self.status = status


_lib = None


def available() -> bool:
    return os.path.exists(LIB)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise RuntimeError(f"{LIB} missing: run `make -C oracle ref` where /root/reference exists")
        L = C.CDLL(LIB)  # RTLD_LOCAL: its b3d_* symbols never interpose the product's
        L.refb_last_error.restype = C.c_char_p
        L.b3d_last_error.restype = C.c_char_p
        for name in ("refb_compose", "refb_inverse", "refb_rotation_matrix", "refb_from_axis_angle",
                     "refb_camera_pose_from_spherical", "refb_camera_pose_to_spherical",
                     "refb_contact_to_pose", "refb_voxel_to_mesh", "refb_render_instances",
                     "refb_windowed_multi", "refb_full_loglik", "refb_score_poses",
                     "refb_sample_observation", "refb_stage0", "refb_propose", "refb_run_smc",
                     "refb_track_camera", "refb_orbit_sequence", "refb_stage0_cell_poses"):
            getattr(L, name).restype = C.c_int
        _lib = L
    return _lib


def _check(rc):
    if rc:
        raise RefError(rc, lib().refb_last_error().decode())


def _p(a):
    # always a c_void_p: a bare Python int would be passed as a 32-bit C int
    return C.c_void_p(a.ctypes.data) if a is not None else None


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def intr(k) -> Intr:
    t = k.as_tuple() if hasattr(k, "as_tuple") else tuple(k)
    return Intr(*t)


D = C.c_double


# ---------------------------------------------------------------- pose math
def compose(a, b):
    a, b, o = _f64(a), _f64(b), np.zeros(7)
    _check(lib().refb_compose(_p(a), _p(b), _p(o)))
    return o


def inverse(a):
    a, o = _f64(a), np.zeros(7)
    _check(lib().refb_inverse(_p(a), _p(o)))
    return o


def rotation_matrix(a):
    a, o = _f64(a), np.zeros(9)
    _check(lib().refb_rotation_matrix(_p(a), _p(o)))
    return o.reshape(3, 3)


def from_axis_angle(axis, angle):
    ax, o = _f64(axis), np.zeros(7)
    _check(lib().refb_from_axis_angle(_p(ax), D(angle), _p(o)))
    return o


def camera_pose_from_spherical(d, az, alt):
    o = np.zeros(7)
    _check(lib().refb_camera_pose_from_spherical(D(d), D(az), D(alt), _p(o)))
    return o


def camera_pose_to_spherical(pose, tol=1e-9):
    p, o, ok = _f64(pose), np.zeros(3), C.c_int()
    _check(lib().refb_camera_pose_to_spherical(_p(p), D(tol), _p(o), C.byref(ok)))
    return tuple(o) if ok.value else None


def contact_to_pose(table_w, table_h, voxels, resolution, origin, face, dx, dy, dtheta):
    v, org, o = np.ascontiguousarray(voxels, dtype=np.int32), _f64(origin), np.zeros(7)
    _check(lib().refb_contact_to_pose(D(table_w), D(table_h), _p(v), C.c_uint64(v.shape[0]),
                                      D(resolution), _p(org), face, D(dx), D(dy), D(dtheta), _p(o)))
    return o


def voxel_to_mesh(voxels, resolution, origin):
    v = np.ascontiguousarray(voxels, dtype=np.int32)
    cap_v, cap_t = 8 * v.shape[0] + 8, 12 * v.shape[0] + 12
    verts, tris = np.zeros((cap_v, 3)), np.zeros((cap_t, 3), dtype=np.uint32)
    nv, nt = C.c_uint64(), C.c_uint64()
    org = _f64(origin)
    _check(lib().refb_voxel_to_mesh(_p(v), C.c_uint64(v.shape[0]), D(resolution), _p(org),
                                    _p(verts), C.c_uint64(cap_v), _p(tris), C.c_uint64(cap_t),
                                    C.byref(nv), C.byref(nt)))
    return verts[: nv.value].copy(), tris[: nt.value].copy()


# ---------------------------------------------------------------- renderer / likelihood
def render(k, instances, camera=None):
    """render_instances (renderer.cpp:174-184): instances = [(vertices, triangles, model_to_world)]."""
    ki = intr(k)
    n = len(instances)
    keep = [(_f64(v), np.ascontiguousarray(t, dtype=np.uint32)) for v, t, _ in instances]
    vptr = (vp * max(n, 1))(*[v.ctypes.data for v, _ in keep])
    tptr = (vp * max(n, 1))(*[t.ctypes.data for _, t in keep])
    nv = np.array([v.shape[0] for v, _ in keep] or [0], dtype=np.uint64)
    nt = np.array([t.shape[0] for _, t in keep] or [0], dtype=np.uint64)
    poses = _f64([p for _, _, p in instances] or [[1, 0, 0, 0, 0, 0, 0]])
    cam = _f64(camera if camera is not None else [1, 0, 0, 0, 0, 0, 0])
    out = np.zeros((ki.height, ki.width), dtype=np.float32)
    _check(lib().refb_render_instances(C.byref(ki), n, vptr, _p(nv), tptr, _p(nt), _p(poses),
                                       _p(cam), _p(out)))
    return out


def windowed_loglik_multi(obs, rend, k, noise, sigma_max, window, prefactor=0):
    ki = intr(k)
    o, r = _f32(obs), _f32(rend)
    p = _f64([a for a, _ in noise])
    s = _f64([b for _, b in noise])
    out = np.zeros(len(noise))
    _check(lib().refb_windowed_multi(C.byref(ki), _p(o), _p(r), len(noise), _p(p), _p(s),
                                     D(sigma_max), window, prefactor, _p(out)))
    return out


def full_loglik(obs, rend, k, noise, sigma_max, prefactor=0):
    ki = intr(k)
    o, r, out = _f32(obs), _f32(rend), D()
    _check(lib().refb_full_loglik(C.byref(ki), _p(o), _p(r), D(noise[0]), D(noise[1]),
                                  D(sigma_max), prefactor, C.byref(out)))
    return out.value


def score_poses(k, observed, verts, tris, poses, noise, sigma_max, window, prefactor=0, threads=0,
                camera=None, base=()):
    """Per hypothesis: base instances [(v, t, pose)] rendered once, the object
    composited at each pose (compose_render), windowed multi-noise score
    (window < 0: full likelihood).  Returns (scores n x n_noise, status)."""
    ki = intr(k)
    o, v = _f32(observed), _f64(verts)
    t = np.ascontiguousarray(tris, dtype=np.uint32)
    poses = _f64(poses).reshape(-1, 7)
    n = poses.shape[0]
    p = _f64([a for a, _ in noise])
    s = _f64([b for _, b in noise])
    nb = len(base)
    keep = [(_f64(bv), np.ascontiguousarray(bt, dtype=np.uint32)) for bv, bt, _ in base]
    bvp = (vp * max(nb, 1))(*[x.ctypes.data for x, _ in keep])
    btp = (vp * max(nb, 1))(*[x.ctypes.data for _, x in keep])
    bnv = np.array([x.shape[0] for x, _ in keep] or [0], dtype=np.uint64)
    bnt = np.array([x.shape[0] for _, x in keep] or [0], dtype=np.uint64)
    bposes = _f64([bp for _, _, bp in base] or [[1, 0, 0, 0, 0, 0, 0]])
    cam = _f64(camera if camera is not None else [1, 0, 0, 0, 0, 0, 0])
    scores = np.zeros((n, len(noise)))
    status = np.zeros(n, dtype=np.int32)
    _check(lib().refb_score_poses(C.byref(ki), _p(o), _p(cam), nb, bvp, _p(bnv), btp, _p(bnt),
                                  _p(bposes), _p(v), C.c_uint64(v.shape[0]), _p(t),
                                  C.c_uint64(t.shape[0]), n, _p(poses), len(noise), _p(p), _p(s),
                                  D(sigma_max), window, prefactor, threads, _p(scores),
                                  _p(status)))
    return scores, status


def sample_observation(rendered, k, p_outlier, sigma, seed, k0=0, k1=0, k2=0):
    """sample_observation (likelihood.cpp:44-80) with rng = Rng(seed).split(k0, k1, k2)."""
    ki = intr(k)
    r = _f32(rendered)
    out = np.empty_like(r)
    _check(lib().refb_sample_observation(C.byref(ki), _p(r), D(p_outlier), D(sigma),
                                         C.c_uint64(seed), C.c_uint64(k0), C.c_uint64(k1),
                                         C.c_uint64(k2), _p(out)))
    return out


# ---------------------------------------------------------------- scene-graph inference
class World:
    """Library of voxel objects + table + model settings (make_inference_context)."""

    def __init__(self, objects, table_w, table_h, sigma_max, window, stage0, refine, noise,
                 threads=0):
        # objects: [(voxels int32 n x 3, resolution, origin)]
        self.voxels = np.ascontiguousarray(np.concatenate([o[0] for o in objects]), dtype=np.int32)
        self.counts = np.array([o[0].shape[0] for o in objects], dtype=np.uint64)
        self.res = _f64([o[1] for o in objects])
        self.origins = _f64([o[2] for o in objects])
        self.refine = np.ascontiguousarray(np.asarray(refine, dtype=np.int32).reshape(-1, 3))
        self.np_ = _f64([a for a, _ in noise])
        self.ns_ = _f64([b for _, b in noise])
        self.spec = SmcSpec(len(objects), self.voxels.ctypes.data, self.counts.ctypes.data,
                            self.res.ctypes.data, self.origins.ctypes.data, table_w, table_h,
                            sigma_max, window, (C.c_int * 3)(*stage0), self.refine.shape[0],
                            self.refine.ctypes.data, len(noise), self.np_.ctypes.data,
                            self.ns_.ctypes.data, threads)
        self.n_stages = 1 + self.refine.shape[0]


def stage0(k, observed, camera, world: World, cap=1 << 22):
    ki = intr(k)
    o, cam = _f32(observed), _f64(camera)
    n = C.c_uint64()
    ints = np.zeros((cap, 3), dtype=np.int32)
    iv = np.zeros((cap, 6))
    sc = np.zeros(cap)
    az = C.c_int()
    _check(lib().refb_stage0(C.byref(ki), _p(o), _p(cam), C.byref(world.spec), C.c_uint64(cap),
                             C.byref(n), _p(ints), _p(iv), _p(sc), C.byref(az)))
    m = n.value
    return ints[:m].copy(), iv[:m].copy(), sc[:m].copy(), bool(az.value)


def stage0_cell_poses(k, world: World, obj, face, cap=1 << 21):
    """World poses of the stage-0 cell centres of one (object, face) branch."""
    ki = intr(k)
    obs = np.full((ki.height, ki.width), ki.far_m, dtype=np.float32)
    n = C.c_uint64()
    out = np.zeros((cap, 7))
    _check(lib().refb_stage0_cell_poses(C.byref(ki), _p(obs), C.byref(world.spec), obj, face,
                                        C.c_uint64(cap), C.byref(n), _p(out)))
    return out[: n.value].copy()


def propose(k, observed, camera, world: World, seed, n_props):
    ki = intr(k)
    o, cam = _f32(observed), _f64(camera)
    paths = np.zeros((n_props, world.n_stages), dtype=np.int32)
    leaf = np.zeros((n_props, 3), dtype=np.int32)
    contact = np.zeros((n_props, 3))
    log_q = np.zeros(n_props)
    _check(lib().refb_propose(C.byref(ki), _p(o), _p(cam), C.byref(world.spec), C.c_uint64(seed),
                              n_props, _p(paths), _p(leaf), _p(contact), _p(log_q)))
    return paths, leaf, contact, log_q


def run_smc(k, observed, camera, world: World, n_objects, n_particles, threshold, seed):
    ki = intr(k)
    o, cam = _f32(observed), _f64(camera)
    ints = np.zeros((n_particles, n_objects, 2), dtype=np.int32)
    contact = np.zeros((n_particles, n_objects, 3))
    noise_index = np.zeros(n_particles, dtype=np.int32)
    log_w = np.zeros(n_particles)
    log_t = np.zeros(n_particles)
    ev = D()
    _check(lib().refb_run_smc(C.byref(ki), _p(o), _p(cam), C.byref(world.spec), n_objects,
                              n_particles, D(threshold), C.c_uint64(seed), _p(ints), _p(contact),
                              _p(noise_index), _p(log_w), _p(log_t), C.byref(ev)))
    return dict(children=ints, contact=contact, noise_index=noise_index, log_weight=log_w,
                log_target=log_t, log_evidence=ev.value)


# ---------------------------------------------------------------- tracking
def track_camera(k, voxels, resolution, origin, frames, initial, *, table_w=0.5, table_h=0.5,
                 sigma_max=0.1, window=2, p_outlier=0.1, sigma=0.005, pos_extent=0.03,
                 angle_extent=0.17453292519943295, points_per_dim=5, refine_stages=2,
                 refine_factor=3.0, beam_width=1, threads=0):
    ki = intr(k)
    v, org = np.ascontiguousarray(voxels, dtype=np.int32), _f64(origin)
    fr = _f32(frames)
    nf = fr.shape[0]
    spec = TrackSpec(table_w, table_h, sigma_max, window, p_outlier, sigma, pos_extent,
                     angle_extent, points_per_dim, refine_stages, refine_factor, beam_width,
                     threads)
    ini = _f64(initial)
    out = np.zeros((nf, 7))
    _check(lib().refb_track_camera(C.byref(ki), _p(v), C.c_uint64(v.shape[0]), D(resolution),
                                   _p(org), C.byref(spec), nf, _p(fr), _p(ini), _p(out)))
    return out


def orbit_sequence(k, voxels, resolution, origin, n_frames, *, distance=0.9,
                   altitude=0.6981317007977318, azimuth_start=0.0, sweep=6.283185307179586476925287,
                   table_w=0.5, table_h=0.5, p_outlier=0.1, sigma=0.005, seed=0):
    ki = intr(k)
    v, org = np.ascontiguousarray(voxels, dtype=np.int32), _f64(origin)
    frames = np.zeros((n_frames, ki.height, ki.width), dtype=np.float32)
    poses = np.zeros((n_frames, 7))
    _check(lib().refb_orbit_sequence(C.byref(ki), _p(v), C.c_uint64(v.shape[0]), D(resolution),
                                     _p(org), n_frames, D(distance), D(altitude), D(azimuth_start),
                                     D(sweep), D(table_w), D(table_h), D(p_outlier), D(sigma),
                                     C.c_uint64(seed), _p(frames), _p(poses)))
    return frames, poses


# ---------------------------------------------------------------- the reference's own C ABI
def capi_log_likelihood(obs, rend, k, p_outlier, sigma, sigma_max, window):
    """b3d_log_likelihood (b3d.h:110-115) of the reference library itself."""
    L = lib()
    ki = intr(k)
    o, r = _f32(obs), _f32(rend)
    ho, hr = vp(), vp()
    _check_capi(L.b3d_depth_image_create(ki.width, ki.height, _p(o), C.byref(ho)))
    _check_capi(L.b3d_depth_image_create(ki.width, ki.height, _p(r), C.byref(hr)))
    try:
        out = D()
        rc = L.b3d_log_likelihood(ho, hr, C.byref(ki), D(p_outlier), D(sigma), D(sigma_max),
                                  window, C.byref(out))
        _check_capi(rc)
        return out.value
    finally:
        L.b3d_depth_image_destroy(ho)
        L.b3d_depth_image_destroy(hr)


def _check_capi(rc):
    if rc:
        raise RefError(rc, lib().b3d_last_error().decode())


def _write_svox(path, voxels, resolution, origin):
    """SVOX (io.hpp:20): "SVOX" | f32 resolution | f32[3] origin | u32 count | count * i32[3]."""
    v = np.ascontiguousarray(voxels, dtype="<i4")
    with open(path, "wb") as f:
        f.write(b"SVOX")
        f.write(np.array([resolution, *origin], dtype="<f4").tobytes())
        f.write(np.array([v.shape[0]], dtype="<u4").tobytes())
        f.write(v.tobytes())


def capi_infer(observed, k, camera, objects, config: dict, seed: int):
    """b3d_infer (b3d.h:121-124) of the reference library: objects =
    [(voxels, resolution, origin)] written as SVOX + manifest.  Returns the
    particle JSONL lines, log evidence and MAP pose of child 0."""
    L = lib()
    ki = intr(k)
    with tempfile.TemporaryDirectory() as d:
        models = []
        for i, (vox, res, org) in enumerate(objects):
            _write_svox(os.path.join(d, f"m{i}.svox"), vox, res, org)
            models.append({"id": i, "path": f"m{i}.svox"})
        with open(os.path.join(d, "manifest.json"), "w") as f:
            json.dump({"models": models}, f)
        hl = vp()
        _check_capi(L.b3d_library_open(os.path.join(d, "manifest.json").encode(), C.byref(hl)))
    o = _f32(observed)
    ho, hp = vp(), vp()
    _check_capi(L.b3d_depth_image_create(ki.width, ki.height, _p(o), C.byref(ho)))
    cam = Pose(*_f64(camera).tolist())
    try:
        _check_capi(L.b3d_infer(ho, C.byref(cam), hl, json.dumps(config).encode(),
                                C.c_uint64(seed), C.byref(hp)))
        s = C.c_void_p()
        L.b3d_particles_to_jsonl.argtypes = [vp, C.POINTER(C.c_void_p)]
        _check_capi(L.b3d_particles_to_jsonl(hp, C.byref(s)))
        text = C.cast(s, C.c_char_p).value.decode()
        L.b3d_string_free(s)
        ev = D()
        _check_capi(L.b3d_particles_log_evidence(hp, C.byref(ev)))
        mp = Pose()
        _check_capi(L.b3d_particles_map_pose(hp, C.c_size_t(0), C.byref(mp)))
        return dict(particles=[json.loads(x) for x in text.splitlines() if x.strip()],
                    log_evidence=ev.value,
                    map_pose=np.array([getattr(mp, n) for n, _ in Pose._fields_]))
    finally:
        L.b3d_depth_image_destroy(ho)
        if hp:
            L.b3d_particles_destroy(hp)
        L.b3d_library_destroy(hl)
