"""ctypes binding of the CPU oracle (oracle/_build/libb3d_oracle.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference leg, as the checker -- never by
the product package.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(_HERE, "_build", "libb3d_oracle.so")
REF_RNG = os.path.join(_HERE, "_ref", "libref_rng.so")


class Intr(C.Structure):
    _fields_ = [("fx", C.c_double), ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("width", C.c_uint32), ("height", C.c_uint32),
                ("near_m", C.c_double), ("far_m", C.c_double)]


class Pose(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("qw", "qx", "qy", "qz", "tx", "ty", "tz")]


class Noise(C.Structure):
    _fields_ = [("p_outlier", C.c_double), ("sigma_noise", C.c_double)]


class Instance(C.Structure):
    _fields_ = [("vertices", C.c_void_p), ("triangles", C.c_void_p),
                ("n_vertices", C.c_uint64), ("n_triangles", C.c_uint64),
                ("model_to_world", Pose)]


class Counters(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in ("vertices", "triangles", "bbox_px", "fragments",
                                          "rend_valid", "obs_valid", "pairs")]

    def as_dict(self):
        return {n: getattr(self, n) for n, _ in self._fields_}


_lib = None


def build():
    subprocess.check_call(["make", "-s", "-C", _HERE])


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        L = C.CDLL(LIB)
        vp = C.c_void_p
        d = C.c_double
        L.orc_rng_uniform.restype = d
        L.orc_rng_normal.restype = d
        L.orc_rng_next_u64.restype = C.c_uint64
        L.orc_rng_uniform_int.restype = C.c_uint64
        L.orc_rng_uniform_int.argtypes = [vp, C.c_uint64]
        L.orc_rng_seed.argtypes = [C.c_uint64, vp]
        L.orc_rng_normal.argtypes = [vp]
        L.orc_rng_uniform.argtypes = [vp]
        L.orc_rng_next_u64.argtypes = [vp]
        L.orc_rng_split.argtypes = [vp, C.c_uint64, C.c_uint64, C.c_uint64, vp]
        L.orc_visible_volume.restype = d
        L.orc_logsumexp.restype = d
        L.orc_logsumexp.argtypes = [vp, C.c_size_t]
        L.orc_sample_categorical.restype = C.c_size_t
        L.orc_sample_categorical.argtypes = [vp, C.c_size_t, vp]
        L.orc_argmax.restype = C.c_size_t
        L.orc_argmax.argtypes = [vp, C.c_size_t]
        L.orc_normalize.argtypes = [vp, C.c_size_t, vp]
        L.orc_lattice.restype = d
        L.orc_lattice.argtypes = [d, d, C.c_int, C.c_int]
        L.orc_from_axis_angle.argtypes = [vp, d, vp]
        L.orc_camera_pose_from_spherical.argtypes = [d, d, d, vp]
        L.orc_contact_to_pose.argtypes = [d, d, vp, vp, C.c_int, d, d, d, vp]
        L.orc_windowed_loglik_multi.argtypes = [vp, vp, vp, vp, C.c_size_t, d, d, C.c_int,
                                                C.c_int, vp, vp]
        L.orc_full_loglik.argtypes = [vp, vp, vp, vp, d, d, C.c_int, vp]
        L.orc_full_loglik_points.argtypes = [vp, C.c_size_t, vp, C.c_size_t, vp, d, d, C.c_int,
                                             vp]
        L.orc_depth_to_cloud.argtypes = [vp, vp, vp, vp]
        L.orc_sample_observation.argtypes = [vp, vp, d, d, vp, vp]
        L.orc_raster_mesh.argtypes = [vp, vp, vp, vp, C.c_uint64, vp, C.c_uint64, vp,
                                      C.c_uint32, vp]
        L.orc_render_instances.argtypes = [vp, vp, vp, C.c_size_t, vp, vp, vp]
        L.orc_score_poses.argtypes = [vp, vp, vp, vp, vp, C.c_uint64, vp, C.c_uint64, vp,
                                      C.c_size_t, vp, C.c_size_t, d, C.c_int, C.c_int, vp, vp,
                                      C.c_int, vp]
        L.orc_voxel_to_mesh.argtypes = [vp, C.c_size_t, d, vp, vp, vp, vp, vp]
        L.orc_compose.argtypes = [vp, vp, vp]
        L.orc_inverse.argtypes = [vp, vp]
        L.orc_rotation_matrix.argtypes = [vp, vp]
        L.orc_rotated_bounds.argtypes = [vp, vp, C.c_int, vp, vp]
        L.orc_box_mesh.argtypes = [vp, vp, vp, vp]
        _lib = L
    return _lib


def intr(k) -> Intr:
    t = k.as_tuple() if hasattr(k, "as_tuple") else tuple(k)
    return Intr(*t)


def pose(p) -> Pose:
    return Pose(*np.asarray(p, dtype=np.float64).reshape(7).tolist())


def _p(a):
    return a.ctypes.data if a is not None else None


# ---------------------------------------------------------------- wrappers
def rng_seed(seed):
    st = np.zeros(5, dtype=np.uint64)
    lib().orc_rng_seed(seed, _p(st))
    return st


def rng_split(st, k0, k1=0, k2=0):
    out = np.zeros(5, dtype=np.uint64)
    lib().orc_rng_split(_p(st), k0, k1, k2, _p(out))
    return out


def rng_u64(st, n):
    return np.array([lib().orc_rng_next_u64(_p(st)) for _ in range(n)], dtype=np.uint64)


def rng_uniform(st):
    return lib().orc_rng_uniform(_p(st))


def rng_uniform_int(st, n):
    return int(lib().orc_rng_uniform_int(_p(st), n))


def rng_normal(st):
    return lib().orc_rng_normal(_p(st))


def voxel_to_mesh(voxels, resolution, origin):
    v = np.ascontiguousarray(voxels, dtype=np.int32)
    n = v.shape[0]
    verts = np.zeros((8 * n, 3), dtype=np.float64)
    tris = np.zeros((12 * n, 3), dtype=np.uint32)
    nv, nt = C.c_size_t(), C.c_size_t()
    o = np.ascontiguousarray(origin, dtype=np.float64)
    rc = lib().orc_voxel_to_mesh(_p(v), n, resolution, _p(o), _p(verts), _p(tris), C.byref(nv),
                                 C.byref(nt))
    assert rc == 0
    return verts[: nv.value].copy(), tris[: nt.value].copy()


def box_mesh(lo, hi):
    v = np.zeros((8, 3), dtype=np.float64)
    t = np.zeros((12, 3), dtype=np.uint32)
    lo_a = np.ascontiguousarray(lo, dtype=np.float64)  # keep alive across the call
    hi_a = np.ascontiguousarray(hi, dtype=np.float64)
    lib().orc_box_mesh(_p(lo_a), _p(hi_a), _p(v), _p(t))
    return v, t


def compose(a, b):
    out = Pose()
    pa, pb = pose(a), pose(b)
    lib().orc_compose(C.byref(pa), C.byref(pb), C.byref(out))
    return np.array([getattr(out, n) for n, _ in Pose._fields_])


def inverse(a):
    out = Pose()
    pa = pose(a)
    lib().orc_inverse(C.byref(pa), C.byref(out))
    return np.array([getattr(out, n) for n, _ in Pose._fields_])


def rotation_matrix(a):
    m = np.zeros(9, dtype=np.float64)
    pa = pose(a)
    lib().orc_rotation_matrix(C.byref(pa), _p(m))
    return m.reshape(3, 3)


def from_axis_angle(axis, angle, t=(0, 0, 0)):
    out = Pose()
    ax = np.ascontiguousarray(axis, dtype=np.float64)
    lib().orc_from_axis_angle(_p(ax), angle, C.byref(out))
    p = np.array([getattr(out, n) for n, _ in Pose._fields_])
    p[4:] = t
    return p


def camera_pose_from_spherical(d, az, alt):
    out = Pose()
    lib().orc_camera_pose_from_spherical(d, az, alt, C.byref(out))
    return np.array([getattr(out, n) for n, _ in Pose._fields_])


def contact_to_pose(table_w, table_h, aabb_min, aabb_max, face, dx, dy, dtheta):
    out = Pose()
    lo_a = np.ascontiguousarray(aabb_min, dtype=np.float64)
    hi_a = np.ascontiguousarray(aabb_max, dtype=np.float64)
    rc = lib().orc_contact_to_pose(table_w, table_h, _p(lo_a), _p(hi_a), face, dx, dy, dtheta,
                                   C.byref(out))
    if rc:
        raise ValueError("contact params out of valid range")
    return np.array([getattr(out, n) for n, _ in Pose._fields_])


def rotated_bounds(aabb_min, aabb_max, face):
    lo = np.zeros(3)
    hi = np.zeros(3)
    lo_a = np.ascontiguousarray(aabb_min, dtype=np.float64)
    hi_a = np.ascontiguousarray(aabb_max, dtype=np.float64)
    lib().orc_rotated_bounds(_p(lo_a), _p(hi_a), face, _p(lo), _p(hi))
    return lo, hi


def render(k, instances, camera=None, with_ids=False, counters=False):
    """render_instances: instances = [(vertices, triangles, model_to_world)]."""
    ki = intr(k)
    W, H = ki.width, ki.height
    keep = []
    arr = (Instance * max(1, len(instances)))()
    for i, (v, t, p) in enumerate(instances):
        v = np.ascontiguousarray(v, dtype=np.float64)
        t = np.ascontiguousarray(t, dtype=np.uint32)
        keep += [v, t]
        arr[i] = Instance(v.ctypes.data, t.ctypes.data, v.shape[0], t.shape[0], pose(p))
    depth = np.zeros((H, W), dtype=np.float32)
    ids = np.zeros((H, W), dtype=np.int32) if with_ids else None
    cam = pose(camera if camera is not None else [1, 0, 0, 0, 0, 0, 0])
    cnt = Counters()
    lib().orc_render_instances(C.byref(ki), C.byref(cam), arr, len(instances), _p(depth),
                               _p(ids), C.byref(cnt))
    out = (depth, ids) if with_ids else depth
    if counters:
        return out, cnt.as_dict()
    return out


def windowed_loglik_multi(obs, rend, k, noise, sigma_max, window, prefactor=0, volume=None,
                          counters=False):
    ki = intr(k)
    arr = (Noise * len(noise))(*[Noise(p, s) for p, s in noise])
    out = np.zeros(len(noise), dtype=np.float64)
    vol = lib().orc_visible_volume(C.byref(ki)) if volume is None else volume
    cnt = Counters()
    o = np.ascontiguousarray(obs, dtype=np.float32)
    r = np.ascontiguousarray(rend, dtype=np.float32)
    rc = lib().orc_windowed_loglik_multi(_p(o), _p(r), C.byref(ki), arr, len(noise), vol,
                                         sigma_max, window, prefactor, _p(out), C.byref(cnt))
    if rc:
        raise ValueError("windowed likelihood: invalid argument or empty rendered cloud")
    return (out, cnt.as_dict()) if counters else out


def full_loglik(obs, rend, k, noise, sigma_max, prefactor=0, volume=None):
    ki = intr(k)
    np_ = Noise(*noise)
    vol = lib().orc_visible_volume(C.byref(ki)) if volume is None else volume
    out = C.c_double()
    o = np.ascontiguousarray(obs, dtype=np.float32)
    r = np.ascontiguousarray(rend, dtype=np.float32)
    rc = lib().orc_full_loglik(_p(o), _p(r), C.byref(ki), C.byref(np_), vol, sigma_max,
                               prefactor, C.byref(out))
    if rc:
        raise ValueError("full likelihood: invalid argument or empty rendered cloud")
    return out.value


def full_loglik_points(obs_pts, rend_pts, noise, volume, sigma_max, prefactor=0):
    o = np.ascontiguousarray(obs_pts, dtype=np.float64).reshape(-1, 3)
    r = np.ascontiguousarray(rend_pts, dtype=np.float64).reshape(-1, 3)
    np_ = Noise(*noise)
    out = C.c_double()
    rc = lib().orc_full_loglik_points(_p(o), o.shape[0], _p(r), r.shape[0], C.byref(np_),
                                      volume, sigma_max, prefactor, C.byref(out))
    if rc:
        raise ValueError("full_log_likelihood: empty rendered cloud or invalid noise")
    return out.value


def depth_to_cloud(depth, k):
    ki = intr(k)
    d = np.ascontiguousarray(depth, dtype=np.float32)
    out = np.zeros((d.size, 3), dtype=np.float64)
    n = C.c_size_t()
    lib().orc_depth_to_cloud(_p(d), C.byref(ki), _p(out), C.byref(n))
    return out[: n.value].copy()


def sample_observation(rendered, k, p_outlier, sigma, st):
    """likelihood.cpp:44-80; st (5 x uint64) advanced in place.  None when the
    reference would throw."""
    r = np.ascontiguousarray(rendered, dtype=np.float32)
    out = np.empty_like(r)
    ki = intr(k)
    if lib().orc_sample_observation(_p(r), C.byref(ki), p_outlier, sigma, _p(st), _p(out)):
        return None
    return out


def visible_volume(k):
    ki = intr(k)
    return lib().orc_visible_volume(C.byref(ki))


def score_poses(k, observed, verts, tris, poses, noise, sigma_max, window, prefactor=0,
                base_depth=None, camera=None, threads=0, counters=False):
    ki = intr(k)
    poses = np.ascontiguousarray(poses, dtype=np.float64)
    n = poses.shape[0]
    arr = (Noise * len(noise))(*[Noise(p, s) for p, s in noise])
    scores = np.zeros((n, len(noise)), dtype=np.float64)
    status = np.zeros(n, dtype=np.uint8)
    v = np.ascontiguousarray(verts, dtype=np.float64)
    t = np.ascontiguousarray(tris, dtype=np.uint32)
    o = np.ascontiguousarray(observed, dtype=np.float32)
    cam = pose(camera if camera is not None else [1, 0, 0, 0, 0, 0, 0])
    cnt = Counters()
    lib().orc_score_poses(C.byref(ki), C.byref(cam), _p(o), _p(base_depth), _p(v), v.shape[0],
                          _p(t), t.shape[0], _p(poses), n, arr, len(noise), sigma_max, window,
                          prefactor, _p(scores), _p(status), threads, C.byref(cnt))
    if counters:
        return scores, status, cnt.as_dict()
    return scores, status


def normalize(lt):
    lt = np.ascontiguousarray(lt, dtype=np.float64)
    p = np.zeros_like(lt)
    az = lib().orc_normalize(_p(lt), lt.shape[0], _p(p))
    return p, bool(az)


def sample_categorical(probs, st):
    probs = np.ascontiguousarray(probs, dtype=np.float64)
    return int(lib().orc_sample_categorical(_p(probs), probs.shape[0], _p(st)))


def argmax(xs):
    xs = np.ascontiguousarray(xs, dtype=np.float64)
    return int(lib().orc_argmax(_p(xs), xs.shape[0]))


def logsumexp(xs):
    xs = np.ascontiguousarray(xs, dtype=np.float64)
    return float(lib().orc_logsumexp(_p(xs), xs.shape[0]))


# ------------------------------------------------ the reference's own RNG
def ref_rng_available() -> bool:
    return os.path.exists(REF_RNG)


def ref_rng_draw(seed, split, k0, k1, k2, kind, m, n):
    L = C.CDLL(REF_RNG)
    out = np.zeros(n, dtype=np.uint64)
    L.ref_rng_draw.argtypes = [C.c_uint64, C.c_int, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int,
                               C.c_uint64, C.c_void_p, C.c_size_t]
    L.ref_rng_draw(seed, split, k0, k1, k2, kind, m, out.ctypes.data, n)
    return out


# ---------------------------------------------------------------- tracking
_HALF_PI = 1.5707963267948966
_TWO_PI = 6.283185307179586476925287


def camera_pose_to_spherical(p, tol=1e-6):
    """generative.cpp:61-85 (libm asin/atan2/fmod as the reference; 3-term
    norms split x2 + (y2 + z2) like Eigen's redux)."""
    import math
    t = [float(p[4]), float(p[5]), float(p[6])]
    d = math.sqrt(t[0] * t[0] + (t[1] * t[1] + t[2] * t[2]))
    if d <= 0:
        return None
    sin_alt = min(max(t[2] / d, -1.0), 1.0)
    alt = math.asin(sin_alt)
    if alt <= 0 or alt >= _HALF_PI:
        return None
    az = math.fmod(math.atan2(t[1], t[0]), _TWO_PI)
    if az < 0:
        az += _TWO_PI
    e = camera_pose_from_spherical(d, az, alt)
    dt = [e[4] - t[0], e[5] - t[1], e[6] - t[2]]
    if math.sqrt(dt[0] * dt[0] + (dt[1] * dt[1] + dt[2] * dt[2])) > tol * max(1.0, d):
        return None
    a = [e[1] - p[1], e[2] - p[2], e[3] - p[3], e[0] - p[0]]
    b = [e[1] + p[1], e[2] + p[2], e[3] + p[3], e[0] + p[0]]
    qa = math.sqrt((a[0] * a[0] + a[1] * a[1]) + (a[2] * a[2] + a[3] * a[3]))
    qb = math.sqrt((b[0] * b[0] + b[1] * b[1]) + (b[2] * b[2] + b[3] * b[3]))
    if min(qa, qb) > tol:
        return None
    return d, az, alt


def _lattice(c, e, n):
    """tracking.cpp:27-37"""
    if n == 1:
        return [c]
    return [c - e + 2.0 * e * i / (n - 1) for i in range(n)]


def track_camera(frames, k, instances, initial, noise, sigma_max, window,
                 pos_extent=0.03, angle_extent=0.17453292519943295, points_per_dim=5,
                 refine_stages=2, refine_factor=3.0, beam_width=1, prefactor=0,
                 stage_log=None):
    """track_camera (tracking.cpp:59-172) over render_instances + the
    windowed likelihood of this oracle; returns the camera pose per frame.
    stage_log, if a list, receives (frame, stage, grid, scores) per stage."""
    start = camera_pose_to_spherical(initial)
    if start is None:
        raise ValueError("track_camera: initial pose must look at the origin with up = +z")
    poses = [np.asarray(initial, dtype=np.float64)]
    beam = [(start, 0.0)]
    n = points_per_dim
    for f in range(1, len(frames)):
        nxt = []
        for seed, _ in beam:
            center = seed
            pe, ae = pos_extent, angle_extent
            stage_best = (center, -np.inf)
            for st in range(refine_stages + 1):
                grid = [(d, az, alt) for d in _lattice(center[0], pe, n)
                        for az in _lattice(center[1], ae, n)
                        for alt in _lattice(center[2], ae, n)]
                scores = []
                for d, az, alt in grid:
                    if d <= 0 or alt <= 0 or alt >= _HALF_PI:
                        scores.append(-np.inf)
                        continue
                    cam = camera_pose_from_spherical(d, az, alt)
                    rend = render(k, instances, camera=cam)
                    scores.append(windowed_loglik_multi(frames[f], rend, k, [noise], sigma_max,
                                                        window, prefactor)[0])
                best = 0
                for i in range(1, len(scores)):
                    if scores[i] > scores[best]:
                        best = i
                if not np.isfinite(scores[best]):
                    raise ValueError("track_camera: every candidate pose scored -inf")
                if stage_log is not None:
                    stage_log.append((f, st, grid, scores))
                center = grid[best]
                stage_best = (center, scores[best])
                if beam_width > 1 and st == refine_stages:
                    order = sorted(range(len(grid)), key=lambda i: -scores[i])
                    for i in order[:beam_width]:
                        nxt.append((grid[i], scores[i]))
                pe /= refine_factor
                ae /= refine_factor
            if beam_width == 1:
                nxt.append(stage_best)
        nxt = sorted(nxt, key=lambda c: -c[1])[:beam_width]
        beam = nxt
        top = beam[0][0]
        poses.append(camera_pose_from_spherical(*top))
    return np.array(poses)


# ---------------------------------------------------------------- SMC
_TWO_PI_C = 6.283185307179586476925287


class _Rng:
    """rng.cpp through the pinned golden-vector restatement (rng_seed/split/uniform)."""

    def __init__(self, st):
        self.st = st

    @classmethod
    def seed(cls, s):
        return cls(rng_seed(s))

    def split(self, k0, k1=0, k2=0):
        return _Rng(rng_split(self.st, k0, k1, k2))

    def uniform(self, lo=None, hi=None):
        u = rng_uniform(self.st)
        return u if lo is None else lo + (hi - lo) * u


def run_smc(k, camera, observed, library, table, schedule, noise_grid, sigma_max, window,
            n_objects, n_particles, resample_threshold, seed, prefactor=0):
    """run_smc (inference.cpp:398-520) restated over this oracle's render and
    windowed likelihood.  library: [(verts, tris, aabb_min, aabb_max)];
    table: (verts, tris, width, height); schedule: (stage0 (nx, ny, nt),
    [refine (nx, ny, nt), ...]).  Returns (particles, log_evidence) with
    particles = [(children [(obj, face, dx, dy, dtheta)], noise_index,
    log_target, log_weight)]."""
    import math
    tv, tt, tw, th = table
    L = len(library)
    ident = np.array([1.0, 0, 0, 0, 0, 0, 0])

    def footprint(obj, face):
        lo, hi = rotated_bounds(library[obj][2], library[obj][3], face)
        return hi[0] - lo[0], hi[1] - lo[1]

    def child_prior(c):  # inference.cpp:26-38
        obj, face, dx, dy, dt = c
        fx, fy = footprint(obj, face)
        dxr, dyr = tw - fx, th - fy
        if dxr <= 0 or dyr <= 0:
            return -np.inf
        if dx < 0 or dx > dxr or dy < 0 or dy > dyr or dt < 0 or dt >= _TWO_PI_C:
            return -np.inf
        return (-math.log(float(L)) - math.log(6.0) - math.log(dxr) - math.log(dyr)
                - math.log(_TWO_PI_C))

    def prior_sum(cs):
        total = 0.0
        for c in cs:
            lp = child_prior(c)
            if not np.isfinite(lp):
                return -np.inf
            total += lp
        return total

    def pose_of(c):
        obj, face, dx, dy, dt = c
        return contact_to_pose(tw, th, library[obj][2], library[obj][3], face, dx, dy, dt)

    def base_depth(partial):  # render_partial
        inst = [(tv, tt, ident)] + [(library[c[0]][0], library[c[0]][1], pose_of(c))
                                    for c in partial]
        return render(k, inst, camera=camera)

    def score(obj, poses, noise, base):
        s, st = score_poses(k, observed, library[obj][0], library[obj][1], np.asarray(poses),
                            noise, sigma_max, window, prefactor, base_depth=base, camera=camera)
        s = s.copy()
        s[st != 0] = -np.inf
        return s

    def normalise(lt):  # inference.cpp:315-330
        m = max(lt)
        if not np.isfinite(m):
            return [1.0 / len(lt)] * len(lt), True
        sc = [math.exp(x - m) for x in lt]
        tot = 0.0
        for x in sc:
            tot += x
        return [x / tot for x in sc], False

    def sample(probs, rng):  # inference.cpp:345-353
        u = rng.uniform()
        acc = 0.0
        for i, p in enumerate(probs):
            acc += p
            if u < acc:
                return i
        return len(probs) - 1

    def center(iv):
        return 0.5 * (iv[0] + iv[1])

    def build_stage0(partial):
        nx, ny, nt = schedule[0]
        bp = prior_sum(partial)
        base = base_depth(partial)
        cells, lt = [], []
        for obj in range(L):
            for face in range(1, 7):
                fx, fy = footprint(obj, face)
                dxr, dyr = tw - fx, th - fy
                if dxr <= 0 or dyr <= 0:
                    continue
                grp = []
                for ix in range(nx):
                    for iy in range(ny):
                        for it in range(nt):
                            grp.append((obj, face, (dxr * ix / nx, dxr * (ix + 1) / nx),
                                        (dyr * iy / ny, dyr * (iy + 1) / ny),
                                        (_TWO_PI_C * it / nt, _TWO_PI_C * (it + 1) / nt)))
                poses = [pose_of((c[0], c[1], center(c[2]), center(c[3]), center(c[4])))
                         for c in grp]
                s = score(obj, poses, noise_grid, base)
                for ci, c in enumerate(grp):
                    cp = child_prior((c[0], c[1], center(c[2]), center(c[3]), center(c[4])))
                    for e in range(len(noise_grid)):
                        cells.append(c + (e,))
                        l = s[ci, e]
                        lt.append(bp + cp + l if np.isfinite(bp) and np.isfinite(cp)
                                  and np.isfinite(l) else -np.inf)
        probs, az = normalise(lt)
        return cells, probs, az

    def subdivide(c, st):
        nx, ny, nt = st
        obj, face, dx, dy, dt, e = c
        out = []
        for ix in range(nx):
            for iy in range(ny):
                for it in range(nt):
                    w0, w1, w2 = dx[1] - dx[0], dy[1] - dy[0], dt[1] - dt[0]
                    out.append((obj, face, (dx[0] + w0 * ix / nx, dx[0] + w0 * (ix + 1) / nx),
                                (dy[0] + w1 * iy / ny, dy[0] + w1 * (iy + 1) / ny),
                                (dt[0] + w2 * it / nt, dt[0] + w2 * (it + 1) / nt), e))
        return out

    def propose(partial, rng, stage0=None):  # inference.cpp:357-396
        cells, probs, _ = stage0 if stage0 is not None else build_stage0(partial)
        pick0 = sample(probs, rng)
        log_q = math.log(probs[pick0])
        cur = cells[pick0]
        for st in schedule[1]:
            ch = subdivide(cur, st)
            if len(ch) == 1:
                cur = ch[0]
                continue
            bp = prior_sum(partial)
            base = base_depth(partial)
            poses = [pose_of((c[0], c[1], center(c[2]), center(c[3]), center(c[4]))) for c in ch]
            s = score(cur[0], poses, [noise_grid[cur[5]]], base)
            lt = []
            for ci, c in enumerate(ch):
                cp = child_prior((c[0], c[1], center(c[2]), center(c[3]), center(c[4])))
                l = s[ci, 0]
                lt.append(bp + cp + l if np.isfinite(bp) and np.isfinite(cp) and np.isfinite(l)
                          else -np.inf)
            sc, _ = normalise(lt)
            pick = sample(sc, rng)
            log_q += math.log(sc[pick])
            cur = ch[pick]
        obj, face, dx, dy, dt, e = cur
        child = (obj, face, rng.uniform(dx[0], dx[1]), rng.uniform(dy[0], dy[1]),
                 rng.uniform(dt[0], dt[1]))
        vol = (dx[1] - dx[0]) * (dy[1] - dy[0]) * (dt[1] - dt[0])
        log_q += -math.log(vol)
        return child, e, log_q

    def target(children, e):  # scene_target_logpdf
        prior = prior_sum(children)
        if not np.isfinite(prior):
            return -np.inf
        s = score(children[-1][0], [pose_of(children[-1])], [noise_grid[e]],
                  base_depth(children[:-1]))
        return prior + s[0, 0] if np.isfinite(s[0, 0]) else -np.inf

    def lse(xs):
        m = max(xs)
        if not np.isfinite(m):
            return -np.inf
        acc = 0.0
        for x in xs:
            acc += math.exp(x - m)
        return m + math.log(acc)

    def weights(ps):
        lw = [p[3] for p in ps]
        l = lse(lw)
        return [math.exp(x - l) for x in lw]

    def resample(ps, rng):
        w = weights(ps)
        log_total = lse([p[3] for p in ps])
        n = len(ps)
        u = rng.uniform()
        out, cum, src = [], 0.0, 0
        for i in range(n):
            pos = (float(i) + u) / float(n)
            while src + 1 < n and cum + w[src] <= pos:
                cum += w[src]
                src += 1
            out.append(ps[src])
        reset = log_total - math.log(float(n))
        return [(p[0], p[1], p[2], reset) for p in out]

    rng = _Rng.seed(seed)
    s0 = build_stage0([])
    if s0[2]:
        raise ValueError("smc_init: all-zero scores at stage 0")
    ps = []
    for i in range(n_particles):
        child, e, log_q = propose([], rng.split(1, i), s0)
        lt = target([child], e)
        ps.append(([child], e, lt, lt - log_q))
    rs = rng.split(0x5e5a, 0)

    def maybe_resample(ps, stage):
        w = weights(ps)
        ess = 1.0 / sum(x * x for x in w)
        if ess < resample_threshold * n_particles:
            return resample(ps, rs.split(stage))
        return ps

    ps = maybe_resample(ps, 1)
    for kk in range(2, n_objects + 1):
        key = len(ps[0][0]) + 1
        nps = []
        for i, (ch, e0, lt0, lw) in enumerate(ps):
            child, e, log_q = propose(ch, rng.split(key, i))
            lt = target(ch + [child], e)
            nps.append((ch + [child], e, lt, lw + lt - lt0 - log_q))
        ps = maybe_resample(nps, kk)
    log_ev = lse([p[3] for p in ps]) - math.log(float(n_particles))
    return ps, log_ev
