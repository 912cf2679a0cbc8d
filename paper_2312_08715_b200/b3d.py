"""ctypes client of libb3d_b200.so (include/b3d_b200.h).

The product is the C ABI + C++ host layer + sm_100a kernels in csrc/; this
module only marshals arguments so tests and bench.py can drive the same
entry points a foreign caller would bind.  There is no CPU
fallback: if the shared library or a GPU is missing, calls fail loudly.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("B3D_LIB") or os.path.join(_HERE, "_lib", "libb3d_b200.so")

B3D_OK = 0
B3D_ERROR = 1
B3D_ERROR_CONFIG = 2
B3D_ERROR_IO = 3
B3D_ERROR_NUMERIC = 4
PREFACTOR_PRINTED = 0
PREFACTOR_UNIFORM = 1
GRID_PRODUCT = 0
GRID_ZIP = 1

# b3d_pose as a numpy row: (qw, qx, qy, qz, tx, ty, tz)
POSE_DTYPE = np.float64


class B3DError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"b3d status {status}: {message}")
        self.status = status


class Intrinsics(C.Structure):
    _fields_ = [("fx", C.c_double), ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("width", C.c_uint32), ("height", C.c_uint32),
                ("near_m", C.c_double), ("far_m", C.c_double)]

    @classmethod
    def make(cls, fx, fy, cx, cy, width, height, near, far):
        return cls(fx, fy, cx, cy, width, height, near, far)


class Pose(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("qw", "qx", "qy", "qz", "tx", "ty", "tz")]


class Noise(C.Structure):
    _fields_ = [("p_outlier", C.c_double), ("sigma_noise", C.c_double)]


class PoseGrid(C.Structure):
    _fields_ = [("center", Pose), ("extent", C.c_double * 3), ("count", C.c_uint32 * 3),
                ("rotations", C.c_void_p), ("n_rot", C.c_uint32), ("mode", C.c_uint32)]


class ContactGrid(C.Structure):
    _fields_ = [("table_w", C.c_double), ("table_h", C.c_double), ("aabb_min", C.c_double * 3),
                ("aabb_max", C.c_double * 3), ("face", C.c_int32), ("count", C.c_uint32 * 3)]

    @classmethod
    def make(cls, table_w, table_h, aabb_min, aabb_max, face, count):
        g = cls()
        g.table_w, g.table_h, g.face = float(table_w), float(table_h), int(face)
        for a in range(3):
            g.aabb_min[a] = float(aabb_min[a])
            g.aabb_max[a] = float(aabb_max[a])
            g.count[a] = int(count[a])
        return g

    @property
    def n(self):
        return self.count[0] * self.count[1] * self.count[2]


class StageSpec(C.Structure):
    _fields_ = [("extent", C.c_double * 3), ("count", C.c_uint32 * 3), ("rotations", C.c_void_p),
                ("n_rot", C.c_uint32), ("mode", C.c_uint32), ("noise", Noise),
                ("window", C.c_int32), ("select", C.c_uint32)]


SELECT_SAMPLE = 0
SELECT_ARGMAX = 1


class TrackSearch(C.Structure):
    """TrackSearch (tracking.hpp:25-34); defaults as the reference's."""
    _fields_ = [("pos_extent", C.c_double), ("angle_extent", C.c_double),
                ("points_per_dim", C.c_int32), ("refine_stages", C.c_int32),
                ("refine_factor", C.c_double), ("beam_width", C.c_int32),
                ("reserved", C.c_int32)]

    @classmethod
    def default(cls, **kw):
        d = dict(pos_extent=0.03, angle_extent=0.17453292519943295, points_per_dim=5,
                 refine_stages=2, refine_factor=3.0, beam_width=1, reserved=0)
        d.update(kw)
        return cls(**d)


class SmcObject(C.Structure):
    _fields_ = [("mesh_id", C.c_int32), ("reserved", C.c_int32),
                ("aabb_min", C.c_double * 3), ("aabb_max", C.c_double * 3)]


class ScheduleStage(C.Structure):
    _fields_ = [("n_dx", C.c_uint32), ("n_dy", C.c_uint32), ("n_dtheta", C.c_uint32)]


class SmcConfig(C.Structure):
    _fields_ = [("table_w", C.c_double), ("table_h", C.c_double), ("table_mesh", C.c_int32),
                ("n_refine", C.c_uint32), ("stage0", ScheduleStage),
                ("refine", C.c_void_p), ("noise_grid", C.c_void_p),
                ("n_noise_grid", C.c_uint32), ("n_objects", C.c_uint32),
                ("n_particles", C.c_uint32), ("resample_threshold", C.c_double),
                ("sigma_max", C.c_double), ("window", C.c_int32), ("prefactor", C.c_int32),
                ("renders", C.c_void_p)]


class SmcChild(C.Structure):
    _fields_ = [("object_id", C.c_int32), ("face", C.c_int32), ("dx", C.c_double),
                ("dy", C.c_double), ("dtheta", C.c_double)]


class SmcParticle(C.Structure):
    _fields_ = [("children", C.POINTER(SmcChild)), ("n_children", C.c_int32),
                ("noise_index", C.c_int32), ("log_target", C.c_double),
                ("log_weight", C.c_double)]


class ShardExchange(C.Structure):
    """b3d_shard_exchange: peer-mapped score arrays (2 x n_total x n_noise
    doubles each) and signal pads (n_ranks u64 each) of every rank."""
    _fields_ = [("n_ranks", C.c_uint32), ("rank", C.c_uint32), ("offset", C.c_uint64),
                ("n_total", C.c_uint64), ("scores", C.c_uint64 * 8), ("signals", C.c_uint64 * 8),
                ("epoch", C.c_uint64)]

    @classmethod
    def make(cls, rank, offset, n_total, score_ptrs, signal_ptrs, epoch):
        ex = cls()
        ex.n_ranks, ex.rank, ex.offset, ex.n_total = len(score_ptrs), rank, offset, n_total
        for r, (a, b) in enumerate(zip(score_ptrs, signal_ptrs)):
            ex.scores[r] = int(a)
            ex.signals[r] = int(b)
        ex.epoch = epoch
        return ex


class StageResult(C.Structure):
    _fields_ = [("argmax", C.c_uint64), ("sample", C.c_uint64), ("max_score", C.c_double),
                ("logsumexp", C.c_double), ("total", C.c_double), ("sample_logp", C.c_double),
                ("all_zero", C.c_uint32), ("n_nonfinite", C.c_uint32),
                ("sample_fallback", C.c_uint32), ("reserved", C.c_uint32)]


_lib = None


def lib() -> C.CDLL:
    """Loads libb3d_b200.so; raises if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} missing: run __graft_entry__.build() (no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    vp, st, u64, i32, u32, dbl = C.c_void_p, C.c_int, C.c_uint64, C.c_int32, C.c_uint32, C.c_double
    sig = {
        "b3d_version": ([], C.c_char_p),
        "b3d_last_error": ([], C.c_char_p),
        "b3d_depth_image_create": ([u32, u32, vp, C.POINTER(vp)], st),
        "b3d_depth_image_width": ([vp], u32),
        "b3d_depth_image_height": ([vp], u32),
        "b3d_depth_image_data": ([vp], vp),
        "b3d_depth_image_destroy": ([vp], None),
        "b3d_log_likelihood": ([vp, vp, C.POINTER(Intrinsics), dbl, dbl, dbl, st,
                                C.POINTER(dbl)], st),
        "b3d_gpu_context_create": ([st, C.POINTER(vp)], st),
        "b3d_gpu_context_destroy": ([vp], None),
        "b3d_gpu_set_stream": ([vp, vp], st),
        "b3d_gpu_synchronize": ([vp], st),
        "b3d_gpu_set_camera": ([vp, C.POINTER(Intrinsics), C.POINTER(Pose)], st),
        "b3d_gpu_upload_mesh": ([vp, vp, u64, vp, u64, C.POINTER(i32)], st),
        "b3d_gpu_set_observation": ([vp, vp], st),
        "b3d_gpu_set_culling": ([vp, st], st),
        "b3d_gpu_set_score_peers": ([vp, vp, u32, u64, u64], st),
        "b3d_gpu_shard_barrier": ([vp, vp, u32, u32, u64], st),
        "b3d_gpu_test_exchange_emulation": ([vp, u32, u32, C.c_int32, u64, vp], st),
        "b3d_gpu_enumerate_shard": ([vp, i32, vp, vp, vp, u64, C.POINTER(ShardExchange), vp, vp],
                                    st),
        "b3d_gpu_set_camera_scene": ([vp, vp, vp, u32], st),
        "b3d_gpu_render_cameras": ([vp, vp, u64, vp, vp], st),
        "b3d_gpu_score_cameras": ([vp, vp, u64, vp, vp], st),
        "b3d_gpu_track_camera": ([vp, vp, u32, C.POINTER(Pose), C.POINTER(TrackSearch), vp, vp],
                                 st),
        "b3d_camera_pose_from_spherical": ([dbl, dbl, dbl, C.POINTER(Pose)], st),
        "b3d_box_mesh": ([vp, vp, vp, vp], st),
        "b3d_depth_image_load": ([C.c_char_p, C.POINTER(vp)], st),
        "b3d_depth_image_save": ([vp, C.c_char_p], st),
        "b3d_model_from_voxels": ([vp, C.c_size_t, dbl, vp, st, C.POINTER(vp)], st),
        "b3d_model_load": ([C.c_char_p, st, C.POINTER(vp)], st),
        "b3d_model_save": ([vp, C.c_char_p], st),
        "b3d_model_bbox": ([vp, vp], st),
        "b3d_model_resolution": ([vp, C.POINTER(dbl)], st),
        "b3d_model_voxel_count": ([vp, C.POINTER(C.c_size_t)], st),
        "b3d_model_mesh": ([vp, C.POINTER(vp), C.POINTER(u64), C.POINTER(vp), C.POINTER(u64)],
                           st),
        "b3d_model_destroy": ([vp], None),
        "b3d_library_open": ([C.c_char_p, C.POINTER(vp)], st),
        "b3d_library_create": ([vp, C.c_size_t, C.POINTER(vp)], st),
        "b3d_library_size": ([vp], C.c_size_t),
        "b3d_library_destroy": ([vp], None),
        "b3d_scene_from_json": ([C.c_char_p, vp, C.POINTER(vp)], st),
        "b3d_scene_to_json": ([vp, C.POINTER(C.c_void_p)], st),
        "b3d_scene_destroy": ([vp], None),
        "b3d_string_free": ([C.c_void_p], None),
        "b3d_render": ([vp, C.POINTER(Pose), C.POINTER(Intrinsics), C.POINTER(vp)], st),
        "b3d_infer": ([vp, C.POINTER(Pose), vp, C.c_char_p, u64, C.POINTER(vp)], st),
        "b3d_particles_count": ([vp], C.c_size_t),
        "b3d_particles_log_evidence": ([vp, C.POINTER(dbl)], st),
        "b3d_particles_to_jsonl": ([vp, C.POINTER(C.c_void_p)], st),
        "b3d_particles_type_marginal": ([vp, vp, C.c_size_t], st),
        "b3d_particles_map_pose": ([vp, C.c_size_t, C.POINTER(Pose)], st),
        "b3d_particles_destroy": ([vp], None),
        "b3d_rotated_bounds": ([vp, vp, i32, vp, vp], st),
        "b3d_gpu_score_contact_cells": ([vp, i32, vp, vp, vp], st),
        "b3d_contact_cells_poses": ([vp, vp], st),
        "b3d_gpu_run_smc": ([vp, vp, u32, C.POINTER(SmcConfig), u64, vp, C.POINTER(dbl)], st),
        "b3d_contact_to_pose": ([dbl, dbl, vp, vp, i32, dbl, dbl, dbl, C.POINTER(Pose)], st),
        "b3d_camera_pose_to_spherical": ([C.POINTER(Pose), dbl, C.POINTER(dbl), C.POINTER(dbl),
                                          C.POINTER(dbl)], C.c_int),
        "b3d_mesh_cull_sign": ([vp, u64, vp, u64, C.POINTER(i32)], st),
        "b3d_gpu_mesh_cull_sign": ([vp, i32, C.POINTER(i32)], st),
        "b3d_gpu_set_likelihood": ([vp, C.POINTER(Noise), u32, dbl, st, st], st),
        "b3d_gpu_score_poses": ([vp, i32, vp, u64, vp, vp], st),
        "b3d_gpu_score_grid": ([vp, i32, C.POINTER(PoseGrid), vp, vp], st),
        "b3d_gpu_render_poses": ([vp, i32, vp, u64, vp, vp], st),
        "b3d_gpu_stage_reduce": ([vp, vp, u64, u32, u32, vp, vp, vp], st),
        "b3d_gpu_coarse_to_fine": ([vp, i32, C.POINTER(Pose), vp, u32, vp, vp, vp], st),
        "b3d_gpu_set_base_scene": ([vp, vp, vp, u32], st),
        "b3d_gpu_sample_many": ([vp, vp, u64, u32, u32, vp, u32, vp, vp], st),
        "b3d_gpu_enumerate_poses": ([vp, i32, vp, u64, vp, vp, vp], st),
        "b3d_gpu_enumerate_observed": ([vp, i32, vp, vp, u64, vp, vp, vp], st),
        "b3d_gpu_enumerate_grid": ([vp, i32, C.POINTER(PoseGrid), vp, vp, vp], st),
        "b3d_gpu_score_grid_range": ([vp, i32, C.POINTER(PoseGrid), u64, u64, vp, vp], st),
        "b3d_gpu_score_contact_grid": ([vp, i32, C.POINTER(ContactGrid), vp, vp], st),
        "b3d_contact_grid_poses": ([C.POINTER(ContactGrid), vp], st),
        "b3d_rng_seed": ([u64, vp], None),
        "b3d_rng_split": ([vp, u64, u64, u64, vp], None),
        "b3d_voxel_to_mesh": ([vp, u64, dbl, vp, vp, vp, C.POINTER(u64), C.POINTER(u64)], st),
        "b3d_gpu_voxel_to_mesh": ([vp, vp, u64, dbl, vp, vp, vp, C.POINTER(u64), C.POINTER(u64)],
                                  st),
        "b3d_sample_observation": ([C.POINTER(Intrinsics), vp, C.POINTER(Noise), vp, vp], st),
        "b3d_sample_observations": ([C.POINTER(Intrinsics), vp, u64, C.POINTER(Noise), vp, u64,
                                     vp], st),
    }
    for name, (args, res) in sig.items():
        if os.environ.get("B3D_LIB") and not hasattr(L, name):
            continue  # same-box A/B against an older build (scripts/gpu_ablib.sh)
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    _lib = L
    return L


def exported_symbols() -> Sequence[str]:
    """Every function include/b3d_b200.h declares (B3D_API)."""
    import re
    hdr = open(os.path.join(_HERE, os.pardir, "include", "b3d_b200.h")).read()
    return re.findall(r"B3D_API[^;]*?\b(b3d_\w+)\s*\(", hdr, flags=re.S)


def _check(status: int) -> None:
    if status != B3D_OK:
        raise B3DError(status, lib().b3d_last_error().decode())


def _ptr(a) -> int:
    """Raw address of a numpy array (host) or a torch tensor (host/device)."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    if isinstance(a, np.ndarray):
        if not a.flags.c_contiguous:
            raise ValueError("arrays must be C-contiguous")
        if a.flags.writeable and a.size:
            # ~0.4 us instead of ~1.3 us for a.ctypes.data (a per-call cost on
            # the end-to-end path, four pointers per stage)
            return C.addressof(C.c_char.from_buffer(a))
        return a.ctypes.data
    raise TypeError(f"unsupported buffer type {type(a)}")


def _pose(p) -> Pose:
    p = np.asarray(p, dtype=np.float64).reshape(7)
    return Pose(*p.tolist())


def rng_seed(seed: int) -> np.ndarray:
    st = np.zeros(5, dtype=np.uint64)
    lib().b3d_rng_seed(C.c_uint64(seed), st.ctypes.data)
    return st


def rng_split(state: np.ndarray, k0: int, k1: int = 0, k2: int = 0) -> np.ndarray:
    out = np.zeros(5, dtype=np.uint64)
    lib().b3d_rng_split(state.ctypes.data, k0, k1, k2, out.ctypes.data)
    return out


def sample_observation(k: Intrinsics, rendered: np.ndarray, p_outlier: float, sigma: float,
                       rng_state: np.ndarray) -> np.ndarray:
    """The reference's sample_observation (likelihood.cpp:44-80): a synthetic
    observed depth image from a rendered one; rng_state (5 x uint64) is
    advanced in place, as the reference's Rng& is."""
    r = np.ascontiguousarray(rendered, dtype=np.float32)
    assert r.shape == (k.height, k.width)
    assert rng_state.dtype == np.uint64 and rng_state.flags.c_contiguous
    out = np.empty_like(r)
    nz = Noise(p_outlier, sigma)
    _check(lib().b3d_sample_observation(C.byref(k), r.ctypes.data, C.byref(nz),
                                        rng_state.ctypes.data, out.ctypes.data))
    return out


def sample_observations(k: Intrinsics, rendered: np.ndarray, p_outlier: float, sigma: float,
                        rng_state: np.ndarray, split_key: int = 0x0F) -> np.ndarray:
    """Frames of generate_orbit_sequence (tracking.cpp:199-202): frame i is
    sample_observation(rendered[i]) with rng_state.split(split_key, i); all host
    threads."""
    r = np.ascontiguousarray(rendered, dtype=np.float32)
    assert r.ndim == 3 and r.shape[1:] == (k.height, k.width)
    st = np.ascontiguousarray(rng_state, dtype=np.uint64)
    out = np.empty_like(r)
    nz = Noise(p_outlier, sigma)
    _check(lib().b3d_sample_observations(C.byref(k), r.ctypes.data, r.shape[0], C.byref(nz),
                                         st.ctypes.data, split_key, out.ctypes.data))
    return out


def voxel_to_mesh(voxels: np.ndarray, resolution: float, origin) -> tuple:
    v = np.ascontiguousarray(voxels, dtype=np.int32)
    n = v.shape[0]
    verts = np.zeros((8 * n, 3), dtype=np.float64)
    tris = np.zeros((12 * n, 3), dtype=np.uint32)
    o = np.ascontiguousarray(origin, dtype=np.float64)
    nv, nt = C.c_uint64(), C.c_uint64()
    _check(lib().b3d_voxel_to_mesh(v.ctypes.data, n, resolution, o.ctypes.data,
                                   verts.ctypes.data, tris.ctypes.data, C.byref(nv), C.byref(nt)))
    return verts[: nv.value].copy(), tris[: nt.value].copy()


def mesh_cull_sign(vertices: np.ndarray, triangles: np.ndarray) -> int:
    """+1 / -1: closed mesh wound outward / inward (back faces may be culled in
    score-many); 0: not closed."""
    v = np.ascontiguousarray(vertices, dtype=np.float64)
    t = np.ascontiguousarray(triangles, dtype=np.uint32)
    out = C.c_int32()
    _check(lib().b3d_mesh_cull_sign(v.ctypes.data, v.shape[0], t.ctypes.data, t.shape[0],
                                    C.byref(out)))
    return out.value


# ---- the reference's handle API (b3d.h), thin Python wrappers --------------
def _owned_string(fn, *args) -> str:
    out = C.c_void_p()
    _check(fn(*args, C.byref(out)))
    try:
        return C.cast(out, C.c_char_p).value.decode()
    finally:
        lib().b3d_string_free(out)


class Model:
    """b3d_object_model handle."""

    def __init__(self, handle):
        self.h = handle

    @classmethod
    def from_voxels(cls, voxels, resolution, origin, id_=0):
        v = np.ascontiguousarray(voxels, dtype=np.int32)
        o = np.ascontiguousarray(origin, dtype=np.float64)
        h = C.c_void_p()
        _check(lib().b3d_model_from_voxels(v.ctypes.data, v.shape[0], resolution, o.ctypes.data,
                                           id_, C.byref(h)))
        return cls(h)

    @classmethod
    def load(cls, path, id_=0):
        h = C.c_void_p()
        _check(lib().b3d_model_load(str(path).encode(), id_, C.byref(h)))
        return cls(h)

    def save(self, path):
        _check(lib().b3d_model_save(self.h, str(path).encode()))

    def bbox(self):
        e = np.zeros(3)
        _check(lib().b3d_model_bbox(self.h, e.ctypes.data))
        return e

    def resolution(self):
        r = C.c_double()
        _check(lib().b3d_model_resolution(self.h, C.byref(r)))
        return r.value

    def voxel_count(self):
        n = C.c_size_t()
        _check(lib().b3d_model_voxel_count(self.h, C.byref(n)))
        return n.value

    def mesh(self):
        vp_, tp_, nv, nt = C.c_void_p(), C.c_void_p(), C.c_uint64(), C.c_uint64()
        _check(lib().b3d_model_mesh(self.h, C.byref(vp_), C.byref(nv), C.byref(tp_), C.byref(nt)))
        v = np.ctypeslib.as_array(C.cast(vp_, C.POINTER(C.c_double)), (nv.value, 3)).copy()
        t = np.ctypeslib.as_array(C.cast(tp_, C.POINTER(C.c_uint32)), (nt.value, 3)).copy()
        return v, t

    def __del__(self):
        try:
            lib().b3d_model_destroy(self.h)
        except Exception:
            pass


class Library:
    def __init__(self, handle):
        self.h = handle

    @classmethod
    def create(cls, models):
        arr = (C.c_void_p * len(models))(*[m.h.value for m in models])
        h = C.c_void_p()
        _check(lib().b3d_library_create(arr, len(models), C.byref(h)))
        return cls(h)

    @classmethod
    def open(cls, manifest):
        h = C.c_void_p()
        _check(lib().b3d_library_open(str(manifest).encode(), C.byref(h)))
        return cls(h)

    def __len__(self):
        return lib().b3d_library_size(self.h)

    def __del__(self):
        try:
            lib().b3d_library_destroy(self.h)
        except Exception:
            pass


class Scene:
    def __init__(self, handle):
        self.h = handle

    @classmethod
    def from_json(cls, text, library):
        h = C.c_void_p()
        _check(lib().b3d_scene_from_json(text.encode(), library.h, C.byref(h)))
        return cls(h)

    def to_json(self) -> str:
        return _owned_string(lib().b3d_scene_to_json, self.h)

    def __del__(self):
        try:
            lib().b3d_scene_destroy(self.h)
        except Exception:
            pass


def _image_from_handle(h) -> np.ndarray:
    L = lib()
    w, hh = L.b3d_depth_image_width(h), L.b3d_depth_image_height(h)
    d = np.ctypeslib.as_array(C.cast(L.b3d_depth_image_data(h), C.POINTER(C.c_float)),
                              (hh, w)).copy()
    L.b3d_depth_image_destroy(h)
    return d


def _image_handle(depth: np.ndarray):
    d = np.ascontiguousarray(depth, dtype=np.float32)
    h = C.c_void_p()
    _check(lib().b3d_depth_image_create(d.shape[1], d.shape[0], d.ctypes.data, C.byref(h)))
    return h


def depth_image_save(depth: np.ndarray, path):
    h = _image_handle(depth)
    try:
        _check(lib().b3d_depth_image_save(h, str(path).encode()))
    finally:
        lib().b3d_depth_image_destroy(h)


def depth_image_load(path) -> np.ndarray:
    h = C.c_void_p()
    _check(lib().b3d_depth_image_load(str(path).encode(), C.byref(h)))
    return _image_from_handle(h)


def render(scene: Scene, camera, k: Intrinsics) -> np.ndarray:
    """b3d_render (reference b3d.h:107-108), device-backed."""
    h = C.c_void_p()
    _check(lib().b3d_render(scene.h, C.byref(_pose(camera)), C.byref(k), C.byref(h)))
    return _image_from_handle(h)


def infer(observed: np.ndarray, camera, library: Library, config_json: str, seed: int):
    """b3d_infer (reference b3d.h:121-124): returns (jsonl lines, log_evidence,
    type marginal or None, map pose of child 0)."""
    L = lib()
    img = _image_handle(observed)
    p = C.c_void_p()
    try:
        _check(L.b3d_infer(img, C.byref(_pose(camera)), library.h, config_json.encode(), seed,
                           C.byref(p)))
    finally:
        L.b3d_depth_image_destroy(img)
    try:
        lines = _owned_string(L.b3d_particles_to_jsonl, p).strip().splitlines()
        le = C.c_double()
        _check(L.b3d_particles_log_evidence(p, C.byref(le)))
        marg = np.zeros(len(library))
        st = L.b3d_particles_type_marginal(p, marg.ctypes.data, len(marg))
        pose = Pose()
        _check(L.b3d_particles_map_pose(p, 0, C.byref(pose)))
        return (lines, le.value, marg if st == B3D_OK else None,
                np.array([getattr(pose, n) for n, _ in Pose._fields_]))
    finally:
        L.b3d_particles_destroy(p)


def rotated_bounds(aabb_min, aabb_max, face):
    """rotated_bounds (scene_graph.cpp:73-89): AABB with `face` down."""
    lo_a = np.ascontiguousarray(aabb_min, dtype=np.float64)
    hi_a = np.ascontiguousarray(aabb_max, dtype=np.float64)
    lo, hi = np.zeros(3), np.zeros(3)
    _check(lib().b3d_rotated_bounds(lo_a.ctypes.data, hi_a.ctypes.data, face, lo.ctypes.data,
                                    hi.ctypes.data))
    return lo, hi


def box_mesh(lo, hi):
    """make_box_mesh (scene_graph.cpp:37-58)."""
    lo_a = np.ascontiguousarray(lo, dtype=np.float64)
    hi_a = np.ascontiguousarray(hi, dtype=np.float64)
    v = np.zeros((8, 3), dtype=np.float64)
    t = np.zeros((12, 3), dtype=np.uint32)
    _check(lib().b3d_box_mesh(lo_a.ctypes.data, hi_a.ctypes.data, v.ctypes.data, t.ctypes.data))
    return v, t


def contact_to_pose(table_w, table_h, aabb_min, aabb_max, face, dx, dy, dtheta) -> np.ndarray:
    """contact_to_pose (scene_graph.cpp:97-121) on the host."""
    lo_a = np.ascontiguousarray(aabb_min, dtype=np.float64)
    hi_a = np.ascontiguousarray(aabb_max, dtype=np.float64)
    out = Pose()
    _check(lib().b3d_contact_to_pose(table_w, table_h, lo_a.ctypes.data, hi_a.ctypes.data, face,
                                     dx, dy, dtheta, C.byref(out)))
    return np.array([getattr(out, n) for n, _ in Pose._fields_])


def camera_pose_from_spherical(distance: float, azimuth: float, altitude: float) -> np.ndarray:
    """generative.cpp:35-59 on the host (the product's libm path)."""
    out = Pose()
    _check(lib().b3d_camera_pose_from_spherical(distance, azimuth, altitude, C.byref(out)))
    return np.array([getattr(out, n) for n, _ in Pose._fields_])


def camera_pose_to_spherical(pose, tol: float = 1e-6):
    """generative.cpp:61-85: (distance, azimuth, altitude) or None."""
    d, a, h = C.c_double(), C.c_double(), C.c_double()
    ok = lib().b3d_camera_pose_to_spherical(C.byref(_pose(pose)), tol, C.byref(d), C.byref(a),
                                            C.byref(h))
    return (d.value, a.value, h.value) if ok else None


def contact_grid_poses(grid: "ContactGrid") -> np.ndarray:
    """Host model-to-world poses of a table-contact grid (b3d_contact_grid_poses)."""
    out = np.zeros((grid.n, 7), dtype=np.float64)
    _check(lib().b3d_contact_grid_poses(C.byref(grid), out.ctypes.data))
    return out


def log_likelihood(observed: np.ndarray, rendered: np.ndarray, k: Intrinsics, p_outlier: float,
                   sigma_noise: float, sigma_max: float, window: int) -> float:
    """b3d_log_likelihood (reference b3d.h:110-115), GPU-backed."""
    L = lib()
    o, r = C.c_void_p(), C.c_void_p()
    obs = np.ascontiguousarray(observed, dtype=np.float32)
    ren = np.ascontiguousarray(rendered, dtype=np.float32)
    _check(L.b3d_depth_image_create(obs.shape[1], obs.shape[0], obs.ctypes.data, C.byref(o)))
    try:
        _check(L.b3d_depth_image_create(ren.shape[1], ren.shape[0], ren.ctypes.data, C.byref(r)))
        try:
            out = C.c_double()
            _check(L.b3d_log_likelihood(o, r, C.byref(k), p_outlier, sigma_noise, sigma_max,
                                        window, C.byref(out)))
            return out.value
        finally:
            L.b3d_depth_image_destroy(r)
    finally:
        L.b3d_depth_image_destroy(o)


@dataclass
class StageOut:
    argmax: int
    sample: int
    max_score: float
    logsumexp: float
    total: float
    sample_logp: float
    all_zero: bool
    n_nonfinite: int
    sample_fallback: bool


class GpuContext:
    """Owns a b3d_gpu_context (device, stream, meshes, observation)."""

    def __init__(self, device: int = 0):
        self._L = lib()
        h = C.c_void_p()
        _check(self._L.b3d_gpu_context_create(device, C.byref(h)))
        self.h = h
        self.device = device
        self.k: Optional[Intrinsics] = None
        self.n_noise = 0

    def close(self):
        if self.h:
            self._L.b3d_gpu_context_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream_handle: int | None):
        _check(self._L.b3d_gpu_set_stream(self.h, stream_handle))

    def synchronize(self):
        _check(self._L.b3d_gpu_synchronize(self.h))

    def set_camera(self, k: Intrinsics, camera=None):
        self.k = k
        _check(self._L.b3d_gpu_set_camera(self.h, C.byref(k),
                                          C.byref(_pose(camera)) if camera is not None else None))

    def upload_mesh(self, vertices: np.ndarray, triangles: np.ndarray) -> int:
        v = np.ascontiguousarray(vertices, dtype=np.float64)
        t = np.ascontiguousarray(triangles, dtype=np.uint32)
        mid = C.c_int32()
        _check(self._L.b3d_gpu_upload_mesh(self.h, v.ctypes.data, v.shape[0], t.ctypes.data,
                                           t.shape[0], C.byref(mid)))
        return mid.value

    def voxel_to_mesh(self, voxels, resolution: float, origin) -> tuple:
        """b3d_gpu_voxel_to_mesh: voxels (n,3) int32 numpy or torch (host/device);
        returns host numpy (vertices, triangles) for numpy input, device torch
        tensors for a device tensor."""
        o = np.ascontiguousarray(origin, dtype=np.float64)
        nv, nt = C.c_uint64(), C.c_uint64()
        if isinstance(voxels, np.ndarray):
            v = np.ascontiguousarray(voxels, dtype=np.int32)
            n = v.shape[0]
            verts = np.zeros((8 * n, 3), dtype=np.float64)
            tris = np.zeros((12 * n, 3), dtype=np.uint32)
        else:
            import torch
            v = voxels.contiguous()
            n = v.shape[0]
            verts = torch.empty((8 * n, 3), dtype=torch.float64, device=v.device)
            tris = torch.empty((12 * n, 3), dtype=torch.int32, device=v.device)
        _check(self._L.b3d_gpu_voxel_to_mesh(self.h, _ptr(v), n, resolution, o.ctypes.data,
                                             _ptr(verts), _ptr(tris), C.byref(nv), C.byref(nt)))
        return verts[: nv.value], tris[: nt.value]

    def set_score_peers(self, peer_ptrs, offset: int, capacity: int = 0):
        """Fused all-gather targets (b3d_gpu_set_score_peers): score (h, e) also
        goes to peer[(offset + h) * n_noise + e] below `capacity` elements;
        [] turns it off."""
        arr = (C.c_uint64 * max(1, len(peer_ptrs)))(*[int(x) for x in peer_ptrs])
        _check(self._L.b3d_gpu_set_score_peers(self.h, arr, len(peer_ptrs), offset, capacity))

    def shard_barrier(self, signal_ptrs, rank: int, epoch: int):
        """b3d_gpu_shard_barrier over the ranks' signal pads."""
        arr = (C.c_uint64 * max(1, len(signal_ptrs)))(*[int(x) for x in signal_ptrs])
        _check(self._L.b3d_gpu_shard_barrier(self.h, arr, len(signal_ptrs), rank, epoch))

    def exchange_emulation(self, n_ranks: int, rounds: int, double_buffered: bool = True,
                           hold_ns: int = 50_000) -> int:
        """b3d_gpu_test_exchange_emulation: the exchange protocol for n_ranks
        ranks emulated in one cooperative launch; returns the stale reads."""
        err = C.c_uint32()
        _check(self._L.b3d_gpu_test_exchange_emulation(self.h, n_ranks, rounds,
                                                       1 if double_buffered else 0, hold_ns,
                                                       C.byref(err)))
        return err.value

    def enumerate_shard(self, mesh: int, ex: "ShardExchange", poses=None, grid=None, depth=None,
                        n_local: int = None, rng_state=None, out=None):
        """b3d_gpu_enumerate_shard: [observation], this rank's shard scored into
        every rank's array, barrier, stage reduction of the whole array.
        Returns a StageOut (host out) or None (device out)."""
        if isinstance(depth, np.ndarray):
            depth = np.ascontiguousarray(depth, dtype=np.float32)
        if isinstance(poses, np.ndarray):
            poses = np.ascontiguousarray(poses, dtype=np.float64)
        if n_local is None:
            n_local = poses.shape[0]
        res = StageResult() if out is None else None
        _check(self._L.b3d_gpu_enumerate_shard(
            self.h, mesh, _ptr(depth), _ptr(poses), C.byref(grid) if grid is not None else None,
            n_local, C.byref(ex), _ptr(rng_state),
            _ptr(out) if out is not None else C.addressof(res)))
        if res is None:
            return None
        return StageOut(res.argmax, res.sample, res.max_score, res.logsumexp, res.total,
                        res.sample_logp, bool(res.all_zero), res.n_nonfinite,
                        bool(res.sample_fallback))

    def set_culling(self, enable: bool):
        _check(self._L.b3d_gpu_set_culling(self.h, 1 if enable else 0))

    def mesh_cull_sign(self, mesh: int) -> int:
        out = C.c_int32()
        _check(self._L.b3d_gpu_mesh_cull_sign(self.h, mesh, C.byref(out)))
        return out.value

    def set_observation(self, depth):
        if isinstance(depth, np.ndarray):
            depth = np.ascontiguousarray(depth, dtype=np.float32)
        _check(self._L.b3d_gpu_set_observation(self.h, _ptr(depth)))

    def set_likelihood(self, noise: Sequence[tuple], sigma_max: float, window: int,
                       prefactor: int = PREFACTOR_PRINTED):
        arr = (Noise * len(noise))(*[Noise(p, s) for p, s in noise])
        _check(self._L.b3d_gpu_set_likelihood(self.h, arr, len(noise), sigma_max, window,
                                              prefactor))
        self.n_noise = len(noise)

    def score_poses(self, mesh: int, poses, scores=None, status=None):
        """poses: (n,7) float64 numpy (host) or torch tensor (host/device)."""
        n = poses.shape[0]
        host = isinstance(poses, np.ndarray)
        if host:
            poses = np.ascontiguousarray(poses, dtype=np.float64)
        if scores is None:
            scores = np.zeros((n, self.n_noise), dtype=np.float64)
            status = np.zeros(n, dtype=np.uint8) if status is None else status
        _check(self._L.b3d_gpu_score_poses(self.h, mesh, _ptr(poses), n, _ptr(scores),
                                           _ptr(status)))
        return scores, status

    def make_grid(self, center, extent, count, rotations, mode=GRID_ZIP) -> PoseGrid:
        g = PoseGrid()
        g.center = _pose(center)
        for a in range(3):
            g.extent[a] = float(extent[a])
            g.count[a] = int(count[a])
        g.rotations = _ptr(rotations)
        g.n_rot = rotations.shape[0]
        g.mode = mode
        g._keep = rotations  # keep the buffer alive
        return g

    @staticmethod
    def grid_size(g: PoseGrid) -> int:
        nt = g.count[0] * g.count[1] * g.count[2]
        return nt * g.n_rot if g.mode == GRID_PRODUCT else nt

    def score_grid(self, mesh: int, grid: PoseGrid, scores=None, status=None):
        n = self.grid_size(grid)
        if scores is None:
            scores = np.zeros((n, self.n_noise), dtype=np.float64)
            status = np.zeros(n, dtype=np.uint8) if status is None else status
        _check(self._L.b3d_gpu_score_grid(self.h, mesh, C.byref(grid), _ptr(scores),
                                          _ptr(status)))
        return scores, status

    def enumerate_grid(self, mesh: int, grid: PoseGrid, rng_state, out, scores):
        """score_grid + stage reduction fused into one launch
        (b3d_gpu_enumerate_grid); device tensors only, asynchronous."""
        _check(self._L.b3d_gpu_enumerate_grid(self.h, mesh, C.byref(grid), _ptr(rng_state),
                                              _ptr(out), _ptr(scores)))

    def render_poses(self, mesh: int, poses, with_ids: bool = True):
        n = poses.shape[0]
        poses = np.ascontiguousarray(poses, dtype=np.float64)
        H, W = self.k.height, self.k.width
        depth = np.zeros((n, H, W), dtype=np.float32)
        ids = np.zeros((n, H, W), dtype=np.int32) if with_ids else None
        _check(self._L.b3d_gpu_render_poses(self.h, mesh, poses.ctypes.data, n,
                                            depth.ctypes.data, _ptr(ids)))
        return depth, ids

    def stage_reduce(self, scores, n=None, stride=1, col=0, rng_state=None, probs=None,
                     out=None):
        if n is None:
            n = scores.shape[0]
        if isinstance(scores, np.ndarray):
            scores = np.ascontiguousarray(scores, dtype=np.float64)
        res = StageResult() if out is None else None
        _check(self._L.b3d_gpu_stage_reduce(self.h, _ptr(scores), n, stride, col,
                                            _ptr(rng_state), _ptr(out) if out is not None
                                            else C.addressof(res), _ptr(probs)))
        if res is None:
            return None
        return StageOut(res.argmax, res.sample, res.max_score, res.logsumexp, res.total,
                        res.sample_logp, bool(res.all_zero), res.n_nonfinite,
                        bool(res.sample_fallback))

    def coarse_to_fine(self, mesh: int, center, stages: Sequence[dict], rng_state=None):
        """b3d_gpu_coarse_to_fine.  stages: dicts with extent, count,
        rotations (n,4), mode, noise (p, sigma), window, select.
        Returns (list of StageOut, centers (n_stages+1, 7))."""
        specs = (StageSpec * len(stages))()
        keep = []
        for i, g in enumerate(stages):
            rot = np.ascontiguousarray(g["rotations"], dtype=np.float64)
            keep.append(rot)
            sp = specs[i]
            for a in range(3):
                sp.extent[a] = float(g["extent"][a])
                sp.count[a] = int(g["count"][a])
            sp.rotations = rot.ctypes.data
            sp.n_rot = rot.shape[0]
            sp.mode = int(g.get("mode", GRID_PRODUCT))
            sp.noise = Noise(*g["noise"])
            sp.window = int(g["window"])
            sp.select = int(g.get("select", SELECT_SAMPLE))
        res = (StageResult * len(stages))()
        centers = np.zeros((len(stages) + 1, 7), dtype=np.float64)
        c = _pose(center)
        _check(self._L.b3d_gpu_coarse_to_fine(self.h, mesh, C.byref(c), specs, len(stages),
                                              _ptr(rng_state), C.addressof(res),
                                              centers.ctypes.data))
        outs = [StageOut(r.argmax, r.sample, r.max_score, r.logsumexp, r.total, r.sample_logp,
                         bool(r.all_zero), r.n_nonfinite, bool(r.sample_fallback)) for r in res]
        return outs, centers

    def set_camera_scene(self, mesh_ids: Sequence[int], poses):
        """Instances (draw order) rendered under camera hypotheses
        (b3d_gpu_set_camera_scene); poses are model-to-world."""
        ids = np.ascontiguousarray(mesh_ids, dtype=np.int32)
        P = np.ascontiguousarray(poses, dtype=np.float64).reshape(-1, 7)
        _check(self._L.b3d_gpu_set_camera_scene(self.h, ids.ctypes.data, P.ctypes.data, len(ids)))

    def render_cameras(self, cameras, with_ids: bool = True):
        cams = np.ascontiguousarray(cameras, dtype=np.float64).reshape(-1, 7)
        n = cams.shape[0]
        H, W = self.k.height, self.k.width
        depth = np.zeros((n, H, W), dtype=np.float32)
        ids = np.zeros((n, H, W), dtype=np.int32) if with_ids else None
        _check(self._L.b3d_gpu_render_cameras(self.h, cams.ctypes.data, n, depth.ctypes.data,
                                              _ptr(ids)))
        return depth, ids

    def score_cameras(self, cameras):
        cams = np.ascontiguousarray(cameras, dtype=np.float64).reshape(-1, 7)
        n = cams.shape[0]
        scores = np.zeros((n, self.n_noise), dtype=np.float64)
        status = np.zeros(n, dtype=np.uint8)
        _check(self._L.b3d_gpu_score_cameras(self.h, cams.ctypes.data, n, scores.ctypes.data,
                                             status.ctypes.data))
        return scores, status

    def track_camera(self, frames, initial, search: "TrackSearch" = None):
        """track_camera (tracking.cpp:59-172): camera poses per frame and the
        per-frame wall time in ms."""
        fr = frames if not isinstance(frames, np.ndarray) else \
            np.ascontiguousarray(frames, dtype=np.float32)
        n = fr.shape[0]
        poses = np.zeros((n, 7), dtype=np.float64)
        ms = np.zeros(n, dtype=np.float64)
        search = search or TrackSearch.default()
        _check(self._L.b3d_gpu_track_camera(self.h, _ptr(fr), n, C.byref(_pose(initial)),
                                            C.byref(search), poses.ctypes.data, ms.ctypes.data))
        return poses, ms

    def run_smc(self, library, table_mesh: int, table_w: float, table_h: float, schedule,
                noise_grid, sigma_max: float, window: int, n_objects: int, n_particles: int,
                resample_threshold: float, seed: int, prefactor: int = PREFACTOR_PRINTED):
        """run_smc (inference.cpp:398-520) with device scoring (b3d_gpu_run_smc).
        library: [(mesh_id, aabb_min, aabb_max)]; schedule: (stage0 (nx, ny, nt),
        [refine ...]).  Returns ([(children [(obj, face, dx, dy, dtheta)],
        noise_index, log_target, log_weight)], log_evidence)."""
        libs = (SmcObject * len(library))()
        for i, (mid, lo, hi) in enumerate(library):
            libs[i].mesh_id = mid
            for a in range(3):
                libs[i].aabb_min[a] = float(lo[a])
                libs[i].aabb_max[a] = float(hi[a])
        nz = (Noise * len(noise_grid))(*[Noise(p, s) for p, s in noise_grid])
        cfg = SmcConfig()
        cfg.table_w, cfg.table_h, cfg.table_mesh = table_w, table_h, table_mesh
        cfg.stage0 = ScheduleStage(*schedule[0])
        cfg.n_refine = len(schedule[1])
        refine = (ScheduleStage * max(1, len(schedule[1])))(*[ScheduleStage(*st)
                                                               for st in schedule[1]])
        cfg.refine = C.cast(refine, C.c_void_p)
        cfg.noise_grid = C.cast(nz, C.c_void_p)
        cfg.n_noise_grid = len(noise_grid)
        cfg.n_objects, cfg.n_particles = n_objects, n_particles
        cfg.resample_threshold, cfg.sigma_max = resample_threshold, sigma_max
        cfg.window, cfg.prefactor = window, prefactor
        renders = C.c_uint64()
        cfg.renders = C.cast(C.byref(renders), C.c_void_p)
        out = (SmcParticle * n_particles)()
        kids = (SmcChild * (n_particles * max(1, n_objects)))()
        for i in range(n_particles):
            out[i].children = C.cast(C.byref(kids, i * max(1, n_objects) * C.sizeof(SmcChild)),
                                     C.POINTER(SmcChild))
        le = C.c_double()
        _check(self._L.b3d_gpu_run_smc(self.h, libs, len(library), C.byref(cfg), seed, out,
                                       C.byref(le)))
        ps = []
        for p in out:
            ch = [(c.object_id, c.face, c.dx, c.dy, c.dtheta)
                  for c in p.children[:p.n_children]]
            ps.append((ch, p.noise_index, p.log_target, p.log_weight))
        self.last_smc_renders = renders.value  # device evaluations of that run
        return ps, le.value

    def set_base_scene(self, mesh_ids: Sequence[int], poses):
        """Fixed instances (table first, then base children) rendered once and
        composited under every hypothesis (b3d_gpu_set_base_scene)."""
        ids = np.ascontiguousarray(mesh_ids, dtype=np.int32)
        P = np.ascontiguousarray(poses, dtype=np.float64).reshape(-1, 7)
        _check(self._L.b3d_gpu_set_base_scene(self.h, ids.ctypes.data if len(ids) else None,
                                              P.ctypes.data if len(ids) else None, len(ids)))

    def score_contact_grid(self, mesh: int, grid: "ContactGrid", scores=None, status=None):
        n = grid.n
        if scores is None:
            scores = np.zeros((n, self.n_noise), dtype=np.float64)
            status = np.zeros(n, dtype=np.uint8) if status is None else status
        _check(self._L.b3d_gpu_score_contact_grid(self.h, mesh, C.byref(grid), _ptr(scores),
                                                  _ptr(status)))
        return scores, status

    def sample_many(self, scores, n_samples: int, rng_state, n=None, stride=1, col=0,
                    samples=None):
        """n_samples posterior draws (b3d_gpu_sample_many); returns (samples, StageOut)."""
        if n is None:
            n = scores.shape[0]
        if isinstance(scores, np.ndarray):
            scores = np.ascontiguousarray(scores, dtype=np.float64)
        if samples is None:
            samples = np.zeros(n_samples, dtype=np.uint64)
        res = StageResult()
        _check(self._L.b3d_gpu_sample_many(self.h, _ptr(scores), n, stride, col, _ptr(rng_state),
                                           n_samples, _ptr(samples), C.addressof(res)))
        return samples, StageOut(res.argmax, res.sample, res.max_score, res.logsumexp, res.total,
                                 res.sample_logp, bool(res.all_zero), res.n_nonfinite,
                                 bool(res.sample_fallback))

    def score_grid_range(self, mesh: int, grid: PoseGrid, first: int, n: int, scores=None,
                         status=None):
        if scores is None:
            scores = np.zeros((n, self.n_noise), dtype=np.float64)
            status = np.zeros(n, dtype=np.uint8) if status is None else status
        _check(self._L.b3d_gpu_score_grid_range(self.h, mesh, C.byref(grid), first, n,
                                                _ptr(scores), _ptr(status)))
        return scores, status

    def enumerate_observed(self, mesh: int, depth, poses, rng_state=None,
                           scores=None) -> "StageOut":
        """b3d_gpu_enumerate_observed: set_observation + enumerate_poses in one call."""
        if isinstance(depth, np.ndarray):
            depth = np.ascontiguousarray(depth, dtype=np.float32)
        if isinstance(poses, np.ndarray):
            poses = np.ascontiguousarray(poses, dtype=np.float64)
        res = StageResult()
        _check(self._L.b3d_gpu_enumerate_observed(self.h, mesh, _ptr(depth), _ptr(poses),
                                                  poses.shape[0], _ptr(rng_state),
                                                  C.addressof(res), _ptr(scores)))
        return StageOut(res.argmax, res.sample, res.max_score, res.logsumexp, res.total,
                        res.sample_logp, bool(res.all_zero), res.n_nonfinite,
                        bool(res.sample_fallback))

    def enumerate_poses(self, mesh: int, poses, rng_state=None, scores=None) -> "StageOut":
        """b3d_gpu_enumerate_poses: score-many + stage reduce in one call."""
        if isinstance(poses, np.ndarray):
            poses = np.ascontiguousarray(poses, dtype=np.float64)
        res = StageResult()
        _check(self._L.b3d_gpu_enumerate_poses(self.h, mesh, _ptr(poses), poses.shape[0],
                                               _ptr(rng_state), C.addressof(res), _ptr(scores)))
        return StageOut(res.argmax, res.sample, res.max_score, res.logsumexp, res.total,
                        res.sample_logp, bool(res.all_zero), res.n_nonfinite,
                        bool(res.sample_fallback))
