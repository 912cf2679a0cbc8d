"""Boundary cases of the reference C ABI (b3d.h), run identically against any
library exporting it: the reference's own (oracle/_ref/libb3d_ref.so, to make
tests/golden/ref_capi.json) and the product's (libb3d_b200.so, checked
against that fixture in tests/test_capi_reference.py).

Each case returns (status, message) -- or a value -- so a drop-in caller sees
the same codes and the same thread-local error text for the same misuse:
bad arguments, invalid intrinsics / noise, dimension mismatches, SDPT / SVOX
format errors, manifest and scene-JSON errors, and the `infer` config schema
(b3d_capi.cpp:22-48, 297-379).  Cases marked gpu need the product's device
work to be reached (the empty-render checks come after a device count).
"""
from __future__ import annotations

import ctypes as C
import hashlib
import json
import os
import struct
import tempfile

import numpy as np

vp = C.c_void_p


class Intr(C.Structure):
    _fields_ = [("fx", C.c_double), ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("width", C.c_uint32), ("height", C.c_uint32),
                ("near_m", C.c_double), ("far_m", C.c_double)]


class Pose(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("qw", "qx", "qy", "qz", "tx", "ty", "tz")]


def _sig(L):
    L.b3d_last_error.restype = C.c_char_p
    L.b3d_depth_image_create.argtypes = [C.c_uint32, C.c_uint32, vp, C.POINTER(vp)]
    L.b3d_depth_image_load.argtypes = [C.c_char_p, C.POINTER(vp)]
    L.b3d_log_likelihood.argtypes = [vp, vp, C.POINTER(Intr), C.c_double, C.c_double, C.c_double,
                                     C.c_int, C.POINTER(C.c_double)]
    L.b3d_model_load.argtypes = [C.c_char_p, C.c_int, C.POINTER(vp)]
    L.b3d_library_open.argtypes = [C.c_char_p, C.POINTER(vp)]
    L.b3d_scene_from_json.argtypes = [C.c_char_p, vp, C.POINTER(vp)]
    L.b3d_render.argtypes = [vp, C.POINTER(Pose), C.POINTER(Intr), C.POINTER(vp)]
    L.b3d_infer.argtypes = [vp, C.POINTER(Pose), vp, C.c_char_p, C.c_uint64, C.POINTER(vp)]
    L.b3d_depth_image_destroy.argtypes = [vp]
    L.b3d_depth_image_data.argtypes = [vp]
    L.b3d_depth_image_data.restype = C.POINTER(C.c_float)
    L.b3d_particles_log_evidence.argtypes = [vp, C.POINTER(C.c_double)]
    L.b3d_particles_to_jsonl.argtypes = [vp, C.POINTER(C.c_void_p)]
    L.b3d_string_free.argtypes = [vp]
    L.b3d_particles_type_marginal.argtypes = [vp, C.POINTER(C.c_double), C.c_size_t]
    L.b3d_particles_map_pose.argtypes = [vp, C.c_size_t, C.POINTER(Pose)]
    L.b3d_library_destroy.argtypes = [vp]
    L.b3d_scene_destroy.argtypes = [vp]
    L.b3d_particles_destroy.argtypes = [vp]
    for n in ("b3d_depth_image_create", "b3d_depth_image_load", "b3d_log_likelihood",
              "b3d_model_load", "b3d_library_open", "b3d_scene_from_json", "b3d_render",
              "b3d_infer"):
        getattr(L, n).restype = C.c_int


def _res(L, st):
    return [int(st), L.b3d_last_error().decode() if st else ""]


def _img(L, w, h, fill):
    d = np.full((h, w), fill, dtype=np.float32)
    hdl = vp()
    assert L.b3d_depth_image_create(w, h, d.ctypes.data, C.byref(hdl)) == 0
    return hdl


def _svox(path, voxels, res=0.01, origin=(0.0, 0.0, 0.0), magic=b"SVOX"):
    v = np.ascontiguousarray(voxels, dtype="<i4")
    with open(path, "wb") as f:
        f.write(magic + struct.pack("<4f", res, *origin) + struct.pack("<I", v.shape[0]))
        f.write(v.tobytes())


K = Intr(60.0, 60.0, 31.5, 23.5, 64, 48, 0.05, 4.0)
CAM = Pose(1, 0, 0, 0, 0, 0, 0)
TOP = Pose(0, 1, 0, 0, 0.2, 0.2, 0.8)  # above the table, looking down


def run_cases(L, gpu: bool):
    """All cases against library L; gpu=False skips the device-reaching ones."""
    _sig(L)
    out = {}
    tmp = tempfile.mkdtemp()
    obs = _img(L, 64, 48, 1.0)
    rend = _img(L, 64, 48, 1.0)
    empty = _img(L, 64, 48, 4.0)  # every pixel = the far sentinel
    small = _img(L, 32, 24, 1.0)
    r = C.c_double()
    h = vp()
    d = np.zeros(4, dtype=np.float32)
    out["depth_create_zero_width"] = _res(L, L.b3d_depth_image_create(0, 3, d.ctypes.data,
                                                                      C.byref(h)))
    out["depth_create_null"] = _res(L, L.b3d_depth_image_create(2, 2, None, C.byref(h)))
    # b3d_log_likelihood (b3d.h:110-115): validation before any work
    ll = lambda o, re, k, p, s, sm, w: _res(L, L.b3d_log_likelihood(o, re, C.byref(k) if k else None,
                                                                   p, s, sm, w, C.byref(r)))
    out["ll_null_observed"] = ll(None, rend, K, 0.1, 0.01, 0.1, 1)
    out["ll_sigma_nonpositive"] = ll(obs, rend, K, 0.1, 0.0, 0.1, 1)
    out["ll_sigma_max_nonpositive"] = ll(obs, rend, K, 0.1, 0.01, 0.0, 1)
    out["ll_p_outlier_above_one"] = ll(obs, rend, K, 1.5, 0.01, 0.1, 1)
    out["ll_p_outlier_negative"] = ll(obs, rend, K, -0.1, 0.01, 0.1, 1)
    out["ll_window_dims"] = ll(obs, small, K, 0.1, 0.01, 0.1, 1)
    out["ll_full_dims"] = ll(obs, small, K, 0.1, 0.01, 0.1, -1)
    bad_k = Intr(60.0, 60.0, 80.0, 23.5, 64, 48, 0.05, 4.0)  # cx outside the image
    out["ll_bad_intrinsics"] = ll(obs, rend, bad_k, 0.1, 0.01, 0.1, 1)
    near_k = Intr(60.0, 60.0, 31.5, 23.5, 64, 48, 5.0, 4.0)  # near >= far
    out["ll_near_far"] = ll(obs, rend, near_k, 0.1, 0.01, 0.1, 1)
    if gpu:
        out["ll_empty_windowed"] = ll(obs, empty, K, 0.1, 0.01, 0.1, 1)
        out["ll_empty_full"] = ll(obs, empty, K, 0.1, 0.01, 0.1, -1)
    # files
    open(os.path.join(tmp, "bad.sdpt"), "wb").write(b"SDPX" + bytes(8))
    out["sdpt_missing"] = _res(L, L.b3d_depth_image_load(os.path.join(tmp, "nope.sdpt").encode(),
                                                         C.byref(h)))
    out["sdpt_bad_magic"] = _res(L, L.b3d_depth_image_load(os.path.join(tmp, "bad.sdpt").encode(),
                                                           C.byref(h)))
    open(os.path.join(tmp, "short.sdpt"), "wb").write(b"SDPT" + struct.pack("<II", 4, 4) + bytes(8))
    out["sdpt_truncated"] = _res(L, L.b3d_depth_image_load(
        os.path.join(tmp, "short.sdpt").encode(), C.byref(h)))
    _svox(os.path.join(tmp, "bad.svox"), [[0, 0, 0]], magic=b"SVOY")
    out["svox_bad_magic"] = _res(L, L.b3d_model_load(os.path.join(tmp, "bad.svox").encode(), 0,
                                                     C.byref(h)))
    _svox(os.path.join(tmp, "a.svox"), [[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]])
    _svox(os.path.join(tmp, "b.svox"), [[0, 0, 0], [1, 0, 0], [2, 0, 0], [0, 1, 0], [0, 0, 1]])

    def manifest(name, obj):
        p = os.path.join(tmp, name)
        open(p, "w").write(obj if isinstance(obj, str) else json.dumps(obj))
        return p.encode()

    lib = vp()
    cases = {
        "manifest_missing": os.path.join(tmp, "none.json").encode(),
        "manifest_not_json": manifest("nj.json", "{not json"),
        "manifest_no_models": manifest("nm.json", {"x": 1}),
        "manifest_sparse_ids": manifest("sp.json", {"models": [{"id": 1, "path": "a.svox"}]}),
        "manifest_duplicate_ids": manifest("dup.json", {"models": [{"id": 0, "path": "a.svox"},
                                                                   {"id": 0, "path": "b.svox"}]}),
        "manifest_bad_entry": manifest("be.json", {"models": [{"id": 0}]}),
    }
    for name, path in cases.items():
        out[name] = _res(L, L.b3d_library_open(path, C.byref(lib)))
    st = L.b3d_library_open(manifest("ok.json", {"models": [{"id": 0, "path": "a.svox"},
                                                            {"id": 1, "path": "b.svox"}]}),
                            C.byref(lib))
    assert st == 0, L.b3d_last_error()
    # scene JSON (scene_graph.cpp:211-234)
    sc = vp()
    scenes = {
        "scene_not_json": "{x",
        "scene_missing_table": json.dumps({"children": []}),
        "scene_object_range": json.dumps({"table": {"width": 1, "height": 1}, "children": [
            {"object_id": 7, "face": 1, "dx": 0, "dy": 0, "dtheta": 0}]}),
        "scene_missing_key": json.dumps({"table": {"width": 1, "height": 1}, "children": [
            {"object_id": 0, "face": 1, "dx": 0, "dy": 0}]}),
        "scene_table_nonpositive": json.dumps({"table": {"width": 0, "height": 1}}),
    }
    for name, text in scenes.items():
        out[name] = _res(L, L.b3d_scene_from_json(text.encode(), lib, C.byref(sc)))
    # render: invalid intrinsics before any device work
    st = L.b3d_scene_from_json(json.dumps({"table": {"width": 0.4, "height": 0.4}, "children": [
        {"object_id": 0, "face": 1, "dx": 0.1, "dy": 0.1, "dtheta": 0.5}]}).encode(), lib,
                               C.byref(sc))
    assert st == 0, L.b3d_last_error()
    img = vp()
    out["render_bad_intrinsics"] = _res(L, L.b3d_render(sc, C.byref(CAM), C.byref(bad_k),
                                                        C.byref(img)))
    out["render_null_scene"] = _res(L, L.b3d_render(None, C.byref(CAM), C.byref(K), C.byref(img)))
    if gpu:  # whole renders, bitwise: a few children (one camera-mode launch) and 20
        for n in (3, 20):  # (more than a camera-mode scene holds: instance after instance)
            ch = [{"object_id": i % 2, "face": 1 + i % 6, "dx": 0.02 + 0.017 * (i % 5),
                   "dy": 0.03 + 0.013 * (i // 5), "dtheta": 0.37 * i % 6.0} for i in range(n)]
            many = vp()
            st = L.b3d_scene_from_json(json.dumps({"table": {"width": 0.4, "height": 0.4},
                                                   "children": ch}).encode(), lib,
                                       C.byref(many))
            assert st == 0, L.b3d_last_error()
            st = L.b3d_render(many, C.byref(TOP), C.byref(K), C.byref(img))
            if st == 0:
                a = np.ctypeslib.as_array(L.b3d_depth_image_data(img), shape=(48 * 64,))
                out[f"render_{n}_children"] = [int((a < 4.0).sum()),
                                               hashlib.sha256(a.tobytes()).hexdigest()]
                L.b3d_depth_image_destroy(img)
            else:
                out[f"render_{n}_children"] = _res(L, st)
            if n == 3 and st == 0:  # this render is the observation of the SMC case below
                st = L.b3d_render(many, C.byref(TOP), C.byref(K), C.byref(img))
                assert st == 0, L.b3d_last_error()
                seen = vp(img.value)
            L.b3d_scene_destroy(many)
        # run_smc placing more objects than any fixed particle layout holds
        cfg = {"intrinsics": dict(fx=60.0, fy=60.0, cx=31.5, cy=23.5, width=64, height=48,
                                  near=0.05, far=4.0),
               "table": {"width": 0.4, "height": 0.4}, "n_objects": 10, "particles": 3,
               "schedule": {"stage0": [2, 2, 2], "refine": [[2, 1, 2]]},
               "noise_grid": {"p_outlier": [0.1], "sigma": [0.01]}}
        marg = (C.c_double * 2)()
        mp = Pose()
        for name, n_obj in (("infer_ten_objects", 10), ("infer_one_object", 1)):
            part = vp()
            st = L.b3d_infer(seen, C.byref(TOP), lib, json.dumps(dict(cfg, n_objects=n_obj)).encode(),
                             5, C.byref(part))
            if st != 0:
                out[name] = _res(L, st)
                continue
            le, txt = C.c_double(), C.c_void_p()
            assert L.b3d_particles_log_evidence(part, C.byref(le)) == 0
            assert L.b3d_particles_to_jsonl(part, C.byref(txt)) == 0
            lines = C.string_at(txt).decode().splitlines()
            L.b3d_string_free(txt)
            ps = [[[c["object_id"], c["face"], c["dx"], c["dy"], c["dtheta"]]
                   for c in json.loads(ln)["children"]] for ln in lines]
            res = {"log_evidence": le.value, "particles": ps}
            st = L.b3d_particles_type_marginal(part, marg, 2)
            if st == 0:
                res["marginal"] = list(marg)
            else:
                out[name + "_marginal"] = _res(L, st)
            st = L.b3d_particles_map_pose(part, 0, C.byref(mp))
            if st == 0:
                res["map_pose"] = [getattr(mp, f) for f, _ in Pose._fields_]
            out[name + "_map_pose_index"] = _res(L, L.b3d_particles_map_pose(part, n_obj,
                                                                              C.byref(mp)))
            out[name + "_marginal_small"] = _res(L, L.b3d_particles_type_marginal(part, marg, 1))
            L.b3d_particles_destroy(part)
            out[name] = [0, res]
        L.b3d_depth_image_destroy(seen)
    # io.cpp:60-102 / 118-130: saved bytes (golden layout), atomic writes that
    # leave nothing behind when the target directory is missing
    L.b3d_depth_image_save.argtypes = [vp, C.c_char_p]
    L.b3d_model_save.argtypes = [vp, C.c_char_p]
    L.b3d_model_load.argtypes = [C.c_char_p, C.c_int, C.POINTER(vp)]
    L.b3d_model_destroy.argtypes = [vp]
    for name, fn in (("depth_save", lambda p: L.b3d_depth_image_save(obs, p)),):
        good = os.path.join(tmp, "saved.sdpt")
        st = fn(good.encode())
        out[name] = [st, hashlib.sha256(open(good, "rb").read()).hexdigest() if st == 0 else
                     L.b3d_last_error().decode()]
        bad = os.path.join(tmp, "no_such_dir", "x.sdpt")
        out[name + "_bad_dir"] = _res(L, fn(bad.encode()))
        out[name + "_bad_dir_leftovers"] = [0, str(sorted(os.listdir(tmp)))]
    mh = vp()
    assert L.b3d_model_load(os.path.join(tmp, "a.svox").encode(), 4, C.byref(mh)) == 0
    good = os.path.join(tmp, "saved.svox")
    st = L.b3d_model_save(mh, good.encode())
    out["model_save"] = [st, hashlib.sha256(open(good, "rb").read()).hexdigest() if st == 0
                         else L.b3d_last_error().decode()]
    out["model_save_bad_dir"] = _res(L, L.b3d_model_save(
        mh, os.path.join(tmp, "no_such_dir", "m.svox").encode()))
    L.b3d_model_destroy(mh)
    # b3d_infer config schema (b3d_capi.cpp:297-379)
    kk = {"fx": 60.0, "fy": 60.0, "cx": 31.5, "cy": 23.5, "width": 64, "height": 48,
          "near": 0.05, "far": 4.0}
    base = {"intrinsics": kk, "table": {"width": 0.4, "height": 0.4}}
    infer = {
        "infer_bad_json": "{nope",
        "infer_no_intrinsics": json.dumps({"table": {"width": 1, "height": 1}}),
        "infer_no_table": json.dumps({"intrinsics": kk}),
        "infer_unknown_key": json.dumps(dict(base, bogus=1)),
        "infer_wrong_type": json.dumps(dict(base, particles="many")),
        "infer_intrinsics_extra": json.dumps(dict(base, intrinsics=dict(kk, extra=1))),
        "infer_stage_shape": json.dumps(dict(base, schedule={"stage0": [2, 2], "refine": []})),
        "infer_stage_zero": json.dumps(dict(base, schedule={"stage0": [2, 0, 2], "refine": []})),
        "infer_noise_outside": json.dumps(dict(base, noise_grid={"p_outlier": [0.1],
                                                                 "sigma": [0.5]})),
        "infer_noise_empty": json.dumps(dict(base, noise_grid={"p_outlier": [], "sigma": [0.1]})),
        "infer_zero_particles": json.dumps(dict(base, particles=0)),
        "infer_zero_objects": json.dumps(dict(base, n_objects=0)),
        "infer_obs_dims": json.dumps(dict(base, intrinsics=dict(kk, width=32, height=24))),
    }
    part = vp()
    for name, text in infer.items():
        if not gpu and name in ("infer_zero_particles", "infer_zero_objects", "infer_noise_outside",
                                "infer_noise_empty", "infer_obs_dims", "infer_stage_zero"):
            continue  # checked after the product sets up its device context
        out[name] = _res(L, L.b3d_infer(obs, C.byref(CAM), lib, text.encode(), 1,
                                        C.byref(part)))
    for hdl in (obs, rend, empty, small):
        L.b3d_depth_image_destroy(hdl)
    L.b3d_scene_destroy(sc)
    L.b3d_library_destroy(lib)
    return {k: [st, msg.replace(tmp, "<tmp>") if isinstance(msg, str) else msg]
            for k, (st, msg) in out.items()}
