"""Seeded random `b3d_infer` configurations (b3d_capi.cpp:297-379): a small
valid configuration with one to three mutations each -- keys deleted, set to
other JSON types or out-of-range values, unknown keys added, the text cut
short -- run identically against the reference's C ABI (to make
tests/golden/ref_infer_fuzz.json) and the product's (tests/test_capi_reference.py).

The world is tiny (16x12 image, one 2-voxel object, a 0.2 m table) so every
configuration that is valid also runs in milliseconds on the reference."""
from __future__ import annotations

import copy
import ctypes as C
import json
import os
import random
import struct
import tempfile

import numpy as np

from capi_cases import Intr, Pose, _sig, _svox  # noqa: F401

BASE = {
    "intrinsics": {"fx": 20.0, "fy": 20.0, "cx": 7.5, "cy": 5.5, "width": 16, "height": 12,
                   "near": 0.05, "far": 4.0},
    "table": {"width": 0.2, "height": 0.2, "thickness": 0.01},
    "schedule": {"stage0": [1, 1, 2], "refine": [[1, 1, 2]]},
    "noise_grid": {"p_outlier": [0.1], "sigma": [0.02]},
    "particles": 2, "n_objects": 1, "window": 1, "sigma_max": 0.1,
    "resample_threshold": 0.5, "threads": 1,
}
VALUES = [0, 1, 2, 3, -1, 2.5, -0.5, 1e-9, 0.07, "s", True, False, None, [], {}, [1, 2, 3],
          [2, 2], [1, [2], 3], 3000000000, 1e300]
CAMERA = Pose(0, 1, 0, 0, 0.1, 0.1, 0.5)  # above the table, looking down


def _paths(cfg, prefix=()):
    out = []
    if isinstance(cfg, dict):
        for k, v in cfg.items():
            out.append(prefix + (k,))
            out.extend(_paths(v, prefix + (k,)))
    elif isinstance(cfg, list):
        for i, v in enumerate(cfg):
            out.append(prefix + (i,))
            out.extend(_paths(v, prefix + (i,)))
    return out


def _get(cfg, path):
    for p in path:
        cfg = cfg[p]
    return cfg


def mutate(rng: random.Random) -> str:
    cfg = copy.deepcopy(BASE)
    for _ in range(rng.randint(1, 3)):
        paths = _paths(cfg)
        if not paths:
            break
        path = rng.choice(paths)
        parent = _get(cfg, path[:-1])
        op = rng.random()
        if op < 0.2 and isinstance(parent, dict):
            del parent[path[-1]]
        elif op < 0.3 and isinstance(parent, dict):
            parent["bogus"] = rng.choice(VALUES)
        elif op < 0.35 and isinstance(parent, list):
            parent.append(rng.choice(VALUES))
        else:
            parent[path[-1]] = copy.deepcopy(rng.choice(VALUES))
    text = json.dumps(cfg)
    if rng.random() < 0.04:
        text = text[: rng.randint(1, len(text) - 1)]
    return text


def configs(seed: int = 2024, n: int = 240) -> list:
    rng = random.Random(seed)
    return [mutate(rng) for _ in range(n)]


def run(L, texts, allow_device: bool):
    """[status, message] per configuration, or [0, {log_evidence, particles}]
    for a valid one; allow_device=False stops before b3d_infer for none --
    the caller filters device errors."""
    _sig(L)
    L.b3d_particles_log_evidence.argtypes = [C.c_void_p, C.POINTER(C.c_double)]
    L.b3d_particles_to_jsonl.argtypes = [C.c_void_p, C.POINTER(C.c_void_p)]
    L.b3d_string_free.argtypes = [C.c_void_p]
    vp = C.c_void_p
    tmp = tempfile.mkdtemp()
    _svox(os.path.join(tmp, "a.svox"), [[0, 0, 0], [1, 0, 0]], res=0.01)
    man = os.path.join(tmp, "m.json")
    with open(man, "w") as f:
        json.dump({"models": [{"id": 0, "path": "a.svox"}]}, f)
    lib = vp()
    assert L.b3d_library_open(man.encode(), C.byref(lib)) == 0, L.b3d_last_error()
    depth = np.full((12, 16), 0.5, dtype=np.float32)
    depth[4:8, 6:10] = 0.48
    obs = vp()
    assert L.b3d_depth_image_create(16, 12, depth.ctypes.data, C.byref(obs)) == 0
    out = []
    for text in texts:
        part = vp()
        st = L.b3d_infer(obs, C.byref(CAMERA), lib, text.encode(), 3, C.byref(part))
        if st != 0:
            out.append([int(st), L.b3d_last_error().decode()])
            continue
        le, txt = C.c_double(), C.c_void_p()
        assert L.b3d_particles_log_evidence(part, C.byref(le)) == 0
        assert L.b3d_particles_to_jsonl(part, C.byref(txt)) == 0
        lines = C.string_at(txt).decode().splitlines()
        L.b3d_string_free(txt)
        L.b3d_particles_destroy(part)
        out.append([0, {"log_evidence": le.value,
                        "particles": [[[c["object_id"], c["face"], c["dx"], c["dy"], c["dtheta"]]
                                       for c in json.loads(ln)["children"]] for ln in lines]}])
    L.b3d_depth_image_destroy(obs)
    L.b3d_library_destroy(lib)
    return out


SCENE = {"table": {"width": 0.3, "height": 0.25, "thickness": 0.02},
         "children": [{"object_id": 0, "face": 2, "dx": 0.05, "dy": 0.04, "dtheta": 1.0},
                      {"object_id": 1, "face": 5, "dx": 0.1, "dy": 0.02, "dtheta": 4.0}]}


def scene_texts(seed: int = 77, n: int = 200) -> list:
    """Seeded random scene JSON documents (scene_graph.cpp:182-204)."""
    rng = random.Random(seed)
    out = []
    for _ in range(n):
        cfg = copy.deepcopy(SCENE)
        for _ in range(rng.randint(1, 3)):
            paths = _paths(cfg)
            if not paths:
                break
            path = rng.choice(paths)
            parent = _get(cfg, path[:-1])
            op = rng.random()
            if op < 0.25 and isinstance(parent, dict):
                del parent[path[-1]]
            elif op < 0.35 and isinstance(parent, dict):
                parent["bogus"] = rng.choice(VALUES)
            elif op < 0.4 and isinstance(parent, list):
                parent.append(copy.deepcopy(rng.choice(VALUES + [SCENE["children"][0]])))
            else:
                parent[path[-1]] = copy.deepcopy(rng.choice(VALUES))
        text = json.dumps(cfg)
        if rng.random() < 0.04:
            text = text[: rng.randint(1, len(text) - 1)]
        out.append(text)
    return out


def run_scenes(L, texts):
    """[status, message], or [0, b3d_scene_to_json text] for a valid scene."""
    _sig(L)
    L.b3d_scene_to_json.argtypes = [C.c_void_p, C.POINTER(C.c_void_p)]
    L.b3d_string_free.argtypes = [C.c_void_p]
    vp = C.c_void_p
    tmp = tempfile.mkdtemp()
    _svox(os.path.join(tmp, "a.svox"), [[0, 0, 0], [1, 0, 0]], res=0.01)
    _svox(os.path.join(tmp, "b.svox"), [[0, 0, 0], [0, 1, 0], [0, 0, 1]], res=0.01)
    man = os.path.join(tmp, "m.json")
    with open(man, "w") as f:
        json.dump({"models": [{"id": 0, "path": "a.svox"}, {"id": 1, "path": "b.svox"}]}, f)
    lib = vp()
    assert L.b3d_library_open(man.encode(), C.byref(lib)) == 0, L.b3d_last_error()
    out = []
    for text in texts:
        sc = vp()
        st = L.b3d_scene_from_json(text.encode(), lib, C.byref(sc))
        if st != 0:
            out.append([int(st), L.b3d_last_error().decode()])
            continue
        js = C.c_void_p()
        assert L.b3d_scene_to_json(sc, C.byref(js)) == 0
        out.append([0, C.string_at(js).decode()])
        L.b3d_string_free(js)
        L.b3d_scene_destroy(sc)
    L.b3d_library_destroy(lib)
    return out
