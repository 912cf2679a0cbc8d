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
        st = L.b3d_infer(obs, C.byref(CAMERA), lib, text.encode("utf-8", "surrogatepass"), 3,
                         C.byref(part))
        if st != 0:
            out.append([int(st), L.b3d_last_error().decode("utf-8", "backslashreplace")])
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


def _sdpt(w, h, vals):
    return b"SDPT" + struct.pack("<II", w, h) + np.asarray(vals, dtype="<f4").tobytes()


def _svox_bytes(res, origin, voxels):
    v = np.asarray(voxels, dtype="<i4").reshape(-1, 3)
    return (b"SVOX" + struct.pack("<4f", res, *origin) + struct.pack("<I", v.shape[0])
            + v.tobytes())


def file_cases(seed: int = 5, n: int = 200) -> list:
    """Seeded random SDPT / SVOX files (io.cpp:93-147): byte flips, cuts,
    appended bytes, edited headers and payloads."""
    rng = random.Random(seed)
    base_sdpt = _sdpt(4, 3, [0.5 + 0.1 * i for i in range(12)])
    base_svox = _svox_bytes(0.01, (0.0, 0.0, 0.0), [[0, 0, 0], [1, 0, 0], [0, 2, -1]])
    out = []
    for _ in range(n):
        kind = rng.choice(["sdpt", "svox"])
        b = bytearray(base_sdpt if kind == "sdpt" else base_svox)
        for _ in range(rng.randint(1, 2)):
            op = rng.random()
            if op < 0.25 and len(b) > 1:
                del b[rng.randint(1, len(b) - 1):]
            elif op < 0.45 and len(b) > 0:
                i = rng.randint(0, len(b) - 1)
                b[i] = rng.randint(0, 255)
            elif op < 0.55:
                b += bytes(rng.randint(0, 255) for _ in range(rng.choice([1, 4, 12])))
            elif op < 0.75 and len(b) >= 12:
                # a header field: dims / resolution / origin / count
                off = rng.choice([4, 8] if kind == "sdpt" else [4, 8, 12, 16, 20])
                val = rng.choice([0, 1, 2, 3, 5, 0xFFFFFFFF, 0x7FFFFFFF])
                if kind == "svox" and off < 20 and rng.random() < 0.7:
                    b[off:off + 4] = struct.pack("<f", rng.choice(
                        [0.0, -0.01, 1e-30, float("nan"), float("inf"), 1e30, 0.5]))
                else:
                    b[off:off + 4] = struct.pack("<I", val)
            else:  # payload values
                if len(b) >= 16:
                    i = rng.randrange(12 if kind == "sdpt" else 24, max(len(b) - 3, 13), 4) \
                        if len(b) > 24 else 12
                    b[i:i + 4] = struct.pack("<f" if kind == "sdpt" else "<i", rng.choice(
                        [0.0, -1.0, 1e30, float("nan"), 2.5]) if kind == "sdpt" else
                        rng.choice([-2147483648, 2147483647, -5, 1000]))
        out.append((kind, bytes(b)))
    return out


def run_files(L, cases):
    """[status, message] per file, or [0, summary]: an image's width, height
    and sha256 of its floats; a model's SVOX re-saved by b3d_model_save."""
    import hashlib
    _sig(L)
    L.b3d_depth_image_width.argtypes = [C.c_void_p]
    L.b3d_depth_image_width.restype = C.c_uint32
    L.b3d_depth_image_height.argtypes = [C.c_void_p]
    L.b3d_depth_image_height.restype = C.c_uint32
    L.b3d_depth_image_data.argtypes = [C.c_void_p]
    L.b3d_depth_image_data.restype = C.POINTER(C.c_float)
    L.b3d_model_save.argtypes = [C.c_void_p, C.c_char_p]
    L.b3d_model_destroy.argtypes = [C.c_void_p]
    tmp = tempfile.mkdtemp()
    out = []
    for kind, data in cases:
        path = os.path.join(tmp, "f." + kind)
        with open(path, "wb") as f:
            f.write(data)
        h = C.c_void_p()
        if kind == "sdpt":
            st = L.b3d_depth_image_load(path.encode(), C.byref(h))
            if st == 0:
                w, hh = L.b3d_depth_image_width(h), L.b3d_depth_image_height(h)
                a = np.ctypeslib.as_array(L.b3d_depth_image_data(h), shape=(w * hh,)) \
                    if w * hh else np.zeros(0, np.float32)
                out.append([0, [w, hh, hashlib.sha256(a.tobytes()).hexdigest()]])
                L.b3d_depth_image_destroy(h)
                continue
        else:
            st = L.b3d_model_load(path.encode(), 3, C.byref(h))
            if st == 0:
                p2 = os.path.join(tmp, "g.svox")
                st2 = L.b3d_model_save(h, p2.encode())
                L.b3d_model_destroy(h)
                if st2 != 0:
                    out.append([int(st2), "save: " + L.b3d_last_error().decode()])
                    continue
                with open(p2, "rb") as f:
                    out.append([0, hashlib.sha256(f.read()).hexdigest()])
                continue
        out.append([int(st), L.b3d_last_error().decode().replace(tmp, "<tmp>")])
    return out


MANIFEST = {"models": [{"id": 0, "path": "a.svox"}, {"id": 1, "path": "b.svox"}]}


def manifest_texts(seed: int = 11, n: int = 150) -> list:
    """Seeded random library manifests (scene_graph.cpp:206-234)."""
    rng = random.Random(seed)
    paths = ["a.svox", "b.svox", "bad.svox", "none.svox", "", "sub/../a.svox"]
    out = []
    for _ in range(n):
        cfg = copy.deepcopy(MANIFEST)
        for _ in range(rng.randint(1, 3)):
            ps = _paths(cfg)
            if not ps:
                break
            path = rng.choice(ps)
            parent = _get(cfg, path[:-1])
            op = rng.random()
            if op < 0.2 and isinstance(parent, dict):
                del parent[path[-1]]
            elif op < 0.3 and isinstance(parent, dict):
                parent["bogus"] = rng.choice(VALUES)
            elif op < 0.4 and isinstance(parent, list):
                parent.append({"id": rng.choice([0, 1, 2, 3, -1, 2.5]), "path": rng.choice(paths)})
            elif op < 0.6 and path[-1] == "path":
                parent["path"] = rng.choice(paths)
            else:
                parent[path[-1]] = copy.deepcopy(rng.choice(VALUES))
        text = json.dumps(cfg)
        if rng.random() < 0.04:
            text = text[: rng.randint(1, len(text) - 1)]
        out.append(text)
    return out


def run_manifests(L, texts):
    """[status, message] per manifest, or [0, number of models]."""
    _sig(L)
    L.b3d_library_size.argtypes = [C.c_void_p]
    L.b3d_library_size.restype = C.c_size_t
    tmp = tempfile.mkdtemp()
    _svox(os.path.join(tmp, "a.svox"), [[0, 0, 0], [1, 0, 0]], res=0.01)
    _svox(os.path.join(tmp, "b.svox"), [[0, 0, 0], [0, 1, 0], [0, 0, 1]], res=0.01)
    _svox(os.path.join(tmp, "bad.svox"), [[0, 0, 0]], magic=b"SVOY")
    os.makedirs(os.path.join(tmp, "sub"), exist_ok=True)
    out = []
    for text in texts:
        man = os.path.join(tmp, "m.json")
        with open(man, "w") as f:
            f.write(text)
        lib = C.c_void_p()
        st = L.b3d_library_open(man.encode(), C.byref(lib))
        if st == 0:
            out.append([0, int(L.b3d_library_size(lib))])
            L.b3d_library_destroy(lib)
        else:
            out.append([int(st), L.b3d_last_error().decode().replace(tmp, "<tmp>")])
    return out


def loglik_cases(seed: int = 13, n: int = 160) -> list:
    """Seeded random b3d_log_likelihood calls (b3d.h:110-115): image pairs
    with random sentinel fractions and sizes, intrinsics, noise, window."""
    rng = random.Random(seed)
    out = []
    for _ in range(n):
        w, h = rng.choice([(8, 6), (8, 6), (8, 6), (6, 8), (1, 1)])  # noqa: E501
        rw, rh = (w, h) if rng.random() < 0.85 else rng.choice([(6, 8), (8, 5)])
        fill_o, fill_r = rng.choice([0.0, 0.3, 0.9, 1.0]), rng.choice([0.0, 0.3, 0.9, 1.0])
        far = rng.choice([4.0, 4.0, 2.0])
        seed_img = rng.randrange(1 << 30)
        k = [rng.choice([10.0, 10.0, 0.0, -5.0]), 10.0,
             rng.choice([(w - 1) / 2, (w - 1) / 2, w + 3.0]), (h - 1) / 2, w, h,
             rng.choice([0.05, 0.05, 5.0]), far]
        if rng.random() < 0.05:
            k[4] = 0
        out.append({"obs": [w, h, fill_o], "rend": [rw, rh, fill_r], "seed": seed_img, "k": k,
                    "p": rng.choice([-0.1, 0.0, 1e-9, 0.05, 0.3, 1.0, 1.5]),
                    "sigma": rng.choice([0.0, -0.01, 1e-4, 0.01, 0.05, 0.2]),
                    "sigma_max": rng.choice([0.0, 0.1, 0.1, 1e-3]),
                    "window": rng.choice([-1, 0, 1, 2, 3, 100])})
    return out


def _img(w, h, fill, far, seed):
    g = np.random.Generator(np.random.PCG64(seed))
    d = g.uniform(0.5, far * 0.9, size=(h, w)).astype(np.float32)
    d[g.random((h, w)) < fill] = np.float32(far)
    return d


def run_loglik(L, cases):
    """[status, message] or [0, value] per call."""
    _sig(L)
    out = []
    for c in cases:
        k = Intr(*c["k"])
        o = _img(*c["obs"], c["k"][7], c["seed"])
        r = _img(*c["rend"], c["k"][7], c["seed"] + 1)
        ho, hr = C.c_void_p(), C.c_void_p()
        assert L.b3d_depth_image_create(o.shape[1], o.shape[0], o.ctypes.data, C.byref(ho)) == 0
        assert L.b3d_depth_image_create(r.shape[1], r.shape[0], r.ctypes.data, C.byref(hr)) == 0
        v = C.c_double()
        st = L.b3d_log_likelihood(ho, hr, C.byref(k), c["p"], c["sigma"], c["sigma_max"],
                                  c["window"], C.byref(v))
        out.append([0, v.value] if st == 0 else [int(st), L.b3d_last_error().decode()])
        L.b3d_depth_image_destroy(ho)
        L.b3d_depth_image_destroy(hr)
    return out


def render_cases(seed: int = 17, n: int = 120) -> list:
    """Seeded random b3d_render calls: scenes of 0-18 children (some with
    invalid contacts), cameras around / inside / behind the table,
    intrinsics (some invalid)."""
    rng = random.Random(seed)
    out = []
    for _ in range(n):
        nch = rng.choice([0, 1, 2, 5, 18])
        ch = []
        for i in range(nch):
            ch.append({"object_id": rng.randrange(2), "face": rng.choice([1, 2, 3, 4, 5, 6, 6, 7]),
                       "dx": rng.choice([0.01, 0.05, 0.1, 0.2, -0.01, 0.35]),
                       "dy": rng.choice([0.01, 0.05, 0.1, 0.15]),
                       "dtheta": rng.choice([0.0, 1.0, 3.0, 6.0, 6.3])})
        cam = rng.choice([[0, 1, 0, 0, 0.15, 0.12, 0.5], [0, 1, 0, 0, 0.15, 0.12, 0.05],
                          [0, 1.001, 0, 0, 0.15, 0.12, 0.5], [0, 0.9999999, 0, 0, 0.15, 0.12, 0.5],
                          [1, 0, 0, 0, 0.1, 0.1, -0.4], [0.9238795, 0.3826834, 0, 0, 0.1, -0.2, 0.4],
                          [0, 1, 0, 0, 0.15, 0.12, 0.01], [0, 1, 0, 0, 3.0, 0.12, 0.5]])
        k = [20.0, 20.0, 7.5, 5.5, 16, 12, rng.choice([0.05, 0.05, 0.3]), 4.0]
        if rng.random() < 0.1:
            k[2] = 40.0
        out.append({"scene": {"table": {"width": 0.3, "height": 0.25}, "children": ch},
                    "camera": cam, "k": k})
    return out


def run_render(L, cases):
    """[status, message] or [0, sha256 of the depth image] per call."""
    import hashlib
    _sig(L)
    L.b3d_depth_image_data.argtypes = [C.c_void_p]
    L.b3d_depth_image_data.restype = C.POINTER(C.c_float)
    tmp = tempfile.mkdtemp()
    _svox(os.path.join(tmp, "a.svox"), [[0, 0, 0], [1, 0, 0]], res=0.01)
    _svox(os.path.join(tmp, "b.svox"), [[0, 0, 0], [0, 1, 0], [0, 0, 1]], res=0.01)
    man = os.path.join(tmp, "m.json")
    with open(man, "w") as f:
        json.dump({"models": [{"id": 0, "path": "a.svox"}, {"id": 1, "path": "b.svox"}]}, f)
    lib = C.c_void_p()
    assert L.b3d_library_open(man.encode(), C.byref(lib)) == 0, L.b3d_last_error()
    out = []
    for c in cases:
        sc = C.c_void_p()
        st = L.b3d_scene_from_json(json.dumps(c["scene"]).encode(), lib, C.byref(sc))
        if st != 0:
            out.append([int(st), L.b3d_last_error().decode()])
            continue
        img = C.c_void_p()
        st = L.b3d_render(sc, C.byref(Pose(*c["camera"])), C.byref(Intr(*c["k"])), C.byref(img))
        if st == 0:
            a = np.ctypeslib.as_array(L.b3d_depth_image_data(img), shape=(c["k"][4] * c["k"][5],))
            out.append([0, hashlib.sha256(a.tobytes()).hexdigest()])
            L.b3d_depth_image_destroy(img)
        else:
            out.append([int(st), L.b3d_last_error().decode()])
        L.b3d_scene_destroy(sc)
    L.b3d_library_destroy(lib)
    return out


def syntax_texts(seed: int = 19, n: int = 200) -> list:
    """The base infer config's JSON text with random character edits:
    brackets, quotes, commas, escapes (\\u, \\n, bad ones), control
    characters, duplicate keys, whitespace -- for the parser's verdicts."""
    rng = random.Random(seed)
    base = json.dumps(BASE)
    pieces = ['{', '}', '[', ']', '"', ',', ':', '\\\\', '\\\\u0041', '\\\\uD83D\\\\uDE00', '\\\\x',
              '\\t', '\\n', ' ', '\\u0001', 'true', 'null', '-', '0', '1e5', '"threads": 1, ',
              '"window": 1, ', '/**/', '\\ufeff', 'é', '"s\\\\"t"']
    out = []
    for _ in range(n):
        t = base
        for _ in range(rng.randint(1, 2)):
            i = rng.randrange(len(t))
            op = rng.random()
            p = rng.choice(pieces).encode().decode("unicode_escape")
            if op < 0.4:
                t = t[:i] + p + t[i:]
            elif op < 0.7:
                t = t[:i] + t[i + 1:]
            else:
                t = t[:i] + p + t[i + 1:]
        out.append(t)
    return out
