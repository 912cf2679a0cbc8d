"""Per-call wall time of the reference C ABI's scoring entry points on the
product (GPU) and, where built, on the reference library (host): b3d_render
and b3d_log_likelihood at cfg1's 160x120, medians of 200 calls."""
import ctypes as C
import json
import os
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, ROOT)
from capi_cases import Intr, Pose, _sig, _svox  # noqa: E402
from paper_2312_08715_b200 import b3d  # noqa: E402

libs = {"product": C.CDLL(b3d.lib()._name)}
ref = os.path.join(ROOT, "oracle", "_ref", "libb3d_ref.so")
if os.path.exists(ref):
    libs["reference"] = C.CDLL(ref)
k = Intr(200.0, 200.0, 79.5, 59.5, 160, 120, 0.05, 4.0)
rng = np.random.Generator(np.random.PCG64(1))
obs = rng.uniform(0.5, 1.5, size=(120, 160)).astype(np.float32)
ren = obs + rng.normal(0, 0.005, size=obs.shape).astype(np.float32)
ren[rng.random(obs.shape) < 0.5] = np.float32(4.0)
for name, L in libs.items():
    _sig(L)
    ho, hr = C.c_void_p(), C.c_void_p()
    L.b3d_depth_image_create(160, 120, obs.ctypes.data, C.byref(ho))
    L.b3d_depth_image_create(160, 120, ren.ctypes.data, C.byref(hr))
    v = C.c_double()
    for window in (1, 3):
        ts = []
        for i in range(220):
            t0 = time.perf_counter()
            st = L.b3d_log_likelihood(ho, hr, C.byref(k), 0.1, 0.01, 0.1, window, C.byref(v))
            ts.append(time.perf_counter() - t0)
            assert st == 0
        print(f"{name:10s} b3d_log_likelihood window {window}: median "
              f"{1e6 * np.median(ts[20:]):8.1f} us")
    tmp = tempfile.mkdtemp()
    vox = [[i % 10, (i // 10) % 10, i // 100] for i in range(300)]
    _svox(os.path.join(tmp, "a.svox"), vox, res=0.005)
    with open(os.path.join(tmp, "m.json"), "w") as f:
        json.dump({"models": [{"id": 0, "path": "a.svox"}]}, f)
    lib = C.c_void_p()
    assert L.b3d_library_open(os.path.join(tmp, "m.json").encode(), C.byref(lib)) == 0
    sc = C.c_void_p()
    scene = {"table": {"width": 0.3, "height": 0.3},
             "children": [{"object_id": 0, "face": 1, "dx": 0.1, "dy": 0.1, "dtheta": 0.5}]}
    assert L.b3d_scene_from_json(json.dumps(scene).encode(), lib, C.byref(sc)) == 0
    cam = Pose(0, 1, 0, 0, 0.15, 0.15, 0.6)
    img = C.c_void_p()
    ts = []
    for i in range(220):
        t0 = time.perf_counter()
        st = L.b3d_render(sc, C.byref(cam), C.byref(k), C.byref(img))
        ts.append(time.perf_counter() - t0)
        assert st == 0
        L.b3d_depth_image_destroy(img)
    print(f"{name:10s} b3d_render: median {1e6 * np.median(ts[20:]):8.1f} us")
