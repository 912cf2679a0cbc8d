import sys, time, ctypes as C, numpy as np
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
from capi_cases import Intr, _sig
from paper_2312_08715_b200 import b3d
L = C.CDLL(b3d.lib()._name); _sig(L)
for (w, h) in ((16, 12), (160, 120)):
    k = Intr(200.0, 200.0, (w-1)/2, (h-1)/2, w, h, 0.05, 4.0)
    rng = np.random.Generator(np.random.PCG64(1))
    obs = rng.uniform(0.5, 1.5, size=(h, w)).astype(np.float32)
    ren = obs.copy(); ren[rng.random(obs.shape) < 0.5] = np.float32(4.0)
    ho, hr = C.c_void_p(), C.c_void_p()
    L.b3d_depth_image_create(w, h, obs.ctypes.data, C.byref(ho)); L.b3d_depth_image_create(w, h, ren.ctypes.data, C.byref(hr))
    v = C.c_double()
    for window in (0, 1, 3, -1):
        if window == -1 and w > 16: continue
        ts = []
        for i in range(120):
            t0 = time.perf_counter(); L.b3d_log_likelihood(ho, hr, C.byref(k), 0.1, 0.01, 0.1, window, C.byref(v)); ts.append(time.perf_counter() - t0)
        print(w, h, window, f"{1e6*np.median(ts[20:]):.1f} us")
