"""Device time of one stage reduction (1,024 / 32,768 / 1M scores, device
buffers, CUDA events around back-to-back launches)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_08715_b200 import b3d  # noqa: E402

ctx = b3d.GpuContext(0)
ctx.set_stream(torch.cuda.current_stream().cuda_stream)
ctx.set_camera(b3d.Intrinsics(200.0, 200.0, 80.0, 60.0, 160, 120, 0.01, 10.0))
for n in (1024, 32768, 1 << 20):
    x = torch.from_numpy(np.random.default_rng(1).normal(-15000, 300, n)).cuda()
    rng = torch.from_numpy(b3d.rng_seed(3).view(np.int64)).cuda()
    out = torch.zeros(8, dtype=torch.float64, device="cuda")
    for _ in range(10):
        ctx.stage_reduce(x, rng_state=rng, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 200
    e0.record()
    for _ in range(reps):
        ctx.stage_reduce(x, rng_state=rng, out=out)
    e1.record()
    torch.cuda.synchronize()
    print(f"n={n:8d}: {e0.elapsed_time(e1) * 1e3 / reps:6.2f} us per reduction (back to back)")
