"""Device-side cost of the e2e step's transfers (pinned host <-> device)."""
import torch

s = torch.cuda.current_stream()
for nbytes in (40, 8192, 57344, 76800, 134184, 1 << 20):
    h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    for direction in ("H2D", "D2H"):
        for _ in range(10):
            (d.copy_(h, non_blocking=True) if direction == "H2D" else h.copy_(d, non_blocking=True))
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(100):
            (d.copy_(h, non_blocking=True) if direction == "H2D" else h.copy_(d, non_blocking=True))
        e1.record(s)
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 10
        print(f"{direction} {nbytes:8d} B: {us:6.2f} us/copy  ({nbytes / us / 1e3:6.2f} GB/s)")
