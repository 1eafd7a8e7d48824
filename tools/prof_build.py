"""MEASUREMENT TOOL: kernel timeline of one warm build_forest (Netflix32) with torch.profiler
(CUPTI): per-kernel device time, and the wall time vs the sum of kernel time (host gaps)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2210_06014_b200 as ft  # noqa: E402

dims = (480_189, 17_770, 2_182)
dev = ft.generate_device(dims, 99_072_112, (1.0, 5.0), seed=0)
for _ in range(2):
    f = ft.build_forest(dev, 128, compact=True)
    for t in f.trees:
        t.ensure_slots(32, 32)
    del f
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    t0 = time.perf_counter()
    f = ft.build_forest(dev, 128, compact=True)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    for t in f.trees:
        t.ensure_slots(32, 32)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
print(f"build_forest wall {1e3 * (t1 - t0):.2f} ms, slot layouts wall {1e3 * (t2 - t1):.2f} ms")
tot = 0.0
rows = []
for e in prof.key_averages():
    if e.device_type.name == "CUDA" or getattr(e, "self_device_time_total", 0) > 0:
        dt = getattr(e, "self_device_time_total", 0) or getattr(e, "self_cuda_time_total", 0)
        if dt > 0:
            rows.append((dt, e.count, e.key))
            tot += dt
rows.sort(reverse=True)
print(f"sum of device time {tot / 1e3:.2f} ms")
for dt, n, k in rows[:30]:
    print(f"{dt / 1e3:8.3f} ms  x{n:3d}  {k[:90]}")
