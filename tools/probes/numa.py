"""Probe: pinned H2D rate with the process pinned to the GPU's local CPUs vs the others."""
import os
import time

import pynvml
import torch

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
words = pynvml.nvmlDeviceGetCpuAffinity(h, (os.cpu_count() + 63) // 64)
local = {w * 64 + b for w, m in enumerate(words) for b in range(64) if (m >> b) & 1}
allc = set(range(os.cpu_count()))
print("cpus", os.cpu_count(), "gpu-local", len(local), sorted(local)[:4], "...")
for name, cpus in (("local", local), ("remote", allc - local), ("all", allc)):
    if not cpus:
        continue
    os.sched_setaffinity(0, cpus)
    n = 2189721600
    hbuf = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    best = 1e9
    for _ in range(3):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        d.copy_(hbuf, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(f"{name}: H2D {n / best / 1e6:.1f} GB/s")
    del hbuf, d
