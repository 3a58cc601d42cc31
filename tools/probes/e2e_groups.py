"""Host-buffer calls (the e2e path) at HV720 / 90 %: pinned host Q/K/V in,
host output out, for several upload/compute/download head-group sizes."""
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_2505_14708_b200 as da  # noqa: E402
from paper_2505_14708_b200 import api  # noqa: E402

plan = da.pad_plan(33, 45, 80, 8, 8)
host = [torch.randn(24, plan.num_valid, 128).to(torch.bfloat16).pin_memory() for _ in range(3)]
out = torch.empty(24, plan.num_valid, 128, dtype=torch.bfloat16).pin_memory()
scale = da.head_dim_scale(128)
for hg in (None, 1, 2, 3, 4, 6):
    run = lambda: api._pipeline_host(*host, plan, 0.9, scale, "average", "logits", True, False, "hnd",
                                     group_heads=hg, out=out, details=False)
    for _ in range(2):
        run()
    ts = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        run()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    print(f"group_heads={hg}: {statistics.median(ts):.2f} ms", flush=True)
t = []
for _ in range(5):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    d = torch.empty(3, 24, plan.num_valid, 128, dtype=torch.bfloat16, device="cuda")
    a.record()
    for i in range(3):
        d[i].copy_(host[i], non_blocking=True)
    b.record()
    torch.cuda.synchronize()
    t.append(a.elapsed_time(b))
print(f"H2D alone (2.19 GB): {statistics.median(t):.2f} ms", flush=True)
