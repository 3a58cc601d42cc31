"""Probe: host-input API (pipelined head groups) at HV720, per group size."""
import sys, time
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_2505_14708_b200 as da
from paper_2505_14708_b200 import api
plan = da.pad_plan(33, 45, 80, 8, 8)
H, n, d = 24, plan.num_valid, 128
host = [torch.randn(H, n, d).to(torch.bfloat16).pin_memory() for _ in range(3)]
out_host = torch.empty(H, n, d, dtype=torch.bfloat16).pin_memory()
for hg in (None, 1, 2, 3, 4, 6, 8, 12):
    def once():
        return api._pipeline_host(host[0], host[1], host[2], plan, 0.9, da.head_dim_scale(d), "average", "logits",
                                  True, False, "hnd", group_heads=hg, out=out_host, details=False)
    once(); once()
    ts = []
    for _ in range(4):
        t0 = time.perf_counter(); once(); ts.append(time.perf_counter() - t0)
    print(f"group_heads={hg}: {min(ts) * 1e3:.1f} ms/call (host in -> host out)", flush=True)
qd = host[0].cuda(); torch.cuda.synchronize()
t0 = time.perf_counter()
for x in host: x.cuda(non_blocking=True)
torch.cuda.synchronize(); print("H2D 3 tensors", (time.perf_counter() - t0) * 1e3, "ms")
