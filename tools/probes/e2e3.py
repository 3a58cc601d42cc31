"""Probe: e2e distribution — the bench's measurement (5 back-to-back calls, averaged) repeated."""
import sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_2505_14708_b200 as da
plan = da.pad_plan(33, 45, 80, 8, 8)
H, n, d = 24, plan.num_valid, 128
host = [torch.randn(H, n, d).to(torch.bfloat16).pin_memory() for _ in range(3)]
out_host = torch.empty(H, n, d, dtype=torch.bfloat16).pin_memory()
once = lambda: da.multi_head_sparse_attention(host[0], host[1], host[2], plan, 0.9, out=out_host)  # noqa: E731
for _ in range(3):
    once()
torch.cuda.synchronize()
for rep in range(6):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(5):
        once()
    e.record()
    torch.cuda.synchronize()
    print(f"rep {rep}: {s.elapsed_time(e) / 5:.1f} ms/call  reserved {torch.cuda.memory_reserved() / 2**30:.1f} GiB", flush=True)
