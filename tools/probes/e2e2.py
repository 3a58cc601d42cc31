import sys, time
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_2505_14708_b200 as da
plan = da.pad_plan(33, 45, 80, 8, 8)
H, n, d = 24, plan.num_valid, 128
host = [torch.randn(H, n, d, dtype=torch.float32).to(torch.bfloat16).pin_memory() for _ in range(3)]
out = torch.empty(H, n, d, dtype=torch.bfloat16).pin_memory()
for i in range(8):
    t0 = time.perf_counter()
    o = da.multi_head_sparse_attention(host[0], host[1], host[2], plan, 0.9, out=out if i % 2 else None)
    print(i, f"{(time.perf_counter() - t0) * 1e3:.1f} ms", o.is_pinned(), flush=True)
