"""Probe: the softmax warpgroup 0's ring walk (TK_TRACE2 build): per step,
5 = before next_step, 6 = after next_step, 7 = owned-step start, 2 = S ready,
4 = P written (CTA 0)."""
import ctypes, sys
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_2505_14708_b200 as da  # noqa: E402
from paper_2505_14708_b200 import _lib, api  # noqa: E402
NT = 4096
plan = da.pad_plan(33, 45, 80, 8, 8)
n, d = plan.num_valid, 128
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v = (torch.randn(24, n, d, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
api._pipeline(q, k, v, plan, 0.9, da.head_dim_scale(d), "average", "logits", True, False, "hnd")
tr = torch.zeros(8 * NT, dtype=torch.int64, device="cuda")
_lib.lib().da_debug_trace(ctypes.c_void_p(tr.data_ptr()))
api._pipeline(q, k, v, plan, 0.9, da.head_dim_scale(d), "average", "logits", True, False, "hnd")
torch.cuda.synchronize()
_lib.lib().da_debug_trace(None)
t = tr.reshape(8, NT).cpu().numpy().astype(np.int64)
base = t[5, 200]
for s in range(200, 214):
    print(s, "before", t[5, s] - base, "after", t[6, s] - base, "own start", (t[7, s] - base) if s % 2 == 0 else "",
          "S ready", (t[2, s] - base) if s % 2 == 0 else "", "P written", (t[4, s] - base) if s % 2 == 0 else "",
          "G1 issue", t[0, s] - base)
lo, hi = 200, 3000
ev = np.arange(lo, hi, 2)
print("next_step wait (owned)", np.median(t[6, ev] - t[5, ev]), "next_step wait (skipped)", np.median(t[6, ev + 1] - t[5, ev + 1]))
print("P written -> before next(s+1)", np.median(t[5, ev + 1] - t[4, ev]))
print("after next(s+1) -> before next(s+2)", np.median(t[5, ev + 2] - t[6, ev + 1]))
