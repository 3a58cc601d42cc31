"""Probe: per-step pipeline timeline of the tcgen05 kernel (CTA 0, clock64).

Region-pair kernel events (row, index = step counter of that role):
  0 K producer issues K(k)      1 V producer issues V(k)
  2 MMA got K(k) (GEMM1 issue)  4 MMA GEMM2 #k issue (after V and P)
  5 softmax waits S(G)          6 softmax got S(G)          7 softmax arrived P(G)
"""
import ctypes
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_2505_14708_b200 as da  # noqa: E402
from paper_2505_14708_b200 import _lib, api  # noqa: E402

heads = int(sys.argv[1]) if len(sys.argv) > 1 else 2
plan = da.pad_plan(33, 45, 80, 8, 8)
n, d = plan.num_valid, 128
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v = (torch.randn(heads, n, d, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
api._pipeline(q, k, v, plan, 0.9, da.head_dim_scale(d), "average", "logits", True, False, "hnd")
tr = torch.zeros(16, 1024, dtype=torch.int64, device="cuda")
_lib.lib().da_debug_trace(ctypes.c_void_p(tr.data_ptr()))
api._pipeline(q, k, v, plan, 0.9, da.head_dim_scale(d), "average", "logits", True, False, "hnd")
torch.cuda.synchronize()
_lib.lib().da_debug_trace(None)
t = tr.cpu().numpy()
base = t[0, 0]
rel = lambda x: int(x - base) if x else -1  # noqa: E731
print("step: Kissue Vissue MMAgotK GEMM2issue | SMwaitS SMgotS SMarrP")
for s in range(200, 232):
    print(f"{s:4d}: {rel(t[0, s]):9d} {rel(t[1, s]):9d} {rel(t[2, s]):9d} {rel(t[4, s]):9d} | "
          f"{rel(t[5, s]):9d} {rel(t[6, s]):9d} {rel(t[7, s]):9d}")


def avg(a, b, lo=100, hi=900):
    return float(np.mean(t[b, lo:hi] - t[a, lo:hi]))


print("avg cycles/step (K issue):", float(np.mean(np.diff(t[0, 100:900]))))
print("avg cycles/step (GEMM1 issue):", float(np.mean(np.diff(t[2, 100:900]))))
print("softmax: gotS->arrivedP", avg(6, 7), " waitS->gotS", avg(5, 6))
print("GEMM1 issue -> softmax got S", avg(2, 6), "  arrivedP -> GEMM2 issue", avg(7, 4))
print("producer K lead (K issue -> GEMM1 issue)", avg(0, 2), " V issue -> GEMM2 issue", avg(1, 4))
