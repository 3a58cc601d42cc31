"""Probe: per-step pipeline timeline of the region-pair tcgen05 kernel (CTA 0, clock64).

Event rows (index = step counter of that role):
  0 K producer issues K(t)     1 V producer issues V(t)
  2 MMA got K(t)               3 MMA issued GEMM1(t)
  4 MMA passed GEMM2(t) waits  5 MMA issued GEMM2(t)
  6 softmax warp 4 got S(t)    7..14 softmax warps 4..11 arrived P(t)
  15 softmax warp 4 starts waiting for S(t)
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
tr = torch.zeros(24, 1024, dtype=torch.int64, device="cuda")
_lib.lib().da_debug_trace(ctypes.c_void_p(tr.data_ptr()))
api._pipeline(q, k, v, plan, 0.9, da.head_dim_scale(d), "average", "logits", True, False, "hnd")
torch.cuda.synchronize()
_lib.lib().da_debug_trace(None)
t = tr.cpu().numpy().astype(np.float64)
lo, hi = 100, 900
last_p = t[7:15, :].max(axis=0)
first_p = t[7:15, :].min(axis=0)
base = t[0, lo]
print("step | Kiss  gotK  G1done  G2pass G2done | S4got  Pfirst Plast   (cycles rel. to K issue of step 100)")
for s in range(200, 224):
    print(f"{s:4d} | " + " ".join(f"{int(t[r, s] - base):7d}" for r in (0, 2, 3, 4, 5)) + " | " +
          " ".join(f"{int(x - base):7d}" for x in (t[6, s], first_p[s], last_p[s])))


def m(x):
    return float(np.mean(x[lo:hi]))


print("cycles/step (GEMM1 issue):", m(np.diff(t[2], prepend=0)))
print("G1 issue duration (gotK->G1done):", m(t[3] - t[2]), "  G2 issue duration:", m(t[5] - t[4]))
print("softmax spread (last P - first P):", m(last_p - first_p))
print("last P(t) -> G2(t) passes waits:", m(t[4] - last_p))
print("G2(t) done -> gotK(t+2):", float(np.mean(t[2, lo + 2:hi + 2] - t[5, lo:hi])))
print("G1(t) issued -> S(t) got by warp 4:", m(t[6] - t[3]))
print("S got -> last P:", m(last_p - t[6]), " per-warp S got -> P:",
      [round(m(t[7 + w] - t[6]), 0) for w in range(8)])
print("warp4 waiting for S:", m(t[6] - t[15]))
print("warp4: S got -> ld done", m(t[16] - t[6]), " ld done -> exps done", m(t[17] - t[16]),
      " exps done -> st waited", m(t[18] - t[17]), " st waited -> P arrive", m(t[7] - t[18]))
print("MMA warp: gotK -> G1 issued+committed", m(t[3] - t[2]))
print("  G1(t+3) committed -> enter gemm2(t)", float(np.mean(t[20, lo:hi] - t[3, lo + 3:hi + 3])))
print("  v_full wait", m(t[21] - t[20]), " p_full+o_empty wait", m(t[4] - t[21]), " G2 issue+commit", m(t[5] - t[4]))
print("  G2(t) committed -> gotK(t+4)", float(np.mean(t[2, lo + 4:hi + 4] - t[5, lo:hi])))
print("scheduler emit period", m(np.diff(t[23], prepend=0)), " emit(t) -> K producer issue(t)", m(t[0] - t[23]),
      " K issue(t) -> MMA gotK(t)", m(t[2] - t[0]))
