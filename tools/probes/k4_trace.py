"""Probe: per-step pipeline timeline of the tcgen05 kernel (CTA 0, clock64).

Events (rows of the trace buffer, index = step counter of that role):
  0 K producer issues K(k)      1 V producer issues V(k)
  15 MMA waits K(k)             2 MMA got K(k) (GEMM1 issue)
  3 MMA GEMM2 #v waits P        4 MMA got P (GEMM2 issue)
  11/14 WG0/WG1 waits S(G)      5/8 WG0/WG1 got S(G)
  6/9 WG0/WG1 before P-buffer wait   7/10 WG0/WG1 arrived P(G)
"""
import ctypes
import sys
from pathlib import Path

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
print("global step k: Kissue Vissue MMAwaitK MMAgotK MMAgotSfree | gemm2#k waitV gotV(waitP) gotP")
for kk in range(200, 232):
    print(f"k={kk:4d}: {rel(t[0, kk]):9d} {rel(t[1, kk]):9d} {rel(t[15, kk]):9d} {rel(t[2, kk]):9d} "
          f"{rel(t[12, kk]):9d} | {rel(t[13, kk]):9d} {rel(t[3, kk]):9d} {rel(t[4, kk]):9d}")
for wg, (ws, gs, pw, pa) in enumerate([(11, 5, 6, 7), (14, 8, 9, 10)]):
    print(f"WG{wg} step G: waitS gotS beforePwait arrivedP")
    for G in range(100, 116):
        print(f"G={G:4d}: {rel(t[ws, G]):9d} {rel(t[gs, G]):9d} {rel(t[pw, G]):9d} {rel(t[pa, G]):9d}")
# averages over steps 100..900
import numpy as np  # noqa: E402

def avg(a, b, lo=100, hi=900):
    return float(np.mean(t[b, lo:hi] - t[a, lo:hi]))

print("avg cycles/global step (K issue):", float(np.mean(np.diff(t[0, 100:900]))))
print("avg cycles/WG0 step:", float(np.mean(np.diff(t[7, 100:450]))))
print("WG0 softmax: gotS->arrivedP", avg(5, 7, 100, 450), " waitS->gotS", avg(11, 5, 100, 450),
      " beforePwait->arrivedP", avg(6, 7, 100, 450))
print("MMA: waitK->gotK", avg(15, 2), " gotK->gotSfree", avg(2, 12), " gemm2 waitV->gotV", avg(13, 3),
      " gemm2 waitP->gotP", avg(3, 4))
print("producer K lead over MMA (K issue -> MMA got K)", avg(0, 2))
