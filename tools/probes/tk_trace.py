"""Probe: per-step event times of the transposed K4 on CTA 0 (library built
with -DDA_K4_TK -DTK_TRACE, loaded through DRAFTATTN_B200_LIB).

Events: 0 GEMM1 issue, 1 GEMM2 issue, 2 softmax S ready (s_full wake),
3 softmax S read (s_free), 4 softmax P written (p_full), 5 K stored, 6 V^T stored.
Prints the median gap between consecutive steps of each event and the median
latency between events of one step.
"""
import ctypes
import sys
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
names = ["G1 issue", "G2 issue", "S ready", "S read", "P written", "K copy / K stored", "V stored", "SM step start"]
lo, hi = 200, 3000
t0 = t[:, lo:hi]
print("median per-step gap (cycles):", {names[e]: float(np.median(np.diff(t0[e]))) for e in range(8)})
def lat(a, b, shift=0):
    return float(np.median(t[b, lo + shift:hi + shift] - t[a, lo:hi]))
print("SM step start -> S ready", lat(7, 2))
print("P written(s) -> SM step start(s+2)", lat(4, 7, 2))
print("K stored -> G1 issue", lat(5, 0))
print("G1 issue -> S ready", lat(0, 2))
print("S ready -> S read", lat(2, 3))
print("S read -> P written", lat(3, 4))
print("P written -> G2 issue", lat(4, 1))
print("V stored -> G2 issue", lat(6, 1))
print("S read(s) -> G1 issue(s+2)", lat(3, 0, 2))
print("G2 issue(s) -> P written(s+2)", lat(1, 4, 2))
print("G1 issue(s) -> K stored(s+2)", lat(0, 5, 2))
print("G2 issue(s) -> V stored(s+2)", lat(1, 6, 2))
print("P written(s) -> SM step start(s+3)", lat(4, 7, 3))
print("S read(s) -> G1 issue(s+3)", lat(3, 0, 3))
print("G2 issue(s) -> P written(s+3)", lat(1, 4, 3))
for s in range(lo, lo + 12):
    print(s, [int(t[e, s] - t[0, lo]) for e in range(8)])
