"""Probe: where the lane-half K4's roles wait (build with DA_NVCC_FLAGS=-DLH_PROF).

Per-CTA cycle sums of each wait, averaged over CTAs, as a share of the CTA's
total cycles (GEMM1 warp, slot 31).
"""
import ctypes
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_2505_14708_b200 as da  # noqa: E402
from paper_2505_14708_b200 import _lib, api  # noqa: E402

heads = int(sys.argv[1]) if len(sys.argv) > 1 else 24
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
t = tr.flatten()[:148 * 32].reshape(148, 32).cpu().numpy().astype(np.float64)
tot = t[:, 31].mean()
names = {0: "K prod: item_empty", 16: "K prod: k_empty", 17: "V prod: v_empty", 18: "V prod: info",
         1: "GEMM1: q_full", 2: "GEMM1: info", 3: "GEMM1: s_free", 4: "GEMM1: k_full",
         5: "GEMM2: info", 6: "GEMM2: v_full", 7: "GEMM2: p_full", 8: "GEMM2: o_empty",
         9: "softmax (2 warps): info", 10: "softmax: s_full", 11: "softmax: p_free", 12: "softmax: o_full",
         13: "softmax: q_empty", 14: "softmax: item-start bar", 15: "softmax: offset bar"}
print(f"CTA cycles (mean) {tot:.3e}")
for k in sorted(names):
    print(f"{names[k]:28s} {t[:, k].mean() / tot * 100:6.1f} %")
