"""Probe: where the transposed K4's roles wait (library built with -DDA_K4_TK
-DTK_PROF, loaded through DRAFTATTN_B200_LIB).

Per-CTA cycle sums of each accounted segment, averaged over CTAs, as a share
of the CTA's total cycles (slot 63).
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
tr = torch.zeros(148 * 64, dtype=torch.int64, device="cuda")
_lib.lib().da_debug_trace(ctypes.c_void_p(tr.data_ptr()))
api._pipeline(q, k, v, plan, 0.9, da.head_dim_scale(d), "average", "logits", True, False, "hnd")
torch.cuda.synchronize()
_lib.lib().da_debug_trace(None)
t = tr.reshape(148, 64).cpu().numpy().astype(np.float64)
tot = t[:, 63].mean()
roles = ["GEMM1", "GEMM2", "V loader 0", "V loader 1", "softmax", "Q loader", "scheduler"]
slots = {
    0: {0: "step info", 1: "q_full", 2: "k_full", 3: "s_free", 4: "MMA issue + commits"},
    1: {0: "step info", 1: "o_empty", 2: "v_full", 3: "p_full", 4: "MMA issue + commits"},
    2: {0: "step info", 2: "buffer empty", 3: "tmem st (incl. LDG latency)"},
    3: {0: "step info", 2: "buffer empty", 3: "tmem st (incl. LDG latency)"},
    4: {0: "step info", 1: "q_full", 2: "s_full", 3: "S ld + exp + P^T stores + sums", 4: "p_free", 5: "o_full"},
    5: {0: "item", 1: "q_empty"},
    6: {1: "ring full (info_empty)", 2: "K slot (k_empty)"},
}
print(f"CTA cycles (mean) {tot:.3e}")
for r, name in enumerate(roles):
    for k, what in slots[r].items():
        print(f"{name:10s} {what:32s} {t[:, 8 * r + k].mean() / tot * 100:6.1f} %")
