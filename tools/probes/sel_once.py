"""Probe driver: three HV720 pipeline calls (for ncu launch timings of the
selection kernels; pick the library with DRAFTATTN_B200_LIB)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_2505_14708_b200 as da  # noqa: E402
from paper_2505_14708_b200 import api  # noqa: E402

plan = da.pad_plan(33, 45, 80, 8, 8)
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v = (torch.randn(24, plan.num_valid, 128, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
for _ in range(3):
    out, mask, _ = api._pipeline(q, k, v, plan, 0.9, da.head_dim_scale(128), "average", "logits", True, False, "hnd")
torch.cuda.synchronize()
print("kept", int(mask.kept_counts.sum()))
