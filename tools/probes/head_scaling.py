"""Probe: what one rank computes at P = 1/2/4/8 head-parallel GPUs, on one GPU
and without collectives: HV720 with 24/P heads, in the head groups
HeadParallelAttention uses (3 by default). Prints ms per call and the
compute-only efficiency T(24) / (P * T(24/P)), the ceiling for the driver's
scaling efficiency."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_2505_14708_b200 as da  # noqa: E402
from paper_2505_14708_b200 import api  # noqa: E402
from paper_2505_14708_b200.headpar import head_groups  # noqa: E402

plan = da.pad_plan(33, 45, 80, 8, 8)
n, d = plan.num_valid, 128
g = torch.Generator(device="cuda").manual_seed(0)
groups_arg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
res = {}
for P in (1, 2, 4, 8):
    hl = 24 // P
    q, k, v = (torch.randn(n, hl, d, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
    out = torch.empty(n, hl, d, device="cuda", dtype=torch.bfloat16)
    grp = head_groups(hl, groups_arg if P > 1 else 1)

    def call():
        for h0, h1 in grp:
            api._pipeline(q[:, h0:h1], k[:, h0:h1], v[:, h0:h1], plan, 0.9, da.head_dim_scale(d), "average",
                          "logits", True, False, "nhd", want_bitmap=False, out_dev=out[:, h0:h1])

    for _ in range(3):
        call()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(10):
        call()
    e.record()
    torch.cuda.synchronize()
    res[P] = s.elapsed_time(e) / 10
    print(json.dumps({"P": P, "heads": hl, "groups": len(grp), "ms": res[P],
                      "compute_only_efficiency": res[1] / (P * res[P])}), flush=True)
