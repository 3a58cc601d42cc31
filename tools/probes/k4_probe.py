"""Probe: K4 time vs heads in flight and input layout (L2 residency study).

    python tools/probes/k4_probe.py --heads 1,2,4,24 --layouts orig,reord --reps 3
"""
import argparse
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_2505_14708_b200 as da  # noqa: E402
from paper_2505_14708_b200 import api  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--heads", default="1,2,4,24")
ap.add_argument("--layouts", default="orig,reord")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--sparsity", type=float, default=0.9)
args = ap.parse_args()

plan = da.pad_plan(33, 45, 80, 8, 8)
n, d = plan.num_valid, 128
for H in [int(x) for x in args.heads.split(",")]:
    g = torch.Generator(device="cuda").manual_seed(H)
    q, k, v = (torch.randn(H, n, d, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
    out, mask, _ = api._pipeline(q, k, v, plan, args.sparsity, da.head_dim_scale(d), "average", "logits", True,
                                 False, "hnd")
    kept = int(mask.kept_counts.sum().item())
    flops = 4.0 * 64 * 64 * d * kept
    for lay in args.layouts.split(","):
        if lay == "orig":
            ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            for e in ev:
                e.record()
            ts = []
            for _ in range(args.reps):
                api._pipeline(q, k, v, plan, args.sparsity, da.head_dim_scale(d), "average", "logits", True,
                              False, "hnd", attn_events=ev)
                torch.cuda.synchronize()
                ts.append(ev[0].elapsed_time(ev[1]))
        else:
            qr, kr, vr = (da.reorder_tokens(x, plan) for x in (q, k, v))
            ts = []
            for _ in range(args.reps):
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                da.block_sparse_attention(qr, kr, vr, mask)
                e.record()
                torch.cuda.synchronize()
                ts.append(s.elapsed_time(e))
        ms = min(ts)
        print(f"heads={H:3d} layout={lay:5s} k4={ms:8.3f} ms  per-head={ms / H:7.3f} ms  "
              f"{flops / ms / 1e9:7.1f} TFLOP/s", flush=True)
