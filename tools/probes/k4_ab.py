"""Probe: K4 on gaussian and smooth synthetic data at HV720 (pair-union statistics of the masks).

    python tools/probes/k4_ab.py --data gaussian,smooth --sparsity 0.9
(build variants with DA_NVCC_FLAGS, e.g. -DLH_KSL=4)
"""
import argparse
import os
import sys
from pathlib import Path

import torch
import torch.nn.functional as F

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_2505_14708_b200 as da  # noqa: E402
from paper_2505_14708_b200 import api  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--data", default="gaussian,smooth")
ap.add_argument("--sparsity", type=float, default=0.9)
ap.add_argument("--heads", type=int, default=24)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--config", default="hv720")
args = ap.parse_args()

f, h, w = {"hv720": (33, 45, 80), "wan720": (21, 45, 80), "hv16": (16, 45, 80), "hv8": (8, 45, 80)}[args.config]
plan = da.pad_plan(f, h, w, 8, 8)
n, d, H = plan.num_valid, 128, args.heads


def smooth(gen):
    # bilinear field over (f, y, x) from a coarse 6x10 grid per frame + 0.1 noise, like synth.py's smooth mode
    lo = torch.randn(H * d, f, 6, 10, device="cuda", generator=gen)
    fld = F.interpolate(lo, size=(h, w), mode="bilinear", align_corners=True)  # (H*d, f, h, w)
    fld = fld.reshape(H, d, f * h * w).transpose(1, 2)
    return (fld + 0.1 * torch.randn(H, n, d, device="cuda", generator=gen)).to(torch.bfloat16).contiguous()


for mode in args.data.split(","):
    g = torch.Generator(device="cuda").manual_seed(7)
    if mode == "gaussian":
        q, k, v = (torch.randn(H, n, d, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
    else:
        q, k, v = (smooth(g) for _ in range(3))
    out, mask, _ = api._pipeline(q, k, v, plan, args.sparsity, da.head_dim_scale(d), "average", "logits", True,
                                 False, "hnd")
    kept = int(mask.kept_counts.sum().item())
    # union size of region pairs (2i, 2i+1)
    rp = mask.row_ptr.cpu()
    ci = mask.col_idx.cpu()
    gg = plan.layout.num_regions
    uni = 0
    for hh in range(min(H, 2)):
        for i in range(0, gg - 1, 2):
            a = set(ci[hh, rp[hh, i]:rp[hh, i + 1]].tolist())
            b = set(ci[hh, rp[hh, i + 1]:rp[hh, i + 2]].tolist())
            uni += len(a | b)
    kept2 = int(mask.kept_counts[:min(H, 2)].sum().item())
    steps_est = uni / min(H, 2) * H  # union steps of the whole call (one key region per step)
    flops = 4.0 * 64 * 64 * d * kept
    ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
    for e in ev:
        e.record()
    ts, tot = [], []
    for _ in range(args.reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        api._pipeline(q, k, v, plan, args.sparsity, da.head_dim_scale(d), "average", "logits", True,
                      False, "hnd", attn_events=ev, want_bitmap=False)
        e.record()
        torch.cuda.synchronize()
        ts.append(ev[0].elapsed_time(ev[1]))
        tot.append(s.elapsed_time(e))
    ms = sorted(ts)[len(ts) // 2]
    print(f"K4={os.environ.get('DA_K4', 'pair'):10s} data={mode:8s} sp={args.sparsity} k4={ms:8.3f} ms "
          f"call={sorted(tot)[len(tot) // 2]:8.3f} ms  {flops / ms / 1e9:7.1f} TFLOP/s  "
          f"pair-union/kept={2 * uni / kept2:.3f}  ~{ms * 1e-3 * 1.8e9 * 148 / steps_est:.0f} cycles/step @1.8GHz",
          flush=True)
