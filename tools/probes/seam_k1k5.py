"""Probe: standalone K1 (permute-in) / K5 (permute-out) seams at HV720, 24 heads.

Times reorder_tokens / restore_tokens with CUDA events and prints achieved
GB/s over their algorithmic bytes (K1: read 3 ... per tensor: n_real rows in,
n_pad rows out; K5: n_pad rows in, n_real rows out). Under ncu, the kernels
are permute_in_kernel / permute_out_kernel.

    python tools/probes/seam_k1k5.py [--reps 10]
"""
import argparse
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_2505_14708_b200 as da  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=10)
args = ap.parse_args()

plan = da.pad_plan(33, 45, 80, 8, 8)
heads, d = 24, 128
x = torch.randn(heads, plan.num_valid, d, device="cuda").to(torch.bfloat16)
xr = da.reorder_tokens(x, plan)
for _ in range(3):
    da.restore_tokens(da.reorder_tokens(x, plan), plan)
torch.cuda.synchronize()
res = {}
for name, fn, nbytes in (("K1 permute_in", lambda: da.reorder_tokens(x, plan),
                          heads * d * 2 * (plan.num_valid + plan.layout.num_tokens)),
                         ("K5 permute_out", lambda: da.restore_tokens(xr, plan),
                          heads * d * 2 * (plan.layout.num_tokens + plan.num_valid))):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(args.reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / args.reps
    res[name] = {"ms": ms, "bytes": nbytes, "GB/s": nbytes / ms / 1e6}
print(json.dumps(res))
