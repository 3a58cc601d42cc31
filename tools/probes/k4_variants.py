"""Probe: A/B of K4 build variants on one box, interleaved.

Build (here, no GPU):   python tools/probes/k4_variants.py build NAME=-DFLAG=1 NAME2=...
Run (GPU box):          python tools/probes/k4_variants.py run NAME NAME2 ... [--rounds 3] [--sparsity 0.9]

Each variant is tools/probes/libs/lib_<NAME>.so (a full library built with
extra -D flags); every run is a fresh process loading that library through
DRAFTATTN_B200_LIB, timing the HV720 call and its K4 launch with CUDA events
and checking the output against the first variant's.
"""
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
LIBS = ROOT / "tools" / "probes" / "libs"

CHILD = r'''
import json, statistics, sys, torch
sys.path.insert(0, sys.argv[1])
import paper_2505_14708_b200 as da
from paper_2505_14708_b200 import api
sp, cfg = float(sys.argv[2]), sys.argv[3]
f, h, w, H = {"hv720": (33, 45, 80, 24), "wan720": (21, 45, 80, 40)}[cfg]
plan = da.pad_plan(f, h, w, 8, 8)
g = torch.Generator(device="cuda").manual_seed(1234)
q, k, v = (torch.randn(H, plan.num_valid, 128, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
run = lambda ev=None: api._pipeline(q, k, v, plan, sp, da.head_dim_scale(128), "average", "logits", True, False,
                                    "hnd", attn_events=ev, want_bitmap=False)
for _ in range(3):
    out = run()
torch.cuda.synchronize()
evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(10)]
for a, b in evs:
    a.record(); b.record()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for ev in evs:
    out = run(ev)
e.record()
torch.cuda.synchronize()
k4 = statistics.median(a.elapsed_time(b) for a, b in evs)
torch.save(out[0][:2].cpu(), sys.argv[4])
print(json.dumps({"call_ms": s.elapsed_time(e) / len(evs), "k4_ms": k4}))
'''


def build(specs):
    sys.path.insert(0, str(ROOT))
    from paper_2505_14708_b200.build import build as b
    LIBS.mkdir(parents=True, exist_ok=True)
    for spec in specs:
        name, _, flags = spec.partition("=")
        out = b(out=LIBS / f"lib_{name}.so", flags=flags.split(",") if flags else [], verbose=True)
        print("built", out)


def run(names, rounds=3, sparsity=0.9, cfg="hv720"):
    import torch
    res = {n: [] for n in names}
    ref = None
    for r in range(rounds):
        for n in names:
            env = dict(os.environ, DRAFTATTN_B200_LIB=str(LIBS / f"lib_{n}.so"))
            outp = f"/tmp/k4v_{n}.pt"
            p = subprocess.run([sys.executable, "-c", CHILD, str(ROOT), str(sparsity), cfg, outp], env=env,
                               capture_output=True, text=True)
            if p.returncode != 0:
                print(n, "FAILED", p.stderr[-2000:], flush=True)
                continue
            line = json.loads(p.stdout.strip().splitlines()[-1])
            o = torch.load(outp).float()
            if ref is None:
                ref = o
            line["max_diff_vs_first"] = float((o - ref).abs().max())
            res[n].append(line)
            print(r, n, line, flush=True)
    for n in names:
        if res[n]:
            print(n, "k4 ms", sorted(x["k4_ms"] for x in res[n]), "call ms", sorted(x["call_ms"] for x in res[n]))


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build(sys.argv[2:])
    else:
        args = sys.argv[2:]
        kw = {}
        for flag, key, typ in (("--rounds", "rounds", int), ("--sparsity", "sparsity", float), ("--config", "cfg", str)):
            if flag in args:
                i = args.index(flag)
                kw[key] = typ(args[i + 1])
                del args[i:i + 2]
        run(args, **kw)
