"""Per-step timeline of one softmax thread (TRACE_T, set at build time) next to the MMA warp.
Rows: 2 gotK, 3 G1 committed, 20 enter gemm2, 21 v ok, 4 p ok, 5 G2 committed,
15 wait S, 6 S got, 16 ld done, 17 exps done, 18 st done, 7+w P arrived (warp 4+w)."""
import ctypes, sys
from pathlib import Path
import numpy as np, torch
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_2505_14708_b200 as da
from paper_2505_14708_b200 import _lib, api
warp = int(sys.argv[1]) if len(sys.argv) > 1 else 5
heads = 24
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
t = tr.cpu().numpy().astype(np.int64)
base = t[3, 300]
print("step |  G1com  G2ent   v_ok   p_ok  G2com | waitS  Sgot  lddone expdone stdone Parr(w)")
for s in range(300, 320):
    mm = " ".join(f"{t[r, s] - base:6d}" for r in (3, 20, 21, 4, 5))
    sm = " ".join(f"{t[r, s] - base:6d}" for r in (15, 6, 16, 17, 18, 7 + warp - 4))
    print(f"{s:4d} | {mm} | {sm}")
lo, hi = 100, 900
print("period", np.mean(np.diff(t[3, lo:hi])))
for name, a, b in (("waitS->Sgot", 15, 6), ("Sgot->lddone", 6, 16), ("ld->exp", 16, 17), ("exp->st", 17, 18),
                   ("st->P", 18, 7 + warp - 4), ("P -> next waitS", 7 + warp - 4, None)):
    if b is None:
        print(name, np.mean(t[15, lo + 1:hi + 1] - t[7 + warp - 4, lo:hi]))
    else:
        print(name, np.mean(t[b, lo:hi] - t[a, lo:hi]))
print("G1com(t) -> Sgot(t)", np.mean(t[6, lo:hi] - t[3, lo:hi]))
