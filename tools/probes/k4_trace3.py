"""Timeline of the two-issuer K4 (rows: 0 Kiss, 1 Viss, 2 G1 gotK, 3 G1 committed, 20 G2 enter, 21 G2 v ok,
4 G2 p ok, 5 G2 committed, 6 S got (TRACE_T), 16 ld, 17 exps, 18 st, 7..14 P arrive per softmax warp, 23 sched emit)."""
import ctypes, sys
from pathlib import Path
import numpy as np, torch
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_2505_14708_b200 as da
from paper_2505_14708_b200 import _lib, api
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
base = t[2, 400]
lastP = t[7:15].max(0)
print("step |   Kiss  G1got  G1com |  G2ent  G2vok  G2pok  G2com |  Sgot   lastP")
for s in range(400, 420):
    row = [t[0, s], t[2, s], t[3, s], t[20, s], t[21, s], t[4, s], t[5, s], t[6, s], lastP[s]]
    print(f"{s:4d} | " + " ".join(f"{x - base:6d}" for x in row[:3]) + " | " + " ".join(f"{x - base:6d}" for x in row[3:7])
          + " | " + " ".join(f"{x - base:6d}" for x in row[7:]))
lo, hi = 100, 900
m = lambda a: float(np.mean(a[lo:hi]))
print("period G1", m(np.diff(t[3], prepend=0)), "period G2", m(np.diff(t[5], prepend=0)))
print("G1: got->com", m(t[3] - t[2]), " com(t)->got(t+1)", float(np.mean(t[2, lo + 1:hi + 1] - t[3, lo:hi])))
print("G2: enter->vok", m(t[21] - t[20]), " vok->pok", m(t[4] - t[21]), " pok->com", m(t[5] - t[4]),
      " com(t)->enter(t+1)", float(np.mean(t[20, lo + 1:hi + 1] - t[5, lo:hi])))
print("G1com(t) -> Sgot(t)", m(t[6] - t[3]), " Sgot -> lastP", m(lastP - t[6]), " lastP(t) -> G2pok(t)", m(t[4] - lastP))
print("G1com(t) - G2com(t)", m(t[3] - t[5]), "(negative: GEMM1 ahead)")
print("Kiss(t) -> G1got(t)", m(t[2] - t[0]), " Viss(t) -> G2vok(t)", m(t[21] - t[1]))
w = 7 + (128 // 32 - 4)
print("softmax warp4 per step: loop top->info ok", m(t[19] - t[22]), " info ok->waitS", m(t[15] - t[19]),
      " waitS->Sgot", m(t[6] - t[15]), " Sgot->ld", m(t[16] - t[6]), " ld->exps", m(t[17] - t[16]),
      " exps->st", m(t[18] - t[17]), " st->arrive", m(t[w] - t[18]), " arrive->next top",
      float(np.mean(t[22, lo + 1:hi + 1] - t[w, lo:hi])))
for s_ in range(400, 410):
    print(s_, [int(t[r, s_] - t[22, s_]) for r in (19, 15, 6, 16, 17, 18, w)], int(t[22, s_ + 1] - t[22, s_]))
