"""Cost of the sequence-shard addressing on one GPU: HV720 / 90 % with the
tokens in 8 local row blocks (the kernels' SPLIT instantiations) vs one
(n, heads, d) tensor, both in the "nhd" layout; call and K4 times by CUDA
events, and the outputs compared bit for bit."""
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_2505_14708_b200 as da  # noqa: E402
from paper_2505_14708_b200 import api  # noqa: E402

plan = da.pad_plan(33, 45, 80, 8, 8)
n, H, d = plan.num_valid, 24, 128
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v = (torch.randn(n, H, d, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
rows = n // 8
split = lambda x: [x[i:i + rows].contiguous() for i in range(0, n, rows)]
qs, ks, vs = split(q), split(k), split(v)
outs = [torch.empty_like(x) for x in qs]
table = api._shard_table(qs, ks, vs, outs)
scale = da.head_dim_scale(d)


def plain(ev=None):
    return api._pipeline(q, k, v, plan, 0.9, scale, "average", "logits", True, False, "nhd", attn_events=ev,
                         want_bitmap=False)[0]


def sharded(ev=None):
    api._run_sharded(table, plan, 0.9, scale, attn_events=ev)
    return outs


for name, fn in (("unsplit", plain), ("8 shards", sharded)):
    for _ in range(3):
        fn()
    calls, k4s = [], []
    for _ in range(10):
        ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn(ev)
        e.record()
        torch.cuda.synchronize()
        calls.append(s.elapsed_time(e))
        k4s.append(ev[0].elapsed_time(ev[1]))
    print(f"{name}: call {statistics.median(calls):.3f} ms, K4 {statistics.median(k4s):.3f} ms", flush=True)
ref = plain()
sharded()
torch.cuda.synchronize()
print("bit-identical:", torch.equal(torch.cat(outs), ref))
