"""CUDA-graph capture of the pipeline call (HV720 / 90 %, all tokens, H heads:
24 = one GPU, 3 = one rank's share at P = 8): eager vs replay, CUDA events,
K4's share, and the outputs compared.  python tools/probes/graph_probe.py [H]"""
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_2505_14708_b200 as da  # noqa: E402
from paper_2505_14708_b200 import api  # noqa: E402

plan = da.pad_plan(33, 45, 80, 8, 8)
g = torch.Generator(device="cuda").manual_seed(0)
H = int(sys.argv[1]) if len(sys.argv) > 1 else 24
q, k, v = (torch.randn(H, plan.num_valid, 128, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
scale = da.head_dim_scale(128)
run = lambda: api._pipeline(q, k, v, plan, 0.9, scale, "average", "logits", True, False, "hnd", want_bitmap=False)
for _ in range(3):
    ref = run()[0]
torch.cuda.synchronize()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    for _ in range(2):
        run()
torch.cuda.current_stream().wait_stream(s)
graph = torch.cuda.CUDAGraph()
with torch.cuda.graph(graph):
    out_g = run()[0]
torch.cuda.synchronize()


def timeit(fn, n=20):
    ts = []
    for _ in range(n):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


for rep in range(2):
    print(f"H={H} eager ms", round(timeit(run), 3), "graph ms", round(timeit(graph.replay), 3), flush=True)
k4 = []
for _ in range(10):
    ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
    api._pipeline(q, k, v, plan, 0.9, scale, "average", "logits", True, False, "hnd", want_bitmap=False, attn_events=ev)
    torch.cuda.synchronize()
    k4.append(ev[0].elapsed_time(ev[1]))
print(f"H={H} K4 (region order + kernel + fallback list) ms", round(statistics.median(k4), 3))
graph.replay()
torch.cuda.synchronize()
print("graph output == eager:", torch.equal(out_g, ref))
