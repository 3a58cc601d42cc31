"""Head groups on concurrent streams: does the next group's pooling and
selection co-run with the current group's K4 (and its K4 fill the previous
one's tail)? HV720 / 90 %: one 24-head call vs G groups on G streams, CUDA
events on the calling stream (which joins every group), outputs compared."""
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_2505_14708_b200 as da  # noqa: E402
from paper_2505_14708_b200 import api  # noqa: E402

plan = da.pad_plan(33, 45, 80, 8, 8)
H = 24
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v = (torch.randn(H, plan.num_valid, 128, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
scale = da.head_dim_scale(128)
streams = [torch.cuda.Stream() for _ in range(8)]
out = torch.empty_like(q)


def one():
    return api._pipeline(q, k, v, plan, 0.9, scale, "average", "logits", True, False, "hnd", want_bitmap=False)[0]


def split(G):
    main = torch.cuda.current_stream()
    bounds = [round(i * H / G) for i in range(G + 1)]
    for i in range(G):
        st = streams[i]
        st.wait_stream(main)
        with torch.cuda.stream(st):
            h0, h1 = bounds[i], bounds[i + 1]
            api._pipeline(q[h0:h1], k[h0:h1], v[h0:h1], plan, 0.9, scale, "average", "logits", True, False, "hnd",
                          want_bitmap=False, out_dev=out[h0:h1])
    for i in range(G):
        main.wait_stream(streams[i])
    return out


def timeit(fn, n=10):
    for _ in range(3):
        r = fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        r = fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts), r


for rep in range(2):
    t1, r1 = timeit(one)
    print(f"one call: {t1:.3f} ms", flush=True)
    for G in (2, 3, 4, 6):
        tg, rg = timeit(lambda: split(G))
        print(f"{G} streams: {tg:.3f} ms  equal={torch.equal(rg, r1)}", flush=True)
