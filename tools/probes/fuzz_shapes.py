"""Randomised cross-checks on the GPU: for random grids, pool shapes (64, 128,
256 and 512 tokens, every aspect the kernels take), head counts and
sparsities, (1) the tcgen05 pipeline against the portable kernel (same masks,
outputs within 1e-2 of the larger magnitude), and (2) the same call over a
random number of sequence shards, bit-identical.

    python tools/probes/fuzz_shapes.py [count] [seed]
"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_2505_14708_b200 as da  # noqa: E402
from paper_2505_14708_b200 import api  # noqa: E402

POOLS = [(8, 8), (4, 16), (16, 4), (2, 32), (8, 16), (16, 8), (4, 32), (16, 16), (8, 32), (32, 8), (16, 32)]


def main(count=200, seed=7):
    rng = np.random.default_rng(seed)
    fails = 0
    for c in range(count):
        ph, pw = POOLS[rng.integers(len(POOLS))]
        f = int(rng.integers(1, 4))
        h = int(rng.integers(ph // 2 + 1, 4 * ph))
        w = int(rng.integers(pw // 2 + 1, 4 * pw))
        heads = int(rng.integers(1, 4))
        sp = float(rng.choice([0.0, 0.5, 0.8, 0.9, 0.95]))
        qmul = float(rng.choice([1.0, 1.0, 1.0, 30.0]))
        plan = da.pad_plan(f, h, w, ph, pw)
        n = plan.num_valid
        gen = torch.Generator(device="cuda").manual_seed(int(rng.integers(1 << 30)))
        q, k, v = (torch.randn(n, heads, 128, device="cuda", generator=gen) for _ in range(3))
        q, k, v = (q * qmul).to(torch.bfloat16), k.to(torch.bfloat16), v.to(torch.bfloat16)
        scale = da.head_dim_scale(128)
        a, ma, _ = api._pipeline(q, k, v, plan, sp, scale, "average", "logits", True, False, "nhd")
        b, mb, _ = api._pipeline(q, k, v, plan, sp, scale, "average", "logits", True, False, "nhd",
                                 force_portable=True)
        same_masks = all(ma.head(i).bitmap_bytes() == mb.head(i).bitmap_bytes() for i in range(heads))
        err = (a.float() - b.float()).abs().max().item()
        tol = 1e-2 * max(1.0, b.float().abs().max().item())
        parts = int(rng.integers(2, 9))
        rows = -(-n // parts)
        while rows * (parts - 1) >= n:  # every shard non-empty
            parts -= 1
        ok_sh = True
        if parts >= 2:
            split = lambda x: [x[i:i + rows].contiguous() for i in range(0, n, rows)]
            outs = da.sharded_sparse_attention(split(q), split(k), split(v), plan, sp)
            ok_sh = torch.equal(torch.cat(outs), a)
        torch.cuda.synchronize()
        ok = same_masks and err <= tol and ok_sh
        fails += not ok
        print(f"{c:4d} {'ok  ' if ok else 'FAIL'} grid {f}x{h}x{w} pool {ph}x{pw} heads {heads} sp {sp} qx{qmul:g} "
              f"err {err:.2e} masks {same_masks} shards {parts} {ok_sh}", flush=True)
    print(f"{count - fails}/{count} ok")
    return fails


if __name__ == "__main__":
    sys.exit(1 if main(*(int(x) for x in sys.argv[1:3])) else 0)
