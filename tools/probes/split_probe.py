"""tcgen05 vs portable on non-8x8 pools, repeated: max-abs per run."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_2505_14708_b200 as da  # noqa: E402
from paper_2505_14708_b200 import api  # noqa: E402

for dims in [(2, 16, 48, 8, 16), (2, 20, 72, 8, 16), (2, 12, 20, 8, 16), (2, 24, 40, 4, 16), (2, 21, 40, 16, 4),
             (2, 24, 40, 8, 8), (2, 21, 40, 8, 8)]:
    plan = da.pad_plan(*dims)
    g = torch.Generator(device="cuda").manual_seed(sum(dims))
    q, k, v = (torch.randn(3, plan.num_valid, 128, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
    scale = da.head_dim_scale(128)
    b, mb, _ = api._pipeline(q, k, v, plan, 0.85, scale, "average", "logits", True, False, "hnd", force_portable=True)
    errs = []
    for _ in range(5):
        a, ma, _ = api._pipeline(q, k, v, plan, 0.85, scale, "average", "logits", True, False, "hnd")
        torch.cuda.synchronize()
        errs.append(round((a.float() - b.float()).abs().max().item(), 4))
    # executor alone with the same mask (kv_tile_kernel tiles instead of the pooling pass's)
    e = api._attend(q, k, v, plan, mb, scale)
    torch.cuda.synchronize()
    print(dims, "pipeline", errs, "executor", round((e.float() - b.float()).abs().max().item(), 4), flush=True)
