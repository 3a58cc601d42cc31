"""Driver for compute-sanitizer runs of the shipped kernels (memcheck,
racecheck, synccheck, initcheck): small shapes of every device path.

    compute-sanitizer --tool memcheck python tools/sanitize.py

* the full pipeline (pooling + region tiles, fp32 draft GEMM and selection,
  lane-half K4, output in original order) on a ragged 720p slice
  (2 x 45 x 80 tokens, 2 heads, d = 128, 8x8 pool, 90 %);
* the fp64 selection fallback (all-zero Q: massive ties), the softmax basis
  and the shared-head mask;
* the portable executor (d = 64, 4x4 pool) and the d % 8 != 0 path;
* the seams: reorder / restore, pool_tokens, draft_logits,
  select_top_fraction, block_sparse_attention;
* sequence shards (the kernels' SPLIT instantiations): the pipeline over 3
  ragged row blocks, max pooling, the portable kernel and the cached-mask
  executor.

Each call is checked against the loose invariants the sanitizer run needs
(finite, right shape); parity proper is tests/test_gpu_parity.py.
"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2505_14708_b200 as da  # noqa: E402


def rnd(*shape, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return torch.randn(*shape, device="cuda", generator=g).to(torch.bfloat16)


def check(name, out):
    torch.cuda.synchronize()
    o = out[0] if isinstance(out, tuple) else getattr(out, "output", out)
    assert torch.isfinite(o.float()).all(), name
    print("ok", name, tuple(o.shape), flush=True)


def main():
    f, h, w, heads, d = 2, 45, 80, 2, 128
    n = f * h * w
    q, k, v = rnd(heads, n, d, seed=1), rnd(heads, n, d, seed=2), rnd(heads, n, d, seed=3)
    plan = da.pad_plan(f, h, w, 8, 8)
    check("pipeline hv slice", da.multi_head_sparse_attention(q, k, v, plan, 0.9))
    check("pipeline padded, details",
          da.padded_sparse_attention(q[0], k[0], v[0], f, h, w, 8, 8, 0.9, return_details=True))
    check("pipeline softmax basis", da.multi_head_sparse_attention(q, k, v, plan, 0.75, select_on="softmax"))
    check("pipeline shared mask", da.multi_head_sparse_attention(q, k, v, plan, 0.5, shared_head_mask=True))
    check("pipeline fp64 fallback (ties)", da.multi_head_sparse_attention(torch.zeros_like(q), k, v, plan, 0.9))
    # portable executor: d = 64, 4x4 pool; and d % 8 != 0
    f2, h2, w2 = 2, 16, 20
    n2 = f2 * h2 * w2
    q2, k2, v2 = rnd(2, n2, 64, seed=4), rnd(2, n2, 64, seed=5), rnd(2, n2, 64, seed=6)
    check("portable d=64", da.multi_head_sparse_attention(q2, k2, v2, da.pad_plan(f2, h2, w2, 4, 4), 0.5))
    check("portable d=36", da.multi_head_sparse_attention(q2[..., :36].contiguous(), k2[..., :36].contiguous(),
                                                          v2[..., :36].contiguous(),
                                                          da.pad_plan(f2, h2, w2, 4, 4), 0.5))
    # seams
    qr = da.reorder_tokens(q, plan)
    check("reorder", qr)
    check("restore", da.restore_tokens(qr, plan))
    kr = da.reorder_tokens(k, plan)
    vr = da.reorder_tokens(v, plan)
    pq = da.pool_tokens(q, plan)
    pk = da.pool_tokens(k, plan)
    check("pool_tokens", pq)
    s = da.draft_logits(pq[0], pk[0], head_dim=d)
    check("draft_logits", s)
    m = da.select_top_fraction(s, 0.1, force_row_keep=True)
    o = da.block_sparse_attention(qr[0], kr[0], vr[0], m)
    check("block_sparse_attention", o)
    # sequence shards: 3 row blocks (the last ragged), "nhd" views
    def split(x, rows):
        xt = x.transpose(0, 1)
        return [xt[i:i + rows].contiguous() for i in range(0, xt.shape[0], rows)]

    qs, ks, vs = split(q, 2500), split(k, 2500), split(v, 2500)
    outs, mask = da.sharded_sparse_attention(qs, ks, vs, plan, 0.9, return_mask=True)
    check("sharded pipeline", torch.cat(outs))
    check("sharded executor (cached mask)", torch.cat(da.sharded_sparse_attention(qs, ks, vs, plan, 0.9, mask=mask)))
    plan_m = da.pad_plan(2, 16, 24, 8, 8)
    qm, km, vm = (rnd(plan_m.num_valid, 2, 128, seed=s_) for s_ in (7, 8, 9))
    sp = lambda x: [x[i:i + 300].contiguous() for i in range(0, x.shape[0], 300)]
    check("sharded max pooling", torch.cat(da.sharded_sparse_attention(sp(qm), sp(km), sp(vm), plan_m, 0.8,
                                                                       pool_mode="max")))
    plan_p = da.pad_plan(f2, h2, w2, 4, 4)
    sp2 = lambda x: [t.contiguous() for t in x.transpose(0, 1).split(200)]
    check("sharded portable", torch.cat(da.sharded_sparse_attention(sp2(q2), sp2(k2), sp2(v2), plan_p, 0.5)))


if __name__ == "__main__":
    main()
