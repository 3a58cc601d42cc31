"""Worker of test_gpu_shards.py::test_peer_transport_two_processes_one_gpu:
one rank of HeadParallelAttention(transport="peer") on cuda:0 (all ranks share
the GPU; gloo carries the IPC handles and the barriers). Each rank checks its
output shard and masks against a single-process call and writes ok<rank>."""

import os
import sys
from pathlib import Path

import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import paper_2505_14708_b200 as da  # noqa: E402
from paper_2505_14708_b200.headpar import HeadParallelAttention  # noqa: E402


def main(out_dir: str) -> None:
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(0)
    dist.init_process_group("gloo")
    plan = da.pad_plan(2, 45, 80, 8, 8) if world == 2 else da.pad_plan(3, 40, 80, 8, 8)
    heads = 2 * world
    n = plan.num_valid
    assert n % world == 0
    nl = n // world
    g = torch.Generator(device="cuda").manual_seed(5)  # identical full inputs on every rank
    q, k, v = (torch.randn(n, heads, 128, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
    ref = da.multi_head_sparse_attention(q, k, v, plan, 0.9, qkv_layout="nhd", return_details=True)
    rows = slice(rank * nl, (rank + 1) * nl)
    hp = HeadParallelAttention(plan, 0.9, world, rank, transport="peer")
    for it in range(3):  # repeated calls reuse the mapped buffers
        out, mask = hp(q[rows].contiguous(), k[rows].contiguous(), v[rows].contiguous())
        torch.cuda.synchronize()
        assert torch.equal(out, ref.output[rows]), f"rank {rank} call {it}: output differs"
        hl = heads // world
        for h in range(hl):
            assert mask.head(h).bitmap_bytes() == ref.mask.head(rank * hl + h).bitmap_bytes()
    # a caller that writes its shards straight into the mapped buffers
    pb = hp.peer_buffers(nl, heads, 128, 128)
    pb.q.copy_(q[rows]); pb.k.copy_(k[rows]); pb.v.copy_(v[rows])
    out, _ = hp(pb.q, pb.k, pb.v)
    torch.cuda.synchronize()
    assert torch.equal(out, ref.output[rows])
    # cached mask: the executor alone on the next step's inputs
    q2 = (q.float() * 0.5).to(torch.bfloat16)
    ref_exec = da.padded_block_sparse_attention(q2, k, v, plan, ref.mask, qkv_layout="nhd")
    out, m2 = hp(q2[rows].contiguous(), k[rows].contiguous(), v[rows].contiguous(), mask=mask)
    torch.cuda.synchronize()
    assert m2 is mask and torch.equal(out, ref_exec[rows]), f"rank {rank}: cached-mask output differs"
    hp.close()
    # the DiT call, sequence parallel: draft step, cached step, refresh
    from paper_2505_14708_b200.dit import DraftAttention

    f, hh, ww = plan.frames, plan.height, plan.width
    att = DraftAttention(f, hh, ww, sparsity=0.9, mask_refresh_every=2, world=world, rank=rank, transport="peer")
    qb, kb, vb = (x[rows].unsqueeze(0).contiguous() for x in (q, k, v))
    o0 = att(qb, kb, vb, step=0)
    assert torch.equal(o0[0], ref.output[rows]) and att.mode(1) == "cached"
    o1 = att(q2[rows].unsqueeze(0).contiguous(), kb, vb, step=1)
    assert torch.equal(o1[0], ref_exec[rows])
    o2 = att(qb, kb, vb, step=2)
    assert torch.equal(o2[0], ref.output[rows])
    att.close()
    Path(out_dir, f"ok{rank}").write_text("ok")
    dist.destroy_process_group()


if __name__ == "__main__":
    main(sys.argv[1])
