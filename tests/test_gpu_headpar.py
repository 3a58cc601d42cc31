"""Head-parallel path on the GPU: HeadParallelAttention under NCCL (world
size 1 on the one GPU of a test box; the cross-rank schedule itself is covered
at world sizes 2 and 3 over gloo in test_headpar_gloo.py)."""

import socket

import pytest
import torch
import torch.distributed as dist

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nccl():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2505_14708_b200.build import build

    build()
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    yield
    dist.destroy_process_group()


def _inputs(heads=6, seed=3):
    import paper_2505_14708_b200 as da

    plan = da.pad_plan(3, 45, 80, 8, 8)
    g = torch.Generator(device="cuda").manual_seed(seed)
    q, k, v = (torch.randn(plan.num_valid, heads, 128, device="cuda", generator=g).to(torch.bfloat16)
               for _ in range(3))
    return plan, q, k, v


@pytest.mark.parametrize("groups", [1, 2, 4])
def test_head_parallel_equals_single_call(nccl, groups):
    # per-head masks: the resharded, head-grouped call computes exactly what one
    # all-head call does (heads are independent, sparse.py:273-279)
    import paper_2505_14708_b200 as da
    from paper_2505_14708_b200.headpar import HeadParallelAttention

    plan, q, k, v = _inputs()
    hp = HeadParallelAttention(plan, 0.9, 1, 0, head_groups=groups)
    events = []
    out, mask = hp(q, k, v, compute_events=events)
    ref = da.multi_head_sparse_attention(q, k, v, plan, 0.9, qkv_layout="nhd", return_details=True)
    torch.cuda.synchronize()
    assert torch.equal(out, ref.output)
    assert mask.heads == 6 and len(events) == min(groups, 6)
    for h in range(6):
        assert mask.head(h).bitmap_bytes() == ref.mask.head(h).bitmap_bytes()


def test_head_parallel_shared_mask_equals_single_call(nccl):
    # shared_head_mask: the head-ordered fold of the bases gives the same mask
    # as the single-process head mean (sparse.py:281-297)
    import paper_2505_14708_b200 as da
    from paper_2505_14708_b200.headpar import HeadParallelAttention

    plan, q, k, v = _inputs(heads=4, seed=4)
    for select_on in ("logits", "softmax"):
        hp = HeadParallelAttention(plan, 0.85, 1, 0, shared_head_mask=True, select_on=select_on)
        out, mask = hp(q, k, v)
        ref = da.multi_head_sparse_attention(q, k, v, plan, 0.85, shared_head_mask=True, select_on=select_on,
                                             qkv_layout="nhd", return_details=True)
        assert mask.bitmap_bytes() == ref.mask.bitmap_bytes()
        assert mask.kept_count == ref.mask.kept_count and mask.threshold == ref.mask.threshold
        assert (out.float() - ref.output.float()).abs().max().item() <= 4e-3


@pytest.mark.parametrize("transport", ["nccl", "peer"])
def test_head_parallel_cached_mask_runs_the_executor(nccl, transport):
    # mask caching across denoising steps: a returned mask fed back runs the
    # executor alone (padded_block_sparse_attention with that mask)
    import paper_2505_14708_b200 as da
    from paper_2505_14708_b200.headpar import HeadParallelAttention

    plan, q, k, v = _inputs(heads=4, seed=6)
    hp = HeadParallelAttention(plan, 0.9, 1, 0, head_groups=2, transport=transport)
    out, mask = hp(q, k, v)
    ref = da.multi_head_sparse_attention(q, k, v, plan, 0.9, qkv_layout="nhd")
    assert torch.equal(out, ref)
    q2 = (q.float() * 0.5).to(torch.bfloat16)  # the next step's inputs, same mask
    out2, mask2 = hp(q2, k, v, mask=mask)
    assert mask2 is mask
    assert torch.equal(out2, da.padded_block_sparse_attention(q2, k, v, plan, mask, qkv_layout="nhd"))
    hp.close()


def test_dit_world1_parallel_api_matches(nccl):
    # DraftAttention's sequence-parallel branch at world 1 would be the plain
    # call; world > 1 runs in tests/_peer_worker.py (two processes, one GPU)
    from paper_2505_14708_b200.dit import DraftAttention

    att = DraftAttention(3, 45, 80, sparsity=0.9, mask_refresh_every=2)
    plan, q, k, v = _inputs(heads=2, seed=8)
    o = att(q.unsqueeze(0), k.unsqueeze(0), v.unsqueeze(0), step=0)
    assert o.shape == (1, plan.num_valid, 2, 128) and att.mode(1) == "cached"
