"""DraftAttention (paper_2505_14708_b200/dit.py): the DiT attention call with a
dense warm-up and a mask cache across denoising steps."""
import pytest
import torch

import paper_2505_14708_b200 as da
from paper_2505_14708_b200.dit import DraftAttention


def test_arguments_validated():
    with pytest.raises(ValueError, match="sparsity"):
        DraftAttention(2, 45, 80, sparsity=1.0)
    with pytest.raises(ValueError, match="dense_warmup_steps"):
        DraftAttention(2, 45, 80, dense_warmup_steps=-1)
    with pytest.raises(ValueError, match="mask_refresh_every"):
        DraftAttention(2, 45, 80, mask_refresh_every=0)
    att = DraftAttention(2, 45, 80)
    x = torch.zeros(1, 7200, 2, 16)
    with pytest.raises(ValueError, match="CUDA"):
        att(x, x, x)
    with pytest.raises(ValueError, match="token count"):
        att(x[:, :100], x[:, :100], x[:, :100])


def test_step_schedule():
    att = DraftAttention(2, 45, 80, dense_warmup_steps=2, mask_refresh_every=3)
    assert [att.mode(s) for s in (0, 1, 2)] == ["dense", "dense", "select"]
    att._mask, att._mask_step = object(), 2  # as after a selection at step 2
    assert [att.mode(s) for s in (2, 3, 4, 5, 6)] == ["cached", "cached", "cached", "select", "select"]
    assert att.mode(1) == "dense" and att.mode(0) == "dense"
    att.reset()
    assert att.mode(4) == "select"


@pytest.mark.gpu
def test_dit_steps_match_the_entries():
    torch.manual_seed(0)
    b, heads, d = 2, 3, 128
    plan = da.pad_plan(2, 45, 80, 8, 8)
    q, k, v = (torch.randn(b, plan.num_valid, heads, d, device="cuda").to(torch.bfloat16) for _ in range(3))
    att = DraftAttention(2, 45, 80, sparsity=0.9, dense_warmup_steps=1, mask_refresh_every=2)
    # step 0: dense
    o0 = att(q, k, v, step=0)
    ref0 = torch.nn.functional.scaled_dot_product_attention(q.transpose(1, 2), k.transpose(1, 2),
                                                           v.transpose(1, 2)).transpose(1, 2)
    assert torch.equal(o0, ref0)
    # step 1: draft pipeline (bnhd), masks cached
    o1 = att(q, k, v, step=1)
    ref1 = da.multi_head_sparse_attention(q, k, v, plan, 0.9, qkv_layout="bnhd")
    assert torch.equal(o1, ref1) and att.mode(2) == "cached"
    # step 2: executor only with the cached masks = the same attention on the same inputs
    o2 = att(q, k, v, step=2)
    assert o2.shape == o1.shape and o2.dtype == o1.dtype
    assert (o2.float() - o1.float()).abs().max().item() <= 4e-3
    # step 3: refresh
    assert att.mode(3) == "select"
    o3 = att(q, k, v, step=3)
    assert torch.equal(o3, ref1)
