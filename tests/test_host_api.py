"""Host-side logic of the drop-in API (CPU only): geometry, counts, FLOP model
and the reference's ValueError contract, raised before any device work."""

import numpy as np
import pytest
import torch

import paper_2505_14708_b200 as da
from oracle import draftattn_oracle as O


def test_layout_validation_matches_reference():
    # layout.py:25-39
    with pytest.raises(ValueError, match="positive integer"):
        da.LatentLayout(0, 4, 4, 2, 2)
    with pytest.raises(ValueError, match="patch_h=3 does not divide height=4"):
        da.LatentLayout(1, 4, 4, 3, 2)
    lay = da.LatentLayout(4, 16, 16, 4, 4)
    assert (lay.num_tokens, lay.region_size, lay.num_regions) == (1024, 16, 64)


def test_pad_plan_geometry():
    plan = da.pad_plan(33, 45, 80, 8, 8)
    assert (plan.layout.height, plan.layout.width) == (48, 80)
    assert plan.num_valid == 118800 and plan.layout.num_tokens == 126720
    assert not plan.is_identity
    assert da.pad_plan(2, 4, 8, 2, 4).is_identity
    with pytest.raises(ValueError, match="positive"):
        da.pad_plan(0, 4, 4, 2, 2)


@pytest.mark.parametrize("n,r", [(100, 0.1), (3920400, 0.1), (3920400, 0.5), (3920400, 0.25),
                                 (3920400, 0.05), (5715360, 0.25), (4096, 0.5), (9, 0.5), (16, 0.001)])
def test_top_fraction_count_equals_oracle(n, r):
    assert da.top_fraction_count(n, r) == O.top_fraction_count(n, r)


def test_hv720_keep_counts():
    # SURVEY 8(a) a8
    g2 = 1980 ** 2
    assert [da.top_fraction_count(g2, 1.0 - s) for s in (0.5, 0.75, 0.9, 0.95)] == \
        [1960200, 980100, 392040, 196020]


def test_flops_model_matches_oracle():
    lay = da.LatentLayout(33, 48, 80, 8, 8)
    f = da.flops_count(lay, 128, kept_count=392040)
    ref = O.flops_count(126720, 1980, 64, 128, 392040)
    assert f.as_dict() == ref
    assert da.flops_count(lay, 128, sparsity=0.9).sparse_logits_flops == ref["sparse_logits_flops"]
    with pytest.raises(ValueError, match="sparsity must be in"):
        da.flops_count(lay, 128, sparsity=1.0)


def _cpu_qkv(n=30, d=8):
    x = torch.zeros(n, d, dtype=torch.bfloat16)
    return x, x, x


def test_pipeline_argument_errors_raise_reference_messages():
    q, k, v = _cpu_qkv()
    with pytest.raises(ValueError, match=r"sparsity must be in \[0, 1\)"):
        da.padded_sparse_attention(q, k, v, 2, 3, 5, 2, 4, 1.0)
    with pytest.raises(ValueError, match="select_on must be 'logits' or 'softmax'"):
        da.padded_sparse_attention(q, k, v, 2, 3, 5, 2, 4, 0.5, select_on="bogus")
    with pytest.raises(ValueError, match="padded grids support average pooling only"):
        da.padded_sparse_attention(q, k, v, 2, 3, 5, 2, 4, 0.5, pool_mode="max")
    with pytest.raises(ValueError, match="real-token rows"):
        da.padded_sparse_attention(q[:29], k[:29], v[:29], 2, 3, 5, 2, 4, 0.5)
    lay = da.LatentLayout(1, 4, 8, 2, 4)
    with pytest.raises(ValueError, match="q rows 30 != layout token count 32"):
        da.draft_sparse_attention(q, k, v, lay, 0.5)
    with pytest.raises(ValueError, match=r"expected \(heads, n, d\)"):
        da.multi_head_sparse_attention(q, k, v, lay, 0.5)


def test_cpu_tensors_are_rejected_not_computed():
    # the B200 path has no CPU fallback: host tensors are staged to the GPU, so
    # without a CUDA device valid arguments raise instead of computing on CPU
    q = torch.zeros(32, 8, dtype=torch.bfloat16)
    with pytest.raises((ValueError, RuntimeError), match="CUDA"):
        da.draft_sparse_attention(q, q, q, da.LatentLayout(1, 4, 8, 2, 4), 0.5)


def test_selection_argument_errors():
    with pytest.raises(ValueError, match="keep_ratio must be in"):
        da.top_fraction_count(10, 0.0)
    with pytest.raises(ValueError, match="square"):
        da.select_top_fraction(torch.zeros(2, 3), 0.5)


@pytest.mark.parametrize("heads,hg", [(24, 2), (40, 4), (2, 1), (3, 1), (5, 1), (24, 1), (7, 2), (13, 2), (1, 1),
                                      (4, 4), (9, 4)])
def test_head_groups_cover_every_head_once(heads, hg):
    from paper_2505_14708_b200.api import _head_groups
    g = _head_groups(heads, hg)
    assert g[0][0] == 0 and g[-1][1] == heads
    assert all(a[1] == b[0] for a, b in zip(g, g[1:]))
    assert all(0 < h1 - h0 <= hg for h0, h1 in g)
    if heads >= 2 * hg and hg > 1:
        assert g[0][1] - g[0][0] == hg // 2  # half-size first group (pipeline fill)


# ---------------------------------------------------------------- mask wire formats (masking.py:128-176)

def _wire_cases():
    import json
    from pathlib import Path
    return json.loads((Path(__file__).resolve().parent / "golden" / "wire.json").read_text())


def test_mask_json_round_trip_matches_reference_export():
    for case in _wire_cases():
        ref = case["json"]
        m = da.mask_from_json_dict(ref, device="cpu")
        assert m.bitmap_bytes().hex() == case["bitmap_hex"]
        assert da.mask_to_json_dict(m) == ref
        assert da.mask_density_stats(m) == case["stats"]


def test_mask_bitmap_round_trip():
    for case in _wire_cases():
        g = case["json"]["g"]
        raw = bytes.fromhex(case["bitmap_hex"])
        kept = da.kept_from_bitmap(raw, g)
        assert kept.dtype == torch.bool and tuple(kept.shape) == (g, g)
        m = da.RegionMask.from_bitmap(raw, g, case["keep_ratio"], case["json"]["threshold"],
                                      case["json"]["forced_row_keeps"], device="cpu")
        assert da.mask_to_bitmap(m) == raw
        assert m.kept_count == case["json"]["kept_count"]
        # executor lists: ascending kept columns per row
        rp, ci = m.row_ptr[0].tolist(), m.col_idx[0].tolist()
        for i in range(g):
            assert ci[rp[i]:rp[i + 1]] == torch.nonzero(kept[i]).flatten().tolist()
    with pytest.raises(ValueError, match="too short"):
        da.kept_from_bitmap(b"\x00", 4)


def test_multi_head_mask_from_kept():
    rng = np.random.default_rng(0)
    kept = rng.random((3, 9, 9)) < 0.3
    m = da.RegionMask.from_kept(kept, 0.3, [0.1, 0.2, 0.3], [0, 1, 2], device="cpu")
    assert m.heads == 3 and not m.single
    assert m.kept_count == kept.reshape(3, -1).sum(1).tolist()
    assert m.threshold == [0.1, 0.2, 0.3] and m.forced_row_keeps == [0, 1, 2]
    for h in range(3):
        assert m.bitmap_bytes(h) == O.mask_bitmap(kept[h])
    with pytest.raises(ValueError, match="boolean"):
        da.RegionMask.from_kept(kept.astype(np.int8), 0.3, 0.0, device="cpu")


# ---------------------------------------------------------------- layouts

def test_bnhd_layout_validation():
    lay = da.LatentLayout(1, 4, 8, 2, 4)
    q = torch.zeros(2, 32, 3, 8, dtype=torch.bfloat16)
    with pytest.raises(ValueError, match="qkv_layout must be one of"):
        da.multi_head_sparse_attention(q[0], q[0], q[0], lay, 0.5, qkv_layout="nchw")
    with pytest.raises(ValueError, match="does not match"):
        da.multi_head_sparse_attention(q, q[:, :, :2], q, lay, 0.5, qkv_layout="bnhd")
    with pytest.raises(ValueError, match="layout token count"):
        da.draft_sparse_attention(q[:, :30], q[:, :30], q[:, :30], lay, 0.5, qkv_layout="bnhd")
    with pytest.raises(ValueError, match="bnhd"):
        da.padded_sparse_attention(q[0], q[0], q[0], 1, 4, 8, 2, 4, 0.5, qkv_layout="bnhd")


def test_feature_padding_is_exact():
    from paper_2505_14708_b200.api import _pad_features
    with pytest.raises(ValueError, match="CUDA"):
        _pad_features(torch.zeros(1, 4, 5))


def test_padded_block_sparse_attention_argument_errors():
    plan = da.pad_plan(2, 13, 20, 4, 4)
    q = torch.zeros(2, plan.num_valid, 16, dtype=torch.bfloat16)
    with pytest.raises(ValueError, match="qkv_layout"):
        da.padded_block_sparse_attention(q, q, q, plan, None, qkv_layout="bhnd")
    with pytest.raises(ValueError, match="do not match"):
        da.padded_block_sparse_attention(q, q[:1], q, plan, None)


def test_shard_table_struct_and_errors():
    # the C-ABI shard table a sequence-sharded call passes (include/draftattn_b200.h
    # da_attn_args.shard_*): pointers per shard, shared strides, rows per shard
    from paper_2505_14708_b200 import _lib, api

    t = api.ShardTable(q=(0x1000, 0x2000), k=(0x3000, 0x4000), v=(0x5000, 0x6000), out=(0x7000, 0x8000),
                       rows=3600, n=7200, heads=4, d=128, dv=64,
                       strides=(128, 3072, 128, 3072, 64, 1536, 64, 1536))
    a = t.struct(0.125)
    assert (a.shard_count, a.shard_rows, a.layout) == (2, 3600, _lib.LAYOUT_ORIGINAL)
    assert list(a.q_shards)[:2] == [0x1000, 0x2000] and list(a.out_shards)[:2] == [0x7000, 0x8000]
    assert a.q_shards[2] is None and len(a.v_shards) == _lib.MAX_SHARDS
    assert (a.q_head_stride, a.q_row_stride, a.v_row_stride, a.o_head_stride) == (128, 3072, 1536, 64)
    assert (a.heads, a.d, a.dv, a.scale) == (4, 128, 64, 0.125)
    x = torch.zeros(10, 2, 8, dtype=torch.bfloat16)
    with pytest.raises(ValueError, match="shards"):
        api._shard_table([x], [x], [x], [x])
    with pytest.raises(ValueError, match="CUDA tensor"):
        api._shard_table([x, x], [x, x], [x, x], [x, x])


def test_head_parallel_transport_argument():
    from paper_2505_14708_b200.headpar import HeadParallelAttention

    plan = da.pad_plan(2, 16, 16, 8, 8)
    with pytest.raises(ValueError, match="transport"):
        HeadParallelAttention(plan, 0.9, 2, 0, transport="shm")
    assert HeadParallelAttention(plan, 0.9, 2, 0, transport="peer").transport == "peer"


def test_documented_entry_points_exist():
    # the README's entry-point table and INTEGRATION.md name these
    import paper_2505_14708_b200.dit as dit
    import paper_2505_14708_b200.headpar as headpar

    for name in ("padded_sparse_attention", "draft_sparse_attention", "multi_head_sparse_attention",
                 "padded_block_sparse_attention", "block_sparse_attention", "select_top_fraction", "draft_logits",
                 "draft_attention_map", "pool_regions", "pool_tokens", "reorder_tokens", "restore_tokens",
                 "RegionMask", "mask_to_json_dict", "mask_from_json_dict", "mask_to_bitmap", "kept_from_bitmap",
                 "mask_density_stats", "flops_count", "sharded_sparse_attention", "pad_plan", "PadPlan",
                 "LatentLayout", "PipelineResult", "FlopsReport", "top_fraction_count", "head_dim_scale"):
        assert callable(getattr(da, name)), name
    assert callable(headpar.HeadParallelAttention) and callable(headpar.PeerShards)
    assert callable(dit.DraftAttention)
