"""GPU parity: every stage of the CUDA path against the CPU oracle and the
reference's golden fixtures, through the C ABI.

Bars (north_star): permutation and pooling bit-exact; selected block set,
forced count and kept count identical (threshold equal to fp64 roundoff);
attention output within bf16 tolerance  max-abs <= 1e-2  and  cosine >= 0.9999
against the float64 oracle on the same bf16 inputs.
"""

from pathlib import Path

import numpy as np
import pytest
import torch

from oracle import draftattn_oracle as O

pytestmark = pytest.mark.gpu

GOLD = Path(__file__).resolve().parent / "golden"
MAX_ABS = 1e-2
MIN_COS = 0.9999

da = None


@pytest.fixture(scope="module", autouse=True)
def _module():
    global da
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2505_14708_b200.build import build

    build()
    import paper_2505_14708_b200 as mod

    da = mod


def _npz(name):
    return np.load(GOLD / f"{name}.npz")


def _inputs(dims, head_ids=None):
    f, h, w, ph, pw, d, heads, seed = (int(x) for x in dims)
    grid = O.Grid(f, h, w, ph, pw)
    q, k, v = O.gen_real_inputs(grid, d, seed, heads, head_ids=head_ids)
    tq, tk, tv = (torch.from_numpy(x).to("cuda").to(torch.bfloat16) for x in (q, k, v))
    f64 = lambda t: t.double().cpu().numpy()  # noqa: E731
    return grid, (tq, tk, tv), (f64(tq), f64(tk), f64(tv))


def _close(out, ref, max_abs=MAX_ABS, min_cos=MIN_COS):
    out = np.asarray(out, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    err = np.abs(out - ref).max() if out.size else 0.0
    cos = float((out * ref).sum() / (np.linalg.norm(out) * np.linalg.norm(ref) + 1e-300))
    assert err <= max_abs, f"max-abs {err:.3e} > {max_abs}"
    assert cos >= min_cos, f"cosine {cos:.8f} < {min_cos}"
    return err, cos


# ---------------------------------------------------------------- K1 / K5

@pytest.mark.parametrize("dims", [(4, 16, 16, 4, 4, 64), (2, 13, 10, 4, 4, 32), (1, 8, 11, 4, 4, 16),
                                  (3, 45, 80, 8, 8, 128), (2, 7, 3, 2, 2, 8)])
def test_permutation_bit_exact(dims):
    f, h, w, ph, pw, d = dims
    grid = O.Grid(f, h, w, ph, pw)
    plan = da.pad_plan(f, h, w, ph, pw)
    x = torch.randn(3, grid.n_real, d, device="cuda").to(torch.bfloat16)
    xr = da.reorder_tokens(x, plan)
    xs = x.view(torch.int16).cpu().numpy()
    ref = np.stack([O.permute_in(xs[hh], grid) for hh in range(3)])
    assert np.array_equal(xr.view(torch.int16).cpu().numpy(), ref)
    back = da.restore_tokens(xr, plan)
    assert torch.equal(back.view(torch.int16), x.view(torch.int16))


def test_permutation_bit_exact_hv720_full():
    grid = O.Grid(33, 45, 80, 8, 8)
    plan = da.pad_plan(33, 45, 80, 8, 8)
    x = torch.randn(24, grid.n_real, 128, device="cuda").to(torch.bfloat16)
    xr = da.reorder_tokens(x, plan)
    xs = x.view(torch.int16)
    src = torch.from_numpy(O.real_source_index(grid)).cuda()
    live = src >= 0
    ref = torch.zeros(24, grid.n_pad, 128, dtype=torch.int16, device="cuda")
    ref[:, live] = xs[:, src[live]]
    assert torch.equal(xr.view(torch.int16), ref)
    assert torch.equal(da.restore_tokens(xr, plan).view(torch.int16), xs)


def test_permutation_nhd_layout():
    grid = O.Grid(2, 45, 80, 8, 8)
    plan = da.pad_plan(2, 45, 80, 8, 8)
    x = torch.randn(grid.n_real, 4, 128, device="cuda").to(torch.bfloat16)  # (n, heads, d)
    xr = da.reorder_tokens(x, plan, qkv_layout="nhd")
    ref = da.reorder_tokens(x.transpose(0, 1).contiguous(), plan)
    assert torch.equal(xr, ref)


# ---------------------------------------------------------------- K2

@pytest.mark.parametrize("dims,mode", [((4, 16, 16, 4, 4, 64), "average"), ((4, 16, 16, 4, 4, 64), "max"),
                                       ((2, 13, 10, 4, 4, 32), "average"), ((3, 45, 80, 8, 8, 128), "average"),
                                       ((2, 8, 16, 8, 16, 64), "average")])
def test_pooling_bit_exact(dims, mode):
    f, h, w, ph, pw, d = dims
    grid = O.Grid(f, h, w, ph, pw)
    plan = da.pad_plan(f, h, w, ph, pw)
    x = torch.randn(2, grid.n_real, d, device="cuda").to(torch.bfloat16)
    got = da.pool_tokens(x, plan, mode).cpu().numpy()
    x64 = x.double().cpu().numpy()
    for hh in range(2):
        xr = O.permute_in(x64[hh], grid)
        if grid.divisible:
            ref = O.pool_regions(xr, grid.region_size, mode)
        else:
            ref = O.pool_valid(xr, O.valid_reordered(grid), grid.region_size)
        assert np.array_equal(got[hh], ref)


def test_pool_regions_seam_matches_reference_fixture():
    z = _npz("pooling")
    x = torch.from_numpy(z["x"]).to(torch.bfloat16).cuda()
    assert np.array_equal(da.pool_regions(x, 16, "average").cpu().numpy(), z["pool_avg"])
    assert np.array_equal(da.pool_regions(x, 16, "max").cpu().numpy(), z["pool_max"])


# ---------------------------------------------------------------- K3

def test_draft_logits_float64():
    rng = np.random.default_rng(0)
    qp = rng.standard_normal((3, 100, 128))
    kp = rng.standard_normal((3, 100, 128))
    got = da.draft_logits(torch.from_numpy(qp).cuda(), torch.from_numpy(kp).cuda()).cpu().numpy()
    for hh in range(3):
        ref = O.draft_logits(qp[hh], kp[hh], O.head_dim_scale(128))
        np.testing.assert_allclose(got[hh], ref, rtol=1e-13, atol=1e-14)
    sm = da.draft_logits(torch.from_numpy(qp).cuda(), torch.from_numpy(kp).cuda(), softmax=True).cpu().numpy()
    np.testing.assert_allclose(sm[0], O.softmax_rows(O.draft_logits(qp[0], kp[0], O.head_dim_scale(128))),
                               rtol=1e-12, atol=1e-15)
    # draft_attention_map (pooling.py:59-65) is the same row-softmaxed map
    dm = da.draft_attention_map(torch.from_numpy(qp[0]).cuda(), torch.from_numpy(kp[0]).cuda()).cpu().numpy()
    np.testing.assert_array_equal(dm, sm[0])


def test_selection_matches_reference_fixtures_bit_exact():
    z = _npz("selection")
    for c in range(int(z["count"])):
        r, force, thr, forced, kept = z[f"c{c}_meta"]
        scores = torch.from_numpy(z[f"c{c}_scores"]).cuda()
        m = da.select_top_fraction(scores, float(r), bool(force))
        assert m.bitmap_bytes() == z[f"c{c}_bitmap"].tobytes(), f"case {c}"
        assert m.threshold == thr and m.forced_row_keeps == forced and m.kept_count == kept
        rows = m.row_kept_counts.cpu().numpy()
        kept_np = m.kept.cpu().numpy()
        assert np.array_equal(rows, kept_np.sum(axis=1))
        cols = m.col_idx[0].cpu().numpy()
        rp = m.row_ptr[0].cpu().numpy()
        for i in range(m.g):
            assert np.array_equal(cols[rp[i]:rp[i + 1]], np.flatnonzero(kept_np[i]))


def test_selection_edge_cases():
    # hand cases (test_masking.py:59-64, :77-81, :95-103) + negative zero + large ties
    m = da.select_top_fraction(torch.tensor([[9.0, 1.0], [5.0, 7.0]], device="cuda"), 0.5)
    assert m.kept.cpu().tolist() == [[True, False], [False, True]] and m.threshold == 7.0
    m = da.select_top_fraction(torch.zeros(3, 3, device="cuda", dtype=torch.float64), 4 / 9)
    assert m.kept.reshape(-1).cpu().tolist() == [True] * 4 + [False] * 5
    s = torch.full((4, 4), -10.0, dtype=torch.float64)
    s[0] = torch.tensor([4.0, 3.0, 2.0, 1.0])
    m = da.select_top_fraction(s.cuda(), 0.25, force_row_keep=True)
    assert m.forced_row_keeps == 3
    z = np.zeros((5, 5))
    z[1, 2] = -0.0
    z[0, 0] = -0.0
    ref = O.select_top_fraction(z, 0.3, True)
    m = da.select_top_fraction(torch.from_numpy(z).cuda(), 0.3, True)
    assert m.bitmap_bytes() == O.mask_bitmap(ref.kept)
    big = np.round(np.random.default_rng(5).standard_normal((300, 300)))  # heavy ties, g^2 = 90000
    for r in (0.1, 0.37, 0.9):
        for force in (False, True):
            ref = O.select_top_fraction(big, r, force)
            m = da.select_top_fraction(torch.from_numpy(big).cuda(), r, force)
            assert m.bitmap_bytes() == O.mask_bitmap(ref.kept)
            assert m.threshold == ref.threshold and m.forced_row_keeps == ref.forced_row_keeps


def test_selection_dead_columns():
    s = np.random.default_rng(3).standard_normal((20, 20))
    ref = O.drop_key_regions(O.select_top_fraction(s, 0.3, True), [3, 7])
    m = da.select_top_fraction(torch.from_numpy(s).cuda(), 0.3, True, dead_columns=[3, 7])
    assert m.bitmap_bytes() == O.mask_bitmap(ref.kept)
    assert m.kept_count == ref.kept_count and m.forced_row_keeps == ref.forced_row_keeps


# ---------------------------------------------------------------- pipelines vs reference fixtures

def _check_mask(mask, h, z, key):
    got = mask.head(h) if not mask.single else mask
    assert got.bitmap_bytes() == z[f"{key}_bitmap"].tobytes()
    thr, forced, kept = z[f"{key}_meta"]
    assert got.forced_row_keeps == forced and got.kept_count == kept
    assert abs(got.threshold - thr) <= 1e-12 * max(1.0, abs(thr))


@pytest.mark.parametrize("name", ["tiny", "ragged_small", "ragged_w", "pool816", "d4"])
def test_pipeline_full_output_vs_reference(name):
    z = _npz(name)
    grid, (q, k, v), _ = _inputs(z["dims"])
    heads = q.shape[0]
    res = da.multi_head_sparse_attention(q, k, v, da.pad_plan(grid.frames, grid.height, grid.width,
                                                              grid.patch_h, grid.patch_w),
                                         float(z["sparsity"]), return_details=True)
    out = res.output.float().cpu().numpy()
    for h in range(heads):
        _check_mask(res.mask, h, z, f"h{h}")
        _close(out[h], z[f"h{h}_out"])
    # the single-head reference-signature entry gives the same result
    one = da.padded_sparse_attention(q[0], k[0], v[0], grid.frames, grid.height, grid.width,
                                     grid.patch_h, grid.patch_w, float(z["sparsity"]))
    assert torch.equal(one, res.output[0])


@pytest.mark.parametrize("name,head_ids", [("hv720_f2", None), ("hv720", [0, 1])])
def test_pipeline_720p_masks_and_sampled_rows(name, head_ids):
    z = _npz(name)
    grid, (q, k, v), _ = _inputs(z["dims"], head_ids)
    plan = da.pad_plan(grid.frames, grid.height, grid.width, grid.patch_h, grid.patch_w)
    res = da.multi_head_sparse_attention(q, k, v, plan, float(z["sparsity"]), return_details=True)
    ids = head_ids or list(range(q.shape[0]))
    src = O.real_source_index(grid)
    out = res.output.float().cpu().numpy()
    for slot, h in enumerate(ids):
        _check_mask(res.mask, slot, z, f"h{h}")
        rows = z[f"h{h}_rows"]
        pos = (rows[:, None] * grid.region_size + np.arange(grid.region_size)[None, :]).reshape(-1)
        live = src[pos] >= 0
        _close(out[slot][src[pos][live]], z[f"h{h}_out_rows"][live])


def _full_output_report(out, ref, grid):
    """max-abs, max-abs / max|ref|, global and minimum per-row cosine over the
    real rows of one head (bars: max-abs <= 1e-2, global cosine >= 0.9999)."""
    out = np.asarray(out, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    err = float(np.abs(out - ref).max())
    cos = float((out * ref).sum() / (np.linalg.norm(out) * np.linalg.norm(ref)))
    num = (out * ref).sum(1)
    den = np.linalg.norm(out, axis=1) * np.linalg.norm(ref, axis=1)
    live = den > 0
    row_cos = float((num[live] / den[live]).min()) if live.any() else 1.0
    assert np.array_equal(np.linalg.norm(ref, axis=1) == 0, np.linalg.norm(out, axis=1) == 0)
    return {"rows": int(out.shape[0]), "max_abs": err, "rel_max_abs": err / float(np.abs(ref).max()),
            "cosine": cos, "min_row_cosine": row_cos}


@pytest.mark.parametrize("sparsity,head_ids", [(0.9, [0, 1]), (0.5, [2]), (0.75, [3]), (0.95, [4])])
def test_hv720_full_head_outputs_vs_oracle(sparsity, head_ids):
    # complete output of whole HV720 heads (all 118,800 real rows) against the
    # float64 oracle on the same bf16 inputs, with masks, threshold, forced and
    # kept counts (padding.py:95-165); two heads at the headline 90 %, one head
    # at each other sweep point
    grid, (q, k, v), (q64, k64, v64) = _inputs((33, 45, 80, 8, 8, 128, 24, 0), head_ids=head_ids)
    plan = da.pad_plan(33, 45, 80, 8, 8)
    res = da.multi_head_sparse_attention(q, k, v, plan, sparsity, return_details=True)
    out = res.output.float().cpu().numpy()
    for slot, h in enumerate(head_ids):
        ref = O.padded_sparse_attention(q64[slot], k64[slot], v64[slot], 33, 45, 80, 8, 8, sparsity,
                                        return_details=True)
        got = res.mask.head(slot)
        assert got.bitmap_bytes() == O.mask_bitmap(ref.mask.kept)
        assert got.kept_count == ref.mask.kept_count and got.forced_row_keeps == ref.mask.forced_row_keeps
        # the m-th ranked fp64 score; its last bits depend on the dot product's
        # summation order (BLAS vs the GPU's sequential FMA chain)
        assert abs(got.threshold - ref.mask.threshold) <= 1e-12 * max(1.0, abs(ref.mask.threshold))
        rep = _full_output_report(out[slot], ref.output, grid)
        print(f"hv720 head {h} sparsity {sparsity}: {rep}")
        assert rep["max_abs"] <= MAX_ABS and rep["cosine"] >= MIN_COS, rep
        assert rep["min_row_cosine"] >= 0.999, rep


def test_hv720_all_24_heads_masks_vs_oracle():
    # every head of the headline call: bitmap, kept and forced counts, threshold
    grid, (q, k, v), (q64, k64, _) = _inputs((33, 45, 80, 8, 8, 128, 24, 0))
    plan = da.pad_plan(33, 45, 80, 8, 8)
    res = da.multi_head_sparse_attention(q, k, v, plan, 0.9, return_details=True)
    for h in range(24):
        ref, _ = O.draft_mask(q64[h], k64[h], grid, 0.9)
        got = res.mask.head(h)
        assert got.bitmap_bytes() == O.mask_bitmap(ref.kept), h
        assert got.kept_count == ref.kept_count and got.forced_row_keeps == ref.forced_row_keeps, h
        assert abs(got.threshold - ref.threshold) <= 1e-12 * max(1.0, abs(ref.threshold)), h


def test_wan720_all_40_heads_masks_vs_oracle():
    # the Wan 720p config (21 x 45 x 80, 40 heads, 75 %): every head's mask
    grid, (q, k, v), (q64, k64, _) = _inputs((21, 45, 80, 8, 8, 128, 40, 0))
    plan = da.pad_plan(21, 45, 80, 8, 8)
    res = da.multi_head_sparse_attention(q, k, v, plan, 0.75, return_details=True)
    for h in range(40):
        ref, _ = O.draft_mask(q64[h], k64[h], grid, 0.75)
        got = res.mask.head(h)
        assert got.bitmap_bytes() == O.mask_bitmap(ref.kept), h
        assert got.kept_count == ref.kept_count and got.forced_row_keeps == ref.forced_row_keeps, h


@pytest.mark.parametrize("sparsity", [0.5, 0.75, 0.95])
def test_hv720_sparsity_sweep_masks(sparsity):
    grid, (q, k, v), (q64, k64, _) = _inputs((33, 45, 80, 8, 8, 128, 24, 0), head_ids=[0])
    res = da.padded_sparse_attention(q[0], k[0], v[0], 33, 45, 80, 8, 8, sparsity, return_details=True)
    ref, _ = O.draft_mask(q64[0], k64[0], grid, sparsity)
    assert res.mask.bitmap_bytes() == O.mask_bitmap(ref.kept)
    assert res.mask.kept_count == ref.kept_count
    assert res.flops.sparse_logits_flops == 2 * ref.kept_count * 64 * 64 * 128


def test_wan720_masks_and_sampled_rows():
    # the second SURVEY config: Wan 720p, 21 x 45 x 80 tokens at 75 % sparsity
    # (two of its 40 heads, generated with the same per-head seed streams)
    grid, (q, k, v), (q64, k64, v64) = _inputs((21, 45, 80, 8, 8, 128, 40, 0), head_ids=[0, 1])
    plan = da.pad_plan(21, 45, 80, 8, 8)
    res = da.multi_head_sparse_attention(q, k, v, plan, 0.75, return_details=True)
    out = res.output.float().cpu().numpy()
    rows = np.arange(0, grid.num_regions, 97)
    for hh in range(2):
        ref = O.padded_sparse_attention(q64[hh], k64[hh], v64[hh], 21, 45, 80, 8, 8, 0.75, return_details=True,
                                        sample_rows=rows)
        got = res.mask.head(hh)
        assert got.bitmap_bytes() == O.mask_bitmap(ref.mask.kept)
        assert got.kept_count == ref.mask.kept_count and got.forced_row_keeps == ref.mask.forced_row_keeps
        src = O.real_source_index(grid)
        pos = (rows[:, None] * grid.region_size + np.arange(grid.region_size)[None, :]).reshape(-1)
        live = src[pos] >= 0
        _close(out[hh][src[pos][live]], ref.output[src[pos][live]])


# ---------------------------------------------------------------- executor seams and edge cases

def _seam_case(g, p, d, heads, density, seed, key_valid=False):
    rng = np.random.default_rng(seed)
    n = g * p
    q = torch.from_numpy(rng.standard_normal((heads, n, d)).astype(np.float32)).cuda().to(torch.bfloat16)
    k = torch.from_numpy(rng.standard_normal((heads, n, d)).astype(np.float32)).cuda().to(torch.bfloat16)
    v = torch.from_numpy(rng.standard_normal((heads, n, d)).astype(np.float32)).cuda().to(torch.bfloat16)
    scores = rng.standard_normal((heads, g, g))
    kv = None
    if key_valid:
        kv = rng.random(n) < 0.7
        kv[p:2 * p] = False  # one key block fully invalid
    return q, k, v, scores, kv


@pytest.mark.parametrize("g,p,d,force_portable", [(40, 64, 128, False), (40, 64, 128, True), (30, 16, 64, False),
                                                   (20, 128, 64, False), (25, 64, 128, False), (12, 256, 128, False),
                                                   (12, 256, 128, True), (8, 512, 128, False)])
def test_block_sparse_seam_vs_oracle(g, p, d, force_portable):
    q, k, v, scores, _ = _seam_case(g, p, d, 2, 0.3, g + p + d)
    mask = da.select_top_fraction(torch.from_numpy(scores).cuda(), 0.3, True)
    out = da.block_sparse_attention(q, k, v, mask, force_portable=force_portable).float().cpu().numpy()
    q64, k64, v64 = (t.double().cpu().numpy() for t in (q, k, v))
    kept = mask.kept.cpu().numpy()
    for h in range(2):
        ref = O.block_sparse_attention(q64[h], k64[h], v64[h], kept[h], O.head_dim_scale(d))
        _close(out[h], ref)


def test_block_sparse_key_valid_and_dropped_rows():
    g, p, d = 24, 64, 128
    q, k, v, scores, kv = _seam_case(g, p, d, 1, 0.3, 9, key_valid=True)
    scores[0, 5, :] = -1e9  # row 5 never selected ...
    mask = da.select_top_fraction(torch.from_numpy(scores).cuda(), 0.3, False)  # ... and not forced
    out = da.block_sparse_attention(q, k, v, mask, key_valid=torch.from_numpy(kv)).float().cpu().numpy()
    q64, k64, v64 = (t.double().cpu().numpy() for t in (q, k, v))
    ref = O.block_sparse_attention(q64[0], k64[0], v64[0], mask.kept.cpu().numpy()[0], O.head_dim_scale(d),
                                   key_valid=kv)
    assert np.all(out[0][5 * p:6 * p] == 0.0)
    _close(out[0], ref)


@pytest.mark.parametrize("p,key_valid", [(64, False), (128, False), (128, True)])
def test_tcgen05_matches_portable_kernel(p, key_valid):
    # p = 128: the tcgen05 kernel runs the regions as their two 64-token halves
    q, k, v, scores, kv = _seam_case(48, p, 128, 3, 0.2, 17 + p, key_valid=key_valid)
    mask = da.select_top_fraction(torch.from_numpy(scores).cuda(), 0.2, True)
    kv_t = None if kv is None else torch.from_numpy(kv).cuda()
    a = da.block_sparse_attention(q, k, v, mask, key_valid=kv_t).float()
    b = da.block_sparse_attention(q, k, v, mask, key_valid=kv_t, force_portable=True).float()
    assert (a - b).abs().max().item() <= 4e-3


@pytest.mark.parametrize("shared,select_on,qmul", [(True, "logits", 1.0), (False, "softmax", 1.0), (True, "softmax", 1.0),
                                                   (False, "logits", 40.0)])
def test_8x16_pools_shared_softmax_and_fallback_rows_vs_oracle(shared, select_on, qmul):
    # 8x16 pools on the tcgen05 half-regions with the other selection options,
    # and with large logits (rows whose fixed offset underflows are recomputed
    # region-wise by the portable kernel at the 128-token geometry)
    dims = (2, 20, 40, 8, 16)
    plan = da.pad_plan(*dims)
    rng = np.random.default_rng(int(qmul) + (2 if shared else 0) + (1 if select_on == "softmax" else 0))
    q, k, v = (torch.from_numpy(rng.standard_normal((2, plan.num_valid, 128))).float().cuda() for _ in range(3))
    q, k, v = (q * qmul).to(torch.bfloat16), k.to(torch.bfloat16), v.to(torch.bfloat16)
    q64, k64, v64 = (x.double().cpu().numpy() for x in (q, k, v))
    res = da.multi_head_sparse_attention(q, k, v, plan, 0.8, shared_head_mask=shared, select_on=select_on,
                                         return_details=True)
    ref = O.multi_head_sparse_attention(q64, k64, v64, *dims, 0.8, shared_head_mask=shared, select_on=select_on)
    out = res.output.float().cpu().numpy()
    for hh in range(2):
        _close(out[hh], ref[hh], max_abs=1e-2 * max(1.0, float(np.abs(ref[hh]).max())))
    assert torch.equal(da.multi_head_sparse_attention(q, k, v, plan, 0.8, shared_head_mask=shared,
                                                      select_on=select_on), res.output)  # deterministic


@pytest.mark.parametrize("dims", [(2, 16, 48, 8, 16), (3, 45, 80, 8, 16), (2, 20, 72, 8, 16), (2, 12, 20, 8, 16),
                                  (2, 13, 37, 8, 16), (2, 24, 40, 4, 16), (2, 21, 40, 16, 4),
                                  # 256- and 512-token regions: four / eight column parts on tcgen05; the
                                  # portable kernel runs them in query chunks
                                  (2, 32, 48, 16, 16), (2, 16, 64, 8, 32), (2, 20, 72, 16, 32), (2, 16, 48, 16, 8)])
def test_pipeline_tcgen05_matches_portable_other_pools(dims):
    # the paper's 8x16 pools (half-regions on tcgen05) and other 64-token pool
    # shapes, padded grids included: same masks, outputs within the bf16 tolerance
    from paper_2505_14708_b200 import api

    plan = da.pad_plan(*dims)
    g = torch.Generator(device="cuda").manual_seed(sum(dims))
    q, k, v = (torch.randn(3, plan.num_valid, 128, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
    scale = da.head_dim_scale(128)
    a, ma, _ = api._pipeline(q, k, v, plan, 0.85, scale, "average", "logits", True, False, "hnd")
    b, mb, _ = api._pipeline(q, k, v, plan, 0.85, scale, "average", "logits", True, False, "hnd", force_portable=True)
    for h in range(3):
        assert ma.head(h).bitmap_bytes() == mb.head(h).bitmap_bytes()
    # the stated output tolerance: one bf16 rounding apart is 7.8e-3 at |o| >= 1
    assert (a.float() - b.float()).abs().max().item() <= 1e-2
    assert torch.nn.functional.cosine_similarity(a.float().flatten(), b.float().flatten(), dim=0).item() >= 0.9999


def test_extreme_logits_stay_finite():
    # test_sparse.py:204-211: huge logits must not overflow (rescale path)
    q, k, v, scores, _ = _seam_case(16, 64, 128, 1, 0.5, 21)
    q = (q.float() * 40).to(torch.bfloat16)
    mask = da.select_top_fraction(torch.from_numpy(scores).cuda(), 0.5, True)
    out = da.block_sparse_attention(q, k, v, mask).float()
    assert torch.isfinite(out).all()
    q64, k64, v64 = (t.double().cpu().numpy() for t in (q, k, v))
    ref = O.block_sparse_attention(q64[0], k64[0], v64[0], mask.kept.cpu().numpy()[0], O.head_dim_scale(128))
    _close(out.cpu().numpy()[0], ref, max_abs=3e-2, min_cos=0.999)


def test_zero_sparsity_equals_dense():
    # test_sparse.py:241-247 / test_padding.py:138-145 on a ragged grid
    grid = O.Grid(2, 13, 16, 8, 8)
    plan = da.pad_plan(2, 13, 16, 8, 8)
    g = torch.Generator(device="cuda").manual_seed(0)
    q, k, v = (torch.randn(2, grid.n_real, 128, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
    out = da.multi_head_sparse_attention(q, k, v, plan, 0.0).float()
    ref = torch.nn.functional.scaled_dot_product_attention(q.float(), k.float(), v.float())
    _close(out.cpu().numpy(), ref.cpu().numpy())


def test_shared_head_mask_and_softmax_selection():
    z = (4, 16, 16, 4, 4, 64, 3, 7)
    grid, (q, k, v), (q64, k64, v64) = _inputs(z)
    lay = da.LatentLayout(4, 16, 16, 4, 4)
    out = da.multi_head_sparse_attention(q, k, v, lay, 0.6, shared_head_mask=True).float().cpu().numpy()
    ref = O.multi_head_sparse_attention(q64, k64, v64, 4, 16, 16, 4, 4, 0.6, shared_head_mask=True)
    _close(out, ref)
    out = da.multi_head_sparse_attention(q, k, v, lay, 0.6, select_on="softmax").float().cpu().numpy()
    ref = O.multi_head_sparse_attention(q64, k64, v64, 4, 16, 16, 4, 4, 0.6, select_on="softmax")
    _close(out, ref)
    out = da.multi_head_sparse_attention(q, k, v, lay, 0.6, pool_mode="max").float().cpu().numpy()
    ref = O.multi_head_sparse_attention(q64, k64, v64, 4, 16, 16, 4, 4, 0.6, pool_mode="max")
    _close(out, ref)


def test_nhd_layout_and_dtype_roundtrip():
    grid, (q, k, v), _ = _inputs((2, 45, 80, 8, 8, 128, 3, 4))
    plan = da.pad_plan(2, 45, 80, 8, 8)
    ref = da.multi_head_sparse_attention(q, k, v, plan, 0.8)
    nhd = da.multi_head_sparse_attention(q.transpose(0, 1), k.transpose(0, 1), v.transpose(0, 1), plan, 0.8,
                                         qkv_layout="nhd")
    assert nhd.shape == (grid.n_real, 3, 128)
    assert torch.equal(nhd.transpose(0, 1), ref)
    f32 = da.multi_head_sparse_attention(q.float(), k.float(), v.float(), plan, 0.8)
    assert f32.dtype == torch.float32 and torch.equal(f32.to(torch.bfloat16), ref)


def test_deterministic():
    grid, (q, k, v), _ = _inputs((3, 45, 80, 8, 8, 128, 2, 5))
    plan = da.pad_plan(3, 45, 80, 8, 8)
    a = da.multi_head_sparse_attention(q, k, v, plan, 0.9)
    b = da.multi_head_sparse_attention(q, k, v, plan, 0.9)
    assert torch.equal(a, b)


def test_host_inputs_pipelined_by_head_group_match_device_call():
    # reference calling convention: host tensors in, host tensor out; head
    # groups overlap upload / compute / download and must not change results
    grid, (q, k, v), _ = _inputs((2, 45, 80, 8, 8, 128, 6, 0), head_ids=None)
    plan = da.pad_plan(2, 45, 80, 8, 8)
    dev = da.multi_head_sparse_attention(q, k, v, plan, 0.9, return_details=True)
    qh, kh, vh = (x.cpu().pin_memory() for x in (q, k, v))
    host = da.multi_head_sparse_attention(qh, kh, vh, plan, 0.9, return_details=True)
    assert host.output.device.type == "cpu"
    assert torch.equal(host.output, dev.output.cpu())
    assert torch.equal(host.mask.bitmap, dev.mask.bitmap)
    assert host.mask.kept_count == dev.mask.kept_count
    single = da.padded_sparse_attention(qh[1], kh[1], vh[1], 2, 45, 80, 8, 8, 0.9)
    assert torch.equal(single, dev.output[1].cpu())
    # float32 host inputs: the output keeps the inputs' dtype (result_type,
    # sparse.py:129-131) and equals the device call on the same values
    qf, kf, vf = (x.float() for x in (qh, kh, vh))
    hf = da.multi_head_sparse_attention(qf, kf, vf, plan, 0.9)
    assert hf.dtype == torch.float32 and hf.device.type == "cpu"
    df = da.multi_head_sparse_attention(qf.cuda(), kf.cuda(), vf.cuda(), plan, 0.9)
    assert torch.equal(hf, df.cpu())
    # caller-provided host output buffer
    buf = torch.empty_like(host.output).pin_memory()
    o2 = da.multi_head_sparse_attention(qh, kh, vh, plan, 0.9, out=buf)
    assert o2.data_ptr() == buf.data_ptr() and torch.equal(buf, dev.output.cpu())


@pytest.mark.parametrize("kind", ["zeros", "constant_rows", "nan_row"])
def test_pipeline_selection_fallback_cases(kind):
    # massive ties (every score equal) overflow the fp32 guard band and
    # non-finite inputs skip it: the gated fp64 selection must then produce
    # the reference mask (masking.py:59-91 tie rule, np.argmax first max)
    grid, (q, k, v), _ = _inputs((2, 45, 80, 8, 8, 128, 2, 3), head_ids=None)
    if kind == "zeros":
        q = torch.zeros_like(q)
    elif kind == "constant_rows":
        k = torch.ones_like(k)
    plan = da.pad_plan(2, 45, 80, 8, 8)
    if kind == "nan_row":
        q = q.clone()
        q[1, 7] = float("nan")
    res = da.multi_head_sparse_attention(q, k, v, plan, 0.9, return_details=True)
    q64, k64, v64 = (t.double().cpu().numpy() for t in (q, k, v))
    for h in range(2):
        ref, _ = O.draft_mask(q64[h], k64[h], grid, 0.9)
        got = res.mask.head(h)
        assert got.bitmap_bytes() == O.mask_bitmap(ref.kept), (kind, h)
        assert got.kept_count == ref.kept_count and got.forced_row_keeps == ref.forced_row_keeps


@pytest.mark.parametrize("dims", [(1, 12, 20, 4, 4, 32, 3, 7), (3, 40, 24, 8, 8, 128, 3, 8),
                                  (3, 17, 20, 8, 8, 128, 2, 9)])
def test_pipeline_odd_region_counts(dims):
    # g odd (15, 45, 27 - the last one also ragged on both axes): per-head score
    # planes are not 16-byte aligned at g * g, and rows are not either
    grid, (q, k, v), (q64, k64, v64) = _inputs(dims)
    f, h, w, ph, pw = dims[:5]
    plan = da.pad_plan(f, h, w, ph, pw)
    res = da.multi_head_sparse_attention(q, k, v, plan, 0.75, return_details=True)
    out = res.output.float().cpu().numpy()
    for hh in range(q.shape[0]):
        ref = O.padded_sparse_attention(q64[hh], k64[hh], v64[hh], f, h, w, ph, pw, 0.75, return_details=True)
        got = res.mask.head(hh)
        assert got.bitmap_bytes() == O.mask_bitmap(ref.mask.kept), hh
        assert got.kept_count == ref.mask.kept_count and got.forced_row_keeps == ref.mask.forced_row_keeps
        _close(out[hh], ref.output)


@pytest.mark.parametrize("sparsity", [0.995, 0.97])
def test_pipeline_without_force_keep_empty_and_short_rows(sparsity):
    # force_row_keep off at high sparsity: many query regions keep 0, 1 or 2
    # key regions (empty items are zero-filled by K4's producer, one-step
    # items leave one TMEM lane half unused)
    grid, (q, k, v), (q64, k64, v64) = _inputs((3, 45, 80, 8, 8, 128, 2, 11))
    plan = da.pad_plan(3, 45, 80, 8, 8)
    res = da.multi_head_sparse_attention(q, k, v, plan, sparsity, force_row_keep=False, return_details=True)
    out = res.output.float().cpu().numpy()
    for hh in range(2):
        ref = O.padded_sparse_attention(q64[hh], k64[hh], v64[hh], 3, 45, 80, 8, 8, sparsity,
                                        force_row_keep=False, return_details=True)
        got = res.mask.head(hh)
        assert got.bitmap_bytes() == O.mask_bitmap(ref.mask.kept)
        counts = ref.mask.kept.sum(1)
        assert (counts == 0).any() and (counts == 1).any()
        _close(out[hh], ref.output)


def test_zero_sparsity_long_lists_equal_dense():
    # g = 4800 regions (80 frames): every kept list (4800 key regions) exceeds
    # K4's staged-list capacity, so the producer reads the list from global
    # memory; at sparsity 0 the result is dense attention
    f, h, w = 80, 45, 80
    plan = da.pad_plan(f, h, w, 8, 8)
    n = plan.num_valid
    g = torch.Generator(device="cuda").manual_seed(3)
    q, k, v = (torch.randn(1, n, 128, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
    out = da.multi_head_sparse_attention(q, k, v, plan, 0.0).float()
    # dense reference: bf16 flash attention (fp32 math would need the full n x n matrix)
    ref = torch.nn.functional.scaled_dot_product_attention(q[None], k[None], v[None])[0].float()
    _close(out.cpu().numpy(), ref.cpu().numpy())


@pytest.mark.parametrize("kind,expect_fallback", [("gaussian", False), ("zeros", True)])
def test_selection_fast_path_decides_the_mask(kind, expect_fallback):
    # the fp32 guard-band selection must decide ordinary masks itself (the
    # fp64 path it hands over to is correct but ~4x slower, so a too-wide band
    # would pass every parity test): check the device flag
    from paper_2505_14708_b200 import api
    grid, (q, k, v), _ = _inputs((4, 45, 80, 8, 8, 128, 3, 4), head_ids=None)
    if kind == "zeros":
        q = torch.zeros_like(q)
    plan = da.pad_plan(4, 45, 80, 8, 8)
    dbg = {}
    api._pipeline(q, k, v, plan, 0.9, da.head_dim_scale(128), "average", "logits", True, False, "hnd", debug=dbg)
    assert dbg["selection_fallback"] == expect_fallback


@pytest.mark.parametrize("dims", [(2, 16, 48, 4, 16, 128, 2, 12), (3, 24, 40, 8, 8, 64, 2, 13),
                                  (2, 16, 48, 8, 16, 128, 2, 14), (2, 20, 40, 8, 16, 128, 2, 15)])
def test_pipeline_other_pools_and_head_dims(dims):
    # 64-token regions that are not 8x8 (4x16), and d = 64 with 8x8 pools:
    # shapes the tcgen05 kernels do not take (the portable executor runs)
    grid, (q, k, v), (q64, k64, v64) = _inputs(dims)
    f, h, w, ph, pw = dims[:5]
    plan = da.pad_plan(f, h, w, ph, pw)
    res = da.multi_head_sparse_attention(q, k, v, plan, 0.8, return_details=True)
    out = res.output.float().cpu().numpy()
    for hh in range(q.shape[0]):
        ref = O.padded_sparse_attention(q64[hh], k64[hh], v64[hh], f, h, w, ph, pw, 0.8, return_details=True)
        got = res.mask.head(hh)
        assert got.bitmap_bytes() == O.mask_bitmap(ref.mask.kept)
        _close(out[hh], ref.output)


@pytest.mark.parametrize("shared,select_on", [(True, "logits"), (False, "softmax"), (True, "softmax")])
def test_720p_slice_shared_mask_and_softmax_selection(shared, select_on):
    # the fp64 selection paths (head-mean basis, row-softmax basis) feeding the
    # lane-half K4 on the 8x8 / d = 128 shape
    grid, (q, k, v), (q64, k64, v64) = _inputs((2, 45, 80, 8, 8, 128, 3, 14))
    plan = da.pad_plan(2, 45, 80, 8, 8)
    out = da.multi_head_sparse_attention(q, k, v, plan, 0.85, shared_head_mask=shared, select_on=select_on)
    ref = O.multi_head_sparse_attention(q64, k64, v64, 2, 45, 80, 8, 8, 0.85, shared_head_mask=shared,
                                        select_on=select_on)
    _close(out.float().cpu().numpy(), ref)


# ---------------------------------------------------------------- public entries, stats, layouts

def _same_stats(got, want):
    # mask_density_stats (masking.py:128-141): everything exact but the
    # threshold's last bits (dot-product summation order)
    assert set(got) == set(want)
    for key in want:
        if key == "threshold":
            assert abs(got[key] - want[key]) <= 1e-12 * max(1.0, abs(want[key]))
        else:
            assert got[key] == want[key], key


def test_draft_sparse_attention_tiny_vs_reference():
    # configs[0] through the divisible-grid entry (sparse.py:193-246), per head,
    # with its details (FlopsReport, mask stats) against the oracle's
    z = _npz("tiny")
    grid, (q, k, v), (q64, k64, v64) = _inputs(z["dims"])
    lay = da.LatentLayout(grid.frames, grid.height, grid.width, grid.patch_h, grid.patch_w)
    for h in range(q.shape[0]):
        res = da.draft_sparse_attention(q[h], k[h], v[h], lay, float(z["sparsity"]), return_details=True)
        _check_mask(res.mask, 0, z, f"h{h}")
        _close(res.output.float().cpu().numpy(), z[f"h{h}_out"])
        ref = O.padded_sparse_attention(q64[h], k64[h], v64[h], grid.frames, grid.height, grid.width,
                                        grid.patch_h, grid.patch_w, float(z["sparsity"]), return_details=True)
        _same_stats(res.mask_stats, ref.mask_stats)
        assert res.flops.as_dict() == ref.flops


def test_mask_density_stats_vs_oracle():
    # masking.py:128-141 on the 720p slice, every head
    grid, (q, k, v), (q64, k64, _) = _inputs((3, 45, 80, 8, 8, 128, 3, 21))
    plan = da.pad_plan(3, 45, 80, 8, 8)
    res = da.multi_head_sparse_attention(q, k, v, plan, 0.8, return_details=True)
    for h in range(3):
        ref, _ = O.draft_mask(q64[h], k64[h], grid, 0.8)
        got = da.mask_density_stats(res.mask, h)
        _same_stats(got, O.mask_stats(ref))
        assert res.mask_stats[h] == got


@pytest.mark.parametrize("d,dv,p", [(128, 64, 64), (64, 128, 16), (128, 32, 64), (128, 128, 128)])
def test_block_sparse_seam_dv_differs_from_d(d, dv, p):
    # test_sparse.py:193-202: value width differs from the key width
    g = 24
    rng = np.random.default_rng(d + dv + p)
    n = g * p
    q = torch.from_numpy(rng.standard_normal((2, n, d)).astype(np.float32)).cuda().to(torch.bfloat16)
    k = torch.from_numpy(rng.standard_normal((2, n, d)).astype(np.float32)).cuda().to(torch.bfloat16)
    v = torch.from_numpy(rng.standard_normal((2, n, dv)).astype(np.float32)).cuda().to(torch.bfloat16)
    mask = da.select_top_fraction(torch.from_numpy(rng.standard_normal((2, g, g))).cuda(), 0.3, True)
    out = da.block_sparse_attention(q, k, v, mask).float().cpu().numpy()
    assert out.shape == (2, n, dv)
    q64, k64, v64 = (t.double().cpu().numpy() for t in (q, k, v))
    kept = mask.kept.cpu().numpy()
    for h in range(2):
        _close(out[h], O.block_sparse_attention(q64[h], k64[h], v64[h], kept[h], O.head_dim_scale(d)))


def test_pipeline_dv_differs_from_d():
    grid, (q, k, _), (q64, k64, _) = _inputs((2, 13, 10, 4, 4, 32, 2, 22))
    v = torch.randn(2, grid.n_real, 48, device="cuda").to(torch.bfloat16)
    v64 = v.double().cpu().numpy()
    plan = da.pad_plan(2, 13, 10, 4, 4)
    out = da.multi_head_sparse_attention(q, k, v, plan, 0.6).float().cpu().numpy()
    for h in range(2):
        ref = O.padded_sparse_attention(q64[h], k64[h], v64[h], 2, 13, 10, 4, 4, 0.6)
        _close(out[h], ref)


def test_head_dims_not_multiple_of_8():
    # the reference's own grids use d in {4, 16, 64} (gridutil.py:9-34); d = 4
    # and d = 12 run zero-padded to 8 / 16 features (exact)
    for d in (4, 12):
        grid, (q, k, v), (q64, k64, v64) = _inputs((2, 8, 12, 4, 4, d, 2, 23))
        plan = da.pad_plan(2, 8, 12, 4, 4)
        res = da.multi_head_sparse_attention(q, k, v, plan, 0.5, return_details=True)
        assert res.output.shape == (2, grid.n_real, d)
        for h in range(2):
            ref = O.padded_sparse_attention(q64[h], k64[h], v64[h], 2, 8, 12, 4, 4, 0.5, return_details=True)
            assert res.mask.head(h).bitmap_bytes() == O.mask_bitmap(ref.mask.kept)
            _close(res.output[h].float().cpu().numpy(), ref.output)
        # the lower seams accept the same widths
        xr = da.reorder_tokens(q, plan)
        assert xr.shape[-1] == d
        assert torch.equal(da.restore_tokens(xr, plan), q)
        pooled = da.pool_tokens(q, plan).cpu().numpy()
        assert np.array_equal(pooled[0], O.pool_valid(O.permute_in(q64[0], grid), O.valid_reordered(grid), 16))


def test_bnhd_batched_layout_equals_per_element_calls():
    # (batch, n, heads, d) DiT inputs: one call per batch element, no copies
    plan = da.pad_plan(2, 45, 80, 8, 8)
    gen = torch.Generator(device="cuda").manual_seed(7)
    q, k, v = (torch.randn(2, plan.num_valid, 3, 128, device="cuda", generator=gen).to(torch.bfloat16)
               for _ in range(3))
    res = da.multi_head_sparse_attention(q, k, v, plan, 0.85, qkv_layout="bnhd", return_details=True)
    assert res.output.shape == (2, plan.num_valid, 3, 128) and res.mask.heads == 6
    for b in range(2):
        ref = da.multi_head_sparse_attention(q[b], k[b], v[b], plan, 0.85, qkv_layout="nhd", return_details=True)
        assert torch.equal(res.output[b], ref.output)
        for h in range(3):
            assert res.mask.head(3 * b + h).bitmap_bytes() == ref.mask.head(h).bitmap_bytes()
    # host inputs, the same layout
    host = da.multi_head_sparse_attention(q.cpu(), k.cpu(), v.cpu(), plan, 0.85, qkv_layout="bnhd")
    assert host.device.type == "cpu" and torch.equal(host, res.output.cpu())


def test_nhd_host_out_buffer():
    # out= in the caller's (n, heads, dv) layout (host inputs)
    grid, (q, k, v), _ = _inputs((2, 45, 80, 8, 8, 128, 3, 24))
    plan = da.pad_plan(2, 45, 80, 8, 8)
    qn, kn, vn = (x.transpose(0, 1).contiguous() for x in (q, k, v))
    ref = da.multi_head_sparse_attention(qn, kn, vn, plan, 0.8, qkv_layout="nhd")
    buf = torch.empty(plan.num_valid, 3, 128, dtype=torch.bfloat16).pin_memory()
    got = da.multi_head_sparse_attention(qn.cpu(), kn.cpu(), vn.cpu(), plan, 0.8, qkv_layout="nhd", out=buf)
    assert got.data_ptr() == buf.data_ptr() and torch.equal(buf, ref.cpu())


def test_cached_mask_through_json_reproduces_the_call():
    # the mask wire format as a cache: export a call's mask, re-import it and
    # run the executor seam on reordered tensors with it
    grid, (q, k, v), _ = _inputs((2, 45, 80, 8, 8, 128, 2, 25))
    plan = da.pad_plan(2, 45, 80, 8, 8)
    res = da.multi_head_sparse_attention(q, k, v, plan, 0.9, return_details=True)
    for h in range(2):
        m = da.mask_from_json_dict(da.mask_to_json_dict(res.mask, h))
        assert m.bitmap_bytes() == res.mask.head(h).bitmap_bytes()
        kv = torch.from_numpy(O.valid_reordered(grid))
        o_r = da.block_sparse_attention(da.reorder_tokens(q[h], plan), da.reorder_tokens(k[h], plan),
                                        da.reorder_tokens(v[h], plan), m, key_valid=kv)
        got = da.restore_tokens(o_r, plan)
        assert (got.float() - res.output[h].float()).abs().max().item() <= 4e-3


@pytest.mark.gpu
def test_smooth_inputs_720p_slice_masks_and_outputs():
    # the reference's secondary data mode (smooth per-frame fields: patches
    # nearly uniform, neighbouring regions alike, so many near-equal draft
    # scores) through the full pipeline: masks identical, outputs within bars
    grid = O.Grid(2, 45, 80, 8, 8)
    q, k, v = O.gen_real_inputs(grid, 128, 11, 2, mode="smooth")
    tq, tk, tv = (torch.from_numpy(x).to("cuda").to(torch.bfloat16) for x in (q, k, v))
    plan = da.pad_plan(2, 45, 80, 8, 8)
    res = da.multi_head_sparse_attention(tq, tk, tv, plan, 0.9, return_details=True)
    out = res.output.float().cpu().numpy()
    for h in range(2):
        ref = O.padded_sparse_attention(tq[h].double().cpu().numpy(), tk[h].double().cpu().numpy(),
                                        tv[h].double().cpu().numpy(), 2, 45, 80, 8, 8, 0.9, return_details=True)
        got = res.mask.head(h)
        assert got.bitmap_bytes() == O.mask_bitmap(ref.mask.kept)
        assert int(got.kept_count) == int(ref.mask.kept.sum())
        assert int(got.forced_row_keeps) == int(ref.mask.forced_row_keeps)
        _close(out[h], ref.output)


@pytest.mark.gpu
@pytest.mark.parametrize("shared", [False, True])
def test_cached_mask_on_original_order_equals_the_call(shared):
    # mask reuse across denoising steps: the executor alone on original-order
    # tensors with a cached (JSON round-tripped) mask reproduces the full call
    grid, (q, k, v), _ = _inputs((2, 45, 80, 8, 8, 128, 3, 27))
    plan = da.pad_plan(2, 45, 80, 8, 8)
    res = da.multi_head_sparse_attention(q, k, v, plan, 0.9, shared_head_mask=shared, return_details=True)
    if shared:
        mask = da.mask_from_json_dict(da.mask_to_json_dict(res.mask, 0))
    else:
        mask = res.mask
    got = da.padded_block_sparse_attention(q, k, v, plan, mask)
    assert got.shape == res.output.shape and got.dtype == res.output.dtype
    assert (got.float() - res.output.float()).abs().max().item() <= 4e-3
    # (n, heads, d) DiT layout, and one head as (n, d)
    got_nhd = da.padded_block_sparse_attention(q.transpose(0, 1), k.transpose(0, 1), v.transpose(0, 1), plan,
                                               mask, qkv_layout="nhd")
    assert torch.equal(got_nhd.transpose(0, 1), got)
    one = da.padded_block_sparse_attention(q[1], k[1], v[1], plan, mask if shared else res.mask.head(1))
    assert torch.equal(one, got[1])


def _random_configs(count, seed=2024):
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < count:
        ph, pw = [(4, 4), (8, 8), (4, 8), (8, 4), (2, 8)][rng.integers(5)]
        f = int(rng.integers(1, 4))
        h = int(rng.integers(ph, 6 * ph))
        w = int(rng.integers(pw, 6 * pw))
        d = int([8, 16, 36, 64, 128][rng.integers(5)])
        heads = int(rng.integers(1, 4))
        sp = float(rng.choice([0.0, 0.3, 0.5, 0.75, 0.9, 0.97]))
        out.append((f, h, w, ph, pw, d, heads, sp, int(rng.integers(1 << 30))))
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("cfg", _random_configs(48))
def test_random_shapes_vs_oracle(cfg):
    # random grids (ragged and divisible), pools, head dims (incl. d % 8 != 0),
    # head counts and sparsities through the full pipeline: masks identical,
    # outputs within the bars
    f, h, w, ph, pw, d, heads, sp, seed = cfg
    grid = O.Grid(f, h, w, ph, pw)
    q, k, v = O.gen_real_inputs(grid, d, seed % 100000, heads)
    tq, tk, tv = (torch.from_numpy(x).to("cuda").to(torch.bfloat16) for x in (q, k, v))
    plan = da.pad_plan(f, h, w, ph, pw)
    res = da.multi_head_sparse_attention(tq, tk, tv, plan, sp, return_details=True)
    out = res.output.float().cpu().numpy()
    for hh in range(heads):
        ref = O.padded_sparse_attention(tq[hh].double().cpu().numpy(), tk[hh].double().cpu().numpy(),
                                        tv[hh].double().cpu().numpy(), f, h, w, ph, pw, sp, return_details=True)
        got = res.mask.head(hh)
        assert got.bitmap_bytes() == O.mask_bitmap(ref.mask.kept), cfg
        assert int(got.forced_row_keeps) == int(ref.mask.forced_row_keeps), cfg
        _close(out[hh], ref.output)


@pytest.mark.gpu
@pytest.mark.parametrize("frames,sparsity", [(129, 0.9), (65, 0.97)])
def test_long_video_masks_vs_oracle(frames, sparsity):
    # longer clips than the paper's 720p shapes (129 frames: 464,400 tokens,
    # g = 7,740 regions, 60 M draft scores per head): the fp32 selection, its
    # guard band and the lane-half executor at that size; masks bit-identical
    grid = O.Grid(frames, 45, 80, 8, 8)
    q, k, v = O.gen_real_inputs(grid, 128, 31, 1)
    tq, tk, tv = (torch.from_numpy(x).to("cuda").to(torch.bfloat16) for x in (q, k, v))
    plan = da.pad_plan(frames, 45, 80, 8, 8)
    res = da.multi_head_sparse_attention(tq, tk, tv, plan, sparsity, return_details=True)
    ref, _ = O.draft_mask(tq[0].double().cpu().numpy(), tk[0].double().cpu().numpy(), grid, sparsity)
    got = res.mask.head(0)
    assert got.bitmap_bytes() == O.mask_bitmap(ref.kept)
    assert int(got.kept_count) == int(ref.kept.sum())
    assert float(got.threshold) == pytest.approx(ref.threshold, rel=1e-12)
    out = res.output.float()
    assert torch.isfinite(out).all() and out.abs().max().item() < 10.0


@pytest.mark.gpu
@pytest.mark.parametrize("config", ["wan720", "hv720_smooth"])
def test_full_head_outputs_other_headline_data(config):
    # complete output of one whole head of the Wan 720p config (75 %) and of
    # HV720 on the reference's smooth data mode (90 %) against the fp64 oracle
    if config == "wan720":
        dims, sp, mode = (21, 45, 80, 8, 8), 0.75, "gaussian"
    else:
        dims, sp, mode = (33, 45, 80, 8, 8), 0.9, "smooth"
    grid = O.Grid(*dims)
    q, k, v = O.gen_real_inputs(grid, 128, 5, 40 if config == "wan720" else 24, head_ids=[7], mode=mode)
    tq, tk, tv = (torch.from_numpy(x).to("cuda").to(torch.bfloat16) for x in (q, k, v))
    plan = da.pad_plan(*dims)
    res = da.multi_head_sparse_attention(tq, tk, tv, plan, sp, return_details=True)
    ref = O.padded_sparse_attention(tq[0].double().cpu().numpy(), tk[0].double().cpu().numpy(),
                                    tv[0].double().cpu().numpy(), *dims, sp, return_details=True)
    got = res.mask.head(0)
    assert got.bitmap_bytes() == O.mask_bitmap(ref.mask.kept)
    rep = _full_output_report(res.output[0].float().cpu().numpy(), ref.output, grid)
    print(f"{config} head 7 sparsity {sp}: {rep}")
    assert rep["max_abs"] <= MAX_ABS and rep["cosine"] >= MIN_COS, rep
    assert rep["min_row_cosine"] >= 0.999, rep


@pytest.mark.gpu
def test_repeated_calls_bit_identical():
    # the persistent K4 claims items dynamically and its roles hand work over
    # through mbarrier rings: any ordering race would show up as run-to-run
    # differences. Full HV720 calls (24 heads) and many small calls, all
    # bit-identical.
    torch.manual_seed(3)
    plan = da.pad_plan(33, 45, 80, 8, 8)
    q, k, v = (torch.randn(24, plan.num_valid, 128, device="cuda").to(torch.bfloat16) for _ in range(3))
    ref = da.multi_head_sparse_attention(q, k, v, plan, 0.9)
    for _ in range(6):
        assert torch.equal(da.multi_head_sparse_attention(q, k, v, plan, 0.9), ref)
    small = da.pad_plan(2, 45, 80, 8, 8)
    qs, ks, vs = (x[:3, :small.num_valid].contiguous() for x in (q, k, v))
    ref_s = da.multi_head_sparse_attention(qs, ks, vs, small, 0.75)
    for _ in range(40):
        assert torch.equal(da.multi_head_sparse_attention(qs, ks, vs, small, 0.75), ref_s)


@pytest.mark.gpu
def test_pipeline_is_cuda_graph_capturable():
    # no host synchronisation or allocation inside the C ABI: one call can be
    # captured into a CUDA graph and replayed (a DiT loop with static buffers)
    from paper_2505_14708_b200 import api

    plan = da.pad_plan(3, 45, 80, 8, 8)
    g = torch.Generator(device="cuda").manual_seed(12)
    q, k, v = (torch.randn(4, plan.num_valid, 128, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
    run = lambda: api._pipeline(q, k, v, plan, 0.9, da.head_dim_scale(128), "average", "logits", True, False, "hnd",
                                want_bitmap=False)[0]
    ref = run().clone()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        run()
    torch.cuda.current_stream().wait_stream(s)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        out = run()
    q.mul_(0.5)  # new contents of the static input buffer
    graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, run())
    q.mul_(2.0)
    graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, ref)
