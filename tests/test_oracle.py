"""Pin the CPU oracle to the reference (CPU only, no GPU).

Every fixture under tests/golden/ was produced by the UNMODIFIED reference
(tests/golden/make_golden.py). The hand vectors below are the reference's own
known-answer tests (cited per test).
"""

from pathlib import Path

import numpy as np
import pytest

from oracle import draftattn_oracle as O

GOLD = Path(__file__).resolve().parent / "golden"


def _npz(name):
    return np.load(GOLD / f"{name}.npz")


def _bf16_inputs(dims, head_ids=None):
    import torch

    f, h, w, ph, pw, d, heads, seed = (int(x) for x in dims)
    grid = O.Grid(f, h, w, ph, pw)
    q, k, v = O.gen_real_inputs(grid, d, seed, heads, head_ids=head_ids)
    rnd = lambda x: torch.from_numpy(x).to(torch.bfloat16).to(torch.float64).numpy()  # noqa: E731
    return grid, rnd(q), rnd(k), rnd(v)


# ---------------------------------------------------------------- permutation

def test_hand_trace_reorder():
    # test_layout.py:41-43 / test_acceptance.py:194-195
    grid = O.Grid(1, 2, 4, 2, 2)
    assert O.reorder_index(grid).tolist() == [0, 1, 4, 5, 2, 3, 6, 7]


def test_single_patch_is_identity():
    # test_layout.py:45-47
    grid = O.Grid(2, 4, 4, 4, 4)
    np.testing.assert_array_equal(O.reorder_index(grid), np.arange(32))


def test_permutation_fixtures():
    z = _npz("permutation")
    for i in range(8):
        f, h, w, ph, pw = (int(x) for x in z[f"case{i}_dims"])
        grid = O.Grid(f, h, w, ph, pw)
        np.testing.assert_array_equal(O.reorder_index(grid), z[f"case{i}_forward"])
        np.testing.assert_array_equal(O.valid_padded(grid), z[f"case{i}_valid"])
        inv = O.invert(O.reorder_index(grid))
        np.testing.assert_array_equal(O.reorder_index(grid)[inv], np.arange(grid.n_pad))


def test_permute_in_out_round_trip_and_zero_padding():
    grid = O.Grid(2, 3, 5, 2, 4)
    x = np.arange(grid.n_real * 3, dtype=np.float32).reshape(grid.n_real, 3)
    xr = O.permute_in(x, grid)
    assert (xr[~O.valid_reordered(grid)] == 0).all()
    np.testing.assert_array_equal(O.permute_out(xr, grid), x)


# ---------------------------------------------------------------- pooling

def test_pooling_hand_case():
    # test_pooling.py:13-21
    x = np.array([[0, 2], [2, 4], [10, 0], [0, 10]], dtype=np.float64)
    np.testing.assert_array_equal(O.pool_regions(x, 2, "average"), [[1, 3], [5, 5]])
    np.testing.assert_array_equal(O.pool_regions(x, 2, "max"), [[2, 4], [10, 10]])


def test_pooling_fixture_bit_exact():
    z = _npz("pooling")
    np.testing.assert_array_equal(O.pool_valid(z["x"], z["valid"], 16), z["pool_valid"])
    np.testing.assert_array_equal(O.pool_regions(z["x"], 16, "average"), z["pool_avg"])
    np.testing.assert_array_equal(O.pool_regions(z["x"], 16, "max"), z["pool_max"])


# ---------------------------------------------------------------- selection

@pytest.mark.parametrize("n,r,expected", [(100, 0.1, 10), (100, 0.25, 25), (100, 0.101, 11),
                                          (9, 0.5, 5), (4, 1.0, 4), (16, 0.001, 1)])
def test_top_fraction_count_table(n, r, expected):
    # test_masking.py:25-34
    assert O.top_fraction_count(n, r) == expected


def test_top_fraction_count_float_guard():
    # test_masking.py:36-39
    for g2 in (100, 400, 1600, 3600, 240 * 240):
        assert O.top_fraction_count(g2, 0.1) == g2 // 10


def test_selection_hand_cases():
    # test_masking.py:59-64, :77-81, :95-103
    m = O.select_top_fraction(np.array([[9.0, 1.0], [5.0, 7.0]]), 0.5)
    assert m.kept.tolist() == [[True, False], [False, True]] and m.threshold == 7.0
    m = O.select_top_fraction(np.zeros((3, 3)), 4 / 9)
    assert m.kept.reshape(-1).tolist() == [True] * 4 + [False] * 5
    s = np.full((4, 4), -10.0)
    s[0] = [4.0, 3.0, 2.0, 1.0]
    m = O.select_top_fraction(s, 0.25, force_row_keep=True)
    assert m.forced_row_keeps == 3 and (m.kept.sum(axis=1) >= 1).all()


def test_selection_fixtures_bit_exact():
    z = _npz("selection")
    for i in range(int(z["count"])):
        r, force, thr, forced, kept = z[f"c{i}_meta"]
        m = O.select_top_fraction(z[f"c{i}_scores"], float(r), bool(force))
        assert np.frombuffer(O.mask_bitmap(m.kept), np.uint8).tolist() == z[f"c{i}_bitmap"].tolist()
        assert m.threshold == thr and m.forced_row_keeps == forced and m.kept_count == kept


# ---------------------------------------------------------------- pipelines

@pytest.mark.parametrize("name", ["tiny", "ragged_small", "ragged_w", "pool816", "d4"])
def test_pipeline_fixtures_full(name):
    z = _npz(name)
    grid, q, k, v = _bf16_inputs(z["dims"])
    for h in range(q.shape[0]):
        res = O.padded_sparse_attention(q[h], k[h], v[h], grid.frames, grid.height, grid.width,
                                        grid.patch_h, grid.patch_w, float(z["sparsity"]),
                                        return_details=True)
        assert O.mask_bitmap(res.mask.kept) == z[f"h{h}_bitmap"].tobytes()
        thr, forced, kept = z[f"h{h}_meta"]
        assert res.mask.threshold == thr and res.mask.forced_row_keeps == forced
        assert res.mask.kept_count == kept
        np.testing.assert_allclose(res.output, z[f"h{h}_out"], rtol=0, atol=1e-12)


def test_pipeline_hv720_two_frames_sampled():
    z = _npz("hv720_f2")
    grid, q, k, v = _bf16_inputs(z["dims"])
    p = grid.region_size
    for h in range(q.shape[0]):
        mask, _ = O.draft_mask(q[h], k[h], grid, float(z["sparsity"]))
        assert O.mask_bitmap(mask.kept) == z[f"h{h}_bitmap"].tobytes()
        assert mask.threshold == z[f"h{h}_meta"][0]
        rows = z[f"h{h}_rows"]
        out_r = O.block_sparse_attention(O.permute_in(q[h], grid), O.permute_in(k[h], grid),
                                         O.permute_in(v[h], grid), mask.kept,
                                         O.head_dim_scale(q.shape[2]),
                                         key_valid=O.valid_reordered(grid), rows=rows)
        idx = (rows[:, None] * p + np.arange(p)[None, :]).reshape(-1)
        np.testing.assert_allclose(out_r[idx], z[f"h{h}_out_rows"], rtol=0, atol=1e-12)


@pytest.mark.slow
def test_pipeline_hv720_full_shape_masks():
    z = _npz("hv720")
    grid, q, k, v = _bf16_inputs(z["dims"], head_ids=[0, 1])
    for slot, h in enumerate((0, 1)):
        mask, _ = O.draft_mask(q[slot], k[slot], grid, float(z["sparsity"]))
        assert O.mask_bitmap(mask.kept) == z[f"h{h}_bitmap"].tobytes()
        thr, forced, kept = z[f"h{h}_meta"]
        assert mask.threshold == thr and mask.forced_row_keeps == forced and mask.kept_count == kept


def test_mask_wire_fixtures():
    # masking.py:128-176: the reference's JSON export, density stats and bitmap
    import json

    for case in json.loads((GOLD / "wire.json").read_text()):
        s = np.asarray(case["scores"])
        m = O.select_top_fraction(s, case["keep_ratio"], case["force_row_keep"])
        assert O.mask_bitmap(m.kept).hex() == case["bitmap_hex"]
        assert [list(x) for x in zip(*np.nonzero(m.kept))] == case["json"]["kept"]
        stats = O.mask_stats(m)
        for key, val in case["stats"].items():
            assert stats[key] == val, key


def test_smooth_generator_matches_reference_fixture():
    # synth.gen_inputs(mode="smooth") (synth.py:44-114), the reference's
    # secondary data mode, restated in the oracle: identical float32 values
    z = np.load(GOLD / "smooth.npz")
    q, k, v = O.gen_smooth_heads(O.Grid(2, 13, 20, 4, 4), 8, 7, 2)
    assert np.array_equal(q, z["q"]) and np.array_equal(k, z["k"]) and np.array_equal(v, z["v"])
