"""Generate the golden fixtures from the UNMODIFIED reference package.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py

It imports ``draftattn`` from /root/reference/pkg/src (read-only; nothing is
copied) and writes small ``.npz`` fixtures next to this script. The GPU box
never runs this file: the tests there read the committed fixtures only.

Inputs follow the SURVEY §8(c)/(d) recipe: seeded ``synth.gen_inputs`` on the
padded layout (real rows kept as ``cli.cmd_gen`` does), cast to bf16 with
torch (round-to-nearest-even), and handed to the reference as exact float64
upcasts of those bf16 values.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import torch

REF_SRC = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent


def _ref():
    sys.path.insert(0, str(REF_SRC))
    import draftattn  # noqa: PLC0415

    return draftattn


def bf16_round(x: np.ndarray) -> np.ndarray:
    """float32 -> bf16 (RNE, torch) -> exact float64."""
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).to(torch.bfloat16).to(torch.float64).numpy()


def real_inputs(da, frames, height, width, ph, pw, d, seed, heads, head_ids=None):
    """Padded-layout synth inputs, real rows kept (cli.py:77-98), bf16-rounded.

    ``head_ids`` generates only those heads, with the per-head seeds
    gen_inputs would use (SeedSequence(seed).spawn(heads), synth.py:108-110).
    """
    plan = da.pad_plan(frames, height, width, ph, pw)
    if head_ids is None:
        q, k, v = da.gen_inputs(plan.layout, d, seed, "gaussian", np.float32, heads=heads)
        if heads == 1:
            q, k, v = q[None], k[None], v[None]
    else:
        kids = np.random.SeedSequence(seed).spawn(heads)
        trip = [da.gen_gaussian(plan.layout, d, kids[h], np.float32) for h in head_ids]
        q, k, v = (np.stack([t[i] for t in trip]) for i in range(3))
    if not plan.is_identity:
        q, k, v = q[:, plan.valid], k[:, plan.valid], v[:, plan.valid]
    return bf16_round(q), bf16_round(k), bf16_round(v)


def gen_permutations(da):
    """Forward reorder indices and validity for padded and divisible grids."""
    cases = [(1, 2, 4, 2, 2), (2, 4, 8, 2, 4), (2, 3, 5, 2, 4), (3, 45, 80, 8, 8),
             (1, 13, 10, 4, 4), (2, 7, 3, 2, 2), (4, 16, 16, 4, 4), (1, 1, 1, 2, 2)]
    out = {}
    for idx, (f, h, w, ph, pw) in enumerate(cases):
        plan = da.pad_plan(f, h, w, ph, pw)
        perm = da.gen_reorder_index(plan.layout)
        out[f"case{idx}_dims"] = np.array([f, h, w, ph, pw])
        out[f"case{idx}_forward"] = perm.forward
        out[f"case{idx}_valid"] = plan.valid
    np.savez_compressed(OUT / "permutation.npz", **out)


def gen_pooling(da):
    from draftattn.padding import pool_regions_valid  # noqa: PLC0415

    rng = np.random.default_rng(7)
    out = {}
    x = bf16_round(rng.standard_normal((6 * 16, 8)))
    valid = rng.random(6 * 16) < 0.7
    valid[16:32] = False  # one empty region
    out["x"] = x
    out["valid"] = valid
    out["pool_valid"] = pool_regions_valid(x, valid, 16)
    out["pool_avg"] = da.pool_regions(x, 16, "average")
    out["pool_max"] = da.pool_regions(x, 16, "max")
    np.savez_compressed(OUT / "pooling.npz", **out)


def gen_selection(da):
    rng = np.random.default_rng(11)
    out = {}
    idx = 0
    for g in (2, 3, 5, 8, 17, 40):
        for r in (0.1, 0.25, 0.5, 0.9, 1.0):
            for kind in ("normal", "tied", "zeros"):
                if kind == "normal":
                    s = rng.standard_normal((g, g))
                elif kind == "tied":
                    s = np.round(rng.standard_normal((g, g)) * 2) / 2
                else:
                    s = np.zeros((g, g))
                for force in (False, True):
                    m = da.select_top_fraction(s, r, force_row_keep=force)
                    out[f"c{idx}_scores"] = s
                    out[f"c{idx}_meta"] = np.array([r, float(force), m.threshold,
                                                    m.forced_row_keeps, m.kept_count])
                    out[f"c{idx}_bitmap"] = np.frombuffer(da.masking.mask_to_bitmap(m), np.uint8)
                    idx += 1
    out["count"] = np.array(idx)
    np.savez_compressed(OUT / "selection.npz", **out)


def gen_wire(da):
    """Mask wire formats (masking.py:128-176): the reference's JSON export and
    density stats of a few selections, as JSON next to their score matrices."""
    import json  # noqa: PLC0415

    from draftattn.masking import mask_density_stats, mask_to_json_dict  # noqa: PLC0415

    rng = np.random.default_rng(13)
    cases = []
    for g, r, force, tied in ((3, 0.5, True, False), (8, 0.25, False, True), (17, 0.1, True, False),
                              (40, 0.3, True, True)):
        s = rng.standard_normal((g, g))
        if tied:
            s = np.round(s * 2) / 2
        m = da.select_top_fraction(s, r, force_row_keep=force)
        cases.append({"scores": s.tolist(), "keep_ratio": r, "force_row_keep": force,
                      "json": mask_to_json_dict(m), "stats": mask_density_stats(m),
                      "bitmap_hex": da.masking.mask_to_bitmap(m).hex()})
    (OUT / "wire.json").write_text(json.dumps(cases))


def _pipeline_case(da, name, frames, height, width, ph, pw, d, heads, sparsity, seed,
                   sample_rows=None, full_output=True, head_ids=None):
    q, k, v = real_inputs(da, frames, height, width, ph, pw, d, seed, heads, head_ids)
    slots = list(range(heads)) if head_ids is None else list(head_ids)
    out = {"dims": np.array([frames, height, width, ph, pw, d, heads, seed]),
           "sparsity": np.array(sparsity)}
    for slot, h in enumerate(slots):
        if head_ids is not None:
            q_h, k_h, v_h = q[slot], k[slot], v[slot]
        else:
            q_h, k_h, v_h = q[h], k[h], v[h]
        if full_output:
            res = da.padded_sparse_attention(q_h, k_h, v_h, frames, height, width, ph, pw,
                                             sparsity, return_details=True)
            mask, o = res.mask, res.output
            out[f"h{h}_out"] = o
        else:
            mask, o = _sampled_reference(da, q_h, k_h, v_h, frames, height, width, ph, pw,
                                         sparsity, sample_rows)
            out[f"h{h}_rows"] = sample_rows
            out[f"h{h}_out_rows"] = o
        out[f"h{h}_bitmap"] = np.frombuffer(da.masking.mask_to_bitmap(mask), np.uint8)
        out[f"h{h}_meta"] = np.array([mask.threshold, mask.forced_row_keeps, mask.kept_count])
    np.savez_compressed(OUT / f"{name}.npz", **out)


def _sampled_reference(da, q, k, v, frames, height, width, ph, pw, sparsity, region_rows):
    """Reference mask in full, reference executor on a sample of query regions.

    Runs the reference's own stages (padding.py:134-157) with the executor fed
    a RegionMask whose unsampled rows are emptied, which the reference skips
    (sparse.py:137-138); returns real-token output rows of the sampled regions.
    """
    from draftattn.masking import RegionMask, drop_key_regions  # noqa: PLC0415
    from draftattn.padding import embed_rows, pool_regions_valid  # noqa: PLC0415

    plan = da.pad_plan(frames, height, width, ph, pw)
    layout = plan.layout
    scale = da.head_dim_scale(q.shape[1])
    perm = da.gen_reorder_index(layout)
    q_r = da.permute_rows(embed_rows(q, plan), perm)
    k_r = da.permute_rows(embed_rows(k, plan), perm)
    v_r = da.permute_rows(embed_rows(v, plan), perm)
    valid_r = da.permute_rows(plan.valid, perm)
    p = layout.region_size
    basis = da.draft_logits(pool_regions_valid(q_r, valid_r, p), pool_regions_valid(k_r, valid_r, p), scale)
    mask = da.select_top_fraction(basis, 1.0 - sparsity, True)
    dead = np.flatnonzero(valid_r.reshape(layout.num_regions, p).sum(axis=1) == 0)
    if dead.size:
        mask = drop_key_regions(mask, dead)
    sub = np.zeros_like(mask.kept)
    sub[region_rows] = mask.kept[region_rows]
    sub.setflags(write=False)
    sub_mask = RegionMask(kept=sub, keep_ratio=mask.keep_ratio, threshold=mask.threshold)
    out_r = da.block_sparse_attention(q_r, k_r, v_r, sub_mask, scale, key_valid=valid_r)
    rows = (np.asarray(region_rows)[:, None] * p + np.arange(p)[None, :]).reshape(-1)
    return mask, out_r[rows]


def gen_smooth(da):
    """synth.gen_inputs(mode="smooth") on a small padded grid (the reference's
    secondary data mode), to pin the oracle's restatement of the generator."""
    from draftattn import synth
    plan = da.pad_plan(2, 13, 20, 4, 4)
    q, k, v = synth.gen_inputs(plan.layout, 8, 7, mode="smooth", dtype=np.float32, heads=2)
    np.savez_compressed(OUT / "smooth.npz", q=q, k=k, v=v)


def main():
    da = _ref()
    if sys.argv[1:] == ["smooth"]:
        gen_smooth(da)
        return
    gen_smooth(da)
    gen_permutations(da)
    gen_pooling(da)
    gen_selection(da)
    gen_wire(da)
    # the paper's 8x16 pool (p = 128) with d = 128 on a ragged grid, and a head
    # dim that is not a multiple of 8 (the reference's own tests use d = 4)
    _pipeline_case(da, "pool816", 2, 12, 20, 8, 16, 128, 2, 0.75, 5)
    _pipeline_case(da, "d4", 2, 8, 12, 4, 4, 4, 2, 0.5, 6)
    # tiny config (BASELINE configs[0]): divisible grid, draft_sparse_attention path
    _pipeline_case(da, "tiny", 4, 16, 16, 4, 4, 64, 2, 0.5, 0)
    # small ragged grids through the padded path
    _pipeline_case(da, "ragged_small", 2, 13, 10, 4, 4, 32, 3, 0.75, 1)
    _pipeline_case(da, "ragged_w", 1, 8, 11, 4, 4, 16, 2, 0.5, 2)
    # 720p frame geometry on 2 frames, d=128, 8x8 pool, 90%
    rows = np.arange(0, 120, 7)
    _pipeline_case(da, "hv720_f2", 2, 45, 80, 8, 8, 128, 2, 0.9, 3,
                   sample_rows=rows, full_output=False)
    # full HunyuanVideo 720p shape (configs[1]): masks of heads 0 and 1 of 24,
    # executor output on a sample of query regions
    rows = np.array([0, 1, 55, 59, 777, 1234, 1979])
    _pipeline_case(da, "hv720", 33, 45, 80, 8, 8, 128, 24, 0.9, 0,
                   sample_rows=rows, full_output=False, head_ids=[0, 1])


if __name__ == "__main__":
    main()
