"""Attention for a video DiT block (HunyuanVideo / Wan style), on the B200 path.

The reference stops at the attention call; a DiT sampler calls attention once
per block per denoising step with (batch, n, heads, d) tensors over a
frames x height x width latent grid. ``DraftAttention`` is that call:

* steps before ``dense_warmup_steps`` run dense attention (the paper keeps the
  first steps dense; dense is cuDNN / flash SDPA, a library call);
* afterwards each step runs the draft pipeline (pool -> draft scores -> global
  top-fraction -> block-sparse attention, ``multi_head_sparse_attention``), or,
  between mask refreshes (``mask_refresh_every`` > 1), the executor alone with
  the cached mask (``padded_block_sparse_attention``: no pooling / selection).

One instance per attention block (each block has its own mask cache). Inputs
are CUDA tensors; the output has the inputs' layout and dtype.
"""

from __future__ import annotations

import torch

from . import api


class DraftAttention:
    def __init__(self, frames: int, height: int, width: int, patch_h: int = 8, patch_w: int = 8,
                 sparsity: float = 0.9, dense_warmup_steps: int = 0, mask_refresh_every: int = 1,
                 scale=None, select_on: str = "logits", force_row_keep: bool = True):
        if dense_warmup_steps < 0:
            raise ValueError(f"dense_warmup_steps must be >= 0, got {dense_warmup_steps}")
        if mask_refresh_every < 1:
            raise ValueError(f"mask_refresh_every must be >= 1, got {mask_refresh_every}")
        api._validate_pipeline_args(sparsity, select_on, "average")
        self.plan = api.pad_plan(frames, height, width, patch_h, patch_w)
        self.sparsity = float(sparsity)
        self.dense_warmup_steps = int(dense_warmup_steps)
        self.mask_refresh_every = int(mask_refresh_every)
        self.scale = scale
        self.select_on = select_on
        self.force_row_keep = force_row_keep
        self._mask = None        # per (batch element, head) masks of the last refresh, batch-major
        self._mask_step = None   # the step they were selected at
        self._mask_shape = None  # (batch, heads) they were selected for

    def reset(self) -> None:
        """Forget the cached masks (a new video)."""
        self._mask = self._mask_step = self._mask_shape = None

    def mode(self, step: int) -> str:
        """What ``__call__`` runs at ``step``: "dense", "select" (full draft
        pipeline, refreshing the mask cache) or "cached" (executor only)."""
        if step < self.dense_warmup_steps:
            return "dense"
        if self._mask is None or step - self._mask_step >= self.mask_refresh_every or step < self._mask_step:
            return "select"
        return "cached"

    def __call__(self, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, step: int = 0) -> torch.Tensor:
        """q, k, v: (batch, n, heads, d) CUDA tensors, n = frames * height * width
        tokens in (f, y, x) order. Returns (batch, n, heads, dv)."""
        if q.ndim != 4 or k.shape != q.shape or v.shape[:3] != q.shape[:3]:
            raise ValueError(f"expected (batch, n, heads, d) q/k and (batch, n, heads, dv) v, got "
                             f"{tuple(q.shape)}, {tuple(k.shape)}, {tuple(v.shape)}")
        if q.shape[1] != self.plan.num_valid:
            raise ValueError(f"q rows {q.shape[1]} != layout token count {self.plan.num_valid}")
        if not q.is_cuda:
            raise ValueError("inputs must be CUDA tensors (the B200 path has no CPU fallback)")
        batch, _, heads, d = q.shape
        scale = self.scale if self.scale is not None else api.head_dim_scale(d)
        mode = self.mode(step)
        if mode == "dense":
            return self._dense(q, k, v, scale)
        if mode == "cached" and self._mask_shape != (batch, heads):
            mode = "select"
        if mode == "select":
            res = api.multi_head_sparse_attention(q, k, v, self.plan, self.sparsity, scale=scale,
                                                  select_on=self.select_on, force_row_keep=self.force_row_keep,
                                                  qkv_layout="bnhd", return_details=True)
            self._mask, self._mask_step, self._mask_shape = res.mask, step, (batch, heads)
            return res.output
        out = torch.empty(q.shape[:3] + (v.shape[3],), dtype=api._out_dtype(q, k, v), device=q.device)
        for b in range(batch):
            out[b] = api.padded_block_sparse_attention(q[b], k[b], v[b], self.plan,
                                                       _mask_rows(self._mask, b * heads, (b + 1) * heads), scale,
                                                       qkv_layout="nhd")
        return out

    @staticmethod
    def _dense(q, k, v, scale):
        import torch.nn.functional as F

        o = F.scaled_dot_product_attention(q.transpose(1, 2), k.transpose(1, 2), v.transpose(1, 2), scale=scale)
        return o.transpose(1, 2)


def _mask_rows(m: api.RegionMask, h0: int, h1: int) -> api.RegionMask:
    """Masks h0 .. h1 - 1 of a stacked RegionMask (views, no copies)."""
    return api.RegionMask(m.g, m.keep_ratio, None if m.packed is None else m.packed[h0:h1], m.row_ptr[h0:h1],
                          m.col_idx[h0:h1], m.thresholds[h0:h1], m.forced[h0:h1], m.kept_counts[h0:h1],
                          single=h1 - h0 == 1)
