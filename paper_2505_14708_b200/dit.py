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

Sequence parallel (``world`` > 1, one process per GPU): every rank passes its
(batch, n/P, heads, d) sequence shard and gets its output shard back. The
draft and cached steps run ``headpar.HeadParallelAttention`` (each rank owns
heads/P heads; ``transport="peer"`` reads the other ranks' rows in place over
NVLink, ``"nccl"`` reshards with all-to-alls) and cache each rank's masks of
its own heads; dense warm-up steps reshard with NCCL all-to-alls around SDPA.
"""

from __future__ import annotations

import torch

from . import api


class DraftAttention:
    def __init__(self, frames: int, height: int, width: int, patch_h: int = 8, patch_w: int = 8,
                 sparsity: float = 0.9, dense_warmup_steps: int = 0, mask_refresh_every: int = 1,
                 scale=None, select_on: str = "logits", force_row_keep: bool = True,
                 world: int = 1, rank: int = 0, group=None, transport: str = "peer", head_groups: int = 2):
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
        self.world, self.rank = int(world), int(rank)
        self._hp = None
        if self.world > 1:
            from .headpar import HeadParallelAttention

            self._hp = HeadParallelAttention(self.plan, self.sparsity, self.world, self.rank, group, scale,
                                             select_on=select_on, force_row_keep=force_row_keep,
                                             head_groups=head_groups, transport=transport)
        self.group = group
        self._mask = None        # per (batch element, head) masks of the last refresh, batch-major
                                 # (world > 1: a list, per batch element, of this rank's heads' masks)
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
        tokens in (f, y, x) order (world > 1: this rank's (batch, n/P, heads, d)
        sequence shard, rows [rank * n/P, (rank + 1) * n/P)). Returns
        (batch, n, heads, dv) (world > 1: the output shard)."""
        if q.ndim != 4 or k.shape != q.shape or v.shape[:3] != q.shape[:3]:
            raise ValueError(f"expected (batch, n, heads, d) q/k and (batch, n, heads, dv) v, got "
                             f"{tuple(q.shape)}, {tuple(k.shape)}, {tuple(v.shape)}")
        if q.shape[1] * self.world != self.plan.num_valid:
            raise ValueError(f"q rows {q.shape[1]} x world {self.world} != layout token count {self.plan.num_valid}")
        if not q.is_cuda:
            raise ValueError("inputs must be CUDA tensors (the B200 path has no CPU fallback)")
        batch, _, heads, d = q.shape
        scale = self.scale if self.scale is not None else api.head_dim_scale(d)
        mode = self.mode(step)
        if self.world > 1:
            return self._call_parallel(q, k, v, scale, mode, step)
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

    def _call_parallel(self, q, k, v, scale, mode, step):
        """world > 1: per batch element, the head-parallel call on the sequence shards."""
        batch, nl, heads, _ = q.shape
        if heads % self.world:
            raise ValueError(f"heads {heads} must be divisible by the world size {self.world}")
        out = torch.empty(q.shape[:3] + (v.shape[3],), dtype=api._out_dtype(q, k, v), device=q.device)
        if mode == "dense":
            from .headpar import head_to_seq, seq_to_head

            for b in range(batch):
                qh, kh, vh = (seq_to_head(x[b].contiguous(), self.world, self.group) for x in (q, k, v))
                oh = self._dense(qh.unsqueeze(0), kh.unsqueeze(0), vh.unsqueeze(0), scale)[0]
                out[b] = head_to_seq(oh.contiguous(), self.world, self.group)
            return out
        if mode == "cached" and (len(self._mask) != batch or self._mask_shape != (batch, heads)):
            mode = "select"
        masks = []
        for b in range(batch):
            o, m = self._hp(q[b].contiguous(), k[b].contiguous(), v[b].contiguous(),
                            mask=self._mask[b] if mode == "cached" else None)
            out[b] = o
            masks.append(m)
        if mode == "select":
            self._mask, self._mask_step, self._mask_shape = masks, step, (batch, heads)
        return out

    def close(self) -> None:
        """world > 1 with the peer transport: unmap the peers' buffers (a collective)."""
        if self._hp is not None:
            self._hp.close()

    @staticmethod
    def _dense(q, k, v, scale):
        import torch.nn.functional as F

        o = F.scaled_dot_product_attention(q.transpose(1, 2), k.transpose(1, 2), v.transpose(1, 2), scale=scale)
        return o.transpose(1, 2)


def _mask_rows(m: api.RegionMask, h0: int, h1: int) -> api.RegionMask:
    """Masks h0 .. h1 - 1 of a stacked RegionMask (views, no copies)."""
    return m.head_range(h0, h1)
