"""Head-parallel execution across GPUs (one process per GPU).

The reference runs heads one after another (sparse.py:273-279); heads are
independent (per-head masks by default), so P ranks each own heads/P heads.
A sequence-parallel caller holds n/P tokens of every head; one NCCL
all-to-all reshards Q/K/V to "all tokens of my heads" before the call and one
reshards the output back (Ulysses-style). No other collective is needed.
"""

from __future__ import annotations

import torch
import torch.distributed as dist

from . import api


def seq_to_head(x: torch.Tensor, world: int, group=None) -> torch.Tensor:
    """(n/P, H, d) sequence shard -> (n, H/P, d) head shard (all-to-all)."""
    nl, heads, d = x.shape
    hl = heads // world
    send = x.reshape(nl, world, hl, d).permute(1, 0, 2, 3).contiguous()  # [dest rank][rows][my heads]
    recv = torch.empty_like(send)                                          # [src rank][its rows][my heads]
    dist.all_to_all_single(recv, send, group=group)
    return recv.reshape(world * nl, hl, d)


def head_to_seq(o: torch.Tensor, world: int, group=None) -> torch.Tensor:
    """(n, H/P, d) head shard -> (n/P, H, d) sequence shard (all-to-all)."""
    n, hl, d = o.shape
    nl = n // world
    send = o.reshape(world, nl, hl, d).contiguous()                        # [dest rank][its rows][my heads]
    recv = torch.empty_like(send)                                          # [src rank = head group][my rows]
    dist.all_to_all_single(recv, send, group=group)
    return recv.permute(1, 0, 2, 3).reshape(nl, world * hl, d)


class HeadParallelAttention:
    """padded_sparse_attention over a sequence-sharded (n/P, H, d) input."""

    def __init__(self, plan: api.PadPlan, sparsity: float, world: int, rank: int, group=None,
                 scale=None, pool_mode="average", select_on="logits", force_row_keep=True):
        self.plan, self.sparsity, self.world, self.rank, self.group = plan, sparsity, world, rank, group
        self.scale, self.pool_mode, self.select_on, self.force = scale, pool_mode, select_on, force_row_keep

    def __call__(self, q, k, v, attn_events=None, a2a_events=None):
        """``a2a_events`` (optional): two (begin, end) CUDA event pairs recorded
        around the input and output all-to-alls, for timing the collectives."""
        if a2a_events is not None:
            a2a_events[0][0].record()
        qh, kh, vh = (seq_to_head(x, self.world, self.group) for x in (q, k, v))
        if a2a_events is not None:
            a2a_events[0][1].record()
        scale = self.scale if self.scale is not None else api.head_dim_scale(q.shape[-1])
        out, mask, _ = api._pipeline(qh, kh, vh, self.plan, self.sparsity, scale, self.pool_mode, self.select_on,
                                     self.force, False, "nhd", attn_events=attn_events, want_bitmap=False)
        if a2a_events is not None:
            a2a_events[1][0].record()
        res = head_to_seq(out, self.world, self.group)
        if a2a_events is not None:
            a2a_events[1][1].record()
        return res, mask
