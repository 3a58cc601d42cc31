"""B200-native (sm_100a) DraftAttention sparse-attention path.

Drop-in for the reference package's draft-attention operators
(/root/reference/pkg/src/draftattn): same names, argument order, defaults and
error messages, computed by hand-written CUDA kernels behind a C ABI
(include/draftattn_b200.h). See DESIGN.md.
"""

from .api import (
    FlopsReport,
    LatentLayout,
    PadPlan,
    PipelineResult,
    RegionMask,
    block_sparse_attention,
    draft_attention_map,
    draft_logits,
    draft_sparse_attention,
    flops_count,
    head_dim_scale,
    kept_from_bitmap,
    mask_density_stats,
    mask_from_json_dict,
    mask_to_bitmap,
    mask_to_json_dict,
    multi_head_sparse_attention,
    pad_plan,
    padded_block_sparse_attention,
    padded_sparse_attention,
    pool_regions,
    pool_tokens,
    reorder_tokens,
    restore_tokens,
    select_top_fraction,
    sharded_sparse_attention,
    top_fraction_count,
)

__version__ = "0.1.0"

__all__ = [
    "FlopsReport", "LatentLayout", "PadPlan", "PipelineResult", "RegionMask",
    "block_sparse_attention", "draft_attention_map", "draft_logits", "draft_sparse_attention", "flops_count",
    "head_dim_scale", "kept_from_bitmap", "mask_density_stats", "mask_from_json_dict", "mask_to_bitmap",
    "mask_to_json_dict", "multi_head_sparse_attention", "pad_plan", "padded_block_sparse_attention",
    "padded_sparse_attention", "pool_regions", "pool_tokens", "reorder_tokens",
    "restore_tokens", "select_top_fraction", "sharded_sparse_attention", "top_fraction_count", "__version__",
]
