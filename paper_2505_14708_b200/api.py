"""Drop-in GPU API for the DraftAttention sparse-attention path.

Mirrors the reference package's operator surface (names, positional order,
defaults and ValueError messages of /root/reference/pkg/src/draftattn):

    padded_sparse_attention   padding.py:95-165
    draft_sparse_attention    sparse.py:193-246
    multi_head_sparse_attention  sparse.py:249-302
    block_sparse_attention    sparse.py:88-166   (reordered seam)
    select_top_fraction       masking.py:59-91
    draft_logits / pool_regions / top_fraction_count / head_dim_scale / flops_count

Tensors are torch tensors (bf16 compute: float32 / float64 inputs are rounded
to bf16 on entry, so masks and outputs are those of the bf16-rounded inputs,
and the output is cast back to the reference's ``result_type(q, k, v)``).
Token matrices are ``(n, d)`` or ``(heads, n, d)``; ``qkv_layout="nhd"``
accepts the DiT ``(n, heads, d)`` layout and ``qkv_layout="bnhd"`` a batch of
them, ``(batch, n, heads, d)``, without a copy. Any head dim works: dims that
are not a multiple of 8 are zero-padded to one (exact: zero features add
nothing to any dot product). Host (CPU) tensors are staged to the GPU. All
work runs in hand-written sm_100a kernels behind the C ABI
(include/draftattn_b200.h); there is no CPU compute path.
"""

from __future__ import annotations

import ctypes
import dataclasses
import math
from dataclasses import dataclass, field

import torch

from . import _lib
from ._lib import DaAttnArgs, DaPipelineArgs, check, lib, make_grid

_CEIL_EPS = 1e-9
POOL_MODES = ("average", "max")
SELECT_MODES = ("logits", "softmax")
QKV_LAYOUTS = ("hnd", "nhd", "bnhd")


# --------------------------------------------------------------------------
# host-side geometry (layout.py:10-60, padding.py:21-56)
# --------------------------------------------------------------------------

@dataclass(frozen=True)
class LatentLayout:
    """Token grid partitioned into pooling patches (layout.py:10-60)."""

    frames: int
    height: int
    width: int
    patch_h: int
    patch_w: int

    def __post_init__(self) -> None:
        for name in ("frames", "height", "width", "patch_h", "patch_w"):
            value = getattr(self, name)
            if not isinstance(value, int) or isinstance(value, bool) or value < 1:
                raise ValueError(f"{name} must be a positive integer, got {value!r}")
        if self.height % self.patch_h != 0:
            raise ValueError(f"patch_h={self.patch_h} does not divide height={self.height}; "
                             "pad the grid first (see draftattn.padding)")
        if self.width % self.patch_w != 0:
            raise ValueError(f"patch_w={self.patch_w} does not divide width={self.width}; "
                             "pad the grid first (see draftattn.padding)")

    @property
    def num_tokens(self) -> int:
        return self.frames * self.height * self.width

    @property
    def region_size(self) -> int:
        return self.patch_h * self.patch_w

    @property
    def patches_h(self) -> int:
        return self.height // self.patch_h

    @property
    def patches_w(self) -> int:
        return self.width // self.patch_w

    @property
    def num_regions(self) -> int:
        return self.frames * self.patches_h * self.patches_w


@dataclass(frozen=True)
class PadPlan:
    """Padded geometry of a real grid (padding.py:21-42); validity is closed form."""

    frames: int
    height: int
    width: int
    layout: LatentLayout

    @property
    def num_valid(self) -> int:
        return self.frames * self.height * self.width

    @property
    def is_identity(self) -> bool:
        return self.layout.height == self.height and self.layout.width == self.width


def pad_plan(frames: int, height: int, width: int, patch_h: int, patch_w: int) -> PadPlan:
    """Smallest patch-divisible grid containing (height, width) (padding.py:45-56)."""
    if min(frames, height, width, patch_h, patch_w) < 1:
        raise ValueError("all grid dimensions must be positive")
    ph = -(-height // patch_h) * patch_h
    pw = -(-width // patch_w) * patch_w
    return PadPlan(frames, height, width, LatentLayout(frames, ph, pw, patch_h, patch_w))


def head_dim_scale(head_dim: int) -> float:
    """1/sqrt(d) (core.py:13-17)."""
    if head_dim < 1:
        raise ValueError(f"head_dim must be positive, got {head_dim}")
    return 1.0 / math.sqrt(head_dim)


def top_fraction_count(num_entries: int, keep_ratio: float) -> int:
    """ceil(r*N - 1e-9) clamped to [1, N] (masking.py:49-56)."""
    if not 0.0 < keep_ratio <= 1.0:
        raise ValueError(f"keep_ratio must be in (0, 1], got {keep_ratio}")
    if num_entries < 1:
        raise ValueError(f"num_entries must be positive, got {num_entries}")
    m = math.ceil(keep_ratio * num_entries - _CEIL_EPS)
    return min(max(m, 1), num_entries)


# --------------------------------------------------------------------------
# result types (masking.py:16-46, sparse.py:15-43, 183-190)
# --------------------------------------------------------------------------

@dataclass(frozen=True, eq=False)
class RegionMask:
    """Block mask of one or more heads, resident on the GPU.

    ``bitmap`` is the reference's packed row-major MSB-first layout
    (masking.py:168-170), one row of ``ceil(g*g/8)`` bytes per head;
    ``row_ptr``/``col_idx`` are the executor feed (ascending kept columns).
    ``threshold``, ``forced_row_keeps`` and ``kept_count`` are per head
    (Python scalars for a single-head mask).
    """

    g: int
    keep_ratio: float
    packed: torch.Tensor | None   # (heads, ceil(g*g/8)) uint8, or None: packed from the lists on first use
    row_ptr: torch.Tensor         # (heads, g+1) int32
    col_idx: torch.Tensor         # (heads, cap) int32
    thresholds: torch.Tensor      # (heads,) float64
    forced: torch.Tensor          # (heads,) int64
    kept_counts: torch.Tensor     # (heads,) int64
    single: bool = True
    _host: dict = field(default_factory=dict, repr=False)

    @property
    def heads(self) -> int:
        return int(self.row_ptr.shape[0])

    @property
    def bitmap(self) -> torch.Tensor:
        """Packed bitmap (heads, ceil(g*g/8)) uint8; calls that did not ask for
        details skip the packing kernel, and it is built here from the lists."""
        if self.packed is not None:
            return self.packed
        if "bitmap" not in self._host:
            g, dev = self.g, self.row_ptr.device
            nbytes = (g * g + 7) // 8
            bits = torch.zeros((self.heads, nbytes * 8), dtype=torch.uint8, device=dev)
            counts = (self.row_ptr[:, 1:] - self.row_ptr[:, :-1]).to(torch.int64)
            rows = torch.arange(g, device=dev, dtype=torch.int64)
            for h in range(self.heads):
                tot = int(self.row_ptr[h, g].item())
                flat = torch.repeat_interleave(rows, counts[h]) * g + self.col_idx[h, :tot].to(torch.int64)
                bits[h, flat] = 1
            w = torch.tensor([128, 64, 32, 16, 8, 4, 2, 1], dtype=torch.int32, device=dev)
            self._host["bitmap"] = (bits.view(self.heads, nbytes, 8).to(torch.int32) * w).sum(-1).to(torch.uint8)
        return self._host["bitmap"]

    def _scalars(self):
        if "s" not in self._host:
            self._host["s"] = (self.thresholds.cpu().tolist(), self.forced.cpu().tolist(),
                               self.kept_counts.cpu().tolist())
        return self._host["s"]

    @property
    def threshold(self):
        t = self._scalars()[0]
        return t[0] if self.single else t

    @property
    def forced_row_keeps(self):
        f = self._scalars()[1]
        return f[0] if self.single else f

    @property
    def kept_count(self):
        k = self._scalars()[2]
        return k[0] if self.single else k

    @property
    def kept(self) -> torch.Tensor:
        """Unpacked boolean (g, g) (or (heads, g, g)) matrix, on the GPU."""
        bits = torch.tensor([128, 64, 32, 16, 8, 4, 2, 1], dtype=torch.uint8, device=self.bitmap.device)
        kept = ((self.bitmap.unsqueeze(-1) & bits) != 0).reshape(self.heads, -1)[:, : self.g * self.g]
        kept = kept.reshape(self.heads, self.g, self.g)
        return kept[0] if self.single else kept

    @property
    def row_kept_counts(self) -> torch.Tensor:
        c = (self.row_ptr[:, 1:] - self.row_ptr[:, :-1]).to(torch.int64)
        return c[0] if self.single else c

    def bitmap_bytes(self, head: int = 0) -> bytes:
        """mask_to_bitmap (masking.py:168-170) of one head."""
        return self.bitmap[head].cpu().numpy().tobytes()

    def head(self, h: int) -> "RegionMask":
        return RegionMask(self.g, self.keep_ratio, None if self.packed is None else self.packed[h:h + 1],
                          self.row_ptr[h:h + 1],
                          self.col_idx[h:h + 1], self.thresholds[h:h + 1], self.forced[h:h + 1],
                          self.kept_counts[h:h + 1], single=True)

    def head_range(self, h0: int, h1: int) -> "RegionMask":
        """Masks h0 .. h1 - 1 of a stacked mask (views, no copies); a shared
        (single) mask is returned as is."""
        if self.single or self.heads == 1:
            return self
        return RegionMask(self.g, self.keep_ratio, None if self.packed is None else self.packed[h0:h1],
                          self.row_ptr[h0:h1], self.col_idx[h0:h1], self.thresholds[h0:h1], self.forced[h0:h1],
                          self.kept_counts[h0:h1], single=h1 - h0 == 1)

    @classmethod
    def from_kept(cls, kept, keep_ratio: float, threshold, forced_row_keeps=0, device=None) -> "RegionMask":
        """A GPU mask (executor lists + packed bitmap) from a boolean (g, g) or
        (heads, g, g) kept matrix (numpy or torch), e.g. a cached mask reused
        across denoising steps. ``threshold`` / ``forced_row_keeps``: scalars or
        one per head."""
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        k = torch.as_tensor(kept, device=dev)
        if k.dtype != torch.bool:
            raise ValueError(f"kept must be a boolean matrix, got {k.dtype}")
        single = k.ndim == 2
        if single:
            k = k.unsqueeze(0)
        if k.ndim != 3 or k.shape[1] != k.shape[2]:
            raise ValueError(f"kept must be a square boolean matrix, got shape {tuple(kept.shape)}")
        heads, g, _ = k.shape
        counts = k.sum(dim=2, dtype=torch.int64)
        row_ptr = torch.zeros((heads, g + 1), dtype=torch.int32, device=dev)
        row_ptr[:, 1:] = torch.cumsum(counts, dim=1).to(torch.int32)
        totals = counts.sum(dim=1)
        cap = max(1, int(totals.max().item()) if heads else 1)
        col_idx = torch.zeros((heads, cap), dtype=torch.int32, device=dev)
        for h in range(heads):
            cols = k[h].nonzero()[:, 1]  # row-major: rows ascending, columns ascending within a row
            col_idx[h, :cols.numel()] = cols.to(torch.int32)
        nbytes = (g * g + 7) // 8
        bits = torch.zeros((heads, nbytes * 8), dtype=torch.int32, device=dev)
        bits[:, :g * g] = k.reshape(heads, -1).to(torch.int32)
        w = torch.tensor([128, 64, 32, 16, 8, 4, 2, 1], dtype=torch.int32, device=dev)
        packed = (bits.view(heads, nbytes, 8) * w).sum(-1).to(torch.uint8)
        thr = torch.as_tensor(threshold, dtype=torch.float64, device=dev).reshape(-1).expand(heads).contiguous()
        forced = torch.as_tensor(forced_row_keeps, dtype=torch.int64, device=dev).reshape(-1).expand(heads)
        return cls(g, float(keep_ratio), packed, row_ptr, col_idx, thr, forced.contiguous(), totals,
                   single=single)

    @classmethod
    def from_bitmap(cls, raw: bytes, g: int, keep_ratio: float, threshold, forced_row_keeps=0,
                    device=None) -> "RegionMask":
        """Inverse of ``bitmap_bytes`` (masking.py:168-176): a GPU mask from the
        reference's packed row-major bitmap of one head."""
        return cls.from_kept(kept_from_bitmap(raw, g), keep_ratio, threshold, forced_row_keeps, device)


def mask_density_stats(mask: RegionMask, head: int = 0) -> dict:
    """Occupancy summary of one head (masking.py:128-141)."""
    m = mask.head(head) if not mask.single else mask
    rows = m.row_kept_counts.double()
    kept = int(m.kept_count)
    return {
        "g": m.g,
        "keep_ratio": m.keep_ratio,
        "threshold": m.threshold,
        "kept_count": kept,
        "kept_fraction": kept / (m.g * m.g),
        "row_kept_min": int(rows.min().item()),
        "row_kept_mean": float(rows.mean().item()),
        "row_kept_max": int(rows.max().item()),
        "forced_row_keeps": m.forced_row_keeps,
    }


def mask_to_bitmap(mask: RegionMask, head: int = 0) -> bytes:
    """Row-major packed bits of one head's kept matrix (masking.py:168-170)."""
    return mask.bitmap_bytes(head)


def kept_from_bitmap(raw: bytes, g: int) -> torch.Tensor:
    """Unpack a row-major bitmap into a (g, g) bool tensor on the CPU (masking.py:173-176)."""
    if g < 1:
        raise ValueError(f"g must be positive, got {g}")
    data = torch.frombuffer(bytearray(raw), dtype=torch.uint8)
    if data.numel() * 8 < g * g:
        raise ValueError(f"bitmap of {data.numel()} bytes is too short for g = {g}")
    bits = torch.tensor([128, 64, 32, 16, 8, 4, 2, 1], dtype=torch.uint8)
    return ((data.unsqueeze(-1) & bits) != 0).reshape(-1)[: g * g].reshape(g, g)


def mask_to_json_dict(mask: RegionMask, head: int = 0) -> dict:
    """JSON-ready export of one head: metadata plus the kept coordinate list in
    row-major order (masking.py:144-155)."""
    m = mask.head(head) if not mask.single else mask
    total = int(m.row_ptr[0, m.g].item())
    rows = torch.repeat_interleave(torch.arange(m.g, device=m.row_ptr.device),
                                   (m.row_ptr[0, 1:] - m.row_ptr[0, :-1]).to(torch.int64))
    cols = m.col_idx[0, :total]
    pairs = torch.stack([rows.to(torch.int64), cols.to(torch.int64)], dim=1).cpu().tolist()
    return {
        "g": m.g,
        "keep_ratio": m.keep_ratio,
        "threshold": m.threshold,
        "kept_count": int(m.kept_count),
        "forced_row_keeps": int(m.forced_row_keeps),
        "kept": pairs,
    }


def mask_from_json_dict(data: dict, device=None) -> RegionMask:
    """Inverse of ``mask_to_json_dict`` (masking.py:158-166), on the GPU."""
    g = int(data["g"])
    kept = torch.zeros((g, g), dtype=torch.bool)
    if data["kept"]:
        idx = torch.as_tensor(data["kept"], dtype=torch.int64)
        kept[idx[:, 0], idx[:, 1]] = True
    return RegionMask.from_kept(kept, float(data["keep_ratio"]), float(data["threshold"]),
                                int(data.get("forced_row_keeps", 0)), device)


@dataclass(frozen=True)
class FlopsReport:
    """Matmul FLOP accounting for one head (sparse.py:15-43)."""

    full_logits_flops: int
    full_av_flops: int
    draft_flops: int
    sparse_logits_flops: int
    sparse_av_flops: int
    overhead_ratio: float
    total_ratio: float

    def as_dict(self) -> dict:
        return dict(self.__dict__)


def flops_count(layout: LatentLayout, head_dim: int, sparsity: float | None = None,
                kept_count: int | None = None, force_row_keep_extras: int = 0) -> FlopsReport:
    """FLOP model (sparse.py:45-85)."""
    if head_dim < 1:
        raise ValueError(f"head_dim must be positive, got {head_dim}")
    n, g, p = layout.num_tokens, layout.num_regions, layout.region_size
    if kept_count is None:
        if sparsity is None:
            raise ValueError("pass sparsity or kept_count")
        if not 0.0 <= sparsity < 1.0:
            raise ValueError(f"sparsity must be in [0, 1), got {sparsity}")
        kept_count = min(top_fraction_count(g * g, 1.0 - sparsity) + force_row_keep_extras, g * g)
    elif not 0 <= kept_count <= g * g:
        raise ValueError(f"kept_count {kept_count} outside [0, {g * g}]")
    full = 2 * n * n * head_dim
    draft = 2 * g * g * head_dim
    sparse = 2 * kept_count * p * p * head_dim
    return FlopsReport(full, full, draft, sparse, sparse, draft / full, (draft + sparse) / full)


@dataclass(frozen=True, eq=False)
class PipelineResult:
    """Output plus the artifacts that produced it (sparse.py:183-190)."""

    output: torch.Tensor
    mask: RegionMask
    flops: FlopsReport | list
    mask_stats: dict | list


# --------------------------------------------------------------------------
# tensor plumbing
# --------------------------------------------------------------------------

def _stream_ptr(device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def _as_heads(x: torch.Tensor, qkv_layout: str, name: str):
    """Return (heads-first 3-d view, squeeze) for (n,d) / (h,n,d) / (n,h,d)."""
    if not isinstance(x, torch.Tensor):
        raise TypeError(f"{name} must be a torch.Tensor on a CUDA device")
    if qkv_layout not in ("hnd", "nhd"):
        raise ValueError(f"qkv_layout must be one of {QKV_LAYOUTS}, got {qkv_layout!r}")
    if x.ndim == 2:
        x3 = x.unsqueeze(0)
        squeeze = True
    elif x.ndim == 3:
        x3 = x if qkv_layout == "hnd" else x.transpose(0, 1)
        squeeze = False
    else:
        raise ValueError(f"{name} must be 2-d (n, d) or 3-d, got shape {tuple(x.shape)}")
    return x3, squeeze


def _prep(x3: torch.Tensor) -> torch.Tensor:
    """bf16, CUDA, unit stride on features, 16-byte aligned rows (copy only if needed)."""
    if not x3.is_cuda:
        raise ValueError("inputs must be CUDA tensors (the B200 path has no CPU fallback)")
    if x3.dtype != torch.bfloat16:
        x3 = x3.to(torch.bfloat16)
    ok = (x3.stride(2) == 1 and x3.stride(0) % 8 == 0 and x3.stride(1) % 8 == 0
          and x3.data_ptr() % 16 == 0 and x3.shape[2] % 8 == 0)
    return x3 if ok else x3.contiguous()


def _out_dtype(q, k, v):
    return torch.promote_types(torch.promote_types(q.dtype, k.dtype), v.dtype)


def _pad_features(x3: torch.Tensor) -> torch.Tensor:
    """(heads, n, d) -> bf16 (heads, n, ceil8(d)) with zero features appended
    (zeros change no dot product, pooled mean or weighted sum)."""
    d = x3.shape[2]
    d8 = -(-d // 8) * 8
    if not x3.is_cuda:
        raise ValueError("inputs must be CUDA tensors (the B200 path has no CPU fallback)")
    out = torch.zeros((x3.shape[0], x3.shape[1], d8), dtype=torch.bfloat16, device=x3.device)
    out[..., :d] = x3
    return out


def _alloc_like_layout(heads, n, dv, qkv_layout, device):
    if qkv_layout == "nhd":
        base = torch.empty((n, heads, dv), dtype=torch.bfloat16, device=device)
        return base, base.transpose(0, 1)
    base = torch.empty((heads, n, dv), dtype=torch.bfloat16, device=device)
    return base, base


def _attn_struct(q3, k3, v3, o3, d, dv, layout_code, scale) -> DaAttnArgs:
    a = DaAttnArgs()
    a.q, a.k, a.v, a.out = q3.data_ptr(), k3.data_ptr(), v3.data_ptr(), o3.data_ptr()
    a.q_head_stride, a.q_row_stride = q3.stride(0), q3.stride(1)
    a.k_head_stride, a.k_row_stride = k3.stride(0), k3.stride(1)
    a.v_head_stride, a.v_row_stride = v3.stride(0), v3.stride(1)
    a.o_head_stride, a.o_row_stride = o3.stride(0), o3.stride(1)
    a.heads = q3.shape[0]
    a.d, a.dv, a.layout = d, dv, layout_code
    a.scale = float(scale)
    return a


def _validate_pipeline_args(sparsity, select_on, pool_mode):
    if not 0.0 <= sparsity < 1.0:
        raise ValueError(f"sparsity must be in [0, 1), got {sparsity}")
    if select_on not in SELECT_MODES:
        raise ValueError(f"select_on must be 'logits' or 'softmax', got {select_on!r}")
    if pool_mode not in POOL_MODES:
        raise ValueError(f"mode must be one of {POOL_MODES}, got {pool_mode!r}")


def _pipeline(q, k, v, plan: PadPlan, sparsity, scale, pool_mode, select_on, force_row_keep,
              shared_head_mask, qkv_layout, force_portable=False, attn_events=None, want_bitmap=True,
              out_dev=None, debug=None):
    """Run the fused C-ABI pipeline; returns (output, mask, squeeze). ``out_dev``
    (internal): a preallocated bf16 device tensor, in the inputs' layout, the
    output is written into."""
    q3, squeeze = _as_heads(q, qkv_layout, "q")
    k3, _ = _as_heads(k, qkv_layout, "k")
    v3, _ = _as_heads(v, qkv_layout, "v")
    heads, n, d = q3.shape
    if k3.shape != q3.shape:
        raise ValueError(f"k shape {tuple(k3.shape)} does not match q shape {tuple(q3.shape)}")
    if v3.shape[:2] != q3.shape[:2]:
        raise ValueError(f"v rows {v3.shape[1]} != key rows {n}")
    out_dtype = _out_dtype(q, k, v)
    if d % 8 or v3.shape[2] % 8:
        # zero-pad the features to a multiple of 8 (exact) and drop the padded
        # output features; the caller's scale is kept
        dv0 = v3.shape[2]
        o, mask, _ = _pipeline(_pad_features(q3), _pad_features(k3), _pad_features(v3), plan, sparsity, scale,
                               pool_mode, select_on, force_row_keep, shared_head_mask, "hnd", force_portable,
                               attn_events, want_bitmap, None, debug)
        o = o[..., :dv0]
        if out_dev is not None:
            _as_heads(out_dev, qkv_layout, "out")[0].copy_(o)
            return out_dev, mask, squeeze
        out = o[0] if squeeze else (o.transpose(0, 1) if qkv_layout == "nhd" else o)
        return (out.to(out_dtype) if out_dtype != out.dtype else out), mask, squeeze
    q3, k3, v3 = _prep(q3), _prep(k3), _prep(v3)
    dv = v3.shape[2]
    dev = q3.device
    if out_dev is not None:
        # the caller's bf16 output buffer, in the inputs' layout
        o3, _ = _as_heads(out_dev, qkv_layout, "out")
        if o3.dtype != torch.bfloat16 or tuple(o3.shape) != (heads, n, dv) or o3.device != dev or \
                o3.stride(2) != 1 or o3.stride(0) % 8 or o3.stride(1) % 8 or o3.data_ptr() % 16:
            raise ValueError("internal output buffer has the wrong shape, dtype or strides")
        o_base = out_dev
    else:
        o_base, o3 = _alloc_like_layout(heads, n, dv, qkv_layout if not squeeze else "hnd", dev)
    a = _attn_struct(q3, k3, v3, o3, d, dv, _lib.LAYOUT_ORIGINAL, scale)
    a.force_portable = 1 if force_portable else 0
    mask = _launch_pipeline(a, plan, sparsity, pool_mode, select_on, force_row_keep, shared_head_mask, dev,
                            want_bitmap, attn_events, debug, single=squeeze or shared_head_mask)
    out = o3[0] if squeeze else (o_base if qkv_layout == "nhd" else o3)
    if out_dtype != torch.bfloat16:
        out = out.to(out_dtype)
    return out, mask, squeeze


def _launch_pipeline(a: DaAttnArgs, plan: PadPlan, sparsity, pool_mode, select_on, force_row_keep,
                     shared_head_mask, dev, want_bitmap=True, attn_events=None, debug=None,
                     single=False) -> RegionMask:
    """Allocate the mask outputs and the workspace, run da_sparse_attention
    with the tensor fields of ``a`` (plain or sharded) and return the mask."""
    heads, d = a.heads, a.d
    layout = plan.layout
    g = layout.num_regions
    grid = make_grid(plan.frames, plan.height, plan.width, layout.patch_h, layout.patch_w)
    m = top_fraction_count(g * g, 1.0 - sparsity)
    mheads = 1 if shared_head_mask else heads
    cap = m + g
    row_ptr = torch.empty((mheads, g + 1), dtype=torch.int32, device=dev)
    col_idx = torch.empty((mheads, cap), dtype=torch.int32, device=dev)
    bitmap = torch.empty((mheads, (g * g + 7) // 8), dtype=torch.uint8, device=dev) if want_bitmap else None
    thr = torch.empty(mheads, dtype=torch.float64, device=dev)
    forced = torch.empty(mheads, dtype=torch.int64, device=dev)
    kept = torch.empty(mheads, dtype=torch.int64, device=dev)
    ws_bytes = lib().da_pipeline_workspace_size(ctypes.byref(grid), heads, d)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    pa = DaPipelineArgs()
    pa.attn = a
    pa.m = m
    pa.force_row_keep = 1 if force_row_keep else 0
    pa.pool_mode = POOL_MODES.index(pool_mode)
    pa.select_softmax = 1 if select_on == "softmax" else 0
    pa.shared_head_mask = 1 if shared_head_mask else 0
    pa.row_ptr, pa.col_idx = row_ptr.data_ptr(), col_idx.data_ptr()
    pa.bitmap = bitmap.data_ptr() if bitmap is not None else None
    pa.threshold, pa.forced, pa.kept = thr.data_ptr(), forced.data_ptr(), kept.data_ptr()
    pa.workspace = ws.data_ptr()
    if attn_events is not None:  # (begin, end) torch.cuda.Event pair around the K4 launch
        for e in attn_events:
            if not e.cuda_event:  # torch creates the CUDA event on its first record
                e.record()
        pa.ev_attn_begin = attn_events[0].cuda_event
        pa.ev_attn_end = attn_events[1].cuda_event
    with torch.cuda.device(dev):
        check(lib().da_sparse_attention(ctypes.byref(pa), ctypes.byref(grid), _stream_ptr(dev)),
              "sparse_attention")
    if debug is not None:  # tests: did the fp32 guard-band selection hand over to the fp64 path?
        off = lib().da_pipeline_fallback_offset(ctypes.byref(grid), heads, d)
        debug["selection_fallback"] = int(ws[off:off + 4].view(torch.int32).item()) != 0
    return RegionMask(g, float(1.0 - sparsity), bitmap, row_ptr, col_idx, thr, forced, kept, single=single)


def _run(q, k, v, plan, sparsity, scale, pool_mode, select_on, force_row_keep, shared_head_mask, qkv_layout, out,
         details=True):
    """Device tensors run on their GPU; host tensors (the reference's calling
    convention) go through the pipelined upload/compute/download path, which
    may write into a caller-provided host ``out``."""
    if q.is_cuda:
        if out is not None:
            raise ValueError("out= is for host inputs; device calls return a fresh tensor")
        o, mask, _ = _pipeline(q, k, v, plan, sparsity, scale, pool_mode, select_on, force_row_keep,
                               shared_head_mask, qkv_layout, want_bitmap=details)
    else:
        o, mask, _ = _pipeline_host(q, k, v, plan, sparsity, scale, pool_mode, select_on, force_row_keep,
                                    shared_head_mask, qkv_layout, out=out, details=details)
    return o, mask


def _run_layout(q, k, v, plan, sparsity, scale, pool_mode, select_on, force_row_keep, shared_head_mask, qkv_layout,
                out, details=True):
    """``_run`` plus the batched DiT layout ``qkv_layout="bnhd"``: (batch, n,
    heads, d) inputs, one pipeline call per batch element on its (n, heads, d)
    slice (no copies), written straight into a (batch, n, heads, dv) output.
    The mask stacks the batch elements' heads, batch-major (per element: one
    mask per head, or one shared mask with ``shared_head_mask``)."""
    if qkv_layout != "bnhd":
        return _run(q, k, v, plan, sparsity, scale, pool_mode, select_on, force_row_keep, shared_head_mask,
                    qkv_layout, out, details)
    for name, x in (("q", q), ("k", k), ("v", v)):
        if not isinstance(x, torch.Tensor) or x.ndim != 4:
            raise ValueError(f"qkv_layout='bnhd' expects (batch, n, heads, d) tensors; {name} has shape "
                             f"{tuple(getattr(x, 'shape', ()))}")
    if k.shape != q.shape:
        raise ValueError(f"k shape {tuple(k.shape)} does not match q shape {tuple(q.shape)}")
    if v.shape[:3] != q.shape[:3]:
        raise ValueError(f"v shape {tuple(v.shape)} does not match q's (batch, n, heads) {tuple(q.shape[:3])}")
    batch, n, heads, _ = q.shape
    dv = v.shape[3]
    out_dtype = _out_dtype(q, k, v)
    masks = []
    if q.is_cuda:
        if out is not None:
            raise ValueError("out= is for host inputs; device calls return a fresh tensor")
        res = torch.empty((batch, n, heads, dv), dtype=torch.bfloat16, device=q.device)
        for b in range(batch):
            _, m_b, _ = _pipeline(q[b], k[b], v[b], plan, sparsity, scale, pool_mode, select_on, force_row_keep,
                                  shared_head_mask, "nhd", want_bitmap=details, out_dev=res[b])
            masks.append(m_b)
        o = res if out_dtype == torch.bfloat16 else res.to(out_dtype)
    else:
        if out is None:
            out = torch.empty((batch, n, heads, dv), dtype=out_dtype, pin_memory=torch.cuda.is_available())
        elif out.shape != (batch, n, heads, dv) or out.dtype != out_dtype or not out.is_contiguous():
            raise ValueError(f"out must be a contiguous CPU tensor of shape {(batch, n, heads, dv)} and dtype {out_dtype}")
        for b in range(batch):
            _, m_b, _ = _pipeline_host(q[b], k[b], v[b], plan, sparsity, scale, pool_mode, select_on, force_row_keep,
                                       shared_head_mask, "nhd", out=out[b], details=details)
            masks.append(m_b)
        o = out
    mask = _cat_masks(masks)
    if mask.single:  # a one-element batch with a shared mask: still indexed per batch element
        mask = dataclasses.replace(mask, single=False)
    return o, mask


def _attend(q, k, v, plan: PadPlan, mask: RegionMask, scale, qkv_layout="hnd", out_dev=None):
    """K4 alone on ORIGINAL-order token tensors with a given mask (one mask
    per head, or one shared by all heads): the executor stage of
    padded_sparse_attention (padding.py:155-157) with the permutation fused.
    Used by the head-parallel path once a cross-rank shared mask is known.
    ``out_dev``: optional bf16 output buffer in the inputs' layout."""
    q3, squeeze = _as_heads(q, qkv_layout, "q")
    k3, _ = _as_heads(k, qkv_layout, "k")
    v3, _ = _as_heads(v, qkv_layout, "v")
    heads, n, d = q3.shape
    if n != plan.num_valid:
        raise ValueError(f"expected {plan.num_valid} real-token rows, got {n}")
    if mask.heads not in (1, heads) or mask.g != plan.layout.num_regions:
        raise ValueError(f"mask of {mask.heads} heads over {mask.g} regions does not fit {heads} heads / "
                         f"{plan.layout.num_regions} regions")
    if d % 8 or v3.shape[2] % 8:
        raise ValueError("_attend needs head dims that are multiples of 8")
    q3, k3, v3 = _prep(q3), _prep(k3), _prep(v3)
    dv = v3.shape[2]
    dev = q3.device
    if out_dev is not None:
        o3, _ = _as_heads(out_dev, qkv_layout, "out")
        if o3.dtype != torch.bfloat16 or tuple(o3.shape) != (heads, n, dv) or o3.stride(2) != 1:
            raise ValueError("output buffer has the wrong shape, dtype or strides")
        o_base = out_dev
    else:
        o_base, o3 = _alloc_like_layout(heads, n, dv, qkv_layout if not squeeze else "hnd", dev)
    lay = plan.layout
    grid = make_grid(plan.frames, plan.height, plan.width, lay.patch_h, lay.patch_w)
    a = _attn_struct(q3, k3, v3, o3, d, dv, _lib.LAYOUT_ORIGINAL, scale)
    a.row_ptr, a.col_idx, a.mask_cap = mask.row_ptr.data_ptr(), mask.col_idx.data_ptr(), mask.col_idx.shape[1]
    a.shared_mask = 1 if mask.heads == 1 else 0
    ws = torch.empty(max(1, lib().da_attn_workspace_size(heads, ctypes.byref(grid))), dtype=torch.uint8, device=dev)
    a.workspace = ws.data_ptr()
    with torch.cuda.device(dev):
        check(lib().da_block_sparse_fwd(ctypes.byref(a), ctypes.byref(grid), _stream_ptr(dev)), "block_sparse_fwd")
    return o3[0] if squeeze else (o_base if qkv_layout == "nhd" else o3)


def padded_block_sparse_attention(q, k, v, plan: PadPlan, mask: RegionMask, scale=None, *, qkv_layout="hnd",
                                  out=None) -> torch.Tensor:
    """The executor stage of padded_sparse_attention (padding.py:155-157:
    embed, permute, block_sparse_attention with key_valid, permute back,
    extract) on ORIGINAL-order tensors with a given mask, the permutation fused
    into the kernel: the way to reuse a cached mask (mask_from_json_dict /
    a previous call's ``res.mask``) across denoising steps without pooling and
    selection. ``mask``: one per head or one shared by all heads, over
    ``plan``'s regions. Inputs as for multi_head_sparse_attention
    ((n, d), (heads, n, d), or (n, heads, d) with qkv_layout="nhd")."""
    if qkv_layout not in ("hnd", "nhd"):
        raise ValueError(f"qkv_layout must be 'hnd' or 'nhd', got {qkv_layout!r}")
    q3, squeeze = _as_heads(q, qkv_layout, "q")
    k3, _ = _as_heads(k, qkv_layout, "k")
    v3, _ = _as_heads(v, qkv_layout, "v")
    if k3.shape != q3.shape or v3.shape[:2] != q3.shape[:2]:
        raise ValueError(f"q {tuple(q3.shape)}, k {tuple(k3.shape)} and v {tuple(v3.shape)} do not match")
    if scale is None:
        scale = head_dim_scale(q3.shape[2])
    out_dtype = _out_dtype(q, k, v)
    dv0 = v3.shape[2]
    if q3.shape[2] % 8 or dv0 % 8:  # exact zero features, as the pipeline does
        o = _attend(_pad_features(q3), _pad_features(k3), _pad_features(v3), plan, mask, scale)[..., :dv0]
        o = o[0] if squeeze else (o.transpose(0, 1) if qkv_layout == "nhd" else o)
    else:
        o = _attend(q, k, v, plan, mask, scale, qkv_layout)
    o = o.to(out_dtype) if o.dtype != out_dtype else o
    if out is not None:
        if tuple(out.shape) != tuple(o.shape) or out.dtype != o.dtype:
            raise ValueError(f"out must have shape {tuple(o.shape)} and dtype {o.dtype}")
        out.copy_(o)
        return out
    return o


# --------------------------------------------------------------------------
# sequence shards (no reference counterpart: the reference is single-process)
# --------------------------------------------------------------------------

@dataclass(frozen=True)
class ShardTable:
    """Token tensors split into row blocks: q/k/v/out[s] are the device
    addresses of element (head 0, local row 0) of shard s, which holds tokens
    [s * rows, s * rows + rows_s) in original order (every shard but the last
    has ``rows`` rows). The addresses may be other GPUs' memory mapped into
    this process (``headpar.PeerShards``); the kernels then read and write the
    peers' rows over NVLink. ``strides``: element strides (head, row) of q, k,
    v and out, shared by all shards."""
    q: tuple
    k: tuple
    v: tuple
    out: tuple
    rows: int
    n: int
    heads: int
    d: int
    dv: int
    strides: tuple  # (qh, qr, kh, kr, vh, vr, oh, orow)

    def struct(self, scale) -> DaAttnArgs:
        a = DaAttnArgs()
        (a.q_head_stride, a.q_row_stride, a.k_head_stride, a.k_row_stride,
         a.v_head_stride, a.v_row_stride, a.o_head_stride, a.o_row_stride) = self.strides
        a.heads, a.d, a.dv, a.layout = self.heads, self.d, self.dv, _lib.LAYOUT_ORIGINAL
        a.scale = float(scale)
        a.shard_count, a.shard_rows = len(self.q), self.rows
        a.q, a.k, a.v, a.out = self.q[0], self.k[0], self.v[0], self.out[0]  # (one shard: a plain tensor)
        for i in range(len(self.q)):
            a.q_shards[i], a.k_shards[i] = self.q[i], self.k[i]
            a.v_shards[i], a.out_shards[i] = self.v[i], self.out[i]
        return a


def _shard_table(qs, ks, vs, outs) -> ShardTable:
    """ShardTable of lists of (rows_s, heads, d) CUDA tensors (the "nhd" layout)."""
    count = len(qs)
    if not 2 <= count <= _lib.MAX_SHARDS or not len(ks) == len(vs) == len(outs) == count:
        raise ValueError(f"need 2..{_lib.MAX_SHARDS} shards of q, k, v and out, got "
                         f"{len(qs)}, {len(ks)}, {len(vs)}, {len(outs)}")
    rows = qs[0].shape[0]
    heads, d = qs[0].shape[1], qs[0].shape[2]
    dv = vs[0].shape[2]
    for s in range(count):
        q, k, v, o = qs[s], ks[s], vs[s], outs[s]
        for x, name, last in ((q, "q", d), (k, "k", d), (v, "v", dv), (o, "out", dv)):
            if not isinstance(x, torch.Tensor) or not x.is_cuda or x.dtype != torch.bfloat16 or x.ndim != 3:
                raise ValueError(f"{name} shard {s} must be a 3-d bf16 CUDA tensor (rows, heads, d)")
            if x.shape[1:] != (heads, last) or x.shape[0] != q.shape[0]:
                raise ValueError(f"{name} shard {s} has shape {tuple(x.shape)}, expected "
                                 f"({q.shape[0]}, {heads}, {last})")
            ref = {"q": qs[0], "k": ks[0], "v": vs[0], "out": outs[0]}[name]
            if x.stride() != ref.stride() or x.stride(2) != 1 or x.data_ptr() % 16:
                raise ValueError(f"{name} shards need identical strides, unit feature stride and 16-byte alignment")
        if (s < count - 1 and q.shape[0] != rows) or not 1 <= q.shape[0] <= rows:
            raise ValueError(f"every shard but the last must hold {rows} rows (the last 1..{rows}), "
                             f"shard {s} holds {q.shape[0]}")
    if d % 8 or dv % 8:
        raise ValueError("sharded calls need head dims that are multiples of 8")
    n = rows * (count - 1) + qs[-1].shape[0]
    q0, k0, v0, o0 = qs[0], ks[0], vs[0], outs[0]
    return ShardTable(tuple(x.data_ptr() for x in qs), tuple(x.data_ptr() for x in ks),
                      tuple(x.data_ptr() for x in vs), tuple(x.data_ptr() for x in outs), rows, n, heads, d, dv,
                      (q0.stride(1), q0.stride(0), k0.stride(1), k0.stride(0), v0.stride(1), v0.stride(0),
                       o0.stride(1), o0.stride(0)))


def _run_sharded(table: ShardTable, plan: PadPlan, sparsity, scale, pool_mode="average", select_on="logits",
                 force_row_keep=True, shared_head_mask=False, device=None, want_bitmap=False, attn_events=None,
                 mask: RegionMask | None = None) -> RegionMask:
    """The pipeline (or, with ``mask``, the executor alone) over a ShardTable,
    on ``device``'s current stream. Returns the mask."""
    if table.n != plan.num_valid:
        raise ValueError(f"shards hold {table.n} rows, the layout has {plan.num_valid} tokens")
    scale = head_dim_scale(table.d) if scale is None else scale
    a = table.struct(scale)
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    if mask is None:
        _validate_pipeline_args(sparsity, select_on, pool_mode)
        return _launch_pipeline(a, plan, sparsity, pool_mode, select_on, force_row_keep, shared_head_mask, dev,
                                want_bitmap, attn_events, single=shared_head_mask)
    if mask.heads not in (1, table.heads) or mask.g != plan.layout.num_regions:
        raise ValueError(f"mask of {mask.heads} heads over {mask.g} regions does not fit {table.heads} heads / "
                         f"{plan.layout.num_regions} regions")
    lay = plan.layout
    grid = make_grid(plan.frames, plan.height, plan.width, lay.patch_h, lay.patch_w)
    a.row_ptr, a.col_idx, a.mask_cap = mask.row_ptr.data_ptr(), mask.col_idx.data_ptr(), mask.col_idx.shape[1]
    a.shared_mask = 1 if mask.heads == 1 else 0
    ws = torch.empty(max(1, lib().da_attn_workspace_size(table.heads, ctypes.byref(grid))), dtype=torch.uint8,
                     device=dev)
    a.workspace = ws.data_ptr()
    with torch.cuda.device(dev):
        check(lib().da_block_sparse_fwd(ctypes.byref(a), ctypes.byref(grid), _stream_ptr(dev)), "block_sparse_fwd")
    return mask


def sharded_sparse_attention(q_shards, k_shards, v_shards, plan: PadPlan, sparsity, scale=None,
                             pool_mode="average", select_on="logits", force_row_keep=True,
                             shared_head_mask=False, *, out_shards=None, mask: RegionMask | None = None,
                             return_mask=False):
    """``multi_head_sparse_attention`` (per-head masks, or ``shared_head_mask``)
    over a sequence held as row blocks: ``q_shards[s]`` etc. are (rows_s,
    heads, d) bf16 CUDA tensors (the DiT "nhd" layout) holding tokens
    [s * rows_0, s * rows_0 + rows_s) in original order, every shard but the
    last with rows_0 rows (2 .. 8 shards). The kernels address the shards in
    place (no gather). ``out_shards``: (rows_s, heads, dv) output buffers (new
    ones if None). ``mask``: run the executor alone with this mask (cached
    masks, ``padded_block_sparse_attention``). Returns the output shards
    (and the mask with ``return_mask``). ``headpar.HeadParallelAttention``
    with ``transport="peer"`` uses the same C-ABI path with other GPUs'
    shards."""
    if out_shards is None:
        out_shards = [torch.empty(q.shape[:2] + (v.shape[2],), dtype=torch.bfloat16, device=q.device)
                      for q, v in zip(q_shards, v_shards)]
    table = _shard_table(list(q_shards), list(k_shards), list(v_shards), list(out_shards))
    m = _run_sharded(table, plan, sparsity, scale, pool_mode, select_on, force_row_keep, shared_head_mask,
                     q_shards[0].device, want_bitmap=return_mask, mask=mask)
    return (list(out_shards), m) if return_mask else list(out_shards)


def _cat_masks(masks) -> RegionMask:
    """Stack per-head-group masks of one call (same g, keep ratio, capacity)."""
    if len(masks) == 1:
        return masks[0]
    m0 = masks[0]
    cat = lambda name: torch.cat([getattr(m, name) for m in masks], 0)  # noqa: E731
    packed = None if any(m.packed is None for m in masks) else cat("packed")
    return RegionMask(m0.g, m0.keep_ratio, packed, cat("row_ptr"), cat("col_idx"), cat("thresholds"),
                      cat("forced"), cat("kept_counts"), single=False)


def _head_groups(heads: int, hg: int):
    """Head ranges [h0, h1) of a pipelined host call: groups of ``hg`` heads,
    except that the first group's upload and the last group's compute +
    download overlap nothing, so those two are half as large."""
    edge = max(1, hg // 2) if heads >= 2 * hg else hg
    bounds = [0] + ([edge] if edge < hg else [])
    while bounds[-1] < heads:
        left = heads - bounds[-1]
        bounds.append(bounds[-1] + (left if left <= edge or left <= hg else min(hg, left - edge)))
    return list(zip(bounds[:-1], bounds[1:]))


def _pipeline_host(q, k, v, plan: PadPlan, sparsity, scale, pool_mode, select_on, force_row_keep,
                   shared_head_mask, qkv_layout, group_heads=None, out=None, details=True):
    """Host (CPU) inputs, the reference's calling convention: the call stages
    Q/K/V to the GPU in head groups on a copy stream, runs each group's
    pipeline on the current stream while the next group uploads, copies each
    group's output back on a third stream, and returns once the output is in
    (pinned) host memory. Heads are independent (per-head masks), so the
    result equals one all-head call. Compute stays on the GPU: without CUDA
    this raises (there is no CPU path)."""
    if not torch.cuda.is_available():
        raise RuntimeError("host inputs are staged to the GPU; no CUDA device is available (no CPU fallback)")
    q3, squeeze = _as_heads(q, qkv_layout, "q")
    k3, _ = _as_heads(k, qkv_layout, "k")
    v3, _ = _as_heads(v, qkv_layout, "v")
    heads, n, _ = q3.shape
    dv = v3.shape[2]
    dev = torch.device("cuda", torch.cuda.current_device())
    out_dtype = _out_dtype(q, k, v)
    main = torch.cuda.current_stream(dev)
    contiguous = all(x.is_contiguous() for x in (q3, k3, v3))
    hg = group_heads or max(1, -(-heads // 12))
    if shared_head_mask or heads == 1 or not contiguous:
        groups = [(0, heads)]  # the head-mean mask needs every head at once
    else:
        groups = _head_groups(heads, hg)
    s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    if out is not None:
        # validated in the caller's own layout: (n, dv), (heads, n, dv) or, for
        # qkv_layout="nhd", (n, heads, dv)
        want = (n, dv) if squeeze else ((n, heads, dv) if qkv_layout == "nhd" else (heads, n, dv))
        if not isinstance(out, torch.Tensor) or out.device.type != "cpu" or tuple(out.shape) != want or \
                out.dtype != out_dtype or not out.is_contiguous():
            raise ValueError(f"out must be a contiguous CPU tensor of shape {want} and dtype {out_dtype}")
        out_host, _ = _as_heads(out, qkv_layout, "out")
    else:
        # pinned so the per-group downloads are asynchronous (pass out= to reuse a buffer)
        out_host = torch.empty((heads, n, dv), dtype=out_dtype, pin_memory=True)
    # Device staging for the whole call, allocated once on the compute stream:
    # the uploads (s_in) and downloads (s_out) only touch slices of these, and
    # every group's compute waits for its upload, so no cross-stream frees.
    dev_in = [torch.empty(x.shape, dtype=x.dtype, device=dev) for x in (q3, k3, v3)]
    direct_out = len(groups) > 1 and out_dtype == torch.bfloat16
    out_dev = torch.empty((heads, n, dv), dtype=torch.bfloat16, device=dev) if direct_out else None
    s_in.wait_stream(main)
    s_out.wait_stream(main)
    masks = []
    for h0, h1 in groups:
        with torch.cuda.stream(s_in):
            for x, y in zip((q3, k3, v3), dev_in):
                y[h0:h1].copy_(x[h0:h1], non_blocking=True)
            ev_in = torch.cuda.Event()
            ev_in.record(s_in)
        main.wait_event(ev_in)
        qd, kd, vd = (y[h0:h1] for y in dev_in)
        out_g, mask_g, _ = _pipeline(qd, kd, vd, plan, sparsity, scale, pool_mode, select_on, force_row_keep,
                                     shared_head_mask, "hnd", want_bitmap=details,
                                     out_dev=out_dev[h0:h1] if direct_out else None)
        if out_g.dtype != out_dtype:
            out_g = out_g.to(out_dtype)
        ev_c = torch.cuda.Event()
        ev_c.record(main)
        with torch.cuda.stream(s_out):
            s_out.wait_event(ev_c)
            out_host[h0:h1].copy_(out_g, non_blocking=True)
        if not direct_out:
            out_g.record_stream(s_out)
        masks.append(mask_g)
    main.wait_stream(s_out)
    s_out.synchronize()
    res = out_host[0] if squeeze else (out_host.transpose(0, 1) if qkv_layout == "nhd" else out_host)
    return res, _cat_masks(masks), squeeze


def _rows_and_dim(q, qkv_layout: str):
    """(token rows, head dim) of q in the caller's layout."""
    if qkv_layout == "bnhd":
        if not isinstance(q, torch.Tensor) or q.ndim != 4:
            raise ValueError(f"qkv_layout='bnhd' expects (batch, n, heads, d) tensors, got shape "
                             f"{tuple(getattr(q, 'shape', ()))}")
        return q.shape[1], q.shape[3]
    q3, _ = _as_heads(q, qkv_layout, "q")
    return q3.shape[1], q3.shape[2]


def _details(out, mask: RegionMask, layout: LatentLayout, d: int):
    if mask.single:
        return PipelineResult(out, mask, flops_count(layout, d, kept_count=int(mask.kept_count)),
                              mask_density_stats(mask))
    flops = [flops_count(layout, d, kept_count=int(c)) for c in mask.kept_count]
    stats = [mask_density_stats(mask, h) for h in range(mask.heads)]
    return PipelineResult(out, mask, flops, stats)


# --------------------------------------------------------------------------
# public operators
# --------------------------------------------------------------------------

def padded_sparse_attention(q, k, v, frames, height, width, patch_h, patch_w, sparsity,
                            scale=None, pool_mode="average", select_on="logits",
                            force_row_keep=True, two_pass=False, return_details=False,
                            *, qkv_layout="hnd", out=None):
    """Draft-guided block-sparse attention on any grid (padding.py:95-165).

    Ragged grids are padded inside the kernels: pooling averages over real
    tokens only, padded keys are masked, padded rows never reach the output.
    ``two_pass`` (the reference's debug executor) computes the same function
    and is accepted for signature compatibility.
    """
    del two_pass
    plan = pad_plan(frames, height, width, patch_h, patch_w)
    _validate_pipeline_args(sparsity, select_on, pool_mode)
    if not plan.is_identity and pool_mode != "average":
        raise ValueError("padded grids support average pooling only")
    rows, d = _rows_and_dim(q, qkv_layout)
    if rows != plan.num_valid:
        raise ValueError(f"expected ({plan.num_valid}, d) real-token rows, got {tuple(q.shape)}")
    if scale is None:
        scale = head_dim_scale(d)
    out, mask = _run_layout(q, k, v, plan, sparsity, scale, pool_mode, select_on, force_row_keep, False, qkv_layout,
                            out, return_details)
    if not return_details:
        return out
    return _details(out, mask, plan.layout, d)


def draft_sparse_attention(q, k, v, layout: LatentLayout, sparsity, scale=None, pool_mode="average",
                           select_on="logits", force_row_keep=True, two_pass=False,
                           return_details=False, *, qkv_layout="hnd", out=None):
    """Full pipeline on a divisible grid (sparse.py:193-246)."""
    del two_pass
    _validate_pipeline_args(sparsity, select_on, pool_mode)
    rows, d = _rows_and_dim(q, qkv_layout)
    if rows != layout.num_tokens:
        raise ValueError(f"q rows {rows} != layout token count {layout.num_tokens}")
    if scale is None:
        scale = head_dim_scale(d)
    plan = PadPlan(layout.frames, layout.height, layout.width, layout)
    out, mask = _run_layout(q, k, v, plan, sparsity, scale, pool_mode, select_on, force_row_keep, False, qkv_layout,
                            out, return_details)
    if not return_details:
        return out
    return _details(out, mask, layout, d)


def multi_head_sparse_attention(q, k, v, layout: LatentLayout, sparsity, shared_head_mask=False,
                                scale=None, pool_mode="average", select_on="logits",
                                force_row_keep=True, *, qkv_layout="hnd", return_details=False, out=None):
    """Stacked (heads, n, d) inputs (sparse.py:249-302); all heads in one launch per stage.

    ``layout`` may also be a PadPlan for ragged grids (the reference has no
    padded multi-head entry; this is the batched form of its per-head loop).
    """
    if q.ndim != (4 if qkv_layout == "bnhd" else 3):
        raise ValueError(f"expected (heads, n, d) inputs, got shape {tuple(q.shape)}")
    _validate_pipeline_args(sparsity, select_on, pool_mode)
    plan = layout if isinstance(layout, PadPlan) else PadPlan(layout.frames, layout.height,
                                                                layout.width, layout)
    if not plan.is_identity and pool_mode != "average":
        raise ValueError("padded grids support average pooling only")
    rows, d = _rows_and_dim(q, qkv_layout)
    if rows != plan.num_valid:
        raise ValueError(f"q rows {rows} != layout token count {plan.num_valid}")
    if scale is None:
        scale = head_dim_scale(d)
    out, mask = _run_layout(q, k, v, plan, sparsity, scale, pool_mode, select_on, force_row_keep, shared_head_mask,
                            qkv_layout, out, return_details)
    if not return_details:
        return out
    return _details(out, mask, plan.layout, d)


# --------------------------------------------------------------------------
# lower seams
# --------------------------------------------------------------------------

def reorder_tokens(x, plan: PadPlan, *, qkv_layout="hnd") -> torch.Tensor:
    """permute_rows(embed_rows(x, plan), perm) (padding.py:140-142): K1, bit-exact.

    Returns dense (heads, n_pad, d) (or (n_pad, d) for 2-d input) in patch-contiguous order.
    """
    x3, squeeze = _as_heads(x, qkv_layout, "x")
    d0 = x3.shape[2]
    x3 = _prep(x3) if d0 % 8 == 0 else _pad_features(x3)
    heads, n, d = x3.shape
    if n != plan.num_valid:
        raise ValueError(f"expected ({plan.num_valid}, d) real-token rows, got {tuple(x.shape)}")
    lay = plan.layout
    out = torch.empty((heads, lay.num_tokens, d), dtype=torch.bfloat16, device=x3.device)
    grid = make_grid(plan.frames, plan.height, plan.width, lay.patch_h, lay.patch_w)
    with torch.cuda.device(x3.device):
        check(lib().da_permute_in(x3.data_ptr(), x3.stride(0), x3.stride(1), out.data_ptr(), heads, d,
                                  ctypes.byref(grid), _stream_ptr(x3.device)), "permute_in")
    out = out[..., :d0] if d0 != d else out
    return out[0] if squeeze else out


def restore_tokens(x_r, plan: PadPlan) -> torch.Tensor:
    """extract_rows(permute_rows(x_r, perm.inverse), plan) (padding.py:157): K5, bit-exact."""
    x3, squeeze = _as_heads(x_r, "hnd", "x_r")
    d0 = x3.shape[2]
    x3 = _prep(x3).contiguous() if d0 % 8 == 0 else _pad_features(x3)
    heads, n_pad, d = x3.shape
    lay = plan.layout
    if n_pad != lay.num_tokens:
        raise ValueError(f"expected {lay.num_tokens} padded rows, got {n_pad}")
    out = torch.empty((heads, plan.num_valid, d), dtype=torch.bfloat16, device=x3.device)
    grid = make_grid(plan.frames, plan.height, plan.width, lay.patch_h, lay.patch_w)
    with torch.cuda.device(x3.device):
        check(lib().da_permute_out(x3.data_ptr(), out.data_ptr(), out.stride(0), out.stride(1), heads, d,
                                   ctypes.byref(grid), _stream_ptr(x3.device)), "permute_out")
    out = out[..., :d0] if d0 != d else out
    return out[0] if squeeze else out


def pool_tokens(x, plan: PadPlan, mode="average", *, qkv_layout="hnd") -> torch.Tensor:
    """Region pooling straight from original token order, float64 result (K2).

    Equals pool_regions_valid(permute_rows(embed_rows(x)), valid_r, p)
    (padding.py:78-92) on ragged grids and pool_regions (pooling.py:12-32) on
    divisible ones.
    """
    if mode not in POOL_MODES:
        raise ValueError(f"mode must be one of {POOL_MODES}, got {mode!r}")
    if mode != "average" and not plan.is_identity:
        raise ValueError("padded grids support average pooling only")
    x3, squeeze = _as_heads(x, qkv_layout, "x")
    d0 = x3.shape[2]
    x3 = _prep(x3) if d0 % 8 == 0 else _pad_features(x3)
    heads, n, d = x3.shape
    lay = plan.layout
    out = torch.empty((heads, lay.num_regions, d), dtype=torch.float64, device=x3.device)
    grid = make_grid(plan.frames, plan.height, plan.width, lay.patch_h, lay.patch_w)
    with torch.cuda.device(x3.device):
        check(lib().da_pool(x3.data_ptr(), x3.stride(0), x3.stride(1), out.data_ptr(), heads, d, ctypes.byref(grid),
                            POOL_MODES.index(mode), _stream_ptr(x3.device)), "pool")
    out = out[..., :d0] if d0 != d else out
    return out[0] if squeeze else out


def pool_regions(x_r, region_size: int, mode="average") -> torch.Tensor:
    """Contiguous region mean/max of reordered rows (pooling.py:12-32), float64 result."""
    if mode not in POOL_MODES:
        raise ValueError(f"mode must be one of {POOL_MODES}, got {mode!r}")
    x3, squeeze = _as_heads(x_r, "hnd", "x")
    n = x3.shape[1]
    if region_size < 1:
        raise ValueError(f"region_size must be positive, got {region_size}")
    if n % region_size != 0:
        raise ValueError(f"row count {n} is not a multiple of region_size {region_size}")
    # contiguous regions == a grid of n/p frames of one 1 x p patch each
    plan = pad_plan(n // region_size, 1, region_size, 1, region_size)
    out = pool_tokens(x3, plan, mode)
    return out[0] if squeeze else out


def draft_logits(q_pooled, k_pooled, scale=None, head_dim=None, *, softmax=False) -> torch.Tensor:
    """scale * q_pooled @ k_pooled^T in float64 (pooling.py:35-56, core.py:20-35): K3a."""
    if scale is not None and head_dim is not None:
        raise ValueError("pass at most one of scale and head_dim")
    qp3, squeeze = _as_heads(q_pooled, "hnd", "q_pooled")
    kp3, _ = _as_heads(k_pooled, "hnd", "k_pooled")
    if qp3.shape[2] != kp3.shape[2]:
        raise ValueError(f"head_dim mismatch: q has {qp3.shape[2]}, k has {kp3.shape[2]}")
    if qp3.shape[1] != kp3.shape[1]:
        raise ValueError("draft scores need the same number of query and key regions")
    if head_dim is not None:
        scale = head_dim_scale(head_dim)
    if scale is None:
        scale = head_dim_scale(qp3.shape[2])
    qp3 = qp3.to(torch.float64).contiguous()
    kp3 = kp3.to(torch.float64).contiguous()
    heads, g, d = qp3.shape
    out = torch.empty((heads, g, g), dtype=torch.float64, device=qp3.device)
    with torch.cuda.device(qp3.device):
        check(lib().da_draft_scores(qp3.data_ptr(), kp3.data_ptr(), out.data_ptr(), heads, g, d, float(scale),
                                    1 if softmax else 0, _stream_ptr(qp3.device)), "draft_scores")
    return out[0] if squeeze else out


def draft_attention_map(q_pooled, k_pooled, scale=None) -> torch.Tensor:
    """Row-softmaxed draft map of the pooled sequences (pooling.py:59-65):
    softmax_rows(draft_logits(q_pooled, k_pooled, scale)), float64."""
    return draft_logits(q_pooled, k_pooled, scale, softmax=True)


def select_top_fraction(scores, keep_ratio: float, force_row_keep: bool = False,
                        dead_columns=None) -> RegionMask:
    """Global top-ceil(r*g^2) with flat-index ties (+ row argmax keep) (masking.py:59-91): K3b.

    ``scores`` is (g, g) or (heads, g, g) on the GPU (computed in float64).
    ``dead_columns`` (optional) are dropped afterwards (masking.py:94-105).
    """
    s3, squeeze = _as_heads(scores, "hnd", "scores")
    if s3.shape[1] != s3.shape[2]:
        raise ValueError(f"expected a square score matrix, got shape {tuple(scores.shape)}")
    heads, g, _ = s3.shape
    m = top_fraction_count(g * g, keep_ratio)
    s3 = s3.to(torch.float64).contiguous()
    dev = s3.device
    cap = m + g
    row_ptr = torch.empty((heads, g + 1), dtype=torch.int32, device=dev)
    col_idx = torch.empty((heads, cap), dtype=torch.int32, device=dev)
    bitmap = torch.empty((heads, (g * g + 7) // 8), dtype=torch.uint8, device=dev)
    thr = torch.empty(heads, dtype=torch.float64, device=dev)
    forced = torch.empty(heads, dtype=torch.int64, device=dev)
    kept = torch.empty(heads, dtype=torch.int64, device=dev)
    ws = torch.empty(lib().da_select_workspace_size(heads, g), dtype=torch.uint8, device=dev)
    dead_ptr = None
    if dead_columns is not None:
        dead = torch.zeros(g, dtype=torch.uint8, device=dev)
        idx = torch.as_tensor(dead_columns, dtype=torch.int64, device=dev)
        if idx.numel():
            dead[idx] = 1
        dead_ptr = dead.data_ptr()
    with torch.cuda.device(dev):
        check(lib().da_select(s3.data_ptr(), heads, g, m, 1 if force_row_keep else 0, dead_ptr, ws.data_ptr(),
                              row_ptr.data_ptr(), col_idx.data_ptr(), bitmap.data_ptr(), thr.data_ptr(),
                              forced.data_ptr(), kept.data_ptr(), _stream_ptr(dev)), "select")
    return RegionMask(g, float(keep_ratio), bitmap, row_ptr, col_idx, thr, forced, kept, single=squeeze)


def block_sparse_attention(q_r, k_r, v_r, mask: RegionMask, scale=None, key_valid=None, two_pass=False,
                           *, force_portable=False) -> torch.Tensor:
    """Executor over reordered inputs, kept key blocks only (sparse.py:88-166): K4.

    q_r/k_r/v_r: (n, d) or (heads, n, d) in patch-contiguous order; ``mask``
    from select_top_fraction (one head, or one per input head). ``key_valid``:
    optional bool (n,) of keys allowed to receive attention. Output stays in
    reordered order.
    """
    del two_pass
    q3, squeeze = _as_heads(q_r, "hnd", "q")
    k3, _ = _as_heads(k_r, "hnd", "k")
    v3, _ = _as_heads(v_r, "hnd", "v")
    heads, n, d = q3.shape
    if k3.shape != q3.shape:
        raise ValueError(f"k shape {tuple(k3.shape)} does not match q shape {tuple(q3.shape)}")
    if v3.shape[1] != n:
        raise ValueError(f"v rows {v3.shape[1]} != key rows {n}")
    g = mask.g
    if n % g != 0:
        raise ValueError(f"token count {n} is not a multiple of region count {g}")
    p = n // g
    if scale is None:
        scale = head_dim_scale(d)
    out_dtype = _out_dtype(q_r, k_r, v_r)
    dv0 = v3.shape[2]
    if d % 8 or dv0 % 8:  # zero features: exact (see _pad_features)
        q3, k3, v3 = _pad_features(q3), _pad_features(k3), _pad_features(v3)
    else:
        q3, k3, v3 = _prep(q3), _prep(k3), _prep(v3)
    d = q3.shape[2]
    dv = v3.shape[2]
    kv_ptr = None
    if key_valid is not None:
        kv = torch.as_tensor(key_valid, device=q3.device).to(torch.bool)
        if tuple(kv.shape) != (n,):
            raise ValueError(f"key_valid shape {tuple(kv.shape)} != ({n},)")
        kv = kv.to(torch.uint8).contiguous()
        kv_ptr = kv.data_ptr()
    if mask.heads not in (1, heads):
        raise ValueError(f"mask has {mask.heads} heads for {heads} input heads")
    out = torch.empty((heads, n, dv), dtype=torch.bfloat16, device=q3.device)
    # a reordered (g*p)-row tensor is the grid of g frames of one 1 x p patch
    grid = make_grid(g, 1, p, 1, p)
    a = _attn_struct(q3, k3, v3, out, d, dv, _lib.LAYOUT_REORDERED, scale)
    a.row_ptr, a.col_idx, a.mask_cap = mask.row_ptr.data_ptr(), mask.col_idx.data_ptr(), mask.col_idx.shape[1]
    a.key_valid = kv_ptr
    a.shared_mask = 1 if mask.heads == 1 else 0
    a.force_portable = 1 if force_portable else 0
    ws = torch.empty(max(1, lib().da_attn_workspace_size(heads, ctypes.byref(grid))), dtype=torch.uint8,
                     device=q3.device)
    a.workspace = ws.data_ptr()
    with torch.cuda.device(q3.device):
        check(lib().da_block_sparse_fwd(ctypes.byref(a), ctypes.byref(grid), _stream_ptr(q3.device)),
              "block_sparse_fwd")
    out = out[..., :dv0] if dv0 != dv else out
    out = out[0] if squeeze else out
    return out.to(out_dtype) if out_dtype != torch.bfloat16 else out
