"""ctypes binding of the C ABI in include/draftattn_b200.h.

The shared library is built in-tree (``python -c "import __graft_entry__ as g;
g.build()"`` or ``python -m paper_2505_14708_b200.build``) and loaded from this
package directory. There is no fallback: if the library is missing, every
entry point raises.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

LIB_NAME = "libdraftattn_b200.so"
LIB_PATH = Path(__file__).resolve().parent / LIB_NAME

DA_OK, DA_EINVAL, DA_ECUDA = 0, 1, 2
ABI_VERSION = 101  # da_version() of the library these struct layouts match
LAYOUT_REORDERED, LAYOUT_ORIGINAL = 0, 1
MAX_SHARDS = 8
IPC_HANDLE_BYTES = 64

c_i32, c_i64, c_f64, c_vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_double, ctypes.c_void_p


class DaGrid(ctypes.Structure):
    _fields_ = [("frames", c_i32), ("height", c_i32), ("width", c_i32),
                ("patch_h", c_i32), ("patch_w", c_i32)]


class DaAttnArgs(ctypes.Structure):
    _fields_ = [
        ("q", c_vp), ("k", c_vp), ("v", c_vp), ("out", c_vp),
        ("q_head_stride", c_i64), ("q_row_stride", c_i64),
        ("k_head_stride", c_i64), ("k_row_stride", c_i64),
        ("v_head_stride", c_i64), ("v_row_stride", c_i64),
        ("o_head_stride", c_i64), ("o_row_stride", c_i64),
        ("heads", c_i32), ("d", c_i32), ("dv", c_i32), ("layout", c_i32),
        ("scale", c_f64),
        ("row_ptr", c_vp), ("col_idx", c_vp), ("mask_cap", c_i64),
        ("key_valid", c_vp),
        ("shared_mask", c_i32), ("force_portable", c_i32),
        ("workspace", c_vp),
        ("shard_count", c_i32), ("shard_rows", c_i64),
        ("q_shards", c_vp * MAX_SHARDS), ("k_shards", c_vp * MAX_SHARDS),
        ("v_shards", c_vp * MAX_SHARDS), ("out_shards", c_vp * MAX_SHARDS),
    ]


class DaPipelineArgs(ctypes.Structure):
    _fields_ = [
        ("attn", DaAttnArgs),
        ("m", c_i64), ("force_row_keep", c_i32), ("pool_mode", c_i32),
        ("select_softmax", c_i32), ("shared_head_mask", c_i32),
        ("row_ptr", c_vp), ("col_idx", c_vp), ("bitmap", c_vp),
        ("threshold", c_vp), ("forced", c_vp), ("kept", c_vp),
        ("workspace", c_vp),
        ("ev_attn_begin", c_vp), ("ev_attn_end", c_vp),
    ]


# name -> (restype, argtypes); every symbol declared in include/draftattn_b200.h
SIGNATURES = {
    "da_num_regions": (c_i32, [ctypes.POINTER(DaGrid)]),
    "da_region_size": (c_i32, [ctypes.POINTER(DaGrid)]),
    "da_padded_tokens": (c_i64, [ctypes.POINTER(DaGrid)]),
    "da_version": (c_i32, []),
    "da_last_error": (ctypes.c_char_p, []),
    "da_mask_capacity": (c_i64, [c_i32, c_i64]),
    "da_permute_in": (ctypes.c_int, [c_vp, c_i64, c_i64, c_vp, c_i32, c_i32, ctypes.POINTER(DaGrid), c_vp]),
    "da_permute_out": (ctypes.c_int, [c_vp, c_vp, c_i64, c_i64, c_i32, c_i32, ctypes.POINTER(DaGrid), c_vp]),
    "da_pool": (ctypes.c_int, [c_vp, c_i64, c_i64, c_vp, c_i32, c_i32, ctypes.POINTER(DaGrid), c_i32, c_vp]),
    "da_draft_scores": (ctypes.c_int, [c_vp, c_vp, c_vp, c_i32, c_i32, c_i32, c_f64, c_i32, c_vp]),
    "da_select_workspace_size": (ctypes.c_size_t, [c_i32, c_i32]),
    "da_select": (ctypes.c_int, [c_vp, c_i32, c_i32, c_i64, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp,
                                 c_vp, c_vp, c_vp, c_vp]),
    "da_attn_workspace_size": (ctypes.c_size_t, [c_i32, ctypes.POINTER(DaGrid)]),
    "da_block_sparse_fwd": (ctypes.c_int, [ctypes.POINTER(DaAttnArgs), ctypes.POINTER(DaGrid), c_vp]),
    "da_pipeline_workspace_size": (ctypes.c_size_t, [ctypes.POINTER(DaGrid), c_i32, c_i32]),
    "da_pipeline_launches": (c_i32, [c_i32, c_i32]),
    "da_pipeline_fallback_offset": (ctypes.c_int64, [ctypes.POINTER(DaGrid), c_i32, c_i32]),
    "da_debug_trace": (ctypes.c_int, [c_vp]),
    "da_ipc_export": (ctypes.c_int, [c_vp, c_vp, ctypes.POINTER(c_i64)]),
    "da_ipc_open": (ctypes.c_int, [c_vp, c_i64, ctypes.POINTER(c_vp)]),
    "da_ipc_close": (ctypes.c_int, [c_vp, c_i64]),
    "da_sparse_attention": (ctypes.c_int, [ctypes.POINTER(DaPipelineArgs), ctypes.POINTER(DaGrid), c_vp]),
}

_LIB = None


def lib() -> ctypes.CDLL:
    """Load the in-tree library (once). Raises if it has not been built."""
    global _LIB
    if _LIB is None:
        path = os.environ.get("DRAFTATTN_B200_LIB", str(LIB_PATH))
        if not Path(path).exists():
            raise RuntimeError(
                f"{LIB_NAME} not found at {path}: build it with "
                "`python -m paper_2505_14708_b200.build` (no CPU fallback exists)")
        handle = ctypes.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        if handle.da_version() != ABI_VERSION:  # a stale build would misread the argument structs
            raise RuntimeError(f"{path} has ABI version {handle.da_version()}, this package needs {ABI_VERSION}: "
                               "rebuild it with `python -m paper_2505_14708_b200.build`")
        _LIB = handle
    return _LIB


def check(rc: int, what: str) -> None:
    """Raise on a nonzero C-ABI status, with the library's thread-local message."""
    if rc == DA_OK:
        return
    msg = lib().da_last_error().decode(errors="replace")
    if rc == DA_EINVAL:
        raise ValueError(f"{what}: {msg}")
    raise RuntimeError(f"{what}: {msg}")


def make_grid(frames, height, width, patch_h, patch_w) -> DaGrid:
    return DaGrid(int(frames), int(height), int(width), int(patch_h), int(patch_w))
