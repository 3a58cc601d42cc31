"""C-ABI library: loads without a GPU, exports every declared symbol, host-only
entry points and argument validation behave (CPU only)."""

import ctypes
import re
from pathlib import Path

import pytest

from paper_2505_14708_b200 import _lib
from paper_2505_14708_b200.build import build

ROOT = Path(__file__).resolve().parents[1]


@pytest.fixture(scope="module")
def L():
    build()
    return _lib.lib()


def _declared_symbols():
    text = (ROOT / "include" / "draftattn_b200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(da_[a-z_0-9]+)\s*\(", text)))


def test_every_declared_symbol_is_exported(L):
    names = _declared_symbols()
    assert len(names) >= 15
    for name in names:
        assert hasattr(L, name), name
    assert set(names) == set(_lib.SIGNATURES), "ctypes table out of sync with the header"


def test_geometry_helpers(L):
    hv = _lib.make_grid(33, 45, 80, 8, 8)
    assert L.da_num_regions(ctypes.byref(hv)) == 1980
    assert L.da_region_size(ctypes.byref(hv)) == 64
    assert L.da_padded_tokens(ctypes.byref(hv)) == 126720
    tiny = _lib.make_grid(4, 16, 16, 4, 4)
    assert L.da_num_regions(ctypes.byref(tiny)) == 64
    assert L.da_padded_tokens(ctypes.byref(tiny)) == 1024
    bad = _lib.make_grid(0, 4, 4, 2, 2)
    assert L.da_num_regions(ctypes.byref(bad)) == -1
    assert L.da_version() >= 100
    assert L.da_mask_capacity(1980, 392040) == 392040 + 1980


def test_workspace_sizes(L):
    hv = _lib.make_grid(33, 45, 80, 8, 8)
    ws = L.da_pipeline_workspace_size(ctypes.byref(hv), 24, 128)
    # pooled q, k (24 x 1980 x 128 f64 each) + scores (24 x 1980^2 f64) at least
    assert ws >= 8 * (2 * 24 * 1980 * 128 + 24 * 1980 * 1980)
    assert L.da_select_workspace_size(24, 1980) > 0
    assert L.da_select_workspace_size(0, 1980) == 0


def test_invalid_arguments_fail_before_any_launch(L):
    g = _lib.make_grid(2, 3, 5, 2, 4)
    rc = L.da_permute_in(None, 0, 8, None, 1, 8, ctypes.byref(g), None)
    assert rc == _lib.DA_EINVAL
    assert b"permute_in" in L.da_last_error()
    bad = _lib.make_grid(2, 0, 5, 2, 4)
    rc = L.da_pool(ctypes.c_void_p(16), 0, 8, ctypes.c_void_p(16), 1, 8, ctypes.byref(bad), 0, None)
    assert rc == _lib.DA_EINVAL and b"positive" in L.da_last_error()
    rc = L.da_pool(ctypes.c_void_p(16), 0, 8, ctypes.c_void_p(16), 1, 8, ctypes.byref(g), 1, None)
    assert rc == _lib.DA_EINVAL and b"average pooling only" in L.da_last_error()
    rc = L.da_select(None, 1, 4, 3, 0, None, None, None, None, None, None, None, None, None)
    assert rc == _lib.DA_EINVAL
    args = _lib.DaAttnArgs()
    rc = L.da_block_sparse_fwd(ctypes.byref(args), ctypes.byref(g), None)
    assert rc == _lib.DA_EINVAL and b"null" in L.da_last_error()


def test_check_maps_status_to_python_errors(L):
    g = _lib.make_grid(2, 0, 5, 2, 4)
    rc = L.da_pool(ctypes.c_void_p(16), 0, 8, ctypes.c_void_p(16), 1, 8, ctypes.byref(g), 0, None)
    with pytest.raises(ValueError, match="positive"):
        _lib.check(rc, "pool")
