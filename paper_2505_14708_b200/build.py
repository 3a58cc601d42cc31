"""Compile the sm_100a shared library in-tree (nvcc; no JIT cache).

    python -m paper_2505_14708_b200.build [--force]
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
OUT = PKG / "libdraftattn_b200.so"
SOURCES = ["api.cu", "prep.cu", "select.cu", "attn_portable.cu", "attn_lh.cu"]
# the transposed TMEM-fed K4 (attn_tk.cu) is an experiment: only builds with
# -DDA_K4_TK link it (tools/probes/k4_variants.py); the shipped library does not
EXPERIMENT_SOURCES = {"-DDA_K4_TK": ["attn_tk.cu"]}
HEADERS = ["common.cuh", "kernels.h", "attn_k4.cuh"]
ARCH = "-gencode=arch=compute_100a,code=sm_100a"


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (Path(cand).exists() or cand == "nvcc"):
            return cand
    return "nvcc"


def _stale() -> bool:
    if not OUT.exists():
        return True
    t = OUT.stat().st_mtime
    deps = [CSRC / s for s in SOURCES + HEADERS] + [PKG.parent / "include" / "draftattn_b200.h"]
    return any(p.stat().st_mtime > t for p in deps)


def build(force: bool = False, verbose: bool = False, out: Path | None = None, flags=()) -> Path:
    """Build libdraftattn_b200.so for sm_100a unless it is up to date.
    ``out`` / ``flags``: experiment builds (tools/probes) into another path
    with extra -D options; the shipped library takes neither."""
    target = Path(out) if out is not None else OUT
    if out is None and not force and not _stale():
        return OUT
    extra = os.environ.get("DA_NVCC_FLAGS", "").split() + list(flags)  # experiments only
    sources = list(SOURCES)
    for flag, more in EXPERIMENT_SOURCES.items():
        if flag in extra:
            sources += more
    cmd = [nvcc(), ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC",
           "-o", str(target)] + extra + [str(CSRC / s) for s in sources]
    if verbose:
        print(" ".join(cmd), flush=True)
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"nvcc failed ({res.returncode})")
    return target


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(OUT)
