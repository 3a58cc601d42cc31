"""The C ABI from plain C: examples/c_abi_demo.c includes only
include/draftattn_b200.h and the CUDA runtime, links the in-tree library and
runs the whole call. CPU: it compiles as C99 against the header. GPU: its
output and kept counts equal the Python API's on the same inputs, bit for bit."""
import shutil
import subprocess
from pathlib import Path

import numpy as np
import pytest
import torch

ROOT = Path(__file__).resolve().parents[1]
LIBDIR = ROOT / "paper_2505_14708_b200"
CUDA = Path("/usr/local/cuda")


def _compile(out: Path) -> Path:
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    exe = out / "c_abi_demo"
    cmd = ["gcc", "-std=c99", "-O2", "-Wall", "-Werror", "-I", str(ROOT / "include"), "-I", str(CUDA / "include"),
           str(ROOT / "examples" / "c_abi_demo.c"), "-o", str(exe), "-L", str(LIBDIR), "-ldraftattn_b200",
           "-L", str(CUDA / "lib64"), "-lcudart", "-lm", f"-Wl,-rpath,{LIBDIR}", f"-Wl,-rpath,{CUDA / 'lib64'}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_c_demo_compiles_against_the_header(tmp_path):
    if not (LIBDIR / "libdraftattn_b200.so").exists():
        pytest.skip("library not built")
    assert _compile(tmp_path).exists()


@pytest.mark.gpu
@pytest.mark.parametrize("dims,heads,sp", [((3, 45, 80, 8, 8), 3, 0.9), ((2, 20, 72, 8, 16), 2, 0.8)])
def test_c_demo_equals_python_api(tmp_path, dims, heads, sp):
    import paper_2505_14708_b200 as da

    exe = _compile(tmp_path)
    plan = da.pad_plan(*dims)
    g = torch.Generator(device="cuda").manual_seed(7)
    q, k, v = (torch.randn(heads, plan.num_valid, 128, device="cuda", generator=g).to(torch.bfloat16)
               for _ in range(3))
    for name, x in (("q", q), ("k", k), ("v", v)):
        x.cpu().view(torch.int16).numpy().tofile(tmp_path / f"{name}.bin")
    r = subprocess.run([str(exe), *map(str, dims), str(heads), "128", str(sp), str(tmp_path)],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr + r.stdout
    res = da.multi_head_sparse_attention(q, k, v, plan, sp, return_details=True)
    out = np.fromfile(tmp_path / "out.bin", dtype=np.int16).reshape(heads, plan.num_valid, 128)
    assert np.array_equal(out, res.output.cpu().view(torch.int16).numpy())
    kept = np.fromfile(tmp_path / "kept.bin", dtype=np.int64)
    assert kept.tolist() == res.mask.kept_counts.cpu().tolist()
