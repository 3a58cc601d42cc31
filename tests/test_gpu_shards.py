"""Sequence shards: the C-ABI pipeline and executor reading Q/K/V rows from,
and writing output rows into, separate row-block buffers give results
bit-identical to the unsplit call. On one GPU the shards are local buffers;
the head-parallel "peer" transport hands the same kernels other ranks' buffers
(CUDA IPC), exercised here by two processes sharing the test box's GPU."""

import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest
import torch

import paper_2505_14708_b200 as da
from paper_2505_14708_b200 import api

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def _split(x, rows):
    return [x[i:i + rows].contiguous() for i in range(0, x.shape[0], rows)]


def _inputs(plan, heads, d, seed, qmul=1.0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    q, k, v = (torch.randn(plan.num_valid, heads, d, device="cuda", generator=g) for _ in range(3))
    return (q * qmul).to(torch.bfloat16), k.to(torch.bfloat16), v.to(torch.bfloat16)


def _assert_same_masks(m, ref, heads):
    assert m.heads == ref.heads
    for h in range(m.heads):
        assert m.head(h).bitmap_bytes() == ref.head(h).bitmap_bytes()
    assert torch.equal(m.kept_counts, ref.kept_counts) and torch.equal(m.thresholds, ref.thresholds)


# (grid, heads, d, rows per shard, sparsity, pool, select_on, shared, q scale)
CASES = [
    ((3, 45, 80, 8, 8), 4, 128, 5400, 0.9, "average", "logits", False, 1.0),     # 2 even shards, tcgen05
    ((3, 45, 80, 8, 8), 4, 128, 4000, 0.9, "average", "logits", False, 1.0),     # ragged last shard
    ((3, 45, 80, 8, 8), 3, 128, 1351, 0.75, "average", "logits", False, 1.0),    # 8 shards (one NVLink node)
    ((3, 45, 80, 8, 8), 4, 128, 3600, 0.85, "average", "softmax", False, 1.0),
    ((3, 45, 80, 8, 8), 4, 128, 3600, 0.85, "average", "logits", True, 1.0),     # shared head mask
    ((2, 16, 24, 8, 8), 2, 128, 300, 0.8, "max", "logits", False, 1.0),          # max pooling
    ((2, 12, 20, 4, 4), 3, 64, 170, 0.7, "average", "logits", False, 1.0),       # portable kernel (p = 16, d = 64)
    ((2, 16, 48, 8, 16), 2, 128, 600, 0.8, "average", "logits", False, 1.0),    # portable, 8x16 pool (key chunks)
    ((2, 45, 80, 8, 8), 2, 128, 2500, 0.9, "average", "logits", False, 40.0),    # K4 fallback rows (portable list)
    ((2, 20, 40, 8, 16), 2, 128, 500, 0.8, "average", "logits", False, 40.0),    # the same with 8x16 half-regions
    ((2, 20, 40, 8, 16), 3, 128, 700, 0.8, "average", "softmax", True, 1.0),     # 8x16, shared mask, softmax basis
]


@pytest.mark.parametrize("case", CASES)
def test_sharded_pipeline_equals_unsplit(case):
    dims, heads, d, rows, sp, pool, select_on, shared, qmul = case
    plan = da.pad_plan(*dims)
    q, k, v = _inputs(plan, heads, d, seed=sum(dims) + heads, qmul=qmul)
    ref, ref_mask, _ = api._pipeline(q, k, v, plan, sp, api.head_dim_scale(d), pool, select_on, True, shared, "nhd")
    outs, mask = da.sharded_sparse_attention(_split(q, rows), _split(k, rows), _split(v, rows), plan, sp,
                                             pool_mode=pool, select_on=select_on, shared_head_mask=shared,
                                             return_mask=True)
    assert len(outs) == -(-plan.num_valid // rows)
    assert torch.equal(torch.cat(outs), ref)
    _assert_same_masks(mask, ref_mask, heads)


@pytest.mark.parametrize("rows,shared", [(4000, False), (3600, True)])
def test_sharded_executor_with_cached_mask(rows, shared):
    plan = da.pad_plan(3, 45, 80, 8, 8)
    q, k, v = _inputs(plan, 4, 128, seed=11)
    res = da.multi_head_sparse_attention(q, k, v, plan, 0.9, shared_head_mask=shared, qkv_layout="nhd",
                                         return_details=True)
    ref = da.padded_block_sparse_attention(q, k, v, plan, res.mask, qkv_layout="nhd")
    outs = da.sharded_sparse_attention(_split(q, rows), _split(k, rows), _split(v, rows), plan, 0.9,
                                       mask=res.mask)
    assert torch.equal(torch.cat(outs), ref)
    assert torch.equal(ref, res.output)


def test_sharded_argument_errors():
    plan = da.pad_plan(2, 16, 24, 8, 8)
    q, k, v = _inputs(plan, 2, 128, seed=1)
    with pytest.raises(ValueError, match="shards"):
        da.sharded_sparse_attention([q], [k], [v], plan, 0.9)                       # one shard
    with pytest.raises(ValueError, match="rows"):
        da.sharded_sparse_attention([q[:300], q[300:400], q[400:]], [k[:300], k[300:400], k[400:]],
                                    [v[:300], v[300:400], v[400:]], plan, 0.9)      # short middle shard
    with pytest.raises(ValueError, match="layout has"):
        da.sharded_sparse_attention(_split(q[:700], 350), _split(k[:700], 350), _split(v[:700], 350), plan, 0.9)
    with pytest.raises(ValueError, match="strides"):
        qs = _split(q, 384)
        qs[1] = qs[1].transpose(0, 1).contiguous().transpose(0, 1)
        da.sharded_sparse_attention(qs, _split(k, 384), _split(v, 384), plan, 0.9)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("world", [2, 3, 4])
def test_peer_transport_two_processes_one_gpu(world, tmp_path):
    # world processes on the one GPU, gloo for the host-side exchange: every
    # rank maps the others' shard buffers through CUDA IPC and the kernels read
    # and write them in place; the output shards and masks must equal one
    # single-process call bit for bit (tests/_peer_worker.py)
    env = dict(os.environ, PYTHONPATH=str(ROOT), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", f"--master-port={env['MASTER_PORT']}",
           str(ROOT / "tests" / "_peer_worker.py"), str(tmp_path)]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    for rank in range(world):
        assert (tmp_path / f"ok{rank}").read_text() == "ok"


def test_bench_multi_rank_code_path_one_gpu():
    # bench.py's N > 1 path (peer transport, max-over-ranks timing, e2e through
    # the mapped buffers) with two ranks sharing the GPU: a code-path check of
    # the driver's scaling command, not a measurement
    import json

    env = dict(os.environ, DA_BENCH_SAME_GPU="1", PYTHONPATH=str(ROOT))
    port = str(_free_port())
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(ROOT / "bench.py"), "--gpus", "2",
           "--config", "tiny", "--steps", "3", "--warmup", "3", "--no-cpu", "--no-dense"]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600, cwd=str(ROOT))
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    line = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["transport"] == "peer" and line["value"] > 0
    assert line["e2e"]["value"] > 0 and "collective_exposed_ms" in line
