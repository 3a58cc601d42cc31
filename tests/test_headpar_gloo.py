"""Sequence <-> head resharding of the multi-GPU path, world_size 2 over gloo (CPU)."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2505_14708_b200.headpar import head_to_seq, seq_to_head

        n, heads, d = 12, 4, 8
        full = torch.arange(n * heads * d, dtype=torch.float32).reshape(n, heads, d)
        nl, hl = n // world, heads // world
        local = full[rank * nl:(rank + 1) * nl].clone()
        mine = seq_to_head(local, world)
        ok1 = torch.equal(mine, full[:, rank * hl:(rank + 1) * hl])
        back = head_to_seq(mine * 2, world)
        ok2 = torch.equal(back, local * 2)
        results[rank] = bool(ok1 and ok2)
    finally:
        dist.destroy_process_group()


def test_seq_head_resharding_world2():
    world = 2
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), results), nprocs=world, join=True)
    assert dict(results) == {0: True, 1: True}
