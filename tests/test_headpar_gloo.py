"""Host-side logic of the multi-GPU path, world_size 2 and 3 over gloo (CPU):
the sequence <-> head resharding, the pipelined head-group schedule with
asynchronous all-to-alls, and the head-ordered cross-rank fold behind the
shared-head mask."""

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


def _init(rank, world, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


def _reshard_worker(rank, world, port, results):
    _init(rank, world, port)
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
    mp.spawn(_reshard_worker, args=(world, _free_port(), results), nprocs=world, join=True)
    assert dict(results) == {0: True, 1: True}


def _pipelined_worker(rank, world, port, groups, results):
    # HeadParallelAttention's schedule with a stand-in per-head compute
    # (out = 2 v + row-sum of q, per head: any function of all of a head's rows
    # would show a resharding error); the pipeline itself needs a GPU
    _init(rank, world, port)
    try:
        from paper_2505_14708_b200 import api
        from paper_2505_14708_b200.headpar import HeadParallelAttention

        n, heads, d = 24, 6 * world, 8
        g = torch.Generator().manual_seed(0)
        full = [torch.randn(n, heads, d, generator=g).to(torch.bfloat16) for _ in range(3)]
        nl = n // world

        def compute(qh, kh, vh, out):  # (n, hg, d) views
            out.copy_((2 * vh.float() + qh.float().sum(0, keepdim=True) + kh.float().mean(0, keepdim=True)).to(torch.bfloat16))
            return None

        plan = api.pad_plan(1, 1, n, 1, 1)
        hp = HeadParallelAttention(plan, 0.5, world, rank, head_groups=groups, compute=compute)
        out, _ = hp(*(x[rank * nl:(rank + 1) * nl].contiguous() for x in full))
        want = torch.empty(n, heads, d, dtype=torch.bfloat16)
        for h in range(heads):
            compute(full[0][:, h:h + 1], full[1][:, h:h + 1], full[2][:, h:h + 1], want[:, h:h + 1])
        results[rank] = bool(torch.equal(out, want[rank * nl:(rank + 1) * nl]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,groups", [(2, 1), (2, 3), (3, 2), (2, 6)])
def test_pipelined_head_groups_world(world, groups):
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_pipelined_worker, args=(world, _free_port(), groups, results), nprocs=world, join=True)
    assert dict(results) == {r: True for r in range(world)}


def _fold_worker(rank, world, port, results):
    _init(rank, world, port)
    try:
        from paper_2505_14708_b200.headpar import ordered_head_sum

        heads = 4 * world
        g = torch.Generator().manual_seed(1)
        # wide dynamic range so that the summation order changes the rounding
        bases = torch.randn(heads, 16, 16, generator=g, dtype=torch.float64) * \
            torch.logspace(-12, 12, heads, dtype=torch.float64)[torch.randperm(heads, generator=g)][:, None, None]
        hl = heads // world
        total = ordered_head_sum(bases[rank * hl:(rank + 1) * hl].clone(), rank, world)
        if rank == world - 1:
            ref = bases[0].clone()
            for h in range(1, heads):
                ref = ref + bases[h]  # sparse.py:296 left fold
            rev = bases[-1].clone()
            for h in range(heads - 2, -1, -1):
                rev = rev + bases[h]  # another order rounds differently on these inputs
            results[rank] = bool(torch.equal(total, ref)) and not bool(torch.equal(ref, rev))
        else:
            results[rank] = total is None
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_ordered_head_sum_is_the_reference_left_fold(world):
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_fold_worker, args=(world, _free_port(), results), nprocs=world, join=True)
    assert dict(results) == {r: True for r in range(world)}


def test_head_groups_split():
    from paper_2505_14708_b200.headpar import head_groups

    assert head_groups(3, 2) == [(0, 2), (2, 3)]
    assert head_groups(12, 1) == [(0, 12)]
    assert head_groups(2, 8) == [(0, 1), (1, 2)]
    for hl in range(1, 20):
        for G in range(1, 6):
            gs = head_groups(hl, G)
            assert gs[0][0] == 0 and gs[-1][1] == hl and all(a[1] == b[0] for a, b in zip(gs, gs[1:]))


class _FakeLib:
    """Stands in for the C library in the PeerShards set-up: export / open
    succeed or fail per rank (no GPU needed for the agreement logic)."""

    def __init__(self, fail_export, fail_open):
        self.fail_export, self.fail_open, self.closed = fail_export, fail_open, []

    def da_ipc_export(self, ptr, handle, offset):
        if self.fail_export:
            return 2
        handle.raw = bytes([dist.get_rank() + 1]) * 64
        return 0

    def da_ipc_open(self, handle, offset, out):
        if self.fail_open:
            return 2
        out._obj.value = 4096 * (1 + handle[0] if isinstance(handle, bytes) else 1)
        return 0

    def da_ipc_close(self, ptr, offset):
        self.closed.append(ptr)
        return 0

    def da_last_error(self):
        return b"simulated failure"


def _peer_setup_worker(rank, world, port, fail_export_rank, fail_open_rank, results):
    # one rank's export or mapping fails: every rank must raise, none may be
    # left waiting in a collective (the next collective below would hang)
    _init(rank, world, port)
    try:
        from paper_2505_14708_b200 import _lib
        from paper_2505_14708_b200.headpar import PeerShards

        fake = _FakeLib(rank == fail_export_rank, rank == fail_open_rank)
        _lib.lib = lambda: fake
        raised = False
        try:
            PeerShards(4, 2, 8, 8, world, rank, device="cpu")
        except (RuntimeError, ValueError):
            raised = True
        flag = torch.tensor([1])
        dist.all_reduce(flag)  # every rank reaches the next collective
        results[rank] = (raised, int(flag.item()), len(fake.closed))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("fail_export_rank,fail_open_rank", [(1, -1), (-1, 1), (-1, -1)])
def test_peer_shard_setup_failures_are_collective(fail_export_rank, fail_open_rank):
    world = 2
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_peer_setup_worker, args=(world, _free_port(), fail_export_rank, fail_open_rank, results),
             nprocs=world, join=True)
    res = dict(results)
    expect_raise = fail_export_rank >= 0 or fail_open_rank >= 0
    assert all(res[r][0] == expect_raise for r in range(world)), res
    assert all(res[r][1] == world for r in range(world))
    if fail_open_rank >= 0:  # the rank whose mapping succeeded unmapped it again
        assert res[1 - fail_open_rank][2] == 1
