"""Head-parallel execution across GPUs (one process per GPU).

The reference runs heads one after another (sparse.py:273-279); heads are
independent (per-head masks by default), so P ranks each own heads/P heads.
A sequence-parallel caller holds n/P tokens of every head; all-to-alls
reshard Q/K/V to "all tokens of my heads" before the pipeline and reshard the
output back (Ulysses-style).

The local heads are processed in head GROUPS so the collectives overlap the
compute: the input all-to-alls of group g+1 are in flight while group g runs
its pipeline, and group g's output all-to-all runs while group g+1 computes.
The collectives are asynchronous NCCL calls (their stream waits for the
packing copies; the compute stream waits for their completion only where it
needs the data).

Layouts (no copies beyond the one pack per input tensor and the one unpack of
the output):
  * send buffer of a group: [dest rank][my rows][its heads of the group][d]
    (one strided copy of the caller's (n/P, H, d) shard);
  * receive buffer: [src rank][its rows][my heads of the group][d], which IS
    the (n, heads_of_group, d) "nhd" layout the pipeline reads in place;
  * the pipeline writes (n, heads_of_group, dv), whose per-destination row
    blocks are contiguous: it is the output all-to-all's send buffer as is.

With ``transport="peer"`` there are no all-to-alls at all: every rank keeps
its (n/P, H, d) shards in buffers the other ranks map (CUDA IPC,
``PeerShards``), and the kernels of rank r read all ranks' rows of r's heads
and write r's output rows into their owners' buffers over NVLink (the
sharded C-ABI path, ``api.ShardTable``). Two stream-ordered barriers per
call (a one-element all-reduce) order the writers and readers.

``shared_head_mask`` (sparse.py:281-297) needs the mean of every head's
selection basis before any head can attend. The ranks fold the per-head fp64
bases in global head order, as the reference's ``basis_sum + basis`` loop does
(rank r continues the running sum it receives from rank r-1 with its own heads
and passes it on), so the mean, and therefore the mask, is bit-identical to
the single-process result; the last rank broadcasts the mean.
"""

from __future__ import annotations

import torch
import torch.distributed as dist

from . import api


def seq_to_head(x: torch.Tensor, world: int, group=None) -> torch.Tensor:
    """(n/P, H, d) sequence shard -> (n, H/P, d) head shard (one blocking all-to-all)."""
    nl, heads, d = x.shape
    hl = heads // world
    send = x.reshape(nl, world, hl, d).permute(1, 0, 2, 3).contiguous()  # [dest rank][rows][my heads]
    recv = torch.empty_like(send)                                          # [src rank][its rows][my heads]
    dist.all_to_all_single(recv, send, group=group)
    return recv.reshape(world * nl, hl, d)


def head_to_seq(o: torch.Tensor, world: int, group=None) -> torch.Tensor:
    """(n, H/P, d) head shard -> (n/P, H, d) sequence shard (one blocking all-to-all)."""
    n, hl, d = o.shape
    nl = n // world
    send = o.reshape(world, nl, hl, d).contiguous()                        # [dest rank][its rows][my heads]
    recv = torch.empty_like(send)                                          # [src rank = head group][my rows]
    dist.all_to_all_single(recv, send, group=group)
    return recv.permute(1, 0, 2, 3).reshape(nl, world * hl, d)


def head_groups(local_heads: int, groups: int):
    """Contiguous [h0, h1) ranges splitting a rank's heads into ``groups`` groups."""
    groups = max(1, min(groups, local_heads))
    base, extra = divmod(local_heads, groups)
    out, h0 = [], 0
    for gi in range(groups):
        h1 = h0 + base + (1 if gi < extra else 0)
        out.append((h0, h1))
        h0 = h1
    return out


def ordered_head_sum(bases: torch.Tensor, rank: int, world: int, group=None) -> torch.Tensor | None:
    """Sum of every rank's per-head bases in global head order, left fold
    ((b_0 + b_1) + b_2) + ... (sparse.py:296), across ranks: rank r receives
    the running sum of ranks < r, adds its own heads in order and sends it on.
    Returns the total on the LAST rank, None elsewhere. ``bases``: this rank's
    (heads, ...) float64 bases, its heads being the next ones in global order."""
    acc = None
    if rank > 0:
        acc = torch.empty_like(bases[0])
        dist.recv(acc, src=_global(rank - 1, group), group=group)
    for h in range(bases.shape[0]):
        acc = bases[h].clone() if acc is None else acc + bases[h]
    if rank < world - 1:
        dist.send(acc, dst=_global(rank + 1, group), group=group)
        return None
    return acc


def _record(events):
    """Start a (begin, end) CUDA event pair on the current stream, or None."""
    if events is None:
        return None
    pair = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
    pair[0].record()
    events.append(pair)
    return pair


def _close(pair):
    if pair is not None:
        pair[1].record()


def _global(rank: int, group) -> int:
    return rank if group is None else dist.get_global_rank(group, rank)


class PeerShards:
    """This rank's sequence-shard buffers (q, k, v: (n/P, H, d); out:
    (n/P, H, dv), bf16, one allocation) and the same buffers of every rank of
    ``group`` mapped into this process through CUDA IPC (``da_ipc_export`` /
    ``da_ipc_open``; peer access over NVLink between GPUs). A collective:
    every rank constructs it with the same shape. ``close()`` (also a
    collective) unmaps the peers' buffers."""

    def __init__(self, rows: int, heads: int, d: int, dv: int, world: int, rank: int, group=None, device=None):
        import contextlib
        import ctypes

        from ._lib import IPC_HANDLE_BYTES, check, lib

        self.rows, self.heads, self.d, self.dv, self.world, self.rank, self.group = rows, heads, d, dv, world, rank, group
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.sizes = [rows * heads * d, rows * heads * d, rows * heads * dv, rows * heads * dv]
        # one allocation, each buffer 256-byte aligned
        self.offsets, off = [], 0
        for n in self.sizes:
            self.offsets.append(off)
            off += -(-n * 2 // 256) * 256
        # a local failure (allocation, export) must not skip the collective
        # below, or the other ranks would wait in it: it is raised after it
        failure, mine = None, None
        try:
            self.arena = torch.empty(off, dtype=torch.uint8, device=dev)
            handle = ctypes.create_string_buffer(IPC_HANDLE_BYTES)
            offset = ctypes.c_int64()
            check(lib().da_ipc_export(self.arena.data_ptr(), handle, ctypes.byref(offset)), "ipc_export")
            mine = (bytes(handle.raw), int(offset.value))
        except Exception as e:  # noqa: BLE001
            failure = e
        everyone = [None] * world
        dist.all_gather_object(everyone, mine, group=group)
        if failure is not None:
            raise failure
        if any(x is None for x in everyone):
            raise RuntimeError("a peer rank could not allocate or export its shard buffers")
        views = [self.arena[o:o + n * 2].view(torch.bfloat16) for o, n in zip(self.offsets, self.sizes)]
        self.q = views[0].view(rows, heads, d)
        self.k = views[1].view(rows, heads, d)
        self.v = views[2].view(rows, heads, dv)
        self.out = views[3].view(rows, heads, dv)
        self._opened = []   # (base pointer, 0) of every mapping this process made
        self.bases = []     # arena address of each rank, in this process
        mapped = {}
        try:
            for r, (h, o) in enumerate(everyone):
                if r == rank:
                    self.bases.append(self.arena.data_ptr())
                    continue
                if h not in mapped:
                    ptr = ctypes.c_void_p()
                    with (torch.cuda.device(dev) if dev.type == "cuda" else contextlib.nullcontext()):
                        check(lib().da_ipc_open(h, 0, ctypes.byref(ptr)), "ipc_open")
                    mapped[h] = ptr.value
                    self._opened.append(ptr.value)
                self.bases.append(mapped[h] + o)
        except Exception as e:  # noqa: BLE001
            failure = e
        # every rank learns whether every rank mapped every peer, and all raise together
        oks = [None] * world
        dist.all_gather_object(oks, failure is None, group=group)
        if not all(oks):
            for base in self._opened:
                lib().da_ipc_close(base, 0)
            self._opened = []
            raise failure if failure is not None else RuntimeError("a peer rank could not map the shard buffers")
        self._flag = torch.zeros(1, dtype=torch.float32, device=dev)

    def table(self, h0: int, h1: int):
        """api.ShardTable of heads [h0, h1) of every rank's shards."""
        from .api import ShardTable

        hd = self.heads
        ptr = lambda t, h, last: tuple(b + self.offsets[t] + h * last * 2 for b in self.bases)
        return ShardTable(ptr(0, h0, self.d), ptr(1, h0, self.d), ptr(2, h0, self.dv), ptr(3, h0, self.dv),
                          self.rows, self.rows * self.world, h1 - h0, self.d, self.dv,
                          (self.d, hd * self.d, self.d, hd * self.d, self.dv, hd * self.dv, self.dv, hd * self.dv))

    def barrier(self):
        """Every rank's prior device work on its current stream is complete
        (and its writes visible) before any rank's next device work: a
        one-element all-reduce with NCCL (stream-ordered), else a host
        barrier after a device synchronise (gloo, tests)."""
        if dist.get_backend(self.group) == "nccl":
            dist.all_reduce(self._flag, group=self.group)
        else:
            torch.cuda.synchronize()
            dist.barrier(group=self.group)

    def close(self):
        from ._lib import check, lib

        if self.arena is None:
            return
        self.barrier()  # nobody reads or writes the mappings any more
        for base in self._opened:
            check(lib().da_ipc_close(base, 0), "ipc_close")
        self._opened = []
        torch.cuda.synchronize()
        dist.barrier(group=self.group)  # every peer unmapped this rank's arena before it is freed
        self.arena = None


class HeadParallelAttention:
    """padded_sparse_attention over a sequence-sharded (n/P, H, d) input.

    ``head_groups``: how many groups the rank's heads are split into for the
    communication / compute overlap (1 = no overlap). ``compute`` (tests):
    replaces the pipeline, called as compute(q, k, v, out) on (n, hg, d) "nhd"
    views and a (n, hg, dv) output buffer; returns a mask or None.
    """

    def __init__(self, plan: api.PadPlan, sparsity: float, world: int, rank: int, group=None,
                 scale=None, pool_mode="average", select_on="logits", force_row_keep=True,
                 shared_head_mask=False, head_groups=2, compute=None, transport="nccl"):
        if transport not in ("nccl", "peer"):
            raise ValueError(f"transport must be 'nccl' or 'peer', got {transport!r}")
        self.plan, self.sparsity, self.world, self.rank, self.group = plan, sparsity, world, rank, group
        self.scale, self.pool_mode, self.select_on, self.force = scale, pool_mode, select_on, force_row_keep
        self.shared = shared_head_mask
        self.groups = head_groups
        self.compute = compute
        # the shared-head mask needs every head's basis before any selection:
        # it keeps the all-to-all schedule (_call_shared) under either transport
        self.transport = transport
        self._peer = None

    def peer_buffers(self, rows: int, heads: int, d: int, dv: int) -> PeerShards:
        """The transport="peer" buffers for (rows, heads, d) shards (made on
        first use; a collective). A caller that writes its shards straight into
        ``.q`` / ``.k`` / ``.v`` saves the copy-in."""
        p = self._peer
        if p is None or (p.rows, p.heads, p.d, p.dv) != (rows, heads, d, dv):
            if p is not None:
                p.close()
            self._peer = PeerShards(rows, heads, d, dv, self.world, self.rank, self.group)
        return self._peer

    def close(self):
        if self._peer is not None:
            self._peer.close()
            self._peer = None

    # ------------------------------------------------------------ collectives
    def _pack(self, x, h0, h1):
        nl, heads, d = x.shape
        hl = heads // self.world
        return x.reshape(nl, self.world, hl, d)[:, :, h0:h1, :].permute(1, 0, 2, 3).contiguous()

    def _a2a(self, recv, send):
        return dist.all_to_all_single(recv, send, group=self.group, async_op=True)

    def _issue_inputs(self, q, k, v, h0, h1):
        bufs, works = [], []
        for x in (q, k, v):
            send = self._pack(x, h0, h1)                      # [dest][nl][hg][d]
            recv = torch.empty_like(send)                     # [src][nl][hg][d] == (n, hg, d)
            works.append(self._a2a(recv, send))
            bufs.append(recv)
        return bufs, works

    # ------------------------------------------------------------ call
    def __call__(self, q, k, v, compute_events=None, k4_events=None, mask=None):
        """q, k, v: this rank's (n/P, H, d) sequence shards. Returns the
        (n/P, H, dv) output shard and this rank's mask(s). ``mask``: a mask
        this rank returned before (its H/P heads, or one shared mask) to run
        the executor alone (mask caching across denoising steps: no pooling or
        selection). ``compute_events``
        (timing): a list that receives one (begin, end) CUDA event pair per
        compute phase on the current stream; the collectives run on NCCL's
        stream, so call time minus compute time is the exposed communication.
        ``k4_events``: likewise, one pair around each group's attention kernel."""
        nl, heads, d = q.shape
        dv = v.shape[2]
        if heads % self.world or k.shape != q.shape or v.shape[:2] != q.shape[:2]:
            raise ValueError("q, k, v must be (n/P, H, d) shards with H divisible by the world size")
        hl = heads // self.world
        n = nl * self.world
        scale = self.scale if self.scale is not None else api.head_dim_scale(d)
        groups = head_groups(hl, self.groups)
        if mask is not None and mask.heads not in (1, hl):
            raise ValueError(f"mask of {mask.heads} heads does not fit this rank's {hl} heads")
        if self.transport == "peer" and (not self.shared or mask is not None) and self.compute is None:
            return self._call_peer(q, k, v, scale, compute_events, k4_events, mask)
        out = torch.empty((nl, heads, dv), dtype=torch.bfloat16, device=q.device)
        if self.shared and mask is None:
            return self._call_shared(q, k, v, out, groups, scale, compute_events)

        inflight = {0: self._issue_inputs(q, k, v, *groups[0])}
        outs, masks = [], []
        for gi, (h0, h1) in enumerate(groups):
            if gi + 1 < len(groups):  # next group's inputs travel while this group computes
                inflight[gi + 1] = self._issue_inputs(q, k, v, *groups[gi + 1])
            (qh, kh, vh), works = inflight.pop(gi)
            for w in works:
                w.wait()
            hg = h1 - h0
            res = torch.empty((n, hg, dv), dtype=torch.bfloat16, device=q.device)
            ev = _record(compute_events)
            if mask is not None:  # cached mask: the executor alone
                api._attend(qh.view(n, hg, d), kh.view(n, hg, d), vh.view(n, hg, dv), self.plan,
                            mask.head_range(h0, h1), scale, qkv_layout="nhd", out_dev=res)
                masks.append(mask.head_range(h0, h1) if mask.heads > 1 else None)
            else:
                masks.append(self._compute(qh.view(n, hg, d), kh.view(n, hg, d), vh.view(n, hg, dv), res, scale,
                                           k4_events))
            _close(ev)
            recv = torch.empty((self.world, nl, hg, dv), dtype=torch.bfloat16, device=q.device)
            outs.append((h0, h1, recv, self._a2a(recv, res.view(self.world, nl, hg, dv))))
        for h0, h1, recv, work in outs:
            work.wait()
            out.view(nl, self.world, hl, dv)[:, :, h0:h1, :].copy_(recv.permute(1, 0, 2, 3))
        if mask is not None:
            return out, mask
        masks = [m for m in masks if m is not None]
        return out, (api._cat_masks(masks) if masks else None)

    def _call_peer(self, q, k, v, scale, compute_events=None, k4_events=None, mask=None):
        """transport="peer": shards copied into the mapped buffers (unless the
        caller wrote them there), a barrier, ONE pipeline call over all of
        this rank's heads reading every rank's rows in place and writing the
        output rows into their owners' buffers, a barrier. The returned output
        shard is a copy (the buffers are reused by the next call)."""
        nl, heads, d = q.shape
        dv = v.shape[2]
        hl = heads // self.world
        pb = self.peer_buffers(nl, heads, d, dv)
        for src, dst in ((q, pb.q), (k, pb.k), (v, pb.v)):
            if src.data_ptr() != dst.data_ptr():
                dst.copy_(src)
        pb.barrier()                                  # every rank's shards are in place
        ev = _record(compute_events)
        k4 = None
        if k4_events is not None and mask is None:
            k4 = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            k4_events.append(k4)
        h0 = self.rank * hl
        mask = api._run_sharded(pb.table(h0, h0 + hl), self.plan, self.sparsity, scale, self.pool_mode,
                                self.select_on, self.force, False, q.device, attn_events=k4, mask=mask)
        _close(ev)
        pb.barrier()                                  # every rank's output rows have landed
        return pb.out.clone(), mask

    def _compute(self, qh, kh, vh, res, scale, k4_events=None):
        if self.compute is not None:
            return self.compute(qh, kh, vh, res)
        ev = None
        if k4_events is not None:
            ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            k4_events.append(ev)
        _, mask, _ = api._pipeline(qh, kh, vh, self.plan, self.sparsity, scale, self.pool_mode, self.select_on,
                                   self.force, False, "nhd", want_bitmap=False, out_dev=res, attn_events=ev)
        return mask

    def _call_shared(self, q, k, v, out, groups, scale, compute_events):
        """One mask for all heads of all ranks: inputs first, then the ordered
        cross-rank fold of the bases, the selection, and the attention."""
        nl, heads, d = q.shape
        dv = v.shape[2]
        hl = heads // self.world
        n = nl * self.world
        inputs = []
        for h0, h1 in groups:
            bufs, works = self._issue_inputs(q, k, v, h0, h1)
            for w in works:
                w.wait()
            hg = h1 - h0
            inputs.append((h0, h1, bufs[0].view(n, hg, d), bufs[1].view(n, hg, d), bufs[2].view(n, hg, dv)))
        ev = _record(compute_events)
        bases = []
        for _, _, qh, kh, _ in inputs:
            qp = api.pool_tokens(qh, self.plan, self.pool_mode, qkv_layout="nhd")
            kp = api.pool_tokens(kh, self.plan, self.pool_mode, qkv_layout="nhd")
            bases.append(api.draft_logits(qp, kp, scale, softmax=self.select_on == "softmax"))
        _close(ev)
        total = ordered_head_sum(torch.cat(bases, 0), self.rank, self.world, self.group)
        g = self.plan.layout.num_regions
        mean = total / heads if total is not None else torch.empty((g, g), dtype=torch.float64, device=q.device)
        dist.broadcast(mean, src=_global(self.world - 1, self.group), group=self.group)
        ev = _record(compute_events)
        mask = api.select_top_fraction(mean, 1.0 - self.sparsity, self.force)
        outs = []
        for h0, h1, qh, kh, vh in inputs:
            hg = h1 - h0
            res = torch.empty((n, hg, dv), dtype=torch.bfloat16, device=q.device)
            api._attend(qh, kh, vh, self.plan, mask, scale, qkv_layout="nhd", out_dev=res)
            recv = torch.empty((self.world, nl, hg, dv), dtype=torch.bfloat16, device=q.device)
            outs.append((h0, h1, recv, self._a2a(recv, res.view(self.world, nl, hg, dv))))
        _close(ev)
        for h0, h1, recv, work in outs:
            work.wait()
            out.view(nl, self.world, hl, dv)[:, :, h0:h1, :].copy_(recv.permute(1, 0, 2, 3))
        return out, mask
