"""Benchmark of the DraftAttention sparse-attention call on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config hv720|wan720|tiny]
                    [--sparsity S] [--impl ours|reference]

One step = one attention call over all heads of the configuration (pool ->
draft scores -> global top-fraction selection -> block-sparse attention, output
in original token order). N = 1: inputs resident in HBM (value); the same call
through the public API with pinned-host inputs and a host copy of the output
(e2e). N > 1: inputs arrive sequence-sharded and each rank runs its heads
(strong scaling: the call's total work is fixed). --transport peer (default):
the kernels read every rank's shard rows in place over NVLink (CUDA IPC) and
write the output rows into their owners' shards, no all-to-all; it is checked
bit-exact against the nccl transport on the first call and falls back to it
on any failure. --transport nccl: NCCL all-to-alls reshard to head-sharded and
back, overlapped with the compute by head groups. Inputs (2.2 GB for HV720) are larger than L2, so
no L2 flush is needed between steps.

The line also carries dense attention at the same shape (cuDNN / flash SDPA,
bf16, the north-star comparator) as ``dense_sdpa_ms`` and
``speedup_vs_dense_sdpa`` (skip with --no-dense).

--impl reference times the UNMODIFIED reference (``draftattn`` installed into
baseline/_ref with ``pip install --no-index --no-deps --target baseline/_ref``,
git-ignored, travels to the GPU box with the snapshot) through its public
``padded_sparse_attention`` on the host cores: whole heads of the same call,
float32 inputs (the reference's default precision) holding the bf16-rounded
values the GPU gets, heads one after another as the reference runs them; ms per
call = the per-head time x heads (labelled extrapolated). Without baseline/_ref
it times the oracle port of the same algorithm (oracle/, kind "port").
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    # name: frames, height, width, patch_h, patch_w, heads, head_dim, sparsity
    "hv720": (33, 45, 80, 8, 8, 24, 128, 0.9),
    "wan720": (21, 45, 80, 8, 8, 40, 128, 0.75),
    "tiny": (4, 16, 16, 4, 4, 2, 64, 0.5),
    # the paper's 8x16 pools (p = 128) on the HV720 grid (the reference's default patch)
    "hv720_8x16": (33, 45, 80, 8, 16, 24, 128, 0.9),
}
METRIC = "ms/attn call at HunyuanVideo 720p, 90% sparse; effective TFLOP/s per B200"


def _peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:  # noqa: BLE001
        return {}


def _profile_traffic(config_name):
    """DRAM bytes per K4 launch from the committed ncu --set full summary, if any."""
    p = ROOT / "profiles" / "ncu_k4_summary.json"
    try:
        data = json.loads(p.read_text())
        return data.get(config_name, {}).get("dram_bytes_per_launch")
    except Exception:  # noqa: BLE001
        return None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region.

    The sampler process starts before the warm-up (``start()``) so it is
    already emitting samples when the timed region opens; ``begin()`` /
    ``end()`` mark the region in wall time and only samples stamped inside it
    count (if the region is shorter than the 100 ms cadence, the first sample
    after it opened stands in, flagged ``nearest``)."""

    FIELDS = ("timestamp,clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.result = None
        self.t0 = self.t1 = None

    def start(self):
        """Start sampling and wait (up to 5 s) for the first sample, so that
        nvidia-smi's own start-up (which can stall the GPU's host thread for
        milliseconds) is over before any timed work."""
        import select

        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            ready, _, _ = select.select([self.proc.stdout], [], [], 5.0)
            if ready:
                self.proc.stdout.readline()
            time.sleep(0.3)  # a few more samples: past the start-up
        except Exception:  # noqa: BLE001
            self.proc = None
        return self

    def begin(self):
        self.t0 = time.time()

    def end(self):
        self.t1 = time.time()
        time.sleep(0.25)  # let the sample after the region arrive
        self._collect()

    def _collect(self):
        import datetime

        self.result = None
        if self.proc is None:
            return
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:  # noqa: BLE001
            self.proc.kill()
            out = ""
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        samples = []
        for line in out.strip().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) != 7:
                continue
            try:
                ts = datetime.datetime.strptime(parts[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                samples.append((ts, float(parts[1]), float(parts[2]),
                                {n for n, v in zip(names, parts[3:]) if v.lower().startswith("active")}))
            except ValueError:
                continue
        inside = [x for x in samples if self.t0 is not None and self.t0 <= x[0] <= self.t1]
        nearest = False
        if not inside:
            after = [x for x in samples if self.t0 is not None and x[0] >= self.t0]
            inside, nearest = after[:1], True
        if inside:
            self.result = {"sm_mhz": statistics.median(x[1] for x in inside), "sm_max_mhz": max(x[2] for x in inside),
                           "reasons": sorted(set().union(*(x[3] for x in inside))), "samples": len(inside)}
            if nearest:
                self.result["nearest"] = True


# --------------------------------------------------------------------------
# CPU reference arm / baseline (oracle port of the reference algorithm)
# --------------------------------------------------------------------------

def _reference_impl():
    """padded_sparse_attention of the unmodified reference from baseline/_ref,
    or None (then the oracle port stands in)."""
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "draftattn" / "padding.py").exists():
        return None
    if str(ref) not in sys.path:
        sys.path.insert(0, str(ref))
    try:
        from draftattn.padding import padded_sparse_attention
    except Exception:  # noqa: BLE001
        return None
    return padded_sparse_attention


def cpu_reference_sample(cfg, seed=0, head_ids=(0, 1), use_reference=True):
    """Time the reference path on whole heads of the call:
    padded_sparse_attention per head (padding.py:95-165), heads sequential,
    float32 inputs holding the bf16-rounded values. The unmodified reference
    (baseline/_ref) when installed, else the oracle port. Returns (ms per call
    extrapolated to every head, sample description, BLAS threads, kind)."""
    import torch
    from oracle import draftattn_oracle as O

    f, h, w, ph, pw, heads, d, sp = cfg
    fn = _reference_impl() if use_reference else None
    kind = "reference" if fn is not None else "port"
    if fn is None:
        fn = O.padded_sparse_attention
    grid = O.Grid(f, h, w, ph, pw)
    q, k, v = O.gen_real_inputs(grid, d, seed, heads, head_ids=list(head_ids))
    rnd = lambda x: torch.from_numpy(x).to(torch.bfloat16).to(torch.float32).numpy()  # noqa: E731
    q, k, v = rnd(q), rnd(k), rnd(v)
    times = []
    for slot in range(len(head_ids)):
        t0 = time.perf_counter()
        fn(q[slot], k[slot], v[slot], f, h, w, ph, pw, sp)
        times.append(time.perf_counter() - t0)
    per_head = statistics.mean(times)
    threads = _blas_threads()
    what = ("unmodified reference draftattn.padded_sparse_attention (baseline/_ref)" if kind == "reference"
            else "oracle port of the reference algorithm")
    sample = (f"{len(head_ids)} of {heads} heads in full ({', '.join(f'{t:.2f}' for t in times)} s), float32 numpy, "
              f"{what}, BLAS threads={threads}, {os.cpu_count()} host cores; ms/call = mean per head x "
              f"{heads} heads (extrapolated)")
    return per_head * heads * 1e3, sample, threads, kind


def _blas_threads():
    try:
        from threadpoolctl import threadpool_info
        n = [i.get("num_threads") for i in threadpool_info() if i.get("user_api") == "blas"]
        return int(n[0]) if n else (os.cpu_count() or 1)
    except Exception:  # noqa: BLE001
        return os.cpu_count() or 1


def run_reference(args, cfg, name):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    vals, threads, kind = [], 1, "port"
    for _ in range(args.warmup_ref):
        cpu_reference_sample(CONFIGS["tiny"], head_ids=(0,))
    heads = cfg[5]
    for s in range(args.steps):  # one whole head per step, a different head each step
        ms, _, threads, kind = cpu_reference_sample(cfg, head_ids=(s % heads,))
        vals.append(ms)
    ms = statistics.median(vals)
    what = ("unmodified reference draftattn.padded_sparse_attention (baseline/_ref)" if kind == "reference"
            else "oracle port of the reference algorithm")
    sample = (f"one whole head per step (heads 0..{args.steps - 1}), float32 numpy, {what}, "
              f"BLAS threads={threads}, {os.cpu_count()} host cores; ms/call = per-head median x {heads} heads "
              f"(extrapolated)")
    line = {
        "impl": "reference", "metric": METRIC, "value": ms, "unit": "ms/call", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic (synth.py gaussian, seeded)",
        "config": _config_dict(name, cfg, args.gpus),
        "cpu_baseline": {"value": ms, "unit": "ms/call", "cores": threads, "kind": kind, "sample": sample},
        "e2e": {"value": ms, "unit": "ms/call", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        # each step times ONE head of the call; value = that x heads
        "extrapolated": {"timed_s_per_step": [v / heads / 1e3 for v in vals], "factor": heads,
                         "what": "whole heads timed, call = per-head time x heads"},
    }
    print(json.dumps(line), flush=True)


def _config_dict(name, cfg, n, head_sharded=False, transport="nccl"):
    f, h, w, ph, pw, heads, d, sp = cfg
    return {"workload": f"{name}: {f}x{h}x{w} tokens ({f * h * w}), {heads} heads, d={d}, "
                        f"{ph}x{pw} pool, {int(sp * 100)}% sparsity",
            "frames": f, "height": h, "width": w, "patch": [ph, pw], "heads": heads, "head_dim": d,
            "sparsity": sp,
            "parallelism": ((f"head-sharded replicas x{n} (no collective)" if head_sharded else
                             (f"head-parallel x{n} (sequence-sharded inputs read in place over NVLink, no all-to-all)"
                              if transport == "peer" else
                              f"head-parallel x{n} (sequence-sharded inputs, NCCL all-to-all)")) if n > 1
                            else "single GPU"),
            "l2": "inputs (3 x heads x n x d bf16) exceed the 126 MB L2; no flush needed"}


# --------------------------------------------------------------------------
# GPU arm
# --------------------------------------------------------------------------

def run_ours(args, cfg, name):
    import torch
    import torch.distributed as dist

    import paper_2505_14708_b200 as da
    from paper_2505_14708_b200 import _lib
    from paper_2505_14708_b200.build import build

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if rank == 0:
        build()
    # DA_BENCH_SAME_GPU=1 (a code-path check on a one-GPU box, not a measurement):
    # every rank on cuda:0, gloo, peer transport without the nccl cross-check
    same_gpu = os.environ.get("DA_BENCH_SAME_GPU") == "1"
    if same_gpu:
        local = 0
    torch.cuda.set_device(local)  # before NCCL: its communicator binds the current device
    dev = torch.device("cuda", local)
    if world > 1:
        if same_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
        dist.barrier()
    f, h, w, ph, pw, heads, d, sp = cfg
    plan = da.pad_plan(f, h, w, ph, pw)
    n = plan.num_valid
    g = plan.layout.num_regions
    p = plan.layout.region_size
    gen = torch.Generator(device=dev).manual_seed(1234 + rank)
    # N > 1: sequence-sharded inputs through the head-parallel all-to-alls, or
    # (--head-sharded) every rank already holds its heads: replicas, no collective
    collective = world > 1 and not args.head_sharded
    if world > 1 and args.head_sharded:
        assert heads % world == 0, "heads must divide the world size"
    hl = heads // world if world > 1 else heads

    if not collective:
        if args.data == "smooth":
            q, k, v = (_smooth_inputs(plan, hl, d, dev, gen) for _ in range(3))
        else:
            q, k, v = (torch.randn(hl, n, d, device=dev, generator=gen, dtype=torch.float32).to(torch.bfloat16)
                       for _ in range(3))

        def step(events=None):
            return da.api._pipeline(q, k, v, plan, sp, da.head_dim_scale(d), "average", "logits", True, False,
                                    "hnd", attn_events=events, want_bitmap=False)
    else:
        from paper_2505_14708_b200.headpar import HeadParallelAttention

        assert n % world == 0 and heads % world == 0, "tokens and heads must divide the world size"
        nl = n // world
        q, k, v = (torch.randn(nl, heads, d, device=dev, generator=gen, dtype=torch.float32).to(torch.bfloat16)
                   for _ in range(3))
        hp = HeadParallelAttention(plan, sp, world, rank, head_groups=args.head_groups)
        transport_note = None
        if args.transport == "peer":
            hp, q, k, v, transport_note = _peer_transport(hp, q, k, v, dev, same_gpu)
        comp_ev = [[] for _ in range(args.steps)]
        k4_ev = [[] for _ in range(args.steps)]
        step_i = [0]

        def step(events=None):
            if events is None:
                return hp(q, k, v)
            s_ = step_i[0]
            step_i[0] += 1
            return hp(q, k, v, compute_events=comp_ev[s_], k4_events=k4_ev[s_])

    clocks = ClockSampler(local).start()  # running (and sampling) before the timed region opens
    res = None
    for _ in range(args.warmup):
        # keep each result alive until the next step returns, as the timed
        # loop does, so the caching allocator has already grown to that
        # footprint (a cudaMalloc inside the timed steps would stall one call)
        res = step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for pair in ev:  # torch creates the CUDA event lazily on first record; the C library records them
        for e_ in pair:
            e_.record()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # step boundaries: per-call times for the median (median of >= 20 calls)
    marks = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps - 1)]
    kept_total = None
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks.begin()
    start.record()
    for s in range(args.steps):
        res = step(ev[s])
        if s < args.steps - 1:
            marks[s].record()
    end.record()
    torch.cuda.synchronize()
    clocks.end()
    elapsed = start.elapsed_time(end)
    bounds = [start] + marks + [end]
    per_call = [bounds[i].elapsed_time(bounds[i + 1]) for i in range(args.steps)]
    ms_median = statistics.median(per_call)
    if world > 1:  # max over ranks, like the value
        tm = torch.tensor([ms_median], device=dev, dtype=torch.float64)
        dist.all_reduce(tm, op=dist.ReduceOp.MAX)
        ms_median = float(tm.item())
    mask = res[1]
    kept_total = int(mask.kept_counts.sum().item())
    a2a_ms = None
    if collective:
        # compute phases and K4 launches of every head group (current stream);
        # the all-to-alls run on NCCL's stream: call - compute = exposed comm
        k4_ms = statistics.mean(sum(b.elapsed_time(e) for b, e in evs) for evs in k4_ev)
        comp_ms = statistics.mean(sum(b.elapsed_time(e) for b, e in evs) for evs in comp_ev)
        a2a_ms = max(0.0, elapsed / args.steps - comp_ms)
        t = torch.tensor([elapsed, k4_ms, a2a_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed, k4_ms, a2a_ms = float(t[0]), float(t[1]), float(t[2])
        kt = torch.tensor([kept_total], device=dev, dtype=torch.int64)
        dist.all_reduce(kt)
        kept_total = int(kt.item())
    else:
        k4_ms = statistics.mean(b.elapsed_time(e) for b, e in ev)
        if world > 1:  # replicas: max over ranks
            t = torch.tensor([elapsed, k4_ms], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            elapsed, k4_ms = float(t[0]), float(t[1])
            kt = torch.tensor([kept_total], device=dev, dtype=torch.int64)
            dist.all_reduce(kt)
            kept_total = int(kt.item())
    ms = elapsed / args.steps

    # effective work: 4 p^2 d per kept block pair (sparse.py:74-84 on the padded layout)
    eff_flops = 4.0 * p * p * d * kept_total
    peaks = _peaks()
    peak_tf = peaks.get("bf16_tflops_sustained") or 1419.7
    k4_tflops = eff_flops / (k4_ms * 1e-3) / 1e12 / world
    e2e = None
    cpu_base = None
    dense_ms = dense_err = None
    if collective:
        e2e = _e2e_sharded(hp, q.shape, dev, args, world)
    elif world > 1:
        e2e = _e2e(da, plan, cfg[:5] + (hl,) + cfg[6:], dev, args, world)
    if world == 1:
        e2e = _e2e(da, plan, cfg, dev, args)
        dense_ms, dense_err = (None, None) if args.no_dense else _dense_sdpa(q, k, v, res[0])
        if not args.no_cpu:
            # one whole head through the unmodified reference (~45 s), else two through the port
            ids = (0,) if _reference_impl() is not None else (0, 1)
            cms, sample, threads, kind = cpu_reference_sample(cfg, head_ids=ids)
            cpu_base = {"value": cms, "unit": "ms/call", "cores": threads, "kind": kind, "sample": sample,
                        "extrapolated": True}
    if rank == 0:
        calls_per_step = 1  # pipeline calls per step: one per head group on the nccl transport
        if collective and hp.transport == "nccl":
            from paper_2505_14708_b200.headpar import head_groups as _hg

            calls_per_step = len(_hg(hl, args.head_groups))
        launches = _lib.lib().da_pipeline_launches(0, 0) * calls_per_step * args.steps
        line = {
            "metric": METRIC, "value": ms, "unit": "ms/call", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False, "scaling": "strong",
            "ms_median": ms_median, "ms_calls": [round(x, 3) for x in per_call],
            "vs_baseline": None, "dtype": "bf16",
            "data": ("synthetic (torch.randn gaussian, seeded)" if args.data == "gaussian" else
                     "synthetic (smooth per-frame bilinear fields + 0.1 noise, synth.py mode, torch RNG, seeded)"),
            "config": _config_dict(name, cfg, world, head_sharded=world > 1 and args.head_sharded,
                                   transport=hp.transport if collective else "nccl"),
            "effective_tflops_per_gpu": eff_flops / (ms * 1e-3) / 1e12 / world,
            "kept_blocks": kept_total,
            "roofline": {"bound": "tensor", "kernel": "sparse_attn_lh_kernel (K4)", "achieved": k4_tflops,
                         "peak": peak_tf, "unit": "TFLOP/s", "frac": k4_tflops / peak_tf,
                         "peak_source": "MEASURED_PEAKS.json bf16_tflops_sustained" if peaks else "fallback",
                         "k4_ms": k4_ms, "k4_share_of_step": k4_ms / ms,
                         "algorithmic_flops_per_launch": eff_flops / world,
                         "traffic": _profile_traffic(name)},
            "gpu_launches": launches,
            "clocks": clocks.result,
        }
        if clocks.result and kept_total and world == 1:
            # K4's structural floor: a kept block is a 64-row tcgen05 tile pair
            # (GEMM1 + GEMM2 at M = 64) = 512 tensor cycles whatever the peak
            # says; at the SM clock measured during the timed steps
            sms = torch.cuda.get_device_properties(dev).multi_processor_count
            f_hz = clocks.result["sm_mhz"] * 1e6
            floor_ms = kept_total * (p // 64) ** 2 * 512 / (sms * f_hz) * 1e3  # (p = 128: four 64x64 blocks)
            line["roofline"]["tile_floor"] = {
                "what": "512 tensor cycles per kept 64x64x128 block (M = 64 tcgen05 tiles), all SMs, measured SM clock",
                "ms": floor_ms, "frac": floor_ms / k4_ms, "sm_mhz": clocks.result["sm_mhz"]}
        if a2a_ms is not None:  # all-to-all time NOT hidden under compute, per call, max over ranks
            line["collective_exposed_ms"] = a2a_ms
            line["transport"] = hp.transport
            if hp.transport == "nccl":
                line["head_groups"] = args.head_groups
            if transport_note:
                line["transport_note"] = transport_note
        if e2e is not None:
            line["e2e"] = e2e
        if dense_ms is not None:
            line["dense_sdpa_ms"] = dense_ms
            line["speedup_vs_dense_sdpa"] = dense_ms / ms
        if dense_err is not None:
            line["sparse_vs_dense_output"] = dense_err
        if cpu_base is not None:
            line["cpu_baseline"] = cpu_base
        print(json.dumps(line), flush=True)
    if world > 1:
        if collective:
            hp.close()  # unmap the peers' shard buffers (peer transport) before any rank frees its own
        dist.destroy_process_group()


def _smooth_inputs(plan, heads, d, dev, gen, field_scale=0.5, noise_scale=0.1):
    """The reference's secondary data mode (synth.py:44-86) on the GPU: per
    frame, a Gaussian field at patch corners, bilinearly upsampled to the token
    grid, plus 0.1-scaled i.i.d. noise; drawn on the padded grid, real rows
    kept (cli.py:77-98). torch RNG, so the values differ from numpy's."""
    import torch

    lay = plan.layout
    ch, cw, hp, wp = lay.patches_h, lay.patches_w, lay.height, lay.width
    ys = torch.linspace(0.0, ch, hp, device=dev, dtype=torch.float64)
    xs = torch.linspace(0.0, cw, wp, device=dev, dtype=torch.float64)
    y0 = ys.long().clamp(0, ch - 1)
    x0 = xs.long().clamp(0, cw - 1)
    fy = (ys - y0)[:, None, None].float()
    fx = (xs - x0)[None, :, None].float()
    knots = torch.randn(heads, lay.frames, ch + 1, cw + 1, d, device=dev, generator=gen) * field_scale
    k00 = knots[:, :, y0][:, :, :, x0]
    k01 = knots[:, :, y0][:, :, :, x0 + 1]
    k10 = knots[:, :, y0 + 1][:, :, :, x0]
    k11 = knots[:, :, y0 + 1][:, :, :, x0 + 1]
    field = k00 * (1 - fy) * (1 - fx) + k01 * (1 - fy) * fx + k10 * fy * (1 - fx) + k11 * fy * fx
    field += noise_scale * torch.randn(field.shape, device=dev, generator=gen)
    real = field[:, :, :plan.height, :plan.width]  # (heads, F, H, W, d): real rows, original order
    return real.reshape(heads, -1, d).to(torch.bfloat16).contiguous()


def _peer_transport(hp, q, k, v, dev, same_gpu):
    """Switch the head-parallel call to transport="peer" with the inputs in
    the mapped shard buffers. Unless ``same_gpu``, the first peer call is
    compared bit for bit with the nccl transport's (the same kernels on the
    same rows: the results are identical); any failure on any rank keeps the
    nccl transport. Returns (hp, q, k, v, note)."""
    import torch
    import torch.distributed as dist

    from paper_2505_14708_b200.headpar import HeadParallelAttention

    nl, heads, d = q.shape
    peer = HeadParallelAttention(hp.plan, hp.sparsity, hp.world, hp.rank, head_groups=hp.groups, transport="peer")
    note = None

    def agree(ok):  # every rank learns whether every rank succeeded (same collective sequence on all ranks)
        flag = torch.tensor([1 if ok else 0], dtype=torch.int32, device=dev)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        return int(flag.item()) == 1

    ok = True
    try:  # the mapping (one all-gather of IPC handles, then local opens)
        pb = peer.peer_buffers(nl, heads, d, v.shape[2])
        pb.q.copy_(q); pb.k.copy_(k); pb.v.copy_(v)
    except Exception as e:  # noqa: BLE001 - reported in the JSON line
        ok, note = False, f"peer mapping failed: {type(e).__name__}: {str(e)[:200]}"
    if not agree(ok):
        return hp, q, k, v, note or "another rank's peer mapping failed; nccl transport used"
    if not same_gpu:  # one call of each transport (both complete on every rank), compared bit for bit
        a, _ = peer(pb.q, pb.k, pb.v)
        b, _ = hp(q, k, v)
        torch.cuda.synchronize()
        ok = torch.equal(a, b)
        if not agree(ok):
            return hp, q, k, v, ("peer output differed from the nccl transport's" if not ok else
                                 "another rank's peer output differed; nccl transport used")
    return peer, pb.q, pb.k, pb.v, None


def _e2e_sharded(hp, shape, dev, args, world):
    """N > 1: each rank's sequence shard starts in pinned host memory; upload,
    the head-parallel call (two NCCL all-to-alls around the pipeline) and the
    download of the output shard are timed; max over ranks."""
    import torch
    import torch.distributed as dist

    host = [torch.randn(*shape, dtype=torch.float32).to(torch.bfloat16).pin_memory() for _ in range(3)]
    out_host = torch.empty(*shape, dtype=torch.bfloat16).pin_memory()

    pb = hp.peer_buffers(*shape[:3], shape[2]) if hp.transport == "peer" else None

    def once():
        if pb is not None:  # the shard lands straight in the mapped buffers
            for x, buf in zip(host, (pb.q, pb.k, pb.v)):
                buf.copy_(x, non_blocking=True)
            o, _ = hp(pb.q, pb.k, pb.v)
        else:
            qd, kd, vd = (x.to(dev, non_blocking=True) for x in host)
            o, _ = hp(qd, kd, vd)
        out_host.copy_(o, non_blocking=True)

    for _ in range(3):
        once()
    torch.cuda.synchronize()
    dist.barrier()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    steps = max(3, min(args.steps, 5))
    s.record()
    for _ in range(steps):
        once()
    e.record()
    torch.cuda.synchronize()
    t = torch.tensor([s.elapsed_time(e) / steps], device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    nb = shape[0] * shape[1] * shape[2] * 2
    return {"value": float(t[0]), "unit": "ms/call", "h2d_bytes_per_step": 3 * nb * world,
            "d2h_bytes_per_step": nb * world}


def _e2e(da, plan, cfg, dev, args, world=1):
    """Public API with pinned host inputs and a host copy of the output (max
    over ranks when replicas run on N > 1 GPUs)."""
    import torch

    f, h, w, ph, pw, heads, d, sp = cfg
    n = plan.num_valid
    host = [torch.randn(heads, n, d, dtype=torch.float32).to(torch.bfloat16).pin_memory() for _ in range(3)]
    out_host = torch.empty(heads, n, d, dtype=torch.bfloat16).pin_memory()

    def once():
        # host tensors in, host tensor out (the reference's calling convention):
        # the API uploads head groups while earlier groups compute and download
        return da.multi_head_sparse_attention(host[0], host[1], host[2], plan, sp, out=out_host)

    for _ in range(3):
        once()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    steps = max(3, min(args.steps, 5))
    s.record()
    for _ in range(steps):
        once()
    e.record()
    torch.cuda.synchronize()
    nb = heads * n * d * 2
    val = s.elapsed_time(e) / steps
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([val], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        val = float(t[0])
    return {"value": val, "unit": "ms/call", "h2d_bytes_per_step": 3 * nb * world, "d2h_bytes_per_step": nb * world}


def _dense_sdpa(q, k, v, sparse_out):
    """Dense attention (cuDNN / flash SDPA, bf16) on the call's own inputs: its
    time per call, and how far the sparse output is from it (the sweep's
    sparse-vs-dense output error)."""
    import torch
    import torch.nn.functional as F
    from torch.nn.attention import SDPBackend, sdpa_kernel

    qd, kd, vd = (x.unsqueeze(0) for x in (q, k, v))  # (1, heads, n, d) views
    try:
        with sdpa_kernel([SDPBackend.CUDNN_ATTENTION, SDPBackend.FLASH_ATTENTION]):
            dense = F.scaled_dot_product_attention(qd, kd, vd)
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for _ in range(3):
                F.scaled_dot_product_attention(qd, kd, vd)
            e.record()
            torch.cuda.synchronize()
        ms = s.elapsed_time(e) / 3
    except Exception:  # noqa: BLE001
        return None, None
    a = sparse_out.float().reshape(-1)
    b = dense[0].float().reshape(-1)
    err = {"rel_l2": float((a - b).norm() / b.norm()), "max_abs": float((a - b).abs().max()),
           "cosine": float(torch.nn.functional.cosine_similarity(a, b, dim=0)),
           "what": "sparse call output vs dense SDPA on the same bf16 inputs (all heads)"}
    del dense, a, b
    return ms, err


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="hv720", choices=sorted(CONFIGS))
    ap.add_argument("--sparsity", type=float, default=None)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline leg")
    ap.add_argument("--no-dense", action="store_true", help="skip timing dense SDPA at the same shape")
    ap.add_argument("--data", default="gaussian", choices=["gaussian", "smooth"],
                    help="synthetic input mode (synth.py): i.i.d. gaussian (primary) or smooth fields")
    ap.add_argument("--head-sharded", action="store_true",
                    help="N > 1: inputs arrive head-sharded (heads/N per rank): replicas, no collective")
    ap.add_argument("--transport", default="peer", choices=["peer", "nccl"],
                    help="N > 1: shard rows read in place over NVLink (peer) or NCCL all-to-alls (nccl)")
    ap.add_argument("--head-groups", type=int, default=3,
                    help="N > 1: head groups per rank (all-to-all / compute overlap)")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    if args.sparsity is not None:
        cfg = cfg[:7] + (args.sparsity,)
    if args.impl == "reference":
        args.warmup_ref = 1 if args.warmup > 0 else 0
        args.steps = max(1, min(args.steps, 3))
        run_reference(args, cfg, args.config)
    else:
        run_ours(args, cfg, args.config)


if __name__ == "__main__":
    main()
