#!/usr/bin/env python
"""Benchmark of the TWED hot path on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload cfg3|cfg3_f32|cfg2|cfg1|cfg5] [--no-batch] [--no-cpu]

Headline (N=1): BASELINE.json's metric "TWED GCUPS at the n=1M pair" on
config 3 (single pair, 3-D random walks, n = 1,000,000, nu = 1, lam = 1,
degree 2, fp64). One step = one full distance of the pair (1e12 DP cells).
The single pair does not shard across GPUs, so with N > 1
(torchrun) the headline becomes the batch half of the metric -- twed_batch
pairs/s on the 10k x 10k tri config 5, strong-scaled over the ranks, the
unpadded gather to rank 0 and the on-device mirror inside the timed region
(--workload cfg5 selects it at any N). At N = 1 the batch is reported in the
"batch" object, and "other_configs" carries the other BASELINE configs, the
precompute's HBM GB/s, config 1's host-call latency, batch e2e (numpy in and
out), the paper's R^28 batch shape and LCS.

  value  : whole-job GCUPS with inputs resident in HBM (device API, CUDA
           events on the launching stream, max over ranks).
  e2e    : the same metric through the public host API (numpy in pinned host
           memory -> H2D -> kernels -> D2H of the distance) = what a user of
           warpband.twed gets.
  roofline: the DP kernel against the MEASURED FP64 add throughput of this
           GPU (add-chain probe in libtwb200; MEASURED_PEAKS.json carries only
           HBM and bf16 tensor peaks, which do not bound a min-plus DP).
  cpu_baseline: the reference package itself (twedband.engine.twed_parallel
           from baseline/_ref, numba per-diagonal parallel band, all host
           cores) on a bounded sample of the same workload, with the C
           restatement in oracle/ beside it; the port alone when baseline/_ref
           is absent.
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))

# Algorithmic ops per interior DP cell: subtractions, the
# lp norm (sqrt counted as 1), the time-gap terms, the three candidate sums
# and the two mins of interior_cost (_kernels.py:61-80).
FLOPS_PER_CELL = {1: 11, 2: 16, 3: 19, 4: 22}
METRIC = "TWED GCUPS (DP cells/s, n=1M pair)"

WORKLOADS = {
    "cfg1": dict(n=1_000, d=1, seed=0, dtype="f64"),
    "cfg2": dict(n=100_000, d=1, seed=1, dtype="f64"),
    "cfg3": dict(n=1_000_000, d=3, seed=2, dtype="f64"),
    "cfg3_f32": dict(n=1_000_000, d=3, seed=2, dtype="f32"),
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        if os.environ.get("TWB_BENCH_NO_CLOCKS"):  # diagnostics: no sampler at all
            return self
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def mark_start(self):
        self.i0 = len(self.lines)

    def mark_end(self):
        time.sleep(0.25)  # the sample in flight at the end of the region
        self.i1 = len(self.lines)

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        lines = self.lines[getattr(self, "i0", 0):getattr(self, "i1", len(self.lines))]
        for line in lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for name, flag in zip(names, parts[5:9]):
                if flag.lower() == "active":
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


# ---------------------------------------------------------------------------
# CPU reference: the reference package itself (baseline/_ref, installed from
# /root/reference with pip; travels to the GPU box with the snapshot) and the
# C restatement in oracle/ (always available) as a second column.
# ---------------------------------------------------------------------------
def load_reference():
    """twedband from baseline/_ref, or None when it is not installed / numba is missing."""
    ref = REPO / "baseline" / "_ref"
    if not (ref / "twedband").is_dir():
        return None
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/twb_numba_cache")
    if str(ref) not in sys.path:
        sys.path.insert(0, str(ref))
    try:
        import twedband
        return twedband
    except Exception as exc:  # numba absent or broken install
        log(f"reference package unavailable: {exc!r}")
        return None


def _ref_solver(kind: str, d: int, seed: int, threads: int):
    """solve(n) -> seconds for one pair of the workload generator at length n."""
    from paper_2007_16135_b200.workloads import make_pair

    if kind == "reference":
        tb = load_reference()
        params = tb.TwedParams(1.0, 1.0, 2)

        def solve(n):
            a, ta, b, tb_ = make_pair(n, d, seed)
            sa, sb = tb.TimeSeries(a, ta), tb.TimeSeries(b, tb_)
            t0 = time.perf_counter()
            tb.twed_parallel(sa, sb, params, threads)
            return time.perf_counter() - t0
    else:
        from oracle import oracle as orc
        orc.build()

        def solve(n):
            a, ta, b, tb_ = make_pair(n, d, seed)
            t0 = time.perf_counter()
            orc.twed(a, ta, b, tb_, 1.0, 1.0, 2, threads=threads)
            return time.perf_counter() - t0
    return solve


def cpu_reference_rate(kind: str, d: int, seed: int, budget_s: float, threads: int):
    """GCUPS of the CPU reference on one pair of the workload's generator,
    sized so that the final solve takes about `budget_s` seconds (cells ~ n^2)."""
    solve = _ref_solver(kind, d, seed, threads)
    solve(600)  # JIT / thread-pool warm-up (parallel path needs n >= 512)
    n = 2048
    dt = solve(n)
    while dt < budget_s / 16 and n < 1_000_000:
        n *= 2
        dt = solve(n)
    n2 = int(min(1_000_000, n * max(1.0, (budget_s / max(dt, 1e-6)) ** 0.5)))
    if n2 > n * 1.2:
        n = n2
        dt = solve(n)
    return n * n / dt / 1e9, n, dt


def reference_kind() -> str:
    return "reference" if load_reference() is not None else "port"


def reference_sample_text(kind, n, d, seed, threads, workload):
    what = ("twedband.engine.twed_parallel (the reference package from baseline/_ref, numba "
            "per-diagonal parallel band, _kernels.py:145-174)" if kind == "reference" else
            "C restatement of twedband.engine.twed_parallel (oracle/twed_oracle.c, per-diagonal "
            "parallel band)")
    return (f"one make_pair(n={n}, d={d}, seed={seed}) solve per step (bounded sample of "
            f"{workload}); {what}, {threads} threads")


def run_reference(args, world, rank):
    """--impl reference: the reference's CPU implementation on the host cores."""
    if rank != 0:
        return
    wl = WORKLOADS[args.workload]
    threads = os.cpu_count() or 1
    kind = reference_kind()
    d, seed = wl["d"], wl["seed"]
    _, n, _ = cpu_reference_rate(kind, d, seed, args.ref_step_s, threads)
    solve = _ref_solver(kind, d, seed, threads)
    for _ in range(args.warmup):
        solve(1024)
    elapsed = 0.0
    for _ in range(args.steps):
        elapsed += solve(n)
    value = args.steps * n * n / elapsed / 1e9
    # the rate at three sizes and the power-law fit t = c * n^a, extrapolated
    # to the workload's n (the reference's CPU rate grows with n: the per-
    # diagonal fork/join amortises)
    sizes = [int(n / 2), int(n / 2 ** 0.5), n]
    secs = [solve(sizes[0]), solve(sizes[1]), elapsed / args.steps]
    a_fit, c_fit = np.polyfit(np.log(sizes), np.log(secs), 1)
    t_full = float(np.exp(c_fit) * wl["n"] ** a_fit)
    fit = {"n": sizes, "seconds": secs, "gcups": [x * x / t / 1e9 for x, t in zip(sizes, secs)],
           "exponent": float(a_fit), "extrapolated_seconds_at_n": t_full,
           "extrapolated_gcups_at_n": wl["n"] ** 2 / t_full / 1e9, "n_target": wl["n"]}
    from oracle import oracle as orc
    line = {
        "impl": "reference", "metric": METRIC, "value": value,
        "unit": "GCUPS", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": elapsed / args.steps * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic random walks (SURVEY.md §8(d) generator)",
        "config": {"workload": args.workload, "n": wl["n"], "d": d, "sample_n": n},
        "cpu_baseline": {"value": value, "unit": "GCUPS", "cores": threads, "kind": kind,
                         "sample": reference_sample_text(kind, n, d, seed, threads,
                                                         args.workload),
                         "host": orc.host_description()},
        "e2e": {"value": value, "unit": "GCUPS", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "fit": fit,
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# Our arm
# ---------------------------------------------------------------------------
def flush_l2(buf):
    buf.add_(1)


def run_ours(args, world, rank, local):
    import torch

    import paper_2007_16135_b200 as twb
    from paper_2007_16135_b200 import _lib
    from paper_2007_16135_b200.workloads import make_pair

    lib = _lib.load()
    _lib.require_device()
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    wl = WORKLOADS[args.workload]
    n, d = wl["n"], wl["d"]
    f32 = wl["dtype"] == "f32"
    npdt = np.float32 if f32 else np.float64
    tdt = torch.float32 if f32 else torch.float64
    a, ta, b, tb = make_pair(n, d, wl["seed"] + 0)  # every replica solves the same pair
    host = [np.ascontiguousarray(x.astype(npdt)) for x in (a, ta, b, tb)]
    dev_in = [torch.from_numpy(x).to(dev) for x in host]
    out = torch.empty(1, dtype=torch.float64, device=dev)
    cells = float(n) * float(n)
    l2_flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)  # 256 MB > L2
    stream = torch.cuda.current_stream(dev)

    def step():
        twb.twed_dev(*dev_in, nu=1.0, lamb=1.0, degree=2, out=out, stream=stream)

    lib.twb_set_kernel_timing(1)
    # nvidia-smi starts (and settles) before the warm-up; only the samples
    # taken during the timed region are kept. The warm-up steps are the timed
    # step exactly (L2 flush included: its kernel is loaded lazily on first
    # use, which cost the first timed step up to 200 ms when it was not), and
    # the timed region follows them without an idle gap.
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    kernel_ms = []
    with ClockSampler(local) as clocks:
        time.sleep(1.0)
        for _ in range(args.warmup):
            flush_l2(l2_flush)
            step()
            lib.twb_last_kernel_ms()
        torch.cuda.synchronize()
        result = out.item()

        # ---- device-resident timed region ---------------------------------
        _lib.take_launch_count()
        # no cyclic-GC pass inside the region: a full collection of this
        # process's objects takes ~100 ms of host time between launches
        gc.collect()
        gc.disable()
        barrier(world)
        torch.cuda.synchronize()
        clocks.mark_start()
        ev0.record(stream)
        step_ev = []
        for _ in range(args.steps):
            e = torch.cuda.Event(enable_timing=True)
            e.record(stream)
            step_ev.append(e)
            flush_l2(l2_flush)
            step()
            kernel_ms.append(lib.twb_last_kernel_ms())
        ev1.record(stream)
        torch.cuda.synchronize()
        clocks.mark_end()
        gc.enable()
    barrier(world)
    launches = _lib.take_launch_count()  # libtwb200 kernels only (the L2 flush is torch's)
    marks = step_ev + [ev1]
    log("timed steps (ms, event-to-event / kernel):",
        [(round(a.elapsed_time(b), 2), round(k, 2)) for a, b, k in zip(marks, marks[1:], kernel_ms)])
    elapsed_ms = max_over_ranks(ev0.elapsed_time(ev1), world)
    value = world * args.steps * cells / (elapsed_ms * 1e-3) / 1e9
    ms_per_step = elapsed_ms / args.steps
    kmean = float(np.mean(kernel_ms))

    # ---- end to end through the public host API ---------------------------
    pinned = []
    for x in host:
        t = torch.empty(x.shape, dtype=tdt, pin_memory=True)
        t.numpy()[...] = x
        pinned.append(t.numpy())
    lib.twb_set_kernel_timing(0)
    twb.twed(*pinned, 1.0, 1.0, 2, dtype=npdt, device=local)  # warm
    barrier(world)
    gc.collect()
    gc.disable()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        r = twb.twed(*pinned, 1.0, 1.0, 2, dtype=npdt, device=local)
    e2e_local = time.perf_counter() - t0
    gc.enable()
    e2e_s = max_over_ranks(e2e_local, world)
    assert (r == result) or f32, (r, result)
    e2e = {"value": world * args.steps * cells / e2e_s / 1e9, "unit": "GCUPS",
           "h2d_bytes_per_step": int(sum(x.nbytes for x in host)), "d2h_bytes_per_step": 8,
           "ms_per_step": e2e_s / args.steps * 1e3, "api": "paper_2007_16135_b200.twed"}

    # ---- roofline -----------------------------------------------------------
    import ctypes
    shape = [ctypes.c_int64(0) for _ in range(3)]
    lib.twb_last_wave_shape(*(ctypes.byref(x) for x in shape))
    stripes, rows_per_stripe, ctas = (int(x.value) for x in shape)
    # bytes a launch must move: the two series (values + times) once, and each
    # stripe's bottom row (z and d, 16 B per column) written and read back once
    # (z is fp64 in every pair mode; d is fp32 in the fp32 mode)
    boundary = 2 * stripes * (n + 1) * (8 + (4 if f32 else 8))
    alg_bytes = sum(x.nbytes for x in host) + boundary
    peak_ops = lib.twb_probe_add_rate(0 if f32 else 1, local)
    achieved_ops = FLOPS_PER_CELL[d] * cells / (kmean * 1e-3)
    traffic = None
    prof = REPO / "profiles" / "ncu_summary.json"
    if prof.exists():
        try:
            traffic = json.loads(prof.read_text()).get(args.workload, {}).get("dram_bytes")
        except (ValueError, AttributeError):
            traffic = None
    roofline = {
        "bound": "fp32" if f32 else "fp64",
        "achieved": achieved_ops / 1e12, "peak": peak_ops / 1e12, "unit": "TFLOP/s",
        "frac": achieved_ops / peak_ops if peak_ops > 0 else None,
        "traffic": traffic,
        "kernel": "twb::wave_kernel (persistent flag-synchronised wavefront)",
        "kernel_ms": kmean, "kernel_share_of_step": kmean / ms_per_step,
        "flops_per_cell": FLOPS_PER_CELL[d], "cells_per_launch": cells,
        "peak_source": ("twb_probe_add_rate: measured independent-add throughput of the "
                        f"{'FP32' if f32 else 'FP64'} pipe on this GPU, 1 op per lane per add "
                        "(MEASURED_PEAKS.json has no FP64/FP32-ALU peak)"),
        "algorithmic_bytes_per_launch": alg_bytes,
        "algorithmic_bytes_per_cell": alg_bytes / cells,
        "sweep_shape": {"stripes": stripes, "rows_per_stripe": rows_per_stripe, "ctas": ctas},
        "traffic_note": ("ncu DRAM bytes of one cfg3 launch (profiles/ncu_summary.json): the "
                         "stripes' bottom rows written back from L2; the next stripe reads "
                         "them from L2"),
    }

    # ---- batch (config 5: tri 10k x 10k, n=128, d=2, fp32), sharded over ranks -------
    batch = None
    if not args.no_batch:
        batch = run_batch_cfg5(args, world, rank, local)
    extra = {} if args.no_extra else run_extra(args, world, rank, local)
    if world > 1 and not args.no_extra:
        extra["cfg3_one_pair_all_gpus"] = run_pair_all_gpus(args, world, rank, host)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        from oracle import oracle as orc
        threads = os.cpu_count() or 1
        kind = reference_kind()
        ref_gcups, ns, dts = cpu_reference_rate(kind, d, wl["seed"], args.cpu_budget_s, threads)
        cpu = {"value": ref_gcups, "unit": "GCUPS", "cores": threads, "kind": kind,
               "sample": reference_sample_text(kind, ns, d, wl["seed"], threads, args.workload)
               + f" ({dts:.1f} s)",
               "host": orc.host_description()}
        if kind == "reference":
            gp, np_, dtp = cpu_reference_rate("port", d, wl["seed"], args.cpu_budget_s / 2,
                                              threads)
            cpu["port"] = {"value": gp, "sample_n": np_,
                           "what": "C restatement of the same band (oracle/), same threads"}

    if rank == 0:
        line = {
            "metric": METRIC,
            "value": value, "unit": "GCUPS", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None,
            "dtype": "f32" if f32 else "f64",
            "data": "synthetic random walks (SURVEY.md §8(d) make_pair), unit timestamps",
            "config": {"workload": args.workload, "n": n, "d": d, "nu": 1.0, "lam": 1.0,
                       "degree": 2, "parallelism": f"replicas x{world} (single pair does not "
                       "shard)", "l2": "256 MB buffer written between timed steps"},
            "result": result,
            "e2e": e2e, "roofline": roofline, "cpu_baseline": cpu,
            "clocks": clocks.summary(), "gpu_launches": launches,
            "batch": batch,
            "other_configs": extra,
        }
        print(json.dumps(line), flush=True)


def run_extra(args, world, rank, local):
    """The other BASELINE configs, kernel-timed on this rank (events inside
    libtwb200, device-resident inputs): cfg3 in fp32 mode, cfg2, cfg1, and the
    cfg4 full 1000 x 1000 fp64 matrix sharded by rows over the ranks."""
    import torch

    import paper_2007_16135_b200 as twb
    from paper_2007_16135_b200 import _lib
    from paper_2007_16135_b200.distributed import row_bounds
    from paper_2007_16135_b200.workloads import make_pair, make_set

    lib = _lib.load()
    lib.twb_set_kernel_timing(1)
    dev = torch.device("cuda", local)
    res = {}
    for name in ("cfg3_f32", "cfg2", "cfg1"):
        wl = WORKLOADS[name]
        dt = np.float32 if wl["dtype"] == "f32" else np.float64
        a, ta, b, tb = (torch.from_numpy(np.ascontiguousarray(x.astype(dt))).to(dev)
                        for x in make_pair(wl["n"], wl["d"], wl["seed"]))
        out = twb.twed_dev(a, ta, b, tb, nu=1.0, lamb=1.0, degree=2)
        torch.cuda.synchronize()
        ks = []
        reps = 2 if wl["n"] >= 1_000_000 else 5
        for _ in range(reps):
            twb.twed_dev(a, ta, b, tb, nu=1.0, lamb=1.0, degree=2, out=out)
            ks.append(lib.twb_last_kernel_ms())
        kms = max_over_ranks(float(np.median(ks)), world)
        res[name] = {"n": wl["n"], "d": wl["d"], "dtype": wl["dtype"], "kernel_ms": kms,
                     "gcups": wl["n"] * wl["n"] / (kms * 1e-3) / 1e9, "result": out.item()}
    res["lcs"] = run_lcs(args, world, rank, local)
    res["precompute"] = run_precompute(args, local)
    res["cfg1_host_latency"] = run_cfg1_latency(args, local)
    res["mnist_shaped_d28"] = run_wide_batch(args, world, rank, local)
    if world == 1:
        res["batch_e2e"] = run_batch_e2e(args, local)
    # cfg4: AA 1000 x 256 (seed 3) against BB 1000 x 256 (seed 4), d = 1, fp64, full
    AA, TAA = make_set(1000, 256, 1, 3)
    BB, TBB = make_set(1000, 256, 1, 4)
    dA = torch.from_numpy(AA.reshape(-1, 1)).to(dev)
    dTA = torch.from_numpy(TAA.reshape(-1)).to(dev)
    dB = torch.from_numpy(BB.reshape(-1, 1)).to(dev)
    dTB = torch.from_numpy(TBB.reshape(-1)).to(dev)
    off = np.arange(1001, dtype=np.int64) * 256
    b0, b1 = row_bounds(1000, world, False)[rank]
    R = torch.empty((b1 - b0, 1000), dtype=torch.float64, device=dev)
    ks = []
    for _ in range(4):
        twb.twed_batch_dev(dA, off, dTA, dB, off, dTB, nu=1.0, lamb=1.0, degree=2, tri=False,
                           row_begin=b0, row_end=b1, out=R)
        ks.append(lib.twb_last_kernel_ms())
    kms = max_over_ranks(float(np.median(ks[1:])), world)
    res["cfg4"] = {"pairs": 1_000_000, "kernel_ms": kms, "pairs_per_s": 1e6 / (kms * 1e-3),
                   "gcups": 1e6 * 256 * 256 / (kms * 1e-3) / 1e9, "n_gpus": world,
                   "sharding": "rows, no collective in the timed kernel"}
    return res


def run_precompute(args, local):
    """The single pair's precompute as twed_dev runs it (twb_prepare_pair_dev:
    both cfg3 series, core.prepare_series C:218-234, fused with the input
    check, bulk-copy staged tiles) timed alone with CUDA events, L2 flushed
    before each launch. Achieved HBM GB/s = algorithmic bytes / time against
    MEASURED_PEAKS.json hbm_gbs."""
    import ctypes

    import torch

    from paper_2007_16135_b200 import _lib
    from paper_2007_16135_b200.workloads import make_pair

    lib = _lib.load()
    dev = torch.device("cuda", local)
    n, d = 1_000_000, 3
    a, ta, b, tb = (torch.from_numpy(np.ascontiguousarray(x)).to(dev) for x in make_pair(n, d, 2))
    V = [torch.empty((n + 1) * d, dtype=torch.float64, device=dev) for _ in range(2)]
    T = [torch.empty(n + 1, dtype=torch.float64, device=dev) for _ in range(2)]
    D = [torch.empty(n + 1, dtype=torch.float64, device=dev) for _ in range(2)]
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    l2 = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    st = torch.cuda.current_stream(dev)

    def launch():
        _lib.check(lib.twb_prepare_pair_dev_f64(
            a.data_ptr(), ta.data_ptr(), n, b.data_ptr(), tb.data_ptr(), n, d, 1.0, 1.0, 2,
            V[0].data_ptr(), T[0].data_ptr(), D[0].data_ptr(), V[1].data_ptr(), T[1].data_ptr(),
            D[1].data_ptr(), flag.data_ptr(), ctypes.c_void_p(st.cuda_stream)))

    for _ in range(3):
        launch()
    times = []
    for _ in range(20):
        flush_l2(l2)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(st)
        launch()
        e1.record(st)
        e1.synchronize()
        times.append(e0.elapsed_time(e1))
    ms = float(np.median(times))
    # per sample: reads d values + 1 time, writes d values + time + deletion cost
    alg = 2 * n * ((d + 1) + (d + 2)) * 8 + 2 * (d + 2) * 8
    peak = None
    mp = REPO / "MEASURED_PEAKS.json"
    if mp.exists():
        try:
            peak = float(json.loads(mp.read_text())["hbm_gbs"])
        except (ValueError, KeyError):
            peak = None
    peak = peak or 6545.6
    traffic = None
    prof = REPO / "profiles" / "ncu_summary.json"
    if prof.exists():
        try:
            traffic = json.loads(prof.read_text()).get("prepare", {}).get("dram_bytes")
        except (ValueError, AttributeError):
            traffic = None
    gbs = alg / (ms * 1e-3) / 1e9
    return {"kernel": "twb::prepare_kernel (both cfg3 series + input check, one launch)",
            "kernel_us": ms * 1e3, "algorithmic_bytes": alg, "achieved_gbs": gbs,
            "roofline": {"bound": "hbm", "achieved": gbs, "peak": peak, "unit": "GB/s",
                         "frac": gbs / peak, "traffic": traffic,
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs"},
            "timing": "CUDA events around one launch, 256 MB L2 flush before each, median of 20",
            "unsafe_flag": int(flag.item())}


def run_cfg1_latency(args, local):
    """Config 1 (n = 1000, d = 1, fp64) through the public host API, one call
    at a time: numpy in, H2D, precompute, sweep, D2H of the distance."""
    import paper_2007_16135_b200 as twb
    from paper_2007_16135_b200.workloads import make_pair

    a, ta, b, tb = make_pair(1_000, 1, 0)
    for _ in range(5):
        r = twb.twed(a, ta, b, tb, 1.0, 1.0, 2, device=local)
    ts = []
    for _ in range(50):
        t0 = time.perf_counter()
        r = twb.twed(a, ta, b, tb, 1.0, 1.0, 2, device=local)
        ts.append(time.perf_counter() - t0)
    return {"api": "paper_2007_16135_b200.twed (numpy in, float out)", "n": 1000, "d": 1,
            "median_ms": float(np.median(ts)) * 1e3, "min_ms": float(np.min(ts)) * 1e3,
            "calls": 50, "result": r, "e2e_gcups": 1e6 / float(np.median(ts)) / 1e9}


def run_wide_batch(args, world, rank, local):
    """The paper's R^28 shape (MNIST digits as 28 rows of 28 pixels,
    PAPER.md:391): 2000 series of n = 28, d = 28, fp64, tri, device-resident,
    through the runtime-d kernels (D = 0); the row blocks sharded over ranks."""
    import torch

    import paper_2007_16135_b200 as twb
    from paper_2007_16135_b200 import _lib
    from paper_2007_16135_b200.distributed import row_bounds
    from paper_2007_16135_b200.workloads import make_set

    lib = _lib.load()
    lib.twb_set_kernel_timing(1)
    dev = torch.device("cuda", local)
    N, n, d = 2000, 28, 28
    S, TS = make_set(N, n, d, 28)
    dS = torch.from_numpy(np.ascontiguousarray(S.reshape(N * n, d))).to(dev)
    dT = torch.from_numpy(np.ascontiguousarray(TS.reshape(N * n))).to(dev)
    off = np.arange(N + 1, dtype=np.int64) * n
    b0, b1 = row_bounds(N, world, True)[rank]
    out = torch.empty((b1 - b0, N), dtype=torch.float64, device=dev)
    ks = []
    for _ in range(4):
        twb.twed_batch_dev(dS, off, dT, nu=1.0, lamb=1.0, degree=2, tri=True, row_begin=b0,
                           row_end=b1, out=out)
        ks.append(lib.twb_last_kernel_ms())
    kms = max_over_ranks(float(np.median(ks[1:])), world)
    pairs = N * (N + 1) // 2
    return {"series": N, "n": n, "d": d, "dtype": "f64", "layout": "tri", "pairs": pairs,
            "kernel_ms": kms, "pairs_per_s": pairs / (kms * 1e-3),
            "gcups": pairs * n * n / (kms * 1e-3) / 1e9, "kernel": "batch_kernel<D = 0> (runtime d)"}


def run_batch_e2e(args, local):
    """configs 4 and 5 through the public host API twed_batch: numpy in, the
    validated lists packed, H2D, precompute, all-pairs kernel (+ on-device
    mirror for tri), D2H of the whole matrix into numpy (8 MB / 400 MB)."""
    import paper_2007_16135_b200 as twb
    from paper_2007_16135_b200.workloads import make_set

    out = {}
    AA, TAA = make_set(1000, 256, 1, 3)
    BB, TBB = make_set(1000, 256, 1, 4)
    S, TS = make_set(10000, 128, 2, 5)
    S32, TS32 = S.astype(np.float32), TS.astype(np.float32)
    cases = {
        "cfg4": (lambda: twb.twed_batch(AA, TAA, BB, TBB, 1.0, 1.0, 2, False, device=local),
                 1000 * 1000, AA.nbytes + TAA.nbytes + BB.nbytes + TBB.nbytes, 8 * 10 ** 6),
        "cfg5": (lambda: twb.twed_batch(S32, TS32, None, None, 1.0, 1.0, 2, True,
                                        dtype=np.float32, device=local),
                 10000 * 10001 // 2, S32.nbytes + TS32.nbytes, 4 * 10 ** 8),
    }
    for name, (call, pairs, h2d, d2h) in cases.items():
        call()
        ts = []
        for _ in range(max(3, args.steps)):
            t0 = time.perf_counter()
            R = call()
            ts.append(time.perf_counter() - t0)
        dt = float(np.median(ts))
        out[name] = {"api": "paper_2007_16135_b200.twed_batch (numpy in, numpy out)",
                     "pairs": pairs, "ms": dt * 1e3, "pairs_per_s": pairs / dt,
                     "h2d_bytes": int(h2d), "d2h_bytes": int(d2h), "shape": list(R.shape)}
    return out


def run_lcs(args, world, rank, local):
    """LCS length of two random DNA strings of 1M symbols:
    the bit-parallel kernel's event time (twb_lcs_i32), and on rank 0 of a 1-GPU
    run the reference's own lcs_band (numba three-diagonal band, one thread) on a
    bounded 20k x 20k sample of the same generator."""
    from paper_2007_16135_b200 import _lib
    from paper_2007_16135_b200.api import lcs_codes

    lib = _lib.load()
    lib.twb_set_kernel_timing(1)
    n = 1_000_000
    rng = np.random.default_rng(2007)
    a = rng.integers(0, 4, n)
    b = rng.integers(0, 4, n)
    lcs_codes(a[:4096], b[:4096], device=local)
    ks = []
    for _ in range(3):
        r = lcs_codes(a, b, device=local)
        ks.append(lib.twb_last_kernel_ms())
    kms = max_over_ranks(float(min(ks)), world)
    out = {"n": n, "alphabet": 4, "kernel_ms": kms, "gcups": n * n / (kms * 1e-3) / 1e9,
           "result": r, "kernel": "lcs_kernel (bit-parallel, 64 cells per word op)"}
    if rank == 0 and world == 1 and not args.no_cpu:
        tb = load_reference()
        if tb is not None:
            m = 20_000
            sa = "".join("ACGT"[x] for x in a[:m])
            sb = "".join("ACGT"[x] for x in b[:m])
            tb.lcs_band(sa[:500], sb[:500])  # JIT
            t0 = time.perf_counter()
            rv = tb.lcs_band(sa, sb)
            dt = time.perf_counter() - t0
            assert rv == lcs_codes(a[:m], b[:m], device=local)
            out["cpu_reference"] = {"gcups": m * m / dt / 1e9, "seconds": dt, "sample": f"{m} x {m}",
                                    "what": "twedband.lcs_band (numba band, 1 thread)"}
    return out


def run_pair_all_gpus(args, world, rank, host):
    """The headline pair as ONE distance over all N GPUs:
    rank 0 drives one kernel per device (twb_twed_multi_*, peer memory between
    consecutive devices) through the public API with host arrays; the other
    ranks keep their GPUs idle behind a CPU-side (gloo) barrier -- an NCCL
    barrier kernel would hold SMs the cooperative launches need."""
    import torch.distributed as dist

    import paper_2007_16135_b200 as twb

    grp = dist.new_group(backend="gloo")
    dist.barrier(group=grp)
    res = None
    if rank == 0:
        try:
            a, ta, b, tb = host
            n = len(a)
            twb.twed(a[:4096], ta[:4096], b[:4096], tb[:4096], 1.0, 1.0, 2,
                     device=list(range(world)))  # warm: contexts, peer access
            t0 = time.perf_counter()
            r = twb.twed(a, ta, b, tb, 1.0, 1.0, 2, device=list(range(world)))
            dt = time.perf_counter() - t0
            res = {"n_gpus": world, "ms": dt * 1e3, "gcups": n * n / dt / 1e9, "result": r,
                   "timing": "wall clock, host arrays (H2D + prepare + sweep + D2H), one run",
                   "path": "twb_twed_multi_f64: one CTA ring over one kernel per GPU"}
        except Exception as exc:  # report, do not fail the bench line
            res = {"n_gpus": world, "error": repr(exc)}
    dist.barrier(group=grp)
    return res


def batch_reference_rate(S, TS, n, d, count=240):
    """The reference's twed_batch (engine.py:183-226: per-pair serial band solves
    on a thread pool, all host cores) on a bounded sample of config 5: the
    symmetric batch of the first `count` series (fp32-rounded inputs, fp64)."""
    tb = load_reference()
    if tb is None:
        return None
    threads = os.cpu_count() or 1
    series = [tb.TimeSeries(S[k * n:(k + 1) * n].astype(np.float64),
                            TS[k * n:(k + 1) * n].astype(np.float64)) for k in range(count)]
    params = tb.TwedParams(1.0, 1.0, 2)
    w8 = series[:8]
    warm = tb.BatchSpec(w8, w8, params, symmetric=True, workers=threads)
    tb.twed_batch(warm)
    t0 = time.perf_counter()
    tb.twed_batch(tb.BatchSpec(series, series, params, symmetric=True, workers=threads))
    dt = time.perf_counter() - t0
    pairs = count * (count + 1) // 2
    return {"value": pairs / dt, "unit": "pairs/s", "cores": threads, "seconds": dt,
            "sample": f"symmetric batch of the first {count} config-5 series ({pairs} pairs)",
            "what": "twedband.twed_batch (the reference package, thread pool of serial band solves)"}


def run_batch_cfg5(args, world, rank, local):
    import torch

    import paper_2007_16135_b200 as twb
    from paper_2007_16135_b200 import _lib
    from paper_2007_16135_b200.distributed import row_bounds
    from paper_2007_16135_b200.workloads import make_set

    N, n, d = args.batch_n, 128, 2
    S, TS = make_set(N, n, d, 5)
    S = S.astype(np.float32).reshape(N * n, d)
    TS = TS.astype(np.float32).reshape(N * n)
    dev = torch.device("cuda", local)
    dS = torch.from_numpy(S).to(dev)
    dT = torch.from_numpy(TS).to(dev)
    off = np.arange(N + 1, dtype=np.int64) * n
    bounds = row_bounds(N, world, True)
    b0, b1 = bounds[rank]
    # rank 0 solves straight into its rows of the full matrix; the others into
    # their block, sent unpadded (exactly rows x N entries) to rank 0
    full = torch.empty((N, N), dtype=torch.float32, device=dev) if rank == 0 else None
    block = full[b0:b1] if rank == 0 else torch.empty((b1 - b0, N), dtype=torch.float32, device=dev)
    lib = _lib.load()
    lib.twb_set_kernel_timing(1)

    def step():
        twb.twed_batch_dev(dS, off, dT, nu=1.0, lamb=1.0, degree=2, tri=True, row_begin=b0,
                           row_end=b1, out=block)
        if world > 1:  # the job's only exchange: the row blocks to rank 0, mirror there
            import torch.distributed as dist
            if rank == 0:
                reqs = [dist.irecv(full[lo:hi], src=r) for r, (lo, hi) in enumerate(bounds)
                        if r > 0 and hi > lo]
                for q in reqs:
                    q.wait()
                twb.mirror_upper_dev(full)
            elif b1 > b0:
                dist.send(block, dst=0)

    for _ in range(max(1, args.warmup)):
        step()
    torch.cuda.synchronize()
    barrier(world)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    ks = []
    gc.collect()
    gc.disable()
    e0.record()
    for _ in range(args.steps):
        step()
        ks.append(lib.twb_last_kernel_ms())
    e1.record()
    torch.cuda.synchronize()
    gc.enable()
    ms = max_over_ranks(e0.elapsed_time(e1), world) / args.steps
    pairs = N * (N + 1) // 2
    cells = pairs * float(n) * n
    peak = lib.twb_probe_add_rate(0, local)
    kms = max_over_ranks(float(np.mean(ks)), world)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = batch_reference_rate(S, TS, n, d)
    return {"cpu_reference": cpu,
            "metric": "twed_batch pairs/s (tri 10k x 10k, n=128, d=2, fp32)",
            "workload": "cfg5", "pairs": pairs, "value": pairs / (ms * 1e-3), "unit": "pairs/s",
            "gcups": cells / (ms * 1e-3) / 1e9, "ms_per_step": ms, "n_gpus": world,
            "scaling": "strong",
            "gather": ("none (one GPU: the kernel writes the mirrored matrix)" if world == 1 else
                       "timed: each rank's rows sent unpadded to rank 0 (NCCL send/recv, "
                       f"{4 * N * (N - (bounds[0][1] - bounds[0][0]))} bytes in all) + "
                       "on-device mirror"),
            "sharding": [list(b) for b in bounds],
            "kernel_ms": kms,
            "roofline": {"bound": "fp32", "achieved": FLOPS_PER_CELL[2] * cells / (kms * 1e-3) / 1e12,
                         "peak": peak / 1e12, "unit": "TFLOP/s",
                         "frac": FLOPS_PER_CELL[2] * cells / (kms * 1e-3) / peak}}


BATCH_METRIC = "twed_batch pairs/s (tri 10k x 10k, n=128, d=2, fp32)"


def run_ours_batch(args, world, rank, local):
    """Headline at N > 1 (BASELINE: batch pairs/s on 1/2/4/8 GPUs): config 5
    strong-scaled over the ranks, the unpadded gather to rank 0 and the
    on-device mirror inside the timed region; e2e through
    distributed.twed_batch_distributed (numpy in on every rank, numpy matrix
    out on rank 0)."""
    import torch

    from paper_2007_16135_b200 import _lib
    from paper_2007_16135_b200.distributed import twed_batch_distributed
    from paper_2007_16135_b200.workloads import make_set

    _lib.load()
    _lib.require_device()
    torch.cuda.set_device(local)
    with ClockSampler(local) as clocks:
        time.sleep(1.0)
        _lib.take_launch_count()
        clocks.mark_start()
        batch = run_batch_cfg5(args, world, rank, local)
        clocks.mark_end()
    launches = _lib.take_launch_count()
    N = args.batch_n
    S, TS = make_set(N, 128, 2, 5)
    S32, TS32 = S.astype(np.float32), TS.astype(np.float32)
    twed_batch_distributed(S32, TS32, tri=True, dtype=np.float32)  # warm
    barrier(world)
    ts = []
    for _ in range(max(1, args.steps)):
        t0 = time.perf_counter()
        R = twed_batch_distributed(S32, TS32, tri=True, dtype=np.float32)
        ts.append(time.perf_counter() - t0)
    e2e_s = max_over_ranks(float(np.median(ts)), world)
    pairs = batch["pairs"]
    if rank == 0:
        assert R.shape == (N, N)
        line = {
            "metric": BATCH_METRIC, "value": batch["value"], "unit": "pairs/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": batch["ms_per_step"],
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic random walks (SURVEY.md §8(d) make_set), unit timestamps",
            "config": {"workload": "cfg5", "series": N, "n": 128, "d": 2, "layout": "tri",
                       "nu": 1.0, "lam": 1.0, "degree": 2, "parallelism": f"row blocks x{world}",
                       "l2": "400 MB output matrix written every step (> L2)"},
            "e2e": {"value": pairs / e2e_s, "unit": "pairs/s",
                    "h2d_bytes_per_step": int(world * (S32.nbytes + TS32.nbytes)),
                    "d2h_bytes_per_step": int(4 * N * N), "ms_per_step": e2e_s * 1e3,
                    "api": "paper_2007_16135_b200.distributed.twed_batch_distributed"},
            "roofline": batch["roofline"] | {"kernel": "twb::batch_kernel", "kernel_ms": batch["kernel_ms"],
                                             "flops_per_cell": FLOPS_PER_CELL[2]},
            "cpu_baseline": None, "clocks": clocks.summary(), "gpu_launches": launches,
            "batch": batch,
        }
        print(json.dumps(line), flush=True)


def run_reference_batch(args, world, rank):
    """--impl reference for the batch headline: the reference's twed_batch
    (engine.py:183-226) on all host cores, a bounded symmetric sample of
    config 5 per step; rank 0 only."""
    if rank != 0:
        return
    from paper_2007_16135_b200.workloads import make_set
    threads = os.cpu_count() or 1
    S, TS = make_set(args.batch_n, 128, 2, 5)
    S = S.astype(np.float32).reshape(-1, 2)
    TS = TS.astype(np.float32).reshape(-1)
    res = batch_reference_rate(S, TS, 128, 2, count=240)
    if res is None:
        print(json.dumps({"impl": "reference", "unavailable": "baseline/_ref not installed"}))
        return
    rates = [res["value"]]
    for _ in range(max(0, args.steps - 1)):
        rates.append(batch_reference_rate(S, TS, 128, 2, count=240)["value"])
    value = float(np.mean(rates))
    line = {"impl": "reference", "metric": BATCH_METRIC, "value": value, "unit": "pairs/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": res["seconds"] * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic random walks (SURVEY.md §8(d) make_set), fp32-rounded",
            "config": {"workload": "cfg5", "series": args.batch_n, "n": 128, "d": 2,
                       "sample_series": 240},
            "cpu_baseline": {"value": value, "unit": "pairs/s", "cores": threads,
                             "kind": "reference", "sample": res["sample"]},
            "e2e": {"value": value, "unit": "pairs/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default=None, choices=sorted(WORKLOADS) + ["cfg5"],
                    help="default: cfg3 (the n = 1M pair) on one GPU, cfg5 (the sharded "
                         "10k x 10k tri batch, BASELINE's 1/2/4/8-GPU metric) on several")
    ap.add_argument("--no-batch", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-extra", action="store_true")
    ap.add_argument("--batch-n", type=int, default=10_000)
    ap.add_argument("--cpu-budget-s", type=float, default=12.0)
    ap.add_argument("--ref-step-s", type=float, default=8.0)
    args = ap.parse_args()
    if args.warmup < 3:
        log("warning: fewer than 3 warm-up steps")
    world, rank, local = (1, 0, 0)
    if args.workload is None:
        args.workload = "cfg3" if int(os.environ.get("WORLD_SIZE", "1")) == 1 else "cfg5"
    if args.impl == "reference":
        world = int(os.environ.get("WORLD_SIZE", "1"))
        rank = int(os.environ.get("RANK", "0"))
        if args.workload == "cfg5":
            run_reference_batch(args, world, rank)
        else:
            run_reference(args, world, rank)
        return
    world, rank, local = dist_setup()
    if args.workload == "cfg5":
        run_ours_batch(args, world, rank, local)
    else:
        run_ours(args, world, rank, local)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
