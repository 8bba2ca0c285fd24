#!/usr/bin/env python
"""Benchmark of the TWED hot path on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload cfg3|cfg3_f32|cfg2|cfg1] [--no-batch] [--no-cpu]

Headline (N=1): BASELINE.json's metric "TWED GCUPS at the n=1M pair" on
config 3 (single pair, 3-D random walks, n = 1,000,000, nu = 1, lam = 1,
degree 2, fp64). One step = one full distance of the pair (1e12 DP cells).
The single pair does not shard across GPUs (replicas only),
so with N > 1 every rank solves its own replica (weak scaling). The batch
half of the metric -- twed_batch pairs/s on the 10k x 10k tri config 5 --
is reported in the "batch" object, sharded over the N GPUs (strong scaling).

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
    max_rows = max(e - b for b, e in bounds)
    block = torch.zeros((max_rows, N), dtype=torch.float32, device=dev)
    full = parts = None
    if world > 1 and rank == 0:
        full = torch.empty((N, N), dtype=torch.float32, device=dev)
        parts = [torch.empty_like(block) for _ in range(world)]
    lib = _lib.load()
    lib.twb_set_kernel_timing(1)

    def step():
        twb.twed_batch_dev(dS, off, dT, nu=1.0, lamb=1.0, degree=2, tri=True, row_begin=b0,
                           row_end=b1, out=block[: b1 - b0])
        if world > 1:  # the job's only collective: gather the row blocks, mirror on rank 0
            import torch.distributed as dist
            dist.gather(block, parts, dst=0)
            if rank == 0:
                for (lo, hi), part in zip(bounds, parts):
                    full[lo:hi].copy_(part[: hi - lo])
                twb.mirror_upper_dev(full)

    for _ in range(max(1, args.warmup // 2)):
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
                       "timed: NCCL gather of the row blocks to rank 0 + on-device mirror"),
            "sharding": [list(b) for b in bounds],
            "kernel_ms": kms,
            "roofline": {"bound": "fp32", "achieved": FLOPS_PER_CELL[2] * cells / (kms * 1e-3) / 1e12,
                         "peak": peak / 1e12, "unit": "TFLOP/s",
                         "frac": FLOPS_PER_CELL[2] * cells / (kms * 1e-3) / peak}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg3", choices=sorted(WORKLOADS))
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
    if args.impl == "reference":
        world = int(os.environ.get("WORLD_SIZE", "1"))
        rank = int(os.environ.get("RANK", "0"))
        run_reference(args, world, rank)
        return
    world, rank, local = dist_setup()
    run_ours(args, world, rank, local)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
