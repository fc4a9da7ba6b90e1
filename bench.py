#!/usr/bin/env python
"""Benchmark of the B200 FP64 epsilon self-join (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--kernel tile]
    python bench.py --impl reference ...      # the reference path on the host cores

One step = one complete self-join of the configured workload: grid index
build, estimator/batching, refine (DMMA or CUDA-core FP64) with pair
emission, canonical CSR output.  `value` is algorithmic FP64 distance
TFLOP/s = 2*d*C / step time (C = candidate pairs the grid produces, the
reference's JoinStats.candidates_refined) with inputs resident in HBM; the
step time in seconds is `ms_per_step`/1000 ("self-join s").  `e2e` repeats
the measurement through the public API `self_join(host Dataset, JoinConfig)`
with H2D of the coordinates and D2H of the CSR pair set inside the timed
region.  N>1 ranks (torchrun) default to config 5 strong-scaled: each rank
holds a 1/N row slice, the step plans equal-cost bin ranges (NCCL all-reduces),
routes every rank's bins + halo points to it (one all-to-all), joins its bins'
cells and all-reduces the per-id counts into the global offsets
(distributed.py); times are the max over ranks.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "self-join s & FP64 dist TFLOP/s (frac of peak), TC vs CUDA-core, 1/2/4/8 B200"
CONFIGS = {  # BASELINE.md §2 / SURVEY.md §8(d); eps for ~64 neighbours per point
    "c1": ("uniform", 100_000, 2, 0.0143667),
    "c2": ("uniform", 2_000_000, 4, 0.051306),
    "c3": ("exponential", 5_000_000, 8, 0.0118508),
    "c4d2": ("uniform", 2_000_000, 2, 0.00320714),
    "c4d4": ("uniform", 2_000_000, 4, 0.051306),
    "c4d8": ("uniform", 2_000_000, 8, 0.244686),
    "c4d16": ("uniform", 2_000_000, 16, 0.657508),
    "c4d32": ("uniform", 2_000_000, 32, 1.31923),
    "c4d64": ("uniform", 2_000_000, 64, 2.27218),
    "c5": ("uniform", 50_000_000, 4, 0.0232204),
    # the paper's best case (Expo3D2M): skewed 3-D data at ~64 neighbours
    "expo3d2m": ("exponential", 2_000_000, 3, 0.00097345),
}
L2_FLUSH_BYTES = 256 << 20  # > 126 MB L2


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines: list[tuple[float, str]] = []
        self.window = None  # (t0, t1) of the timed region

    def wait_first(self, timeout: float = 3.0):
        t = time.monotonic()
        while self.proc is not None and not self.lines and time.monotonic() - t < timeout:
            time.sleep(0.02)

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.monotonic(), line.strip()))

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        lines = self.lines
        if self.window is not None:
            t0, t1 = self.window
            inside = [x for x in lines if t0 - 0.25 <= x[0] <= t1 + 0.25]
            lines = inside or lines  # timed region shorter than the 200 ms period: use the load phase
        for _, ln in lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------- helpers
def host_info() -> dict:
    model = ""
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"cpu": model, "cpu_count": os.cpu_count(), "affinity": len(os.sched_getaffinity(0))}


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if args.impl == "reference":
            dist.init_process_group("gloo")
        elif os.environ.get("TJ_DIST_BACKEND", "nccl") == "gloo":
            # test hook: several ranks sharing the visible GPU(s) (NCCL refuses that)
            local = local % max(torch.cuda.device_count(), 1)
            torch.cuda.set_device(local)
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    return world, rank, local


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    dev = "cpu" if dist.get_backend() == "gloo" else "cuda"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    dev = "cpu" if dist.get_backend() == "gloo" else "cuda"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def barrier(world: int):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def refine_kernel_name(kernel: str, d: int) -> str:
    """The refine kernel tj_refine dispatches to (capi.cu)."""
    if kernel == "scalar":
        return "refine_core_kernel"
    return "refine_lowd_kernel" if d <= 4 else "refine_tc_kernel"


def traffic_from_profiles(config: str, kernel: str):
    """DRAM bytes per launch of `kernel` (function name) at `config`, from the committed
    ncu --set full summary (profiles/ncu_summary.json), if any."""
    p = ROOT / "profiles" / "ncu_summary.json"
    try:
        data = json.loads(p.read_text())
        return data.get(config, {}).get(kernel, {}).get("dram_bytes_per_launch")
    except (OSError, ValueError):
        return None


# ----------------------------------------------------------------- CPU side
def measured_hbm_gbs() -> tuple[float, str]:
    """HBM copy bandwidth from MEASURED_PEAKS.json (driver-written), else the guide's fallback."""
    try:
        return float(json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs"
    except (OSError, ValueError, KeyError):
        return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


def secondary_rooflines(n: int, d: int, dp: int, timings) -> list:
    """HBM rooflines of the phases around the refine, from the phase CUDA events.

    index: algorithmic bytes = n * (read d_pad coords + write d_pad cell-ordered
    coords + ceil(d/4) chunk norms + 8 B norm + 12 B key/id);
    output (finalize): 4 B per result pair written + 8 B offsets per point.
    """
    peak, src = measured_hbm_gbs()
    idx_ms = float(np.mean([t["index_ms"] for t in timings]))
    fin_ms = float(np.mean([t["finalize_ms"] for t in timings]))
    idx_bytes = n * (8 * dp * 2 + 8 * ((d + 3) // 4) + 8 + 12)
    out_bytes = 4 * timings[0]["pairs"] + 8 * (n + 1)
    rows = []
    for name, b, ms in (("index (grid build, all kernels)", idx_bytes, idx_ms),
                        ("canonical output (count scan + emit + long rows)", out_bytes, fin_ms)):
        gbs = b / (ms * 1e-3) / 1e9
        rows.append({"phase": name, "bound": "hbm", "achieved": gbs, "peak": peak, "unit": "GB/s",
                     "frac": gbs / peak, "algorithmic_bytes": b, "ms": ms, "peak_source": src})
    return rows


def host_threads() -> int:
    """Every host core this process may run on (torchrun sets OMP_NUM_THREADS=1;
    the reference arm and the CPU baseline pass an explicit thread count)."""
    try:
        return len(os.sched_getaffinity(0))
    except (AttributeError, OSError):
        return os.cpu_count() or 1


def cpu_reference(ds, eps: float, d: int, info_candidates: int, costs, budget_s: float = 20.0,
                  seed: int = 0, grid_s: float | None = None) -> dict:
    """Reference algorithm (oracle C port of grid.py + the scalar refiner, all host
    threads) on a bounded sample: the grid is built over all points (timed once),
    a seeded sample of query cells (the 10 costliest + random ones, ~budget_s of
    work) is refined in one emitting pass; the full-join time is extrapolated as
    grid + refine_sample * C / C_sample."""
    import oracle

    threads = host_threads()
    n_cells = len(costs)
    total = int(costs.sum())
    rng = np.random.default_rng(seed)
    probe = np.sort(rng.choice(n_cells, size=min(n_cells, 2000), replace=False))
    g_s, r_s, _ = oracle.time_join(ds, eps, cells=probe, threads=threads)
    if grid_s is None:
        grid_s = g_s
    rate = max(int(costs[probe].sum()), 1) / max(r_s, 1e-6)  # candidate pairs / s
    if total / rate <= budget_s:
        cells, label, c_sample = None, "full workload", total
    else:
        want = rate * budget_s * 0.8
        top = np.argsort(-costs, kind="stable")[:10]
        pick = set(int(c) for c in top)
        acc = int(costs[top].sum())
        for c in rng.permutation(n_cells):
            if acc >= want:
                break
            if int(c) not in pick:
                pick.add(int(c))
                acc += int(costs[c])
        cells = np.sort(np.fromiter(pick, dtype=np.int64))
        c_sample = int(costs[cells].sum())
        label = (f"{len(cells)} of {n_cells} query cells (10 costliest + seeded random), "
                 f"{c_sample} of {total} candidate pairs; grid over all points")
    _, r_s, pairs = oracle.time_join(ds, eps, cells=cells, threads=threads)
    full_s = grid_s + r_s * total / max(c_sample, 1)
    return {"value": 2.0 * d * total / full_s / 1e12, "unit": "TFLOP/s", "cores": threads,
            "kind": "port", "sample": label, "seconds": grid_s + r_s,
            "grid_seconds": grid_s, "refine_seconds": r_s, "sample_pairs": pairs,
            "candidate_pairs_per_s": c_sample / r_s,
            "extrapolated_full_join_s": full_s}


def run_reference(args, world, rank):
    """--impl reference: the reference algorithm (oracle C port of grid.py + join.py scalar
    refinement) on the host cores, rank 0 only."""
    dist_name, n, d, eps = CONFIGS[args.config]
    if rank != 0:
        return
    import oracle
    from paper_2209_11287_b200.datasets import GenSpec, generate

    ds = generate(GenSpec(dist_name, n, d, seed=0))
    order, cstart, ccoord, cand = oracle.grid(ds, eps, min(d, 6))
    costs = np.diff(cstart) * cand
    grid_s, _, _ = oracle.time_join(ds, eps, cells=np.zeros(1, np.int64), threads=host_threads())
    vals = []
    per_step = args.cpu_budget / max(args.steps + args.warmup, 1)
    for i in range(args.warmup + args.steps):
        r = cpu_reference(ds, eps, d, int(costs.sum()), costs, budget_s=per_step, seed=i,
                          grid_s=grid_s)
        if i >= args.warmup:
            vals.append(r)
    v = float(np.median([r["value"] for r in vals]))
    secs = float(np.median([r["extrapolated_full_join_s"] for r in vals]))
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "TFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": secs * 1e3,
        # throughput of one workload on the host cores; under weak scaling N
        # workloads take N times as long, so the value stands for every N
        "higher_is_better": True,
        "scaling": "weak" if world > 1 and args.scaling == "weak" else "strong",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference generator, seed 0)",
        "config": workload_config(args, world),
        "cpu_baseline": {k: vals[-1][k] for k in ("kind", "cores", "sample")} | {"value": v, "unit": "TFLOP/s"},
        "e2e": {"value": v, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "host": host_info(),
    }
    print(json.dumps(line), flush=True)


def workload_config(args, world: int) -> dict:
    """The JSON line's `config`: identical in both arms (ours and --impl reference)."""
    dist_name, n, d, eps = CONFIGS[args.config]
    weak = world > 1 and args.scaling == "weak"
    return {"workload": args.config, "dist": dist_name, "n": n * (world if weak else 1), "d": d,
            "eps": eps, "kernel": args.kernel, "short_circuit": not args.no_short_circuit,
            "l2": "256 MiB write between steps",
            "parallelism": (f"weak: {world} slabs of the workload side by side along dim 0"
                            if weak else f"strong: one workload over {world} rank(s)")}


# ------------------------------------------------------------------ GPU side
def weak_local_dataset(dist_name: str, n: int, d: int, eps: float, rank: int, world: int):
    """Rank `rank`'s part of the weak-scaled workload.

    The global dataset is `world` copies of the configured workload laid side by
    side along dimension 0 (slab r = the generator with seed r, x0 shifted by r:
    same density, same epsilon, world x the points).  Rank r owns the query
    cells whose dimension-0 index covers its slab and holds its slab plus a
    one-cell halo from each neighbouring slab (the candidates of those cells);
    no data crosses ranks inside the step.  Returns (local Dataset, own points,
    (lo, hi) dimension-0 cell indices of the owned cells).
    """
    from paper_2209_11287_b200.datasets import Dataset, GenSpec, generate

    def slab(r):
        x = generate(GenSpec(dist_name, n, d, seed=r)).coords
        x[:, 0] += r
        return x

    own = slab(rank)
    c0 = np.floor(own[:, 0] / eps)
    lo, hi = int(c0.min()), int(c0.max())
    parts = [own]
    if rank > 0:
        h = slab(rank - 1)
        parts.append(h[np.floor(h[:, 0] / eps) >= lo - 1])
    if rank < world - 1:
        h = slab(rank + 1)
        parts.append(h[np.floor(h[:, 0] / eps) <= hi + 1])
    coords = np.ascontiguousarray(np.concatenate(parts))
    return Dataset._wrap(coords, d), len(own), (lo, hi)


def run_ours(args, world, rank, local):
    import torch

    from paper_2209_11287_b200 import _native
    from paper_2209_11287_b200.datasets import Dataset, GenSpec, generate
    from paper_2209_11287_b200.join import DeviceJoin, JoinConfig, self_join

    dist_name, n, d, eps = CONFIGS[args.config]
    dev = local
    torch.cuda.set_device(dev)
    weak = world > 1 and args.scaling == "weak"
    if weak:  # every rank holds its own slab + halo; nothing is broadcast
        ds, n_own, (c_lo, c_hi) = weak_local_dataset(dist_name, n, d, eps, rank, world)
        n = ds.n
    else:
        ds = generate(GenSpec(dist_name, n, d, seed=0))
    cfg = JoinConfig(epsilon=eps, kernel=args.kernel, short_circuit=not args.no_short_circuit,
                     device=dev)
    # device-resident input on rank 0 (strong: other ranks receive it inside the
    # step) or on every rank (weak: its own slab + halo)
    coords0 = torch.from_numpy(ds.coords).to(f"cuda:{dev}")
    weak_range = {}  # owned cell range of the (deterministic) local grid, found once
    dp = 4 * ((d + 3) // 4)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.int32, device=f"cuda:{dev}")
    stream = torch.cuda.current_stream(dev)

    def one_step(kernel_cfg, timings=None):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
        ev[0].record(stream)
        coords = coords0  # N = 1, or weak: this rank's slab + halo, resident
        ev[1].record(stream)
        # non-root ranks hold only the shape on the host (np.empty touches no pages)
        work = ds if ds is not None else Dataset._wrap(np.empty((n, dp)), d)
        job = DeviceJoin(work, kernel_cfg, device=dev)
        info = job.build(coords)
        ev[2].record(stream)
        cell_range = None
        if weak:
            if not weak_range:  # first (warm-up) step: locate the owned cells once
                cc = job.ctx.export(info, job.k_idx)[2][:, 0]
                cb = int(np.searchsorted(cc, c_lo, side="left"))
                ce = int(np.searchsorted(cc, c_hi, side="right"))
                weak_range["r"] = (cb, ce)
                weak_range["C"] = int(job.ctx.cell_costs(info.n_cells)[cb:ce].sum())
            cell_range = weak_range["r"]
        job.refine(cell_range=cell_range)
        refine_ms = job.ctx.last_refine_ms()
        ev[3].record(stream)
        job.finalize()
        ev[4].record(stream)
        torch.cuda.synchronize(dev)
        st = job.ctx.stats()
        if timings is not None:
            timings.append({
                "step_ms": ev[0].elapsed_time(ev[4]),
                "bcast_ms": ev[0].elapsed_time(ev[1]),
                "index_ms": ev[1].elapsed_time(ev[2]),
                "refine_ms": ev[2].elapsed_time(ev[3]),
                "refine_kernel_ms": refine_ms,
                "finalize_ms": ev[3].elapsed_time(ev[4]),
                "candidates": int(info.candidates),
                "rank_candidates": int(st.candidates_refined),
                "pairs": int(job.total),
                "n_cells": int(info.n_cells),
                "rechecks": int(st.guard_rechecks),
                "emit_kernel_ms": job.ctx.last_emit_ms() if job.appends_pairs() is False else None,
            })
        return job

    def measure(kernel_cfg, steps, warmup, min_warm_s=1.0):
        with ClockSampler(dev) as clk:
            clk.wait_first()
            # >= `warmup` steps and >= min_warm_s of load, so the clock sampler sees the GPU
            # busy; ranks agree on every extra step (each step holds a collective)
            t_w, done = time.monotonic(), 0
            while True:
                more = done < warmup or time.monotonic() - t_w < min_warm_s
                if world > 1:
                    more = max_over_ranks(1.0 if more else 0.0, world) > 0.5
                if not more:
                    break
                one_step(kernel_cfg)
                flush.zero_()
                done += 1
            torch.cuda.synchronize(dev)
            barrier(world)
            timings = []
            launches0 = _native.launch_count()
            t0 = time.monotonic()
            for _ in range(steps):
                one_step(kernel_cfg, timings)
                flush.zero_()  # L2 flush between steps, outside the step events
            torch.cuda.synchronize(dev)
            barrier(world)
            # the timed steps are shorter than the 200 ms sampling period: report the
            # whole loaded phase (>= 1 s warm-up + timed steps)
            clk.window = (t_w, time.monotonic())
            launches = _native.launch_count() - launches0
            time.sleep(0.25)
        return timings, clk.summary(), launches

    timings, clocks, launches = measure(cfg, args.steps, args.warmup)
    step_ms = max_over_ranks(float(np.mean([t["step_ms"] for t in timings])), world)
    C = timings[0]["candidates"]
    if weak:  # whole-job work: the owned cells of every rank
        C = int(round(sum_over_ranks(float(weak_range["C"]), world)))
    value = 2.0 * d * C / (step_ms * 1e-3) / 1e12

    # TC vs CUDA-core: every other kernel on the same harness -- the reference's
    # exact scalar order, the FMA direct form and the expanded form in DFMA
    others = {}
    for other in ("tile", "scalar", "core_fma", "core_expanded"):
        if other == args.kernel:
            continue
        ocfg = JoinConfig(epsilon=eps, kernel=other, short_circuit=cfg.short_circuit, device=dev)
        o_t, _, _ = measure(ocfg, max(1, min(args.steps, 3)), 1)
        others[other] = (max_over_ranks(float(np.mean([t["step_ms"] for t in o_t])), world),
                         max_over_ranks(float(np.mean([t["refine_kernel_ms"] for t in o_t])), world))

    # roofline of the dominant kernel (refine), FP64 peak measured in-run
    peak_dmma, _ = _native.fp64_peak(1)
    peak_dfma, _ = _native.fp64_peak(0)
    peak = max(peak_dmma, peak_dfma)
    ref_ms = float(np.mean([t["refine_kernel_ms"] for t in timings]))
    rank_c = timings[0]["rank_candidates"]
    achieved = 2.0 * d * rank_c / (ref_ms * 1e-3) / 1e12
    share = ref_ms / float(np.mean([t["step_ms"] for t in timings]))

    # e2e through the public API with host buffers
    e2e_val = None
    h2d = n * dp * 8
    d2h = (n + 1) * 8 + timings[0]["pairs"] * 4
    if world == 1:
        # warm-up keeps the previous result alive like the timed loop does, so the
        # pinned host buffers of two results are cached (no cudaHostAlloc when timed)
        r = None
        for _ in range(max(2, args.warmup)):
            r = self_join(ds, cfg)
        ts = []
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize(dev)
            t = time.perf_counter()
            r = self_join(ds, cfg)
            ts.append(time.perf_counter() - t)
        e2e_s = float(np.mean(ts))
        d2h = (n + 1) * 8 + r.total_pairs * 4
        e2e_val = 2.0 * d * C / e2e_s / 1e12
    elif weak:
        # per rank: H2D of its slab + halo, join of its owned cells, D2H of its rows
        ts = []
        for i in range(args.warmup + args.steps):
            barrier(world)
            t = time.perf_counter()
            job = DeviceJoin(ds, cfg, device=dev)
            job.build()
            job.refine(cell_range=weak_range["r"])
            off_h, nbr_h = job.finalize_fetch()
            el = max_over_ranks(time.perf_counter() - t, world)
            if i >= args.warmup:
                ts.append(el)
        e2e_s = float(np.mean(ts))
        e2e_val = 2.0 * d * C / e2e_s / 1e12
        h2d = int(sum_over_ranks(float(ds.coords.nbytes), world))
        d2h = int(sum_over_ranks(float(off_h.nbytes + nbr_h.nbytes), world))
    if rank != 0:
        return
    cpu = None
    if world == 1 and not args.skip_cpu:
        import oracle

        order, cstart, ccoord, cand = oracle.grid(ds, eps, min(d, 6))
        costs = np.diff(cstart) * cand
        cpu = cpu_reference(ds, eps, d, C, costs, budget_s=args.cpu_budget)
    mean = lambda k: float(np.mean([t[k] for t in timings]))
    # the dominant kernel by its measured share of the step: the refine (FP64
    # roofline) or the row emission (HBM roofline, 4 B per result pair written)
    refine_roof = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                   "frac": achieved / peak,
                   "traffic": traffic_from_profiles(args.config, refine_kernel_name(args.kernel, d)),
                   "kernel": refine_kernel_name(args.kernel, d),
                   "peak_source": f"in-run FP64 microbenchmark max(DMMA {peak_dmma:.2f}, DFMA "
                                  f"{peak_dfma:.2f}) TFLOP/s; MEASURED_PEAKS.json has no FP64 entry",
                   "work": "2*d FLOP per candidate pair (SURVEY.md 8(d))",
                   "share_of_step": share}
    secondary = secondary_rooflines(n, d, dp, timings)
    emit_ms = [t["emit_kernel_ms"] for t in timings if t.get("emit_kernel_ms")]
    primary = refine_roof
    if emit_ms:
        e_ms = float(np.mean(emit_ms))
        hbm, hbm_src = measured_hbm_gbs()
        e_bytes = 4 * timings[0]["pairs"]
        emit_roof = {"bound": "hbm", "achieved": e_bytes / (e_ms * 1e-3) / 1e9, "peak": hbm,
                     "unit": "GB/s", "frac": e_bytes / (e_ms * 1e-3) / 1e9 / hbm,
                     "traffic": traffic_from_profiles(args.config, "emit_rows_kernel"),
                     "kernel": "emit_rows_kernel", "peak_source": hbm_src,
                     "work": "4 B written per result pair (the canonical neighbour ids)",
                     "ms": e_ms, "share_of_step": e_ms / float(np.mean([t["step_ms"] for t in timings]))}
        if e_ms > ref_ms:
            primary, secondary = emit_roof, [refine_roof] + secondary
        else:
            secondary = [emit_roof] + secondary
    line = {
        "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms,
        "self_join_s": step_ms / 1e3,
        "higher_is_better": True, "scaling": "weak" if weak else "strong", "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (reference generator restated, seed 0; checksum pinned in tests/golden)"
                if not weak else "synthetic: rank r = reference generator seed r, dim 0 shifted by r",
        "config": workload_config(args, world),
        "workload_stats": {"candidate_pairs": C, "result_pairs": timings[0]["pairs"],
                           "n_cells": timings[0]["n_cells"],
                           "layout": ("rank r owns slab r's cells + a one-cell halo, no "
                                      "collectives in the step") if weak else "single device"},
        "phases_ms": {k: mean(k) for k in ("bcast_ms", "index_ms", "refine_ms", "refine_kernel_ms",
                                           "finalize_ms")},
        "roofline": primary,
        "secondary_rooflines": secondary,
        "tc_vs_core": {args.kernel: {"step_ms": step_ms, "refine_kernel_ms": ref_ms,
                                     "refine_tflops": achieved}} | {
            k: {"step_ms": o_step, "refine_kernel_ms": o_ref,
                "refine_tflops": 2.0 * d * rank_c / (o_ref * 1e-3) / 1e12}
            for k, (o_step, o_ref) in others.items()},
        "e2e": {"value": e2e_val, "unit": "TFLOP/s", "seconds": e2e_s,
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "api": "self_join(host Dataset, JoinConfig) -> CSR in pinned host memory"
                       if world == 1 else
                       "per rank: DeviceJoin over its slab + halo (H2D, join of its cells, D2H "
                       "of its rows); max over ranks"},
        "gpu_launches": launches,
        "guard_rechecks": timings[0]["rechecks"],
        "clocks": clocks,
        "cpu_baseline": cpu,
        "host": host_info(),
    }
    print(json.dumps(line), flush=True)


def run_strong(args, world, rank, local):
    """N > 1, strong scaling (the default): ONE workload (config 5 unless --config)
    split by estimated cost over the ranks with the strong layout of
    distributed.py -- every step all-reduces the bin bounds/histogram, routes every
    rank's rows to the ranks needing them (one NCCL all-to-all: bins + halo), builds
    the local grid, refines the owned cells, emits canonical rows and all-reduces
    the per-id counts into the global CSR offsets.  Inputs at step start: each
    rank's 1/N row slice resident on its device.  Times are CUDA events on each
    rank, max over ranks."""
    import torch
    import torch.distributed as dist

    from paper_2209_11287_b200 import _native
    from paper_2209_11287_b200.datasets import GenSpec, generate
    from paper_2209_11287_b200.distributed import (
        SharedHostCSR,
        assemble_host_csr,
        row_slice,
        strong_self_join,
    )
    from paper_2209_11287_b200.join import JoinConfig

    dist_name, n, d, eps = CONFIGS[args.config]
    dev = local
    torch.cuda.set_device(dev)
    ds = generate(GenSpec(dist_name, n, d, seed=0))  # each host process reads its slice from it
    a, b = row_slice(n, rank, world)
    host_rows = torch.from_numpy(ds.coords[a:b]).pin_memory()
    rows = host_rows.to(f"cuda:{dev}")
    cfg = JoinConfig(epsilon=eps, kernel=args.kernel, short_circuit=not args.no_short_circuit,
                     device=dev)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.int32, device=f"cuda:{dev}")
    stream = torch.cuda.current_stream(dev)
    phases = ("plan", "exchange", "index", "refine", "offsets")

    def one_step(timings=None):
        evs = {"start": torch.cuda.Event(enable_timing=True)}
        evs["start"].record(stream)

        def mark(name):
            e = torch.cuda.Event(enable_timing=True)
            e.record(stream)
            evs[name] = e

        shard = strong_self_join(rows, n, d, cfg, timer=mark)
        torch.cuda.synchronize(dev)
        if timings is not None:
            st = shard.job.ctx.stats()
            t, prev = {}, "start"
            for ph in phases:
                t[ph + "_ms"] = evs[prev].elapsed_time(evs[ph])
                prev = ph
            t["step_ms"] = evs["start"].elapsed_time(evs["offsets"])
            t["refine_kernel_ms"] = shard.job.ctx.last_refine_ms() if shard.pairs else 0.0
            t["rank_candidates"] = int(st.candidates_refined)
            t["rank_pairs"] = shard.pairs
            t["pairs"] = shard.total_pairs
            t["n_local"] = shard.n_local
            timings.append(t)
        return shard

    with ClockSampler(dev) as clk:
        clk.wait_first()
        t_w = time.monotonic()
        for _ in range(max(args.warmup, 3)):
            one_step()
            flush.zero_()
        torch.cuda.synchronize(dev)
        barrier(world)
        launches0 = _native.launch_count()
        timings = []
        for _ in range(args.steps):
            one_step(timings)
            flush.zero_()
        torch.cuda.synchronize(dev)
        barrier(world)
        launches = _native.launch_count() - launches0
        clk.window = (t_w, time.monotonic())
        time.sleep(0.25)
    mean = lambda k: float(np.mean([t[k] for t in timings]))
    step_ms = max_over_ranks(mean("step_ms"), world)
    phase_max = {ph: max_over_ranks(mean(ph + "_ms"), world) for ph in phases}
    C = int(round(sum_over_ranks(float(timings[0]["rank_candidates"]), world)))
    value = 2.0 * d * C / (step_ms * 1e-3) / 1e12
    ref_ms = mean("refine_kernel_ms")
    achieved = 2.0 * d * timings[0]["rank_candidates"] / max(ref_ms * 1e-3, 1e-12) / 1e12
    peak_dmma, _ = _native.fp64_peak(1)
    peak_dfma, _ = _native.fp64_peak(0)
    peak = max(peak_dmma, peak_dfma)

    # e2e: each rank uploads its row slice (pinned), runs the step, and writes its
    # rows into the shared page-locked host CSR; root also copies the offsets
    total = timings[0]["pairs"]
    shared = SharedHostCSR(total)
    ts = []
    for i in range(args.warmup + args.steps):
        barrier(world)
        t = time.perf_counter()
        r_dev = host_rows.to(f"cuda:{dev}", non_blocking=True)
        shard = strong_self_join(r_dev, n, d, cfg)
        csr = assemble_host_csr(shard, shared)
        el = max_over_ranks(time.perf_counter() - t, world)
        if i >= args.warmup:
            ts.append(el)
    shared.close()
    e2e_s = float(np.mean(ts))
    nbytes_h2d = int(sum_over_ranks(float(host_rows.numel() * 8), world))
    if rank != 0:
        return
    assert csr is not None and int(csr[0][-1]) == total
    line = {
        "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms,
        "self_join_s": step_ms / 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference generator restated, seed 0; checksum pinned in tests/golden)",
        "config": workload_config(args, world),
        "workload_stats": {"candidate_pairs": C, "result_pairs": total,
                           "layout": f"{world} ranks own equal-cost contiguous (x0, x1) bin "
                                     "ranges; NCCL all-reduce of bounds, histogram and per-id "
                                     "counts + all-to-all of each rank's bins + halo points inside the step"},
        "phases_ms_max_over_ranks": phase_max,
        "rank0": {"n_local": timings[0]["n_local"], "pairs": timings[0]["rank_pairs"],
                  "refine_kernel_ms": ref_ms},
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak, "traffic": None,
                     "kernel": refine_kernel_name(args.kernel, d) + " (rank 0)",
                     "peak_source": f"in-run FP64 microbenchmark max(DMMA {peak_dmma:.2f}, "
                                    f"DFMA {peak_dfma:.2f}) TFLOP/s",
                     "work": "2*d FLOP per candidate pair (SURVEY.md 8(d))"},
        "e2e": {"value": 2.0 * d * C / e2e_s / 1e12, "unit": "TFLOP/s", "seconds": e2e_s,
                "h2d_bytes_per_step": nbytes_h2d,
                "d2h_bytes_per_step": 8 * (n + 1) + 4 * total,
                "api": "distributed.strong_self_join + assemble_host_csr (each rank uploads its "
                       "row slice and writes its rows into one shared mapped host CSR)"},
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "cpu_baseline": None,
        "host": host_info(),
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default=None,
                    help="workload (default: c2 on one GPU, c5 strong-scaled over N > 1)")
    ap.add_argument("--kernel", choices=("tile", "scalar", "core_fma", "core_expanded"), default="tile")
    ap.add_argument("--no-short-circuit", action="store_true")
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--scaling", choices=("weak", "strong"), default="strong",
                    help="N > 1: strong = one workload (default c5) split by estimated cost "
                         "(the default); weak = each rank owns one workload-sized slab")
    ap.add_argument("--cpu-budget", type=float, default=20.0,
                    help="seconds of host-core reference work per run (sampled cells)")
    args = ap.parse_args()
    world, rank, local = dist_setup(args)
    if args.config is None:
        args.config = "c5" if world > 1 and args.scaling == "strong" else "c2"
    if args.impl == "reference":
        run_reference(args, world, rank)
    elif world > 1 and args.scaling == "strong":
        run_strong(args, world, rank, local)
    else:
        run_ours(args, world, rank, local)
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
