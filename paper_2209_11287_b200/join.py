"""Epsilon self-join on B200: the drop-in for tilejoin.join (join.py:1-349).

`self_join(dataset, JoinConfig(epsilon=...)) -> JoinResult` keeps the
reference's signature, validation, error types, batching/capacity-guard
behaviour, counters and canonical (query id, neighbour id) ordering.  The
work runs on the GPU through libtedjoin.so:

    H2D coords -> tj_build_grid (cell keys, radix sort, cell table, candidate
    runs, estimates) -> per batch tj_refine (DMMA or CUDA-core FP64 + pair
    append) -> tj_finalize (CSR by original id, rows sorted) -> D2H CSR.

`kernel="tile"` selects the paper's tensor-core formulation (mma.sync m8n8k4
f64), `kernel="scalar"` the CUDA-core direct form (GDS-Join style); as in the
reference, only epsilon changes the pair set.  The pair set is the reference
direct-form set exactly: the tile path re-decides every pair whose expanded
value lies inside its rounding guard band with the direct form.
"""

from __future__ import annotations

import math
import os
import time
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .datasets import Dataset, as_dataset, reorder_dims_by_variance
from .errors import ResourceError, ValidationError

DEFAULT_K_IDX_CAP = 6  # grid.py:22


def default_k_idx(d: int) -> int:
    return min(d, DEFAULT_K_IDX_CAP)


@dataclass(frozen=True)
class JoinConfig:
    """Join parameters (join.py:30-46); only epsilon affects which pairs are returned.

    kernel: 'tile' = DMMA tensor-core path, 'scalar' = CUDA-core FP64 path,
        'auto' = the faster one for this d from measured throughput (extension);
        'core_fma' / 'core_expanded' = CUDA-core FMA direct / expanded form (extension).
    batch_size: target estimated pairs per batch (None = one batch).
    k_idx: indexed dimensions, default min(d, 6); the device grid supports <= 8.
    thread_count: accepted for compatibility (host threading has no role here).
    device: CUDA device index (extension; None = torch's current device).
    """

    epsilon: float
    kernel: str = "tile"
    short_circuit: bool = True
    k_idx: int | None = None
    batch_size: int | None = None
    thread_count: int = 1
    reorder_dims: bool = False
    device: int | None = None


@dataclass
class JoinStats:
    """Counters and phase timings from one join run (join.py:49-77)."""

    tiles_processed: int = 0
    chunks_executed: int = 0
    chunks_skipped: int = 0
    candidates_refined: int = 0
    pairs_emitted: int = 0
    index_seconds: float = 0.0
    refine_seconds: float = 0.0
    total_seconds: float = 0.0
    guard_rechecks: int = 0

    @property
    def pairs_per_second(self) -> float:
        return self.pairs_emitted / self.total_seconds if self.total_seconds > 0 else 0.0

    def as_dict(self) -> dict:
        return {
            "tiles_processed": self.tiles_processed,
            "chunks_executed": self.chunks_executed,
            "chunks_skipped": self.chunks_skipped,
            "candidates_refined": self.candidates_refined,
            "pairs_emitted": self.pairs_emitted,
            "index_seconds": self.index_seconds,
            "refine_seconds": self.refine_seconds,
            "total_seconds": self.total_seconds,
            "pairs_per_second": self.pairs_per_second,
        }


class _PairsField:
    """`JoinResult.pairs` as a dataclass field that is built on first read.

    Assigned explicitly (the reference's constructor, join.py:80-91), it is a
    plain value.  Left unset by the engine, the first read expands the CSR with
    the native multi-threaded tj_expand_pairs and caches the array.
    """

    def __set_name__(self, owner, name):
        self.slot = "_" + name

    def __get__(self, obj, owner=None):
        if obj is None:
            return None  # the dataclass default
        value = obj.__dict__.get(self.slot)
        if value is None and obj.__dict__.get("offsets") is not None:
            value = _native.expand_pairs(obj.offsets, obj.neighbors)
            obj.__dict__[self.slot] = value
        return value

    def __set__(self, obj, value):
        obj.__dict__[self.slot] = None if value is None else np.asarray(value)


@dataclass
class JoinResult:
    """Pair set of the join: ordered (query id, neighbour id), self-pairs included.

    The reference's dataclass (join.py:80-91): ``pairs`` (m, 2) int64 sorted by
    (query, neighbour), ``total_pairs``, ``selectivity`` = (|R| - n) / n,
    ``stats``.  The engine fills the CSR form -- ``offsets`` (int64, n+1) and
    ``neighbors`` (int32, ascending within each row), i.e. per-point neighbour
    lists -- and ``pairs`` is expanded from it on first access.  A result built
    from ``pairs`` alone (as reference callers do) derives the CSR on demand.
    """

    pairs: np.ndarray = _PairsField()
    total_pairs: int = 0
    selectivity: float = 0.0
    stats: JoinStats = field(default_factory=JoinStats)
    offsets: np.ndarray | None = field(default=None, repr=False, compare=False)
    neighbors: np.ndarray | None = field(default=None, repr=False, compare=False)

    def __post_init__(self):
        if self.offsets is None and self.__dict__.get("_pairs") is not None:
            pr = self.__dict__["_pairs"]
            n = int(pr[:, 0].max()) + 1 if len(pr) else 0
            self.offsets = np.concatenate(
                [[0], np.cumsum(np.bincount(pr[:, 0], minlength=n))]).astype(np.int64)
            self.neighbors = pr[:, 1].astype(np.int32)

    def neighbors_of(self, i: int) -> np.ndarray:
        return self.neighbors[self.offsets[i]: self.offsets[i + 1]]


@dataclass(frozen=True)
class BatchPlan:
    """Cell ranges (into the lexicographic cell list) per batch (join.py:94-99)."""

    batches: list = field(default_factory=list)
    estimated_pairs: list = field(default_factory=list)


def selectivity(result: JoinResult, n: int) -> float:
    """Average neighbours per query excluding self: (|R| - n) / n (join.py:102-106)."""
    if n < 1:
        raise ValidationError(f"n must be >= 1, got {n}")
    return (result.total_pairs - n) / n


def join_stats(result: JoinResult) -> JoinStats:
    return result.stats


def plan_from_estimates(cell_estimates, batch_size) -> BatchPlan:
    """Greedy contiguous batches closing once the running estimate reaches batch_size.

    Same partition as _plan_from_estimates (join.py:128-147), computed with a
    prefix sum + binary search per batch instead of a per-cell Python loop.
    """
    if batch_size is not None and batch_size < 1:
        raise ValidationError(f"batch_size must be >= 1, got {batch_size}")
    est = np.asarray(cell_estimates, dtype=np.int64)
    n_cells = len(est)
    if batch_size is None:
        return BatchPlan(batches=[(0, n_cells)], estimated_pairs=[int(est.sum())])
    csum = np.cumsum(est)
    batches, estimates = [], []
    start, base = 0, 0
    while start < n_cells:
        # first i >= start with csum[i] - base >= batch_size
        i = int(np.searchsorted(csum, base + batch_size, side="left"))
        if i >= n_cells:
            batches.append((start, n_cells))
            estimates.append(int(csum[-1] - base))
            break
        batches.append((start, i + 1))
        estimates.append(int(csum[i] - base))
        base = int(csum[i])
        start = i + 1
    return BatchPlan(batches=batches, estimated_pairs=estimates)


def plan_batches(index, config: JoinConfig) -> BatchPlan:
    """Batch plan over a built index (join.py:114-125): estimate |cell| * |cand(cell)|."""
    return plan_from_estimates(index.cell_costs(), config.batch_size)


def _validate_config(config: JoinConfig) -> None:
    """join.py:218-226."""
    if not np.isfinite(config.epsilon) or config.epsilon <= 0:
        raise ValidationError(f"epsilon must be positive and finite, got {config.epsilon}")
    if config.kernel not in KERNEL_CODES and config.kernel != "auto":
        raise ValidationError(
            f"kernel must be 'tile', 'scalar' or 'auto' (or {', '.join(CORE_VARIANTS)}), "
            f"got {config.kernel!r}")
    if config.batch_size is not None and config.batch_size < 1:
        raise ValidationError(f"batch_size must be >= 1, got {config.batch_size}")
    if config.thread_count < 1:
        raise ValidationError(f"thread_count must be >= 1, got {config.thread_count}")


def resolve_k_idx(config: JoinConfig, d: int) -> int:
    k_idx = config.k_idx if config.k_idx is not None else default_k_idx(d)
    if not 1 <= k_idx <= d:  # grid.py:79-80
        raise ValidationError(f"k_idx must be in [1, {d}], got {k_idx}")
    if k_idx > _native.TJ_MAX_K_IDX:
        raise ValidationError(
            f"k_idx must be <= {_native.TJ_MAX_K_IDX} on the device grid, got {k_idx}")
    return k_idx


# Refine-kernel throughput measured on one B200, round 2 (FP64 TFLOP/s, 2*d flops
# per candidate pair, short_circuit off; profiles/r2i/kncu, profiles/r2i/sweep_core.jsonl,
# profiles/r2g/sweep_hd.jsonl): (d, DMMA tile, best CUDA-core variant).  The CUDA-core
# kernels are issue-bound (ncu: 72-90 % issue-active, FP64 pipe 25-54 %); the DMMA
# formulation does 256 FMAs per instruction and wins at every measured d.  Above
# the DMMA instantiation (d > 64) only the CUDA-core kernel exists.
MEASURED_KERNEL_TFLOPS = ((2, 4.44, 1.39), (4, 9.64, 4.72), (8, 17.3, 6.38), (16, 23.8, 4.92),
                          (32, 27.0, 5.36), (64, 27.9, 3.2))
DMMA_MAX_DIM = 64

# JoinConfig.kernel -> tj_refine kernel code.  'tile' and 'scalar' are the
# reference's two kernels (join.py:34-41); the two extra CUDA-core variants do the
# FMA direct form and the expanded form in DFMA (same pair set, for the
# tensor-core vs CUDA-core comparison; refine_core.cu).
CORE_VARIANTS = ("core_fma", "core_expanded")
KERNEL_CODES = {"tile": _native.TJ_KERNEL_DMMA, "scalar": _native.TJ_KERNEL_CORE,
                "core_fma": _native.TJ_KERNEL_CORE_FMA,
                "core_expanded": _native.TJ_KERNEL_CORE_EXPANDED}


def resolve_kernel(kernel: str, d: int) -> str:
    """'tile' / 'scalar' as given; 'auto' picks the faster measured kernel for d
    (the nearest measured dimensionality), the CUDA-core one beyond d = 64."""
    if kernel != "auto":
        return kernel
    if d > DMMA_MAX_DIM:
        return "scalar"
    nearest = min(MEASURED_KERNEL_TFLOPS, key=lambda row: abs(row[0] - d))
    return "tile" if nearest[1] >= nearest[2] else "scalar"


_pinned: dict = {}


def _pin(arr: np.ndarray) -> bool:
    """Page-lock a host array once so H2D runs at full link speed.

    Memory torch already page-locked (read_dataset(pinned=True)) is used as is.
    Otherwise tj_host_register (cudaHostRegister; a failure leaves no stale CUDA
    error behind) pins it for the array's lifetime.  Returns False when the
    array stays pageable (small, non-contiguous, or registration refused).
    """
    import weakref

    import torch

    key = arr.__array_interface__["data"][0]
    if key in _pinned:
        return True
    if not arr.flags.c_contiguous or arr.nbytes < (1 << 20):
        return False
    if torch.from_numpy(arr).is_pinned():
        return True
    try:
        _native.host_register(key, arr.nbytes)
    except (RuntimeError, ValidationError):
        return False

    def _unregister(ptr=key):
        _pinned.pop(ptr, None)
        try:
            _native.host_unregister(ptr)
        except Exception:
            pass

    _pinned[key] = weakref.finalize(arr, _unregister)
    return True


def upload(work: Dataset, device: int):
    """Host Dataset.coords -> device tensor with the same (n, d_padded) layout."""
    import torch

    pinned = _pin(work.coords)
    host = torch.from_numpy(work.coords)
    out = host.to(device=f"cuda:{device}", non_blocking=pinned)
    return out


class DeviceJoin:
    """The join pipeline on one device, split into the steps bench.py times.

    prepare(): H2D + grid build; refine(): all batches; finalize(): canonical CSR
    on device; fetch(): D2H.  `self_join` chains them.
    """

    def __init__(self, work: Dataset, config: JoinConfig, device: int | None = None):
        import torch

        self.work = work
        self.config = config
        self.k_idx = resolve_k_idx(config, work.d)
        self.ctx = _native.context(device if device is not None else config.device)
        self.device = self.ctx.device
        self.kernel_name = resolve_kernel(config.kernel, work.d)
        self.kernel = KERNEL_CODES[self.kernel_name]
        self.torch = torch
        self.coords = None
        self.info = None
        self.total = 0

    def build(self, coords=None):
        w = self.work
        self.coords = coords if coords is not None else upload(w, self.device)
        self.ctx.build_grid(self.coords, w.n, w.d, int(self.coords.stride(0)), self.k_idx,
                            self.config.epsilon)
        self.info = self.ctx.grid_info()
        return self.info

    def plan(self) -> BatchPlan:
        if self.config.batch_size is None:
            return BatchPlan(batches=[(0, self.info.n_cells)],
                             estimated_pairs=[int(self.info.candidates)])
        return plan_from_estimates(self.ctx.cell_costs(self.info.n_cells), self.config.batch_size)

    # ---- output-budget batcher (join.py:184-202) ----
    SAMPLE_ITEMS = 256         # query blocks refined to estimate |R| (tj_estimate_pairs)
    SAMPLE_ABOVE = 1 << 24     # candidate pairs below which the buffer is just sized to C

    def appends_pairs(self) -> bool:
        """Every kernel but the low-d DMMA one (hit masks) appends (query, candidate)
        pairs to the ctx's pair buffer, whose size the batcher manages."""
        return not (self.kernel == _native.TJ_KERNEL_DMMA and self.work.d_padded == 4)

    def estimate_pairs(self, batches, costs=None) -> int:
        """Result pairs of `batches` from a sampled selectivity: SAMPLE_ITEMS query
        blocks of cost-weighted random cells run on the refine kernel with nothing
        stored (tj_estimate_pairs); pairs per candidate pair x candidate pairs,
        +25% and a floor for the sampling error."""
        if costs is None:
            costs = self.ctx.cell_costs(self.info.n_cells)
        csum = np.concatenate([[0], np.cumsum(costs)])
        total_c = int(sum(csum[b] - csum[a] for a, b in batches))
        if total_c <= self.SAMPLE_ABOVE:
            return total_c
        lo, hi = min(a for a, _ in batches), max(b for _, b in batches)
        rate = self.ctx.estimate_pairs(self.kernel, lo, hi, self.SAMPLE_ITEMS)
        return int(min(total_c, rate * total_c * 1.25 + (1 << 20)))

    def refine(self, cell_range=None, max_result_pairs=None, plan=None):
        """Run every batch; returns the exact pair count.

        Appending kernels write into a pair buffer sized from a sampled estimate
        (estimate_pairs).  The kernels count appends past its capacity, so after a
        batch the exact total is known: an overflowing batch is rolled back
        (counters + its per-query counts), the buffer grows to the exact size --
        keeping the earlier batches' pairs -- and the batch runs again, so no
        batch runs more than twice.  `max_result_pairs` is checked after every
        batch (join.py:198-202)."""
        cfg = self.config
        if plan is None:
            plan = self.plan()
        batches = plan.batches
        if cell_range is not None:
            lo, hi = cell_range
            batches = [(max(a, lo), min(b, hi)) for a, b in batches if min(b, hi) > max(a, lo)]
        # the low-d symmetric join (TJ_SYMMETRIC=1; measured slower on the device
        # step) reads every earlier cell's masks: for a cell range
        # past cell 0 (a multi-GPU shard) the earlier cells -- the shard's halo --
        # are refined for their masks only, below
        symmetric = os.environ.get("TJ_SYMMETRIC", "0") == "1"
        self.ctx.set_symmetric(symmetric)
        appends = self.appends_pairs()
        if appends and batches:
            est = self.estimate_pairs(batches)
        self.ctx.reset_results()
        if appends and batches:
            self.ctx.reserve_results(est)
        if symmetric and batches and batches[0][0] > 0:
            self.ctx.refine_masks(self.kernel, cfg.short_circuit, 0, batches[0][0])
        total = 0
        for batch_no, (start, stop) in enumerate(batches):
            if appends:
                self.ctx.checkpoint_results()
            self.ctx.refine(self.kernel, cfg.short_circuit, start, stop)
            if not (appends or max_result_pairs is not None):
                continue
            total, over = self.ctx.result_count()
            if over:  # exact total known: roll back, grow, run the batch again
                self.ctx.rollback_results(start, stop)
                self.ctx.reserve_results(total + (total >> 4) + 1024)
                self.ctx.refine(self.kernel, cfg.short_circuit, start, stop)
                total, over = self.ctx.result_count()
                if over:
                    raise RuntimeError(f"batch {batch_no}: pair buffer overflowed after growing")
            if max_result_pairs is not None and total > max_result_pairs:
                raise ResourceError(
                    f"batch {batch_no}: result grew to {total} pairs, "
                    f"beyond the container capacity of {max_result_pairs}")
        total, over = self.ctx.result_count()
        if over:  # a kernel appended where none was expected (non-finite norms): redo once
            self.ctx.reset_results()
            self.ctx.reserve_results(total + 1024)
            for start, stop in batches:
                self.ctx.refine(self.kernel, cfg.short_circuit, start, stop)
            total, over = self.ctx.result_count()
            if over:
                raise RuntimeError("pair buffer overflowed after growing")
        self.total = total
        return total

    def finalize(self):
        torch = self.torch
        n = self.work.n
        dev = f"cuda:{self.device}"
        self.offsets_d = torch.empty(n + 1, dtype=torch.int64, device=dev)
        self.neighbors_d = torch.empty(max(self.total, 1), dtype=torch.int32, device=dev)
        self.ctx.finalize(self.offsets_d, self.neighbors_d)
        return self.offsets_d, self.neighbors_d

    def fetch(self):
        torch = self.torch
        off = torch.empty(self.offsets_d.shape, dtype=torch.int64, pin_memory=True)
        nbr = torch.empty((self.total,), dtype=torch.int32, pin_memory=True)
        off.copy_(self.offsets_d, non_blocking=True)
        nbr.copy_(self.neighbors_d[: self.total], non_blocking=True)
        torch.cuda.current_stream(self.device).synchronize()
        return off.numpy(), nbr.numpy()

    # id ranges of the result pipeline, one D2H copy each (measured at c2,
    # profiles/r2aj/e2e_pipeline.txt: 16 ranges 10.46 ms for rows + copies, 8
    # ranges 10.64; grouping ranges into growing copies leaves a long last copy
    # exposed: 12.0)
    PIPELINE_CHUNKS = 16
    PIPELINE_COPIES = None

    def finalize_fetch(self, chunks: int | None = None, copies=None):
        """finalize() + fetch() as a pipeline into pinned host memory; returns numpy
        (offsets, neighbors).

        The offsets go first (their D2H on the copy stream overlaps the first rows).
        The rows are then built in `chunks` ranges of original ids
        (tj_finalize_rows_chunk): each range is one contiguous part of the CSR, final
        when its kernels end.  The ranges are copied in groups (`copies`: ranges per
        D2H, summing to `chunks`) on a copy stream while the next ranges are emitted
        -- the double-buffered result pipeline of the north star, with the PCIe copy
        engine running while the SMs emit."""
        torch = self.torch
        n = self.work.n
        dev = f"cuda:{self.device}"
        if chunks is None:
            chunks, copies = self.PIPELINE_CHUNKS, self.PIPELINE_COPIES
        if copies is None:
            copies = (1,) * chunks
        if sum(copies) != chunks:
            raise ValueError("copies must sum to chunks")
        main = torch.cuda.current_stream(self.device)
        self.offsets_d = torch.empty(n + 1, dtype=torch.int64, device=dev)
        self.neighbors_d = torch.empty(max(self.total, 1), dtype=torch.int32, device=dev)
        off = torch.empty((n + 1,), dtype=torch.int64, pin_memory=True)
        nbr = torch.empty((max(self.total, 1),), dtype=torch.int32, pin_memory=True)
        if not hasattr(self, "_copy_stream"):
            self._copy_stream = torch.cuda.Stream(device=self.device)
        cs = self._copy_stream
        self.ctx.finalize_offsets(self.offsets_d)
        cs.wait_stream(main)
        with torch.cuda.stream(cs):
            off.copy_(self.offsets_d, non_blocking=True)
            off_ready = torch.cuda.Event()
            off_ready.record(cs)
        bounds = [(k * n + chunks - 1) // chunks for k in range(chunks + 1)]  # tj_finalize_rows_chunk
        k = 0
        for g, m in enumerate(copies):
            k0 = k
            for _ in range(m):
                self.ctx.finalize_rows_chunk(self.offsets_d, self.neighbors_d, k, chunks)
                k += 1
            done = torch.cuda.Event()
            done.record(main)
            if g == 0:
                off_ready.synchronize()  # host needs the offsets to size the copies
            lo, hi = int(off[bounds[k0]]), int(off[bounds[k]])
            if hi > lo:
                cs.wait_event(done)
                with torch.cuda.stream(cs):
                    nbr[lo:hi].copy_(self.neighbors_d[lo:hi], non_blocking=True)
        cs.synchronize()
        main.synchronize()
        return off.numpy(), nbr[: self.total].numpy()

    def stats(self) -> JoinStats:
        st = self.ctx.stats()
        s = JoinStats(
            candidates_refined=int(st.candidates_refined),
            pairs_emitted=int(st.pairs_emitted),
            guard_rechecks=int(st.guard_rechecks),
        )
        if self.kernel_name == "tile":
            n_chunks = self.work.d_padded // 4
            if st.tiles_processed or st.candidates_refined == 0:
                s.tiles_processed = int(st.tiles_processed)
                s.chunks_executed = int(st.chunks_executed)
                s.chunks_skipped = int(st.chunks_skipped)
            else:  # d > 64 or non-finite norms: the exact kernel ran; report the tiling
                s.tiles_processed = int(self.info.tiles)
                s.chunks_executed = int(self.info.tiles) * n_chunks
        return s


# Variances closer than this (relative) are re-ranked on the host with numpy's own
# var(axis=0): compensated device sums are accurate to a few ulp, numpy's
# sequential ones to ~n ulp, so only such near-ties could order differently.
_VAR_TIE_REL = 1e-8


def variance_order(ctx, coords, dataset: Dataset) -> np.ndarray:
    """np.argsort(-var, kind="stable") of the columns (datasets.py:119-122), var on the GPU."""
    _, var = ctx.column_moments(coords, dataset.n, dataset.d)
    v = np.sort(var)
    if dataset.d > 1 and np.any(np.diff(v) <= _VAR_TIE_REL * np.abs(v[1:])):
        var = dataset.logical.var(axis=0)  # near-tie: the reference's exact values decide
    return np.argsort(-var, kind="stable")


def reorder_dims_on_device(ctx, coords, dataset: Dataset):
    """Device copy of the coordinates with columns in non-increasing variance order."""
    perm = variance_order(ctx, coords, dataset)
    if np.array_equal(perm, np.arange(dataset.d)):
        return coords
    out = coords.new_empty(coords.shape)
    ctx.permute_columns(coords, dataset.n, dataset.d, perm, out)
    return out


def self_join(dataset, config: JoinConfig, max_result_pairs: int | None = None) -> JoinResult:
    """Find every ordered pair within config.epsilon, self-pairs included (join.py:150-215).

    The pair set depends only on the data and epsilon.  ``max_result_pairs``
    caps the result and raises ResourceError naming the offending batch.
    """
    t_start = time.perf_counter()
    dataset = as_dataset(dataset)
    _validate_config(config)
    job = DeviceJoin(dataset, config)
    # one native context per device holds the grid and result buffers: joins on
    # the same device from several host threads run one after another
    with job.ctx.lock:
        coords = upload(dataset, job.device)
        if config.reorder_dims and dataset.n >= 2:  # join.py:163-164, on the device
            coords = reorder_dims_on_device(job.ctx, coords, dataset)
        job.build(coords)
        t_indexed = time.perf_counter()
        total = job.refine(max_result_pairs=max_result_pairs)
        offsets, neighbors = job.finalize_fetch()
        t_end = time.perf_counter()
        stats = job.stats()
    stats.pairs_emitted = total
    stats.index_seconds = t_indexed - t_start
    stats.refine_seconds = t_end - t_indexed
    stats.total_seconds = t_end - t_start
    return JoinResult(total_pairs=total, selectivity=(total - dataset.n) / dataset.n, stats=stats,
                      offsets=offsets, neighbors=neighbors)
