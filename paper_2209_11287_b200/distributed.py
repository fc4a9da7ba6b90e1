"""Multi-GPU self-join: one process per GPU, each owning a cost-balanced cell range.

Replaces the reference's only data-parallel executor -- a thread pool mapping a
batch's cells (join.py:184-197) -- with the strong layout of SURVEY.md 8(e):

1. every rank holds a 1/G slice of the input rows (its own PCIe upload);
2. prefix bins (the first min(2, k_idx) indexed dims of each point's cell,
   floor(x_j / eps), grid.py:81): one MIN/MAX all-reduce of the bounds and
   one SUM all-reduce of the per-bin point counts (a few KB);
3. every rank derives the same plan on the host: per-bin cost = count x the
   3x3 neighbourhood count (the reference estimator |cell| * |cand(cell)|,
   join.py:122-124, at bin granularity), cut into G contiguous lexicographic
   bin ranges of equal cost -- contiguous cell ranges of the reference order;
4. every rank routes its own rows to the ranks that need them -- a point goes to
   the owner of its bin and to the ranks whose bins are in its one-cell halo
   (one counting pass + a stable compaction per destination, tj_shard_route) -- and
   one all-to-all (NCCL over NVLink) delivers each rank its bins' points plus
   its halo, in global id order;
5. each rank builds the grid over those points, refines only its owned cells
   (tj_shard_cell_range) and emits its canonical CSR rows with global neighbour
   ids (tj_set_output_ids: local ids are monotone in global ids, so rows stay
   sorted);
6. global row offsets: each rank scatters its row counts to global ids
   (tj_scatter_counts_u8), one SUM all-reduce of n one-byte counts (int32 when
   a row reaches 256 ids), one scan.
The pair set then sits on the devices, each rank holding its rows and every
rank the global offsets: no O(|R|) buffer exists on any rank.  To land it on
the host, every rank writes its rows straight to their final places in one
shared, page-locked, device-mapped host CSR (`assemble_host_csr`: one
/dev/shm segment, tj_place_rows over each rank's own PCIe link).

The bin planning, the halo predicate and the placement are restated in numpy
below (`plan_bins`, `halo_mask`) for the gloo CPU tests; the device kernels are
csrc/shard.cu.
"""

from __future__ import annotations

import mmap
import os
import uuid
from dataclasses import dataclass, field

import numpy as np

from .datasets import Dataset

PREFIX_DIMS = 2  # bins over the first min(2, k_idx) indexed dims


# ------------------------------------------------------------------ host planning
def balanced_cell_ranges(costs, parts: int) -> list[tuple[int, int]]:
    """Cut items into `parts` contiguous half-open ranges of ~equal total cost.

    Range r ends at the first item whose inclusive prefix cost reaches
    (r+1)/parts of the total; contiguity keeps each rank's candidate runs local.
    """
    costs = np.asarray(costs, dtype=np.int64)
    n = len(costs)
    if parts < 1:
        raise ValueError("parts must be >= 1")
    csum = np.cumsum(costs)
    total = int(csum[-1]) if n else 0
    bounds = [0]
    for r in range(1, parts):
        target = (total * r + parts - 1) // parts
        cut = int(np.searchsorted(csum, target, side="left")) + 1 if total else 0
        bounds.append(min(max(cut, bounds[-1]), n))
    bounds.append(n)
    return [(bounds[r], bounds[r + 1]) for r in range(parts)]


def bin_costs(hist: np.ndarray, span) -> np.ndarray:
    """count(b) * sum of counts over b's 3x3 neighbourhood (3-neighbourhood for 1 dim)."""
    h = np.asarray(hist, dtype=np.int64).reshape(int(span[0]), -1)
    pad = np.pad(h, 1)
    nb = np.zeros_like(h)
    rows = (0, 1, 2)
    cols = (0, 1, 2) if h.shape[1] > 1 else (1,)
    for a in rows:
        for b in cols:
            nb += pad[a: a + h.shape[0], b: b + h.shape[1]]
    return (h * nb).reshape(-1)


@dataclass(frozen=True)
class ShardPlan:
    """Agreed partition: prefix dims, bin origin/span and each rank's owned bin range."""

    pdims: int
    origin: tuple
    span: tuple
    ranges: tuple  # per rank (own_lo, own_hi) inclusive lexicographic bin indices
    bin_cost: np.ndarray = field(repr=False, compare=False, default=None)

    def owned(self, rank: int) -> tuple[int, int]:
        return self.ranges[rank]

    def cost_share(self) -> list[int]:
        return [int(self.bin_cost[lo: hi + 1].sum()) if hi >= lo else 0 for lo, hi in self.ranges]


def plan_bins(hist, pdims: int, origin, span, world: int) -> ShardPlan:
    """Equal-cost contiguous bin ranges (inclusive) for `world` ranks."""
    costs = bin_costs(hist, span)
    ranges = tuple((lo, hi - 1) for lo, hi in balanced_cell_ranges(costs, world))
    return ShardPlan(pdims, tuple(int(v) for v in origin), tuple(int(v) for v in span), ranges,
                     costs)


def point_bins(x: np.ndarray, eps: float, pdims: int, origin) -> tuple[np.ndarray, np.ndarray]:
    """(b0, b1) bin coordinates of rows of x: floor(x_j / eps) - origin_j (numpy mirror)."""
    b0 = np.floor(x[:, 0] / eps).astype(np.int64) - origin[0]
    b1 = (np.floor(x[:, 1] / eps).astype(np.int64) - origin[1]) if pdims > 1 else np.zeros_like(b0)
    return b0, b1


def halo_mask(b0, b1, span, pdims: int, lo: int, hi: int) -> np.ndarray:
    """Numpy restatement of shard.cu bin_needed: some bin within Chebyshev distance 1
    of (b0, b1) lies in the owned lexicographic interval [lo, hi]."""
    s0, s1 = int(span[0]), int(span[1]) if pdims > 1 else 1
    w = 1 if pdims > 1 else 0
    need = np.zeros(len(b0), dtype=bool)
    for dq in (-1, 0, 1):
        q0 = b0 + dq
        ok = (q0 >= 0) & (q0 < s0)
        lo_l = q0 * s1 + np.maximum(b1 - w, 0)
        hi_l = q0 * s1 + np.minimum(b1 + w, s1 - 1)
        need |= ok & (lo_l <= hi) & (hi_l >= lo)
    return need


def prefix_dims(d: int, k_idx: int) -> int:
    return max(1, min(PREFIX_DIMS, d, k_idx))


# ------------------------------------------------------------------ device path
def _all_reduce(t, op, group):
    import torch.distributed as dist

    dist.all_reduce(t, op=op, group=group)
    return t


def plan_shards(ctx, rows, eps: float, pdims: int, group=None) -> ShardPlan:
    """Steps 2-3: bounds + histogram of this rank's rows, all-reduced, planned on the host."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    n = rows.shape[0]
    lo, hi = ctx.shard_bounds(rows, n, pdims, eps)
    dev = rows.device if dist.get_backend(group) != "gloo" else torch.device("cpu")
    big = np.iinfo(np.int64).max
    lo_t = torch.tensor(list(lo) if n else [big] * pdims, dtype=torch.int64, device=dev)
    hi_t = torch.tensor(list(-np.asarray(hi)) if n else [big] * pdims, dtype=torch.int64, device=dev)
    both = torch.cat([lo_t, hi_t])  # one MIN all-reduce: (lo, -hi)
    _all_reduce(both, dist.ReduceOp.MIN, group)
    both = both.cpu().numpy()
    origin = both[:pdims]
    span = -both[pdims:] - origin + 1
    span_full = (int(span[0]), int(span[1]) if pdims > 1 else 1)
    hist = torch.zeros(span_full[0] * span_full[1], dtype=torch.int64, device=rows.device)
    ctx.shard_histogram(rows, n, pdims, eps, origin, span_full, hist)
    if dev.type == "cpu":
        hist = hist.cpu()
    _all_reduce(hist, dist.ReduceOp.SUM, group)
    return plan_bins(hist.cpu().numpy(), pdims, (int(origin[0]), int(origin[1]) if pdims > 1 else 0),
                     span_full, world)


@dataclass
class ShardResult:
    """One rank's part of the distributed join (device tensors)."""

    plan: ShardPlan
    rank: int
    n: int                  # global points
    n_local: int            # points this rank holds (owned + halo)
    gid: object             # uint32 (as int32) [n_local] global id of each local point
    offsets: object         # int64 [n_local + 1] local CSR (rows of owned points only)
    neighbors: object       # int32 [pairs] global neighbour ids, rows ascending
    global_offsets: object  # int64 [n + 1] the global CSR offsets (every rank)
    pairs: int              # pairs this rank emitted
    total_pairs: int        # pairs of the whole join
    cells: tuple            # owned cell range of the local grid
    job: object = field(repr=False, default=None)
    times: dict = field(default_factory=dict)


def _a2a(out, inp, out_splits, in_splits, group):
    """all_to_all_single; the gloo backend moves CUDA tensors through host memory."""
    import torch.distributed as dist

    if dist.get_backend(group) == "gloo" and inp.is_cuda:
        o = out.cpu()
        dist.all_to_all_single(o, inp.cpu(), out_splits, in_splits, group=group)
        out.copy_(o)
    else:
        dist.all_to_all_single(out, inp, out_splits, in_splits, group=group)
    return out


def exchange_points(ctx, rows, gid_base: int, d: int, eps: float, plan: ShardPlan, group=None):
    """Step 4: route this rank's rows (global ids gid_base + i) to every rank that needs
    them and receive this rank's bins + halo.  Returns (coords (n_local, d_pad) f64,
    gid int32 [n_local], n_local); rows come in global id order (sources are ordered
    by id range, each source's rows stay in order)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    n_my, width = rows.shape[0], rows.shape[1]
    pdims = plan.pdims
    dev = rows.device
    # one counting pass over the rows for every destination, then the stable writes
    counts = ctx.shard_route(rows, n_my, d, pdims, eps, plan.origin, plan.span, plan.ranges)
    total = sum(counts)
    send = torch.empty((max(total, 1), width), dtype=torch.float64, device=dev)
    send_gid = torch.empty(max(total, 1), dtype=torch.int32, device=dev)
    if total:
        ctx.shard_route(rows, n_my, d, pdims, eps, plan.origin, plan.span, plan.ranges,
                        counts=counts, out=send, gid=send_gid, gid_base=gid_base)
    cdev = dev if dist.get_backend(group) != "gloo" else torch.device("cpu")
    sc = torch.tensor(counts, dtype=torch.int64, device=cdev)
    rc = torch.empty_like(sc)
    dist.all_to_all_single(rc, sc, group=group)
    recv_counts = [int(v) for v in rc.cpu().tolist()]
    n_local = sum(recv_counts)
    local = torch.empty((max(n_local, 1), width), dtype=torch.float64, device=dev)
    gid = torch.empty(max(n_local, 1), dtype=torch.int32, device=dev)
    _a2a(local[:n_local], send[:total], recv_counts, counts, group)
    _a2a(gid[:n_local], send_gid[:total], recv_counts, counts, group)
    return local, gid, n_local


def gather_rows(rows, n: int, group=None):
    """All-gather the ranks' row slices into the full (n, d_pad) coordinates (NCCL)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    per = -(-n // world)
    width = rows.shape[1]
    if dist.get_backend(group) == "gloo":
        parts = [torch.empty((per, width), dtype=rows.dtype) for _ in range(world)]
        mine = torch.zeros((per, width), dtype=rows.dtype)
        mine[: rows.shape[0]] = rows.cpu()
        dist.all_gather(parts, mine, group=group)
        return torch.cat(parts)[:n].to(rows.device)
    mine = rows
    if rows.shape[0] != per:
        mine = torch.zeros((per, width), dtype=rows.dtype, device=rows.device)
        mine[: rows.shape[0]] = rows
    full = torch.empty((per * world, width), dtype=rows.dtype, device=rows.device)
    dist.all_gather_into_tensor(full, mine.contiguous(), group=group)
    return full[:n]


def row_slice(n: int, rank: int, world: int) -> tuple[int, int]:
    """This rank's slice of the input rows (equal ceil(n/world) slices, the last shorter)."""
    per = -(-n // world)
    return min(n, rank * per), min(n, (rank + 1) * per)


def exchange_counts(ctx, loff, n_local: int, gid, n: int, dev, group=None, stream=None):
    """Global per-id row counts: every rank scatters its rows' lengths to their
    global ids and the ranks SUM-all-reduce the n counts (each id is owned by one
    rank).  One byte per id while every row is shorter than 256 (a 4-byte MAX
    all-reduce of the overflow flag decides), else int32.

    stream: run the counts' all-reduce there (NCCL), so it overlaps whatever the
    caller enqueues next on its own stream; the caller waits on `stream` before
    reading the counts."""
    import torch
    import torch.distributed as dist

    gloo = dist.get_backend(group) == "gloo"

    def reduce(t, op):
        if gloo:  # gloo reduces host tensors
            c = t.cpu()
            _all_reduce(c, op, group)
            return c.to(dev)
        _all_reduce(t, op, group)
        return t

    c8 = torch.zeros(n, dtype=torch.uint8, device=dev)
    ovf = torch.zeros(1, dtype=torch.int32, device=dev)
    if n_local:
        ctx.scatter_counts(loff, n_local, gid, c8, ovf)
    if int(reduce(ovf, dist.ReduceOp.MAX).item()):
        del c8
        c8 = torch.zeros(n, dtype=torch.int32, device=dev)
        if n_local:
            ctx.scatter_counts(loff, n_local, gid, c8)
    if stream is None:
        return reduce(c8, dist.ReduceOp.SUM)
    stream.wait_stream(torch.cuda.current_stream(dev))
    with torch.cuda.stream(stream):
        c8 = reduce(c8, dist.ReduceOp.SUM)
    c8.record_stream(stream)  # used on both streams (gloo returns a copy made on `stream`)
    c8.record_stream(torch.cuda.current_stream(dev))
    return c8


_SIDE_STREAMS: dict = {}


def _side_stream(dev):
    """One high-priority side stream per device for the collectives that overlap
    the emit (its NCCL kernels get SM slots before the emit's persistent CTAs)."""
    import torch

    if dev.index not in _SIDE_STREAMS:
        _SIDE_STREAMS[dev.index] = torch.cuda.Stream(device=dev, priority=-1)
    return _SIDE_STREAMS[dev.index]


def strong_self_join(rows, n: int, d: int, config, group=None, timer=None) -> ShardResult:
    """The strong layout's join step over the process group (steps 2-6 above).

    rows: this rank's slice of the input (device tensor, (len, d_pad) f64, rows
    row_slice(n, rank, world) -- the id order the exchange relies on).  `timer(name)` (optional) is called at phase
    boundaries (the bench records CUDA events there).
    """
    import torch
    import torch.distributed as dist

    from .join import DeviceJoin, resolve_k_idx

    mark = timer or (lambda name: None)
    rank = dist.get_rank(group)
    eps = float(config.epsilon)
    dev = rows.device
    work_shape = Dataset._wrap(np.empty((1, rows.shape[1])), d)
    k_idx = resolve_k_idx(config, d)
    pdims = prefix_dims(d, k_idx)
    from . import _native

    ctx = _native.context(dev.index)
    plan = plan_shards(ctx, rows, eps, pdims, group)
    mark("plan")
    a, _ = row_slice(n, rank, dist.get_world_size(group))
    local, gid, n_local = exchange_points(ctx, rows, a, d, eps, plan, group)
    mark("exchange")
    lo, hi = plan.owned(rank)
    work = Dataset._wrap(np.empty((max(n_local, 1), rows.shape[1])), d) if n_local else work_shape
    job = DeviceJoin(work, config, device=dev.index)
    pairs = 0
    if n_local:
        job.build(local[:n_local])
        cb, ce = ctx.shard_cell_range(pdims, plan.origin, plan.span, lo, hi)
        mark("index")
        pairs = job.refine(cell_range=(cb, ce))
        mark("refine")
        ctx.set_output_ids(gid)  # rows carry global neighbour ids (gid is monotone)
        # local row offsets first: the global counts they give are all-reduced on a
        # side stream while this rank's rows are emitted
        loff = torch.empty(n_local + 1, dtype=torch.int64, device=dev)
        lnbr = torch.empty(max(pairs, 1), dtype=torch.int32, device=dev)
        job.offsets_d, job.neighbors_d = loff, lnbr
        ctx.finalize_offsets(loff)
        side = _side_stream(dev)
        counts = exchange_counts(ctx, loff, n_local, gid, n, dev, group, stream=side)
        ctx.finalize_rows(loff, lnbr)
        torch.cuda.current_stream(dev).wait_stream(side)
    else:
        cb = ce = 0
        loff = torch.zeros(1, dtype=torch.int64, device=dev)
        lnbr = torch.empty(1, dtype=torch.int32, device=dev)
        mark("index")
        mark("refine")
        counts = exchange_counts(ctx, loff, n_local, gid, n, dev, group)
    goff = torch.empty(n + 1, dtype=torch.int64, device=dev)
    ctx.counts_to_offsets(counts, n, goff)
    mark("offsets")
    total = int(goff[-1].item())
    return ShardResult(plan, rank, n, n_local, gid[:n_local], loff, lnbr[:pairs], goff, pairs,
                       total, (cb, ce), job)


# ------------------------------------------------------------------ host CSR
class SharedHostCSR:
    """A neighbour array in one /dev/shm segment shared by every rank on the node,
    page-locked and mapped into each rank's device address space, so every rank
    writes its rows straight to their final places over its own PCIe link."""

    def __init__(self, total: int, group=None, root: int = 0):
        import torch.distributed as dist

        from . import _native

        self.bytes = max(int(total), 1) * 4
        name = [f"/dev/shm/tedjoin-{uuid.uuid4().hex}" if dist.get_rank(group) == root else None]
        dist.broadcast_object_list(name, src=dist.get_global_rank(group, root) if group else root,
                                   group=group)
        self.path = name[0]
        if dist.get_rank(group) == root:
            with open(self.path, "wb") as fh:
                fh.truncate(self.bytes)
        dist.barrier(group=group)
        self._fd = os.open(self.path, os.O_RDWR)
        self._map = mmap.mmap(self._fd, self.bytes)
        self.array = np.frombuffer(self._map, dtype=np.uint32)
        self.host_ptr = self.array.ctypes.data
        self.device_ptr = _native.host_register(self.host_ptr, self.bytes, mapped=True)
        self._root = dist.get_rank(group) == root

    def close(self):
        from . import _native

        if self._map is None:
            return
        try:
            _native.host_unregister(self.host_ptr)
        finally:
            self.array = None
            self._map.close()
            os.close(self._fd)
            self._map = None
            if self._root:
                try:
                    os.unlink(self.path)
                except FileNotFoundError:
                    pass


def assemble_host_csr(shard: ShardResult, shared: SharedHostCSR | None = None, group=None,
                      root: int = 0):
    """Every rank places its rows in the shared host CSR; returns (offsets, neighbors)
    numpy arrays on `root` (None elsewhere).  Pass a SharedHostCSR of at least
    shard.total_pairs entries to reuse its page-locked mapping across joins."""
    import torch
    import torch.distributed as dist

    from . import _native

    own = shared is None
    if own:
        shared = SharedHostCSR(shard.total_pairs, group=group, root=root)
    ctx = _native.context(shard.global_offsets.device.index)
    if shard.pairs:
        ctx.place_rows(shard.offsets, shard.neighbors, shard.n_local, shard.gid,
                       shard.global_offsets, shared.device_ptr)
    off = shard.global_offsets.cpu().numpy() if dist.get_rank(group) == root else None
    torch.cuda.synchronize(shard.global_offsets.device)
    dist.barrier(group=group)
    out = None
    if dist.get_rank(group) == root:
        out = (off, np.array(shared.array[: shard.total_pairs]).view(np.int32))
    dist.barrier(group=group)
    if own:
        shared.close()
    return out


def broadcast_dataset(ds: Dataset | None, root: int = 0, group=None, device=None) -> tuple:
    """Replicate the (n, d_padded) coordinates from `root` to every rank (one broadcast).

    Returns (Dataset on host or None, coords tensor on `device`, d).
    """
    import torch
    import torch.distributed as dist

    rank = dist.get_rank(group)
    dev = torch.device("cpu") if device is None else torch.device(device)
    hdr = torch.zeros(3, dtype=torch.int64, device=dev)
    if rank == root:
        hdr[0], hdr[1], hdr[2] = ds.n, ds.d, ds.d_padded
    dist.broadcast(hdr, src=root, group=group)
    n, d, dp = (int(v) for v in hdr.tolist())
    if rank == root:
        coords = torch.from_numpy(ds.coords).to(dev)
    else:
        coords = torch.empty((n, dp), dtype=torch.float64, device=dev)
    dist.broadcast(coords, src=root, group=group)
    host = ds if rank == root else None
    if host is None and dev.type == "cpu":
        host = Dataset._wrap(coords.numpy(), d)
    return host, coords, d


def shard_self_join(ds: Dataset | None, config, root: int = 0, group=None):
    """Library entry point: rank `root` holds the dataset.  Each rank takes its row
    slice (one scatter), runs `strong_self_join`, and the pair set is assembled in
    a shared host CSR.  Returns (ShardResult, (offsets, neighbors) on root / None)."""
    import torch
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    device = torch.cuda.current_device()
    _, coords, d = broadcast_dataset(ds, root=root, group=group, device=f"cuda:{device}")
    n = coords.shape[0]
    a, b = row_slice(n, rank, world)
    shard = strong_self_join(coords[a:b], n, d, config, group=group)
    return shard, assemble_host_csr(shard, group=group, root=root)


def gather_csr(offsets: np.ndarray, neighbors: np.ndarray, root: int = 0, group=None):
    """Host (gloo) combine of per-rank CSR shards with disjoint non-empty rows on root.

    Every rank passes its full-length offsets (n+1; rows it does not own are
    empty) and its neighbour ids.  Returns (offsets, neighbors) on root, None elsewhere.
    """
    import torch
    import torch.distributed as dist

    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    counts = torch.from_numpy(np.diff(np.asarray(offsets, dtype=np.int64)))
    total_counts = counts.clone()
    dist.all_reduce(total_counts, op=dist.ReduceOp.SUM, group=group)
    sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(sizes, torch.tensor([len(neighbors)], dtype=torch.int64), group=group)
    max_size = max(int(s.item()) for s in sizes)
    mine = torch.zeros(max(max_size, 1), dtype=torch.int64)
    mine[: len(neighbors)] = torch.from_numpy(np.asarray(neighbors, dtype=np.int64))
    all_counts = [torch.zeros_like(counts) for _ in range(world)] if rank == root else None
    all_nbrs = [torch.zeros_like(mine) for _ in range(world)] if rank == root else None
    dist.gather(counts, all_counts, dst=root, group=group)
    dist.gather(mine, all_nbrs, dst=root, group=group)
    if rank != root:
        return None
    tc = total_counts.numpy()
    goff = np.zeros(len(tc) + 1, dtype=np.int64)
    np.cumsum(tc, out=goff[1:])
    out = np.empty(int(goff[-1]), dtype=np.int64)
    for r in range(world):
        c = all_counts[r].numpy()
        rows = np.flatnonzero(c)
        if rows.size == 0:
            continue
        seg = c[rows]
        m = int(seg.sum())
        starts = np.repeat(goff[rows], seg)
        within = np.arange(m, dtype=np.int64) - np.repeat(np.cumsum(seg) - seg, seg)
        out[starts + within] = all_nbrs[r].numpy()[:m]
    return goff, out
