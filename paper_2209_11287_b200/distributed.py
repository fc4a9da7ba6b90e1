"""Multi-GPU self-join: one process per GPU, cells sharded by estimated cost.

North-star layout: the dataset is replicated to every rank
with one broadcast (NCCL over NVLink on GPUs, gloo in the CPU tests), every
rank rebuilds the same deterministic grid, the lexicographic cell list is cut
into contiguous ranges of equal estimated cost (|cell| * |cand(cell)|, the
reference estimator join.py:122-124), each rank refines only its query cells
and emits canonical CSR rows for its own queries, and the rows are combined on
the devices (count all-reduce + one reduce of the disjoint rows) and copied to
the root host once.  There is no collective on the refine path itself.
`gather_csr` is the host-memory (gloo) variant used by the CPU tests.
"""

from __future__ import annotations

import numpy as np

from .datasets import Dataset


def balanced_cell_ranges(costs, parts: int) -> list[tuple[int, int]]:
    """Cut cells into `parts` contiguous ranges of ~equal total cost.

    Range r ends at the first cell whose inclusive prefix cost reaches
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


def broadcast_dataset(ds: Dataset | None, root: int = 0, group=None, device=None) -> tuple:
    """Replicate the (n, d_padded) coordinates from `root` to every rank.

    Returns (Dataset on host or None, coords tensor on `device`).  With the NCCL
    backend the tensor is a CUDA tensor and the broadcast runs over NVLink;
    with gloo it is a CPU tensor.
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


def gather_csr(offsets: np.ndarray, neighbors: np.ndarray, root: int = 0, group=None):
    """Combine per-rank CSR shards with disjoint non-empty rows into the global CSR on root.

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
        # destination of each shard element: row start in the global CSR + rank in the row
        starts = np.repeat(goff[rows], seg)
        within = np.arange(m, dtype=np.int64) - np.repeat(np.cumsum(seg) - seg, seg)
        out[starts + within] = all_nbrs[r].numpy()[:m]
    return goff, out


def gather_csr_device(offsets, neighbors, total: int, root: int = 0, group=None):
    """Device-side gather of per-rank CSR shards (disjoint non-empty rows) to `root`.

    offsets: device int64[n+1] of this rank's rows (rows it does not own are
    empty); neighbors: device int32[>= total].  The per-row counts are summed
    with one all-reduce (NCCL over NVLink on GPUs), every rank places its rows
    at their global offsets in a full-length buffer and one reduce(SUM) lands
    the union on `root`'s device (rows are disjoint, so the sum is the union).
    Returns (offsets, neighbors) device tensors on root, None elsewhere.
    """
    import torch
    import torch.distributed as dist

    rank = dist.get_rank(group)
    counts = offsets[1:] - offsets[:-1]
    gcounts = counts.clone()
    dist.all_reduce(gcounts, op=dist.ReduceOp.SUM, group=group)
    goff = torch.zeros_like(offsets)
    torch.cumsum(gcounts, 0, out=goff[1:])
    m = int(goff[-1].item())
    full = torch.zeros(max(m, 1), dtype=torch.int32, device=offsets.device)
    if total > 0:
        rows = torch.repeat_interleave(torch.arange(len(counts), device=offsets.device), counts)
        dest = goff[rows] + (torch.arange(total, device=offsets.device) - offsets[rows])
        full.index_copy_(0, dest, neighbors[:total])
    if dist.get_backend(group) == "gloo":  # gloo has no GPU reduce; all-reduce instead
        dist.all_reduce(full, op=dist.ReduceOp.SUM, group=group)
    else:
        dist.reduce(full, dst=root, op=dist.ReduceOp.SUM, group=group)
    return (goff, full[:m]) if rank == root else None


def shard_self_join(ds: Dataset | None, config, root: int = 0, group=None):
    """Distributed self-join over the current process group (one GPU per rank).

    Rank `root` holds the dataset; the coordinates are broadcast (NCCL over
    NVLink), every rank refines its cost-balanced cell range, the CSR shards are
    combined on the device (gather_csr_device) and only `root` copies the
    result to its host.  Returns (local device CSR, root host CSR or None, job).
    """
    import torch
    import torch.distributed as dist

    from .join import DeviceJoin

    device = torch.cuda.current_device()
    host, coords, d = broadcast_dataset(ds, root=root, group=group, device=f"cuda:{device}")
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    n = coords.shape[0]
    work = host if host is not None else Dataset._wrap(np.empty((n, coords.shape[1])), d)
    job = DeviceJoin(work, config, device=device)
    info = job.build(coords)
    costs = job.ctx.cell_costs(info.n_cells)
    lo, hi = balanced_cell_ranges(costs, world)[rank]
    job.refine(cell_range=(lo, hi))
    off_d, nbr_d = job.finalize()
    merged = gather_csr_device(off_d, nbr_d, job.total, root=root, group=group)
    host_csr = None
    if merged is not None:
        host_csr = (merged[0].cpu().numpy(), merged[1].cpu().numpy())
    return (off_d, nbr_d), host_csr, job


_host_groups: dict = {}


def _host_group(group=None):
    """A gloo group over the same ranks for host-memory gathers (NCCL moves only device tensors)."""
    import torch.distributed as dist

    if dist.get_backend(group) == "gloo":
        return group
    key = id(group)
    if key not in _host_groups:
        ranks = None if group is None else dist.get_process_group_ranks(group)
        _host_groups[key] = dist.new_group(ranks=ranks, backend="gloo")
    return _host_groups[key]
