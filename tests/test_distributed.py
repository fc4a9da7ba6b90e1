"""CPU, world_size 2 over gloo: the multi-GPU host path (dataset broadcast, cost-balanced
cell split, CSR gather).  The per-rank refine is the oracle restricted to the
rank's cells here; on GPUs it is tj_refine over the same cell range."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle
from paper_2209_11287_b200.datasets import GenSpec, generate


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, eps, out_q):
    import torch.distributed as dist

    from paper_2209_11287_b200.distributed import (
        balanced_cell_ranges,
        broadcast_dataset,
        gather_csr,
    )

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ds = generate(GenSpec("exponential", 3000, 3, seed=9)) if rank == 0 else None
        host, coords, d = broadcast_dataset(ds, root=0)
        assert host.n == 3000 and d == 3
        order, cstart, ccoord, cand = oracle.grid(host, eps)
        costs = np.diff(cstart) * cand
        lo, hi = balanced_cell_ranges(costs, world)[rank]
        off, nb = oracle.join_csr(host, eps, cells=np.arange(lo, hi))
        merged = gather_csr(off, nb, root=0)
        if rank == 0:
            out_q.put((merged[0], merged[1], host.checksum(), [int(costs[lo:hi].sum())]))
        else:
            out_q.put((None, None, host.checksum(), [int(costs[lo:hi].sum())]))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_join_equals_single_process():
    world, eps = 2, 0.02
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, eps, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ds = generate(GenSpec("exponential", 3000, 3, seed=9))
    full_off, full_nb = oracle.join_csr(ds, eps)
    merged = [r for r in results if r[0] is not None][0]
    assert all(r[2] == ds.checksum() for r in results)  # broadcast delivered the same bytes
    assert np.array_equal(merged[0], full_off)
    assert np.array_equal(merged[1], full_nb.astype(np.int64))
    shares = [r[3][0] for r in results]
    assert min(shares) > 0


def _strong_worker(rank, world, port, eps, shm_path, out_q):
    """The strong layout's host logic with numpy/oracle standing in for the CUDA kernels
    (shard.cu restated in distributed.point_bins / halo_mask): row slices, all-reduced
    bounds + bin histogram, equal-cost bin ranges, all-gather, halo select, the owned
    cells' rows, global offsets from all-reduced counts, rows placed in one shared
    host segment at their global offsets."""
    import torch
    import torch.distributed as dist

    from paper_2209_11287_b200.distributed import (
        halo_mask,
        plan_bins,
        point_bins,
        row_slice,
    )

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ds = generate(GenSpec("exponential", 6000, 3, seed=11))  # every rank reads its slice
        n, pdims = ds.n, 2
        a, b = row_slice(n, rank, world)
        rows = ds.coords[a:b]
        c = np.floor(rows[:, :pdims] / eps).astype(np.int64)
        bounds = torch.tensor(np.concatenate([c.min(0), -c.max(0)]))
        dist.all_reduce(bounds, op=dist.ReduceOp.MIN)
        origin = bounds[:pdims].numpy()
        span = -bounds[pdims:].numpy() - origin + 1
        b0, b1 = point_bins(rows, eps, pdims, origin)
        hist = torch.from_numpy(np.bincount(b0 * span[1] + b1, minlength=int(span[0] * span[1])))
        dist.all_reduce(hist, op=dist.ReduceOp.SUM)
        plan = plan_bins(hist.numpy(), pdims, origin, span, world)
        lo, hi = plan.owned(rank)
        # route this rank's rows to every rank needing them, one all-to-all
        rb0, rb1 = point_bins(rows, eps, pdims, origin)
        sends, send_gids, counts = [], [], []
        for (olo, ohi) in plan.ranges:
            m = halo_mask(rb0, rb1, span, pdims, olo, ohi)
            sends.append(rows[m])
            send_gids.append(a + np.flatnonzero(m))
            counts.append(int(m.sum()))
        rc = torch.empty(world, dtype=torch.int64)
        dist.all_to_all_single(rc, torch.tensor(counts, dtype=torch.int64))
        rcounts = rc.tolist()
        recv = torch.empty((sum(rcounts), rows.shape[1]), dtype=torch.float64)
        dist.all_to_all_single(recv, torch.from_numpy(np.concatenate(sends)), rcounts, counts)
        rgid = torch.empty(sum(rcounts), dtype=torch.int64)
        dist.all_to_all_single(rgid, torch.from_numpy(np.concatenate(send_gids)), rcounts, counts)
        gid = rgid.numpy()
        assert np.all(np.diff(gid) > 0)  # global id order: local ids monotone in global ids
        local = np.ascontiguousarray(recv.numpy())
        _, cstart, ccoord, _ = oracle.grid(local, eps)
        cell_bin = (ccoord[:, 0] - origin[0]) * span[1] + (ccoord[:, 1] - origin[1])
        owned = np.flatnonzero((cell_bin >= lo) & (cell_bin <= hi))
        assert np.all(np.diff(owned) == 1) or len(owned) <= 1  # one contiguous cell range
        loff, lnb = oracle.join_csr(local, eps, cells=owned)
        gnb = gid[lnb.astype(np.int64)]
        # global offsets as distributed.exchange_counts: one byte per id unless a
        # row reaches 256 ids on some rank (MAX all-reduce of the flag), else int32
        lens = np.diff(loff)
        ovf = torch.tensor([int(np.any(lens > 255))], dtype=torch.int32)
        dist.all_reduce(ovf, op=dist.ReduceOp.MAX)
        counts = torch.zeros(n, dtype=torch.uint8 if int(ovf) == 0 else torch.int32)
        counts[gid] = torch.from_numpy(np.minimum(lens, 255) if int(ovf) == 0 else lens).to(counts.dtype)
        dist.all_reduce(counts, op=dist.ReduceOp.SUM)
        goff = np.concatenate([[0], np.cumsum(counts.numpy().astype(np.int64))])
        if rank == 0:
            np.zeros(int(goff[-1]), np.int64).tofile(shm_path)
        dist.barrier()
        out = np.memmap(shm_path, dtype=np.int64, mode="r+", shape=(int(goff[-1]),))
        for l in np.flatnonzero(np.diff(loff)):  # rows straight to their global places
            out[goff[gid[l]]: goff[gid[l] + 1]] = gnb[loff[l]: loff[l + 1]]
        out.flush()
        dist.barrier()
        share = int(plan.cost_share()[rank])
        out_q.put((rank, goff if rank == 0 else None,
                   np.array(out) if rank == 0 else None, share, len(local), len(rows)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_strong_layout_gloo_equals_single_process(world, tmp_path):
    eps = 0.02
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    shm = str(tmp_path / "csr.bin")
    procs = [ctx.Process(target=_strong_worker, args=(r, world, port, eps, shm, q))
             for r in range(world)]
    for p in procs:
        p.start()
    results = sorted([q.get(timeout=180) for _ in range(world)], key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ds = generate(GenSpec("exponential", 6000, 3, seed=11))
    full_off, full_nb = oracle.join_csr(ds, eps)
    assert np.array_equal(results[0][1], full_off)
    assert np.array_equal(results[0][2], full_nb.astype(np.int64))
    shares = [r[3] for r in results]
    assert min(shares) > 0  # every rank owns work (skewed 6000 points: coarse bins)
    assert sum(r[4] for r in results) < world * ds.n  # ranks hold bins + halo, not all of it


def test_plan_bins_balances_uniform_costs():
    """c5's shape: 44 x 44 bins of ~equal density over 8 ranks -> shares within 2%."""
    from paper_2209_11287_b200.distributed import plan_bins

    rng = np.random.default_rng(1)
    hist = rng.poisson(25_800, size=44 * 44)
    plan = plan_bins(hist, 2, (0, 0), (44, 44), 8)
    shares = np.array(plan.cost_share(), dtype=float)
    assert shares.min() > 0.98 * shares.mean() and shares.max() < 1.02 * shares.mean()
    lo = [r[0] for r in plan.ranges]
    hi = [r[1] for r in plan.ranges]
    assert lo[0] == 0 and hi[-1] == 44 * 44 - 1 and all(lo[i + 1] == hi[i] + 1 for i in range(7))


def test_halo_mask_matches_definition():
    """halo_mask (the numpy twin of shard.cu bin_needed) = 'some Chebyshev-1 neighbour
    bin is owned', checked by enumeration."""
    from paper_2209_11287_b200.distributed import halo_mask

    rng = np.random.default_rng(5)
    for pdims, span in ((2, (7, 5)), (1, (9, 1))):
        b0 = rng.integers(0, span[0], 400)
        b1 = rng.integers(0, span[1], 400)
        for lo, hi in ((0, 0), (3, 17), (12, 12), (20, span[0] * span[1] - 1), (5, 4)):
            got = halo_mask(b0, b1, span, pdims, lo, hi)
            for i in range(len(b0)):
                want = False
                for a in (-1, 0, 1):
                    for c in ((-1, 0, 1) if pdims > 1 else (0,)):
                        q0, q1 = b0[i] + a, b1[i] + c
                        if 0 <= q0 < span[0] and 0 <= q1 < span[1]:
                            want |= lo <= q0 * span[1] + q1 <= hi
                assert got[i] == want


def _gpu_worker(rank, world, port, case, kernel, out_q):
    """The real strong layout (strong_self_join: bin plan, all-gather, tj_shard_select,
    tj_refine of the owned cells, global offsets, rows placed in the shared mapped host
    CSR) with two ranks sharing cuda:0 over gloo (NCCL needs distinct GPUs)."""
    import torch
    import torch.distributed as dist

    from paper_2209_11287_b200 import JoinConfig
    from paper_2209_11287_b200.distributed import shard_self_join

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        dist_, n, d, eps = case
        ds = generate(GenSpec(dist_, n, d, seed=4)) if rank == 0 else None
        shard, merged = shard_self_join(ds, JoinConfig(epsilon=eps, kernel=kernel, device=0))
        info = (shard.pairs, shard.n_local, shard.total_pairs)
        if rank == 0:
            out_q.put((merged[0], merged[1], info))
        else:
            out_q.put((None, None, info))
    finally:
        dist.destroy_process_group()


# (uniform 4-D: one-byte count exchange; uniform 2-D at ~250 neighbours per point:
#  rows of 256+ ids force the int32 fallback of distributed.exchange_counts)
GPU_CASES = [("uniform", 40_000, 4, 0.06), ("uniform", 8_000, 2, 0.1)]


@pytest.mark.gpu
@pytest.mark.parametrize("case", GPU_CASES)
@pytest.mark.parametrize("kernel", ["tile", "scalar"])
def test_two_rank_shard_self_join_on_gpu(kernel, case):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gpu_worker, args=(r, world, port, case, kernel, q))
             for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    dist_, n, d, eps = case
    ds = generate(GenSpec(dist_, n, d, seed=4))
    full_off, full_nb = oracle.join_csr(ds, eps)
    if d == 2:
        assert np.diff(full_off).max() > 255  # the int32 count exchange runs
    merged = [r for r in results if r[0] is not None][0]
    assert np.array_equal(merged[0], full_off)
    assert np.array_equal(np.asarray(merged[1], np.int64), full_nb.astype(np.int64))
    infos = [r[2] for r in results]
    assert all(i[0] > 0 for i in infos) and sum(i[0] for i in infos) == int(full_off[-1])
    assert all(i[1] < ds.n for i in infos)  # each rank holds its bins + halo, not everything


def test_weak_scaling_partition_is_exact():
    """bench.py's weak-scaled partition: each rank's slab + one-cell halo holds every
    candidate of its owned cells, so its rows equal the global join's rows."""
    import sys

    sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parents[1]))
    from bench import weak_local_dataset

    n, d, eps, world = 4000, 3, 0.06, 3
    parts = [weak_local_dataset("uniform", n, d, eps, r, world) for r in range(world)]
    glob = np.concatenate([p[0].coords[: p[1]] for p in parts])  # slabs in rank order
    g_off, g_nb = oracle.join_csr(glob, eps)
    for r, (local, n_own, _) in enumerate(parts):
        l_off, l_nb = oracle.join_csr(local, eps)
        # local ids: own slab first (global ids r*n .. r*n+n_own), then halo points
        halo_gid = []
        if r > 0:
            lo_slab = parts[r - 1][0].coords[: n]
            halo_gid.append((r - 1) * n + np.flatnonzero(
                np.floor(lo_slab[:, 0] / eps) >= parts[r][2][0] - 1))
        if r < world - 1:
            hi_slab = parts[r + 1][0].coords[: n]
            halo_gid.append((r + 1) * n + np.flatnonzero(
                np.floor(hi_slab[:, 0] / eps) <= parts[r][2][1] + 1))
        gid = np.concatenate([r * n + np.arange(n_own)] + halo_gid)
        for i in range(0, n_own, 97):  # own rows, mapped to global ids
            mine = np.sort(gid[l_nb[l_off[i]:l_off[i + 1]]])
            want = g_nb[g_off[r * n + i]:g_off[r * n + i + 1]]
            assert np.array_equal(mine, want.astype(np.int64)), (r, i)
