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


def _gpu_worker(rank, world, port, eps, kernel, out_q):
    """The real multi-GPU path (shard_self_join: broadcast, cost-balanced tj_refine,
    gather) with two ranks sharing cuda:0 over gloo (NCCL needs distinct GPUs)."""
    import torch
    import torch.distributed as dist

    from paper_2209_11287_b200 import JoinConfig
    from paper_2209_11287_b200.distributed import shard_self_join

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ds = generate(GenSpec("uniform", 40_000, 4, seed=4)) if rank == 0 else None
        (off, nb), merged, job = shard_self_join(ds, JoinConfig(epsilon=eps, kernel=kernel, device=0))
        own = int(job.total)
        if rank == 0:
            out_q.put((merged[0], merged[1], own))
        else:
            out_q.put((None, None, own))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("kernel", ["tile", "scalar"])
def test_two_rank_shard_self_join_on_gpu(kernel):
    world, eps = 2, 0.06
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gpu_worker, args=(r, world, port, eps, kernel, q))
             for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    ds = generate(GenSpec("uniform", 40_000, 4, seed=4))
    full_off, full_nb = oracle.join_csr(ds, eps)
    merged = [r for r in results if r[0] is not None][0]
    assert np.array_equal(merged[0], full_off)
    assert np.array_equal(np.asarray(merged[1], np.int64), full_nb.astype(np.int64))
    assert all(r[2] > 0 for r in results) and sum(r[2] for r in results) == int(full_off[-1])


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
