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
