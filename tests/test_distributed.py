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
