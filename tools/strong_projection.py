"""Per-rank device time of the strong multi-GPU layout, measured on ONE GPU.

    python tools/strong_projection.py [config] [G ...]

For G ranks, every rank's step (distributed.strong_self_join without the
collectives: routing of its row slice, local grid over its bins + halo, refine
of the owned cells, canonical rows, id remap, count scatter, global offsets) is
run in turn on this device with CUDA
events; the step time of G GPUs is the slowest rank plus the collectives,
estimated from their byte counts at a stated NVLink bus bandwidth.  Efficiency
= T_1 / (G * T_G).  This is a projection (one GPU measures each rank's share);
the collectives are not measured here.
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np
import torch

from bench import CONFIGS
from paper_2209_11287_b200 import GenSpec, JoinConfig, _native, generate
from paper_2209_11287_b200.datasets import Dataset
from paper_2209_11287_b200.distributed import plan_bins, prefix_dims
from paper_2209_11287_b200.join import DeviceJoin

NVLINK_BUS_GBS = 500.0  # assumed NCCL bus bandwidth per GPU (B200 NVLink 5: 900 GB/s per direction)

name = sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].isdigit() else "c5"
Gs = [int(a) for a in sys.argv[1:] if a.isdigit()] or [1, 2, 4, 8]
dist, n, d, eps = CONFIGS[name]
ds = generate(GenSpec(dist, n, d, seed=0))
dev = "cuda:0"
coords = torch.from_numpy(ds.coords).to(dev)
cfg = JoinConfig(epsilon=eps)
ctx = _native.context(0)
pdims = prefix_dims(d, min(d, 6))


def ev():
    e = torch.cuda.Event(enable_timing=True)
    e.record()
    return e


def full_join():
    t = [ev()]
    job = DeviceJoin(ds, cfg)
    job.build(coords)
    t.append(ev())
    job.refine()
    t.append(ev())
    job.finalize()
    t.append(ev())
    torch.cuda.synchronize()
    del job
    return [t[i].elapsed_time(t[i + 1]) for i in range(3)]


for _ in range(2):
    full_join()
T1 = float(np.median([sum(full_join()) for _ in range(3)]))
lo, hi = ctx.shard_bounds(coords, n, pdims, eps)
origin = lo
span = (int(hi[0] - lo[0] + 1), int(hi[1] - lo[1] + 1) if pdims > 1 else 1)
hist = torch.zeros(span[0] * span[1], dtype=torch.int64, device=dev)
ctx.shard_histogram(coords, n, pdims, eps, origin, span, hist)
h = hist.cpu().numpy()


def rank_step(plan, r, G):
    lo_b, hi_b = plan.owned(r)
    # exchange, this rank's side: route its own row slice to every rank (G selects);
    # the all-to-all itself is estimated from the bytes received
    per = -(-n // G)
    sl = coords[r * per: min(n, (r + 1) * per)]
    t = [ev()]
    cnts = ctx.shard_route(sl, sl.shape[0], d, pdims, eps, plan.origin, plan.span, plan.ranges)
    send = torch.empty((max(sum(cnts), 1), coords.shape[1]), dtype=torch.float64, device=dev)
    sgid = torch.empty(max(sum(cnts), 1), dtype=torch.int32, device=dev)
    ctx.shard_route(sl, sl.shape[0], d, pdims, eps, plan.origin, plan.span, plan.ranges,
                    counts=cnts, out=send, gid=sgid, gid_base=r * per)
    t.append(ev())
    # what this rank receives (the same set, in global id order)
    n_local = ctx.shard_select(coords, n, d, pdims, eps, plan.origin, plan.span, lo_b, hi_b)
    local = torch.empty((max(n_local, 1), coords.shape[1]), dtype=torch.float64, device=dev)
    gid = torch.empty(max(n_local, 1), dtype=torch.int32, device=dev)
    ctx.shard_select(coords, n, d, pdims, eps, plan.origin, plan.span, lo_b, hi_b, out=local, gid=gid)
    torch.cuda.synchronize()
    t.append(ev())
    job = DeviceJoin(Dataset._wrap(np.empty((n_local, coords.shape[1])), d), cfg)
    job.build(local[:n_local])
    cb, ce = ctx.shard_cell_range(pdims, plan.origin, plan.span, lo_b, hi_b)
    t.append(ev())
    pairs = job.refine(cell_range=(cb, ce))
    t.append(ev())
    ctx.set_output_ids(gid)
    # distributed.strong_self_join: local offsets, the count scatter (its all-reduce
    # runs on a side stream while the rows are emitted), the rows, global offsets
    loff = torch.empty(n_local + 1, dtype=torch.int64, device=dev)
    lnbr = torch.empty(max(pairs, 1), dtype=torch.int32, device=dev)
    ctx.finalize_offsets(loff)
    counts = torch.zeros(n, dtype=torch.uint8, device=dev)  # distributed.exchange_counts
    ovf = torch.zeros(1, dtype=torch.int32, device=dev)
    ctx.scatter_counts(loff, n_local, gid, counts, ovf)
    if int(ovf.item()):
        counts = torch.zeros(n, dtype=torch.int32, device=dev)
        ctx.scatter_counts(loff, n_local, gid, counts)
    te = ev()
    ctx.finalize_rows(loff, lnbr)
    te2 = ev()
    goff = torch.empty(n + 1, dtype=torch.int64, device=dev)
    ctx.counts_to_offsets(counts, n, goff)
    t.append(ev())
    torch.cuda.synchronize()
    ph = [t[i].elapsed_time(t[i + 1]) for i in range(5)]
    return {"rank": r, "n_local": n_local, "pairs": pairs, "emit_ms": te.elapsed_time(te2),
            "route_ms": ph[0], "index_ms": ph[2],
            "refine_ms": ph[3], "output_ms": ph[4], "step_ms": ph[0] + ph[2] + ph[3] + ph[4],
            "recv_bytes": n_local * (coords.shape[1] * 8 + 4), "count_bytes": counts.element_size()}


out = {"config": name, "n": n, "d": d, "T1_ms": T1, "nvlink_bus_gbs_assumed": NVLINK_BUS_GBS,
       "projection": []}
for G in Gs:
    if G == 1:
        continue
    plan = plan_bins(h, pdims, origin, span, G)
    ranks = [rank_step(plan, r, G) for r in range(G)]  # first pass: warm allocator
    # per rank, the median step of three measured passes (host jitter in the
    # read-backs inside the phases moves single samples by ~0.1 ms)
    passes = [[rank_step(plan, r, G) for r in range(G)] for _ in range(3)]
    ranks = [sorted((p[r] for p in passes), key=lambda x: x["step_ms"])[1] for r in range(G)]
    worst = max(ranks, key=lambda x: x["step_ms"])
    coll_bytes = {"all_to_all_points": (G - 1) / G * worst["recv_bytes"],
                  "all_reduce_counts": 2 * (G - 1) / G * n * max(x["count_bytes"] for x in ranks)}
    coll = {k: b / (NVLINK_BUS_GBS * 1e9) * 1e3 for k, b in coll_bytes.items()}
    # the counts' all-reduce runs on a side stream during the row emission
    # (distributed.strong_self_join): only what outlasts the emit adds to the step
    hidden = min(coll["all_reduce_counts"], min(x["emit_ms"] for x in ranks))
    coll_ms = sum(coll.values()) - hidden
    TG = worst["step_ms"] + coll_ms
    TG_serial = worst["step_ms"] + sum(coll.values())
    row = {"G": G, "slowest_rank": worst, "mean_rank_ms": float(np.mean([x["step_ms"] for x in ranks])),
           "collectives_ms_est": coll, "collectives_overlapped_ms": hidden, "T_G_ms": TG,
           "efficiency": T1 / (G * TG), "efficiency_serial_collectives": T1 / (G * TG_serial),
           "efficiency_device_only": T1 / (G * worst["step_ms"]),
           "pairs_total": int(sum(x["pairs"] for x in ranks))}
    out["projection"].append(row)
    print(json.dumps(row), flush=True)
print(json.dumps(out))
