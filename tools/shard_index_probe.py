"""Index phase of one strong-layout rank (c5, G ranks, rank r): the rank's
bins + halo are selected on the device, then DeviceJoin.build is timed alone
(CUDA events) and with the cell-range lookup, to separate the grid build from
host-side overhead.  Under ncu it gives the rank's per-kernel split.

    python tools/shard_index_probe.py [G] [rank] [reps]
"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np
import torch

from bench import CONFIGS
from paper_2209_11287_b200 import GenSpec, JoinConfig, _native, generate
from paper_2209_11287_b200.datasets import Dataset
from paper_2209_11287_b200.distributed import plan_bins, prefix_dims
from paper_2209_11287_b200.join import DeviceJoin

G = int(sys.argv[1]) if len(sys.argv) > 1 else 8
r = int(sys.argv[2]) if len(sys.argv) > 2 else G - 1
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
dist, n, d, eps = CONFIGS["c5"]
ds = generate(GenSpec(dist, n, d, seed=0))
dev = "cuda:0"
coords = torch.from_numpy(ds.coords).to(dev)
ctx = _native.context(0)
pdims = prefix_dims(d, min(d, 6))
lo, hi = ctx.shard_bounds(coords, n, pdims, eps)
span = (int(hi[0] - lo[0] + 1), int(hi[1] - lo[1] + 1) if pdims > 1 else 1)
hist = torch.zeros(span[0] * span[1], dtype=torch.int64, device=dev)
ctx.shard_histogram(coords, n, pdims, eps, lo, span, hist)
plan = plan_bins(hist.cpu().numpy(), pdims, lo, span, G)
lo_b, hi_b = plan.owned(r)
n_local = ctx.shard_select(coords, n, d, pdims, eps, plan.origin, plan.span, lo_b, hi_b)
local = torch.empty((n_local, coords.shape[1]), dtype=torch.float64, device=dev)
gid = torch.empty(n_local, dtype=torch.int32, device=dev)
ctx.shard_select(coords, n, d, pdims, eps, plan.origin, plan.span, lo_b, hi_b, out=local, gid=gid)
# the rank's routing of its own row slice (distributed.exchange_points, this side)
per = -(-n // G)
sl = coords[r * per: min(n, (r + 1) * per)]
rt = []
for i in range(6):
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e[0].record()
    cnts = ctx.shard_route(sl, sl.shape[0], d, pdims, eps, plan.origin, plan.span, plan.ranges)
    e[1].record()
    send = torch.empty((max(sum(cnts), 1), coords.shape[1]), dtype=torch.float64, device=dev)
    sgid = torch.empty(max(sum(cnts), 1), dtype=torch.int32, device=dev)
    ctx.shard_route(sl, sl.shape[0], d, pdims, eps, plan.origin, plan.span, plan.ranges,
                    counts=cnts, out=send, gid=sgid, gid_base=r * per)
    e[2].record()
    torch.cuda.synchronize()
    rt.append([e[0].elapsed_time(e[1]), e[1].elapsed_time(e[2])])
    del send, sgid
rm = np.median(np.array(rt[1:]), axis=0)
print(f"G={G} rank={r}: route count {rm[0]:.3f} ms, route write {rm[1]:.3f} ms", flush=True)
cfg = JoinConfig(epsilon=eps)
wrap = Dataset._wrap(np.empty((n_local, coords.shape[1])), d)
del coords, sl
torch.cuda.synchronize()
rows = []
for i in range(reps):
    e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    t0 = time.perf_counter()
    e[0].record()
    job = DeviceJoin(wrap, cfg)
    e[1].record()
    job.build(local)
    e[2].record()
    ctx.shard_cell_range(pdims, plan.origin, plan.span, lo_b, hi_b)
    e[3].record()
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    rows.append([e[0].elapsed_time(e[1]), e[1].elapsed_time(e[2]), e[2].elapsed_time(e[3]),
                 (t1 - t0) * 1e3])
    del job
m = np.median(np.array(rows[1:]), axis=0)
print(f"G={G} rank={r} n_local={n_local}: DeviceJoin() {m[0]:.3f} ms, build {m[1]:.3f} ms, "
      f"cell_range {m[2]:.3f} ms, host wall {m[3]:.3f} ms", flush=True)
