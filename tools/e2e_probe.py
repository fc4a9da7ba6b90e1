"""Break the public self_join() call of a bench workload into host/device phases.

python tools/e2e_probe.py c2 [reps]
"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch

from bench import CONFIGS
from paper_2209_11287_b200 import GenSpec, JoinConfig, generate
from paper_2209_11287_b200.datasets import reorder_dims_by_variance
from paper_2209_11287_b200.join import DeviceJoin, self_join

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
dist, n, d, eps = CONFIGS[name]
ds = generate(GenSpec(dist, n, d, seed=0))
cfg = JoinConfig(epsilon=eps)
keep = [self_join(ds, cfg) for _ in range(2)]
for r in range(reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    work, _ = reorder_dims_by_variance(ds)
    t1 = time.perf_counter()
    job = DeviceJoin(work, cfg)
    job.build()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    total = job.refine()
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    job.finalize()
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    off, nbr = job.fetch()
    t5 = time.perf_counter()
    keep = [keep[-1], (off, nbr)]
    t6 = time.perf_counter()
    res = self_join(ds, cfg)
    t7 = time.perf_counter()
    print(f"{name} rep {r}: reorder {1e3 * (t1 - t0):.1f} ms, upload+build {1e3 * (t2 - t1):.1f}, "
          f"refine {1e3 * (t3 - t2):.1f}, finalize {1e3 * (t4 - t3):.1f}, fetch {1e3 * (t5 - t4):.1f} "
          f"({(off.nbytes + nbr.nbytes) / (t5 - t4) / 1e9:.1f} GB/s) | self_join {1e3 * (t7 - t6):.1f} ms",
          flush=True)
