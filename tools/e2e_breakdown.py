"""Phase timing of the public self_join path (host buffers in, CSR out): python tools/e2e_breakdown.py c2"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch

from bench import CONFIGS
from paper_2209_11287_b200 import GenSpec, JoinConfig, generate
from paper_2209_11287_b200.join import DeviceJoin, upload

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
dist, n, d, eps = CONFIGS[name]
ds = generate(GenSpec(dist, n, d, seed=0))
cfg = JoinConfig(epsilon=eps, device=0)
for rep in range(4):
    t = [time.perf_counter()]
    job = DeviceJoin(ds, cfg)
    coords = upload(ds, 0)
    torch.cuda.synchronize()
    t.append(time.perf_counter())
    job.build(coords)
    t.append(time.perf_counter())
    job.refine()
    t.append(time.perf_counter())
    job.finalize()
    torch.cuda.synchronize()
    t.append(time.perf_counter())
    off, nbr = job.fetch()
    t.append(time.perf_counter())
    st = job.stats()
    t.append(time.perf_counter())
    names = ["upload", "build", "refine", "finalize", "fetch", "stats"]
    print(f"rep {rep}: " + " ".join(f"{k}={1e3 * (b - a):.2f}ms" for k, a, b in zip(names, t, t[1:]))
          + f" total={1e3 * (t[-1] - t[0]):.2f}ms pairs={job.total}", flush=True)
