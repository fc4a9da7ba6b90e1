"""Run a few self-joins of a bench workload (for ncu captures): python tools/run_join.py c2 tile [reps]"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch

from bench import CONFIGS
from paper_2209_11287_b200 import GenSpec, JoinConfig, generate
from paper_2209_11287_b200.join import DeviceJoin

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
kernel = sys.argv[2] if len(sys.argv) > 2 else "tile"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
dist, n, d, eps = CONFIGS[name]
ds = generate(GenSpec(dist, n, d, seed=0))
coords = torch.from_numpy(ds.coords).cuda()
for r in range(reps):
    job = DeviceJoin(ds, JoinConfig(epsilon=eps, kernel=kernel, device=0))
    t = time.perf_counter()
    info = job.build(coords)
    total = job.refine()
    job.finalize()
    torch.cuda.synchronize()
    print(f"{name} {kernel} rep {r}: {time.perf_counter() - t:.4f}s pairs={total} "
          f"refine_kernel={job.ctx.last_refine_ms():.3f}ms C={info.candidates}", flush=True)
