"""Run only the refine kernel of a workload (for ncu captures): grid built, pair
buffer sized generously, short_circuit off (the roofline setting), then
`reps` tj_refine launches over all cells.

    python tools/refine_only.py <config|n:d:eps> <kernel> [reps]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch

from bench import CONFIGS
from paper_2209_11287_b200 import GenSpec, JoinConfig, generate
from paper_2209_11287_b200.join import DeviceJoin

spec, kernel = sys.argv[1], sys.argv[2]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
if spec in CONFIGS:
    dist, n, d, eps = CONFIGS[spec]
else:
    n_, d_, e_ = spec.split(":")
    dist, n, d, eps = "uniform", int(n_), int(d_), float(e_)
ds = generate(GenSpec(dist, n, d, seed=0))
job = DeviceJoin(ds, JoinConfig(epsilon=eps, kernel=kernel, short_circuit=False))
info = job.build()
job.ctx.reset_results()
job.ctx.reserve_results(min(int(info.candidates), 400_000_000))
for r in range(reps):
    job.ctx.reset_results()
    job.ctx.refine(job.kernel, False, 0, info.n_cells)
    ms = job.ctx.last_refine_ms()
    total, over = job.ctx.result_count()
    print(f"{spec} {kernel}: refine {ms:.2f} ms, {2 * d * info.candidates / ms / 1e9:.2f} TFLOP/s, "
          f"pairs {total}{' (overflow)' if over else ''}", flush=True)
