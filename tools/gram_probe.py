"""A reduced brute-force workload for profiling the Gram DMMA kernel under ncu.

    python tools/gram_probe.py [n] [d] [reps]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch

from paper_2209_11287_b200 import GenSpec, JoinConfig, generate
from paper_2209_11287_b200.join import DeviceJoin

n = int(sys.argv[1]) if len(sys.argv) > 1 else 400_000
d = int(sys.argv[2]) if len(sys.argv) > 2 else 16
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
eps = {16: 0.657508, 32: 1.31923, 64: 2.27218}.get(d, 0.2 * d ** 0.5)
ds = generate(GenSpec("uniform", n, d, seed=0))
coords = torch.from_numpy(ds.coords).cuda()
for r in range(reps):
    job = DeviceJoin(ds, JoinConfig(epsilon=eps, short_circuit=False))
    info = job.build(coords)
    job.refine()
    ms = job.ctx.last_refine_ms()
    print(f"n={n} d={d} cells={info.n_cells} C={info.candidates} refine {ms:.1f} ms "
          f"{2 * d * info.candidates / ms / 1e9:.2f} TFLOP/s", flush=True)
