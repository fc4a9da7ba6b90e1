"""One join of a synthetic workload, for ncu captures of a single refine launch.

    python tools/profile_join.py <dist> <n> <d> <eps> [tile|scalar] [--no-short-circuit] [--reps=K]

With --reps=K the refine is repeated K times and the median kernel time is
reported (the first launch of a process runs on cold clocks).
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch

from paper_2209_11287_b200 import GenSpec, JoinConfig, generate
from paper_2209_11287_b200.join import DeviceJoin

dist, n, d, eps = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), float(sys.argv[4])
kernel = sys.argv[5] if len(sys.argv) > 5 and not sys.argv[5].startswith("--") else "tile"
sc = "--no-short-circuit" not in sys.argv
ds = generate(GenSpec(dist, n, d, seed=0))
coords = torch.from_numpy(ds.coords).cuda()
job = DeviceJoin(ds, JoinConfig(epsilon=eps, kernel=kernel, short_circuit=sc, device=0))
info = job.build(coords)
reps = int(next((a.split("=")[1] for a in sys.argv if a.startswith("--reps=")), "1"))
times = []
for _ in range(reps):
    job.refine()
    times.append(job.ctx.last_refine_ms())
ms = sorted(times)[len(times) // 2]
st = job.ctx.stats()
C = int(info.candidates)
print(f"{dist} n={n} d={d} eps={eps} {kernel} sc={sc}: C={C:.4g} pairs={int(job.total)} "
      f"refine {ms:.3f} ms = {2 * d * C / ms / 1e9:.2f} TFLOP/s, tiles {st.tiles_processed} "
      f"skipped chunks {st.chunks_skipped}", flush=True)
