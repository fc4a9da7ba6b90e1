"""Time the grid build (index phase) alone: CUDA events around tj_build_grid on
resident coordinates, L2 flushed between repetitions.  Under
`ncu --metrics gpu__time_duration.sum` it gives the per-kernel split of one build.

    python tools/index_probe.py <config> [reps]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch

from bench import CONFIGS
from paper_2209_11287_b200 import GenSpec, JoinConfig, generate
from paper_2209_11287_b200.join import DeviceJoin

spec = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
dist, n, d, eps = CONFIGS[spec]
ds = generate(GenSpec(dist, n, d, seed=0))
job = DeviceJoin(ds, JoinConfig(epsilon=eps))
info = job.build()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream()
times = []
for r in range(reps):
    flush.fill_(r & 0xFF)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    job.ctx.build_grid(job.coords, n, d, int(job.coords.stride(0)), job.k_idx, eps)
    e1.record(s)
    torch.cuda.synchronize()
    times.append(e0.elapsed_time(e1))
info = job.ctx.grid_info()
times.sort()
print(f"{spec}: build_grid median {times[len(times) // 2]:.4f} ms min {times[0]:.4f} ms "
      f"(cells {info.n_cells}, runs {info.n_runs}, candidates {info.candidates})", flush=True)
