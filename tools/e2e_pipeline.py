"""Phases of the public self_join() call (host wall clock, synchronised per phase)
and the chunked result pipeline at several chunk counts.

    python tools/e2e_pipeline.py [config] [reps]
"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np
import torch

from bench import CONFIGS
from paper_2209_11287_b200 import GenSpec, JoinConfig, generate
from paper_2209_11287_b200.join import DeviceJoin, self_join, upload

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
dist, n, d, eps = CONFIGS[name]
ds = generate(GenSpec(dist, n, d, seed=0))
cfg = JoinConfig(epsilon=eps)
keep = [self_join(ds, cfg) for _ in range(2)]


def sync():
    torch.cuda.synchronize()
    return time.perf_counter()


for chunks, copies in ((1, None), (8, None), (16, None), (24, None), (32, None),
                       (32, (1, 2, 4, 8, 17))):
    rows = []
    for r in range(reps):
        t0 = sync()
        job = DeviceJoin(ds, cfg)
        coords = upload(ds, job.device)
        t1 = sync()
        job.build(coords)
        t2 = sync()
        job.refine()
        t3 = sync()
        off, nbr = job.finalize_fetch(chunks=chunks, copies=copies)
        t4 = sync()
        rows.append((t1 - t0, t2 - t1, t3 - t2, t4 - t3, t4 - t0))
    m = np.median(np.array(rows), axis=0) * 1e3
    print(f"{name} chunks={chunks:2d} copies={copies}: upload {m[0]:.2f} build {m[1]:.2f} refine {m[2]:.2f} "
          f"finalize+fetch {m[3]:.2f} | total {m[4]:.2f} ms", flush=True)
ts = []
for r in range(reps):
    t0 = sync()
    self_join(ds, cfg)
    ts.append(sync() - t0)
print(f"{name} self_join: {np.median(ts) * 1e3:.2f} ms (median of {reps})")
