"""Per-config device timings for both kernels (BASELINE configs 1-5, the d sweep).

    python tools/sweep.py [c1 c2 ...] [--reps 3] [--no-short-circuit]

One JSON line per (config, kernel): index / refine / finalize ms (CUDA events,
inputs resident in HBM, median of reps), refine kernel ms, FP64 distance
TFLOP/s (2*d*C / refine kernel time) and the step-level rate.
"""
import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np
import torch

from bench import CONFIGS
from paper_2209_11287_b200 import GenSpec, JoinConfig, generate
from paper_2209_11287_b200.join import DeviceJoin


def run(name, kernel, reps, sc):
    dist, n, d, eps = CONFIGS[name]
    ds = generate(GenSpec(dist, n, d, seed=0))
    coords = torch.from_numpy(ds.coords).cuda()
    cfg = JoinConfig(epsilon=eps, kernel=kernel, short_circuit=sc, device=0)
    rows = []
    for _ in range(reps + 1):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        ev[0].record()
        job = DeviceJoin(ds, cfg)
        info = job.build(coords)
        ev[1].record()
        job.refine()
        rk = job.ctx.last_refine_ms()
        ev[2].record()
        job.finalize()
        ev[3].record()
        torch.cuda.synchronize()
        st = job.ctx.stats()
        rows.append({"index_ms": ev[0].elapsed_time(ev[1]), "refine_ms": ev[1].elapsed_time(ev[2]),
                     "refine_kernel_ms": rk, "finalize_ms": ev[2].elapsed_time(ev[3]),
                     "step_ms": ev[0].elapsed_time(ev[3])})
        del job
    rows = rows[1:]
    med = {k: float(np.median([r[k] for r in rows])) for k in rows[0]}
    C = int(info.candidates)
    return {"config": name, "dist": dist, "n": n, "d": d, "eps": eps, "kernel": kernel,
            "short_circuit": sc, "candidates": C, "pairs": int(st.pairs_emitted),
            "n_cells": int(info.n_cells), "tiles": int(st.tiles_processed),
            "chunks_skipped": int(st.chunks_skipped), "rechecks": int(st.guard_rechecks),
            **med,
            "refine_tflops": 2.0 * d * C / (med["refine_kernel_ms"] * 1e-3) / 1e12,
            "step_tflops": 2.0 * d * C / (med["step_ms"] * 1e-3) / 1e12}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["c1", "c2", "c4d2", "c4d8", "c3", "c4d16",
                                                   "c4d32", "c5"])
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--kernels", default="tile,scalar")
    ap.add_argument("--no-short-circuit", action="store_true")
    args = ap.parse_args()
    for name in args.configs:
        for kernel in args.kernels.split(","):
            t = time.time()
            try:
                line = run(name, kernel, args.reps, not args.no_short_circuit)
            except Exception as e:  # keep sweeping; report the failure
                line = {"config": name, "kernel": kernel, "error": repr(e)[:300]}
            line["wall_s"] = time.time() - t
            print(json.dumps(line), flush=True)
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
