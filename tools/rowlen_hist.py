"""Row-length histogram of a bench workload's result (which finalize paths it exercises)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np

from bench import CONFIGS
from paper_2209_11287_b200 import GenSpec, JoinConfig, generate
from paper_2209_11287_b200.join import self_join

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
dist, n, d, eps = CONFIGS[name]
r = self_join(generate(GenSpec(dist, n, d, seed=0)), JoinConfig(epsilon=eps))
lens = np.diff(r.offsets)
edges = [0, 32, 64, 96, 128, 256, 512, 1024, 2048, 4096, 8192, 1 << 40]
h, _ = np.histogram(lens, bins=edges)
tot = lens.sum()
for lo, hi, c in zip(edges[:-1], edges[1:], h):
    sel = (lens >= lo) & (lens < hi)
    print(f"[{lo},{hi}): rows {c} ({100 * c / len(lens):.2f}%), ids {100 * lens[sel].sum() / tot:.2f}%")
print("max", lens.max(), "mean", lens.mean())
