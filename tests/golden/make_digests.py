"""Full-set pair digests of the BASELINE configs from the golden-pinned C oracle.

    python tests/golden/make_digests.py [config ...]   ->  tests/golden/full_digests.json

The oracle (oracle/direct_join.c, the reference grid + direct form restated in C
with -ffp-contract=off) is pinned against the reference itself by the other
fixtures here (sweep.json, config1.json, sampled.*).  This script runs it over
the FULL inputs of configs 1, 2, 3, 4 (d = 2, 4, 8) and 5 and records the
order-independent digest of each pair set (count, two 64-bit sums of
splitmix64(q << 32 | c); tests/digest.py), so the GPU suite can check the whole
pair set at full size without a multi-GB fixture.  Configs 4 d >= 16 are
brute force over 4e12 candidate pairs (hours of this container's 8 cores, the
early exit of the running sum helps); they are also checked against the GPU's
exact direct-form brute force (tj_brute_force, bf_digests.json), itself pinned
to the oracle at full size on config 2.

    TJ_ORACLE_THREADS=6 python tests/golden/make_digests.py c4d16 c4d32 c4d64
"""

from __future__ import annotations

import json
import os
import sys
import time
from pathlib import Path

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT))

import oracle  # noqa: E402
from paper_2209_11287_b200.datasets import GenSpec, generate  # noqa: E402

CONFIGS = {
    "c1": ("uniform", 100_000, 2, 0.0143667),
    "c2": ("uniform", 2_000_000, 4, 0.051306),
    "c4d2": ("uniform", 2_000_000, 2, 0.00320714),
    "c5": ("uniform", 50_000_000, 4, 0.0232204),
    "c4d8": ("uniform", 2_000_000, 8, 0.244686),
    "c3": ("exponential", 5_000_000, 8, 0.0118508),
    "expo3d2m": ("exponential", 2_000_000, 3, 0.00097345),
    # brute force over 4e12 candidate pairs: hours on 8 cores, run in the background
    "c4d16": ("uniform", 2_000_000, 16, 0.657508),
    "c4d32": ("uniform", 2_000_000, 32, 1.31923),
    "c4d64": ("uniform", 2_000_000, 64, 2.27218),
}


def main(names):
    path = HERE / "full_digests.json"
    out = json.loads(path.read_text()) if path.exists() else {}
    for name in names or list(CONFIGS):
        dist, n, d, eps = CONFIGS[name]
        ds = generate(GenSpec(dist, n, d, seed=0))
        t = time.perf_counter()
        dg = oracle.digest(ds, eps, threads=int(os.environ.get("TJ_ORACLE_THREADS", "0")))
        dg.update({"dist": dist, "n": n, "d": d, "eps": eps, "checksum": ds.checksum(),
                   "oracle_seconds": round(time.perf_counter() - t, 1),
                   "oracle_threads": oracle.num_threads()})
        print(name, dg, flush=True)
        out = json.loads(path.read_text()) if path.exists() else {}  # entries written meanwhile
        out[name] = dg
        path.write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1:])
