"""GPU exact brute-force digests for the configs beyond the CPU oracle (run on the GPU box).

    python tools/make_bf_digests.py [c2 c4d16 c4d32 c4d64]  ->  tests/golden/bf_digests.json

Every ordered pair of the full input is decided by tj_brute_force -- the
reference direct form with __d*_rn intrinsics, no grid (csrc/verify.cu) -- and
the resulting CSR is digested on the device (tests/digest.py).  c2 is included
so the test suite can pin this brute force to the CPU oracle at full size.
"""

from __future__ import annotations

import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]

import torch  # noqa: E402

from digest import csr_digest_torch  # noqa: E402
from paper_2209_11287_b200 import _native  # noqa: E402
from paper_2209_11287_b200.datasets import GenSpec, generate  # noqa: E402

CONFIGS = {
    "c2": ("uniform", 2_000_000, 4, 0.051306),
    "c4d16": ("uniform", 2_000_000, 16, 0.657508),
    "c4d32": ("uniform", 2_000_000, 32, 1.31923),
    "c4d64": ("uniform", 2_000_000, 64, 2.27218),
}


def main(names):
    path = ROOT / "tests" / "golden" / "bf_digests.json"
    out = json.loads(path.read_text()) if path.exists() else {}
    ctx = _native.context(0)
    for name in names or list(CONFIGS):
        dist, n, d, eps = CONFIGS[name]
        ds = generate(GenSpec(dist, n, d, seed=0))
        coords = torch.from_numpy(ds.coords).cuda()
        t = time.perf_counter()
        offsets = torch.empty(n + 1, dtype=torch.int64, device="cuda")
        total = ctx.brute_force(coords, n, d, eps, offsets)
        nbr = torch.empty(max(total, 1), dtype=torch.int32, device="cuda")
        ctx.brute_force(coords, n, d, eps, offsets, nbr)
        torch.cuda.synchronize()
        secs = time.perf_counter() - t
        dg = csr_digest_torch(offsets, nbr)
        assert dg["ascending"]
        dg.pop("ascending")
        dg.update({"dist": dist, "n": n, "d": d, "eps": eps, "checksum": ds.checksum(),
                   "source": "tj_brute_force (GPU exact direct form, all n^2 pairs)",
                   "gpu_seconds": round(secs, 1)})
        out[name] = dg
        print(name, dg, flush=True)
        path.write_text(json.dumps(out, indent=1))
        del coords, offsets, nbr


if __name__ == "__main__":
    main(sys.argv[1:])
