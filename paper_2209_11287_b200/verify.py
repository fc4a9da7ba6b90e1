"""GPU brute-force verification (the reference's oracle.brute_force_join, oracle.py:55-86).

Every ordered pair is decided by the reference direct form on the GPU
(tj_brute_force), independently of the grid index.  The default guard is the
reference's (oracle.BRUTE_FORCE_GUARD = 50,000, cli.py:165-171); with
force=True the GPU checks inputs far beyond what the CPU oracle can.
"""

from __future__ import annotations

import numpy as np

from . import _native
from .datasets import as_dataset
from .errors import ResourceError, ValidationError
from .join import JoinResult, JoinStats

# Largest n verified without force=True: the reference's guard (oracle.py:22), so
# `verify` refuses the same inputs; with force=True the GPU takes any n.
BRUTE_FORCE_GUARD = 50_000


def brute_force_join(dataset, epsilon: float, force: bool = False,
                     device: int | None = None) -> JoinResult:
    """All ordered pairs with direct-form squared distance <= fl(eps*eps), as a JoinResult."""
    import torch

    ds = as_dataset(dataset)
    if not np.isfinite(epsilon) or epsilon <= 0:
        raise ValidationError(f"epsilon must be positive and finite, got {epsilon}")
    if ds.n > BRUTE_FORCE_GUARD and not force:
        raise ResourceError(
            f"n={ds.n} exceeds the verification guard of {BRUTE_FORCE_GUARD}; "
            "pass force=True to run anyway")
    ctx = _native.context(device)
    dev = f"cuda:{ctx.device}"
    coords = torch.from_numpy(ds.coords).to(dev)
    offsets = torch.empty(ds.n + 1, dtype=torch.int64, device=dev)
    total = ctx.brute_force(coords, ds.n, ds.d, epsilon, offsets)
    nbr = torch.empty(max(total, 1), dtype=torch.int32, device=dev)
    ctx.brute_force(coords, ds.n, ds.d, epsilon, offsets, nbr)
    off = offsets.cpu().numpy()
    nb = nbr[:total].cpu().numpy()
    stats = JoinStats(candidates_refined=ds.n * ds.n, pairs_emitted=total)
    return JoinResult(total_pairs=total, selectivity=(total - ds.n) / ds.n, stats=stats,
                      offsets=off, neighbors=nb)


def pair_set_diff(reference: JoinResult, engine: JoinResult):
    """(missing, extra): pairs only in the reference / only in the engine (cli.py:292-298)."""
    ref = {(int(i), int(j)) for i, j in reference.pairs}
    eng = {(int(i), int(j)) for i, j in engine.pairs}
    return sorted(ref - eng), sorted(eng - ref)
