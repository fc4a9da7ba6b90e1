"""Pairs file: canonical "i j sq_dist" lines of a join result (cli.py:270-289).

`canonical_pair_sq_dists` computes, on the GPU, the reference's canonical
squared distance of every emitted pair -- the direct form summed over
ascending dimensions with one correctly rounded op each (cli.py:270-283) --
whichever kernel produced the pair.  `write_pairs` formats the lines with the
native multi-threaded writer (tj_write_pairs); the text is byte-identical to
the reference's f"{i} {j} {s:.17g}" lines.
"""

from __future__ import annotations

import numpy as np

from . import _native
from .datasets import Dataset, as_dataset


def canonical_pair_sq_dists(dataset, result, device: int | None = None) -> np.ndarray:
    """float64[total_pairs]: direct-form squared distance of each CSR pair, in pair order."""
    import torch

    ds: Dataset = as_dataset(dataset)
    ctx = _native.context(device)
    dev = f"cuda:{ctx.device}"
    m = int(result.total_pairs)
    coords = torch.from_numpy(ds.coords).to(dev)
    offsets = torch.from_numpy(np.ascontiguousarray(result.offsets, dtype=np.int64)).to(dev)
    nbr = torch.from_numpy(np.ascontiguousarray(result.neighbors[:m]).view(np.int32)).to(dev)
    out = torch.empty(max(m, 1), dtype=torch.float64, device=dev)
    ctx.pair_sq_dists(coords, ds.d, offsets, nbr, m, out)
    return out[:m].cpu().numpy()


def write_pairs(dataset, result, path, device: int | None = None,
                threads: int | None = None) -> None:
    """One "i j sq_dist" line per pair, sorted by (i, j) (cli._write_pairs, cli.py:285-289)."""
    sq = canonical_pair_sq_dists(dataset, result, device)
    _native.write_pairs(path, result.offsets, result.neighbors[: result.total_pairs], sq, threads)
