"""Order-independent pair-set digest (test infrastructure).

The same digest as oracle/direct_join.c oracle_digest: for every pair (q, c),
key = q << 32 | c; s1 = sum splitmix64(key), s2 = sum splitmix64(key + K2), both
mod 2^64, plus the pair count.  `csr_digest_torch` computes it from a CSR held in
device memory (torch int64 arithmetic wraps mod 2^64; right shifts are masked to
be logical), so full-size GPU results are checked without a host copy.
"""

from __future__ import annotations

import numpy as np

K2 = 0x632BE59BD9B4E019
C1 = 0xBF58476D1CE4E5B9
C2 = 0x94D049BB133111EB
M64 = (1 << 64) - 1


def _s64(v: int) -> int:
    return v - (1 << 64) if v >= (1 << 63) else v


def _mix_torch(z):
    import torch  # noqa: F401

    def lsr(x, s):
        return (x >> s) & ((1 << (64 - s)) - 1)

    z = z ^ lsr(z, 30)
    z = z * _s64(C1)
    z = z ^ lsr(z, 27)
    z = z * _s64(C2)
    z = z ^ lsr(z, 31)
    return z


def keys_digest_torch(keys) -> dict:
    """Digest of an int64 tensor of keys (q << 32 | c)."""
    s1 = int(_mix_torch(keys).sum().item()) & M64
    s2 = int(_mix_torch(keys + _s64(K2)).sum().item()) & M64
    return {"pairs": int(keys.numel()), "s1": s1, "s2": s2}


def csr_digest_torch(offsets, neighbors, chunk_rows: int = 1 << 22) -> dict:
    """Digest + row checks of a CSR (offsets int64[n+1], neighbors int32/uint32 ids)
    in device memory: also returns max_row and whether every row is strictly
    ascending (canonical order)."""
    import torch

    n = offsets.numel() - 1
    counts = offsets[1:] - offsets[:-1]
    s1 = s2 = 0
    ascending = True
    for r0 in range(0, n, chunk_rows):
        r1 = min(n, r0 + chunk_rows)
        a, b = int(offsets[r0].item()), int(offsets[r1].item())
        if a == b:
            continue
        rows = torch.repeat_interleave(
            torch.arange(r0, r1, device=offsets.device, dtype=torch.int64), counts[r0:r1])
        nb = neighbors[a:b].to(torch.int64) & 0xFFFFFFFF
        keys = (rows << 32) | nb
        s1 += int(_mix_torch(keys).sum().item())
        s2 += int(_mix_torch(keys + _s64(K2)).sum().item())
        # strictly ascending inside each row: key order is (row, id) lexicographic
        if keys.numel() > 1 and not bool((keys[1:] > keys[:-1]).all().item()):
            ascending = False
        del rows, nb, keys
    return {"pairs": int(offsets[-1].item()), "s1": s1 & M64, "s2": s2 & M64,
            "max_row": int(counts.max().item()) if n else 0, "ascending": ascending}


def csr_digest_numpy(offsets, neighbors) -> dict:
    """Host version for small CSRs (uint64 numpy arithmetic wraps)."""
    off = np.asarray(offsets, np.int64)
    n = len(off) - 1
    rows = np.repeat(np.arange(n, dtype=np.uint64), np.diff(off))
    keys = (rows << np.uint64(32)) | np.asarray(neighbors[: off[-1]], np.uint64)

    def mix(z):
        z = z ^ (z >> np.uint64(30))
        z = z * np.uint64(C1)
        z = z ^ (z >> np.uint64(27))
        z = z * np.uint64(C2)
        return z ^ (z >> np.uint64(31))

    with np.errstate(over="ignore"):
        s1 = int(mix(keys).sum(dtype=np.uint64))
        s2 = int(mix(keys + np.uint64(K2)).sum(dtype=np.uint64))
    return {"pairs": int(off[-1]), "s1": s1, "s2": s2,
            "max_row": int(np.diff(off).max()) if n else 0}
