"""ORACLE — TEST INFRASTRUCTURE ONLY.

CPU restatements of the reference tilejoin self-join used to check the CUDA
path.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline and
--impl reference legs may import this package; the product package
paper_2209_11287_b200 never does.

* `join_csr` / `grid` wrap liboracle.so (direct_join.c): the reference grid
  (grid.py:66-133) + scalar refinement (join.py:286-349) in C with
  -ffp-contract=off, OpenMP over cells.  Pinned bit-for-bit against the
  reference's own outputs by tests/golden (made by tests/golden/make_golden.py
  with the reference imported from /root/reference).
* `brute_force` restates oracle.brute_force_join (oracle.py:55-86) in numpy.
"""

from __future__ import annotations

import ctypes
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "liboracle.so"
_lib = None


def build() -> Path:
    """Compile liboracle.so with the committed Makefile (gcc, OpenMP)."""
    res = subprocess.run(["make", "-s", "-C", str(HERE), "liboracle.so"], capture_output=True,
                         text=True)
    if res.returncode != 0:
        raise RuntimeError(f"oracle build failed:\n{res.stdout}\n{res.stderr}")
    return LIB


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not LIB.exists() or LIB.stat().st_mtime < (HERE / "direct_join.c").stat().st_mtime:
            build()
        L = ctypes.CDLL(str(LIB))
        vp, i64, i32, f64 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
        L.oracle_self_join.restype = i32
        L.oracle_self_join.argtypes = [vp, i64, i32, i64, i32, f64, vp, i64, vp, vp, vp, i32]
        L.oracle_grid.restype = i64
        L.oracle_grid.argtypes = [vp, i64, i32, i64, i32, f64, vp, vp, vp, vp]
        L.oracle_sqdist.restype = f64
        L.oracle_sqdist.argtypes = [vp, i64, i32, i64, i64]
        L.oracle_num_threads.restype = i32
        L.oracle_time_join.restype = i64
        L.oracle_time_join.argtypes = [vp, i64, i32, i64, i32, f64, vp, i64, i32,
                                       ctypes.POINTER(f64), ctypes.POINTER(f64)]
        L.oracle_rows.restype = i32
        L.oracle_rows.argtypes = [vp, i64, i32, i64, i32, f64, vp, i64, vp, vp, i32]
        L.oracle_digest.restype = i32
        L.oracle_digest.argtypes = [vp, i64, i32, i64, i32, f64, i32, vp]
        L.oracle_digest_keys.restype = None
        L.oracle_digest_keys.argtypes = [vp, i64, vp]
        _lib = L
    return _lib


def _coords(data):
    x = getattr(data, "coords", None)
    if x is None:
        x = np.ascontiguousarray(np.asarray(data, dtype=np.float64))
        return x, x.shape[1]
    return np.ascontiguousarray(x), int(data.d)


def join_csr(data, eps: float, k_idx: int | None = None, cells=None, threads: int = 0):
    """Reference direct-form self-join -> (offsets int64[n+1], neighbours uint32[m]).

    cells: optional int64 indices into the lexicographic cell list; only those
    cells' queries are refined (their rows are complete, others empty).
    """
    x, d = _coords(data)
    n, ld = x.shape
    k = min(d, 6) if k_idx is None else int(k_idx)
    L = lib()
    offsets = np.zeros(n + 1, dtype=np.int64)
    total = ctypes.c_int64(0)
    sel = None if cells is None else np.ascontiguousarray(cells, dtype=np.int64)
    sel_ptr = None if sel is None else sel.ctypes.data
    n_sel = 0 if sel is None else len(sel)
    rc = L.oracle_self_join(x.ctypes.data, n, d, ld, k, float(eps), sel_ptr, n_sel,
                            offsets.ctypes.data, None, ctypes.byref(total), threads)
    if rc != 0:
        raise RuntimeError(f"oracle_self_join failed ({rc})")
    nbrs = np.empty(max(total.value, 1), dtype=np.uint32)
    rc = L.oracle_self_join(x.ctypes.data, n, d, ld, k, float(eps), sel_ptr, n_sel,
                            offsets.ctypes.data, nbrs.ctypes.data, ctypes.byref(total), threads)
    if rc != 0:
        raise RuntimeError(f"oracle_self_join failed ({rc})")
    return offsets, nbrs[: total.value]


def rows(data, eps: float, qids, k_idx: int | None = None, threads: int = 0):
    """Reference rows of selected query ids -> (counts int64[len(qids)], concatenated ids)."""
    x, d = _coords(data)
    n, ld = x.shape
    k = min(d, 6) if k_idx is None else int(k_idx)
    q = np.ascontiguousarray(qids, dtype=np.int64)
    counts = np.zeros(len(q), dtype=np.int64)
    L = lib()
    rc = L.oracle_rows(x.ctypes.data, n, d, ld, k, float(eps), q.ctypes.data, len(q),
                       counts.ctypes.data, None, threads)
    if rc != 0:
        raise RuntimeError(f"oracle_rows failed ({rc})")
    nbrs = np.empty(max(int(counts.sum()), 1), dtype=np.uint32)
    rc = L.oracle_rows(x.ctypes.data, n, d, ld, k, float(eps), q.ctypes.data, len(q),
                       counts.ctypes.data, nbrs.ctypes.data, threads)
    if rc != 0:
        raise RuntimeError(f"oracle_rows failed ({rc})")
    return counts, nbrs[: int(counts.sum())]


def grid(data, eps: float, k_idx: int | None = None):
    """(point_order, cell_start, cell_coords, cand_counts) in the reference's grid order."""
    x, d = _coords(data)
    n, ld = x.shape
    k = min(d, 6) if k_idx is None else int(k_idx)
    order = np.empty(n, dtype=np.uint32)
    cstart = np.empty(n + 1, dtype=np.int64)
    ccoord = np.empty(n * k, dtype=np.int64)
    cand = np.empty(n, dtype=np.int64)
    nc = lib().oracle_grid(x.ctypes.data, n, d, ld, k, float(eps), order.ctypes.data,
                           cstart.ctypes.data, ccoord.ctypes.data, cand.ctypes.data)
    if nc < 0:
        raise RuntimeError("oracle_grid failed")
    return order, cstart[: nc + 1], ccoord[: nc * k].reshape(nc, k), cand[:nc]


def sqdist(data, i: int, j: int) -> float:
    """Reference direct-form squared distance of points i and j (oracle.py:78-81)."""
    x, d = _coords(data)
    return lib().oracle_sqdist(x.ctypes.data, x.shape[1], d, int(i), int(j))


def time_join(data, eps: float, cells=None, k_idx: int | None = None, threads: int = 0):
    """(grid seconds, refine seconds, pairs) of the reference algorithm on the host cores.

    The grid over all points is built once; only `cells` (indices into the
    lexicographic cell list; None = all) are refined, in one emitting pass.
    """
    x, d = _coords(data)
    n, ld = x.shape
    k = min(d, 6) if k_idx is None else int(k_idx)
    sel = None if cells is None else np.ascontiguousarray(cells, dtype=np.int64)
    gs, rs = ctypes.c_double(), ctypes.c_double()
    pairs = lib().oracle_time_join(x.ctypes.data, n, d, ld, k, float(eps),
                                   None if sel is None else sel.ctypes.data,
                                   0 if sel is None else len(sel), threads,
                                   ctypes.byref(gs), ctypes.byref(rs))
    if pairs < 0:
        raise RuntimeError("oracle_time_join failed")
    return gs.value, rs.value, int(pairs)


def digest(data, eps: float, k_idx: int | None = None, threads: int = 0) -> dict:
    """Order-independent digest of the full reference pair set (direct_join.c
    oracle_digest): {"pairs", "s1", "s2", "max_row"}; no output is materialised."""
    x, d = _coords(data)
    n, ld = x.shape
    k = min(d, 6) if k_idx is None else int(k_idx)
    out = np.zeros(4, dtype=np.uint64)
    if lib().oracle_digest(x.ctypes.data, n, d, ld, k, float(eps), threads, out.ctypes.data) != 0:
        raise RuntimeError("oracle_digest failed")
    return {"pairs": int(out[0]), "s1": int(out[1]), "s2": int(out[2]), "max_row": int(out[3])}


def digest_keys(keys) -> dict:
    """The same digest over explicit keys (q << 32 | c), uint64."""
    k = np.ascontiguousarray(keys, dtype=np.uint64)
    out = np.zeros(3, dtype=np.uint64)
    lib().oracle_digest_keys(k.ctypes.data, len(k), out.ctypes.data)
    return {"pairs": int(out[0]), "s1": int(out[1]), "s2": int(out[2])}


def num_threads() -> int:
    return int(lib().oracle_num_threads())


def brute_force(data, eps: float) -> np.ndarray:
    """All ordered pairs with direct-form squared distance <= fl(eps*eps), sorted (m, 2) int64.

    Restates oracle.brute_force_join (oracle.py:55-86): 256-row blocks,
    ascending-dimension accumulation, numpy's unfused subtract/multiply/add.
    """
    x, d = _coords(data)
    x = x[:, :d]
    n = x.shape[0]
    eps_sq = eps * eps
    out_i, out_j = [], []
    for s in range(0, n, 256):
        q = x[s: s + 256]
        acc = np.zeros((q.shape[0], n))
        for dim in range(d):
            diff = q[:, dim, None] - x[None, :, dim]
            acc += diff * diff
        ii, jj = np.nonzero(acc <= eps_sq)
        out_i.append(ii + s)
        out_j.append(jj)
    return np.column_stack([np.concatenate(out_i), np.concatenate(out_j)]).astype(np.int64)


def csr_to_pairs(offsets, nbrs) -> np.ndarray:
    n = len(offsets) - 1
    out = np.empty((int(offsets[-1]), 2), dtype=np.int64)
    out[:, 0] = np.repeat(np.arange(n, dtype=np.int64), np.diff(offsets))
    out[:, 1] = nbrs[: offsets[-1]]
    return out
