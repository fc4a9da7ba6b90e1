"""ctypes binding of libtedjoin.so (include/tedjoin.h) and the per-device context.

The CUDA library is the only compute path: if it cannot be loaded, or no CUDA
device is visible, every entry point raises RuntimeError — there is no CPU
fallback.  Device buffers are torch tensors (data_ptr()), streams are torch's
current CUDA stream on the context's device.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

from .errors import ResourceError, ValidationError

LIB_PATH = Path(__file__).resolve().parent / "libtedjoin.so"

TJ_OK, TJ_EINVAL, TJ_ECAPACITY, TJ_ECUDA, TJ_ENOMEM = 0, 1, 2, 3, 4
TJ_KERNEL_CORE, TJ_KERNEL_DMMA, TJ_KERNEL_CORE_FMA, TJ_KERNEL_CORE_EXPANDED = 0, 1, 2, 3
TJ_MAX_K_IDX = 8
TJ_MAX_DIM = 128

_i32, _i64, _f64, _vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_double, ctypes.c_void_p


class GridInfo(ctypes.Structure):
    _fields_ = [
        ("n", _i64), ("d", _i32), ("d_pad", _i32), ("k_idx", _i32), ("key_bits", _i32),
        ("eps", _f64), ("eps_sq", _f64), ("n_cells", _i64), ("n_runs", _i64),
        ("candidates", _i64), ("tiles", _i64), ("max_cell", _i64),
    ]


class Stats(ctypes.Structure):
    _fields_ = [
        ("tiles_processed", _i64), ("chunks_executed", _i64), ("chunks_skipped", _i64),
        ("candidates_refined", _i64), ("pairs_emitted", _i64), ("guard_rechecks", _i64),
    ]


# name -> (restype, argtypes); every symbol include/tedjoin.h declares
SIGNATURES = {
    "tj_version": (_i32, []),
    "tj_ctx_create": (_i32, [_i32, ctypes.POINTER(_vp)]),
    "tj_ctx_destroy": (None, [_vp]),
    "tj_last_error": (ctypes.c_char_p, [_vp]),
    "tj_build_grid": (_i32, [_vp, _vp, _i64, _i32, _i64, _i32, _f64, _vp]),
    "tj_get_grid_info": (_i32, [_vp, ctypes.POINTER(GridInfo)]),
    "tj_grid_export": (_i32, [_vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "tj_refine": (_i32, [_vp, _i32, _i32, _i64, _i64, _vp]),
    "tj_result_count": (_i32, [_vp, ctypes.POINTER(_i64), ctypes.POINTER(_i32)]),
    "tj_reset_results": (_i32, [_vp, _vp]),
    "tj_reserve_results": (_i32, [_vp, _i64]),
    "tj_checkpoint_results": (_i32, [_vp, _vp]),
    "tj_set_symmetric": (_i32, [_vp, _i32]),
    "tj_set_output_ids": (_i32, [_vp, _vp]),
    "tj_refine_masks": (_i32, [_vp, _i32, _i32, _i64, _i64, _vp]),
    "tj_estimate_pairs": (_i32, [_vp, _i32, _i64, _i64, _i32, ctypes.c_uint64,
                                 ctypes.POINTER(_f64), _vp]),
    "tj_rollback_results": (_i32, [_vp, _i64, _i64, _vp]),
    "tj_finalize": (_i32, [_vp, _vp, _vp, _vp]),
    "tj_finalize_offsets": (_i32, [_vp, _vp, _vp]),
    "tj_finalize_rows": (_i32, [_vp, _vp, _vp, _vp]),
    "tj_finalize_rows_chunk": (_i32, [_vp, _vp, _vp, _i32, _i32, _vp]),
    "tj_get_stats": (_i32, [_vp, ctypes.POINTER(Stats)]),
    "tj_cell_costs": (_i32, [_vp, _vp]),
    "tj_pair_sq_dists": (_i32, [_vp, _vp, _i64, _i32, _vp, _i64, _vp, _i64, _vp, _vp]),
    "tj_write_pairs": (_i32, [ctypes.c_char_p, _vp, _i64, _vp, _vp, _i32]),
    "tj_expand_pairs": (_i32, [_vp, _i64, _vp, _vp, _i32]),
    "tj_column_moments": (_i32, [_vp, _vp, _i64, _i32, _i64, _vp, _vp, _vp]),
    "tj_permute_columns": (_i32, [_vp, _vp, _i64, _i32, _i64, _vp, _vp, _i64, _vp]),
    "tj_brute_force": (_i32, [_vp, _vp, _i64, _i32, _i64, _f64, _vp, _vp, _vp, _vp]),
    "tj_host_register": (_i32, [_vp, _i64, _i32, ctypes.POINTER(_vp)]),
    "tj_host_unregister": (_i32, [_vp]),
    "tj_shard_bounds": (_i32, [_vp, _vp, _i64, _i64, _i32, _f64, _vp, _vp, _vp]),
    "tj_shard_histogram": (_i32, [_vp, _vp, _i64, _i64, _i32, _f64, _vp, _vp, _vp, _vp]),
    "tj_shard_select": (_i32, [_vp, _vp, _i64, _i64, _i32, _i32, _f64, _vp, _vp, _i64, _i64,
                               _vp, _i64, _vp, _i64, _i64, ctypes.POINTER(_i64), _vp]),
    "tj_shard_route": (_i32, [_vp, _vp, _i64, _i64, _i32, _i32, _f64, _vp, _vp, _vp, _vp, _i32,
                              _vp, _vp, _i64, _vp, _i64, _i64, _vp]),
    "tj_shard_cell_range": (_i32, [_vp, _i32, _vp, _vp, _i64, _i64, ctypes.POINTER(_i64),
                                   ctypes.POINTER(_i64)]),
    "tj_remap_ids": (_i32, [_vp, _vp, _i64, _vp, _vp]),
    "tj_scatter_counts": (_i32, [_vp, _vp, _i64, _vp, _vp, _vp]),
    "tj_counts_to_offsets": (_i32, [_vp, _vp, _i64, _vp, _vp]),
    "tj_scatter_counts_u8": (_i32, [_vp, _vp, _i64, _vp, _vp, _vp, _vp]),
    "tj_counts_u8_to_offsets": (_i32, [_vp, _vp, _i64, _vp, _vp]),
    "tj_place_rows": (_i32, [_vp, _vp, _vp, _i64, _vp, _vp, _vp, _vp]),
    "tj_fp64_peak": (_i32, [_i32, _i32, ctypes.POINTER(_f64), ctypes.POINTER(_f64)]),
    "tj_dmma_known_answer": (_i32, [_vp, _vp, _vp, _vp]),
    "tj_last_refine_ms": (_i32, [_vp, ctypes.POINTER(_f64)]),
    "tj_last_emit_ms": (_i32, [_vp, ctypes.POINTER(_f64)]),
    "tj_launch_count": (_i64, []),
}

_lib = None
_lib_lock = threading.Lock()


def load_library(path: str | os.PathLike | None = None) -> ctypes.CDLL:
    """Load libtedjoin.so and bind every declared symbol (no GPU needed)."""
    global _lib
    with _lib_lock:
        if _lib is not None and path is None:
            return _lib
        p = Path(path) if path is not None else LIB_PATH
        if not p.exists():
            raise RuntimeError(
                f"{p} is missing: build the CUDA extension first "
                "(python -m paper_2209_11287_b200.build); there is no CPU fallback"
            )
        lib = ctypes.CDLL(str(p))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if path is None:
            _lib = lib
        return lib


def _raise(status: int, msg: str):
    if status == TJ_EINVAL:
        raise ValidationError(msg)
    if status == TJ_ECAPACITY:
        raise ResourceError(msg)
    raise RuntimeError(f"tedjoin CUDA error ({status}): {msg}")


class Context:
    """One tj_ctx on one CUDA device (owns the device grid and result buffers)."""

    def __init__(self, device: int):
        import torch

        if not torch.cuda.is_available():
            raise RuntimeError("tedjoin requires a CUDA device (sm_100a); none is visible")
        self.lib = load_library()
        self.device = int(device)
        handle = _vp()
        st = self.lib.tj_ctx_create(self.device, ctypes.byref(handle))
        if st != TJ_OK:
            _raise(st, self.lib.tj_last_error(None).decode())
        self.handle = handle
        self.lock = threading.RLock()

    def __del__(self):
        h = getattr(self, "handle", None)
        if h and getattr(self, "lib", None) is not None:
            try:
                self.lib.tj_ctx_destroy(h)
            except Exception:
                pass
            self.handle = None

    def _check(self, st: int):
        if st != TJ_OK:
            _raise(st, self.lib.tj_last_error(self.handle).decode())

    def stream(self):
        import torch

        return torch.cuda.current_stream(self.device)

    def build_grid(self, coords, n: int, d: int, ld: int, k_idx: int, eps: float, stream=None):
        s = stream or self.stream()
        self._check(self.lib.tj_build_grid(self.handle, coords.data_ptr(), n, d, ld, k_idx,
                                           float(eps), s.cuda_stream))

    def grid_info(self) -> GridInfo:
        info = GridInfo()
        self._check(self.lib.tj_get_grid_info(self.handle, ctypes.byref(info)))
        return info

    def export(self, info: GridInfo, k: int):
        import numpy as np

        order = np.empty(info.n, dtype=np.uint32)
        cstart = np.empty(info.n_cells + 1, dtype=np.int64)
        coords = np.empty((info.n_cells, k), dtype=np.int64)
        cands = np.empty(info.n_cells, dtype=np.int64)
        cruns = np.empty(info.n_cells + 1, dtype=np.int64)
        runs = np.empty((max(info.n_runs, 1), 2), dtype=np.uint32)
        self._check(self.lib.tj_grid_export(
            self.handle, order.ctypes.data, cstart.ctypes.data, coords.ctypes.data,
            cands.ctypes.data, cruns.ctypes.data, runs.ctypes.data))
        return order, cstart, coords, cands, cruns, runs[: info.n_runs]

    def cell_costs(self, n_cells: int):
        import numpy as np

        out = np.empty(n_cells, dtype=np.int64)
        self._check(self.lib.tj_cell_costs(self.handle, out.ctypes.data))
        return out

    def refine(self, kernel: int, short_circuit: bool, cell_begin: int, cell_end: int, stream=None):
        s = stream or self.stream()
        self._check(self.lib.tj_refine(self.handle, kernel, int(bool(short_circuit)),
                                       cell_begin, cell_end, s.cuda_stream))

    def reset_results(self, stream=None):
        s = stream or self.stream()
        self._check(self.lib.tj_reset_results(self.handle, s.cuda_stream))

    def reserve_results(self, pairs: int):
        self._check(self.lib.tj_reserve_results(self.handle, int(pairs)))

    def estimate_pairs(self, kernel: int, cell_begin: int, cell_end: int, samples: int = 256,
                       seed: int = 0, stream=None) -> float:
        """Sampled result pairs per candidate pair of the cell range (tj_estimate_pairs)."""
        s = stream or self.stream()
        rate = _f64()
        self._check(self.lib.tj_estimate_pairs(self.handle, int(kernel), int(cell_begin),
                                               int(cell_end), int(samples), int(seed),
                                               ctypes.byref(rate), s.cuda_stream))
        return float(rate.value)

    def refine_masks(self, kernel: int, short_circuit: bool, cell_begin: int, cell_end: int,
                     stream=None):
        s = stream or self.stream()
        self._check(self.lib.tj_refine_masks(self.handle, kernel, int(bool(short_circuit)),
                                             cell_begin, cell_end, s.cuda_stream))

    def set_output_ids(self, id_map):
        self._check(self.lib.tj_set_output_ids(self.handle,
                                               id_map.data_ptr() if id_map is not None else None))

    def set_symmetric(self, on: bool):
        self._check(self.lib.tj_set_symmetric(self.handle, int(bool(on))))

    def checkpoint_results(self, stream=None):
        s = stream or self.stream()
        self._check(self.lib.tj_checkpoint_results(self.handle, s.cuda_stream))

    def rollback_results(self, cell_begin: int, cell_end: int, stream=None):
        s = stream or self.stream()
        self._check(self.lib.tj_rollback_results(self.handle, int(cell_begin), int(cell_end),
                                                 s.cuda_stream))

    def result_count(self):
        total, over = _i64(), _i32()
        self._check(self.lib.tj_result_count(self.handle, ctypes.byref(total), ctypes.byref(over)))
        return int(total.value), bool(over.value)

    def finalize(self, offsets, neighbors, stream=None):
        s = stream or self.stream()
        self._check(self.lib.tj_finalize(self.handle, offsets.data_ptr(),
                                         neighbors.data_ptr() if neighbors is not None else None,
                                         s.cuda_stream))

    def finalize_offsets(self, offsets, stream=None):
        s = stream or self.stream()
        self._check(self.lib.tj_finalize_offsets(self.handle, offsets.data_ptr(), s.cuda_stream))

    def finalize_rows(self, offsets, neighbors, stream=None):
        s = stream or self.stream()
        self._check(self.lib.tj_finalize_rows(
            self.handle, offsets.data_ptr(),
            neighbors.data_ptr() if neighbors is not None else None, s.cuda_stream))

    def finalize_rows_chunk(self, offsets, neighbors, chunk: int, chunks: int, stream=None):
        s = stream or self.stream()
        self._check(self.lib.tj_finalize_rows_chunk(
            self.handle, offsets.data_ptr(), neighbors.data_ptr() if neighbors is not None else None,
            int(chunk), int(chunks), s.cuda_stream))

    def stats(self) -> Stats:
        st = Stats()
        self._check(self.lib.tj_get_stats(self.handle, ctypes.byref(st)))
        return st

    def pair_sq_dists(self, coords, d: int, offsets, neighbors, m: int, out, stream=None):
        """Canonical direct-form squared distance of every CSR pair (device tensors)."""
        s = stream or self.stream()
        n = offsets.shape[0] - 1
        self._check(self.lib.tj_pair_sq_dists(
            self.handle, coords.data_ptr(), int(coords.stride(0)), int(d), offsets.data_ptr(), n,
            neighbors.data_ptr() if m else None, int(m), out.data_ptr() if m else None,
            s.cuda_stream))

    def column_moments(self, coords, n: int, d: int):
        """(mean, var) numpy arrays of the first d columns of a device tensor."""
        import numpy as np

        mean, var = np.empty(d), np.empty(d)
        self._check(self.lib.tj_column_moments(self.handle, coords.data_ptr(), int(n), int(d),
                                               int(coords.stride(0)), mean.ctypes.data,
                                               var.ctypes.data, self.stream().cuda_stream))
        return mean, var

    def permute_columns(self, src, n: int, d: int, perm, dst):
        import numpy as np

        p = np.ascontiguousarray(perm, dtype=np.int32)
        self._check(self.lib.tj_permute_columns(self.handle, src.data_ptr(), int(n), int(d),
                                                int(src.stride(0)), p.ctypes.data, dst.data_ptr(),
                                                int(dst.stride(0)), self.stream().cuda_stream))

    def brute_force(self, coords, n: int, d: int, eps: float, offsets, neighbors=None):
        """Two-phase GPU brute force: without neighbors returns the pair count."""
        total = _i64()
        self._check(self.lib.tj_brute_force(
            self.handle, coords.data_ptr(), int(n), int(d), int(coords.stride(0)), float(eps),
            offsets.data_ptr(), neighbors.data_ptr() if neighbors is not None else None,
            ctypes.byref(total) if neighbors is None else None, self.stream().cuda_stream))
        return int(total.value)

    # ---- multi-GPU strong layout (shard.cu) ----
    @staticmethod
    def _bins(pdims, origin, span):
        import numpy as np

        o = np.ascontiguousarray(origin, dtype=np.int64)[:pdims]
        sp = np.ascontiguousarray(span, dtype=np.int64)[:pdims]
        return o, sp

    def shard_bounds(self, coords, n: int, pdims: int, eps: float):
        """(lo, hi) numpy int64[pdims]: floor(x_j / eps) bounds of the rows."""
        import numpy as np

        lo, hi = np.zeros(2, np.int64), np.zeros(2, np.int64)
        self._check(self.lib.tj_shard_bounds(
            self.handle, coords.data_ptr() if n else None, int(n), int(coords.stride(0)),
            int(pdims), float(eps), lo.ctypes.data, hi.ctypes.data, self.stream().cuda_stream))
        return lo[:pdims], hi[:pdims]

    def shard_histogram(self, coords, n: int, pdims: int, eps: float, origin, span, hist):
        o, sp = self._bins(pdims, origin, span)
        self._check(self.lib.tj_shard_histogram(
            self.handle, coords.data_ptr() if n else None, int(n), int(coords.stride(0)),
            int(pdims), float(eps), o.ctypes.data, sp.ctypes.data, hist.data_ptr(),
            self.stream().cuda_stream))

    def shard_select(self, coords, n: int, d: int, pdims: int, eps: float, origin, span,
                     own_lo: int, own_hi: int, out=None, gid=None, gid_base: int = 0) -> int:
        o, sp = self._bins(pdims, origin, span)
        sel = _i64()
        self._check(self.lib.tj_shard_select(
            self.handle, coords.data_ptr() if n else None, int(n), int(coords.stride(0)), int(d),
            int(pdims), float(eps), o.ctypes.data, sp.ctypes.data, int(own_lo), int(own_hi),
            out.data_ptr() if out is not None else None,
            int(out.stride(0)) if out is not None else 0,
            gid.data_ptr() if gid is not None else None, int(gid_base),
            int(out.shape[0]) if out is not None else 0, ctypes.byref(sel),
            self.stream().cuda_stream))
        return int(sel.value)

    def shard_route(self, coords, n: int, d: int, pdims: int, eps: float, origin, span, ranges,
                    counts=None, out=None, gid=None, gid_base: int = 0):
        """Count (out None) or write the rows each rank needs (tj_shard_route)."""
        import numpy as np

        o, sp = self._bins(pdims, origin, span)
        lo = np.ascontiguousarray([r[0] for r in ranges], dtype=np.int64)
        hi = np.ascontiguousarray([r[1] for r in ranges], dtype=np.int64)
        cnt = (np.zeros(len(ranges), np.int64) if counts is None
               else np.ascontiguousarray(counts, dtype=np.int64))
        self._check(self.lib.tj_shard_route(
            self.handle, coords.data_ptr() if n else None, int(n), int(coords.stride(0)), int(d),
            int(pdims), float(eps), o.ctypes.data, sp.ctypes.data, lo.ctypes.data, hi.ctypes.data,
            len(ranges), cnt.ctypes.data, out.data_ptr() if out is not None else None,
            int(out.stride(0)) if out is not None else 0,
            gid.data_ptr() if gid is not None else None, int(gid_base),
            int(out.shape[0]) if out is not None else 0, self.stream().cuda_stream))
        return [int(v) for v in cnt]

    def shard_cell_range(self, pdims: int, origin, span, own_lo: int, own_hi: int):
        o, sp = self._bins(pdims, origin, span)
        b, e = _i64(), _i64()
        self._check(self.lib.tj_shard_cell_range(self.handle, int(pdims), o.ctypes.data,
                                                 sp.ctypes.data, int(own_lo), int(own_hi),
                                                 ctypes.byref(b), ctypes.byref(e)))
        return int(b.value), int(e.value)

    def remap_ids(self, ids, m: int, gid):
        self._check(self.lib.tj_remap_ids(self.handle, ids.data_ptr() if m else None, int(m),
                                          gid.data_ptr(), self.stream().cuda_stream))

    def scatter_counts(self, offsets, n_rows: int, gid, counts, overflow=None):
        """counts (int32, or uint8 with an int32 `overflow` flag) [gid[l]] = row l's length."""
        import torch

        if counts.dtype == torch.uint8:
            self._check(self.lib.tj_scatter_counts_u8(self.handle, offsets.data_ptr(), int(n_rows),
                                                      gid.data_ptr(), counts.data_ptr(),
                                                      overflow.data_ptr(), self.stream().cuda_stream))
        else:
            self._check(self.lib.tj_scatter_counts(self.handle, offsets.data_ptr(), int(n_rows),
                                                   gid.data_ptr(), counts.data_ptr(),
                                                   self.stream().cuda_stream))

    def counts_to_offsets(self, counts, n: int, offsets):
        import torch

        fn = (self.lib.tj_counts_u8_to_offsets if counts.dtype == torch.uint8
              else self.lib.tj_counts_to_offsets)
        self._check(fn(self.handle, counts.data_ptr(), int(n), offsets.data_ptr(),
                       self.stream().cuda_stream))

    def place_rows(self, offsets, neighbors, n_rows: int, gid, global_offsets, dst_ptr: int):
        self._check(self.lib.tj_place_rows(self.handle, offsets.data_ptr(), neighbors.data_ptr(),
                                           int(n_rows), gid.data_ptr(),
                                           global_offsets.data_ptr(), int(dst_ptr),
                                           self.stream().cuda_stream))

    def last_emit_ms(self) -> float | None:
        ms = _f64()
        if self.lib.tj_last_emit_ms(self.handle, ctypes.byref(ms)) != TJ_OK:
            return None
        return float(ms.value)

    def last_refine_ms(self) -> float:
        ms = _f64()
        self._check(self.lib.tj_last_refine_ms(self.handle, ctypes.byref(ms)))
        return float(ms.value)


_contexts: dict[int, Context] = {}
_ctx_lock = threading.Lock()


def context(device: int | None = None) -> Context:
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("tedjoin requires a CUDA device (sm_100a); none is visible")
    dev = torch.cuda.current_device() if device is None else int(device)
    with _ctx_lock:
        ctx = _contexts.get(dev)
        if ctx is None:
            ctx = _contexts[dev] = Context(dev)
        return ctx


def write_pairs(path, offsets, neighbors, sq, threads: int | None = None) -> None:
    """Pairs file from host CSR arrays + squared distances (native, multi-threaded)."""
    import numpy as np

    lib = load_library()
    off = np.ascontiguousarray(offsets, dtype=np.int64)
    nb = np.ascontiguousarray(neighbors, dtype=np.uint32)
    sq = np.ascontiguousarray(sq, dtype=np.float64)
    th = threads or min(16, os.cpu_count() or 1)
    st = lib.tj_write_pairs(os.fsencode(os.fspath(path)), off.ctypes.data, len(off) - 1,
                            nb.ctypes.data, sq.ctypes.data, int(th))
    if st != TJ_OK:
        _raise(st, lib.tj_last_error(None).decode())


def expand_pairs(offsets, neighbors, threads: int | None = None):
    """(m, 2) int64 (query id, neighbour id) rows of a host CSR (native, multi-threaded)."""
    import numpy as np

    lib = load_library()
    off = np.ascontiguousarray(offsets, dtype=np.int64)
    m = int(off[-1])
    nb = np.ascontiguousarray(neighbors[:m]).view(np.uint32) if m else np.zeros(1, np.uint32)
    out = np.empty((m, 2), dtype=np.int64)
    th = threads or min(32, os.cpu_count() or 1)
    st = lib.tj_expand_pairs(off.ctypes.data, len(off) - 1, nb.ctypes.data, out.ctypes.data,
                             int(th))
    if st != TJ_OK:
        _raise(st, lib.tj_last_error(None).decode())
    return out


def host_register(ptr: int, nbytes: int, mapped: bool = False) -> int | None:
    """Page-lock host memory; returns the device alias when mapped (else None)."""
    lib = load_library()
    dptr = _vp()
    st = lib.tj_host_register(ctypes.c_void_p(ptr), int(nbytes), int(bool(mapped)),
                              ctypes.byref(dptr) if mapped else None)
    if st != TJ_OK:
        _raise(st, lib.tj_last_error(None).decode())
    return int(dptr.value) if mapped else None


def host_unregister(ptr: int) -> None:
    lib = load_library()
    st = lib.tj_host_unregister(ctypes.c_void_p(ptr))
    if st != TJ_OK:
        _raise(st, lib.tj_last_error(None).decode())


def launch_count() -> int:
    """Kernels libtedjoin.so has launched in this process."""
    return int(load_library().tj_launch_count())


def fp64_peak(kind: int, iters: int = 8192) -> tuple[float, float]:
    """(TFLOP/s, ms) of the FP64 microbenchmark on the current device."""
    lib = load_library()
    tf, ms = _f64(), _f64()
    st = lib.tj_fp64_peak(kind, iters, ctypes.byref(tf), ctypes.byref(ms))
    if st != TJ_OK:
        raise RuntimeError(f"tj_fp64_peak failed with status {st}")
    return float(tf.value), float(ms.value)
