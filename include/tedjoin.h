/* tedjoin — C ABI of the B200 (sm_100a) FP64 epsilon self-join engine.
 *
 * This is the boundary below the Python drop-in for the reference package's
 * `tilejoin.join.self_join(dataset, JoinConfig(epsilon=...)) -> JoinResult`
 * (/root/reference/pkg/src/tilejoin/join.py:150).  The reference is pure
 * Python/NumPy and has no FFI of its own; each entry point below names the
 * reference function whose work it replaces.  A maintainer binds it with
 * ctypes.
 *
 * Conventions
 *  - every call returns an int status: TJ_OK, or TJ_EINVAL (maps to
 *    tilejoin.errors.ValidationError), TJ_ECAPACITY (ResourceError),
 *    TJ_ECUDA / TJ_ENOMEM (RuntimeError).  Message text: tj_last_error().
 *  - pointers documented "device" are caller-owned CUDA device memory
 *    (torch tensors' data_ptr()); "host" pointers are plain host memory.
 *  - `stream` is a cudaStream_t passed as void*; calls that only enqueue work
 *    are asynchronous, calls documented "synchronous" block on the stream.
 *  - one tj_ctx per device.  A ctx is not thread-safe; distinct ctxs may be
 *    driven from distinct host threads.  The ctx owns the grid index, the
 *    pair-append buffer and all scratch.
 */
#ifndef TEDJOIN_H
#define TEDJOIN_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TJ_OK 0
#define TJ_EINVAL 1
#define TJ_ECAPACITY 2
#define TJ_ECUDA 3
#define TJ_ENOMEM 4

#define TJ_KERNEL_CORE 0 /* CUDA-core FP64 direct form, GDS-Join style ("scalar") */
#define TJ_KERNEL_DMMA 1 /* mma.sync m8n8k4 f64 expanded form, paper Alg. 2 ("tile") */
/* CUDA-core comparison kernels (same pair set; values near eps^2 re-decided exactly): */
#define TJ_KERNEL_CORE_FMA 2      /* direct form with fused multiply-add ("core_fma") */
#define TJ_KERNEL_CORE_EXPANDED 3 /* expanded form |q|^2+|c|^2-2q.c in DFMA ("core_expanded") */

/* Largest k_idx the device grid enumerates (3^(k-1) neighbour rows per cell). */
#define TJ_MAX_K_IDX 8
/* Largest logical dimensionality the refine kernels are instantiated for. */
#define TJ_MAX_DIM 128

typedef struct tj_ctx tj_ctx;

typedef struct {
  int64_t n;                /* points */
  int32_t d;                /* logical dimensionality */
  int32_t d_pad;            /* 4*ceil(d/4): row stride of the cell-ordered coordinates */
  int32_t k_idx;            /* indexed dimensions requested */
  int32_t key_bits;         /* bits of the packed cell key */
  double eps;               /* epsilon */
  double eps_sq;            /* fl(eps*eps), the join threshold (join.py:176) */
  int64_t n_cells;          /* non-empty cells (GridIndex.n_cells, grid.py:48-50) */
  int64_t n_runs;           /* contiguous candidate runs over all cells */
  int64_t candidates;       /* C = sum_cells |cell|*|cand(cell)| (JoinStats.candidates_refined) */
  int64_t tiles;            /* sum_cells ceil(|cell|/8)*ceil(|cand|/8) (join.py:257-261) */
  int64_t max_cell;         /* largest cell population */
} tj_grid_info;

typedef struct {
  int64_t tiles_processed;    /* DMMA kernel: 8x8 tiles evaluated            (join.py:270) */
  int64_t chunks_executed;    /* DMMA kernel: 4-dim chunks executed          (join.py:271) */
  int64_t chunks_skipped;     /* DMMA kernel: chunks skipped by short-circuit (join.py:272) */
  int64_t candidates_refined; /* candidate pairs refined                     (join.py:273) */
  int64_t pairs_emitted;      /* result pairs, self-pairs included           (join.py:207) */
  int64_t guard_rechecks;     /* DMMA pairs re-decided by the exact direct form */
} tj_stats;

/* ---- context ----------------------------------------------------------- */
int tj_version(void);
int tj_ctx_create(int device, tj_ctx** out);
void tj_ctx_destroy(tj_ctx* ctx);
/* Message of the last failed call on ctx (or of the last failed tj_ctx_create when ctx is NULL). */
const char* tj_last_error(const tj_ctx* ctx);

/* ---- grid index: replaces grid.build_index (grid.py:66-101) + kernels.precompute_chunk_norms
 *      (kernels.py:115-131) + candidates_for_cell for every cell (grid.py:121-133, join.py:169)
 *      + the per-cell estimate |cell|*|cand| (join.py:170-173).
 * coords: device, n rows of FP64 coordinates, row stride ld >= d doubles (the
 * reference Dataset.coords layout is ld = 4*ceil(d/4), datasets.py:46-48).  Only
 * the first d columns are read.  The grid keeps a cell-ordered zero-padded
 * copy, chunk norms, the non-empty cell table and the compacted candidate runs.
 * k_idx in [1, min(d, TJ_MAX_K_IDX)]; eps > 0 finite. */
int tj_build_grid(tj_ctx* ctx, const double* coords, int64_t n, int32_t d, int64_t ld,
                  int32_t k_idx, double eps, void* stream);
/* synchronous */
int tj_get_grid_info(tj_ctx* ctx, tj_grid_info* out);

/* Export the index to host arrays (synchronous).  Any pointer may be NULL.
 * point_order:  n      original ids in cell order (GridIndex.point_order, grid.py:94)
 * cell_start:   n_cells+1 offsets into point_order
 * cell_coords:  n_cells*k_idx int64 cell coordinates, lexicographic (GridIndex.ordered_cells)
 * cell_cands:   n_cells |cand(cell)|
 * cell_runs:    n_cells+1 offsets into runs
 * runs:         n_runs*2 uint32 [begin,end) ranges of cell-ordered positions */
int tj_grid_export(tj_ctx* ctx, uint32_t* point_order, int64_t* cell_start, int64_t* cell_coords,
                   int64_t* cell_cands, int64_t* cell_runs, uint32_t* runs);

/* ---- refine + emit: replaces the per-batch loop of self_join (join.py:184-202) with
 *      _TileRefiner/distance_tile_v2 (kernel=TJ_KERNEL_DMMA, join.py:238-283, kernels.py:184-263)
 *      or _ScalarRefiner (kernel=TJ_KERNEL_CORE, join.py:286-349).
 * Refines the query cells [cell_begin, cell_end) and appends their pairs to the
 * ctx result buffer.  Asynchronous. */
int tj_refine(tj_ctx* ctx, int32_t kernel, int32_t short_circuit, int64_t cell_begin,
              int64_t cell_end, void* stream);
/* Neighbour ids of the canonical output written as id_map[original id] (device
 * uint32[n] of the current grid, caller-owned, alive until the rows are built;
 * NULL = the original ids).  A multi-GPU shard passes its local -> global id map
 * (monotone, so rows stay sorted) and skips a remap pass over the rows.  Reset by
 * tj_build_grid. */
int tj_set_output_ids(tj_ctx* ctx, const uint32_t* id_map);
/* Low-d DMMA symmetric join (default off; TJ_SYMMETRIC=1 in the environment turns
 * the default on): the refine covers each cell's candidates from the cell itself
 * on, so every pair of neighbour cells is multiplied once, and the rows of a
 * cell's queries take their pairs with earlier cells from those cells' hit masks.
 * It needs every earlier cell refined in the same result set: callers refining a
 * cell range that does not start at cell 0 (the multi-GPU shards) turn it off.
 * Takes effect at the next tj_refine. */
int tj_set_symmetric(tj_ctx* ctx, int32_t on);
/* Symmetric low-d join over a cell range past cell 0 (a multi-GPU shard): refine
 * the earlier cells [cell_begin, cell_end) for their hit masks only -- their rows,
 * counts and stats are not part of the result set; the rows of the cells refined
 * next read their pairs with these cells from the masks.  No-op for other kernels
 * or with the symmetric join off.  Asynchronous. */
int tj_refine_masks(tj_ctx* ctx, int32_t kernel, int32_t short_circuit, int64_t cell_begin,
                    int64_t cell_end, void* stream);
/* Result pairs since the last tj_reset_results (synchronous).  The count is exact
 * even past the append buffer's capacity (CUDA-core and high-d DMMA kernels
 * append pairs; the low-d DMMA kernel records hit masks and never overflows);
 * *overflowed = 1 when appends were dropped -- the caller then rolls the batch
 * back (tj_rollback_results), grows the buffer (tj_reserve_results) and re-runs it
 * (the output-budget batcher of DeviceJoin.refine, join.py:184-202). */
int tj_result_count(tj_ctx* ctx, int64_t* total, int32_t* overflowed);
int tj_reset_results(tj_ctx* ctx, void* stream);
/* Sampled selectivity estimate for sizing the pair buffer (the output-budget
 * batcher): `samples` work items -- cells of [cell_begin, cell_end) drawn with
 * probability |cell|*|cand| (join.py:122-124), one query block at a random offset
 * against the cell's whole candidate list -- run on `kernel`'s refine kernel with
 * nothing stored; *pairs_per_candidate = result pairs / candidate pairs of the
 * sample.  Counters and per-query counts are left as they were.  Not for the low-d
 * DMMA kernel (hit masks, nothing to size).  Synchronous. */
int tj_estimate_pairs(tj_ctx* ctx, int32_t kernel, int64_t cell_begin, int64_t cell_end,
                      int32_t samples, uint64_t seed, double* pairs_per_candidate, void* stream);
/* Grow the pair append buffer to `pairs` entries, keeping what was appended so far. */
int tj_reserve_results(tj_ctx* ctx, int64_t pairs);
/* Snapshot the result counters (stream-ordered) before a batch ... */
int tj_checkpoint_results(tj_ctx* ctx, void* stream);
/* ... and undo that batch: counters back to the snapshot, the per-query counts of
 * the cells [cell_begin, cell_end) zeroed.  Asynchronous. */
int tj_rollback_results(tj_ctx* ctx, int64_t cell_begin, int64_t cell_end, void* stream);

/* Canonical output (replaces the concat + lexsort of join.py:203-204): CSR by
 * original query id with neighbour ids ascending.  offsets: device int64[n+1];
 * neighbors: device uint32[total].  Only rows of queries refined since the last
 * reset are non-empty.  Asynchronous. */
int tj_finalize(tj_ctx* ctx, int64_t* offsets, uint32_t* neighbors, void* stream);

/* tj_finalize in two steps, so the caller can copy the offsets to the host
 * (another stream) while the rows are built: tj_finalize_offsets writes
 * offsets (device int64[n+1]); tj_finalize_rows then writes the rows using
 * those offsets.  Asynchronous. */
int tj_finalize_offsets(tj_ctx* ctx, int64_t* offsets, void* stream);
int tj_finalize_rows(tj_ctx* ctx, const int64_t* offsets, uint32_t* neighbors, void* stream);

/* The rows of one of `chunks` (<= 256) equal original-id ranges only: chunk j
 * covers ids [ceil(j n / chunks), ceil((j+1) n / chunks)), one contiguous part of
 * the CSR (offsets from tj_finalize_offsets).  Once the stream passes this call
 * the part is final, so a caller copies it to the host while the next chunk is
 * built (the chunked, pinned result pipeline of DeviceJoin.finalize_fetch).  Low-d
 * DMMA results are emitted per chunk from the hit masks; for other kernels the
 * first call builds every row.  Asynchronous. */
int tj_finalize_rows_chunk(tj_ctx* ctx, const int64_t* offsets, uint32_t* neighbors,
                           int32_t chunk, int32_t chunks, void* stream);

/* Counters accumulated since the last tj_reset_results (synchronous). */
int tj_get_stats(tj_ctx* ctx, tj_stats* out);

/* Per-cell cost |cell|*|cand(cell)| to host (synchronous); feeds plan_batches
 * (join.py:114-147) and the multi-GPU cost-balanced cell split. */
int tj_cell_costs(tj_ctx* ctx, int64_t* costs);

/* ---- callers either side of the path --------------------- */
/* Canonical squared distance of every emitted pair, for the pairs file
 * (cli._canonical_pair_sq_dists + _write_pairs, cli.py:270-289): out[e] = the
 * direct form sum over ascending dims of fl(fl(x_i - x_j)^2) for the e-th pair
 * (i, neighbors[e]) of the CSR.  coords: device, original point order, row
 * stride ld; offsets: device int64[n+1]; neighbors: device uint32[m]; out:
 * device double[m].  Asynchronous. */
int tj_pair_sq_dists(tj_ctx* ctx, const double* coords, int64_t ld, int32_t d,
                     const int64_t* offsets, int64_t n, const uint32_t* neighbors, int64_t m,
                     double* out, void* stream);

/* Write the pairs file: one "i j sq" line per CSR pair, sq formatted like
 * Python's f"{sq:.17g}" (cli._write_pairs, cli.py:285-289).  All pointers are
 * host arrays (offsets int64[n+1], neighbors uint32[offsets[n]], sq double[..]);
 * `threads` host threads format blocks in parallel.  Synchronous. */
int tj_write_pairs(const char* path, const int64_t* offsets, int64_t n,
                   const uint32_t* neighbors, const double* sq, int32_t threads);

/* JoinResult.pairs (join.py:80-91): expand the CSR into (query id, neighbour id)
 * int64 rows, out[2e] = row, out[2e+1] = neighbors[e].  Host arrays (offsets
 * int64[n+1], neighbors uint32[offsets[n]], out int64[2*offsets[n]]); `threads`
 * host threads write disjoint row ranges.  Synchronous. */
int tj_expand_pairs(const int64_t* offsets, int64_t n, const uint32_t* neighbors, int64_t* out,
                    int32_t threads);

/* Per-column mean and variance of coords (device, n rows, stride ld, first d
 * columns) into host arrays mean[d], var[d] (synchronous).  Feeds the variance
 * dimension reordering (datasets.reorder_dims_by_variance, datasets.py:113-123);
 * compensated summation: accurate to a few ulp, order-independent. */
int tj_column_moments(tj_ctx* ctx, const double* coords, int64_t n, int32_t d, int64_t ld,
                      double* mean, double* var, void* stream);
/* dst[:, j] = src[:, perm[j]] for j < d, zero for d <= j < ld_out.  src/dst
 * device (distinct buffers), perm host int32[d].  Synchronous. */
int tj_permute_columns(tj_ctx* ctx, const double* src, int64_t n, int32_t d, int64_t ld,
                       const int32_t* perm, double* dst, int64_t ld_out, void* stream);

/* Brute-force self-join over all n^2 ordered pairs with the reference direct
 * form (oracle.brute_force_join, oracle.py:55-86): the GPU verification oracle
 * of cli verify for n beyond the CPU guard.  Two calls: with neighbors == NULL
 * it fills offsets (device int64[n+1]) and *total (host); then with a device
 * uint32[*total] buffer it writes the rows (ascending).  d <= 128. */
int tj_brute_force(tj_ctx* ctx, const double* coords, int64_t n, int32_t d, int64_t ld,
                   double eps, int64_t* offsets, uint32_t* neighbors, int64_t* total,
                   void* stream);

/* ---- page-locked host memory ---------------------------------------------------- */
/* Page-lock a host range (cudaHostRegister, portable; mapped != 0 also maps it
 * into the device address space and returns the device alias in *device_ptr,
 * which may be NULL).  A range that is already page-locked is accepted as is;
 * failures never leave a stale CUDA error behind.  Synchronous. */
int tj_host_register(void* ptr, int64_t bytes, int32_t mapped, void** device_ptr);
int tj_host_unregister(void* ptr);

/* ---- multi-GPU strong layout: cell-partitioned shards of one join ----------------
 * Replaces the reference's data-parallel executor (join.py:184-197, a thread pool
 * over a batch's cells) with one process per GPU owning a contiguous, cost-balanced
 * range of the lexicographic cell order.  Bins are the first
 * `pdims` (1 or 2) indexed dims of a point's cell, b_j = floor(x_j/eps) - origin[j]
 * (grid.py:81), numbered L = b_0*span[1] + b_1; a rank owns bins [own_lo, own_hi]
 * (inclusive).  origin/span are host arrays of pdims entries. */
/* floor(x_j/eps) bounds of coords (device rows, stride ld) -> host lo[pdims],
 * hi[pdims].  Synchronous. */
int tj_shard_bounds(tj_ctx* ctx, const double* coords, int64_t n, int64_t ld, int32_t pdims,
                    double eps, int64_t* lo, int64_t* hi, void* stream);
/* Points per bin -> device int64 hist[span0*span1] (zeroed first): the estimator's
 * input (join.py:122-124) at bin granularity.  Asynchronous. */
int tj_shard_histogram(tj_ctx* ctx, const double* coords, int64_t n, int64_t ld, int32_t pdims,
                       double eps, const int64_t* origin, const int64_t* span, int64_t* hist,
                       void* stream);
/* Stable compaction of the points a rank needs: those whose bin is within
 * Chebyshev distance 1 of an owned bin (its cells' candidates, grid.py:104-133).
 * out: device (capacity, ld_out) f64, columns >= d zeroed; gid: device uint32
 * (gid_base + row index of each kept point).  out == NULL only counts.
 * *selected = kept points.  Synchronous. */
int tj_shard_select(tj_ctx* ctx, const double* coords, int64_t n, int64_t ld, int32_t d,
                    int32_t pdims, double eps, const int64_t* origin, const int64_t* span,
                    int64_t own_lo, int64_t own_hi, double* out, int64_t ld_out, uint32_t* gid,
                    int64_t gid_base, int64_t capacity, int64_t* selected, void* stream);
/* Route this rank's rows to `ranks` (<= 64) ranks (rank r owns bins [own_lo[r],
 * own_hi[r]]): a row goes to every rank whose bins or one-cell halo hold it.
 * out == NULL: one pass, counts[r] = rows for rank r (host int64[ranks];
 * synchronous), the rows' destination sets kept in the ctx.  Otherwise (right
 * after that call, same rows and counts): the rows for rank r, stably compacted, at row
 * sum(counts[<r]) of out (device (capacity, ld_out) f64) with gid_base + index in
 * gid; asynchronous.  The send side of the shard exchange (one all-to-all). */
int tj_shard_route(tj_ctx* ctx, const double* coords, int64_t n, int64_t ld, int32_t d,
                   int32_t pdims, double eps, const int64_t* origin, const int64_t* span,
                   const int64_t* own_lo, const int64_t* own_hi, int32_t ranks, int64_t* counts,
                   double* out, int64_t ld_out, uint32_t* gid, int64_t gid_base, int64_t capacity,
                   void* stream);
/* The owned cells [*cell_begin, *cell_end) of the grid built on ctx (lexicographic
 * cell order, so contiguous).  Synchronous. */
int tj_shard_cell_range(tj_ctx* ctx, int32_t pdims, const int64_t* origin, const int64_t* span,
                        int64_t own_lo, int64_t own_hi, int64_t* cell_begin, int64_t* cell_end);
/* ids[e] = gid[ids[e]] (device arrays): local neighbour ids -> global ids.  Async. */
int tj_remap_ids(tj_ctx* ctx, uint32_t* ids, int64_t m, const uint32_t* gid, void* stream);
/* counts[gid[l]] = offsets[l+1] - offsets[l] for the non-empty local rows (device).
 * Summing the ranks' count arrays gives the global per-id counts.  Async. */
int tj_scatter_counts(tj_ctx* ctx, const int64_t* offsets, int64_t n_rows, const uint32_t* gid,
                      int32_t* counts, void* stream);
/* offsets[0..n] = exclusive prefix sum of counts[0..n-1] (device).  Async. */
int tj_counts_to_offsets(tj_ctx* ctx, const int32_t* counts, int64_t n, int64_t* offsets,
                         void* stream);
/* The same exchange with one byte per id: counts[gid[l]] = min(row length, 255)
 * and *overflow |= 1 when a row is longer (device int32, zeroed by the caller;
 * any overflow on any rank -> use the int32 pair above).  The all-reduce of the
 * counts then moves n bytes instead of 4n.  Async. */
int tj_scatter_counts_u8(tj_ctx* ctx, const int64_t* offsets, int64_t n_rows, const uint32_t* gid,
                         uint8_t* counts, int32_t* overflow, void* stream);
int tj_counts_u8_to_offsets(tj_ctx* ctx, const uint8_t* counts, int64_t n, int64_t* offsets,
                            void* stream);
/* Copy every non-empty local row l (neighbors already global ids) to
 * dst[global_offsets[gid[l]] ...]; dst may be device memory or mapped pinned
 * host memory (cudaHostRegisterMapped), so ranks write one shared host CSR.  Async. */
int tj_place_rows(tj_ctx* ctx, const int64_t* offsets, const uint32_t* neighbors, int64_t n_rows,
                  const uint32_t* gid, const int64_t* global_offsets, uint32_t* dst, void* stream);

/* ---- measurement helpers ------------------------------------------------ */
/* FP64 throughput microbenchmark on the current device: kind 0 = DFMA,
 * 1 = DMMA m8n8k4, 2 = both interleaved.  Reports FLOP/s counting 2 per FMA. */
int tj_fp64_peak(int32_t kind, int32_t iters, double* tflops, double* ms);
/* One m8n8k4 f64 MMA on device; A 8x4, B 4x8, C/D 8x8 row-major host arrays. */
int tj_dmma_known_answer(const double* a, const double* b, const double* c, double* d);
/* Average duration (ms) of the last tj_refine launch's refine kernel, measured
 * with CUDA events on the launching stream (synchronous). */
int tj_last_refine_ms(tj_ctx* ctx, double* ms);
/* Duration (ms) of the last low-d row-emission kernel (emit_rows_kernel, the canonical
 * output's dominant kernel), CUDA events on its stream (synchronous). */
int tj_last_emit_ms(tj_ctx* ctx, double* ms);
/* Kernels this library has launched so far in the process (all contexts). */
int64_t tj_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* TEDJOIN_H */
