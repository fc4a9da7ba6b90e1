// Library-internal declarations: the context, device buffers, work items and
// the host-side launchers shared between translation units.
#pragma once
#include <algorithm>
#include <string>
#include <vector>

#include "common.cuh"

namespace tj {

struct ScanScratch;

// Grow-only device buffer on the stream-ordered allocator.
struct DevBuf {
  void* ptr = nullptr;
  size_t bytes = 0;
  template <class T>
  T* as() const {
    return static_cast<T*>(ptr);
  }
  void ensure(size_t need, cudaStream_t s) {
    if (need <= bytes) return;
    if (ptr) TJ_CUDA(cudaFreeAsync(ptr, s));
    ptr = nullptr;
    bytes = 0;
    size_t want = std::max<size_t>(need, 256);
    cudaError_t e = cudaMallocAsync(&ptr, want, s);
    if (e != cudaSuccess) {
      (void)cudaGetLastError();
      ptr = nullptr;
      fail(TJ_ENOMEM, "device allocation of " + std::to_string(want) + " bytes failed: " +
                          cudaGetErrorString(e));
    }
    bytes = want;
  }
  void release(cudaStream_t s) {
    if (ptr) cudaFreeAsync(ptr, s);
    ptr = nullptr;
    bytes = 0;
  }
};

// One unit of refine work: queries [q0, q0+nq) (cell-ordered positions, all in
// `cell`) against the candidate slice [s0, s1) of that cell's concatenated
// candidate list (grid.py:121-133 order).  s0 is a multiple of 8 so 8-candidate
// tiles line up with the reference's tiling of the concatenation (join.py:261).
struct WorkItem {
  uint32_t cell;
  uint32_t q0;
  uint32_t nq;
  uint32_t s0;
  uint32_t s1;
  uint32_t pad;
};

// Device-side counters, one struct per ctx.
struct DevCounters {
  unsigned long long pairs;         // appended pairs (keeps counting past capacity)
  unsigned long long tiles;         // DMMA tiles evaluated
  unsigned long long chunks_exec;   // DMMA chunks executed
  unsigned long long chunks_skip;   // DMMA chunks skipped by the short-circuit
  unsigned long long refined;       // candidate pairs refined
  unsigned long long rechecks;      // guard-band rechecks
  unsigned long long item_next;     // persistent-kernel work counter
  unsigned long long hits;          // pairs recorded as low-d hit masks
  unsigned long long max_row;       // longest low-d row (count_rows_kernel)
  unsigned long long n_items;       // work items of the current launch (device-side count)
};

// Low-d output: one 64-bit hit mask per (query group, 8-candidate block) tile,
// dense per cell (see build_mask_bases).  Bit L (< 32) = pair (query 2*(L&3),
// candidate L>>2) of the tile, bit 32 + L = pair (query 2*(L&3) + 1, candidate L>>2).

// Everything a refine kernel needs, passed by value.
struct RefineArgs {
  const double* P;         // (n, d_pad) cell-ordered coordinates
  const double* NRM;       // (n) squared norms (any rounding order; the guard covers it)
  const double* CN;        // (n, nchunks) chunk norms, reference order (kernels.py:126-130)
  const double* SFX;       // (n, 2): chunk-norm suffix after the short-circuit check, |c|^2
  const uint2* runs;       // (n_runs) candidate position ranges [begin, end)
  const uint32_t* run_off; // (n_runs) offset of each run inside its cell's concatenation
  const int64_t* cell_runs;   // (n_cells+1)
  const int64_t* cell_start;  // (n_cells+1)
  const WorkItem* items;
  int64_t n_items;                       // item count, or an upper bound when n_items_dev is set
  const unsigned long long* n_items_dev; // exact count on the device (nullptr: n_items is exact)
  DevCounters* ctr;
  uint2* pairs;            // append buffer of (query pos, candidate pos)
  unsigned long long pair_cap;
  uint32_t* qcount;        // (n) per-query pair counts (cell-ordered positions)
  unsigned long long* masks;     // low-d hit masks
  const int64_t* cell_mbase;     // first mask of cell c at cell_mbase[c - cell_base]
  int64_t cell_base;
  const uint32_t* fwd;           // low-d symmetric join: first candidate offset refined per cell
                                 // (the cell's own position in its list); nullptr = 0
  int d, d_pad, nchunks;
  double eps_sq;
  double guard_rel;        // guard band = guard_rel * (qn + max_norm)
  double max_norm;
  int short_circuit;
};

struct GridState {
  bool built = false;
  int64_t n = 0;
  int d = 0, d_pad = 0, k = 0, nchunks = 0;
  double eps = 0, eps_sq = 0;
  int key_bits = 0;
  // cell keys wider than 63 bits: two words, dims [0, split) in the high word
  bool wide = false;
  int lo_bits = 0, hi_bits = 0;
  int bits[TJ_MAX_K_IDX] = {};
  int word[TJ_MAX_K_IDX] = {};     // 0: low word, 1: high word
  int shift[TJ_MAX_K_IDX] = {};    // inside the dim's word
  int64_t cmin[TJ_MAX_K_IDX] = {};
  int64_t n_cells = 0, n_runs = 0, candidates = 0, tiles = 0, max_cell = 0;
  double max_norm = 0;
};

}  // namespace tj

struct tj_ctx {
  int device = 0;
  std::string err;
  cudaStream_t last_stream = nullptr;
  tj::GridState g;
  // grid buffers
  tj::DevBuf P, NRM, CN, perm, keys, keys_hi, cell_key, cell_key_hi, cell_start, cell_runs, runs, run_off, cell_cand,
      cell_cost, dense, SFX;
  // scratch
  tj::DevBuf keys_alt, vals_alt, sort_hist, scan_partial, scan_total, minmax, tmp64, items;
  // results
  tj::DevBuf pairs, qcount, counters, fill, masks, cell_mbase, win_cell;
  // low-d symmetric join: per-cell forward offset, backward-cell table (CSR by cell)
  tj::DevBuf fwd, bt_start, bt, bt_desc;
  // output id map (tj_set_output_ids): neighbour ids written as out_ids[original id]
  const uint32_t* out_ids = nullptr;
  tj::DevBuf route_dest;   // shard_route: destination mask of each routed row
  tj::DevBuf route_tiles;  // shard_route: per (destination, warp tile) counts -> offsets
  tj::DevBuf nid;
  bool nid_ready = false;
  bool symmetric = true;
  tj::DevBuf pos_off, rows_tmp;  // finalize: rows in cell (position) order before the sort
  tj::DevBuf ipos, pcell;        // id-range position lists (2 x n: sort ping-pong), position -> cell
  tj::DevBuf chunk_key;          // sort keys of the position lists
  int64_t chunk_pos_off = 0;     // which half of ipos holds the sorted lists
  int chunk_lists = 0;           // id ranges the lists were built for
  bool id_maps_ready = false;    // lists / pcell built for the current grid
  bool rows_range_done = false;  // pair-path rows built by an earlier range call
  unsigned long long pair_cap = 0;
  int64_t mask_cells_begin = 0, mask_cells_end = 0;  // cells whose masks are in `masks`
  int64_t n_items = 0;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  cudaEvent_t ev2 = nullptr, ev3 = nullptr;  // around the last row-emission kernel
  bool have_refine_timing = false;
  bool have_emit_timing = false;
  bool masks_ready = false;  // low-d mask layout built for the current grid
  bool ctr_valid = false;    // `ctr` holds the device counters (no refine since the read)
  tj::DevCounters ctr{};
};

namespace tj {
// sort.cu
int64_t radix_sort_scratch_elems(int64_t n);
int radix_sort_pairs(uint64_t* k0, uint32_t* v0, uint64_t* k1, uint32_t* v1, int64_t n,
                     int key_bits, bool identity_values, int64_t* hist, ScanScratch scan,
                     cudaStream_t stream);
int radix_sort_pairs32(uint32_t* k0, uint32_t* v0, uint32_t* k1, uint32_t* v1, int64_t n,
                       int key_bits, bool identity_values, int64_t* hist, ScanScratch scan,
                       cudaStream_t stream);
// grid.cu
void build_grid(tj_ctx* ctx, const double* coords, int64_t n, int d, int64_t ld, int k,
                double eps, cudaStream_t s);
int64_t build_work_items(tj_ctx* ctx, int64_t cell_begin, int64_t cell_end, int q_per_item,
                         int64_t slice, cudaStream_t s, unsigned long long* total_dev = nullptr);
ScanScratch scan_scratch(tj_ctx* ctx, int64_t n, cudaStream_t s);
void build_mask_bases(tj_ctx* ctx, int64_t cell_begin, int64_t cell_end, cudaStream_t s);
// refine_core.cu / refine_dmma.cu
// variant: 0 exact reference order, 1 FMA direct form, 2 expanded form (refine_core.cu)
void launch_refine_core(const RefineArgs& a, int variant, cudaStream_t s);
void launch_refine_tc(const RefineArgs& a, int64_t n, int64_t n_cells,
                      cudaStream_t s);  // DMMA, 5 <= d <= 64
void launch_refine_lowd(const RefineArgs& a, int64_t n, int64_t n_cells,
                        cudaStream_t s);  // d <= 4, unsliced items
int lowd_queries_per_item(int64_t n, int64_t n_cells);
// refine_gram.cu: CTA-blocked DMMA for big cells at d_pad >= 12
constexpr int kGramQueries = 64;
constexpr int64_t kGramSlice = 32768;
bool gram_applies(int d_pad, int64_t n, int64_t n_cells);
void launch_refine_gram(const RefineArgs& a, bool cuda_cores, cudaStream_t s);
int core_queries_per_item(int d, int d_pad);
int tc_queries_per_item(int d_pad, int64_t n, int64_t n_cells);
// finalize.cu
// output.cu / reorder.cu / verify.cu
void launch_pair_sq_dists(const double* x, int64_t ld, int d, const int64_t* offsets, int64_t n,
                          const uint32_t* nbr, int64_t m, double* out, cudaStream_t s);
void write_pairs_file(const char* path, const int64_t* offsets, int64_t n, const uint32_t* nbr,
                      const double* sq, int threads);
void expand_pairs(const int64_t* offsets, int64_t n, const uint32_t* nbr, int64_t* out,
                  int threads);
void column_moments(tj_ctx* ctx, const double* x, int64_t n, int d, int64_t ld, double* h_mean,
                    double* h_var, cudaStream_t s);
void permute_columns(const double* src, int64_t n, int d, int64_t ld, const int* h_perm,
                     double* dst, int64_t ld_out, cudaStream_t s);
void brute_force_join(tj_ctx* ctx, const double* x, int64_t n, int d, int64_t ld, double eps,
                      int64_t* offsets, uint32_t* nbr, int64_t* total, cudaStream_t s);
void build_window_cells(tj_ctx* ctx, cudaStream_t s);
void build_symmetric_tables(tj_ctx* ctx, cudaStream_t s);
void build_bt_desc(tj_ctx* ctx, cudaStream_t s);
// shard.cu (multi-GPU strong layout)
void shard_bounds(tj_ctx* ctx, const double* x, int64_t n, int64_t ld, int pdims, double eps,
                  int64_t* lo, int64_t* hi, cudaStream_t s);
void shard_histogram(const double* x, int64_t n, int64_t ld, int pdims, double eps,
                     const int64_t* origin, const int64_t* span, int64_t* hist, cudaStream_t s);
int64_t shard_select(tj_ctx* ctx, const double* x, int64_t n, int64_t ld, int d, int pdims,
                     double eps, const int64_t* origin, const int64_t* span, int64_t own_lo,
                     int64_t own_hi, double* out, int64_t ld_out, uint32_t* gid, int64_t gid_base,
                     int64_t capacity, cudaStream_t s);
void shard_route(tj_ctx* ctx, const double* x, int64_t n, int64_t ld, int d, int pdims, double eps,
                 const int64_t* origin, const int64_t* span, const int64_t* lo, const int64_t* hi,
                 int G, int64_t* counts, double* out, int64_t ld_out, uint32_t* gid,
                 int64_t gid_base, int64_t capacity, cudaStream_t s);
void shard_cell_range(tj_ctx* ctx, int pdims, const int64_t* origin, const int64_t* span,
                      int64_t own_lo, int64_t own_hi, int64_t* begin, int64_t* end, cudaStream_t s);
void shard_remap_ids(uint32_t* ids, int64_t m, const uint32_t* gid, cudaStream_t s);
void shard_scatter_counts(const int64_t* loff, int64_t n_rows, const uint32_t* gid, int32_t* counts,
                          cudaStream_t s);
void shard_place_rows(const int64_t* loff, const uint32_t* nbr, int64_t n_rows, const uint32_t* gid,
                      const int64_t* goff, uint32_t* dst, cudaStream_t s);
void counts_to_offsets(tj_ctx* ctx, const int32_t* counts, int64_t n, int64_t* offsets,
                       cudaStream_t s);
void shard_scatter_counts_u8(const int64_t* loff, int64_t n_rows, const uint32_t* gid,
                             uint8_t* counts, int32_t* overflow, cudaStream_t s);
void counts_to_offsets_u8(tj_ctx* ctx, const uint8_t* counts, int64_t n, int64_t* offsets,
                          cudaStream_t s);
void launch_count_rows(tj_ctx* ctx, int64_t cb, int64_t ce, unsigned long long* hits,
                       unsigned long long* max_row, cudaStream_t s);
void finalize_csr(tj_ctx* ctx, int64_t* offsets, uint32_t* neighbors, int64_t n_pairs,
                  int64_t n_mask_hits, int64_t max_mask_row, cudaStream_t s, int phase = 3);
void finalize_rows_range(tj_ctx* ctx, const int64_t* offsets, uint32_t* nbr, int64_t n_pairs,
                         int64_t n_mask_hits, int64_t max_mask_row, int chunk, int chunks,
                         cudaStream_t s);
}  // namespace tj
