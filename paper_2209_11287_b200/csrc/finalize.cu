// Canonical output: CSR by original query id with neighbour ids ascending.
//
// Replaces the concatenate + np.lexsort((j, i)) of join.py:203-204.  Per-query
// pair counts (cell-ordered positions) move to original-id order and are
// scanned into int64 row offsets; a second scan in position order gives every
// row a contiguous slot range in a cell-ordered staging array.  Then:
//  * low-d path (hit masks, refine_lowd.cu): emit_rows_kernel expands the masks
//    of 32 consecutive query positions straight into a shared-memory pool,
//    sorts one row per lane in registers and writes the rows to their places;
//  * pair path (other kernels): every (query, candidate) pair is scattered to
//    a staging row in cell order through a per-row atomic cursor (a second
//    scan in position order places the rows), then sort_rows_kernel reads 32
//    consecutive staging rows (coalesced), sorts one row per lane and writes
//    each row to its final place.
//  Rows longer than 88 ids are sorted in place by a warp (<= 256), one CTA
//  (shared-memory bitonic, <= 8192) or, beyond that, by a composite-key radix
//  sort.
#include "internal.cuh"
#include "scan.cuh"

namespace tj {

__global__ void counts_to_orig_kernel(const uint32_t* __restrict__ qcount,
                                      const uint32_t* __restrict__ perm, int64_t n,
                                      int64_t* __restrict__ cnt_orig) {
  for (int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p < n;
       p += int64_t(gridDim.x) * blockDim.x)
    cnt_orig[perm[p]] = qcount[p];
}

// Pair path: (query position, candidate position) -> the query's row in cell
// (position) order through a per-row atomic cursor; ids are original ids.
__global__ void scatter_pairs_kernel(const uint2* __restrict__ pairs, int64_t total,
                                     const uint32_t* __restrict__ nid,
                                     const int64_t* __restrict__ pos_off,
                                     uint32_t* __restrict__ fill, uint32_t* __restrict__ rows) {
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const uint2 pr = pairs[e];
    const uint32_t slot = atomicAdd(&fill[pr.x], 1u);
    rows[pos_off[pr.x] + slot] = nid[pr.y];
  }
}

// Bitonic sort of 32*R keys held as v[r] (element index r*32 + lane), ascending.
template <int R>
__device__ __forceinline__ void warp_bitonic(uint32_t (&v)[R]) {
  const int lane = lane_id();
  constexpr int N = 32 * R;
#pragma unroll
  for (int k = 2; k <= N; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j >= 32) {
        const int rj = j >> 5;
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int p = r ^ rj;
          if (p > r) {
            const int i = r * 32 + lane;
            const bool asc = (i & k) == 0;
            const uint32_t a = v[r], b = v[p];
            const bool swap = asc ? (a > b) : (a < b);
            v[r] = swap ? b : a;
            v[p] = swap ? a : b;
          }
        }
      } else {
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int i = r * 32 + lane;
          const bool asc = (i & k) == 0;
          const uint32_t o = __shfl_xor_sync(0xffffffffu, v[r], j);
          const bool lower = (lane & j) == 0;
          // lower element keeps min when ascending, max when descending
          const uint32_t mn = min(v[r], o), mx = max(v[r], o);
          v[r] = (lower == asc) ? mn : mx;
        }
      }
    }
  }
}

template <int R>
__device__ __forceinline__ void warp_sort_row(uint32_t* row, int len) {
  uint32_t v[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int i = r * 32 + lane_id();
    v[r] = i < len ? row[i] : 0xffffffffu;
  }
  warp_bitonic<R>(v);
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int i = r * 32 + lane_id();
    if (i < len) row[i] = v[r];
  }
}

constexpr int kWarpSortMax = 1024;
constexpr int kBlockSortMax = 8192;

// ---------------------------------------------------------------- row batches
// Short rows are sorted one per lane: a warp holds up to 32 rows in a
// transposed shared-memory pool (slot i of column c at pool[i * kPoolLd + c];
// the odd leading dimension keeps both the per-lane column walk and the
// per-row copy-out conflict-free), each lane pulls its row into registers and
// runs Batcher's odd-even merge sort on them.  The network is a compile-time
// constant; slots past the row end hold 0xffffffff, so every comparator that
// touches the padding folds away and a network of N slots costs only its
// data-dependent min/max pairs (N = 64: 543 comparators, ~34 warp
// instructions per row when the warp is full) -- versus ~300 for a warp-wide
// bitonic sort of the same row.
constexpr int kPoolSlots = 88;
constexpr int kPoolLd = 33;

// Comparator list of Batcher's odd-even merge sort for N keys (the network of
// the next power of two restricted to the first N slots), built at compile time.
template <int N>
struct OemNet {
  static constexpr int NP = N <= 16 ? 16 : N <= 32 ? 32 : N <= 64 ? 64 : 128;
  template <typename F>
  __host__ __device__ static constexpr void walk(F&& f) {
    for (int p = 1; p < NP; p <<= 1)
      for (int k = p; k >= 1; k >>= 1)
        for (int j = k % p; j + k < NP; j += 2 * k)
          for (int i = 0; i < k; ++i) {
            const int x = i + j, y = i + j + k;
            if (y < N && (x / (2 * p)) == (y / (2 * p))) f(x, y);
          }
  }
  __host__ __device__ static constexpr int count() {
    int c = 0;
    walk([&](int, int) { ++c; });
    return c;
  }
  static constexpr int C = count();
  struct List {
    unsigned char x[C], y[C];
  };
  __host__ __device__ static constexpr List list() {
    List l{};
    int c = 0;
    walk([&](int x, int y) {
      l.x[c] = (unsigned char)x;
      l.y[c] = (unsigned char)y;
      ++c;
    });
    return l;
  }
};

template <int N>
__device__ __forceinline__ void oem_sort(uint32_t (&v)[N]) {
  constexpr auto net = OemNet<N>::list();
#pragma unroll
  for (int t = 0; t < OemNet<N>::C; ++t) {
    const uint32_t a = v[net.x[t]], b = v[net.y[t]];
    v[net.x[t]] = min(a, b);
    v[net.y[t]] = max(a, b);
  }
}

template <int N>
__device__ __noinline__ void pool_sort_n(uint32_t* pool, int len) {
  const int lane = lane_id();
  uint32_t v[N];
#pragma unroll
  for (int i = 0; i < N; ++i) v[i] = i < len ? pool[i * kPoolLd + lane] : 0xffffffffu;
  oem_sort<N>(v);
#pragma unroll
  for (int i = 0; i < N; ++i)
    if (i < len) pool[i * kPoolLd + lane] = v[i];
}

// Sort column `lane` of the pool (len <= kPoolSlots ids; 0 = no row).
__device__ __noinline__ void pool_sort(uint32_t* pool, int len) {
  int mx = len;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (mx <= 1) return;
  // three network sizes only: warps of one launch mostly share one network, so
  // the straight-line code stays resident in the instruction cache
  if (mx <= 32) pool_sort_n<32>(pool, len);
  else if (mx <= 64) pool_sort_n<64>(pool, len);
  else pool_sort_n<88>(pool, len);
}

// Rows with more than kPoolSlots ids are written straight to their place and
// sorted there: by the warp (<= kWarpSortMax) or listed for the CTA/radix path.
__device__ __noinline__ void sort_long_row(uint32_t* row, int len, uint32_t id, uint32_t* big_rows,
                                           unsigned long long* n_big) {
  if (len <= 128) warp_sort_row<4>(row, len);
  else if (len <= 256) warp_sort_row<8>(row, len);
  else if (len <= 512) warp_sort_row<16>(row, len);
  else if (len <= kWarpSortMax) warp_sort_row<32>(row, len);
  else if (lane_id() == 0) big_rows[atomicAdd(n_big, 1ull)] = id;
}

// Rows in cell order -> final CSR.  Warp per 32 consecutive query positions:
// their rows are one contiguous segment of `rows` (position-order offsets
// pos_off), read row by row with 16 rows' loads in flight before their
// shared-memory stores into the rows' pool columns.  Each lane then sorts one
// row in registers (odd-even merge network) and the warp writes the sorted rows
// to their places.  Rows longer than kPoolSlots are copied to their place and
// sorted there (warp bitonic <= kWarpSortMax, else listed for the CTA / radix
// path).
constexpr int kSortWarps = 4;
constexpr int kSortGroup = 16;  // rows loaded per group

__global__ void __launch_bounds__(kSortWarps * 32)
    sort_rows_kernel(const int64_t* __restrict__ pos_off, const uint32_t* __restrict__ rows,
                     const uint32_t* __restrict__ perm, const int64_t* __restrict__ offsets,
                     int64_t n, uint32_t* __restrict__ nbr, uint32_t* __restrict__ big_rows,
                     unsigned long long* n_big) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = lane_id();
  uint32_t* pool = reinterpret_cast<uint32_t*>(smem_raw) + warp * kPoolSlots * kPoolLd;
  const int64_t warps = int64_t(gridDim.x) * kSortWarps;
  for (int64_t p0 = (int64_t(blockIdx.x) * kSortWarps + warp) * 32; p0 < n; p0 += warps * 32) {
    const int64_t p = p0 + lane;
    const int64_t src = p < n ? pos_off[p] : 0;
    const int len = p < n ? int(pos_off[p + 1] - src) : 0;
    const uint32_t id = p < n ? perm[p] : 0u;
    const int64_t dst = p < n ? offsets[id] : 0;
    const int nrows = int(min(int64_t(32), n - p0));
    __syncwarp();
    for (int k0 = 0; k0 < nrows; k0 += kSortGroup) {
      uint32_t v[kSortGroup][3];
#pragma unroll
      for (int kk = 0; kk < kSortGroup; ++kk) {
        const int L = __shfl_sync(0xffffffffu, len, (k0 + kk) & 31);
        const int64_t S = __shfl_sync(0xffffffffu, src, (k0 + kk) & 31);
        const bool ok = k0 + kk < nrows && L <= kPoolSlots;
#pragma unroll
        for (int t = 0; t < 3; ++t) {
          const int e = lane + 32 * t;
          v[kk][t] = (ok && e < L) ? __ldg(rows + S + e) : 0u;
        }
      }
#pragma unroll
      for (int kk = 0; kk < kSortGroup; ++kk) {
        const int L = __shfl_sync(0xffffffffu, len, (k0 + kk) & 31);
        const bool ok = k0 + kk < nrows && L <= kPoolSlots;
#pragma unroll
        for (int t = 0; t < 3; ++t) {
          const int e = lane + 32 * t;
          if (ok && e < L) pool[e * kPoolLd + k0 + kk] = v[kk][t];
        }
      }
    }
    __syncwarp();
    pool_sort(pool, len <= kPoolSlots ? len : 0);
    __syncwarp();
    for (int k = 0; k < nrows; ++k) {
      const int L = __shfl_sync(0xffffffffu, len, k);
      const int64_t D = __shfl_sync(0xffffffffu, dst, k);
      if (L <= kPoolSlots) {
        for (int e = lane; e < L; e += 32) nbr[D + e] = pool[e * kPoolLd + k];
      } else {
        const int64_t S = __shfl_sync(0xffffffffu, src, k);
        for (int e = lane; e < L; e += 32) nbr[D + e] = rows[S + e];
        __syncwarp();
        sort_long_row(nbr + D, L, __shfl_sync(0xffffffffu, id, k), big_rows, n_big);
      }
    }
  }
}

// ------------------------------------------------------------ low-d masks
// Rows of the low-d path are read straight out of the refine kernel's hit
// masks.  Query position p of cell c sits in group g = (p - cs) / 8 of its
// cell, column (p - cs) % 8; its hits against block b are the bits
// 4r + col/2 (+32 for odd columns) of mask (g, b), i.e. candidate 8b + r of
// the cell's concatenated list.  Every kernel below walks windows of 32
// consecutive positions, lane j = position 32w + j.

// Cell of this lane's position: c0 = cell containing the window start; the
// cells starting inside the window are found with one load per lane.
__device__ __forceinline__ int64_t window_lane_cell(const int64_t* __restrict__ cell_start,
                                                    int64_t n_cells, int64_t c0, int64_t p0) {
  const int lane = lane_id();
  const int64_t cl = c0 + lane;
  const int64_t cs_l = cl <= n_cells ? cell_start[cl] : INT64_MAX;
  const int64_t off = cs_l - p0;
  const unsigned bit = (off >= 0 && off < 32) ? (1u << unsigned(off)) : 0u;
  const unsigned starts = __reduce_or_sync(0xffffffffu, bit);
  const unsigned upto = (2u << lane) - 1u;  // lanes <= this one (wraps to all at lane 31)
  return c0 + __popc(starts & upto) - int(starts & 1u);
}

// Symmetric join tables (build_symmetric_tables); fwd == nullptr: plain join.
// One backward entry of cell c: an earlier neighbour cell X, with what a row of c
// needs to read X's masks (built once per grid after the mask layout).
struct alignas(16) BtDesc {
  long long mbase;   // X's first mask
  unsigned nblk;     // X's refined blocks per query group
  unsigned rel;      // offset of c's first point in X's refined suffix
  unsigned qbase;    // X's first position
  unsigned ng;       // X's query groups
  unsigned pad[2];
};

struct SymTables {
  const uint32_t* fwd;       // per cell: list offset of the cell's own first point
  const int64_t* bt_start;   // per cell: backward entries [bt_start[c], bt_start[c+1])
  const BtDesc* desc;        // the entries
};

struct MaskRow {
  const unsigned long long* m;  // the row's group: nblk masks
  int nblk;
  int shift;                    // 32 * (col & 1) + col / 2
  uint32_t fwd;                 // list offset of block 0 (symmetric join), else 0
};

__device__ __forceinline__ MaskRow mask_row(const unsigned long long* __restrict__ masks,
                                            const int64_t* __restrict__ cell_mbase,
                                            const int64_t* __restrict__ cell_cand, int64_t c,
                                            int64_t rel, const uint32_t* __restrict__ fwd) {
  MaskRow r;
  r.fwd = fwd ? fwd[c] : 0u;
  r.nblk = int((cell_cand[c] - r.fwd + 7) >> 3);
  r.m = masks + cell_mbase[c] + (rel >> 3) * r.nblk;
  const int col = int(rel & 7);
  r.shift = 32 * (col & 1) + (col >> 1);
  return r;
}

// The 8 query bits of candidate row r of a tile mask: bit j < 4 -> query 2j,
// bit 4 + j -> query 2j + 1 (the layout of refine_lowd.cu's ballots).
__device__ __forceinline__ unsigned cand_row_bits(unsigned long long m, int r) {
  return unsigned((m >> (4 * r)) & 0xFu) | (unsigned((m >> (32 + 4 * r)) & 0xFu) << 4);
}

// Backward part of a row (symmetric join): the point at offset `rel` of cell c
// is a candidate of every earlier neighbour cell X; its pairs with X's queries
// are candidate row (off & 7) of block (off >> 3) in each of X's query groups.
// Entries go four at a time: their descriptors, then their masks, are loaded
// before any is used (the loads are independent; only their latency matters).
template <class F>
__device__ __forceinline__ void for_backward_hits(const SymTables& sym,
                                                  const unsigned long long* __restrict__ masks,
                                                  int64_t c, uint32_t rel, F&& f) {
  const int64_t e1 = sym.bt_start[c + 1];
  for (int64_t e0 = sym.bt_start[c]; e0 < e1; e0 += 4) {
    BtDesc dd[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (e0 + u < e1) {
        dd[u] = sym.desc[e0 + u];
      } else {
        dd[u].ng = 0;
        dd[u].mbase = 0;
        dd[u].nblk = dd[u].rel = dd[u].qbase = 0;
      }
    }
    unsigned long long mv[4][2];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const unsigned long long* m = masks + dd[u].mbase + ((dd[u].rel + rel) >> 3);
      mv[u][0] = dd[u].ng > 0 ? __ldg(m) : 0ull;
      mv[u][1] = dd[u].ng > 1 ? __ldg(m + dd[u].nblk) : 0ull;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int r = int((dd[u].rel + rel) & 7);
      if (dd[u].ng > 0) f(cand_row_bits(mv[u][0], r), dd[u].qbase);
      if (dd[u].ng > 1) f(cand_row_bits(mv[u][1], r), dd[u].qbase + 8);
      for (unsigned g = 2; g < dd[u].ng; ++g) {  // cells of > 16 points: rare at low d
        const unsigned long long* m = masks + dd[u].mbase + ((dd[u].rel + rel) >> 3);
        f(cand_row_bits(__ldg(m + int64_t(g) * dd[u].nblk), r), dd[u].qbase + 8 * g);
      }
    }
  }
}

__device__ __forceinline__ int backward_count(const SymTables& sym,
                                              const unsigned long long* __restrict__ masks,
                                              const int64_t* __restrict__ cell_mbase,
                                              const int64_t* __restrict__ cell_start,
                                              const int64_t* __restrict__ cell_cand, int64_t c,
                                              uint32_t rel) {
  (void)cell_mbase;
  (void)cell_start;
  (void)cell_cand;
  int cnt = 0;
  for_backward_hits(sym, masks, c, rel, [&](unsigned bits, unsigned) { cnt += __popc(bits); });
  return cnt;
}

// Query column of bit j of cand_row_bits: bits 0..3 -> 0, 2, 4, 6; 4..7 -> 1, 3, 5, 7.
__device__ __forceinline__ int cand_bit_query(int j) { return j < 4 ? 2 * j : 2 * (j - 4) + 1; }

// Positions of a row's backward hits into its pool column from `slot` on.
__device__ __noinline__ void emit_backward(const SymTables& sym,
                                           const unsigned long long* __restrict__ masks,
                                           int64_t c, uint32_t rel, uint32_t* col, int slot) {
  for_backward_hits(sym, masks, c, rel, [&](unsigned bits, unsigned qbase) {
    while (bits) {
      const int j = __ffs(bits) - 1;
      bits &= bits - 1u;
      col[slot * kPoolLd] = qbase + unsigned(cand_bit_query(j));
      ++slot;
    }
  });
}

// desc[e] for every backward entry (after the mask layout is known).
__global__ void bt_desc_kernel(const uint2* __restrict__ bt, const int64_t* __restrict__ n_entries_dev,
                               const int64_t* __restrict__ cell_start,
                               const int64_t* __restrict__ cell_cand,
                               const int64_t* __restrict__ cell_mbase,
                               const uint32_t* __restrict__ fwd, BtDesc* __restrict__ desc) {
  const int64_t n_entries = *n_entries_dev;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n_entries;
       e += int64_t(gridDim.x) * blockDim.x) {
    const uint2 xo = bt[e];
    const int64_t x = xo.x;
    BtDesc d;
    d.mbase = cell_mbase[x];
    d.nblk = unsigned((cell_cand[x] - fwd[x] + 7) >> 3);
    d.rel = xo.y;
    d.qbase = unsigned(cell_start[x]);
    d.ng = unsigned((cell_start[x + 1] - cell_start[x] + 7) >> 3);
    d.pad[0] = d.pad[1] = 0;
    desc[e] = d;
  }
}

__device__ __forceinline__ unsigned row_bits(unsigned long long m, int shift) {
  return unsigned(m >> shift) & 0x11111111u;  // bit 4r: candidate r of the block
}

// Pairs per query of the cells [cb, ce) (their masks were just written).
__global__ void __launch_bounds__(256)
    count_rows_kernel(const unsigned long long* __restrict__ masks,
                      const int64_t* __restrict__ cell_mbase, const int64_t* __restrict__ cell_start,
                      const int64_t* __restrict__ cell_cand, int64_t n_cells,
                      const uint32_t* __restrict__ win_cell, int64_t cb, int64_t ce,
                      uint32_t* __restrict__ qcount, unsigned long long* hits,
                      unsigned long long* max_row, SymTables sym) {
  const int lane = lane_id();
  const int64_t pb = cell_start[cb], pe = cell_start[ce];
  const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
  unsigned long long tot = 0;
  unsigned mx = 0;
  for (int64_t w = (pb >> 5) + (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) / 32;
       (w << 5) < pe; w += warps) {
    const int64_t p0 = w << 5, p = p0 + lane;
    const int64_t c = window_lane_cell(cell_start, n_cells, win_cell[w], p0);
    if (p < pb || p >= pe) continue;
    const MaskRow mr = mask_row(masks, cell_mbase, cell_cand, c, p - cell_start[c], sym.fwd);
    unsigned cnt = 0;
    int b = 0;
    for (; b + 4 <= mr.nblk; b += 4) {
      unsigned long long v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = __ldg(mr.m + b + u);
#pragma unroll
      for (int u = 0; u < 4; ++u) cnt += __popc(row_bits(v[u], mr.shift));
    }
    for (; b < mr.nblk; ++b) cnt += __popc(row_bits(__ldg(mr.m + b), mr.shift));
    if (sym.fwd)
      cnt += backward_count(sym, masks, cell_mbase, cell_start, cell_cand, c,
                            uint32_t(p - cell_start[c]));
    qcount[p] = cnt;
    tot += cnt;
    mx = max(mx, cnt);
  }
  mx = __reduce_max_sync(0xffffffffu, mx);
  if (lane == 0 && mx) atomicMax(max_row, (unsigned long long)mx);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
  if (lane == 0 && tot) atomicAdd(hits, tot);
}

// Candidate list offset t of a cell -> cell-ordered position (runs [rb, rb+nr)).
__device__ __forceinline__ uint32_t run_position(const uint2* __restrict__ runs,
                                                 const uint32_t* __restrict__ run_off, int64_t rb,
                                                 int nr, uint32_t t) {
  int lo = 0, hi = nr;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (run_off[rb + mid] <= t) lo = mid;
    else hi = mid;
  }
  return runs[rb + lo].x + (t - run_off[rb + lo]);
}

// Short rows (<= kPoolSlots ids), one per lane, expanded, sorted and placed in
// one pass.  The lane's mask row (its query group, ~1 KB) is first prefetched
// into L1 with independent prefetches, then walked 16 masks per batch of
// independent loads (what the prefetch missed costs one round trip per batch);
// four blocks' row bits are packed into one word (bit 4r + u = candidate r of
// block u), so the divergent hit loop runs once per four blocks; hit offsets go to column `lane`
// of a transposed shared-memory pool (order is irrelevant: rows are sorted by
// id at the end).  Offsets map to positions through the cell's run table with a
// per-block run hint (both staged in shared memory once per window for up to
// kEmitCells cells), positions to original ids with 16 gathers in flight; the
// warp sorts the 32 rows in registers (odd-even merge network per lane) and
// writes them to their places.  Longer rows are listed for long_rows_kernel.
constexpr int kEmitWarps = 2;
constexpr int kEmitCells = 4;   // cells of one window whose run tables are staged
constexpr int kRunTab = 32;     // >= 27 runs (k <= 4) + the list-length sentinel
constexpr int kBlkTab = 256;    // block -> run hints per staged cell (2048 candidates)

struct EmitSmem {
  uint32_t pool[kPoolSlots * kPoolLd];
  uint32_t roff[kEmitCells][kRunTab];      // run offsets, padded with 0xffffffff
  uint32_t rpos[kEmitCells][kRunTab];      // run start positions
  unsigned char brun[kEmitCells][kBlkTab]; // run holding candidate 8b of block b
};

__device__ __forceinline__ void prefetch_l1(const void* p) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}

// LIST = false: windows of 32 consecutive positions.  LIST = true: windows of 32
// consecutive entries of a position list (ascending positions of the rows of one
// original-id range, tj_finalize_rows_chunk): the rows land at the same final
// places, but the range is complete when the launch ends.
struct RowList {
  const uint32_t* pos;   // ascending positions
  int64_t begin, end;    // entries of this launch
  const uint32_t* pcell; // cell of every position
};

template <int MINB, bool LIST>
__global__ void __launch_bounds__(kEmitWarps * 32, MINB)
    emit_rows_kernel(const unsigned long long* __restrict__ masks,
                     const int64_t* __restrict__ cell_mbase, const int64_t* __restrict__ cell_start,
                     const int64_t* __restrict__ cell_runs, const uint2* __restrict__ runs,
                     const uint32_t* __restrict__ run_off, const int64_t* __restrict__ cell_cand,
                     int64_t n_cells, const uint32_t* __restrict__ win_cell,
                     const uint32_t* __restrict__ qcount, const uint32_t* __restrict__ perm,
                     const uint32_t* __restrict__ nid,
                     const int64_t* __restrict__ offsets, int64_t n, uint32_t* __restrict__ nbr,
                     uint2* __restrict__ long_rows, unsigned long long* n_long, RowList rl,
                     SymTables sym) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = lane_id();
  EmitSmem& sm = reinterpret_cast<EmitSmem*>(smem_raw)[warp];
  uint32_t* pool = sm.pool;
  const int64_t n_win = LIST ? (rl.end - rl.begin + 31) >> 5 : (n + 31) >> 5;
  const int64_t stride = int64_t(gridDim.x) * kEmitWarps;
  for (int64_t w = int64_t(blockIdx.x) * kEmitWarps + warp; w < n_win; w += stride) {
    int64_t p;
    bool valid;
    if constexpr (LIST) {
      const int64_t e = rl.begin + (w << 5) + lane;
      valid = e < rl.end;
      p = valid ? int64_t(rl.pos[e]) : 0;
    } else {
      p = (w << 5) + lane;
      valid = p < n;
    }
    const int len = valid ? int(qcount[p]) : 0;
    // windows of cells another rank / batch refined: nothing to do
    if (__ballot_sync(0xffffffffu, len > 0) == 0u) continue;
    const uint32_t id = valid ? perm[p] : 0u;
    const int64_t dst = valid ? offsets[id] : 0;
    int64_t c0, c, c_last;
    if constexpr (LIST) {  // positions ascend along the window: lane 0 has the first cell
      const int cv = valid ? int(rl.pcell[p]) : -1;
      c0 = __shfl_sync(0xffffffffu, cv, 0);
      c_last = __reduce_max_sync(0xffffffffu, cv);  // the last valid lane's cell
      c = valid ? cv : c0;
    } else {
      c0 = win_cell[w];
      c = window_lane_cell(cell_start, n_cells, c0, w << 5);
      c_last = __shfl_sync(0xffffffffu, c, 31);
    }
    const bool pooled = len > 0 && len <= kPoolSlots;
    if (len > kPoolSlots) long_rows[atomicAdd(n_long, 1ull)] = make_uint2(uint32_t(p), uint32_t(c));
    MaskRow mr{};
    if (pooled) {
      mr = mask_row(masks, cell_mbase, cell_cand, c, p - cell_start[c], sym.fwd);
      for (int b = 0; b < mr.nblk; b += 4) prefetch_l1(mr.m + b);
    }
    // run tables + block hints of the window's first kEmitCells cells
    const int ncw = int(min(c_last + 1, n_cells) - c0);
    __syncwarp();
    for (int ci = 0; ci < min(ncw, kEmitCells); ++ci) {
      const int64_t rb = cell_runs[c0 + ci], nr = cell_runs[c0 + ci + 1] - rb;
      sm.roff[ci][lane] = lane < nr ? run_off[rb + lane] : 0xffffffffu;
      sm.rpos[ci][lane] = lane < nr ? runs[rb + lane].x : 0u;
    }
    __syncwarp();
    for (int ci = 0; ci < min(ncw, kEmitCells); ++ci) {
      const int nblk = int(min((cell_cand[c0 + ci] + 7) >> 3, int64_t(kBlkTab)));
      const uint32_t* ro = sm.roff[ci];
      for (int b = lane; b < nblk; b += 32) {
        const uint32_t t = 8u * uint32_t(b);
        int r = 0;
#pragma unroll
        for (int step = 16; step > 0; step >>= 1)
          if (ro[r + step] <= t) r += step;
        sm.brun[ci][b] = (unsigned char)r;
      }
    }
    __syncwarp();
    if (pooled) {
      uint32_t* col = pool + lane;
      const int ci = int(c - c0);
      // 1. candidate offsets (in the cell's list): 16 masks per batch, four blocks
      //    per packed word
      int slot = 0;
      for (int b0 = 0; b0 < mr.nblk; b0 += 16) {
        unsigned long long mv[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) mv[u] = b0 + u < mr.nblk ? mr.m[b0 + u] : 0ull;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          unsigned wbits = 0u;
#pragma unroll
          for (int u = 0; u < 4; ++u) wbits |= row_bits(mv[4 * q + u], mr.shift) << u;
          while (wbits) {
            const int j = __ffs(wbits) - 1;
            wbits &= wbits - 1u;
            col[slot * kPoolLd] = mr.fwd + uint32_t(8 * (b0 + 4 * q + (j & 3)) + (j >> 2));
            ++slot;
          }
        }
      }
      const int nf = slot;  // forward hits; the symmetric join's backward ones follow
      // 2. offsets -> positions: the block's run hint, then the (rare) steps to
      //    later runs when the block straddles a run boundary
      if (ci < kEmitCells && ((cell_cand[c] + 7) >> 3) <= kBlkTab) {
        const uint32_t* ro = sm.roff[ci];
        const uint32_t* rp = sm.rpos[ci];
        const unsigned char* br = sm.brun[ci];
        for (int i = 0; i < nf; ++i) {
          const uint32_t t = col[i * kPoolLd];
          int r = br[t >> 3];
          while (ro[r + 1] <= t) ++r;
          col[i * kPoolLd] = rp[r] + (t - ro[r]);
        }
      } else {
        // many cells in the window (small cells, or a position list), or a very
        // long list: walk the cell's run table in global memory from the previous
        // hit's run (offsets come out nearly ascending: a step or two per hit)
        const int64_t rb = cell_runs[c];
        const int nr = int(cell_runs[c + 1] - rb);
        const uint32_t* ro = run_off + rb;
        int r = 0;
        uint32_t r_lo = __ldg(ro), r_hi = nr > 1 ? __ldg(ro + 1) : 0xffffffffu;
        for (int i = 0; i < nf; ++i) {
          const uint32_t t = col[i * kPoolLd];
          while (t >= r_hi) {
            ++r;
            r_lo = r_hi;
            r_hi = r + 1 < nr ? __ldg(ro + r + 1) : 0xffffffffu;
          }
          while (t < r_lo) {
            --r;
            r_hi = r_lo;
            r_lo = __ldg(ro + r);
          }
          col[i * kPoolLd] = runs[rb + r].x + (t - r_lo);
        }
      }
      // 3. symmetric join: positions of the pairs with earlier neighbour cells,
      //    from their masks
      if (sym.fwd) emit_backward(sym, masks, c, uint32_t(p - cell_start[c]), col, nf);
      // 4. positions -> original ids, 16 gathers in flight
      for (int i0 = 0; i0 < len; i0 += 16) {
        uint32_t v[16];
#pragma unroll
        for (int u = 0; u < 16; ++u)
          v[u] = i0 + u < len ? __ldg(nid + col[(i0 + u) * kPoolLd]) : 0u;
#pragma unroll
        for (int u = 0; u < 16; ++u)
          if (i0 + u < len) col[(i0 + u) * kPoolLd] = v[u];
      }
    }
    __syncwarp();
    pool_sort(pool, pooled ? len : 0);
    __syncwarp();
    const unsigned todo = __ballot_sync(0xffffffffu, pooled);
    for (unsigned m = todo; m; m &= m - 1u) {
      const int k = __ffs(m) - 1;
      const int L = __shfl_sync(0xffffffffu, len, k);
      const int64_t D = __shfl_sync(0xffffffffu, dst, k);
#pragma unroll
      for (int e0 = 0; e0 < kPoolSlots; e0 += 32)
        if (e0 + lane < L) nbr[D + e0 + lane] = pool[(e0 + lane) * kPoolLd + k];
    }
  }
}

// pcell[p] = cell of position p; key[p] = the original-id range (of `chunks`
// equal ranges) holding perm[p] -- a stable sort by key lists every range's
// positions in ascending order (tj_finalize_rows_chunk).
__global__ void chunk_keys_kernel(const uint32_t* __restrict__ perm,
                                  const int64_t* __restrict__ cell_start, int64_t n,
                                  int64_t n_cells, int chunks, uint64_t* __restrict__ key,
                                  uint32_t* __restrict__ pcell) {
  for (int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p < n;
       p += int64_t(gridDim.x) * blockDim.x)
    key[p] = uint64_t((int64_t(perm[p]) * chunks) / n);
  for (int64_t c = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; c < n_cells;
       c += int64_t(gridDim.x) * blockDim.x)
    for (int64_t p = cell_start[c]; p < cell_start[c + 1]; ++p) pcell[p] = uint32_t(c);
}

// Rows longer than kPoolSlots: warp per row.  Lanes take blocks, a warp scan of
// the per-block hit counts places every candidate offset in ascending order at
// the row's destination, offsets are mapped to original ids in place, and the
// row is sorted there (warp bitonic <= kWarpSortMax, else listed for the CTA /
// radix path).
__global__ void __launch_bounds__(256)
    long_rows_kernel(const unsigned long long* __restrict__ masks,
                     const int64_t* __restrict__ cell_mbase, const int64_t* __restrict__ cell_start,
                     const int64_t* __restrict__ cell_runs, const uint2* __restrict__ runs,
                     const uint32_t* __restrict__ run_off, const int64_t* __restrict__ cell_cand,
                     int64_t n_cells, const uint32_t* __restrict__ perm,
                     const uint32_t* __restrict__ nid,
                     const int64_t* __restrict__ offsets, uint32_t* __restrict__ nbr,
                     const uint2* __restrict__ long_rows, const unsigned long long* n_long,
                     uint32_t* __restrict__ big_rows, unsigned long long* n_big, SymTables sym) {
  const int lane = lane_id();
  const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
  const int64_t nl = int64_t(*n_long);
  for (int64_t i = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) / 32; i < nl; i += warps) {
    const uint2 pc = long_rows[i];  // (position, its cell), listed by the emit kernel
    const uint32_t p = pc.x;
    const int64_t c = pc.y;
    const uint32_t id = perm[p];
    const int64_t dst = offsets[id];
    const int len = int(offsets[id + 1] - dst);
    const MaskRow mr = mask_row(masks, cell_mbase, cell_cand, c, int64_t(p) - cell_start[c],
                                sym.fwd);
    uint32_t* row = nbr + dst;
    int base = 0;
    for (int b0 = 0; b0 < mr.nblk; b0 += 32) {
      const int b = b0 + lane;
      unsigned bits = b < mr.nblk ? row_bits(__ldg(mr.m + b), mr.shift) : 0u;
      const int cnt = __popc(bits);
      int incl = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      int at = base + incl - cnt;
      while (bits) {
        const int r = (__ffs(bits) - 1) >> 2;
        bits &= bits - 1u;
        row[at++] = mr.fwd + uint32_t(8 * b + r);
      }
      base += __shfl_sync(0xffffffffu, incl, 31);
    }
    __syncwarp();
    const int64_t rb = cell_runs[c];
    const int nr = int(cell_runs[c + 1] - rb);
    if (nr <= 32) {
      // the cell's runs in the lanes (lane r: run r); each offset finds its run
      // by a 5-step search over the lanes (no dependent global loads)
      const uint32_t ro = lane < nr ? run_off[rb + lane] : 0xffffffffu;
      const uint32_t rp = lane < nr ? runs[rb + lane].x : 0u;
      for (int e0 = 0; e0 < base; e0 += 32) {
        const int e = e0 + lane;
        const uint32_t t = e < base ? row[e] : 0u;
        int r = 0;
#pragma unroll
        for (int step = 16; step > 0; step >>= 1) {
          const uint32_t o = __shfl_sync(0xffffffffu, ro, r + step);
          if (o <= t) r += step;
        }
        const uint32_t pos = __shfl_sync(0xffffffffu, rp, r) + (t - __shfl_sync(0xffffffffu, ro, r));
        if (e < base) row[e] = nid[pos];
      }
    } else {
      for (int e = lane; e < base; e += 32) row[e] = nid[run_position(runs, run_off, rb, nr, row[e])];
    }
    // symmetric join: the pairs with earlier neighbour cells (rare long rows: one lane)
    if (sym.fwd && lane == 0) {
      int at = base;
      for_backward_hits(sym, masks, c, uint32_t(int64_t(p) - cell_start[c]),
                        [&](unsigned bits, unsigned qbase) {
                          while (bits) {
                            const int j = __ffs(bits) - 1;
                            bits &= bits - 1u;
                            row[at++] = nid[qbase + cand_bit_query(j)];
                          }
                        });
    }
    __syncwarp();
    sort_long_row(row, len, id, big_rows, n_big);
  }
}

// win_cell[w] = the cell containing position 32 w.
__global__ void window_cells_kernel(const int64_t* __restrict__ cell_start, int64_t n_cells,
                                    uint32_t* __restrict__ win_cell) {
  for (int64_t c = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; c < n_cells;
       c += int64_t(gridDim.x) * blockDim.x) {
    const int64_t cs = cell_start[c], ce = cell_start[c + 1];
    for (int64_t w = (cs + 31) >> 5; (w << 5) < ce; ++w) win_cell[w] = uint32_t(c);
  }
}

// One CTA per listed row of 257..8192 ids: shared-memory bitonic sort.
__global__ void __launch_bounds__(1024)
    sort_rows_block_kernel(const int64_t* __restrict__ offsets, uint32_t* __restrict__ nbr,
                           const uint32_t* __restrict__ rows, const unsigned long long* n_rows,
                           uint32_t* __restrict__ huge_rows, unsigned long long* n_huge) {
  __shared__ uint32_t s[kBlockSortMax];
  for (unsigned long long ri = blockIdx.x; ri < *n_rows; ri += gridDim.x) {
    const uint32_t i = rows[ri];
    const int64_t b = offsets[i];
    const int64_t len = offsets[i + 1] - b;
    if (len > kBlockSortMax) {
      if (threadIdx.x == 0) huge_rows[atomicAdd(n_huge, 1ull)] = i;
      continue;
    }
    int N = 512;
    while (N < len) N <<= 1;
    __syncthreads();
    for (int t = threadIdx.x; t < N; t += blockDim.x) s[t] = t < len ? nbr[b + t] : 0xffffffffu;
    __syncthreads();
    for (int k = 2; k <= N; k <<= 1) {
      for (int j = k >> 1; j > 0; j >>= 1) {
        for (int t = threadIdx.x; t < N; t += blockDim.x) {
          const int p = t ^ j;
          if (p > t) {
            const bool asc = (t & k) == 0;
            const uint32_t x = s[t], y = s[p];
            if (asc ? (x > y) : (x < y)) {
              s[t] = y;
              s[p] = x;
            }
          }
        }
        __syncthreads();
      }
    }
    for (int t = threadIdx.x; t < len; t += blockDim.x) nbr[b + t] = s[t];
  }
}

// Rows longer than kBlockSortMax: gather (row rank << 32 | id) keys, radix sort, scatter back.
__global__ void huge_gather_kernel(const int64_t* __restrict__ offsets, const uint32_t* nbr,
                                   const uint32_t* __restrict__ huge, int n_huge,
                                   const int64_t* __restrict__ base, uint64_t* __restrict__ keys) {
  for (int h = blockIdx.y; h < n_huge; h += gridDim.y) {
    const int64_t b = offsets[huge[h]];
    const int64_t len = offsets[huge[h] + 1] - b;
    for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < len;
         t += int64_t(gridDim.x) * blockDim.x)
      keys[base[h] + t] = (uint64_t(h) << 32) | nbr[b + t];
  }
}
__global__ void huge_scatter_kernel(const int64_t* __restrict__ offsets, uint32_t* nbr,
                                    const uint32_t* __restrict__ huge, int n_huge,
                                    const int64_t* __restrict__ base,
                                    const uint64_t* __restrict__ keys) {
  for (int h = blockIdx.y; h < n_huge; h += gridDim.y) {
    const int64_t b = offsets[huge[h]];
    const int64_t len = offsets[huge[h] + 1] - b;
    for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < len;
         t += int64_t(gridDim.x) * blockDim.x)
      nbr[b + t] = uint32_t(keys[base[h] + t]);
  }
}

// ---------------------------------------------------------- symmetric join
// Low-d symmetric join: the refine covers, for every cell B, only the suffix of
// B's candidate list from B's own first point on (the cells >= B; fwd[B] is that
// offset).  The pairs of B's queries with a neighbour cell X < B then sit in X's
// masks, where B's points are candidates: the backward table lists, per cell B,
// every such X with the offset of B's first point in X's refined suffix.
// Position of pos in the list of cell c (runs are position-sorted): list offset.
__device__ __forceinline__ uint32_t list_offset(const uint2* __restrict__ runs,
                                                const uint32_t* __restrict__ run_off, int64_t rb,
                                                int nr, uint32_t pos) {
  int lo = 0, hi = nr;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (runs[rb + mid].x <= pos) lo = mid;
    else hi = mid;
  }
  return run_off[rb + lo] + (pos - runs[rb + lo].x);
}

__global__ void sym_fwd_kernel(const int64_t* __restrict__ cell_start,
                               const int64_t* __restrict__ cell_runs, const uint2* __restrict__ runs,
                               const uint32_t* __restrict__ run_off, const uint32_t* __restrict__ pcell,
                               int64_t n_cells, uint32_t* __restrict__ fwd,
                               int64_t* __restrict__ bt_count) {
  for (int64_t c = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; c < n_cells;
       c += int64_t(gridDim.x) * blockDim.x) {
    const int64_t rb = cell_runs[c];
    const int nr = int(cell_runs[c + 1] - rb);
    const uint32_t own = uint32_t(cell_start[c]);
    fwd[c] = list_offset(runs, run_off, rb, nr, own);
    int64_t cnt = 0;  // neighbour cells before c
    for (int r = 0; r < nr; ++r) {
      const uint2 run = runs[rb + r];
      if (run.x >= own) break;
      const int64_t first = pcell[run.x];
      const int64_t last = run.y <= own ? int64_t(pcell[run.y - 1]) : c - 1;
      cnt += last - first + 1;
    }
    bt_count[c] = cnt;
  }
}

__global__ void sym_fill_kernel(const int64_t* __restrict__ cell_start,
                                const int64_t* __restrict__ cell_runs, const uint2* __restrict__ runs,
                                const uint32_t* __restrict__ run_off, const uint32_t* __restrict__ pcell,
                                const uint32_t* __restrict__ fwd, int64_t n_cells,
                                const int64_t* __restrict__ bt_start, uint2* __restrict__ bt) {
  for (int64_t c = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; c < n_cells;
       c += int64_t(gridDim.x) * blockDim.x) {
    const int64_t rb = cell_runs[c];
    const int nr = int(cell_runs[c + 1] - rb);
    const uint32_t own = uint32_t(cell_start[c]);
    int64_t out = bt_start[c];
    for (int r = 0; r < nr; ++r) {
      const uint2 run = runs[rb + r];
      if (run.x >= own) break;
      const int64_t first = pcell[run.x];
      const int64_t last = run.y <= own ? int64_t(pcell[run.y - 1]) : c - 1;
      for (int64_t x = first; x <= last; ++x) {
        const int64_t xb = cell_runs[x];
        const uint32_t off = list_offset(runs, run_off, xb, int(cell_runs[x + 1] - xb), own);
        bt[out++] = make_uint2(uint32_t(x), off - fwd[x]);
      }
    }
  }
}

// Warp per cell (lanes stride over its points: big cells stay parallel).
__global__ void pcell_kernel(const int64_t* __restrict__ cell_start, int64_t n_cells,
                             uint32_t* __restrict__ pcell) {
  const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
  for (int64_t c = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5; c < n_cells; c += warps)
    for (int64_t p = cell_start[c] + lane_id(); p < cell_start[c + 1]; p += 32) pcell[p] = uint32_t(c);
}

__global__ void compose_ids_kernel(const uint32_t* __restrict__ perm,
                                   const uint32_t* __restrict__ id_map, int64_t n,
                                   uint32_t* __restrict__ out) {
  for (int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p < n;
       p += int64_t(gridDim.x) * blockDim.x)
    out[p] = id_map[perm[p]];
}

// Id written for a neighbour at cell-ordered position p: the original id perm[p],
// or id_map[perm[p]] when the caller set an output id map (tj_set_output_ids: a
// multi-GPU shard writes global ids straight away, no remap pass over the rows).
static const uint32_t* neighbour_ids(tj_ctx* ctx, cudaStream_t s) {
  if (!ctx->out_ids) return ctx->perm.as<uint32_t>();
  if (!ctx->nid_ready) {
    const int64_t n = ctx->g.n;
    ctx->nid.ensure(sizeof(uint32_t) * std::max<int64_t>(n, 1), s);
    compose_ids_kernel<<<unsigned(std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 256),
                                                                          kNumSMs * 16))),
                         256, 0, s>>>(ctx->perm.as<uint32_t>(), ctx->out_ids, n,
                                      ctx->nid.as<uint32_t>());
    TJ_CHECK_LAUNCH();
    ctx->nid_ready = true;
  }
  return ctx->nid.as<uint32_t>();
}

static SymTables sym_tables(const tj_ctx* ctx) {
  if (!ctx->symmetric) return SymTables{nullptr, nullptr, nullptr};
  return SymTables{ctx->fwd.as<uint32_t>(), ctx->bt_start.as<int64_t>(),
                   ctx->bt_desc.as<BtDesc>()};
}

static unsigned blocks_for(int64_t n, int threads) {
  return unsigned(std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, threads), kNumSMs * 16)));
}

void build_symmetric_tables(tj_ctx* ctx, cudaStream_t s) {
  const int64_t n = ctx->g.n, nc = ctx->g.n_cells;
  ctx->pcell.ensure(sizeof(uint32_t) * std::max<int64_t>(n, 1), s);
  pcell_kernel<<<blocks_for(nc * 32, 256), 256, 0, s>>>(ctx->cell_start.as<int64_t>(), nc,
                                                        ctx->pcell.as<uint32_t>());
  TJ_CHECK_LAUNCH();
  ctx->fwd.ensure(sizeof(uint32_t) * std::max<int64_t>(nc, 1), s);
  ctx->bt_start.ensure(sizeof(int64_t) * (nc + 1), s);
  ctx->tmp64.ensure(sizeof(int64_t) * (nc + 1), s);
  sym_fwd_kernel<<<blocks_for(nc, 128), 128, 0, s>>>(
      ctx->cell_start.as<int64_t>(), ctx->cell_runs.as<int64_t>(), ctx->runs.as<uint2>(),
      ctx->run_off.as<uint32_t>(), ctx->pcell.as<uint32_t>(), nc, ctx->fwd.as<uint32_t>(),
      ctx->tmp64.as<int64_t>());
  TJ_CHECK_LAUNCH();
  ScanScratch sc = scan_scratch(ctx, std::max<int64_t>(nc, 1), s);
  scan_exclusive(LoadAt<int64_t>{ctx->tmp64.as<int64_t>()},
                 StoreAt<int64_t>{ctx->bt_start.as<int64_t>()}, nc, sc, s);
  TJ_CUDA(cudaMemcpyAsync(ctx->bt_start.as<int64_t>() + nc, sc.total, sizeof(int64_t),
                          cudaMemcpyDeviceToDevice, s));
  // bound: every neighbour row of a cell holds <= 3 cells (13 backward cells at k = 4)
  int rows = 1;
  for (int j = 0; j < ctx->g.k - 1; ++j) rows *= 3;
  ctx->bt.ensure(sizeof(uint2) * std::max<int64_t>(nc * int64_t(rows) * 3 / 2 + 1, 1), s);
  sym_fill_kernel<<<blocks_for(nc, 128), 128, 0, s>>>(
      ctx->cell_start.as<int64_t>(), ctx->cell_runs.as<int64_t>(), ctx->runs.as<uint2>(),
      ctx->run_off.as<uint32_t>(), ctx->pcell.as<uint32_t>(), ctx->fwd.as<uint32_t>(), nc,
      ctx->bt_start.as<int64_t>(), ctx->bt.as<uint2>());
  TJ_CHECK_LAUNCH();
}

void build_bt_desc(tj_ctx* ctx, cudaStream_t s) {
  const int64_t nc = ctx->g.n_cells;
  int rows = 1;
  for (int j = 0; j < ctx->g.k - 1; ++j) rows *= 3;
  const int64_t bound = std::max<int64_t>(nc * int64_t(rows) * 3 / 2 + 1, 1);
  ctx->bt_desc.ensure(sizeof(BtDesc) * bound, s);
  bt_desc_kernel<<<blocks_for(bound, 256), 256, 0, s>>>(
      ctx->bt.as<uint2>(), ctx->bt_start.as<int64_t>() + nc, ctx->cell_start.as<int64_t>(),
      ctx->cell_cand.as<int64_t>(), ctx->cell_mbase.as<int64_t>(), ctx->fwd.as<uint32_t>(),
      ctx->bt_desc.as<BtDesc>());
  TJ_CHECK_LAUNCH();
}

void build_window_cells(tj_ctx* ctx, cudaStream_t s) {
  const int64_t n_win = ceil_div(ctx->g.n, 32);
  ctx->win_cell.ensure(sizeof(uint32_t) * std::max<int64_t>(n_win, 1), s);
  window_cells_kernel<<<blocks_for(ctx->g.n_cells, 256), 256, 0, s>>>(
      ctx->cell_start.as<int64_t>(), ctx->g.n_cells, ctx->win_cell.as<uint32_t>());
  TJ_CHECK_LAUNCH();
}

void launch_count_rows(tj_ctx* ctx, int64_t cb, int64_t ce, unsigned long long* hits,
                       unsigned long long* max_row, cudaStream_t s) {
  count_rows_kernel<<<kNumSMs * 8, 256, 0, s>>>(
      ctx->masks.as<unsigned long long>(), ctx->cell_mbase.as<int64_t>(),
      ctx->cell_start.as<int64_t>(), ctx->cell_cand.as<int64_t>(), ctx->g.n_cells,
      ctx->win_cell.as<uint32_t>(), cb, ce, ctx->qcount.as<uint32_t>(), hits, max_row,
      sym_tables(ctx));
  TJ_CHECK_LAUNCH();
}

// Sort the rows listed in big_rows (> kWarpSortMax ids) in place.
static void sort_big_rows(tj_ctx* ctx, int64_t* offsets, uint32_t* nbr, uint32_t* big_rows,
                          unsigned long long* nbig, cudaStream_t s) {
  const int64_t n = ctx->g.n;
  unsigned long long h_nbig = 0;
  TJ_CUDA(cudaMemcpyAsync(&h_nbig, nbig, sizeof(h_nbig), cudaMemcpyDeviceToHost, s));
  TJ_CUDA(cudaStreamSynchronize(s));
  if (h_nbig == 0) return;
  ctx->vals_alt.ensure(sizeof(uint32_t) * h_nbig, s);
  uint32_t* huge = ctx->vals_alt.as<uint32_t>();
  sort_rows_block_kernel<<<unsigned(std::min<unsigned long long>(h_nbig, kNumSMs * 4)), 1024, 0,
                           s>>>(offsets, nbr, big_rows, nbig, huge, nbig + 1);
  TJ_CHECK_LAUNCH();
  unsigned long long h_nhuge = 0;
  TJ_CUDA(cudaMemcpyAsync(&h_nhuge, nbig + 1, sizeof(h_nhuge), cudaMemcpyDeviceToHost, s));
  TJ_CUDA(cudaStreamSynchronize(s));
  if (h_nhuge == 0) return;

  // composite-key radix sort over all huge rows together
  std::vector<uint32_t> hh(h_nhuge);
  TJ_CUDA(cudaMemcpyAsync(hh.data(), huge, sizeof(uint32_t) * h_nhuge, cudaMemcpyDeviceToHost, s));
  TJ_CUDA(cudaStreamSynchronize(s));
  std::vector<int64_t> hbase(h_nhuge + 1, 0);
  for (size_t h = 0; h < hh.size(); ++h) {
    int64_t se[2];
    TJ_CUDA(cudaMemcpy(se, offsets + hh[h], 2 * sizeof(int64_t), cudaMemcpyDeviceToHost));
    hbase[h + 1] = hbase[h] + (se[1] - se[0]);
  }
  const int64_t m = hbase[h_nhuge];
  DevBuf kb, kb2, vb, vb2, bb, hb;
  kb.ensure(sizeof(uint64_t) * m, s);
  kb2.ensure(sizeof(uint64_t) * m, s);
  vb.ensure(sizeof(uint32_t) * m, s);
  vb2.ensure(sizeof(uint32_t) * m, s);
  bb.ensure(sizeof(int64_t) * (h_nhuge + 1), s);
  TJ_CUDA(cudaMemcpyAsync(bb.ptr, hbase.data(), sizeof(int64_t) * (h_nhuge + 1),
                          cudaMemcpyHostToDevice, s));
  dim3 g(unsigned(std::min<int64_t>(ceil_div(m, 256), 1024)),
         unsigned(std::min<unsigned long long>(h_nhuge, 65535)));
  huge_gather_kernel<<<g, 256, 0, s>>>(offsets, nbr, huge, int(h_nhuge), bb.as<int64_t>(),
                                       kb.as<uint64_t>());
  TJ_CHECK_LAUNCH();
  int hbits = 0;
  while ((1ull << hbits) < h_nhuge) ++hbits;
  hb.ensure(sizeof(int64_t) * radix_sort_scratch_elems(m), s);
  ScanScratch sc2 = scan_scratch(ctx, std::max<int64_t>(radix_sort_scratch_elems(m), n), s);
  const int where = radix_sort_pairs(kb.as<uint64_t>(), vb.as<uint32_t>(), kb2.as<uint64_t>(),
                                     vb2.as<uint32_t>(), m, 32 + hbits, true, hb.as<int64_t>(),
                                     sc2, s);
  huge_scatter_kernel<<<g, 256, 0, s>>>(offsets, nbr, huge, int(h_nhuge), bb.as<int64_t>(),
                                        where ? kb2.as<uint64_t>() : kb.as<uint64_t>());
  TJ_CHECK_LAUNCH();
  TJ_CUDA(cudaStreamSynchronize(s));
  kb.release(s);
  kb2.release(s);
  vb.release(s);
  vb2.release(s);
  bb.release(s);
  hb.release(s);
}

// Rows of id range `chunk` of the split of [0, n) into `chunks` equal ranges
// (offsets from phase 1).  Low-d mask
// results: the range's positions (a stable partition of the positions by id
// range, built once per grid) are emitted by emit_rows_kernel<LIST>, windows of
// 32 ascending positions.  Other results have no per-id source, so the first call
// builds every row (later calls find them done).
void finalize_rows_range(tj_ctx* ctx, const int64_t* offsets, uint32_t* nbr, int64_t n_pairs,
                         int64_t n_mask_hits, int64_t max_mask_row, int chunk, int chunks,
                         cudaStream_t s) {
  const int64_t n = ctx->g.n;
  if (n_mask_hits == 0) {
    if (!ctx->rows_range_done)
      finalize_csr(ctx, const_cast<int64_t*>(offsets), nbr, n_pairs, 0, 0, s, 2);
    ctx->rows_range_done = true;
    return;
  }
  // the chunk lists: positions of every id range, ascending (once per grid and K)
  const int K = int(std::min<int64_t>(std::max<int64_t>(chunks, 1), 256));
  if (!ctx->id_maps_ready || ctx->chunk_lists != K) {
    ctx->pcell.ensure(sizeof(uint32_t) * std::max<int64_t>(n, 1), s);
    ctx->chunk_key.ensure(sizeof(uint64_t) * 2 * std::max<int64_t>(n, 1), s);
    ctx->ipos.ensure(sizeof(uint32_t) * 2 * std::max<int64_t>(n, 1), s);
    uint64_t* k0 = ctx->chunk_key.as<uint64_t>();
    uint32_t* v0 = ctx->ipos.as<uint32_t>();
    chunk_keys_kernel<<<blocks_for(std::max(n, ctx->g.n_cells), 256), 256, 0, s>>>(
        ctx->perm.as<uint32_t>(), ctx->cell_start.as<int64_t>(), n, ctx->g.n_cells, K, k0,
        ctx->pcell.as<uint32_t>());
    TJ_CHECK_LAUNCH();
    DevBuf hb;
    hb.ensure(sizeof(int64_t) * radix_sort_scratch_elems(n), s);
    ScanScratch sc = scan_scratch(ctx, std::max<int64_t>(radix_sort_scratch_elems(n), n), s);
    int kb = 0;
    while ((1 << kb) < K) ++kb;
    const int where = radix_sort_pairs(k0, v0, k0 + n, v0 + n, n, std::max(kb, 1), true,
                                       hb.as<int64_t>(), sc, s);
    ctx->chunk_pos_off = where ? n : 0;
    hb.release(s);
    ctx->chunk_lists = K;
    ctx->id_maps_ready = true;
  }
  // chunk j holds the ids [ceil(j n / K), ceil((j+1) n / K)): one position each,
  // so its list entries start after the ceil(j n / K) positions of smaller ids
  auto first_entry = [&](int64_t j) -> int64_t { return (j * n + K - 1) / K; };
  const int64_t lb = first_entry(chunk), le = first_entry(chunk + 1);
  ctx->fill.ensure(sizeof(uint32_t) * n + 4 * sizeof(unsigned long long), s);
  uint32_t* fill = ctx->fill.as<uint32_t>();
  unsigned long long* nbig = reinterpret_cast<unsigned long long*>(ctx->minmax.as<long long>());
  TJ_CUDA(cudaMemsetAsync(nbig, 0, 3 * sizeof(unsigned long long), s));
  ctx->pos_off.ensure(sizeof(int64_t) * (n + 1), s);
  uint2* long_rows = reinterpret_cast<uint2*>(ctx->pos_off.as<int64_t>());
  if (le > lb) {
    auto kern = emit_rows_kernel<8, true>;
    const size_t smem = sizeof(EmitSmem) * kEmitWarps;
    TJ_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    int per_sm = 0;
    TJ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kEmitWarps * 32, smem));
    const int64_t grid = std::min<int64_t>(ceil_div(ceil_div(le - lb, 32), kEmitWarps),
                                           int64_t(kNumSMs) * std::max(per_sm, 1));
    RowList rl{ctx->ipos.as<uint32_t>() + ctx->chunk_pos_off, lb, le, ctx->pcell.as<uint32_t>()};
    kern<<<unsigned(std::max<int64_t>(grid, 1)), kEmitWarps * 32, smem, s>>>(
        ctx->masks.as<unsigned long long>(), ctx->cell_mbase.as<int64_t>(),
        ctx->cell_start.as<int64_t>(), ctx->cell_runs.as<int64_t>(), ctx->runs.as<uint2>(),
        ctx->run_off.as<uint32_t>(), ctx->cell_cand.as<int64_t>(), ctx->g.n_cells,
        ctx->win_cell.as<uint32_t>(), ctx->qcount.as<uint32_t>(), ctx->perm.as<uint32_t>(),
        neighbour_ids(ctx, s), offsets, n, nbr, long_rows, nbig + 2, rl, sym_tables(ctx));
    TJ_CHECK_LAUNCH();
  }
  long_rows_kernel<<<kNumSMs * 3, 256, 0, s>>>(
      ctx->masks.as<unsigned long long>(), ctx->cell_mbase.as<int64_t>(),
      ctx->cell_start.as<int64_t>(), ctx->cell_runs.as<int64_t>(), ctx->runs.as<uint2>(),
      ctx->run_off.as<uint32_t>(), ctx->cell_cand.as<int64_t>(), ctx->g.n_cells,
      ctx->perm.as<uint32_t>(), neighbour_ids(ctx, s), offsets, nbr, long_rows, nbig + 2, fill,
      nbig, sym_tables(ctx));
  TJ_CHECK_LAUNCH();
  if (max_mask_row > kWarpSortMax)
    sort_big_rows(ctx, const_cast<int64_t*>(offsets), nbr, fill, nbig, s);
}

// phase 1: row offsets by original id; phase 2: the rows (needs phase 1's
// offsets); 3: both.  Splitting lets a caller copy the offsets to the host
// while the rows are being built.
void finalize_csr(tj_ctx* ctx, int64_t* offsets, uint32_t* nbr, int64_t n_pairs,
                  int64_t n_mask_hits, int64_t max_mask_row, cudaStream_t s, int phase) {
  const int64_t n = ctx->g.n;
  ScanScratch sc = scan_scratch(ctx, n, s);
  if (phase & 1) {
    ctx->tmp64.ensure(sizeof(int64_t) * (n + 1), s);
    int64_t* cnt = ctx->tmp64.as<int64_t>();
    counts_to_orig_kernel<<<blocks_for(n, 256), 256, 0, s>>>(ctx->qcount.as<uint32_t>(),
                                                            ctx->perm.as<uint32_t>(), n, cnt);
    TJ_CHECK_LAUNCH();
    scan_exclusive(LoadAt<int64_t>{cnt}, StoreAt<int64_t>{offsets}, n, sc, s);
    TJ_CUDA(cudaMemcpyAsync(offsets + n, sc.total, sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
  }
  if (!(phase & 2) || (n_pairs == 0 && n_mask_hits == 0)) return;

  // `fill` doubles as the list of rows too long for the in-register sorts
  ctx->fill.ensure(sizeof(uint32_t) * n + 4 * sizeof(unsigned long long), s);
  uint32_t* fill = ctx->fill.as<uint32_t>();
  unsigned long long* nbig = reinterpret_cast<unsigned long long*>(ctx->minmax.as<long long>());
  TJ_CUDA(cudaMemsetAsync(nbig, 0, 3 * sizeof(unsigned long long), s));
  if (n_mask_hits > 0) {
    // low-d masks: short rows expanded, sorted and placed in one pass; long rows
    // by a warp each
    const int64_t nc = ctx->g.n_cells;
    const int64_t n_win = ceil_div(n, 32);
    ctx->pos_off.ensure(sizeof(int64_t) * (n + 1), s);
    uint2* long_rows = reinterpret_cast<uint2*>(ctx->pos_off.as<int64_t>());
    {
      // 4 CTAs/SM (<= 128 registers): measured on par with the unbounded build
      // (158 registers, 3 CTAs) and well ahead of 5 CTAs (spills)
      auto kern = emit_rows_kernel<8, false>;
      const size_t smem = sizeof(EmitSmem) * kEmitWarps;
      TJ_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   int(smem)));
      int per_sm = 0;
      TJ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern,
                                                            kEmitWarps * 32, smem));
      const int64_t grid = std::min<int64_t>(ceil_div(n_win, kEmitWarps),
                                             int64_t(kNumSMs) * std::max(per_sm, 1));
      TJ_CUDA(cudaEventRecord(ctx->ev2, s));
      kern<<<unsigned(std::max<int64_t>(grid, 1)), kEmitWarps * 32, smem, s>>>(
          ctx->masks.as<unsigned long long>(), ctx->cell_mbase.as<int64_t>(),
          ctx->cell_start.as<int64_t>(), ctx->cell_runs.as<int64_t>(), ctx->runs.as<uint2>(),
          ctx->run_off.as<uint32_t>(), ctx->cell_cand.as<int64_t>(), nc,
          ctx->win_cell.as<uint32_t>(), ctx->qcount.as<uint32_t>(), ctx->perm.as<uint32_t>(),
          neighbour_ids(ctx, s), offsets, n, nbr, long_rows, nbig + 2, RowList{}, sym_tables(ctx));
      TJ_CHECK_LAUNCH();
      TJ_CUDA(cudaEventRecord(ctx->ev3, s));
      ctx->have_emit_timing = true;
    }
    long_rows_kernel<<<kNumSMs * 3, 256, 0, s>>>(
        ctx->masks.as<unsigned long long>(), ctx->cell_mbase.as<int64_t>(),
        ctx->cell_start.as<int64_t>(), ctx->cell_runs.as<int64_t>(), ctx->runs.as<uint2>(),
        ctx->run_off.as<uint32_t>(), ctx->cell_cand.as<int64_t>(), nc, ctx->perm.as<uint32_t>(),
        neighbour_ids(ctx, s), offsets, nbr, long_rows, nbig + 2, fill, nbig, sym_tables(ctx));
    TJ_CHECK_LAUNCH();
  } else {
    // pair path: rows in cell (position) order first, then sorted into place
    ctx->pos_off.ensure(sizeof(int64_t) * (n + 1), s);
    int64_t* pos_off = ctx->pos_off.as<int64_t>();
    scan_exclusive(LoadAt<uint32_t>{ctx->qcount.as<uint32_t>()}, StoreAt<int64_t>{pos_off}, n, sc,
                   s);
    TJ_CUDA(cudaMemcpyAsync(pos_off + n, sc.total, sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
    ctx->rows_tmp.ensure(sizeof(uint32_t) * std::max<int64_t>(n_pairs, 1), s);
    uint32_t* rows = ctx->rows_tmp.as<uint32_t>();
    TJ_CUDA(cudaMemsetAsync(fill, 0, sizeof(uint32_t) * n, s));
    scatter_pairs_kernel<<<blocks_for(n_pairs, 256), 256, 0, s>>>(
        ctx->pairs.as<uint2>(), n_pairs, neighbour_ids(ctx, s), pos_off, fill, rows);
    TJ_CHECK_LAUNCH();
    const size_t smem = sizeof(uint32_t) * kPoolSlots * kPoolLd * kSortWarps;
    TJ_CUDA(cudaFuncSetAttribute(sort_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(smem)));
    int per_sm = 0;
    TJ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sort_rows_kernel,
                                                          kSortWarps * 32, smem));
    const int64_t grid = std::min<int64_t>(ceil_div(n, 32 * kSortWarps),
                                           int64_t(kNumSMs) * std::max(per_sm, 1));
    sort_rows_kernel<<<unsigned(std::max<int64_t>(grid, 1)), kSortWarps * 32, smem, s>>>(
        pos_off, rows, ctx->perm.as<uint32_t>(), offsets, n, nbr, fill, nbig);
    TJ_CHECK_LAUNCH();
  }
  // low-d rows are at most max_mask_row long (count_rows_kernel): rows the
  // in-warp sorts cannot take exist only beyond kWarpSortMax
  if (n_mask_hits == 0 || max_mask_row > kWarpSortMax) sort_big_rows(ctx, offsets, nbr, fill, nbig, s);
}

}  // namespace tj
