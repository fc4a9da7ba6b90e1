// Canonical output: CSR by original query id with neighbour ids ascending.
//
// Replaces the concatenate + np.lexsort((j, i)) of join.py:203-204.  Per-query
// pair counts (cell-ordered positions) move to original-id order and are
// scanned into int64 row offsets; a second scan in position order gives every
// row a contiguous slot range in a cell-ordered staging array.  Then:
//  * low-d path (hit masks, refine_lowd.cu): warp per cell expands the masks of
//    its query slices into the staging rows (expand_masks_kernel);
//  * pair path (other kernels): every (query, candidate) pair is scattered to
//    its staging row through a per-row atomic cursor;
//  * sort_rows_kernel reads 32 consecutive staging rows (coalesced), sorts one
//    row per lane in registers (odd-even merge network) and writes each row to
//    its final place.  Rows longer than 96 ids are sorted in place by a warp
//    (<= 256), one CTA (shared-memory bitonic, <= 8192) or, beyond that, by a
//    composite-key radix sort.
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
                                     const uint32_t* __restrict__ perm,
                                     const int64_t* __restrict__ pos_off,
                                     uint32_t* __restrict__ fill, uint32_t* __restrict__ rows) {
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const uint2 pr = pairs[e];
    const uint32_t slot = atomicAdd(&fill[pr.x], 1u);
    rows[pos_off[pr.x] + slot] = perm[pr.y];
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

constexpr int kWarpSortMax = 256;
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
constexpr int kPoolSlots = 96;
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
  if (mx <= 16) pool_sort_n<16>(pool, len);
  else if (mx <= 32) pool_sort_n<32>(pool, len);
  else if (mx <= 48) pool_sort_n<48>(pool, len);
  else if (mx <= 64) pool_sort_n<64>(pool, len);
  else if (mx <= 80) pool_sort_n<80>(pool, len);
  else pool_sort_n<96>(pool, len);
}

// Rows with more than kPoolSlots ids are written straight to their place and
// sorted there: by the warp (<= kWarpSortMax) or listed for the CTA/radix path.
__device__ __noinline__ void sort_long_row(uint32_t* row, int len, uint32_t id, uint32_t* big_rows,
                                           unsigned long long* n_big) {
  if (len <= 128) warp_sort_row<4>(row, len);
  else if (len <= kWarpSortMax) warp_sort_row<8>(row, len);
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

// Low-d hit masks -> rows in cell order (unsorted; sort_rows_kernel orders).  Warp
// per cell: the cell's candidate runs are re-flattened into 8-candidate blocks
// exactly as the refine kernel tiled them.  For each chunk of blocks the
// original ids of the blocks' candidates and the current query slice's masks
// (<= 4 groups of 8 queries) are staged with wide independent loads; the masks
// are split into 32-bit halves and compacted to the non-empty ones.  Lanes then
// drain one hit per iteration and grab the next half from a shared counter
// (hits cluster in the blocks nearest the query cell, so any static split
// leaves most lanes idle); bit 4r + c of a low / high half is candidate r of the
// block against query column 2c / 2c + 1.  A per-query shared-memory cursor
// hands out slots in a flat slice buffer (row order is irrelevant before the
// sort), and the slice's rows are copied out with coalesced stores.  Rows that
// do not fit the buffer are written straight to their place.
constexpr int kExpandBlk = 64;     // blocks staged per chunk
constexpr int kExpandWarps = 8;
constexpr int kSliceBuf = 1536;    // ids buffered per query slice

struct ExpandSmem {
  uint32_t buf[kSliceBuf];
  uint32_t pos[kExpandBlk];
  uint32_t ids[kExpandBlk * 8];
  uint2 units[kExpandBlk * 8];  // non-empty mask halves: (bits, ids index << 8 | column)
  int64_t dst[32];              // row start per query of the slice
  uint32_t slot[32];            // next free slot per query (buffer index or row index)
  uint32_t next;                // dynamic unit counter
  uint32_t direct;              // bit j: query j writes straight to its row
};

__global__ void __launch_bounds__(kExpandWarps * 32)
    expand_masks_kernel(const unsigned long long* __restrict__ masks,
                        const int64_t* __restrict__ cell_mbase,
                        const int64_t* __restrict__ cell_start,
                        const int64_t* __restrict__ cell_runs, const uint2* __restrict__ runs,
                        int64_t n_cells, const uint32_t* __restrict__ qcount,
                        const uint32_t* __restrict__ perm, const int64_t* __restrict__ pos_off,
                        uint32_t* __restrict__ rows_out, uint32_t n_points) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = lane_id();
  ExpandSmem& sm = reinterpret_cast<ExpandSmem*>(smem_raw)[warp];
  const unsigned lt = lanemask_lt();

  const int64_t stride = int64_t(gridDim.x) * kExpandWarps;
  for (int64_t c = int64_t(blockIdx.x) * kExpandWarps + warp; c < n_cells; c += stride) {
    const int64_t cs = cell_start[c];
    const int nq = int(cell_start[c + 1] - cs);
    if (qcount[cs] == 0) continue;  // cell not refined in this result set (self pair missing)
    const int ngc = (nq + 7) >> 3;
    // flatten the runs (<= 27 for k <= 4) into blocks
    const int64_t rb = cell_runs[c], re = cell_runs[c + 1];
    const int nr = int(re - rb);
    uint2 myrun = make_uint2(0u, 0u);
    if (lane < nr) myrun = runs[rb + lane];
    const int mynblk = int(myrun.y - myrun.x + 7) >> 3;
    int incl = mynblk;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    const int myfirst = incl - mynblk;
    const unsigned long long* mb = masks + cell_mbase[c];
    for (int q0 = 0; q0 < nq; q0 += 32) {
      const int nqs = min(32, nq - q0);
      const int ngs = (nqs + 7) >> 3;
      const int gs = q0 >> 3;  // first group of the slice
      // query j of the slice (lane j): length, buffer offset, row start
      const bool qa = lane < nqs;
      const int cnt = qa ? int(qcount[cs + q0 + lane]) : 0;
      int ci = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, ci, o);
        if (lane >= o) ci += t;
      }
      const int poff = ci - cnt;
      const bool pooled = poff + cnt <= kSliceBuf;
      const int64_t dst = qa ? pos_off[cs + q0 + lane] : 0;  // row start, position order
      __syncwarp();
      if (qa) {
        sm.dst[lane] = dst;
        sm.slot[lane] = pooled ? uint32_t(poff) : 0u;
      }
      {
        const unsigned dm = __ballot_sync(0xffffffffu, qa && !pooled);
        if (lane == 0) sm.direct = dm;
      }
      for (int b0 = 0; b0 < total; b0 += kExpandBlk) {
        const int nb = min(kExpandBlk, total - b0);
        __syncwarp();
        {
          const int lo = max(myfirst, b0), hi = min(myfirst + mynblk, b0 + nb);
          for (int b = lo; b < hi; ++b) sm.pos[b - b0] = myrun.x + 8u * uint32_t(b - myfirst);
        }
        __syncwarp();
        // original ids of the chunk's candidates: 4 loads in flight per lane
        for (int i0 = 0; i0 < nb * 8; i0 += 128) {
          uint32_t v[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int i = i0 + 32 * k + lane;
            const uint32_t p = i < nb * 8 ? sm.pos[i >> 3] + uint32_t(i & 7) : n_points;
            v[k] = p < n_points ? __ldg(perm + p) : 0u;  // rows past a run end never hit
          }
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int i = i0 + 32 * k + lane;
            if (i < nb * 8) sm.ids[i] = v[k];
          }
        }
        // the slice's mask words, split into halves and compacted to the non-empty ones
        const int nw = nb * ngs;  // word w = (block w / ngs, group w % ngs)
        int nunits = 0;
        for (int i0 = 0; i0 < nw; i0 += 128) {
          unsigned long long v[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int w = i0 + 32 * k + lane;
            const int b = ngs == 3 ? int((unsigned(w) * 0xAAABu) >> 17) : (w >> (ngs >> 1));
            v[k] = w < nw ? __ldg(mb + size_t(b0 + b) * ngc + gs + (w - b * ngs)) : 0ull;
          }
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int w = i0 + 32 * k + lane;
            const int b = ngs == 3 ? int((unsigned(w) * 0xAAABu) >> 17) : (w >> (ngs >> 1));
            const unsigned meta = (unsigned(8 * b) << 8) | unsigned(8 * (w - b * ngs));
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const unsigned bits = unsigned(v[k] >> (32 * h));
              const unsigned bal = __ballot_sync(0xffffffffu, bits != 0u);
              if (bits) sm.units[nunits + __popc(bal & lt)] = make_uint2(bits, meta + h);
              nunits += __popc(bal);
            }
          }
        }
        if (lane == 0) sm.next = 32;
        __syncwarp();
        const unsigned direct = sm.direct;
        int k = lane;
        uint2 e = k < nunits ? sm.units[k] : make_uint2(0u, 0u);
        while (__any_sync(0xffffffffu, k < nunits)) {
          if (k < nunits) {
            const int j = __ffs(e.x) - 1;
            e.x &= e.x - 1u;
            const int col = int(e.y & 0xffu) + 2 * (j & 3);
            const uint32_t v = sm.ids[(e.y >> 8) + (j >> 2)];
            const uint32_t slot = atomicAdd(&sm.slot[col], 1u);
            if (!((direct >> col) & 1u)) sm.buf[slot] = v;
            else rows_out[sm.dst[col] + slot] = v;
            if (e.x == 0u) {
              k = int(atomicAdd(&sm.next, 1u));
              if (k < nunits) e = sm.units[k];
            }
          }
        }
      }
      __syncwarp();
      // the buffered rows (a prefix of the slice) are contiguous in rows_out too
      int pend = (qa && pooled) ? poff + cnt : 0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) pend = max(pend, __shfl_xor_sync(0xffffffffu, pend, o));
      const int64_t d0 = __shfl_sync(0xffffffffu, dst, 0);
      for (int i = lane; i < pend; i += 32) rows_out[d0 + i] = sm.buf[i];
    }
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

static unsigned blocks_for(int64_t n, int threads) {
  return unsigned(std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, threads), kNumSMs * 16)));
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

void finalize_csr(tj_ctx* ctx, int64_t* offsets, uint32_t* nbr, int64_t n_pairs,
                  int64_t n_mask_hits, cudaStream_t s) {
  const int64_t n = ctx->g.n;
  ctx->tmp64.ensure(sizeof(int64_t) * (n + 1), s);
  int64_t* cnt = ctx->tmp64.as<int64_t>();
  counts_to_orig_kernel<<<blocks_for(n, 256), 256, 0, s>>>(ctx->qcount.as<uint32_t>(),
                                                          ctx->perm.as<uint32_t>(), n, cnt);
  TJ_CHECK_LAUNCH();
  ScanScratch sc = scan_scratch(ctx, n, s);
  scan_exclusive(LoadAt<int64_t>{cnt}, StoreAt<int64_t>{offsets}, n, sc, s);
  TJ_CUDA(cudaMemcpyAsync(offsets + n, sc.total, sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
  if (n_pairs == 0 && n_mask_hits == 0) return;

  // rows in cell (position) order first: offsets by position, then the ids
  ctx->pos_off.ensure(sizeof(int64_t) * (n + 1), s);
  int64_t* pos_off = ctx->pos_off.as<int64_t>();
  scan_exclusive(LoadAt<uint32_t>{ctx->qcount.as<uint32_t>()}, StoreAt<int64_t>{pos_off}, n, sc, s);
  TJ_CUDA(cudaMemcpyAsync(pos_off + n, sc.total, sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
  const int64_t total = n_pairs + n_mask_hits;
  ctx->rows_tmp.ensure(sizeof(uint32_t) * std::max<int64_t>(total, 1), s);
  uint32_t* rows = ctx->rows_tmp.as<uint32_t>();
  ctx->fill.ensure(sizeof(uint32_t) * n + 4 * sizeof(unsigned long long), s);
  uint32_t* fill = ctx->fill.as<uint32_t>();
  unsigned long long* nbig = reinterpret_cast<unsigned long long*>(ctx->minmax.as<long long>());
  TJ_CUDA(cudaMemsetAsync(nbig, 0, 2 * sizeof(unsigned long long), s));
  if (n_mask_hits > 0) {
    const int64_t nc = ctx->g.n_cells;
    const size_t smem = sizeof(ExpandSmem) * kExpandWarps;
    TJ_CUDA(cudaFuncSetAttribute(expand_masks_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(smem)));
    int per_sm = 0;
    TJ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, expand_masks_kernel,
                                                          kExpandWarps * 32, smem));
    const int64_t grid = std::min<int64_t>(ceil_div(nc, kExpandWarps),
                                           int64_t(kNumSMs) * std::max(per_sm, 1));
    expand_masks_kernel<<<unsigned(std::max<int64_t>(grid, 1)), kExpandWarps * 32, smem, s>>>(
        ctx->masks.as<unsigned long long>(), ctx->cell_mbase.as<int64_t>(),
        ctx->cell_start.as<int64_t>(), ctx->cell_runs.as<int64_t>(), ctx->runs.as<uint2>(), nc,
        ctx->qcount.as<uint32_t>(), ctx->perm.as<uint32_t>(), pos_off, rows, uint32_t(n));
    TJ_CHECK_LAUNCH();
  } else {
    TJ_CUDA(cudaMemsetAsync(fill, 0, sizeof(uint32_t) * n, s));
    scatter_pairs_kernel<<<blocks_for(n_pairs, 256), 256, 0, s>>>(
        ctx->pairs.as<uint2>(), n_pairs, ctx->perm.as<uint32_t>(), pos_off, fill, rows);
    TJ_CHECK_LAUNCH();
  }
  // sort each row into its final place; `fill` becomes the list of long rows
  {
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
  sort_big_rows(ctx, offsets, nbr, fill, nbig, s);
}

}  // namespace tj
