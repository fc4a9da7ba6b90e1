// Device epsilon-grid index: cell keys, radix sort by cell, cell-ordered
// coordinates + chunk norms, the non-empty cell table, compacted candidate runs
// and the per-cell estimate.
//
// Reference semantics (grid.py):
//   coords = floor(x[:, :k] / eps) (FP64 true divide, grid.py:81) — here
//     __ddiv_rn + round-down conversion, bit-identical per coordinate;
//   stable lexsort, dim 0 primary (grid.py:83) — here a packed key with dim 0
//     in the high bits and a stable LSD radix sort of (key, id);
//   cells dict + ordered_cells + point_order (grid.py:85-94) — the sorted run
//     table (cell_key, cell_start) and perm;
//   candidates_for_cell = members of the occupied Chebyshev-1 neighbours in
//     lexicographic order (grid.py:104-133) — every neighbour row that differs
//     only in the last indexed dim is one contiguous position range of the
//     cell-ordered array, so a cell's candidate list is <= 3^(k-1) runs found by
//     two binary searches each, already in the reference's concatenation order.
#include <climits>
#include <cmath>
#include <cstring>

#include "internal.cuh"
#include "scan.cuh"

namespace tj {

struct KeyParams {
  int k;
  int shift[TJ_MAX_K_IDX];
  int word[TJ_MAX_K_IDX];
  long long cmin[TJ_MAX_K_IDX];
};

// Signed integer image of a double with the same order (finite values and infinities).
__host__ __device__ __forceinline__ long long ordered_bits(double v) {
  long long b;
  memcpy(&b, &v, sizeof(b));
  return b >= 0 ? b : (b ^ 0x7fffffffffffffffll);
}
__host__ __device__ __forceinline__ double from_ordered_bits(long long b) {
  if (b < 0) b ^= 0x7fffffffffffffffll;
  double v;
  memcpy(&v, &b, sizeof(v));
  return v;
}

__device__ __forceinline__ long long cell_coord(double x, double eps) {
  return __double2ll_rd(__ddiv_rn(x, eps));  // floor(x / eps), IEEE division
}

__global__ void minmax_init_kernel(long long* mm, int k) {
  int j = threadIdx.x;
  if (j < k) {
    mm[2 * j] = LLONG_MAX;
    mm[2 * j + 1] = LLONG_MIN;
  }
  if (j == 0) mm[2 * TJ_MAX_K_IDX] = 0;  // max squared norm, as bits of a non-negative double
}

// Coordinate bounds per indexed dim.  floor(x / eps) is monotone in x for eps > 0
// (IEEE division by a positive constant and floor both are), so the cell bounds
// are floor(min x / eps) and floor(max x / eps): the kernel only compares raw
// coordinates and the host divides the 2k extremes (bit-identical rounding).
__global__ void cell_minmax_kernel(const double* __restrict__ x, int64_t n, int ld, int k,
                                   double eps, long long* mm) {
  (void)eps;
  double lo[TJ_MAX_K_IDX], hi[TJ_MAX_K_IDX];
#pragma unroll
  for (int j = 0; j < TJ_MAX_K_IDX; ++j) {
    lo[j] = INFINITY;
    hi[j] = -INFINITY;
  }
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const double* row = x + i * ld;
#pragma unroll
    for (int j = 0; j < TJ_MAX_K_IDX; j += 2) {
      if (j < k) {
        double2 v;
        if (j + 1 < k && (ld & 1) == 0) v = *reinterpret_cast<const double2*>(row + j);
        else v = make_double2(row[j], j + 1 < k ? row[j + 1] : row[j]);
        lo[j] = fmin(lo[j], v.x);
        hi[j] = fmax(hi[j], v.x);
        if (j + 1 < k) {
          lo[j + 1] = fmin(lo[j + 1], v.y);
          hi[j + 1] = fmax(hi[j + 1], v.y);
        }
      }
    }
  }
  // warp -> block -> one atomic per block and dimension (doubles as ordered bit
  // patterns: min/max on the sign-adjusted integer image)
  __shared__ double s_lo[TJ_MAX_K_IDX][32], s_hi[TJ_MAX_K_IDX][32];
  const int warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
#pragma unroll
  for (int j = 0; j < TJ_MAX_K_IDX; ++j) {
    if (j >= k) break;
    double a = lo[j], b = hi[j];
    for (int o = 16; o > 0; o >>= 1) {
      a = fmin(a, __shfl_xor_sync(0xffffffffu, a, o));
      b = fmax(b, __shfl_xor_sync(0xffffffffu, b, o));
    }
    if (lane_id() == 0) {
      s_lo[j][warp] = a;
      s_hi[j][warp] = b;
    }
  }
  __syncthreads();
  if (threadIdx.x < k) {
    const int j = threadIdx.x;
    double a = INFINITY, b = -INFINITY;
    for (int w = 0; w < nwarps; ++w) {
      a = fmin(a, s_lo[j][w]);
      b = fmax(b, s_hi[j][w]);
    }
    atomicMin(&mm[2 * j], ordered_bits(a));
    atomicMax(&mm[2 * j + 1], ordered_bits(b));
  }
}

// K = uint32_t when the packed key has <= 32 bits (the radix sort moves 4 bytes less per key).
template <class K>
__global__ void cell_key_kernel(const double* __restrict__ x, int64_t n, int ld, double eps,
                                KeyParams kp, K* __restrict__ keys) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    uint64_t key = 0;
#pragma unroll
    for (int j = 0; j < TJ_MAX_K_IDX; ++j) {
      if (j < kp.k) {
        long long c = cell_coord(x[i * ld + j], eps);
        key |= uint64_t(c - kp.cmin[j] + 1) << kp.shift[j];
      }
    }
    keys[i] = K(key);
  }
}

// Two-word cell keys (> 63 bits): dims with word 1 in `hi`, the rest in `lo`;
// row i of x, or row perm[i] when perm is given (the keys in sorted order).
__global__ void cell_key2_kernel(const double* __restrict__ x, int64_t n, int ld, double eps,
                                 KeyParams kp, const uint32_t* __restrict__ perm,
                                 uint64_t* __restrict__ lo, uint64_t* __restrict__ hi) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t row = perm ? int64_t(perm[i]) : i;
    uint64_t kl = 0, kh = 0;
#pragma unroll
    for (int j = 0; j < TJ_MAX_K_IDX; ++j) {
      if (j < kp.k) {
        const long long c = cell_coord(x[row * ld + j], eps);
        const uint64_t f = uint64_t(c - kp.cmin[j] + 1) << kp.shift[j];
        if (kp.word[j]) kh |= f;
        else kl |= f;
      }
    }
    lo[i] = kl;
    hi[i] = kh;
  }
}

__global__ void gather_u64_kernel(const uint64_t* __restrict__ src, const uint32_t* __restrict__ idx,
                                  int64_t n, uint64_t* __restrict__ dst) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    dst[i] = src[idx[i]];
}

// Cell-ordered zero-padded coordinates, chunk norms in the reference order
// ((((0+x0^2)+x1^2)+x2^2)+x3^2 per chunk, kernels.py:126-130) and full norms.
// One chunk (d <= 4): the chunk norm is the norm, CN is not written (only the
// d > 4 kernels read it).  Rows are read as double2 when the row stride is even.
template <bool VEC>
__global__ void permute_kernel(const double* __restrict__ x, int64_t n, int ld, int d, int d_pad,
                               const uint32_t* __restrict__ perm, double* __restrict__ P,
                               double* __restrict__ CN, double* __restrict__ NRM,
                               unsigned long long* max_norm_bits) {
  const int nchunks = d_pad / 4;
  unsigned long long local_max = 0;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p < n;
       p += stride) {
    const int64_t id = perm[p];
    const double* src = x + id * ld;
    double* dst = P + p * d_pad;
    double total = 0.0;
    for (int c = 0; c < nchunks; ++c) {
      double v[4];
      if (VEC && 4 * c + 4 <= d) {
        const double2 lo = __ldg(reinterpret_cast<const double2*>(src + 4 * c));
        const double2 hi = __ldg(reinterpret_cast<const double2*>(src + 4 * c + 2));
        v[0] = lo.x;
        v[1] = lo.y;
        v[2] = hi.x;
        v[3] = hi.y;
      } else {
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const int j = 4 * c + t;
          v[t] = j < d ? __ldg(src + j) : 0.0;
        }
      }
      double s = 0.0;
#pragma unroll
      for (int t = 0; t < 4; ++t) s = __dadd_rn(s, __dmul_rn(v[t], v[t]));
      // d <= 3: the padding coordinate carries |x|^2 for the norm-in-K DMMA tile
      // (refine_lowd.cu); every reader of P uses only the first d coordinates otherwise.
      if (nchunks == 1 && d <= 3) v[3] = s;
      double2* dst2 = reinterpret_cast<double2*>(dst + 4 * c);
      dst2[0] = make_double2(v[0], v[1]);
      dst2[1] = make_double2(v[2], v[3]);
      if (nchunks > 1) CN[p * nchunks + c] = s;
      total = __dadd_rn(total, s);
    }
    NRM[p] = total;
    local_max = max(local_max, (unsigned long long)__double_as_longlong(total));
  }
  for (int o = 16; o > 0; o >>= 1)
    local_max = max(local_max, __shfl_xor_sync(0xffffffffu, local_max, o));
  if (lane_id() == 0) atomicMax(max_norm_bits, local_max);
}

// Short-circuit record (d > 4): SFX[p] = (sum of p's chunk norms from chunk
// nchunks/2 on, |p|^2) -- the one 16-byte record a DMMA tile needs besides the
// coordinates (the check point sits after half of the chunks, refine_tc.cu).
__global__ void suffix_kernel(const double* __restrict__ CN, const double* __restrict__ NRM,
                              int64_t n, int nchunks, double* __restrict__ SFX) {
  const int ch = nchunks / 2;
  for (int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p < n;
       p += int64_t(gridDim.x) * blockDim.x) {
    double acc = 0.0;
    for (int j = ch; j < nchunks; ++j) acc += CN[p * nchunks + j];
    reinterpret_cast<double2*>(SFX)[p] = make_double2(acc, NRM[p]);
  }
}

template <class K>
struct HeadFlag {
  const K* keys;
  __device__ int64_t operator()(int64_t i) const { return i == 0 || keys[i] != keys[i - 1]; }
};
template <class K>
struct CellTableOut {
  const K* keys;
  uint64_t* cell_key;
  int64_t* cell_start;
  __device__ void operator()(int64_t i, int64_t excl) const {
    if (i == 0 || keys[i] != keys[i - 1]) {
      cell_key[excl] = uint64_t(keys[i]);
      cell_start[excl] = i;
    }
  }
};

struct HeadFlag2 {
  const uint64_t* lo;
  const uint64_t* hi;
  __device__ int64_t operator()(int64_t i) const {
    return i == 0 || lo[i] != lo[i - 1] || hi[i] != hi[i - 1];
  }
};
struct CellTableOut2 {
  const uint64_t* lo;
  const uint64_t* hi;
  uint64_t* cell_key;
  uint64_t* cell_key_hi;
  int64_t* cell_start;
  __device__ void operator()(int64_t i, int64_t excl) const {
    if (i == 0 || lo[i] != lo[i - 1] || hi[i] != hi[i - 1]) {
      cell_key[excl] = lo[i];
      cell_key_hi[excl] = hi[i];
      cell_start[excl] = i;
    }
  }
};

// (hi, lo) lexicographic bounds over the two-word cell keys.
__device__ __forceinline__ bool key2_less(uint64_t ah, uint64_t al, uint64_t bh, uint64_t bl) {
  return ah < bh || (ah == bh && al < bl);
}
__device__ __forceinline__ int64_t lower_bound_key2(const uint64_t* kh, const uint64_t* kl,
                                                    int64_t n, uint64_t vh, uint64_t vl) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (key2_less(kh[mid], kl[mid], vh, vl)) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}
__device__ __forceinline__ int64_t upper_bound_key2(const uint64_t* kh, const uint64_t* kl,
                                                    int64_t n, uint64_t vh, uint64_t vl) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (!key2_less(vh, vl, kh[mid], kl[mid])) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ int64_t lower_bound_u64(const uint64_t* a, int64_t n, uint64_t v) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (a[mid] < v) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}
__device__ __forceinline__ int64_t upper_bound_u64(const uint64_t* a, int64_t n, uint64_t v) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (a[mid] <= v) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

struct RowParams {
  int k;
  int n_rows;                     // 3^(k-1)
  long long shift[TJ_MAX_K_IDX];  // as 64-bit for the offset arithmetic
  // Dense cell lookup (when the guarded coordinate box is small): the position
  // range {start, end} of the cell at each mixed-radix box index, {~0, ~0} when
  // empty (one dependent load to a row's range).  Null: binary search on cell_key.
  const uint2* dense;
  long long dstride[TJ_MAX_K_IDX];
  unsigned long long fmask[TJ_MAX_K_IDX];
  // two-word keys: high words of the cell keys (null: one word), word of each dim
  const uint64_t* key_hi;
  int word[TJ_MAX_K_IDX];
};

__device__ __forceinline__ long long dense_index(const RowParams& rp, uint64_t key) {
  long long idx = 0;
  for (int j = 0; j < rp.k; ++j) idx += (long long)((key >> rp.shift[j]) & rp.fmask[j]) * rp.dstride[j];
  return idx;
}

// Position range of the three box entries of a row (left to right along the last dim).
__device__ __forceinline__ void dense_range(uint2 c0, uint2 c1, uint2 c2, int64_t& b, int64_t& e) {
  constexpr uint32_t kEmpty = 0xffffffffu;
  const uint32_t first = c0.x != kEmpty ? c0.x : (c1.x != kEmpty ? c1.x : c2.x);
  const uint32_t last = c2.x != kEmpty ? c2.y : (c1.x != kEmpty ? c1.y : c0.y);
  if (first == kEmpty) {
    b = e = 0;
  } else {
    b = first;
    e = last;
  }
}

// Position range [b, e) of neighbour row r of the cell with key `key`.
__device__ __forceinline__ void neighbour_row(const RowParams& rp, uint64_t key, uint64_t key_hi,
                                              int r,
                                              const uint64_t* cell_key, const int64_t* cell_start,
                                              int64_t n_cells, int64_t& b, int64_t& e) {
  if (rp.dense) {
    // the row's three cells along the last dim are adjacent box entries
    long long idx = dense_index(rp, key);
    int rr = r;
    for (int j = rp.k - 2; j >= 0; --j) {
      idx += (long long)(rr % 3 - 1) * rp.dstride[j];
      rr /= 3;
    }
    const uint2 c0 = rp.dense[idx - 1], c1 = rp.dense[idx], c2 = rp.dense[idx + 1];
    dense_range(c0, c1, c2, b, e);
    return;
  }
  long long delta = 0, delta_hi = 0;
  int rr = r;
  for (int j = rp.k - 2; j >= 0; --j) {  // dim k-2 is the fastest-varying digit
    const int o = rr % 3 - 1;
    rr /= 3;
    if (rp.word[j]) delta_hi += (long long)o << rp.shift[j];
    else delta += (long long)o << rp.shift[j];
  }
  const uint64_t last = 1ull << rp.shift[rp.k - 1];  // dim k-1 is always in the low word
  if (rp.key_hi) {  // fields never carry into each other (coordinates are offset by 1)
    const uint64_t kh = key_hi + uint64_t(delta_hi);
    const int64_t a = lower_bound_key2(rp.key_hi, cell_key, n_cells, kh, key + uint64_t(delta) - last);
    const int64_t z = upper_bound_key2(rp.key_hi, cell_key, n_cells, kh, key + uint64_t(delta) + last);
    b = cell_start[a];
    e = cell_start[z];
    return;
  }
  const uint64_t lo_key = key + uint64_t(delta) - last;
  const uint64_t hi_key = key + uint64_t(delta) + last;
  const int64_t a = lower_bound_u64(cell_key, n_cells, lo_key);
  const int64_t z = upper_bound_u64(cell_key, n_cells, hi_key);
  b = cell_start[a];
  e = cell_start[z];
}

// Dense lookup of U cells at once (lane = neighbour row): the three box entries
// of every cell's row, then their position ranges -- U independent load chains
// per lane instead of one (the kernels below are load-latency bound).
template <int U>
__device__ __forceinline__ void dense_rows(const RowParams& rp, const uint64_t (&key)[U], int r,
                                           const int64_t* __restrict__ cell_start,
                                           int64_t (&b)[U], int64_t (&e)[U]) {
  long long delta = 0;
  int rr = r;
  for (int j = rp.k - 2; j >= 0; --j) {
    delta += (long long)(rr % 3 - 1) * rp.dstride[j];
    rr /= 3;
  }
  uint2 cc[U][3];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const long long idx = dense_index(rp, key[u]) + delta;
#pragma unroll
    for (int t = 0; t < 3; ++t) cc[u][t] = __ldg(rp.dense + idx - 1 + t);
  }
#pragma unroll
  for (int u = 0; u < U; ++u) dense_range(cc[u][0], cc[u][1], cc[u][2], b[u], e[u]);
}

// Galloping searches: the same neighbour row of consecutive cells (ascending
// keys) has non-decreasing bounds, so a warp that walks a contiguous range of
// cells starts every search at the row's previous answer (a few probes instead
// of a full binary search).
// first i >= from with a[i] >= v; a[from - 1] < v
__device__ __forceinline__ int64_t gallop_lb(const uint64_t* __restrict__ a, int64_t n, uint64_t v,
                                             int64_t from) {
  if (from >= n || a[from] >= v) return from;
  int64_t lo = from, hi = from + 1, step = 1;  // a[lo] < v
  while (hi < n && a[hi] < v) {
    lo = hi;
    step <<= 1;
    hi = from + step;
  }
  if (hi > n) hi = n;
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) >> 1;
    if (a[mid] < v) lo = mid;
    else hi = mid;
  }
  return hi;
}
// first i >= from with a[i] > v; a[from - 1] <= v
__device__ __forceinline__ int64_t gallop_ub(const uint64_t* __restrict__ a, int64_t n, uint64_t v,
                                             int64_t from) {
  if (from >= n || a[from] > v) return from;
  int64_t lo = from, hi = from + 1, step = 1;  // a[lo] <= v
  while (hi < n && a[hi] <= v) {
    lo = hi;
    step <<= 1;
    hi = from + step;
  }
  if (hi > n) hi = n;
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) >> 1;
    if (a[mid] <= v) lo = mid;
    else hi = mid;
  }
  return hi;
}

// Key range [lo, hi] of neighbour row r (one-word keys).
__device__ __forceinline__ void row_key_range(const RowParams& rp, uint64_t key, int r,
                                              uint64_t& lo, uint64_t& hi) {
  long long delta = 0;
  int rr = r;
  for (int j = rp.k - 2; j >= 0; --j) {
    delta += (long long)(rr % 3 - 1) << rp.shift[j];
    rr /= 3;
  }
  const uint64_t last = 1ull << rp.shift[rp.k - 1];
  lo = key + uint64_t(delta) - last;
  hi = key + uint64_t(delta) + last;
}

constexpr int kGallopSlots = 8;  // rows per lane: k_idx <= 6 (243 rows)

__device__ __forceinline__ bool use_gallop(const RowParams& rp) {
  return !rp.dense && !rp.key_hi && rp.n_rows <= 32 * kGallopSlots;
}

constexpr int kCandU = 4;  // cells per warp iteration (dense lookup)

// Warp per cell: number of non-empty runs and candidates.
__global__ void cand_count_kernel(RowParams rp, const uint64_t* __restrict__ cell_key,
                                  const int64_t* __restrict__ cell_start, int64_t n_cells,
                                  int64_t* __restrict__ run_count, int64_t* __restrict__ cand_count) {
  const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
  const int64_t w0 = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  if (rp.dense && rp.n_rows <= 32) {
    const int r = lane_id();
    for (int64_t c0 = w0 * kCandU; c0 < n_cells; c0 += warps * kCandU) {
      uint64_t key[kCandU];
#pragma unroll
      for (int u = 0; u < kCandU; ++u) key[u] = c0 + u < n_cells ? cell_key[c0 + u] : cell_key[c0];
      int64_t b[kCandU], e[kCandU];
      if (r < rp.n_rows) {
        dense_rows<kCandU>(rp, key, r, cell_start, b, e);
      } else {
#pragma unroll
        for (int u = 0; u < kCandU; ++u) b[u] = e[u] = 0;
      }
#pragma unroll
      for (int u = 0; u < kCandU; ++u) {
        const int64_t runs = __popc(__ballot_sync(0xffffffffu, e[u] > b[u]));
        const int64_t cands = warp_sum(e[u] - b[u]);
        if (lane_id() == 0 && c0 + u < n_cells) {
          run_count[c0 + u] = runs;
          cand_count[c0 + u] = cands;
        }
      }
    }
    return;
  }
  if (use_gallop(rp) && rp.n_rows <= 16) {
    // k_idx <= 3: each half-warp walks every other cell of the warp's range
    // (lane = row), so 2 cells per step instead of one with half the lanes idle
    const int64_t per = (n_cells + warps - 1) / warps;
    const int64_t cb = w0 * per, ce = min(n_cells, cb + per);
    const int h = int(lane_id()) >> 4, r = int(lane_id()) & 15;
    int64_t pa = 0, pz = 0;
    for (int64_t c0 = cb; c0 < ce; c0 += 2) {
      const int64_t c = c0 + h;
      const bool vc = c < ce;
      int64_t runs = 0, cands = 0;
      if (vc && r < rp.n_rows) {
        uint64_t lo, hi;
        row_key_range(rp, cell_key[c], r, lo, hi);
        const int64_t a = gallop_lb(cell_key, n_cells, lo, pa);
        const int64_t z = gallop_ub(cell_key, n_cells, hi, max(pz, a));
        pa = a;
        pz = z;
        const int64_t b = cell_start[a], e = cell_start[z];
        if (e > b) {
          runs = 1;
          cands = e - b;
        }
      }
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) {  // sums inside each half
        runs += __shfl_xor_sync(0xffffffffu, runs, o);
        cands += __shfl_xor_sync(0xffffffffu, cands, o);
      }
      if (r == 0 && vc) {
        run_count[c] = runs;
        cand_count[c] = cands;
      }
    }
    return;
  }
  if (use_gallop(rp)) {  // contiguous cells per warp, galloping row searches
    const int64_t per = (n_cells + warps - 1) / warps;
    const int64_t cb = w0 * per, ce = min(n_cells, cb + per);
    int64_t pa[kGallopSlots], pz[kGallopSlots];
#pragma unroll
    for (int i = 0; i < kGallopSlots; ++i) pa[i] = pz[i] = 0;
    for (int64_t c = cb; c < ce; ++c) {
      const uint64_t key = cell_key[c];
      int64_t runs = 0, cands = 0;
#pragma unroll
      for (int i = 0; i < kGallopSlots; ++i) {
        const int r = int(lane_id()) + 32 * i;
        if (r < rp.n_rows) {
          uint64_t lo, hi;
          row_key_range(rp, key, r, lo, hi);
          const int64_t a = gallop_lb(cell_key, n_cells, lo, pa[i]);
          const int64_t z = gallop_ub(cell_key, n_cells, hi, max(pz[i], a));
          pa[i] = a;
          pz[i] = z;
          const int64_t b = cell_start[a], e = cell_start[z];
          if (e > b) {
            runs += 1;
            cands += e - b;
          }
        }
      }
      runs = warp_sum(runs);
      cands = warp_sum(cands);
      if (lane_id() == 0) {
        run_count[c] = runs;
        cand_count[c] = cands;
      }
    }
    return;
  }
  for (int64_t c = w0; c < n_cells; c += warps) {
    const uint64_t key = cell_key[c];
    int64_t runs = 0, cands = 0;
    for (int r = lane_id(); r < rp.n_rows; r += 32) {
      int64_t b, e;
      neighbour_row(rp, key, rp.key_hi ? rp.key_hi[c] : 0ull, r, cell_key, cell_start, n_cells, b,
                    e);
      if (e > b) {
        runs += 1;
        cands += e - b;
      }
    }
    runs = warp_sum(runs);
    cands = warp_sum(cands);
    if (lane_id() == 0) {
      run_count[c] = runs;
      cand_count[c] = cands;
    }
  }
}

__global__ void cand_fill_kernel(RowParams rp, const uint64_t* __restrict__ cell_key,
                                 const int64_t* __restrict__ cell_start, int64_t n_cells,
                                 const int64_t* __restrict__ cell_runs, uint2* __restrict__ runs,
                                 uint32_t* __restrict__ run_off) {
  const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
  const unsigned lt = lanemask_lt();
  const int64_t w0 = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  if (rp.dense && rp.n_rows <= 32) {
    const int r = lane_id();
    for (int64_t c0 = w0 * kCandU; c0 < n_cells; c0 += warps * kCandU) {
      uint64_t key[kCandU];
      int64_t out[kCandU];
#pragma unroll
      for (int u = 0; u < kCandU; ++u) {
        key[u] = c0 + u < n_cells ? cell_key[c0 + u] : cell_key[c0];
        out[u] = c0 + u < n_cells ? cell_runs[c0 + u] : 0;
      }
      int64_t b[kCandU], e[kCandU];
      if (r < rp.n_rows) {
        dense_rows<kCandU>(rp, key, r, cell_start, b, e);
      } else {
#pragma unroll
        for (int u = 0; u < kCandU; ++u) b[u] = e[u] = 0;
      }
#pragma unroll
      for (int u = 0; u < kCandU; ++u) {
        const unsigned m = __ballot_sync(0xffffffffu, e[u] > b[u]);
        const int64_t len = e[u] - b[u];
        const int64_t inc = warp_inclusive_scan(len);
        if (e[u] > b[u] && c0 + u < n_cells) {
          runs[out[u] + __popc(m & lt)] = make_uint2(uint32_t(b[u]), uint32_t(e[u]));
          run_off[out[u] + __popc(m & lt)] = uint32_t(inc - len);
        }
      }
    }
    return;
  }
  if (use_gallop(rp) && rp.n_rows <= 16) {  // two cells per step, one per half-warp
    const int64_t per = (n_cells + warps - 1) / warps;
    const int64_t cb = w0 * per, ce = min(n_cells, cb + per);
    const int h = int(lane_id()) >> 4, r = int(lane_id()) & 15;
    const unsigned lt16 = (1u << r) - 1u;
    int64_t pa = 0, pz = 0;
    for (int64_t c0 = cb; c0 < ce; c0 += 2) {
      const int64_t c = c0 + h;
      const bool vc = c < ce;
      int64_t b = 0, e = 0, out = 0;
      if (vc && r < rp.n_rows) {
        uint64_t lo, hi;
        row_key_range(rp, cell_key[c], r, lo, hi);
        const int64_t a = gallop_lb(cell_key, n_cells, lo, pa);
        const int64_t z = gallop_ub(cell_key, n_cells, hi, max(pz, a));
        pa = a;
        pz = z;
        b = cell_start[a];
        e = cell_start[z];
        out = cell_runs[c];
      }
      const unsigned mh = (__ballot_sync(0xffffffffu, e > b) >> (16 * h)) & 0xffffu;
      const int64_t len = e - b;
      int64_t inc = len;
#pragma unroll
      for (int o = 1; o < 16; o <<= 1) {  // inclusive scan inside each half
        const int64_t t = __shfl_up_sync(0xffffffffu, inc, o, 16);
        if (r >= o) inc += t;
      }
      if (e > b) {
        runs[out + __popc(mh & lt16)] = make_uint2(uint32_t(b), uint32_t(e));
        run_off[out + __popc(mh & lt16)] = uint32_t(inc - len);
      }
    }
    return;
  }
  if (use_gallop(rp)) {
    const int64_t per = (n_cells + warps - 1) / warps;
    const int64_t cb = w0 * per, ce = min(n_cells, cb + per);
    int64_t pa[kGallopSlots], pz[kGallopSlots];
#pragma unroll
    for (int i = 0; i < kGallopSlots; ++i) pa[i] = pz[i] = 0;
    for (int64_t c = cb; c < ce; ++c) {
      const uint64_t key = cell_key[c];
      int64_t out = cell_runs[c];
      int64_t off = 0;
#pragma unroll
      for (int i = 0; i < kGallopSlots; ++i) {
        if (32 * i >= rp.n_rows) break;
        const int r = int(lane_id()) + 32 * i;
        int64_t b = 0, e = 0;
        if (r < rp.n_rows) {
          uint64_t lo, hi;
          row_key_range(rp, key, r, lo, hi);
          const int64_t a = gallop_lb(cell_key, n_cells, lo, pa[i]);
          const int64_t z = gallop_ub(cell_key, n_cells, hi, max(pz[i], a));
          pa[i] = a;
          pz[i] = z;
          b = cell_start[a];
          e = cell_start[z];
        }
        const unsigned m = __ballot_sync(0xffffffffu, e > b);
        const int64_t len = e - b;
        const int64_t inc = warp_inclusive_scan(len);
        if (e > b) {
          runs[out + __popc(m & lt)] = make_uint2(uint32_t(b), uint32_t(e));
          run_off[out + __popc(m & lt)] = uint32_t(off + inc - len);
        }
        out += __popc(m);
        off += __shfl_sync(0xffffffffu, inc, 31);
      }
    }
    return;
  }
  for (int64_t c = w0; c < n_cells; c += warps) {
    const uint64_t key = cell_key[c];
    int64_t out = cell_runs[c];
    int64_t off = 0;  // offset of the next run inside the concatenated candidate list
    for (int r0 = 0; r0 < rp.n_rows; r0 += 32) {
      const int r = r0 + lane_id();
      int64_t b = 0, e = 0;
      if (r < rp.n_rows)
        neighbour_row(rp, key, rp.key_hi ? rp.key_hi[c] : 0ull, r, cell_key, cell_start, n_cells,
                      b, e);
      const unsigned m = __ballot_sync(0xffffffffu, e > b);
      const int64_t len = e - b;
      const int64_t inc = warp_inclusive_scan(len);
      if (e > b) {
        runs[out + __popc(m & lt)] = make_uint2(uint32_t(b), uint32_t(e));
        run_off[out + __popc(m & lt)] = uint32_t(off + inc - len);
      }
      out += __popc(m);
      off += __shfl_sync(0xffffffffu, inc, 31);
    }
  }
}

__global__ void dense_fill_kernel(RowParams rp, const uint64_t* __restrict__ cell_key,
                                  const int64_t* __restrict__ cell_start, int64_t n_cells,
                                  uint2* __restrict__ dense) {
  for (int64_t c = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; c < n_cells;
       c += int64_t(gridDim.x) * blockDim.x)
    dense[dense_index(rp, cell_key[c])] = make_uint2(uint32_t(cell_start[c]), uint32_t(cell_start[c + 1]));
}

// cost = |cell|*|cand|, tiles = ceil(|cell|/8)*ceil(|cand|/8) (join.py:170-173, 257-261).
__global__ void cell_cost_kernel(const int64_t* __restrict__ cell_start,
                                 const int64_t* __restrict__ cand, int64_t n_cells,
                                 int64_t* __restrict__ cost, unsigned long long* totals) {
  unsigned long long c_sum = 0, t_sum = 0, mx = 0;
  for (int64_t c = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; c < n_cells;
       c += int64_t(gridDim.x) * blockDim.x) {
    const int64_t nq = cell_start[c + 1] - cell_start[c];
    const int64_t nc = cand[c];
    cost[c] = nq * nc;
    c_sum += nq * nc;
    t_sum += ((nq + 7) / 8) * ((nc + 7) / 8);
    mx = max(mx, (unsigned long long)nq);
  }
  for (int o = 16; o > 0; o >>= 1) {
    c_sum += __shfl_xor_sync(0xffffffffu, c_sum, o);
    t_sum += __shfl_xor_sync(0xffffffffu, t_sum, o);
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  if (lane_id() == 0) {
    atomicAdd(&totals[0], c_sum);
    atomicAdd(&totals[1], t_sum);
    atomicMax(&totals[2], mx);
  }
}

static unsigned grid_for(int64_t n, int threads) {
  return unsigned(std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, threads), kNumSMs * 16)));
}

ScanScratch scan_scratch(tj_ctx* ctx, int64_t n, cudaStream_t s) {
  ctx->scan_partial.ensure(sizeof(int64_t) * (scan_tiles(n) + 1), s);
  ctx->scan_total.ensure(sizeof(int64_t) * 4, s);
  return ScanScratch{ctx->scan_partial.as<int64_t>(), ctx->scan_total.as<int64_t>()};
}

template <class T>
static T read_scalar(const void* dptr, cudaStream_t s) {
  T v;
  TJ_CUDA(cudaMemcpyAsync(&v, dptr, sizeof(T), cudaMemcpyDeviceToHost, s));
  TJ_CUDA(cudaStreamSynchronize(s));
  return v;
}

void build_grid(tj_ctx* ctx, const double* x, int64_t n, int d, int64_t ld64, int k, double eps,
                cudaStream_t s) {
  GridState& g = ctx->g;
  g = GridState{};
  g.n = n;
  g.d = d;
  g.d_pad = int(ceil_div(d, 4) * 4);
  g.nchunks = g.d_pad / 4;
  g.k = k;
  g.eps = eps;
  g.eps_sq = eps * eps;  // fl(eps*eps) as in join.py:176
  const int ld = int(ld64);

  // 1. cell coordinate bounds -> packed key layout
  ctx->minmax.ensure(sizeof(long long) * (2 * TJ_MAX_K_IDX + 2), s);
  long long* mm = ctx->minmax.as<long long>();
  minmax_init_kernel<<<1, 32, 0, s>>>(mm, k);
  TJ_CHECK_LAUNCH();
  cell_minmax_kernel<<<unsigned(std::min<int64_t>(ceil_div(n, 256), 8 * kNumSMs)), 256, 0, s>>>(
      x, n, ld, k, eps, mm);
  TJ_CHECK_LAUNCH();
  long long hmm[2 * TJ_MAX_K_IDX];
  TJ_CUDA(cudaMemcpyAsync(hmm, mm, sizeof(long long) * 2 * k, cudaMemcpyDeviceToHost, s));
  TJ_CUDA(cudaStreamSynchronize(s));
  for (int j = 0; j < 2 * k; ++j)  // coordinate extremes -> cell extremes (grid.py:81)
    hmm[j] = (long long)std::floor(from_ordered_bits(hmm[j]) / eps);
  int bits[TJ_MAX_K_IDX];
  int total_bits = 0;
  for (int j = 0; j < k; ++j) {
    const unsigned long long span = (unsigned long long)(hmm[2 * j + 1] - hmm[2 * j]) + 2ull;
    int b = 0;
    while (b < 64 && (span >> b) != 0) ++b;
    bits[j] = b;
    total_bits += b;
    g.cmin[j] = hmm[2 * j];
  }
  g.wide = total_bits > 63;
  for (int j = 0; j < k; ++j) g.bits[j] = bits[j];
  {
    // dim 0 most significant; one word when the key fits in 63 bits, else the
    // last dims fill the low word and the rest go to the high word
    int sh = 0, j = k - 1;
    for (; j >= 0 && (!g.wide || sh + bits[j] <= 63); --j) {
      g.shift[j] = sh;
      g.word[j] = 0;
      sh += bits[j];
    }
    g.lo_bits = sh;
    sh = 0;
    for (; j >= 0; --j) {
      if (sh + bits[j] > 63)
        fail(TJ_EINVAL, "cell key over k_idx=" + std::to_string(k) + " indexed dimensions needs " +
                            std::to_string(total_bits) +
                            " bits (> 126); use a smaller k_idx or a larger epsilon");
      g.shift[j] = sh;
      g.word[j] = 1;
      sh += bits[j];
    }
    g.hi_bits = sh;
  }
  g.key_bits = total_bits;

  // 2. keys, 3. stable radix sort of (key, id)
  ctx->keys.ensure(sizeof(uint64_t) * n, s);
  ctx->keys_alt.ensure(sizeof(uint64_t) * n, s);
  ctx->perm.ensure(sizeof(uint32_t) * n, s);
  ctx->vals_alt.ensure(sizeof(uint32_t) * n, s);
  KeyParams kp{};
  kp.k = k;
  for (int j = 0; j < k; ++j) {
    kp.shift[j] = g.shift[j];
    kp.word[j] = g.word[j];
    kp.cmin[j] = g.cmin[j];
  }
  const int64_t hist_elems = radix_sort_scratch_elems(n);
  ctx->sort_hist.ensure(sizeof(int64_t) * hist_elems, s);
  ScanScratch sc = scan_scratch(ctx, std::max<int64_t>(hist_elems, n), s);
  ctx->cell_key.ensure(sizeof(uint64_t) * (n + 1), s);
  ctx->cell_start.ensure(sizeof(int64_t) * (n + 1), s);
  if (g.wide) {
    // lo word first, then the hi word (stable), as two LSD sorts; the sorted
    // keys are recomputed from the coordinates in the final order
    uint64_t* k0 = ctx->keys.as<uint64_t>();
    uint64_t* k1 = ctx->keys_alt.as<uint64_t>();
    ctx->keys_hi.ensure(sizeof(uint64_t) * n, s);
    ctx->cell_key_hi.ensure(sizeof(uint64_t) * (n + 1), s);
    uint64_t* kh = ctx->keys_hi.as<uint64_t>();
    cell_key2_kernel<<<grid_for(n, 256), 256, 0, s>>>(x, n, ld, eps, kp, nullptr, k0, kh);
    TJ_CHECK_LAUNCH();
    const int w1 = radix_sort_pairs(k0, ctx->perm.as<uint32_t>(), k1, ctx->vals_alt.as<uint32_t>(),
                                    n, g.lo_bits, true, ctx->sort_hist.as<int64_t>(), sc, s);
    uint32_t* pa = w1 ? ctx->vals_alt.as<uint32_t>() : ctx->perm.as<uint32_t>();
    uint32_t* pb = w1 ? ctx->perm.as<uint32_t>() : ctx->vals_alt.as<uint32_t>();
    gather_u64_kernel<<<grid_for(n, 256), 256, 0, s>>>(kh, pa, n, k0);
    TJ_CHECK_LAUNCH();
    const int w2 = radix_sort_pairs(k0, pa, k1, pb, n, g.hi_bits, false,
                                    ctx->sort_hist.as<int64_t>(), sc, s);
    if ((w2 ? pb : pa) != ctx->perm.as<uint32_t>()) std::swap(ctx->perm, ctx->vals_alt);
    cell_key2_kernel<<<grid_for(n, 256), 256, 0, s>>>(x, n, ld, eps, kp, ctx->perm.as<uint32_t>(),
                                                       k0, kh);
    TJ_CHECK_LAUNCH();
    scan_exclusive(HeadFlag2{k0, kh},
                   CellTableOut2{k0, kh, ctx->cell_key.as<uint64_t>(),
                                 ctx->cell_key_hi.as<uint64_t>(), ctx->cell_start.as<int64_t>()},
                   n, sc, s);
  } else if (total_bits <= 32) {
    uint32_t* k0 = ctx->keys.as<uint32_t>();
    uint32_t* k1 = ctx->keys_alt.as<uint32_t>();
    cell_key_kernel<uint32_t><<<grid_for(n, 256), 256, 0, s>>>(x, n, ld, eps, kp, k0);
    TJ_CHECK_LAUNCH();
    const int where = radix_sort_pairs32(k0, ctx->perm.as<uint32_t>(), k1,
                                         ctx->vals_alt.as<uint32_t>(), n, total_bits, true,
                                         ctx->sort_hist.as<int64_t>(), sc, s);
    if (where == 1) {
      std::swap(ctx->keys, ctx->keys_alt);
      std::swap(ctx->perm, ctx->vals_alt);
    }
    // 4. run table of non-empty cells
    const uint32_t* keys = ctx->keys.as<uint32_t>();
    scan_exclusive(HeadFlag<uint32_t>{keys},
                   CellTableOut<uint32_t>{keys, ctx->cell_key.as<uint64_t>(),
                                          ctx->cell_start.as<int64_t>()},
                   n, sc, s);
  } else {
    uint64_t* k0 = ctx->keys.as<uint64_t>();
    uint64_t* k1 = ctx->keys_alt.as<uint64_t>();
    cell_key_kernel<uint64_t><<<grid_for(n, 256), 256, 0, s>>>(x, n, ld, eps, kp, k0);
    TJ_CHECK_LAUNCH();
    const int where = radix_sort_pairs(k0, ctx->perm.as<uint32_t>(), k1,
                                       ctx->vals_alt.as<uint32_t>(), n, total_bits, true,
                                       ctx->sort_hist.as<int64_t>(), sc, s);
    if (where == 1) {
      std::swap(ctx->keys, ctx->keys_alt);
      std::swap(ctx->perm, ctx->vals_alt);
    }
    const uint64_t* keys = ctx->keys.as<uint64_t>();
    scan_exclusive(HeadFlag<uint64_t>{keys},
                   CellTableOut<uint64_t>{keys, ctx->cell_key.as<uint64_t>(),
                                          ctx->cell_start.as<int64_t>()},
                   n, sc, s);
  }
  g.n_cells = read_scalar<int64_t>(sc.total, s);
  TJ_CUDA(cudaMemcpyAsync(ctx->cell_start.as<int64_t>() + g.n_cells, &n, sizeof(int64_t),
                          cudaMemcpyHostToDevice, s));

  // 5. cell-ordered coordinates + norms
  ctx->P.ensure(sizeof(double) * n * g.d_pad, s);
  if (g.nchunks > 1) ctx->CN.ensure(sizeof(double) * n * g.nchunks, s);
  ctx->NRM.ensure(sizeof(double) * n, s);
  const bool vec = ld % 2 == 0 && d >= 4 && (reinterpret_cast<uintptr_t>(x) & 15) == 0;
  auto permute = vec ? permute_kernel<true> : permute_kernel<false>;
  permute<<<grid_for(n, 256), 256, 0, s>>>(
      x, n, ld, d, g.d_pad, ctx->perm.as<uint32_t>(), ctx->P.as<double>(), ctx->CN.as<double>(),
      ctx->NRM.as<double>(), reinterpret_cast<unsigned long long*>(mm + 2 * TJ_MAX_K_IDX));
  TJ_CHECK_LAUNCH();
  if (g.nchunks > 1) {
    ctx->SFX.ensure(sizeof(double) * 2 * n, s);
    suffix_kernel<<<grid_for(n, 256), 256, 0, s>>>(ctx->CN.as<double>(), ctx->NRM.as<double>(), n,
                                                    g.nchunks, ctx->SFX.as<double>());
    TJ_CHECK_LAUNCH();
  }

  // 6. candidate runs
  RowParams rp{};
  rp.k = k;
  rp.n_rows = 1;
  for (int j = 0; j < k - 1; ++j) rp.n_rows *= 3;
  for (int j = 0; j < k; ++j) {
    rp.shift[j] = g.shift[j];
    rp.word[j] = g.word[j];
  }
  rp.key_hi = g.wide ? ctx->cell_key_hi.as<uint64_t>() : nullptr;
  const int64_t nc = g.n_cells;
  // dense box lookup when the guarded box is small (<= max(8 * cells, 4M) entries)
  {
    long long box = 1;
    bool small = true;
    for (int j = k - 1; j >= 0; --j) {
      rp.dstride[j] = box;
      const int fbits = g.bits[j];
      rp.fmask[j] = fbits >= 64 ? ~0ull : (1ull << fbits) - 1;
      const long long span = (long long)(hmm[2 * j + 1] - hmm[2 * j]) + 3;  // fields 0..range+2
      if (box > (1ll << 40) / span) small = false;
      else box *= span;
    }
    if (!g.wide && small && box <= std::max<long long>(8 * nc, 1ll << 22)) {
      ctx->dense.ensure(sizeof(uint2) * box, s);
      TJ_CUDA(cudaMemsetAsync(ctx->dense.ptr, 0xff, sizeof(uint2) * box, s));
      rp.dense = ctx->dense.as<uint2>();
      dense_fill_kernel<<<grid_for(nc, 256), 256, 0, s>>>(rp, ctx->cell_key.as<uint64_t>(),
                                                          ctx->cell_start.as<int64_t>(), nc,
                                                          ctx->dense.as<uint2>());
      TJ_CHECK_LAUNCH();
    } else {
      rp.dense = nullptr;
    }
  }
  ctx->cell_runs.ensure(sizeof(int64_t) * (nc + 1), s);
  ctx->cell_cand.ensure(sizeof(int64_t) * (nc + 1), s);
  ctx->cell_cost.ensure(sizeof(int64_t) * (nc + 1), s);
  ctx->tmp64.ensure(sizeof(int64_t) * (nc + 1), s);
  const unsigned warp_blocks = grid_for(ceil_div(nc, rp.dense ? kCandU : 1) * 32, 256);
  cand_count_kernel<<<warp_blocks, 256, 0, s>>>(rp, ctx->cell_key.as<uint64_t>(),
                                                ctx->cell_start.as<int64_t>(), nc,
                                                ctx->tmp64.as<int64_t>(),
                                                ctx->cell_cand.as<int64_t>());
  TJ_CHECK_LAUNCH();
  sc = scan_scratch(ctx, std::max<int64_t>(hist_elems, n), s);
  scan_exclusive(LoadAt<int64_t>{ctx->tmp64.as<int64_t>()},
                 StoreAt<int64_t>{ctx->cell_runs.as<int64_t>()}, nc, sc, s);
  // the run count stays on the device (read back with the totals below): the run
  // table is sized for its bound, 3^(k-1) rows per cell
  TJ_CUDA(cudaMemcpyAsync(ctx->cell_runs.as<int64_t>() + nc, sc.total, sizeof(int64_t),
                          cudaMemcpyDeviceToDevice, s));
  const int64_t runs_bound = std::max<int64_t>(nc * rp.n_rows, 1);
  ctx->runs.ensure(sizeof(uint2) * runs_bound, s);
  ctx->run_off.ensure(sizeof(uint32_t) * runs_bound, s);
  cand_fill_kernel<<<warp_blocks, 256, 0, s>>>(rp, ctx->cell_key.as<uint64_t>(),
                                               ctx->cell_start.as<int64_t>(), nc,
                                               ctx->cell_runs.as<int64_t>(), ctx->runs.as<uint2>(),
                                               ctx->run_off.as<uint32_t>());
  TJ_CHECK_LAUNCH();

  // 7. per-cell estimate and totals
  unsigned long long* totals = reinterpret_cast<unsigned long long*>(ctx->scan_total.as<int64_t>());
  TJ_CUDA(cudaMemsetAsync(totals, 0, 4 * sizeof(int64_t), s));
  cell_cost_kernel<<<grid_for(nc, 256), 256, 0, s>>>(ctx->cell_start.as<int64_t>(),
                                                     ctx->cell_cand.as<int64_t>(), nc,
                                                     ctx->cell_cost.as<int64_t>(), totals);
  TJ_CHECK_LAUNCH();
  unsigned long long ht[3];
  unsigned long long maxnorm_bits;
  TJ_CUDA(cudaMemcpyAsync(&g.n_runs, ctx->cell_runs.as<int64_t>() + nc, sizeof(int64_t),
                          cudaMemcpyDeviceToHost, s));
  TJ_CUDA(cudaMemcpyAsync(ht, totals, sizeof(ht), cudaMemcpyDeviceToHost, s));
  TJ_CUDA(cudaMemcpyAsync(&maxnorm_bits, mm + 2 * TJ_MAX_K_IDX, sizeof(maxnorm_bits),
                          cudaMemcpyDeviceToHost, s));
  TJ_CUDA(cudaStreamSynchronize(s));
  g.candidates = int64_t(ht[0]);
  g.tiles = int64_t(ht[1]);
  g.max_cell = int64_t(ht[2]);
  double mn;
  memcpy(&mn, &maxnorm_bits, sizeof(mn));
  g.max_norm = mn;
  g.built = true;
}

// ---------------------------------------------------------------- work items
struct ItemCountIn {
  const int64_t* cell_start;
  const int64_t* cand;
  int64_t cb;
  int qpi;
  int64_t target;
  __device__ int64_t operator()(int64_t i) const {
    const int64_t c = cb + i;
    const int64_t nq = cell_start[c + 1] - cell_start[c];
    const int64_t nc = cand[c];
    const int64_t qeff = nq < qpi ? nq : qpi;
    int64_t slice = (target / (qeff > 0 ? qeff : 1) + 7) / 8 * 8;
    if (slice < 256) slice = 256;
    const int64_t nqb = (nq + qpi - 1) / qpi;
    const int64_t nsl = (nc + slice - 1) / slice;
    return nqb * nsl;
  }
};

__global__ void item_fill_kernel(const int64_t* __restrict__ cell_start,
                                 const int64_t* __restrict__ cand, int64_t cb, int64_t n,
                                 int qpi, int64_t target, const int64_t* __restrict__ offs,
                                 WorkItem* __restrict__ items) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t c = cb + i;
    const int64_t q_begin = cell_start[c];
    const int64_t nq = cell_start[c + 1] - q_begin;
    const int64_t nc = cand[c];
    const int64_t qeff = nq < qpi ? nq : qpi;
    int64_t slice = (target / (qeff > 0 ? qeff : 1) + 7) / 8 * 8;
    if (slice < 256) slice = 256;
    int64_t o = offs[i];
    for (int64_t q = 0; q < nq; q += qpi) {
      for (int64_t s0 = 0; s0 < nc; s0 += slice) {
        WorkItem w;
        w.cell = uint32_t(c);
        w.q0 = uint32_t(q_begin + q);
        w.nq = uint32_t(min(int64_t(qpi), nq - q));
        w.s0 = uint32_t(s0);
        w.s1 = uint32_t(min(nc, s0 + slice));
        w.pad = 0;
        items[o++] = w;
      }
    }
  }
}

// Low-d hit masks: every (query group, 8-candidate block) tile of the cells
// [cb, ce) owns one 64-bit mask.  Cell c's masks start at mbase[c - cb] and are
// ordered (group, block); block b = candidates [8b, 8b+8) of the concatenated
// list, i.e. the reference's tiling (join.py:257-261).
struct MaskCountIn {
  const int64_t* cell_start;
  const int64_t* cand;
  int64_t cb;
  const uint32_t* fwd;  // symmetric join: only blocks from the cell's own offset on
  __device__ int64_t operator()(int64_t i) const {
    const int64_t c = cb + i;
    const int64_t nc = cand[c] - (fwd ? int64_t(fwd[c]) : 0);
    return ((cell_start[c + 1] - cell_start[c] + 7) / 8) * ((nc + 7) / 8);
  }
};

// (The total over all cells is GridState::tiles, already on the host: no read-back.)
void build_mask_bases(tj_ctx* ctx, int64_t cb, int64_t ce, cudaStream_t s) {
  const int64_t n = ce - cb;
  if (n <= 0) return;
  ScanScratch sc = scan_scratch(ctx, std::max<int64_t>(n, 1), s);
  ctx->cell_mbase.ensure(sizeof(int64_t) * (n + 1), s);
  scan_exclusive(MaskCountIn{ctx->cell_start.as<int64_t>(), ctx->cell_cand.as<int64_t>(), cb,
                             ctx->symmetric ? ctx->fwd.as<uint32_t>() : nullptr},
                 StoreAt<int64_t>{ctx->cell_mbase.as<int64_t>()}, n, sc, s);
}

// Returns the item count.  With total_dev != nullptr (unsliced items, bound =
// cells + points/qpi) the count stays on the device (*total_dev) and the
// returned value is only an upper bound: no host round trip.
int64_t build_work_items(tj_ctx* ctx, int64_t cb, int64_t ce, int qpi, int64_t target,
                         cudaStream_t s, unsigned long long* total_dev) {
  const int64_t n = ce - cb;
  if (n <= 0) return 0;
  ScanScratch sc = scan_scratch(ctx, std::max<int64_t>(n, 1), s);
  ctx->tmp64.ensure(sizeof(int64_t) * (n + 1), s);
  ItemCountIn in{ctx->cell_start.as<int64_t>(), ctx->cell_cand.as<int64_t>(), cb, qpi, target};
  scan_exclusive(in, StoreAt<int64_t>{ctx->tmp64.as<int64_t>()}, n, sc, s);
  int64_t total;
  if (total_dev) {
    total = n + ctx->g.n / qpi + 1;
    TJ_CUDA(cudaMemcpyAsync(total_dev, sc.total, sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
  } else {
    total = read_scalar<int64_t>(sc.total, s);
  }
  ctx->items.ensure(sizeof(WorkItem) * std::max<int64_t>(total, 1), s);
  item_fill_kernel<<<grid_for(n, 256), 256, 0, s>>>(ctx->cell_start.as<int64_t>(),
                                                    ctx->cell_cand.as<int64_t>(), cb, n, qpi,
                                                    target, ctx->tmp64.as<int64_t>(),
                                                    ctx->items.as<WorkItem>());
  TJ_CHECK_LAUNCH();
  return total;
}

}  // namespace tj
