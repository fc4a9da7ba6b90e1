// Multi-GPU strong layout: cell-partitioned shards of one join.
//
// Replaces the reference's only data-parallel executor, a thread pool over a
// batch's cells (join.py:184-197), with one process per GPU owning a
// contiguous, cost-balanced range of the lexicographic cell order:
//  * bins: the first `pdims` (<= 2) indexed dims of a point's cell,
//    b_j = floor(x_j / eps) - origin_j (the grid's own IEEE division + floor,
//    grid.py:81), numbered lexicographically L = b_0 * span_1 + b_1 -- the
//    prefix of the reference's lexicographic cell order (grid.py:83);
//  * a rank owns the bins [own_lo, own_hi] (inclusive, lexicographic), hence
//    every grid cell whose prefix falls there -- one contiguous cell range;
//  * it needs the points of its own bins plus the one-cell halo: a point is
//    kept when some bin within Chebyshev distance 1 of its own is owned.  For
//    a neighbour row q0 in {b0-1, b0, b0+1} the candidate bins are the
//    lexicographic interval q0*span1 + [b1-1, b1+1] (clipped), so the test is
//    three interval intersections;
//  * the kept points are compacted stably, so local ids are monotone in global
//    ids: cells, candidate lists and sorted rows of the local grid are exactly
//    the global grid's for the owned cells (ids mapped through `gid`).
// Kernels here: prefix bounds, prefix histogram (the estimator's input), the
// halo select, the owned cell range of a local grid, id remapping, per-row
// counts scattered to global ids, and row placement at global CSR offsets
// (device memory or mapped pinned host memory).
#include <climits>

#include "internal.cuh"
#include "scan.cuh"

namespace tj {

struct Bins {
  int pdims;
  long long origin0, origin1;
  long long span0, span1;
  double eps;
};

__device__ __forceinline__ long long bin_coord(double x, double eps) {
  return __double2ll_rd(__ddiv_rn(x, eps));  // floor(x / eps), as grid.cu cell_coord
}

__device__ __forceinline__ void point_bins(const double* row, const Bins& b, long long& b0,
                                           long long& b1) {
  b0 = bin_coord(row[0], b.eps) - b.origin0;
  b1 = b.pdims > 1 ? bin_coord(row[1], b.eps) - b.origin1 : 0;
}

// Does the Chebyshev-1 neighbourhood of bin (b0, b1) meet the owned interval?
__device__ __forceinline__ bool bin_needed(long long b0, long long b1, const Bins& b,
                                           long long lo, long long hi) {
  bool need = false;
#pragma unroll
  for (int dq = -1; dq <= 1; ++dq) {
    const long long q0 = b0 + dq;
    if (q0 < 0 || q0 >= b.span0) continue;
    const long long l = q0 * b.span1 + max(b1 - (b.pdims > 1 ? 1 : 0), 0ll);
    const long long h = q0 * b.span1 + min(b1 + (b.pdims > 1 ? 1 : 0), b.span1 - 1);
    need |= (l <= hi) && (h >= lo);
  }
  return need;
}

__global__ void shard_bounds_kernel(const double* __restrict__ x, int64_t n, int64_t ld, int pdims,
                                    double eps, long long* mm) {
  long long lo0 = LLONG_MAX, hi0 = LLONG_MIN, lo1 = LLONG_MAX, hi1 = LLONG_MIN;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const long long c0 = bin_coord(x[i * ld], eps);
    lo0 = min(lo0, c0);
    hi0 = max(hi0, c0);
    if (pdims > 1) {
      const long long c1 = bin_coord(x[i * ld + 1], eps);
      lo1 = min(lo1, c1);
      hi1 = max(hi1, c1);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lo0 = min(lo0, __shfl_xor_sync(0xffffffffu, lo0, o));
    hi0 = max(hi0, __shfl_xor_sync(0xffffffffu, hi0, o));
    lo1 = min(lo1, __shfl_xor_sync(0xffffffffu, lo1, o));
    hi1 = max(hi1, __shfl_xor_sync(0xffffffffu, hi1, o));
  }
  if (lane_id() == 0) {
    atomicMin(&mm[0], lo0);
    atomicMax(&mm[1], hi0);
    atomicMin(&mm[2], lo1);
    atomicMax(&mm[3], hi1);
  }
}

__global__ void shard_bounds_init(long long* mm) {
  mm[0] = LLONG_MAX;
  mm[1] = LLONG_MIN;
  mm[2] = LLONG_MAX;
  mm[3] = LLONG_MIN;
}

// Per-bin point counts; a shared-memory histogram per block when the bins fit.
__global__ void shard_hist_kernel(const double* __restrict__ x, int64_t n, int64_t ld, Bins b,
                                  unsigned long long* __restrict__ hist, int smem_bins) {
  extern __shared__ unsigned int s_hist[];
  const long long nbins = b.span0 * b.span1;
  const bool local = nbins <= smem_bins;
  if (local)
    for (int i = threadIdx.x; i < nbins; i += blockDim.x) s_hist[i] = 0;
  __syncthreads();
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    long long b0, b1;
    point_bins(x + i * ld, b, b0, b1);
    const long long L = b0 * b.span1 + b1;
    if (L < 0 || L >= nbins) continue;  // outside the agreed bounds: caller error, dropped
    if (local) atomicAdd(&s_hist[L], 1u);
    else atomicAdd(&hist[L], 1ull);
  }
  __syncthreads();
  if (local)
    for (int i = threadIdx.x; i < nbins; i += blockDim.x)
      if (s_hist[i]) atomicAdd(&hist[i], (unsigned long long)s_hist[i]);
}

struct HaloPred {
  const double* x;
  int64_t ld;
  Bins b;
  long long lo, hi;
  __device__ bool operator()(int64_t i) const {
    long long b0, b1;
    point_bins(x + i * ld, b, b0, b1);
    return bin_needed(b0, b1, b, lo, hi);
  }
};

struct HaloCount {
  HaloPred p;
  __device__ int64_t operator()(int64_t i) const { return p(i) ? 1 : 0; }
};

struct HaloWrite {
  HaloPred p;
  int d;
  double* out;
  int64_t ld_out;
  uint32_t* gid;
  int64_t gid_base;
  __device__ void operator()(int64_t i, int64_t at) const {
    if (!p(i)) return;
    const double* src = p.x + i * p.ld;
    double* dst = out + at * ld_out;
    for (int j = 0; j < ld_out; ++j) dst[j] = j < d ? src[j] : 0.0;
    gid[at] = uint32_t(gid_base + i);
  }
};

struct NoStore {
  __device__ void operator()(int64_t, int64_t) const {}
};

// Points of this rank's rows needed by each of G <= 64 ranks (owned bins + halo):
// the destination set of every row (a bit mask, kept for the write pass) and the
// count per destination.
__global__ void route_count_kernel(const double* __restrict__ x, int64_t n, int64_t ld, Bins b,
                                   const long long* __restrict__ lo, const long long* __restrict__ hi,
                                   int G, unsigned long long* __restrict__ counts,
                                   unsigned long long* __restrict__ dest) {
  extern __shared__ unsigned int s_cnt[];
  for (int r = threadIdx.x; r < G; r += blockDim.x) s_cnt[r] = 0;
  __syncthreads();
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    long long b0, b1;
    point_bins(x + i * ld, b, b0, b1);
    unsigned long long m = 0;
    for (int r = 0; r < G; ++r)
      if (bin_needed(b0, b1, b, lo[r], hi[r])) {
        m |= 1ull << r;
        atomicAdd(&s_cnt[r], 1u);
      }
    dest[i] = m;
  }
  __syncthreads();
  for (int r = threadIdx.x; r < G; r += blockDim.x)
    if (s_cnt[r]) atomicAdd(&counts[r], (unsigned long long)s_cnt[r]);
}

// Warp-tiled stable routing: warp w of the grid owns rows [w * kRouteRows, +kRouteRows).
// Pass 1 counts, per destination, the rows of every warp tile (dest-major table);
// one exclusive scan gives every (destination, tile) its first output row, so the
// send buffer is destination-major and stable; pass 2 writes.
constexpr int kRouteRows = 512;

__global__ void route_tile_count_kernel(const unsigned long long* __restrict__ dest, int64_t n,
                                        int G, int64_t n_tiles, int64_t* __restrict__ tile_cnt) {
  const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
  for (int64_t t = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5; t < n_tiles; t += warps) {
    const int64_t i0 = t * kRouteRows, i1 = min(n, (t + 1) * kRouteRows);
    for (int r = 0; r < G; ++r) {  // the tile's masks stay in L1 across destinations
      unsigned c = 0;
      for (int64_t i = i0 + lane_id(); i < i1; i += 32) c += unsigned((dest[i] >> r) & 1ull);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
      if (lane_id() == 0) tile_cnt[int64_t(r) * n_tiles + t] = c;
    }
  }
}

// One pass over the tile's rows: every 32-row round loads its destination
// masks and rows once, then places the rows of each destination present in the
// round (ballot rank = stable order) -- no per-destination re-walk of the tile.
// The per-destination cursors live in shared memory (G <= 64).
template <bool VEC>
__global__ void __launch_bounds__(256)
    route_tile_write_kernel(const unsigned long long* __restrict__ dest, int64_t n, int G,
                            int64_t n_tiles, const int64_t* __restrict__ tile_off,
                            const double* __restrict__ x, int64_t ld, int d,
                            double* __restrict__ out, int64_t ld_out, uint32_t* __restrict__ gid,
                            int64_t gid_base) {
  __shared__ int64_t s_at[8][64];
  const int warp = threadIdx.x >> 5, lane = lane_id();
  int64_t* at = s_at[warp];
  const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
  const unsigned lt = lanemask_lt();
  for (int64_t t = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5; t < n_tiles; t += warps) {
    const int64_t i0 = t * kRouteRows, i1 = min(n, (t + 1) * kRouteRows);
    __syncwarp();
    for (int r = lane; r < G; r += 32) at[r] = tile_off[int64_t(r) * n_tiles + t];
    __syncwarp();
    for (int64_t base = i0; base < i1; base += 32) {
      const int64_t i = base + lane;
      const unsigned long long m = i < i1 ? dest[i] : 0ull;
      double2 v0 = make_double2(0.0, 0.0), v1 = v0;
      if (VEC && m) {
        const double2* src = reinterpret_cast<const double2*>(x + i * ld);
        v0 = __ldg(src);
        if (ld_out > 2) v1 = __ldg(src + 1);
      }
      unsigned long long present = m;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) present |= __shfl_xor_sync(0xffffffffu, present, o);
      while (present) {
        const int r = __ffsll(present) - 1;
        present &= present - 1ull;
        const bool hit = (m >> r) & 1ull;
        const unsigned bal = __ballot_sync(0xffffffffu, hit);
        const int64_t a = at[r];
        if (hit) {
          const int64_t o = a + __popc(bal & lt);
          double* dst = out + o * ld_out;
          if (VEC) {
            if (ld_out == 4) {
              reinterpret_cast<double2*>(dst)[0] = v0;
              reinterpret_cast<double2*>(dst)[1] = v1;
            } else {
              const double* src = x + i * ld;
              for (int j = 0; j < ld_out; j += 2)
                *reinterpret_cast<double2*>(dst + j) = __ldg(reinterpret_cast<const double2*>(src + j));
            }
          } else {
            const double* src = x + i * ld;
            for (int j = 0; j < ld_out; ++j) dst[j] = j < d ? src[j] : 0.0;
          }
          gid[o] = uint32_t(gid_base + i);
        }
        __syncwarp();
        if (lane == 0) at[r] = a + __popc(bal);
        __syncwarp();
      }
    }
  }
}

// First cell c of the local grid whose bin index is >= target (cells are
// lexicographic, so their prefix bins are non-decreasing).
__global__ void cell_bound_kernel(const double* __restrict__ P, const int64_t* __restrict__ cell_start,
                                  int64_t n_cells, int d_pad, Bins b, long long lo, long long hi,
                                  int64_t* out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  for (int side = 0; side < 2; ++side) {
    const long long target = side == 0 ? lo : hi + 1;
    int64_t a = 0, z = n_cells;
    while (a < z) {
      const int64_t mid = (a + z) >> 1;
      long long b0, b1;
      point_bins(P + cell_start[mid] * d_pad, b, b0, b1);
      if (b0 * b.span1 + b1 < target) a = mid + 1;
      else z = mid;
    }
    out[side] = a;
  }
}

__global__ void remap_ids_kernel(uint32_t* __restrict__ ids, int64_t m, const uint32_t* __restrict__ gid) {
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < m;
       e += int64_t(gridDim.x) * blockDim.x)
    ids[e] = gid[ids[e]];
}

__global__ void scatter_counts_kernel(const int64_t* __restrict__ loff, int64_t n_rows,
                                      const uint32_t* __restrict__ gid, int32_t* __restrict__ counts) {
  for (int64_t l = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; l < n_rows;
       l += int64_t(gridDim.x) * blockDim.x) {
    const int64_t c = loff[l + 1] - loff[l];
    if (c) counts[gid[l]] = int32_t(c);
  }
}

// One byte per id when every row is shorter than 256 (the usual case: the
// all-reduce then moves n bytes instead of 4n); longer rows set *overflow and
// the caller falls back to the int32 counts.
__global__ void scatter_counts_u8_kernel(const int64_t* __restrict__ loff, int64_t n_rows,
                                         const uint32_t* __restrict__ gid,
                                         uint8_t* __restrict__ counts, int32_t* overflow) {
  bool over = false;
  for (int64_t l = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; l < n_rows;
       l += int64_t(gridDim.x) * blockDim.x) {
    const int64_t c = loff[l + 1] - loff[l];
    if (c) counts[gid[l]] = uint8_t(c > 255 ? 255 : c);
    over |= c > 255;
  }
  if (__any_sync(0xffffffffu, over) && lane_id() == 0) atomicOr(overflow, 1);
}

// Warp per local row: copy the row (ids already global) to its global offset.
__global__ void place_rows_kernel(const int64_t* __restrict__ loff, const uint32_t* __restrict__ nbr,
                                  int64_t n_rows, const uint32_t* __restrict__ gid,
                                  const int64_t* __restrict__ goff, uint32_t* __restrict__ dst) {
  const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
  for (int64_t l = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5; l < n_rows; l += warps) {
    const int64_t a = loff[l], z = loff[l + 1];
    if (a == z) continue;
    uint32_t* out = dst + goff[gid[l]];
    for (int64_t e = a + lane_id(); e < z; e += 32) out[e - a] = nbr[e];
  }
}

static unsigned grid_for(int64_t n, int threads) {
  return unsigned(std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, threads), int64_t(kNumSMs) * 16)));
}

static Bins make_bins(int pdims, double eps, const int64_t* origin, const int64_t* span) {
  Bins b;
  b.pdims = pdims;
  b.eps = eps;
  b.origin0 = origin[0];
  b.origin1 = pdims > 1 ? origin[1] : 0;
  b.span0 = span[0];
  b.span1 = pdims > 1 ? span[1] : 1;
  return b;
}

void shard_bounds(tj_ctx* ctx, const double* x, int64_t n, int64_t ld, int pdims, double eps,
                  int64_t* lo, int64_t* hi, cudaStream_t s) {
  ctx->minmax.ensure(sizeof(long long) * (2 * TJ_MAX_K_IDX + 4), s);
  long long* mm = ctx->minmax.as<long long>();
  shard_bounds_init<<<1, 1, 0, s>>>(mm);
  TJ_CHECK_LAUNCH();
  if (n > 0) {
    shard_bounds_kernel<<<grid_for(n, 256), 256, 0, s>>>(x, n, ld, pdims, eps, mm);
    TJ_CHECK_LAUNCH();
  }
  long long h[4];
  TJ_CUDA(cudaMemcpyAsync(h, mm, sizeof(h), cudaMemcpyDeviceToHost, s));
  TJ_CUDA(cudaStreamSynchronize(s));
  lo[0] = h[0];
  hi[0] = h[1];
  if (pdims > 1) {
    lo[1] = h[2];
    hi[1] = h[3];
  }
}

void shard_histogram(const double* x, int64_t n, int64_t ld, int pdims, double eps,
                     const int64_t* origin, const int64_t* span, int64_t* hist, cudaStream_t s) {
  const Bins b = make_bins(pdims, eps, origin, span);
  const int64_t nbins = b.span0 * b.span1;
  TJ_CUDA(cudaMemsetAsync(hist, 0, sizeof(int64_t) * nbins, s));
  if (n == 0) return;
  constexpr int kSmemBins = 12288;  // 48 KB of 32-bit counters
  const size_t smem = nbins <= kSmemBins ? sizeof(unsigned) * size_t(nbins) : 0;
  shard_hist_kernel<<<grid_for(n, 256), 256, smem, s>>>(
      x, n, ld, b, reinterpret_cast<unsigned long long*>(hist), kSmemBins);
  TJ_CHECK_LAUNCH();
}

int64_t shard_select(tj_ctx* ctx, const double* x, int64_t n, int64_t ld, int d, int pdims,
                     double eps, const int64_t* origin, const int64_t* span, int64_t own_lo,
                     int64_t own_hi, double* out, int64_t ld_out, uint32_t* gid, int64_t gid_base,
                     int64_t capacity, cudaStream_t s) {
  const Bins b = make_bins(pdims, eps, origin, span);
  const HaloPred pred{x, ld, b, own_lo, own_hi};
  ScanScratch sc = scan_scratch(ctx, std::max<int64_t>(n, 1), s);
  if (!out) {
    scan_exclusive(HaloCount{pred}, NoStore{}, n, sc, s);
  } else {
    scan_exclusive(HaloCount{pred}, HaloWrite{pred, d, out, ld_out, gid, gid_base}, n, sc, s);
  }
  int64_t total = 0;
  TJ_CUDA(cudaMemcpyAsync(&total, sc.total, sizeof(total), cudaMemcpyDeviceToHost, s));
  TJ_CUDA(cudaStreamSynchronize(s));
  if (out && total > capacity) fail(TJ_ECAPACITY, "shard_select: output capacity too small");
  return total;
}

void shard_route(tj_ctx* ctx, const double* x, int64_t n, int64_t ld, int d, int pdims, double eps,
                 const int64_t* origin, const int64_t* span, const int64_t* lo, const int64_t* hi,
                 int G, int64_t* counts, double* out, int64_t ld_out, uint32_t* gid,
                 int64_t gid_base, int64_t capacity, cudaStream_t s) {
  const Bins b = make_bins(pdims, eps, origin, span);
  if (G > 64) fail(TJ_EINVAL, "shard_route supports up to 64 ranks");
  if (!out) {  // counts only: one pass over the rows, one read-back
    ctx->tmp64.ensure(sizeof(long long) * (2 * G) + sizeof(unsigned long long) * G + 64, s);
    long long* dlo = reinterpret_cast<long long*>(ctx->tmp64.ptr);
    long long* dhi = dlo + G;
    unsigned long long* dcnt = reinterpret_cast<unsigned long long*>(dhi + G);
    std::vector<long long> hlh(2 * G);
    for (int r = 0; r < G; ++r) {
      hlh[r] = lo[r];
      hlh[G + r] = hi[r];
    }
    TJ_CUDA(cudaMemcpyAsync(dlo, hlh.data(), sizeof(long long) * 2 * G, cudaMemcpyHostToDevice, s));
    TJ_CUDA(cudaMemsetAsync(dcnt, 0, sizeof(unsigned long long) * G, s));
    ctx->route_dest.ensure(sizeof(unsigned long long) * std::max<int64_t>(n, 1), s);
    if (n > 0) {
      route_count_kernel<<<grid_for(n, 256), 256, sizeof(unsigned) * G, s>>>(
          x, n, ld, b, dlo, dhi, G, dcnt, ctx->route_dest.as<unsigned long long>());
      TJ_CHECK_LAUNCH();
    }
    std::vector<unsigned long long> hc(G);
    TJ_CUDA(cudaMemcpyAsync(hc.data(), dcnt, sizeof(unsigned long long) * G, cudaMemcpyDeviceToHost, s));
    TJ_CUDA(cudaStreamSynchronize(s));
    for (int r = 0; r < G; ++r) counts[r] = int64_t(hc[r]);
    return;
  }
  // write (after the count call on the same rows: its destination masks):
  // destination r's rows at [sum(counts[<r]), ...), stable, no read-back
  const unsigned long long* dest = ctx->route_dest.as<unsigned long long>();
  int64_t total = 0;
  for (int r = 0; r < G; ++r) total += counts[r];
  if (total > capacity) fail(TJ_ECAPACITY, "shard_route: output capacity too small");
  if (n == 0 || total == 0) return;
  const int64_t n_tiles = ceil_div(n, kRouteRows);
  ctx->route_tiles.ensure(sizeof(int64_t) * (G * n_tiles + 1), s);
  int64_t* tiles = ctx->route_tiles.as<int64_t>();
  const unsigned warp_grid = grid_for(n_tiles * 32, 256);
  route_tile_count_kernel<<<warp_grid, 256, 0, s>>>(dest, n, G, n_tiles, tiles);
  TJ_CHECK_LAUNCH();
  ScanScratch sc = scan_scratch(ctx, G * n_tiles, s);
  scan_exclusive(LoadAt<int64_t>{tiles}, StoreAt<int64_t>{tiles}, G * n_tiles, sc, s);
  // unpadded even-width rows copy as double2
  const bool vec = ld == ld_out && ld % 2 == 0 && d == ld &&
                   ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(out)) & 15) == 0;
  auto write = vec ? route_tile_write_kernel<true> : route_tile_write_kernel<false>;
  write<<<warp_grid, 256, 0, s>>>(dest, n, G, n_tiles, tiles, x, ld, d, out, ld_out, gid, gid_base);
  TJ_CHECK_LAUNCH();
}

void shard_cell_range(tj_ctx* ctx, int pdims, const int64_t* origin, const int64_t* span,
                      int64_t own_lo, int64_t own_hi, int64_t* begin, int64_t* end, cudaStream_t s) {
  const GridState& g = ctx->g;
  const Bins b = make_bins(pdims, g.eps, origin, span);
  ctx->tmp64.ensure(sizeof(int64_t) * std::max<int64_t>(g.n + 1, 2), s);
  int64_t* out = ctx->tmp64.as<int64_t>();
  cell_bound_kernel<<<1, 32, 0, s>>>(ctx->P.as<double>(), ctx->cell_start.as<int64_t>(), g.n_cells,
                                     g.d_pad, b, own_lo, own_hi, out);
  TJ_CHECK_LAUNCH();
  int64_t h[2];
  TJ_CUDA(cudaMemcpyAsync(h, out, sizeof(h), cudaMemcpyDeviceToHost, s));
  TJ_CUDA(cudaStreamSynchronize(s));
  *begin = h[0];
  *end = h[1];
}

void shard_remap_ids(uint32_t* ids, int64_t m, const uint32_t* gid, cudaStream_t s) {
  if (m <= 0) return;
  remap_ids_kernel<<<grid_for(m, 256), 256, 0, s>>>(ids, m, gid);
  TJ_CHECK_LAUNCH();
}

void shard_scatter_counts(const int64_t* loff, int64_t n_rows, const uint32_t* gid, int32_t* counts,
                          cudaStream_t s) {
  if (n_rows <= 0) return;
  scatter_counts_kernel<<<grid_for(n_rows, 256), 256, 0, s>>>(loff, n_rows, gid, counts);
  TJ_CHECK_LAUNCH();
}

void shard_scatter_counts_u8(const int64_t* loff, int64_t n_rows, const uint32_t* gid,
                             uint8_t* counts, int32_t* overflow, cudaStream_t s) {
  if (n_rows <= 0) return;
  scatter_counts_u8_kernel<<<grid_for(n_rows, 256), 256, 0, s>>>(loff, n_rows, gid, counts, overflow);
  TJ_CHECK_LAUNCH();
}

void shard_place_rows(const int64_t* loff, const uint32_t* nbr, int64_t n_rows, const uint32_t* gid,
                      const int64_t* goff, uint32_t* dst, cudaStream_t s) {
  if (n_rows <= 0) return;
  place_rows_kernel<<<grid_for(n_rows * 32, 256), 256, 0, s>>>(loff, nbr, n_rows, gid, goff, dst);
  TJ_CHECK_LAUNCH();
}

template <class T>
static void counts_to_offsets_t(tj_ctx* ctx, const T* counts, int64_t n, int64_t* offsets,
                                cudaStream_t s) {
  ScanScratch sc = scan_scratch(ctx, std::max<int64_t>(n, 1), s);
  scan_exclusive(LoadAt<T>{counts}, StoreAt<int64_t>{offsets}, n, sc, s);
  TJ_CUDA(cudaMemcpyAsync(offsets + n, sc.total, sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
}

void counts_to_offsets(tj_ctx* ctx, const int32_t* counts, int64_t n, int64_t* offsets,
                       cudaStream_t s) {
  counts_to_offsets_t(ctx, counts, n, offsets, s);
}

void counts_to_offsets_u8(tj_ctx* ctx, const uint8_t* counts, int64_t n, int64_t* offsets,
                          cudaStream_t s) {
  counts_to_offsets_t(ctx, counts, n, offsets, s);
}

}  // namespace tj
