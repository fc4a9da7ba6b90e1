// Stable LSD radix sort of (uint64 key, uint32 value) pairs, 8-bit digits.
//
// Replaces the stable np.lexsort of grid.py:83 (cell coordinates, dim 0 most
// significant; ids ascending within a cell because the sort is stable and the
// values start as 0..n-1) and sorts the composite keys of oversized CSR rows in
// the canonical output.  Only ceil(key_bits/8) passes run.
//
// Per pass: (1) per-tile digit histograms, (2) one device-wide exclusive scan
// over the digit-major histogram table, (3) a stable scatter in which each
// 4096-key tile ranks its keys per digit with warp match_any + per-warp digit
// counters in shared memory, processing the tile in index order.
#include "internal.cuh"
#include "scan.cuh"

namespace tj {

constexpr int kSortThreads = 256;
constexpr int kSortRounds = 16;
constexpr int kSortTile = kSortThreads * kSortRounds;  // 4096 keys
constexpr int kRadix = 256;
constexpr int kSortWarps = kSortThreads / kWarp;

__global__ void __launch_bounds__(kSortThreads)
    radix_hist_kernel(const uint64_t* __restrict__ keys, int64_t n, int shift,
                      int64_t* __restrict__ hist, int64_t n_tiles) {
  __shared__ unsigned s_hist[kSortWarps][kRadix];
  for (int i = threadIdx.x; i < kSortWarps * kRadix; i += kSortThreads) (&s_hist[0][0])[i] = 0;
  __syncthreads();
  const int warp = threadIdx.x >> 5;
  const int64_t base = int64_t(blockIdx.x) * kSortTile;
#pragma unroll 4
  for (int r = 0; r < kSortRounds; ++r) {
    int64_t i = base + r * kSortThreads + threadIdx.x;
    if (i < n) atomicAdd(&s_hist[warp][(keys[i] >> shift) & 0xff], 1u);
  }
  __syncthreads();
  for (int dgt = threadIdx.x; dgt < kRadix; dgt += kSortThreads) {
    unsigned s = 0;
#pragma unroll
    for (int w = 0; w < kSortWarps; ++w) s += s_hist[w][dgt];
    hist[int64_t(dgt) * n_tiles + blockIdx.x] = s;
  }
}

__global__ void __launch_bounds__(kSortThreads)
    radix_scatter_kernel(const uint64_t* __restrict__ keys_in, const uint32_t* __restrict__ vals_in,
                         uint64_t* __restrict__ keys_out, uint32_t* __restrict__ vals_out,
                         int64_t n, int shift, const int64_t* __restrict__ offsets,
                         int64_t n_tiles) {
  __shared__ unsigned s_wcnt[kSortWarps][kRadix];
  __shared__ unsigned s_wpre[kSortWarps][kRadix];
  __shared__ unsigned s_run[kRadix];
  __shared__ int64_t s_goff[kRadix];
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < kSortWarps * kRadix; i += kSortThreads) (&s_wcnt[0][0])[i] = 0;
  for (int dgt = threadIdx.x; dgt < kRadix; dgt += kSortThreads) {
    s_run[dgt] = 0;
    s_goff[dgt] = offsets[int64_t(dgt) * n_tiles + blockIdx.x];
  }
  __syncthreads();
  const int64_t base = int64_t(blockIdx.x) * kSortTile;
  const unsigned lt = lanemask_lt();
  for (int r = 0; r < kSortRounds; ++r) {
    const int64_t i = base + r * kSortThreads + threadIdx.x;
    const bool valid = i < n;
    uint64_t key = 0;
    uint32_t val = 0;
    unsigned dgt = kRadix;  // sentinel for lanes past the end
    if (valid) {
      key = keys_in[i];
      val = vals_in ? vals_in[i] : uint32_t(i);
      dgt = unsigned(key >> shift) & 0xffu;
    }
    const unsigned peers = __match_any_sync(0xffffffffu, dgt);
    const unsigned rank = __popc(peers & lt);
    if (valid && rank == 0) s_wcnt[warp][dgt] = __popc(peers);
    __syncthreads();
    for (int d2 = threadIdx.x; d2 < kRadix; d2 += kSortThreads) {
      unsigned run = s_run[d2];
#pragma unroll
      for (int w = 0; w < kSortWarps; ++w) {
        unsigned c = s_wcnt[w][d2];
        s_wpre[w][d2] = run;
        run += c;
        s_wcnt[w][d2] = 0;
      }
      s_run[d2] = run;
    }
    __syncthreads();
    if (valid) {
      const int64_t dst = s_goff[dgt] + s_wpre[warp][dgt] + rank;
      keys_out[dst] = key;
      vals_out[dst] = val;
    }
  }
}

int64_t radix_sort_scratch_elems(int64_t n) {
  const int64_t tiles = ceil_div(n, kSortTile);
  return tiles * kRadix;
}

__global__ void iota_kernel(uint32_t* v, int64_t n) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    v[i] = uint32_t(i);
}

// Sorts by the low key_bits bits.  Returns 0 if the result is in (k0,v0), 1 if in (k1,v1).
// identity_values: v0's contents are ignored and the values start as 0..n-1.
int radix_sort_pairs(uint64_t* k0, uint32_t* v0, uint64_t* k1, uint32_t* v1, int64_t n,
                     int key_bits, bool identity_values, int64_t* hist, ScanScratch scan,
                     cudaStream_t stream) {
  const int passes = key_bits <= 0 ? 0 : (key_bits + 7) / 8;
  if (n <= 1 || passes == 0) {
    if (n > 0 && identity_values) {
      iota_kernel<<<unsigned(std::min<int64_t>(ceil_div(n, 256), 4096)), 256, 0, stream>>>(v0, n);
      TJ_CHECK_LAUNCH();
    }
    return 0;
  }
  const int64_t tiles = ceil_div(n, kSortTile);
  const uint32_t* vin = identity_values ? nullptr : v0;
  uint64_t* kin = k0;
  uint64_t* kout = k1;
  uint32_t* vout = v1;
  int cur = 0;
  for (int p = 0; p < passes; ++p) {
    const int shift = 8 * p;
    radix_hist_kernel<<<unsigned(tiles), kSortThreads, 0, stream>>>(kin, n, shift, hist, tiles);
    TJ_CHECK_LAUNCH();
    scan_exclusive(LoadAt<int64_t>{hist}, StoreAt<int64_t>{hist}, tiles * kRadix, scan, stream);
    radix_scatter_kernel<<<unsigned(tiles), kSortThreads, 0, stream>>>(kin, vin, kout, vout, n,
                                                                      shift, hist, tiles);
    TJ_CHECK_LAUNCH();
    // next pass reads what we just wrote
    cur ^= 1;
    kin = cur ? k1 : k0;
    kout = cur ? k0 : k1;
    vin = cur ? v1 : v0;
    vout = cur ? v0 : v1;
  }
  return cur;
}

}  // namespace tj
