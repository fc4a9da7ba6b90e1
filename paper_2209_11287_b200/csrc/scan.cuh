// Device-wide exclusive prefix sum (int64), warp-tiled reduce-then-scan.
//
// Used for every offset computation on the path: cell numbering from sort-run
// heads, candidate-run offsets, work-item offsets, radix digit offsets and the
// CSR row offsets of the canonical output.  Each warp owns a tile of
// kScanItems*32 consecutive elements, read coalesced in 32-wide rounds.
#pragma once
#include "common.cuh"

namespace tj {

constexpr int kScanItems = 16;                   // rounds per warp tile
constexpr int kScanTile = kScanItems * kWarp;    // 512 elements per warp
constexpr int kScanBlock = 256;                  // 8 warps
constexpr int kScanWarps = kScanBlock / kWarp;

__device__ __forceinline__ int64_t warp_inclusive_scan(int64_t v) {
  const unsigned lane = lane_id();
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int64_t t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= (unsigned)o) v += t;
  }
  return v;
}

__device__ __forceinline__ int64_t warp_sum(int64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <class In>
__global__ void __launch_bounds__(kScanBlock) scan_reduce_kernel(In in, int64_t n, int64_t* partial,
                                                                 int64_t n_tiles) {
  const int64_t tile = int64_t(blockIdx.x) * kScanWarps + (threadIdx.x >> 5);
  if (tile >= n_tiles) return;
  const int64_t base = tile * kScanTile;
  int64_t s = 0;
#pragma unroll 4
  for (int r = 0; r < kScanItems; ++r) {
    int64_t i = base + r * kWarp + lane_id();
    if (i < n) s += in(i);
  }
  s = warp_sum(s);
  if (lane_id() == 0) partial[tile] = s;
}

// Single block: exclusive scan of the tile partials in place; total -> *total.
template <int kThreads = 1024>
__global__ void __launch_bounds__(kThreads) scan_partials_kernel(int64_t* partial, int64_t n_tiles,
                                                                 int64_t* total) {
  __shared__ int64_t warp_tot[kThreads / kWarp];
  __shared__ int64_t carry_s;
  if (threadIdx.x == 0) carry_s = 0;
  __syncthreads();
  const int warp = threadIdx.x >> 5;
  for (int64_t base = 0; base < n_tiles; base += kThreads) {
    const int64_t i = base + threadIdx.x;
    const int64_t v = i < n_tiles ? partial[i] : 0;
    const int64_t inc = warp_inclusive_scan(v);
    if (lane_id() == 31) warp_tot[warp] = inc;
    __syncthreads();
    if (warp == 0) {
      int64_t t = lane_id() < kThreads / kWarp ? warp_tot[lane_id()] : 0;
      int64_t ti = warp_inclusive_scan(t);
      if (lane_id() < kThreads / kWarp) warp_tot[lane_id()] = ti - t;
    }
    __syncthreads();
    const int64_t carry = carry_s;
    if (i < n_tiles) partial[i] = carry + warp_tot[warp] + inc - v;
    __syncthreads();
    if (threadIdx.x == kThreads - 1) carry_s = carry + warp_tot[warp] + inc;
    __syncthreads();
  }
  if (threadIdx.x == 0) *total = carry_s;
}

template <class In, class Out>
__global__ void __launch_bounds__(kScanBlock) scan_downsweep_kernel(In in, Out out, int64_t n,
                                                                    const int64_t* partial,
                                                                    int64_t n_tiles) {
  const int64_t tile = int64_t(blockIdx.x) * kScanWarps + (threadIdx.x >> 5);
  if (tile >= n_tiles) return;
  const int64_t base = tile * kScanTile;
  int64_t carry = partial[tile];
  for (int r = 0; r < kScanItems; ++r) {
    int64_t i = base + r * kWarp + lane_id();
    int64_t v = i < n ? in(i) : 0;
    int64_t inc = warp_inclusive_scan(v);
    if (i < n) out(i, carry + inc - v);
    carry += __shfl_sync(0xffffffffu, inc, 31);
  }
}

struct ScanScratch {
  int64_t* partial;  // >= scan_partials_needed(n) elements
  int64_t* total;    // device scalar
};

inline int64_t scan_tiles(int64_t n) { return ceil_div(n, kScanTile); }

// out(i, exclusive_prefix) is called for every i in [0, n); *scratch.total gets the sum.
template <class In, class Out>
void scan_exclusive(In in, Out out, int64_t n, ScanScratch scratch, cudaStream_t stream) {
  const int64_t tiles = scan_tiles(n);
  if (tiles == 0) {
    TJ_CUDA(cudaMemsetAsync(scratch.total, 0, sizeof(int64_t), stream));
    return;
  }
  const unsigned blocks = unsigned(ceil_div(tiles, kScanWarps));
  scan_reduce_kernel<<<blocks, kScanBlock, 0, stream>>>(in, n, scratch.partial, tiles);
  TJ_CHECK_LAUNCH();
  scan_partials_kernel<1024><<<1, 1024, 0, stream>>>(scratch.partial, tiles, scratch.total);
  TJ_CHECK_LAUNCH();
  scan_downsweep_kernel<<<blocks, kScanBlock, 0, stream>>>(in, out, n, scratch.partial, tiles);
  TJ_CHECK_LAUNCH();
}

// Common functors -----------------------------------------------------------
template <class T>
struct LoadAt {
  const T* p;
  __device__ int64_t operator()(int64_t i) const { return int64_t(p[i]); }
};
template <class T>
struct StoreAt {
  T* p;
  __device__ void operator()(int64_t i, int64_t v) const { p[i] = T(v); }
};

}  // namespace tj
