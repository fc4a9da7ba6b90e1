// Stable LSD radix sort of (uint32 or uint64 key, uint32 value) pairs.
//
// Replaces the stable np.lexsort of grid.py:83 (cell coordinates, dim 0 most
// significant; ids ascending within a cell because the sort is stable and the
// values start as 0..n-1) and sorts the composite keys of oversized CSR rows in
// the canonical output.  Only the key's significant bits are sorted, in the
// fewest passes of <= 11-bit digits (a 20-bit cell key: two 10-bit passes).
// Cell keys of <= 32 bits are sorted as uint32 (8 bytes per element moved per
// pass instead of 12).
//
// Per pass: (1) per-tile digit histograms, (2) one device-wide exclusive scan
// over the digit-major histogram table, (3) a stable scatter.  In the scatter
// each warp ranks its own 512 consecutive keys of the 4096-key tile (warp
// match_any + warp-private digit counters in shared memory, no block barrier),
// one barrier, then the per-digit prefix over the 8 warps adds the tile's
// global digit offset and every key goes straight to its place from registers:
// two block barriers per tile.
#include "internal.cuh"
#include "scan.cuh"

#include <cstdlib>

namespace tj {

constexpr int kSortThreads = 256;
constexpr int kSortRounds = 16;  // keys per thread
constexpr int kSortTile = kSortThreads * kSortRounds;  // 4096 keys
constexpr int kSortWarps = kSortThreads / kWarp;
constexpr int kSortWarpKeys = kSortRounds * kWarp;     // 512 consecutive keys per warp
constexpr int kMaxDigitBits = 11;
constexpr int kDefaultDigitBits = 10;

template <class K>
__device__ __forceinline__ unsigned digit_of(K key, int shift, unsigned mask) {
  return unsigned(key >> shift) & mask;
}

template <class K>
__global__ void __launch_bounds__(kSortThreads)
    radix_hist_kernel(const K* __restrict__ keys, int64_t n, int shift, int bits,
                      int64_t* __restrict__ hist, int64_t n_tiles) {
  extern __shared__ unsigned s_hist[];  // 1 << bits counters
  const int R = 1 << bits;
  const unsigned mask = unsigned(R - 1);
  for (int i = threadIdx.x; i < R; i += kSortThreads) s_hist[i] = 0;
  __syncthreads();
  const int64_t base = int64_t(blockIdx.x) * kSortTile;
#pragma unroll 4
  for (int r = 0; r < kSortRounds; ++r) {
    const int64_t i = base + r * kSortThreads + threadIdx.x;
    if (i < n) atomicAdd(&s_hist[digit_of(keys[i], shift, mask)], 1u);
  }
  __syncthreads();
  for (int dgt = threadIdx.x; dgt < R; dgt += kSortThreads)
    hist[int64_t(dgt) * n_tiles + blockIdx.x] = s_hist[dgt];
}

// offsets: exclusive scan of the digit-major histogram table (global offset of
// digit d's keys of tile t at offsets[d * n_tiles + t]).
// Shared memory: [kSortWarps][R] warp digit counts (then warp bases inside the
// tile), R digit adjustments (global offset - tile-local start), and the
// tile's keys + values in digit order, so the global writes go out as
// contiguous per-digit runs (consecutive threads, consecutive addresses).
template <class K>
__global__ void __launch_bounds__(kSortThreads)
    radix_scatter_kernel(const K* __restrict__ keys_in, const uint32_t* __restrict__ vals_in,
                         K* __restrict__ keys_out, uint32_t* __restrict__ vals_out, int64_t n,
                         int shift, int bits, const int64_t* __restrict__ offsets,
                         int64_t n_tiles) {
  extern __shared__ __align__(16) unsigned char s_raw[];
  const int R = 1 << bits;
  const unsigned mask = unsigned(R - 1);
  K* s_key = reinterpret_cast<K*>(s_raw);                                   // [kSortTile]
  uint32_t* s_val = reinterpret_cast<uint32_t*>(s_key + kSortTile);         // [kSortTile]
  int64_t* s_adj = reinterpret_cast<int64_t*>(s_val + kSortTile);          // [R]
  unsigned* s_cnt = reinterpret_cast<unsigned*>(s_adj + R);                 // [kSortWarps][R]
  __shared__ unsigned s_wsum[kSortWarps];
  const int warp = threadIdx.x >> 5, lane = lane_id();
  for (int i = threadIdx.x; i < kSortWarps * R; i += kSortThreads) s_cnt[i] = 0;
  __syncthreads();
  unsigned* wc = s_cnt + warp * R;
  const unsigned lt = lanemask_lt();
  const int64_t tile0 = int64_t(blockIdx.x) * kSortTile;
  const int64_t base = tile0 + warp * kSortWarpKeys;
  const int tile_n = n - tile0 < kSortTile ? int(n - tile0) : kSortTile;
  K key[kSortRounds];
  uint32_t val[kSortRounds];
  unsigned rank[kSortRounds];
#pragma unroll
  for (int r = 0; r < kSortRounds; ++r) {
    const int64_t i = base + r * kWarp + lane;
    key[r] = i < n ? keys_in[i] : K(0);
    val[r] = i < n ? (vals_in ? vals_in[i] : uint32_t(i)) : 0u;
  }
#pragma unroll
  for (int r = 0; r < kSortRounds; ++r) {
    const bool valid = base + r * kWarp + lane < n;
    const unsigned dgt = valid ? digit_of(key[r], shift, mask) : 0xffffffffu;
    const unsigned peers = __match_any_sync(0xffffffffu, dgt);
    const unsigned before = valid ? wc[dgt] : 0u;
    __syncwarp();
    if (valid && (peers & lt) == 0u) wc[dgt] = before + __popc(peers);
    __syncwarp();
    rank[r] = before + __popc(peers & lt);
  }
  __syncthreads();
  // per digit: counts of the earlier warps (bases inside the digit), the digit's
  // tile total; thread t owns the R / 256 consecutive digits [t * per, (t+1) * per)
  const int per = R >= kSortThreads ? R / kSortThreads : 1;
  const int d0 = threadIdx.x * per;
  unsigned tsum = 0;
  if (d0 < R) {
    for (int d = d0; d < d0 + per; ++d) {
      unsigned run = 0;
#pragma unroll
      for (int w = 0; w < kSortWarps; ++w) {
        const unsigned c = s_cnt[w * R + d];
        s_cnt[w * R + d] = run;
        run += c;
      }
      s_adj[d] = run;  // digit total for now
      tsum += run;
    }
  }
  // exclusive scan of the per-thread digit totals -> tile-local digit starts
  unsigned inc = tsum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned t = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += t;
  }
  if (lane == 31) s_wsum[warp] = inc;
  __syncthreads();
  unsigned wbase = 0;
#pragma unroll
  for (int w = 0; w < kSortWarps; ++w) wbase += w < warp ? s_wsum[w] : 0u;
  if (d0 < R) {
    unsigned start = wbase + inc - tsum;
    for (int d = d0; d < d0 + per; ++d) {
      const unsigned tot = unsigned(s_adj[d]);
      // warp bases become tile-local positions
#pragma unroll
      for (int w = 0; w < kSortWarps; ++w) s_cnt[w * R + d] += start;
      s_adj[d] = offsets[int64_t(d) * n_tiles + blockIdx.x] - int64_t(start);
      start += tot;
    }
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kSortRounds; ++r) {
    if (base + r * kWarp + lane < n) {
      const unsigned pos = wc[digit_of(key[r], shift, mask)] + rank[r];
      s_key[pos] = key[r];
      s_val[pos] = val[r];
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < tile_n; i += kSortThreads) {
    const K k = s_key[i];
    const int64_t dst = s_adj[digit_of(k, shift, mask)] + i;
    keys_out[dst] = k;
    vals_out[dst] = s_val[i];
  }
}

template <class K>
static size_t scatter_smem(int bits) {
  return (sizeof(K) + sizeof(uint32_t)) * kSortTile +
         (sizeof(int64_t) + sizeof(unsigned) * kSortWarps) * (size_t(1) << bits);
}

int64_t radix_sort_scratch_elems(int64_t n) {
  const int64_t tiles = ceil_div(n, kSortTile);
  return tiles << kMaxDigitBits;
}

__global__ void iota_kernel(uint32_t* v, int64_t n) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    v[i] = uint32_t(i);
}

template <class K>
static int radix_sort_t(K* k0, uint32_t* v0, K* k1, uint32_t* v1, int64_t n, int key_bits,
                        bool identity_values, int64_t* hist, ScanScratch scan, cudaStream_t stream) {
  // digit width: wider digits mean fewer passes but per-tile work (counters,
  // digit prefix, histogram rows) grows with the radix (TJ_SORT_DIGIT_BITS: A/B)
  static const int max_bits = [] {
    const char* e = std::getenv("TJ_SORT_DIGIT_BITS");
    const int v = e ? std::atoi(e) : kDefaultDigitBits;
    return v < 4 ? 4 : (v > kMaxDigitBits ? kMaxDigitBits : v);
  }();
  const int passes = key_bits <= 0 ? 0 : (key_bits + max_bits - 1) / max_bits;
  if (n <= 1 || passes == 0) {
    if (n > 0 && identity_values) {
      iota_kernel<<<unsigned(std::min<int64_t>(ceil_div(n, 256), 4096)), 256, 0, stream>>>(v0, n);
      TJ_CHECK_LAUNCH();
    }
    return 0;
  }
  // up to 8 x 2048 counters (64 KB) in the scatter (per device: set on every call)
  TJ_CUDA(cudaFuncSetAttribute(radix_scatter_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               int(scatter_smem<K>(kMaxDigitBits))));
  const int64_t tiles = ceil_div(n, kSortTile);
  const uint32_t* vin = identity_values ? nullptr : v0;
  K* kin = k0;
  K* kout = k1;
  uint32_t* vout = v1;
  int cur = 0;
  int shift = 0;
  for (int p = 0; p < passes; ++p) {
    // equal digit widths, <= 11 bits each
    const int bits = (key_bits - shift + (passes - p) - 1) / (passes - p);
    const size_t hsm = sizeof(unsigned) << bits;
    radix_hist_kernel<K><<<unsigned(tiles), kSortThreads, hsm, stream>>>(kin, n, shift, bits,
                                                                        hist, tiles);
    TJ_CHECK_LAUNCH();
    scan_exclusive(LoadAt<int64_t>{hist}, StoreAt<int64_t>{hist}, tiles << bits, scan, stream);
    radix_scatter_kernel<K><<<unsigned(tiles), kSortThreads, scatter_smem<K>(bits), stream>>>(
        kin, vin, kout, vout, n, shift, bits, hist, tiles);
    TJ_CHECK_LAUNCH();
    shift += bits;
    // next pass reads what we just wrote
    cur ^= 1;
    kin = cur ? k1 : k0;
    kout = cur ? k0 : k1;
    vin = cur ? v1 : v0;
    vout = cur ? v0 : v1;
  }
  return cur;
}

// Sorts by the low key_bits bits.  Returns 0 if the result is in (k0,v0), 1 if in (k1,v1).
// identity_values: v0's contents are ignored and the values start as 0..n-1.
int radix_sort_pairs(uint64_t* k0, uint32_t* v0, uint64_t* k1, uint32_t* v1, int64_t n,
                     int key_bits, bool identity_values, int64_t* hist, ScanScratch scan,
                     cudaStream_t stream) {
  return radix_sort_t<uint64_t>(k0, v0, k1, v1, n, key_bits, identity_values, hist, scan, stream);
}
int radix_sort_pairs32(uint32_t* k0, uint32_t* v0, uint32_t* k1, uint32_t* v1, int64_t n,
                       int key_bits, bool identity_values, int64_t* hist, ScanScratch scan,
                       cudaStream_t stream) {
  return radix_sort_t<uint32_t>(k0, v0, k1, v1, n, key_bits, identity_values, hist, scan, stream);
}

}  // namespace tj
