// Pieces shared by the refine kernels: the reference direct form, the warp
// pair buffer and the statistics flush.
#pragma once
#include "internal.cuh"

namespace tj {

constexpr int kHitBuf = 256;            // pairs per warp buffer (2 KB of shared memory)
constexpr double kPadNorm = 1e300;      // norm of padded candidate slots: never within eps

// Reference direct form (oracle.py:78-81, kernels.py:286-292, join.py:314-318):
// acc = fl(acc + fl(fl(q_i - c_i)^2)) over ascending logical dims, then acc <= eps^2.
// __d*_rn keeps nvcc from contracting into FMA, so the value is bit-identical.
__device__ __forceinline__ bool direct_form_le(const double* __restrict__ P, int dp, int d,
                                               uint32_t q, uint32_t c, double eps_sq) {
  const double* x = P + size_t(q) * dp;
  const double* y = P + size_t(c) * dp;
  double acc = 0.0;
  for (int j = 0; j < d; ++j) {
    const double t = __dsub_rn(x[j], y[j]);
    acc = __dadd_rn(acc, __dmul_rn(t, t));
  }
  return acc <= eps_sq;
}

// Warp-private pair buffer in shared memory; `count` is warp-uniform.
struct HitBuffer {
  int count = 0;
  __device__ __forceinline__ void flush(uint2* buf, const RefineArgs& a) {
    __syncwarp();
    if (count == 0) return;
    unsigned long long base = 0;
    if (lane_id() == 0) base = atomicAdd(&a.ctr->pairs, (unsigned long long)count);
    base = __shfl_sync(0xffffffffu, base, 0);
    for (int i = lane_id(); i < count; i += kWarp) {
      const unsigned long long e = base + i;
      if (e < a.pair_cap) a.pairs[e] = buf[i];
    }
    __syncwarp();
    count = 0;
  }
  __device__ __forceinline__ void reserve(int n, uint2* buf, const RefineArgs& a) {
    if (count + n > kHitBuf) flush(buf, a);
  }
};

__device__ __forceinline__ void flush_stats(const RefineArgs& a, unsigned long long tiles,
                                            unsigned long long exec, unsigned long long skip,
                                            unsigned long long rechecks) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    tiles += __shfl_xor_sync(0xffffffffu, tiles, o);
    exec += __shfl_xor_sync(0xffffffffu, exec, o);
    skip += __shfl_xor_sync(0xffffffffu, skip, o);
    rechecks += __shfl_xor_sync(0xffffffffu, rechecks, o);
  }
  if (lane_id() == 0) {
    if (tiles) atomicAdd(&a.ctr->tiles, tiles);
    if (exec) atomicAdd(&a.ctr->chunks_exec, exec);
    if (skip) atomicAdd(&a.ctr->chunks_skip, skip);
    if (rechecks) atomicAdd(&a.ctr->rechecks, rechecks);
  }
}

}  // namespace tj
