// Pieces shared by the two refine kernels: candidate staging from the
// contiguous runs, the reference direct form, the warp pair buffer and the
// statistics flush.
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

// Copy candidates [w0, w0+cnt) of a cell's concatenated candidate list into
// shared memory.  The list is the runs [rb, re) (position ranges of the
// cell-ordered arrays, each with its offset in the concatenation).  Warps take
// whole runs; lanes move 16-byte pieces, so every run segment is one coalesced
// sweep over contiguous rows.  Slots [cnt, roundup8(cnt)) get zero coordinates
// and a huge norm.  Optional extras:
//   fold:  s_pts[t*STRIDE + 3] = |c|^2 (d <= 3 norm-in-K trick);
//   NCHECK > 0: s_sfx[c*kStageN + t] = sum of chunk norms after check point c.
// DP is the staged row width; the global row stride is a.d_pad (== DP for the
// DMMA kernel, <= DP for the CUDA-core kernel's shared instantiations).
template <int DP, int STRIDE, int NCHECK, int NWARPS, int kStageN = 256>
__device__ __forceinline__ void stage_candidates(const RefineArgs& a, int64_t rb, int64_t re,
                                                 uint32_t w0, int cnt, double* s_pts,
                                                 double* s_nrm, double* s_sfx, uint32_t* s_pos,
                                                 bool fold, int check_every) {
  const int gdp = a.d_pad;
  const int PP = gdp / 2;  // double2 pieces per row
  const int warp = threadIdx.x >> 5;
  const int lane = lane_id();
  const uint32_t w1 = w0 + uint32_t(cnt);
  // first run with off <= w0 (runs are sorted by offset)
  int64_t lo = rb, hi = re;
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) >> 1;
    if (a.run_off[mid] <= w0) lo = mid;
    else hi = mid;
  }
  for (int64_t r = lo + warp; r < re; r += NWARPS) {
    const uint32_t off = a.run_off[r];
    if (off >= w1) break;
    const uint2 run = a.runs[r];
    const uint32_t len = run.y - run.x;
    const uint32_t g0 = max(off, w0), g1 = min(off + len, w1);
    if (g1 <= g0) continue;
    const int t0 = int(g0 - w0);
    const int seg = int(g1 - g0);
    const uint32_t pos0 = run.x + (g0 - off);
    if constexpr (STRIDE % 2 == 0) {
      const double2* src = reinterpret_cast<const double2*>(a.P + size_t(pos0) * gdp);
      for (int i = lane; i < seg * PP; i += kWarp) {
        const int cnd = i / PP, piece = i - cnd * PP;
        *reinterpret_cast<double2*>(s_pts + (t0 + cnd) * STRIDE + 2 * piece) = src[i];
      }
    } else {  // odd row stride (conflict-free per-lane row reads): 8-byte moves
      const double* src = a.P + size_t(pos0) * gdp;
      for (int i = lane; i < seg * gdp; i += kWarp) {
        const int cnd = i / gdp, j = i - cnd * gdp;
        s_pts[(t0 + cnd) * STRIDE + j] = src[i];
      }
    }
    __syncwarp();
    for (int i = lane; i < seg; i += kWarp) {
      const uint32_t p = pos0 + i;
      const double nrm = a.NRM[p];
      s_nrm[t0 + i] = nrm;
      s_pos[t0 + i] = p;
      if (fold) s_pts[(t0 + i) * STRIDE + 3] = nrm;
      if constexpr (NCHECK > 0) {
        const double* cn = a.CN + size_t(p) * (gdp / 4);
        for (int c = 0; c < NCHECK; ++c) {
          double acc = 0.0;  // chunk norms after check point c
          for (int j = (c + 1) * check_every; j < gdp / 4; ++j) acc += cn[j];
          s_sfx[c * kStageN + t0 + i] = acc;
        }
      }
    }
  }
  const int padded = (cnt + 7) & ~7;
  for (int t = cnt + threadIdx.x; t < padded; t += blockDim.x) {
    for (int j = 0; j < DP; ++j) s_pts[t * STRIDE + j] = 0.0;
    if (fold) s_pts[t * STRIDE + 3] = kPadNorm;
    s_nrm[t] = kPadNorm;
    s_pos[t] = 0;
    if constexpr (NCHECK > 0)
      for (int c = 0; c < NCHECK; ++c) s_sfx[c * kStageN + t] = 0.0;
  }
}

}  // namespace tj
