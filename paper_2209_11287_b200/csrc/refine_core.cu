// CUDA-core FP64 refine in the style of GDS-Join: the reference's scalar
// running-sum kernel, bit-exact.
//
// Reference: _ScalarRefiner (join.py:286-349) / scalar_distance_sq
// (kernels.py:274-292): for every query of a cell and every candidate,
// acc = fl(acc + fl(fl(q_i - c_i)^2)) over ascending dims, short-circuiting
// between blocks of min(8, d) dims once acc > eps^2 (exact: partial sums of
// squares are monotone under round-to-nearest).
//
// B200 mapping: one warp per work item (<= QC queries of one cell x a slice of
// its concatenated candidate list).  The item's queries sit in shared memory
// (broadcast reads); each lane owns one candidate of a 32-wide window that
// slides over the flattened candidate runs (coalesced row loads, no padding
// between runs), keeps it in registers (32 dims at a time) and evaluates the
// direct form against every query with __dsub_rn/__dmul_rn/__dadd_rn (no FMA
// contraction, so every value is bit-identical to the reference).  A ballot per
// query feeds the warp pair buffer; per-query counts accumulate per lane.
//
// Three CUDA-core variants share this kernel (template V), so the tensor-core
// formulation is compared against CUDA cores doing the same algebra
// (GDS-Join configuration PAPER.md:291-293):
//  * kExact     the reference order above: 3 FP64 ops per dim (sub, mul, add);
//  * kFma       direct form with fused multiply-add, acc = fma(t, t, acc):
//               2 ops per dim; values within (4d + 8) ulp of eps^2 (relative to
//               eps^2) are re-decided by the exact direct form;
//  * kExpanded  the paper's expanded form on CUDA cores, acc = |c|^2 + |q|^2 +
//               sum fma(-2 q_i, c_i, .): 1 op per dim; values inside the DMMA
//               path's guard band are re-decided exactly.  No short-circuit
//               (partial sums of the expanded form are not monotone).
// All three emit the reference direct-form pair set exactly.
#include "internal.cuh"
#include "refine_common.cuh"

namespace tj {

constexpr int kCoreWarps = 4;
constexpr int kCoreThreads = kCoreWarps * kWarp;

template <int DP>
struct CoreShape {
  static constexpr int DCH = DP < 32 ? DP : 32;  // dims held in registers at once
  static constexpr int QC = DP <= 32 ? 16 : 8;    // queries per work item
  static constexpr bool kMulti = DP > DCH;        // several register chunks of dims
};

enum CoreVariant { kExact = 0, kFma = 1, kExpanded = 2 };

// Decision of one value of a non-exact variant: pass below the band, fail above
// it, and inside it the exact direct form decides.
__device__ __forceinline__ bool core_decide(double acc, double band, const RefineArgs& a,
                                            uint32_t q, uint32_t c, unsigned long long& rechecks) {
  const double e = a.eps_sq;
  if (acc <= e - band) return true;
  if (acc > e + band) return false;
  ++rechecks;
  return direct_form_le(a.P, a.d_pad, a.d, q, c, e);
}

template <int DP, int V>
__global__ void __launch_bounds__(kCoreThreads) refine_core_kernel(RefineArgs a) {
  using S = CoreShape<DP>;
  constexpr int DCH = S::DCH, QC = S::QC;
  __shared__ double s_q[kCoreWarps][QC * DP];
  __shared__ double s_qn[kCoreWarps][QC];  // kExpanded: |q|^2
  __shared__ uint2 s_hits[kCoreWarps][kHitBuf];
  __shared__ uint32_t s_roff[kCoreWarps][33];  // concat offsets of the staged runs (+ end)
  __shared__ uint32_t s_rpos[kCoreWarps][32];  // their first positions
  const int warp = threadIdx.x >> 5;
  const int lane = lane_id();
  const unsigned lt = lanemask_lt();
  double* q_s = s_q[warp];
  uint32_t* roff = s_roff[warp];
  uint32_t* rpos = s_rpos[warp];
  uint2* hits = s_hits[warp];
  HitBuffer hb;
  const int d = a.d;
  const int gdp = a.d_pad;
  const double eps_sq = a.eps_sq;
  // reference unroll = min(8, d) (join.py:301); the expanded form cannot stop early
  const bool sc = V != kExpanded && a.short_circuit && d > 8;
  // kFma: |fma-order sum - reference sum| <= (2d + 4) ulp of the sum near eps^2
  const double fma_band = (4.0 * d + 8.0) * 1.1102230246251565e-16 * eps_sq + 1e-300;
  const double fma_stop = eps_sq + fma_band;  // monotone partial sums: safe early exit
  unsigned long long rechecks = 0;

  for (;;) {
    unsigned long long idx = 0;
    if (lane == 0) idx = atomicAdd(&a.ctr->item_next, 1ull);
    idx = __shfl_sync(0xffffffffu, idx, 0);
    if (idx >= (unsigned long long)a.n_items) break;
    const WorkItem it = a.items[idx];
    const int nq = int(it.nq);
    __syncwarp();
    for (int i = lane; i < nq * gdp; i += kWarp) {
      const int q = i / gdp, j = i - q * gdp;
      const double v = a.P[size_t(it.q0) * gdp + i];
      q_s[q * DP + j] = V == kExpanded ? -2.0 * v : v;
    }
    if (V == kExpanded && lane < nq) s_qn[warp][lane] = a.NRM[it.q0 + lane];
    unsigned mycnt = 0;  // lane q < nq counts query q's pairs

    // runs of the cell, staged 32 at a time; the window [w, w+32) of the slice
    // spans a few consecutive runs
    const int64_t re = a.cell_runs[it.cell + 1];
    int64_t r0;
    {
      int64_t lo = a.cell_runs[it.cell], hi = re;  // first run with offset <= s0
      while (hi - lo > 1) {
        const int64_t mid = (lo + hi) >> 1;
        if (a.run_off[mid] <= it.s0) lo = mid;
        else hi = mid;
      }
      r0 = lo;
    }
    int nrun = 0;
    int kw = 0;  // staged run containing w
    auto stage = [&](int64_t from) {
      __syncwarp();
      const int64_t r = from + lane;
      if (r < re) {
        const uint2 run = a.runs[r];
        const uint32_t o = a.run_off[r];
        rpos[lane] = run.x;
        roff[lane] = o;
        if (r + 1 == re || lane == 31) roff[lane + 1] = o + (run.y - run.x);
      }
      nrun = int(min(int64_t(32), re - from));
      r0 = from;
      kw = 0;
      __syncwarp();
    };
    stage(r0);
#pragma unroll 1
    for (uint32_t w = it.s0; w < it.s1; w += kWarp) {
      const uint32_t wend = min(w + uint32_t(kWarp), it.s1);
      while (kw + 1 < nrun && roff[kw + 1] <= w) ++kw;
      if (roff[nrun] < wend && r0 + nrun < re) stage(r0 + kw);  // window runs past the staged runs
      const uint32_t off = w + uint32_t(lane);
      const bool valid = off < wend;
      uint32_t cpos = 0;
      if (valid) {
        int k = kw;
        while (k + 1 < nrun && roff[k + 1] <= off) ++k;
        cpos = rpos[k] + (off - roff[k]);
      }
      const double* crow = a.P + size_t(cpos) * gdp;
      if constexpr (!S::kMulti) {
        double c[DP];
#pragma unroll
        for (int j = 0; j < DP; ++j) c[j] = (valid && j < gdp) ? __ldg(crow + j) : 0.0;
        const double cn = V == kExpanded && valid ? __ldg(a.NRM + cpos) : 0.0;
#pragma unroll 1
        for (int q = 0; q < nq; ++q) {
          const double* qrow = q_s + q * DP;
          double acc = V == kExpanded ? cn : 0.0;
          bool alive = valid;
#pragma unroll
          for (int j = 0; j < DP; ++j) {
            if (j < d) {
              if constexpr (V == kExpanded) {
                acc = __fma_rn(qrow[j], c[j], acc);
              } else if constexpr (V == kFma) {
                const double t = __dsub_rn(qrow[j], c[j]);
                acc = __fma_rn(t, t, acc);
              } else {
                const double t = __dsub_rn(qrow[j], c[j]);
                acc = __dadd_rn(acc, __dmul_rn(t, t));
              }
              if (sc && ((j + 1) & 7) == 0 && j + 1 < d) {
                alive = alive && acc <= (V == kFma ? fma_stop : eps_sq);
                if (!__any_sync(0xffffffffu, alive)) break;
              }
            }
          }
          bool hit;
          if constexpr (V == kExact) {
            hit = alive && acc <= eps_sq;
          } else if constexpr (V == kFma) {
            hit = alive && core_decide(acc, fma_band, a, it.q0 + q, cpos, rechecks);
          } else {
            const double qn = s_qn[warp][q];
            acc = __dadd_rn(acc, qn);
            hit = alive && core_decide(acc, a.guard_rel * (qn + a.max_norm) + 1e-300, a,
                                       it.q0 + q, cpos, rechecks);
          }
          const unsigned bal = __ballot_sync(0xffffffffu, hit);
          if (bal == 0) continue;
          const int nh = __popc(bal);
          hb.reserve(nh, hits, a);
          if (hit) hits[hb.count + __popc(bal & lt)] = make_uint2(it.q0 + q, cpos);
          hb.count += nh;
          if (lane == q) mycnt += nh;
        }
      } else {
        // several 32-dim register chunks: per-query running sums in registers
        double acc[QC];
        unsigned alive = valid ? ((1u << nq) - 1u) : 0u;
        const double cn = V == kExpanded && valid ? __ldg(a.NRM + cpos) : 0.0;
#pragma unroll
        for (int q = 0; q < QC; ++q) acc[q] = cn;
#pragma unroll 1
        for (int k0 = 0; k0 < d; k0 += DCH) {
          double c[DCH];
#pragma unroll
          for (int j = 0; j < DCH; ++j) c[j] = (valid && k0 + j < gdp) ? __ldg(crow + k0 + j) : 0.0;
#pragma unroll
          for (int q = 0; q < QC; ++q) {
            if (q < nq && ((alive >> q) & 1u)) {
              const double* qrow = q_s + q * DP + k0;
              double s = acc[q];
#pragma unroll
              for (int j = 0; j < DCH; ++j) {
                if (k0 + j < d) {
                  if constexpr (V == kExpanded) {
                    s = __fma_rn(qrow[j], c[j], s);
                  } else if constexpr (V == kFma) {
                    const double t = __dsub_rn(qrow[j], c[j]);
                    s = __fma_rn(t, t, s);
                  } else {
                    const double t = __dsub_rn(qrow[j], c[j]);
                    s = __dadd_rn(s, __dmul_rn(t, t));
                  }
                  if (sc && ((k0 + j + 1) & 7) == 0 && k0 + j + 1 < d &&
                      s > (V == kFma ? fma_stop : eps_sq)) {
                    alive &= ~(1u << q);
                    break;
                  }
                }
              }
              acc[q] = s;
            }
          }
          if (!__any_sync(0xffffffffu, alive != 0)) break;
        }
#pragma unroll
        for (int q = 0; q < QC; ++q) {
          if (q < nq) {
            bool hit = (alive >> q) & 1u;
            if constexpr (V == kExact) {
              hit = hit && acc[q] <= eps_sq;
            } else if constexpr (V == kFma) {
              hit = hit && core_decide(acc[q], fma_band, a, it.q0 + q, cpos, rechecks);
            } else {
              const double qn = s_qn[warp][q];
              hit = hit && core_decide(__dadd_rn(acc[q], qn),
                                       a.guard_rel * (qn + a.max_norm) + 1e-300, a, it.q0 + q,
                                       cpos, rechecks);
            }
            const unsigned bal = __ballot_sync(0xffffffffu, hit);
            if (bal) {
              const int nh = __popc(bal);
              hb.reserve(nh, hits, a);
              if (hit) hits[hb.count + __popc(bal & lt)] = make_uint2(it.q0 + q, cpos);
              hb.count += nh;
              if (lane == q) mycnt += nh;
            }
          }
        }
      }
    }
    if (lane < nq && mycnt) atomicAdd(&a.qcount[it.q0 + lane], mycnt);
    if (lane == 0) atomicAdd(&a.ctr->refined, (unsigned long long)it.nq * (it.s1 - it.s0));
  }
  hb.flush(hits, a);
  flush_stats(a, 0, 0, 0, rechecks);
}

int core_queries_per_item(int /*d*/, int d_pad) { return d_pad <= 32 ? 16 : 8; }  // == QC

template <int DP, int V>
static void launch_core_t(const RefineArgs& a, cudaStream_t s) {
  auto kern = refine_core_kernel<DP, V>;
  int per_sm = 0;
  TJ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kCoreThreads, 0));
  per_sm = std::max(per_sm, 1);
  const int64_t grid = std::min<int64_t>(ceil_div(a.n_items, kCoreWarps), int64_t(kNumSMs) * per_sm);
  kern<<<unsigned(std::max<int64_t>(grid, 1)), kCoreThreads, 0, s>>>(a);
  TJ_CHECK_LAUNCH();
}

template <int V>
static void launch_core_v(const RefineArgs& a, cudaStream_t s) {
  if (a.d_pad <= 4) return launch_core_t<4, V>(a, s);
  if (a.d_pad <= 8) return launch_core_t<8, V>(a, s);
  if (a.d_pad <= 16) return launch_core_t<16, V>(a, s);
  if (a.d_pad <= 32) return launch_core_t<32, V>(a, s);
  if (a.d_pad <= 64) return launch_core_t<64, V>(a, s);
  if (a.d_pad <= 128) return launch_core_t<128, V>(a, s);
  fail(TJ_EINVAL, "CUDA-core refine supports d <= 128, got d=" + std::to_string(a.d));
}

void launch_refine_core(const RefineArgs& a, int variant, cudaStream_t s) {
  switch (variant) {
    case kFma: return launch_core_v<kFma>(a, s);
    case kExpanded: return launch_core_v<kExpanded>(a, s);
    default: return launch_core_v<kExact>(a, s);
  }
}

}  // namespace tj
