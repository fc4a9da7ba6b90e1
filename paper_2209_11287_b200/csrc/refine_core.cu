// CUDA-core FP64 refine in the style of GDS-Join: the reference's scalar
// running-sum kernel, bit-exact.
//
// Reference: _ScalarRefiner (join.py:286-349) / scalar_distance_sq
// (kernels.py:274-292): for every query of a cell and every candidate,
// acc = fl(acc + fl(fl(q_i - c_i)^2)) over ascending dims, short-circuiting
// between blocks of min(8, d) dims once acc > eps^2 (exact: partial sums of
// squares are monotone under round-to-nearest).
//
// B200 design: the same persistent work-item loop and shared-memory candidate
// stages as the DMMA kernel; here each lane owns one staged candidate (kept in
// registers, up to 32 dims at a time) and the item's queries are broadcast from
// shared memory, so each warp evaluates 32 pairs per query step with
// sub/mul/add as __dsub_rn/__dmul_rn/__dadd_rn (no FMA contraction), then a
// ballot feeds the warp pair buffer.
#include "internal.cuh"
#include "refine_common.cuh"

namespace tj {

constexpr int kCoreWarps = 4;
constexpr int kCoreThreads = kCoreWarps * kWarp;

template <int DP>
struct CoreShape {
  static constexpr int STRIDE = DP + 1;        // odd: conflict-free per-lane rows
  static constexpr int DCH = DP < 32 ? DP : 32;  // dims held in registers at once
  static constexpr int QC = DP <= 32 ? 32 : 16;  // queries per work item
  static constexpr int STAGE = DP <= 16 ? 256 : 128;
};

template <int DP>
__global__ void __launch_bounds__(kCoreThreads) refine_core_kernel(RefineArgs a) {
  using S = CoreShape<DP>;
  constexpr int STRIDE = S::STRIDE;
  constexpr int DCH = S::DCH;
  constexpr int QC = S::QC;
  constexpr int kCoreStage = S::STAGE;
  constexpr bool kMulti = DP > DCH;  // dims processed in several register chunks
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* s_pts = reinterpret_cast<double*>(smem_raw);        // kCoreStage * STRIDE
  double* s_nrm = s_pts + kCoreStage * STRIDE;                // kCoreStage (+8)
  uint32_t* s_pos = reinterpret_cast<uint32_t*>(s_nrm + kCoreStage + 8);
  double* s_q = reinterpret_cast<double*>(s_pos + kCoreStage);  // QC * DP
  uint2* s_hits = reinterpret_cast<uint2*>(s_q + QC * DP);      // kCoreWarps * kHitBuf
  __shared__ uint32_t s_qc[QC];
  __shared__ WorkItem s_item;
  __shared__ int64_t s_item_idx;

  const int warp = threadIdx.x >> 5;
  const int lane = lane_id();
  const unsigned lt = lanemask_lt();
  uint2* my_hits = s_hits + warp * kHitBuf;
  HitBuffer hb;
  const int d = a.d;
  const double eps_sq = a.eps_sq;
  const bool sc = a.short_circuit && d > 8;
  for (int q = threadIdx.x; q < QC; q += kCoreThreads) s_qc[q] = 0;

  for (;;) {
    if (threadIdx.x == 0) {
      s_item_idx = int64_t(atomicAdd(&a.ctr->item_next, 1ull));
      if (s_item_idx < a.n_items) s_item = a.items[s_item_idx];
    }
    __syncthreads();
    if (s_item_idx >= a.n_items) break;
    const WorkItem it = s_item;
    const int nq = int(it.nq);
    const int gdp = a.d_pad;
    for (int i = threadIdx.x; i < nq * gdp; i += kCoreThreads) {
      const int q = i / gdp, j = i - q * gdp;
      s_q[q * DP + j] = a.P[size_t(it.q0) * gdp + i];
    }

    const int64_t rb = a.cell_runs[it.cell], re = a.cell_runs[it.cell + 1];
    for (uint32_t w0 = it.s0; w0 < it.s1; w0 += kCoreStage) {
      const int cnt = int(min(uint32_t(kCoreStage), it.s1 - w0));
      __syncthreads();
      stage_candidates<DP, STRIDE, 0, kCoreWarps, kCoreStage>(a, rb, re, w0, cnt, s_pts, s_nrm,
                                                               nullptr, s_pos, false, 1);
      __syncthreads();
      for (int base = warp * kWarp; base < cnt; base += kCoreThreads) {
        const int t = base + lane;
        const bool valid = t < cnt;
        const double* crow = s_pts + (valid ? t : 0) * STRIDE;
        const uint32_t cpos = valid ? s_pos[t] : 0;
        if constexpr (!kMulti) {
          double c[DP];
#pragma unroll
          for (int j = 0; j < DP; ++j) c[j] = crow[j];
          for (int q = 0; q < nq; ++q) {
            const double* qrow = s_q + q * DP;
            double acc = 0.0;
            bool alive = valid;
#pragma unroll
            for (int j = 0; j < DP; ++j) {
              if (j < d) {
                const double tq = __dsub_rn(qrow[j], c[j]);
                acc = __dadd_rn(acc, __dmul_rn(tq, tq));
                if (sc && ((j + 1) & 7) == 0 && j + 1 < d && acc > eps_sq) {
                  alive = false;
                  break;
                }
              }
            }
            const bool hit = alive && acc <= eps_sq;
            const unsigned bal = __ballot_sync(0xffffffffu, hit);
            if (bal == 0) continue;
            const int nh = __popc(bal);
            hb.reserve(nh, my_hits, a);
            if (hit) my_hits[hb.count + __popc(bal & lt)] = make_uint2(it.q0 + q, cpos);
            hb.count += nh;
            if (lane == 0) atomicAdd(&s_qc[q], unsigned(nh));
          }
        } else {
          // several 32-dim register chunks: per-query running sums in registers
          double acc[QC];
          unsigned alive = valid ? (nq >= 32 ? 0xffffffffu : ((1u << nq) - 1u)) : 0u;
#pragma unroll
          for (int q = 0; q < QC; ++q) acc[q] = 0.0;
          for (int k0 = 0; k0 < d; k0 += DCH) {
            double c[DCH];
#pragma unroll
            for (int j = 0; j < DCH; ++j) c[j] = (k0 + j < DP) ? crow[k0 + j] : 0.0;
#pragma unroll
            for (int q = 0; q < QC; ++q) {
              if (q < nq && ((alive >> q) & 1u)) {
                const double* qrow = s_q + q * DP + k0;
                double s = acc[q];
#pragma unroll
                for (int j = 0; j < DCH; ++j) {
                  if (k0 + j < d) {
                    const double tq = __dsub_rn(qrow[j], c[j]);
                    s = __dadd_rn(s, __dmul_rn(tq, tq));
                    if (sc && ((k0 + j + 1) & 7) == 0 && k0 + j + 1 < d && s > eps_sq) {
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
              const bool hit = ((alive >> q) & 1u) && acc[q] <= eps_sq;
              const unsigned bal = __ballot_sync(0xffffffffu, hit);
              if (bal) {
                const int nh = __popc(bal);
                hb.reserve(nh, my_hits, a);
                if (hit) my_hits[hb.count + __popc(bal & lt)] = make_uint2(it.q0 + q, cpos);
                hb.count += nh;
                if (lane == 0) atomicAdd(&s_qc[q], unsigned(nh));
              }
            }
          }
        }
      }
    }
    __syncthreads();
    for (int q = threadIdx.x; q < nq; q += kCoreThreads) {
      const uint32_t c = s_qc[q];
      if (c) atomicAdd(&a.qcount[it.q0 + q], c);
      s_qc[q] = 0;
    }
    if (threadIdx.x == 0)
      atomicAdd(&a.ctr->refined, (unsigned long long)it.nq * (it.s1 - it.s0));
  }
  hb.flush(my_hits, a);
}

int core_queries_per_item(int /*d*/, int d_pad) { return d_pad <= 32 ? 32 : 16; }  // == CoreShape::QC

template <int DP>
static void launch_core_t(const RefineArgs& a, cudaStream_t s) {
  using S = CoreShape<DP>;
  constexpr int kCoreStage = S::STAGE;
  const size_t smem = sizeof(double) * (kCoreStage * S::STRIDE + kCoreStage + 8) +
                      sizeof(uint32_t) * kCoreStage + sizeof(double) * S::QC * DP +
                      sizeof(uint2) * kCoreWarps * kHitBuf;
  auto kern = refine_core_kernel<DP>;
  TJ_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  int per_sm = 0;
  TJ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kCoreThreads, smem));
  per_sm = std::max(per_sm, 1);
  const int64_t grid = std::min<int64_t>(a.n_items, int64_t(kNumSMs) * per_sm);
  kern<<<unsigned(std::max<int64_t>(grid, 1)), kCoreThreads, smem, s>>>(a);
  TJ_CHECK_LAUNCH();
}

void launch_refine_core(const RefineArgs& a, cudaStream_t s) {
  if (a.d_pad <= 4) return launch_core_t<4>(a, s);
  if (a.d_pad <= 8) return launch_core_t<8>(a, s);
  if (a.d_pad <= 16) return launch_core_t<16>(a, s);
  if (a.d_pad <= 32) return launch_core_t<32>(a, s);
  if (a.d_pad <= 64) return launch_core_t<64>(a, s);
  if (a.d_pad <= 128) return launch_core_t<128>(a, s);
  fail(TJ_EINVAL, "CUDA-core refine supports d <= 128, got d=" + std::to_string(a.d));
}

}  // namespace tj
