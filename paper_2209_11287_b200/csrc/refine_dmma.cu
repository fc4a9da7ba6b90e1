// Tensor-core FP64 refine: the paper's Algorithm 2 (expanded form) on
// warp-level mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4), with exact decisions.
//
// Reference: _TileRefiner (join.py:238-283) driving distance_tile_v2
// (kernels.py:184-263): 8 queries of one cell x 8 candidates of the cell's
// concatenated candidate list per tile, per 4-dim chunk D = (-2Q) * C^T + acc,
// short-circuit when every valid entry already exceeds eps^2, emit <= eps^2.
//
// B200 design:
//  * a persistent grid of 4-warp CTAs pulls work items (cell, up to 8*QG
//    queries, candidate slice).  All four warps hold the same QG query groups
//    as A fragments in registers (-2*q, loaded once per item) and split the
//    8-candidate tiles of each shared-memory stage between them, so every
//    staged candidate feeds QG DMMAs per warp.
//  * a stage holds kStage candidates of the slice: coordinates (row stride
//    padded against bank conflicts), norms and cell-ordered positions, copied
//    from the contiguous candidate runs with coalesced 16-byte loads.
//  * d <= 3: the candidate norm rides in the free 4th K column (A col 3 = 1,
//    B row 3 = |c|^2) and C = |q|^2, so one DMMA yields the squared distance.
//    d >= 4: C = |c|^2 and the comparison uses eps^2 - |q|^2 per query row.
//  * exactness: the hardware accumulation order of DMMA is unpinned (measured:
//    up to 4 ulp of the absolute sum vs exact), so the expanded value decides a
//    pair only outside a guard band of width guard_rel*(|q|^2+max|c|^2); pairs
//    inside it are re-decided with the reference direct form
//    acc = fl(acc + fl(fl(q-c)^2)) (oracle.py:78-81) on CUDA cores.  The
//    emitted set therefore equals the reference direct-form pair set exactly.
//  * short-circuit (join.py:250-253): a group's tile stops after chunk j when
//    every entry's partial distance exceeds eps^2 + guard; partials use the
//    candidate chunk-norm suffix and the query chunk-norm prefix.
//  * emission: per-warp shared-memory pair buffer, flushed with one global
//    atomicAdd per 256 pairs (warp-aggregated append); per-query counts are
//    flushed once per item.
#include "internal.cuh"
#include "refine_common.cuh"

namespace tj {

constexpr int kDmmaWarps = 4;
constexpr int kDmmaThreads = kDmmaWarps * kWarp;

template <int NCH>
struct DmmaShape {
  static constexpr int DP = 4 * NCH;
  static constexpr int STRIDE = (DP % 8 == 0) ? DP + 4 : DP;  // doubles per staged row
  static constexpr int NCHECK = NCH > 1 ? (NCH - 1) / ((NCH + 3) / 4) : 0;  // short-circuit points
  static constexpr int CHECK_EVERY = (NCH + 3) / 4;
  static constexpr int STAGE = NCH <= 4 ? 256 : 128;  // candidates per shared-memory stage
};

template <int NCH, int QG, bool FOLD>
__global__ void __launch_bounds__(kDmmaThreads)
    refine_dmma_kernel(RefineArgs a) {
  using S = DmmaShape<NCH>;
  constexpr int DP = S::DP;
  constexpr int STRIDE = S::STRIDE;
  constexpr int NCHECK = S::NCHECK;
  constexpr int kStage = S::STAGE;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* s_pts = reinterpret_cast<double*>(smem_raw);                 // kStage * STRIDE
  double* s_nrm = s_pts + kStage * STRIDE;                             // kStage (+8 pad)
  double* s_sfx = s_nrm + kStage + 8;                                  // NCHECK * kStage
  uint32_t* s_pos = reinterpret_cast<uint32_t*>(s_sfx + NCHECK * kStage);  // kStage
  uint2* s_hits = reinterpret_cast<uint2*>(s_pos + kStage);            // kDmmaWarps * kHitBuf
  __shared__ WorkItem s_item;
  __shared__ int64_t s_item_idx;

  const int warp = threadIdx.x >> 5;
  const int lane = lane_id();
  const int row = lane >> 2;  // fragment row: query slot in the group
  const int col = lane & 3;   // fragment k / column pair
  const unsigned lt = lanemask_lt();
  uint2* my_hits = s_hits + warp * kHitBuf;
  HitBuffer hb;

  unsigned long long st_tiles = 0, st_exec = 0, st_skip = 0, st_rechecks = 0;

  for (;;) {
    if (threadIdx.x == 0) {
      s_item_idx = int64_t(atomicAdd(&a.ctr->item_next, 1ull));
      if (s_item_idx < a.n_items) s_item = a.items[s_item_idx];
    }
    __syncthreads();
    if (s_item_idx >= a.n_items) break;
    const WorkItem it = s_item;

    // ---- A fragments and per-row thresholds for this item's query groups
    double afr[QG][NCH];
    double thr_hi[QG], thr_lo[QG], guard[QG];
    double cinit[QG];
    double qpre[QG][NCHECK > 0 ? NCHECK : 1];
    uint32_t qpos[QG];
    bool qvalid[QG];
#pragma unroll
    for (int g = 0; g < QG; ++g) {
      const int slot = 8 * g + row;
      qvalid[g] = slot < int(it.nq);
      qpos[g] = it.q0 + slot;
      const double qn = qvalid[g] ? a.NRM[qpos[g]] : 0.0;
      guard[g] = a.guard_rel * (qn + a.max_norm) + 1e-300;
#pragma unroll
      for (int j = 0; j < NCH; ++j) {
        double v = qvalid[g] ? a.P[size_t(qpos[g]) * DP + 4 * j + col] : 0.0;
        afr[g][j] = (FOLD && col == 3) ? (qvalid[g] ? 1.0 : 0.0) : -2.0 * v;
      }
      if (FOLD) {
        cinit[g] = qn;
        thr_hi[g] = qvalid[g] ? a.eps_sq + guard[g] : -INFINITY;
        thr_lo[g] = a.eps_sq - guard[g];
      } else {
        cinit[g] = 0.0;
        thr_hi[g] = qvalid[g] ? (a.eps_sq - qn) + guard[g] : -INFINITY;
        thr_lo[g] = (a.eps_sq - qn) - guard[g];
      }
#pragma unroll
      for (int c = 0; c < NCHECK; ++c) {
        // eps^2 + guard - (query chunk norms up to the check point)
        double pre = 0.0;
        const int upto = (c + 1) * S::CHECK_EVERY;
        for (int j = 0; j < upto; ++j) pre += qvalid[g] ? a.CN[size_t(qpos[g]) * NCH + j] : 0.0;
        qpre[g][c] = qvalid[g] ? a.eps_sq + 2.0 * guard[g] - pre : -INFINITY;
      }
    }
    uint32_t qcnt[QG];
#pragma unroll
    for (int g = 0; g < QG; ++g) qcnt[g] = 0;

    const int64_t rb = a.cell_runs[it.cell], re = a.cell_runs[it.cell + 1];
    for (uint32_t w0 = it.s0; w0 < it.s1; w0 += kStage) {
      const int cnt = int(min(uint32_t(kStage), it.s1 - w0));
      __syncthreads();  // previous stage fully consumed
      stage_candidates<DP, STRIDE, NCHECK, kDmmaWarps, kStage>(a, rb, re, w0, cnt, s_pts, s_nrm, s_sfx,
                                                       s_pos, FOLD, S::CHECK_EVERY);
      __syncthreads();
      const int nblk = (cnt + 7) >> 3;
      for (int b = warp; b < nblk; b += kDmmaWarps) {
        const int cb = 8 * b;
        // B fragments: candidate cb + row, dims 4j + col
        double bfr[NCH];
#pragma unroll
        for (int j = 0; j < NCH; ++j) bfr[j] = s_pts[(cb + row) * STRIDE + 4 * j + col];
        double2 cn2 = make_double2(0.0, 0.0);
        if (!FOLD) cn2 = *reinterpret_cast<const double2*>(s_nrm + cb + 2 * col);
#pragma unroll
        for (int g = 0; g < QG; ++g) {
          if (__all_sync(0xffffffffu, !qvalid[g])) continue;  // group beyond nq
          double d0 = FOLD ? cinit[g] : cn2.x;
          double d1 = FOLD ? cinit[g] : cn2.y;
          int executed = NCH;
          bool pruned = false;
#pragma unroll
          for (int j = 0; j < NCH; ++j) {
            dmma_8x8x4(d0, d1, afr[g][j], bfr[j], d0, d1);
            if constexpr (NCHECK > 0) {
              if (a.short_circuit && (j + 1) % S::CHECK_EVERY == 0 &&
                  (j + 1) / S::CHECK_EVERY <= NCHECK) {
                const int c = (j + 1) / S::CHECK_EVERY - 1;
                const double sf0 = s_sfx[c * kStage + cb + 2 * col];
                const double sf1 = s_sfx[c * kStage + cb + 2 * col + 1];
                // partial distance > eps^2 + guard for every entry of the tile
                const bool far = (d0 - sf0 > qpre[g][c]) && (d1 - sf1 > qpre[g][c]);
                if (__all_sync(0xffffffffu, far)) {
                  executed = j + 1;
                  pruned = true;
                  break;
                }
              }
            }
          }
          st_tiles += 1;
          st_exec += executed;
          st_skip += NCH - executed;
          if (pruned) continue;
          bool p0 = d0 <= thr_hi[g];
          bool p1 = d1 <= thr_hi[g];
          if ((p0 && d0 > thr_lo[g]) || (p1 && d1 > thr_lo[g])) {
            // guard band: decide with the reference direct form
            const uint32_t c0 = s_pos[cb + 2 * col], c1 = s_pos[cb + 2 * col + 1];
            if (p0 && d0 > thr_lo[g]) {
              p0 = direct_form_le(a.P, DP, a.d, qpos[g], c0, a.eps_sq);
              ++st_rechecks;
            }
            if (p1 && d1 > thr_lo[g]) {
              p1 = direct_form_le(a.P, DP, a.d, qpos[g], c1, a.eps_sq);
              ++st_rechecks;
            }
          }
          const unsigned b0 = __ballot_sync(0xffffffffu, p0);
          const unsigned b1 = __ballot_sync(0xffffffffu, p1);
          if ((b0 | b1) == 0) continue;
          const int n0 = __popc(b0), n1 = __popc(b1);
          hb.reserve(n0 + n1, my_hits, a);
          if (p0) my_hits[hb.count + __popc(b0 & lt)] = make_uint2(qpos[g], s_pos[cb + 2 * col]);
          if (p1)
            my_hits[hb.count + n0 + __popc(b1 & lt)] =
                make_uint2(qpos[g], s_pos[cb + 2 * col + 1]);
          hb.count += n0 + n1;
          qcnt[g] += unsigned(p0) + unsigned(p1);
        }
      }
    }
    // per-query pair counts: reduce the 4 lanes of each fragment row
#pragma unroll
    for (int g = 0; g < QG; ++g) {
      uint32_t c = qcnt[g];
      c += __shfl_xor_sync(0xffffffffu, c, 1);
      c += __shfl_xor_sync(0xffffffffu, c, 2);
      if (col == 0 && qvalid[g] && c) atomicAdd(&a.qcount[qpos[g]], c);
    }
    if (threadIdx.x == 0)
      atomicAdd(&a.ctr->refined, (unsigned long long)it.nq * (it.s1 - it.s0));
  }
  hb.flush(my_hits, a);
  if (lane != 0) st_tiles = st_exec = st_skip = 0;  // warp-uniform counters: count once
  flush_stats(a, st_tiles, st_exec, st_skip, st_rechecks);
}

int dmma_queries_per_item(int d, int d_pad) {
  const int nch = d_pad / 4;
  if (d <= 3 || nch <= 2) return 32;
  return nch <= 8 ? 16 : 8;
}

template <int NCH, int QG, bool FOLD>
static void launch_dmma_t(const RefineArgs& a, cudaStream_t s) {
  using S = DmmaShape<NCH>;
  constexpr int kStage = S::STAGE;
  const size_t smem = sizeof(double) * (kStage * S::STRIDE + kStage + 8 + S::NCHECK * kStage) +
                      sizeof(uint32_t) * kStage + sizeof(uint2) * kDmmaWarps * kHitBuf;
  auto kern = refine_dmma_kernel<NCH, QG, FOLD>;
  TJ_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  int per_sm = 0;
  TJ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kDmmaThreads, smem));
  per_sm = std::max(per_sm, 1);
  const int64_t grid = std::min<int64_t>(a.n_items, int64_t(kNumSMs) * per_sm);
  kern<<<unsigned(std::max<int64_t>(grid, 1)), kDmmaThreads, smem, s>>>(a);
  TJ_CHECK_LAUNCH();
}

void launch_refine_dmma(const RefineArgs& a, cudaStream_t s) {
  if (a.d <= 3) return launch_dmma_t<1, 4, true>(a, s);
  switch (a.nchunks) {
    case 1: return launch_dmma_t<1, 4, false>(a, s);
    case 2: return launch_dmma_t<2, 4, false>(a, s);
    case 3: return launch_dmma_t<3, 2, false>(a, s);
    case 4: return launch_dmma_t<4, 2, false>(a, s);
    case 5: return launch_dmma_t<5, 2, false>(a, s);
    case 6: return launch_dmma_t<6, 2, false>(a, s);
    case 7: return launch_dmma_t<7, 2, false>(a, s);
    case 8: return launch_dmma_t<8, 2, false>(a, s);
    case 9: return launch_dmma_t<9, 1, false>(a, s);
    case 10: return launch_dmma_t<10, 1, false>(a, s);
    case 11: return launch_dmma_t<11, 1, false>(a, s);
    case 12: return launch_dmma_t<12, 1, false>(a, s);
    case 13: return launch_dmma_t<13, 1, false>(a, s);
    case 14: return launch_dmma_t<14, 1, false>(a, s);
    case 15: return launch_dmma_t<15, 1, false>(a, s);
    case 16: return launch_dmma_t<16, 1, false>(a, s);
    default: break;
  }
  fail(TJ_EINVAL, "DMMA refine is instantiated for d <= 64, got d=" + std::to_string(a.d));
}

}  // namespace tj
