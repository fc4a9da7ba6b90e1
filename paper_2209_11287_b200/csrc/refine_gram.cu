// DMMA refine for big cells at d >= 12 (d_pad >= 12): the brute-force regime of
// config 4 d = 16 / 32 / 64 (64 cells or one cell, every pair a candidate).
//
// Reference: _TileRefiner / distance_tile_v2 (join.py:238-283, kernels.py:184-263):
// D = (-2Q) * C^T + |c|^2 accumulated chunk by chunk, + |q|^2, emit <= eps^2.
//
// There the join is a dense Gram computation, and what limits the per-warp
// kernel (refine_tc.cu: 16 queries per item, each staged candidate used by two
// query groups) is operand traffic, not the DMMA pipe.  This kernel is blocked
// like a GEMM:
//  * a CTA (4 warps) owns a work item of <= 64 queries of one cell x a slice of
//    its concatenated candidate list and sweeps the slice in 64-candidate stages;
//  * the item's queries are staged once, scaled by -2, in shared memory; every
//    stage's candidates arrive through a 2-deep cp.async ring (positions mapped
//    from the cell's runs once per stage); rows are padded to a conflict-free
//    stride and carry |c|^2 as the accumulator's start value;
//  * warp w computes a 32 x 32 block (4 candidate blocks x 4 query groups = 16
//    independent DMMA accumulator chains): per 4-dim chunk 4 A + 4 B fragment
//    loads feed 16 DMMAs, so each staged candidate is used by 64 queries;
//  * epilogue as refine_tc.cu: one branch per stage on the OR of the compare
//    ballots; tiles with a passing value are handled one by one, guard-band
//    values re-decided by the reference direct form, pairs through a per-warp
//    shared-memory buffer;
//  * no short-circuit: at these sizes every chunk is executed (chunks_skipped
//    stays 0, chunks_executed = tiles * NCH in the reference's tiling).
#include "internal.cuh"
#include "refine_common.cuh"

namespace tj {

constexpr int kGramWarps = 4;
constexpr int kGramThreads = kGramWarps * kWarp;
constexpr int kGramQ = 64;   // queries per item
constexpr int kGramC = 64;   // candidates per stage
constexpr int kGramStages = 2;

// CORE = false: DMMA fragments.  CORE = true: the same blocking on CUDA cores --
// the expanded form in DFMA, each thread a 4-query x 8-candidate register block
// (kernel="core_expanded" on big cells: the tensor-core comparison with identical
// algebra, staging and epilogue).
template <int NCH, bool CORE = false>
struct GramShape {
  static constexpr int DP = 4 * NCH;
  // DMMA: conflict-free fragment rows; CORE: rows 8 apart (a thread's candidates)
  // and 16 apart (its queries) hit distinct banks with 16-byte loads
  static constexpr int STRIDE = CORE ? DP + 2 : ((DP % 8 == 0) ? DP + 4 : DP);
  static constexpr int PPR = DP / 2;                           // 16-byte pieces per row
};

template <int NCH, bool CORE = false>
struct GramSmem {
  using S = GramShape<NCH, CORE>;
  double q[kGramQ][S::STRIDE];                   // -2 * query coordinates
  double c[kGramStages][kGramC][S::STRIDE];      // candidate coordinates
  double cn[kGramStages][kGramC];                // |c|^2 (padding rows: kPadNorm)
  double thr[kGramQ], tlo[kGramQ];               // per query: guard band edges (see below)
  uint32_t pos[3][kGramC];                       // cell-ordered positions, by stage % 3
  uint2 hits[kGramWarps][kHitBuf];
};

__device__ __forceinline__ void gram_cp16(void* smem, const void* gmem) {
  const unsigned s = unsigned(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void gram_cp8(void* smem, const void* gmem) {
  const unsigned s = unsigned(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void gram_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void gram_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// m8n8k4 f64 without `volatile`, so the scheduler may interleave the chains.
__device__ __forceinline__ void gram_mma(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

__device__ __noinline__ uint2 gram_recheck(const double* P, int dp, int d, double eps_sq, bool b0,
                                           bool b1, unsigned m0, unsigned m1, uint32_t qa,
                                           uint32_t c, unsigned long long* ctr) {
  bool p0 = (m0 >> lane_id()) & 1u, p1 = (m1 >> lane_id()) & 1u;
  if (b0) p0 = direct_form_le(P, dp, d, qa, c, eps_sq);
  if (b1) p1 = direct_form_le(P, dp, d, qa + 1, c, eps_sq);
  const unsigned nb = __popc(__ballot_sync(0xffffffffu, b0)) + __popc(__ballot_sync(0xffffffffu, b1));
  if (lane_id() == 0) atomicAdd(ctr, (unsigned long long)nb);
  return make_uint2(__ballot_sync(0xffffffffu, p0), __ballot_sync(0xffffffffu, p1));
}

// One 64 x 64 stage on CUDA cores: thread (qg, cg) = (threadIdx.x >> 3, & 7) owns
// queries qg + 16k (k < 4) x candidates cg + 8i (i < 8); two dims per 16-byte load,
// 64 DFMA per 12 loads; acc starts at |c|^2 and adds (-2q).c (the expanded form).
template <class S, class Q, class C>
__device__ __forceinline__ void gram_core_stage(const RefineArgs& a, const Q& sq, const C& sc,
                                                const double* cn, const double* thr_s,
                                                const double* tlo_s, const uint32_t* pos,
                                                uint32_t q0, HitBuffer& hb, uint2* hits,
                                                unsigned (&qc)[4][2],
                                                unsigned long long& rechecks) {
  const int qg = threadIdx.x >> 3, cg = threadIdx.x & 7;
  const unsigned lt = lanemask_lt();
  double acc[4][8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const double c0 = cn[cg + 8 * i];
#pragma unroll
    for (int k = 0; k < 4; ++k) acc[k][i] = c0;
  }
#pragma unroll 2
  for (int j = 0; j < S::DP; j += 2) {
    double2 qv[4], cv[8];
#pragma unroll
    for (int k = 0; k < 4; ++k) qv[k] = *reinterpret_cast<const double2*>(&sq[qg + 16 * k][j]);
#pragma unroll
    for (int i = 0; i < 8; ++i) cv[i] = *reinterpret_cast<const double2*>(&sc[cg + 8 * i][j]);
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        acc[k][i] = __fma_rn(qv[k].x, cv[i].x, acc[k][i]);
        acc[k][i] = __fma_rn(qv[k].y, cv[i].y, acc[k][i]);
      }
  }
  double thr[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) thr[k] = thr_s[qg + 16 * k];
  bool pk[4] = {false, false, false, false};
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int k = 0; k < 4; ++k) pk[k] = pk[k] || (acc[k][i] <= thr[k]);
  if (!__any_sync(0xffffffffu, (pk[0] || pk[1]) || (pk[2] || pk[3]))) return;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const double tlo = tlo_s[qg + 16 * k];
    const uint32_t qpos = q0 + qg + 16 * k;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      bool p = acc[k][i] <= thr[k];
      if (!__any_sync(0xffffffffu, p)) continue;
      const uint32_t cpos = pos[cg + 8 * i];
      const bool band = p && acc[k][i] > tlo;
      if (band) {  // inside the guard band: the reference direct form decides
        ++rechecks;
        p = direct_form_le(a.P, S::DP, a.d, qpos, cpos, a.eps_sq);
      }
      const unsigned m = __ballot_sync(0xffffffffu, p);
      if (!m) continue;
      hb.reserve(__popc(m), hits, a);
      if (p) hits[hb.count + __popc(m & lt)] = make_uint2(qpos, cpos);
      hb.count += __popc(m);
      qc[k][0] += p;
    }
  }
}

template <int NCH, int MINB, bool CORE>
__global__ void __launch_bounds__(kGramThreads, MINB) refine_gram_kernel(RefineArgs a) {
  using S = GramShape<NCH, CORE>;
  constexpr int DP = S::DP, PPR = S::PPR;
  constexpr int kUnroll = NCH >= 8 ? 4 : 2;  // chunks whose fragment loads are hoisted together
  extern __shared__ __align__(16) unsigned char smem_raw[];
  GramSmem<NCH, CORE>& sm = *reinterpret_cast<GramSmem<NCH, CORE>*>(smem_raw);
  const int warp = threadIdx.x >> 5, lane = lane_id();
  const int row = lane >> 2, col = lane & 3;
  const unsigned lt = lanemask_lt();
  const int wc = warp & 1, wq = warp >> 1;  // the warp's 32 x 32 block of the 64 x 64 stage
  uint2* hits = sm.hits[warp];
  HitBuffer hb;
  const double eps_sq = a.eps_sq;
  unsigned long long st_tiles_ref = 0, rechecks = 0;
  __shared__ unsigned long long s_item;

  for (;;) {
    __syncthreads();  // previous item's buffers are free
    if (threadIdx.x == 0) s_item = atomicAdd(&a.ctr->item_next, 1ull);
    __syncthreads();
    const unsigned long long idx = s_item;
    if (idx >= (unsigned long long)a.n_items) break;
    const WorkItem it = a.items[idx];
    const int nq = int(it.nq);
    const int64_t rb = a.cell_runs[it.cell];
    const int nr = int(a.cell_runs[it.cell + 1] - rb);
    const uint32_t s0 = it.s0, s1 = it.s1;
    const int nst = int((s1 - s0 + kGramC - 1) / kGramC);

    // queries, scaled by -2 (exact), rows >= nq zero
    for (int i = threadIdx.x; i < kGramQ * PPR; i += kGramThreads) {
      const int r = i / PPR, pc = i - r * PPR;
      double2 v = make_double2(0.0, 0.0);
      if (r < nq) v = *reinterpret_cast<const double2*>(a.P + size_t(it.q0 + r) * DP + 2 * pc);
      sm.q[r][2 * pc] = -2.0 * v.x;
      sm.q[r][2 * pc + 1] = -2.0 * v.y;
    }
    // guard band edges per query (shared: registers go to the accumulators)
    if (threadIdx.x < kGramQ) {
      const int q = threadIdx.x;
      const bool v = q < nq;
      const double qn = v ? a.NRM[it.q0 + q] : 0.0;
      const double guard = a.guard_rel * (qn + a.max_norm) + 1e-300;
      sm.thr[q] = v ? eps_sq - qn + guard : -INFINITY;
      sm.tlo[q] = v ? eps_sq - qn - guard : INFINITY;
    }
    unsigned qc[4][2] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};  // CORE: qc[k][0], query qg + 16k
    if (threadIdx.x == 0) st_tiles_ref += uint64_t((nq + 7) >> 3) * ((s1 - s0 + 7) >> 3);

    // stage st: candidates s0 + 64 st + r.  Thread r < 64 follows offsets
    // s0 + r, s0 + r + 64, ... through the cell's runs with a cursor (one binary
    // search per item; per stage a compare, a load only when a run ends), and
    // writes slot st % 3 (the epilogue of stage st - 1 may still read its slot).
    int rk = 0;
    uint32_t r_off = 0, r_pos = 0, r_end = 0xffffffffu;
    if (threadIdx.x < kGramC) {
      const uint32_t t0 = s0 + threadIdx.x;
      int lo = 0, hi = nr;
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (a.run_off[rb + mid] <= t0) lo = mid;
        else hi = mid;
      }
      rk = lo;
      r_off = a.run_off[rb + rk];
      r_pos = a.runs[rb + rk].x;
      r_end = rk + 1 < nr ? a.run_off[rb + rk + 1] : 0xffffffffu;
    }
    auto map_positions = [&](int st) {
      if (st < nst && threadIdx.x < kGramC) {
        const uint32_t t = s0 + uint32_t(st) * kGramC + threadIdx.x;
        while (t >= r_end) {
          ++rk;
          r_off = r_end;
          r_pos = a.runs[rb + rk].x;
          r_end = rk + 1 < nr ? a.run_off[rb + rk + 1] : 0xffffffffu;
        }
        sm.pos[st % 3][threadIdx.x] = t < s1 ? r_pos + (t - r_off) : 0xffffffffu;
      }
    };
    // cp.async of stage st into buffer st % 2 (its positions are visible)
    auto issue = [&](int st) {
      if (st < nst) {
        const int buf = st % kGramStages;
        const uint32_t* pos = sm.pos[st % 3];
        for (int i = threadIdx.x; i < kGramC * PPR; i += kGramThreads) {
          const int r = i / PPR, pc = i - r * PPR;
          const uint32_t p = pos[r];
          if (p != 0xffffffffu) gram_cp16(&sm.c[buf][r][2 * pc], a.P + size_t(p) * DP + 2 * pc);
          else *reinterpret_cast<double2*>(&sm.c[buf][r][2 * pc]) = make_double2(0.0, 0.0);
        }
        if (threadIdx.x < kGramC) {
          const uint32_t p = pos[threadIdx.x];
          if (p != 0xffffffffu) gram_cp8(&sm.cn[buf][threadIdx.x], a.NRM + p);
          else sm.cn[buf][threadIdx.x] = kPadNorm;
        }
      }
      gram_commit();
    };
    map_positions(0);
    __syncthreads();
    issue(0);
    // two barriers per stage: (1) stage st+1's positions visible and every warp
    // done with stage st-1 (its buffer is refilled next); (2) stage st landed
#pragma unroll 1
    for (int st = 0; st < nst; ++st) {
      map_positions(st + 1);
      __syncthreads();
      issue(st + 1);
      gram_wait<1>();
      __syncthreads();
      const int buf = st % kGramStages;
      if constexpr (CORE) {
        gram_core_stage<S>(a, sm.q, sm.c[buf], sm.cn[buf], sm.thr, sm.tlo, sm.pos[st % 3], it.q0,
                           hb, hits, qc, rechecks);
      } else {
      double acc[4][4][2];  // [candidate block][query group][value]
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const double cn = sm.cn[buf][32 * wc + 8 * b + row];
#pragma unroll
        for (int g = 0; g < 4; ++g) acc[b][g][0] = acc[b][g][1] = cn;
      }
#pragma unroll(kUnroll)
      for (int j = 0; j < NCH; ++j) {
        double av[4], bv[4];
#pragma unroll
        for (int b = 0; b < 4; ++b) av[b] = sm.c[buf][32 * wc + 8 * b + row][4 * j + col];
#pragma unroll
        for (int g = 0; g < 4; ++g) bv[g] = sm.q[32 * wq + 8 * g + row][4 * j + col];
#pragma unroll
        for (int b = 0; b < 4; ++b)
#pragma unroll
          for (int g = 0; g < 4; ++g) gram_mma(acc[b][g][0], acc[b][g][1], av[b], bv[g]);
      }
      // epilogue: one branch per stage; this lane's queries 32*wq + 8*g + 2*col + jj
      double thr[4][2];
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        const double2 t = *reinterpret_cast<const double2*>(&sm.thr[32 * wq + 8 * g + 2 * col]);
        thr[g][0] = t.x;
        thr[g][1] = t.y;
      }
      // one predicate per lane (DSETP with OR-accumulate, four independent chains
      // so their latencies overlap), one vote per stage
      bool pb[4] = {false, false, false, false};
#pragma unroll
      for (int g = 0; g < 4; ++g)
#pragma unroll
        for (int b = 0; b < 4; ++b)
          pb[b] = pb[b] || (acc[b][g][0] <= thr[g][0]) || (acc[b][g][1] <= thr[g][1]);
      if (__any_sync(0xffffffffu, (pb[0] || pb[1]) || (pb[2] || pb[3]))) {
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const uint32_t cpos = sm.pos[st % 3][32 * wc + 8 * b + row];
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            const bool p0 = acc[b][g][0] <= thr[g][0];
            const bool p1 = acc[b][g][1] <= thr[g][1];
            unsigned m0 = __ballot_sync(0xffffffffu, p0);
            unsigned m1 = __ballot_sync(0xffffffffu, p1);
            if ((m0 | m1) == 0) continue;
            const uint32_t qa = it.q0 + 32 * wq + 8 * g + 2 * col;
            const double2 tl = *reinterpret_cast<const double2*>(&sm.tlo[32 * wq + 8 * g + 2 * col]);
            const bool b0 = p0 && acc[b][g][0] > tl.x;
            const bool b1 = p1 && acc[b][g][1] > tl.y;
            if (__any_sync(0xffffffffu, b0 || b1)) {
              const uint2 m = gram_recheck(a.P, DP, a.d, eps_sq, b0, b1, m0, m1, qa, cpos,
                                           &a.ctr->rechecks);
              m0 = m.x;
              m1 = m.y;
              if ((m0 | m1) == 0) continue;
            }
            const bool h0 = (m0 >> lane) & 1u, h1 = (m1 >> lane) & 1u;
            const int n0 = __popc(m0), n1 = __popc(m1);
            hb.reserve(n0 + n1, hits, a);
            if (h0) hits[hb.count + __popc(m0 & lt)] = make_uint2(qa, cpos);
            if (h1) hits[hb.count + n0 + __popc(m1 & lt)] = make_uint2(qa + 1, cpos);
            hb.count += n0 + n1;
            qc[g][0] += h0;
            qc[g][1] += h1;
          }
        }
      }
      }  // DMMA path
    }
    gram_wait<0>();
    // per-query counts (items of one cell share queries across slices: atomics)
    if constexpr (CORE) {
      // the 8 lanes of a query group (threadIdx.x >> 3) hold its 4 queries' counts
      const int qg = threadIdx.x >> 3;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        unsigned c = qc[k][0];
        c += __shfl_xor_sync(0xffffffffu, c, 1);
        c += __shfl_xor_sync(0xffffffffu, c, 2);
        c += __shfl_xor_sync(0xffffffffu, c, 4);
        const int q = qg + 16 * k;
        if ((threadIdx.x & 7) == 0 && q < nq && c) atomicAdd(&a.qcount[it.q0 + q], c);
      }
    } else {
#pragma unroll
    for (int g = 0; g < 4; ++g)
#pragma unroll
      for (int jj = 0; jj < 2; ++jj) {
        unsigned c = qc[g][jj];
        c += __shfl_xor_sync(0xffffffffu, c, 4);
        c += __shfl_xor_sync(0xffffffffu, c, 8);
        c += __shfl_xor_sync(0xffffffffu, c, 16);
        const int q = 32 * wq + 8 * g + 2 * col + jj;
        if (row == 0 && q < nq && c) atomicAdd(&a.qcount[it.q0 + q], c);
      }
    }
    if (threadIdx.x == 0) atomicAdd(&a.ctr->refined, (unsigned long long)nq * (s1 - s0));
  }
  hb.flush(hits, a);
  if (CORE) st_tiles_ref = 0;  // CUDA-core kernels report no tiles (join.py:328)
  flush_stats(a, st_tiles_ref, st_tiles_ref * NCH, 0, rechecks);
}

// Items of <= 64 queries x candidate slices of ~32k (a multiple of 64).
bool gram_applies(int d_pad, int64_t n, int64_t n_cells) {
  return d_pad >= 12 && n >= int64_t(256) * n_cells;
}

template <int NCH, bool CORE>
static void launch_gram_t(const RefineArgs& a, cudaStream_t s) {
  const size_t smem = sizeof(GramSmem<NCH, CORE>);
  // 3 CTAs (12 warps, <= 168 registers) per SM while the shared memory allows
  constexpr int kMinBlocks = NCH <= 10 ? 3 : 2;
  auto kern = refine_gram_kernel<NCH, kMinBlocks, CORE>;
  TJ_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  int per_sm = 0;
  TJ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kGramThreads, smem));
  per_sm = std::max(per_sm, 1);
  const int64_t grid = std::min<int64_t>(a.n_items, int64_t(kNumSMs) * per_sm);
  kern<<<unsigned(std::max<int64_t>(grid, 1)), kGramThreads, smem, s>>>(a);
  TJ_CHECK_LAUNCH();
}

template <bool CORE>
static void launch_gram_c(const RefineArgs& a, cudaStream_t s) {
  switch (a.nchunks) {
    case 3: return launch_gram_t<3, CORE>(a, s);
    case 4: return launch_gram_t<4, CORE>(a, s);
    case 5: return launch_gram_t<5, CORE>(a, s);
    case 6: return launch_gram_t<6, CORE>(a, s);
    case 7: return launch_gram_t<7, CORE>(a, s);
    case 8: return launch_gram_t<8, CORE>(a, s);
    case 9: return launch_gram_t<9, CORE>(a, s);
    case 10: return launch_gram_t<10, CORE>(a, s);
    case 11: return launch_gram_t<11, CORE>(a, s);
    case 12: return launch_gram_t<12, CORE>(a, s);
    case 13: return launch_gram_t<13, CORE>(a, s);
    case 14: return launch_gram_t<14, CORE>(a, s);
    case 15: return launch_gram_t<15, CORE>(a, s);
    case 16: return launch_gram_t<16, CORE>(a, s);
    default: break;
  }
  fail(TJ_EINVAL, "Gram refine is instantiated for 9 <= d <= 64, got d=" + std::to_string(a.d));
}

void launch_refine_gram(const RefineArgs& a, bool cuda_cores, cudaStream_t s) {
  if (cuda_cores) launch_gram_c<true>(a, s);
  else launch_gram_c<false>(a, s);
}

}  // namespace tj
