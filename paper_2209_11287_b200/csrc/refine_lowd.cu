// DMMA refine for d <= 4 (one 4-dim chunk): the hot kernel of configs 1, 2,
// 4(d<=4) and 5.
//
// Same math as refine_dmma.cu (paper Alg. 2, exact decisions through a guard
// band), mapped for the fewest instructions per m8n8k4 tile:
//  * one warp per work item (<= 16 queries of one cell), no CTA barriers;
//  * transposed roles: candidates are the A operand (rows) and the queries the
//    B operand (columns), so the C operand is the candidates' norms and each
//    lane loads exactly the norm of the candidate whose coordinate it loads;
//    query fragments and thresholds stay in registers for the whole item;
//  * d <= 3: |c|^2 sits in the padding coordinate of P (A col 3), B row 3 = 1,
//    C = |q|^2: D is the squared distance with no norm load at all;
//  * the item's candidate runs are flattened into a shared-memory list of
//    8-candidate blocks; blocks are staged four at a time into a per-warp
//    shared-memory ring with cp.async, kLowStages-1 stages ahead;
//  * hit test: one DSETP per value against the guard-inflated threshold; in a
//    tile with hits the guard band is screened with integer ops on the high
//    word of the double and, when a band bit is set (rare), re-decided out of
//    line by the reference direct form;
//  * output: the tile's two ballots form one 64-bit hit mask, stored densely
//    (one 8-byte store per tile, no atomics, no ranking); per-query counts
//    accumulate in registers.  finalize.cu expands the masks into sorted rows.
// Keep the hot loop small: the whole kernel must stay within the instruction
// cache (rare paths are __noinline__).
// JoinStats tiles are the reference formula ceil(nq/8) * ceil(|cand|/8) per item
// (join.py:257-261); chunks = tiles since d <= 4 has one chunk (kernels.py:250).
#include "internal.cuh"
#include "refine_common.cuh"

namespace tj {

constexpr int kLowWarps = 4;
constexpr int kLowThreads = kLowWarps * kWarp;
constexpr int kLowStages = 4;  // cp.async ring depth per warp (stages of 4 blocks)
constexpr int kBlkList = 256;  // block descriptors per list chunk

__device__ __forceinline__ unsigned hi_word(double v) { return unsigned(__double2hiint(v)); }

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = unsigned(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned s = unsigned(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

struct LowStage {
  double pts[32][4];  // candidate coordinates (d <= 3: slot 3 holds |c|^2)
  double nrm[32];     // |c|^2 (C operand, d == 4)
  uint32_t pos[4];    // position of each block's first candidate
};

struct QuerySide {
  double bq[2];                 // B fragments per group
  double cq[2][2];              // FOLD: C operand |q|^2 per column
  double thr[2][2];             // pass iff D <= thr (guard-inflated)
  unsigned h1[2][2], hw[2][2];  // guard band as a high-word range [h1, h1+hw]
};

// Guard-band pairs of one tile, re-decided by the reference direct form.
// Returns the corrected (m0, m1); out of line because it is rare.
__device__ __noinline__ uint2 recheck_tile(const double* P, int d, double eps_sq, bool b0,
                                           bool b1, bool p0, bool p1, uint32_t qa, uint32_t c,
                                           unsigned long long* ctr) {
  if (b0) p0 = direct_form_le(P, 4, d, qa, c, eps_sq);
  if (b1) p1 = direct_form_le(P, 4, d, qa + 1, c, eps_sq);
  const unsigned nb = __popc(__ballot_sync(0xffffffffu, b0)) + __popc(__ballot_sync(0xffffffffu, b1));
  if (lane_id() == 0) atomicAdd(ctr, (unsigned long long)nb);
  return make_uint2(__ballot_sync(0xffffffffu, p0), __ballot_sync(0xffffffffu, p1));
}

template <bool FOLD>
__device__ __forceinline__ void lowd_tile(const RefineArgs& a, const QuerySide& qs,
                                          unsigned (&qc)[2][2], int ng, double av, double cn,
                                          uint32_t p, uint32_t q0, unsigned long long* mrow,
                                          int ngc) {
  const int lane = lane_id();
#pragma unroll
  for (int g = 0; g < 2; ++g) {
    if (g >= ng) break;
    double d0, d1;
    dmma_8x8x4(d0, d1, av, qs.bq[g], FOLD ? qs.cq[g][0] : cn, FOLD ? qs.cq[g][1] : cn);
    bool p0 = d0 <= qs.thr[g][0];
    bool p1 = d1 <= qs.thr[g][1];
    unsigned m0 = __ballot_sync(0xffffffffu, p0);
    unsigned m1 = __ballot_sync(0xffffffffu, p1);
    if (m0 | m1) {
      const bool b0 = p0 && (hi_word(d0) - qs.h1[g][0]) <= qs.hw[g][0];
      const bool b1 = p1 && (hi_word(d1) - qs.h1[g][1]) <= qs.hw[g][1];
      if (__any_sync(0xffffffffu, b0 || b1)) {
        const uint2 m = recheck_tile(a.P, a.d, a.eps_sq, b0, b1, p0, p1,
                                     q0 + 8 * g + 2 * (lane & 3), p + (lane >> 2),
                                     &a.ctr->rechecks);
        m0 = m.x;
        m1 = m.y;
        p0 = (m0 >> lane) & 1u;
        p1 = (m1 >> lane) & 1u;
      }
      qc[g][0] += p0;
      qc[g][1] += p1;
    }
    if (lane == 0) mrow[g] = (static_cast<unsigned long long>(m1) << 32) | m0;
  }
  (void)ngc;
}

template <bool FOLD>
__device__ __forceinline__ void lowd_item(const RefineArgs& a, const QuerySide& qs,
                                          unsigned (&qc)[2][2], int ng, uint2* blk,
                                          LowStage* ring, uint32_t q0, int64_t rb, int64_t re,
                                          unsigned long long* mbase, int ngc) {
  const int lane = lane_id();
  const int row = lane >> 2, col = lane & 3;
  constexpr int R = kLowStages;
  // lane r holds run r (<= 27 runs for k <= 4) and its first block's flat index
  const int nr = int(re - rb);
  uint2 myrun = make_uint2(0u, 0u);
  if (lane < nr) myrun = a.runs[rb + lane];
  const int mynblk = int(myrun.y - myrun.x + 7) >> 3;
  int incl = mynblk;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  const int total = __shfl_sync(0xffffffffu, incl, 31);
  const int myfirst = incl - mynblk;
  const int cblk = lane >> 3, crow = lane & 7;  // the candidate row this lane stages
#pragma unroll 1
  for (int c0 = 0; c0 < total; c0 += kBlkList) {
    const int cn = min(kBlkList, total - c0);
    // descriptors of blocks [c0, c0+cn): (position, valid rows)
    __syncwarp();
    {
      const int lo = max(myfirst, c0), hi = min(myfirst + mynblk, c0 + cn);
      for (int b = lo; b < hi; ++b) {
        const uint32_t pos = myrun.x + 8u * uint32_t(b - myfirst);
        blk[b - c0] = make_uint2(pos, min(8u, myrun.y - pos));
      }
    }
    __syncwarp();
    const int nst = (cn + 3) >> 2;
    auto issue = [&](int st, LowStage* s) {
      const int b = 4 * st + cblk;
      uint2 bd = make_uint2(0u, 0u);
      if (b < cn) bd = blk[b];
      const uint32_t pidx = bd.x + uint32_t(crow);
      if (uint32_t(crow) < bd.y) {
        cp_async16(&s->pts[lane][0], a.P + size_t(pidx) * 4);
        cp_async16(&s->pts[lane][2], a.P + size_t(pidx) * 4 + 2);
        if (!FOLD) cp_async8(&s->nrm[lane], a.NRM + pidx);
      } else {  // padding row: never within eps
        *reinterpret_cast<double2*>(&s->pts[lane][0]) = make_double2(0.0, 0.0);
        *reinterpret_cast<double2*>(&s->pts[lane][2]) = make_double2(0.0, FOLD ? kPadNorm : 0.0);
        s->nrm[lane] = kPadNorm;
      }
      if (crow == 0) s->pos[cblk] = bd.x;
      cp_async_commit();
    };
#pragma unroll
    for (int k = 0; k < R - 1; ++k) {
      if (k < nst) issue(k, ring + k);
      else cp_async_commit();
    }
#pragma unroll 1
    for (int st = 0; st < nst; ++st) {
      cp_async_wait<R - 2>();
      __syncwarp();
      const LowStage* s = ring + (st % R);
      const int nb = min(4, cn - 4 * st);
#pragma unroll 1
      for (int k = 0; k < nb; ++k) {
        const double av = s->pts[8 * k + row][col];
        const double cv = FOLD ? 0.0 : s->nrm[8 * k + row];
        lowd_tile<FOLD>(a, qs, qc, ng, av, cv, s->pos[k], q0,
                        mbase + size_t(c0 + 4 * st + k) * ngc, ngc);
      }
      __syncwarp();
      if (st + R - 1 < nst) issue(st + R - 1, ring + ((st + R - 1) % R));
      else cp_async_commit();
    }
    cp_async_wait<0>();
  }
}

template <bool FOLD>
__global__ void __launch_bounds__(kLowThreads, 5) refine_lowd_kernel(RefineArgs a) {
  __shared__ uint2 s_blk[kLowWarps][kBlkList];
  __shared__ LowStage s_ring[kLowWarps][kLowStages];
  const int warp = threadIdx.x >> 5;
  const int lane = lane_id();
  const int row = lane >> 2;
  const int col = lane & 3;
  unsigned long long st_tiles = 0;
  const double eps_sq = a.eps_sq;

  for (;;) {
    unsigned long long idx = 0;
    if (lane == 0) idx = atomicAdd(&a.ctr->item_next, 1ull);
    idx = __shfl_sync(0xffffffffu, idx, 0);
    if (idx >= (unsigned long long)a.n_items) break;
    const WorkItem it = a.items[idx];
    const int nq = int(it.nq);
    const int ng = (nq + 7) >> 3;
    QuerySide qs;
#pragma unroll
    for (int g = 0; g < 2; ++g) {
      const int qb = 8 * g + row;
      const bool vb = qb < nq;
      const double x = vb ? a.P[size_t(it.q0 + qb) * 4 + col] : 0.0;
      qs.bq[g] = (FOLD && col == 3) ? (vb ? 1.0 : 0.0) : -2.0 * x;
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int q = 8 * g + 2 * col + j;
        const bool v = q < nq;
        const double qn = v ? a.NRM[it.q0 + q] : 0.0;
        const double guard = a.guard_rel * (qn + a.max_norm) + 1e-300;
        const double center = FOLD ? eps_sq : eps_sq - qn;
        const double hi = center + guard, lo = center - guard;
        qs.cq[g][j] = qn;
        qs.thr[g][j] = v ? hi : -INFINITY;
        if (!v) {
          qs.h1[g][j] = 0u;
          qs.hw[g][j] = 0u;
        } else if ((hi < 0.0) == (lo < 0.0) && lo != 0.0 && hi != 0.0) {
          const unsigned a1 = hi_word(hi), a2 = hi_word(lo);
          qs.h1[g][j] = min(a1, a2);
          qs.hw[g][j] = max(a1, a2) - min(a1, a2);
        } else {  // band straddles zero: decide every passing pair exactly
          qs.h1[g][j] = 0u;
          qs.hw[g][j] = 0xffffffffu;
        }
      }
    }
    // reference tiling of the concatenated list (join.py:257-261)
    st_tiles += uint64_t(ng) * ((it.s1 - it.s0 + 7) >> 3);
    const int64_t rb = a.cell_runs[it.cell], re = a.cell_runs[it.cell + 1];
    // this item's masks: cell base + block * groups_in_cell + (first group of the item)
    const int64_t cs = a.cell_start[it.cell];
    const int ngc = int((a.cell_start[it.cell + 1] - cs + 7) >> 3);
    unsigned long long* mbase =
        a.masks + a.cell_mbase[it.cell - a.cell_base] + (int64_t(it.q0) - cs) / 8;
    unsigned qc[2][2] = {{0u, 0u}, {0u, 0u}};
    lowd_item<FOLD>(a, qs, qc, ng, s_blk[warp], s_ring[warp], it.q0, rb, re, mbase, ngc);
    // per-query counts: sum the 8 fragment rows holding the same columns
    unsigned item_hits = 0;
#pragma unroll
    for (int g = 0; g < 2; ++g) {
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        unsigned c = qc[g][j];
        c += __shfl_xor_sync(0xffffffffu, c, 4);
        c += __shfl_xor_sync(0xffffffffu, c, 8);
        c += __shfl_xor_sync(0xffffffffu, c, 16);
        const int q = 8 * g + 2 * col + j;
        if (row == 0 && q < nq) {
          a.qcount[it.q0 + q] = c;  // each query lives in one item
          item_hits += c;
        }
      }
    }
    item_hits = __reduce_add_sync(0xffffffffu, item_hits);
    if (lane == 0) {
      atomicAdd(&a.ctr->refined, (unsigned long long)nq * (it.s1 - it.s0));
      atomicAdd(&a.ctr->hits, (unsigned long long)item_hits);
    }
  }
  if (lane != 0) st_tiles = 0;
  flush_stats(a, st_tiles, st_tiles, 0, 0);
}

int lowd_queries_per_item() { return 16; }

template <bool FOLD>
static void launch_lowd_t(const RefineArgs& a, cudaStream_t s) {
  auto kern = refine_lowd_kernel<FOLD>;
  int per_sm = 0;
  TJ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kLowThreads, 0));
  per_sm = std::max(per_sm, 1);
  const int64_t grid = std::min<int64_t>(ceil_div(a.n_items, kLowWarps), int64_t(kNumSMs) * per_sm);
  kern<<<unsigned(std::max<int64_t>(grid, 1)), kLowThreads, 0, s>>>(a);
  TJ_CHECK_LAUNCH();
}

void launch_refine_lowd(const RefineArgs& a, cudaStream_t s) {
  if (a.d_pad != 4) fail(TJ_EINVAL, "low-d DMMA refine needs d <= 4");
  if (a.d <= 3) launch_lowd_t<true>(a, s);
  else launch_lowd_t<false>(a, s);
}

}  // namespace tj
