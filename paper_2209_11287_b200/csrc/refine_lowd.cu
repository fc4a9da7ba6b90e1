// DMMA refine for d <= 4 (one 4-dim chunk): the hot kernel of configs 1, 2,
// 4(d<=4) and 5.
//
// Same math as refine_dmma.cu (paper Alg. 2, exact decisions through a guard
// band), mapped for minimum instructions per m8n8k4 tile:
//  * one warp per work item (a cell's query groups), no CTA barriers: the warp
//    streams the cell's candidate runs straight from L2 (256 contiguous bytes
//    per 8-candidate block) with the next block's loads in flight (ping-pong
//    registers, two blocks per loop trip);
//  * transposed roles: candidates are the A operand (rows) and the item's
//    queries the B operand (columns), so the C operand is the candidates'
//    norms and each lane loads exactly the norm of the candidate whose
//    coordinate it loads; query fragments and thresholds live in registers;
//  * d <= 3: |c|^2 sits in the padding coordinate of P (A col 3), B row 3 = 1,
//    C = |q|^2: D is the squared distance with no norm load at all;
//  * hit test: one DSETP per value against the guard-inflated threshold; the
//    guard band is screened with integer ops on the high word of the double;
//  * emission is deferred: a tile with hits logs its hit and band masks to a
//    per-warp shared-memory log; every ~32 entries the warp expands the log:
//    band pairs are re-decided with the exact direct form, hits become
//    (query, candidate) pairs behind one global atomicAdd, and per-query
//    counts come from the masks with warp reductions.
// JoinStats tiles are the reference formula ceil(nq/8) * ceil(|cand|/8) per item
// (join.py:257-261); chunks = tiles since d <= 4 has one chunk (kernels.py:250).
#include "internal.cuh"
#include "refine_common.cuh"

namespace tj {

constexpr int kLowWarps = 4;
constexpr int kLowThreads = kLowWarps * kWarp;
constexpr int kLogEntries = 32;

struct LogMasks {
  unsigned m0, m1;    // ballot hit masks: bit L -> (candidate L>>2, query 2*(L&3) + {0,1})
  unsigned bm0, bm1;  // subset inside the guard band (to re-decide exactly)
};
struct LogWhere {
  uint32_t pos;  // position of the block's first candidate
  uint32_t g;    // query group
};

__device__ __forceinline__ unsigned hi_word(double v) { return unsigned(__double2hiint(v)); }

// Expand `ns` log entries into pairs; returns this lane's query-count increment
// (lane L < 16 owns query column L of the item).
__device__ __forceinline__ unsigned expand_log(const LogMasks* lm, const LogWhere* lw, int ns,
                                               uint32_t q0, const RefineArgs& a,
                                               unsigned long long& rechecks) {
  const int lane = lane_id();
  LogMasks e = {0u, 0u, 0u, 0u};
  LogWhere w = {0u, 0u};
  if (lane < ns) {
    e = lm[lane];
    w = lw[lane];
  }
  const uint32_t qbase = q0 + 8 * w.g;
  if (__any_sync(0xffffffffu, (e.bm0 | e.bm1) != 0)) {
    // guard band: the reference direct form decides (rare)
    for (int h = 0; h < 2; ++h) {
      unsigned bm = h ? e.bm1 : e.bm0;
      unsigned m = h ? e.m1 : e.m0;
      while (bm) {
        const int L = __ffs(bm) - 1;
        bm &= bm - 1;
        const bool keep = direct_form_le(a.P, 4, a.d, qbase + 2 * (L & 3) + h, w.pos + (L >> 2),
                                         a.eps_sq);
        m = keep ? (m | (1u << L)) : (m & ~(1u << L));
        ++rechecks;
      }
      if (h) e.m1 = m;
      else e.m0 = m;
    }
  }
  const int cnt = __popc(e.m0) + __popc(e.m1);
  int incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  const int total = __shfl_sync(0xffffffffu, incl, 31);
  unsigned long long base = 0;
  if (lane == 0 && total) base = atomicAdd(&a.ctr->pairs, (unsigned long long)total);
  base = __shfl_sync(0xffffffffu, base, 0) + (incl - cnt);
  for (int h = 0; h < 2; ++h) {
    unsigned m = h ? e.m1 : e.m0;
    while (m) {
      const int L = __ffs(m) - 1;
      m &= m - 1;
      if (base < a.pair_cap) a.pairs[base] = make_uint2(qbase + 2 * (L & 3) + h, w.pos + (L >> 2));
      ++base;
    }
  }
  // per-query counts: column c of group g is bits 4r + (c>>1) of m0 (c even) / m1 (c odd)
  unsigned mine = 0;
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    const unsigned mm = (q & 1) ? e.m1 : e.m0;
    const unsigned v = (w.g == unsigned(q >> 3)) ? __popc(mm & (0x11111111u << ((q & 7) >> 1))) : 0u;
    const unsigned s = __reduce_add_sync(0xffffffffu, v);
    if (lane == q) mine = s;
  }
  return mine;
}

struct QuerySide {
  double bq[2];                 // B fragments per group
  double cq[2][2];              // FOLD: C operand |q|^2 per column
  double thr[2][2];             // pass iff D <= thr (guard-inflated)
  unsigned h1[2][2], hw[2][2];  // guard band as a high-word range [h1, h1+hw]
};

template <int NG, bool FOLD>
__device__ __forceinline__ int lowd_tile(const QuerySide& qs, LogMasks* lm, LogWhere* lw, int ns,
                                         double av, double cn, uint32_t p) {
  const int lane = lane_id();
#pragma unroll
  for (int g = 0; g < NG; ++g) {
    double d0, d1;
    dmma_8x8x4(d0, d1, av, qs.bq[g], FOLD ? qs.cq[g][0] : cn, FOLD ? qs.cq[g][1] : cn);
    const bool p0 = d0 <= qs.thr[g][0];
    const bool p1 = d1 <= qs.thr[g][1];
    const unsigned m0 = __ballot_sync(0xffffffffu, p0);
    const unsigned m1 = __ballot_sync(0xffffffffu, p1);
    if (m0 | m1) {
      const unsigned bm0 =
          __ballot_sync(0xffffffffu, p0 && (hi_word(d0) - qs.h1[g][0]) <= qs.hw[g][0]);
      const unsigned bm1 =
          __ballot_sync(0xffffffffu, p1 && (hi_word(d1) - qs.h1[g][1]) <= qs.hw[g][1]);
      if (lane == 0) {
        lm[ns] = LogMasks{m0, m1, bm0, bm1};
        lw[ns] = LogWhere{p, uint32_t(g)};
      }
      ++ns;
    }
  }
  return ns;
}

template <int NG, bool FOLD>
__device__ __forceinline__ unsigned lowd_runs(const RefineArgs& a, const QuerySide& qs,
                                              LogMasks* lm, LogWhere* lw, uint32_t q0,
                                              int64_t rb, int64_t re,
                                              unsigned long long& rechecks) {
  const int lane = lane_id();
  const int row = lane >> 2, col = lane & 3;
  const double pad_a = (FOLD && col == 3) ? kPadNorm : 0.0;
  constexpr int kRoom = kLogEntries - 2 * NG;  // room for one loop trip's entries
  unsigned qcnt = 0;
  int ns = 0;
#pragma unroll 1
  for (int64_t r = rb; r < re; ++r) {
    const uint2 run = a.runs[r];
    const int len = int(run.y - run.x);
    const int nblk = (len + 7) >> 3;
    const double* pa = a.P + size_t(run.x + row) * 4 + col;
    const double* pn = a.NRM + run.x + row;
    // block b covers rows 8b..8b+7 of the run; invalid rows read as padding
    bool v = row < len;
    double a0 = v ? pa[0] : pad_a;
    double c0 = FOLD ? 0.0 : (v ? pn[0] : kPadNorm);
#pragma unroll 1
    for (int b = 0; b < nblk; b += 2) {
      double a1 = pad_a, c1 = kPadNorm;
      const bool has1 = b + 1 < nblk;
      if (has1) {
        v = 8 * (b + 1) + row < len;
        a1 = v ? pa[32 * (b + 1)] : pad_a;
        if (!FOLD) c1 = v ? pn[8 * (b + 1)] : kPadNorm;
      }
      ns = lowd_tile<NG, FOLD>(qs, lm, lw, ns, a0, c0, run.x + 8 * b);
      if (b + 2 < nblk) {
        v = 8 * (b + 2) + row < len;
        a0 = v ? pa[32 * (b + 2)] : pad_a;
        if (!FOLD) c0 = v ? pn[8 * (b + 2)] : kPadNorm;
      }
      if (has1) ns = lowd_tile<NG, FOLD>(qs, lm, lw, ns, a1, c1, run.x + 8 * (b + 1));
      if (ns > kRoom) {
        __syncwarp();
        qcnt += expand_log(lm, lw, ns, q0, a, rechecks);
        __syncwarp();
        ns = 0;
      }
    }
  }
  if (ns) {
    __syncwarp();
    qcnt += expand_log(lm, lw, ns, q0, a, rechecks);
    __syncwarp();
  }
  return qcnt;
}

template <bool FOLD>
__global__ void __launch_bounds__(kLowThreads, 6) refine_lowd_kernel(RefineArgs a) {
  __shared__ LogMasks s_lm[kLowWarps][kLogEntries];
  __shared__ LogWhere s_lw[kLowWarps][kLogEntries];
  const int warp = threadIdx.x >> 5;
  const int lane = lane_id();
  const int row = lane >> 2;
  const int col = lane & 3;
  unsigned long long st_rechecks = 0, st_tiles = 0;
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
    const unsigned qcnt =
        ng == 1 ? lowd_runs<1, FOLD>(a, qs, s_lm[warp], s_lw[warp], it.q0, rb, re, st_rechecks)
                : lowd_runs<2, FOLD>(a, qs, s_lm[warp], s_lw[warp], it.q0, rb, re, st_rechecks);
    // each query lives in exactly one item: plain store of its count
    if (lane < nq) a.qcount[it.q0 + lane] = qcnt;
    if (lane == 0) atomicAdd(&a.ctr->refined, (unsigned long long)nq * (it.s1 - it.s0));
  }
  if (lane != 0) st_tiles = 0;
  flush_stats(a, st_tiles, st_tiles, 0, st_rechecks);
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
