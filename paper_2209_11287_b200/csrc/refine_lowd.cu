// DMMA refine for d <= 4 (one 4-dim chunk): the hot kernel of configs 1, 2,
// 4(d<=4) and 5.
//
// Same math as refine_tc.cu (paper Alg. 2, exact decisions through a guard
// band), mapped for the fewest instructions per m8n8k4 tile:
//  * one warp per work item (<= 32 queries of one cell = NG <= 4 query groups,
//    a compile-time parameter of the block loop), no CTA barriers;
//  * transposed roles: candidates are the A operand (rows) and the queries the
//    B operand (columns), so the C operand is the candidates' norms and each
//    lane loads exactly the norm of the candidate whose coordinate it loads;
//    query fragments and thresholds stay in registers for the whole item;
//  * d <= 3: |c|^2 sits in the padding coordinate of P (A col 3), B row 3 = 1,
//    C = |q|^2: D is the squared distance with no norm load at all;
//  * 8-candidate blocks tile the cell's *concatenated* candidate list exactly
//    as the reference tiles it (join.py:257-261): blocks straddle run
//    boundaries, only the list's last block is padded.  Candidates are staged
//    64 at a time (two per lane, one coalesced 32-byte row each) into a
//    2-stage per-warp cp.async ring (5 CTAs = 20 warps per SM: the measured
//    best ring depth / occupancy); a warp-uniform run cursor maps list offsets
//    to cell-ordered positions;
//  * hit test: one DSETP + ballot per value against the guard band's upper
//    edge; the band itself is pre-tested on the integer pipe (the high word of
//    D between the band edges' high words, IADD + ISETP), so the FP64 pipe runs
//    only the DMMA and one DSETP per value; the rare steps where a value is that
//    near the band re-decide its passing values out of line by the reference
//    direct form;
//  * output: the tile's two ballots form one 64-bit hit mask.  One lane writes
//    each step's masks to the warp's window buffer in shared memory (vector
//    stores); a 32-block window is flushed with one coalesced 256-byte store per
//    query group.  No atomics, no ranking, no counting: finalize.cu counts each
//    row from the masks (count_rows_kernel) and expands them into sorted CSR
//    rows.
// Keep the hot loop small: the whole kernel must stay within the instruction
// cache (rare paths are __noinline__).
// JoinStats tiles are ceil(nq/8) * ceil(|cand|/8) per item -- exactly the tiles
// executed, and the reference formula (join.py:257-261); chunks = tiles since
// d <= 4 has one chunk (kernels.py:250).
#include "internal.cuh"
#include "refine_common.cuh"

namespace tj {

constexpr int kLowWarps = 4;
constexpr int kLowThreads = kLowWarps * kWarp;
constexpr int kLowStages = 2;  // cp.async ring depth per warp (stages of 8 blocks)
constexpr int kStageCands = 64;

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

constexpr int kWinLd = 8;  // window buffer row: <= 4 groups x (low, high) mask words

struct LowStage {
  double pts[kStageCands][4];  // candidate coordinates (d <= 3: slot 3 holds |c|^2)
  double2 nrm[kStageCands];    // (|c|^2, |c|^2): the C operand pair (d == 4)
  uint32_t pos[kStageCands];   // cell-ordered positions (guard-band recheck only)
};

template <int NG>
struct QuerySide {
  double bq[NG];                 // B fragments per group
  double cq[NG][2];              // FOLD: C operand |q|^2 per column
  double thr[NG][2];             // pass iff D <= thr (upper edge of the guard band)
  uint32_t hlo[NG][2], hrg[NG][2];  // band pre-test: high word of D in [hlo, hlo + hrg]
};

// Guard-band pairs of one tile, re-decided by the reference direct form.
// (m0, m1): the tile's ballots; returns them corrected.  Out of line: rare.
__device__ __noinline__ uint2 recheck_tile(const double* P, int d, double eps_sq, bool b0,
                                           bool b1, unsigned m0, unsigned m1, uint32_t qa,
                                           uint32_t c, unsigned long long* ctr) {
  bool p0 = (m0 >> lane_id()) & 1u, p1 = (m1 >> lane_id()) & 1u;
  if (b0) p0 = direct_form_le(P, 4, d, qa, c, eps_sq);
  if (b1) p1 = direct_form_le(P, 4, d, qa + 1, c, eps_sq);
  const unsigned nb = __popc(__ballot_sync(0xffffffffu, b0)) + __popc(__ballot_sync(0xffffffffu, b1));
  if (lane_id() == 0) atomicAdd(ctr, (unsigned long long)nb);
  return make_uint2(__ballot_sync(0xffffffffu, p0), __ballot_sync(0xffffffffu, p1));
}

// U consecutive staged blocks k .. k+U-1 against the NG query groups: all
// U * NG DMMAs are issued before the first compare, then one DSETP + ballot and
// the integer band pre-test per value; only steps with a value near the band
// leave the fast path.  Lane 0
// writes the blocks' masks to the warp's window buffer (vector stores).
template <bool FOLD, int NG, int U>
__device__ __forceinline__ void lowd_blocks(const RefineArgs& a, const QuerySide<NG>& qs,
                                            const LowStage* s, int k, uint32_t* wbuf,
                                            uint32_t q0) {
  const int lane = lane_id();
  const int row = lane >> 2, col = lane & 3;
  double av[U];
  double2 cv[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    av[u] = s->pts[8 * (k + u) + row][col];
    cv[u] = FOLD ? make_double2(0.0, 0.0) : s->nrm[8 * (k + u) + row];
  }
  double dv[U][NG][2];
#pragma unroll
  for (int u = 0; u < U; ++u)
#pragma unroll
    for (int g = 0; g < NG; ++g)
      dmma_8x8x4(dv[u][g][0], dv[u][g][1], av[u], qs.bq[g], FOLD ? qs.cq[g][0] : cv[u].x,
                 FOLD ? qs.cq[g][1] : cv[u].y);
  unsigned m[U][NG][2];
  // band pre-test on the integer pipe: a value inside the guard band has the
  // high word of a double between the band edges' high words (same-sign edges:
  // bit patterns are monotone in magnitude), so one IADD + ISETP per value
  // replaces a second DSETP on the FP64 pipe the DMMAs use
  bool near = false;
#pragma unroll
  for (int u = 0; u < U; ++u)
#pragma unroll
    for (int g = 0; g < NG; ++g)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        m[u][g][j] = __ballot_sync(0xffffffffu, dv[u][g][j] <= qs.thr[g][j]);
        near |= uint32_t(__double2hiint(dv[u][g][j])) - qs.hlo[g][j] <= qs.hrg[g][j];
      }
  if (__any_sync(0xffffffffu, near)) {  // rare: re-decide passing values near the band exactly
    unsigned bm[U][NG][2];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int g = 0; g < NG; ++g)
#pragma unroll
        for (int j = 0; j < 2; ++j)
          bm[u][g][j] = __ballot_sync(0xffffffffu, uint32_t(__double2hiint(dv[u][g][j])) - qs.hlo[g][j] <=
                                                       qs.hrg[g][j]) &
                        m[u][g][j];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int g = 0; g < NG; ++g) {
        if (bm[u][g][0] | bm[u][g][1]) {
          const uint2 mm = recheck_tile(a.P, a.d, a.eps_sq, (bm[u][g][0] >> lane) & 1u,
                                        (bm[u][g][1] >> lane) & 1u, m[u][g][0], m[u][g][1],
                                        q0 + 8 * g + 2 * col, s->pos[8 * (k + u) + row],
                                        &a.ctr->rechecks);
          m[u][g][0] = mm.x;
          m[u][g][1] = mm.y;
        }
      }
  }
  // the block's masks into the window buffer (one lane, vector stores)
  if (lane == 0) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      uint32_t* w = wbuf + (k + u) * kWinLd;
#pragma unroll
      for (int g = 0; g < NG; g += 2) {
        if (g + 1 < NG)
          *reinterpret_cast<uint4*>(w + 2 * g) = make_uint4(m[u][g][0], m[u][g][1], m[u][g + 1][0], m[u][g + 1][1]);
        else
          *reinterpret_cast<uint2*>(w + 2 * g) = make_uint2(m[u][g][0], m[u][g][1]);
      }
    }
  }
}

// All tiles of one work item with NG query groups (compile-time, so the block
// loop has no group branches): the item's candidate list is staged 64
// candidates at a time and every 8-candidate block is multiplied against the
// NG query fragments back to back (independent DMMAs in flight), then
// compared and balloted.
// Blocks cover the item's candidates [s0, total) of the cell's list (s0 = 0, or the
// cell's own offset in the symmetric join).
template <bool FOLD, int NG, int R, bool U2ALL>
__device__ __forceinline__ void lowd_item(const RefineArgs& a, const WorkItem& it, LowStage* ring,
                                          uint32_t* wbuf, unsigned long long* mrow, int nblk,
                                          uint32_t s0, uint32_t total, uint32_t r_off,
                                          uint32_t r_pos, int nr) {
  const int lane = lane_id();
  const int row = lane >> 2, col = lane & 3;
  const int nq = int(it.nq);
  const double eps_sq = a.eps_sq;
  QuerySide<NG> qs;
#pragma unroll
  for (int g = 0; g < NG; ++g) {
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
      const uint32_t hh = uint32_t(__double2hiint(hi)), hl = uint32_t(__double2hiint(lo));
      if ((hh ^ hl) >> 31) {  // edges of opposite signs (band around 0): always re-decide
        qs.hlo[g][j] = 0u;
        qs.hrg[g][j] = 0xffffffffu;
      } else {
        qs.hlo[g][j] = min(hh, hl);
        qs.hrg[g][j] = max(hh, hl) - min(hh, hl);
      }
    }
  }
  const int nst = (nblk + 7) >> 3;
  // run containing the first candidate of the next stage to issue
  int rc = __popc(__ballot_sync(0xffffffffu, lane < nr && r_off <= s0)) - 1;
  auto issue = [&](int st, LowStage* s) {
    const uint32_t base = s0 + uint32_t(st) * kStageCands;
    const uint32_t t0 = base + lane, t1 = t0 + 32;
    uint32_t p0 = 0, p1 = 0;
    int r = rc;
    for (;;) {
      const uint32_t o = __shfl_sync(0xffffffffu, r_off, r);
      const uint32_t ps = __shfl_sync(0xffffffffu, r_pos, r);
      if (t0 >= o) p0 = ps + (t0 - o);
      if (t1 >= o) p1 = ps + (t1 - o);
      const uint32_t on = __shfl_sync(0xffffffffu, r_off, r + 1);
      if (r + 1 >= nr || on >= base + kStageCands) break;
      ++r;
    }
    rc = r;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint32_t t = h ? t1 : t0;
      const uint32_t p = h ? p1 : p0;
      const int slot = lane + 32 * h;
      if (t < total) {
        const double* src = a.P + size_t(p) * 4;
        cp_async16(&s->pts[slot][0], src);
        cp_async16(&s->pts[slot][2], src + 2);
        if (!FOLD) {
          cp_async8(&s->nrm[slot].x, a.NRM + p);
          cp_async8(&s->nrm[slot].y, a.NRM + p);
        }
        s->pos[slot] = p;
      } else {  // padding row: never within eps
        *reinterpret_cast<double2*>(&s->pts[slot][0]) = make_double2(0.0, 0.0);
        *reinterpret_cast<double2*>(&s->pts[slot][2]) = make_double2(0.0, FOLD ? kPadNorm : 0.0);
        s->nrm[slot] = make_double2(kPadNorm, kPadNorm);
        s->pos[slot] = 0;
      }
    }
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
    const int nb = min(8, nblk - 8 * st);
    uint32_t* wb = wbuf + ((st & 3) << 3) * kWinLd;  // this stage's 8 blocks of the window
    // NG <= 2: two blocks per step (2 * NG independent DMMAs in flight); an odd
    // stage end runs one padding block, whose rows never pass
    constexpr int U = (NG <= 2 || U2ALL) ? 2 : 1;
#pragma unroll 1
    for (int k = 0; k < nb; k += U) lowd_blocks<FOLD, NG, U>(a, qs, s, k, wb, it.q0);
    // window of 32 blocks complete: lane k stores block (window + k) of each group
    if ((st & 3) == 3 || st + 1 == nst) {
      __syncwarp();
      const int b = ((st >> 2) << 5) + lane;
      if (b < nblk) {
        const uint2* w = reinterpret_cast<const uint2*>(wbuf + lane * kWinLd);
#pragma unroll
        for (int g = 0; g < NG; ++g) {
          const uint2 v = w[g];
          mrow[int64_t(g) * nblk + b] = (static_cast<unsigned long long>(v.y) << 32) | v.x;
        }
      }
    }
    __syncwarp();
    if (st + R - 1 < nst) issue(st + R - 1, ring + ((st + R - 1) % R));
    else cp_async_commit();
  }
  cp_async_wait<0>();
}

// NGMAX: largest query-group count of an item (items hold <= 8 * NGMAX queries);
// NGMAX = 2 keeps the kernel within 102 registers (5 CTAs = 20 warps per SM).
template <bool FOLD, int NGMAX, int R, bool U2ALL, int MINB>
__global__ void __launch_bounds__(kLowThreads, MINB) refine_lowd_kernel(RefineArgs a) {
  __shared__ LowStage s_ring[kLowWarps][R];
  __shared__ __align__(16) uint32_t s_win[kLowWarps][32 * kWinLd];
  const int warp = threadIdx.x >> 5;
  const int lane = lane_id();
  LowStage* ring = s_ring[warp];
  uint32_t* wbuf = s_win[warp];
  unsigned long long st_tiles = 0, st_refined = 0;
  const unsigned long long n_items = a.n_items_dev ? *a.n_items_dev : (unsigned long long)a.n_items;

  for (;;) {
    unsigned long long idx = 0;
    if (lane == 0) idx = atomicAdd(&a.ctr->item_next, 1ull);
    idx = __shfl_sync(0xffffffffu, idx, 0);
    if (idx >= n_items) break;
    const WorkItem it = a.items[idx];
    const int ng = (int(it.nq) + 7) >> 3;
    // candidate list = the cell's runs concatenated; lane r holds run r
    // (<= 27 runs for k <= 4); lanes past the last run hold the list length
    const int64_t rb = a.cell_runs[it.cell], re = a.cell_runs[it.cell + 1];
    const int nr = int(re - rb);
    const uint32_t total = it.s1;  // low-d items reach the end of the list
    // symmetric join: only candidates from the cell itself on (cells >= it.cell);
    // the pairs with earlier cells come from those cells' masks (finalize.cu)
    const uint32_t s0 = a.fwd ? a.fwd[it.cell] : 0u;
    uint32_t r_off = total, r_pos = 0;
    if (lane < nr) {
      r_off = a.run_off[rb + lane];
      r_pos = a.runs[rb + lane].x;
    }
    const int nblk = int((total - s0 + 7) >> 3);
    // JoinStats in the reference's tiling of the whole list (join.py:257-261, 273)
    st_tiles += uint64_t(ng) * uint64_t((total + 7) >> 3);
    st_refined += uint64_t(it.nq) * total;
    // this item's masks: (group, block) order, group (q0 - cell start) / 8 of the cell
    const int64_t cs = a.cell_start[it.cell];
    unsigned long long* mrow = a.masks + a.cell_mbase[it.cell - a.cell_base] +
                               ((int64_t(it.q0) - cs) >> 3) * nblk;
    switch (ng) {
      case 1: lowd_item<FOLD, 1, R, U2ALL>(a, it, ring, wbuf, mrow, nblk, s0, total, r_off, r_pos, nr); break;
      case 2: lowd_item<FOLD, 2, R, U2ALL>(a, it, ring, wbuf, mrow, nblk, s0, total, r_off, r_pos, nr); break;
      case 3:
        if constexpr (NGMAX >= 3)
          lowd_item<FOLD, 3, R, U2ALL>(a, it, ring, wbuf, mrow, nblk, s0, total, r_off, r_pos, nr);
        break;
      default:
        if constexpr (NGMAX >= 4)
          lowd_item<FOLD, 4, R, U2ALL>(a, it, ring, wbuf, mrow, nblk, s0, total, r_off, r_pos, nr);
        break;
    }
  }
  if (lane == 0 && st_refined) atomicAdd(&a.ctr->refined, st_refined);
  if (lane != 0) st_tiles = 0;
  flush_stats(a, st_tiles, st_tiles, 0, 0);
}

// Items of <= 32 queries (measured on c2: fewer partial groups and less restaging
// beat the higher occupancy of 16-query items).
int lowd_queries_per_item(int64_t, int64_t) { return 32; }  // NG <= 4 query groups

template <bool FOLD, int NGMAX, int R, bool U2ALL, int MINB>
static void launch_lowd_t(const RefineArgs& a, cudaStream_t s) {
  auto kern = refine_lowd_kernel<FOLD, NGMAX, R, U2ALL, MINB>;
  int per_sm = 0;
  TJ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kLowThreads, 0));
  per_sm = std::max(per_sm, 1);
  const int64_t grid = std::min<int64_t>(ceil_div(a.n_items, kLowWarps), int64_t(kNumSMs) * per_sm);
  kern<<<unsigned(std::max<int64_t>(grid, 1)), kLowThreads, 0, s>>>(a);
  TJ_CHECK_LAUNCH();
}

// Configuration measured best on c2/c4 d<=3 (tools/var_lowd.sh sweep): a
// 2-stage ring (64 candidates each), two-block steps for NG <= 2, 5 CTAs = 20
// warps per SM (<= 102 registers).
template <bool FOLD>
static void launch_lowd_v(const RefineArgs& a, cudaStream_t s) {
  launch_lowd_t<FOLD, 4, kLowStages, false, 5>(a, s);
}

void launch_refine_lowd(const RefineArgs& a, int64_t n, int64_t n_cells, cudaStream_t s) {
  if (a.d_pad != 4) fail(TJ_EINVAL, "low-d DMMA refine needs d <= 4");
  (void)n;
  (void)n_cells;
  if (a.d <= 3) launch_lowd_v<true>(a, s);
  else launch_lowd_v<false>(a, s);
}

}  // namespace tj
