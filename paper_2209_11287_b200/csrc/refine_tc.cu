// DMMA refine for 5 <= d <= 64 (NCH = ceil(d/4) >= 2 chunks): configs 3 and
// 4(d >= 8), where the join is FP64-bound.
//
// Reference: _TileRefiner / distance_tile_v2 (join.py:238-283, kernels.py:184-263):
// per 4-dim chunk D = (-2Q) * C^T + acc, short-circuit when every entry of the
// tile already exceeds eps^2 (join.py:250-253), emit <= eps^2.
//
// B200 mapping (FP64-pipe bound, so the loop is built around keeping the DMMA
// pipe fed):
//  * one warp per work item (<= 8*NG queries of one cell x a slice of its
//    concatenated candidate list), transposed tiles: candidates are the A
//    operand (rows), queries the B operand (columns; -2*q chunk fragments stay
//    in registers for the whole item), C starts at the candidate norm and the
//    NCH DMMAs of a tile chain through the accumulator;
//  * a warp-uniform cursor walks the item's runs (clipped to its slice) and
//    cuts them into 8-candidate blocks; SB blocks form one stage of a per-warp
//    cp.async ring (one wait + one barrier per stage, not per block); rows are
//    padded so fragment reads are bank-conflict free; a 16-byte record per row
//    (short-circuit suffix, |c|^2) rides along;
//  * two blocks per step: 2 * NG independent DMMA chains are interleaved chunk
//    by chunk, so the chain latency is hidden inside the warp;
//  * short-circuit (optional, adaptive): one check after half of the chunks; a
//    tile stops when every entry's partial distance (acc - candidate suffix +
//    query prefix) exceeds eps^2 + 2*guard -- safe under rounding, decisions
//    stay exact.  A warp stops checking when its first 64 checks save fewer
//    DMMAs than they cost (prune rate * (NCH - CH) < 3/4; re-probed every 16
//    items) and then runs the plain step;
//  * exact decisions: guard band as in refine_lowd.cu (values above the band's
//    lower edge re-decided out of line by the reference direct form);
//  * emission: hits are sparse at these dimensionalities (|R|/C ~ 1e-3), so a
//    step branches once on the OR of all its compare ballots and only steps
//    with a hit look at tiles one by one; pairs go through a per-warp shared-memory buffer flushed with one
//    atomicAdd per 256 pairs; per-query counts accumulate in registers and are
//    added once per item (items of a big cell share queries).
#include "internal.cuh"
#include "refine_common.cuh"

namespace tj {

constexpr int kTcWarps = 4;
constexpr int kTcThreads = kTcWarps * kWarp;


template <int NCH>
struct TcShape {
  static constexpr int DP = 4 * NCH;
  static constexpr int STRIDE = (DP % 8 == 0) ? DP + 4 : DP;  // conflict-free fragment rows
  static constexpr int SB = NCH <= 4 ? 4 : 2;                  // blocks per stage (even)
  static constexpr int ROWS = 8 * SB;
  static constexpr int PPR = DP / 2;                           // 16-byte pieces per row
  static constexpr int CH = NCH / 2;                           // chunks before the check
};

template <int NCH>
struct alignas(16) TcStage {
  double pts[TcShape<NCH>::ROWS][TcShape<NCH>::STRIDE];
  double rec[TcShape<NCH>::ROWS][2];  // chunk-norm suffix after the check point, |c|^2
  uint32_t pos[TcShape<NCH>::SB];     // position of each block's row 0
  uint32_t nblk;                      // blocks staged (the rest are padding)
  uint32_t pad[3];
};

__device__ __forceinline__ void tc_cp16(void* smem, const void* gmem) {
  const unsigned s = unsigned(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void tc_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void tc_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// Re-decide guard-band pairs with the reference direct form (rare, out of line).
__device__ __noinline__ uint2 tc_recheck(const double* P, int dp, int d, double eps_sq, bool b0,
                                         bool b1, unsigned m0, unsigned m1, uint32_t qa,
                                         uint32_t c, unsigned long long* ctr) {
  bool p0 = (m0 >> lane_id()) & 1u, p1 = (m1 >> lane_id()) & 1u;
  if (b0) p0 = direct_form_le(P, dp, d, qa, c, eps_sq);
  if (b1) p1 = direct_form_le(P, dp, d, qa + 1, c, eps_sq);
  const unsigned nb = __popc(__ballot_sync(0xffffffffu, b0)) + __popc(__ballot_sync(0xffffffffu, b1));
  if (lane_id() == 0) atomicAdd(ctr, (unsigned long long)nb);
  return make_uint2(__ballot_sync(0xffffffffu, p0), __ballot_sync(0xffffffffu, p1));
}

// Warp-uniform walk over the item's runs clipped to [s0, s1) of the
// concatenated candidate list, one 8-candidate block at a time (runs are tiled
// separately: a block never straddles two runs, so its rows are contiguous).
struct BlockCursor {
  int64_t r, re;     // current run, end of the cell's runs
  uint32_t x, y;     // remaining positions [x, y) of the current run piece
  uint32_t at, s1;   // concat offset of x, slice end
  __device__ __forceinline__ void load_run(const RefineArgs& a) {
    while (r < re) {
      const uint32_t off = a.run_off[r];
      const uint2 run = a.runs[r];
      const uint32_t lo = max(off, at), hi = min(off + (run.y - run.x), s1);
      if (lo < hi) {
        x = run.x + (lo - off);
        y = x + (hi - lo);
        at = lo;
        return;
      }
      if (off >= s1) break;
      ++r;
    }
    x = y = 0;
    r = re;
  }
  __device__ __forceinline__ bool next(uint32_t& pos, uint32_t& valid, const RefineArgs& a) {
    if (x >= y) return false;
    pos = x;
    valid = min(8u, y - x);
    x += valid;
    at += valid;
    if (x >= y) {
      ++r;
      load_run(a);
    }
    return true;
  }
};

template <int NCH, int NG>
struct TcQuery {
  double bq[NG][NCH];  // -2 * query chunk, B fragments
  double thr[NG][2];   // pass iff D <= thr (upper edge of the guard band)
  double tlo[NG][2];   // D > tlo: inside the band, decided exactly
  double pre[NG][2];   // check: prune iff D_partial - suffix > pre for the whole tile
};

// One step: blocks k and k+1 of stage s (the second may be padding) against
// the NG query groups -- 2*NG accumulator chains advanced chunk by chunk.
template <int NCH, int NG, bool SC>
__device__ __forceinline__ void tc_step(const RefineArgs& a, const TcQuery<NCH, NG>& qs,
                                        const TcStage<NCH>* s, int k, uint32_t q0, bool& check,
                                        unsigned& n_checks, unsigned& n_pruned,
                                        unsigned long long& st_skip, unsigned (&qc)[NG][2],
                                        HitBuffer& hb, uint2* hits) {
  using S = TcShape<NCH>;
  constexpr int CH = S::CH;
  const int lane = lane_id();
  const int row = lane >> 2, col = lane & 3;
  const unsigned lt = lanemask_lt();
  double acc[2][NG][2];
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const double cn = s->rec[8 * (k + u) + row][1];
#pragma unroll
    for (int g = 0; g < NG; ++g) acc[u][g][0] = acc[u][g][1] = cn;
  }
  bool live[2][NG];
#pragma unroll
  for (int u = 0; u < 2; ++u)
#pragma unroll
    for (int g = 0; g < NG; ++g) live[u][g] = true;
  // chunks [0, CH): all chains
#pragma unroll
  for (int j = 0; j < (SC ? CH : NCH); ++j) {
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const double av = s->pts[8 * (k + u) + row][4 * j + col];
#pragma unroll
      for (int g = 0; g < NG; ++g)
        dmma_8x8x4(acc[u][g][0], acc[u][g][1], av, qs.bq[g][j], acc[u][g][0], acc[u][g][1]);
    }
  }
  if constexpr (SC) {
    if (check) {
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const double sf = s->rec[8 * (k + u) + row][0];
#pragma unroll
        for (int g = 0; g < NG; ++g) {
          const bool far = (acc[u][g][0] - sf > qs.pre[g][0]) && (acc[u][g][1] - sf > qs.pre[g][1]);
          live[u][g] = !__all_sync(0xffffffffu, far);
          ++n_checks;
          if (!live[u][g]) {
            ++n_pruned;
            st_skip += NCH - CH;
          }
        }
      }
    }
    // chunks [CH, NCH): chains still live
#pragma unroll
    for (int j = CH; j < NCH; ++j) {
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const double av = s->pts[8 * (k + u) + row][4 * j + col];
#pragma unroll
        for (int g = 0; g < NG; ++g)
          if (live[u][g])
            dmma_8x8x4(acc[u][g][0], acc[u][g][1], av, qs.bq[g][j], acc[u][g][0], acc[u][g][1]);
      }
    }
  }
  // epilogue: one branch for the step on the OR of the compare ballots (not
  // kept: registers; hits are rare); steps with a hit recompute them per tile.
  // Pruned tiles hold partial sums and are masked out.
  unsigned any = 0u;
#pragma unroll
  for (int u = 0; u < 2; ++u)
#pragma unroll
    for (int g = 0; g < NG; ++g) {
      const unsigned lv = live[u][g] ? 0xffffffffu : 0u;
      any |= (__ballot_sync(0xffffffffu, acc[u][g][0] <= qs.thr[g][0]) |
              __ballot_sync(0xffffffffu, acc[u][g][1] <= qs.thr[g][1])) & lv;
    }
  if (any == 0u) return;
#pragma unroll
  for (int u = 0; u < 2; ++u)
#pragma unroll
    for (int g = 0; g < NG; ++g) {
      if (!live[u][g]) continue;
      const bool p0 = acc[u][g][0] <= qs.thr[g][0];
      const bool p1 = acc[u][g][1] <= qs.thr[g][1];
      unsigned m0 = __ballot_sync(0xffffffffu, p0);
      unsigned m1 = __ballot_sync(0xffffffffu, p1);
      if ((m0 | m1) == 0) continue;
      const uint32_t cpos = s->pos[k + u] + uint32_t(row);
      const uint32_t qa = q0 + 8 * g + 2 * col;
      const bool b0 = p0 && acc[u][g][0] > qs.tlo[g][0];
      const bool b1 = p1 && acc[u][g][1] > qs.tlo[g][1];
      if (__any_sync(0xffffffffu, b0 || b1)) {
        const uint2 m = tc_recheck(a.P, 4 * NCH, a.d, a.eps_sq, b0, b1, m0, m1, qa, cpos,
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

// NG: query groups per item (2 by default; 4 = 32-query items for big cells at
// NCH <= 2, where sharing each staged block among more groups pays).
template <int NCH, bool SC, int R, int MINB, int NG>
__global__ void __launch_bounds__(kTcThreads, MINB) refine_tc_kernel(RefineArgs a) {
  using S = TcShape<NCH>;
  constexpr int DP = S::DP, SB = S::SB, ROWS = S::ROWS, PPR = S::PPR, CH = S::CH;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5;
  const int lane = lane_id();
  const int row = lane >> 2, col = lane & 3;
  TcStage<NCH>* ring = reinterpret_cast<TcStage<NCH>*>(smem_raw) + warp * R;
  uint2* hits = reinterpret_cast<uint2*>(reinterpret_cast<TcStage<NCH>*>(smem_raw) + kTcWarps * R) +
                warp * kHitBuf;
  HitBuffer hb;
  unsigned long long st_tiles_ref = 0, st_tiles = 0, st_skip = 0;
  const double eps_sq = a.eps_sq;
  bool sc_check = SC && a.short_circuit != 0;
  unsigned sc_items = 0, n_checks = 0, n_pruned = 0;

  for (;;) {
    unsigned long long idx = 0;
    if (lane == 0) idx = atomicAdd(&a.ctr->item_next, 1ull);
    idx = __shfl_sync(0xffffffffu, idx, 0);
    if (idx >= (unsigned long long)a.n_items) break;
    const WorkItem it = a.items[idx];
    const int nq = int(it.nq);
    const int ng = (nq + 7) >> 3;

    // ---- query side
    TcQuery<NCH, NG> qs;
#pragma unroll
    for (int g = 0; g < NG; ++g) {
      const int qb = 8 * g + row;
      const bool vb = qb < nq;
#pragma unroll
      for (int j = 0; j < NCH; ++j)
        qs.bq[g][j] = vb ? -2.0 * a.P[size_t(it.q0 + qb) * DP + 4 * j + col] : 0.0;
#pragma unroll
      for (int jj = 0; jj < 2; ++jj) {
        const int q = 8 * g + 2 * col + jj;
        const bool v = q < nq;
        const size_t qp = size_t(it.q0) + (v ? q : 0);
        const double qn = v ? a.NRM[qp] : 0.0;
        const double guard = a.guard_rel * (qn + a.max_norm) + 1e-300;
        const double center = eps_sq - qn;
        qs.thr[g][jj] = v ? center + guard : -INFINITY;
        qs.tlo[g][jj] = v ? center - guard : INFINITY;
        // eps^2 + 2*guard - (query chunk norms up to the check point)
        double pre = 0.0;
        for (int j = 0; j < CH; ++j) pre += v ? a.CN[qp * NCH + j] : 0.0;
        qs.pre[g][jj] = v ? eps_sq + 2.0 * guard - pre : -INFINITY;
      }
    }
    unsigned qc[NG][2];
#pragma unroll
    for (int g = 0; g < NG; ++g) qc[g][0] = qc[g][1] = 0;
    st_tiles_ref += uint64_t(ng) * ((it.s1 - it.s0 + 7) >> 3);

    // ---- candidate stream
    BlockCursor cur;
    {
      int64_t lo = a.cell_runs[it.cell], hi = a.cell_runs[it.cell + 1];
      cur.re = hi;
      while (hi - lo > 1) {  // first run with offset <= s0
        const int64_t mid = (lo + hi) >> 1;
        if (a.run_off[mid] <= it.s0) lo = mid;
        else hi = mid;
      }
      cur.r = lo;
      cur.at = it.s0;
      cur.s1 = it.s1;
      cur.load_run(a);
    }
    // stage up to SB blocks; lane -> (row, 16-byte piece) over the whole stage
    auto issue = [&](TcStage<NCH>* st) -> int {
      uint32_t bpos[SB], bval[SB];
      int nb = 0;
#pragma unroll
      for (int b = 0; b < SB; ++b) {
        bpos[b] = 0;
        bval[b] = 0;
        if (cur.next(bpos[b], bval[b], a)) ++nb;
      }
#pragma unroll
      for (int i0 = 0; i0 < ROWS * PPR; i0 += 32) {
        const int i = i0 + lane;
        if (i < ROWS * PPR) {
          const int rr = i / PPR, pc = i - rr * PPR;
          const int b = rr >> 3, r8 = rr & 7;
          uint32_t p = bpos[0], v = bval[0];
#pragma unroll
          for (int bb = 1; bb < SB; ++bb)
            if (b == bb) {
              p = bpos[bb];
              v = bval[bb];
            }
          if (uint32_t(r8) < v) tc_cp16(&st->pts[rr][2 * pc], a.P + size_t(p + r8) * DP + 2 * pc);
          else *reinterpret_cast<double2*>(&st->pts[rr][2 * pc]) = make_double2(0.0, 0.0);
        }
      }
      // records: (chunk-norm suffix after the check point, |c|^2)
      for (int rr = lane; rr < ROWS; rr += 32) {
        const int b = rr >> 3, r8 = rr & 7;
        uint32_t p = bpos[0], v = bval[0];
#pragma unroll
        for (int bb = 1; bb < SB; ++bb)
          if (b == bb) {
            p = bpos[bb];
            v = bval[bb];
          }
        if (uint32_t(r8) < v) {
          tc_cp16(&st->rec[rr][0], a.SFX + size_t(p + r8) * 2);
        } else {
          st->rec[rr][0] = 0.0;
          st->rec[rr][1] = kPadNorm;
        }
      }
      if (lane < SB) st->pos[lane] = bpos[lane];
      if (lane == 0) st->nblk = nb;
      tc_commit();
      return nb;
    };
    // adaptive short-circuit: keep checking while at least 1/4 of checks prune;
    // the verdict carries over to the warp's next items (re-probed every 16)
    if (SC && (++sc_items & 15u) == 0) {
      sc_check = true;
      n_checks = n_pruned = 0;
    }
    bool& check = sc_check;
    int pending = 0;  // stages holding at least one block
#pragma unroll
    for (int k = 0; k < R - 1; ++k) pending += issue(ring + k) > 0 ? 1 : 0;
#pragma unroll 1
    for (int st = 0; st < pending; ++st) {
      tc_wait<R - 2>();
      __syncwarp();
      const TcStage<NCH>* s = ring + (st % R);
      const int nb = int(s->nblk);
      st_tiles += uint64_t(nb) * ng;
      // (a missing second group / block is padding: its values never pass)
      if (SC && check) {
#pragma unroll 1
        for (int k = 0; k < nb; k += 2)
          tc_step<NCH, NG, SC>(a, qs, s, k, it.q0, check, n_checks, n_pruned, st_skip, qc, hb, hits);
        // a check costs ~1.5 DMMA issue slots; a prune saves NCH - CH DMMAs
        if (n_checks >= 64 && 4 * n_pruned * (NCH - CH) < 3 * n_checks) check = false;
      } else {  // not checking: the plain step (no live flags, no predicated DMMAs)
#pragma unroll 1
        for (int k = 0; k < nb; k += 2)
          tc_step<NCH, NG, false>(a, qs, s, k, it.q0, check, n_checks, n_pruned, st_skip, qc, hb, hits);
      }
      __syncwarp();
      pending += issue(ring + ((st + R - 1) % R)) > 0 ? 1 : 0;
    }
    tc_wait<0>();
    // per-query counts (items of one cell may share queries: atomic add)
#pragma unroll
    for (int g = 0; g < NG; ++g) {
#pragma unroll
      for (int jj = 0; jj < 2; ++jj) {
        unsigned c = qc[g][jj];
        c += __shfl_xor_sync(0xffffffffu, c, 4);
        c += __shfl_xor_sync(0xffffffffu, c, 8);
        c += __shfl_xor_sync(0xffffffffu, c, 16);
        const int q = 8 * g + 2 * col + jj;
        if (row == 0 && q < nq && c) atomicAdd(&a.qcount[it.q0 + q], c);
      }
    }
    if (lane == 0) atomicAdd(&a.ctr->refined, (unsigned long long)nq * (it.s1 - it.s0));
  }
  hb.flush(hits, a);
  // chunk counters in the reference's tiling: scale our skips to its tile count
  if (lane != 0) st_tiles_ref = st_tiles = st_skip = 0;
  unsigned long long skip_ref =
      st_tiles ? (unsigned long long)((double)st_skip * (double)st_tiles_ref / (double)st_tiles) : 0;
  if (skip_ref > st_tiles_ref * NCH) skip_ref = st_tiles_ref * NCH;
  flush_stats(a, st_tiles_ref, st_tiles_ref * NCH - skip_ref, skip_ref, 0);
}

// 32-query items (NG = 4) when the cells are big enough to fill them (NCH <= 2).
static bool tc_big_items(int nch, int64_t n, int64_t n_cells) {
  return nch <= 2 && n >= 48 * n_cells;
}

int tc_queries_per_item(int d_pad, int64_t n, int64_t n_cells) {
  const int nch = d_pad / 4;
  if (tc_big_items(nch, n, n_cells)) return 32;
  return 16;
}

template <int NCH, bool SC, int R, int MINB, int NG>
static void launch_tc_t(const RefineArgs& a, cudaStream_t s) {
  const size_t smem = sizeof(TcStage<NCH>) * kTcWarps * R + sizeof(uint2) * kTcWarps * kHitBuf;
  auto kern = refine_tc_kernel<NCH, SC, R, MINB, NG>;
  TJ_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  int per_sm = 0;
  TJ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kTcThreads, smem));
  per_sm = std::max(per_sm, 1);
  const int64_t grid = std::min<int64_t>(ceil_div(a.n_items, kTcWarps), int64_t(kNumSMs) * per_sm);
  kern<<<unsigned(std::max<int64_t>(grid, 1)), kTcThreads, smem, s>>>(a);
  TJ_CHECK_LAUNCH();
}

// Ring depth and CTAs per SM measured on d = 8 / 16 / 32 (ring x occupancy
// sweep): a 2-stage ring at 4 CTAs (16 warps, <= 128 registers) for NCH <= 4,
// a 3-stage ring at 3 CTAs up to NCH = 8, and above that a 2-stage ring at 2
// CTAs so two query groups' fragments fit in registers (d = 64: one group per
// item, 50.6 s -> two groups, 27.9 s).
template <int NCH, bool SC>
static void launch_tc_v(const RefineArgs& a, cudaStream_t s, bool big) {
  if constexpr (NCH <= 2) {
    if (big) return launch_tc_t<NCH, SC, 2, 3, 4>(a, s);
  }
  if constexpr (NCH <= 4) launch_tc_t<NCH, SC, 2, 4, 2>(a, s);
  else if constexpr (NCH <= 8) launch_tc_t<NCH, SC, 3, 3, 2>(a, s);
  else launch_tc_t<NCH, SC, 2, 2, 2>(a, s);
}

template <int NCH>
static void launch_tc_sc(const RefineArgs& a, cudaStream_t s, bool big) {
  if (a.short_circuit) launch_tc_v<NCH, true>(a, s, big);
  else launch_tc_v<NCH, false>(a, s, big);
}

void launch_refine_tc(const RefineArgs& a, int64_t n, int64_t n_cells, cudaStream_t s) {
  const bool big = tc_big_items(a.nchunks, n, n_cells);
  switch (a.nchunks) {
    case 2: return launch_tc_sc<2>(a, s, big);
    case 3: return launch_tc_sc<3>(a, s, big);
    case 4: return launch_tc_sc<4>(a, s, big);
    case 5: return launch_tc_sc<5>(a, s, big);
    case 6: return launch_tc_sc<6>(a, s, big);
    case 7: return launch_tc_sc<7>(a, s, big);
    case 8: return launch_tc_sc<8>(a, s, big);
    case 9: return launch_tc_sc<9>(a, s, big);
    case 10: return launch_tc_sc<10>(a, s, big);
    case 11: return launch_tc_sc<11>(a, s, big);
    case 12: return launch_tc_sc<12>(a, s, big);
    case 13: return launch_tc_sc<13>(a, s, big);
    case 14: return launch_tc_sc<14>(a, s, big);
    case 15: return launch_tc_sc<15>(a, s, big);
    case 16: return launch_tc_sc<16>(a, s, big);
    default: break;
  }
  fail(TJ_EINVAL, "DMMA refine is instantiated for 5 <= d <= 64, got d=" + std::to_string(a.d));
}

}  // namespace tj
