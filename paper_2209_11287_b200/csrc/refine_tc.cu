// DMMA refine for 5 <= d <= 64 (NCH = ceil(d/4) >= 2 chunks): configs 3 and
// 4(d >= 8), where the join is FP64-bound.
//
// Reference: _TileRefiner / distance_tile_v2 (join.py:238-283, kernels.py:184-263):
// per 4-dim chunk D = (-2Q) * C^T + acc, short-circuit when every entry of the
// tile already exceeds eps^2 (join.py:250-253), emit <= eps^2.
//
// B200 mapping (same ideas as refine_lowd.cu, generalised to several chunks):
//  * one warp per work item (<= 8*NGM queries of one cell x a slice of its
//    concatenated candidate list), transposed tiles: candidates are the A operand
//    (rows), queries the B operand (columns, -2*q chunk fragments held in
//    registers for the whole item), C starts at the candidate norm and the NCH
//    DMMAs of a tile chain through the accumulator;
//  * a warp-uniform cursor walks the item's runs (clipped to its slice) block by
//    block; each 8-candidate block is staged into a per-warp shared-memory ring
//    with cp.async using a fixed lane -> (row, 16-byte piece) map (no index
//    division), rows padded so fragment reads are bank-conflict free; the 32-byte
//    record (3 short-circuit suffixes + |c|^2) rides along;
//  * short-circuit at up to 3 check points: a tile stops when every entry's
//    partial distance (acc - candidate suffix + query prefix) exceeds
//    eps^2 + 2*guard — safe under rounding, decisions stay exact.  The check costs
//    FP64 issue slots, so a warp turns it off for the rest of an item when fewer
//    than a quarter of its first checks prune;
//  * exact decisions: guard band as in refine_lowd.cu (integer high-word screen,
//    rare out-of-line direct-form recheck);
//  * emission: hits are sparse at these dimensionalities (|R|/C ~ 1e-3), so
//    pairs go through a per-warp shared-memory buffer flushed with one atomicAdd
//    per 256 pairs; per-query counts accumulate in registers and are added once
//    per item (items of a big cell share queries).
#include "internal.cuh"
#include "refine_common.cuh"

namespace tj {

constexpr int kTcWarps = 4;
constexpr int kTcThreads = kTcWarps * kWarp;
constexpr int kTcStages = 4;  // blocks in the per-warp ring

template <int NCH>
struct TcShape {
  static constexpr int DP = 4 * NCH;
  static constexpr int STRIDE = (DP % 8 == 0) ? DP + 4 : DP;  // conflict-free fragment rows
  static constexpr int NGM = NCH <= 8 ? 2 : 1;                 // query groups per item
  static constexpr int CE = (NCH + 3) / 4;                     // chunks per check interval
  static constexpr int NCHECK = (NCH - 1) / CE;                // check points (<= 3)
  static constexpr int PPR = DP / 2;                           // 16-byte pieces per row
};

template <int NCH>
struct alignas(16) TcBlock {
  double pts[8][TcShape<NCH>::STRIDE];
  double rec[8][4];  // suffixes after check points 0..2, |c|^2
  uint32_t pos;      // position of row 0
  uint32_t pad[3];
};

__device__ __forceinline__ unsigned tc_hi_word(double v) { return unsigned(__double2hiint(v)); }

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
                                         bool b1, bool p0, bool p1, uint32_t qa, uint32_t c,
                                         unsigned long long* ctr) {
  if (b0) p0 = direct_form_le(P, dp, d, qa, c, eps_sq);
  if (b1) p1 = direct_form_le(P, dp, d, qa + 1, c, eps_sq);
  const unsigned nb = __popc(__ballot_sync(0xffffffffu, b0)) + __popc(__ballot_sync(0xffffffffu, b1));
  if (lane_id() == 0) atomicAdd(ctr, (unsigned long long)nb);
  return make_uint2(__ballot_sync(0xffffffffu, p0), __ballot_sync(0xffffffffu, p1));
}

// Warp-uniform walk over the item's runs clipped to [s0, s1) of the
// concatenated candidate list, one 8-candidate block at a time.
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

template <int NCH>
__global__ void __launch_bounds__(kTcThreads, 4) refine_tc_kernel(RefineArgs a) {
  using S = TcShape<NCH>;
  constexpr int DP = S::DP, NGM = S::NGM, CE = S::CE, NCHECK = S::NCHECK, PPR = S::PPR;
  constexpr int R = kTcStages;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5;
  const int lane = lane_id();
  const int row = lane >> 2, col = lane & 3;
  const unsigned lt = lanemask_lt();
  TcBlock<NCH>* ring = reinterpret_cast<TcBlock<NCH>*>(smem_raw) + warp * R;
  uint2* hits = reinterpret_cast<uint2*>(reinterpret_cast<TcBlock<NCH>*>(smem_raw) + kTcWarps * R) +
                warp * kHitBuf;
  HitBuffer hb;
  unsigned long long st_tiles_ref = 0, st_tiles = 0, st_skip = 0;
  const double eps_sq = a.eps_sq;

  for (;;) {
    unsigned long long idx = 0;
    if (lane == 0) idx = atomicAdd(&a.ctr->item_next, 1ull);
    idx = __shfl_sync(0xffffffffu, idx, 0);
    if (idx >= (unsigned long long)a.n_items) break;
    const WorkItem it = a.items[idx];
    const int nq = int(it.nq);
    const int ng = (nq + 7) >> 3;

    // ---- query side
    double bq[NGM][NCH];
    double thr[NGM][2];
    unsigned h1[NGM][2], hw[NGM][2];
    double qpre[NGM][NCHECK > 0 ? NCHECK : 1][2];
#pragma unroll
    for (int g = 0; g < NGM; ++g) {
      const int qb = 8 * g + row;
      const bool vb = qb < nq;
#pragma unroll
      for (int j = 0; j < NCH; ++j)
        bq[g][j] = vb ? -2.0 * a.P[size_t(it.q0 + qb) * DP + 4 * j + col] : 0.0;
#pragma unroll
      for (int jj = 0; jj < 2; ++jj) {
        const int q = 8 * g + 2 * col + jj;
        const bool v = q < nq;
        const size_t qp = size_t(it.q0) + (v ? q : 0);
        const double qn = v ? a.NRM[qp] : 0.0;
        const double guard = a.guard_rel * (qn + a.max_norm) + 1e-300;
        const double center = eps_sq - qn;
        const double hi = center + guard, lo = center - guard;
        thr[g][jj] = v ? hi : -INFINITY;
        if (!v) {
          h1[g][jj] = 0u;
          hw[g][jj] = 0u;
        } else if ((hi < 0.0) == (lo < 0.0) && lo != 0.0 && hi != 0.0) {
          const unsigned a1 = tc_hi_word(hi), a2 = tc_hi_word(lo);
          h1[g][jj] = min(a1, a2);
          hw[g][jj] = max(a1, a2) - min(a1, a2);
        } else {
          h1[g][jj] = 0u;
          hw[g][jj] = 0xffffffffu;
        }
        // eps^2 + 2*guard - (query chunk norms up to each check point)
#pragma unroll
        for (int c = 0; c < NCHECK; ++c) {
          double pre = 0.0;
          for (int j = 0; j < (c + 1) * CE; ++j) pre += v ? a.CN[qp * NCH + j] : 0.0;
          qpre[g][c][jj] = v ? eps_sq + 2.0 * guard - pre : -INFINITY;
        }
      }
    }
    unsigned qc[NGM][2];
#pragma unroll
    for (int g = 0; g < NGM; ++g) qc[g][0] = qc[g][1] = 0;
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
    // stage one block into slot s: lane -> (row, piece) fixed map
    auto issue = [&](TcBlock<NCH>* blk) -> bool {
      uint32_t pos = 0, valid = 0;
      const bool any = cur.next(pos, valid, a);
      constexpr int RPI = 32 / PPR > 0 ? 32 / PPR : 1;  // rows per pass
#pragma unroll
      for (int r0 = 0; r0 < 8; r0 += (PPR >= 32 ? 1 : RPI)) {
#pragma unroll
        for (int p0 = 0; p0 < PPR; p0 += 32) {
          const int rr = r0 + (PPR >= 32 ? 0 : lane / PPR);
          const int pc = p0 + (PPR >= 32 ? lane : lane % PPR);
          if (rr < 8 && pc < PPR) {
            if (uint32_t(rr) < valid)
              tc_cp16(&blk->pts[rr][2 * pc], a.P + size_t(pos + rr) * DP + 2 * pc);
            else
              *reinterpret_cast<double2*>(&blk->pts[rr][2 * pc]) = make_double2(0.0, 0.0);
          }
        }
      }
      if (lane < 16) {  // 8 records x 2 pieces
        const int rr = lane >> 1, pc = lane & 1;
        if (uint32_t(rr) < valid)
          tc_cp16(&blk->rec[rr][2 * pc], a.SFX + size_t(pos + rr) * 4 + 2 * pc);
        else
          *reinterpret_cast<double2*>(&blk->rec[rr][2 * pc]) =
              make_double2(pc ? 0.0 : 0.0, pc ? kPadNorm : 0.0);
      }
      if (lane == 0) blk->pos = pos;
      tc_commit();
      return any;
    };
    int nstaged = 0;
#pragma unroll
    for (int k = 0; k < R - 1; ++k) nstaged += issue(ring + k) ? 1 : 0;
    // adaptive short-circuit: keep checking while at least 1/4 of checks prune
    bool check = a.short_circuit != 0;
    unsigned n_checks = 0, n_pruned = 0;
#pragma unroll 1
    for (int b = 0; b < nstaged; ++b) {
      tc_wait<R - 2>();
      __syncwarp();
      const TcBlock<NCH>* s = ring + (b % R);
      const double cn = s->rec[row][3];
      const uint32_t cpos = s->pos + uint32_t(row);
#pragma unroll
      for (int g = 0; g < NGM; ++g) {
        if (g >= ng) break;
        double d0 = cn, d1 = cn;
        bool pruned = false;
#pragma unroll
        for (int j = 0; j < NCH; ++j) {
          dmma_8x8x4(d0, d1, s->pts[row][4 * j + col], bq[g][j], d0, d1);
          if constexpr (NCHECK > 0) {
            if ((j + 1) % CE == 0 && (j + 1) / CE <= NCHECK && check) {
              const int c = (j + 1) / CE - 1;
              const double sf = s->rec[row][c];
              const bool far = (d0 - sf > qpre[g][c][0]) && (d1 - sf > qpre[g][c][1]);
              ++n_checks;
              if (__all_sync(0xffffffffu, far)) {
                st_skip += NCH - (j + 1);
                ++n_pruned;
                pruned = true;
                break;
              }
            }
          }
        }
        ++st_tiles;
        if (pruned) continue;
        bool p0 = d0 <= thr[g][0];
        bool p1 = d1 <= thr[g][1];
        unsigned m0 = __ballot_sync(0xffffffffu, p0);
        unsigned m1 = __ballot_sync(0xffffffffu, p1);
        if ((m0 | m1) == 0) continue;
        const bool b0 = p0 && (tc_hi_word(d0) - h1[g][0]) <= hw[g][0];
        const bool b1 = p1 && (tc_hi_word(d1) - h1[g][1]) <= hw[g][1];
        const uint32_t qa = it.q0 + 8 * g + 2 * col;
        if (__any_sync(0xffffffffu, b0 || b1)) {
          const uint2 m = tc_recheck(a.P, DP, a.d, eps_sq, b0, b1, p0, p1, qa, cpos,
                                     &a.ctr->rechecks);
          m0 = m.x;
          m1 = m.y;
          p0 = (m0 >> lane) & 1u;
          p1 = (m1 >> lane) & 1u;
          if ((m0 | m1) == 0) continue;
        }
        const int n0 = __popc(m0), n1 = __popc(m1);
        hb.reserve(n0 + n1, hits, a);
        if (p0) hits[hb.count + __popc(m0 & lt)] = make_uint2(qa, cpos);
        if (p1) hits[hb.count + n0 + __popc(m1 & lt)] = make_uint2(qa + 1, cpos);
        hb.count += n0 + n1;
        qc[g][0] += p0;
        qc[g][1] += p1;
      }
      if (check && n_checks >= 64 && 4 * n_pruned < n_checks) check = false;
      __syncwarp();
      nstaged += issue(ring + ((b + R - 1) % R)) ? 1 : 0;
    }
    tc_wait<0>();
    // per-query counts (items of one cell may share queries: atomic add)
#pragma unroll
    for (int g = 0; g < NGM; ++g) {
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

int tc_queries_per_item(int d_pad) { return d_pad / 4 <= 8 ? 16 : 8; }

template <int NCH>
static void launch_tc_t(const RefineArgs& a, cudaStream_t s) {
  const size_t smem = sizeof(TcBlock<NCH>) * kTcWarps * kTcStages + sizeof(uint2) * kTcWarps * kHitBuf;
  auto kern = refine_tc_kernel<NCH>;
  TJ_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  int per_sm = 0;
  TJ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kTcThreads, smem));
  per_sm = std::max(per_sm, 1);
  const int64_t grid = std::min<int64_t>(ceil_div(a.n_items, kTcWarps), int64_t(kNumSMs) * per_sm);
  kern<<<unsigned(std::max<int64_t>(grid, 1)), kTcThreads, smem, s>>>(a);
  TJ_CHECK_LAUNCH();
}

void launch_refine_tc(const RefineArgs& a, cudaStream_t s) {
  switch (a.nchunks) {
    case 2: return launch_tc_t<2>(a, s);
    case 3: return launch_tc_t<3>(a, s);
    case 4: return launch_tc_t<4>(a, s);
    case 5: return launch_tc_t<5>(a, s);
    case 6: return launch_tc_t<6>(a, s);
    case 7: return launch_tc_t<7>(a, s);
    case 8: return launch_tc_t<8>(a, s);
    case 9: return launch_tc_t<9>(a, s);
    case 10: return launch_tc_t<10>(a, s);
    case 11: return launch_tc_t<11>(a, s);
    case 12: return launch_tc_t<12>(a, s);
    case 13: return launch_tc_t<13>(a, s);
    case 14: return launch_tc_t<14>(a, s);
    case 15: return launch_tc_t<15>(a, s);
    case 16: return launch_tc_t<16>(a, s);
    default: break;
  }
  fail(TJ_EINVAL, "DMMA refine is instantiated for 5 <= d <= 64, got d=" + std::to_string(a.d));
}

}  // namespace tj
