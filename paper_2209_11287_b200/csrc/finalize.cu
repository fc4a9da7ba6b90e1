// Canonical output: CSR by original query id with neighbour ids ascending.
//
// Replaces the concatenate + np.lexsort((j, i)) of join.py:203-204.  Per-query
// pair counts (cell-ordered positions) move to original-id order and are
// scanned into int64 row offsets.  Then:
//  * low-d path (row segments, refine_lowd.cu): one warp per query gathers its
//    segment chain, maps candidate positions to original ids, sorts the row in
//    registers (bitonic network) and writes it to its final place;
//  * pair path (other kernels): every (query, candidate) pair is scattered to
//    its row through a per-row atomic cursor, then each row is sorted in place.
// Rows longer than 256 ids are sorted by one CTA (shared-memory bitonic, <= 8192)
// or, beyond that, by a composite-key radix sort.
#include "internal.cuh"
#include "scan.cuh"

namespace tj {

__global__ void counts_to_orig_kernel(const uint32_t* __restrict__ qcount,
                                      const uint32_t* __restrict__ perm, int64_t n,
                                      int64_t* __restrict__ cnt_orig) {
  for (int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p < n;
       p += int64_t(gridDim.x) * blockDim.x)
    cnt_orig[perm[p]] = qcount[p];
}

__global__ void scatter_pairs_kernel(const uint2* __restrict__ pairs, int64_t total,
                                     const uint32_t* __restrict__ perm,
                                     const int64_t* __restrict__ offsets,
                                     uint32_t* __restrict__ fill, uint32_t* __restrict__ nbr) {
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const uint2 pr = pairs[e];
    const uint32_t row = perm[pr.x];
    const uint32_t slot = atomicAdd(&fill[row], 1u);
    nbr[offsets[row] + slot] = perm[pr.y];
  }
}

// Bitonic sort of 32*R keys held as v[r] (element index r*32 + lane), ascending.
template <int R>
__device__ __forceinline__ void warp_bitonic(uint32_t (&v)[R]) {
  const int lane = lane_id();
  constexpr int N = 32 * R;
#pragma unroll
  for (int k = 2; k <= N; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j >= 32) {
        const int rj = j >> 5;
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int p = r ^ rj;
          if (p > r) {
            const int i = r * 32 + lane;
            const bool asc = (i & k) == 0;
            const uint32_t a = v[r], b = v[p];
            const bool swap = asc ? (a > b) : (a < b);
            v[r] = swap ? b : a;
            v[p] = swap ? a : b;
          }
        }
      } else {
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int i = r * 32 + lane;
          const bool asc = (i & k) == 0;
          const uint32_t o = __shfl_xor_sync(0xffffffffu, v[r], j);
          const bool lower = (lane & j) == 0;
          // lower element keeps min when ascending, max when descending
          const uint32_t mn = min(v[r], o), mx = max(v[r], o);
          v[r] = (lower == asc) ? mn : mx;
        }
      }
    }
  }
}

template <int R>
__device__ __forceinline__ void warp_sort_row(uint32_t* row, int len) {
  uint32_t v[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int i = r * 32 + lane_id();
    v[r] = i < len ? row[i] : 0xffffffffu;
  }
  warp_bitonic<R>(v);
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int i = r * 32 + lane_id();
    if (i < len) row[i] = v[r];
  }
}

constexpr int kWarpSortMax = 256;
constexpr int kBlockSortMax = 8192;

__global__ void sort_rows_warp_kernel(const int64_t* __restrict__ offsets, int64_t n,
                                      uint32_t* __restrict__ nbr, uint32_t* __restrict__ big_rows,
                                      unsigned long long* n_big) {
  const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
  for (int64_t i = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5; i < n; i += warps) {
    const int64_t b = offsets[i];
    const int64_t len = offsets[i + 1] - b;
    if (len <= 1) continue;
    uint32_t* row = nbr + b;
    if (len <= 32) warp_sort_row<1>(row, int(len));
    else if (len <= 64) warp_sort_row<2>(row, int(len));
    else if (len <= 128) warp_sort_row<4>(row, int(len));
    else if (len <= kWarpSortMax) warp_sort_row<8>(row, int(len));
    else if (lane_id() == 0) big_rows[atomicAdd(n_big, 1ull)] = uint32_t(i);
  }
}

// Low-d hit masks -> rows.  Warp per cell: the cell's candidate runs are
// re-flattened into 8-candidate blocks exactly as the refine kernel tiled them;
// lane j owns query j of the current 32-query slice, walks the blocks, extracts
// its column of each tile mask (bit 4r + (c>>1) of the low / high word for even /
// odd column c) and writes the original ids of its hits to its final row; then
// the warp sorts the slice's rows (bitonic in registers, long rows deferred).
// Rows of the slice are built in a per-warp shared-memory pool and sorted from
// there (one coalesced store per row); masks and the original ids of each
// block's candidates are staged in shared memory first, so the per-hit work is
// shared-memory only.
constexpr int kExpandBlk = 64;  // blocks staged per chunk
constexpr int kExpandPool = 1536;
constexpr int kExpandWarps = 4;

template <int R>
__device__ __forceinline__ void sort_store_row(const uint32_t* src, int len, uint32_t* dst) {
  uint32_t v[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int i = r * 32 + lane_id();
    v[r] = i < len ? src[i] : 0xffffffffu;
  }
  warp_bitonic<R>(v);
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int i = r * 32 + lane_id();
    if (i < len) dst[i] = v[r];
  }
}

__global__ void __launch_bounds__(kExpandWarps * 32)
    expand_masks_kernel(const unsigned long long* __restrict__ masks,
                        const int64_t* __restrict__ cell_mbase,
                        const int64_t* __restrict__ cell_start,
                        const int64_t* __restrict__ cell_runs, const uint2* __restrict__ runs,
                        int64_t n_cells, const uint32_t* __restrict__ qcount,
                        const uint32_t* __restrict__ perm, const int64_t* __restrict__ offsets,
                        uint32_t* __restrict__ nbr, uint32_t* __restrict__ big_rows,
                        unsigned long long* n_big, uint32_t n_points) {
  __shared__ uint32_t s_pos[kExpandWarps][kExpandBlk];
  __shared__ uint32_t s_ids[kExpandWarps][kExpandBlk * 8];
  __shared__ unsigned long long s_msk[kExpandWarps][kExpandBlk * 4];
  __shared__ uint32_t s_pool[kExpandWarps][kExpandPool];
  const int warp = threadIdx.x >> 5, lane = lane_id();
  uint32_t* bpos = s_pos[warp];
  uint32_t* bids = s_ids[warp];
  unsigned long long* bmsk = s_msk[warp];
  uint32_t* pool = s_pool[warp];
  const int64_t stride = int64_t(gridDim.x) * kExpandWarps;
  for (int64_t c = int64_t(blockIdx.x) * kExpandWarps + warp; c < n_cells; c += stride) {
    const int64_t cs = cell_start[c];
    const int nq = int(cell_start[c + 1] - cs);
    if (qcount[cs] == 0) continue;  // cell not refined in this result set
    const int ngc = (nq + 7) >> 3;
    // flatten the runs (<= 27 for k <= 4) into blocks
    const int64_t rb = cell_runs[c], re = cell_runs[c + 1];
    const int nr = int(re - rb);
    uint2 myrun = make_uint2(0u, 0u);
    if (lane < nr) myrun = runs[rb + lane];
    const int mynblk = int(myrun.y - myrun.x + 7) >> 3;
    int incl = mynblk;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    const int myfirst = incl - mynblk;
    const unsigned long long* mb = masks + cell_mbase[c];
    for (int q0 = 0; q0 < nq; q0 += 32) {
      const int j = q0 + lane;  // query index within the cell
      const bool active = j < nq;
      const int cnt = active ? int(qcount[cs + j]) : 0;
      int ci = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, ci, o);
        if (lane >= o) ci += t;
      }
      const int poff = ci - cnt;
      const bool pooled = poff + cnt <= kExpandPool;  // otherwise straight to the final row
      const uint32_t qrow = active ? perm[cs + j] : 0u;
      uint32_t* dst = nbr + (active ? offsets[qrow] : 0);
      const int gs = q0 >> 3;                    // first group of the slice
      const int ngs = min(4, ngc - gs);          // groups in the slice
      const int gl = lane >> 3, col = lane & 7;  // my group within the slice, my column
      const unsigned word = col & 1, sh = col >> 1;
      int o = 0;
      for (int b0 = 0; b0 < total; b0 += kExpandBlk) {
        const int nb = min(kExpandBlk, total - b0);
        __syncwarp();
        {
          const int lo = max(myfirst, b0), hi = min(myfirst + mynblk, b0 + nb);
          for (int b = lo; b < hi; ++b) bpos[b - b0] = myrun.x + 8u * uint32_t(b - myfirst);
        }
        __syncwarp();
        // original ids of the blocks' candidates and the slice's masks (coalesced)
        for (int i = lane; i < nb * 8; i += 32) {
          const int b = i >> 3;
          const uint32_t p = bpos[b] + uint32_t(i & 7);
          bids[i] = p < n_points ? __ldg(perm + p) : 0u;  // rows past a run end: never hit
        }
        for (int i = lane; i < nb * 4; i += 32) {
          const int b = i >> 2, g = i & 3;
          bmsk[i] = g < ngs ? __ldg(mb + size_t(b0 + b) * ngc + gs + g) : 0ull;
        }
        __syncwarp();
        if (active) {
          for (int b = 0; b < nb; ++b) {
            unsigned bits =
                (unsigned(bmsk[4 * b + gl] >> (32 * word)) >> sh) & 0x11111111u;
            while (bits) {
              const int r = (__ffs(bits) - 1) >> 2;
              bits &= bits - 1;
              const uint32_t v = bids[8 * b + r];
              if (pooled) pool[poff + o] = v;
              else dst[o] = v;
              ++o;
            }
          }
        }
      }
      __syncwarp();
      // sort the slice's rows and store them
      const int nrows = min(32, nq - q0);
      for (int k = 0; k < nrows; ++k) {
        const int len = __shfl_sync(0xffffffffu, cnt, k);
        const int off = __shfl_sync(0xffffffffu, poff, k);
        const bool pk = __shfl_sync(0xffffffffu, pooled ? 1 : 0, k) != 0;
        const uint32_t rrow = __shfl_sync(0xffffffffu, qrow, k);
        uint32_t* row = nbr + offsets[rrow];
        if (pk && len <= kWarpSortMax) {
          if (len <= 32) sort_store_row<1>(pool + off, len, row);
          else if (len <= 64) sort_store_row<2>(pool + off, len, row);
          else if (len <= 128) sort_store_row<4>(pool + off, len, row);
          else sort_store_row<8>(pool + off, len, row);
        } else if (pk) {  // long pooled row: copy out, the CTA / radix path sorts it
          for (int i = lane; i < len; i += 32) row[i] = pool[off + i];
          if (lane == 0) big_rows[atomicAdd(n_big, 1ull)] = rrow;
        } else if (len > 1) {  // written in place
          if (len <= kWarpSortMax) {
            if (len <= 32) warp_sort_row<1>(row, len);
            else if (len <= 64) warp_sort_row<2>(row, len);
            else if (len <= 128) warp_sort_row<4>(row, len);
            else warp_sort_row<8>(row, len);
          } else if (lane == 0) {
            big_rows[atomicAdd(n_big, 1ull)] = rrow;
          }
        }
      }
      __syncwarp();
    }
  }
}

// One CTA per listed row of 257..8192 ids: shared-memory bitonic sort.
__global__ void __launch_bounds__(1024)
    sort_rows_block_kernel(const int64_t* __restrict__ offsets, uint32_t* __restrict__ nbr,
                           const uint32_t* __restrict__ rows, const unsigned long long* n_rows,
                           uint32_t* __restrict__ huge_rows, unsigned long long* n_huge) {
  __shared__ uint32_t s[kBlockSortMax];
  for (unsigned long long ri = blockIdx.x; ri < *n_rows; ri += gridDim.x) {
    const uint32_t i = rows[ri];
    const int64_t b = offsets[i];
    const int64_t len = offsets[i + 1] - b;
    if (len > kBlockSortMax) {
      if (threadIdx.x == 0) huge_rows[atomicAdd(n_huge, 1ull)] = i;
      continue;
    }
    int N = 512;
    while (N < len) N <<= 1;
    __syncthreads();
    for (int t = threadIdx.x; t < N; t += blockDim.x) s[t] = t < len ? nbr[b + t] : 0xffffffffu;
    __syncthreads();
    for (int k = 2; k <= N; k <<= 1) {
      for (int j = k >> 1; j > 0; j >>= 1) {
        for (int t = threadIdx.x; t < N; t += blockDim.x) {
          const int p = t ^ j;
          if (p > t) {
            const bool asc = (t & k) == 0;
            const uint32_t x = s[t], y = s[p];
            if (asc ? (x > y) : (x < y)) {
              s[t] = y;
              s[p] = x;
            }
          }
        }
        __syncthreads();
      }
    }
    for (int t = threadIdx.x; t < len; t += blockDim.x) nbr[b + t] = s[t];
  }
}

// Rows longer than kBlockSortMax: gather (row rank << 32 | id) keys, radix sort, scatter back.
__global__ void huge_gather_kernel(const int64_t* __restrict__ offsets, const uint32_t* nbr,
                                   const uint32_t* __restrict__ huge, int n_huge,
                                   const int64_t* __restrict__ base, uint64_t* __restrict__ keys) {
  for (int h = blockIdx.y; h < n_huge; h += gridDim.y) {
    const int64_t b = offsets[huge[h]];
    const int64_t len = offsets[huge[h] + 1] - b;
    for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < len;
         t += int64_t(gridDim.x) * blockDim.x)
      keys[base[h] + t] = (uint64_t(h) << 32) | nbr[b + t];
  }
}
__global__ void huge_scatter_kernel(const int64_t* __restrict__ offsets, uint32_t* nbr,
                                    const uint32_t* __restrict__ huge, int n_huge,
                                    const int64_t* __restrict__ base,
                                    const uint64_t* __restrict__ keys) {
  for (int h = blockIdx.y; h < n_huge; h += gridDim.y) {
    const int64_t b = offsets[huge[h]];
    const int64_t len = offsets[huge[h] + 1] - b;
    for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < len;
         t += int64_t(gridDim.x) * blockDim.x)
      nbr[b + t] = uint32_t(keys[base[h] + t]);
  }
}

static unsigned blocks_for(int64_t n, int threads) {
  return unsigned(std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, threads), kNumSMs * 16)));
}

// Sort the rows listed in big_rows (> kWarpSortMax ids) in place.
static void sort_big_rows(tj_ctx* ctx, int64_t* offsets, uint32_t* nbr, uint32_t* big_rows,
                          unsigned long long* nbig, cudaStream_t s) {
  const int64_t n = ctx->g.n;
  unsigned long long h_nbig = 0;
  TJ_CUDA(cudaMemcpyAsync(&h_nbig, nbig, sizeof(h_nbig), cudaMemcpyDeviceToHost, s));
  TJ_CUDA(cudaStreamSynchronize(s));
  if (h_nbig == 0) return;
  ctx->vals_alt.ensure(sizeof(uint32_t) * h_nbig, s);
  uint32_t* huge = ctx->vals_alt.as<uint32_t>();
  sort_rows_block_kernel<<<unsigned(std::min<unsigned long long>(h_nbig, kNumSMs * 4)), 1024, 0,
                           s>>>(offsets, nbr, big_rows, nbig, huge, nbig + 1);
  TJ_CHECK_LAUNCH();
  unsigned long long h_nhuge = 0;
  TJ_CUDA(cudaMemcpyAsync(&h_nhuge, nbig + 1, sizeof(h_nhuge), cudaMemcpyDeviceToHost, s));
  TJ_CUDA(cudaStreamSynchronize(s));
  if (h_nhuge == 0) return;

  // composite-key radix sort over all huge rows together
  std::vector<uint32_t> hh(h_nhuge);
  TJ_CUDA(cudaMemcpyAsync(hh.data(), huge, sizeof(uint32_t) * h_nhuge, cudaMemcpyDeviceToHost, s));
  TJ_CUDA(cudaStreamSynchronize(s));
  std::vector<int64_t> hbase(h_nhuge + 1, 0);
  for (size_t h = 0; h < hh.size(); ++h) {
    int64_t se[2];
    TJ_CUDA(cudaMemcpy(se, offsets + hh[h], 2 * sizeof(int64_t), cudaMemcpyDeviceToHost));
    hbase[h + 1] = hbase[h] + (se[1] - se[0]);
  }
  const int64_t m = hbase[h_nhuge];
  DevBuf kb, kb2, vb, vb2, bb, hb;
  kb.ensure(sizeof(uint64_t) * m, s);
  kb2.ensure(sizeof(uint64_t) * m, s);
  vb.ensure(sizeof(uint32_t) * m, s);
  vb2.ensure(sizeof(uint32_t) * m, s);
  bb.ensure(sizeof(int64_t) * (h_nhuge + 1), s);
  TJ_CUDA(cudaMemcpyAsync(bb.ptr, hbase.data(), sizeof(int64_t) * (h_nhuge + 1),
                          cudaMemcpyHostToDevice, s));
  dim3 g(unsigned(std::min<int64_t>(ceil_div(m, 256), 1024)),
         unsigned(std::min<unsigned long long>(h_nhuge, 65535)));
  huge_gather_kernel<<<g, 256, 0, s>>>(offsets, nbr, huge, int(h_nhuge), bb.as<int64_t>(),
                                       kb.as<uint64_t>());
  TJ_CHECK_LAUNCH();
  int hbits = 0;
  while ((1ull << hbits) < h_nhuge) ++hbits;
  hb.ensure(sizeof(int64_t) * radix_sort_scratch_elems(m), s);
  ScanScratch sc2 = scan_scratch(ctx, std::max<int64_t>(radix_sort_scratch_elems(m), n), s);
  const int where = radix_sort_pairs(kb.as<uint64_t>(), vb.as<uint32_t>(), kb2.as<uint64_t>(),
                                     vb2.as<uint32_t>(), m, 32 + hbits, true, hb.as<int64_t>(),
                                     sc2, s);
  huge_scatter_kernel<<<g, 256, 0, s>>>(offsets, nbr, huge, int(h_nhuge), bb.as<int64_t>(),
                                        where ? kb2.as<uint64_t>() : kb.as<uint64_t>());
  TJ_CHECK_LAUNCH();
  TJ_CUDA(cudaStreamSynchronize(s));
  kb.release(s);
  kb2.release(s);
  vb.release(s);
  vb2.release(s);
  bb.release(s);
  hb.release(s);
}

void finalize_csr(tj_ctx* ctx, int64_t* offsets, uint32_t* nbr, int64_t n_pairs,
                  int64_t n_mask_hits, cudaStream_t s) {
  const int64_t n = ctx->g.n;
  ctx->tmp64.ensure(sizeof(int64_t) * (n + 1), s);
  int64_t* cnt = ctx->tmp64.as<int64_t>();
  counts_to_orig_kernel<<<blocks_for(n, 256), 256, 0, s>>>(ctx->qcount.as<uint32_t>(),
                                                          ctx->perm.as<uint32_t>(), n, cnt);
  TJ_CHECK_LAUNCH();
  ScanScratch sc = scan_scratch(ctx, n, s);
  scan_exclusive(LoadAt<int64_t>{cnt}, StoreAt<int64_t>{offsets}, n, sc, s);
  TJ_CUDA(cudaMemcpyAsync(offsets + n, sc.total, sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
  if (n_pairs == 0 && n_mask_hits == 0) return;

  ctx->fill.ensure(sizeof(uint32_t) * n + 4 * sizeof(unsigned long long), s);
  uint32_t* fill = ctx->fill.as<uint32_t>();
  unsigned long long* nbig = reinterpret_cast<unsigned long long*>(ctx->minmax.as<long long>());
  TJ_CUDA(cudaMemsetAsync(nbig, 0, 2 * sizeof(unsigned long long), s));
  if (n_mask_hits > 0) {
    const int64_t nc = ctx->g.n_cells;
    expand_masks_kernel<<<unsigned(std::min<int64_t>(ceil_div(nc, 4), kNumSMs * 64)), 128, 0, s>>>(
        ctx->masks.as<unsigned long long>(), ctx->cell_mbase.as<int64_t>(),
        ctx->cell_start.as<int64_t>(), ctx->cell_runs.as<int64_t>(), ctx->runs.as<uint2>(), nc,
        ctx->qcount.as<uint32_t>(), ctx->perm.as<uint32_t>(), offsets, nbr, fill, nbig,
        uint32_t(n));
    TJ_CHECK_LAUNCH();
  } else {
    TJ_CUDA(cudaMemsetAsync(fill, 0, sizeof(uint32_t) * n, s));
    scatter_pairs_kernel<<<blocks_for(n_pairs, 256), 256, 0, s>>>(
        ctx->pairs.as<uint2>(), n_pairs, ctx->perm.as<uint32_t>(), offsets, fill, nbr);
    TJ_CHECK_LAUNCH();
    // `fill` becomes the list of long rows once the scatter is done (same stream)
    sort_rows_warp_kernel<<<blocks_for(n * 32, 256), 256, 0, s>>>(offsets, n, nbr, fill, nbig);
    TJ_CHECK_LAUNCH();
  }
  sort_big_rows(ctx, offsets, nbr, fill, nbig, s);
}

}  // namespace tj
