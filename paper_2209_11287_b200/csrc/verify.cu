// GPU brute-force self-join: the verification oracle for inputs beyond the
// reference's CPU guard (oracle.brute_force_join, oracle.py:55-86, refuses
// n > 50,000 without --force; cli.cmd_verify, cli.py:165-192).
//
// Every ordered pair (i, j) is decided by the reference direct form
// acc = fl(acc + fl(fl(x_i - x_j)^2)) over ascending dims (oracle.py:78-81)
// with __d*_rn intrinsics, so the result is the reference pair set exactly,
// with no grid involved -- an independent check of the indexed join.
// Layout: CTA = 8 warps = 8 query rows; candidate rows are staged through
// shared memory in tiles shared by the 8 warps; a warp's lanes take 32
// consecutive candidates, so a ballot gives each hit its rank and rows come
// out ascending.  Two launches: count (offsets) and fill.
#include "internal.cuh"
#include "scan.cuh"

namespace tj {

constexpr int kBfWarps = 8;
constexpr int kBfSmemDoubles = 4096;  // 32 KB candidate tile

__global__ void __launch_bounds__(kBfWarps * 32)
    brute_force_kernel(const double* __restrict__ x, int64_t n, int d, int64_t ld, double eps_sq,
                       int64_t* __restrict__ counts, const int64_t* __restrict__ offsets,
                       uint32_t* __restrict__ nbr) {
  __shared__ double s_c[kBfSmemDoubles];
  extern __shared__ double s_q[];  // kBfWarps * d
  const int warp = threadIdx.x >> 5, lane = lane_id();
  const unsigned lt = lanemask_lt();
  const int tile = kBfSmemDoubles / d;  // candidate rows per tile
  for (int64_t q0 = int64_t(blockIdx.x) * kBfWarps; q0 < n; q0 += int64_t(gridDim.x) * kBfWarps) {
    const int64_t q = q0 + warp;
    __syncthreads();
    for (int i = threadIdx.x; i < kBfWarps * d; i += blockDim.x) {
      const int64_t r = q0 + i / d;
      s_q[i] = r < n ? x[r * ld + (i % d)] : 0.0;
    }
    int64_t cnt = 0;
    int64_t out = (nbr && q < n) ? offsets[q] : 0;
    for (int64_t c0 = 0; c0 < n; c0 += tile) {
      const int rows = int(min(int64_t(tile), n - c0));
      __syncthreads();
      for (int i = threadIdx.x; i < rows * d; i += blockDim.x)
        s_c[i] = x[(c0 + i / d) * ld + (i % d)];
      __syncthreads();
      if (q >= n) continue;
      const double* qr = s_q + warp * d;
      for (int j0 = 0; j0 < rows; j0 += 32) {
        const int j = j0 + lane;
        bool hit = false;
        if (j < rows) {
          const double* cr = s_c + j * d;
          double acc = 0.0;
          for (int k = 0; k < d; ++k) {
            const double t = __dsub_rn(qr[k], cr[k]);
            acc = __dadd_rn(acc, __dmul_rn(t, t));
          }
          hit = acc <= eps_sq;
        }
        const unsigned bal = __ballot_sync(0xffffffffu, hit);
        if (nbr && hit) nbr[out + __popc(bal & lt)] = uint32_t(c0 + j);
        out += __popc(bal);
        cnt += __popc(bal);
      }
    }
    if (!nbr && q < n && lane == 0) counts[q] = cnt;
  }
}

void brute_force_join(tj_ctx* ctx, const double* x, int64_t n, int d, int64_t ld, double eps,
                      int64_t* offsets, uint32_t* nbr, int64_t* total, cudaStream_t s) {
  if (d > kBfSmemDoubles / 32) fail(TJ_EINVAL, "brute force supports d <= 128");
  const double eps_sq = eps * eps;
  const size_t qsm = sizeof(double) * kBfWarps * d;
  const unsigned grid =
      unsigned(std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, kBfWarps), int64_t(kNumSMs) * 8)));
  if (!nbr) {
    ctx->tmp64.ensure(sizeof(int64_t) * (n + 1), s);
    int64_t* cnt = ctx->tmp64.as<int64_t>();
    brute_force_kernel<<<grid, kBfWarps * 32, qsm, s>>>(x, n, d, ld, eps_sq, cnt, nullptr, nullptr);
    TJ_CHECK_LAUNCH();
    ScanScratch sc = scan_scratch(ctx, n, s);
    scan_exclusive(LoadAt<int64_t>{cnt}, StoreAt<int64_t>{offsets}, n, sc, s);
    TJ_CUDA(cudaMemcpyAsync(offsets + n, sc.total, sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
    TJ_CUDA(cudaMemcpyAsync(total, sc.total, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    TJ_CUDA(cudaStreamSynchronize(s));
  } else {
    brute_force_kernel<<<grid, kBfWarps * 32, qsm, s>>>(x, n, d, ld, eps_sq, nullptr, offsets, nbr);
    TJ_CHECK_LAUNCH();
  }
}

}  // namespace tj
