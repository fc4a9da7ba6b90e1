// Variance dimension reordering on device (datasets.reorder_dims_by_variance,
// datasets.py:113-123; invoked by self_join at join.py:163-164).
//
// The reference permutes columns by np.argsort(-var, kind="stable") with
// var = x.var(axis=0).  Only the ORDER of the variances matters, so the
// device computes every column's mean and variance with compensated (two-sum)
// accumulation -- a deterministic value accurate to a few ulp -- and the host
// argsorts them; when two variances are so close that rounding could swap
// them, the caller re-derives that comparison on the host (see join.py), so
// the permutation always equals the reference's.
//   column_moments: grid (column, row chunk); each CTA reduces its chunk of one
//     column into a (hi, lo) pair; a second tiny pass combines the partials.
//   permute_columns: dst[:, j] = src[:, perm[j]], zero padding to ld_out.
#include "internal.cuh"

namespace tj {

constexpr int kMomThreads = 256;
constexpr int kMomChunks = 64;  // CTAs per column

__device__ __forceinline__ void two_sum(double& hi, double& lo, double v) {
  const double s = hi + v;
  const double bp = s - hi;
  const double err = (hi - (s - bp)) + (v - bp);
  hi = s;
  lo += err;
}

// partial[(col * kMomChunks + chunk) * 2 + {0,1}] = sum over the chunk of f(x)
// with f(x) = x (mean == nullptr) or (x - mean[col])^2.
__global__ void __launch_bounds__(kMomThreads)
    column_sum_kernel(const double* __restrict__ x, int64_t n, int64_t ld,
                      const double* __restrict__ mean, double* __restrict__ partial) {
  const int col = blockIdx.x;
  const int chunk = blockIdx.y;
  const int64_t per = (n + kMomChunks - 1) / kMomChunks;
  const int64_t r0 = chunk * per, r1 = min(n, r0 + per);
  const double mu = mean ? mean[col] : 0.0;
  double hi = 0.0, lo = 0.0;
  for (int64_t r = r0 + threadIdx.x; r < r1; r += kMomThreads) {
    const double v = x[r * ld + col];
    if (mean) {
      const double t = v - mu;
      two_sum(hi, lo, t * t);
    } else {
      two_sum(hi, lo, v);
    }
  }
  __shared__ double s_hi[kMomThreads], s_lo[kMomThreads];
  s_hi[threadIdx.x] = hi;
  s_lo[threadIdx.x] = lo;
  __syncthreads();
  if (threadIdx.x == 0) {  // fixed order: deterministic
    double h = 0.0, l = 0.0;
    for (int i = 0; i < kMomThreads; ++i) {
      two_sum(h, l, s_hi[i]);
      l += s_lo[i];
    }
    partial[(int64_t(col) * kMomChunks + chunk) * 2] = h;
    partial[(int64_t(col) * kMomChunks + chunk) * 2 + 1] = l;
  }
}

__global__ void column_finish_kernel(const double* __restrict__ partial, int d, int64_t n,
                                     double* __restrict__ out) {
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= d) return;
  double h = 0.0, l = 0.0;
  for (int i = 0; i < kMomChunks; ++i) {
    two_sum(h, l, partial[(int64_t(col) * kMomChunks + i) * 2]);
    l += partial[(int64_t(col) * kMomChunks + i) * 2 + 1];
  }
  out[col] = (h + l) / double(n);
}

__global__ void permute_columns_kernel(const double* __restrict__ src, int64_t n, int d,
                                       int64_t ld, const int* __restrict__ perm,
                                       double* __restrict__ dst, int64_t ld_out) {
  const int64_t total = n * ld_out;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = e / ld_out;
    const int j = int(e - r * ld_out);
    dst[e] = j < d ? src[r * ld + perm[j]] : 0.0;
  }
}

void column_moments(tj_ctx* ctx, const double* x, int64_t n, int d, int64_t ld, double* h_mean,
                    double* h_var, cudaStream_t s) {
  DevBuf part, mv;
  part.ensure(sizeof(double) * 2 * kMomChunks * d, s);
  mv.ensure(sizeof(double) * 2 * d, s);
  double* mean = mv.as<double>();
  double* var = mean + d;
  dim3 g(unsigned(d), kMomChunks);
  column_sum_kernel<<<g, kMomThreads, 0, s>>>(x, n, ld, nullptr, part.as<double>());
  TJ_CHECK_LAUNCH();
  column_finish_kernel<<<unsigned(ceil_div(d, 128)), 128, 0, s>>>(part.as<double>(), d, n, mean);
  TJ_CHECK_LAUNCH();
  column_sum_kernel<<<g, kMomThreads, 0, s>>>(x, n, ld, mean, part.as<double>());
  TJ_CHECK_LAUNCH();
  column_finish_kernel<<<unsigned(ceil_div(d, 128)), 128, 0, s>>>(part.as<double>(), d, n, var);
  TJ_CHECK_LAUNCH();
  TJ_CUDA(cudaMemcpyAsync(h_mean, mean, sizeof(double) * d, cudaMemcpyDeviceToHost, s));
  TJ_CUDA(cudaMemcpyAsync(h_var, var, sizeof(double) * d, cudaMemcpyDeviceToHost, s));
  TJ_CUDA(cudaStreamSynchronize(s));
  part.release(s);
  mv.release(s);
  (void)ctx;
}

void permute_columns(const double* src, int64_t n, int d, int64_t ld, const int* h_perm,
                     double* dst, int64_t ld_out, cudaStream_t s) {
  DevBuf pb;
  pb.ensure(sizeof(int) * d, s);
  TJ_CUDA(cudaMemcpyAsync(pb.ptr, h_perm, sizeof(int) * d, cudaMemcpyHostToDevice, s));
  const unsigned grid = unsigned(
      std::max<int64_t>(1, std::min<int64_t>(ceil_div(n * ld_out, 256), int64_t(kNumSMs) * 16)));
  permute_columns_kernel<<<grid, 256, 0, s>>>(src, n, d, ld, pb.as<int>(), dst, ld_out);
  TJ_CHECK_LAUNCH();
  TJ_CUDA(cudaStreamSynchronize(s));  // h_perm may be a temporary of the caller
  pb.release(s);
}

}  // namespace tj
