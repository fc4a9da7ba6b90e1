// FP64 pipe microbenchmarks (DFMA on CUDA cores vs DMMA.8x8x4 on the tensor
// pipe) and a known-answer test pinning the m8n8k4 f64 fragment layout.
// These give the roofline denominator the bench reports: B200's FP64 peak is
// not in MEASURED_PEAKS.json.
#include "common.cuh"

namespace tj {

template <int KIND>
__global__ void __launch_bounds__(256) fp64_peak_kernel(double* out, int iters, double seed) {
  // 8 independent DFMA chains and 4 independent DMMA accumulators per thread/warp.
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = seed * (threadIdx.x + i + 1);
  double d0[4], d1[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    d0[i] = seed * i;
    d1[i] = seed * (i + 2);
  }
  const double a = 1.0 + 1e-9 * threadIdx.x, b = 0.999999;
  for (int it = 0; it < iters; ++it) {
    if (KIND == 0 || KIND == 2) {
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = fma(x[i], b, a);
    }
    if (KIND == 1 || KIND == 2) {
#pragma unroll
      for (int i = 0; i < 4; ++i) dmma_8x8x4(d0[i], d1[i], a, b, d0[i], d1[i]);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
#pragma unroll
  for (int i = 0; i < 4; ++i) s += d0[i] + d1[i];
  if (s == 12345.678) out[threadIdx.x] = s;  // keep the work alive
}

__global__ void dmma_kat_kernel(const double* a, const double* b, const double* c, double* d) {
  const int lane = threadIdx.x;
  const int g = lane >> 2, t = lane & 3;
  double a0 = a[g * 4 + t];             // A[g][t]
  double b0 = b[t * 8 + g];             // B[t][g]
  double c0 = c[g * 8 + 2 * t], c1 = c[g * 8 + 2 * t + 1];
  double d0, d1;
  dmma_8x8x4(d0, d1, a0, b0, c0, c1);
  d[g * 8 + 2 * t] = d0;
  d[g * 8 + 2 * t + 1] = d1;
}

}  // namespace tj

using namespace tj;

extern "C" int tj_fp64_peak(int32_t kind, int32_t iters, double* tflops, double* ms) {
  if (kind < 0 || kind > 2 || iters < 1) return TJ_EINVAL;
  double* out = nullptr;
  if (cudaMalloc(&out, 256 * sizeof(double)) != cudaSuccess) return TJ_ECUDA;
  const int blocks = kNumSMs * 8;
  auto launch = [&](int it) {
    if (kind == 0) fp64_peak_kernel<0><<<blocks, 256>>>(out, it, 1.0);
    if (kind == 1) fp64_peak_kernel<1><<<blocks, 256>>>(out, it, 1.0);
    if (kind == 2) fp64_peak_kernel<2><<<blocks, 256>>>(out, it, 1.0);
  };
  launch(16);  // warm-up
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  launch(iters);
  cudaEventRecord(e1);
  cudaError_t err = cudaEventSynchronize(e1);
  float t = 0;
  cudaEventElapsedTime(&t, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  if (err != cudaSuccess) return TJ_ECUDA;
  const double threads = double(blocks) * 256.0;
  double flops = 0;
  if (kind == 0 || kind == 2) flops += threads * iters * 8 * 2.0;
  if (kind == 1 || kind == 2) flops += threads / 32.0 * iters * 4 * 512.0;
  *ms = t;
  *tflops = flops / (t * 1e-3) / 1e12;
  return TJ_OK;
}

extern "C" int tj_dmma_known_answer(const double* a, const double* b, const double* c, double* d) {
  double* buf = nullptr;
  if (cudaMalloc(&buf, (32 + 32 + 64 + 64) * sizeof(double)) != cudaSuccess) return TJ_ECUDA;
  cudaMemcpy(buf, a, 32 * sizeof(double), cudaMemcpyHostToDevice);
  cudaMemcpy(buf + 32, b, 32 * sizeof(double), cudaMemcpyHostToDevice);
  cudaMemcpy(buf + 64, c, 64 * sizeof(double), cudaMemcpyHostToDevice);
  dmma_kat_kernel<<<1, 32>>>(buf, buf + 32, buf + 64, buf + 128);
  cudaError_t err = cudaMemcpy(d, buf + 128, 64 * sizeof(double), cudaMemcpyDeviceToHost);
  cudaFree(buf);
  return err == cudaSuccess ? TJ_OK : TJ_ECUDA;
}
