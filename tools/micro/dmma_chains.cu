// DMMA.8x8x4 throughput vs independent accumulator chains per warp and warps
// per SM (guides the refine kernels' step structure).  nvcc -arch=sm_100a.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int C>
__global__ void chains(double* out, int iters) {
  double d0[C], d1[C];
  for (int i = 0; i < C; ++i) { d0[i] = threadIdx.x * 1e-3 + i; d1[i] = i * 0.5; }
  const double a = 1.0 + 1e-9 * threadIdx.x, b = 0.999999;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < C; ++i) dmma(d0[i], d1[i], a, b);
  double s = 0;
  for (int i = 0; i < C; ++i) s += d0[i] + d1[i];
  if (s == 1.2345) out[threadIdx.x] = s;
}

template <int C>
void run(int warps_per_sm, double* out) {
  const int iters = 4096;
  const int threads = 32 * (warps_per_sm < 4 ? warps_per_sm : 4);
  const int blocks = 148 * warps_per_sm * 32 / threads;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  chains<C><<<blocks, threads>>>(out, 16);
  cudaEventRecord(e0);
  chains<C><<<blocks, threads>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double flops = 2.0 * 256 * C * double(iters) * blocks * (threads / 32);
  printf("chains/warp %d warps/SM %2d : %6.2f TFLOP/s\n", C, warps_per_sm, flops / ms / 1e9);
}

int main() {
  double* out; cudaMalloc(&out, 1024 * sizeof(double));
  int ws[] = {4, 8, 12, 16, 24, 32};
  for (int w : ws) { run<1>(w, out); run<2>(w, out); run<4>(w, out); run<8>(w, out); }
  return 0;
}
