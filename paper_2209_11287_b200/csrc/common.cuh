// Shared helpers for the tedjoin sm_100a kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string>

#include "../../include/tedjoin.h"

namespace tj {

constexpr int kWarp = 32;
constexpr int kNumSMs = 148;

// Thrown inside the library only; every extern "C" entry point catches it and
// converts it to a status code plus tj_last_error() text.
struct Error {
  int status;
  std::string msg;
};

[[noreturn]] void fail(int status, const std::string& msg);

#define TJ_CUDA(expr)                                                              \
  do {                                                                             \
    cudaError_t _e = (expr);                                                       \
    if (_e != cudaSuccess)                                                         \
      ::tj::fail(TJ_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(_e) +    \
                               " (" __FILE__ ":" + std::to_string(__LINE__) + ")"); \
  } while (0)

// Every kernel launch of the library goes through TJ_CHECK_LAUNCH, which also
// counts it (tj_launch_count: the bench's gpu_launches evidence).
void note_launch();
#define TJ_CHECK_LAUNCH()          \
  do {                             \
    ::tj::note_launch();           \
    TJ_CUDA(cudaGetLastError());   \
  } while (0)

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }
__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Warp-level FP64 MMA D(8x8) = A(8x4) * B(4x8) + C(8x8); SASS DMMA.8x8x4 on sm_100a.
// Fragments (PTX ISA, m8n8k4 .f64): a = A[lane>>2][lane&3], b = B[lane&3][lane>>2],
// c/d = C[lane>>2][2*(lane&3) + {0,1}].
__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b,
                                           double c0, double c1) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};\n"
               : "=d"(d0), "=d"(d1)
               : "d"(a), "d"(b), "d"(c0), "d"(c1));
}

}  // namespace tj
