// rserve-b200 — shared CUDA helpers for the sm_100a kernels.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "host/status.hpp"

namespace rserve {

#define RS_CUDA_CHECK(expr)                                                     \
  do {                                                                          \
    cudaError_t rs_err__ = (expr);                                              \
    if (rs_err__ != cudaSuccess)                                                \
      throw ::rserve::DeviceError(RS_ERR_CUDA, std::string(#expr) + ": " +      \
                                                   cudaGetErrorString(rs_err__) + \
                                                   " (" __FILE__ ":" +          \
                                                   std::to_string(__LINE__) + ")"); \
  } while (0)

#define RS_LAUNCH_CHECK() RS_CUDA_CHECK(cudaGetLastError())

using bf16 = __nv_bfloat16;

constexpr int kNumSMs = 148;

// Counts launches of our kernels (for bench.py's gpu_launches claim).
void count_launch(std::uint64_t n = 1);
std::uint64_t launches_so_far();

// Optional live per-kernel-class timing (CUDA events on the launch stream),
// enabled per engine run for bench.py's roofline figures.
namespace prof {
bool enabled();
void enable(bool on);
/// Returns a token for end(); -1 when disabled.
int begin(cudaStream_t st);
void end(int token, cudaStream_t st, const char* klass, double flops, double bytes);
/// "klass launches ms flops bytes" lines, aggregated; resets the counters.
std::string drain();
}  // namespace prof

__host__ __device__ inline int ceil_div(int a, int b) { return (a + b - 1) / b; }
__host__ __device__ inline std::int64_t ceil_div64(std::int64_t a, std::int64_t b) {
  return (a + b - 1) / b;
}

#ifdef __CUDACC__
__device__ __forceinline__ float bf2f(bf16 v) { return __bfloat162float(v); }
__device__ __forceinline__ bf16 f2bf(float v) { return __float2bfloat16_rn(v); }

__device__ __forceinline__ std::uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 p = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<std::uint32_t*>(&p);
}
__device__ __forceinline__ float2 unpack_bf16x2(std::uint32_t v) {
  __nv_bfloat162 p = *reinterpret_cast<__nv_bfloat162*>(&v);
  return __bfloat1622float2(p);
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
#endif

}  // namespace rserve
