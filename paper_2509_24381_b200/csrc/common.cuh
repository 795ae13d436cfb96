// rserve-b200 — shared CUDA helpers for the sm_100a kernels.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <chrono>
#include <cstdint>
#include <string>
#include <utility>

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
// RS_HOST_TRACE=<ms>: host phases (launch path) longer than <ms> are
// reported on stderr with their label (diagnostics for launch-path stalls).
double host_trace_ms();
struct HostPhase {
  const char* label;
  std::chrono::steady_clock::time_point t0;
  explicit HostPhase(const char* l) : label(l), t0(std::chrono::steady_clock::now()) {}
  ~HostPhase();
};

namespace prof {
bool enabled();
void enable(bool on);
/// Returns a token for end(); -1 when disabled.
int begin(cudaStream_t st);
void end(int token, cudaStream_t st, const char* klass, double flops, double bytes);
/// "klass launches ms flops bytes" lines, aggregated; resets the counters.
std::string drain();
}  // namespace prof

// Programmatic dependent launch (PDL): kernels of the hot path are launched
// with programmatic stream serialization, so the next kernel of a stream is
// scheduled while the current one drains (its CTAs queue at the stream's
// priority instead of the other stream's kernel slipping into the gap, and
// launch latency / prologue overlap the previous tail). Every such kernel
// calls pdl_wait() before touching global memory. RS_PDL=0 disables.
bool pdl_enabled();
/// Longest single kernel-launch API call since the last reset (host stall
/// diagnostics: a full launch queue blocks the calling thread), in ms.
void note_launch_ms(double ms);
double take_max_launch_ms();

/// cudaLaunchKernelEx with the PDL attribute (when enabled) and an optional
/// cluster dimension.
template <typename... KArgs, typename... Args>
inline void launch_kernel(void (*kernel)(KArgs...), dim3 grid, dim3 block, std::size_t smem,
                          cudaStream_t st, int cluster_x, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  unsigned n = 0;
  if (pdl_enabled()) {
    attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  if (cluster_x > 1) {
    attr[n].id = cudaLaunchAttributeClusterDimension;
    attr[n].val.clusterDim.x = static_cast<unsigned>(cluster_x);
    attr[n].val.clusterDim.y = 1;
    attr[n].val.clusterDim.z = 1;
    ++n;
  }
  cfg.attrs = attr;
  cfg.numAttrs = n;
  const auto t0 = std::chrono::steady_clock::now();
  RS_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
  note_launch_ms(std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
}

__host__ __device__ inline int ceil_div(int a, int b) { return (a + b - 1) / b; }
__host__ __device__ inline std::int64_t ceil_div64(std::int64_t a, std::int64_t b) {
  return (a + b - 1) / b;
}

#ifdef __CUDACC__
// PDL device side: wait for the prerequisite grid (no-op without PDL), and
// let the dependent grid launch early.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ float bf2f(bf16 v) { return __bfloat162float(v); }
// Packed fp32x2 arithmetic (sm_100 FFMA2 / FADD2 / FMUL2: two lanes per instruction).
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;"
      : "=l"(r)
      : "l"(*reinterpret_cast<unsigned long long*>(&a)), "l"(*reinterpret_cast<unsigned long long*>(&b)),
        "l"(*reinterpret_cast<unsigned long long*>(&c)));
  return *reinterpret_cast<float2*>(&r);
}
__device__ __forceinline__ float2 add2(float2 a, float2 b) {
  unsigned long long r;
  asm("add.rn.f32x2 %0, %1, %2;"
      : "=l"(r)
      : "l"(*reinterpret_cast<unsigned long long*>(&a)), "l"(*reinterpret_cast<unsigned long long*>(&b)));
  return *reinterpret_cast<float2*>(&r);
}
__device__ __forceinline__ float2 mul2(float2 a, float2 b) {
  unsigned long long r;
  asm("mul.rn.f32x2 %0, %1, %2;"
      : "=l"(r)
      : "l"(*reinterpret_cast<unsigned long long*>(&a)), "l"(*reinterpret_cast<unsigned long long*>(&b)));
  return *reinterpret_cast<float2*>(&r);
}
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
