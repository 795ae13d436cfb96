// Dev microbenchmark: back-to-back tcgen05.mma issue rate from one thread,
// 128 x N x 16 bf16 (SS: both operands in smem; TS: A from TMEM), M = 128,
// cta_group::1. Prints clocks per MMA for N = 64 / 128 / 256.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 -I paper_2509_24381_b200/csrc scripts/dev/mma_rate.cu -o /tmp/mma_rate -lcuda
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "sm100.cuh"

using namespace rserve;

template <int N, bool TS>
__global__ void k(unsigned long long* out, int iters) {
  extern __shared__ __align__(1024) std::uint8_t smem[];
  __shared__ std::uint64_t bar;
  __shared__ std::uint32_t holder;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) { sm100::mbar_init(&bar, 1); sm100::fence_mbar_init(); }
  if (warp == 0) sm100::tmem_alloc(&holder, 512);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const std::uint32_t tmem = holder;
  if (threadIdx.x == 0) {
    constexpr std::uint32_t idesc = sm100::idesc_bf16_f32(128, N);
    const std::uint64_t ad = sm100::sw128_kmajor_desc(sm100::smem_u32(smem));
    const std::uint64_t bd = sm100::sw128_kmajor_desc(sm100::smem_u32(smem + 16384));
    // warm
    for (int i = 0; i < 8; ++i) {
      if (TS) sm100::umma_bf16_ts(tmem + 256, tmem + 8 * (i & 3), bd, idesc, 1u);
      else sm100::umma_bf16(tmem, ad, bd, idesc, 1u);
    }
    sm100::umma_commit(&bar);
    sm100::mbar_wait(&bar, 0);
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      if (TS) sm100::umma_bf16_ts(tmem + 256, tmem + 8 * (i & 3), bd + 2 * (i & 3), idesc, 1u);
      else sm100::umma_bf16(tmem, ad + 2 * (i & 3), bd + 2 * (i & 3), idesc, 1u);
    }
    long long t1 = clock64();
    sm100::umma_commit(&bar);
    sm100::mbar_wait(&bar, 1);
    long long t2 = clock64();
    out[0] = t1 - t0;  // issue time
    out[1] = t2 - t0;  // issue + drain
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 0) sm100::tmem_dealloc(tmem, 512);
}

template <int N, bool TS>
void run(int iters) {
  unsigned long long* d;
  cudaMalloc(&d, 16);
  auto f = k<N, TS>;
  cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  f<<<1, 128, 100 * 1024>>>(d, iters);
  unsigned long long h[2];
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("%s N=%3d: issue %.1f clk/mma, issue+drain %.1f clk/mma (nominal %d)\n", TS ? "TS" : "SS", N,
         double(h[0]) / iters, double(h[1]) / iters, 128 * N / 256);
  cudaFree(d);
}

int main() {
  for (int it : {64, 1024}) {
    printf("iters %d\n", it);
    run<64, false>(it); run<128, false>(it); run<256, false>(it);
    run<128, true>(it); run<256, true>(it);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
}
