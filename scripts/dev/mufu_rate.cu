// Dev microbenchmark: MUFU.EX2 and packed FFMA2 throughput per SM sub-partition
// (warps per SMSP = W / 4), independent chains. Prints clocks per warp-instruction.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 scripts/dev/mufu_rate.cu -o scripts/dev/mufu_rate
#include <cstdio>
#include <cuda_runtime.h>

template <int KIND>
__global__ void k(float* out, int iters, long long* clk) {
  float a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = -0.001f * (threadIdx.x + i);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (KIND == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
      else if (KIND == 1) {
        float2 v = make_float2(a[i], a[i] + 1.f);
        asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(*reinterpret_cast<unsigned long long*>(&v))
                     : "l"(*reinterpret_cast<unsigned long long*>(&v)), "l"(*reinterpret_cast<unsigned long long*>(&v)));
        a[i] = v.x;
      } else {
        unsigned u;
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(u) : "f"(a[i]), "f"(a[i] * 0.5f));
        a[i] = __uint_as_float(u & 0x7fffffu);
      }
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int KIND>
void run(int warps, const char* name) {
  const int iters = 4096;
  float* o; long long* c;
  cudaMalloc(&o, 4 << 20); cudaMalloc(&c, 8 * 148);
  k<KIND><<<148, 32 * warps>>>(o, iters, c);
  long long h;
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  // warp-instructions per SMSP = iters * 8 * (warps / 4)
  const double per = double(h) / (double(iters) * 8 * (warps / 4.0));
  printf("%-8s warps/SM %2d: %.2f clk per warp-instruction per SMSP (=> %.1f lanes/clk/SM)\n", name, warps, per,
         4 * 32 / per);
  cudaFree(o); cudaFree(c);
}

int main() {
  for (int w : {4, 8, 16}) { run<0>(w, "ex2"); run<1>(w, "ffma2"); run<2>(w, "f2fp"); }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
