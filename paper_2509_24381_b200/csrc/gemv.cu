// rserve-b200 — skinny GEMM (M <= 8 rows: decode steps) on the CUDA cores.
//
// At batch-1 decode every LLM weight is read once per step, so the step is
// bound by streaming B from HBM; the tcgen05 kernel's 128-row tiles would
// leave most of the SMs idle (e.g. 36 tiles for the QKV projection). Here a
// CTA owns 32 consecutive B rows (one SwiGLU interleave group), each of its 8
// warps streams 4 rows over the full K with 16-byte loads (A rows come
// through L1), lanes reduce by shuffles, and the block applies the same
// fused epilogues as the tcgen05 GEMM (bias, residual + folded-norm sums of
// squares, SwiGLU, GELU, fp32 row-mapped logits, folded-norm row scale).
#include <cuda_runtime.h>

#include "gemm.cuh"

namespace rserve {
namespace {

constexpr int kRowsPerBlock = 32, kWarps = 8, kRowsPerWarp = 4, kMaxM = 8;

__device__ __forceinline__ float gelu_erf_v(float x) { return 0.5f * x * (1.f + erff(x * 0.70710678118654752f)); }
__device__ __forceinline__ float silu_v(float x) { return __fdividef(x, 1.f + __expf(-x)); }

template <int MM, int EPI>
__global__ void __launch_bounds__(kWarps * 32) gemv_kernel(GemmArgs a) {
  __shared__ float res[kRowsPerBlock][MM];
  pdl_wait();
  pdl_launch_dependents();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n0 = blockIdx.x * kRowsPerBlock;
  const int r0 = n0 + warp * kRowsPerWarp;
  float acc[kRowsPerWarp][MM];
#pragma unroll
  for (int r = 0; r < kRowsPerWarp; ++r)
#pragma unroll
    for (int m = 0; m < MM; ++m) acc[r][m] = 0.f;
  const int k8n = a.K / 8;
  const uint4* brow[kRowsPerWarp];
#pragma unroll
  for (int r = 0; r < kRowsPerWarp; ++r)
    brow[r] = reinterpret_cast<const uint4*>(a.B + static_cast<std::int64_t>(min(r0 + r, a.N - 1)) * a.ldb);
#pragma unroll 2
  for (int k8 = lane; k8 < k8n; k8 += 32) {
    uint4 bv[kRowsPerWarp];
#pragma unroll
    for (int r = 0; r < kRowsPerWarp; ++r) bv[r] = __ldcs(brow[r] + k8);  // streamed once
#pragma unroll
    for (int m = 0; m < MM; ++m) {
      if (m >= a.M) break;
      const uint4 av = __ldg(reinterpret_cast<const uint4*>(a.A + static_cast<std::int64_t>(m) * a.lda) + k8);
      const std::uint32_t aw[4] = {av.x, av.y, av.z, av.w};
#pragma unroll
      for (int r = 0; r < kRowsPerWarp; ++r) {
        const std::uint32_t bw[4] = {bv[r].x, bv[r].y, bv[r].z, bv[r].w};
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const float2 fa = unpack_bf16x2(aw[t]), fb = unpack_bf16x2(bw[t]);
          acc[r][m] = fmaf(fa.x, fb.x, fmaf(fa.y, fb.y, acc[r][m]));
        }
      }
    }
  }
#pragma unroll
  for (int r = 0; r < kRowsPerWarp; ++r)
#pragma unroll
    for (int m = 0; m < MM; ++m) {
      float v = acc[r][m];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) res[warp * kRowsPerWarp + r][m] = v;
    }
  __syncthreads();
  // ---- fused epilogue: thread -> (row m, column c of the block) ----
  const int tid = threadIdx.x;
  const int m = tid / kRowsPerBlock, c = tid % kRowsPerBlock;
  if (m >= a.M || m >= MM) return;
  float rs = 1.f;
  if (a.ss_in != nullptr)
    rs = rsqrtf(static_cast<float>(__ldcg(a.ss_in + m)) * (1.f / kSsFixedScale) * a.ss_inv_dim + a.ss_eps);
  const int out_row = a.row_map != nullptr ? a.row_map[m] : m;
  if constexpr (EPI == static_cast<int>(Epi::SwiGLU)) {
    if (c >= 16) return;
    const int gr = n0 + c, ur = n0 + 16 + c;  // 16-row gate / up interleave
    float g = rs * res[c][m], u = rs * res[16 + c][m];
    if (a.bias != nullptr) {
      g += __bfloat162float(a.bias[gr]);
      u += __bfloat162float(a.bias[ur]);
    }
    bf16* C = static_cast<bf16*>(a.C);
    C[static_cast<std::int64_t>(out_row) * a.ldc + (n0 / 32) * 16 + c] = __float2bfloat16_rn(silu_v(g) * u);
  } else {
    const int col = n0 + c;
    float v = 0.f;
    const bool ok = col < a.N;
    if (ok) {
      v = rs * res[c][m];
      if (a.bias != nullptr) v += __bfloat162float(a.bias[col]);
      if constexpr (EPI == static_cast<int>(Epi::Gelu)) v = gelu_erf_v(v);
      if constexpr (EPI == static_cast<int>(Epi::Residual))
        v += __bfloat162float(a.residual[static_cast<std::int64_t>(out_row) * a.ldr + col]);
      if constexpr (EPI == static_cast<int>(Epi::StoreF32)) {
        static_cast<float*>(a.C)[static_cast<std::int64_t>(out_row) * a.ldc + col] = v;
      } else {
        const bf16 o = __float2bfloat16_rn(v);
        static_cast<bf16*>(a.C)[static_cast<std::int64_t>(out_row) * a.ldc + col] = o;
        v = __bfloat162float(o);
      }
    }
    if constexpr (EPI == static_cast<int>(Epi::Residual)) {
      if (a.ss_out != nullptr) {  // sum of squares of this block's 32 output columns of row m
        float sq = ok ? v * v : 0.f;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
        if (c == 0)
          atomicAdd(a.ss_out + out_row, static_cast<unsigned long long>(__float2ull_rn(sq * kSsFixedScale)));
      }
    }
  }
}

__global__ void clear_u64_kernel(unsigned long long* p, int n) {
  pdl_wait();
  pdl_launch_dependents();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) p[i] = 0ull;
}

template <int MM>
void launch_m(const GemmArgs& a, Epi epi, cudaStream_t st) {
  const dim3 grid((a.N + kRowsPerBlock - 1) / kRowsPerBlock), block(kWarps * 32);
  switch (epi) {
    case Epi::Store: return launch_kernel(gemv_kernel<MM, 0>, grid, block, 0, st, 1, a);
    case Epi::Residual: return launch_kernel(gemv_kernel<MM, 1>, grid, block, 0, st, 1, a);
    case Epi::SwiGLU: return launch_kernel(gemv_kernel<MM, 2>, grid, block, 0, st, 1, a);
    case Epi::Gelu: return launch_kernel(gemv_kernel<MM, 3>, grid, block, 0, st, 1, a);
    case Epi::StoreF32: return launch_kernel(gemv_kernel<MM, 4>, grid, block, 0, st, 1, a);
  }
}

}  // namespace

bool gemv_small_m(const GemmArgs& a, Epi epi, cudaStream_t st) {
  if (a.M > kMaxM || a.M_dev != nullptr || a.K % 8 != 0 || a.lda % 8 != 0 || a.ldb % 8 != 0) return false;
  if (epi == Epi::SwiGLU && a.N % kRowsPerBlock != 0) return false;
  if (a.ss_clear != nullptr && a.ss_clear_n > 0)
    launch_kernel(clear_u64_kernel, dim3((a.ss_clear_n + 255) / 256), dim3(256), 0, st, 1, a.ss_clear, a.ss_clear_n);
  if (a.M <= 1) launch_m<1>(a, epi, st);
  else if (a.M <= 2) launch_m<2>(a, epi, st);
  else if (a.M <= 4) launch_m<4>(a, epi, st);
  else launch_m<8>(a, epi, st);
  RS_LAUNCH_CHECK();
  count_launch(a.ss_clear != nullptr && a.ss_clear_n > 0 ? 2 : 1);
  return true;
}

}  // namespace rserve
