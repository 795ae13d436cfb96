// rserve-b200 — skinny GEMM (M <= 8 rows: decode steps) on the CUDA cores.
//
// At batch-1 decode every LLM weight is read once per step, so the step is
// bound by streaming B from HBM; the tcgen05 kernel's 128-row tiles would
// leave most of the SMs idle (e.g. 36 tiles for the QKV projection). Here a
// CTA owns 4 B rows (for SwiGLU: 2 gate rows and their 2 up rows of one
// 32-row interleave group) and its 8 warps split K, streaming the rows with
// 16-byte loads (A rows come through L1); warp partials are summed in warp
// order (deterministic) and the CTA applies the same fused epilogues as the
// tcgen05 GEMM (bias, residual + folded-norm sums of squares, SwiGLU, GELU,
// fp32 row-mapped logits, folded-norm row scale, and the QKV projection's
// M-RoPE + paged K / V append: a block of q / k columns holds two
// rotate-half pairs (i, i + hd/2), (i + 1, i + 1 + hd/2) of one head).
#include <cuda_runtime.h>

#include "gemm.cuh"
#include "kernels.cuh"

namespace rserve {
namespace {

#ifndef RS_GEMV_UNROLL
#define RS_GEMV_UNROLL 2
#endif
constexpr int kRows = 4, kWarps = 8, kMaxM = 8;
constexpr int kUnroll = RS_GEMV_UNROLL;  // k iterations in flight per thread

__device__ __forceinline__ float gelu_erf_v(float x) { return 0.5f * x * (1.f + erff(x * 0.70710678118654752f)); }
__device__ __forceinline__ float silu_v(float x) { return __fdividef(x, 1.f + __expf(-x)); }

// B row of local row r (0..3) of block b
template <bool SWIGLU>
__device__ __forceinline__ int brow_of(int b, int r) {
  if constexpr (SWIGLU) {
    const int group = b >> 3, pair = b & 7;  // 8 blocks per 32-row group
    return group * 32 + (r < 2 ? 2 * pair + r : 16 + 2 * pair + (r - 2));
  } else {
    return b * kRows + r;
  }
}
// QkvRope: q / k heads take rotate-half pairs, r = {i, i + hd/2, i + 1, i + 1 + hd/2}
// with i = 2 (b mod hd/4); v heads take 4 consecutive columns
__device__ __forceinline__ int brow_rope(int b, int r, int hd, int qk_heads) {
  const int per_head = hd / 4, head = b / per_head, j = b % per_head;
  if (head >= qk_heads) return b * kRows + r;
  return head * hd + 2 * j + (r >> 1) + (r & 1) * (hd / 2);
}

template <int MM, int EPI>
__global__ void __launch_bounds__(kWarps * 32) gemv_kernel(GemmArgs a) {
  constexpr bool kSwi = EPI == static_cast<int>(Epi::SwiGLU);
  constexpr bool kRope = EPI == static_cast<int>(Epi::QkvRope);
  auto brow = [&](int bb, int r) {
    if constexpr (kRope) return brow_rope(bb, r, a.rope_hd, a.rope_hq + a.rope_hkv);
    else return brow_of<kSwi>(bb, r);
  };
  __shared__ float part[kWarps][kRows][MM];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = blockIdx.x;
  // The weights are not written by the kernels this one depends on: start
  // pulling this thread's first k iterations into L2 before waiting on the
  // previous kernel (PDL), so the stream overlaps its tail.
#ifndef RS_GEMV_NO_PREFETCH
  {
    const int k8n0 = a.K / 8;
#pragma unroll
    for (int r = 0; r < kRows; ++r) {
      const uint4* row = reinterpret_cast<const uint4*>(
          a.B + static_cast<std::int64_t>(min(brow(b, r), a.N - 1)) * a.ldb);
#pragma unroll
      for (int i = 0; i < kUnroll; ++i) {
        const int k8 = warp * 32 + lane + i * kWarps * 32;
        if (k8 < k8n0) asm volatile("prefetch.global.L2 [%0];" ::"l"(row + k8));
      }
    }
  }
#endif
  pdl_wait();
  pdl_launch_dependents();
  float acc[kRows][MM];
#pragma unroll
  for (int r = 0; r < kRows; ++r)
#pragma unroll
    for (int m = 0; m < MM; ++m) acc[r][m] = 0.f;
  const int k8n = a.K / 8;
  const uint4* brow_p[kRows];
#pragma unroll
  for (int r = 0; r < kRows; ++r)
    brow_p[r] = reinterpret_cast<const uint4*>(a.B + static_cast<std::int64_t>(min(brow(b, r), a.N - 1)) * a.ldb);
#pragma unroll kUnroll
  for (int k8 = warp * 32 + lane; k8 < k8n; k8 += kWarps * 32) {
    uint4 bv[kRows];
#pragma unroll
    for (int r = 0; r < kRows; ++r) bv[r] = __ldcs(brow_p[r] + k8);  // streamed once
#pragma unroll
    for (int m = 0; m < MM; ++m) {
      if (m >= a.M) break;
      const uint4 av = __ldg(reinterpret_cast<const uint4*>(a.A + static_cast<std::int64_t>(m) * a.lda) + k8);
      const std::uint32_t aw[4] = {av.x, av.y, av.z, av.w};
#pragma unroll
      for (int r = 0; r < kRows; ++r) {
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
  for (int r = 0; r < kRows; ++r)
#pragma unroll
    for (int m = 0; m < MM; ++m) {
      float v = acc[r][m];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) part[warp][r][m] = v;
    }
  __syncthreads();
  // ---- fused epilogue: thread -> (row m, local column r) ----
  const int tid = threadIdx.x;
  if (tid >= kRows * MM) return;
  const int m = tid / kRows, r = tid % kRows;
  if (m >= a.M) return;
  auto dot = [&](int rr) {
    float s = 0.f;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) s += part[w][rr][m];  // warp order: deterministic
    return s;
  };
  float rs = 1.f;
  if (a.ss_in != nullptr)
    rs = rsqrtf(static_cast<float>(__ldcg(a.ss_in + m)) * (1.f / kSsFixedScale) * a.ss_inv_dim + a.ss_eps);
  const int out_row = a.row_map != nullptr ? a.row_map[m] : m;
  if constexpr (kRope) {
    // x = rs * acc + bias, rotated with its rotate-half partner (q / k), then
    // stored to C; k / v rows also go to this token's KV page (as the tcgen05
    // QkvRope epilogue: fp32 rotation, one bf16 rounding)
    const int hd = a.rope_hd, half = hd / 2;
    const int col = brow(b, r);
    if (col >= a.N) return;
    const int head = col / hd, i0 = col % hd;
    float x = rs * dot(r);
    if (a.bias != nullptr) x += __bfloat162float(a.bias[col]);
    if (head < a.rope_hq + a.rope_hkv) {
      const int pc = brow(b, r ^ 1);  // partner column i0 -/+ hd/2
      float w = rs * dot(r ^ 1);
      if (a.bias != nullptr) w += __bfloat162float(a.bias[pc]);
      const float2 cs = a.rope_table[static_cast<std::int64_t>(m) * half + (i0 % half)];
      x = i0 < half ? x * cs.x - w * cs.y : x * cs.x + w * cs.y;
    }
    const bf16 o = __float2bfloat16_rn(x);
    static_cast<bf16*>(a.C)[static_cast<std::int64_t>(out_row) * a.ldc + col] = o;
    if (head >= a.rope_hq) {
      const ChunkRowInfo ri = static_cast<const ChunkRowInfo*>(a.rope_rows)[m];
      const std::int64_t page = a.page_tables[ri.req_slot][ri.pos / a.page_size];
      const int off = ri.pos % a.page_size;
      if (head < a.rope_hq + a.rope_hkv) {  // K: [page][kv head][token][hd]
        const int kvh = head - a.rope_hq;
        a.k_cache[((page * a.rope_hkv + kvh) * a.page_size + off) * hd + i0] = o;
      } else {  // V transposed: [page][kv head][hd][token]
        const int kvh = head - a.rope_hq - a.rope_hkv;
        a.v_cache[((page * a.rope_hkv + kvh) * hd + i0) * a.page_size + off] = o;
      }
    }
  } else if constexpr (kSwi) {
    if (r >= 2) return;
    const int gr = brow_of<true>(b, r), ur = brow_of<true>(b, r + 2);
    float g = rs * dot(r), u = rs * dot(r + 2);
    if (a.bias != nullptr) {
      g += __bfloat162float(a.bias[gr]);
      u += __bfloat162float(a.bias[ur]);
    }
    const int col = (gr / 32) * 16 + gr % 32;  // output column of gate row gr
    static_cast<bf16*>(a.C)[static_cast<std::int64_t>(out_row) * a.ldc + col] = __float2bfloat16_rn(silu_v(g) * u);
  } else {
    const int col = brow_of<false>(b, r);
    float v = 0.f;
    const bool ok = col < a.N;
    if (ok) {
      v = rs * dot(r);
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
      if (a.ss_out != nullptr) {  // the block's 4 columns of row m (lanes 4m..4m+3 of warp 0)
        const unsigned long long q =
            ok ? static_cast<unsigned long long>(__float2ull_rn(v * v * kSsFixedScale)) : 0ull;
        const unsigned mask = __activemask();  // rows m < M: whole 4-lane groups
        unsigned long long t = q + __shfl_down_sync(mask, q, 1, kRows);
        t += __shfl_down_sync(mask, t, 2, kRows);
        if (r == 0) atomicAdd(a.ss_out + out_row, t);  // 2^-16 fixed point: order-free
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
  const dim3 grid((a.N + kRows - 1) / kRows), block(kWarps * 32);
  switch (epi) {
    case Epi::Store: return launch_kernel(gemv_kernel<MM, 0>, grid, block, 0, st, 1, a);
    case Epi::Residual: return launch_kernel(gemv_kernel<MM, 1>, grid, block, 0, st, 1, a);
    case Epi::SwiGLU: return launch_kernel(gemv_kernel<MM, 2>, grid, block, 0, st, 1, a);
    case Epi::Gelu: return launch_kernel(gemv_kernel<MM, 3>, grid, block, 0, st, 1, a);
    case Epi::StoreF32: return launch_kernel(gemv_kernel<MM, 4>, grid, block, 0, st, 1, a);
    case Epi::QkvRope: return launch_kernel(gemv_kernel<MM, 5>, grid, block, 0, st, 1, a);
  }
}

}  // namespace

bool gemv_small_m(const GemmArgs& a, Epi epi, cudaStream_t st) {
  if (a.M > kMaxM || a.M_dev != nullptr || a.K % 8 != 0 || a.lda % 8 != 0 || a.ldb % 8 != 0) return false;
  if (epi == Epi::SwiGLU && a.N % 32 != 0) return false;
  if (epi == Epi::QkvRope && (a.rope_hd % 4 != 0 || a.N % a.rope_hd != 0 || a.rope_rows == nullptr ||
                              a.rope_table == nullptr || a.page_tables == nullptr || a.row_map != nullptr))
    return false;
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
