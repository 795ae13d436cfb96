// rserve-b200 — persistent, warp-specialised tcgen05 GEMM for sm_100a.
//
//   C[M, N] = epilogue( A[M, K] . B[N, K]^T )      (A, B bf16, K-major)
//
// One CTA per SM (grid = min(tiles, 148)), 128 x BN output tiles, BK = 64.
// warp 0: TMA producer (128B-swizzled tiles, multi-stage mbarrier ring);
// warp 1: single-thread tcgen05.mma issuer (M=128, N=BN, K=16, FP32 in
//         TMEM, double-buffered accumulators so the epilogue of tile i
//         overlaps the MMAs of tile i+1);
// warp 2: TMEM allocator; warps 4-7: epilogue (tcgen05.ld -> fused op ->
//         bf16/fp32 global stores).
// Fused epilogues cover every linear layer of the ViT and the LLM: bias,
// in-place residual add, SwiGLU (gate/up interleaved in 16-row blocks),
// exact-erf GELU, fp32 logits, and an optional output-row map used to scatter
// merger rows straight into LLM token order / embedding slots.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "common.cuh"

namespace rserve {

enum class Epi : int {
  Store = 0,     // C = acc (+ bias)                       bf16
  Residual = 1,  // C = acc (+ bias) + R   (R may alias C)  bf16
  SwiGLU = 2,    // C[:, j] = silu(g_j) * u_j, N/2 columns  bf16
  Gelu = 3,      // C = gelu_erf(acc + bias)                bf16
  StoreF32 = 4,  // C = acc (+ bias)                       fp32
  QkvRope = 5,   // LLM QKV: C = acc (+ bias), q / k rotated (M-RoPE), k / v
                 // appended to the paged KV cache (V transposed)   bf16
};

struct GemmArgs {
  const bf16* A = nullptr;  // [M, K] row stride lda (elements)
  int lda = 0;
  const bf16* B = nullptr;  // [N, K] row stride ldb
  int ldb = 0;
  void* C = nullptr;        // [M, N] (SwiGLU: [M, N/2]) row stride ldc
  int ldc = 0;
  const bf16* bias = nullptr;      // [N] or null
  const bf16* residual = nullptr;  // Residual epilogue, row stride ldr
  int ldr = 0;
  const int* row_map = nullptr;    // optional: output row of input row m
  int M = 0, N = 0, K = 0;
  const int* M_dev = nullptr;      // optional device-side M (<= M), graph-friendly
  // RMSNorm folded into the GEMMs around it (model.cu). A norm's consumer
  // GEMM reads the un-normalised residual stream x and scales output row r by
  // rsqrt(ss_in[r] * 2^-16 * ss_inv_dim + ss_eps) before the bias (the norm
  // weight is folded into B's columns at load). The residual GEMM producing x
  // adds each epilogue thread's sum of squares of its bf16 output row segment
  // to ss_out[r] as 2^-16 fixed point (64-bit integer atomics: the total is
  // independent of the order, so runs stay bit-reproducible) and zeroes
  // ss_clear[0, ss_clear_n) for the next producer (ping-pong buffers).
  const unsigned long long* ss_in = nullptr;
  float ss_inv_dim = 0.f, ss_eps = 0.f;
  unsigned long long* ss_out = nullptr;
  unsigned long long* ss_clear = nullptr;
  int ss_clear_n = 0;
  // Epi::QkvRope: per-row chunk info (ChunkRowInfo: req slot, position), the
  // chunk's [M, hd/2] (cos, sin) table, paged KV of this layer
  const void* rope_rows = nullptr;
  const float2* rope_table = nullptr;
  const int* const* page_tables = nullptr;
  bf16* k_cache = nullptr;
  bf16* v_cache = nullptr;
  int rope_hq = 0, rope_hkv = 0, rope_hd = 0, page_size = 0;
  // B is not written by the kernels launched before this GEMM on its stream
  // (model weights): its first tiles may load before the PDL wait. The
  // public op (rs_op_gemm) clears it: there B may be a preceding op's output.
  bool b_stable = true;
};
constexpr float kSsFixedScale = 65536.f;  // 2^16

/// Launches the tcgen05 GEMM. Requires K % 8 == 0, N % 16 == 0,
/// 16-byte aligned rows. Tile width is picked for wave efficiency.
void gemm(const GemmArgs& args, Epi epi, cudaStream_t stream, int force_bn = 0);

/// Skinny GEMM for M <= 8 rows (decode) on the CUDA cores, same epilogues
/// (gemv.cu). Returns false when the shape is not supported (caller falls
/// back to the tcgen05 kernel). gemm() routes here by default.
/// Frees the split-K workspace of a stream that is about to be destroyed.
void gemm_release_stream(cudaStream_t st);

bool gemv_small_m(const GemmArgs& args, Epi epi, cudaStream_t stream);

}  // namespace rserve
