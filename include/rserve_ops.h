/* rserve-b200 — op-level C-ABI: one product kernel per call, raw device
 * pointers, explicit cudaStream_t (passed as void*; NULL = legacy default).
 * Used by the parity tests (tests/test_ops_gpu.py) and the micro-benchmarks.
 * These ops have no reference counterpart (the reference has no device
 * code); each one implements a piece of the work hidden
 * behind encode_time_ms / stage_time_ms (cost_model.hpp:68-82).           */
#ifndef RSERVE_OPS_H_
#define RSERVE_OPS_H_

#include "rserve.h"

#ifdef __cplusplus
extern "C" {
#endif

enum { RS_EPI_STORE = 0, RS_EPI_RESIDUAL = 1, RS_EPI_SWIGLU = 2, RS_EPI_GELU = 3,
       RS_EPI_STORE_F32 = 4 };

/* C[M,N] = epi(A[M,K] . B[N,K]^T) on tcgen05 (K-major bf16 operands). */
RS_API rs_status rs_op_gemm(const void* A, int lda, const void* B, int ldb, void* C, int ldc,
                     const void* bias, const void* residual, int ldr, const int* row_map,
                     int M, int N, int K, int epi, int force_bn, void* stream);
/* y = rmsnorm(x) * w (Qwen2 semantics: fp32 normalise, bf16 cast, scale). */
RS_API rs_status rs_op_rmsnorm(const void* x, int ldx, const void* w, void* y, int ldy, int rows,
                        int dim, float eps, void* stream);
/* Varlen bidirectional attention over packed QKV [total, 3*heads*hd]. */
RS_API rs_status rs_op_attention_varlen(const void* qkv, int ld_qkv, void* out, int ld_out,
                                 const int* cu_seqlens, int n_seqs, int max_seqlen, int total,
                                 int heads, int head_dim, float scale, void* stream);
/* Same contract as rs_op_attention_varlen, on the tcgen05 path used by the
 * ViT (head-padded operands built by vit_qkv_split with identity RoPE).
 * Synchronous. */
RS_API rs_status rs_op_attention_varlen_tc(const void* qkv, int ld_qkv, void* out, int ld_out,
                                           const int* cu_seqlens, int n_seqs, int total,
                                           int heads, int head_dim, float scale, void* stream);
/* ViT window attention on the tcgen05 / TMA kernel the encoder runs
 * (attention_win.cu): Q / K / V read in place from packed QKV, windows of
 * <= 128 rows (cu_seqlens, device int32), 2D RoPE (theta) applied to q / k at
 * pos_hw (device int32 [total, 2] = (h, w) per row; NULL = identity).
 * Synchronous. */
RS_API rs_status rs_op_attention_window_tc(const void* qkv, int ld_qkv, void* out, int ld_out,
                                           const int* cu_seqlens, int n_seqs, int total, int heads,
                                           int head_dim, float scale, const int* pos_hw,
                                           float rope_theta, void* stream);
/* Causal chunked-prefill attention (tcgen05) of ONE slice: q rows
 * [0, q_rows) at prompt positions q_pos0.. attend to keys [0, q_pos0+q_rows)
 * of a paged cache: K [pages][kv_heads][64][hd], V^T [pages][kv_heads][hd][64],
 * page_table (device int32) maps key page -> cache page. Synchronous. */
RS_API rs_status rs_op_attention_prefill(const void* q, int ld_q, int rows_alloc, void* out,
                                         int ld_out, int q_pos0, int q_rows, const void* k_cache,
                                         const void* v_cache, long long kv_pages,
                                         const int* page_table, int q_heads, int kv_heads,
                                         int head_dim, float scale, void* stream);
/* Decode attention: q row i (one token of request i, at prompt position
 * q_pos[i], host array) attends keys [0, q_pos[i]] of the paged cache through
 * page_tables[i] (host array of n_req device int32 page tables); GQA with
 * q_heads / kv_heads <= 16, head_dim 64 or 128. Synchronous. */
RS_API rs_status rs_op_attention_decode(const void* q, int ld_q, void* out, int ld_out, int n_req,
                                        const int* q_pos, const int* const* page_tables, const void* k_cache,
                                        const void* v_cache, int q_heads, int kv_heads, int head_dim,
                                        float scale, void* stream);
/* Kernel launches issued by this process so far (our kernels only). */
RS_API unsigned long long rs_kernel_launches(void);
/* Live per-kernel-class timing: CUDA events recorded on each launch stream
 * around our kernels while enabled. drain -> lines
 * "<class> <launches> <ms> <algorithmic flops> <algorithmic bytes>". */
RS_API rs_status rs_profile_enable(int on);
RS_API rs_status rs_profile_drain(char** out_text);

#ifdef __cplusplus
}
#endif
#endif /* RSERVE_OPS_H_ */
