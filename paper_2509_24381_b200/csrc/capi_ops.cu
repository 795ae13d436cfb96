// rserve-b200 — op-level C-ABI entry points (parity tests and micro-bench).
//
// Each op takes raw device pointers and runs ONE of the product kernels on
// the given stream; tests compare them against a plain fp32 reference.
#include "attention.cuh"
#include "common.cuh"
#include "gemm.cuh"
#include "host/status.hpp"
#include "kernels.cuh"
#include "rserve_ops.h"

using namespace rserve;

extern "C" {

rs_status rs_op_gemm(const void* A, int lda, const void* B, int ldb, void* C, int ldc,
                     const void* bias, const void* residual, int ldr, const int* row_map, int M,
                     int N, int K, int epi, int force_bn, void* stream) {
  return guarded([&] {
    GemmArgs a;
    a.A = static_cast<const bf16*>(A);
    a.lda = lda;
    a.B = static_cast<const bf16*>(B);
    a.ldb = ldb;
    a.C = C;
    a.ldc = ldc;
    a.bias = static_cast<const bf16*>(bias);
    a.residual = static_cast<const bf16*>(residual);
    a.ldr = ldr;
    a.row_map = row_map;
    a.M = M;
    a.N = N;
    a.K = K;
    gemm(a, static_cast<Epi>(epi), static_cast<cudaStream_t>(stream), force_bn);
  });
}

rs_status rs_op_rmsnorm(const void* x, int ldx, const void* w, void* y, int ldy, int rows,
                        int dim, float eps, void* stream) {
  return guarded([&] {
    rmsnorm(static_cast<const bf16*>(x), ldx, static_cast<const bf16*>(w), static_cast<bf16*>(y),
            ldy, rows, dim, eps, static_cast<cudaStream_t>(stream));
  });
}

rs_status rs_op_attention_varlen(const void* qkv, int ld_qkv, void* out, int ld_out,
                                 const int* cu_seqlens, int n_seqs, int max_seqlen, int total,
                                 int heads, int head_dim, float scale, void* stream) {
  return guarded([&] {
    attention_varlen_bidir(static_cast<const bf16*>(qkv), ld_qkv, static_cast<bf16*>(out),
                           ld_out, cu_seqlens, n_seqs, max_seqlen, total, heads, head_dim, scale,
                           static_cast<cudaStream_t>(stream));
  });
}

unsigned long long rs_kernel_launches(void) { return launches_so_far(); }

rs_status rs_profile_enable(int on) {
  return guarded([&] { prof::enable(on != 0); });
}

rs_status rs_profile_drain(char** out_text) {
  return guarded([&] { *out_text = c_string(prof::drain()); });
}

}  // extern "C"
