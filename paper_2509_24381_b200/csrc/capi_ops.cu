// rserve-b200 — op-level C-ABI entry points (parity tests and micro-bench).
//
// Each op takes raw device pointers and runs ONE of the product kernels on
// the given stream; tests compare them against a plain fp32 reference.
#include <algorithm>
#include <cstring>
#include <vector>

#include "attention.cuh"
#include "common.cuh"
#include "gemm.cuh"
#include "host/status.hpp"
#include "kernels.cuh"
#include "model.cuh"
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
    a.b_stable = false;
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

rs_status rs_op_attention_varlen_tc(const void* qkv, int ld_qkv, void* out, int ld_out,
                                    const int* cu_seqlens, int n_seqs, int total, int heads,
                                    int head_dim, float scale, void* stream) {
  return guarded([&] {
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    std::vector<int> cu(static_cast<std::size_t>(n_seqs) + 1);
    RS_CUDA_CHECK(cudaMemcpyAsync(cu.data(), cu_seqlens, cu.size() * 4, cudaMemcpyDeviceToHost, st));
    RS_CUDA_CHECK(cudaStreamSynchronize(st));
    std::vector<AttnBlock> blocks;
    std::size_t s = 0;
    const int unit = attn_unit_rows();
    for (int r = 0; r < total; r += unit) {
      const int r1 = std::min(total, r + unit);
      while (s + 1 < cu.size() && cu[s + 1] <= r) ++s;
      std::size_t e = s;
      while (e + 1 < cu.size() && cu[e + 1] < r1) ++e;
      blocks.push_back({r, r1 - r, cu[s], cu[e + 1]});
    }
    const int rows_alloc = (total + 7) / 8 * 8;
    const std::size_t padded = static_cast<std::size_t>(rows_alloc) * heads * 128 * 2;
    void *qp, *kp, *vt, *pos, *bd;
    RS_CUDA_CHECK(cudaMallocAsync(&qp, padded, st));
    RS_CUDA_CHECK(cudaMallocAsync(&kp, padded, st));
    RS_CUDA_CHECK(cudaMallocAsync(&vt, padded, st));
    RS_CUDA_CHECK(cudaMallocAsync(&pos, static_cast<std::size_t>(total) * 8, st));
    RS_CUDA_CHECK(cudaMallocAsync(&bd, blocks.size() * sizeof(AttnBlock), st));
    RS_CUDA_CHECK(cudaMemsetAsync(qp, 0, padded, st));
    RS_CUDA_CHECK(cudaMemsetAsync(kp, 0, padded, st));
    RS_CUDA_CHECK(cudaMemsetAsync(vt, 0, padded, st));
    RS_CUDA_CHECK(cudaMemsetAsync(pos, 0, static_cast<std::size_t>(total) * 8, st));  // RoPE = id
    RS_CUDA_CHECK(cudaMemcpyAsync(bd, blocks.data(), blocks.size() * sizeof(AttnBlock),
                                  cudaMemcpyHostToDevice, st));
    void* table;
    RS_CUDA_CHECK(cudaMallocAsync(&table, static_cast<std::size_t>(total) * head_dim / 2 * sizeof(float2), st));
    vit_rope_table(static_cast<const std::int32_t*>(pos), total, head_dim, 10000.f,
                   static_cast<float2*>(table), st);
    vit_qkv_split(static_cast<const bf16*>(qkv), ld_qkv, static_cast<const float2*>(table), total,
                  heads, head_dim, static_cast<bf16*>(qp), static_cast<bf16*>(kp),
                  static_cast<bf16*>(vt), rows_alloc, st);
    RS_CUDA_CHECK(cudaFreeAsync(table, st));
    attention_varlen_tc(static_cast<bf16*>(qp), static_cast<bf16*>(kp), static_cast<bf16*>(vt),
                        rows_alloc, heads, static_cast<bf16*>(out), ld_out, head_dim,
                        static_cast<const AttnBlock*>(bd), blocks.data(), static_cast<int>(blocks.size()),
                        cu_seqlens, n_seqs, scale, st);
    RS_CUDA_CHECK(cudaStreamSynchronize(st));
    for (void* p : {qp, kp, vt, pos, bd}) RS_CUDA_CHECK(cudaFreeAsync(p, st));
  });
}

rs_status rs_op_attention_window_tc(const void* qkv, int ld_qkv, void* out, int ld_out,
                                    const int* cu_seqlens, int n_seqs, int total, int heads,
                                    int head_dim, float scale, const int* pos_hw, float rope_theta,
                                    void* stream) {
  return guarded([&] {
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    std::vector<int> cu(static_cast<std::size_t>(n_seqs) + 1);
    RS_CUDA_CHECK(cudaMemcpyAsync(cu.data(), cu_seqlens, cu.size() * 4, cudaMemcpyDeviceToHost, st));
    std::vector<std::int32_t> pos(static_cast<std::size_t>(total) * 2, 0);
    if (pos_hw != nullptr)
      RS_CUDA_CHECK(cudaMemcpyAsync(pos.data(), pos_hw, pos.size() * 4, cudaMemcpyDeviceToHost, st));
    RS_CUDA_CHECK(cudaStreamSynchronize(st));
    int max_window = 0, n_pos = 1;
    for (int i = 0; i < n_seqs; ++i) max_window = std::max(max_window, cu[i + 1] - cu[i]);
    for (std::int32_t v : pos) n_pos = std::max(n_pos, v + 1);
    if (!attention_window_tc_supported(head_dim, max_window, n_pos))
      throw lmmsim::InputError("rs_op_attention_window_tc: unsupported head_dim / window / positions");
    // the model's tile plan (finalize_plan): whole consecutive windows of <= 128 rows
    VitBatchPlan plan;
    plan.patches = total;
    plan.cu_window.assign(cu.begin(), cu.end());
    finalize_plan(plan);
    std::vector<std::uint8_t> buf(plan.win_blocks.size() * sizeof(AttnBlock) + plan.win_row.size() * 4);
    std::memcpy(buf.data(), plan.win_blocks.data(), plan.win_blocks.size() * sizeof(AttnBlock));
    std::memcpy(buf.data() + plan.win_blocks.size() * sizeof(AttnBlock), plan.win_row.data(),
                plan.win_row.size() * 4);
    void *bd, *posd, *freq;
    RS_CUDA_CHECK(cudaMallocAsync(&bd, buf.size(), st));
    RS_CUDA_CHECK(cudaMallocAsync(&posd, pos.size() * 4, st));
    RS_CUDA_CHECK(cudaMallocAsync(&freq, static_cast<std::size_t>(n_pos) * (head_dim / 4) * sizeof(float2), st));
    RS_CUDA_CHECK(cudaMemcpyAsync(bd, buf.data(), buf.size(), cudaMemcpyHostToDevice, st));
    RS_CUDA_CHECK(cudaMemcpyAsync(posd, pos.data(), pos.size() * 4, cudaMemcpyHostToDevice, st));
    vit_rope_freq_table(n_pos, head_dim, rope_theta, static_cast<float2*>(freq), st);
    double flops = 0;
    for (int i = 0; i < n_seqs; ++i) flops += 4.0 * (cu[i + 1] - cu[i]) * (cu[i + 1] - cu[i]) * head_dim * heads;
    attention_window_tc(static_cast<const bf16*>(qkv), ld_qkv, total, static_cast<bf16*>(out), ld_out,
                        static_cast<const AttnBlock*>(bd), static_cast<int>(plan.win_blocks.size()), heads,
                        head_dim, scale, static_cast<const std::int32_t*>(posd), static_cast<const float2*>(freq),
                        n_pos, flops, st);
    RS_CUDA_CHECK(cudaStreamSynchronize(st));
    for (void* p : {bd, posd, freq}) RS_CUDA_CHECK(cudaFreeAsync(p, st));
  });
}

rs_status rs_op_attention_prefill(const void* q, int ld_q, int rows_alloc, void* out, int ld_out,
                                  int q_pos0, int q_rows, const void* k_cache,
                                  const void* v_cache, long long kv_pages, const int* page_table,
                                  int q_heads, int kv_heads, int head_dim, float scale,
                                  void* stream) {
  return guarded([&] {
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    std::vector<PrefillWork> work;
    const int unit = attn_unit_rows();
    for (int r = 0; r < q_rows; r += unit)
      work.push_back({r, std::min(unit, q_rows - r), q_pos0 + r, 0});
    PrefillWork* wd = nullptr;
    const int** ptd = nullptr;
    RS_CUDA_CHECK(cudaMallocAsync(reinterpret_cast<void**>(&wd), work.size() * sizeof(PrefillWork), st));
    RS_CUDA_CHECK(cudaMallocAsync(reinterpret_cast<void**>(&ptd), sizeof(int*), st));
    RS_CUDA_CHECK(cudaMemcpyAsync(wd, work.data(), work.size() * sizeof(PrefillWork),
                                  cudaMemcpyHostToDevice, st));
    RS_CUDA_CHECK(cudaMemcpyAsync(ptd, &page_table, sizeof(int*), cudaMemcpyHostToDevice, st));
    PagedKV kv{const_cast<bf16*>(static_cast<const bf16*>(k_cache)),
               const_cast<bf16*>(static_cast<const bf16*>(v_cache)), ptd, 64};
    attention_prefill_paged_tc(static_cast<const bf16*>(q), ld_q, rows_alloc, static_cast<bf16*>(out),
                               ld_out, wd, work.data(), static_cast<int>(work.size()), q_pos0 + q_rows, kv, kv_pages, q_heads,
                               kv_heads, head_dim, scale, st);
    RS_CUDA_CHECK(cudaStreamSynchronize(st));  // host vectors above go out of scope
    RS_CUDA_CHECK(cudaFreeAsync(wd, st));
    RS_CUDA_CHECK(cudaFreeAsync(ptd, st));
  });
}

rs_status rs_op_attention_decode(const void* q, int ld_q, void* out, int ld_out, int n_req, const int* q_pos,
                                 const int* const* page_tables, const void* k_cache, const void* v_cache,
                                 int q_heads, int kv_heads, int head_dim, float scale, void* stream) {
  return guarded([&] {
    if (n_req <= 0) return;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    std::vector<PrefillWork> work;
    int max_keys = 0;
    for (int i = 0; i < n_req; ++i) {
      if (q_pos[i] < 0) throw lmmsim::ConfigError("rs_op_attention_decode: negative position");
      work.push_back({i, 1, q_pos[i], i});
      max_keys = std::max(max_keys, q_pos[i] + 1);
    }
    PrefillWork* wd = nullptr;
    const int** ptd = nullptr;
    RS_CUDA_CHECK(cudaMallocAsync(reinterpret_cast<void**>(&wd), work.size() * sizeof(PrefillWork), st));
    RS_CUDA_CHECK(cudaMallocAsync(reinterpret_cast<void**>(&ptd), n_req * sizeof(int*), st));
    RS_CUDA_CHECK(cudaMemcpyAsync(wd, work.data(), work.size() * sizeof(PrefillWork), cudaMemcpyHostToDevice, st));
    RS_CUDA_CHECK(cudaMemcpyAsync(ptd, page_tables, n_req * sizeof(int*), cudaMemcpyHostToDevice, st));
    PagedKV kv{const_cast<bf16*>(static_cast<const bf16*>(k_cache)),
               const_cast<bf16*>(static_cast<const bf16*>(v_cache)), ptd, 64};
    attention_decode_paged(static_cast<const bf16*>(q), ld_q, static_cast<bf16*>(out), ld_out, wd, n_req, max_keys,
                           kv, q_heads, kv_heads, head_dim, scale, st);
    RS_CUDA_CHECK(cudaStreamSynchronize(st));  // host vectors above go out of scope
    RS_CUDA_CHECK(cudaFreeAsync(wd, st));
    RS_CUDA_CHECK(cudaFreeAsync(ptd, st));
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
