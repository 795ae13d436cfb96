// rserve-b200 — memory-bound kernels of the pipeline (HBM roofline):
// norms, rotary embeddings, paged-KV append, the embedding-tracker data
// plane (K6 scatter + bitmap, K7 ready prefix, K8 text gather, chunk
// gather), LM-head helpers and the seeded weight / payload generators.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "common.cuh"

namespace rserve {

// ---- deterministic synthetic values (mirrored by oracle/model_oracle.py) ----
// u = splitmix64(seed*G + stream*H + i) >> 40, scaled to [0, 1) with 24 bits.
__host__ __device__ inline std::uint64_t mix64(std::uint64_t seed, std::uint64_t stream,
                                               std::uint64_t i) {
  std::uint64_t z = seed * 0x9E3779B97F4A7C15ull + stream * 0xD1B54A32D192ED03ull + i;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

/// dst[i] = bf16((2u - 1) * scale) (+ offset), i < n, row-padded: element
/// (r, c) of a [rows, cols] tensor stored with stride ld; c >= cols -> 0.
/// The hash index is r * cols + c (independent of padding).
void fill_uniform(bf16* dst, std::int64_t rows, int cols, int ld, std::uint64_t seed,
                  std::uint64_t stream, float scale, float offset, cudaStream_t st);
/// SwiGLU weight layout: logical rows r < rows_valid of a [rows_pad, cols]
/// gate (which = 0) or up (which = 1) matrix land at interleaved row
/// (r / 16) * 32 + which * 16 + r % 16 of the [2 * rows_pad, ld] buffer;
/// padding rows are zero. Hash index = r * cols + c, as for fill_uniform.
void fill_uniform_interleaved(bf16* dst, int rows_valid, int rows_pad, int cols, int ld,
                              std::uint64_t seed, std::uint64_t stream, float scale, int which,
                              cudaStream_t st, int row0 = 0);
/// fill_uniform of the sub-block [row0, row0+rows) x [col0, col0+cols) of a
/// [*, cols_full] tensor (hash index (row0 + r) * cols_full + col0 + c):
/// tensor-parallel shards generate exactly their slice of the full weight.
void fill_uniform_slice(bf16* dst, std::int64_t rows, int cols, int ld, std::uint64_t seed,
                        std::uint64_t stream, float scale, std::int64_t row0, int col0, int cols_full,
                        cudaStream_t st);
void fill_const(bf16* dst, std::int64_t n, float v, cudaStream_t st);
/// Folds an RMSNorm weight into the consumer linear: W[r, c] *= g[c]
/// ([rows, cols] with row stride ld), so the GEMM may read the
/// un-normalised stream and apply the per-row rsqrt scale in its epilogue.
void fold_norm_weight(bf16* W, std::int64_t rows, int cols, int ld, const bf16* g, cudaStream_t st);
/// int32 ids in [0, modulo): id = mix64(seed, stream, i) % modulo.
void fill_ids(std::int32_t* dst, std::int64_t n, std::uint64_t seed, std::uint64_t stream,
              std::uint32_t modulo, cudaStream_t st);

// ---- norms -------------------------------------------------------------------
/// y[m] = x[src(m)] * rsqrt(mean(x^2) + eps) * w ; src(m) = row_map ? row_map[m] : m.
/// When x_copy != null the raw source row is also copied to x_copy[m].
void rmsnorm(const bf16* x, int ldx, const bf16* w, bf16* y, int ldy, int rows, int dim,
             float eps, cudaStream_t st, const std::int64_t* row_map = nullptr,
             bf16* x_copy = nullptr, int ld_copy = 0, const int* rows_dev = nullptr);

// ---- rotary --------------------------------------------------------------------
/// ViT 2D RoPE in place on packed QKV rows [P, 3*H*hd]: q and k of every
/// head; pair (i, i + hd/2) rotated by pos_h * f_i (i < hd/4) or
/// pos_w * f_{i - hd/4}, f_j = theta^(-4j/hd). pos: [P, 2] (h, w).
void rope_vit(bf16* qkv, int ld, const std::int32_t* pos_hw, int rows, int heads, int hd,
              float theta, cudaStream_t st);

/// ViT attention operands: 2D RoPE on q, k of packed QKV rows [P, 3*H*hd]
/// (as rope_vit) written head-padded to 128 columns into qp / kp
/// [P, H*128], and V transposed into vt [H*128, ld_vt] (row h*128+d, column
/// = token). Pad columns / rows are never written (zero-initialised once).
void vit_qkv_split(const bf16* qkv, int ld, const float2* rope_table, int rows, int heads, int hd,
                   bf16* qp, bf16* kp, bf16* vt, int ld_vt, cudaStream_t st);
/// cos / sin table [rows, hd/2] of the ViT 2D RoPE (shared by all layers).
/// ViT q / k RoPE in place on the packed qkv rows (window layers, whose
/// attention reads qkv directly).
void vit_qk_rope_inplace(bf16* qkv, int ld, const float2* rope_table, int rows, int heads, int hd,
                         cudaStream_t st);
/// Compact ViT 2D-RoPE table: out[pos * (hd/4) + j] = (cos, sin)(pos * theta^(-4j/hd))
/// for pos < n_pos — the same values vit_rope_table stores per row and pair.
void vit_rope_freq_table(int n_pos, int hd, float theta, float2* out, cudaStream_t st);
void vit_rope_table(const std::int32_t* pos_hw, int rows, int hd, float theta, float2* table,
                    cudaStream_t st);

struct ChunkRowInfo {  // one chunk row (prefill token)
  std::int32_t req_slot;  // per-request tables index
  std::int32_t pos;       // prompt position (KV index)
  std::int32_t rope[3];   // M-RoPE (t, h, w) position ids
  std::int32_t pad;
};
/// LLM M-RoPE on q and k of packed QKV rows [M, (Hq + 2 Hkv) hd], then the
/// rotated k and v are appended to the paged KV cache of the row's request.
/// Sections over the hd/2 frequency pairs: t [0, hd/8), h [hd/8, 5hd/16),
/// w [5hd/16, hd/2) (Qwen2-VL mrope_section [16, 24, 24] at hd = 128).
/// table (optional): the chunk's [rows, hd/2] (cos, sin) from mrope_table(),
/// computed once per chunk instead of once per layer.
void rope_kv_append(bf16* qkv, int ld, const ChunkRowInfo* rows_info, int rows, int q_heads,
                    int kv_heads, int hd, float theta, bf16* k_cache, bf16* v_cache,
                    const int* const* page_tables, int page_size, cudaStream_t st,
                    const int* rows_dev = nullptr, const float2* table = nullptr);
/// Tensor-parallel reduction of the residual stream: x[m] += sum_t parts[t][m]
/// (fp32, in shard order: identical on every shard), and ss[m] += sum of
/// squares of the new bf16 row (2^-16 fixed point) for the folded norm.
/// parts: device array of `n_parts` pointers to [rows, d] bf16.
void tp_reduce_residual(bf16* x, int rows, int d, bf16* const* parts, int n_parts, unsigned long long* ss,
                        cudaStream_t st);
/// Tensor-parallel group reduction over peer memory: T ranks
/// (one per GPU over NVSwitch, or contexts sharing a GPU) each hold their O /
/// down partial in an exchange buffer every rank can address. Every block
/// signals each rank (release, system scope) that this rank's partial of
/// `epoch` is complete, waits for all ranks' signals of the same block
/// (acquire), then reduces its rows reading the T partials in rank order:
/// x += sum_t parts[t] and ss = sum of squares of the new bf16 row — the same
/// bits on every rank. No NCCL: the reads go straight over NVLink.
constexpr int kMaxTpRanks = 8;
constexpr int kTpBlocks = 64;  // reduce grid (flag slots per rank: kTpBlocks x kMaxTpRanks)
struct TpGroupArgs {
  bf16* x;
  int rows, d, T, rank;
  unsigned epoch;
  const bf16* parts[kMaxTpRanks];  // this phase's partial of each rank
  unsigned* flags[kMaxTpRanks];    // each rank's flag slots [kTpBlocks][kMaxTpRanks]
  unsigned long long* ss;
};
void tp_group_reduce(const TpGroupArgs& a, cudaStream_t st);
/// M-RoPE (cos, sin) of every chunk row and rotary frequency: [rows, hd/2].
void mrope_table(const ChunkRowInfo* rows_info, int rows, int hd, float theta, float2* table,
                 cudaStream_t st);

// ---- embedding tracker data plane (K6 / K7 / K8) ----------------------------------
/// K6: dst rows (slot rows of the slab) <- src rows, d bf16 each; and set
/// readiness bits [bit_begin[i], bit_end[i]) of `bitmap` for n_ranges ranges.
void scatter_rows_and_mark(const bf16* src, int n_rows, const std::int64_t* dst_rows, bf16* slab,
                           int d, std::uint32_t* bitmap, const std::uint64_t* ranges,
                           int n_ranges, cudaStream_t st);
/// K7: first clear bit at or after `frontier` (capped at total) -> *out.
void ready_prefix(const std::uint32_t* bitmap, std::uint64_t frontier, std::uint64_t total,
                  std::uint64_t* out, cudaStream_t st);
/// K8: slab[dst_rows[i]] <- vocab[ids[i]] for n text tokens.
void gather_text_embeddings(const bf16* vocab, const std::int32_t* ids, int n,
                            const std::int64_t* dst_rows, bf16* slab, int d, cudaStream_t st);
/// out[i] = src[idx[i]], i < n (decode: per-request argmax of the logits table).
void gather_slots_i32(const std::int32_t* src, const std::int32_t* idx, int n, std::int32_t* out,
                      cudaStream_t st);
/// Set bits [begin, end) for n ranges (text ranges at creation).
void bitmap_set_ranges(std::uint32_t* bitmap, const std::uint64_t* ranges, int n_ranges,
                       cudaStream_t st);

// ---- PD KV transfer -------------------------------------------------------------------
struct PageCopy {  // one KV page: src -> dst, page_bytes each (16-byte aligned)
  const void* src;
  void* dst;
};
/// Copies n pages of page_bytes (multiple of 16) — the KV image pack / unpack
/// (one CTA per page, 16-byte vector loads: HBM-bound). label: profiler class.
void copy_pages(const PageCopy* list_dev, int n, std::size_t page_bytes, cudaStream_t st, const char* label);

// ---- LM head helpers ---------------------------------------------------------------------
/// out[row(i)] = argmax(logits[row(i), :vocab]) (first max); row(i) =
/// rows_idx ? rows_idx[i] : i.
void argmax_rows(const float* logits, int rows, int vocab, std::int32_t* out, cudaStream_t st,
                 const std::int32_t* rows_idx = nullptr);

}  // namespace rserve
