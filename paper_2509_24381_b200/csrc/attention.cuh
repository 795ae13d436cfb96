// rserve-b200 — attention kernels.
//
// (a) ViT varlen bidirectional attention over packed QKV rows (window
//     layers: one sequence per 8x8-patch window; full layers: one sequence
//     per image), head_dim 64 / 80.
// (b) LLM causal chunked-prefill attention: the chunk's query rows (one or
//     more request slices) attend to their request's paged KV cache up to
//     their own position, GQA, head_dim 64 / 128.
// Both are flash-style (online softmax, fp32 statistics) on bf16 tensor-core
// MMAs with cp.async double-buffered K/V tiles.
#pragma once

#include <cuda_runtime.h>

#include "common.cuh"

namespace rserve {

/// rope_table (optional, [total, head_dim/2] float2 cos/sin per packed row):
/// q and k are rotated (rotate-half pairs) in shared memory after loading,
/// i.e. the ViT 2D RoPE fused into the attention.
void attention_varlen_bidir(const bf16* qkv, int ld_qkv, bf16* out, int ld_out,
                            const int* cu_seqlens, int n_seqs, int max_seqlen, int total,
                            int heads, int head_dim, float scale, cudaStream_t stream,
                            const float2* rope_table = nullptr);

// One unit of chunked-prefill attention work: up to attn_unit_rows() query
// rows of one slice.
struct PrefillWork {
  int q_row0;     // first chunk row of this block
  int q_rows;     // valid rows (<= attn_unit_rows())
  int q_pos0;     // prompt position of q_row0
  int req_slot;   // index into the per-request page-table array
};
constexpr int kPrefillRows = 128;
/// Query rows per tcgen05 attention work unit: 256 for the two-tile
/// ping-pong kernel (default), 128 for the single-tile kernel
/// (RS_ATTN_PINGPONG=0). Callers build PrefillWork / AttnBlock units of
/// this many rows.
int attn_unit_rows();

struct PagedKV {
  bf16* k;  // [pages][kv_heads][64 tokens][head_dim] for one layer
  bf16* v;  // TRANSPOSED: [pages][kv_heads][head_dim][64 tokens]
  const int* const* page_tables;  // device array: req_slot -> int* page ids
  int page_size;
};

/// A 128-row query block of packed varlen sequences and the key range it
/// may touch (the union of its rows' sequences).
struct AttnBlock {
  int q_row0, q_rows, key_begin, key_end;
};

/// tcgen05 varlen bidirectional attention (ViT). qp / kp: [rows_alloc,
/// heads*128] (head-padded, rotated); vt: [heads*128, rows_alloc] (V^T,
/// head-padded). out: [rows, heads*out_hd]. Visible keys of row t: its own
/// sequence [cu[s], cu[s+1]).
void attention_varlen_tc(const bf16* qp, const bf16* kp, const bf16* vt, int rows_alloc,
                         int heads, bf16* out, int ld_out, int out_hd, const AttnBlock* blocks,
                         const AttnBlock* blocks_host, int n_blocks, const int* cu_seqlens, int n_seqs,
                         float scale, cudaStream_t stream);

/// tcgen05 / TMA ViT window attention (attention_win.cu): qkv [rows, 3 H hd]
/// read in place (q | k | v head blocks), 2D RoPE applied to q / k from the
/// compact table freq [n_pos, hd/4] (cos, sin) at the rows' pos_hw [rows, 2];
/// tiles: whole consecutive windows of <= 128 rows, {q_row0, q_rows, first
/// window, windows} (finalize_plan), followed in the same device buffer by
/// [rows] u32 per-row windows as tile columns (lo | hi << 16); out
/// [rows, H hd]. flops: profiler label.
bool attention_window_tc_supported(int head_dim, int max_window, int n_pos);
void attention_window_tc(const bf16* qkv, int ld_qkv, int rows, bf16* out, int ld_out, const AttnBlock* tiles,
                         int n_tiles, int heads, int head_dim, float scale, const std::int32_t* pos_hw,
                         const float2* freq, int n_pos, double flops, cudaStream_t st);

/// Decode attention (one query row per work item, q_rows == 1, keys
/// [0, q_pos0]) over the paged KV: split along the keys, GQA-packed,
/// deterministic split merge (attention.cu). max_keys >= every item's keys.
void attention_decode_paged(const bf16* qkv, int ld_q, bf16* out, int ld_out, const PrefillWork* work,
                            int n_req, int max_keys, const PagedKV& kv, int q_heads, int kv_heads,
                            int head_dim, float scale, cudaStream_t st);

/// tcgen05 / TMEM flash attention (attention_tc.cu). q: packed QKV rows of
/// the chunk ([q_rows_alloc, (Hq + 2 Hkv) hd], q columns first); work /
/// blocks: device list, *_host: the same list on the host (inlined into the
/// kernel parameters). max_keys:
/// the longest item's key count (0: unknown); with few (item, head) units and
/// long keys the keys are split over more CTAs and merged (split-KV).
void attention_prefill_paged_tc(const bf16* q, int ld_q, int q_rows_alloc, bf16* out, int ld_out,
                                const PrefillWork* work, const PrefillWork* work_host, int n_work,
                                int max_keys, const PagedKV& kv, std::int64_t kv_pages, int q_heads,
                                int kv_heads, int head_dim, float scale, cudaStream_t stream);

/// Frees the per-stream attention workspaces (split-KV partials) of a stream
/// that is about to be destroyed.
void attention_tc_release_stream(cudaStream_t st);
void attention_release_stream(cudaStream_t st);

}  // namespace rserve
