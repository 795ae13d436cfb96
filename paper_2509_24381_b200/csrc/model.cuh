// rserve-b200 — Qwen2.5-VL-shaped vision encoder + decoder LLM on the B200.
//
// The reference has no model; these are the computations that
// stand behind its cost seam: encode_time_ms (cost_model.hpp:68-71) is one
// Vit::encode of an Algorithm-1 batch, stage_time_ms (76-82) is one
// Llm::forward_stage of a micro-batch over this stage's layers.
//
// Weights are random-init from seeded hashes (kernels.cuh mix64), laid out
// for the kernels: every linear is [out, in] K-major bf16; SwiGLU gate/up
// rows are interleaved in 16-row blocks; widths that TMA cannot stride
// (ViT ff 3420) are zero-padded to a multiple of 16 (3424) — mathematically
// identical. oracle/model_oracle.py regenerates the same values.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "attention.cuh"
#include "common.cuh"
#include "gemm.cuh"
#include "kernels.cuh"
#include "rserve.h"

namespace rserve {

struct Shapes {
  rs_model_config cfg{};
  // ViT
  int vd = 0, vl = 0, vh = 0, vhd = 0, vff = 0, vff_pad = 0, win = 0, full_every = 0, pdim = 0;
  int merge_in = 0;  // 4 * vd
  // LLM
  int d = 0, L = 0, hq = 0, hkv = 0, hd = 0, ff = 0, vocab = 0, qkv_dim = 0;
  float eps = 1e-6f;

  static Shapes from(const rs_model_config& c);
  bool full_attention_layer(int l) const { return full_every > 0 && (l % full_every) == full_every - 1; }
};

/// Hash stream ids of every synthetic tensor (shared with the oracle).
namespace wid {
constexpr std::uint64_t kVit = 1, kMerger = 2, kLlm = 3, kTop = 4;
inline std::uint64_t id(std::uint64_t comp, std::uint64_t layer, std::uint64_t t) {
  return (comp << 32) | (layer << 8) | t;
}
// tensor indices
enum : std::uint64_t {
  kQkvW = 1, kQkvB = 2, kOW = 3, kOB = 4, kGateW = 5, kGateB = 6, kUpW = 7, kUpB = 8,
  kDownW = 9, kDownB = 10, kPatch = 11, kFc1W = 12, kFc1B = 13, kFc2W = 14, kFc2B = 15,
  kEmbed = 16, kHead = 17
};
}  // namespace wid
constexpr float kWeightScale = 0.0346410162f;  // uniform +-a has std 0.02
constexpr float kPixelScale = 1.7320508076f;   // unit-variance uniform

struct VitLayer {
  bf16 *ln1, *qkv_w, *qkv_b, *o_w, *o_b, *ln2, *gu_w, *gu_b, *down_w, *down_b;
};
struct LlmLayer {
  bf16 *ln1, *qkv_w, *qkv_b, *o_w, *ln2, *gu_w, *down_w;
  bf16 *k_cache, *v_cache;  // [pages][hkv][page][hd]
};

/// Device buffers owned by a context; freed together.
class DeviceArena {
 public:
  ~DeviceArena();
  void* alloc(std::size_t bytes);
  std::size_t bytes() const { return total_; }

 private:
  std::vector<void*> blocks_;
  std::size_t total_ = 0;
};

struct VitBatchPlan {  // host-side metadata of one encode batch
  int patches = 0, tokens = 0;
  std::vector<std::int32_t> pos_hw;     // [P, 2]
  std::vector<std::int32_t> cu_window;  // window sequences
  std::vector<std::int32_t> cu_item;    // image sequences
  std::vector<std::int32_t> out_row;    // merged row (window-major) -> output row (LLM order)
  int max_window = 0, max_item = 0;
  std::vector<AttnBlock> win_blocks, full_blocks;  // tcgen05 attention work (finalize_plan)
  std::vector<std::uint32_t> win_row;  // [P] window of each row as columns of its win_blocks tile (lo | hi << 16)
};

/// 128-row attention blocks for the window and full-attention layers.
void finalize_plan(VitBatchPlan& plan);

/// Merged-token grid of an item of `tokens` LLM tokens: (gh, gw), gh <= gw.
void item_grid(std::uint64_t tokens, int* gh, int* gw);
/// Window-major patch order of one item; appends to `plan`.
void plan_item(int gh, int gw, int window, int out_row_base, VitBatchPlan& plan);

/// Patch positions (per axis) covered by the ViT's compact 2D-RoPE table.
constexpr int kVitRopePositions = 512;

class Vit {
 public:
  void init(const Shapes& s, DeviceArena& arena, int max_patches, cudaStream_t st);
  /// patches [P, pdim] bf16 (device) -> out [tokens, d_llm] (LLM row order).
  /// meta_dev: uploaded VitBatchPlan arrays (see encode_meta_bytes()).
  void encode(const VitBatchPlan& plan, const bf16* patches, const std::int32_t* pos_hw_dev,
              const std::int32_t* cu_window_dev, const std::int32_t* cu_item_dev,
              const std::int32_t* out_row_dev, const AttnBlock* win_blocks_dev,
              const AttnBlock* full_blocks_dev, bf16* out, cudaStream_t st);
  std::uint64_t flops_per_batch(const VitBatchPlan& plan) const;
  int max_patches() const { return max_p_; }

 private:
  Shapes s_;
  int max_p_ = 0;
  bf16* patch_w_ = nullptr;
  std::vector<VitLayer> layers_;
  bf16 *merger_ln_ = nullptr, *fc1_w_ = nullptr, *fc1_b_ = nullptr, *fc2_w_ = nullptr,
       *fc2_b_ = nullptr;
  // activations
  bf16 *x_ = nullptr, *xn_ = nullptr, *qkv_ = nullptr, *att_ = nullptr, *h_ = nullptr,
       *mh_ = nullptr;
  bf16 *qp_ = nullptr, *kp_ = nullptr, *vt_ = nullptr;  // head-padded tcgen05 attention operands
  // folded RMSNorm: unit weight for the explicit norms (the layers' norm
  // weights live in their consumer GEMMs' columns) and the per-row sums of
  // squares handed from residual GEMMs to norm consumers (ping-pong)
  bf16* unit_ln_ = nullptr;
  unsigned long long *ss_a_ = nullptr, *ss_b_ = nullptr;  // [max patches], 2^-16 fixed point
  float2* rope_table_ = nullptr;                         // [P, hd/2] cos/sin, per batch
  float2* rope_freq_ = nullptr;                          // [kVitRopePositions, hd/4] cos/sin per (position, freq)
};

/// Per-chunk device descriptor (uploaded before a stage runs).
struct ChunkDev {
  const ChunkRowInfo* rows = nullptr;
  const std::int64_t* gather_rows = nullptr;  // slab rows (first stage)
  const PrefillWork* work = nullptr;
  const PrefillWork* work_host = nullptr;  // same list on the host (alive during the launches)
  int n_work = 0;
  int M = 0;
  const std::int64_t* done_rows = nullptr;    // chunk rows that end a prompt
  const std::int32_t* done_slots = nullptr;   // their logits-table slots
  int n_done = 0;
  bool decode = false;  // one row per work item (decode step): split-KV decode attention
  int max_keys = 0;     // longest key range (prefill: picks the attention KV split)
};

class Llm {
 public:
  /// tp_size > 1: this object is tensor-parallel shard tp_rank (SURVEY §8
  /// f4): q / kv heads and the SwiGLU width split T ways, O / down by input
  /// columns; weights are the exact slices of the full (hashed) tensors.
  void init(const Shapes& s, DeviceArena& arena, int layer_begin, int layer_end, bool with_embed,
            bool with_head, int max_chunk, std::int64_t kv_pages, int page_size,
            int logits_slots, cudaStream_t st, int tp_rank = 0, int tp_size = 1);
  /// Tensor-parallel layer phases (tp_forward in device_context.cu drives all
  /// shards): attention block -> this shard's O-projection partial [M, d];
  /// MLP block -> this shard's down-projection partial. The residual stream x
  /// is read (never written) and normalised on the fly from ss (the previous
  /// reduction's sums of squares) or explicitly on the stage's first layer.
  void tp_attn_partial(int layer, const ChunkDev& c, const bf16* slab, bf16* x, bool first,
                       const unsigned long long* ss, const int* const* page_tables, bf16* part,
                       cudaStream_t st);
  void tp_mlp_partial(int layer, const ChunkDev& c, const bf16* x, const unsigned long long* ss,
                      bf16* part, cudaStream_t st);
  /// QKV GEMM + M-RoPE + KV append (fused epilogue for chunks).
  void qkv_rope_append(GemmArgs g, const ChunkDev& c, const LlmLayer& L, const int* const* page_tables,
                       cudaStream_t st);
  /// Per-chunk setup of a tensor-parallel pass (the M-RoPE table).
  void tp_begin(const ChunkDev& c, cudaStream_t st);
  /// Final norm + LM head + argmax for the rows of c that end a prompt.
  void head_phase(const ChunkDev& c, const bf16* x, cudaStream_t st);
  const Shapes& shapes() const { return s_; }
  /// One micro-batch through layers [begin, end). x: [M, d] residual stream
  /// (in/out). First stage: x is gathered from the embedding slab.
  void forward_stage(const ChunkDev& c, const bf16* slab, bf16* x, const int* const* page_tables,
                     cudaStream_t st, int layer_from = -1, int layer_to = -1);
  const bf16* embed() const { return embed_; }
  float* logits_row(int slot) { return logits_ + static_cast<std::int64_t>(slot) * s_.vocab; }
  std::int32_t* argmax_dev() { return argmax_; }
  int layer_begin() const { return lb_; }
  int layer_end() const { return le_; }
  bool has_head() const { return head_ != nullptr; }
  /// Paged KV of local layer l in [layer_begin, layer_end): K [pages][hkv][page][hd],
  /// V^T [pages][hkv][hd][page] (this shard's kv heads).
  bf16* k_cache(int l) const { return layers_[static_cast<std::size_t>(l - lb_)].k_cache; }
  bf16* v_cache(int l) const { return layers_[static_cast<std::size_t>(l - lb_)].v_cache; }
  std::uint64_t dense_flops(std::uint64_t tokens) const;

 private:
  Shapes s_;
  int lb_ = 0, le_ = 0, page_size_ = 64;
  std::int64_t kv_pages_ = 0;
  bf16* embed_ = nullptr;
  std::vector<LlmLayer> layers_;
  bf16 *final_ln_ = nullptr, *head_ = nullptr;
  bf16 *xn_ = nullptr, *qkv_ = nullptr, *att_ = nullptr, *h_ = nullptr, *xf_ = nullptr;
  bf16* unit_ln_ = nullptr;                  // folded RMSNorm (see Vit)
  float2* rope_table_ = nullptr;             // [max chunk, hd/2] M-RoPE cos/sin of the chunk
  unsigned long long *ss_a_ = nullptr, *ss_b_ = nullptr;
  float* logits_ = nullptr;
  std::int32_t* argmax_ = nullptr;
  float* head_scratch_ = nullptr;
  int max_m_ = 0, slots_ = 0;
};

}  // namespace rserve
