// rserve-b200 — model weights + ViT / LLM forward passes (see model.cuh).
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "attention.cuh"
#include "gemm.cuh"
#include "kernels.cuh"
#include "model.cuh"

namespace rserve {

// ---- shapes -----------------------------------------------------------------------
Shapes Shapes::from(const rs_model_config& c) {
  Shapes s;
  s.cfg = c;
  s.vd = c.vit_dim;
  s.vl = c.vit_layers;
  s.vh = c.vit_heads;
  s.vhd = c.vit_heads > 0 ? c.vit_dim / c.vit_heads : 0;
  s.vff = c.vit_ff;
  s.vff_pad = (c.vit_ff + 15) / 16 * 16;
  s.win = c.vit_window;
  s.full_every = c.vit_fullatt_every;
  s.pdim = c.patch_dim;
  s.merge_in = 4 * c.vit_dim;
  s.d = c.llm_dim;
  s.L = c.llm_layers;
  s.hq = c.llm_q_heads;
  s.hkv = c.llm_kv_heads;
  s.hd = c.llm_head_dim;
  s.ff = c.llm_ff;
  s.vocab = c.vocab;
  s.qkv_dim = (c.llm_q_heads + 2 * c.llm_kv_heads) * c.llm_head_dim;
  s.eps = c.rms_eps;
  if (s.d % 256 != 0 && s.d % 8 != 0) throw lmmsim::ConfigError("model: llm_dim must be a multiple of 8");
  if (s.ff % 16 != 0) throw lmmsim::ConfigError("model: llm_ff must be a multiple of 16");
  if (s.hq % s.hkv != 0) throw lmmsim::ConfigError("model: q heads must be a multiple of kv heads");
  return s;
}

// ---- arena ------------------------------------------------------------------------
DeviceArena::~DeviceArena() {
  for (void* p : blocks_) cudaFree(p);
}
void* DeviceArena::alloc(std::size_t bytes) {
  void* p = nullptr;
  bytes = (bytes + 255) / 256 * 256;
  RS_CUDA_CHECK(cudaMalloc(&p, bytes));
  blocks_.push_back(p);
  total_ += bytes;
  return p;
}

namespace {
bf16* alloc_bf16(DeviceArena& a, std::int64_t n) {
  return static_cast<bf16*>(a.alloc(static_cast<std::size_t>(n) * sizeof(bf16)));
}
// [rows, cols] linear weight, row stride ld (>= cols, zero-padded).
bf16* make_linear(DeviceArena& a, std::int64_t rows, int cols, int ld, std::uint64_t seed,
                  std::uint64_t stream, cudaStream_t st) {
  bf16* w = alloc_bf16(a, rows * ld);
  fill_uniform(w, rows, cols, ld, seed, stream, kWeightScale, 0.f, st);
  return w;
}
bf16* make_ones(DeviceArena& a, int n, cudaStream_t st) {
  bf16* w = alloc_bf16(a, n);
  fill_const(w, n, 1.f, st);
  return w;
}
// Interleaved gate/up weight [2*ff_pad, ld] (+ bias [2*ff_pad] when requested).
bf16* make_gate_up(DeviceArena& a, int ff, int ff_pad, int cols, int ld, std::uint64_t seed,
                   std::uint64_t gate_id, std::uint64_t up_id, cudaStream_t st) {
  bf16* w = alloc_bf16(a, 2LL * ff_pad * ld);
  fill_uniform_interleaved(w, ff, ff_pad, cols, ld, seed, gate_id, kWeightScale, 0, st);
  fill_uniform_interleaved(w, ff, ff_pad, cols, ld, seed, up_id, kWeightScale, 1, st);
  return w;
}
}  // namespace

// ---- vision batch planning --------------------------------------------------------
void item_grid(std::uint64_t tokens, int* gh, int* gw) {
  int best = 1;
  for (std::uint64_t h = 1; h * h <= tokens; ++h)
    if (tokens % h == 0) best = static_cast<int>(h);
  *gh = best;
  *gw = static_cast<int>(tokens / static_cast<std::uint64_t>(best));
}

void plan_item(int gh, int gw, int window, int out_row_base, VitBatchPlan& plan) {
  const int p_base = plan.patches;
  plan.cu_item.push_back(p_base + 4 * gh * gw);
  plan.max_item = std::max(plan.max_item, 4 * gh * gw);
  for (int wy = 0; wy < gh; wy += window) {
    for (int wx = 0; wx < gw; wx += window) {
      const int y1 = std::min(gh, wy + window), x1 = std::min(gw, wx + window);
      for (int r = wy; r < y1; ++r) {
        for (int c = wx; c < x1; ++c) {
          plan.out_row.push_back(out_row_base + r * gw + c);
          for (int dy = 0; dy < 2; ++dy)
            for (int dx = 0; dx < 2; ++dx) {
              plan.pos_hw.push_back(2 * r + dy);
              plan.pos_hw.push_back(2 * c + dx);
            }
        }
      }
      plan.patches += 4 * (y1 - wy) * (x1 - wx);
      plan.cu_window.push_back(plan.patches);
      plan.max_window = std::max(plan.max_window, 4 * (y1 - wy) * (x1 - wx));
    }
  }
  plan.tokens += gh * gw;
}

// ---- ViT --------------------------------------------------------------------------
void Vit::init(const Shapes& s, DeviceArena& a, int max_patches, cudaStream_t st) {
  s_ = s;
  max_p_ = max_patches;
  const std::uint64_t seed = s.cfg.weight_seed;
  using namespace wid;
  patch_w_ = make_linear(a, s.vd, s.pdim, s.pdim, seed, id(kVit, 0, kPatch), st);
  layers_.resize(static_cast<std::size_t>(s.vl));
  for (int l = 0; l < s.vl; ++l) {
    VitLayer& L = layers_[static_cast<std::size_t>(l)];
    const std::uint64_t lid = static_cast<std::uint64_t>(l);
    L.ln1 = make_ones(a, s.vd, st);
    L.ln2 = make_ones(a, s.vd, st);
    L.qkv_w = make_linear(a, 3LL * s.vd, s.vd, s.vd, seed, id(kVit, lid, kQkvW), st);
    L.qkv_b = make_linear(a, 1, 3 * s.vd, 3 * s.vd, seed, id(kVit, lid, kQkvB), st);
    L.o_w = make_linear(a, s.vd, s.vd, s.vd, seed, id(kVit, lid, kOW), st);
    L.o_b = make_linear(a, 1, s.vd, s.vd, seed, id(kVit, lid, kOB), st);
    L.gu_w = make_gate_up(a, s.vff, s.vff_pad, s.vd, s.vd, seed, id(kVit, lid, kGateW),
                          id(kVit, lid, kUpW), st);
    L.gu_b = make_gate_up(a, s.vff, s.vff_pad, 1, 1, seed, id(kVit, lid, kGateB),
                          id(kVit, lid, kUpB), st);
    L.down_w = make_linear(a, s.vd, s.vff, s.vff_pad, seed, id(kVit, lid, kDownW), st);
    L.down_b = make_linear(a, 1, s.vd, s.vd, seed, id(kVit, lid, kDownB), st);
  }
  // RMSNorm weights folded into the consumer GEMMs (QKV <- ln1, gate/up <- ln2)
  for (VitLayer& L : layers_) {
    fold_norm_weight(L.qkv_w, 3LL * s.vd, s.vd, s.vd, L.ln1, st);
    fold_norm_weight(L.gu_w, 2LL * s.vff_pad, s.vd, s.vd, L.ln2, st);
  }
  unit_ln_ = make_ones(a, s.vd, st);
  merger_ln_ = make_ones(a, s.vd, st);
  fc1_w_ = make_linear(a, s.merge_in, s.merge_in, s.merge_in, seed, id(kMerger, 0, kFc1W), st);
  fc1_b_ = make_linear(a, 1, s.merge_in, s.merge_in, seed, id(kMerger, 0, kFc1B), st);
  fc2_w_ = make_linear(a, s.d, s.merge_in, s.merge_in, seed, id(kMerger, 0, kFc2W), st);
  fc2_b_ = make_linear(a, 1, s.d, s.d, seed, id(kMerger, 0, kFc2B), st);

  const std::int64_t P = max_patches;
  x_ = alloc_bf16(a, P * s.vd);
  xn_ = alloc_bf16(a, P * s.vd);
  qkv_ = alloc_bf16(a, P * 3 * s.vd);
  att_ = alloc_bf16(a, P * s.vd);
  h_ = alloc_bf16(a, P * s.vff_pad);
  mh_ = alloc_bf16(a, (P / 4 + 1) * s.merge_in);
  // tcgen05 attention operands, head-padded to 128 (pad never written: zero)
  const std::int64_t padded = P * s.vh * 128;
  qp_ = alloc_bf16(a, padded);
  kp_ = alloc_bf16(a, padded);
  vt_ = alloc_bf16(a, padded);
  RS_CUDA_CHECK(cudaMemsetAsync(qp_, 0, padded * 2, st));
  RS_CUDA_CHECK(cudaMemsetAsync(kp_, 0, padded * 2, st));
  RS_CUDA_CHECK(cudaMemsetAsync(vt_, 0, padded * 2, st));
  rope_table_ = static_cast<float2*>(a.alloc(static_cast<std::size_t>(P) * (s.vhd / 2) * sizeof(float2)));
  rope_freq_ = static_cast<float2*>(a.alloc(static_cast<std::size_t>(kVitRopePositions) * (s.vhd / 4) * sizeof(float2)));
  vit_rope_freq_table(kVitRopePositions, s.vhd, s.cfg.rope_theta_vit, rope_freq_, st);
  ss_a_ = static_cast<unsigned long long*>(a.alloc(static_cast<std::size_t>(P) * 8));
  ss_b_ = static_cast<unsigned long long*>(a.alloc(static_cast<std::size_t>(P) * 8));
}

void finalize_plan(VitBatchPlan& plan) {
  plan.full_blocks.clear();
  plan.win_blocks.clear();
  for (std::size_t i = 0; i + 1 < plan.cu_item.size(); ++i) {
    const int a = plan.cu_item[i], b = plan.cu_item[i + 1];
    const int unit = attn_unit_rows();
    for (int r = a; r < b; r += unit)
      plan.full_blocks.push_back({r, std::min(unit, b - r), a, b});
  }
  // largest images first (LPT issue order, see attention_tc.cu)
  std::stable_sort(plan.full_blocks.begin(), plan.full_blocks.end(), [](const AttnBlock& x, const AttnBlock& y) {
    return x.key_end - x.key_begin > y.key_end - y.key_begin;
  });
  // window layers: tiles of WHOLE consecutive windows of <= 128 packed rows
  // (two 8x8-patch windows in the common case) — one S tile per (tile, head)
  // holds every key its rows can see (attention_win.cu).
  const std::vector<std::int32_t>& cu = plan.cu_window;
  plan.win_row.assign(static_cast<std::size_t>(plan.patches) + 128, 0u);  // padded: unguarded loads
  for (std::size_t w = 0; w + 1 < cu.size();) {
    const int r0 = cu[w];
    std::size_t e = w + 1;
    while (e + 1 < cu.size() && cu[e + 1] - r0 <= kPrefillRows) ++e;
    plan.win_blocks.push_back({r0, cu[e] - r0, static_cast<int>(w), static_cast<int>(e - w)});
    for (std::size_t k = w; k < e; ++k)
      for (int row = cu[k]; row < cu[k + 1]; ++row)
        plan.win_row[static_cast<std::size_t>(row)] =
            static_cast<std::uint32_t>(cu[k] - r0) | (static_cast<std::uint32_t>(cu[k + 1] - r0) << 16);
    w = e;
  }
}

void Vit::encode(const VitBatchPlan& plan, const bf16* patches, const std::int32_t* pos_hw,
                 const std::int32_t* cu_window, const std::int32_t* cu_item,
                 const std::int32_t* out_row, const AttnBlock* win_blocks,
                 const AttnBlock* full_blocks, bf16* out, cudaStream_t st) {
  const int P = plan.patches;
  if (P > max_p_)
    throw DeviceError(RS_ERR_CUDA, "vit: batch of " + std::to_string(P) +
                                       " patches exceeds max_encode_tokens capacity");
  const Shapes& s = s_;
  const float scale = 1.0f / std::sqrt(static_cast<float>(s.vhd));
  GemmArgs g;
  // patch embedding (Conv3d as GEMM; K = 1176 tail zero-filled by TMA)
  g = GemmArgs{};
  g.A = patches; g.lda = s.pdim; g.B = patch_w_; g.ldb = s.pdim; g.C = x_; g.ldc = s.vd;
  g.M = P; g.N = s.vd; g.K = s.pdim;
  gemm(g, Epi::Store, st);
  const int n_win = static_cast<int>(plan.cu_window.size()) - 1;
  const int n_items = static_cast<int>(plan.cu_item.size()) - 1;
  vit_rope_table(pos_hw, P, s.vhd, s.cfg.rope_theta_vit, rope_table_, st);
  // Folded RMSNorm (gemm.cuh): the residual GEMMs hand per-row sums of
  // squares (ss_a_ after down, ss_b_ after O) to the norm-consumer GEMMs
  // (QKV, gate/up), each zeroing the other buffer for the next producer;
  // layer 0's ln1 input comes from the patch embedding: explicit norm.
  RS_CUDA_CHECK(cudaMemsetAsync(ss_b_, 0, static_cast<std::size_t>(P) * 8, st));
  const float inv_vd = 1.0f / static_cast<float>(s.vd);
  static const bool win_tc_env = [] {
    const char* e = std::getenv("RS_VIT_WIN_TC");
    return e == nullptr || e[0] != '0';
  }();
  int n_pos = 0;
  for (std::int32_t v : plan.pos_hw) n_pos = std::max(n_pos, v + 1);
  const bool win_tc = win_tc_env && n_pos <= kVitRopePositions &&
                      attention_window_tc_supported(s.vhd, plan.max_window, n_pos);
  double win_flops = 0;  // 4 n^2 hd per head per window
  for (std::size_t i = 0; i + 1 < plan.cu_window.size(); ++i) {
    const double n = plan.cu_window[i + 1] - plan.cu_window[i];
    win_flops += 4.0 * n * n * s.vhd * s.vh;
  }
  for (int l = 0; l < s.vl; ++l) {
    const VitLayer& L = layers_[static_cast<std::size_t>(l)];
    g = GemmArgs{};
    if (l == 0) {
      rmsnorm(x_, s.vd, unit_ln_, xn_, s.vd, P, s.vd, s.eps, st);
      g.A = xn_;
    } else {
      g.A = x_;
      g.ss_in = ss_a_; g.ss_inv_dim = inv_vd; g.ss_eps = s.eps;
    }
    g.lda = s.vd; g.B = L.qkv_w; g.ldb = s.vd; g.C = qkv_; g.ldc = 3 * s.vd;
    g.bias = L.qkv_b; g.M = P; g.N = 3 * s.vd; g.K = s.vd;
    gemm(g, Epi::Store, st);
    if (s.full_attention_layer(l)) {
      // full image attention: tcgen05 flash attention over head-padded q / k
      // and transposed v (long sequences, tensor-bound)
      vit_qkv_split(qkv_, 3 * s.vd, rope_table_, P, s.vh, s.vhd, qp_, kp_, vt_, max_p_, st);
      attention_varlen_tc(qp_, kp_, vt_, max_p_, s.vh, att_, s.vd, s.vhd, full_blocks,
                          plan.full_blocks.data(), static_cast<int>(plan.full_blocks.size()), cu_item, n_items, scale, st);
    } else {
      // 8x8-patch windows (<= 64 keys): tcgen05 over tiles of whole windows,
      // Q / K / V read in place by TMA (no padding / transpose pass), 2D RoPE
      // applied in shared memory (attention_win.cu); the mma.sync kernel
      // covers head sizes / windows it does not (and RS_VIT_WIN_TC=0)
      if (win_tc)
        attention_window_tc(qkv_, 3 * s.vd, P, att_, s.vd, win_blocks,
                            static_cast<int>(plan.win_blocks.size()), s.vh, s.vhd, scale, pos_hw, rope_freq_,
                            n_pos, win_flops, st);
      else
        attention_varlen_bidir(qkv_, 3 * s.vd, att_, s.vd, cu_window, n_win, plan.max_window, P, s.vh,
                               s.vhd, scale, st, rope_table_);
    }
    g = GemmArgs{};
    g.A = att_; g.lda = s.vd; g.B = L.o_w; g.ldb = s.vd; g.C = x_; g.ldc = s.vd; g.bias = L.o_b;
    g.residual = x_; g.ldr = s.vd; g.M = P; g.N = s.vd; g.K = s.vd;
    g.ss_out = ss_b_; g.ss_clear = ss_a_; g.ss_clear_n = P;
    gemm(g, Epi::Residual, st);
    g = GemmArgs{};
    g.A = x_; g.lda = s.vd; g.B = L.gu_w; g.ldb = s.vd; g.C = h_; g.ldc = s.vff_pad;
    g.bias = L.gu_b; g.M = P; g.N = 2 * s.vff_pad; g.K = s.vd;
    g.ss_in = ss_b_; g.ss_inv_dim = inv_vd; g.ss_eps = s.eps;
    gemm(g, Epi::SwiGLU, st);
    g = GemmArgs{};
    g.A = h_; g.lda = s.vff_pad; g.B = L.down_w; g.ldb = s.vff_pad; g.C = x_; g.ldc = s.vd;
    g.bias = L.down_b; g.residual = x_; g.ldr = s.vd; g.M = P; g.N = s.vd; g.K = s.vff_pad;
    g.ss_out = ss_a_; g.ss_clear = ss_b_; g.ss_clear_n = P;
    gemm(g, Epi::Residual, st);
  }
  // patch merger: RMSNorm per patch, 2x2 groups are 4 consecutive rows ->
  // a free [P/4, 4*vd] view; fc1 + GELU; fc2 scattered to LLM row order.
  rmsnorm(x_, s.vd, merger_ln_, xn_, s.vd, P, s.vd, s.eps, st);
  g = GemmArgs{};
  g.A = xn_; g.lda = s.merge_in; g.B = fc1_w_; g.ldb = s.merge_in; g.C = mh_; g.ldc = s.merge_in;
  g.bias = fc1_b_; g.M = P / 4; g.N = s.merge_in; g.K = s.merge_in;
  gemm(g, Epi::Gelu, st);
  g = GemmArgs{};
  g.A = mh_; g.lda = s.merge_in; g.B = fc2_w_; g.ldb = s.merge_in; g.C = out; g.ldc = s.d;
  g.bias = fc2_b_; g.row_map = out_row; g.M = P / 4; g.N = s.d; g.K = s.merge_in;
  gemm(g, Epi::Store, st);
}

std::uint64_t Vit::flops_per_batch(const VitBatchPlan& plan) const {
  const std::uint64_t P = static_cast<std::uint64_t>(plan.patches);
  const std::uint64_t vd = static_cast<std::uint64_t>(s_.vd), ff = static_cast<std::uint64_t>(s_.vff);
  std::uint64_t f = 2 * P * vd * static_cast<std::uint64_t>(s_.pdim);
  f += static_cast<std::uint64_t>(s_.vl) * 2 * P * (4 * vd * vd + 3 * vd * ff);
  // attention: 4 * n * d per token per layer
  for (int l = 0; l < s_.vl; ++l) {
    const std::vector<std::int32_t>& cu = s_.full_attention_layer(l) ? plan.cu_item : plan.cu_window;
    for (std::size_t i = 0; i + 1 < cu.size(); ++i) {
      const std::uint64_t n = static_cast<std::uint64_t>(cu[i + 1] - cu[i]);
      f += 4 * n * n * vd;
    }
  }
  const std::uint64_t T = P / 4, mi = static_cast<std::uint64_t>(s_.merge_in);
  f += 2 * T * (mi * mi + mi * static_cast<std::uint64_t>(s_.d));
  return f;
}

// ---- LLM --------------------------------------------------------------------------
void Llm::init(const Shapes& sg, DeviceArena& a, int lb, int le, bool with_embed, bool with_head,
               int max_chunk, std::int64_t kv_pages, int page_size, int logits_slots,
               cudaStream_t st, int tp_rank, int tp_size) {
  // local (shard) shapes; sg = the full model the weights are sliced from
  Shapes s = sg;
  if (tp_size > 1) {
    if (sg.hq % tp_size != 0 || sg.hkv % tp_size != 0 || sg.ff % (16 * tp_size) != 0)
      throw lmmsim::ConfigError("tensor parallelism: " + std::to_string(tp_size) +
                                " does not divide the heads / SwiGLU width");
    s.hq = sg.hq / tp_size;
    s.hkv = sg.hkv / tp_size;
    s.ff = sg.ff / tp_size;
    s.qkv_dim = (s.hq + 2 * s.hkv) * s.hd;
  }
  s_ = s;
  lb_ = lb;
  le_ = le;
  page_size_ = page_size;
  max_m_ = max_chunk;
  slots_ = logits_slots;
  const std::uint64_t seed = s.cfg.weight_seed;
  using namespace wid;
  if (with_embed)
    embed_ = make_linear(a, s.vocab, s.d, s.d, seed, id(kTop, 0, kEmbed), st);
  layers_.resize(static_cast<std::size_t>(le - lb));
  const std::int64_t kv_elems = kv_pages * s.hkv * page_size * s.hd;
  for (int l = lb; l < le; ++l) {
    LlmLayer& L = layers_[static_cast<std::size_t>(l - lb)];
    const std::uint64_t lid = static_cast<std::uint64_t>(l);
    L.ln1 = make_ones(a, s.d, st);
    L.ln2 = make_ones(a, s.d, st);
    if (tp_size == 1) {
      L.qkv_w = make_linear(a, s.qkv_dim, s.d, s.d, seed, id(kLlm, lid, kQkvW), st);
      L.qkv_b = make_linear(a, 1, s.qkv_dim, s.qkv_dim, seed, id(kLlm, lid, kQkvB), st);
      L.o_w = make_linear(a, s.d, s.hq * s.hd, s.hq * s.hd, seed, id(kLlm, lid, kOW), st);
      L.gu_w = make_gate_up(a, s.ff, s.ff, s.d, s.d, seed, id(kLlm, lid, kGateW),
                            id(kLlm, lid, kUpW), st);
      L.down_w = make_linear(a, s.d, s.ff, s.ff, seed, id(kLlm, lid, kDownW), st);
    } else {
      // this shard's slices: q / k / v head rows, O and down input columns, gate / up rows
      const int hd = s.hd;
      const std::int64_t q0 = static_cast<std::int64_t>(tp_rank) * s.hq * hd;
      const std::int64_t k0 = static_cast<std::int64_t>(sg.hq) * hd + static_cast<std::int64_t>(tp_rank) * s.hkv * hd;
      const std::int64_t v0 = static_cast<std::int64_t>(sg.hq + sg.hkv) * hd +
                              static_cast<std::int64_t>(tp_rank) * s.hkv * hd;
      const std::int64_t nq = static_cast<std::int64_t>(s.hq) * hd, nk = static_cast<std::int64_t>(s.hkv) * hd;
      L.qkv_w = alloc_bf16(a, static_cast<std::int64_t>(s.qkv_dim) * s.d);
      L.qkv_b = alloc_bf16(a, s.qkv_dim);
      const std::uint64_t wq = id(kLlm, lid, kQkvW), bq = id(kLlm, lid, kQkvB);
      fill_uniform_slice(L.qkv_w, nq, s.d, s.d, seed, wq, kWeightScale, q0, 0, s.d, st);
      fill_uniform_slice(L.qkv_w + nq * s.d, nk, s.d, s.d, seed, wq, kWeightScale, k0, 0, s.d, st);
      fill_uniform_slice(L.qkv_w + (nq + nk) * s.d, nk, s.d, s.d, seed, wq, kWeightScale, v0, 0, s.d, st);
      fill_uniform_slice(L.qkv_b, 1, static_cast<int>(nq), static_cast<int>(nq), seed, bq, kWeightScale, 0,
                         static_cast<int>(q0), sg.qkv_dim, st);
      fill_uniform_slice(L.qkv_b + nq, 1, static_cast<int>(nk), static_cast<int>(nk), seed, bq, kWeightScale, 0,
                         static_cast<int>(k0), sg.qkv_dim, st);
      fill_uniform_slice(L.qkv_b + nq + nk, 1, static_cast<int>(nk), static_cast<int>(nk), seed, bq,
                         kWeightScale, 0, static_cast<int>(v0), sg.qkv_dim, st);
      L.o_w = alloc_bf16(a, static_cast<std::int64_t>(s.d) * nq);
      fill_uniform_slice(L.o_w, s.d, static_cast<int>(nq), static_cast<int>(nq), seed, id(kLlm, lid, kOW),
                         kWeightScale, 0, static_cast<int>(q0), sg.hq * hd, st);
      L.gu_w = alloc_bf16(a, 2LL * s.ff * s.d);
      fill_uniform_interleaved(L.gu_w, s.ff, s.ff, s.d, s.d, seed, id(kLlm, lid, kGateW), kWeightScale, 0, st,
                               tp_rank * s.ff);
      fill_uniform_interleaved(L.gu_w, s.ff, s.ff, s.d, s.d, seed, id(kLlm, lid, kUpW), kWeightScale, 1, st,
                               tp_rank * s.ff);
      L.down_w = alloc_bf16(a, static_cast<std::int64_t>(s.d) * s.ff);
      fill_uniform_slice(L.down_w, s.d, s.ff, s.ff, seed, id(kLlm, lid, kDownW), kWeightScale, 0, tp_rank * s.ff,
                         sg.ff, st);
    }
    L.k_cache = alloc_bf16(a, kv_elems);
    L.v_cache = alloc_bf16(a, kv_elems);
    // Zero-init: masked keys of a partial page must be finite (P = 0 x V).
    RS_CUDA_CHECK(cudaMemsetAsync(L.k_cache, 0, static_cast<std::size_t>(kv_elems) * 2, st));
    RS_CUDA_CHECK(cudaMemsetAsync(L.v_cache, 0, static_cast<std::size_t>(kv_elems) * 2, st));
  }
  kv_pages_ = kv_pages;
  // RMSNorm weights folded into the consumer GEMMs (QKV <- ln1, gate/up <- ln2)
  for (LlmLayer& L : layers_) {
    fold_norm_weight(L.qkv_w, s.qkv_dim, s.d, s.d, L.ln1, st);
    fold_norm_weight(L.gu_w, 2LL * s.ff, s.d, s.d, L.ln2, st);
  }
  unit_ln_ = make_ones(a, s.d, st);
  if (with_head) {
    final_ln_ = make_ones(a, s.d, st);
    head_ = make_linear(a, s.vocab, s.d, s.d, seed, id(kTop, 0, kHead), st);
    logits_ = static_cast<float*>(a.alloc(static_cast<std::size_t>(logits_slots) * s.vocab * 4));
    argmax_ = static_cast<std::int32_t*>(a.alloc(static_cast<std::size_t>(logits_slots) * 4));
    xf_ = alloc_bf16(a, static_cast<std::int64_t>(max_chunk) * s.d);
  }
  const std::int64_t M = max_chunk;
  rope_table_ = static_cast<float2*>(a.alloc(static_cast<std::size_t>(M) * (s.hd / 2) * sizeof(float2)));
  ss_a_ = static_cast<unsigned long long*>(a.alloc(static_cast<std::size_t>(M) * 8));
  ss_b_ = static_cast<unsigned long long*>(a.alloc(static_cast<std::size_t>(M) * 8));
  xn_ = alloc_bf16(a, M * s.d);
  qkv_ = alloc_bf16(a, M * s.qkv_dim);
  att_ = alloc_bf16(a, M * s.hq * s.hd);
  h_ = alloc_bf16(a, M * s.ff);
}

void Llm::forward_stage(const ChunkDev& c, const bf16* slab, bf16* x,
                        const int* const* page_tables, cudaStream_t st, int layer_from,
                        int layer_to) {
  const int l_from = layer_from < 0 ? lb_ : layer_from;
  const int l_to = layer_to < 0 ? le_ : layer_to;
  const Shapes& s = s_;
  const int M = c.M;
  if (M > max_m_) throw DeviceError(RS_ERR_CUDA, "llm: chunk exceeds max_chunk_tokens");
  const float scale = 1.0f / std::sqrt(static_cast<float>(s.hd));
  GemmArgs g;
  // Folded RMSNorm (gemm.cuh): the residual GEMMs hand per-row sums of
  // squares (ss_a_ after down, ss_b_ after O) to the norm-consumer GEMMs
  // (QKV, gate/up), each zeroing the other buffer for the next producer. The
  // first layer of the call normalises explicitly (unit weight: ln1 lives in
  // qkv_w).
  RS_CUDA_CHECK(cudaMemsetAsync(ss_b_, 0, static_cast<std::size_t>(M) * 8, st));
  const float inv_d = 1.0f / static_cast<float>(s.d);
  mrope_table(c.rows, M, s.hd, s.cfg.rope_theta_llm, rope_table_, st);  // shared by every layer
  for (int l = l_from; l < l_to; ++l) {
    HostPhase ph("llm.layer");
    const LlmLayer& L = layers_[static_cast<std::size_t>(l - lb_)];
    g = GemmArgs{};
    if (l == l_from) {
      if (l == 0 && c.gather_rows != nullptr)  // chunk input: gather slot rows (K8 fused into the first norm)
        rmsnorm(slab, s.d, unit_ln_, xn_, s.d, M, s.d, s.eps, st, c.gather_rows, x, s.d);
      else
        rmsnorm(x, s.d, unit_ln_, xn_, s.d, M, s.d, s.eps, st);
      g.A = xn_;
    } else {
      g.A = x;
      g.ss_in = ss_a_; g.ss_inv_dim = inv_d; g.ss_eps = s.eps;
    }
    g.lda = s.d; g.B = L.qkv_w; g.ldb = s.d; g.C = qkv_; g.ldc = s.qkv_dim;
    g.bias = L.qkv_b; g.M = M; g.N = s.qkv_dim; g.K = s.d;
    qkv_rope_append(g, c, L, page_tables, st);
    PagedKV kv{L.k_cache, L.v_cache, page_tables, page_size_};
    if (c.decode)
      attention_decode_paged(qkv_, s.qkv_dim, att_, s.hq * s.hd, c.work, c.n_work, c.max_keys, kv, s.hq,
                             s.hkv, s.hd, scale, st);
    else
      attention_prefill_paged_tc(qkv_, s.qkv_dim, max_m_, att_, s.hq * s.hd, c.work, c.work_host, c.n_work, c.max_keys, kv,
                                 kv_pages_, s.hq, s.hkv, s.hd, scale, st);
    g = GemmArgs{};
    g.A = att_; g.lda = s.hq * s.hd; g.B = L.o_w; g.ldb = s.hq * s.hd; g.C = x; g.ldc = s.d;
    g.residual = x; g.ldr = s.d; g.M = M; g.N = s.d; g.K = s.hq * s.hd;
    g.ss_out = ss_b_; g.ss_clear = ss_a_; g.ss_clear_n = M;
    gemm(g, Epi::Residual, st);
    g = GemmArgs{};
    g.A = x; g.lda = s.d; g.B = L.gu_w; g.ldb = s.d; g.C = h_; g.ldc = s.ff;
    g.M = M; g.N = 2 * s.ff; g.K = s.d;
    g.ss_in = ss_b_; g.ss_inv_dim = inv_d; g.ss_eps = s.eps;
    gemm(g, Epi::SwiGLU, st);
    g = GemmArgs{};
    g.A = h_; g.lda = s.ff; g.B = L.down_w; g.ldb = s.ff; g.C = x; g.ldc = s.d;
    g.residual = x; g.ldr = s.d; g.M = M; g.N = s.d; g.K = s.ff;
    g.ss_out = ss_a_; g.ss_clear = ss_b_; g.ss_clear_n = M;
    gemm(g, Epi::Residual, st);
  }
  if (head_ != nullptr && l_to == le_ && c.n_done > 0) {
    rmsnorm(x, s.d, final_ln_, xf_, s.d, c.n_done, s.d, s.eps, st, c.done_rows);
    g = GemmArgs{};
    g.A = xf_; g.lda = s.d; g.B = head_; g.ldb = s.d; g.C = logits_; g.ldc = s.vocab;
    g.row_map = c.done_slots; g.M = c.n_done; g.N = s.vocab; g.K = s.d;
    gemm(g, Epi::StoreF32, st);
    argmax_rows(logits_, c.n_done, s.vocab, argmax_, st, c.done_slots);
  }
}

// QKV projection + M-RoPE + paged-KV append: fused into the GEMM
// epilogue (Epi::QkvRope) for chunks; decode-sized M goes through the skinny
// GEMM and the separate rope / append kernel. RS_QKV_FUSE=0: unfused (A/B).
void Llm::qkv_rope_append(GemmArgs g, const ChunkDev& c, const LlmLayer& L, const int* const* page_tables,
                          cudaStream_t st) {
  const Shapes& s = s_;
  static const bool fuse = [] {
    const char* e = std::getenv("RS_QKV_FUSE");
    return e == nullptr || e[0] != '0';
  }();
  // chunks: the tcgen05 GEMM's QkvRope epilogue; decode-sized steps (M <= 8):
  // the skinny GEMM's (same math: fp32 rotation, one rounding)
  if (fuse && s.hd % 64 == 0) {
    g.rope_rows = c.rows;
    g.rope_table = rope_table_;
    g.page_tables = page_tables;
    g.k_cache = L.k_cache;
    g.v_cache = L.v_cache;
    g.rope_hq = s.hq;
    g.rope_hkv = s.hkv;
    g.rope_hd = s.hd;
    g.page_size = page_size_;
    gemm(g, Epi::QkvRope, st);
    return;
  }
  gemm(g, Epi::Store, st);
  rope_kv_append(qkv_, s.qkv_dim, c.rows, g.M, s.hq, s.hkv, s.hd, s.cfg.rope_theta_llm, L.k_cache, L.v_cache,
                 page_tables, page_size_, st, nullptr, rope_table_);
}

// ---- tensor-parallel phases (tp_forward, device_context.cu) --------------------------
void Llm::tp_attn_partial(int l, const ChunkDev& c, const bf16* slab, bf16* x, bool first,
                          const unsigned long long* ss, const int* const* page_tables, bf16* part,
                          cudaStream_t st) {
  const Shapes& s = s_;
  const LlmLayer& L = layers_[static_cast<std::size_t>(l - lb_)];
  const int M = c.M;
  const float scale = 1.0f / std::sqrt(static_cast<float>(s.hd));
  GemmArgs g;
  if (first) {
    if (l == 0 && c.gather_rows != nullptr)  // chunk input gathered from the slab into x (K8)
      rmsnorm(slab, s.d, unit_ln_, xn_, s.d, M, s.d, s.eps, st, c.gather_rows, x, s.d);
    else
      rmsnorm(x, s.d, unit_ln_, xn_, s.d, M, s.d, s.eps, st);
    g.A = xn_;
  } else {
    g.A = x;
    g.ss_in = ss; g.ss_inv_dim = 1.0f / static_cast<float>(s.d); g.ss_eps = s.eps;
  }
  g.lda = s.d; g.B = L.qkv_w; g.ldb = s.d; g.C = qkv_; g.ldc = s.qkv_dim;
  g.bias = L.qkv_b; g.M = M; g.N = s.qkv_dim; g.K = s.d;
  qkv_rope_append(g, c, L, page_tables, st);
  PagedKV kv{L.k_cache, L.v_cache, page_tables, page_size_};
  if (c.decode)
    attention_decode_paged(qkv_, s.qkv_dim, att_, s.hq * s.hd, c.work, c.n_work, c.max_keys, kv, s.hq,
                           s.hkv, s.hd, scale, st);
  else
    attention_prefill_paged_tc(qkv_, s.qkv_dim, max_m_, att_, s.hq * s.hd, c.work, c.work_host, c.n_work, c.max_keys, kv,
                               kv_pages_, s.hq, s.hkv, s.hd, scale, st);
  g = GemmArgs{};
  g.A = att_; g.lda = s.hq * s.hd; g.B = L.o_w; g.ldb = s.hq * s.hd; g.C = part; g.ldc = s.d;
  g.M = M; g.N = s.d; g.K = s.hq * s.hd;
  gemm(g, Epi::Store, st);
}

void Llm::tp_mlp_partial(int l, const ChunkDev& c, const bf16* x, const unsigned long long* ss, bf16* part,
                         cudaStream_t st) {
  const Shapes& s = s_;
  const LlmLayer& L = layers_[static_cast<std::size_t>(l - lb_)];
  const int M = c.M;
  GemmArgs g;
  g.A = x; g.lda = s.d; g.B = L.gu_w; g.ldb = s.d; g.C = h_; g.ldc = s.ff;
  g.M = M; g.N = 2 * s.ff; g.K = s.d;
  g.ss_in = ss; g.ss_inv_dim = 1.0f / static_cast<float>(s.d); g.ss_eps = s.eps;
  gemm(g, Epi::SwiGLU, st);
  g = GemmArgs{};
  g.A = h_; g.lda = s.ff; g.B = L.down_w; g.ldb = s.ff; g.C = part; g.ldc = s.d;
  g.M = M; g.N = s.d; g.K = s.ff;
  gemm(g, Epi::Store, st);
}

void Llm::tp_begin(const ChunkDev& c, cudaStream_t st) {
  mrope_table(c.rows, c.M, s_.hd, s_.cfg.rope_theta_llm, rope_table_, st);
}

void Llm::head_phase(const ChunkDev& c, const bf16* x, cudaStream_t st) {
  if (head_ == nullptr || c.n_done <= 0) return;
  const Shapes& s = s_;
  rmsnorm(x, s.d, final_ln_, xf_, s.d, c.n_done, s.d, s.eps, st, c.done_rows);
  GemmArgs g;
  g.A = xf_; g.lda = s.d; g.B = head_; g.ldb = s.d; g.C = logits_; g.ldc = s.vocab;
  g.row_map = c.done_slots; g.M = c.n_done; g.N = s.vocab; g.K = s.d;
  gemm(g, Epi::StoreF32, st);
  argmax_rows(logits_, c.n_done, s.vocab, argmax_, st, c.done_slots);
}

std::uint64_t Llm::dense_flops(std::uint64_t tokens) const {
  const std::uint64_t d = static_cast<std::uint64_t>(s_.d);
  const std::uint64_t per_layer = 2 * (d * static_cast<std::uint64_t>(s_.qkv_dim) +
                                       static_cast<std::uint64_t>(s_.hq * s_.hd) * d +
                                       3 * d * static_cast<std::uint64_t>(s_.ff));
  return tokens * per_layer * static_cast<std::uint64_t>(le_ - lb_);
}

}  // namespace rserve
