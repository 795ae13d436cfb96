// rserve-b200 — flash attention on tcgen05 tensor cores (sm_100a).
//
// One kernel, two key sources:
//   * kPaged  — LLM chunked prefill: a 128-query block of one slice attends
//     causally to its request's paged KV cache (GQA: kv head = h / g).
//   * kVarlen — ViT: a 128-token block of the packed sequence attends
//     bidirectionally within each row's own sequence (window or image,
//     cu_seqlens); Q / K are head-padded to 128 columns and V is transposed
//     by vit_qkv_split (elementwise.cu) so the tiles are plain SW128 K-major.
// Per iteration of 128 keys:
//   S_j  = Q . K_j^T      tcgen05.mma (SS), S double-buffered in TMEM
//   P_j  = softmax rows   4 warps, one query row per thread (tcgen05.ld), fp32
//                         online max / sum, P -> smem bf16 in the SW128 layout
//   O   += P_j . V_j      tcgen05.mma into one TMEM accumulator; the running max
//                         is raised lazily (only when it grows by > 2^8) and O
//                         is then rescaled in TMEM (tcgen05.ld / st)
// V is held transposed ([hd][keys]) so both MMAs read K-major SW128 operands
// with the same descriptors as the GEMM.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <unordered_map>
#include <vector>

#include "attention.cuh"
#include "common.cuh"
#include "sm100.cuh"

namespace rserve {
namespace {

constexpr int kTcThreads = 256;
constexpr int kAtom = 128 * 128;  // one [128 rows x 128 B] SW128 region

template <int HD>
struct TcCfg {
  static constexpr int kHdAtoms = HD / 64;             // K-dim atoms of Q / K tiles
  static constexpr int kQBytes = kHdAtoms * kAtom;     // Q [128 x HD]
  static constexpr int kKBytes = kHdAtoms * kAtom;     // K [128 keys x HD]
  static constexpr int kVAtom = HD * 128;              // V^T [HD x 64 keys]
  static constexpr int kVBytes = 2 * kVAtom;           // 128 keys
  static constexpr int kStages = 3;                    // K and V rings (independent)
  static constexpr int kSmem = kQBytes + kStages * (kKBytes + kVBytes) + 1024 + 512;
};
// TMEM columns: S[0] 0, S[1] 128, O 256 (HD), P[0] 384, P[1] 448 (bf16 pairs)
constexpr std::uint32_t kTmemS = 0, kTmemO = 256, kTmemP = 384;

enum class KvMode { kPaged, kVarlen };

constexpr int kInlineUnits = 128;  // work items per launch (larger launches are batched)
constexpr int kMaxPieces = 256;    // item key-splits per launch

struct TcParams {
  const PrefillWork* work;          // kPaged
  const int* const* page_tables;    // kPaged
  const AttnBlock* blocks;          // kVarlen
  const int* cu_seqlens;            // kVarlen
  int n_seqs;
  int q_heads, kv_heads;
  int q_head_stride;                // q / k column stride between heads
  int out_hd;                       // output columns per head (<= HD)
  float scale_log2;
  bf16* out;
  int ld_out;
  // The launch's work items / blocks, inlined in the kernel parameters
  // (constant bank): the ping-pong kernel's MMA warp derives its loop bounds
  // and ring stages from them, so they stay in uniform registers and the
  // tcgen05.mma operands need no per-instruction uniformisation.
  int4 inl[kInlineUnits];
  // Pieces (ping-pong kernel): an item's keys may be split S ways (kPaged);
  // piece = (item, split s, S, first piece of the item), in descending cost
  // order; unit u = piece u / H, head u % H. Split s covers key tiles
  // [s n / S, (s + 1) n / S) of the item's n tiles and writes unnormalised
  // fp32 O plus (m, l) per row to the workspace (row (u * 256 + r));
  // pp_merge_kernel combines an item's splits in order.
  int4 pieces[kMaxPieces];
  int2 item_split[kInlineUnits];    // (S, first piece) per item
  int n_pieces;
  int max_split;                    // > 1: the workspace / merge are in use
  int max_keys;                     // kPaged: longest item's keys (host info, profiling label)
  float* part_o;                    // [n_pieces * H * 256, HD]
  float* part_ml;                   // [n_pieces * H * 256, 2]
  // RS_PP_TRACE (dev): globaltimer stamps of CTA 0's pipeline handshakes
  // [role][iteration][event], else null
  unsigned long long* trace;
};
constexpr int kPpTraceIters = 24;  // key-tile iterations traced (first unit of CTA 0)
constexpr int kPpTraceEv = 8;
__device__ __forceinline__ unsigned long long pp_gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// role: 0 MMA warp (tile 0 events), 1 MMA warp (tile 1), 2 softmax tile 0, 3 softmax tile 1
#ifdef RS_PP_TRACE_BUILD  // dev builds only: the stamps sit in the hot loops
#define PP_TRACE(role, it, ev)                                                                      \
  do {                                                                                              \
    if (p.trace != nullptr && blockIdx.x == 0 && (it) >= 0 && (it) < kPpTraceIters)                 \
      p.trace[((role) * kPpTraceIters + (it)) * kPpTraceEv + (ev)] = pp_gtimer();                  \
  } while (0)
#else
#define PP_TRACE(role, it, ev) \
  do {                         \
  } while (0)
#endif

__host__ __device__ __forceinline__ void kv_split_range(int n_tiles, int splits, int s, int& jb, int& je) {
  jb = s * n_tiles / splits;
  je = (s + 1) * n_tiles / splits;
}

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// MUFU ex2 (flush-to-zero); ex2(-inf) = +0.
__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// exp2 on the FMA pipe (x <= ~8): 2^x = 2^n * 2^f, n = floor(x), f in [0,1),
// 2^f by a degree-3 minimax polynomial (rel. err ~9e-5, below bf16's 4e-3);
// x < -127 -> 0 (matches ftz ex2 for the masked -inf entries).
__device__ __forceinline__ float poly_exp2(float x) {
  x = fmaxf(x, -127.f);
  const float n = floorf(x);
  const float f = x - n;
  float p = fmaf(0.0790209f, f, 0.2249531f);
  p = fmaf(p, f, 0.6960277f);
  p = fmaf(p, f, 0.99998863f);
  const int bits = __float_as_int(p) + (static_cast<int>(n) << 23);
  return x <= -127.f ? 0.f : __int_as_float(bits);
}
// poly_exp2_fma below on a pair, with the FMAs packed.
__device__ __forceinline__ float2 poly_exp2_fma2(float2 x) {
  x.x = fmaxf(x.x, -125.5f);
  x.y = fmaxf(x.y, -125.5f);
  const float2 magic = make_float2(12582912.f, 12582912.f);
  const float2 t = add2(x, magic);
  const float2 n = add2(t, make_float2(-12582912.f, -12582912.f));
  const float2 f = add2(x, make_float2(-n.x, -n.y));
  float2 p = fma2(make_float2(0.05517166f, 0.05517166f), f, make_float2(0.24261116f, 0.24261116f));
  p = fma2(p, f, make_float2(0.69326099f, 0.69326099f));
  p = fma2(p, f, make_float2(0.99992807f, 0.99992807f));
  return make_float2(__int_as_float(__float_as_int(p.x) + (__float_as_int(t.x) << 23)),
                     __int_as_float(__float_as_int(p.y) + (__float_as_int(t.y) << 23)));
}

// Same on the FMA / ALU pipes only (no FRND / F2I, which share the MUFU
// (XU) pipe): round(x) by the 1.5 * 2^23 magic add, whose low mantissa bits
// then hold the integer part for the exponent add; 2^f on [-0.5, 0.5] by a
// degree-3 minimax polynomial (rel. err 7.5e-5, below bf16's 3.9e-3).
// x <= -125.5 -> 2^-125.5 (~1e-38; masked keys, vanishing next to the row max's 1).
__device__ __forceinline__ float poly_exp2_fma(float x) {
  x = fmaxf(x, -125.5f);
  const float t = __fadd_rn(x, 12582912.f);
  const float f = x - __fsub_rn(t, 12582912.f);
  float p = fmaf(0.05517166f, f, 0.24261116f);
  p = fmaf(p, f, 0.69326099f);
  p = fmaf(p, f, 0.99992807f);
  return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}

template <int HD, KvMode MODE>
__global__ void __launch_bounds__(kTcThreads, 1)
    fa_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                 const __grid_constant__ CUtensorMap tmV, const __grid_constant__ TcParams p) {
  using C = TcCfg<HD>;
  constexpr int S = C::kStages;
  extern __shared__ __align__(1024) std::uint8_t smem_raw[];
  std::uint8_t* smem = reinterpret_cast<std::uint8_t*>(
      (reinterpret_cast<std::uintptr_t>(smem_raw) + 1023) & ~std::uintptr_t(1023));
  std::uint8_t* sQ = smem;
  std::uint8_t* sK = sQ + C::kQBytes;
  std::uint8_t* sV = sK + S * C::kKBytes;
  std::uint64_t* bars = reinterpret_cast<std::uint64_t*>(sV + S * C::kVBytes);
  std::uint64_t* q_full = bars;
  std::uint64_t* k_full = bars + 1;
  std::uint64_t* k_empty = k_full + S;
  std::uint64_t* v_full = k_empty + S;
  std::uint64_t* v_empty = v_full + S;
  std::uint64_t* s_full = v_empty + S;   // [2]
  std::uint64_t* s_empty = s_full + 2;   // [2]
  std::uint64_t* p_full = s_empty + 2;   // [2]
  std::uint64_t* o_full = p_full + 2;    // [2]  PV_i completes o_full[i & 1]
  std::uint32_t* tmem_holder = reinterpret_cast<std::uint32_t*>(o_full + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  pdl_wait();
  pdl_launch_dependents();
  // grid (heads, blocks): heads vary fastest, so blocks issue in work-list
  // order — callers list the most expensive (most keys) first, which makes
  // the hardware's in-order block dispatch an LPT schedule over the SMs.
  const int head = blockIdx.x;
  const int kvh = head / (p.q_heads / p.kv_heads);
  int q_row0, q_rows, key_begin, key_end;
  const int* pt = nullptr;
  int q_pos0 = 0;
  if constexpr (MODE == KvMode::kPaged) {
    const PrefillWork w = p.work[blockIdx.y];
    q_row0 = w.q_row0;
    q_rows = w.q_rows;
    q_pos0 = w.q_pos0;
    key_begin = 0;
    key_end = w.q_pos0 + w.q_rows;
    pt = p.page_tables[w.req_slot];
  } else {
    const AttnBlock b = p.blocks[blockIdx.y];
    q_row0 = b.q_row0;
    q_rows = b.q_rows;
    // The V^T tile is a TMA load along the key dimension, whose start must be
    // 16-byte aligned: start at a multiple of 8 keys. The extra leading keys
    // belong to the previous sequence and are masked by the per-row [lo, hi).
    key_begin = b.key_begin & ~7;
    key_end = b.key_end;
  }
  const int n_keys = key_end - key_begin;
  const int n_it = (n_keys + 127) / 128;

  if (threadIdx.x == 0) {
    sm100::tma_prefetch_desc(&tmQ);
    sm100::tma_prefetch_desc(&tmK);
    sm100::tma_prefetch_desc(&tmV);
    sm100::mbar_init(q_full, 1);
    for (int i = 0; i < S; ++i) {
      sm100::mbar_init(&k_full[i], 1);
      sm100::mbar_init(&k_empty[i], 1);
      sm100::mbar_init(&v_full[i], 1);
      sm100::mbar_init(&v_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      sm100::mbar_init(&s_full[i], 1);
      sm100::mbar_init(&s_empty[i], 128);
      sm100::mbar_init(&p_full[i], 128);
      sm100::mbar_init(&o_full[i], 1);
    }
    sm100::fence_mbar_init();
  }
  if (warp == 2) sm100::tmem_alloc(tmem_holder, 512);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const std::uint32_t tmem = *tmem_holder;

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer: K and V rings run ahead independently ----------------
    sm100::mbar_expect_tx(q_full, C::kQBytes);
    for (int h = 0; h < C::kHdAtoms; ++h)
      sm100::tma_load_2d(sQ + h * kAtom, &tmQ, q_full, head * p.q_head_stride + h * 64, q_row0);
    const int n_pages = (n_keys + 63) / 64;
    for (int j = 0; j < n_it; ++j) {
      const int st = j % S;
      const std::uint32_t par = ((j / S) & 1) ^ 1;
      int pa = 0, pb = 0;
      if constexpr (MODE == KvMode::kPaged) {
        pa = pt[2 * j];
        pb = 2 * j + 1 < n_pages ? pt[2 * j + 1] : pa;  // duplicate: finite, masked
      }
      std::uint8_t* k = sK + st * C::kKBytes;
      sm100::mbar_wait(&k_empty[st], par);
      sm100::mbar_expect_tx(&k_full[st], C::kKBytes);
      if constexpr (MODE == KvMode::kPaged) {
        for (int h = 0; h < C::kHdAtoms; ++h) {
          sm100::tma_load_2d(k + h * kAtom, &tmK, &k_full[st], h * 64, (pa * p.kv_heads + kvh) * 64);
          sm100::tma_load_2d(k + h * kAtom + 64 * 128, &tmK, &k_full[st], h * 64,
                             (pb * p.kv_heads + kvh) * 64);
        }
      } else {
        for (int h = 0; h < C::kHdAtoms; ++h)
          sm100::tma_load_2d(k + h * kAtom, &tmK, &k_full[st], kvh * p.q_head_stride + h * 64,
                             key_begin + 128 * j);
      }
      std::uint8_t* v = sV + st * C::kVBytes;
      sm100::mbar_wait(&v_empty[st], par);
      sm100::mbar_expect_tx(&v_full[st], C::kVBytes);
      if constexpr (MODE == KvMode::kPaged) {
        sm100::tma_load_2d(v, &tmV, &v_full[st], 0, (pa * p.kv_heads + kvh) * HD);
        sm100::tma_load_2d(v + C::kVAtom, &tmV, &v_full[st], 0, (pb * p.kv_heads + kvh) * HD);
      } else {
        const int k0 = key_begin + 128 * j;
        sm100::tma_load_2d(v, &tmV, &v_full[st], k0, kvh * HD);
        sm100::tma_load_2d(v + C::kVAtom, &tmV, &v_full[st], k0 + 64, kvh * HD);
      }
    }
  } else if (warp == 1 && lane == 0) {
    // ---------------- MMA issuer ----------------
    constexpr std::uint32_t idesc_s = sm100::idesc_bf16_f32(128, 128);
    constexpr std::uint32_t idesc_o = sm100::idesc_bf16_f32(128, HD);
    sm100::mbar_wait(q_full, 0);
    auto issue_pv = [&](int i) {
      const int b = i & 1, st = i % S;
      sm100::mbar_wait(&v_full[st], (i / S) & 1);
      sm100::mbar_wait(&p_full[b], (i >> 1) & 1);
      sm100::tc_fence_after();
      std::uint8_t* v = sV + st * C::kVBytes;
      // O += P V: P (A operand) from TMEM, 8 columns (16 keys) per MMA
#pragma unroll
      for (int a = 0; a < 2; ++a) {
        const std::uint64_t vd = sm100::sw128_kmajor_desc(sm100::smem_u32(v + a * C::kVAtom));
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          sm100::umma_bf16_ts(tmem + kTmemO, tmem + kTmemP + 64 * b + 32 * a + 8 * kk, vd + 2 * kk,
                              idesc_o, (i | a | kk) != 0 ? 1u : 0u);
      }
      sm100::umma_commit(&o_full[b]);
      sm100::umma_commit(&v_empty[st]);
    };
    for (int j = 0; j < n_it; ++j) {
      const int b = j & 1, st = j % S;
      sm100::mbar_wait(&k_full[st], (j / S) & 1);
      sm100::mbar_wait(&s_empty[b], ((j >> 1) & 1) ^ 1);
      sm100::tc_fence_after();
      std::uint8_t* k = sK + st * C::kKBytes;
#pragma unroll
      for (int h = 0; h < C::kHdAtoms; ++h) {
        const std::uint64_t qd = sm100::sw128_kmajor_desc(sm100::smem_u32(sQ + h * kAtom));
        const std::uint64_t kd = sm100::sw128_kmajor_desc(sm100::smem_u32(k + h * kAtom));
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          sm100::umma_bf16(tmem + kTmemS + 128 * b, qd + 2 * kk, kd + 2 * kk, idesc_s,
                           (h | kk) != 0 ? 1u : 0u);
      }
      sm100::umma_commit(&s_full[b]);
      sm100::umma_commit(&k_empty[st]);  // K stage free as soon as S_j is computed
      if (j >= 1) issue_pv(j - 1);
    }
    issue_pv(n_it - 1);
  } else if (warp >= 4) {
    // ---------------- softmax (one query row per thread) ----------------
    const int q = warp - 4;
    const int r = q * 32 + lane;
    const std::uint32_t lane_off = static_cast<std::uint32_t>(q * 32) << 16;
    const std::uint32_t o_tmem = tmem + lane_off + kTmemO;
    // Visible keys of this row: absolute key index in [lo, hi).
    int lo, hi;
    if constexpr (MODE == KvMode::kPaged) {
      lo = 0;
      hi = min(q_pos0 + r + 1, key_end);
    } else {
      const int t = q_row0 + min(r, q_rows - 1);
      int a = 0, b = p.n_seqs;  // largest s with cu[s] <= t
      while (b - a > 1) {
        const int mid = (a + b) >> 1;
        if (p.cu_seqlens[mid] <= t) a = mid;
        else b = mid;
      }
      lo = p.cu_seqlens[a];
      hi = p.cu_seqlens[a + 1];
    }
    float m = -INFINITY, l = 0.f;
    for (int j = 0; j < n_it; ++j) {
      const int b = j & 1;
      sm100::mbar_wait(&s_full[b], (j >> 1) & 1);
      sm100::tc_fence_after();
      const int key0 = key_begin + j * 128;
      const int c_lo = lo - key0, c_hi = hi - key0;  // visible columns [c_lo, c_hi)
      // Whole S row in registers (one TMEM pass); masked entries -> -inf.
      std::uint32_t sv[128];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        std::uint32_t(&v)[32] = *reinterpret_cast<std::uint32_t(*)[32]>(&sv[32 * c]);
        sm100::tmem_ld_32x32b_x32(tmem + lane_off + kTmemS + 128 * b + 32 * c, v);
      }
      sm100::tmem_ld_wait();
      sm100::tc_fence_before();
      sm100::mbar_arrive(&s_empty[b]);  // S buffer may be overwritten now
      if (!(c_lo <= 0 && c_hi >= 128)) {
#pragma unroll
        for (int t = 0; t < 128; ++t)
          if (t < c_lo || t >= c_hi) sv[t] = __float_as_uint(-INFINITY);
      }
      // max: 8 independent chains, then a tree
      float mx8[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) mx8[u] = __uint_as_float(sv[u]);
#pragma unroll
      for (int t = 8; t < 128; ++t) mx8[t & 7] = fmaxf(mx8[t & 7], __uint_as_float(sv[t]));
      float mx = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                       fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7])));
      mx *= p.scale_log2;
      // P buffer b was last read by PV_{j-2} (o_full[b]); PV_{j-4} was awaited
      // two steps ago, so this parity wait cannot alias.
      if (j >= 2) sm100::mbar_wait(&o_full[b], ((j - 2) >> 1) & 1);
      const bool raise = mx > m + 8.f || (m == -INFINITY && mx != -INFINITY);
      float alpha = 1.f;
      if (raise) {
        alpha = m == -INFINITY ? 0.f : exp2f(m - mx);
        m = mx;
      }
      if (j > 0 && __any_sync(0xffffffffu, raise && alpha != 1.f)) {
        // rare: O must hold PV_{j-1} before it is rescaled in TMEM
        sm100::mbar_wait(&o_full[(j - 1) & 1], ((j - 1) >> 1) & 1);
        sm100::tc_fence_after();
#pragma unroll
        for (int c = 0; c < HD / 32; ++c) {
          std::uint32_t v[32];
          sm100::tmem_ld_32x32b_x32(o_tmem + 32 * c, v);
          sm100::tmem_ld_wait();
#pragma unroll
          for (int t = 0; t < 32; ++t) v[t] = __float_as_uint(__uint_as_float(v[t]) * alpha);
          sm100::tmem_st_32x32b_x32(o_tmem + 32 * c, v);
        }
        sm100::tmem_st_wait();
      }
      const float mneg = m == -INFINITY ? 0.f : -m;
      float rs8[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        std::uint32_t packed[32];  // 64 keys as bf16 pairs
#pragma unroll
        for (int t = 0; t < 32; ++t) {
          // exp2(-inf) = 0 for masked entries; every 4th pair on the FMA pipe
          const float x0 = fmaf(__uint_as_float(sv[64 * c + 2 * t]), p.scale_log2, mneg);
          const float x1 = fmaf(__uint_as_float(sv[64 * c + 2 * t + 1]), p.scale_log2, mneg);
          const bool poly = (t & 3) == 3;
          const float p0 = poly ? poly_exp2(x0) : fast_exp2(x0);
          const float p1 = poly ? poly_exp2(x1) : fast_exp2(x1);
          rs8[(2 * t) & 7] += p0;
          rs8[(2 * t + 1) & 7] += p1;
          packed[t] = pack_bf16x2(p0, p1);
        }
        sm100::tmem_st_32x32b_x32(tmem + lane_off + kTmemP + 64 * b + 32 * c, packed);
      }
      sm100::tmem_st_wait();
      sm100::tc_fence_before();
      sm100::mbar_arrive(&p_full[b]);
      l = l * alpha + (((rs8[0] + rs8[1]) + (rs8[2] + rs8[3])) + ((rs8[4] + rs8[5]) + (rs8[6] + rs8[7])));
    }
    // PV complete in issue order: the last one implies all
    sm100::mbar_wait(&o_full[(n_it - 1) & 1], ((n_it - 1) >> 1) & 1);
    sm100::tc_fence_after();
    const float inv = l > 0.f ? 1.f / l : 0.f;
    bf16* orow = p.out + static_cast<std::int64_t>(q_row0 + r) * p.ld_out + head * p.out_hd;
#pragma unroll
    for (int c = 0; c < HD / 32; ++c) {
      std::uint32_t v[32];
      sm100::tmem_ld_32x32b_x32(o_tmem + 32 * c, v);
      sm100::tmem_ld_wait();
      if (r < q_rows) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (32 * c + 8 * u < p.out_hd)
            reinterpret_cast<uint4*>(orow + 32 * c)[u] = make_uint4(
                pack_bf16x2(__uint_as_float(v[8 * u]) * inv, __uint_as_float(v[8 * u + 1]) * inv),
                pack_bf16x2(__uint_as_float(v[8 * u + 2]) * inv, __uint_as_float(v[8 * u + 3]) * inv),
                pack_bf16x2(__uint_as_float(v[8 * u + 4]) * inv, __uint_as_float(v[8 * u + 5]) * inv),
                pack_bf16x2(__uint_as_float(v[8 * u + 6]) * inv, __uint_as_float(v[8 * u + 7]) * inv));
        }
      }
    }
  }
  __syncthreads();
  if (warp == 2) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc(tmem, 512);
  }
}

// ---- two-tile ping-pong kernel -------------------------------------------------
// A CTA owns a unit of up to 256 query rows (two 128-row tiles Q0 / Q1 of one
// head) that share every K / V tile. The tensor core alternates between the
// tiles — PV0_{j-1}, S0_j, PV1_{j-1}, S1_j, ... — so while one softmax
// warpgroup turns S_t,j into P_t,j the tensor core works on the other tile:
// the MMA pipe no longer idles for the softmax, and K / V are read from L2
// once per 256 queries instead of per 128.
// TMEM (512 columns): tile t owns [256t, 256t + 256): S_t (fp32, 128 cols) with
// P_t (bf16 pairs) written over its first 64 columns, then O_t (HD cols).
// S_t,j+1 is issued after PV_t,j (in-order tensor pipe), so P_t,j is never
// overwritten early, and S_t,j's commit implies PV_t,j-1 is complete — the
// softmax may rescale O_t right after S_t,j arrives, without another wait.
// Warps: 0 TMA producer (Q, K ring), 1 MMA issuer (+ TMEM allocation), 2-5
// softmax of Q0, 6-9 softmax of Q1 (warp w reads TMEM lanes 32 * (w % 4)),
// 10 TMA producer (V ring).
constexpr int kPpThreads = 352;
#ifndef RS_PP_POLY_EVERY
#define RS_PP_POLY_EVERY 4
#endif
constexpr int kPolyEvery = RS_PP_POLY_EVERY;  // exp2 pairs on the FMA pipe: 1 in kPolyEvery (0: none)
#ifndef RS_PP_POLY_EVERY_VIT
#define RS_PP_POLY_EVERY_VIT 4
#endif
constexpr int kPolyEveryVit = RS_PP_POLY_EVERY_VIT;  // kVarlen (ViT: fewer MMAs per key with hd 80)
// dev timing builds only (wrong results): -DRS_PP_TIMING_NOEXP / -DRS_PP_TIMING_SKIP_SOFTMAX
#ifdef RS_PP_TIMING_NOEXP
constexpr bool kTimingNoExp = true;
#else
constexpr bool kTimingNoExp = false;
#endif
#ifdef RS_PP_TIMING_NO_PV
constexpr bool kTimingNoPv = true;
#else
constexpr bool kTimingNoPv = false;
#endif
#ifdef RS_PP_TIMING_NO_S
constexpr bool kTimingNoS = true;
#else
constexpr bool kTimingNoS = false;
#endif
#ifdef RS_PP_TIMING_NO_PWAIT
constexpr bool kTimingNoPWait = true;
#else
constexpr bool kTimingNoPWait = false;
#endif
#ifdef RS_PP_TIMING_NO_LOAD
constexpr bool kTimingNoLoad = true;
#else
constexpr bool kTimingNoLoad = false;
#endif
// P in two halves (keys 0-63, 64-127), each signalled as soon as it is in
// TMEM: the PV MMAs of the first half start while the softmax still
// exponentiates the second (-DRS_PP_PHALF=0: one signal per tile).
#ifndef RS_PP_PHALF
#define RS_PP_PHALF 1
#endif
constexpr bool kPHalf = RS_PP_PHALF != 0;
// Row sum of P after P is handed to the MMA warp (the exp loop only does
// scale, exp2, pack): -DRS_PP_SUM_AFTER_P=0 sums inside the loop.
#ifndef RS_PP_SUM_AFTER_P
#define RS_PP_SUM_AFTER_P 1
#endif
constexpr bool kSumAfterP = RS_PP_SUM_AFTER_P != 0;
// Softmax turn-taking (FA3-style ping-pong between the two softmax
// warpgroups): named barriers hand a token back and forth so only one tile's
// exp loop runs at a time while the tensor pipe works on the other tile.
// 0: off; 1: the token covers S load + max + exp; 2: the exp loop only.
#ifndef RS_PP_ORDER
#define RS_PP_ORDER 0
#endif
constexpr int kOrder = RS_PP_ORDER;
constexpr int kTurnBar0 = 8;  // named barrier ids 8 (tile 0's turn), 9 (tile 1's turn)
#ifdef RS_PP_TIMING_NO_SLOAD
constexpr bool kTimingNoSLoad = true;
#else
constexpr bool kTimingNoSLoad = false;
#endif
#ifdef RS_PP_TIMING_NO_PSTORE
constexpr bool kTimingNoPStore = true;
#else
constexpr bool kTimingNoPStore = false;
#endif
#ifdef RS_PP_TIMING_SKIP_SOFTMAX
constexpr bool kTimingSkipSoftmax = true;
#else
constexpr bool kTimingSkipSoftmax = false;
#endif

template <int HD>
struct PpCfg {
  static constexpr int kHdAtoms = HD / 64;
  static constexpr int kQBytes = kHdAtoms * kAtom;     // one 128-row Q tile
  static constexpr int kKBytes = kHdAtoms * kAtom;     // 128 keys
  static constexpr int kVAtom = HD * 128;              // V^T [HD x 64 keys]
  static constexpr int kVBytes = 2 * kVAtom;           // 128 keys
  // V ring: 2 stages (4 for small heads); K ring gets what is left (K_j is
  // needed a full PV earlier than V_j in the issue order)
  static constexpr int kBudget = 227 * 1024 - 2 * kQBytes - 1024 - 512;
  static constexpr int kVStages = HD <= 64 ? 4 : 2;
  static constexpr int kKFit = (kBudget - kVStages * kVBytes) / kKBytes;
  static constexpr int kKStages = kKFit > 4 ? 4 : kKFit;
  static constexpr int kSmem = 2 * kQBytes + kKStages * kKBytes + kVStages * kVBytes + 1024 + 512;
};

// Persistent: grid = min(units, 148) CTAs; unit u = (work item u / H, head
// u % H) in the callers' longest-first order, dealt to CTAs in a snake
// (round r: CTA c takes r*G + c, or r*G + G-1-c on odd rounds) so each SM
// gets a balanced mix of long and short units. Barrier phases, the K / V
// rings and the TMEM tiles carry over from unit to unit.
struct PpUnit {
  int head, kvh, q_row0, q_rows, q_pos0, key_begin, key_end;
  int rows_t[2], n_t[2], n_max;
  int ws_unit;     // index into the split workspace
  int splits;      // > 1: this unit writes a partial (split-KV)
  int jb, je;      // key tiles [jb, je) of this split (all of them without a split)
  int e_t[2];      // tile t's end: min(je, n_t); tile t takes part iff e_t > jb
  const int* pt;
};

template <KvMode MODE>
__device__ __forceinline__ PpUnit pp_unit(const TcParams& p, int u) {
  PpUnit x;
  x.ws_unit = u;
  const int pi = u / p.q_heads;
  x.head = u - pi * p.q_heads;
  const int4 pc = p.pieces[pi];
  const int w = pc.x, split = pc.y;
  x.splits = pc.z;
  x.kvh = x.head / (p.q_heads / p.kv_heads);
  x.q_pos0 = 0;
  x.pt = nullptr;
  const int4 it = p.inl[w];  // PrefillWork / AttnBlock, both 4 ints
  if constexpr (MODE == KvMode::kPaged) {
    x.q_row0 = it.x;
    x.q_rows = it.y;
    x.q_pos0 = it.z;
    x.key_begin = 0;
    x.key_end = it.z + it.y;
    x.pt = p.page_tables[it.w];  // producers only
  } else {
    x.q_row0 = it.x;
    x.q_rows = it.y;
    x.key_begin = it.z & ~7;  // 16-B aligned V^T tile start (extra keys masked)
    x.key_end = it.w;
  }
  x.rows_t[0] = min(x.q_rows, 128);
  x.rows_t[1] = max(x.q_rows - 128, 0);
#pragma unroll
  for (int t = 0; t < 2; ++t) {
    const int hi = MODE == KvMode::kPaged ? x.q_pos0 + 128 * t + x.rows_t[t] : x.key_end;
    x.n_t[t] = x.rows_t[t] > 0 ? (hi - x.key_begin + 127) / 128 : 0;
  }
  x.n_max = max(x.n_t[0], x.n_t[1]);
  kv_split_range(x.n_max, x.splits, split, x.jb, x.je);
  x.e_t[0] = min(x.je, x.n_t[0]);
  x.e_t[1] = min(x.je, x.n_t[1]);
  return x;
}

// unit of CTA c in round r (snake order), -1 when past the end
__device__ __forceinline__ int pp_unit_index(int r, int n_units) {
  const int G = static_cast<int>(gridDim.x), c = static_cast<int>(blockIdx.x);
  const int u = r * G + ((r & 1) ? G - 1 - c : c);
  return u < n_units ? u : -1;
}

template <int HD, KvMode MODE>
__global__ void __launch_bounds__(kPpThreads, 1)
    fa_pp_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                 const __grid_constant__ CUtensorMap tmV, const __grid_constant__ TcParams p, int n_units) {
  using C = PpCfg<HD>;
  constexpr int SK = C::kKStages, SV = C::kVStages;
  extern __shared__ __align__(1024) std::uint8_t smem_raw[];
  std::uint8_t* smem = reinterpret_cast<std::uint8_t*>(
      (reinterpret_cast<std::uintptr_t>(smem_raw) + 1023) & ~std::uintptr_t(1023));
  std::uint8_t* sQ = smem;  // [2][kQBytes]
  std::uint8_t* sK = sQ + 2 * C::kQBytes;
  std::uint8_t* sV = sK + SK * C::kKBytes;
  std::uint64_t* bars = reinterpret_cast<std::uint64_t*>(sV + SV * C::kVBytes);
  std::uint64_t* q_full = bars;            // [2]
  std::uint64_t* q_empty = bars + 2;       // [2] last S of the tile's unit issued+done
  std::uint64_t* k_full = bars + 4;        // [SK]
  std::uint64_t* k_empty = k_full + SK;    // [SK]
  std::uint64_t* v_full = k_empty + SK;    // [SV]
  std::uint64_t* v_empty = v_full + SV;    // [SV]
  std::uint64_t* s_full = v_empty + SV;    // [2] S_t,j ready (and PV_t,j-1 done)
  std::uint64_t* p_full = s_full + 2;      // [2 tiles][2 halves] P_t,j keys 0-63 / 64-127 written (4 softmax warps)
  std::uint64_t* o_final = p_full + 4;     // [2] last PV_t of a unit done
  std::uint32_t* tmem_holder = reinterpret_cast<std::uint32_t*>(o_final + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  pdl_launch_dependents();

  if (threadIdx.x == 0) {
    sm100::tma_prefetch_desc(&tmQ);
    sm100::tma_prefetch_desc(&tmK);
    sm100::tma_prefetch_desc(&tmV);
    for (int t = 0; t < 2; ++t) {
      sm100::mbar_init(&q_full[t], 1);
      sm100::mbar_init(&q_empty[t], 1);
      sm100::mbar_init(&s_full[t], 1);
      sm100::mbar_init(&p_full[2 * t], 4);  // one arrive per softmax warp
      sm100::mbar_init(&p_full[2 * t + 1], 4);
      sm100::mbar_init(&o_final[t], 1);
    }
    for (int i = 0; i < SK; ++i) {
      sm100::mbar_init(&k_full[i], 1);
      sm100::mbar_init(&k_empty[i], 1);
    }
    for (int i = 0; i < SV; ++i) {
      sm100::mbar_init(&v_full[i], 1);
      sm100::mbar_init(&v_empty[i], 1);
    }
    sm100::fence_mbar_init();
  }
  if (warp == 1) sm100::tmem_alloc(tmem_holder, 512);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const std::uint32_t tmem = *tmem_holder;
  pdl_wait();  // setup overlapped the previous kernel's tail
#ifdef RS_PP_TRACE_BUILD  // per-CTA span + work (dev): [start, end, units, tile products]
  unsigned long long* cta_tr = p.trace != nullptr ? p.trace + 4 * kPpTraceIters * kPpTraceEv + 4 * blockIdx.x : nullptr;
  if (cta_tr != nullptr && threadIdx.x == 0) {
    cta_tr[0] = pp_gtimer();
    unsigned long long nu = 0, np = 0;
    for (int r = 0;; ++r) {
      const int u = pp_unit_index(r, n_units);
      if (u < 0) break;
      const PpUnit x = pp_unit<MODE>(p, u);
      ++nu;
      np += max(0, x.e_t[0] - x.jb) + max(0, x.e_t[1] - x.jb);
    }
    cta_tr[2] = nu;
    cta_tr[3] = np;
  }
#endif

  auto pages = [&](const PpUnit& x, int j, int& pa, int& pb) {
    const int n_real_pages = (x.key_end - x.key_begin + 63) / 64;
    pa = x.pt[2 * j];
    pb = 2 * j + 1 < n_real_pages ? x.pt[2 * j + 1] : pa;  // duplicate: finite, masked
  };

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer: Q tiles and the K ring ----------------
    std::uint32_t qn[2] = {0, 0};
    std::uint32_t kn = 0;
    for (int r = 0;; ++r) {
      const int u = pp_unit_index(r, n_units);
      if (u < 0) break;
      const PpUnit x = pp_unit<MODE>(p, u);
      for (int t = 0; t < 2; ++t) {
        if (x.e_t[t] <= x.jb) continue;
        sm100::mbar_wait(&q_empty[t], (qn[t] & 1) ^ 1);
        ++qn[t];
        sm100::mbar_expect_tx(&q_full[t], C::kQBytes);
        for (int h = 0; h < C::kHdAtoms; ++h)
          sm100::tma_load_2d(sQ + t * C::kQBytes + h * kAtom, &tmQ, &q_full[t],
                             x.head * p.q_head_stride + h * 64, x.q_row0 + 128 * t);
      }
      for (int j = x.jb; j < x.je; ++j, ++kn) {
        const int st = static_cast<int>(kn % SK);
        std::uint8_t* k = sK + st * C::kKBytes;
        sm100::mbar_wait(&k_empty[st], ((kn / SK) & 1) ^ 1);
        if (kTimingNoLoad && kn >= SK) {
          sm100::mbar_arrive(&k_full[st]);
          continue;
        }
        sm100::mbar_expect_tx(&k_full[st], C::kKBytes);
        if constexpr (MODE == KvMode::kPaged) {
          int pa, pb;
          pages(x, j, pa, pb);
          for (int h = 0; h < C::kHdAtoms; ++h) {
            sm100::tma_load_2d(k + h * kAtom, &tmK, &k_full[st], h * 64, (pa * p.kv_heads + x.kvh) * 64);
            sm100::tma_load_2d(k + h * kAtom + 64 * 128, &tmK, &k_full[st], h * 64,
                               (pb * p.kv_heads + x.kvh) * 64);
          }
        } else {
          for (int h = 0; h < C::kHdAtoms; ++h)
            sm100::tma_load_2d(k + h * kAtom, &tmK, &k_full[st], x.kvh * p.q_head_stride + h * 64,
                               x.key_begin + 128 * j);
        }
      }
    }
  } else if (warp == kPpThreads / 32 - 1 && lane == 0) {
    // ---------------- TMA producer: the V ring (own thread: never queued behind K) ----------------
    std::uint32_t vn = 0;
    for (int r = 0;; ++r) {
      const int u = pp_unit_index(r, n_units);
      if (u < 0) break;
      const PpUnit x = pp_unit<MODE>(p, u);
      for (int j = x.jb; j < x.je; ++j, ++vn) {
        const int st = static_cast<int>(vn % SV);
        std::uint8_t* v = sV + st * C::kVBytes;
        sm100::mbar_wait(&v_empty[st], ((vn / SV) & 1) ^ 1);
        if (kTimingNoLoad && vn >= SV) {
          sm100::mbar_arrive(&v_full[st]);
          continue;
        }
        sm100::mbar_expect_tx(&v_full[st], C::kVBytes);
        if constexpr (MODE == KvMode::kPaged) {
          int pa, pb;
          pages(x, j, pa, pb);
          sm100::tma_load_2d(v, &tmV, &v_full[st], 0, (pa * p.kv_heads + x.kvh) * HD);
          sm100::tma_load_2d(v + C::kVAtom, &tmV, &v_full[st], 0, (pb * p.kv_heads + x.kvh) * HD);
        } else {
          const int k0 = x.key_begin + 128 * j;
          sm100::tma_load_2d(v, &tmV, &v_full[st], k0, x.kvh * HD);
          sm100::tma_load_2d(v + C::kVAtom, &tmV, &v_full[st], k0 + 64, x.kvh * HD);
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer: the whole warp runs the loop (converged,
    // every value derived from the kernel parameters: uniform registers);
    // one elected lane issues each tcgen05.mma / commit. The 512-column
    // allocation can only start at column 0: TMEM addresses are constants.
    if (tmem != 0) __trap();
    constexpr std::uint32_t idesc_s = sm100::idesc_bf16_f32(128, 128);
    // head-padded inputs (ViT: hd 80 in 128-wide tiles): the zero columns need
    // no MMA — S uses ceil(out_hd / 16) K steps, PV writes out_hd (rounded to 16) columns
    const int k_steps = (p.out_hd + 15) / 16;
    const std::uint32_t idesc_o = sm100::idesc_bf16_f32(128, min(HD, k_steps * 16));
    std::uint32_t qn[2] = {0, 0}, pn[2] = {0, 0};
    std::uint32_t kbase = 0;  // K / V tiles consumed before this unit
    for (int r = 0;; ++r) {
      const int u = pp_unit_index(r, n_units);
      if (u < 0) break;
      const PpUnit x = pp_unit<MODE>(p, u);
      for (int t = 0; t < 2; ++t)
        if (x.e_t[t] > x.jb) {
          sm100::mbar_wait(&q_full[t], qn[t] & 1);
          ++qn[t];
        }
      // last consumer of K_j / V_j (tile 1 covers every key tile tile 0 does)
      auto last_user = [&](int j) { return j < x.e_t[1] ? 1 : 0; };
      auto mma_s = [&](int t, int j) {
        const std::uint32_t kn = kbase + static_cast<std::uint32_t>(j - x.jb);
        const int st = static_cast<int>(kn % SK);
        sm100::mbar_wait(&k_full[st], (kn / SK) & 1);
        sm100::tc_fence_after();
        std::uint8_t* k = sK + st * C::kKBytes;
        if (sm100::elect_one()) {
#pragma unroll
          for (int h = 0; h < C::kHdAtoms; ++h) {
            const std::uint64_t qd = sm100::sw128_kmajor_desc(sm100::smem_u32(sQ + t * C::kQBytes + h * kAtom));
            const std::uint64_t kd = sm100::sw128_kmajor_desc(sm100::smem_u32(k + h * kAtom));
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              if (!kTimingNoS && 4 * h + kk < k_steps)
                sm100::umma_bf16(256u * t, qd + 2 * kk, kd + 2 * kk, idesc_s, (h | kk) != 0 ? 1u : 0u);
          }
        }
        __syncwarp();
        if (r == 0 && lane == 0) PP_TRACE(t, j - x.jb, 2);
        if (sm100::elect_one()) {
          sm100::umma_commit(&s_full[t]);
          if (t == last_user(j)) sm100::umma_commit(&k_empty[st]);
          if (j == (t == 0 ? x.e_t[0] : x.e_t[1]) - 1) sm100::umma_commit(&q_empty[t]);
        }
        __syncwarp();
      };
      auto mma_pv = [&](int t, int j) {
        const std::uint32_t vn = kbase + static_cast<std::uint32_t>(j - x.jb);
        const int st = static_cast<int>(vn % SV);
        sm100::mbar_wait(&v_full[st], (vn / SV) & 1);
        if (r == 0 && lane == 0) PP_TRACE(t, j - x.jb, 0);
        std::uint8_t* v = sV + st * C::kVBytes;
#pragma unroll
        for (int a = 0; a < 2; ++a) {  // key half a: P columns [32a, 32a + 32), V^T atom a
          if (a == 0 || kPHalf) {
            if (!kTimingNoPWait) sm100::mbar_wait(&p_full[2 * t + a], pn[t] & 1);
            sm100::tc_fence_after();
          }
          if (a == 0 && r == 0 && lane == 0) PP_TRACE(t, j - x.jb, 1);
          if (sm100::elect_one()) {
            const std::uint64_t vd = sm100::sw128_kmajor_desc(sm100::smem_u32(v + a * C::kVAtom));
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              if (!kTimingNoPv)
                sm100::umma_bf16_ts(256u * t + 128, 256u * t + 32 * a + 8 * kk, vd + 2 * kk, idesc_o,
                                    (j > x.jb || (a | kk) != 0) ? 1u : 0u);
          }
          __syncwarp();
        }
        ++pn[t];
        if (sm100::elect_one()) {
          if (t == last_user(j)) sm100::umma_commit(&v_empty[st]);
          if (j == (t == 0 ? x.e_t[0] : x.e_t[1]) - 1) sm100::umma_commit(&o_final[t]);
        }
        __syncwarp();
      };
      if (x.e_t[0] > x.jb) mma_s(0, x.jb);
      if (x.e_t[1] > x.jb) mma_s(1, x.jb);
      for (int j = x.jb + 1; j <= x.je; ++j) {
        if (j - 1 < x.e_t[0]) mma_pv(0, j - 1);
        if (j < x.e_t[0]) mma_s(0, j);
        if (j - 1 < x.e_t[1]) mma_pv(1, j - 1);
        if (j < x.e_t[1]) mma_s(1, j);
      }
      kbase += static_cast<std::uint32_t>(x.je - x.jb);
    }
  } else if (warp >= 2 && warp < 10) {
    // ---------------- softmax: tile t, one query row per thread ----------------
    const int t = (warp - 2) >> 2;
    const int quad = warp & 3;
    const int r = quad * 32 + lane;  // row within the tile
    const std::uint32_t lane_off = static_cast<std::uint32_t>(quad * 32) << 16;
    const std::uint32_t s_tm = tmem + lane_off + 256 * t;
    const std::uint32_t o_tm = s_tm + 128;
    std::uint32_t sn = 0, on = 0;
    if (kOrder != 0 && t == 1) sm100::named_bar_arrive(kTurnBar0, 256);  // tile 0 goes first
    for (int rr = 0;; ++rr) {
      const int u = pp_unit_index(rr, n_units);
      if (u < 0) break;
      const PpUnit x = pp_unit<MODE>(p, u);
      // iterations both tiles run take turns; a tile's extra ones do not
      const int n_common = max(0, min(x.e_t[0], x.e_t[1]) - x.jb);
      const int j_end = t == 0 ? x.e_t[0] : x.e_t[1];
      const int my_rows = t == 0 ? x.rows_t[0] : x.rows_t[1];
      if (j_end <= x.jb) continue;
      int lo, hi;
      if constexpr (MODE == KvMode::kPaged) {
        lo = 0;
        hi = min(x.q_pos0 + 128 * t + r + 1, x.key_end);
      } else {
        const int row = x.q_row0 + 128 * t + min(r, my_rows - 1);
        int a = 0, b = p.n_seqs;  // largest s with cu[s] <= row
        while (b - a > 1) {
          const int mid = (a + b) >> 1;
          if (p.cu_seqlens[mid] <= row) a = mid;
          else b = mid;
        }
        lo = p.cu_seqlens[a];
        hi = p.cu_seqlens[a + 1];
      }
      float m = -INFINITY, l = 0.f;
      for (int j = x.jb; j < j_end; ++j) {
        if (rr == 0 && r == 0) PP_TRACE(2 + t, j - x.jb, 0);
        sm100::mbar_wait(&s_full[t], sn & 1);
        if (rr == 0 && r == 0) PP_TRACE(2 + t, j - x.jb, 1);
        ++sn;
        sm100::tc_fence_after();
        const bool turn = kOrder != 0 && j - x.jb < n_common;
        if (kOrder == 1 && turn) sm100::named_bar_sync(kTurnBar0 + t, 256);
        if constexpr (kTimingSkipSoftmax) {  // dev timing: pipeline floor (P = raw S bits)
          sm100::tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            sm100::mbar_arrive(&p_full[2 * t]);
            if (kPHalf) sm100::mbar_arrive(&p_full[2 * t + 1]);
          }
          continue;
        }
        const int key0 = x.key_begin + j * 128;
        const int c_lo = lo - key0, c_hi = hi - key0;  // visible columns [c_lo, c_hi)
        std::uint32_t sv[128];
        if constexpr (kTimingNoSLoad) {  // dev timing: S not read from TMEM (wrong results)
#pragma unroll
          for (int c = 0; c < 128; ++c) sv[c] = __float_as_uint(static_cast<float>((c * 7 + lane) & 15) * 0.25f);
        } else {
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            std::uint32_t(&v)[32] = *reinterpret_cast<std::uint32_t(*)[32]>(&sv[32 * c]);
            sm100::tmem_ld_32x32b_x32(s_tm + 32 * c, v);
          }
          sm100::tmem_ld_wait();
        }
        if (rr == 0 && r == 0) PP_TRACE(2 + t, j - x.jb, 3);
        if (!(c_lo <= 0 && c_hi >= 128)) {
#pragma unroll
          for (int q = 0; q < 128; ++q)
            if (q < c_lo || q >= c_hi) sv[q] = __float_as_uint(-INFINITY);
        }
        float mx8[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) mx8[q] = __uint_as_float(sv[q]);
#pragma unroll
        for (int q = 8; q < 128; ++q) mx8[q & 7] = fmaxf(mx8[q & 7], __uint_as_float(sv[q]));
        float mx = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                         fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7])));
        mx *= p.scale_log2;
        if (rr == 0 && r == 0) PP_TRACE(2 + t, j - x.jb, 4);
        const bool raise = mx > m + 8.f || (m == -INFINITY && mx != -INFINITY);
        float alpha = 1.f;
        if (raise) {
          alpha = m == -INFINITY ? 0.f : exp2f(m - mx);
          m = mx;
        }
        if (j > x.jb && __any_sync(0xffffffffu, raise && alpha != 1.f)) {
          // rare: rescale O_t in TMEM (PV_t,j-1 is complete: S_t,j was issued after it)
#pragma unroll 1
          for (int c = 0; c < HD / 32; ++c) {
            std::uint32_t v[32];
            sm100::tmem_ld_32x32b_x32(o_tm + 32 * c, v);
            sm100::tmem_ld_wait();
#pragma unroll
            for (int q = 0; q < 32; ++q) v[q] = __float_as_uint(__uint_as_float(v[q]) * alpha);
            sm100::tmem_st_32x32b_x32(o_tm + 32 * c, v);
          }
        }
        if (kOrder == 2 && turn) sm100::named_bar_sync(kTurnBar0 + t, 256);
        const float mneg = m == -INFINITY ? 0.f : -m;
        const float2 scale2 = make_float2(p.scale_log2, p.scale_log2), mneg2 = make_float2(mneg, mneg);
        float2 rs2[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                         make_float2(0.f, 0.f)};
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          std::uint32_t packed[16];  // 32 keys as bf16 pairs
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            const float2 x = fma2(make_float2(__uint_as_float(sv[32 * c + 2 * q]),
                                              __uint_as_float(sv[32 * c + 2 * q + 1])),
                                  scale2, mneg2);
            float2 e;
            constexpr int kPe = MODE == KvMode::kVarlen ? kPolyEveryVit : kPolyEvery;
            if (kPe > 0 && q % kPe == kPe - 1) {  // every kPe-th pair on the FMA pipe
              e = poly_exp2_fma2(x);
            } else if (kTimingNoExp) {
              e = x;
            } else {
              e.x = fast_exp2(x.x);
              e.y = fast_exp2(x.y);
            }
            if constexpr (kSumAfterP) {  // keep e: the row sum runs after P is released
              sv[32 * c + 2 * q] = __float_as_uint(e.x);
              sv[32 * c + 2 * q + 1] = __float_as_uint(e.y);
            } else {
              rs2[q & 3] = add2(rs2[q & 3], e);
            }
            packed[q] = pack_bf16x2(e.x, e.y);
          }
          if constexpr (!kTimingNoPStore) sm100::tmem_st_32x32b_x16(s_tm + 16 * c, packed);
          else if (packed[0] == 0x12345u && packed[15] == 0x54321u) sm100::tmem_st_32x32b_x16(s_tm + 16 * c, packed);
          if (kPHalf && c == 1) {  // keys 0-63 in TMEM: their PV MMAs may start
            sm100::tmem_st_wait();
            sm100::tc_fence_before();
            __syncwarp();
            if (lane == 0) sm100::mbar_arrive(&p_full[2 * t]);
          }
        }
        if (rr == 0 && r == 0) PP_TRACE(2 + t, j - x.jb, 5);
        if (turn) sm100::named_bar_arrive(kTurnBar0 + (t ^ 1), 256);  // the other tile's turn
        sm100::tmem_st_wait();
        if (rr == 0 && r == 0) PP_TRACE(2 + t, j - x.jb, 6);
        sm100::tc_fence_before();
        __syncwarp();  // the warp's P stores are complete
        if (rr == 0 && r == 0) PP_TRACE(2 + t, j - x.jb, 2);
        if (lane == 0) sm100::mbar_arrive(&p_full[kPHalf ? 2 * t + 1 : 2 * t]);
        if constexpr (kSumAfterP) {  // off the S -> P -> PV critical path
#pragma unroll
          for (int q = 0; q < 64; ++q)
            rs2[q & 3] = add2(rs2[q & 3], make_float2(__uint_as_float(sv[2 * q]), __uint_as_float(sv[2 * q + 1])));
        }
        const float2 r01 = add2(rs2[0], rs2[1]), r23 = add2(rs2[2], rs2[3]);
        const float2 rsum = add2(r01, r23);
        l = l * alpha + (rsum.x + rsum.y);
      }
      sm100::mbar_wait(&o_final[t], on & 1);
      ++on;
      sm100::tc_fence_after();
      if constexpr (MODE == KvMode::kPaged) {
        if (x.splits > 1) {  // unnormalised partial + (m, l) for pp_merge_kernel
          const std::int64_t prow = static_cast<std::int64_t>(x.ws_unit) * 256 + 128 * t + r;
          float4* po = reinterpret_cast<float4*>(p.part_o + prow * HD);
#pragma unroll
          for (int c = 0; c < HD / 32; ++c) {
            std::uint32_t v[32];
            sm100::tmem_ld_32x32b_x32(o_tm + 32 * c, v);
            sm100::tmem_ld_wait();
            if (r < my_rows) {
#pragma unroll
              for (int q = 0; q < 8; ++q)
                po[8 * c + q] = make_float4(__uint_as_float(v[4 * q]), __uint_as_float(v[4 * q + 1]),
                                            __uint_as_float(v[4 * q + 2]), __uint_as_float(v[4 * q + 3]));
            }
          }
          if (r < my_rows) reinterpret_cast<float2*>(p.part_ml)[prow] = make_float2(m, l);
          sm100::tc_fence_before();
          continue;
        }
      }
      const float inv = l > 0.f ? 1.f / l : 0.f;
      bf16* orow = p.out + static_cast<std::int64_t>(x.q_row0 + 128 * t + r) * p.ld_out + x.head * p.out_hd;
#pragma unroll
      for (int c = 0; c < HD / 32; ++c) {
        if (32 * c >= p.out_hd) break;  // head padding (uniform)
        std::uint32_t v[32];
        sm100::tmem_ld_32x32b_x32(o_tm + 32 * c, v);
        sm100::tmem_ld_wait();
        if (r < my_rows) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            if (32 * c + 8 * q < p.out_hd)
              reinterpret_cast<uint4*>(orow + 32 * c)[q] = make_uint4(
                  pack_bf16x2(__uint_as_float(v[8 * q]) * inv, __uint_as_float(v[8 * q + 1]) * inv),
                  pack_bf16x2(__uint_as_float(v[8 * q + 2]) * inv, __uint_as_float(v[8 * q + 3]) * inv),
                  pack_bf16x2(__uint_as_float(v[8 * q + 4]) * inv, __uint_as_float(v[8 * q + 5]) * inv),
                  pack_bf16x2(__uint_as_float(v[8 * q + 6]) * inv, __uint_as_float(v[8 * q + 7]) * inv));
          }
        }
      }
      // O_t is read out (tcgen05.ld waited): the next unit's first PV may overwrite it
      sm100::tc_fence_before();
    }
    if (kOrder != 0 && t == 0) sm100::named_bar_sync(kTurnBar0, 256);  // tile 1's last hand-back
  }
  __syncthreads();
#ifdef RS_PP_TRACE_BUILD
  if (cta_tr != nullptr && threadIdx.x == 0) cta_tr[1] = pp_gtimer();
#endif
  if (warp == 1) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc(tmem, 512);
  }
}

// Split-KV merge: one warp per (work item, head, query row) of the items
// with S > 1, splits combined in index order (deterministic):
// O = sum_s 2^(m_s - M) O_s / sum_s 2^(m_s - M) l_s. Split s holds row q iff
// its range is non-empty and starts at or below q (then key jb * 128 <= q is
// visible and m_s is finite).
template <int HD>
__global__ void __launch_bounds__(256) pp_merge_kernel(const __grid_constant__ TcParams p) {
  pdl_wait();
  pdl_launch_dependents();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wh = blockIdx.x;
  const int w = wh / p.q_heads, head = wh - w * p.q_heads;
  const int2 sp = p.item_split[w];
  const int S = sp.x;
  if (S <= 1) return;
  const int row = blockIdx.y * 8 + warp;
  const int4 wk = p.inl[w];  // PrefillWork
  if (row >= wk.y) return;
  const int q = wk.z + row;
  const int n_tiles = (wk.z + wk.y + 127) / 128;
  auto prow = [&](int s) {  // workspace row of split s
    return (static_cast<std::int64_t>(sp.y + s) * p.q_heads + head) * 256 + row;
  };
  const float2* ml = reinterpret_cast<const float2*>(p.part_ml);
  float M = -INFINITY;
  for (int s = 0; s < S; ++s) {
    int jb, je;
    kv_split_range(n_tiles, S, s, jb, je);
    if (je > jb && q >= jb * 128) M = fmaxf(M, ml[prow(s)].x);
  }
  constexpr int kPer = HD / 32;
  float acc[kPer];
#pragma unroll
  for (int i = 0; i < kPer; ++i) acc[i] = 0.f;
  float L = 0.f;
  for (int s = 0; s < S; ++s) {
    int jb, je;
    kv_split_range(n_tiles, S, s, jb, je);
    if (!(je > jb && q >= jb * 128)) continue;
    const float2 v = ml[prow(s)];
    const float wgt = exp2f(v.x - M);
    L += wgt * v.y;
    const float* po = p.part_o + prow(s) * HD + lane * kPer;
    if constexpr (kPer == 4) {
      const float4 o = *reinterpret_cast<const float4*>(po);
      acc[0] += wgt * o.x;
      acc[1] += wgt * o.y;
      acc[2] += wgt * o.z;
      acc[3] += wgt * o.w;
    } else {
      const float2 o = *reinterpret_cast<const float2*>(po);
      acc[0] += wgt * o.x;
      acc[1] += wgt * o.y;
    }
  }
  const float inv = L > 0.f ? 1.f / L : 0.f;
  bf16* orow = p.out + static_cast<std::int64_t>(wk.x + row) * p.ld_out + head * p.out_hd + lane * kPer;
  if constexpr (kPer == 4)
    *reinterpret_cast<uint2*>(orow) = make_uint2(pack_bf16x2(acc[0] * inv, acc[1] * inv),
                                                 pack_bf16x2(acc[2] * inv, acc[3] * inv));
  else
    *reinterpret_cast<std::uint32_t*>(orow) = pack_bf16x2(acc[0] * inv, acc[1] * inv);
}

// ---- tensor maps ----------------------------------------------------------------
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q{};
    RS_CUDA_CHECK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q));
    if (ptr == nullptr || q != cudaDriverEntryPointSuccess)
      throw DeviceError(RS_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    return reinterpret_cast<EncodeTiledFn>(ptr);
  }();
  return fn;
}

// 2D bf16 [rows, cols] row-major (stride ld), box [box_rows, 64 cols], SW128.
CUtensorMap map_2d(const void* base, std::int64_t rows, std::int64_t cols, std::int64_t ld,
                   int box_rows) {
  CUtensorMap tm;
  std::memset(&tm, 0, sizeof tm);
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 2};
  const cuuint32_t box[2] = {64u, static_cast<cuuint32_t>(box_rows)};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode_fn()(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base),
                                 dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw DeviceError(RS_ERR_CUDA, "attention tensor map failed (" + std::to_string(r) + ")");
  return tm;
}

struct MapKey {
  const void* p;
  std::int64_t rows, cols, ld;
  int box;
  bool operator==(const MapKey& o) const {
    return p == o.p && rows == o.rows && cols == o.cols && ld == o.ld && box == o.box;
  }
};
struct MapHash {
  std::size_t operator()(const MapKey& k) const {
    return std::hash<const void*>()(k.p) ^ (static_cast<std::size_t>(k.rows) * 31) ^
           (static_cast<std::size_t>(k.cols) << 20) ^ (static_cast<std::size_t>(k.box) << 40);
  }
};

CUtensorMap cached_map(const void* base, std::int64_t rows, std::int64_t cols, std::int64_t ld,
                       int box_rows) {
  static std::mutex mu;
  static std::unordered_map<MapKey, CUtensorMap, MapHash> cache;
  const MapKey key{base, rows, cols, ld, box_rows};
  std::lock_guard<std::mutex> g(mu);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  if (cache.size() > 4096) cache.clear();
  return cache.emplace(key, map_2d(base, rows, cols, ld, box_rows)).first->second;
}

template <int HD, KvMode MODE>
void launch(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv, const TcParams& p,
            int n_blocks, cudaStream_t st, const char* klass) {
  static bool set = false;
  if (!set) {
    RS_CUDA_CHECK(cudaFuncSetAttribute(fa_tc_kernel<HD, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       TcCfg<HD>::kSmem));
    RS_CUDA_CHECK(cudaFuncSetAttribute(fa_pp_kernel<HD, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       PpCfg<HD>::kSmem));
    set = true;
  }
  if (n_blocks > 65535) throw DeviceError(RS_ERR_CUDA, "tc attention: too many blocks for grid.y");
  dim3 grid(p.q_heads, n_blocks);
  const int tok = prof::begin(st);
  if (attn_unit_rows() == 256) {
    const int units = p.q_heads * p.n_pieces;
    static const bool trace = std::getenv("RS_PP_TRACE") != nullptr;
    TcParams q = p;
    const std::size_t tn = 4 * kPpTraceIters * kPpTraceEv + 4 * kNumSMs;
    if (trace) {
      RS_CUDA_CHECK(cudaMallocAsync(reinterpret_cast<void**>(&q.trace), tn * 8, st));
      RS_CUDA_CHECK(cudaMemsetAsync(q.trace, 0, tn * 8, st));
    }
    launch_kernel(fa_pp_kernel<HD, MODE>, dim3(std::min(units, kNumSMs)), dim3(kPpThreads), PpCfg<HD>::kSmem,
                  st, 1, tq, tk, tv, q, units);
    if (trace) {  // ns relative to the first stamp: MMA (wait-P begin, end, S issued), softmax (wait-S begin, end, P arrive)
      std::vector<unsigned long long> h(tn);
      RS_CUDA_CHECK(cudaMemcpyAsync(h.data(), q.trace, tn * 8, cudaMemcpyDeviceToHost, st));
      RS_CUDA_CHECK(cudaStreamSynchronize(st));
      RS_CUDA_CHECK(cudaFree(q.trace));
      unsigned long long t0 = ~0ull;
      for (std::size_t i = 0; i < 4 * kPpTraceIters * kPpTraceEv; ++i) if (h[i]) t0 = std::min(t0, h[i]);
      {  // per-CTA spans (dev build): start / end spread, work per CTA
        const unsigned long long* c = h.data() + 4 * kPpTraceIters * kPpTraceEv;
        const int G = std::min(units, kNumSMs);
        unsigned long long s0 = ~0ull, s1 = 0, e0 = ~0ull, e1 = 0, p0 = ~0ull, p1 = 0, u1 = 0;
        double ps = 0;
        for (int i = 0; i < G; ++i) {
          if (c[4 * i] == 0) continue;
          s0 = std::min(s0, c[4 * i]); s1 = std::max(s1, c[4 * i]);
          e0 = std::min(e0, c[4 * i + 1]); e1 = std::max(e1, c[4 * i + 1]);
          p0 = std::min(p0, c[4 * i + 3]); p1 = std::max(p1, c[4 * i + 3]); u1 = std::max(u1, c[4 * i + 2]);
          ps += static_cast<double>(c[4 * i + 3]);
        }
        std::fprintf(stderr, "[pp-cta] ctas %d units %d: start spread %llu ns, end first %llu last %llu ns; "
                     "products/CTA min %llu mean %.1f max %llu; max units/CTA %llu\n", G, units, s1 - s0, e0 - s0,
                     e1 - s0, p0, ps / G, p1, u1);
      }
      auto at = [&](int role, int it, int ev) {
        const unsigned long long v = h[(static_cast<std::size_t>(role) * kPpTraceIters + it) * kPpTraceEv + ev];
        return v ? static_cast<long long>(v - t0) : -1ll;
      };
      std::fprintf(stderr, "[pp-trace] it | mma t0: waitP0 gotP0 S0issued | mma t1: waitP1 gotP1 S1issued | "
                           "sm0: waitS gotS ldS max expd stw Parrive (ns)\n");
      for (int it = 0; it < kPpTraceIters; ++it)
        std::fprintf(stderr, "[pp-trace] %2d | %6lld %6lld %6lld | %6lld %6lld %6lld | %6lld %6lld %6lld %6lld %6lld %6lld %6lld\n", it,
                     at(0, it, 0), at(0, it, 1), at(0, it, 2), at(1, it, 0), at(1, it, 1), at(1, it, 2),
                     at(2, it, 0), at(2, it, 1), at(2, it, 3), at(2, it, 4), at(2, it, 5), at(2, it, 6), at(2, it, 2));
    }
    if (p.max_split > 1) {
      launch_kernel(pp_merge_kernel<HD>, dim3(p.q_heads * n_blocks, 256 / 8), dim3(256), 0, st, 1, p);
      count_launch();
    }
  }
  else
    launch_kernel(fa_tc_kernel<HD, MODE>, grid, dim3(kTcThreads), TcCfg<HD>::kSmem, st, 1, tq, tk, tv, p);
  RS_LAUNCH_CHECK();
  // algorithmic FLOPs (4 hd per (query, visible key) per head): paged items
  // see keys [0, q_pos0 + r]; varlen blocks their sequence [key_begin, key_end)
  double flops = 0;
  if (tok >= 0) {
    for (int i = 0; i < n_blocks; ++i) {
      const int4 it = p.inl[i];
      if (MODE == KvMode::kPaged)
        flops += static_cast<double>(it.y) * it.z + 0.5 * static_cast<double>(it.y) * (it.y + 1);
      else
        flops += static_cast<double>(it.y) * (it.w - it.z);
    }
    flops *= 4.0 * p.out_hd * p.q_heads;
  }
  if (tok >= 0 && MODE == KvMode::kPaged) {
    // per-shape class "attn_prefill_tcgen05|items|max_keys|splits" (bench groups on the prefix)
    char label[96];
    std::snprintf(label, sizeof label, "%s|%d|%d|%d", klass, n_blocks, p.max_keys, p.n_pieces);
    prof::end(tok, st, label, flops, 0);
  } else {
    prof::end(tok, st, klass, flops, 0);
  }
  count_launch();
}

}  // namespace

int attn_unit_rows() {
  static const int rows = [] {
    const char* e = std::getenv("RS_ATTN_PINGPONG");
    return e != nullptr && e[0] == '0' ? 128 : 256;
  }();
  return rows;
}

// split-KV workspace per stream (stream-ordered; released with the stream)
struct PpWs {
  float* buf = nullptr;
  std::size_t floats = 0;
};
std::mutex& pp_ws_mutex() {
  static std::mutex mu;
  return mu;
}
std::unordered_map<cudaStream_t, PpWs>& pp_ws_all() {
  static std::unordered_map<cudaStream_t, PpWs> all;
  return all;
}

// ---- piece planning (host) -------------------------------------------------
// Cost of one (item, split) piece in (query tile, key tile) pairs plus a fixed
// per-unit cost (Q load, pipeline fill, epilogue) and, for splits, the partial
// write + merge; mirrors pp_unit's ranges.
double piece_cost(const int4& it, bool paged, int S, int s) {
  const int q_rows = it.y;
  const int q_pos0 = paged ? it.z : 0;
  const int key_begin = paged ? 0 : (it.z & ~7);
  const int key_end = paged ? it.z + it.y : it.w;
  const int rows_t[2] = {std::min(q_rows, 128), std::max(q_rows - 128, 0)};
  int n_t[2];
  for (int t = 0; t < 2; ++t) {
    const int hi = paged ? q_pos0 + 128 * t + rows_t[t] : key_end;
    n_t[t] = rows_t[t] > 0 ? (hi - key_begin + 127) / 128 : 0;
  }
  int jb, je;
  kv_split_range(std::max(n_t[0], n_t[1]), S, s, jb, je);
  int pairs = 0;
  for (int t = 0; t < 2; ++t) pairs += std::max(0, std::min(je, n_t[t]) - jb);
  return pairs + 4.0 + (S > 1 ? 6.0 : 0.0);
}

struct PiecePlan {
  std::vector<int4> items;  // cache key
  int heads = 0;
  bool paged = false;
  int forced = 0;
  std::vector<int4> pieces;
  std::vector<int2> item_split;
  int max_split = 1;
};

void build_pieces(PiecePlan& pl, const std::vector<int>& S, std::vector<double>* costs) {
  struct P {
    int4 pc;
    double cost;
  };
  std::vector<P> ps;
  const int n = static_cast<int>(pl.items.size());
  pl.item_split.assign(static_cast<std::size_t>(n), make_int2(1, 0));
  for (int w = 0; w < n; ++w)
    for (int s = 0; s < S[w]; ++s)
      ps.push_back({make_int4(w, s, S[w], 0), piece_cost(pl.items[w], pl.paged, S[w], s)});
  std::stable_sort(ps.begin(), ps.end(), [](const P& a, const P& b) { return a.cost > b.cost; });
  // each item's splits must be contiguous for the merge: order items by their
  // largest piece, splits of an item adjacent
  std::vector<int> first(static_cast<std::size_t>(n), -1);
  std::vector<P> out;
  for (const P& x : ps) {
    const int w = x.pc.x;
    if (first[w] >= 0) continue;
    first[w] = static_cast<int>(out.size());
    for (int s = 0; s < S[w]; ++s)
      out.push_back({make_int4(w, s, S[w], first[w]), piece_cost(pl.items[w], pl.paged, S[w], s)});
    pl.item_split[w] = make_int2(S[w], first[w]);
  }
  pl.pieces.clear();
  if (costs) costs->clear();
  pl.max_split = 1;
  for (const P& x : out) {
    pl.pieces.push_back(x.pc);
    if (costs) costs->push_back(x.cost);
    pl.max_split = std::max(pl.max_split, x.pc.z);
  }
}

// Longest CTA of the kernel's snake dealing (grid = min(units, SMs)).
double snake_makespan(const std::vector<double>& cost, int heads) {
  const int units = static_cast<int>(cost.size()) * heads;
  const int G = std::min(units, kNumSMs);
  std::vector<double> load(static_cast<std::size_t>(G), 0.0);
  for (int u = 0; u < units; ++u) {
    const int r = u / G, i = u - r * G;
    load[static_cast<std::size_t>((r & 1) ? G - 1 - i : i)] += cost[static_cast<std::size_t>(u / heads)];
  }
  return *std::max_element(load.begin(), load.end());
}

// Pieces of a launch: no split for kVarlen; for kPaged, items are split
// greedily (the item owning the costliest piece first, up to 8 ways, >= 2 key
// tiles per split) while that shortens the snake makespan. Cached: the 28
// layers of a chunk plan the same list.
const PiecePlan& plan_pieces(const int4* items, int n, int heads, bool paged) {
  // several live plans: the encoder's and the prefill's launches interleave
  // on the host thread (a single entry would re-plan every prefill layer)
  static thread_local std::vector<PiecePlan> cache;
  int forced = 0;
  if (paged) {
    const char* e = std::getenv("RS_ATTN_KV_SPLITS");  // A/B and tests: every item split S ways
    if (e != nullptr && e[0] != '\0') forced = std::max(1, std::min(16, std::atoi(e)));
  }
  for (std::size_t i = 0; i < cache.size(); ++i) {
    const PiecePlan& c = cache[i];
    if (c.heads == heads && c.paged == paged && c.forced == forced && static_cast<int>(c.items.size()) == n &&
        std::memcmp(c.items.data(), items, static_cast<std::size_t>(n) * sizeof(int4)) == 0) {
      if (i != 0) std::swap(cache[0], cache[i]);  // most recent first
      return cache[0];
    }
  }
  if (cache.size() >= 16) cache.pop_back();
  cache.insert(cache.begin(), PiecePlan{});
  PiecePlan& pl = cache[0];
  pl.items.assign(items, items + n);
  pl.heads = heads;
  pl.paged = paged;
  pl.forced = forced;
  std::vector<int> S(static_cast<std::size_t>(n), 1);
  std::vector<double> cost;
  if (forced > 0) {
    std::fill(S.begin(), S.end(), std::max(1, std::min(forced, kMaxPieces / std::max(1, n))));
    build_pieces(pl, S, nullptr);
    return pl;
  }
  build_pieces(pl, S, &cost);
  // host cost matters (planned once per chunk, on the launch path): only
  // launches of at most two waves are planned, one candidate per step
  if (!paged || attn_unit_rows() != 256 || n * heads > 2 * kNumSMs) return pl;
  double best = snake_makespan(cost, heads);
  PiecePlan trial = pl;
  std::vector<double> c2;
  for (int iter = 0; iter < 16; ++iter) {
    const int w = pl.pieces.front().x;  // the item owning the costliest piece
    const int4& it = pl.items[static_cast<std::size_t>(w)];
    const int n_tiles = (it.z + it.y + 127) / 128;
    if (S[w] >= 8 || n_tiles < 2 * (S[w] + 1) || static_cast<int>(pl.pieces.size()) + 1 > kMaxPieces) break;
    ++S[w];
    build_pieces(trial, S, &c2);
    const double m = snake_makespan(c2, heads);
    if (!(m < 0.97 * best)) break;  // clear gains only (the merge and partial writes are not free)
    best = m;
    pl.pieces.swap(trial.pieces);
    pl.item_split.swap(trial.item_split);
    pl.max_split = trial.max_split;
  }
  return pl;
}

void set_pieces(TcParams& p, const PiecePlan& pl) {
  std::memcpy(p.pieces, pl.pieces.data(), pl.pieces.size() * sizeof(int4));
  std::memcpy(p.item_split, pl.item_split.data(), pl.item_split.size() * sizeof(int2));
  p.n_pieces = static_cast<int>(pl.pieces.size());
  p.max_split = pl.max_split;
}

void attention_prefill_paged_tc(const bf16* q, int ld_q, int q_rows_alloc, bf16* out, int ld_out,
                                const PrefillWork* work, const PrefillWork* work_host, int n_work,
                                int max_keys, const PagedKV& kv, std::int64_t kv_pages, int q_heads,
                                int kv_heads, int head_dim, float scale, cudaStream_t stream) {
  if (n_work <= 0) return;
  if (kv.page_size != 64) throw DeviceError(RS_ERR_CUDA, "tc attention needs 64-token pages");
  if (work_host == nullptr) throw DeviceError(RS_ERR_CUDA, "tc attention: host work list required");
  if (n_work > kInlineUnits) {  // batches of inlined work items (independent rows)
    for (int o = 0; o < n_work; o += kInlineUnits)
      attention_prefill_paged_tc(q, ld_q, q_rows_alloc, out, ld_out, work + o, work_host + o,
                                 std::min(kInlineUnits, n_work - o), max_keys, kv, kv_pages, q_heads,
                                 kv_heads, head_dim, scale, stream);
    return;
  }
  TcParams p{};
  static_assert(sizeof(PrefillWork) == sizeof(int4), "inline work item layout");
  std::memcpy(p.inl, work_host, static_cast<std::size_t>(n_work) * sizeof(int4));
  {
    HostPhase ph("attn.plan");
    set_pieces(p, plan_pieces(p.inl, n_work, q_heads, true));
  }
  p.max_keys = max_keys;
  if (p.max_split > 1) {
    std::lock_guard<std::mutex> g(pp_ws_mutex());
    PpWs& ws = pp_ws_all()[stream];
    const std::size_t rows = static_cast<std::size_t>(p.n_pieces) * q_heads * 256;
    const std::size_t need = rows * (head_dim + 2);
    if (ws.floats < need) {
      if (ws.buf != nullptr) RS_CUDA_CHECK(cudaFreeAsync(ws.buf, stream));
      RS_CUDA_CHECK(cudaMallocAsync(reinterpret_cast<void**>(&ws.buf), need * sizeof(float), stream));
      ws.floats = need;
    }
    p.part_o = ws.buf;
    p.part_ml = ws.buf + rows * head_dim;
  }
  p.work = work;
  p.page_tables = kv.page_tables;
  p.q_heads = q_heads;
  p.kv_heads = kv_heads;
  p.q_head_stride = head_dim;
  p.out_hd = head_dim;
  p.scale_log2 = scale * 1.4426950408889634f;
  p.out = out;
  p.ld_out = ld_out;
  const CUtensorMap tq = cached_map(q, q_rows_alloc, (q_heads + 2 * kv_heads) * head_dim, ld_q, 128);
  const CUtensorMap tk = cached_map(kv.k, kv_pages * kv_heads * 64, head_dim, head_dim, 64);
  const CUtensorMap tv = cached_map(kv.v, kv_pages * kv_heads * head_dim, 64, 64, head_dim);
  switch (head_dim) {
    case 64: return launch<64, KvMode::kPaged>(tq, tk, tv, p, n_work, stream, "attn_prefill_tcgen05");
    case 128: return launch<128, KvMode::kPaged>(tq, tk, tv, p, n_work, stream, "attn_prefill_tcgen05");
    default: throw DeviceError(RS_ERR_CUDA, "tc attention: unsupported head_dim " + std::to_string(head_dim));
  }
}

void attention_varlen_tc(const bf16* qp, const bf16* kp, const bf16* vt, int rows_alloc,
                         int heads, bf16* out, int ld_out, int out_hd, const AttnBlock* blocks,
                         const AttnBlock* blocks_host, int n_blocks, const int* cu_seqlens, int n_seqs,
                         float scale, cudaStream_t stream) {
  if (n_blocks <= 0) return;
  if (blocks_host == nullptr) throw DeviceError(RS_ERR_CUDA, "tc attention: host block list required");
  if (n_blocks > kInlineUnits) {
    for (int o = 0; o < n_blocks; o += kInlineUnits)
      attention_varlen_tc(qp, kp, vt, rows_alloc, heads, out, ld_out, out_hd, blocks + o, blocks_host + o,
                          std::min(kInlineUnits, n_blocks - o), cu_seqlens, n_seqs, scale, stream);
    return;
  }
  constexpr int HD = 128;
  TcParams p{};
  static_assert(sizeof(AttnBlock) == sizeof(int4), "inline block layout");
  std::memcpy(p.inl, blocks_host, static_cast<std::size_t>(n_blocks) * sizeof(int4));
  set_pieces(p, plan_pieces(p.inl, n_blocks, heads, false));
  p.blocks = blocks;
  p.cu_seqlens = cu_seqlens;
  p.n_seqs = n_seqs;
  p.q_heads = heads;
  p.kv_heads = heads;
  p.q_head_stride = HD;
  p.out_hd = out_hd;
  p.scale_log2 = scale * 1.4426950408889634f;
  p.out = out;
  p.ld_out = ld_out;
  const CUtensorMap tq = cached_map(qp, rows_alloc, heads * HD, heads * HD, 128);
  const CUtensorMap tk = cached_map(kp, rows_alloc, heads * HD, heads * HD, 128);
  const CUtensorMap tv = cached_map(vt, static_cast<std::int64_t>(heads) * HD, rows_alloc, rows_alloc, HD);
  launch<HD, KvMode::kVarlen>(tq, tk, tv, p, n_blocks, stream, "attn_vit_tcgen05");
}

void attention_tc_release_stream(cudaStream_t st) {
  std::lock_guard<std::mutex> g(pp_ws_mutex());
  auto it = pp_ws_all().find(st);
  if (it == pp_ws_all().end()) return;
  if (it->second.buf) cudaFreeAsync(it->second.buf, st);
  pp_ws_all().erase(it);
}

}  // namespace rserve
