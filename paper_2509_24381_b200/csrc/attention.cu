// rserve-b200 — flash attention kernels (see attention.cuh).
//
// CTA = 4 warps x 16 query rows = 64 queries of one head; K/V tiles of 64
// keys double-buffered in shared memory via cp.async; S = QK^T and O += PV
// on bf16 m16n8k16 tensor-core MMAs with fp32 accumulation; online softmax
// in base-2 with fp32 running max / sum.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
#include <mutex>
#include <unordered_map>

#include "attention.cuh"
#include "common.cuh"

namespace rserve {
namespace {

constexpr int kQ = 64;   // queries per CTA
constexpr int kKV = 64;  // keys per tile

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  const std::uint32_t s = static_cast<std::uint32_t>(__cvta_generic_to_shared(smem));
  const int n = valid ? 16 : 0;  // 0 -> zero fill
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(n)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void ldsm_x4(std::uint32_t (&r)[4], const void* p) {
  const std::uint32_t s = static_cast<std::uint32_t>(__cvta_generic_to_shared(p));
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(s));
}
__device__ __forceinline__ void ldsm_x4_t(std::uint32_t (&r)[4], const void* p) {
  const std::uint32_t s = static_cast<std::uint32_t>(__cvta_generic_to_shared(p));
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(s));
}
__device__ __forceinline__ void mma_bf16(float (&d)[4], const std::uint32_t (&a)[4],
                                         std::uint32_t b0, std::uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 "
      "{%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// Where the keys of a CTA come from.
struct BidirSource {  // packed QKV rows of one sequence
  const bf16* base;   // row 0 of the sequence, K columns of this head
  const bf16* vbase;  // V columns
  int ld;
  int n_keys;
  __device__ const bf16* k_row(int key) const { return base + static_cast<std::int64_t>(key) * ld; }
  __device__ const bf16* v_row(int key) const { return vbase + static_cast<std::int64_t>(key) * ld; }
};
// NBUF = 2: K/V tiles double-buffered; 1: single tile (windows of <= 64
// keys): half the shared memory, so more CTAs are resident per SM.
template <int HD, int NBUF = 2>
struct Smem {
  static constexpr int kLd = HD + 8;  // +16 B pad: conflict-free ldmatrix
  bf16 q[kQ][kLd];
  bf16 k[NBUF][kKV][kLd];
  bf16 v[NBUF][kKV][kLd];
};

// Rotary (rotate-half pairs (i, i + HD/2), cos / sin from a [rows, HD/2]
// float2 table) applied in shared memory to `rows` rows of a tile: the ViT's
// 2D RoPE fused into the window attention (no separate q / k pass).
template <int HD>
__device__ __forceinline__ void rope_tile_smem(bf16 (*t)[HD + 8], int rows, const float2* table) {
  constexpr int kHalf = HD / 2, kPairs = kHalf / 2;  // bf16x2 pairs per half row
  for (int e = threadIdx.x; e < rows * kPairs; e += blockDim.x) {
    const int r = e / kPairs, i = (e % kPairs) * 2;
    std::uint32_t* pa = reinterpret_cast<std::uint32_t*>(&t[r][i]);
    std::uint32_t* pb = reinterpret_cast<std::uint32_t*>(&t[r][i + kHalf]);
    const float2 a = unpack_bf16x2(*pa), b = unpack_bf16x2(*pb);
    const float2 c0 = table[r * kHalf + i], c1 = table[r * kHalf + i + 1];
    *pa = pack_bf16x2(a.x * c0.x - b.x * c0.y, a.y * c1.x - b.y * c1.y);
    *pb = pack_bf16x2(b.x * c0.x + a.x * c0.y, b.y * c1.x + a.y * c1.y);
  }
}

// Core: q rows [q_row0, q_row0 + q_rows) (row stride ld_q, head columns at
// q_ptr), keys [0, src.n_keys). Causal when q_pos0 >= 0: key j visible to
// query i iff j <= q_pos0 + i. With q_rope / k_rope (tables at query row 0 /
// key 0) q and k are rotated in shared memory after their loads.
template <int HD, int NBUF, typename Src>
__device__ void flash_block(const bf16* q_ptr, int ld_q, int q_rows, int q_pos0, const Src& src,
                            bf16* o_ptr, int ld_o, float scale_log2, Smem<HD, NBUF>& sm,
                            const float2* q_rope = nullptr, const float2* k_rope = nullptr) {
  constexpr int kDC = HD / 16;  // d chunks (k dim of QK^T)
  constexpr int kNT = HD / 8;   // d n-tiles of O
  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;
  const int g = lane >> 2, tig = lane & 3;
  const bool causal = q_pos0 >= 0;

  // Load Q (zero rows past the end).
  for (int i = tid; i < kQ * (HD / 8); i += blockDim.x) {
    const int r = i / (HD / 8), c = (i % (HD / 8)) * 8;
    const bool ok = r < q_rows;
    cp_async16(&sm.q[r][c], q_ptr + static_cast<std::int64_t>(ok ? r : 0) * ld_q + c, ok);
  }
  int n_keys = src.n_keys;
  if (causal) n_keys = min(n_keys, q_pos0 + q_rows);
  const int n_tiles = (n_keys + kKV - 1) / kKV;
  auto load_kv = [&](int t, int buf) {
    for (int i = tid; i < kKV * (HD / 8); i += blockDim.x) {
      const int r = i / (HD / 8), c = (i % (HD / 8)) * 8;
      const int key = t * kKV + r;
      const bool ok = key < n_keys;
      cp_async16(&sm.k[buf][r][c], src.k_row(ok ? key : 0) + c, ok);
      cp_async16(&sm.v[buf][r][c], src.v_row(ok ? key : 0) + c, ok);
    }
  };
  if (n_tiles > 0) load_kv(0, 0);
  cp_async_commit();

  std::uint32_t qf[kDC][4];
  float oacc[kNT][4];
#pragma unroll
  for (int j = 0; j < kNT; ++j) oacc[j][0] = oacc[j][1] = oacc[j][2] = oacc[j][3] = 0.f;
  float m_run[2] = {-INFINITY, -INFINITY};
  float l_run[2] = {0.f, 0.f};
  const int q_base = warp * 16;

  for (int t = 0; t < n_tiles; ++t) {
    const int buf = NBUF == 2 ? (t & 1) : 0;
    if (NBUF == 2 && t + 1 < n_tiles) load_kv(t + 1, buf ^ 1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    if (k_rope != nullptr) {
      if (t == 0) rope_tile_smem<HD>(sm.q, q_rows, q_rope);
      rope_tile_smem<HD>(sm.k[buf], min(kKV, n_keys - t * kKV), k_rope + static_cast<std::int64_t>(t) * kKV * (HD / 2));
      __syncthreads();
    }
    if (t == 0) {
#pragma unroll
      for (int c = 0; c < kDC; ++c) {
        const int row = q_base + (lane & 7) + ((lane >> 3) & 1) * 8;
        const int col = c * 16 + (lane >> 4) * 8;
        ldsm_x4(qf[c], &sm.q[row][col]);
      }
    }
    // S = Q K^T : 16 x 64 per warp
    float s[8][4];
#pragma unroll
    for (int j = 0; j < 8; ++j) s[j][0] = s[j][1] = s[j][2] = s[j][3] = 0.f;
#pragma unroll
    for (int c = 0; c < kDC; ++c) {
#pragma unroll
      for (int jp = 0; jp < 4; ++jp) {
        std::uint32_t kb[4];
        const int row = jp * 16 + (lane & 7) + ((lane >> 4) << 3);
        const int col = c * 16 + ((lane >> 3) & 1) * 8;
        ldsm_x4(kb, &sm.k[buf][row][col]);
        mma_bf16(s[2 * jp], qf[c], kb[0], kb[1]);
        mma_bf16(s[2 * jp + 1], qf[c], kb[2], kb[3]);
      }
    }
    // Scale + mask + online softmax (rows g and g+8 of this warp).
    float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
    for (int j = 0; j < 8; ++j) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int key = t * kKV + j * 8 + tig * 2 + (e & 1);
        const int qi = q_base + g + (e >> 1) * 8;
        bool ok = key < n_keys;
        if (causal) ok = ok && key <= q_pos0 + qi;
        const float v = ok ? s[j][e] * scale_log2 : -INFINITY;
        s[j][e] = v;
        mx[e >> 1] = fmaxf(mx[e >> 1], v);
      }
    }
    float alpha[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      mx[h] = fmaxf(mx[h], __shfl_xor_sync(0xffffffffu, mx[h], 1));
      mx[h] = fmaxf(mx[h], __shfl_xor_sync(0xffffffffu, mx[h], 2));
      const float m_new = fmaxf(m_run[h], mx[h]);
      alpha[h] = m_new == -INFINITY ? 1.f : exp2f(m_run[h] - m_new);
      m_run[h] = m_new;
    }
    float rs[2] = {0.f, 0.f};
    std::uint32_t pf[4][4];  // P as A fragments, 4 key chunks of 16
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      float p[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float m = m_run[e >> 1];
        p[e] = m == -INFINITY ? 0.f : exp2f(s[j][e] - m);
        rs[e >> 1] += p[e];
      }
      const int kc = j >> 1;
      if ((j & 1) == 0) {
        pf[kc][0] = pack_bf16x2(p[0], p[1]);
        pf[kc][1] = pack_bf16x2(p[2], p[3]);
      } else {
        pf[kc][2] = pack_bf16x2(p[0], p[1]);
        pf[kc][3] = pack_bf16x2(p[2], p[3]);
      }
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      rs[h] += __shfl_xor_sync(0xffffffffu, rs[h], 1);
      rs[h] += __shfl_xor_sync(0xffffffffu, rs[h], 2);
      l_run[h] = l_run[h] * alpha[h] + rs[h];
    }
#pragma unroll
    for (int j = 0; j < kNT; ++j) {
      oacc[j][0] *= alpha[0];
      oacc[j][1] *= alpha[0];
      oacc[j][2] *= alpha[1];
      oacc[j][3] *= alpha[1];
    }
    // O += P V
#pragma unroll
    for (int kc = 0; kc < 4; ++kc) {
#pragma unroll
      for (int np = 0; np < kNT / 2; ++np) {
        std::uint32_t vb[4];
        const int row = kc * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
        const int col = np * 16 + (lane >> 4) * 8;
        ldsm_x4_t(vb, &sm.v[buf][row][col]);
        mma_bf16(oacc[2 * np], pf[kc], vb[0], vb[1]);
        mma_bf16(oacc[2 * np + 1], pf[kc], vb[2], vb[3]);
      }
    }
    __syncthreads();
  }
  cp_async_wait<0>();
  // Normalise and store.
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int r = q_base + g + h * 8;
    if (r >= q_rows) continue;
    const float inv = l_run[h] > 0.f ? 1.f / l_run[h] : 0.f;
    bf16* orow = o_ptr + static_cast<std::int64_t>(r) * ld_o;
#pragma unroll
    for (int j = 0; j < kNT; ++j) {
      *reinterpret_cast<std::uint32_t*>(orow + j * 8 + tig * 2) =
          pack_bf16x2(oacc[j][2 * h] * inv, oacc[j][2 * h + 1] * inv);
    }
  }
}

template <int HD, int NBUF>
__global__ void __launch_bounds__(128, NBUF == 1 ? 4 : 1) varlen_bidir_kernel(const bf16* __restrict__ qkv, int ld,
                                                           bf16* __restrict__ out, int ld_out,
                                                           const int* __restrict__ cu, int heads,
                                                           float scale_log2, const float2* rope) {
  extern __shared__ __align__(16) std::uint8_t smem_raw[];
  Smem<HD, NBUF>& sm = *reinterpret_cast<Smem<HD, NBUF>*>(smem_raw);
  pdl_wait();
  pdl_launch_dependents();
  const int seq = blockIdx.y, head = blockIdx.z;
  const int s0 = cu[seq], s1 = cu[seq + 1];
  const int q0 = blockIdx.x * kQ;
  const int len = s1 - s0;
  if (q0 >= len) return;
  BidirSource src{qkv + static_cast<std::int64_t>(s0) * ld + (heads + head) * HD,
                  qkv + static_cast<std::int64_t>(s0) * ld + (2 * heads + head) * HD, ld, len};
  flash_block<HD, NBUF>(qkv + static_cast<std::int64_t>(s0 + q0) * ld + head * HD, ld, min(kQ, len - q0),
                  -1, src, out + static_cast<std::int64_t>(s0 + q0) * ld_out + head * HD, ld_out,
                  scale_log2, sm,
                  rope != nullptr ? rope + static_cast<std::int64_t>(s0 + q0) * (HD / 2) : nullptr,
                  rope != nullptr ? rope + static_cast<std::int64_t>(s0) * (HD / 2) : nullptr);
}

constexpr float kLog2e = 1.4426950408889634f;

template <int HD, int NBUF>
void launch_bidir_n(const bf16* qkv, int ld, bf16* out, int ld_out, const int* cu, int n_seqs,
                    int max_seqlen, int heads, float scale, cudaStream_t st, const float2* rope) {
  const int smem = sizeof(Smem<HD, NBUF>);
  static bool set = false;
  if (!set) {
    RS_CUDA_CHECK(cudaFuncSetAttribute(varlen_bidir_kernel<HD, NBUF>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    set = true;
  }
  dim3 grid(ceil_div(max_seqlen, kQ), n_seqs, heads);
  const int tok = prof::begin(st);
  launch_kernel(varlen_bidir_kernel<HD, NBUF>, grid, dim3(128), smem, st, 1, qkv, ld, out, ld_out, cu, heads,
                scale * kLog2e, rope);
  RS_LAUNCH_CHECK();
  prof::end(tok, st, "attn_vit_mma", 0, 0);
  count_launch();
}

template <int HD>
void launch_bidir(const bf16* qkv, int ld, bf16* out, int ld_out, const int* cu, int n_seqs,
                  int max_seqlen, int heads, float scale, cudaStream_t st, const float2* rope) {
  if (max_seqlen <= kKV)  // one key tile per sequence (ViT windows)
    launch_bidir_n<HD, 1>(qkv, ld, out, ld_out, cu, n_seqs, max_seqlen, heads, scale, st, rope);
  else
    launch_bidir_n<HD, 2>(qkv, ld, out, ld_out, cu, n_seqs, max_seqlen, heads, scale, st, rope);
}

}  // namespace

void attention_varlen_bidir(const bf16* qkv, int ld_qkv, bf16* out, int ld_out,
                            const int* cu_seqlens, int n_seqs, int max_seqlen, int /*total*/,
                            int heads, int head_dim, float scale, cudaStream_t stream,
                            const float2* rope_table) {
  if (n_seqs <= 0 || max_seqlen <= 0) return;
  switch (head_dim) {
    case 64: return launch_bidir<64>(qkv, ld_qkv, out, ld_out, cu_seqlens, n_seqs, max_seqlen, heads, scale, stream, rope_table);
    case 80: return launch_bidir<80>(qkv, ld_qkv, out, ld_out, cu_seqlens, n_seqs, max_seqlen, heads, scale, stream, rope_table);
    case 128: return launch_bidir<128>(qkv, ld_qkv, out, ld_out, cu_seqlens, n_seqs, max_seqlen, heads, scale, stream, rope_table);
    default: throw DeviceError(RS_ERR_CUDA, "attention: unsupported head_dim " + std::to_string(head_dim));
  }
}


// ---- decode attention -----------------------------------------------
// One query row per request (the token being decoded) against its paged KV.
// HBM-bound: each K / V byte is read once per kv head, so the kernel is built
// to keep the whole KV stream in flight, not for FLOPs:
//   * a CTA = 4 warps over a contiguous range of key tiles (64-token pages) of
//     one (request, kv head); every warp cp.asyncs its own K and V^T page pair
//     (32 KB for hd 128) into a private swizzled smem slot, so one CTA per SM
//     has 4 pages in flight and a 8.6k-token request's 4 kv heads spread over
//     all SMs with ~one page per warp;
//   * the G = Hq / Hkv query heads of the kv head are the M rows of bf16
//     m16n8k16 MMAs (padded to 16): S = Q K^T takes K rows as the B operand
//     (ldmatrix, no transpose), S's accumulator layout is P's A-operand layout,
//     and O = P V takes the cached V^T rows as B (no transpose either);
//   * every page but the one holding this step's token is loaded before the
//     PDL wait (overlapping the QKV GEMV / RoPE-append kernels before it);
//   * online softmax per warp in base 2, the 4 warps merged in shared memory,
//     the CTAs of a (request, kv head) merged by a one-warp-per-head merge
//     kernel launched under PDL, all in split order: deterministic.
namespace {

constexpr int kDecWarps = 4;
constexpr int kDecThreads = 32 * kDecWarps;
constexpr int kDecMaxG = 16;  // MMA rows
constexpr int kDecTile = 64;  // keys per tile = one KV page

template <int HD>
struct DecCfg {
  static constexpr int kKChunks = HD / 8;                    // 16-B chunks per K row
  static constexpr int kTileBytes = 2 * kDecTile * HD * 2;   // K + V^T of one page
  static constexpr int kScratch = kDecWarps * (kDecMaxG * HD + 2 * kDecMaxG) * 4;
  static constexpr int kSmem = kDecWarps * kTileBytes > kScratch ? kDecWarps * kTileBytes : kScratch;
};

// swizzled byte offsets: 16-B chunk c of row r (8 consecutive rows hit 8 distinct bank groups)
template <int HD>
__device__ __forceinline__ std::uint32_t dec_k_off(int r, int c) {
  return static_cast<std::uint32_t>(r * HD * 2 + ((c ^ (r & 7)) << 4));
}
__device__ __forceinline__ std::uint32_t dec_v_off(int r, int c) {  // V^T rows: 64 keys = 128 B
  return static_cast<std::uint32_t>(r * 128 + ((c ^ (r & 7)) << 4));
}

template <int HD>
__global__ void __launch_bounds__(kDecThreads, 1) decode_attn_kernel(
    const bf16* __restrict__ qkv, int ld_q, const PrefillWork* __restrict__ work,
    const bf16* __restrict__ k_cache, const bf16* __restrict__ v_cache, const int* const* page_tables,
    int q_heads, int kv_heads, int tiles_per_split, float scale_log2, float* part_o, float* part_ml,
    int splits, bf16* out, int ld_out, unsigned long long* trace) {
  using C = DecCfg<HD>;
  // RS_DEC_TRACE (dev): globaltimer per CTA at the phase boundaries
  auto stamp = [&](int k) {
    if (trace != nullptr && threadIdx.x == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      trace[(static_cast<std::size_t>(blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x) * 8 + k] = t;
    }
  };
  extern __shared__ __align__(128) std::uint8_t dsm[];
  stamp(0);
  const int split = blockIdx.x, kvh = blockIdx.y, req = blockIdx.z;
  const int G = q_heads / kv_heads;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t4 = lane & 3;  // MMA fragment row group / column pair
  // work items and page tables are host uploads (stream-ordered before this
  // launch), and every page but the one holding this step's token is stable:
  // those K / V loads are issued before the PDL wait, overlapping the
  // preceding kernels (QKV GEMV, RoPE + KV append)
  const PrefillWork w = work[req];
  const int n_keys = w.q_pos0 + 1;  // keys [0, pos] (this token's K / V appended by the preceding kernel)
  const int n_tiles = (n_keys + kDecTile - 1) / kDecTile;
  const int t_new = n_tiles - 1;
  const int t0 = split * tiles_per_split, t1 = min(n_tiles, t0 + tiles_per_split);
  const int* pt = page_tables[w.req_slot];
  std::uint8_t* my = dsm + warp * C::kTileBytes;
  auto issue = [&](int t) {
    const std::int64_t page = pt[t];
    const bf16* kp = k_cache + (page * kv_heads + kvh) * kDecTile * HD;
    const bf16* vp = v_cache + (page * kv_heads + kvh) * HD * kDecTile;
#pragma unroll
    for (int i = 0; i < kDecTile * HD / 8 / 32; ++i) {
      const int q = lane + 32 * i;
      cp_async16(my + dec_k_off<HD>(q / C::kKChunks, q % C::kKChunks), kp + 8 * q, true);
      cp_async16(my + kDecTile * HD * 2 + dec_v_off(q / 8, q % 8), vp + 8 * q, true);
    }
    cp_async_commit();
  };
  bool issued = t0 + warp < t1 && t0 + warp != t_new;
  if (issued) issue(t0 + warp);
  stamp(1);
  pdl_wait();  // q and this token's K / V come from the preceding kernels
  pdl_launch_dependents();

  // Q as the A operand (rows = heads g, g + 8; zero beyond G), unscaled bf16
  const bf16* qrow = qkv + static_cast<std::int64_t>(w.q_row0) * ld_q + kvh * G * HD;
  std::uint32_t qa[HD / 16][4];
#pragma unroll
  for (int kk = 0; kk < HD / 16; ++kk) {
    const int d = 16 * kk + 2 * t4;
    qa[kk][0] = g < G ? *reinterpret_cast<const std::uint32_t*>(qrow + g * HD + d) : 0u;
    qa[kk][1] = g + 8 < G ? *reinterpret_cast<const std::uint32_t*>(qrow + (g + 8) * HD + d) : 0u;
    qa[kk][2] = g < G ? *reinterpret_cast<const std::uint32_t*>(qrow + g * HD + d + 8) : 0u;
    qa[kk][3] = g + 8 < G ? *reinterpret_cast<const std::uint32_t*>(qrow + (g + 8) * HD + d + 8) : 0u;
  }
  float o[HD / 8][4];
#pragma unroll
  for (int j = 0; j < HD / 8; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;
  float m_r[2] = {-INFINITY, -INFINITY}, l_r[2] = {0.f, 0.f};  // rows g, g + 8 (l: this thread's columns)

  for (int t = t0 + warp; t < t1; t += kDecWarps) {
    if (!issued) issue(t);
    issued = false;
    if (t == t0 + warp) stamp(2);
    cp_async_wait<0>();
    if (t == t0 + warp) stamp(3);
    const int valid = min(kDecTile, n_keys - t * kDecTile);
    if (valid < kDecTile) {  // keys past the end: V^T columns zeroed (P is 0 there; keep 0 * V finite)
      __syncwarp();  // every lane's copies have landed before any lane overwrites part of them
      for (int r = lane; r < HD; r += 32)
        for (int k = valid; k < kDecTile; ++k)
          *reinterpret_cast<bf16*>(my + kDecTile * HD * 2 + dec_v_off(r, k >> 3) + 2 * (k & 7)) = f2bf(0.f);
    }
    __syncwarp();
    // S = Q K^T: 8 key n-tiles x HD/16 k-steps; K rows are the col-major B operand
    float s[kDecTile / 8][4];
#pragma unroll
    for (int n = 0; n < kDecTile / 8; ++n) s[n][0] = s[n][1] = s[n][2] = s[n][3] = 0.f;
#pragma unroll
    for (int n = 0; n < kDecTile / 8; n += 2) {
#pragma unroll
      for (int kk = 0; kk < HD / 16; ++kk) {
        std::uint32_t b[4];  // (keys 8n.., d chunk 2kk), (.., 2kk+1), (keys 8n+8.., 2kk), (.., 2kk+1)
        const int r = 8 * (n + (lane >> 4)) + (lane & 7), c = 2 * kk + ((lane >> 3) & 1);
        ldsm_x4(b, my + dec_k_off<HD>(r, c));
        mma_bf16(s[n], qa[kk], b[0], b[1]);
        mma_bf16(s[n + 1], qa[kk], b[2], b[3]);
      }
    }
    // online softmax (rows g: s[n][0..1], g + 8: s[n][2..3]; keys 8n + 2 t4 + {0, 1})
    float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
    for (int n = 0; n < kDecTile / 8; ++n)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int key = 8 * n + 2 * t4 + (e & 1);
        s[n][e] = key < valid ? s[n][e] * scale_log2 : -INFINITY;
        mx[e >> 1] = fmaxf(mx[e >> 1], s[n][e]);
      }
    float alpha[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      mx[h] = fmaxf(mx[h], __shfl_xor_sync(0xffffffffu, mx[h], 1));
      mx[h] = fmaxf(mx[h], __shfl_xor_sync(0xffffffffu, mx[h], 2));
      const float m_new = fmaxf(m_r[h], mx[h]);  // finite: every tile has >= 1 valid key
      alpha[h] = exp2f(m_r[h] - m_new);
      m_r[h] = m_new;
      l_r[h] *= alpha[h];
    }
#pragma unroll
    for (int j = 0; j < HD / 8; ++j) {
      o[j][0] *= alpha[0];
      o[j][1] *= alpha[0];
      o[j][2] *= alpha[1];
      o[j][3] *= alpha[1];
    }
#pragma unroll
    for (int n = 0; n < kDecTile / 8; ++n)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        s[n][e] = exp2f(s[n][e] - m_r[e >> 1]);
        l_r[e >> 1] += s[n][e];
      }
    // O += P V: P from S's accumulators (A layout), V^T rows as the B operand
#pragma unroll
    for (int kk = 0; kk < kDecTile / 16; ++kk) {
      const std::uint32_t pa[4] = {pack_bf16x2(s[2 * kk][0], s[2 * kk][1]), pack_bf16x2(s[2 * kk][2], s[2 * kk][3]),
                                   pack_bf16x2(s[2 * kk + 1][0], s[2 * kk + 1][1]),
                                   pack_bf16x2(s[2 * kk + 1][2], s[2 * kk + 1][3])};
#pragma unroll
      for (int j = 0; j < HD / 8; j += 2) {
        std::uint32_t b[4];  // (d 8j.., key chunk 2kk), (.., 2kk+1), (d 8j+8.., 2kk), (.., 2kk+1)
        const int r = 8 * (j + (lane >> 4)) + (lane & 7), c = 2 * kk + ((lane >> 3) & 1);
        ldsm_x4(b, my + kDecTile * HD * 2 + dec_v_off(r, c));
        mma_bf16(o[j], pa, b[0], b[1]);
        mma_bf16(o[j + 1], pa, b[2], b[3]);
      }
    }
    __syncwarp();  // this tile's ldmatrix reads are done before the next cp.async overwrites the slot
  }
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    l_r[h] += __shfl_xor_sync(0xffffffffu, l_r[h], 1);
    l_r[h] += __shfl_xor_sync(0xffffffffu, l_r[h], 2);
  }
  stamp(4);
  // merge the 4 warps (in warp order) through shared memory (the K / V slots are dead)
  __syncthreads();
  float* so = reinterpret_cast<float*>(dsm);                       // [warp][16][HD]
  float* sml = so + kDecWarps * kDecMaxG * HD;                     // [warp][16][2]
  float* swt = sml + kDecWarps * kDecMaxG * 2;                     // [warp][16] weights
  float* sL = swt + kDecWarps * kDecMaxG;                          // [16] (M, l) of the CTA
#pragma unroll
  for (int j = 0; j < HD / 8; ++j) {
    float* r0 = so + (warp * kDecMaxG + g) * HD + 8 * j + 2 * t4;
    float* r1 = so + (warp * kDecMaxG + g + 8) * HD + 8 * j + 2 * t4;
    *reinterpret_cast<float2*>(r0) = make_float2(o[j][0], o[j][1]);
    *reinterpret_cast<float2*>(r1) = make_float2(o[j][2], o[j][3]);
  }
  if (t4 == 0) {
    *reinterpret_cast<float2*>(sml + (warp * kDecMaxG + g) * 2) = make_float2(m_r[0], l_r[0]);
    *reinterpret_cast<float2*>(sml + (warp * kDecMaxG + g + 8) * 2) = make_float2(m_r[1], l_r[1]);
  }
  __syncthreads();
  if (tid < G) {  // per head: the warps' weights 2^(m_w - M) and the CTA's (M, l)
    float M = -INFINITY;
#pragma unroll
    for (int v = 0; v < kDecWarps; ++v) M = fmaxf(M, sml[(v * kDecMaxG + tid) * 2]);
    float l = 0.f;
#pragma unroll
    for (int v = 0; v < kDecWarps; ++v) {
      const float wv = M == -INFINITY ? 0.f : exp2f(sml[(v * kDecMaxG + tid) * 2] - M);  // idle warp: 0
      swt[v * kDecMaxG + tid] = wv;
      l += wv * sml[(v * kDecMaxG + tid) * 2 + 1];
    }
    *reinterpret_cast<float2*>(sL + 2 * tid) = make_float2(M, l);
  }
  __syncthreads();
  const std::int64_t head0 = static_cast<std::int64_t>(req) * q_heads + kvh * G;
  constexpr int kQ4 = HD / 4;
  for (int i = tid; i < G * kQ4; i += kDecThreads) {
    const int h = i / kQ4, d = 4 * (i % kQ4);
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int v = 0; v < kDecWarps; ++v) {
      const float wv = swt[v * kDecMaxG + h];
      const float4 x = *reinterpret_cast<const float4*>(so + (v * kDecMaxG + h) * HD + d);
      acc.x += wv * x.x;
      acc.y += wv * x.y;
      acc.z += wv * x.z;
      acc.w += wv * x.w;
    }
    if (splits == 1) {
      const float l = sL[2 * h + 1], inv = l > 0.f ? 1.f / l : 0.f;
      bf16* o4 = out + static_cast<std::int64_t>(w.q_row0) * ld_out + (kvh * G + h) * HD + d;
      *reinterpret_cast<uint2*>(o4) =
          make_uint2(pack_bf16x2(acc.x * inv, acc.y * inv), pack_bf16x2(acc.z * inv, acc.w * inv));
    } else {
      *reinterpret_cast<float4*>(part_o + ((head0 + h) * splits + split) * HD + d) = acc;
    }
  }
  if (splits == 1) return;
  if (tid < G) *reinterpret_cast<float2*>(part_ml + ((head0 + tid) * splits + split) * 2) =
      *reinterpret_cast<const float2*>(sL + 2 * tid);
  __syncthreads();
  stamp(5);
}

// Split merge: one warp per (query head, request), HD / 32 columns per lane;
// split weights 2^(m_s - M) computed once per lane-strided split and
// broadcast by shuffles, up to kMergeChunk partial rows in flight, summed in
// split order (deterministic). PDL: launched while the split kernel runs.
constexpr int kMergeChunk = 40;
template <int HD>
__global__ void __launch_bounds__(32) decode_attn_merge_kernel(const float* part_o, const float* part_ml, int q_heads,
                                                               int splits, bf16* out, int ld_out,
                                                               const PrefillWork* __restrict__ work) {
  constexpr int V = HD / 32;
  const int head = blockIdx.x, req = blockIdx.y, lane = threadIdx.x;
  const int row0 = work[req].q_row0;  // host upload: read before the wait
  pdl_wait();
  pdl_launch_dependents();
  const std::int64_t base = (static_cast<std::int64_t>(req) * q_heads + head) * splits;
  const float2* ml = reinterpret_cast<const float2*>(part_ml) + base;
  float M = -INFINITY;
  for (int s2 = lane; s2 < splits; s2 += 32) M = fmaxf(M, __ldcg(&ml[s2].x));
  M = warp_max(M);
  float acc[V];
#pragma unroll
  for (int v = 0; v < V; ++v) acc[v] = 0.f;
  float lpart = 0.f;
  for (int s0 = 0; s0 < splits; s0 += kMergeChunk) {
    float wl[2];  // weights of splits s0 + lane, s0 + 32 + lane
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int s2 = s0 + 32 * q + lane;
      wl[q] = 0.f;
      if (32 * q + lane < kMergeChunk && s2 < splits && M != -INFINITY) {
        const float2 v = __ldcg(&ml[s2]);
        wl[q] = exp2f(v.x - M);
        lpart += wl[q] * v.y;
      }
    }
    float x[kMergeChunk][V];
#pragma unroll
    for (int k = 0; k < kMergeChunk; ++k) {
      const float* src = part_o + (base + s0 + k) * HD + V * lane;
#pragma unroll
      for (int v = 0; v < V; ++v) x[k][v] = s0 + k < splits ? __ldcg(src + v) : 0.f;
    }
#pragma unroll
    for (int k = 0; k < kMergeChunk; ++k) {
      const float wv = __shfl_sync(0xffffffffu, wl[k >> 5], k & 31);
#pragma unroll
      for (int v = 0; v < V; ++v) acc[v] += wv * x[k][v];
    }
  }
  const float l = warp_sum(lpart);
  const float inv = l > 0.f ? 1.f / l : 0.f;
  bf16* o = out + static_cast<std::int64_t>(row0) * ld_out + head * HD + V * lane;
#pragma unroll
  for (int v = 0; v < V; v += 2) *reinterpret_cast<std::uint32_t*>(o + v) = pack_bf16x2(acc[v] * inv, acc[v + 1] * inv);
}

struct DecodeWs {
  float* buf = nullptr;
  std::size_t floats = 0;
};
std::mutex& decode_ws_mutex() {
  static std::mutex mu;
  return mu;
}
std::unordered_map<cudaStream_t, DecodeWs>& decode_ws_all() {  // per stream, released with it
  static std::unordered_map<cudaStream_t, DecodeWs> all;
  return all;
}

template <int HD>
void launch_decode(dim3 grid, cudaStream_t st, const bf16* qkv, int ld_q, const PrefillWork* work,
                   const PagedKV& kv, int q_heads, int kv_heads, int tiles_per_split, float scale_log2,
                   float* part_o, float* part_ml, int splits, bf16* out, int ld_out) {
  static const bool attr = [] {
    RS_CUDA_CHECK(cudaFuncSetAttribute(decode_attn_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       DecCfg<HD>::kSmem));
    return true;
  }();
  (void)attr;
  static const bool trace = std::getenv("RS_DEC_TRACE") != nullptr;
  unsigned long long* tr = nullptr;
  const std::size_t n_cta = static_cast<std::size_t>(grid.x) * grid.y * grid.z;
  if (trace) {
    RS_CUDA_CHECK(cudaMalloc(reinterpret_cast<void**>(&tr), n_cta * 8 * 8));
    RS_CUDA_CHECK(cudaMemsetAsync(tr, 0, n_cta * 8 * 8, st));
  }
  launch_kernel(decode_attn_kernel<HD>, grid, dim3(kDecThreads), DecCfg<HD>::kSmem, st, 1, qkv, ld_q, work, kv.k,
                kv.v, kv.page_tables, q_heads, kv_heads, tiles_per_split, scale_log2, part_o, part_ml, splits, out,
                ld_out, tr);
  if (splits > 1)
    launch_kernel(decode_attn_merge_kernel<HD>, dim3(q_heads, grid.z), dim3(32), 0, st, 1,
                  static_cast<const float*>(part_o), static_cast<const float*>(part_ml), q_heads, splits, out, ld_out,
                  work);
  if (trace) {  // ns from the earliest CTA start: mean / max over CTAs per phase
    std::vector<unsigned long long> h(n_cta * 8);
    RS_CUDA_CHECK(cudaStreamSynchronize(st));
    RS_CUDA_CHECK(cudaMemcpy(h.data(), tr, h.size() * 8, cudaMemcpyDeviceToHost));
    RS_CUDA_CHECK(cudaFree(tr));
    unsigned long long t0 = ~0ull;
    for (std::size_t i = 0; i < n_cta; ++i) t0 = std::min(t0, h[i * 8]);
    std::fprintf(stderr, "[dec-trace] ctas %zu splits %u:", n_cta, grid.x);
    for (int k = 0; k < 7; ++k) {
      double sum = 0, mx = 0;
      int n = 0;
      for (std::size_t i = 0; i < n_cta; ++i)
        if (h[i * 8 + k] != 0) {
          const double v = static_cast<double>(h[i * 8 + k] - t0);
          sum += v;
          mx = std::max(mx, v);
          ++n;
        }
      std::fprintf(stderr, " p%d %.0f/%.0f(n%d)", k, n ? sum / n : 0.0, mx, n);
    }
    std::fprintf(stderr, "\n");
  }
}

}  // namespace

void attention_decode_paged(const bf16* qkv, int ld_q, bf16* out, int ld_out, const PrefillWork* work,
                            int n_req, int max_keys, const PagedKV& kv, int q_heads, int kv_heads,
                            int head_dim, float scale, cudaStream_t st) {
  if (n_req <= 0) return;
  const int G = q_heads / kv_heads;
  if (G > kDecMaxG || q_heads % kv_heads != 0)
    throw DeviceError(RS_ERR_CUDA, "decode attention: GQA group above 16");
  if (kv.page_size != kDecTile) throw DeviceError(RS_ERR_CUDA, "decode attention needs 64-token pages");
  if (head_dim != 64 && head_dim != 128)
    throw DeviceError(RS_ERR_CUDA, "decode attention: unsupported head_dim " + std::to_string(head_dim));
  const int max_tiles = (max_keys + kDecTile - 1) / kDecTile;
  // one CTA per SM (4 pages in flight each): splits so that all (request,
  // kv head) pairs together fill the SMs
  const int pairs = n_req * kv_heads;
  int splits = std::max(1, (kNumSMs + pairs - 1) / pairs);
  splits = std::min(splits, max_tiles);
  const int tiles_per_split = (max_tiles + splits - 1) / splits;
  splits = (max_tiles + tiles_per_split - 1) / tiles_per_split;
  std::lock_guard<std::mutex> g(decode_ws_mutex());
  DecodeWs& ws = decode_ws_all()[st];
  const std::size_t need = static_cast<std::size_t>(n_req) * q_heads * splits * (head_dim + 2);
  if (ws.floats < need) {
    if (ws.buf != nullptr) RS_CUDA_CHECK(cudaFreeAsync(ws.buf, st));
    RS_CUDA_CHECK(cudaMallocAsync(reinterpret_cast<void**>(&ws.buf), need * sizeof(float), st));
    ws.floats = need;
  }
  float* part_o = ws.buf;
  float* part_ml = ws.buf + static_cast<std::size_t>(n_req) * q_heads * splits * head_dim;
  const float scale_log2 = scale * kLog2e;
  const int tok = prof::begin(st);
  const dim3 grid(splits, kv_heads, n_req);
  if (head_dim == 64)
    launch_decode<64>(grid, st, qkv, ld_q, work, kv, q_heads, kv_heads, tiles_per_split, scale_log2, part_o,
                      part_ml, splits, out, ld_out);
  else
    launch_decode<128>(grid, st, qkv, ld_q, work, kv, q_heads, kv_heads, tiles_per_split, scale_log2, part_o,
                       part_ml, splits, out, ld_out);
  RS_LAUNCH_CHECK();
  // algorithmic bytes: every valid key's K and V row of every kv head, once
  prof::end(tok, st, "attn_decode", 0, 0);
  count_launch(splits > 1 ? 2 : 1);
}

void attention_release_stream(cudaStream_t st) {
  attention_tc_release_stream(st);
  std::lock_guard<std::mutex> g(decode_ws_mutex());
  auto it = decode_ws_all().find(st);
  if (it == decode_ws_all().end()) return;
  if (it->second.buf) cudaFreeAsync(it->second.buf, st);
  decode_ws_all().erase(it);
}

}  // namespace rserve
