// rserve-b200 — flash attention kernels (see attention.cuh).
//
// CTA = 4 warps x 16 query rows = 64 queries of one head; K/V tiles of 64
// keys double-buffered in shared memory via cp.async; S = QK^T and O += PV
// on bf16 m16n8k16 tensor-core MMAs with fp32 accumulation; online softmax
// in base-2 with fp32 running max / sum.
#include <cuda_runtime.h>

#include <algorithm>
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
// One query row per request (the token being decoded) against its paged KV:
// memory-bound (each K / V byte is read once per kv head), so CUDA-core math,
// GQA-packed (the G = Hq / Hkv query heads of a kv head share every K / V tile
// in shared memory) and split along the keys (flash-decoding) so a single
// request still spreads over the SMs; a second kernel merges the splits in
// split order (deterministic).
namespace {

constexpr int kDecThreads = 128;
constexpr int kDecMaxG = 8;
constexpr int kDecTile = 64;  // keys per tile = one KV page

template <int HD>
struct DecSmem {
  float q[kDecMaxG][HD];
  bf16 k[kDecTile][HD + 8];      // +16 B row pad: conflict-free column reads
  bf16 vt[HD][kDecTile + 8];     // V^T tile [hd][keys]
  float p[kDecMaxG][kDecTile];   // scores -> probabilities
  float alpha[kDecMaxG];
};

template <int HD>
__global__ void __launch_bounds__(kDecThreads) decode_attn_split_kernel(
    const bf16* __restrict__ qkv, int ld_q, const PrefillWork* __restrict__ work,
    const bf16* __restrict__ k_cache, const bf16* __restrict__ v_cache, const int* const* page_tables,
    int q_heads, int kv_heads, int tiles_per_split, float scale_log2, float* part_o, float* part_ml,
    int splits) {
  __shared__ DecSmem<HD> sm;
  pdl_wait();
  pdl_launch_dependents();
  const int split = blockIdx.x, kvh = blockIdx.y, req = blockIdx.z;
  const int G = q_heads / kv_heads;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const PrefillWork w = work[req];
  const int n_keys = w.q_pos0 + 1;  // keys [0, pos] (this token's K/V already appended)
  const int n_tiles = (n_keys + kDecTile - 1) / kDecTile;
  const int t0 = split * tiles_per_split, t1 = min(n_tiles, t0 + tiles_per_split);
  const int* pt = page_tables[w.req_slot];
  // q rows of the G heads (fp32, pre-scaled into the exp2 domain)
  const bf16* qrow = qkv + static_cast<std::int64_t>(w.q_row0) * ld_q + kvh * G * HD;
  for (int i = tid; i < G * HD; i += kDecThreads) sm.q[i / HD][i % HD] = bf2f(qrow[i]) * scale_log2;
  float m_run = -INFINITY, l_run = 0.f;  // per (g = warp*2 + {0,1}) on lane 0.. (see below)
  float acc[kDecMaxG];
#pragma unroll
  for (int g = 0; g < kDecMaxG; ++g) acc[g] = 0.f;
  // running max / sum of row g live in warp (g / 2), replicated over its lanes
  float mrow[2] = {-INFINITY, -INFINITY}, lrow[2] = {0.f, 0.f};
  (void)m_run;
  (void)l_run;
  for (int t = t0; t < t1; ++t) {
    const std::int64_t page = pt[t];
    const bf16* kp = k_cache + (page * kv_heads + kvh) * kDecTile * HD;
    const bf16* vp = v_cache + (page * kv_heads + kvh) * HD * kDecTile;
    // every 16-byte load of the K and V^T pages in flight before the first
    // shared-memory store (the kernel is bound by the loads' latency)
    constexpr int kVec = kDecTile * HD / 8 / kDecThreads;  // uint4 per thread per page
    uint4 kr[kVec], vr[kVec];
#pragma unroll
    for (int j = 0; j < kVec; ++j) {
      const int i = tid + j * kDecThreads;
      kr[j] = __ldcs(reinterpret_cast<const uint4*>(kp) + i);
      vr[j] = __ldcs(reinterpret_cast<const uint4*>(vp) + i);
    }
    __syncthreads();  // previous tile's k / vt / p consumed
#pragma unroll
    for (int j = 0; j < kVec; ++j) {
      const int i = tid + j * kDecThreads;
      *reinterpret_cast<uint4*>(&sm.k[i / (HD / 8)][(i % (HD / 8)) * 8]) = kr[j];
      *reinterpret_cast<uint4*>(&sm.vt[i / (kDecTile / 8)][(i % (kDecTile / 8)) * 8]) = vr[j];
    }
    __syncthreads();
    // S[g][key]: thread -> key (tid % 64), heads g = tid / 64 + 2j
    {
      const int key = tid & (kDecTile - 1);
      const int g0 = tid >> 6;
      float s[kDecMaxG / 2];
#pragma unroll
      for (int j = 0; j < kDecMaxG / 2; ++j) s[j] = 0.f;
#pragma unroll 8
      for (int d = 0; d < HD; d += 2) {
        const float2 kk = unpack_bf16x2(*reinterpret_cast<const std::uint32_t*>(&sm.k[key][d]));
#pragma unroll
        for (int j = 0; j < kDecMaxG / 2; ++j) {
          const int g = g0 + 2 * j;
          if (g < G) s[j] = fmaf(sm.q[g][d], kk.x, fmaf(sm.q[g][d + 1], kk.y, s[j]));
        }
      }
      const bool ok = t * kDecTile + key < n_keys;
#pragma unroll
      for (int j = 0; j < kDecMaxG / 2; ++j) {
        const int g = g0 + 2 * j;
        if (g < G) sm.p[g][key] = ok ? s[j] : -INFINITY;
      }
    }
    __syncthreads();
    // online softmax: warp w owns rows 2w, 2w+1 (G <= 8), 2 keys per lane
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int g = 2 * warp + h;
      if (g >= G) continue;
      const float a = sm.p[g][lane], b = sm.p[g][lane + 32];
      float mx = fmaxf(a, b);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      const float m_new = fmaxf(mrow[h], mx);
      const float alpha = m_new == -INFINITY ? 1.f : exp2f(mrow[h] - m_new);
      const float pa = m_new == -INFINITY ? 0.f : exp2f(a - m_new);
      const float pb = m_new == -INFINITY ? 0.f : exp2f(b - m_new);
      float rs = pa + pb;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) rs += __shfl_xor_sync(0xffffffffu, rs, o);
      lrow[h] = lrow[h] * alpha + rs;
      mrow[h] = m_new;
      sm.p[g][lane] = pa;
      sm.p[g][lane + 32] = pb;
      if (lane == 0) sm.alpha[g] = alpha;
    }
    __syncthreads();
    // O[g][d] += sum_k P[g][k] V[k][d]: thread -> d
    for (int d = tid; d < HD; d += kDecThreads) {
      float part[kDecMaxG];
#pragma unroll
      for (int g = 0; g < kDecMaxG; ++g) part[g] = 0.f;
#pragma unroll 4
      for (int k = 0; k < kDecTile; k += 2) {
        const float2 vv = unpack_bf16x2(*reinterpret_cast<const std::uint32_t*>(&sm.vt[d][k]));
#pragma unroll
        for (int g = 0; g < kDecMaxG; ++g)
          if (g < G) part[g] = fmaf(sm.p[g][k], vv.x, fmaf(sm.p[g][k + 1], vv.y, part[g]));
      }
#pragma unroll
      for (int g = 0; g < kDecMaxG; ++g)
        if (g < G) acc[g] = acc[g] * sm.alpha[g] + part[g];
    }
  }
  // partials: o [req][head][split][HD] (unnormalised), ml [req][head][split][2]
  for (int d = tid; d < HD; d += kDecThreads)
    for (int g = 0; g < G; ++g) {
      const int head = kvh * G + g;
      part_o[((static_cast<std::int64_t>(req) * q_heads + head) * splits + split) * HD + d] = acc[g];
    }
  if (lane == 0) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int g = 2 * warp + h;
      if (g >= G) continue;
      float* ml = part_ml + ((static_cast<std::int64_t>(req) * q_heads + kvh * G + g) * splits + split) * 2;
      ml[0] = mrow[h];
      ml[1] = lrow[h];
    }
  }
}

template <int HD>
__global__ void __launch_bounds__(HD) decode_attn_merge_kernel(const float* part_o, const float* part_ml,
                                                               int q_heads, int splits, bf16* out,
                                                               int ld_out, const PrefillWork* work) {
  pdl_wait();
  pdl_launch_dependents();
  const int head = blockIdx.x, req = blockIdx.y, d = threadIdx.x;
  const std::int64_t base = (static_cast<std::int64_t>(req) * q_heads + head) * splits;
  float M = -INFINITY;
  for (int s = 0; s < splits; ++s) M = fmaxf(M, part_ml[(base + s) * 2]);
  float o = 0.f, l = 0.f;
  for (int s = 0; s < splits; ++s) {
    const float m = part_ml[(base + s) * 2];
    if (m == -INFINITY) continue;
    const float w = exp2f(m - M);
    o += w * part_o[(base + s) * HD + d];
    l += w * part_ml[(base + s) * 2 + 1];
  }
  out[static_cast<std::int64_t>(work[req].q_row0) * ld_out + head * HD + d] = f2bf(l > 0.f ? o / l : 0.f);
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

}  // namespace

void attention_decode_paged(const bf16* qkv, int ld_q, bf16* out, int ld_out, const PrefillWork* work,
                            int n_req, int max_keys, const PagedKV& kv, int q_heads, int kv_heads,
                            int head_dim, float scale, cudaStream_t st) {
  if (n_req <= 0) return;
  const int G = q_heads / kv_heads;
  if (G > kDecMaxG || q_heads % kv_heads != 0)
    throw DeviceError(RS_ERR_CUDA, "decode attention: GQA group above 8");
  if (kv.page_size != kDecTile) throw DeviceError(RS_ERR_CUDA, "decode attention needs 64-token pages");
  const int max_tiles = (max_keys + kDecTile - 1) / kDecTile;
  // splits: ~2 CTAs per SM over all requests and kv heads
  const int ctas_wanted = 2 * kNumSMs;
  int splits = std::max(1, ctas_wanted / std::max(1, n_req * kv_heads));
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
  switch (head_dim) {
    case 64:
      launch_kernel(decode_attn_split_kernel<64>, grid, dim3(kDecThreads), 0, st, 1, qkv, ld_q, work, kv.k, kv.v,
                    kv.page_tables, q_heads, kv_heads, tiles_per_split, scale_log2, part_o, part_ml, splits);
      launch_kernel(decode_attn_merge_kernel<64>, dim3(q_heads, n_req), dim3(64), 0, st, 1,
                    static_cast<const float*>(part_o), static_cast<const float*>(part_ml), q_heads, splits, out,
                    ld_out, work);
      break;
    case 128:
      launch_kernel(decode_attn_split_kernel<128>, grid, dim3(kDecThreads), 0, st, 1, qkv, ld_q, work, kv.k, kv.v,
                    kv.page_tables, q_heads, kv_heads, tiles_per_split, scale_log2, part_o, part_ml, splits);
      launch_kernel(decode_attn_merge_kernel<128>, dim3(q_heads, n_req), dim3(128), 0, st, 1,
                    static_cast<const float*>(part_o), static_cast<const float*>(part_ml), q_heads, splits, out,
                    ld_out, work);
      break;
    default:
      throw DeviceError(RS_ERR_CUDA, "decode attention: unsupported head_dim " + std::to_string(head_dim));
  }
  RS_LAUNCH_CHECK();
  prof::end(tok, st, "attn_decode", 0, 0);
  count_launch(2);
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
