// rserve-b200 — flash attention kernels (see attention.cuh).
//
// CTA = 4 warps x 16 query rows = 64 queries of one head; K/V tiles of 64
// keys double-buffered in shared memory via cp.async; S = QK^T and O += PV
// on bf16 m16n8k16 tensor-core MMAs with fp32 accumulation; online softmax
// in base-2 with fp32 running max / sum.
#include <cuda_runtime.h>

#include <cmath>

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
template <int HD>
struct Smem {
  static constexpr int kLd = HD + 8;  // +16 B pad: conflict-free ldmatrix
  bf16 q[kQ][kLd];
  bf16 k[2][kKV][kLd];
  bf16 v[2][kKV][kLd];
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
template <int HD, typename Src>
__device__ void flash_block(const bf16* q_ptr, int ld_q, int q_rows, int q_pos0, const Src& src,
                            bf16* o_ptr, int ld_o, float scale_log2, Smem<HD>& sm,
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
    const int buf = t & 1;
    if (t + 1 < n_tiles) load_kv(t + 1, buf ^ 1);
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

template <int HD>
__global__ void __launch_bounds__(128) varlen_bidir_kernel(const bf16* __restrict__ qkv, int ld,
                                                           bf16* __restrict__ out, int ld_out,
                                                           const int* __restrict__ cu, int heads,
                                                           float scale_log2, const float2* rope) {
  extern __shared__ __align__(16) std::uint8_t smem_raw[];
  Smem<HD>& sm = *reinterpret_cast<Smem<HD>*>(smem_raw);
  pdl_wait();
  pdl_launch_dependents();
  const int seq = blockIdx.y, head = blockIdx.z;
  const int s0 = cu[seq], s1 = cu[seq + 1];
  const int q0 = blockIdx.x * kQ;
  const int len = s1 - s0;
  if (q0 >= len) return;
  BidirSource src{qkv + static_cast<std::int64_t>(s0) * ld + (heads + head) * HD,
                  qkv + static_cast<std::int64_t>(s0) * ld + (2 * heads + head) * HD, ld, len};
  flash_block<HD>(qkv + static_cast<std::int64_t>(s0 + q0) * ld + head * HD, ld, min(kQ, len - q0),
                  -1, src, out + static_cast<std::int64_t>(s0 + q0) * ld_out + head * HD, ld_out,
                  scale_log2, sm,
                  rope != nullptr ? rope + static_cast<std::int64_t>(s0 + q0) * (HD / 2) : nullptr,
                  rope != nullptr ? rope + static_cast<std::int64_t>(s0) * (HD / 2) : nullptr);
}

constexpr float kLog2e = 1.4426950408889634f;

template <int HD>
void launch_bidir(const bf16* qkv, int ld, bf16* out, int ld_out, const int* cu, int n_seqs,
                  int max_seqlen, int heads, float scale, cudaStream_t st, const float2* rope) {
  const int smem = sizeof(Smem<HD>);
  static bool set = false;
  if (!set) {
    RS_CUDA_CHECK(cudaFuncSetAttribute(varlen_bidir_kernel<HD>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    set = true;
  }
  dim3 grid(ceil_div(max_seqlen, kQ), n_seqs, heads);
  const int tok = prof::begin(st);
  launch_kernel(varlen_bidir_kernel<HD>, grid, dim3(128), smem, st, 1, qkv, ld, out, ld_out, cu, heads,
                scale * kLog2e, rope);
  RS_LAUNCH_CHECK();
  prof::end(tok, st, "attn_vit_mma", 0, 0);
  count_launch();
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

}  // namespace rserve
