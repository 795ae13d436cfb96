// rserve-b200 — HBM-bound kernels (see kernels.cuh). All row kernels use one
// warp per row with 16-byte vector accesses; grids are sized to whole waves
// of the 148 SMs and loop over rows.
#include <cuda_runtime.h>

#include <cmath>

#include "common.cuh"
#include "gemm.cuh"
#include "kernels.cuh"

namespace rserve {
namespace {

constexpr int kWarpsPerBlock = 8;

int row_grid(std::int64_t rows) {
  const std::int64_t blocks = ceil_div64(rows, kWarpsPerBlock);
  const std::int64_t cap = static_cast<std::int64_t>(kNumSMs) * 16;
  return static_cast<int>(blocks < cap ? (blocks > 0 ? blocks : 1) : cap);
}

__global__ void fill_uniform_kernel(bf16* dst, std::int64_t rows, int cols, int ld,
                                    std::uint64_t seed, std::uint64_t stream, float scale,
                                    float offset, std::int64_t row0, int col0, int cols_full) {
  const std::int64_t total = rows * ld;
  for (std::int64_t e = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
    const std::int64_t r = e / ld;
    const int c = static_cast<int>(e % ld);
    float v = 0.f;
    if (c < cols) {
      const std::uint64_t z =
          mix64(seed, stream, static_cast<std::uint64_t>(row0 + r) * cols_full + (col0 + c));
      const float u = static_cast<float>(z >> 40) * (1.0f / 16777216.0f);
      v = (2.0f * u - 1.0f) * scale + offset;
    }
    dst[e] = __float2bfloat16_rn(v);
  }
}

__global__ void fill_interleaved_kernel(bf16* dst, int rows_valid, int rows_pad, int cols, int ld,
                                        std::uint64_t seed, std::uint64_t stream, float scale,
                                        int which, int row0) {
  const std::int64_t total = static_cast<std::int64_t>(rows_pad) * ld;
  for (std::int64_t e = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(e / ld);
    const int c = static_cast<int>(e % ld);
    float v = 0.f;
    if (r < rows_valid && c < cols) {
      const std::uint64_t z = mix64(seed, stream, static_cast<std::uint64_t>(row0 + r) * cols + c);
      const float u = static_cast<float>(z >> 40) * (1.0f / 16777216.0f);
      v = (2.0f * u - 1.0f) * scale;
    }
    const std::int64_t dst_row = static_cast<std::int64_t>(r / 16) * 32 + which * 16 + r % 16;
    dst[dst_row * ld + c] = __float2bfloat16_rn(v);
  }
}

__global__ void fill_const_kernel(bf16* dst, std::int64_t n, float v) {
  for (std::int64_t e = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<std::int64_t>(gridDim.x) * blockDim.x)
    dst[e] = __float2bfloat16_rn(v);
}

__global__ void fold_norm_weight_kernel(bf16* W, std::int64_t rows, int cols, int ld, const bf16* g) {
  const std::int64_t n = rows * cols;
  for (std::int64_t e = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
    const std::int64_t r = e / cols;
    const int c = static_cast<int>(e - r * cols);
    bf16& w = W[r * ld + c];
    w = __float2bfloat16_rn(__bfloat162float(w) * __bfloat162float(g[c]));
  }
}

__global__ void fill_ids_kernel(std::int32_t* dst, std::int64_t n, std::uint64_t seed,
                                std::uint64_t stream, std::uint32_t modulo) {
  for (std::int64_t e = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<std::int64_t>(gridDim.x) * blockDim.x)
    dst[e] = static_cast<std::int32_t>(mix64(seed, stream, static_cast<std::uint64_t>(e)) % modulo);
}

// Single-pass RMSNorm: the row stays in registers (VPL 16-byte vectors per
// lane, dim = 256 * VPL), so HBM sees one read and one write per element.
template <int VPL>
__global__ void rmsnorm_reg_kernel(const bf16* __restrict__ x, int ldx, const bf16* __restrict__ w,
                                   bf16* __restrict__ y, int ldy, int rows, float eps,
                                   const std::int64_t* __restrict__ row_map,
                                   bf16* __restrict__ x_copy, int ld_copy) {
  constexpr int kDim = VPL * 256;
  const int lane = threadIdx.x & 31;
  for (int m = blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5); m < rows;
       m += gridDim.x * kWarpsPerBlock) {
    const std::int64_t src = row_map != nullptr ? row_map[m] : m;
    const bf16* xr = x + src * ldx;
    uint4 v[VPL];
#pragma unroll
    for (int k = 0; k < VPL; ++k) v[k] = *reinterpret_cast<const uint4*>(xr + lane * 8 + k * 256);
    float ss = 0.f;
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
      const std::uint32_t vw[4] = {v[k].x, v[k].y, v[k].z, v[k].w};
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const float2 f = unpack_bf16x2(vw[t]);
        ss += f.x * f.x + f.y * f.y;
      }
    }
    if (x_copy != nullptr) {
#pragma unroll
      for (int k = 0; k < VPL; ++k)
        *reinterpret_cast<uint4*>(x_copy + static_cast<std::int64_t>(m) * ld_copy + lane * 8 + k * 256) = v[k];
    }
    ss = warp_sum(ss);
    const float inv = rsqrtf(ss / static_cast<float>(kDim) + eps);
    bf16* yr = y + static_cast<std::int64_t>(m) * ldy;
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
      const uint4 g = *reinterpret_cast<const uint4*>(w + lane * 8 + k * 256);
      const std::uint32_t vw[4] = {v[k].x, v[k].y, v[k].z, v[k].w};
      const std::uint32_t gw[4] = {g.x, g.y, g.z, g.w};
      std::uint32_t o[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const float2 f = unpack_bf16x2(vw[t]);
        const float2 gg = unpack_bf16x2(gw[t]);
        o[t] = pack_bf16x2(bf2f(f2bf(f.x * inv)) * gg.x, bf2f(f2bf(f.y * inv)) * gg.y);
      }
      *reinterpret_cast<uint4*>(yr + lane * 8 + k * 256) = make_uint4(o[0], o[1], o[2], o[3]);
    }
  }
}

__global__ void rmsnorm_kernel(const bf16* __restrict__ x, int ldx, const bf16* __restrict__ w,
                               bf16* __restrict__ y, int ldy, int rows, int dim, float eps,
                               const std::int64_t* __restrict__ row_map, bf16* __restrict__ x_copy,
                               int ld_copy, const int* rows_dev) {
  const int lane = threadIdx.x & 31;
  const int n = rows_dev != nullptr ? min(*rows_dev, rows) : rows;
  for (int m = blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5); m < n;
       m += gridDim.x * kWarpsPerBlock) {
    const std::int64_t src = row_map != nullptr ? row_map[m] : m;
    const bf16* xr = x + src * ldx;
    float ss = 0.f;
    for (int c = lane * 8; c < dim; c += 256) {
      const uint4 v = *reinterpret_cast<const uint4*>(xr + c);
      const std::uint32_t vw[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const float2 f = unpack_bf16x2(vw[t]);
        ss += f.x * f.x + f.y * f.y;
      }
      if (x_copy != nullptr)
        *reinterpret_cast<uint4*>(x_copy + static_cast<std::int64_t>(m) * ld_copy + c) = v;
    }
    ss = warp_sum(ss);
    const float inv = rsqrtf(ss / static_cast<float>(dim) + eps);
    bf16* yr = y + static_cast<std::int64_t>(m) * ldy;
    for (int c = lane * 8; c < dim; c += 256) {
      const uint4 v = *reinterpret_cast<const uint4*>(xr + c);
      const uint4 g = *reinterpret_cast<const uint4*>(w + c);
      const std::uint32_t vw[4] = {v.x, v.y, v.z, v.w};
      const std::uint32_t gw[4] = {g.x, g.y, g.z, g.w};
      std::uint32_t o[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const float2 f = unpack_bf16x2(vw[t]);
        const float2 gg = unpack_bf16x2(gw[t]);
        // Qwen2 RMSNorm: normalise in fp32, cast to bf16, then scale.
        const float a = bf2f(f2bf(f.x * inv)) * gg.x;
        const float b = bf2f(f2bf(f.y * inv)) * gg.y;
        o[t] = pack_bf16x2(a, b);
      }
      *reinterpret_cast<uint4*>(yr + c) = make_uint4(o[0], o[1], o[2], o[3]);
    }
  }
}

// One warp per (row, head) pair of rotations for q and k.
__global__ void rope_vit_kernel(bf16* qkv, int ld, const std::int32_t* __restrict__ pos_hw,
                                int rows, int heads, int hd, float log2_theta) {
  const int lane = threadIdx.x & 31;
  const int half = hd / 2, quarter = hd / 4;
  const std::int64_t items = static_cast<std::int64_t>(rows) * heads * 2;
  for (std::int64_t it = blockIdx.x * static_cast<std::int64_t>(kWarpsPerBlock) + (threadIdx.x >> 5);
       it < items; it += static_cast<std::int64_t>(gridDim.x) * kWarpsPerBlock) {
    const int which = static_cast<int>(it % 2);  // 0 = q, 1 = k
    const int head = static_cast<int>((it / 2) % heads);
    const std::int64_t row = it / (2 * heads);
    bf16* v = qkv + row * ld + (which * heads + head) * hd;
    const float ph = static_cast<float>(pos_hw[2 * row]);
    const float pw = static_cast<float>(pos_hw[2 * row + 1]);
    for (int i = lane; i < half; i += 32) {
      const int j = i < quarter ? i : i - quarter;
      const float freq = exp2f(-log2_theta * (4.0f * j) / static_cast<float>(hd));
      const float ang = (i < quarter ? ph : pw) * freq;
      float s, c;
      sincosf(ang, &s, &c);
      const float a = bf2f(v[i]), b = bf2f(v[i + half]);
      v[i] = f2bf(a * c - b * s);
      v[i + half] = f2bf(b * c + a * s);
    }
  }
}

// cos / sin of the ViT 2D RoPE per (token, pair), shared by all layers.
__global__ void vit_rope_table_kernel(const std::int32_t* __restrict__ pos_hw, int rows, int hd,
                                      float log2_theta, float2* __restrict__ table) {
  const int half = hd / 2, quarter = hd / 4;
  const std::int64_t n = static_cast<std::int64_t>(rows) * half;
  for (std::int64_t e = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
    const int t = static_cast<int>(e / half), i = static_cast<int>(e % half);
    const int j = i < quarter ? i : i - quarter;
    const float freq = exp2f(-log2_theta * (4.0f * j) / static_cast<float>(hd));
    float s, c;
    sincosf(static_cast<float>(pos_hw[2 * t + (i < quarter ? 0 : 1)]) * freq, &s, &c);
    table[e] = make_float2(c, s);
  }
}

__global__ void vit_rope_freq_kernel(int n_pos, int hd, float log2_theta, float2* __restrict__ out) {
  const int quarter = hd / 4;
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n_pos * quarter) return;
  const int pos = e / quarter, j = e % quarter;
  // the same expression as vit_rope_table_kernel: bit-identical entries
  const float freq = exp2f(-log2_theta * (4.0f * j) / static_cast<float>(hd));
  float s, c;
  sincosf(static_cast<float>(pos) * freq, &s, &c);
  out[e] = make_float2(c, s);
}

// q / k RoPE: one thread per (token, q|k, head, 8 pairs); 16-byte loads of
// x[i..i+7] and x[i+half..], 16-byte stores. Destination row stride `ldp`,
// head stride `hs`: head-padded qp / kp (ldp = heads*128, hs = 128) or in
// place (qp = qkv, kp = qkv + heads*hd, ldp = ld, hs = hd; each thread
// rewrites exactly the elements it read).
__global__ void vit_qk_rope_pad_kernel(const bf16* qkv, int ld, const float2* __restrict__ table,
                                       int rows, int heads, int hd, bf16* qp, bf16* kp, int ldp,
                                       int hs) {
  pdl_wait();
  pdl_launch_dependents();
  const int half = hd / 2, chunks = half / 8;
  const std::int64_t n = static_cast<std::int64_t>(rows) * 2 * heads * chunks;
  for (std::int64_t e = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
    const int ch = static_cast<int>(e % chunks);
    const int h = static_cast<int>((e / chunks) % heads);
    const int which = static_cast<int>((e / (chunks * heads)) % 2);
    const int t = static_cast<int>(e / (2 * chunks * heads));
    const int i0 = ch * 8;
    const bf16* src = qkv + static_cast<std::int64_t>(t) * ld + (which * heads + h) * hd;
    const uint4 a = *reinterpret_cast<const uint4*>(src + i0);
    const uint4 b = *reinterpret_cast<const uint4*>(src + i0 + half);
    const float2* cs = table + static_cast<std::int64_t>(t) * half + i0;
    const std::uint32_t aw[4] = {a.x, a.y, a.z, a.w}, bw[4] = {b.x, b.y, b.z, b.w};
    std::uint32_t lo[4], hi[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float2 fa = unpack_bf16x2(aw[k]), fb = unpack_bf16x2(bw[k]);
      const float2 c0 = cs[2 * k], c1 = cs[2 * k + 1];
      lo[k] = pack_bf16x2(fa.x * c0.x - fb.x * c0.y, fa.y * c1.x - fb.y * c1.y);
      hi[k] = pack_bf16x2(fb.x * c0.x + fa.x * c0.y, fb.y * c1.x + fa.y * c1.y);
    }
    bf16* dst = (which == 0 ? qp : kp) + static_cast<std::int64_t>(t) * ldp + h * hs;
    *reinterpret_cast<uint4*>(dst + i0) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
    *reinterpret_cast<uint4*>(dst + i0 + half) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
  }
}

// V [64 tokens, hd] of one head -> vt[head*128 + d][t0 .. t0+64) via smem.
__global__ void vit_v_transpose_kernel(const bf16* __restrict__ qkv, int ld, int rows, int heads,
                                       int hd, bf16* __restrict__ vt, int ld_vt) {
  __shared__ bf16 tile[128][64 + 8];
  pdl_wait();
  pdl_launch_dependents();
  const int t0 = blockIdx.x * 64, h = blockIdx.y;
  const int vec = hd / 8;
  for (int e = threadIdx.x; e < 64 * vec; e += blockDim.x) {
    const int tt = e / vec, c = (e % vec) * 8;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (t0 + tt < rows)
      v = *reinterpret_cast<const uint4*>(qkv + static_cast<std::int64_t>(t0 + tt) * ld +
                                          (2 * heads + h) * hd + c);
    const bf16* pv = reinterpret_cast<const bf16*>(&v);
#pragma unroll
    for (int k = 0; k < 8; ++k) tile[c + k][tt] = pv[k];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < hd * 8; e += blockDim.x) {
    const int d = e / 8, c = (e % 8) * 8;
    if (t0 + c + 8 <= rows)
      *reinterpret_cast<uint4*>(vt + static_cast<std::int64_t>(h * 128 + d) * ld_vt + t0 + c) =
          *reinterpret_cast<const uint4*>(&tile[d][c]);
    else
      for (int k = 0; k < 8 && t0 + c + k < rows; ++k)
        vt[static_cast<std::int64_t>(h * 128 + d) * ld_vt + t0 + c + k] = tile[d][c + k];
  }
}

__global__ void rope_kv_append_kernel(bf16* qkv, int ld, const ChunkRowInfo* __restrict__ info,
                                      int rows, int q_heads, int kv_heads, int hd,
                                      float log2_theta, bf16* k_cache, bf16* v_cache,
                                      const int* const* page_tables, int page_size,
                                      const int* rows_dev) {
  const int lane = threadIdx.x & 31;
  const int half = hd / 2;
  const int s_t = hd / 8, s_h = hd / 8 + (3 * hd) / 16;
  const int n = rows_dev != nullptr ? min(*rows_dev, rows) : rows;
  const int heads_total = q_heads + 2 * kv_heads;
  const std::int64_t items = static_cast<std::int64_t>(n) * heads_total;
  for (std::int64_t it = blockIdx.x * static_cast<std::int64_t>(kWarpsPerBlock) + (threadIdx.x >> 5);
       it < items; it += static_cast<std::int64_t>(gridDim.x) * kWarpsPerBlock) {
    const int head = static_cast<int>(it % heads_total);
    const int row = static_cast<int>(it / heads_total);
    const ChunkRowInfo ri = info[row];
    bf16* v = qkv + static_cast<std::int64_t>(row) * ld + head * hd;
    const bool is_v = head >= q_heads + kv_heads;
    if (!is_v) {
      for (int i = lane; i < half; i += 32) {
        const int sec = i < s_t ? 0 : (i < s_h ? 1 : 2);
        const float freq = exp2f(-log2_theta * (2.0f * i) / static_cast<float>(hd));
        const float ang = static_cast<float>(ri.rope[sec]) * freq;
        float s, c;
        sincosf(ang, &s, &c);
        const float a = bf2f(v[i]), b = bf2f(v[i + half]);
        v[i] = f2bf(a * c - b * s);
        v[i + half] = f2bf(b * c + a * s);
      }
    }
    if (head >= q_heads) {
      __syncwarp();
      const int kvh = is_v ? head - q_heads - kv_heads : head - q_heads;
      const int* pt = page_tables[ri.req_slot];
      const std::int64_t page_head = static_cast<std::int64_t>(pt[ri.pos / page_size]) * kv_heads + kvh;
      const int off = ri.pos % page_size;
      if (!is_v) {  // K: [page][kv head][token][hd]
        bf16* dst = k_cache + (page_head * page_size + off) * hd;
        for (int c = lane * 8; c < hd; c += 256)
          *reinterpret_cast<uint4*>(dst + c) = *reinterpret_cast<const uint4*>(v + c);
      } else {      // V transposed: [page][kv head][hd][token]
        bf16* dst = v_cache + page_head * hd * page_size + off;
        for (int c = lane; c < hd; c += 32) dst[static_cast<std::int64_t>(c) * page_size] = v[c];
      }
    }
  }
}

// M-RoPE + paged KV append, vectorised (rope_kv_append_kernel is the
// reference-shaped scalar version kept for rows_dev / odd head sizes).
// blockIdx.y == 0: one warp per (chunk row, group of 32 / (HD/16) heads):
// cos / sin of 8 frequencies per lane, applied with 16-byte loads; k heads
// are also copied into the page. blockIdx.y == 1: one warp per (32 rows, kv
// head, 16 head dims), lane = row: V is written transposed, so for each head
// dim the 32 lanes store 32 consecutive tokens of a page.
template <int HD>
__global__ void rope_kv_append_vec_kernel(bf16* qkv, int ld, const ChunkRowInfo* __restrict__ info,
                                          int rows, int q_heads, int kv_heads, float log2_theta,
                                          bf16* k_cache, bf16* v_cache,
                                          const int* const* page_tables, int page_size,
                                          const float2* __restrict__ table) {
  constexpr int kHalf = HD / 2, kLph = kHalf / 8, kHpp = 32 / kLph;
  pdl_wait();
  pdl_launch_dependents();
  const int lane = threadIdx.x & 31;
  const int warps_total = gridDim.x * kWarpsPerBlock;
  const int wid = blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
  if (blockIdx.y == 0) {
    const int i0 = (lane % kLph) * 8;
    const int hsub = lane / kLph;
    constexpr int s_t = HD / 8, s_h = HD / 8 + (3 * HD) / 16;
    const int heads = q_heads + kv_heads;
    const int passes = (heads + kHpp - 1) / kHpp;
    for (int item = wid; item < rows * passes; item += warps_total) {
      const int row = item / passes;
      const int h = (item % passes) * kHpp + hsub;
      const ChunkRowInfo ri = info[row];
      float cs[8], sn[8];
      if (table != nullptr) {  // per-chunk cos / sin table (mrope_table): shared by every layer
        const float4* tp = reinterpret_cast<const float4*>(table + static_cast<std::int64_t>(row) * kHalf + i0);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float4 q = tp[j];
          cs[2 * j] = q.x;
          sn[2 * j] = q.y;
          cs[2 * j + 1] = q.z;
          sn[2 * j + 1] = q.w;
        }
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int i = i0 + j;
          const int sec = i < s_t ? 0 : (i < s_h ? 1 : 2);
          const float freq = exp2f(-log2_theta * (2.0f * i) / static_cast<float>(HD));
          sincosf(static_cast<float>(ri.rope[sec]) * freq, &sn[j], &cs[j]);
        }
      }
      const int* pt = page_tables[ri.req_slot];
      const std::int64_t page = pt[ri.pos / page_size];
      const int off = ri.pos % page_size;
      bf16* base = qkv + static_cast<std::int64_t>(row) * ld;
      if (h < heads) {
        bf16* v = base + h * HD;
        const uint4 a = *reinterpret_cast<const uint4*>(v + i0);
        const uint4 b = *reinterpret_cast<const uint4*>(v + i0 + kHalf);
        const std::uint32_t aw[4] = {a.x, a.y, a.z, a.w}, bw[4] = {b.x, b.y, b.z, b.w};
        std::uint32_t oa[4], ob[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const float2 fa = unpack_bf16x2(aw[t]), fb = unpack_bf16x2(bw[t]);
          const float c0 = cs[2 * t], s0 = sn[2 * t], c1 = cs[2 * t + 1], s1 = sn[2 * t + 1];
          oa[t] = pack_bf16x2(fa.x * c0 - fb.x * s0, fa.y * c1 - fb.y * s1);
          ob[t] = pack_bf16x2(fb.x * c0 + fa.x * s0, fb.y * c1 + fa.y * s1);
        }
        const uint4 ua = make_uint4(oa[0], oa[1], oa[2], oa[3]), ub = make_uint4(ob[0], ob[1], ob[2], ob[3]);
        *reinterpret_cast<uint4*>(v + i0) = ua;
        *reinterpret_cast<uint4*>(v + i0 + kHalf) = ub;
        if (h >= q_heads) {  // K: [page][kv head][token][hd]
          bf16* dst = k_cache + ((page * kv_heads + (h - q_heads)) * page_size + off) * HD;
          *reinterpret_cast<uint4*>(dst + i0) = ua;
          *reinterpret_cast<uint4*>(dst + i0 + kHalf) = ub;
        }
      }
    }
  } else {
    constexpr int kSlices = HD / 16;
    const int groups = ((rows + 31) / 32) * kv_heads * kSlices;
    for (int g = wid; g < groups; g += warps_total) {
      const int sl = g % kSlices;
      const int kvh = (g / kSlices) % kv_heads;
      const int r = (g / (kSlices * kv_heads)) * 32 + lane;
      if (r >= rows) continue;
      const ChunkRowInfo ri = info[r];
      const std::int64_t page = page_tables[ri.req_slot][ri.pos / page_size];
      const bf16* v = qkv + static_cast<std::int64_t>(r) * ld + (q_heads + kv_heads + kvh) * HD;
      bf16* dst = v_cache + (page * kv_heads + kvh) * HD * page_size + ri.pos % page_size;
#pragma unroll
      for (int c0 = sl * 16; c0 < sl * 16 + 16; c0 += 8) {
        const uint4 x = *reinterpret_cast<const uint4*>(v + c0);
        const bf16* e = reinterpret_cast<const bf16*>(&x);
#pragma unroll
        for (int t = 0; t < 8; ++t) dst[static_cast<std::int64_t>(c0 + t) * page_size] = e[t];
      }
    }
  }
}

__global__ void scatter_rows_kernel(const bf16* __restrict__ src, int n_rows,
                                    const std::int64_t* __restrict__ dst_rows, bf16* slab, int d,
                                    std::uint32_t* bitmap, const std::uint64_t* __restrict__ ranges,
                                    int n_ranges) {
  const int lane = threadIdx.x & 31;
  const int warp_global = blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
  const int warps = gridDim.x * kWarpsPerBlock;
  // Bitmap bits: one thread per 32-bit word per range (few words).
  if (blockIdx.x == 0) {
    for (int r = 0; r < n_ranges; ++r) {
      const std::uint64_t b = ranges[2 * r], e = ranges[2 * r + 1];
      for (std::uint64_t w = (b >> 5) + threadIdx.x; w <= ((e - 1) >> 5); w += blockDim.x) {
        const std::uint64_t lo = max(b, w << 5), hi = min(e, (w + 1) << 5);
        const unsigned span = static_cast<unsigned>(hi - lo);
        const std::uint32_t mask =
            span == 32 ? 0xFFFFFFFFu : (((1u << span) - 1u) << static_cast<unsigned>(lo & 31));
        atomicOr(bitmap + w, mask);
      }
    }
  }
  const int vec = d / 8;
  for (int r = warp_global; r < n_rows; r += warps) {
    const uint4* s = reinterpret_cast<const uint4*>(src + static_cast<std::int64_t>(r) * d);
    uint4* o = reinterpret_cast<uint4*>(slab + dst_rows[r] * d);
    for (int c = lane; c < vec; c += 32) o[c] = s[c];
  }
}

__global__ void ready_prefix_kernel(const std::uint32_t* __restrict__ bitmap, std::uint64_t frontier,
                                    std::uint64_t total, std::uint64_t* out) {
  const int lane = threadIdx.x;
  const std::uint64_t n_words = (total + 31) >> 5;
  std::uint64_t result = total;
  for (std::uint64_t w0 = frontier >> 5; w0 < n_words; w0 += 32) {
    const std::uint64_t w = w0 + lane;
    std::uint32_t word = w < n_words ? bitmap[w] : 0u;
    if (w == (frontier >> 5)) word |= (1u << (frontier & 31)) - 1u;  // bits below frontier
    const unsigned has_zero = __ballot_sync(0xffffffffu, w < n_words && word != 0xFFFFFFFFu);
    if (has_zero != 0) {
      const int first = __ffs(has_zero) - 1;
      const std::uint32_t fw = __shfl_sync(0xffffffffu, word, first);
      const std::uint64_t hit = ((w0 + first) << 5) + static_cast<std::uint64_t>(__ffs(~fw) - 1);
      result = hit < total ? hit : total;
      break;
    }
  }
  if (lane == 0) *out = result;
}

__global__ void gather_text_kernel(const bf16* __restrict__ vocab, const std::int32_t* __restrict__ ids,
                                   int n, const std::int64_t* __restrict__ dst_rows, bf16* slab,
                                   int d) {
  const int lane = threadIdx.x & 31;
  const int vec = d / 8;
  for (int r = blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5); r < n;
       r += gridDim.x * kWarpsPerBlock) {
    const uint4* s = reinterpret_cast<const uint4*>(vocab + static_cast<std::int64_t>(ids[r]) * d);
    uint4* o = reinterpret_cast<uint4*>(slab + dst_rows[r] * d);
    for (int c = lane; c < vec; c += 32) o[c] = s[c];
  }
}

__global__ void bitmap_set_kernel(std::uint32_t* bitmap, const std::uint64_t* ranges, int n_ranges) {
  for (int r = 0; r < n_ranges; ++r) {
    const std::uint64_t b = ranges[2 * r], e = ranges[2 * r + 1];
    if (e <= b) continue;
    for (std::uint64_t w = (b >> 5) + threadIdx.x + static_cast<std::uint64_t>(blockIdx.x) * blockDim.x;
         w <= ((e - 1) >> 5); w += static_cast<std::uint64_t>(gridDim.x) * blockDim.x) {
      const std::uint64_t lo = max(b, w << 5), hi = min(e, (w + 1) << 5);
      const unsigned span = static_cast<unsigned>(hi - lo);
      const std::uint32_t mask =
          span == 32 ? 0xFFFFFFFFu : (((1u << span) - 1u) << static_cast<unsigned>(lo & 31));
      atomicOr(bitmap + w, mask);
    }
  }
}

// One CTA of 1024 threads per row: 16-byte loads, four in flight per thread
// (the vocabulary row is 608 KB for 152064 logits: a 256-thread scalar loop
// was latency bound at ~2 GB/s, 283 us on the TTFT path). Ties -> lowest index.
__device__ __forceinline__ void argmax_take(float v, int i, float& best, int& idx) {
  if (v > best || (v == best && i < idx)) {
    best = v;
    idx = i;
  }
}

__global__ void __launch_bounds__(1024) argmax_kernel(const float* __restrict__ logits, int vocab,
                                                      std::int32_t* out, const std::int32_t* rows_idx) {
  const int rix = rows_idx != nullptr ? rows_idx[blockIdx.x] : static_cast<int>(blockIdx.x);
  const float* row = logits + static_cast<std::int64_t>(rix) * vocab;
  float best = -INFINITY;
  int idx = 0x7fffffff;
  const bool vec = (vocab & 3) == 0;
  const int n4 = vec ? vocab / 4 : 0;
  const float4* r4 = reinterpret_cast<const float4*>(row);
  constexpr int kU = 4;
  int i = threadIdx.x;
  for (; i + (kU - 1) * static_cast<int>(blockDim.x) < n4; i += kU * blockDim.x) {
    float4 v[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) v[u] = __ldcs(r4 + i + u * blockDim.x);
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int b = 4 * (i + u * static_cast<int>(blockDim.x));
      argmax_take(v[u].x, b, best, idx);
      argmax_take(v[u].y, b + 1, best, idx);
      argmax_take(v[u].z, b + 2, best, idx);
      argmax_take(v[u].w, b + 3, best, idx);
    }
  }
  for (; i < n4; i += blockDim.x) {
    const float4 v = __ldcs(r4 + i);
    argmax_take(v.x, 4 * i, best, idx);
    argmax_take(v.y, 4 * i + 1, best, idx);
    argmax_take(v.z, 4 * i + 2, best, idx);
    argmax_take(v.w, 4 * i + 3, best, idx);
  }
  for (int j = 4 * n4 + threadIdx.x; j < vocab; j += blockDim.x) argmax_take(row[j], j, best, idx);
  __shared__ float sb[32];
  __shared__ int si[32];
  for (int o = 16; o > 0; o >>= 1) {
    const float ob = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
    argmax_take(ob, oi, best, idx);
  }
  if ((threadIdx.x & 31) == 0) {
    sb[threadIdx.x >> 5] = best;
    si[threadIdx.x >> 5] = idx;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    const int nw = static_cast<int>(blockDim.x >> 5);
    best = threadIdx.x < nw ? sb[threadIdx.x] : -INFINITY;
    idx = threadIdx.x < nw ? si[threadIdx.x] : 0x7fffffff;
    for (int o = 16; o > 0; o >>= 1) {
      const float ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
      argmax_take(ob, oi, best, idx);
    }
    if (threadIdx.x == 0) out[rix] = idx;
  }
}

int elem_grid(std::int64_t n) {
  const std::int64_t b = ceil_div64(n, 256);
  const std::int64_t cap = static_cast<std::int64_t>(kNumSMs) * 32;
  return static_cast<int>(b < 1 ? 1 : (b < cap ? b : cap));
}

}  // namespace

void fill_uniform(bf16* dst, std::int64_t rows, int cols, int ld, std::uint64_t seed,
                  std::uint64_t stream, float scale, float offset, cudaStream_t st) {
  if (rows <= 0) return;
  fill_uniform_kernel<<<elem_grid(rows * ld), 256, 0, st>>>(dst, rows, cols, ld, seed, stream,
                                                           scale, offset, 0, 0, cols);
  RS_LAUNCH_CHECK();
  count_launch();
}

void fill_uniform_slice(bf16* dst, std::int64_t rows, int cols, int ld, std::uint64_t seed,
                        std::uint64_t stream, float scale, std::int64_t row0, int col0, int cols_full,
                        cudaStream_t st) {
  if (rows <= 0) return;
  fill_uniform_kernel<<<elem_grid(rows * ld), 256, 0, st>>>(dst, rows, cols, ld, seed, stream, scale, 0.f,
                                                           row0, col0, cols_full);
  RS_LAUNCH_CHECK();
  count_launch();
}

void fill_uniform_interleaved(bf16* dst, int rows_valid, int rows_pad, int cols, int ld,
                              std::uint64_t seed, std::uint64_t stream, float scale, int which,
                              cudaStream_t st, int row0) {
  fill_interleaved_kernel<<<elem_grid(static_cast<std::int64_t>(rows_pad) * ld), 256, 0, st>>>(
      dst, rows_valid, rows_pad, cols, ld, seed, stream, scale, which, row0);
  RS_LAUNCH_CHECK();
  count_launch();
}

__global__ void __launch_bounds__(256) copy_pages_kernel(const PageCopy* __restrict__ list, int n,
                                                         int vec_per_page) {
  pdl_wait();
  pdl_launch_dependents();
  for (int pg = blockIdx.x; pg < n; pg += gridDim.x) {
    const PageCopy c = list[pg];
    const uint4* src = static_cast<const uint4*>(c.src);
    uint4* dst = static_cast<uint4*>(c.dst);
    int i = threadIdx.x;
    for (; i + 3 * 256 < vec_per_page; i += 4 * 256) {  // 4 loads in flight per thread
      const uint4 a = __ldcs(src + i), b = __ldcs(src + i + 256), d = __ldcs(src + i + 512),
                  e = __ldcs(src + i + 768);
      __stcs(dst + i, a);
      __stcs(dst + i + 256, b);
      __stcs(dst + i + 512, d);
      __stcs(dst + i + 768, e);
    }
    for (; i < vec_per_page; i += 256) __stcs(dst + i, __ldcs(src + i));
  }
}

void copy_pages(const PageCopy* list_dev, int n, std::size_t page_bytes, cudaStream_t st, const char* label) {
  if (n <= 0) return;
  if (page_bytes % 16 != 0) throw DeviceError(RS_ERR_CUDA, "copy_pages: page bytes must be a multiple of 16");
  const int tok = prof::begin(st);
  const int grid = std::min(n, 8 * kNumSMs);
  launch_kernel(copy_pages_kernel, dim3(grid), dim3(256), 0, st, 1, list_dev, n,
                static_cast<int>(page_bytes / 16));
  RS_LAUNCH_CHECK();
  prof::end(tok, st, label, 0, 2.0 * static_cast<double>(page_bytes) * n);
  count_launch();
}

__global__ void gather_slots_i32_kernel(const std::int32_t* src, const std::int32_t* idx, int n,
                                        std::int32_t* out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) out[i] = src[idx[i]];
}

void gather_slots_i32(const std::int32_t* src, const std::int32_t* idx, int n, std::int32_t* out,
                      cudaStream_t st) {
  if (n <= 0) return;
  gather_slots_i32_kernel<<<(n + 255) / 256, 256, 0, st>>>(src, idx, n, out);
  RS_LAUNCH_CHECK();
  count_launch();
}

void fold_norm_weight(bf16* W, std::int64_t rows, int cols, int ld, const bf16* g, cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return;
  fold_norm_weight_kernel<<<elem_grid(rows * cols), 256, 0, st>>>(W, rows, cols, ld, g);
  RS_LAUNCH_CHECK();
  count_launch();
}

void fill_const(bf16* dst, std::int64_t n, float v, cudaStream_t st) {
  if (n <= 0) return;
  fill_const_kernel<<<elem_grid(n), 256, 0, st>>>(dst, n, v);
  RS_LAUNCH_CHECK();
  count_launch();
}

void fill_ids(std::int32_t* dst, std::int64_t n, std::uint64_t seed, std::uint64_t stream,
              std::uint32_t modulo, cudaStream_t st) {
  if (n <= 0) return;
  fill_ids_kernel<<<elem_grid(n), 256, 0, st>>>(dst, n, seed, stream, modulo);
  RS_LAUNCH_CHECK();
  count_launch();
}

void rmsnorm(const bf16* x, int ldx, const bf16* w, bf16* y, int ldy, int rows, int dim, float eps,
             cudaStream_t st, const std::int64_t* row_map, bf16* x_copy, int ld_copy,
             const int* rows_dev) {
  if (rows <= 0) return;
  if (dim % 8 != 0) throw DeviceError(RS_ERR_CUDA, "rmsnorm: dim % 8 != 0");
  const int tok = prof::begin(st);
  const int grid = row_grid(rows);
  const int blk = 32 * kWarpsPerBlock;
  if (rows_dev == nullptr && dim % 256 == 0 && dim / 256 <= 32) {
    switch (dim / 256) {
#define RS_RMS_CASE(V) \
  case V: rmsnorm_reg_kernel<V><<<grid, blk, 0, st>>>(x, ldx, w, y, ldy, rows, eps, row_map, x_copy, ld_copy); break;
      RS_RMS_CASE(1) RS_RMS_CASE(2) RS_RMS_CASE(4) RS_RMS_CASE(5) RS_RMS_CASE(14) RS_RMS_CASE(20)
      RS_RMS_CASE(32)
#undef RS_RMS_CASE
      default:
        rmsnorm_kernel<<<grid, blk, 0, st>>>(x, ldx, w, y, ldy, rows, dim, eps, row_map, x_copy,
                                             ld_copy, rows_dev);
    }
  } else {
    rmsnorm_kernel<<<grid, blk, 0, st>>>(x, ldx, w, y, ldy, rows, dim, eps, row_map, x_copy, ld_copy,
                                         rows_dev);
  }
  RS_LAUNCH_CHECK();
  prof::end(tok, st, row_map != nullptr ? "rmsnorm_gather" : "rmsnorm", 0,
            2.0 * rows * dim * (x_copy != nullptr ? 3.0 : 2.0));
  count_launch();
}

void rope_vit(bf16* qkv, int ld, const std::int32_t* pos_hw, int rows, int heads, int hd,
              float theta, cudaStream_t st) {
  if (rows <= 0) return;
  rope_vit_kernel<<<row_grid(static_cast<std::int64_t>(rows) * heads * 2), 32 * kWarpsPerBlock, 0,
                    st>>>(qkv, ld, pos_hw, rows, heads, hd, std::log2(theta));
  RS_LAUNCH_CHECK();
  count_launch();
}

void vit_rope_freq_table(int n_pos, int hd, float theta, float2* out, cudaStream_t st) {
  const int n = n_pos * (hd / 4);
  vit_rope_freq_kernel<<<ceil_div(n, 256), 256, 0, st>>>(n_pos, hd, std::log2(theta), out);
  RS_LAUNCH_CHECK();
  count_launch();
}

void vit_rope_table(const std::int32_t* pos_hw, int rows, int hd, float theta, float2* table,
                    cudaStream_t st) {
  if (rows <= 0) return;
  vit_rope_table_kernel<<<elem_grid(static_cast<std::int64_t>(rows) * hd / 2), 256, 0, st>>>(
      pos_hw, rows, hd, std::log2(theta), table);
  RS_LAUNCH_CHECK();
  count_launch();
}

void vit_qkv_split(const bf16* qkv, int ld, const float2* rope_table, int rows, int heads, int hd,
                   bf16* qp, bf16* kp, bf16* vt, int ld_vt, cudaStream_t st) {
  if (rows <= 0) return;
  if (hd > 128 || hd % 16 != 0) throw DeviceError(RS_ERR_CUDA, "vit_qkv_split: head_dim must be a multiple of 16, <= 128");
  const int tok = prof::begin(st);
  const std::int64_t items = static_cast<std::int64_t>(rows) * 2 * heads * (hd / 16);
  launch_kernel(vit_qk_rope_pad_kernel, dim3(elem_grid(items)), dim3(256), 0, st, 1, qkv, ld, rope_table,
                rows, heads, hd, qp, kp, heads * 128, 128);
  RS_LAUNCH_CHECK();
  launch_kernel(vit_v_transpose_kernel, dim3(ceil_div(rows, 64), heads), dim3(256), 0, st, 1, qkv, ld, rows,
                heads, hd, vt, ld_vt);
  RS_LAUNCH_CHECK();
  prof::end(tok, st, "vit_qkv_split", 0, 2.0 * rows * heads * hd * 3 * 2);
  count_launch(2);
}

void vit_qk_rope_inplace(bf16* qkv, int ld, const float2* rope_table, int rows, int heads, int hd,
                         cudaStream_t st) {
  if (rows <= 0) return;
  if (hd % 16 != 0) throw DeviceError(RS_ERR_CUDA, "vit_qk_rope_inplace: head_dim must be a multiple of 16");
  const int tok = prof::begin(st);
  const std::int64_t items = static_cast<std::int64_t>(rows) * 2 * heads * (hd / 16);
  vit_qk_rope_pad_kernel<<<elem_grid(items), 256, 0, st>>>(qkv, ld, rope_table, rows, heads, hd, qkv,
                                                           qkv + heads * hd, ld, hd);
  RS_LAUNCH_CHECK();
  prof::end(tok, st, "vit_rope", 0, 2.0 * rows * heads * hd * 2 * 2);
  count_launch();
}

void rope_kv_append(bf16* qkv, int ld, const ChunkRowInfo* rows_info, int rows, int q_heads,
                    int kv_heads, int hd, float theta, bf16* k_cache, bf16* v_cache,
                    const int* const* page_tables, int page_size, cudaStream_t st,
                    const int* rows_dev, const float2* table) {
  if (rows <= 0) return;
  if (rows_dev == nullptr && (hd == 64 || hd == 128)) {
    const int tok = prof::begin(st);
    const int passes = (q_heads + kv_heads + 32 / (hd / 16) - 1) / (32 / (hd / 16));
    const dim3 grid(row_grid(static_cast<std::int64_t>(rows) * passes), 2);
    launch_kernel(hd == 128 ? rope_kv_append_vec_kernel<128> : rope_kv_append_vec_kernel<64>, grid,
                  dim3(32 * kWarpsPerBlock), 0, st, 1, qkv, ld, rows_info, rows, q_heads, kv_heads,
                  std::log2(theta), k_cache, v_cache, page_tables, page_size, table);
    RS_LAUNCH_CHECK();
    // algorithmic bytes: q, k read + written, k and v appended (v read once)
    prof::end(tok, st, "rope_kv_append", 0,
              2.0 * rows * hd * (2.0 * (q_heads + kv_heads) + 2.0 * kv_heads));
    count_launch();
    return;
  }
  rope_kv_append_kernel<<<row_grid(static_cast<std::int64_t>(rows) * (q_heads + 2 * kv_heads)),
                          32 * kWarpsPerBlock, 0, st>>>(qkv, ld, rows_info, rows, q_heads, kv_heads,
                                                        hd, std::log2(theta), k_cache, v_cache,
                                                        page_tables, page_size, rows_dev);
  RS_LAUNCH_CHECK();
  count_launch();
}

__global__ void tp_reduce_kernel(bf16* x, int rows, int d, bf16* const* parts, int n_parts,
                                 unsigned long long* ss) {
  pdl_wait();
  pdl_launch_dependents();
  // one warp per row, 8 bf16 per lane per step
  const int lane = threadIdx.x & 31;
  for (int row = blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5); row < rows; row += gridDim.x * kWarpsPerBlock) {
    float sq = 0.f;
    bf16* xr = x + static_cast<std::int64_t>(row) * d;
    for (int c = lane * 8; c < d; c += 256) {
      const uint4 xv = *reinterpret_cast<const uint4*>(xr + c);
      const std::uint32_t xw[4] = {xv.x, xv.y, xv.z, xv.w};
      float acc[8];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const float2 f = unpack_bf16x2(xw[t]);
        acc[2 * t] = f.x;
        acc[2 * t + 1] = f.y;
      }
      float part[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      for (int p = 0; p < n_parts; ++p) {
        const uint4 pv = *reinterpret_cast<const uint4*>(parts[p] + static_cast<std::int64_t>(row) * d + c);
        const std::uint32_t pw[4] = {pv.x, pv.y, pv.z, pv.w};
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const float2 f = unpack_bf16x2(pw[t]);
          part[2 * t] += f.x;
          part[2 * t + 1] += f.y;
        }
      }
      std::uint32_t o[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        o[t] = pack_bf16x2(acc[2 * t] + part[2 * t], acc[2 * t + 1] + part[2 * t + 1]);
        const float2 f = unpack_bf16x2(o[t]);
        sq = fmaf(f.x, f.x, fmaf(f.y, f.y, sq));
      }
      *reinterpret_cast<uint4*>(xr + c) = make_uint4(o[0], o[1], o[2], o[3]);
    }
    sq = warp_sum(sq);
    if (lane == 0) ss[row] = static_cast<unsigned long long>(__float2ull_rn(sq * kSsFixedScale));
  }
}

void tp_reduce_residual(bf16* x, int rows, int d, bf16* const* parts, int n_parts, unsigned long long* ss,
                        cudaStream_t st) {
  if (rows <= 0) return;
  if (d % 256 != 0) throw DeviceError(RS_ERR_CUDA, "tp reduce: d % 256 != 0");
  launch_kernel(tp_reduce_kernel, dim3(row_grid(rows)), dim3(32 * kWarpsPerBlock), 0, st, 1, x, rows, d, parts,
                n_parts, ss);
  RS_LAUNCH_CHECK();
  count_launch();
}

__global__ void __launch_bounds__(128, 16) tp_group_reduce_kernel(const TpGroupArgs a) {
  pdl_wait();  // this rank's partial (previous kernel) is complete
  const int t = threadIdx.x;
  if (t < a.T) {
    unsigned* peer = a.flags[t] + blockIdx.x * kMaxTpRanks + a.rank;
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(peer), "r"(a.epoch) : "memory");
    const unsigned* mine = a.flags[a.rank] + blockIdx.x * kMaxTpRanks + t;
    unsigned v;
    unsigned long long t0 = 0;
    for (unsigned spins = 0;; ++spins) {
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(mine) : "memory");
      if (static_cast<int>(v - a.epoch) >= 0) break;
      if ((spins & 1023u) == 1023u) {  // a rank that never joins: fail the launch instead of hanging the GPU
        unsigned long long now;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
        if (t0 == 0) t0 = now;
        else if (now - t0 > 30ull * 1000 * 1000 * 1000) __trap();
      }
    }
  }
  __syncthreads();
  // only now may the next kernel of this stream start (PDL): a dependent grid
  // holding SMs while a peer sharing this GPU has not signalled could starve it
  pdl_launch_dependents();
  const int lane = t & 31, wpb = blockDim.x >> 5;
  for (int row = blockIdx.x * wpb + (t >> 5); row < a.rows; row += gridDim.x * wpb) {
    float sq = 0.f;
    bf16* xr = a.x + static_cast<std::int64_t>(row) * a.d;
    for (int c = lane * 8; c < a.d; c += 256) {
      const uint4 xv = *reinterpret_cast<const uint4*>(xr + c);
      const std::uint32_t xw[4] = {xv.x, xv.y, xv.z, xv.w};
      float part[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      for (int r = 0; r < a.T; ++r) {  // rank order: the same sum on every rank
        const uint4 pv = __ldcv(reinterpret_cast<const uint4*>(a.parts[r] + static_cast<std::int64_t>(row) * a.d + c));
        const std::uint32_t pw[4] = {pv.x, pv.y, pv.z, pv.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float2 f = unpack_bf16x2(pw[k]);
          part[2 * k] += f.x;
          part[2 * k + 1] += f.y;
        }
      }
      std::uint32_t o[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float2 xf = unpack_bf16x2(xw[k]);
        o[k] = pack_bf16x2(xf.x + part[2 * k], xf.y + part[2 * k + 1]);
        const float2 f = unpack_bf16x2(o[k]);
        sq = fmaf(f.x, f.x, fmaf(f.y, f.y, sq));
      }
      *reinterpret_cast<uint4*>(xr + c) = make_uint4(o[0], o[1], o[2], o[3]);
    }
    sq = warp_sum(sq);
    if (lane == 0) a.ss[row] = static_cast<unsigned long long>(__float2ull_rn(sq * kSsFixedScale));
  }
}

void tp_group_reduce(const TpGroupArgs& a, cudaStream_t st) {
  if (a.rows <= 0) return;
  if (a.d % 256 != 0) throw DeviceError(RS_ERR_CUDA, "tp group reduce: d % 256 != 0");
  if (a.T < 1 || a.T > kMaxTpRanks) throw DeviceError(RS_ERR_CUDA, "tp group reduce: 1..8 ranks");
  const int tok = prof::begin(st);
  // a fixed grid: every rank must use the same flag slots
  launch_kernel(tp_group_reduce_kernel, dim3(kTpBlocks), dim3(128), 0, st, 1, a);
  RS_LAUNCH_CHECK();
  prof::end(tok, st, "tp_group_reduce", 0, 2.0 * a.rows * a.d * (a.T + 2));
  count_launch();
}

__global__ void mrope_table_kernel(const ChunkRowInfo* __restrict__ info, int rows, int hd,
                                   float log2_theta, float2* table) {
  pdl_wait();
  pdl_launch_dependents();
  const int half = hd / 2, s_t = hd / 8, s_h = hd / 8 + (3 * hd) / 16;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < rows * half; e += gridDim.x * blockDim.x) {
    const int row = e / half, i = e % half;
    const int sec = i < s_t ? 0 : (i < s_h ? 1 : 2);
    const float freq = exp2f(-log2_theta * (2.0f * i) / static_cast<float>(hd));
    float sn, cs;
    sincosf(static_cast<float>(info[row].rope[sec]) * freq, &sn, &cs);
    table[e] = make_float2(cs, sn);
  }
}

void mrope_table(const ChunkRowInfo* rows_info, int rows, int hd, float theta, float2* table, cudaStream_t st) {
  if (rows <= 0) return;
  const int n = rows * hd / 2;
  launch_kernel(mrope_table_kernel, dim3(std::min((n + 255) / 256, kNumSMs * 8)), dim3(256), 0, st, 1,
                rows_info, rows, hd, std::log2(theta), table);
  RS_LAUNCH_CHECK();
  count_launch();
}

void scatter_rows_and_mark(const bf16* src, int n_rows, const std::int64_t* dst_rows, bf16* slab,
                           int d, std::uint32_t* bitmap, const std::uint64_t* ranges, int n_ranges,
                           cudaStream_t st) {
  if (d % 8 != 0) throw DeviceError(RS_ERR_CUDA, "scatter: d % 8 != 0");
  const int tok = prof::begin(st);
  scatter_rows_kernel<<<row_grid(n_rows > 0 ? n_rows : 1), 32 * kWarpsPerBlock, 0, st>>>(
      src, n_rows, dst_rows, slab, d, bitmap, ranges, n_ranges);
  RS_LAUNCH_CHECK();
  // algorithmic bytes: rows read + written, row indices, bitmap words
  prof::end(tok, st, "tracker_scatter_k6", 0,
            4.0 * n_rows * d + 8.0 * n_rows + 16.0 * n_ranges);
  count_launch();
}

void ready_prefix(const std::uint32_t* bitmap, std::uint64_t frontier, std::uint64_t total,
                  std::uint64_t* out, cudaStream_t st) {
  ready_prefix_kernel<<<1, 32, 0, st>>>(bitmap, frontier, total, out);
  RS_LAUNCH_CHECK();
  count_launch();
}

void gather_text_embeddings(const bf16* vocab, const std::int32_t* ids, int n,
                            const std::int64_t* dst_rows, bf16* slab, int d, cudaStream_t st) {
  if (n <= 0) return;
  gather_text_kernel<<<row_grid(n), 32 * kWarpsPerBlock, 0, st>>>(vocab, ids, n, dst_rows, slab, d);
  RS_LAUNCH_CHECK();
  count_launch();
}

void bitmap_set_ranges(std::uint32_t* bitmap, const std::uint64_t* ranges, int n_ranges,
                       cudaStream_t st) {
  if (n_ranges <= 0) return;
  bitmap_set_kernel<<<1, 256, 0, st>>>(bitmap, ranges, n_ranges);
  RS_LAUNCH_CHECK();
  count_launch();
}

void argmax_rows(const float* logits, int rows, int vocab, std::int32_t* out, cudaStream_t st,
                 const std::int32_t* rows_idx) {
  if (rows <= 0) return;
  argmax_kernel<<<rows, 1024, 0, st>>>(logits, vocab, out, rows_idx);
  RS_LAUNCH_CHECK();
  count_launch();
}

}  // namespace rserve
