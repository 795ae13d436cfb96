// rserve-b200 — tcgen05 / TMEM / TMA GEMM (see gemm.cuh for the contract).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <unordered_map>

#include "common.cuh"
#include "gemm.cuh"
#include "kernels.cuh"
#include "sm100.cuh"

namespace rserve {
namespace {

constexpr int kBM = 128;
constexpr int kBK = 64;  // 64 bf16 = 128 B = one swizzle row
constexpr int kEpiWarps = 8;  // two per TMEM lane quadrant, splitting the tile's columns
constexpr int kThreads = 128 + 32 * kEpiWarps;

struct GemmParams {
  void* C;
  int ldc;
  const bf16* bias;
  const bf16* residual;
  int ldr;
  const int* row_map;
  int M, N, K;
  const int* M_dev;
  // Tail split-K schedule (host-chosen, see launch()): tiles [0, dp_tiles)
  // are whole-K units striding over the grid; each of the remaining sk_tiles
  // is split into sk_splits equal k ranges, and those units are handed out
  // split-major, so CTAs running at the same time work on the same k range
  // of different tiles (the A / B slices stay shared in L2).
  int dp_tiles, sk_tiles, sk_splits;
  float* ws;     // split partials: [sk_splits][sk_tiles][kBM x BN] fp32
  int* counters; // per split tile arrival counts (self-resetting)
  int sk_debug;  // RS_GEMM_SK_DEBUG: 1 = no partial stores / fixup, 2 = no finisher epilogue
  // folded RMSNorm (gemm.cuh GemmArgs)
  const unsigned long long* ss_in;
  float ss_inv_dim, ss_eps;
  unsigned long long* ss_out;
  unsigned long long* ss_clear;
  int ss_clear_n;
  // Epi::QkvRope
  const ChunkRowInfo* rope_rows;
  const float2* rope_table;
  const int* const* page_tables;
  bf16* k_cache;
  bf16* v_cache;
  int rope_hq, rope_hkv, rope_hd, page_size;
  int early_b;   // issue the first ring's B tiles before the PDL wait (RS_GEMM_EARLY_B=0: off)
};

// Row scale of a norm-consumer GEMM (1 when the GEMM has no folded norm).
__device__ __forceinline__ float row_scale(const GemmParams& p, int row) {
  if (p.ss_in == nullptr || row >= p.M) return 1.f;
  const float ss = static_cast<float>(__ldcg(p.ss_in + row)) * (1.f / kSsFixedScale);
  return rsqrtf(ss * p.ss_inv_dim + p.ss_eps);
}
__device__ __forceinline__ void ss_accumulate(const GemmParams& p, int row, float ss) {
  atomicAdd(p.ss_out + row, static_cast<unsigned long long>(__float2ull_rn(ss * kSsFixedScale)));
}

// ---- work units ---------------------------------------------------------------
// A unit is (tile, [kb0, kb1)). Producer, MMA issuer and epilogue walk the same
// unit sequence. The split-K fixup never waits: each unit of a split tile
// stores its fp32 partial and bumps the tile's counter; the unit completing
// the count sums all partials in k order (deterministic) and runs the fused
// epilogue, so GEMMs sharing the SMs from several streams cannot deadlock.
struct Unit {
  int tile, kb0, kb1, split;  // split: k-range index, -1 for a whole tile
};
struct UnitIter {
  int dp_next, sk_next;
};
struct Sched {
  int dp_tiles, sk_tiles, sk_splits, num_kb, grid;
  __device__ UnitIter begin(int c) const { return {c, c}; }
  __device__ bool next(UnitIter& it, Unit& u) const {
    if (it.dp_next < dp_tiles) {
      u = {it.dp_next, 0, num_kb, -1};
      it.dp_next += grid;
      return true;
    }
    if (it.sk_next < sk_tiles * sk_splits) {
      const int sp = it.sk_next / sk_tiles, t = it.sk_next % sk_tiles;
      u = {dp_tiles + t, sp * num_kb / sk_splits, (sp + 1) * num_kb / sk_splits, sp};
      it.sk_next += grid;
      return true;
    }
    return false;
  }
};
constexpr int kMaxParts = 8;  // units per split tile (launch() guarantees the bound)

// CG = CTAs per tile: 1, or 2 for a CTA pair (cluster of 2 on one TPC) running
// 256 x BN tiles with cta_group::2 MMAs — each CTA stages its own 128 A rows
// and half of the B rows, halving per-SM shared-memory operand traffic.
// QkvRope epilogue staging (ROPE): the tile's 128 rows of the chunk's M-RoPE
// (cos, sin) table (hd = 128: 512 B per row, as 4 SW128 boxes of 32 floats)
// and the tile's BN bias values, loaded while the tile's MMAs run.
constexpr int kRopeTableBytes = 4 * 128 * 128;
// Wide pair tiles (BN = 320 / 448 / 512, CG = 2 only): the tile is issued as
// kSub = 2 MMAs of N = BN / 2 per k-step into adjacent TMEM columns; each CTA
// stages its half of each sub-tile's B rows ([sub 0: BN/4 rows][sub 1: BN/4
// rows]). One accumulator (2 x BN columns do not fit in TMEM): meant for
// launches of <= 1 wave, where the per-SM operand feed (A + B bytes per MMA
// FLOP, from L2) of the narrower tiles is the limit — e.g. the N = 1280 ViT
// projections as 64 tiles of 256 x 320 instead of 128 of 256 x 160.
// Residual epilogues prefetch EVERY residual chunk of a warp's share of the
// tile (one 2 KB buffer + mbarrier each, <= 5 per warp) before the
// accumulator wait, and store each output chunk from its residual buffer:
// the epilogue no longer waits one HBM round trip per chunk, which was the
// tail of single-wave launches (the N = 1280 ViT projections). Other
// epilogues keep a 2-buffer store ring.
template <int BN, int EPI, bool TMA_OUT>
constexpr bool res_deep() {
  return TMA_OUT && EPI == 1 /* Epi::Residual */ && (BN / 32 + 1) / 2 <= 5;
}
template <int BN, int EPI, bool TMA_OUT>
constexpr int epi_bufs() {
  return res_deep<BN, EPI, TMA_OUT>() && (BN / 32 + 1) / 2 > 2 ? (BN / 32 + 1) / 2 : 2;
}
template <int BN, bool TMA_OUT = false, int CG = 1, bool ROPE = false, int NB = 2>
struct Cfg {
  static_assert(BN % 32 == 0 && BN >= 128 &&
                    (BN <= 256 || ((BN == 320 || BN == 448 || BN == 512) && CG == 2 && !ROPE)),
                "tile width");
  static_assert(CG == 1 || (CG == 2 && BN % 32 == 0), "pair tiles split B in halves of 16-row multiples");
  static constexpr int kSub = BN > 256 ? 2 : 1;       // MMAs per k-step
  static constexpr int kSubN = BN / kSub;             // N of one MMA
  static constexpr int kSubRows = kSubN / CG;         // B rows per CTA per sub-tile (one TMA box)
  static constexpr int kAccBufs = 2 * BN <= 512 ? 2 : 1;
  static constexpr int kABytes = kBM * kBK * 2;
  static constexpr int kBBytes = (BN / CG) * kBK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  // epilogue staging: 8 warps x NB buffers x [32 rows x 64 B] (bf16 TMA stores)
  static constexpr int kEpiBuf = 2048;
  static constexpr int kEpiBytes = TMA_OUT ? kEpiWarps * NB * kEpiBuf : 0;
  static constexpr int kRopeBytes = ROPE ? kRopeTableBytes + 2 * BN : 0;
  // as many pipeline stages as the 227 KB of shared memory allow (<= 8)
  static constexpr int kStagesFit = (227 * 1024 - 1024 - 512 - kEpiBytes - kRopeBytes) / kStageBytes;
  static constexpr int kStages = kStagesFit > 8 ? 8 : kStagesFit;
  // double-buffered accumulator (kAccBufs), allocation rounded up to a power of two
  static constexpr int kTmemCols = kAccBufs * BN <= 256 ? 256 : 512;
  static constexpr int kSmem = kStages * kStageBytes + kEpiBytes + kRopeBytes + 1024 /*align*/ + 512 /*barriers*/;
};

__device__ __forceinline__ float gelu_erf(float x) {
  return 0.5f * x * (1.f + erff(x * 0.70710678118654752f));
}
__device__ __forceinline__ float silu(float x) {
  return __fdividef(x, 1.f + __expf(-x));
}
__device__ __forceinline__ float bias_add(float x, const bf16* bias, int col) {
  return bias != nullptr ? x + __bfloat162float(bias[col]) : x;
}
__device__ __forceinline__ float silu_plus(float x, const bf16* bias, int col) {
  return silu(bias_add(x, bias, col));
}

// Epilogue of one accumulator tile through shared memory and TMA stores:
// per warp (32 rows) and per 32-column output chunk, the accumulator is
// read from TMEM, the fused op applied, the bf16 / fp32 row written to a
// SW128-swizzled [32 x 32] smem box (conflict-free: 4 wavefronts per 512 B)
// and stored by one TMA (coalesced, asynchronous). Residual tiles are
// TMA-loaded one chunk ahead into the alternate buffer.
// Sum of the stream-K partials of one split tile at (row, col..col+31), in
// unit (k) order.
template <int BN>
__device__ __forceinline__ void ws_sum32(const float* const (&parts)[kMaxParts], int n_parts, int row,
                                         int col, std::uint32_t (&v)[32]) {
  float a[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) a[i] = 0.f;
  // partial layout: float4 (chunk, q, row) -> ((col/32) * 8 + q) * kBM + row, so
  // a warp's 32 rows of one float4 column are 512 contiguous bytes
  for (int k = 0; k < n_parts; ++k) {
    const float4* src = reinterpret_cast<const float4*>(parts[k]) + (col / 32) * 8 * kBM + row;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const float4 f = __ldcg(src + q * kBM);
      a[4 * q] += f.x;
      a[4 * q + 1] += f.y;
      a[4 * q + 2] += f.z;
      a[4 * q + 3] += f.w;
    }
  }
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(a[i]);
}

// The first residual chunk of a tile, issued by lane 0 of the epilogue warp
// before it waits for the accumulator (its latency hides behind the mainloop).
template <int BN, int EPI, bool DEEP = false>
__device__ __forceinline__ void prefetch_residual(const CUtensorMap* tmR, std::uint8_t* bufs,
                                                  std::uint64_t* rbar, std::uint32_t ec, int m0, int n0,
                                                  int quad, int half, int lane) {
  constexpr int kChunks = BN / 32;
  const int c_begin = half == 0 ? 0 : (kChunks + 1) / 2;
  const int c_end = half == 0 ? (kChunks + 1) / 2 : kChunks;
  if constexpr (DEEP) {
    if (lane == 0 && c_begin < c_end) {
      sm100::bulk_wait_read<0>();  // the previous tile's stores no longer read the buffers
      for (int i = 0; i < c_end - c_begin; ++i) {
        sm100::mbar_expect_tx(&rbar[i], 32 * 64);
        sm100::tma_load_2d(bufs + i * 2048, tmR, &rbar[i], n0 + (c_begin + i) * 32, m0 + quad * 32);
      }
    }
    return;
  }
  if (lane == 0 && c_begin < c_end) {
    sm100::bulk_wait_read<0>();  // the previous tile's stores no longer read the buffers
    const std::uint32_t b = ec & 1;
    sm100::mbar_expect_tx(&rbar[b], 32 * 64);
    sm100::tma_load_2d(bufs + b * 2048, tmR, &rbar[b], n0 + c_begin * 32, m0 + quad * 32);
  }
}

template <int BN, int EPI, bool FROM_WS = false, bool DEEP = false>
__device__ __forceinline__ void epilogue_tile_tma(const GemmParams& p, const CUtensorMap* tmC,
                                                  const CUtensorMap* tmR, std::uint8_t* bufs,
                                                  std::uint64_t* rbar, std::uint32_t& rphase,
                                                  std::uint32_t& ec, std::uint32_t t_row, int m0,
                                                  int n0, int quad, int half, int lane,
                                                  const float* const (&parts)[kMaxParts] = {},
                                                  int n_parts = 0, bool res_issued = false,
                                                  const std::uint8_t* rope_smem = nullptr) {
  const int my_row = m0 + quad * 32 + lane;
  const float rs = row_scale(p, my_row);
  float ss = 0.f;  // sum of squares of this thread's output row segment (ss_out)
  constexpr bool kRope = EPI == static_cast<int>(Epi::QkvRope);
  std::int64_t kv_page = 0;
  int kv_off = 0;
  if constexpr (kRope) {
    if (my_row < p.M) {
      const ChunkRowInfo ri = p.rope_rows[my_row];
      kv_page = p.page_tables[ri.req_slot][ri.pos / p.page_size];
      kv_off = ri.pos % p.page_size;
    }
  }
  constexpr bool kRes = EPI == static_cast<int>(Epi::Residual);
  constexpr bool kSwi = EPI == static_cast<int>(Epi::SwiGLU);
  constexpr bool kF32 = EPI == static_cast<int>(Epi::StoreF32);
  static_assert(!kF32, "fp32 outputs use the direct epilogue");
  constexpr int kAccPerChunk = kSwi ? 64 : 32;  // accumulator columns per output chunk
  constexpr int kChunks = BN / kAccPerChunk;
  constexpr int kRowBytes = kF32 ? 128 : 64;    // 32 output columns
  constexpr int kBuf = 2048;
  // the two warps of a lane quadrant split the chunks
  const int c_begin = half == 0 ? 0 : (kChunks + 1) / 2;
  const int c_end = half == 0 ? (kChunks + 1) / 2 : kChunks;
  const int row0 = m0 + quad * 32;
  const int out_col0 = kSwi ? n0 / 2 : n0;
  auto issue_res = [&](int chunk, std::uint32_t b) {
    sm100::mbar_expect_tx(&rbar[b], 32 * 64);
    sm100::tma_load_2d(bufs + b * kBuf, tmR, &rbar[b], n0 + chunk * 32, row0);
  };
  if constexpr (kRes) {
    if (lane == 0 && c_begin < c_end && !res_issued) {
      sm100::bulk_wait_read<0>();
      if constexpr (DEEP) {
        for (int i = 0; i < c_end - c_begin; ++i) issue_res(c_begin + i, i);
      } else {
        issue_res(c_begin, ec & 1);
      }
    }
  }
#pragma unroll 1
  for (int c = c_begin; c < c_end; ++c, ++ec) {
    // DEEP: chunk i of the warp's share has its own residual / output buffer
    const std::uint32_t b = DEEP ? static_cast<std::uint32_t>(c - c_begin) : ec & 1;
    std::uint8_t* buf = bufs + b * kBuf;
    if (lane == 0) {
      if constexpr (kRes && DEEP) {
        // every residual chunk already in flight; no buffer is reused within the tile
      } else if constexpr (kRes) {
        sm100::bulk_wait_read<0>();  // buffer b^1 (chunk c-1's store) drained
        if (c + 1 < c_end) issue_res(c + 1, b ^ 1);
      } else {
        sm100::bulk_wait_read<1>();  // buffer b (chunk c-2's store) drained
      }
    }
    __syncwarp();
    float x[32];
    {
      std::uint32_t v[32];
      const int prow = quad * 32 + lane;  // row within the tile (stream-K partials)
      if constexpr (FROM_WS) ws_sum32<BN>(parts, n_parts, prow, c * kAccPerChunk, v);
      else sm100::tmem_ld_32x32b_x32(t_row + static_cast<std::uint32_t>(c * kAccPerChunk), v);
      if constexpr (kSwi) {
        std::uint32_t u[32];
        if constexpr (FROM_WS) {
          ws_sum32<BN>(parts, n_parts, prow, c * kAccPerChunk + 32, u);
        } else {
          sm100::tmem_ld_32x32b_x32(t_row + static_cast<std::uint32_t>(c * kAccPerChunk + 32), u);
          sm100::tmem_ld_wait();
        }
        // [g0..15 u0..15 | g16..31 u16..31] -> 32 outputs
#pragma unroll
        for (int t = 0; t < 16; ++t) {
          x[t] = silu_plus(rs * __uint_as_float(v[t]), p.bias, n0 + c * 64 + t) *
                 bias_add(rs * __uint_as_float(v[16 + t]), p.bias, n0 + c * 64 + 16 + t);
          x[16 + t] = silu_plus(rs * __uint_as_float(u[t]), p.bias, n0 + c * 64 + 32 + t) *
                      bias_add(rs * __uint_as_float(u[16 + t]), p.bias, n0 + c * 64 + 48 + t);
        }
      } else {
        if constexpr (!FROM_WS) sm100::tmem_ld_wait();
        const int col = n0 + c * 32;
        // staged tile bias (QkvRope): [BN] bf16 after the rope table
        const std::uint8_t* sbias = kRope && rope_smem != nullptr ? rope_smem + kRopeTableBytes : nullptr;
        if (p.ss_in != nullptr || (p.bias != nullptr && col < p.N)) {
          // v = rs * acc + bias, two columns per packed FFMA2
          const float2 rs2 = make_float2(rs, rs);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            uint4 bb = make_uint4(0, 0, 0, 0);
            if (sbias != nullptr) bb = *reinterpret_cast<const uint4*>(sbias + (c * 32 + q * 8) * 2);
            else if (p.bias != nullptr && col < p.N) bb = *reinterpret_cast<const uint4*>(p.bias + col + q * 8);
            const std::uint32_t bw[4] = {bb.x, bb.y, bb.z, bb.w};
#pragma unroll
            for (int t = 0; t < 4; ++t) {
              const float2 y = fma2(make_float2(__uint_as_float(v[q * 8 + 2 * t]), __uint_as_float(v[q * 8 + 2 * t + 1])),
                                    rs2, unpack_bf16x2(bw[t]));
              v[q * 8 + 2 * t] = __float_as_uint(y.x);
              v[q * 8 + 2 * t + 1] = __float_as_uint(y.y);
            }
          }
        }
#pragma unroll
        for (int t = 0; t < 32; ++t) x[t] = __uint_as_float(v[t]);
        if constexpr (EPI == static_cast<int>(Epi::Gelu)) {
#pragma unroll
          for (int t = 0; t < 32; ++t) x[t] = gelu_erf(x[t]);
        }
        if constexpr (kRope) {
          // M-RoPE on q / k (rotate-half partner 64 columns away, in this tile:
          // tiles are whole heads), then k / v into the paged cache
          const int hd = p.rope_hd, half_hd = hd / 2;
          const int head = col / hd, i0 = col % hd;
          const bool is_v = head >= p.rope_hq + p.rope_hkv;
          if (!is_v && col < p.N) {
            const int delta = i0 < half_hd ? half_hd : -half_hd;
            std::uint32_t w[32];
            if constexpr (FROM_WS) ws_sum32<BN>(parts, n_parts, prow, c * 32 + delta, w);
            else {
              sm100::tmem_ld_32x32b_x32(t_row + static_cast<std::uint32_t>(c * 32 + delta), w);
              sm100::tmem_ld_wait();
            }
            const float4* cs = reinterpret_cast<const float4*>(
                p.rope_table + static_cast<std::int64_t>(min(my_row, p.M - 1)) * half_hd + (i0 % half_hd));
            const float sgn = i0 < half_hd ? -1.f : 1.f;
            const float2 rs2 = make_float2(rs, rs);
#pragma unroll
            for (int q = 0; q < 4; ++q) {  // partner: rs * acc + bias (8 columns per 16-byte load)
              uint4 bb = make_uint4(0, 0, 0, 0);
              if (sbias != nullptr) bb = *reinterpret_cast<const uint4*>(sbias + (c * 32 + delta + q * 8) * 2);
              else if (p.bias != nullptr) bb = *reinterpret_cast<const uint4*>(p.bias + col + delta + q * 8);
              const std::uint32_t bw[4] = {bb.x, bb.y, bb.z, bb.w};
#pragma unroll
              for (int t = 0; t < 4; ++t) {
                const float2 y = fma2(make_float2(__uint_as_float(w[q * 8 + 2 * t]), __uint_as_float(w[q * 8 + 2 * t + 1])),
                                      rs2, unpack_bf16x2(bw[t]));
                w[q * 8 + 2 * t] = __float_as_uint(y.x);
                w[q * 8 + 2 * t + 1] = __float_as_uint(y.y);
              }
            }
            // staged table row (4 SW128 boxes of [128 rows x 32 floats]): pair j at byte 8 j
            const int trow = quad * 32 + lane;
            const std::uint32_t tsm = rope_smem != nullptr ? sm100::smem_u32(rope_smem) : 0u;
#pragma unroll
            for (int q = 0; q < 16; ++q) {  // (cos, sin) of two columns per 16-byte load
              float4 c4;
              if (rope_smem != nullptr) {
                const int off = (i0 % half_hd) * 8 + q * 16;  // byte offset in the table row
                const std::uint32_t a = tsm + static_cast<std::uint32_t>((off >> 7) * 16384 + trow * 128 +
                                                                         ((((off >> 4) & 7) ^ (trow & 7)) << 4));
                asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
                             : "=f"(c4.x), "=f"(c4.y), "=f"(c4.z), "=f"(c4.w) : "r"(a));
              } else {
                c4 = __ldg(cs + q);
              }
              const float2 xr = fma2(make_float2(__uint_as_float(w[2 * q]), __uint_as_float(w[2 * q + 1])),
                                     make_float2(sgn * c4.y, sgn * c4.w),
                                     mul2(make_float2(x[2 * q], x[2 * q + 1]), make_float2(c4.x, c4.z)));
              x[2 * q] = xr.x;
              x[2 * q + 1] = xr.y;
            }
          }
          if (head >= p.rope_hq && my_row < p.M && col < p.N) {
            std::uint32_t o[16];
#pragma unroll
            for (int t = 0; t < 16; ++t) o[t] = pack_bf16x2(x[2 * t], x[2 * t + 1]);
            if (!is_v) {  // K: [page][kv head][token][hd]
              const int kvh = head - p.rope_hq;
              uint4* dst = reinterpret_cast<uint4*>(
                  p.k_cache + ((kv_page * p.rope_hkv + kvh) * p.page_size + kv_off) * hd + i0);
#pragma unroll
              for (int q = 0; q < 4; ++q) dst[q] = make_uint4(o[4 * q], o[4 * q + 1], o[4 * q + 2], o[4 * q + 3]);
            } else {      // V transposed: [page][kv head][hd][token]
              const int kvh = head - p.rope_hq - p.rope_hkv;
              bf16* dst = p.v_cache + ((kv_page * p.rope_hkv + kvh) * hd + i0) * p.page_size + kv_off;
#pragma unroll
              for (int t = 0; t < 32; ++t) dst[static_cast<std::int64_t>(t) * p.page_size] = __float2bfloat16_rn(x[t]);
            }
          }
        }
      }
    }
    if constexpr (kRes) {
      // lane 0 waits for the residual tile's TMA bytes, __syncwarp orders the
      // other lanes' smem reads after it
      if (lane == 0) sm100::mbar_wait(&rbar[b], (rphase >> b) & 1);
      __syncwarp();
      rphase ^= 1u << b;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint4 rv = *reinterpret_cast<const uint4*>(buf + sm100::sw64(lane * 64 + q * 16));
        const std::uint32_t rw[4] = {rv.x, rv.y, rv.z, rv.w};
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const float2 f = unpack_bf16x2(rw[t]);
          x[q * 8 + 2 * t] += f.x;
          x[q * 8 + 2 * t + 1] += f.y;
        }
      }
    }
    if constexpr (kF32) {
#pragma unroll
      for (int q = 0; q < 8; ++q)
        *reinterpret_cast<float4*>(buf + sm100::sw128(lane * kRowBytes + q * 16)) =
            make_float4(x[4 * q], x[4 * q + 1], x[4 * q + 2], x[4 * q + 3]);
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint4 o = make_uint4(pack_bf16x2(x[8 * q], x[8 * q + 1]), pack_bf16x2(x[8 * q + 2], x[8 * q + 3]),
                                   pack_bf16x2(x[8 * q + 4], x[8 * q + 5]), pack_bf16x2(x[8 * q + 6], x[8 * q + 7]));
        *reinterpret_cast<uint4*>(buf + sm100::sw64(lane * kRowBytes + q * 16)) = o;
        if constexpr (kRes) {
          if (p.ss_out != nullptr) {  // the bf16 values the next GEMM reads
            const std::uint32_t ow[4] = {o.x, o.y, o.z, o.w};
#pragma unroll
            for (int t = 0; t < 4; ++t) {
              const float2 f = unpack_bf16x2(ow[t]);
              ss = fmaf(f.x, f.x, fmaf(f.y, f.y, ss));
            }
          }
        }
      }
    }
    sm100::fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
      sm100::tma_store_2d(tmC, buf, out_col0 + c * 32, row0);
      sm100::bulk_commit();
    }
  }
  if constexpr (kRes) {
    if (p.ss_out != nullptr && c_begin < c_end && my_row < p.M) ss_accumulate(p, my_row, ss);
  }
}

template <int EPI>
__device__ __forceinline__ void epilogue_chunk(const GemmParams& p, int row, int col,
                                               const std::uint32_t (&v)[32], float rs, float& ss) {
  float x[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) x[i] = rs * __uint_as_float(v[i]);
  const int nvalid = min(32, p.N - col);  // 16 or 32 (N % 16 == 0)
  if (p.bias != nullptr) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (q * 8 < nvalid) {
        const uint4 b = *reinterpret_cast<const uint4*>(p.bias + col + q * 8);
        const std::uint32_t bw[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const float2 f = unpack_bf16x2(bw[t]);
          x[q * 8 + 2 * t] += f.x;
          x[q * 8 + 2 * t + 1] += f.y;
        }
      }
    }
  }
  const int out_row = p.row_map != nullptr ? p.row_map[row] : row;
  if constexpr (EPI == static_cast<int>(Epi::StoreF32)) {
    float* c = static_cast<float*>(p.C) + static_cast<std::int64_t>(out_row) * p.ldc + col;
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (q * 4 < nvalid)
        *reinterpret_cast<float4*>(c + q * 4) =
            make_float4(x[4 * q], x[4 * q + 1], x[4 * q + 2], x[4 * q + 3]);
  } else if constexpr (EPI == static_cast<int>(Epi::SwiGLU)) {
    // Columns [col, col+16) are gate rows, [col+16, col+32) the matching up
    // rows (weights interleaved in 16-row blocks by the model loader).
    bf16* c = static_cast<bf16*>(p.C) + static_cast<std::int64_t>(out_row) * p.ldc + col / 2;
    std::uint32_t o[8];
#pragma unroll
    for (int t = 0; t < 8; ++t)
      o[t] = pack_bf16x2(silu(x[2 * t]) * x[16 + 2 * t], silu(x[2 * t + 1]) * x[17 + 2 * t]);
    reinterpret_cast<uint4*>(c)[0] = make_uint4(o[0], o[1], o[2], o[3]);
    reinterpret_cast<uint4*>(c)[1] = make_uint4(o[4], o[5], o[6], o[7]);
  } else {
    if constexpr (EPI == static_cast<int>(Epi::Gelu)) {
#pragma unroll
      for (int i = 0; i < 32; ++i) x[i] = gelu_erf(x[i]);
    }
    if constexpr (EPI == static_cast<int>(Epi::Residual)) {
      const bf16* r = p.residual + static_cast<std::int64_t>(out_row) * p.ldr + col;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (q * 8 < nvalid) {
          const uint4 rv = *reinterpret_cast<const uint4*>(r + q * 8);
          const std::uint32_t rw[4] = {rv.x, rv.y, rv.z, rv.w};
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const float2 f = unpack_bf16x2(rw[t]);
            x[q * 8 + 2 * t] += f.x;
            x[q * 8 + 2 * t + 1] += f.y;
          }
        }
      }
    }
    bf16* c = static_cast<bf16*>(p.C) + static_cast<std::int64_t>(out_row) * p.ldc + col;
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (q * 8 < nvalid) {
        const uint4 o = make_uint4(pack_bf16x2(x[8 * q], x[8 * q + 1]), pack_bf16x2(x[8 * q + 2], x[8 * q + 3]),
                                   pack_bf16x2(x[8 * q + 4], x[8 * q + 5]),
                                   pack_bf16x2(x[8 * q + 6], x[8 * q + 7]));
        reinterpret_cast<uint4*>(c)[q] = o;
        if (EPI == static_cast<int>(Epi::Residual) && p.ss_out != nullptr) {
          const std::uint32_t ow[4] = {o.x, o.y, o.z, o.w};
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const float2 f = unpack_bf16x2(ow[t]);
            ss = fmaf(f.x, f.x, fmaf(f.y, f.y, ss));
          }
        }
      }

  }
}

// One CTA's share of a pair tile's B k-block (tile column tn): per sub-tile,
// rows [tn * BN + sub * kSubN + rank * kSubRows, + kSubRows).
template <class C>
__device__ __forceinline__ void load_b_cg2(std::uint8_t* dst, const CUtensorMap* tmB, std::uint32_t fb, int k0,
                                           int tn, std::uint32_t rank) {
#pragma unroll
  for (int sub = 0; sub < C::kSub; ++sub)
    sm100::tma_load_2d_cg2(dst + sub * C::kSubRows * kBK * 2, tmB, fb, k0,
                           tn * C::kSub * C::kSubN + sub * C::kSubN + static_cast<int>(rank) * C::kSubRows);
}

template <int BN, int EPI, bool TMA_OUT, int CG>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tcgen05_kernel(const __grid_constant__ CUtensorMap tmA,
                        const __grid_constant__ CUtensorMap tmB,
                        const __grid_constant__ CUtensorMap tmC,
                        const __grid_constant__ CUtensorMap tmR, const GemmParams p) {
  // QkvRope: tmR maps the chunk's M-RoPE table, staged per tile into smem
  constexpr bool kRopeStage = TMA_OUT && EPI == static_cast<int>(Epi::QkvRope);
  constexpr bool kDeep = res_deep<BN, EPI, TMA_OUT>();
  constexpr int kNB = epi_bufs<BN, EPI, TMA_OUT>();
  using C = Cfg<BN, TMA_OUT, CG, kRopeStage, kNB>;
  static_assert(2 * C::kStages + 4 + kNB * kEpiWarps + 1 <= 60, "barrier slots overlap the rope-table barrier");
  extern __shared__ __align__(1024) std::uint8_t smem_raw[];
  std::uint8_t* smem = reinterpret_cast<std::uint8_t*>(
      (reinterpret_cast<std::uintptr_t>(smem_raw) + 1023) & ~std::uintptr_t(1023));
  std::uint8_t* smem_a = smem;
  std::uint8_t* smem_b = smem + C::kStages * C::kABytes;
  std::uint8_t* smem_epi = smem + C::kStages * C::kStageBytes;  // 1024-aligned
  std::uint8_t* rope_smem = smem_epi + C::kEpiBytes;  // [kRopeTableBytes] table + [BN] bias (kRopeStage)
  std::uint64_t* bars = reinterpret_cast<std::uint64_t*>(rope_smem + C::kRopeBytes);
  std::uint64_t* full = bars;
  std::uint64_t* empty = bars + C::kStages;
  std::uint64_t* tfull = bars + 2 * C::kStages;
  std::uint64_t* tempty = tfull + 2;
  std::uint64_t* rbar = tempty + 2;  // [epilogue warps][kNB] residual-load barriers
  std::uint32_t* tmem_holder = reinterpret_cast<std::uint32_t*>(rbar + kNB * kEpiWarps);
  volatile int* sk_finisher = reinterpret_cast<volatile int*>(tmem_holder + 1);
  std::uint64_t* tbar = bars + 60;  // rope table TMA (kRopeStage)

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  pdl_launch_dependents();
  // CTA pair: rank 0 (leader) issues the MMAs; both CTAs load and drain.
  const std::uint32_t rank = CG == 2 ? sm100::cluster_ctarank() : 0u;
  const int M = p.M_dev != nullptr ? min(*p.M_dev, p.M) : p.M;
  const int m_tiles = (M + kBM * CG - 1) / (kBM * CG);
  const int n_tiles = (p.N + BN - 1) / BN;
  const int num_tiles = m_tiles * n_tiles;
  const int num_kb = (p.K + kBK - 1) / kBK;
  // data-parallel only unless the host chose a stream-K tail
  const Sched sched{p.sk_tiles > 0 ? p.dp_tiles : num_tiles, p.sk_tiles, p.sk_tiles > 0 ? p.sk_splits : 0,
                    num_kb, static_cast<int>(gridDim.x) / CG};
  const int unit0 = static_cast<int>(blockIdx.x) / CG;

  if (warp == 0 && lane == 0) {
    sm100::tma_prefetch_desc(&tmA);
    sm100::tma_prefetch_desc(&tmB);
    for (int s = 0; s < C::kStages; ++s) {
      sm100::mbar_init(&full[s], 1);
      sm100::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      sm100::mbar_init(&tfull[a], 1);
      sm100::mbar_init(&tempty[a], kEpiWarps * CG);  // pair: both CTAs' epilogue warps
    }
    for (int r = 0; r < kNB * kEpiWarps; ++r) sm100::mbar_init(&rbar[r], 1);
    sm100::mbar_init(tbar, 1);
    if constexpr (TMA_OUT) {
      sm100::tma_prefetch_desc(&tmC);
      if (EPI == static_cast<int>(Epi::Residual) || kRopeStage) sm100::tma_prefetch_desc(&tmR);
    }
    sm100::fence_mbar_init();
  }
  if (warp == 2) {
    if constexpr (CG == 2) sm100::tmem_alloc_cg2(tmem_holder, C::kTmemCols);
    else sm100::tmem_alloc(tmem_holder, C::kTmemCols);
  }
  sm100::tc_fence_before();
  if constexpr (CG == 2) sm100::cluster_sync();  // peer barriers initialised before any remote use
  else __syncthreads();
  sm100::tc_fence_after();
  const std::uint32_t tmem_base = *tmem_holder;
  // B (the weights) is never produced by the kernels this one depends on:
  // the producer issues the first ring's B tiles before the PDL wait, so the
  // weight stream starts under the previous kernel's tail; A follows the wait.
  int pre_b = 0;  // leading k-blocks whose B (and expect_tx) were issued early
  if (warp == 0 && lane == 0 && p.early_b) {
    UnitIter it0 = sched.begin(unit0);
    Unit u0;
    if (sched.next(it0, u0)) {
      const int n0 = (u0.tile / m_tiles) * BN + static_cast<int>(rank) * (BN / CG);
      for (int kb = u0.kb0; kb < u0.kb1 && pre_b < C::kStages; ++kb, ++pre_b) {
        if constexpr (CG == 2) {
          if (rank == 0) sm100::mbar_expect_tx(&full[pre_b], 2 * C::kStageBytes);
          const std::uint32_t fb = sm100::mapa(sm100::smem_u32(&full[pre_b]), 0);
          load_b_cg2<C>(smem_b + pre_b * C::kBBytes, &tmB, fb, kb * kBK, u0.tile / m_tiles, rank);
        } else {
          sm100::mbar_expect_tx(&full[pre_b], C::kStageBytes);
          sm100::tma_load_2d(smem_b + pre_b * C::kBBytes, &tmB, &full[pre_b], kb * kBK, n0);
        }
      }
    }
  }
  // PDL: the setup above (barriers, TMEM, descriptor prefetch) overlapped the
  // previous kernel's tail; its outputs are visible from here on.
  pdl_wait();
  for (int i = blockIdx.x * kThreads + threadIdx.x; i < p.ss_clear_n; i += gridDim.x * kThreads)
    p.ss_clear[i] = 0ull;

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer ----------------
    int stage = 0;
    std::uint32_t phase = 0;
    UnitIter it = sched.begin(unit0);
    Unit u;
    while (sched.next(it, u)) {
      const int m0 = (u.tile % m_tiles) * (kBM * CG) + static_cast<int>(rank) * kBM;
      const int n0 = (u.tile / m_tiles) * BN + static_cast<int>(rank) * (BN / CG);
      for (int kb = u.kb0; kb < u.kb1; ++kb) {
        sm100::mbar_wait(&empty[stage], phase ^ 1);
        const bool early = pre_b > 0;  // B + expect_tx already issued (first ring, first unit)
        if (early) --pre_b;
        if constexpr (CG == 2) {
          // both CTAs' bytes complete on the leader's full barrier
          if (rank == 0 && !early) sm100::mbar_expect_tx(&full[stage], 2 * C::kStageBytes);
          const std::uint32_t fb = sm100::mapa(sm100::smem_u32(&full[stage]), 0);
          sm100::tma_load_2d_cg2(smem_a + stage * C::kABytes, &tmA, fb, kb * kBK, m0);
          if (!early) load_b_cg2<C>(smem_b + stage * C::kBBytes, &tmB, fb, kb * kBK, u.tile / m_tiles, rank);
        } else {
          if (!early) sm100::mbar_expect_tx(&full[stage], C::kStageBytes);
          sm100::tma_load_2d(smem_a + stage * C::kABytes, &tmA, &full[stage], kb * kBK, m0);
          if (!early) sm100::tma_load_2d(smem_b + stage * C::kBBytes, &tmB, &full[stage], kb * kBK, n0);
        }
        if (++stage == C::kStages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1 && lane == 0 && rank == 0) {
    // ---------------- MMA issuer (single thread; pair leader) ----------------
    constexpr std::uint32_t idesc = sm100::idesc_bf16_f32(kBM * CG, C::kSubN);
    int stage = 0;
    std::uint32_t phase = 0;
    int local = 0;
    UnitIter it = sched.begin(unit0);
    Unit u;
    for (; sched.next(it, u); ++local) {
      const int acc = local % C::kAccBufs;
      const std::uint32_t acc_phase = (local / C::kAccBufs) & 1;
      sm100::mbar_wait(&tempty[acc], acc_phase ^ 1);
      sm100::tc_fence_after();
      const std::uint32_t d_tmem = tmem_base + static_cast<std::uint32_t>(acc * BN);
      for (int kb = u.kb0; kb < u.kb1; ++kb) {
        sm100::mbar_wait(&full[stage], phase);
        sm100::tc_fence_after();
        const std::uint64_t adesc =
            sm100::sw128_kmajor_desc(sm100::smem_u32(smem_a + stage * C::kABytes));
        const std::uint64_t bdesc =
            sm100::sw128_kmajor_desc(sm100::smem_u32(smem_b + stage * C::kBBytes));
#pragma unroll
        for (int kk = 0; kk < kBK / 16; ++kk) {
          // +32 B along K inside the 128B swizzle atom = +2 in the >>4 field.
#pragma unroll
          for (int sub = 0; sub < C::kSub; ++sub) {
            // sub-tile B rows start kSubRows * 128 B further (whole 1 KB swizzle atoms)
            const std::uint64_t bd = bdesc + 2 * kk + static_cast<std::uint64_t>(sub * C::kSubRows * 128 / 16);
            const std::uint32_t dt = d_tmem + static_cast<std::uint32_t>(sub * C::kSubN);
            if constexpr (CG == 2)
              sm100::umma_bf16_cg2(dt, adesc + 2 * kk, bd, idesc, (kb != u.kb0 || kk != 0) ? 1u : 0u);
            else
              sm100::umma_bf16(dt, adesc + 2 * kk, bd, idesc, (kb != u.kb0 || kk != 0) ? 1u : 0u);
          }
        }
        // frees the smem slot (in both CTAs of a pair) when the MMAs finish
        if constexpr (CG == 2) sm100::umma_commit_cg2(&empty[stage], 3);
        else sm100::umma_commit(&empty[stage]);
        if (++stage == C::kStages) {
          stage = 0;
          phase ^= 1;
        }
      }
      // accumulator ready for the epilogue (both CTAs' halves of a pair tile)
      if constexpr (CG == 2) sm100::umma_commit_cg2(&tfull[acc], 3);
      else sm100::umma_commit(&tfull[acc]);
    }
  } else if (warp >= 4) {
    // ---------------- epilogue warps ----------------
    const int quad = warp & 3;         // TMEM lanes [32*quad, 32*quad + 32) (warp % 4 rule)
    const int half = (warp - 4) >> 2;  // which half of the tile's columns
    int local = 0;
    std::uint32_t ec = 0, rphase = 0, tphase = 0;  // TMA-epilogue chunk counter / residual / rope-table phases
    UnitIter it = sched.begin(unit0);
    Unit u;
    // accumulator-free signal goes to the MMA issuer's CTA (the pair leader)
    auto release_acc = [&](int acc) {
      if constexpr (CG == 2) sm100::mbar_arrive_cluster(sm100::mapa(sm100::smem_u32(&tempty[acc]), 0));
      else sm100::mbar_arrive(&tempty[acc]);
    };
    for (; sched.next(it, u); ++local) {
      const int m0 = (u.tile % m_tiles) * (kBM * CG) + static_cast<int>(rank) * kBM;
      const int n0 = (u.tile / m_tiles) * BN;
      const int acc = local % C::kAccBufs;
      const std::uint32_t acc_phase = (local / C::kAccBufs) & 1;
      const std::uint32_t t_row =
          tmem_base + (static_cast<std::uint32_t>(quad * 32) << 16) + static_cast<std::uint32_t>(acc * BN);
      if (TMA_OUT && u.split >= 0) {
        // ---- split unit: store the fp32 partial, count, maybe finish ----
        // split tile index of this CTA's 128-row half (pairs: one per rank)
        const int t_sk = (u.tile - sched.dp_tiles) * CG + static_cast<int>(rank);
        const int n_parts = sched.sk_splits;
        auto part_ptr = [&](int sp) {
          return p.ws + (static_cast<std::int64_t>(sp) * sched.sk_tiles * CG + t_sk) * (kBM * BN);
        };
        sm100::mbar_wait(&tfull[acc], acc_phase);
        sm100::tc_fence_after();
        if (p.sk_debug == 1) {
          sm100::tc_fence_before();
          __syncwarp();
          if (lane == 0) release_acc(acc);
          continue;
        }
        {
          // coalesced partial layout (ws_sum32): warp stores of 512 contiguous bytes
          float4* mine = reinterpret_cast<float4*>(part_ptr(u.split)) + quad * 32 + lane;
          constexpr int kCh = BN / 32;
          const int c0 = half == 0 ? 0 : (kCh + 1) / 2, c1 = half == 0 ? (kCh + 1) / 2 : kCh;
#pragma unroll 1
          for (int c = c0; c < c1; ++c) {
            std::uint32_t v[32];
            sm100::tmem_ld_32x32b_x32(t_row + static_cast<std::uint32_t>(c * 32), v);
            sm100::tmem_ld_wait();
            float4* dst = mine + c * 8 * kBM;
#pragma unroll
            for (int q = 0; q < 8; ++q)
              __stcg(dst + q * kBM, make_float4(__uint_as_float(v[4 * q]), __uint_as_float(v[4 * q + 1]),
                                          __uint_as_float(v[4 * q + 2]), __uint_as_float(v[4 * q + 3])));
          }
        }
        sm100::tc_fence_before();
        __syncwarp();
        if (lane == 0) release_acc(acc);  // TMEM buffer free
        __threadfence();
        asm volatile("bar.sync 1, %0;" ::"n"(32 * kEpiWarps));
        if (warp == 4 && lane == 0) {
          const int old = atomicAdd(p.counters + t_sk, 1);
          const int fin = old == n_parts - 1;
          if (fin) p.counters[t_sk] = 0;  // ready for the next launch on this stream
          *sk_finisher = fin;
        }
        asm volatile("bar.sync 1, %0;" ::"n"(32 * kEpiWarps));
        if (*sk_finisher && p.sk_debug != 2) {
          __threadfence();
          const float* parts[kMaxParts];
#pragma unroll
          for (int k = 0; k < kMaxParts; ++k) parts[k] = k < n_parts ? part_ptr(k) : nullptr;
          if constexpr (TMA_OUT)
            epilogue_tile_tma<BN, EPI, true, kDeep>(p, &tmC, &tmR, smem_epi + (warp - 4) * kNB * C::kEpiBuf,
                                             rbar + kNB * (warp - 4), rphase, ec, t_row, m0, n0, quad, half,
                                             lane, parts, n_parts);
        }
        asm volatile("bar.sync 1, %0;" ::"n"(32 * kEpiWarps));  // sk_finisher reuse
        continue;
      }
      if constexpr (TMA_OUT) {
        constexpr bool kRes = EPI == static_cast<int>(Epi::Residual);
        if constexpr (kRes)
          prefetch_residual<BN, EPI, kDeep>(&tmR, smem_epi + (warp - 4) * kNB * C::kEpiBuf, rbar + kNB * (warp - 4), ec,
                                     m0, n0, quad, half, lane);
        if constexpr (kRopeStage) {
          // stage this tile's table rows + bias while its MMAs run (the
          // previous tile's epilogue has finished reading them)
          asm volatile("bar.sync 2, %0;" ::"n"(32 * kEpiWarps));
          if (warp == 4 && lane == 0) {
            sm100::mbar_expect_tx(tbar, static_cast<std::uint32_t>(p.rope_hd) * 4 * kBM);
            for (int b = 0; b < p.rope_hd / 32; ++b)
              sm100::tma_load_2d(rope_smem + b * (kBM * 128), &tmR, tbar, b * 32, m0);
          }
          const int t = static_cast<int>(threadIdx.x) - 128;
          if (t < BN) {
            bf16 bv = __float2bfloat16_rn(0.f);
            if (p.bias != nullptr && n0 + t < p.N) bv = p.bias[n0 + t];
            reinterpret_cast<bf16*>(rope_smem + kRopeTableBytes)[t] = bv;
          }
          asm volatile("bar.sync 2, %0;" ::"n"(32 * kEpiWarps));
        }
        sm100::mbar_wait(&tfull[acc], acc_phase);
        sm100::tc_fence_after();
        if constexpr (kRopeStage) {
          sm100::mbar_wait(tbar, tphase);
          tphase ^= 1;
        }
        const float* const no_parts[kMaxParts] = {};
        epilogue_tile_tma<BN, EPI, false, kDeep>(p, &tmC, &tmR, smem_epi + (warp - 4) * kNB * C::kEpiBuf,
                                   rbar + kNB * (warp - 4), rphase, ec, t_row, m0, n0, quad, half,
                                   lane, no_parts, 0, kRes, kRopeStage ? rope_smem : nullptr);
      } else {
        sm100::mbar_wait(&tfull[acc], acc_phase);
        sm100::tc_fence_after();
        const int row = m0 + quad * 32 + lane;
        constexpr int kCh = BN / 32;
        const int c0 = half == 0 ? 0 : (kCh + 1) / 2, c1 = half == 0 ? (kCh + 1) / 2 : kCh;
        const float rs = row_scale(p, row);
        float ss = 0.f;
#pragma unroll 1
        for (int c = 32 * c0; c < 32 * c1; c += 32) {
          std::uint32_t v[32];
          sm100::tmem_ld_32x32b_x32(t_row + static_cast<std::uint32_t>(c), v);
          sm100::tmem_ld_wait();
          if (row < M && n0 + c < p.N) epilogue_chunk<EPI>(p, row, n0 + c, v, rs, ss);
        }
        if (EPI == static_cast<int>(Epi::Residual) && p.ss_out != nullptr && row < M && c0 < c1)
          ss_accumulate(p, row, ss);
      }
      sm100::tc_fence_before();
      __syncwarp();
      if (lane == 0) release_acc(acc);
    }
    if constexpr (TMA_OUT) {
      if (lane == 0) sm100::bulk_wait<0>();  // stores complete before smem is released
      __syncwarp();
    }
  }
  if constexpr (CG == 2) sm100::cluster_sync();  // peer done with our smem / TMEM / barriers
  else __syncthreads();
  if (warp == 2) {
    sm100::tc_fence_after();
    if constexpr (CG == 2) sm100::tmem_dealloc_cg2(tmem_base, C::kTmemCols);
    else sm100::tmem_dealloc(tmem_base, C::kTmemCols);
  }
}

// ---- host side: tensor maps --------------------------------------------------
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

// 2D row-major matrix [rows, cols] (row stride ld elements), SW128 tiles of
// [box_rows, box_cols]; cached per (pointer, shape, box).
CUtensorMap make_map(const void* base, bool f32, int rows, int cols, int ld, int box_cols,
                     int box_rows) {
  // Swizzle span = box row width: 128 B (SW128) or 64 B (SW64, 32 bf16 columns).
  const bool sw64 = box_cols * (f32 ? 4 : 2) == 64;
  struct Key {
    const void* base;
    int rows, cols, ld, bc, br;
    bool f32;
    bool operator==(const Key& o) const {
      return base == o.base && rows == o.rows && cols == o.cols && ld == o.ld && bc == o.bc &&
             br == o.br && f32 == o.f32;
    }
  };
  struct KeyHash {
    std::size_t operator()(const Key& x) const {
      std::size_t h = reinterpret_cast<std::uintptr_t>(x.base);
      for (int v : {x.rows, x.cols, x.ld, x.bc, x.br, static_cast<int>(x.f32)})
        h = h * 1000003u ^ static_cast<std::size_t>(v);
      return h;
    }
  };
  static std::mutex mu;
  static std::unordered_map<Key, CUtensorMap, KeyHash> cache;
  const Key key{base, rows, cols, ld, box_cols, box_rows, f32};
  {
    std::lock_guard<std::mutex> g(mu);
    const auto it = cache.find(key);
    if (it != cache.end()) return it->second;
  }
  CUtensorMap tm;
  std::memset(&tm, 0, sizeof tm);
  const int esize = f32 ? 4 : 2;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * esize};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(box_cols), static_cast<cuuint32_t>(box_rows)};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode_fn()(
      &tm, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
      const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
      sw64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw DeviceError(RS_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(r) +
                                       ") rows=" + std::to_string(rows) + " cols=" +
                                       std::to_string(cols) + " ld=" + std::to_string(ld));
  std::lock_guard<std::mutex> g(mu);
  if (cache.size() > 4096) cache.clear();
  cache.emplace(key, tm);
  return tm;
}

// Stream-K workspace of one stream (GEMMs on a stream are serialised, so one
// workspace per stream suffices): 2 partial slots per CTA + tile counters.
// Stream-ordered allocation from the device pool (no host synchronisation on
// the launch path); released with the stream (gemm_release_stream).
struct SkWorkspace {
  float* ws = nullptr;
  int* counters = nullptr;
};
constexpr std::size_t kSkWsBytes = 64ull << 20;
std::mutex& sk_mutex() {
  static std::mutex mu;
  return mu;
}
std::unordered_map<cudaStream_t, SkWorkspace>& sk_all() {
  static std::unordered_map<cudaStream_t, SkWorkspace> all;
  return all;
}
SkWorkspace& sk_workspace(cudaStream_t st) {
  std::lock_guard<std::mutex> g(sk_mutex());
  SkWorkspace& w = sk_all()[st];
  if (w.ws == nullptr) {
    RS_CUDA_CHECK(cudaMallocAsync(reinterpret_cast<void**>(&w.ws), kSkWsBytes, st));
    RS_CUDA_CHECK(cudaMallocAsync(reinterpret_cast<void**>(&w.counters), sizeof(int) * kNumSMs, st));
    RS_CUDA_CHECK(cudaMemsetAsync(w.counters, 0, sizeof(int) * kNumSMs, st));
  }
  return w;
}

bool streamk_enabled() {
  static const bool on = [] {
    const char* v = std::getenv("RS_GEMM_STREAMK");
    return v == nullptr || v[0] != '0';
  }();
  return on;
}

// Split-K plan of a single-CTA GEMM (tiles of 128 x bn, num_kb k-blocks).
//  * tail: the last, partial wave of whole tiles (R tiles) costs one full
//    tile time; splitting each of those tiles into S k ranges turns it into
//    ceil(R*S / 148) rounds of 1/S tile. Long-K GEMMs only (>= 48 k-blocks):
//    the fp32 partials' round trip must stay small next to the saved tail.
//  * small grid (tiles <= 74, e.g. the 128-token first chunk): every tile is
//    split, so the weight stream (the bound at small M) is read by ~148 SMs.
// cost = tile-times the launch takes (whole tiles = 1 each).
struct SplitPlan {
  int sk_tiles = 0, splits = 1;
  double cost = 0;
};
// cg = 2: pair tiles (256 x bn) on 74 cluster slots; each CTA of a pair keeps
// its own 128-row partials / counter.
SplitPlan plan_split(int tiles, int num_kb, int bn, int cg = 1, bool small_m = false) {
  SplitPlan best;
  const int slots = kNumSMs / cg;
  const int rem = tiles % slots;
  const int full = tiles / slots;
  best.cost = full + (rem > 0 ? 1.0 : 0.0);
  // small grids split K from RS_GEMM_SMALL_MIN_KB k-blocks (r1, strided partial
  // layout: at K = 3584 the partials' round trip ate the gain; K = 18944 won 30%).
  // r2, coalesced partials: the <= 256-row QKV and O projections of the first /
  // last prefill chunk gain 17.5 -> 14.5 / 18.1 -> 16.3 us when split from 32
  // k-blocks (profiles/r02_gemm_smallm.txt); other shapes keep the r1 threshold.
  static const char* const min_kb_env = std::getenv("RS_GEMM_SMALL_MIN_KB");  // A/B: one threshold for all
  const int small_min_kb = min_kb_env != nullptr ? std::atoi(min_kb_env) : (small_m ? 32 : 128);
  const bool small = tiles <= slots / 2 && num_kb >= small_min_kb;
  const bool tail = tiles > slots && rem > 0 && num_kb >= 48;
  // Pair tiles: measured slower with split tails at every cfg2 shape (both
  // CTAs' fp32 partials round-trip), so they run whole tiles only; the kernel
  // path is kept and tested (RS_GEMM_PAIR_SPLIT=1).
  if (cg == 2 && !small_m) {  // (<= 256-row launches: pair split tails measured faster, above)
    const char* e = std::getenv("RS_GEMM_PAIR_SPLIT");
    if (e == nullptr || e[0] != '1') return best;
  }
  if (!small && !tail) return best;
  static const int force_sp = [] {  // A/B only: fixed split count for small grids
    const char* e = std::getenv("RS_GEMM_FORCE_SPLITS");
    return e != nullptr ? std::atoi(e) : 0;
  }();
  if (small && force_sp >= 2 && force_sp <= kMaxParts && num_kb / force_sp >= 4 &&
      static_cast<std::size_t>(rem) * cg * force_sp * kBM * bn * sizeof(float) <= kSkWsBytes) {
    best.sk_tiles = rem;
    best.splits = force_sp;
    best.cost = static_cast<double>(ceil_div(rem * force_sp, slots)) / force_sp;
    return best;
  }
  const int min_kb = 16;
  for (int sp = 2; sp <= kMaxParts && num_kb / sp >= min_kb; ++sp) {
    if (static_cast<std::size_t>(rem) * cg * sp * kBM * bn * sizeof(float) > kSkWsBytes) break;
    if (rem * cg > kNumSMs) break;  // tile counters
    // partial round trip: ~4% of a tile per extra split
    const double tail_c = static_cast<double>(ceil_div(rem * sp, slots)) / sp + 0.04 * (sp - 1);
    if (tail_c <= 0.85 && full + tail_c < best.cost - 1e-9) {
      best.cost = full + tail_c;
      best.sk_tiles = rem;
      best.splits = sp;
    }
  }
  return best;
}

template <int BN, int EPI, bool TMA_OUT, int CG>
void launch(const GemmArgs& a, cudaStream_t stream) {
  using C = Cfg<BN, TMA_OUT, CG, TMA_OUT && EPI == static_cast<int>(Epi::QkvRope), epi_bufs<BN, EPI, TMA_OUT>()>;
  auto* kernel = gemm_tcgen05_kernel<BN, EPI, TMA_OUT, CG>;
  static bool attr_set = false;
  if (!attr_set) {
    RS_CUDA_CHECK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem));
    attr_set = true;
  }
  const CUtensorMap tmA = make_map(a.A, false, a.M, a.K, a.lda, kBK, kBM);
  const CUtensorMap tmB = make_map(a.B, false, a.N, a.K, a.ldb, kBK, C::kSubRows);
  CUtensorMap tmC = tmA, tmR = tmA;  // unused placeholders unless TMA_OUT
  if constexpr (TMA_OUT) {
    constexpr bool f32 = EPI == static_cast<int>(Epi::StoreF32);
    const int out_cols = EPI == static_cast<int>(Epi::SwiGLU) ? a.N / 2 : a.N;
    tmC = make_map(a.C, f32, a.M, out_cols, a.ldc, 32, 32);
    if constexpr (EPI == static_cast<int>(Epi::Residual))
      tmR = make_map(a.residual, false, a.M, a.N, a.ldr, 32, 32);
    if constexpr (EPI == static_cast<int>(Epi::QkvRope)) {
      // the chunk's M-RoPE (cos, sin) table [M, hd/2] float2 = [M, hd] fp32, boxes of 32 floats x 128 rows
      if (a.rope_hd % 32 != 0 || a.rope_hd > 128)
        throw DeviceError(RS_ERR_CUDA, "gemm: QkvRope staging needs head_dim % 32 == 0, <= 128");
      tmR = make_map(a.rope_table, true, a.M, a.rope_hd, a.rope_hd, 32, kBM);
    }
  }
  GemmParams p{a.C, a.ldc, a.bias, a.residual, a.ldr, a.row_map, a.M, a.N, a.K, a.M_dev,
               0, 0, 0, nullptr, nullptr, 0,
               a.ss_in, a.ss_inv_dim, a.ss_eps, a.ss_out, a.ss_clear, a.ss_clear_n,
               static_cast<const ChunkRowInfo*>(a.rope_rows), a.rope_table, a.page_tables, a.k_cache, a.v_cache,
               a.rope_hq, a.rope_hkv, a.rope_hd, a.page_size};
  if (const char* dbg = std::getenv("RS_GEMM_SK_DEBUG")) p.sk_debug = std::atoi(dbg);
  static const int early_b = [] {
    const char* e = std::getenv("RS_GEMM_EARLY_B");
    return e != nullptr && e[0] == '0' ? 0 : 1;
  }();
  p.early_b = early_b && a.b_stable ? 1 : 0;
  const int tiles = ceil_div(a.M, kBM * CG) * ceil_div(a.N, BN);
  int grid = CG * (tiles < kNumSMs / CG ? tiles : kNumSMs / CG);
  // Tail split-K: the last, partial wave of whole tiles (R tiles) costs one
  // full tile time. Splitting each of those tiles into S k ranges turns it
  // into ceil(R*S / 148) rounds of 1/S tile; pick the S (<= kMaxParts, k
  // ranges >= 16 blocks) minimising that, if it saves >= 15% of the tail.
  // Long-K GEMMs only: the fp32 partials' round trip must stay small next to
  // the saved tail.
  if (TMA_OUT && a.M_dev == nullptr && streamk_enabled()) {
    const SplitPlan sp = plan_split(tiles, ceil_div(a.K, kBK), BN, CG, a.M <= 2 * kBM);
    if (sp.splits > 1) {
      SkWorkspace& w = sk_workspace(stream);
      p.dp_tiles = tiles - sp.sk_tiles;
      p.sk_tiles = sp.sk_tiles;
      p.sk_splits = sp.splits;
      p.ws = w.ws;
      p.counters = w.counters;
      grid = CG * std::min(kNumSMs / CG, p.dp_tiles + sp.sk_tiles * sp.splits);
    }
  }
  launch_kernel(kernel, dim3(grid), dim3(kThreads), C::kSmem, stream, CG, tmA, tmB, tmC, tmR, p);
  RS_LAUNCH_CHECK();
  count_launch();
}

template <int BN, int CG>
void dispatch_epi(const GemmArgs& a, Epi epi, cudaStream_t s) {
  // Row-mapped outputs (scatter) keep the direct-store epilogue; everything
  // else goes through smem + TMA stores.
  const bool tma = a.row_map == nullptr && a.M_dev == nullptr;
  switch (epi) {
    case Epi::Store: return tma ? launch<BN, 0, true, CG>(a, s) : launch<BN, 0, false, CG>(a, s);
    case Epi::Residual: return tma ? launch<BN, 1, true, CG>(a, s) : launch<BN, 1, false, CG>(a, s);
    case Epi::SwiGLU:
      if constexpr (BN % 64 == 0)
        return tma ? launch<BN, 2, true, CG>(a, s) : launch<BN, 2, false, CG>(a, s);
      else
        return launch<BN, 2, false, CG>(a, s);
    case Epi::Gelu: return tma ? launch<BN, 3, true, CG>(a, s) : launch<BN, 3, false, CG>(a, s);
    case Epi::StoreF32: return launch<BN, 4, false, CG>(a, s);  // LM-head logits (row-mapped)
    case Epi::QkvRope:
      if constexpr (BN % 64 == 0 && BN <= 256) return launch<BN, 5, true, CG>(a, s);
      else throw DeviceError(RS_ERR_CUDA, "gemm: QkvRope needs whole-head tiles");
  }
}

// Tile shape with the least wave-quantised time. A wave of the persistent
// kernel costs ~BN (per-tile work at fixed BM and K): 148 single-CTA 128 x BN
// tiles per wave, or 74 pair tiles of 256 x BN, whose per-FLOP cost is lower
// (half the shared-memory operand traffic per SM). Calibrated on B200
// (scripts/gemm_sweep.py, profiles/r01_gemm_sweep_pair.txt): pairs gain ~15%
// on long K, ~7% on short K, and lose ~5-10% on short-K GEMMs of <= 2 waves
// (per-tile fixed costs dominate). Ties go to the wider tile (fewer A
// re-reads). RS_GEMM_CG=1/2 forces the CTA mode.
struct TileChoice {
  int bn, cg;
};
int cg_override() {
  static const int v = [] {
    const char* e = std::getenv("RS_GEMM_CG");
    return e != nullptr ? std::atoi(e) : 0;
  }();
  return v;
}
TileChoice pick_tile(int M, int N, int K, bool swiglu, int tile_multiple = 0, bool residual = false) {
  static constexpr int kCandidates[] = {256, 224, 192, 160, 128};
  const int num_kb = ceil_div(K, kBK);
  // first / last prefill chunks (M <= 256): few tiles, weight-streaming and
  // latency bound; measured fastest with the most 128 x 128 tiles (+ split-K
  // on long K) except SwiGLU (scripts/gemm_sweep.py --small-m)
  static const bool small_m_rule = [] {  // RS_GEMM_SMALLM=0: A/B
    const char* e = std::getenv("RS_GEMM_SMALLM");
    return e == nullptr || e[0] != '0';
  }();
  if (small_m_rule && M <= 2 * kBM && !swiglu && N % 128 == 0 && cg_override() == 0) {
    // 129-256 rows with long K (the last chunk's down projection): one 256 x 160
    // pair tile row with a split-K tail reads A once per 160 columns instead of
    // per 128 and B once, not twice (L2 -> SM traffic, not HBM, was the limit):
    // 49.3 -> 43.5 us (profiles/r02_gemm_smallm_sweep.txt)
    if (M > kBM && num_kb >= 128 && tile_multiple == 0) return {160, 2};
    return {128, 1};
  }
  TileChoice best{256, 1};
  double best_cost = -1;
  for (int cg = 1; cg <= 2; ++cg) {
    if (cg_override() != 0 && cg != cg_override()) continue;
    for (int bn : kCandidates) {
      if (swiglu && bn % 64 != 0) continue;  // 64-column gate/up chunks (TMA epilogue)
      if (tile_multiple > 0 && bn % tile_multiple != 0) continue;  // QkvRope: whole heads per tile
      const long tiles = static_cast<long>(ceil_div(M, kBM * cg)) * ceil_div(N, bn);
      const long slots = kNumSMs / cg;
      const long waves = (tiles + slots - 1) / slots;
      const double pair_gain = num_kb >= 32 ? 0.85 : (waves <= 2 ? 1.05 : 0.93);
      // long runs (>= 4 waves): narrow tiles are limited by the per-SM operand
      // feed (A + B bytes per MMA clock: 8192/bn + 32 for a pair CTA, + 64 for a
      // single CTA), above ~68 / ~80 B/clk measured (profiles/r02_gemm_ab.txt:
      // 8192x3840x1280 256x128 pairs 75 us vs 256x256 57 us)
      const double demand = 8192.0 / bn + (cg == 2 ? 32.0 : 64.0);
      const double feed = waves >= 4 ? std::max(1.0, demand / (cg == 2 ? 68.0 : 80.0)) : 1.0;
      const double cost = plan_split(static_cast<int>(tiles), num_kb, bn, cg).cost * bn *
                          (cg == 2 ? pair_gain : 1.0) * feed;
      if (best_cost < 0 || cost < best_cost - 1e-9) {
        best = {bn, cg};
        best_cost = cost;
      }
    }
  }
  // 256 x 320 pair tiles (one wave, one accumulator): twice the operand reuse
  // per SM of 256 x 160. Measured on B200 (scripts/gemm_probe.py --wide,
  // profiles/r02_gemm_wide.txt): ViT down 4096 x 1280 x 3424 35.9 -> 31.4 us;
  // neutral at short K with a residual epilogue (ViT O, K = 1280) and slower
  // past one wave (ViT QKV), so single-wave launches with long K or a plain
  // store (patch embed 4096 x 1280 x 1176: 21.6 -> 14.9 us in a same-process
  // A/B, profiles/r02_gemm_ab.txt). The 448 / 512 widths measured no better
  // than 224 / 256 on the LLM shapes and are left to force_bn.
  static const bool wide = [] {
    const char* e = std::getenv("RS_GEMM_WIDE");
    return e == nullptr || e[0] != '0';
  }();
  if (wide && !swiglu && tile_multiple == 0 && cg_override() != 1 && N % 320 == 0 && (num_kb >= 32 || !residual) &&
      static_cast<long>(ceil_div(M, 2 * kBM)) * (N / 320) <= kNumSMs / 2) {
    const double pair_gain = 0.85;
    if (320 * pair_gain * 0.9 < best_cost) best = {320, 2};
  }
  return best;
}

}  // namespace

void gemm(const GemmArgs& a, Epi epi, cudaStream_t stream, int force_bn) {
  HostPhase phase_("gemm");
  if (a.M <= 0 || a.N <= 0) return;
  if (a.K % 8 != 0 || a.N % 16 != 0 || a.lda % 8 != 0 || a.ldb % 8 != 0)
    throw DeviceError(RS_ERR_CUDA, "gemm: need K%8==0, N%16==0, lda/ldb%8==0 (K=" +
                                       std::to_string(a.K) + ", N=" + std::to_string(a.N) + ")");
  if (epi == Epi::SwiGLU && a.N % 32 != 0)
    throw DeviceError(RS_ERR_CUDA, "gemm: SwiGLU needs N%32==0");
  if (force_bn == 0 && a.M <= 8) {  // decode-sized: weight streaming on the CUDA cores
    const int tok = prof::begin(stream);
    if (gemv_small_m(a, epi, stream)) {
      prof::end(tok, stream, "gemv_small_m", 2.0 * a.M * a.N * a.K, 2.0 * a.N * a.K);
      return;
    }
  }
  // force_bn > 0: single-CTA tiles of that width; < 0: CTA-pair tiles of |force_bn|
  const TileChoice tc = force_bn > 0   ? TileChoice{force_bn, 1}
                        : force_bn < 0 ? TileChoice{-force_bn, 2}
                                       : pick_tile(a.M, a.N, a.K, epi == Epi::SwiGLU,
                                                   epi == Epi::QkvRope ? a.rope_hd : 0, epi == Epi::Residual);
  const int tok = prof::begin(stream);
  const int key = tc.bn * 4 + tc.cg;
  switch (key) {
    case 256 * 4 + 1: dispatch_epi<256, 1>(a, epi, stream); break;
    case 224 * 4 + 1: dispatch_epi<224, 1>(a, epi, stream); break;
    case 192 * 4 + 1: dispatch_epi<192, 1>(a, epi, stream); break;
    case 160 * 4 + 1: dispatch_epi<160, 1>(a, epi, stream); break;
    case 128 * 4 + 1: dispatch_epi<128, 1>(a, epi, stream); break;
    case 256 * 4 + 2: dispatch_epi<256, 2>(a, epi, stream); break;
    case 224 * 4 + 2: dispatch_epi<224, 2>(a, epi, stream); break;
    case 192 * 4 + 2: dispatch_epi<192, 2>(a, epi, stream); break;
    case 160 * 4 + 2: dispatch_epi<160, 2>(a, epi, stream); break;
    case 128 * 4 + 2: dispatch_epi<128, 2>(a, epi, stream); break;
    case 320 * 4 + 2: dispatch_epi<320, 2>(a, epi, stream); break;
    case 448 * 4 + 2: dispatch_epi<448, 2>(a, epi, stream); break;
    case 512 * 4 + 2: dispatch_epi<512, 2>(a, epi, stream); break;
    default:
      throw DeviceError(RS_ERR_CUDA, "gemm: unsupported tile " + std::to_string(tc.bn) + " x cg" +
                                         std::to_string(tc.cg));
  }
  const double m = a.M, n = a.N, k = a.K;
  const double out_bytes = epi == Epi::StoreF32 ? 4.0 : (epi == Epi::SwiGLU ? 1.0 : 2.0);
  if (tok < 0) return;
  // per-shape class "gemm_tcgen05|M|N|K|epi|BN|CG" (the bench groups on the prefix)
  char label[96];
  std::snprintf(label, sizeof label, "gemm_tcgen05|%d|%d|%d|%d|%d|%d", a.M, a.N, a.K,
                static_cast<int>(epi), tc.bn, tc.cg);
  prof::end(tok, stream, label, 2.0 * m * n * k,
            2.0 * (m * k + n * k) + out_bytes * m * n + (epi == Epi::Residual ? 2.0 * m * n : 0.0));
}

void gemm_release_stream(cudaStream_t st) {
  std::lock_guard<std::mutex> g(sk_mutex());
  auto it = sk_all().find(st);
  if (it == sk_all().end()) return;
  if (it->second.ws) cudaFreeAsync(it->second.ws, st);
  if (it->second.counters) cudaFreeAsync(it->second.counters, st);
  sk_all().erase(it);
}

}  // namespace rserve
