// rserve-b200 — ViT window attention on tcgen05 / TMEM with TMA (sm_100a).
//
// The 28 window layers of the Qwen2.5-VL vision tower attend inside 8x8-patch
// windows (<= 64 keys). A work unit is one (tile, head): a tile is a run of
// WHOLE consecutive windows of <= 128 packed rows (two 64-patch windows in the
// common case), so a single 128 x 128 S tile holds every key a row can see and
// the softmax is exact in one pass (block-diagonal mask, no online rescale).
//
// Operands are read straight from the QKV GEMM's output [P, 3 H hd] (no
// head padding / transpose pass):
//   * Q, K  K-major: dims 0..63 by a [128 rows x 64] SW128 TMA box, the 16-dim
//     tail of hd 80 by a [128 x 16] SW32 box; S = Q K^T is 4 + 1 MMAs (K = 16).
//   * V     MN-major (rows = keys, dims contiguous) from the same two boxes:
//     O = P V is 8 x (N = 64 + N = 16) MMAs with the B operand MN-major, so V
//     needs no transpose.
//   * 2D RoPE is applied to Q and K in shared memory (swizzle-aware) by two
//     prep warps between the TMA arrival and the S MMA.
//   * P (bf16) goes back into S's TMEM columns and is the A operand of the
//     TS-MMA for O.
// Warp roles (256 threads, one CTA per SM, persistent over the units):
//   warp 0 TMA producer (3-stage smem ring), warp 1 MMA issuer, warps 2-3
//   RoPE prep, warps 4-7 softmax + epilogue (one query row per thread; warp w
//   owns TMEM lanes 32 (w % 4)). TMEM: S/P and O double-buffered (512 cols).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <mutex>
#include <unordered_map>

#include "attention.cuh"
#include "common.cuh"
#include "sm100.cuh"

namespace rserve {
namespace {

constexpr int kWinThreads = 256;
constexpr int kWinStages = 3;

template <int HD>
struct WinCfg {
  static_assert(HD == 64 || HD == 80, "window attention: head_dim 64 or 80");
  static constexpr int kTail = HD - 64;                    // 16 (hd 80) or 0
  static constexpr int kMainBytes = 128 * 128;             // [128 rows x 64] bf16, SW128
  static constexpr int kTailBytes = 128 * kTail * 2;       // [128 rows x 16] bf16, SW32
  // stage: Qm Km Vm (1024-aligned) then Qt Kt Vt (256-aligned)
  static constexpr int kStageBytes = 3 * kMainBytes + 3 * kTailBytes;
  static constexpr int kSmem = kWinStages * kStageBytes + 1024 + 256;
  static constexpr int kChunkPairs = HD / 16;              // 16-B chunk pairs (i, i + hd/2) per row
};
static_assert(WinCfg<80>::kStageBytes % 1024 == 0, "stage alignment");

// TMEM columns: S/P of buffer b at 128 b, O of buffer b at 256 + 128 b.
constexpr std::uint32_t kTmemO = 256;

struct WinParams {
  const AttnBlock* tiles;   // q_row0 / q_rows of each tile (whole windows)
  const int* cu_window;     // window boundaries over the packed rows
  int n_win;
  int n_units;              // tiles * heads
  int heads;
  int rows_total;
  const float2* rope;       // [rows_total, hd/2] (cos, sin)
  float scale_log2;
  bf16* out;
  int ld_out;
};

__device__ __forceinline__ std::uint64_t make_desc(std::uint32_t saddr, std::uint32_t lbo, std::uint32_t sbo,
                                                   std::uint32_t layout) {
  std::uint64_t d = 0;
  d |= static_cast<std::uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<std::uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
  d |= static_cast<std::uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
  d |= static_cast<std::uint64_t>(1) << 46;            // descriptor version (sm_100)
  d |= static_cast<std::uint64_t>(layout) << 61;       // 2 = SW128, 6 = SW32
  return d;
}
constexpr std::uint32_t kLayoutSW128 = 2, kLayoutSW32 = 6;

__device__ __forceinline__ void tmem_ld_32x32b_x16(std::uint32_t taddr, std::uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
        "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}

__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Byte offset of 16-B chunk `c` (dims 8c..8c+7) of row r inside a stage's
// Q / K region: chunks 0-7 in the SW128 main tile, 8-9 in the SW32 tail.
template <int HD>
__device__ __forceinline__ std::uint32_t chunk_off(int r, int c, std::uint32_t main_off, std::uint32_t tail_off) {
  if (c < 8) return main_off + static_cast<std::uint32_t>(r * 128 + ((c ^ (r & 7)) << 4));
  return tail_off + static_cast<std::uint32_t>(r * 32 + (((c - 8) ^ ((r >> 2) & 1)) << 4));
}

template <int HD>
__global__ void __launch_bounds__(kWinThreads, 1)
    win_attn_tc_kernel(const __grid_constant__ CUtensorMap tmMain, const __grid_constant__ CUtensorMap tmTail,
                       const __grid_constant__ WinParams p) {
  using C = WinCfg<HD>;
  extern __shared__ __align__(1024) std::uint8_t smem_raw[];
  std::uint8_t* base = reinterpret_cast<std::uint8_t*>((reinterpret_cast<std::uintptr_t>(smem_raw) + 1023) & ~std::uintptr_t(1023));
  auto* bars = reinterpret_cast<std::uint64_t*>(base + kWinStages * C::kStageBytes);
  std::uint64_t* full = bars;              // [3] TMA bytes
  std::uint64_t* prepped = bars + 3;       // [3] 64 prep threads
  std::uint64_t* empty = bars + 6;         // [3] MMA commit after O
  std::uint64_t* s_full = bars + 9;        // [2] MMA commit
  std::uint64_t* p_full = bars + 11;       // [2] 128 softmax threads
  std::uint64_t* o_full = bars + 13;       // [2] MMA commit
  std::uint64_t* tmem_free = bars + 15;    // [2] 128 epilogue threads
  auto* tmem_slot = reinterpret_cast<std::uint32_t*>(bars + 17);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 3; ++i) {
      sm100::mbar_init(&full[i], 1);
      sm100::mbar_init(&prepped[i], 64);
      sm100::mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      sm100::mbar_init(&s_full[i], 1);
      sm100::mbar_init(&p_full[i], 128);
      sm100::mbar_init(&o_full[i], 1);
      sm100::mbar_init(&tmem_free[i], 128);
    }
    sm100::fence_mbar_init();
    sm100::tma_prefetch_desc(&tmMain);
    if (C::kTail) sm100::tma_prefetch_desc(&tmTail);
  }
  if (warp == 0) sm100::tmem_alloc(tmem_slot, 512);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const std::uint32_t tmem = *tmem_slot;
  pdl_wait();
  pdl_launch_dependents();
  const int H = p.heads;
  const int qcol = 0, kcol = H * HD, vcol = 2 * H * HD;
  const std::uint32_t sbase = sm100::smem_u32(base);
  auto stage_off = [&](int s) { return static_cast<std::uint32_t>(s * C::kStageBytes); };
  constexpr std::uint32_t kQm = 0, kKm = C::kMainBytes, kVm = 2 * C::kMainBytes;
  constexpr std::uint32_t kQt = 3 * C::kMainBytes, kKt = kQt + C::kTailBytes, kVt = kQt + 2 * C::kTailBytes;

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (sm100::elect_one()) {
      int it = 0;
      for (int u = blockIdx.x; u < p.n_units; u += gridDim.x, ++it) {
        const int s = it % kWinStages;
        const AttnBlock t = p.tiles[u / H];
        const int h = u % H;
        sm100::mbar_wait(&empty[s], ((it / kWinStages) & 1) ^ 1);
        sm100::mbar_expect_tx(&full[s], C::kStageBytes);
        std::uint8_t* st = base + stage_off(s);
        sm100::tma_load_2d(st + kQm, &tmMain, &full[s], qcol + h * HD, t.q_row0);
        sm100::tma_load_2d(st + kKm, &tmMain, &full[s], kcol + h * HD, t.q_row0);
        sm100::tma_load_2d(st + kVm, &tmMain, &full[s], vcol + h * HD, t.q_row0);
        if constexpr (C::kTail > 0) {
          sm100::tma_load_2d(st + kQt, &tmTail, &full[s], qcol + h * HD + 64, t.q_row0);
          sm100::tma_load_2d(st + kKt, &tmTail, &full[s], kcol + h * HD + 64, t.q_row0);
          sm100::tma_load_2d(st + kVt, &tmTail, &full[s], vcol + h * HD + 64, t.q_row0);
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    if (sm100::elect_one()) {
      constexpr std::uint32_t idesc_s = sm100::idesc_bf16_f32(128, 128);
      constexpr std::uint32_t kMnB = 1u << 16;  // B operand MN-major (V rows = keys)
      constexpr std::uint32_t idesc_o64 = sm100::idesc_bf16_f32(128, 64) | kMnB;
      constexpr std::uint32_t idesc_o16 = sm100::idesc_bf16_f32(128, 16) | kMnB;
      auto issue_pv = [&](int j) {
        const int s = j % kWinStages, b = j & 1;
        sm100::mbar_wait(&p_full[b], (j >> 1) & 1);
        sm100::tc_fence_after();
        const std::uint32_t so = sbase + stage_off(s);
        const std::uint64_t vm = make_desc(so + kVm, 16384, 1024, kLayoutSW128);
        const std::uint32_t o = tmem + kTmemO + 128 * b, pa = tmem + 128 * b;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {  // 16 keys per MMA
          sm100::umma_bf16_ts(o, pa + 8 * kk, vm + (2048 >> 4) * kk, idesc_o64, kk != 0 ? 1u : 0u);
          if constexpr (C::kTail > 0) {
            const std::uint64_t vt = make_desc(so + kVt, 4096, 256, kLayoutSW32);
            sm100::umma_bf16_ts(o + 64, pa + 8 * kk, vt + (512 >> 4) * kk, idesc_o16, kk != 0 ? 1u : 0u);
          }
        }
        sm100::umma_commit(&o_full[b]);
        sm100::umma_commit(&empty[s]);
      };
      int it = 0;
      for (int u = blockIdx.x; u < p.n_units; u += gridDim.x, ++it) {
        const int s = it % kWinStages, b = it & 1;
        sm100::mbar_wait(&prepped[s], (it / kWinStages) & 1);
        sm100::mbar_wait(&tmem_free[b], ((it >> 1) & 1) ^ 1);
        sm100::tc_fence_after();
        const std::uint32_t so = sbase + stage_off(s);
        const std::uint64_t qd = sm100::sw128_kmajor_desc(so + kQm);
        const std::uint64_t kd = sm100::sw128_kmajor_desc(so + kKm);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          sm100::umma_bf16(tmem + 128 * b, qd + 2 * kk, kd + 2 * kk, idesc_s, kk != 0 ? 1u : 0u);
        if constexpr (C::kTail > 0)
          sm100::umma_bf16(tmem + 128 * b, make_desc(so + kQt, 16, 256, kLayoutSW32),
                           make_desc(so + kKt, 16, 256, kLayoutSW32), idesc_s, 1u);
        sm100::umma_commit(&s_full[b]);
        if (it > 0) issue_pv(it - 1);
      }
      if (it > 0) issue_pv(it - 1);
    }
  } else if (warp < 4) {
    // ---------------- RoPE prep (64 threads) ----------------
    const int t64 = threadIdx.x - 64;
    int it = 0;
    for (int u = blockIdx.x; u < p.n_units; u += gridDim.x, ++it) {
      const int s = it % kWinStages;
      const AttnBlock t = p.tiles[u / H];
      sm100::mbar_wait(&full[s], (it / kWinStages) & 1);
      std::uint8_t* st = base + stage_off(s);
      const float2* tab = p.rope + static_cast<std::int64_t>(t.q_row0) * (HD / 2);
      for (int task = t64; task < t.q_rows * C::kChunkPairs; task += 64) {
        const int r = task / C::kChunkPairs, c = task % C::kChunkPairs;
        const float4* cs = reinterpret_cast<const float4*>(tab + r * (HD / 2) + 8 * c);  // 8 x (cos, sin)
        float2 cz[8];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float4 v = __ldg(cs + i);
          cz[2 * i] = make_float2(v.x, v.y);
          cz[2 * i + 1] = make_float2(v.z, v.w);
        }
#pragma unroll
        for (int which = 0; which < 2; ++which) {  // Q, K
          const std::uint32_t mo = which == 0 ? kQm : kKm, to = which == 0 ? kQt : kKt;
          uint4* pa = reinterpret_cast<uint4*>(st + chunk_off<HD>(r, c, mo, to));
          uint4* pb = reinterpret_cast<uint4*>(st + chunk_off<HD>(r, c + C::kChunkPairs, mo, to));
          uint4 a = *pa, bv = *pb;
          std::uint32_t* aw = reinterpret_cast<std::uint32_t*>(&a);
          std::uint32_t* bw = reinterpret_cast<std::uint32_t*>(&bv);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float2 x = unpack_bf16x2(aw[i]), y = unpack_bf16x2(bw[i]);
            const float2 c0 = cz[2 * i], c1 = cz[2 * i + 1];
            aw[i] = pack_bf16x2(x.x * c0.x - y.x * c0.y, x.y * c1.x - y.y * c1.y);
            bw[i] = pack_bf16x2(y.x * c0.x + x.x * c0.y, y.y * c1.x + x.y * c1.y);
          }
          *pa = a;
          *pb = bv;
        }
      }
      sm100::fence_proxy_async_smem();  // generic-proxy writes -> visible to the MMA (async proxy)
      sm100::mbar_arrive(&prepped[s]);
    }
  } else {
    // ---------------- softmax + epilogue (one query row per thread) ----------------
    const int q = warp & 3;
    const int r = q * 32 + lane;
    const std::uint32_t lane_off = static_cast<std::uint32_t>(q * 32) << 16;
    int it = 0;
    for (int u = blockIdx.x; u < p.n_units; u += gridDim.x, ++it) {
      const int b = it & 1;
      const AttnBlock t = p.tiles[u / H];
      const int h = u % H;
      // this row's window [lo, hi) as tile columns
      int c_lo = 0, c_hi = 0;
      if (r < t.q_rows) {
        const int row = t.q_row0 + r;
        int a = 0, e = p.n_win;  // largest w with cu[w] <= row
        while (e - a > 1) {
          const int mid = (a + e) >> 1;
          if (p.cu_window[mid] <= row) a = mid;
          else e = mid;
        }
        c_lo = p.cu_window[a] - t.q_row0;
        c_hi = p.cu_window[a + 1] - t.q_row0;
      }
      sm100::mbar_wait(&s_full[b], (it >> 1) & 1);
      sm100::tc_fence_after();
      std::uint32_t sv[128];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        std::uint32_t(&v)[32] = *reinterpret_cast<std::uint32_t(*)[32]>(&sv[32 * c]);
        sm100::tmem_ld_32x32b_x32(tmem + lane_off + 128 * b + 32 * c, v);
      }
      sm100::tmem_ld_wait();
      float mx8[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) mx8[i] = -INFINITY;
#pragma unroll
      for (int c = 0; c < 128; ++c) {
        const bool vis = c >= c_lo && c < c_hi;
        const float v = vis ? __uint_as_float(sv[c]) : -INFINITY;
        sv[c] = __float_as_uint(v);
        mx8[c & 7] = fmaxf(mx8[c & 7], v);
      }
      const float mx = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                             fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7])));
      const float mneg = mx == -INFINITY ? 0.f : -mx * p.scale_log2;
      float rs8[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        std::uint32_t packed[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const float p0 = fast_exp2(fmaf(__uint_as_float(sv[64 * c + 2 * i]), p.scale_log2, mneg));
          const float p1 = fast_exp2(fmaf(__uint_as_float(sv[64 * c + 2 * i + 1]), p.scale_log2, mneg));
          rs8[(2 * i) & 7] += p0;
          rs8[(2 * i + 1) & 7] += p1;
          packed[i] = pack_bf16x2(p0, p1);
        }
        sm100::tmem_st_32x32b_x32(tmem + lane_off + 128 * b + 32 * c, packed);
      }
      sm100::tmem_st_wait();
      sm100::tc_fence_before();
      sm100::mbar_arrive(&p_full[b]);
      const float l = ((rs8[0] + rs8[1]) + (rs8[2] + rs8[3])) + ((rs8[4] + rs8[5]) + (rs8[6] + rs8[7]));
      // epilogue: O row -> bf16 -> global
      sm100::mbar_wait(&o_full[b], (it >> 1) & 1);
      sm100::tc_fence_after();
      std::uint32_t ov[HD];
      {
        std::uint32_t(&v0)[32] = *reinterpret_cast<std::uint32_t(*)[32]>(&ov[0]);
        std::uint32_t(&v1)[32] = *reinterpret_cast<std::uint32_t(*)[32]>(&ov[32]);
        sm100::tmem_ld_32x32b_x32(tmem + lane_off + kTmemO + 128 * b, v0);
        sm100::tmem_ld_32x32b_x32(tmem + lane_off + kTmemO + 128 * b + 32, v1);
        if constexpr (C::kTail > 0) {
          std::uint32_t(&v2)[16] = *reinterpret_cast<std::uint32_t(*)[16]>(&ov[64]);
          tmem_ld_32x32b_x16(tmem + lane_off + kTmemO + 128 * b + 64, v2);
        }
      }
      sm100::tmem_ld_wait();
      sm100::tc_fence_before();
      sm100::mbar_arrive(&tmem_free[b]);
      if (r < t.q_rows) {
        const float inv = l > 0.f ? 1.f / l : 0.f;
        bf16* orow = p.out + static_cast<std::int64_t>(t.q_row0 + r) * p.ld_out + h * HD;
#pragma unroll
        for (int c = 0; c < HD / 8; ++c) {
          uint4 w;
          w.x = pack_bf16x2(__uint_as_float(ov[8 * c + 0]) * inv, __uint_as_float(ov[8 * c + 1]) * inv);
          w.y = pack_bf16x2(__uint_as_float(ov[8 * c + 2]) * inv, __uint_as_float(ov[8 * c + 3]) * inv);
          w.z = pack_bf16x2(__uint_as_float(ov[8 * c + 4]) * inv, __uint_as_float(ov[8 * c + 5]) * inv);
          w.w = pack_bf16x2(__uint_as_float(ov[8 * c + 6]) * inv, __uint_as_float(ov[8 * c + 7]) * inv);
          *reinterpret_cast<uint4*>(orow + 8 * c) = w;
        }
      }
    }
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 0) sm100::tmem_dealloc(tmem, 512);
}

// ---- host ----------------------------------------------------------------------------------
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

// bf16 [rows, cols] row-major (stride ld elements), box [128 rows, box_cols].
CUtensorMap qkv_map(const void* base, int rows, int cols, int ld, int box_cols, CUtensorMapSwizzle sw) {
  CUtensorMap tm;
  std::memset(&tm, 0, sizeof tm);
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 2};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(box_cols), 128u};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode_fn()(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims,
                                 strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw DeviceError(RS_ERR_CUDA, "window attention tensor map failed (" + std::to_string(r) + ")");
  return tm;
}

struct MapPair {
  CUtensorMap main, tail;
};

const MapPair& cached_maps(const void* base, int rows, int cols, int ld) {
  static std::mutex mu;
  static std::unordered_map<std::uint64_t, MapPair> cache;
  const std::uint64_t key = reinterpret_cast<std::uintptr_t>(base) ^ (static_cast<std::uint64_t>(rows) << 44) ^
                            (static_cast<std::uint64_t>(cols) << 32) ^ static_cast<std::uint64_t>(ld);
  std::lock_guard<std::mutex> g(mu);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  if (cache.size() > 1024) cache.clear();
  MapPair m{qkv_map(base, rows, cols, ld, 64, CU_TENSOR_MAP_SWIZZLE_128B),
            qkv_map(base, rows, cols, ld, 16, CU_TENSOR_MAP_SWIZZLE_32B)};
  return cache.emplace(key, m).first->second;
}

template <int HD>
void launch_win(const MapPair& m, const WinParams& p, double flops, cudaStream_t st) {
  static std::once_flag once;
  std::call_once(once, [] {
    RS_CUDA_CHECK(cudaFuncSetAttribute(win_attn_tc_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       WinCfg<HD>::kSmem));
  });
  const int grid = std::min(p.n_units, kNumSMs);
  const int tok = prof::begin(st);
  launch_kernel(win_attn_tc_kernel<HD>, dim3(grid), dim3(kWinThreads), WinCfg<HD>::kSmem, st, 1, m.main,
                m.tail, p);
  RS_LAUNCH_CHECK();
  prof::end(tok, st, "attn_vit_window_tc", flops, 0);
  count_launch();
}

}  // namespace

bool attention_window_tc_supported(int head_dim, int max_window) {
  return (head_dim == 64 || head_dim == 80) && max_window <= 128;
}

void attention_window_tc(const bf16* qkv, int ld_qkv, int rows, bf16* out, int ld_out, const AttnBlock* tiles,
                         int n_tiles, const int* cu_window, int n_win, int heads, int head_dim, float scale,
                         const float2* rope_table, double flops, cudaStream_t st) {
  if (n_tiles <= 0 || rows <= 0) return;
  if (rope_table == nullptr) throw DeviceError(RS_ERR_CUDA, "window attention: rope table required");
  WinParams p{};
  p.tiles = tiles;
  p.cu_window = cu_window;
  p.n_win = n_win;
  p.n_units = n_tiles * heads;
  p.heads = heads;
  p.rows_total = rows;
  p.rope = rope_table;
  p.scale_log2 = scale * 1.4426950408889634f;
  p.out = out;
  p.ld_out = ld_out;
  const MapPair& m = cached_maps(qkv, rows, 3 * heads * head_dim, ld_qkv);
  switch (head_dim) {
    case 80: return launch_win<80>(m, p, flops, st);
    case 64: return launch_win<64>(m, p, flops, st);
    default: throw DeviceError(RS_ERR_CUDA, "window attention: unsupported head_dim " + std::to_string(head_dim));
  }
}

}  // namespace rserve
