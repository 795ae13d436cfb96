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
//     prep warps between the TMA arrival and the S MMA, from a compact
//     (position, frequency) cos/sin table staged in shared memory.
//   * P (bf16) goes back into S's TMEM columns and is the A operand of the
//     TS-MMA for O.
// Warp roles (384 threads, one CTA per SM, persistent over the units):
//   warp 0 TMA producer (3-stage smem ring), warp 1 MMA issuer, warps 2-3 and
//   8-11 RoPE prep, warps 4-7 softmax + epilogue (one query row per thread; warp w
//   owns TMEM lanes 32 (w % 4)). TMEM: S/P and O double-buffered (512 cols).
//   A warp whose rows all lie in one 64-column half of the tile (the common
//   two-window tile) reads / exponentiates only that half. O leaves through
//   the stage's Q slot (dead after S) by TMA store; the stage is refilled once
//   both the O MMAs and that store have read it.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cstring>
#include <mutex>
#include <unordered_map>

#include "attention.cuh"
#include "common.cuh"
#include "sm100.cuh"

namespace rserve {
namespace {

constexpr int kWinThreads = 384;
constexpr int kPrepThreads = 192;  // warps 2-3 and 8-11
constexpr int kWinStages = 3;
constexpr int kMaxFreqBytes = 24 * 1024;  // smem for the staged frequency table

template <int HD>
struct WinCfg {
  static_assert(HD == 64 || HD == 80, "window attention: head_dim 64 or 80");
  static constexpr int kTail = HD - 64;                    // 16 (hd 80) or 0
  static constexpr int kMainBytes = 128 * 128;             // [128 rows x 64] bf16, SW128
  static constexpr int kTailBytes = 128 * kTail * 2;       // [128 rows x 16] bf16, SW32
  // stage: Qm Km Vm (1024-aligned) then Qt Kt Vt (256-aligned)
  static constexpr int kStageBytes = 3 * kMainBytes + 3 * kTailBytes;
  static constexpr int kSmem = kWinStages * kStageBytes + kMaxFreqBytes + 1024 + 256;
  static constexpr int kChunkPairs = HD / 16;              // 16-B chunk pairs (i, i + hd/2) per row
};
static_assert(WinCfg<80>::kStageBytes % 1024 == 0, "stage alignment");

// TMEM columns: S/P of buffer b at 128 b, O of buffer b at 256 + 128 b.
constexpr std::uint32_t kTmemO = 256;

struct WinParams {
  const AttnBlock* tiles;   // {q_row0, q_rows, first window, windows} of each tile
  const std::uint32_t* win_row;  // [rows] this row's window as tile columns: lo | hi << 16
  int n_units;              // tiles * heads
  int heads;
  const int2* pos_hw;       // [rows] (h, w) patch position
  const float2* freq;       // [n_pos, hd/4] (cos, sin)(pos * theta^(-4j/hd)): the 2D RoPE
  int n_pos;                // positions the batch uses (table rows staged in smem)
  float scale_log2;
  bf16* out;
  int ld_out;
  unsigned long long* trace;  // RS_WIN_TRACE: per-CTA phase timestamps (diagnostics), else null
  int skip_rope;              // RS_WIN_SKIP_ROPE=1 in a -DRS_WIN_DEV_BUILD build: timing only (no RoPE)
};
constexpr int kTraceUnits = 8, kTraceSlots = 2 + 6 * kTraceUnits;

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define WIN_TRACE(slot)                                                                   \
  do {                                                                                    \
    if (p.trace != nullptr && (slot) < kTraceSlots)                                       \
      p.trace[static_cast<std::size_t>(blockIdx.x) * kTraceSlots + (slot)] = gtimer();    \
  } while (0)

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

// exp2 of a pair on the FMA pipe (no MUFU): round(x) by the 1.5 * 2^23 magic
// add, 2^f on [-0.5, 0.5] by a degree-3 minimax polynomial (rel. err 7.5e-5,
// below bf16's 3.9e-3); x <= -125.5 -> ~1e-38 (masked keys). Same as
// attention_tc.cu's poly_exp2_fma2: offloads part of the softmax from MUFU.
__device__ __forceinline__ float2 poly_exp2_pair(float2 x) {
  x.x = fmaxf(x.x, -125.5f);
  x.y = fmaxf(x.y, -125.5f);
  const float2 t = add2(x, make_float2(12582912.f, 12582912.f));
  const float2 n = add2(t, make_float2(-12582912.f, -12582912.f));
  const float2 f = add2(x, make_float2(-n.x, -n.y));
  float2 q = fma2(make_float2(0.05517166f, 0.05517166f), f, make_float2(0.24261116f, 0.24261116f));
  q = fma2(q, f, make_float2(0.69326099f, 0.69326099f));
  q = fma2(q, f, make_float2(0.99992807f, 0.99992807f));
  return make_float2(__int_as_float(__float_as_int(q.x) + (__float_as_int(t.x) << 23)),
                     __int_as_float(__float_as_int(q.y) + (__float_as_int(t.y) << 23)));
}

__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ uint4 lds128(std::uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts128(std::uint32_t a, uint4 v) {
  asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ float4 lds_f4(std::uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ void named_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
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
                       const __grid_constant__ CUtensorMap tmOutMain, const __grid_constant__ CUtensorMap tmOutTail,
                       const __grid_constant__ WinParams p) {
  using C = WinCfg<HD>;
  extern __shared__ __align__(1024) std::uint8_t smem_raw[];
  std::uint8_t* base = reinterpret_cast<std::uint8_t*>((reinterpret_cast<std::uintptr_t>(smem_raw) + 1023) & ~std::uintptr_t(1023));
  auto* sfreq = reinterpret_cast<float2*>(base + kWinStages * C::kStageBytes);
  auto* bars = reinterpret_cast<std::uint64_t*>(base + kWinStages * C::kStageBytes + kMaxFreqBytes);
  std::uint64_t* full = bars;              // [3] TMA bytes
  std::uint64_t* prepped = bars + 3;       // [3] prep threads
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
      sm100::mbar_init(&prepped[i], kPrepThreads);
      sm100::mbar_init(&empty[i], 2);  // MMA commit after O + the epilogue's store of O out of Q's slot
    }
    for (int i = 0; i < 2; ++i) {
      sm100::mbar_init(&s_full[i], 1);
      sm100::mbar_init(&p_full[i], 128);
      sm100::mbar_init(&o_full[i], 1);
      sm100::mbar_init(&tmem_free[i], 128);
    }
    sm100::fence_mbar_init();
    sm100::tma_prefetch_desc(&tmMain);
    sm100::tma_prefetch_desc(&tmOutMain);
    if (C::kTail) {
      sm100::tma_prefetch_desc(&tmTail);
      sm100::tma_prefetch_desc(&tmOutTail);
    }
  }
  if (warp == 0) sm100::tmem_alloc(tmem_slot, 512);
  // the frequency table is a model constant (not written by the preceding
  // kernel): staged before the PDL wait
  constexpr int kQuarter = HD / 4;
  for (int i = threadIdx.x; i < p.n_pos * kQuarter; i += kWinThreads) sfreq[i] = __ldg(p.freq + i);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const std::uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 0) WIN_TRACE(0);
  pdl_wait();
  if (threadIdx.x == 0) WIN_TRACE(1);
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
        // PV of the previous unit as soon as its P is in TMEM, unless this
        // unit's prep finishes first (then S first): whichever is ready
        bool pv_done = it == 0;
        if (!pv_done) {
          for (;;) {
            if (sm100::mbar_test(&p_full[(it - 1) & 1], ((it - 1) >> 1) & 1)) {
              issue_pv(it - 1);
              pv_done = true;
              break;
            }
            if (sm100::mbar_test(&prepped[s], (it / kWinStages) & 1)) break;
          }
        }
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
        if (!pv_done) issue_pv(it - 1);
      }
      if (it > 0) issue_pv(it - 1);
    }
  } else if (warp < 4 || warp >= 8) {
    // ---------------- RoPE prep (warps 2-3, 8-11) ----------------
    // warp task = (32-row group g, 16-B chunk pair c), lane = row: rotate-half
    // pairs (i, i + hd/2) of Q and K; consecutive rows hit distinct swizzled
    // 16-B slots (conflict-free). Pair i < hd/4 turns with the row position
    // h, the rest with w: (cos, sin) = freq[pos][i mod hd/4] (bit-identical
    // to vit_rope_table's per-row table).
    const int pw = warp < 4 ? warp - 2 : warp - 6;  // prep warp 0..5
    constexpr int kPrepWarps = kPrepThreads / 32;
    constexpr int kTasks = 4 * C::kChunkPairs;      // 20 (hd 80) / 16 (hd 64)
    const std::uint32_t sf = sm100::smem_u32(sfreq);
    int it = 0;
    for (int u = blockIdx.x; u < p.n_units; u += gridDim.x, ++it) {
      const int s = it % kWinStages;
      const AttnBlock t = p.tiles[u / H];
      int2 pos[4];  // this lane's row in each 32-row group (loaded before the wait)
#pragma unroll
      for (int g = 0; g < 4; ++g)
        pos[g] = 32 * g + lane < t.q_rows ? __ldg(p.pos_hw + t.q_row0 + 32 * g + lane) : make_int2(0, 0);
      sm100::mbar_wait(&full[s], (it / kWinStages) & 1);
      if (pw == 0 && lane == 0 && it < kTraceUnits) WIN_TRACE(2 + 6 * it);
      const std::uint32_t so = sbase + stage_off(s);
#pragma unroll 1
      for (int task = pw; task < (p.skip_rope ? 0 : kTasks); task += kPrepWarps) {
        const int g = task / C::kChunkPairs, c = task % C::kChunkPairs;
        const int r = 32 * g + lane;
        if (32 * g >= t.q_rows) continue;  // warp-uniform
        if (r < t.q_rows) {
          const int2 ps = g == 0 ? pos[0] : g == 1 ? pos[1] : g == 2 ? pos[2] : pos[3];
          const std::uint32_t fh = sf + static_cast<std::uint32_t>(ps.x * kQuarter) * 8u;
          const std::uint32_t fw = sf + static_cast<std::uint32_t>(ps.y * kQuarter) * 8u;
          float2 cz[8];
#pragma unroll
          for (int e = 0; e < 8; e += 2) {  // pairs 8c+e, 8c+e+1 (never straddle hd/4: both even)
            const int i = 8 * c + e;
            const float4 v = lds_f4(i < kQuarter ? fh + 8u * i : fw + 8u * (i - kQuarter));
            cz[e] = make_float2(v.x, v.y);
            cz[e + 1] = make_float2(v.z, v.w);
          }
          // all four chunk loads (Q, K halves) in flight before any math / store
          std::uint32_t pa[2], pb[2];
          uint4 a[2], bv[2];
#pragma unroll
          for (int which = 0; which < 2; ++which) {  // Q, K
            const std::uint32_t mo = which == 0 ? kQm : kKm, to = which == 0 ? kQt : kKt;
            pa[which] = so + chunk_off<HD>(r, c, mo, to);
            pb[which] = so + chunk_off<HD>(r, c + C::kChunkPairs, mo, to);
            a[which] = lds128(pa[which]);
            bv[which] = lds128(pb[which]);
          }
#pragma unroll
          for (int which = 0; which < 2; ++which) {
            std::uint32_t* aw = reinterpret_cast<std::uint32_t*>(&a[which]);
            std::uint32_t* bw = reinterpret_cast<std::uint32_t*>(&bv[which]);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float2 x = unpack_bf16x2(aw[e]), y = unpack_bf16x2(bw[e]);
              const float2 c0 = cz[2 * e], c1 = cz[2 * e + 1];
              aw[e] = pack_bf16x2(x.x * c0.x - y.x * c0.y, x.y * c1.x - y.y * c1.y);
              bw[e] = pack_bf16x2(y.x * c0.x + x.x * c0.y, y.y * c1.x + x.y * c1.y);
            }
          }
#pragma unroll
          for (int which = 0; which < 2; ++which) {
            sts128(pa[which], a[which]);
            sts128(pb[which], bv[which]);
          }
        }
      }
      sm100::fence_proxy_async_smem();  // generic-proxy writes -> visible to the MMA (async proxy)
      sm100::mbar_arrive(&prepped[s]);
      if (pw == 0 && lane == 0 && it < kTraceUnits) WIN_TRACE(3 + 6 * it);
    }
  } else {
    // ---------------- softmax + epilogue (one query row per thread) ----------------
    const int q = warp & 3;
    const int r = q * 32 + lane;
    const std::uint32_t lane_off = static_cast<std::uint32_t>(q * 32) << 16;
    int it = 0;
    int pend_stage = -1;  // stage whose O store is still reading Q's slot
    // this row's window [c_lo, c_hi) as tile columns (host table), loaded one
    // unit ahead so the load latency hides behind the current unit
    // (the table is padded by 128 rows: no bound check on the load path)
    auto win_of = [&](int uu) -> std::uint32_t {
      if (uu >= p.n_units) return 0u;
      return __ldg(p.win_row + p.tiles[uu / H].q_row0 + r);
    };
    std::uint32_t wr_next = win_of(blockIdx.x);
    for (int u = blockIdx.x; u < p.n_units; u += gridDim.x, ++it) {
      const int s = it % kWinStages, b = it & 1;
      const AttnBlock t = p.tiles[u / H];
      const int h = u % H;
      const std::uint32_t wr = r < t.q_rows ? wr_next : 0u;
      wr_next = win_of(u + gridDim.x);
      const int c_lo = static_cast<int>(wr & 0xFFFFu), c_hi = static_cast<int>(wr >> 16);
      // columns this warp needs: one 64-column half when every row's window
      // lies in it (two 64-patch windows per tile: the common case)
      const int w_lo = __reduce_min_sync(0xffffffffu, r < t.q_rows ? c_lo : 128);
      const int w_hi = __reduce_max_sync(0xffffffffu, c_hi);
      const int half = w_hi <= 64 ? 0 : (w_lo >= 64 ? 1 : -1);  // -1: both halves
      sm100::mbar_wait(&s_full[b], (it >> 1) & 1);
      sm100::tc_fence_after();
      if (r == 0 && it < kTraceUnits) WIN_TRACE(4 + 6 * it);
      const std::uint32_t srow = tmem + lane_off + 128 * b;
      // 64 columns of S (one half) -> registers, window-masked to -inf
      auto load_half = [&](int hh, std::uint32_t (&sv)[64]) {
#pragma unroll
        for (int c = 0; c < 2; ++c)
          sm100::tmem_ld_32x32b_x32(srow + 64 * hh + 32 * c, *reinterpret_cast<std::uint32_t(*)[32]>(&sv[32 * c]));
        sm100::tmem_ld_wait();
        const int lo = c_lo - 64 * hh, hi = c_hi - 64 * hh;
        if (__all_sync(0xffffffffu, lo <= 0 && hi >= 64)) return;  // whole half visible (aligned windows)
#pragma unroll
        for (int c = 0; c < 64; ++c)
          sv[c] = (c >= lo && c < hi) ? sv[c] : __float_as_uint(-INFINITY);
      };
      auto half_max = [](const std::uint32_t (&sv)[64]) {
        float mx8[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) mx8[i] = __uint_as_float(sv[i]);
#pragma unroll
        for (int c = 8; c < 64; ++c) mx8[c & 7] = fmaxf(mx8[c & 7], __uint_as_float(sv[c]));
        return fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                     fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7])));
      };
      // P = exp2(s * scale - max) of one half -> bf16 pairs over S's columns
      auto exp_half = [&](int hh, const std::uint32_t (&sv)[64], float mneg) {
        float rs8[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        std::uint32_t packed[32];
        const float2 sc2 = make_float2(p.scale_log2, p.scale_log2), mn2 = make_float2(mneg, mneg);
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const float2 x = fma2(make_float2(__uint_as_float(sv[2 * i]), __uint_as_float(sv[2 * i + 1])), sc2, mn2);
          float2 e;
          if (i & 1) {  // every other pair on the FMA pipe: MUFU and FMA share the work
            e = poly_exp2_pair(x);
          } else {
            e.x = fast_exp2(x.x);
            e.y = fast_exp2(x.y);
          }
          rs8[(2 * i) & 7] += e.x;
          rs8[(2 * i + 1) & 7] += e.y;
          packed[i] = pack_bf16x2(e.x, e.y);
        }
        sm100::tmem_st_32x32b_x32(srow + 32 * hh, packed);
        return ((rs8[0] + rs8[1]) + (rs8[2] + rs8[3])) + ((rs8[4] + rs8[5]) + (rs8[6] + rs8[7]));
      };
      float l = 0.f;
      std::uint32_t sv[64];
      if (half >= 0) {  // one 64-column half holds every row's window of this warp
        load_half(half, sv);
        const float mx = half_max(sv);
        l = exp_half(half, sv, mx == -INFINITY ? 0.f : -mx * p.scale_log2);
        std::uint32_t zeros[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) zeros[i] = 0u;
        sm100::tmem_st_32x32b_x32(srow + 32 * (1 - half), zeros);
      } else {  // windows across the halves: max over both, then exp per half
        // P of half h lands on S columns [32 h, 32 h + 32): half 0's P only
        // covers S columns half 0 has already consumed, half 1's would
        // overwrite half 0's upper S columns, so half 0 is exponentiated first
        load_half(1, sv);
        const float mx1 = half_max(sv);
        load_half(0, sv);
        const float mx = fmaxf(mx1, half_max(sv));
        const float mneg = mx == -INFINITY ? 0.f : -mx * p.scale_log2;
        l = exp_half(0, sv, mneg);
        load_half(1, sv);  // (re-read: one half of S in registers at a time; S columns 64-127 intact)
        l += exp_half(1, sv, mneg);
      }
      sm100::tmem_st_wait();
      sm100::tc_fence_before();
      sm100::mbar_arrive(&p_full[b]);
      if (r == 0 && it < kTraceUnits) WIN_TRACE(5 + 6 * it);
      // epilogue: O row -> bf16 -> Q's slot of this stage (dead since S) -> TMA store
      sm100::mbar_wait(&o_full[b], (it >> 1) & 1);
      sm100::tc_fence_after();
      if (r == 0 && it < kTraceUnits) WIN_TRACE(6 + 6 * it);
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
      const float inv = l > 0.f ? 1.f / l : 0.f;
      const float2 inv2 = make_float2(inv, inv);
      uint4 w[HD / 8];
#pragma unroll
      for (int c = 0; c < HD / 8; ++c) {
        std::uint32_t* ww = reinterpret_cast<std::uint32_t*>(&w[c]);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 y = mul2(make_float2(__uint_as_float(ov[8 * c + 2 * e]), __uint_as_float(ov[8 * c + 2 * e + 1])), inv2);
          ww[e] = pack_bf16x2(y.x, y.y);
        }
      }
      const std::uint32_t so = sbase + stage_off(s);
      if (t.q_rows == 128) {
        // whole tile: rows into Q's (swizzled) slot, one TMA store per box
#pragma unroll
        for (int c = 0; c < HD / 8; ++c) sts128(so + chunk_off<HD>(r, c, kQm, kQt), w[c]);
        sm100::fence_proxy_async_smem();
        named_sync(1, 128);
        if (r == 0) {
          sm100::tma_store_2d(&tmOutMain, base + stage_off(s) + kQm, h * HD, t.q_row0);
          if constexpr (C::kTail > 0)
            sm100::tma_store_2d(&tmOutTail, base + stage_off(s) + kQt, h * HD + 64, t.q_row0);
          sm100::bulk_commit();
          // the previous unit's store has read its slot by now (at most this
          // one in flight): release that stage, not this one (no wait here)
          if (pend_stage >= 0) {
            sm100::bulk_wait_read<1>();
            sm100::mbar_arrive(&empty[pend_stage]);
          }
          pend_stage = s;
        }
      } else {
        // partial tile (its last rows belong to the next tile): direct stores
        if (r < t.q_rows) {
          bf16* orow = p.out + static_cast<std::int64_t>(t.q_row0 + r) * p.ld_out + h * HD;
#pragma unroll
          for (int c = 0; c < HD / 8; ++c) *reinterpret_cast<uint4*>(orow + 8 * c) = w[c];
        }
        if (r == 0) {
          if (pend_stage >= 0) {
            sm100::bulk_wait_read<0>();
            sm100::mbar_arrive(&empty[pend_stage]);
            pend_stage = -1;
          }
          sm100::mbar_arrive(&empty[s]);
        }
      }
      if (r == 0 && it < kTraceUnits) WIN_TRACE(7 + 6 * it);
    }
    if (r == 0) {
      if (pend_stage >= 0) {
        sm100::bulk_wait_read<0>();
        sm100::mbar_arrive(&empty[pend_stage]);
      }
      sm100::bulk_wait<0>();  // stores complete before the CTA retires
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

const MapPair& cached_maps(const void* base, int rows, int cols, int ld) {  // keyed by base (qkv or out)
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
void launch_win(const MapPair& m, const MapPair& mo, const WinParams& p, double flops, double bytes,
                cudaStream_t st) {
  static std::once_flag once;
  std::call_once(once, [] {
    RS_CUDA_CHECK(cudaFuncSetAttribute(win_attn_tc_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       WinCfg<HD>::kSmem));
  });
  const int grid = std::min(p.n_units, kNumSMs);
  static const bool trace = std::getenv("RS_WIN_TRACE") != nullptr;
  WinParams q = p;
#ifdef RS_WIN_DEV_BUILD  // dev timing builds only (-DRS_WIN_DEV_BUILD): results are wrong with the knob set
  static const int skip_rope = std::getenv("RS_WIN_SKIP_ROPE") != nullptr ? std::atoi(std::getenv("RS_WIN_SKIP_ROPE")) : 0;
  q.skip_rope = skip_rope;
#else
  q.skip_rope = 0;
#endif
  unsigned long long* tbuf = nullptr;
  if (trace) {
    RS_CUDA_CHECK(cudaMallocAsync(reinterpret_cast<void**>(&tbuf), grid * kTraceSlots * 8, st));
    RS_CUDA_CHECK(cudaMemsetAsync(tbuf, 0, grid * kTraceSlots * 8, st));
    q.trace = tbuf;
  }
  const int tok = prof::begin(st);
  launch_kernel(win_attn_tc_kernel<HD>, dim3(grid), dim3(kWinThreads), WinCfg<HD>::kSmem, st, 1, m.main,
                m.tail, mo.main, mo.tail, q);
  RS_LAUNCH_CHECK();
  if (trace) {  // per-phase times relative to each CTA's start, averaged over CTAs
    std::vector<unsigned long long> h(static_cast<std::size_t>(grid) * kTraceSlots);
    RS_CUDA_CHECK(cudaMemcpyAsync(h.data(), tbuf, h.size() * 8, cudaMemcpyDeviceToHost, st));
    RS_CUDA_CHECK(cudaStreamSynchronize(st));
    RS_CUDA_CHECK(cudaFree(tbuf));
    unsigned long long t0 = ~0ull;
    for (int b = 0; b < grid; ++b) t0 = std::min(t0, h[static_cast<std::size_t>(b) * kTraceSlots]);
    std::fprintf(stderr, "[win-trace] grid %d units %d (ns from the first CTA start; CTA 0 / mean over CTAs)\n",
                 grid, p.n_units);
    for (int k = 0; k < kTraceSlots; ++k) {
      double sum = 0;
      int n = 0;
      for (int b = 0; b < grid; ++b) {
        const unsigned long long v = h[static_cast<std::size_t>(b) * kTraceSlots + k];
        if (v) { sum += static_cast<double>(v - t0); ++n; }
      }
      const unsigned long long v0 = h[static_cast<std::size_t>(k)];
      if (n) std::fprintf(stderr, "[win-trace] slot %2d cta0 %8.0f mean %8.0f (n=%d)\n", k,
                          v0 ? static_cast<double>(v0 - t0) : -1.0, sum / n, n);
    }
  }
  prof::end(tok, st, "attn_vit_window_tc", flops, bytes);
  count_launch();
}

}  // namespace

bool attention_window_tc_supported(int head_dim, int max_window, int n_pos) {
  return (head_dim == 64 || head_dim == 80) && max_window <= 128 &&
         static_cast<long>(n_pos) * (head_dim / 4) * sizeof(float2) <= kMaxFreqBytes;
}

void attention_window_tc(const bf16* qkv, int ld_qkv, int rows, bf16* out, int ld_out, const AttnBlock* tiles,
                         int n_tiles, int heads, int head_dim, float scale, const std::int32_t* pos_hw,
                         const float2* freq, int n_pos, double flops, cudaStream_t st) {
  if (n_tiles <= 0 || rows <= 0) return;
  if (!attention_window_tc_supported(head_dim, 128, n_pos))
    throw DeviceError(RS_ERR_CUDA, "window attention: unsupported head_dim / positions");
  WinParams p{};
  p.tiles = tiles;
  p.win_row = reinterpret_cast<const std::uint32_t*>(tiles + n_tiles);  // uploaded behind the tiles
  p.n_units = n_tiles * heads;
  p.heads = heads;
  p.pos_hw = reinterpret_cast<const int2*>(pos_hw);
  p.freq = freq;
  p.n_pos = n_pos;
  p.scale_log2 = scale * 1.4426950408889634f;
  p.out = out;
  p.ld_out = ld_out;
  const MapPair m = cached_maps(qkv, rows, 3 * heads * head_dim, ld_qkv);
  const MapPair mo = cached_maps(out, rows, heads * head_dim, ld_out);
  switch (head_dim) {
    // algorithmic bytes: packed q | k | v rows read once, o written once
    case 80: return launch_win<80>(m, mo, p, flops, 2.0 * 4 * heads * 80 * static_cast<double>(rows), st);
    case 64: return launch_win<64>(m, mo, p, flops, 2.0 * 4 * heads * 64 * static_cast<double>(rows), st);
    default: throw DeviceError(RS_ERR_CUDA, "window attention: unsupported head_dim " + std::to_string(head_dim));
  }
}

}  // namespace rserve
