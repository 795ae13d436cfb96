// rserve-b200 — chunked-prefill causal attention over the paged KV cache on
// tcgen05 tensor cores (sm_100a).
//
// CTA = one 128-query block of one slice x one q head (GQA: kv head = h / g).
// Per iteration of 128 keys (two 64-token KV pages):
//   S_j  = Q . K_j^T      tcgen05.mma, Q and K from smem (TMA, SW128), S in TMEM
//   P_j  = softmax rows   4 warps, one query row per thread, read S via
//                         tcgen05.ld, online max / sum in fp32, P written to smem
//                         as bf16 in the SW128 K-major layout
//   O~_j = P_j . V_j      tcgen05.mma into TMEM (fresh accumulator); the softmax
//                         warps fold it into their fp32 register accumulator
//                         O = O * exp2(m_{j-1} - m_j) + O~_j
// S and O~ are double-buffered in TMEM (4 x 128 columns) and K/V in smem, so the
// tensor core computes S_{j+1} while the softmax warps work on P_j.
// V is stored TRANSPOSED in the cache ([page][kv head][hd][64 tokens]) so that
// both MMAs read K-major SW128 operands (the GEMM's descriptor path).
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

constexpr int kTcThreads = 256;
constexpr int kAtom = 128 * 128;  // one [128 rows x 128 B] SW128 region

template <int HD>
struct TcCfg {
  static constexpr int kHdAtoms = HD / 64;             // K-dim atoms of Q / K tiles
  static constexpr int kQBytes = kHdAtoms * kAtom;     // Q [128 x HD]
  static constexpr int kKBytes = kHdAtoms * kAtom;     // K [128 keys x HD]
  static constexpr int kVAtom = HD * 128;              // V^T page [HD x 64 keys]
  static constexpr int kVBytes = 2 * kVAtom;           // two pages
  static constexpr int kPBytes = 2 * kAtom;            // P [128 q x 128 keys]
  static constexpr int kStages = 2;
  static constexpr int kSmem = kQBytes + kStages * (kKBytes + kVBytes) + 2 * kPBytes + 1024 + 512;
  static constexpr int kPageBytes = 64 * HD * 2 * 2;   // K + V of one page
};

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

template <int HD>
__global__ void __launch_bounds__(kTcThreads, 1)
    fa_prefill_tc_kernel(const __grid_constant__ CUtensorMap tmQ,
                         const __grid_constant__ CUtensorMap tmK,
                         const __grid_constant__ CUtensorMap tmV,
                         const PrefillWork* __restrict__ work, const int* const* page_tables,
                         int q_heads, int kv_heads, float scale_log2, bf16* __restrict__ out,
                         int ld_out) {
  using C = TcCfg<HD>;
  extern __shared__ __align__(1024) std::uint8_t smem_raw[];
  std::uint8_t* smem = reinterpret_cast<std::uint8_t*>(
      (reinterpret_cast<std::uintptr_t>(smem_raw) + 1023) & ~std::uintptr_t(1023));
  std::uint8_t* sQ = smem;
  std::uint8_t* sK = sQ + C::kQBytes;
  std::uint8_t* sV = sK + C::kStages * C::kKBytes;
  std::uint8_t* sP = sV + C::kStages * C::kVBytes;
  std::uint64_t* bars = reinterpret_cast<std::uint64_t*>(sP + 2 * C::kPBytes);
  std::uint64_t* q_full = bars;
  std::uint64_t* kv_full = bars + 1;
  std::uint64_t* kv_empty = bars + 3;
  std::uint64_t* s_full = bars + 5;
  std::uint64_t* s_empty = bars + 7;
  std::uint64_t* p_full = bars + 9;
  std::uint64_t* o_full = bars + 11;
  std::uint64_t* o_empty = bars + 13;
  std::uint32_t* tmem_holder = reinterpret_cast<std::uint32_t*>(bars + 16);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const PrefillWork w = work[blockIdx.x];
  const int head = blockIdx.y;
  const int kvh = head / (q_heads / kv_heads);
  const int n_keys = w.q_pos0 + w.q_rows;
  const int n_pages = (n_keys + 63) / 64;
  const int n_it = (n_keys + 127) / 128;
  const int* pt = page_tables[w.req_slot];

  if (threadIdx.x == 0) {
    sm100::tma_prefetch_desc(&tmQ);
    sm100::tma_prefetch_desc(&tmK);
    sm100::tma_prefetch_desc(&tmV);
    sm100::mbar_init(q_full, 1);
    for (int i = 0; i < 2; ++i) {
      sm100::mbar_init(&kv_full[i], 1);
      sm100::mbar_init(&kv_empty[i], 1);
      sm100::mbar_init(&s_full[i], 1);
      sm100::mbar_init(&s_empty[i], 128);
      sm100::mbar_init(&p_full[i], 128);
      sm100::mbar_init(&o_full[i], 1);
      sm100::mbar_init(&o_empty[i], 128);
    }
    sm100::fence_mbar_init();
  }
  if (warp == 2) sm100::tmem_alloc(tmem_holder, 512);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const std::uint32_t tmem = *tmem_holder;
  // TMEM columns: S[0] 0, S[1] 128, O~[0] 256, O~[1] 384

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer ----------------
    sm100::mbar_expect_tx(q_full, C::kQBytes);
    for (int h = 0; h < C::kHdAtoms; ++h)
      sm100::tma_load_2d(sQ + h * kAtom, &tmQ, q_full, head * HD + h * 64, w.q_row0);
    for (int j = 0; j < n_it; ++j) {
      const int st = j & 1;
      sm100::mbar_wait(&kv_empty[st], ((j >> 1) & 1) ^ 1);
      sm100::mbar_expect_tx(&kv_full[st], 2 * C::kPageBytes);
      const int pa = pt[2 * j];
      const int pb = 2 * j + 1 < n_pages ? pt[2 * j + 1] : pa;  // duplicate: finite, masked
      std::uint8_t* k = sK + st * C::kKBytes;
      std::uint8_t* v = sV + st * C::kVBytes;
      for (int h = 0; h < C::kHdAtoms; ++h) {
        sm100::tma_load_2d(k + h * kAtom, &tmK, &kv_full[st], h * 64, (pa * kv_heads + kvh) * 64);
        sm100::tma_load_2d(k + h * kAtom + 64 * 128, &tmK, &kv_full[st], h * 64,
                           (pb * kv_heads + kvh) * 64);
      }
      sm100::tma_load_2d(v, &tmV, &kv_full[st], 0, (pa * kv_heads + kvh) * HD);
      sm100::tma_load_2d(v + C::kVAtom, &tmV, &kv_full[st], 0, (pb * kv_heads + kvh) * HD);
    }
  } else if (warp == 1 && lane == 0) {
    // ---------------- MMA issuer ----------------
    constexpr std::uint32_t idesc_s = sm100::idesc_bf16_f32(128, 128);
    constexpr std::uint32_t idesc_o = sm100::idesc_bf16_f32(128, HD);
    sm100::mbar_wait(q_full, 0);
    // O accumulates in one TMEM region (cols 256..) across all iterations.
    auto issue_pv = [&](int i) {
      const int b = i & 1;
      sm100::mbar_wait(&p_full[b], (i >> 1) & 1);
      sm100::tc_fence_after();
      const std::uint32_t d = tmem + 256;
      std::uint8_t* v = sV + b * C::kVBytes;
      std::uint8_t* p = sP + b * C::kPBytes;
#pragma unroll
      for (int a = 0; a < 2; ++a) {
        const std::uint64_t pd = sm100::sw128_kmajor_desc(sm100::smem_u32(p + a * kAtom));
        const std::uint64_t vd = sm100::sw128_kmajor_desc(sm100::smem_u32(v + a * C::kVAtom));
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          sm100::umma_bf16(d, pd + 2 * kk, vd + 2 * kk, idesc_o, (i | a | kk) != 0 ? 1u : 0u);
      }
      sm100::umma_commit(&o_full[0]);  // completion count = PV index + 1
      sm100::umma_commit(&kv_empty[b]);
    };
    for (int j = 0; j < n_it; ++j) {
      const int b = j & 1;
      sm100::mbar_wait(&kv_full[b], (j >> 1) & 1);
      sm100::mbar_wait(&s_empty[b], ((j >> 1) & 1) ^ 1);
      sm100::tc_fence_after();
      const std::uint32_t d = tmem + 128 * b;
      std::uint8_t* k = sK + b * C::kKBytes;
#pragma unroll
      for (int h = 0; h < C::kHdAtoms; ++h) {
        const std::uint64_t qd = sm100::sw128_kmajor_desc(sm100::smem_u32(sQ + h * kAtom));
        const std::uint64_t kd = sm100::sw128_kmajor_desc(sm100::smem_u32(k + h * kAtom));
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          sm100::umma_bf16(d, qd + 2 * kk, kd + 2 * kk, idesc_s, (h | kk) != 0 ? 1u : 0u);
      }
      sm100::umma_commit(&s_full[b]);
      if (j >= 1) issue_pv(j - 1);
    }
    issue_pv(n_it - 1);
  } else if (warp >= 4) {
    // ---------------- softmax / accumulation (one query row per thread) ----------------
    const int q = warp - 4;
    const int r = q * 32 + lane;
    const int q_pos = w.q_pos0 + r;
    const std::uint32_t lane_off = static_cast<std::uint32_t>(q * 32) << 16;
    const std::uint32_t o_tmem = tmem + lane_off + 256;
    // Running max used for P (lazily raised: only when the true max exceeds it
    // by > 8 in log2 units, which bounds P by 2^8; O in TMEM is then rescaled).
    float m = -INFINITY, l = 0.f;
    for (int j = 0; j < n_it; ++j) {
      const int b = j & 1;
      sm100::mbar_wait(&s_full[b], (j >> 1) & 1);
      sm100::tc_fence_after();
      const int key0 = j * 128;
      const int lim = min(q_pos, n_keys - 1);  // keys <= lim are visible
      float mx = -INFINITY;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        std::uint32_t v[32];
        sm100::tmem_ld_32x32b_x32(tmem + lane_off + 128 * b + 32 * c, v);
        sm100::tmem_ld_wait();
#pragma unroll
        for (int t = 0; t < 32; ++t)
          if (key0 + 32 * c + t <= lim) mx = fmaxf(mx, __uint_as_float(v[t]) * scale_log2);
      }
      // PV_{j-1} must be complete before O may be rescaled (and, in order,
      // before this step's P feeds PV_j).
      if (j > 0) sm100::mbar_wait(&o_full[0], (j - 1) & 1);
      const bool raise = mx > m + 8.f || (m == -INFINITY && mx != -INFINITY);
      float alpha = 1.f;
      if (raise) {
        alpha = m == -INFINITY ? 0.f : exp2f(m - mx);
        m = mx;
      }
      if (j > 0 && __any_sync(0xffffffffu, raise && alpha != 1.f)) {
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
      const float m_new = m;
      float rs = 0.f;
      std::uint8_t* prow = sP + b * C::kPBytes + r * 128;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        std::uint32_t v[32];
        sm100::tmem_ld_32x32b_x32(tmem + lane_off + 128 * b + 32 * c, v);
        sm100::tmem_ld_wait();
        std::uint32_t packed[16];
#pragma unroll
        for (int t = 0; t < 16; ++t) {
          const int k0 = key0 + 32 * c + 2 * t;
          const float s0 = __uint_as_float(v[2 * t]) * scale_log2;
          const float s1 = __uint_as_float(v[2 * t + 1]) * scale_log2;
          const float p0 = (k0 <= lim && m_new != -INFINITY) ? exp2f(s0 - m_new) : 0.f;
          const float p1 = (k0 + 1 <= lim && m_new != -INFINITY) ? exp2f(s1 - m_new) : 0.f;
          rs += p0 + p1;
          packed[t] = pack_bf16x2(p0, p1);
        }
        // 32 keys = 4 16-byte chunks; atom = c / 2 (64 keys), chunk = (c % 2) * 4 + u
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int chunk = (c & 1) * 4 + u;
          uint4* dst = reinterpret_cast<uint4*>(prow + (c >> 1) * kAtom + ((chunk ^ (r & 7)) << 4));
          *dst = make_uint4(packed[4 * u], packed[4 * u + 1], packed[4 * u + 2], packed[4 * u + 3]);
        }
      }
      sm100::tc_fence_before();
      sm100::mbar_arrive(&s_empty[b]);
      fence_proxy_async_smem();
      sm100::mbar_arrive(&p_full[b]);
      l = l * alpha + rs;
    }
    sm100::mbar_wait(&o_full[0], (n_it - 1) & 1);
    sm100::tc_fence_after();
    const float inv = l > 0.f ? 1.f / l : 0.f;
    bf16* orow = out + static_cast<std::int64_t>(w.q_row0 + r) * ld_out + head * HD;
#pragma unroll
    for (int c = 0; c < HD / 32; ++c) {
      std::uint32_t v[32];
      sm100::tmem_ld_32x32b_x32(o_tmem + 32 * c, v);
      sm100::tmem_ld_wait();
      if (r < w.q_rows) {
#pragma unroll
        for (int u = 0; u < 4; ++u)
          reinterpret_cast<uint4*>(orow + 32 * c)[u] = make_uint4(
              pack_bf16x2(__uint_as_float(v[8 * u]) * inv, __uint_as_float(v[8 * u + 1]) * inv),
              pack_bf16x2(__uint_as_float(v[8 * u + 2]) * inv, __uint_as_float(v[8 * u + 3]) * inv),
              pack_bf16x2(__uint_as_float(v[8 * u + 4]) * inv, __uint_as_float(v[8 * u + 5]) * inv),
              pack_bf16x2(__uint_as_float(v[8 * u + 6]) * inv, __uint_as_float(v[8 * u + 7]) * inv));
      }
    }
  }
  __syncthreads();
  if (warp == 2) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc(tmem, 512);
  }
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
CUtensorMap map_2d(const void* base, std::int64_t rows, int cols, int ld, int box_rows) {
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
  std::int64_t rows;
  int cols, ld, box;
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

CUtensorMap cached_map(const void* base, std::int64_t rows, int cols, int ld, int box_rows) {
  static std::mutex mu;
  static std::unordered_map<MapKey, CUtensorMap, MapHash> cache;
  const MapKey key{base, rows, cols, ld, box_rows};
  std::lock_guard<std::mutex> g(mu);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  if (cache.size() > 4096) cache.clear();
  return cache.emplace(key, map_2d(base, rows, cols, ld, box_rows)).first->second;
}

template <int HD>
void launch_tc(const bf16* q, int ld_q, int q_rows_alloc, bf16* out, int ld_out,
               const PrefillWork* work, int n_work, const PagedKV& kv, std::int64_t kv_pages,
               int qh, int kvh, float scale, cudaStream_t st) {
  using C = TcCfg<HD>;
  static bool set = false;
  if (!set) {
    RS_CUDA_CHECK(cudaFuncSetAttribute(fa_prefill_tc_kernel<HD>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem));
    set = true;
  }
  const CUtensorMap tq = cached_map(q, q_rows_alloc, (qh + 2 * kvh) * HD, ld_q, 128);
  const CUtensorMap tk = cached_map(kv.k, kv_pages * kvh * 64, HD, HD, 64);
  const CUtensorMap tv = cached_map(kv.v, kv_pages * kvh * HD, 64, 64, HD);
  dim3 grid(n_work, qh);
  const int tok = prof::begin(st);
  fa_prefill_tc_kernel<HD><<<grid, kTcThreads, C::kSmem, st>>>(
      tq, tk, tv, work, kv.page_tables, qh, kvh, scale * 1.4426950408889634f, out, ld_out);
  RS_LAUNCH_CHECK();
  prof::end(tok, st, "attn_prefill_tcgen05", 0, 0);
  count_launch();
}

}  // namespace

void attention_prefill_paged_tc(const bf16* q, int ld_q, int q_rows_alloc, bf16* out, int ld_out,
                                const PrefillWork* work, int n_work, const PagedKV& kv,
                                std::int64_t kv_pages, int q_heads, int kv_heads, int head_dim,
                                float scale, cudaStream_t stream) {
  if (n_work <= 0) return;
  if (kv.page_size != 64) throw DeviceError(RS_ERR_CUDA, "tc attention needs 64-token pages");
  switch (head_dim) {
    case 64: return launch_tc<64>(q, ld_q, q_rows_alloc, out, ld_out, work, n_work, kv, kv_pages, q_heads, kv_heads, scale, stream);
    case 128: return launch_tc<128>(q, ld_q, q_rows_alloc, out, ld_out, work, n_work, kv, kv_pages, q_heads, kv_heads, scale, stream);
    default: throw DeviceError(RS_ERR_CUDA, "tc attention: unsupported head_dim " + std::to_string(head_dim));
  }
}

}  // namespace rserve
