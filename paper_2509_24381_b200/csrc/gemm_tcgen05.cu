// rserve-b200 — tcgen05 / TMEM / TMA GEMM (see gemm.cuh for the contract).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstring>
#include <mutex>
#include <unordered_map>

#include "common.cuh"
#include "gemm.cuh"
#include "sm100.cuh"

namespace rserve {
namespace {

constexpr int kBM = 128;
constexpr int kBK = 64;  // 64 bf16 = 128 B = one swizzle row
constexpr int kThreads = 256;

struct GemmParams {
  void* C;
  int ldc;
  const bf16* bias;
  const bf16* residual;
  int ldr;
  const int* row_map;
  int M, N, K;
  const int* M_dev;
};

template <int BN>
struct Cfg {
  static constexpr int kStages = BN >= 256 ? 4 : 6;
  static constexpr int kABytes = kBM * kBK * 2;
  static constexpr int kBBytes = BN * kBK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kTmemCols = 2 * BN;  // double-buffered accumulator
  static constexpr int kSmem = kStages * kStageBytes + 1024 /*align*/ + 256 /*barriers*/;
};

__device__ __forceinline__ float gelu_erf(float x) {
  return 0.5f * x * (1.f + erff(x * 0.70710678118654752f));
}
__device__ __forceinline__ float silu(float x) { return x / (1.f + __expf(-x)); }

template <int EPI>
__device__ __forceinline__ void epilogue_chunk(const GemmParams& p, int row, int col,
                                               const std::uint32_t (&v)[32]) {
  float x[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) x[i] = __uint_as_float(v[i]);
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
      if (q * 8 < nvalid)
        reinterpret_cast<uint4*>(c)[q] =
            make_uint4(pack_bf16x2(x[8 * q], x[8 * q + 1]), pack_bf16x2(x[8 * q + 2], x[8 * q + 3]),
                       pack_bf16x2(x[8 * q + 4], x[8 * q + 5]),
                       pack_bf16x2(x[8 * q + 6], x[8 * q + 7]));
  }
}

template <int BN, int EPI>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tcgen05_kernel(const __grid_constant__ CUtensorMap tmA,
                        const __grid_constant__ CUtensorMap tmB, const GemmParams p) {
  using C = Cfg<BN>;
  extern __shared__ __align__(1024) std::uint8_t smem_raw[];
  std::uint8_t* smem = reinterpret_cast<std::uint8_t*>(
      (reinterpret_cast<std::uintptr_t>(smem_raw) + 1023) & ~std::uintptr_t(1023));
  std::uint8_t* smem_a = smem;
  std::uint8_t* smem_b = smem + C::kStages * C::kABytes;
  std::uint64_t* bars = reinterpret_cast<std::uint64_t*>(smem + C::kStages * C::kStageBytes);
  std::uint64_t* full = bars;
  std::uint64_t* empty = bars + C::kStages;
  std::uint64_t* tfull = bars + 2 * C::kStages;
  std::uint64_t* tempty = tfull + 2;
  std::uint32_t* tmem_holder = reinterpret_cast<std::uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int M = p.M_dev != nullptr ? min(*p.M_dev, p.M) : p.M;
  const int m_tiles = (M + kBM - 1) / kBM;
  const int n_tiles = (p.N + BN - 1) / BN;
  const int num_tiles = m_tiles * n_tiles;
  const int num_kb = (p.K + kBK - 1) / kBK;

  if (warp == 0 && lane == 0) {
    sm100::tma_prefetch_desc(&tmA);
    sm100::tma_prefetch_desc(&tmB);
    for (int s = 0; s < C::kStages; ++s) {
      sm100::mbar_init(&full[s], 1);
      sm100::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      sm100::mbar_init(&tfull[a], 1);
      sm100::mbar_init(&tempty[a], 4);
    }
    sm100::fence_mbar_init();
  }
  if (warp == 2) sm100::tmem_alloc(tmem_holder, C::kTmemCols);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const std::uint32_t tmem_base = *tmem_holder;

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer ----------------
    int stage = 0;
    std::uint32_t phase = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
      const int m0 = (tile % m_tiles) * kBM;
      const int n0 = (tile / m_tiles) * BN;
      for (int kb = 0; kb < num_kb; ++kb) {
        sm100::mbar_wait(&empty[stage], phase ^ 1);
        sm100::mbar_expect_tx(&full[stage], C::kStageBytes);
        sm100::tma_load_2d(smem_a + stage * C::kABytes, &tmA, &full[stage], kb * kBK, m0);
        sm100::tma_load_2d(smem_b + stage * C::kBBytes, &tmB, &full[stage], kb * kBK, n0);
        if (++stage == C::kStages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1 && lane == 0) {
    // ---------------- MMA issuer (single thread) ----------------
    constexpr std::uint32_t idesc = sm100::idesc_bf16_f32(kBM, BN);
    int stage = 0;
    std::uint32_t phase = 0;
    int local = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++local) {
      const int acc = local & 1;
      const std::uint32_t acc_phase = (local >> 1) & 1;
      sm100::mbar_wait(&tempty[acc], acc_phase ^ 1);
      sm100::tc_fence_after();
      const std::uint32_t d_tmem = tmem_base + static_cast<std::uint32_t>(acc * BN);
      for (int kb = 0; kb < num_kb; ++kb) {
        sm100::mbar_wait(&full[stage], phase);
        sm100::tc_fence_after();
        const std::uint64_t adesc =
            sm100::sw128_kmajor_desc(sm100::smem_u32(smem_a + stage * C::kABytes));
        const std::uint64_t bdesc =
            sm100::sw128_kmajor_desc(sm100::smem_u32(smem_b + stage * C::kBBytes));
#pragma unroll
        for (int kk = 0; kk < kBK / 16; ++kk) {
          // +32 B along K inside the 128B swizzle atom = +2 in the >>4 field.
          sm100::umma_bf16(d_tmem, adesc + 2 * kk, bdesc + 2 * kk, idesc,
                           (kb | kk) != 0 ? 1u : 0u);
        }
        sm100::umma_commit(&empty[stage]);  // frees the smem slot when MMAs finish
        if (++stage == C::kStages) {
          stage = 0;
          phase ^= 1;
        }
      }
      sm100::umma_commit(&tfull[acc]);  // accumulator ready for the epilogue
    }
  } else if (warp >= 4) {
    // ---------------- epilogue warps ----------------
    const int quad = warp - 4;  // TMEM lanes [32*quad, 32*quad + 32)
    int local = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++local) {
      const int m0 = (tile % m_tiles) * kBM;
      const int n0 = (tile / m_tiles) * BN;
      const int acc = local & 1;
      const std::uint32_t acc_phase = (local >> 1) & 1;
      sm100::mbar_wait(&tfull[acc], acc_phase);
      sm100::tc_fence_after();
      const int row = m0 + quad * 32 + lane;
      const std::uint32_t t_row =
          tmem_base + (static_cast<std::uint32_t>(quad * 32) << 16) + static_cast<std::uint32_t>(acc * BN);
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        std::uint32_t v[32];
        sm100::tmem_ld_32x32b_x32(t_row + static_cast<std::uint32_t>(c), v);
        sm100::tmem_ld_wait();
        if (row < M && n0 + c < p.N) epilogue_chunk<EPI>(p, row, n0 + c, v);
      }
      sm100::tc_fence_before();
      __syncwarp();
      if (lane == 0) sm100::mbar_arrive(&tempty[acc]);
    }
  }
  __syncthreads();
  if (warp == 2) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc(tmem_base, C::kTmemCols);
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

// K-major bf16 matrix [rows, k] (row stride ld elements), box [box_rows, 64].
CUtensorMap make_kmajor_map(const void* base, int rows, int k, int ld, int box_rows) {
  struct Key {
    const void* base;
    int rows, k, ld, box;
    bool operator==(const Key& o) const {
      return base == o.base && rows == o.rows && k == o.k && ld == o.ld && box == o.box;
    }
  };
  struct KeyHash {
    std::size_t operator()(const Key& x) const {
      std::size_t h = reinterpret_cast<std::uintptr_t>(x.base);
      h = h * 1000003u ^ static_cast<std::size_t>(x.rows);
      h = h * 1000003u ^ static_cast<std::size_t>(x.k);
      h = h * 1000003u ^ static_cast<std::size_t>(x.ld);
      return h * 1000003u ^ static_cast<std::size_t>(x.box);
    }
  };
  static std::mutex mu;
  static std::unordered_map<Key, CUtensorMap, KeyHash> cache;
  const Key key{base, rows, k, ld, box_rows};
  {
    std::lock_guard<std::mutex> g(mu);
    const auto it = cache.find(key);
    if (it != cache.end()) return it->second;
  }
  CUtensorMap tm;
  std::memset(&tm, 0, sizeof tm);
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(k), static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 2};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(kBK), static_cast<cuuint32_t>(box_rows)};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode_fn()(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base),
                                 dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw DeviceError(RS_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(r) +
                                       ") rows=" + std::to_string(rows) + " k=" + std::to_string(k) +
                                       " ld=" + std::to_string(ld));
  std::lock_guard<std::mutex> g(mu);
  if (cache.size() > 4096) cache.clear();
  cache.emplace(key, tm);
  return tm;
}

template <int BN, int EPI>
void launch(const GemmArgs& a, cudaStream_t stream) {
  using C = Cfg<BN>;
  static bool attr_set = false;
  if (!attr_set) {
    RS_CUDA_CHECK(cudaFuncSetAttribute(gemm_tcgen05_kernel<BN, EPI>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem));
    attr_set = true;
  }
  const CUtensorMap tmA = make_kmajor_map(a.A, a.M, a.K, a.lda, kBM);
  const CUtensorMap tmB = make_kmajor_map(a.B, a.N, a.K, a.ldb, BN);
  GemmParams p{a.C, a.ldc, a.bias, a.residual, a.ldr, a.row_map, a.M, a.N, a.K, a.M_dev};
  const int tiles = ceil_div(a.M, kBM) * ceil_div(a.N, BN);
  const int grid = tiles < kNumSMs ? tiles : kNumSMs;
  gemm_tcgen05_kernel<BN, EPI><<<grid, kThreads, C::kSmem, stream>>>(tmA, tmB, p);
  RS_LAUNCH_CHECK();
  count_launch();
}

template <int BN>
void dispatch_epi(const GemmArgs& a, Epi epi, cudaStream_t s) {
  switch (epi) {
    case Epi::Store: return launch<BN, 0>(a, s);
    case Epi::Residual: return launch<BN, 1>(a, s);
    case Epi::SwiGLU: return launch<BN, 2>(a, s);
    case Epi::Gelu: return launch<BN, 3>(a, s);
    case Epi::StoreF32: return launch<BN, 4>(a, s);
  }
}

// Wave efficiency of a tile width: useful tiles / (waves * SMs).
double wave_eff(int M, int N, int bn) {
  const int tiles = ceil_div(M, kBM) * ceil_div(N, bn);
  const int waves = ceil_div(tiles, kNumSMs);
  return static_cast<double>(tiles) / (static_cast<double>(waves) * kNumSMs);
}

}  // namespace

void gemm(const GemmArgs& a, Epi epi, cudaStream_t stream, int force_bn) {
  if (a.M <= 0 || a.N <= 0) return;
  if (a.K % 8 != 0 || a.N % 16 != 0 || a.lda % 8 != 0 || a.ldb % 8 != 0)
    throw DeviceError(RS_ERR_CUDA, "gemm: need K%8==0, N%16==0, lda/ldb%8==0 (K=" +
                                       std::to_string(a.K) + ", N=" + std::to_string(a.N) + ")");
  if (epi == Epi::SwiGLU && a.N % 32 != 0)
    throw DeviceError(RS_ERR_CUDA, "gemm: SwiGLU needs N%32==0");
  int bn = force_bn;
  if (bn == 0) {
    // Prefer the wide tile (half the A re-reads) unless the narrow one
    // fills the 148 SMs clearly better.
    bn = wave_eff(a.M, a.N, 128) > wave_eff(a.M, a.N, 256) + 0.15 ? 128 : 256;
  }
  const int tok = prof::begin(stream);
  if (bn == 256)
    dispatch_epi<256>(a, epi, stream);
  else
    dispatch_epi<128>(a, epi, stream);
  const double m = a.M, n = a.N, k = a.K;
  const double out_bytes = epi == Epi::StoreF32 ? 4.0 : (epi == Epi::SwiGLU ? 1.0 : 2.0);
  prof::end(tok, stream, "gemm_tcgen05", 2.0 * m * n * k,
            2.0 * (m * k + n * k) + out_bytes * m * n + (epi == Epi::Residual ? 2.0 * m * n : 0.0));
}

}  // namespace rserve
