// tcgen05 / TMEM / TMA GEMM for sm_100a with fused epilogues.
//
//   C[M,N] = sum_k A[m,k] * B[k,n]     bf16 operands, fp32 accumulation in TMEM
//
// One kernel template covers the three GEMM shapes of the reversible block
// (ref:proj/core/src/ops.cpp:48-92 matmul / matmul_tn / matmul_nt):
//   forward / recompute  x . W        A K-major  [T][in],  B MN-major W[in][out]
//   dgrad                dy . W^T     A K-major  [T][out], B K-major  W[in][out]
//   wgrad                x^T . dy     A MN-major [T][in],  B MN-major [T][out]   (K = T rows)
// so no operand is ever transposed in memory.
//
// Structure (persistent, warp-specialised, 1 CTA per SM):
//   warp 0      TMA producer (one lane)      smem ring of STAGES x (A 128x64 | B BNx64)
//   warp 1      TMEM allocator + MMA issuer  2 accumulators x BN fp32 columns in TMEM
//   warps 2..5  epilogue                     TMEM -> registers -> fused op -> global
// The tile -> CTA map is static (tile = blockIdx.x + i*gridDim.x), every tile and every
// split-K partial is computed by the same instruction sequence whatever the grid size,
// so results are bit-identical for any CTA cap (this is what lets PaReprop partition the
// SMs between its two lanes and still match Reprop bit for bit).
#include <cstdio>
#include <mutex>

#include "gemm.h"
#include "kernels.h"
#include "ptx.cuh"

namespace rp {

constexpr int kBM = 128;
constexpr int kBK = 64;
constexpr int kThreads = 192;

template <int BN>
struct GemmCfg {
  static constexpr int kStages = BN == 256 ? 4 : 6;
  static constexpr int kABytes = kBM * kBK * 2;
  static constexpr int kBBytes = BN * kBK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kTmemCols = 2 * BN;  // double-buffered accumulator
  static constexpr int kSmemBytes = 1024 + kStages * kStageBytes + 256;
};

struct GemmShape {
  int64_t M, N, K;
  int32_t m_tiles, n_tiles, k_blocks, splits;
};

template <int EPI>
__device__ __forceinline__ void epilogue_chunk(const GemmEpi& ep, const GemmShape& sh,
                                               int64_t row, int64_t col, int split,
                                               const float* v) {
  if (row >= sh.M || col >= sh.N) return;
  if constexpr (EPI == RP_EPI_BF16) {
    uint4* o = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(ep.out) + row * ep.ldo + col);
    o[0] = make_uint4(pack_bf16x2(v[0], v[1]), pack_bf16x2(v[2], v[3]),
                      pack_bf16x2(v[4], v[5]), pack_bf16x2(v[6], v[7]));
    o[1] = make_uint4(pack_bf16x2(v[8], v[9]), pack_bf16x2(v[10], v[11]),
                      pack_bf16x2(v[12], v[13]), pack_bf16x2(v[14], v[15]));
  } else if constexpr (EPI == RP_EPI_F32) {
    float4* o = reinterpret_cast<float4*>(static_cast<float*>(ep.out) +
                                          static_cast<int64_t>(split) * ep.split_stride +
                                          row * ep.ldo + col);
#pragma unroll
    for (int i = 0; i < 4; ++i) o[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
  } else if constexpr (EPI == RP_EPI_BIAS_GELU) {
    float u[16], a[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      u[i] = v[i] + (ep.bias ? ep.bias[col + i] : 0.0f);
      a[i] = gelu_tanh(u[i]);
    }
    uint4* o = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(ep.out) + row * ep.ldo + col);
    o[0] = make_uint4(pack_bf16x2(a[0], a[1]), pack_bf16x2(a[2], a[3]),
                      pack_bf16x2(a[4], a[5]), pack_bf16x2(a[6], a[7]));
    o[1] = make_uint4(pack_bf16x2(a[8], a[9]), pack_bf16x2(a[10], a[11]),
                      pack_bf16x2(a[12], a[13]), pack_bf16x2(a[14], a[15]));
    if (ep.out2) {
      uint4* o2 =
          reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(ep.out2) + row * ep.ldo2 + col);
      o2[0] = make_uint4(pack_bf16x2(u[0], u[1]), pack_bf16x2(u[2], u[3]),
                         pack_bf16x2(u[4], u[5]), pack_bf16x2(u[6], u[7]));
      o2[1] = make_uint4(pack_bf16x2(u[8], u[9]), pack_bf16x2(u[10], u[11]),
                         pack_bf16x2(u[12], u[13]), pack_bf16x2(u[14], u[15]));
    }
  } else if constexpr (EPI == RP_EPI_RESID) {
    const float4* r =
        reinterpret_cast<const float4*>(static_cast<const float*>(ep.aux) + row * ep.ldaux + col);
    float4* o = reinterpret_cast<float4*>(static_cast<float*>(ep.out) + row * ep.ldo + col);
    const float s = ep.sign;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float4 rv = r[i];
      float b0 = 0.f, b1 = 0.f, b2 = 0.f, b3 = 0.f;
      if (ep.bias) {
        b0 = ep.bias[col + 4 * i];
        b1 = ep.bias[col + 4 * i + 1];
        b2 = ep.bias[col + 4 * i + 2];
        b3 = ep.bias[col + 4 * i + 3];
      }
      o[i] = make_float4(rv.x + s * (v[4 * i] + b0), rv.y + s * (v[4 * i + 1] + b1),
                         rv.z + s * (v[4 * i + 2] + b2), rv.w + s * (v[4 * i + 3] + b3));
    }
  } else if constexpr (EPI == RP_EPI_GELU_BWD) {
    const uint4* up = reinterpret_cast<const uint4*>(
        static_cast<const __nv_bfloat16*>(ep.aux) + row * ep.ldaux + col);
    const uint4 u0 = up[0], u1 = up[1];
    const uint32_t uu[8] = {u0.x, u0.y, u0.z, u0.w, u1.x, u1.y, u1.z, u1.w};
    float d[16];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float2 f = unpack_bf16x2(uu[i]);
      d[2 * i] = v[2 * i] * gelu_tanh_slope(f.x);
      d[2 * i + 1] = v[2 * i + 1] * gelu_tanh_slope(f.y);
    }
    uint4* o = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(ep.out) + row * ep.ldo + col);
    o[0] = make_uint4(pack_bf16x2(d[0], d[1]), pack_bf16x2(d[2], d[3]),
                      pack_bf16x2(d[4], d[5]), pack_bf16x2(d[6], d[7]));
    o[1] = make_uint4(pack_bf16x2(d[8], d[9]), pack_bf16x2(d[10], d[11]),
                      pack_bf16x2(d[12], d[13]), pack_bf16x2(d[14], d[15]));
  }
}

template <int BN, bool A_MN, bool B_MN, int EPI>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_sm100_kernel(const __grid_constant__ CUtensorMap tmA,
                      const __grid_constant__ CUtensorMap tmB, const GemmShape sh,
                      const GemmEpi ep) {
  using Cfg = GemmCfg<BN>;
  constexpr int S = Cfg::kStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + S * Cfg::kABytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * Cfg::kStageBytes);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 4);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, Cfg::kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int tiles = sh.m_tiles * sh.n_tiles;
  const int units = tiles * sh.splits;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer
      int stage = 0;
      uint32_t phase = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const int split = u / tiles, tile = u % tiles;
        const int m0 = (tile / sh.n_tiles) * kBM, n0 = (tile % sh.n_tiles) * BN;
        const int kb0 = static_cast<int>((static_cast<int64_t>(split) * sh.k_blocks) / sh.splits);
        const int kb1 =
            static_cast<int>((static_cast<int64_t>(split + 1) * sh.k_blocks) / sh.splits);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* a = sA + stage * Cfg::kABytes;
          uint8_t* b = sB + stage * Cfg::kBBytes;
          const int k0 = kb * kBK;
          if constexpr (A_MN) {
            tma_load_2d(a, &tmA, &full[stage], m0, k0);
            tma_load_2d(a + 8192, &tmA, &full[stage], m0 + 64, k0);
          } else {
            tma_load_2d(a, &tmA, &full[stage], k0, m0);
          }
          if constexpr (B_MN) {
#pragma unroll
            for (int j = 0; j < BN / 64; ++j)
              tma_load_2d(b + 8192 * j, &tmB, &full[stage], n0 + 64 * j, k0);
          } else {
            tma_load_2d(b, &tmB, &full[stage], k0, n0);
          }
          mbar_arrive_expect_tx(&full[stage], Cfg::kStageBytes);
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer (single thread issues and commits)
      constexpr uint32_t idesc = make_idesc_bf16(kBM, BN, A_MN, B_MN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const int split = u / tiles;
        const int kb0 = static_cast<int>((static_cast<int64_t>(split) * sh.k_blocks) / sh.splits);
        const int kb1 =
            static_cast<int>((static_cast<int64_t>(split + 1) * sh.k_blocks) / sh.splits);
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + static_cast<uint32_t>(acc * BN);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(sA + stage * Cfg::kABytes);
          const uint32_t b_addr = smem_u32(sB + stage * Cfg::kBBytes);
#pragma unroll
          for (int kk = 0; kk < kBK / 16; ++kk) {
            const uint64_t ad = A_MN ? make_sdesc_sw128(a_addr + kk * 2048, 8192, 1024)
                                     : make_sdesc_sw128(a_addr + kk * 32, 16, 1024);
            const uint64_t bd = B_MN ? make_sdesc_sw128(b_addr + kk * 2048, 8192, 1024)
                                     : make_sdesc_sw128(b_addr + kk * 32, 16, 1024);
            umma_bf16(tmem_d, ad, bd, idesc, (kb > kb0 || kk > 0) ? 1u : 0u);
          }
          umma_commit(&empty[stage]);
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit(&tfull[acc]);
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else {
    // ---------------- epilogue warps 2..5; warp w reads TMEM lanes [32*(w%4), +32)
    const uint32_t q = warp & 3u;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      const int split = u / tiles, tile = u % tiles;
      const int64_t m0 = static_cast<int64_t>(tile / sh.n_tiles) * kBM;
      const int64_t n0 = static_cast<int64_t>(tile % sh.n_tiles) * BN;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t tbase = tmem_base + ((q * 32u) << 16) + static_cast<uint32_t>(acc * BN);
      const int64_t row = m0 + q * 32 + lane;
#pragma unroll 1
      for (int c = 0; c < BN; c += 16) {
        float v[16];
        tmem_ld16(tbase + c, v);
        epilogue_chunk<EPI>(ep, sh, row, n0 + c, split, v);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }

  __syncwarp();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tmem_base, Cfg::kTmemCols);
}

// Deterministic split-K reduction: out[i] = sum_{s=0..S-1} part[s][i], fixed order.
__global__ void splitk_reduce_kernel(const float* __restrict__ part, int splits,
                                     int64_t stride, int64_t n4, float* __restrict__ out) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n4;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float4 acc = reinterpret_cast<const float4*>(part)[i];
    for (int s = 1; s < splits; ++s) {
      const float4 v = reinterpret_cast<const float4*>(part + s * stride)[i];
      acc.x += v.x;
      acc.y += v.y;
      acc.z += v.z;
      acc.w += v.w;
    }
    reinterpret_cast<float4*>(out)[i] = acc;
  }
}

// ------------------------------------------------------------------ host side
typedef CUresult (*PFN_encodeTiled_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                      const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                      const cuuint32_t*, CUtensorMapInterleave,
                                      CUtensorMapSwizzle, CUtensorMapL2promotion,
                                      CUtensorMapFloatOOBfill);

static PFN_encodeTiled_t get_encode_fn() {
  static PFN_encodeTiled_t fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled_t>(p);
  });
  return fn;
}

// bf16 row-major matrix [rows][cols], pitch ld elements; box = {64 cols, box_rows rows}.
static int encode_map(CUtensorMap* m, const void* ptr, int64_t rows, int64_t cols, int64_t ld,
                      uint32_t box_rows) {
  PFN_encodeTiled_t fn = get_encode_fn();
  if (!fn) return RP_ERR_CUDA;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides,
                  box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? RP_OK : RP_ERR_CUDA;
}

typedef void (*GemmKernelPtr)(CUtensorMap, CUtensorMap, GemmShape, GemmEpi);

template <int BN, bool A_MN, bool B_MN, int EPI>
static GemmKernelPtr kernel_ptr() {
  static std::once_flag once;
  auto k = &gemm_sm100_kernel<BN, A_MN, B_MN, EPI>;
  std::call_once(once, [k] {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         GemmCfg<BN>::kSmemBytes);
  });
  return reinterpret_cast<GemmKernelPtr>(k);
}

template <int BN, bool A_MN, bool B_MN>
static GemmKernelPtr pick_epi(int epi) {
  switch (epi) {
    case RP_EPI_BF16: return kernel_ptr<BN, A_MN, B_MN, RP_EPI_BF16>();
    case RP_EPI_F32: return kernel_ptr<BN, A_MN, B_MN, RP_EPI_F32>();
    case RP_EPI_BIAS_GELU: return kernel_ptr<BN, A_MN, B_MN, RP_EPI_BIAS_GELU>();
    case RP_EPI_RESID: return kernel_ptr<BN, A_MN, B_MN, RP_EPI_RESID>();
    case RP_EPI_GELU_BWD: return kernel_ptr<BN, A_MN, B_MN, RP_EPI_GELU_BWD>();
  }
  return nullptr;
}

template <int BN>
static GemmKernelPtr pick(bool a_mn, bool b_mn, int epi) {
  if (!a_mn && !b_mn) return pick_epi<BN, false, false>(epi);
  if (!a_mn && b_mn) return pick_epi<BN, false, true>(epi);
  if (a_mn && !b_mn) return pick_epi<BN, true, false>(epi);
  return pick_epi<BN, true, true>(epi);
}

static int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

}  // namespace rp

using namespace rp;

struct RpGemmPlan {
  CUtensorMap tmA, tmB;
  GemmShape sh;
  GemmEpi ep;
  GemmKernelPtr kern;
  int bn;
  int grid;
  int smem;
  // split-K reduction (only when splits > 1)
  float* red_out;
  int64_t red_n;
};

extern "C" int rp_gemm_plan_create(const RpGemmDesc* d, RpGemmPlan** out) {
  if (!d || !out) return rp_fail(RP_ERR_CONTRACT, "gemm: null descriptor");
  *out = nullptr;
  const int64_t M = d->M, N = d->N, K = d->K;
  if (M <= 0 || N <= 0 || K <= 0) return rp_fail(RP_ERR_SHAPE, "gemm: empty M/N/K");
  if (N % 16 != 0) return rp_fail(RP_ERR_SHAPE, "gemm: N must be a multiple of 16");
  if (d->lda % 8 || d->ldb % 8 || d->ldo % (d->epi == RP_EPI_F32 || d->epi == RP_EPI_RESID ? 4 : 8))
    return rp_fail(RP_ERR_SHAPE, "gemm: leading dimensions must be 16-byte multiples");
  if ((reinterpret_cast<uintptr_t>(d->A) | reinterpret_cast<uintptr_t>(d->B)) & 15)
    return rp_fail(RP_ERR_SHAPE, "gemm: operands must be 16-byte aligned");
  const int bn = (d->bn == 128) ? 128 : 256;
  RpGemmPlan* p = new RpGemmPlan();
  p->bn = bn;
  p->sh.M = M;
  p->sh.N = N;
  p->sh.K = K;
  p->sh.m_tiles = static_cast<int32_t>((M + kBM - 1) / kBM);
  p->sh.n_tiles = static_cast<int32_t>((N + bn - 1) / bn);
  p->sh.k_blocks = static_cast<int32_t>((K + kBK - 1) / kBK);
  int splits = d->splits < 1 ? 1 : d->splits;
  if (splits > p->sh.k_blocks) splits = p->sh.k_blocks;
  if (splits > 1 && d->epi != RP_EPI_F32) {
    delete p;
    return rp_fail(RP_ERR_CONTRACT, "gemm: split-K needs the fp32 (wgrad) epilogue");
  }
  p->sh.splits = splits;
  p->ep.out = d->out;
  p->ep.ldo = d->ldo;
  p->ep.out2 = d->out2;
  p->ep.ldo2 = d->ldo2;
  p->ep.aux = d->aux;
  p->ep.ldaux = d->ldaux;
  p->ep.bias = d->bias;
  p->ep.sign = d->sign;
  p->ep.split_stride = M * d->ldo;
  p->red_out = nullptr;
  p->red_n = 0;
  if (splits > 1) {
    if (!d->workspace || d->ldo != N) {
      delete p;
      return rp_fail(RP_ERR_CONTRACT, "gemm: split-K needs a workspace and ldo == N");
    }
    p->ep.out = d->workspace;  // partials [splits][M][N]
    p->red_out = static_cast<float*>(d->out);
    p->red_n = M * N;
  }
  int rc;
  // A: K-major stored [M][K]; MN-major stored [K][M]
  if (d->a_mn)
    rc = encode_map(&p->tmA, d->A, K, M, d->lda, 64);
  else
    rc = encode_map(&p->tmA, d->A, M, K, d->lda, kBM);
  if (rc == RP_OK) {
    if (d->b_mn)
      rc = encode_map(&p->tmB, d->B, K, N, d->ldb, 64);
    else
      rc = encode_map(&p->tmB, d->B, N, K, d->ldb, static_cast<uint32_t>(bn));
  }
  if (rc != RP_OK) {
    delete p;
    return rp_fail(rc, "gemm: cuTensorMapEncodeTiled failed");
  }
  p->kern = bn == 256 ? pick<256>(d->a_mn, d->b_mn, d->epi) : pick<128>(d->a_mn, d->b_mn, d->epi);
  if (!p->kern) {
    delete p;
    return rp_fail(RP_ERR_CONFIG, "gemm: unknown epilogue");
  }
  p->smem = bn == 256 ? GemmCfg<256>::kSmemBytes : GemmCfg<128>::kSmemBytes;
  const int units = p->sh.m_tiles * p->sh.n_tiles * splits;
  int cap = d->max_ctas > 0 ? d->max_ctas : num_sms();
  p->grid = units < cap ? units : cap;
  *out = p;
  return RP_OK;
}

extern "C" int rp_gemm_plan_launch(const RpGemmPlan* p, rp_stream_t stream_) {
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  if (!p) return RP_ERR_CONTRACT;
  p->kern<<<p->grid, kThreads, p->smem, stream>>>(p->tmA, p->tmB, p->sh, p->ep);
  if (cudaPeekAtLastError() != cudaSuccess) return rp_check_launch("gemm");
  if (p->sh.splits > 1) {
    const int64_t n4 = p->red_n / 4;
    int blocks = static_cast<int>((n4 + 255) / 256);
    if (blocks > 4 * num_sms()) blocks = 4 * num_sms();
    splitk_reduce_kernel<<<blocks, 256, 0, stream>>>(static_cast<const float*>(p->ep.out),
                                                     p->sh.splits, p->ep.split_stride, n4,
                                                     p->red_out);
  }
  return rp_check_launch("gemm");
}

extern "C" int rp_gemm_plan_set_max_ctas(RpGemmPlan* p, int max_ctas) {
  if (!p) return RP_ERR_CONTRACT;
  const int units = p->sh.m_tiles * p->sh.n_tiles * p->sh.splits;
  const int cap = max_ctas > 0 ? max_ctas : num_sms();
  p->grid = units < cap ? units : cap;
  return RP_OK;
}

extern "C" void rp_gemm_plan_destroy(RpGemmPlan* p) { delete p; }

extern "C" int rp_gemm_plan_shape(const RpGemmPlan* p, int64_t* M, int64_t* N, int64_t* K) {
  if (!p) return RP_ERR_CONTRACT;
  *M = p->sh.M;
  *N = p->sh.N;
  *K = p->sh.K;
  return RP_OK;
}

extern "C" int rp_gemm(const RpGemmDesc* d, rp_stream_t stream) {
  RpGemmPlan* p = nullptr;
  int rc = rp_gemm_plan_create(d, &p);
  if (rc != RP_OK) return rc;
  rc = rp_gemm_plan_launch(p, stream);
  rp_gemm_plan_destroy(p);
  return rc;
}
