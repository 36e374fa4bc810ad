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
#include "launch.h"

namespace rp {

constexpr int kBM = 128;

// Instrumentation (tools/gemm_trace.py): when set, the CTA-pair kernel's cluster 0 records
// per tile (first 64 of its tiles, 8 uint64 each): MMA warp waits for the accumulator /
// gets it / cycles spent waiting for operand stages / last MMA issued; epilogue warp 2 gets
// the accumulator / releases it.
__device__ unsigned long long* g_gemm_trace = nullptr;
#define GEMM_TRACE(t, slot, val)                                                        \
  do {                                                                                  \
    if (gtr && (t) < 64) gtr[(t) * 8 + (slot)] = static_cast<unsigned long long>(val);  \
  } while (0)
constexpr int kBK = 64;
constexpr int kThreads = 64 + 8 * 32;  // TMA warp, MMA warp, 8 epilogue warps

template <int BN>
struct GemmCfg {
  static constexpr int kStages = BN == 256 ? 4 : 6;
  static constexpr int kABytes = kBM * kBK * 2;
  static constexpr int kBBytes = BN * kBK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kTmemCols = 2 * BN;  // double-buffered accumulator
  static constexpr int kEpiBytes = 8 * 4096;
  static constexpr int kSmemBytes = 1024 + kStages * kStageBytes + kEpiBytes + 256;
};

struct GemmShape {
  int64_t M, N, K;
  int32_t m_tiles, n_tiles, k_blocks, splits;
  int32_t issue;  // MMA issue form: 1 warp-converged (predicated), 0 one diverged lane
};

// Work unit u -> (split, tile, k-block range). splits == 1 (every non-wgrad GEMM) needs no
// division: the per-tile index math sits between two tiles' MMA streams on the issuing warp.
struct UnitRange {
  int split, tile, kb0, kb1;
};
__device__ __forceinline__ UnitRange unit_range(const GemmShape& sh, int u, int tiles) {
  if (sh.splits == 1) return {0, u, 0, sh.k_blocks};
  const int split = u / tiles;
  return {split, u - split * tiles, (split * sh.k_blocks) / sh.splits,
          ((split + 1) * sh.k_blocks) / sh.splits};
}

// ---------------------------------------------------------------- epilogue
// Each epilogue warp owns 32 accumulator rows (its TMEM lane quarter) and half of the BN
// columns, processed in 32x32 chunks. tcgen05.ld gives one row per thread; the chunk is
// bounced through a warp-private, XOR-swizzled 4 KB smem tile so that every global load
// (residual / saved pre-activation) and store is row-contiguous across the warp (coalesced)
// and every smem access is bank-conflict free.
constexpr int kEpiWarps = 8;
constexpr int kEpiStage = 4096;  // bytes per warp

// fp32 tile: 32 rows x 128 B, 16 B chunk c of row r at r*128 + ((c ^ (r & 7)) << 4)
__device__ __forceinline__ uint32_t sw32(int r, int c) {
  return static_cast<uint32_t>(r * 128 + ((c ^ (r & 7)) << 4));
}
// bf16 tile: 32 rows x 64 B, chunk c (0..3) of row r at r*64 + ((c ^ ((r >> 1) & 3)) << 4)
__device__ __forceinline__ uint32_t sw16(int r, int c) {
  return static_cast<uint32_t>(r * 64 + ((c ^ ((r >> 1) & 3)) << 4));
}

__device__ __forceinline__ void sts128(uint32_t a, uint4 v) {
  asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}
__device__ __forceinline__ uint4 lds128(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(a)
               : "memory");
  return v;
}

// row-owner -> staging (fp32 values)
__device__ __forceinline__ void stage_rows_f32(uint32_t st, int lane, const float* v) {
#pragma unroll
  for (int c = 0; c < 8; ++c)
    sts128(st + sw32(lane, c),
           make_uint4(__float_as_uint(v[4 * c]), __float_as_uint(v[4 * c + 1]),
                      __float_as_uint(v[4 * c + 2]), __float_as_uint(v[4 * c + 3])));
}
// row-owner -> staging (bf16 values)
__device__ __forceinline__ void stage_rows_bf16(uint32_t st, int lane, const float* v) {
#pragma unroll
  for (int c = 0; c < 4; ++c)
    sts128(st + sw16(lane, c),
           make_uint4(pack_bf16x2(v[8 * c], v[8 * c + 1]), pack_bf16x2(v[8 * c + 2], v[8 * c + 3]),
                      pack_bf16x2(v[8 * c + 4], v[8 * c + 5]),
                      pack_bf16x2(v[8 * c + 6], v[8 * c + 7])));
}
// staging -> global, coalesced: 8 lanes per 128 B fp32 row
__device__ __forceinline__ void store_tile_f32(uint32_t st, int lane, float* g, int64_t ld,
                                               int64_t row0, int64_t rows_left) {
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int r = (lane >> 3) + 4 * i, c = lane & 7;
    const uint4 x = lds128(st + sw32(r, c));
    if (r < rows_left) *reinterpret_cast<uint4*>(g + (row0 + r) * ld + 4 * c) = x;
  }
}
// staging -> global, coalesced: 4 lanes per 64 B bf16 row
__device__ __forceinline__ void store_tile_bf16(uint32_t st, int lane, __nv_bfloat16* g,
                                                int64_t ld, int64_t row0, int64_t rows_left) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = (lane >> 2) + 8 * i, c = lane & 3;
    const uint4 x = lds128(st + sw16(r, c));
    if (r < rows_left) *reinterpret_cast<uint4*>(g + (row0 + r) * ld + 8 * c) = x;
  }
}
// Internal epilogue kinds (not in the C ABI): kEpiTma + k is epilogue k with its outputs
// stored through TMA, chosen for CTA-pair tiles with a short K loop, where the epilogue's
// stores, not the MMA, bound the tile.
constexpr int kEpiTma = 100;   // two staging buffers per warp, one pipeline stage fewer
constexpr int kEpiTma1 = 200;  // one staging buffer per warp, full pipeline (long K)
constexpr int base_epi(int epi) {
  return epi >= kEpiTma1 ? epi - kEpiTma1 : (epi >= kEpiTma ? epi - kEpiTma : epi);
}
constexpr bool is_resid(int epi) { return base_epi(epi) == RP_EPI_RESID; }

// Epilogue inputs of one chunk, fetched one chunk ahead (software pipelining) so the
// global-load latency of the residual / saved pre-activation overlaps the previous chunk.
// A chunk is 32 rows x 128 B: 32 fp32 columns (fp32 outputs) or 64 bf16 columns (bf16
// outputs), so every staged row is one full 128-byte line.
struct ChunkIn {
  uint4 aux[8];  // 32 rows x 128 B of the residual (fp32) or of u (bf16), coalesced
};

template <int EPI>
__device__ __forceinline__ void prefetch_chunk(const GemmEpi& ep, int lane, int64_t row0,
                                               int64_t rows_left, int64_t col, ChunkIn& in) {
  if constexpr (is_resid(EPI) || base_epi(EPI) == RP_EPI_GELU_BWD || base_epi(EPI) == RP_EPI_MUL ||
                base_epi(EPI) == RP_EPI_ROWDOT) {
    const int esz = is_resid(EPI) ? 4 : 2;
    const uint8_t* g = static_cast<const uint8_t*>(ep.aux) + col * esz;
    const int64_t ldb = ep.ldaux * esz;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int r = (lane >> 3) + 4 * i, c = lane & 7;
      in.aux[i] = r < rows_left ? *reinterpret_cast<const uint4*>(g + (row0 + r) * ldb + 16 * c)
                                : make_uint4(0, 0, 0, 0);
    }
  }
}

// staging (32 x 128 B, swizzled) -> global, 8 lanes per row: 4 full lines per instruction
__device__ __forceinline__ void store_tile(uint32_t st, int lane, void* g, int64_t ldb,
                                           int64_t row0, int64_t rows_left) {
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int r = (lane >> 3) + 4 * i, c = lane & 7;
    const uint4 x = lds128(st + sw32(r, c));
    if (r < rows_left)
      *reinterpret_cast<uint4*>(static_cast<uint8_t*>(g) + (row0 + r) * ldb + 16 * c) = x;
  }
}
// prefetched coalesced aux -> staging -> this lane's row (8 x 16 B)
__device__ __forceinline__ void aux_rows(uint32_t st, int lane, const ChunkIn& in, uint4* row) {
#pragma unroll
  for (int i = 0; i < 8; ++i) sts128(st + sw32((lane >> 3) + 4 * i, lane & 7), in.aux[i]);
  __syncwarp();
#pragma unroll
  for (int c = 0; c < 8; ++c) row[c] = lds128(st + sw32(lane, c));
  __syncwarp();
}
__device__ __forceinline__ float lds32(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a) : "memory");
  return v;
}
// Column sums of a 32-row x 64-column chunk (this lane holds one row, v[64]) by a
// register butterfly (reduce-scatter over the 32 lanes: 5 rounds of shfl.xor, halving the
// live columns each round), so no shared-memory traffic competes with the tensor core's
// operand reads. Afterwards lane j holds the sums of columns 2j and 2j+1 ->
// ep.colsum[row0 / 32][col + 2j .. +1]. Fixed association order (deterministic).
__device__ __forceinline__ void colsum_chunk64(const GemmEpi& ep, uint32_t /*st*/, int lane,
                                               int64_t row0, int64_t col, const float* v) {
  float a[64];
#pragma unroll
  for (int i = 0; i < 64; ++i) a[i] = v[i];
#pragma unroll
  for (int k = 16, n = 64; k >= 1; k >>= 1, n >>= 1) {
    const bool up = (lane & k) != 0;  // keep the upper half of the live columns
#pragma unroll
    for (int i = 0; i < n / 2; ++i) {
      const float send = up ? a[i] : a[i + n / 2];
      const float keep = up ? a[i + n / 2] : a[i];
      a[i] = keep + __shfl_xor_sync(0xffffffffu, send, k);
    }
  }
  float2* dst = reinterpret_cast<float2*>(ep.colsum + (row0 >> 5) * ep.ldcs + col) + lane;
  *dst = make_float2(a[0], a[1]);
}
// this lane's 64 bf16 values -> staging
__device__ __forceinline__ void stage_row_bf16x64(uint32_t st, int lane, const float* v) {
#pragma unroll
  for (int c = 0; c < 8; ++c)
    sts128(st + sw32(lane, c),
           make_uint4(pack_bf16x2(v[8 * c], v[8 * c + 1]), pack_bf16x2(v[8 * c + 2], v[8 * c + 3]),
                      pack_bf16x2(v[8 * c + 4], v[8 * c + 5]),
                      pack_bf16x2(v[8 * c + 6], v[8 * c + 7])));
}

template <int EPI>
struct EpiTraits {
  static constexpr int kCW = (base_epi(EPI) == RP_EPI_F32 || is_resid(EPI)) ? 32 : 64;
};

// Output staging. Register path (TMA = false): one staging buffer per warp, staged chunk ->
// global by coalesced 16-byte stores. TMA path: two buffers per warp used in turn; a chunk is
// staged into a buffer whose previous bulk store has finished reading it, then lane 0
// issues one cp.async.bulk.tensor store (its own bulk group; rows / columns past M / N are
// clipped by the tensor map).
struct StageRing {
  uint32_t base;
  int idx;
  int nbuf;  // 1 or 2 staging buffers
};
template <bool TMA>
__device__ __forceinline__ uint32_t stage_acquire(uint32_t st, StageRing& ring, int lane) {
  if constexpr (!TMA) {
    return st;
  } else {
    if (lane == 0) {
      if (ring.nbuf == 2)
        asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      else
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    }
    __syncwarp();
    return ring.base + static_cast<uint32_t>(ring.idx * kEpiStage);
  }
}
template <bool TMA>
__device__ __forceinline__ void stage_emit(uint32_t buf, StageRing& ring, int lane, void* g,
                                           int64_t ldb, int64_t row0, int64_t rows_left,
                                           const CUtensorMap* tm, int64_t col) {
  if constexpr (TMA) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) {
      asm volatile(
          "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
              reinterpret_cast<uint64_t>(tm)),
          "r"(static_cast<int32_t>(col)), "r"(static_cast<int32_t>(row0)), "r"(buf)
          : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    __syncwarp();
    ring.idx = ring.nbuf == 2 ? ring.idx ^ 1 : 0;
  } else {
    __syncwarp();
    store_tile(buf, lane, g, ldb, row0, rows_left);
    __syncwarp();
  }
}

// One chunk: rows [row0, row0+32), cols [col, col+CW); v = this lane's row (CW values).
// EPI is a base kind (< kEpiTma); TMA selects the output path (see StageRing).
template <int EPI, bool TMA>
__device__ __forceinline__ void epilogue_chunk(const GemmEpi& ep, const GemmShape& sh,
                                               uint32_t st, StageRing& ring,
                                               const CUtensorMap* tmO, const CUtensorMap* tmO2,
                                               int lane, int64_t row0, int64_t col, int split,
                                               float* v, const ChunkIn& in) {
  const int64_t rows_left = sh.M - row0;
  if constexpr (EPI == RP_EPI_BF16) {
    const uint32_t b = stage_acquire<TMA>(st, ring, lane);
    stage_row_bf16x64(b, lane, v);
    stage_emit<TMA>(b, ring, lane, static_cast<__nv_bfloat16*>(ep.out) + col, ep.ldo * 2, row0,
                    rows_left, tmO, col);
  } else if constexpr (EPI == RP_EPI_F32) {
    if (ep.quant > 0.f) {  // a residual-stream start (embedding / patch merge) on the grid
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = rintf(v[i] * ep.inv_quant) * ep.quant;
    }
    stage_rows_f32(st, lane, v);
    __syncwarp();
    store_tile(st, lane,
               static_cast<float*>(ep.out) + static_cast<int64_t>(split) * ep.split_stride + col,
               ep.ldo * 4, row0, rows_left);
  } else if constexpr (EPI == RP_EPI_BIAS_GELU) {
    if (ep.bias) {
      const float4* b4 = reinterpret_cast<const float4*>(ep.bias + col);
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const float4 b = __ldg(b4 + i);
        v[4 * i] += b.x;
        v[4 * i + 1] += b.y;
        v[4 * i + 2] += b.z;
        v[4 * i + 3] += b.w;
      }
    }
    if (ep.out2) {  // pre-activation u (kept for the backward's gelu')
      const uint32_t b = stage_acquire<TMA>(st, ring, lane);
      stage_row_bf16x64(b, lane, v);
      stage_emit<TMA>(b, ring, lane, static_cast<__nv_bfloat16*>(ep.out2) + col, ep.ldo2 * 2,
                      row0, rows_left, tmO2, col);
    }
#pragma unroll
    for (int i = 0; i < 64; ++i) v[i] = gelu_tanh_fast(v[i]);
    const uint32_t b = stage_acquire<TMA>(st, ring, lane);
    stage_row_bf16x64(b, lane, v);
    stage_emit<TMA>(b, ring, lane, static_cast<__nv_bfloat16*>(ep.out) + col, ep.ldo * 2, row0,
                    rows_left, tmO, col);
  } else if constexpr (EPI == RP_EPI_RESID) {
    const uint32_t b = stage_acquire<TMA>(st, ring, lane);
    uint4 rr[8];
    aux_rows(b, lane, in, rr);
    const float s = ep.sign;
    const float4* b4 = ep.bias ? reinterpret_cast<const float4*>(ep.bias + col) : nullptr;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const float4 bb = b4 ? __ldg(b4 + c) : make_float4(0.f, 0.f, 0.f, 0.f);
      v[4 * c] += bb.x;
      v[4 * c + 1] += bb.y;
      v[4 * c + 2] += bb.z;
      v[4 * c + 3] += bb.w;
    }
    if (ep.quant > 0.f) {  // exact-coupling grid: the sum below is then exact in fp32
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = rintf(v[i] * ep.inv_quant) * ep.quant;
    }
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      v[4 * c] = __fadd_rn(__uint_as_float(rr[c].x), s * v[4 * c]);
      v[4 * c + 1] = __fadd_rn(__uint_as_float(rr[c].y), s * v[4 * c + 1]);
      v[4 * c + 2] = __fadd_rn(__uint_as_float(rr[c].z), s * v[4 * c + 2]);
      v[4 * c + 3] = __fadd_rn(__uint_as_float(rr[c].w), s * v[4 * c + 3]);
    }
    stage_rows_f32(b, lane, v);
    stage_emit<TMA>(b, ring, lane, static_cast<float*>(ep.out) + col, ep.ldo * 4, row0,
                    rows_left, tmO, col);
  } else if constexpr (EPI == RP_EPI_BIAS_GELU_SLOPE) {
    if (ep.bias) {
      const float4* b4 = reinterpret_cast<const float4*>(ep.bias + col);
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const float4 b = __ldg(b4 + i);
        v[4 * i] += b.x;
        v[4 * i + 1] += b.y;
        v[4 * i + 2] += b.z;
        v[4 * i + 3] += b.w;
      }
    }
    float sl[64];
#pragma unroll
    for (int i = 0; i < 64; ++i) gelu_and_slope_fast(v[i], v[i], sl[i]);
    uint32_t b = stage_acquire<TMA>(st, ring, lane);
    stage_row_bf16x64(b, lane, sl);
    stage_emit<TMA>(b, ring, lane, static_cast<__nv_bfloat16*>(ep.out2) + col, ep.ldo2 * 2, row0,
                    rows_left, tmO2, col);
    b = stage_acquire<TMA>(st, ring, lane);
    stage_row_bf16x64(b, lane, v);
    stage_emit<TMA>(b, ring, lane, static_cast<__nv_bfloat16*>(ep.out) + col, ep.ldo * 2, row0,
                    rows_left, tmO, col);
  } else if constexpr (EPI == RP_EPI_ROWDOT) {
    // bf16 output unchanged; D of this lane's row for head col / 64, from the bf16-rounded
    // output (what the attention backward reads as dO) and aux = O
    const uint32_t b = stage_acquire<TMA>(st, ring, lane);
    uint4 uu[8];
    aux_rows(b, lane, in, uu);
    float dot = 0.f;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const uint32_t w[4] = {uu[c].x, uu[c].y, uu[c].z, uu[c].w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float2 o = unpack_bf16x2(w[k]);
        const float2 g = unpack_bf16x2(pack_bf16x2(v[8 * c + 2 * k], v[8 * c + 2 * k + 1]));
        dot = fmaf(g.x, o.x, dot);
        dot = fmaf(g.y, o.y, dot);
      }
    }
    const int64_t row = row0 + lane;
    if (lane < rows_left) {
      const int64_t sq = row / ep.rd_seq, t = row % ep.rd_seq, h = col >> 6;
      ep.rowdot[(sq * ep.rd_heads + h) * ep.rd_seq + t] = dot;
    }
    stage_row_bf16x64(b, lane, v);
    stage_emit<TMA>(b, ring, lane, static_cast<__nv_bfloat16*>(ep.out) + col, ep.ldo * 2, row0,
                    rows_left, tmO, col);
  } else if constexpr (EPI == RP_EPI_MUL || EPI == RP_EPI_GELU_BWD) {
    const uint32_t b = stage_acquire<TMA>(st, ring, lane);
    uint4 uu[8];
    aux_rows(b, lane, in, uu);
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const uint32_t w[4] = {uu[c].x, uu[c].y, uu[c].z, uu[c].w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float2 f = unpack_bf16x2(w[k]);
        if constexpr (EPI == RP_EPI_MUL) {
          v[8 * c + 2 * k] *= f.x;
          v[8 * c + 2 * k + 1] *= f.y;
        } else {
          v[8 * c + 2 * k] *= gelu_tanh_slope_fast(f.x);
          v[8 * c + 2 * k + 1] *= gelu_tanh_slope_fast(f.y);
        }
      }
    }
    if (ep.colsum) colsum_chunk64(ep, b, lane, row0, col, v);
    stage_row_bf16x64(b, lane, v);
    stage_emit<TMA>(b, ring, lane, static_cast<__nv_bfloat16*>(ep.out) + col, ep.ldo * 2, row0,
                    rows_left, tmO, col);
  }
  __syncwarp();
}

template <int BN, bool A_MN, bool B_MN, int EPI>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_sm100_kernel(const __grid_constant__ CUtensorMap tmA,
                      const __grid_constant__ CUtensorMap tmB,
                      const __grid_constant__ CUtensorMap /*tmO: 2-SM TMA store only*/,
                      const __grid_constant__ CUtensorMap /*tmO2*/,
                      const GemmShape sh,
                      const GemmEpi ep) {
  pdl_trigger();

  using Cfg = GemmCfg<BN>;
  constexpr int S = Cfg::kStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + S * Cfg::kABytes;
  uint8_t* sEpi = smem + S * Cfg::kStageBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(sEpi + Cfg::kEpiBytes);
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
      mbar_init(&tempty[i], kEpiWarps);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, Cfg::kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait();

  const int tiles = sh.m_tiles * sh.n_tiles;
  const int units = tiles * sh.splits;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer
      int stage = 0;
      uint32_t phase = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const UnitRange ur = unit_range(sh, u, tiles);
        const int tile = ur.tile, kb0 = ur.kb0, kb1 = ur.kb1;
        const int m0 = (tile / sh.n_tiles) * kBM, n0 = (tile % sh.n_tiles) * BN;
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
    if (sh.issue == 1) {
      // ---------------- MMA issuer, warp-converged: all lanes walk the pipeline, lane 0's
      // predicate issues (same instruction stream and order as below)
      constexpr uint32_t idesc = make_idesc_bf16(kBM, BN, A_MN, B_MN);
      const uint32_t is0 = lane == 0 ? 1u : 0u;
      int stage = 0;
      uint32_t phase = 0;
      const uint64_t adesc0 = A_MN ? make_sdesc_sw128(smem_u32(sA), 8192, 1024)
                                   : make_sdesc_sw128(smem_u32(sA), 16, 1024);
      const uint64_t bdesc0 = B_MN ? make_sdesc_sw128(smem_u32(sB), 8192, 1024)
                                   : make_sdesc_sw128(smem_u32(sB), 16, 1024);
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const UnitRange ur = unit_range(sh, u, tiles);
        const int kb0 = ur.kb0, kb1 = ur.kb1;
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + static_cast<uint32_t>(acc * BN);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint64_t soa = static_cast<uint64_t>((stage * Cfg::kABytes) >> 4);
          const uint64_t sob = static_cast<uint64_t>((stage * Cfg::kBBytes) >> 4);
#pragma unroll
          for (int kk = 0; kk < kBK / 16; ++kk) {
            const uint64_t ad = adesc0 + soa + static_cast<uint64_t>(A_MN ? kk * 128 : kk * 2);
            const uint64_t bd = bdesc0 + sob + static_cast<uint64_t>(B_MN ? kk * 128 : kk * 2);
            umma_bf16_pred(tmem_d, ad, bd, idesc, (kb > kb0 || kk > 0) ? 1u : 0u, is0);
          }
          umma_commit_pred(&empty[stage], is0);
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit_pred(&tfull[acc], is0);
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
      __syncwarp();
    } else if (lane == 0) {
      // ---------------- MMA issuer (single thread issues and commits)
      constexpr uint32_t idesc = make_idesc_bf16(kBM, BN, A_MN, B_MN);
      int stage = 0;
      uint32_t phase = 0;
      const uint64_t adesc0 = A_MN ? make_sdesc_sw128(smem_u32(sA), 8192, 1024)
                                   : make_sdesc_sw128(smem_u32(sA), 16, 1024);
      const uint64_t bdesc0 = B_MN ? make_sdesc_sw128(smem_u32(sB), 8192, 1024)
                                   : make_sdesc_sw128(smem_u32(sB), 16, 1024);
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const UnitRange ur = unit_range(sh, u, tiles);
        const int kb0 = ur.kb0, kb1 = ur.kb1;
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + static_cast<uint32_t>(acc * BN);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint64_t soa = static_cast<uint64_t>((stage * Cfg::kABytes) >> 4);
          const uint64_t sob = static_cast<uint64_t>((stage * Cfg::kBBytes) >> 4);
#pragma unroll
          for (int kk = 0; kk < kBK / 16; ++kk) {
            const uint64_t ad = adesc0 + soa + static_cast<uint64_t>(A_MN ? kk * 128 : kk * 2);
            const uint64_t bd = bdesc0 + sob + static_cast<uint64_t>(B_MN ? kk * 128 : kk * 2);
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
    // ---------------- epilogue warps 2..9: warp w reads TMEM lanes [32*(w%4), +32),
    // column half (w-2)/4 of the tile
    const uint32_t q = warp & 3u;
    const int half = (static_cast<int>(warp) - 2) >> 2;
    const uint32_t st = smem_u32(sEpi + (warp - 2) * kEpiStage);
    StageRing ring{st, 0, 1};
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      const UnitRange ur = unit_range(sh, u, tiles);
      const int split = ur.split, tile = ur.tile;
      const int64_t m0 = static_cast<int64_t>(tile / sh.n_tiles) * kBM;
      const int64_t n0 = static_cast<int64_t>(tile % sh.n_tiles) * BN;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t tbase = tmem_base + ((q * 32u) << 16) + static_cast<uint32_t>(acc * BN);
      const int64_t row0 = m0 + q * 32;
      const int c_begin = half * (BN / 2), c_end = (half + 1) * (BN / 2);
      constexpr int CW = EpiTraits<EPI>::kCW;
      const bool rows_ok = row0 < sh.M;
      ChunkIn nxt;
      if (rows_ok && n0 + c_begin < sh.N)
        prefetch_chunk<EPI>(ep, static_cast<int>(lane), row0, sh.M - row0, n0 + c_begin, nxt);
#pragma unroll 1
      for (int c = c_begin; c < c_end; c += CW) {
        float v[CW];
        if constexpr (CW == 64)
          tmem_ld64(tbase + c, v);
        else
          tmem_ld32(tbase + c, v);
        const ChunkIn cur = nxt;
        if (rows_ok && c + CW < c_end && n0 + c + CW < sh.N)
          prefetch_chunk<EPI>(ep, static_cast<int>(lane), row0, sh.M - row0, n0 + c + CW, nxt);
        if (rows_ok && n0 + c < sh.N)
          epilogue_chunk<EPI, false>(ep, sh, st, ring, nullptr, nullptr, static_cast<int>(lane),
                                     row0, n0 + c, split, v, cur);
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

// ============================================================ 2-SM (CTA pair) variant
// cta_group::2: a cluster of two CTAs on one TPC computes a 256 x 256 tile. CTA r loads
// A rows [m0 + 128 r, +128) and B rows [n0 + 128 r, +128) into its own smem; the leader
// (r = 0) issues tcgen05.mma.cta_group::2 (M = 256, N = 256) which reads both CTAs'
// halves; each CTA's TMEM receives its 128 accumulator rows. Per SM this moves 32 KB of
// operands per 128x256x64 step instead of 48 KB, which is what the L2 can sustain.
// The TMA-store epilogues (kEpiTma + k) store from two staging buffers per warp (the store
// of one chunk drains while the next is computed), paid for with one pipeline stage -- a
// win for short K loops (residual, K = 768: 95.7 -> 87.1 us), a loss for long ones
// (K = 3072: 182 -> 187 us), so plans pick them by K.
template <int EPI>
struct Gemm2Cfg {
  static constexpr bool kTmaStore = EPI >= kEpiTma;
  static constexpr int kTmaBufs = (kTmaStore && EPI < kEpiTma1) ? 2 : 1;
  static constexpr int kStages = kTmaBufs == 2 ? 5 : 6;
  static constexpr int kHalfBytes = 128 * kBK * 2;         // 16 KB: one A or B half stage
  static constexpr int kStageBytes = 2 * kHalfBytes;       // per CTA
  static constexpr int kTmemCols = 512;                    // 2 x 256 accumulator columns
  static constexpr int kEpiBytes = 8 * 4096 * kTmaBufs;
  static constexpr int kSmemBytes = 1024 + kStages * kStageBytes + kEpiBytes + 256;
};

template <bool A_MN, bool B_MN, int EPI>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    gemm_sm100_2sm_kernel(const __grid_constant__ CUtensorMap tmA,
                          const __grid_constant__ CUtensorMap tmB,
                          const __grid_constant__ CUtensorMap tmO,
                          const __grid_constant__ CUtensorMap tmO2, const GemmShape sh,
                          const GemmEpi ep) {
  pdl_trigger();

  using Cfg = Gemm2Cfg<EPI>;
  constexpr int S = Cfg::kStages;
  constexpr int BN = 256;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + S * Cfg::kHalfBytes;
  uint8_t* sEpi = smem + S * Cfg::kStageBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(sEpi + Cfg::kEpiBytes);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  unsigned long long* const gtr = blockIdx.x == 0 ? g_gemm_trace : nullptr;  // instrumentation

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 2 * kEpiWarps);  // both CTAs' epilogue warps (leader's copy)
    }
    fence_barrier_init();
  }
  cluster_sync_all();
  if (warp == 1) tmem_alloc_2sm(tmem_slot, Cfg::kTmemCols);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait();

  const int tiles = sh.m_tiles * sh.n_tiles;  // m_tiles counts 256-row pair tiles
  const int units = tiles * sh.splits;
  const int cluster_id = blockIdx.x >> 1;
  const int nclusters = gridDim.x >> 1;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer (both CTAs, each its own halves)
      int stage = 0;
      uint32_t phase = 0;
      for (int u = cluster_id; u < units; u += nclusters) {
        const UnitRange ur = unit_range(sh, u, tiles);
        const int tile = ur.tile, kb0 = ur.kb0, kb1 = ur.kb1;
        const int m0 = (tile / sh.n_tiles) * 256 + 128 * static_cast<int>(rank);
        // a last tile column of <= 128 valid columns runs as an N = 128 product: each CTA of
        // the pair then supplies 64 columns of B (its first atom / 64 rows)
        const int nt = tile % sh.n_tiles;
        const bool narrow = nt == sh.n_tiles - 1 && sh.N - nt * BN <= 128;
        const int n0 = nt * BN + (narrow ? 64 : 128) * static_cast<int>(rank);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          const uint32_t lbar = mapa_shared(smem_u32(&full[stage]), 0);
          if (leader) mbar_arrive_expect_tx(&full[stage], 2 * Cfg::kStageBytes);
          uint8_t* a = sA + stage * Cfg::kHalfBytes;
          uint8_t* b = sB + stage * Cfg::kHalfBytes;
          const int k0 = kb * kBK;
          if constexpr (A_MN) {
            tma_load_2d_2sm(a, &tmA, lbar, m0, k0);
            tma_load_2d_2sm(a + 8192, &tmA, lbar, m0 + 64, k0);
          } else {
            tma_load_2d_2sm(a, &tmA, lbar, k0, m0);
          }
          if constexpr (B_MN) {
            tma_load_2d_2sm(b, &tmB, lbar, n0, k0);
            tma_load_2d_2sm(b + 8192, &tmB, lbar, n0 + 64, k0);
          } else {
            tma_load_2d_2sm(b, &tmB, lbar, k0, n0);
          }
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (leader && sh.issue == 1) {
      // ---------------- MMA issuer (leader CTA), warp-converged, lane 0's predicate issues
      constexpr uint32_t idesc_full = make_idesc_bf16(256, BN, A_MN, B_MN);
      constexpr uint32_t idesc_narrow = make_idesc_bf16(256, 128, A_MN, B_MN);
      const uint32_t is0 = lane == 0 ? 1u : 0u;
      const uint64_t adesc0 = A_MN ? make_sdesc_sw128(smem_u32(sA), 8192, 1024)
                                   : make_sdesc_sw128(smem_u32(sA), 16, 1024);
      const uint64_t bdesc0 = B_MN ? make_sdesc_sw128(smem_u32(sB), 8192, 1024)
                                   : make_sdesc_sw128(smem_u32(sB), 16, 1024);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      int ti = 0;
      for (int u = cluster_id; u < units; u += nclusters, ++ti) {
        const UnitRange ur = unit_range(sh, u, tiles);
        const int kb0 = ur.kb0, kb1 = ur.kb1;
        const int nt = ur.tile % sh.n_tiles;
        const uint32_t idesc =
            nt == sh.n_tiles - 1 && sh.N - nt * BN <= 128 ? idesc_narrow : idesc_full;
        if (lane == 0) GEMM_TRACE(ti, 0, clock64());
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        if (lane == 0) GEMM_TRACE(ti, 1, clock64());
        long long wfull = 0;
        const uint32_t tmem_d = tmem_base + static_cast<uint32_t>(acc * BN);
        for (int kb = kb0; kb < kb1; ++kb) {
          const long long w0 = clock64();
          mbar_wait(&full[stage], phase);
          wfull += clock64() - w0;
          tc_fence_after();
          // descriptors = stage-0 descriptor + (byte offset >> 4) in the start-address field
          // (no carry: shared addresses < 256 KB), so the issue loop is additions only
          const uint64_t soff = static_cast<uint64_t>((stage * Cfg::kHalfBytes) >> 4);
#pragma unroll
          for (int kk = 0; kk < kBK / 16; ++kk) {
            const uint64_t ad = adesc0 + soff + static_cast<uint64_t>(A_MN ? kk * 128 : kk * 2);
            const uint64_t bd = bdesc0 + soff + static_cast<uint64_t>(B_MN ? kk * 128 : kk * 2);
            umma_bf16_2sm_pred(tmem_d, ad, bd, idesc, (kb > kb0 || kk > 0) ? 1u : 0u, is0);
          }
          umma_commit_2sm_mc_pred(&empty[stage], 0x3, is0);
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit_2sm_mc_pred(&tfull[acc], 0x3, is0);
        if (lane == 0) {
          GEMM_TRACE(ti, 2, wfull);
          GEMM_TRACE(ti, 3, clock64());
        }
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
      __syncwarp();
    } else if (lane == 0 && leader) {
      // ---------------- MMA issuer (leader CTA only)
      constexpr uint32_t idesc_full = make_idesc_bf16(256, BN, A_MN, B_MN);
      constexpr uint32_t idesc_narrow = make_idesc_bf16(256, 128, A_MN, B_MN);
      const uint64_t adesc0 = A_MN ? make_sdesc_sw128(smem_u32(sA), 8192, 1024)
                                   : make_sdesc_sw128(smem_u32(sA), 16, 1024);
      const uint64_t bdesc0 = B_MN ? make_sdesc_sw128(smem_u32(sB), 8192, 1024)
                                   : make_sdesc_sw128(smem_u32(sB), 16, 1024);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int u = cluster_id; u < units; u += nclusters) {
        const UnitRange ur = unit_range(sh, u, tiles);
        const int kb0 = ur.kb0, kb1 = ur.kb1;
        const int nt = ur.tile % sh.n_tiles;
        const uint32_t idesc =
            nt == sh.n_tiles - 1 && sh.N - nt * BN <= 128 ? idesc_narrow : idesc_full;
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + static_cast<uint32_t>(acc * BN);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint64_t soff = static_cast<uint64_t>((stage * Cfg::kHalfBytes) >> 4);
#pragma unroll
          for (int kk = 0; kk < kBK / 16; ++kk) {
            const uint64_t ad = adesc0 + soff + static_cast<uint64_t>(A_MN ? kk * 128 : kk * 2);
            const uint64_t bd = bdesc0 + soff + static_cast<uint64_t>(B_MN ? kk * 128 : kk * 2);
            umma_bf16_2sm(tmem_d, ad, bd, idesc, (kb > kb0 || kk > 0) ? 1u : 0u);
          }
          umma_commit_2sm_mc(&empty[stage], 0x3);
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit_2sm_mc(&tfull[acc], 0x3);
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else {
    // ---------------- epilogue warps 2..9 (both CTAs; this CTA's 128 rows of the tile)
    const uint32_t q = warp & 3u;
    const int half = (static_cast<int>(warp) - 2) >> 2;
    const uint32_t st = smem_u32(sEpi + (warp - 2) * kEpiStage * Cfg::kTmaBufs);
    const uint32_t leader_tempty0 = mapa_shared(smem_u32(&tempty[0]), 0);
    StageRing ring{st, 0, Cfg::kTmaBufs};  // TMA-store staging buffers (kTmaStore)
    int acc = 0;
    uint32_t acc_phase = 0;
    int ti = 0;
    for (int u = cluster_id; u < units; u += nclusters, ++ti) {
      const UnitRange ur = unit_range(sh, u, tiles);
      const int split = ur.split, tile = ur.tile;
      const int64_t m0 = static_cast<int64_t>(tile / sh.n_tiles) * 256 + 128 * rank;
      const int64_t n0 = static_cast<int64_t>(tile % sh.n_tiles) * BN;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      if (warp == 2 && lane == 0) GEMM_TRACE(ti, 4, clock64());
      const uint32_t tbase = tmem_base + ((q * 32u) << 16) + static_cast<uint32_t>(acc * BN);
      const int64_t row0 = m0 + q * 32;
      const int c_begin = half * (BN / 2), c_end = (half + 1) * (BN / 2);
      constexpr int CW = EpiTraits<EPI>::kCW;
      const bool rows_ok = row0 < sh.M;
      ChunkIn nxt;
      if (rows_ok && n0 + c_begin < sh.N)
        prefetch_chunk<EPI>(ep, static_cast<int>(lane), row0, sh.M - row0, n0 + c_begin, nxt);
#pragma unroll 1
      for (int c = c_begin; c < c_end; c += CW) {
        float v[CW];
        if constexpr (CW == 64)
          tmem_ld64(tbase + c, v);
        else
          tmem_ld32(tbase + c, v);
        const ChunkIn cur = nxt;
        if (rows_ok && c + CW < c_end && n0 + c + CW < sh.N)
          prefetch_chunk<EPI>(ep, static_cast<int>(lane), row0, sh.M - row0, n0 + c + CW, nxt);
        if (rows_ok && n0 + c < sh.N)
          epilogue_chunk<base_epi(EPI), Cfg::kTmaStore>(ep, sh, st, ring, &tmO, &tmO2,
                                                        static_cast<int>(lane), row0, n0 + c,
                                                        split, v, cur);
      }
      tc_fence_before();
      __syncwarp();
      if (warp == 2 && lane == 0) GEMM_TRACE(ti, 5, clock64());
      if (lane == 0) mbar_arrive_cluster(leader_tempty0 + static_cast<uint32_t>(acc * 8));
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }

  if constexpr (Cfg::kTmaStore) {
    if (warp >= 2 && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  __syncwarp();
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  if (warp == 1) tmem_dealloc_2sm(tmem_base, Cfg::kTmemCols);
}

// Deterministic split-K reduction: out[i] = sum_{s=0..S-1} part[s][i], fixed order.
__global__ void splitk_reduce_kernel(const float* __restrict__ part, int splits,
                                     int64_t stride, int64_t n4, float* __restrict__ out) {
  pdl_trigger();
  pdl_wait();

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

static int encode_map(CUtensorMap* m, const void* ptr, int64_t rows, int64_t cols, int64_t ld,
                      uint32_t box_rows);
// bf16 output [rows][cols]: box = {64 cols, box_rows rows} (one 32-row epilogue chunk)
static int encode_map_rows(CUtensorMap* m, const void* ptr, int64_t rows, int64_t cols,
                           int64_t ld, uint32_t box_rows) {
  return encode_map(m, ptr, rows, cols, ld, box_rows);
}
// fp32 row-major [rows][cols], pitch ld elements; box = {32 cols, 32 rows} = one epilogue
// chunk, 128-byte swizzle (the staging layout sw32).
static int encode_map_f32(CUtensorMap* m, const void* ptr, int64_t rows, int64_t cols, int64_t ld) {
  PFN_encodeTiled_t fn = get_encode_fn();
  if (!fn) return RP_ERR_CUDA;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 4};
  cuuint32_t box[2] = {32, 32};
  cuuint32_t es[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(ptr), dims, strides,
                  box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? RP_OK : RP_ERR_CUDA;
}

typedef void (*GemmKernelPtr)(CUtensorMap, CUtensorMap, CUtensorMap, CUtensorMap, GemmShape,
                              GemmEpi);

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
    case RP_EPI_BIAS_GELU_SLOPE: return kernel_ptr<BN, A_MN, B_MN, RP_EPI_BIAS_GELU_SLOPE>();
    case RP_EPI_MUL: return kernel_ptr<BN, A_MN, B_MN, RP_EPI_MUL>();
    case RP_EPI_ROWDOT: return kernel_ptr<BN, A_MN, B_MN, RP_EPI_ROWDOT>();
  }
  return nullptr;
}

template <bool A_MN, bool B_MN, int EPI>
static GemmKernelPtr kernel_ptr_2sm() {
  static std::once_flag once;
  auto k = &gemm_sm100_2sm_kernel<A_MN, B_MN, EPI>;
  std::call_once(once, [k] {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         Gemm2Cfg<EPI>::kSmemBytes);
  });
  return reinterpret_cast<GemmKernelPtr>(k);
}

template <bool A_MN, bool B_MN>
static GemmKernelPtr pick_epi_2sm(int epi) {
  switch (epi) {
    case RP_EPI_BF16: return kernel_ptr_2sm<A_MN, B_MN, RP_EPI_BF16>();
    case RP_EPI_F32: return kernel_ptr_2sm<A_MN, B_MN, RP_EPI_F32>();
    case RP_EPI_BIAS_GELU: return kernel_ptr_2sm<A_MN, B_MN, RP_EPI_BIAS_GELU>();
    case RP_EPI_RESID: return kernel_ptr_2sm<A_MN, B_MN, RP_EPI_RESID>();
    case RP_EPI_GELU_BWD: return kernel_ptr_2sm<A_MN, B_MN, RP_EPI_GELU_BWD>();
    case RP_EPI_BIAS_GELU_SLOPE: return kernel_ptr_2sm<A_MN, B_MN, RP_EPI_BIAS_GELU_SLOPE>();
    case RP_EPI_MUL: return kernel_ptr_2sm<A_MN, B_MN, RP_EPI_MUL>();
    case RP_EPI_ROWDOT: return kernel_ptr_2sm<A_MN, B_MN, RP_EPI_ROWDOT>();
    case kEpiTma + RP_EPI_ROWDOT: return kernel_ptr_2sm<A_MN, B_MN, kEpiTma + RP_EPI_ROWDOT>();
    case kEpiTma1 + RP_EPI_ROWDOT:
      return kernel_ptr_2sm<A_MN, B_MN, kEpiTma1 + RP_EPI_ROWDOT>();
    case kEpiTma + RP_EPI_BF16: return kernel_ptr_2sm<A_MN, B_MN, kEpiTma + RP_EPI_BF16>();
    case kEpiTma + RP_EPI_BIAS_GELU:
      return kernel_ptr_2sm<A_MN, B_MN, kEpiTma + RP_EPI_BIAS_GELU>();
    case kEpiTma + RP_EPI_RESID: return kernel_ptr_2sm<A_MN, B_MN, kEpiTma + RP_EPI_RESID>();
    case kEpiTma + RP_EPI_GELU_BWD:
      return kernel_ptr_2sm<A_MN, B_MN, kEpiTma + RP_EPI_GELU_BWD>();
    case kEpiTma + RP_EPI_BIAS_GELU_SLOPE:
      return kernel_ptr_2sm<A_MN, B_MN, kEpiTma + RP_EPI_BIAS_GELU_SLOPE>();
    case kEpiTma + RP_EPI_MUL: return kernel_ptr_2sm<A_MN, B_MN, kEpiTma + RP_EPI_MUL>();
    case kEpiTma1 + RP_EPI_RESID: return kernel_ptr_2sm<A_MN, B_MN, kEpiTma1 + RP_EPI_RESID>();
    case kEpiTma1 + RP_EPI_BF16: return kernel_ptr_2sm<A_MN, B_MN, kEpiTma1 + RP_EPI_BF16>();
    case kEpiTma1 + RP_EPI_BIAS_GELU:
      return kernel_ptr_2sm<A_MN, B_MN, kEpiTma1 + RP_EPI_BIAS_GELU>();
    case kEpiTma1 + RP_EPI_GELU_BWD:
      return kernel_ptr_2sm<A_MN, B_MN, kEpiTma1 + RP_EPI_GELU_BWD>();
    case kEpiTma1 + RP_EPI_BIAS_GELU_SLOPE:
      return kernel_ptr_2sm<A_MN, B_MN, kEpiTma1 + RP_EPI_BIAS_GELU_SLOPE>();
    case kEpiTma1 + RP_EPI_MUL: return kernel_ptr_2sm<A_MN, B_MN, kEpiTma1 + RP_EPI_MUL>();
  }
  return nullptr;
}

static GemmKernelPtr pick_2sm(bool a_mn, bool b_mn, int epi) {
  if (!a_mn && !b_mn) return pick_epi_2sm<false, false>(epi);
  if (!a_mn && b_mn) return pick_epi_2sm<false, true>(epi);
  if (a_mn && !b_mn) return pick_epi_2sm<true, false>(epi);
  return pick_epi_2sm<true, true>(epi);
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
  CUtensorMap tmA, tmB, tmO, tmO2;  // tmO / tmO2: output maps of the TMA-store epilogues
  GemmShape sh;
  GemmEpi ep;
  GemmKernelPtr kern;
  int bn;
  bool two_sm;
  int grid;
  int smem;
  // split-K reduction (only when splits > 1)
  float* red_out;
  int64_t red_n;
};

extern "C" int rp_gemm_plan_set_max_ctas(RpGemmPlan* p, int max_ctas);

extern "C" int rp_gemm_plan_create(const RpGemmDesc* d, RpGemmPlan** out) {
  if (!d || !out) return rp_fail(RP_ERR_CONTRACT, "gemm: null descriptor");
  *out = nullptr;
  const int64_t M = d->M, N = d->N, K = d->K;
  if (M <= 0 || N <= 0 || K <= 0) return rp_fail(RP_ERR_SHAPE, "gemm: empty M/N/K");
  if (N % 64 != 0) return rp_fail(RP_ERR_SHAPE, "gemm: N must be a multiple of 64");
  if (d->lda % 8 || d->ldb % 8 || d->ldo % (d->epi == RP_EPI_F32 || d->epi == RP_EPI_RESID ? 4 : 8))
    return rp_fail(RP_ERR_SHAPE, "gemm: leading dimensions must be 16-byte multiples");
  if ((reinterpret_cast<uintptr_t>(d->A) | reinterpret_cast<uintptr_t>(d->B)) & 15)
    return rp_fail(RP_ERR_SHAPE, "gemm: operands must be 16-byte aligned");
  const bool two_sm = d->bn == 512;  // CTA-pair 256x256 tiles
  const int bn = (d->bn == 128) ? 128 : 256;
  RpGemmPlan* p = new RpGemmPlan();
  p->bn = bn;
  p->two_sm = two_sm;
  p->sh.M = M;
  p->sh.N = N;
  p->sh.K = K;
  p->sh.m_tiles = static_cast<int32_t>((M + (two_sm ? 255 : kBM - 1)) / (two_sm ? 256 : kBM));
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
  p->ep.colsum = d->colsum_part;
  p->ep.ldcs = N;
  p->ep.rowdot = d->rowdot;
  p->ep.rd_seq = d->rd_seq;
  p->ep.rd_heads = N / 64;
  p->ep.quant = 0.f;
  p->ep.inv_quant = 0.f;
  if (d->quantum != 0.f) {
    int ex = 0;
    const float mant = frexpf(d->quantum, &ex);
    if (d->quantum < 0.f || mant != 0.5f || (d->epi != RP_EPI_RESID && d->epi != RP_EPI_F32) ||
        splits > 1) {
      delete p;
      return rp_fail(RP_ERR_CONTRACT,
                     "gemm: quantum must be a power of two, for RESID / unsplit F32 outputs");
    }
    p->ep.quant = d->quantum;
    p->ep.inv_quant = 1.0f / d->quantum;
  }
  if (d->epi == RP_EPI_ROWDOT && (!d->rowdot || !d->aux || d->rd_seq < 1 || N % 64)) {
    delete p;
    return rp_fail(RP_ERR_CONTRACT, "gemm: ROWDOT needs rowdot, aux, rd_seq >= 1, N % 64 == 0");
  }
  if (d->colsum_part && d->epi != RP_EPI_MUL && d->epi != RP_EPI_GELU_BWD) {
    delete p;
    return rp_fail(RP_ERR_CONTRACT, "gemm: colsum_part needs the MUL or GELU_BWD epilogue");
  }
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
      rc = encode_map(&p->tmB, d->B, N, K, d->ldb, two_sm ? 128u : static_cast<uint32_t>(bn));
  }
  // TMA stores pay off for epilogues that also read an input (residual, saved slope / u)
  // or write two outputs; a plain single bf16 output is a little faster on the register
  // path (same-box A/B, K = 768: bf16 134.5 -> 137.4 us; gelu' multiply 286 -> 240-256;
  // bias + GELU + u 226.5 -> 219.4; residual 95.7 -> 87.1)
  int tma_kind = 0;  // 0: register stores; kEpiTma: two buffers; kEpiTma1: one buffer
  // Interleaved same-box A/B (µs, K = 768 unless noted): two staging buffers (one pipeline
  // stage fewer) win for the epilogues that read a bf16 input (gelu' multiply 250 vs 258);
  // one buffer with the full pipeline wins or ties everywhere else (bias + GELU + u 216 vs
  // 221, residual 87.4 vs 88.7 and K = 3072 180.6 vs 187, plain bf16 132.5 vs 135.2 on
  // register stores; bias + GELU + slope 271.4 vs 271.8, tools/gemm_epi_ab.py). The split-K
  // fp32 partials keep register stores.
  if (two_sm && d->epi != RP_EPI_F32)
    tma_kind = (K <= 1024 && (d->epi == RP_EPI_GELU_BWD || d->epi == RP_EPI_MUL ||
                              d->epi == RP_EPI_ROWDOT))
                   ? kEpiTma
                   : kEpiTma1;
  const bool tma_store = tma_kind != 0;
  if (rc == RP_OK && tma_store) {
    if (d->epi == RP_EPI_RESID) {
      rc = encode_map_f32(&p->tmO, d->out, M, N, d->ldo);
    } else {
      rc = encode_map_rows(&p->tmO, d->out, M, N, d->ldo, 32);
      if (rc == RP_OK && d->out2 &&
          (d->epi == RP_EPI_BIAS_GELU || d->epi == RP_EPI_BIAS_GELU_SLOPE))
        rc = encode_map_rows(&p->tmO2, d->out2, M, N, d->ldo2, 32);
    }
  }
  if (rc != RP_OK) {
    delete p;
    return rp_fail(rc, "gemm: cuTensorMapEncodeTiled failed");
  }
  p->kern = two_sm ? pick_2sm(d->a_mn, d->b_mn, tma_store ? tma_kind + d->epi : d->epi)
                   : (bn == 256 ? pick<256>(d->a_mn, d->b_mn, d->epi)
                                : pick<128>(d->a_mn, d->b_mn, d->epi));
  if (!p->kern) {
    delete p;
    return rp_fail(RP_ERR_CONFIG, "gemm: unknown epilogue");
  }
  p->smem = two_sm ? (tma_kind == kEpiTma ? Gemm2Cfg<kEpiTma + RP_EPI_BF16>::kSmemBytes
                              : Gemm2Cfg<RP_EPI_F32>::kSmemBytes)
                   : (bn == 256 ? GemmCfg<256>::kSmemBytes : GemmCfg<128>::kSmemBytes);
  rp_gemm_plan_set_max_ctas(p, d->max_ctas);
  *out = p;
  return RP_OK;
}

extern "C" int rp_set_gemm_trace(void* device_buffer) {
  unsigned long long* p = static_cast<unsigned long long*>(device_buffer);
  return cudaMemcpyToSymbol(g_gemm_trace, &p, sizeof(p)) == cudaSuccess ? RP_OK
                                                                          : rp_fail(RP_ERR_CUDA, "gemm trace");
}

// MMA issue form of the GEMM kernels (A/B switch, read at launch): 1 warp-converged
// predicated issue, 0 a single diverged lane
static int g_mma_issue = 1;
extern "C" int rp_set_mma_issue(int mode) {
  if (mode < 0 || mode > 1) return rp_fail(RP_ERR_CONFIG, "mma issue mode must be 0 or 1");
  g_mma_issue = mode;
  return RP_OK;
}

extern "C" int rp_gemm_plan_launch(const RpGemmPlan* p, rp_stream_t stream_) {
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  if (!p) return RP_ERR_CONTRACT;
  GemmShape sh = p->sh;
  sh.issue = g_mma_issue;
  launch_k(p->kern, dim3(p->grid), dim3(kThreads), p->smem, stream, p->tmA, p->tmB, p->tmO,
           p->tmO2, sh, p->ep);
  if (cudaPeekAtLastError() != cudaSuccess) return rp_check_launch("gemm");
  if (p->sh.splits > 1) {
    const int64_t n4 = p->red_n / 4;
    int blocks = static_cast<int>((n4 + 255) / 256);
    if (blocks > 4 * num_sms()) blocks = 4 * num_sms();
    launch_k(splitk_reduce_kernel, dim3(blocks), dim3(256), 0, stream, static_cast<const float*>(p->ep.out),
                                                     p->sh.splits, p->ep.split_stride, n4,
                                                     p->red_out);
  }
  return rp_check_launch("gemm");
}

extern "C" int rp_gemm_plan_set_max_ctas(RpGemmPlan* p, int max_ctas) {
  if (!p) return RP_ERR_CONTRACT;
  const int units = p->sh.m_tiles * p->sh.n_tiles * p->sh.splits;
  int cap = max_ctas > 0 ? max_ctas : num_sms();
  if (p->two_sm) {  // one unit per CTA pair; grid is a whole number of clusters
    int pairs = cap / 2;
    if (pairs < 1) pairs = 1;
    p->grid = 2 * (units < pairs ? units : pairs);
  } else {
    p->grid = units < cap ? units : cap;
  }
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
