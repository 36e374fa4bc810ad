// tcgen05 attention forward for short sequences (N <= 256 keys, head_dim 64).
//
// Same contract as attn_fwd_kernel in attention.cu (ref:proj/core/src/layers.cpp:150-166:
// scores = (q k^T) * 1/sqrt(hd), row softmax, probs . v), but the two products run on the
// 5th-gen tensor cores with TMEM accumulators:
//   S = Q K^T      tcgen05.mma kind::f16, A = Q (smem), B = K (smem)  -> TMEM cols [0, Nk)
//   softmax        4 warps, one query row per thread, exact (the whole key row fits):
//                  pass 1 row max, pass 2 p = exp2(s*scale*log2e - m) -> bf16 P written
//                  back into TMEM over the already-consumed S columns [0, Nk/2)
//   O = P V        tcgen05.mma with A = P straight from TMEM, B = V (smem, MN-major)
//                  -> TMEM cols [192, 256)
// One CTA per (sequence, head, 128-query tile): 80 KB smem + 256 TMEM columns, so two
// CTAs share an SM and one's loads overlap the other's softmax. Eight softmax warps: warp
// w reads TMEM lane quarter w%4 and key half w/4; the two halves exchange row max / sum
// through smem. P of key half k is written over that half's own (consumed) S columns,
// so no warp overwrites columns another warp may still be reading. Keys beyond N (the next
// sequence's rows, or TMA zero fill past the end) are masked to -inf.
#include <mutex>

#include "../../include/revprop_b200.h"
#include "kernels.h"
#include "ptx.cuh"
#include "launch.h"

namespace rp {
namespace attn_tc {

constexpr int kThreads = 288;  // warps 0-7 softmax / epilogue, warp 8 TMA + MMA issue
constexpr int kTmemCols = 256;
constexpr int kOCol = 192;

struct Geom {
  int B, N, H, Nk;  // sequences, tokens, heads, padded key count (multiple of 32, <= 256)
  int64_t ld_o;
  float scale_log2;
};

__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t* r) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(
                   taddr),
               "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]),
               "r"(r[7])
               : "memory");
}

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// two 16-column TMEM loads behind one tcgen05.wait::ld
__device__ __forceinline__ void tmem_ld16x2(uint32_t ta, uint32_t tb, float* a, float* b) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%32];\n\t"
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%33];\n\t"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
        "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
        "=r"(r[31])
      : "r"(ta), "r"(tb)
      : "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    a[i] = __uint_as_float(r[i]);
    b[i] = __uint_as_float(r[16 + i]);
  }
}

// four 16-column TMEM loads behind one tcgen05.wait::ld
__device__ __forceinline__ void tmem_ld16x4(uint32_t t0, uint32_t t1, uint32_t t2, uint32_t t3,
                                            float* a, float* b, float* c, float* d) {
  uint32_t r[64];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%64];\n\t"
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%65];\n\t"
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47}, [%66];\n\t"
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%67];\n\t"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
        "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
        "=r"(r[31]), "=r"(r[32]), "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]),
        "=r"(r[37]), "=r"(r[38]), "=r"(r[39]), "=r"(r[40]), "=r"(r[41]), "=r"(r[42]),
        "=r"(r[43]), "=r"(r[44]), "=r"(r[45]), "=r"(r[46]), "=r"(r[47]), "=r"(r[48]),
        "=r"(r[49]), "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]),
        "=r"(r[55]), "=r"(r[56]), "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]),
        "=r"(r[61]), "=r"(r[62]), "=r"(r[63])
      : "r"(t0), "r"(t1), "r"(t2), "r"(t3)
      : "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    a[i] = __uint_as_float(r[i]);
    b[i] = __uint_as_float(r[16 + i]);
    c[i] = __uint_as_float(r[32 + i]);
    d[i] = __uint_as_float(r[48 + i]);
  }
}

__device__ __forceinline__ void named_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15])
      : "memory");
}

// D[tmem] (+)= A[tmem] . B[smem]   (A K-major, 16-bit elements packed two per column)
__device__ __forceinline__ void umma_ts_bf16(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc,
                                             uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

__global__ void __launch_bounds__(kThreads, 2)
    attn_fwd_tc_kernel(const __grid_constant__ CUtensorMap tm_q,
                       const __grid_constant__ CUtensorMap tm_kv, __nv_bfloat16* __restrict__ out,
                       float* __restrict__ lse, Geom g) {
  pdl_trigger();

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sQ = smem;                 // 128 x 128 B
  uint8_t* sK = sQ + 128 * 128;       // Nk x 128 B
  uint8_t* sV = sK + 256 * 128;       // Nk x 128 B
  float* red = reinterpret_cast<float*>(sV + 256 * 128);  // [2 halves][128 rows] x 2
  uint64_t* bars = reinterpret_cast<uint64_t*>(red + 4 * 128);
  uint64_t* bar_load = bars;      // TMA bytes
  uint64_t* bar_s = bars + 1;     // S ready (tcgen05.commit)
  uint64_t* bar_p = bars + 2;     // P written to TMEM (4 warp arrivals)
  uint64_t* bar_o = bars + 3;     // O ready (tcgen05.commit)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 4);

  const uint32_t warp = warp_id(), lane = lane_id();
  const int q0 = blockIdx.x * 128, h = blockIdx.y, b = blockIdx.z;
  const int Nk = g.Nk;
  if (warp == 8) {
    if (lane == 0) {
      tma_prefetch_desc(&tm_q);
      tma_prefetch_desc(&tm_kv);
      mbar_init(bar_load, 1);
      mbar_init(bar_s, 1);
      mbar_init(bar_p, 8);
      mbar_init(bar_o, 1);
      fence_barrier_init();
    }
    tmem_alloc(tmem_slot, kTmemCols);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();
  const int row_seq = b * g.N;  // first row of this sequence in qkv [T, 3d]
  const int d = g.H * 64;

  if (warp == 8) {
    if (lane == 0) {
      // ---- loads: Q tile, K and V rows [0, Nk) of this sequence / head
      mbar_arrive_expect_tx(bar_load, (128 + 2 * Nk) * 128);
      tma_load_2d(sQ, &tm_q, bar_load, h * 64, row_seq + q0);
      tma_load_2d(sK, &tm_kv, bar_load, d + h * 64, row_seq);
      tma_load_2d(sV, &tm_kv, bar_load, 2 * d + h * 64, row_seq);
      mbar_wait(bar_load, 0);
      tc_fence_after();
      // ---- S = Q K^T : M = 128, N = Nk, K = 64 (4 x 16)
      const uint32_t idesc_s = make_idesc_bf16(128, static_cast<uint32_t>(Nk), false, false);
      const uint32_t aq = smem_u32(sQ), bk = smem_u32(sK), bv = smem_u32(sV);
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
        umma_bf16(tmem, make_sdesc_sw128(aq + kk * 32, 16, 1024),
                  make_sdesc_sw128(bk + kk * 32, 16, 1024), idesc_s, kk > 0 ? 1u : 0u);
      umma_commit(bar_s);
      // ---- O = P V : M = 128, N = 64, K = Nk (Nk/16 steps); A = P in TMEM cols [0, Nk/2)
      mbar_wait(bar_p, 0);
      tc_fence_after();
      const uint32_t idesc_o = make_idesc_bf16(128, 64, false, true);
      const int half = Nk / 2;
      for (int ks = 0; ks < Nk / 16; ++ks) {
        // key half 0: P at cols [0, half/2); key half 1: P at cols [half, half + half/2)
        const int kcol = ks * 16 < half ? ks * 8 : half + (ks * 16 - half) / 2;
        umma_ts_bf16(tmem + kOCol, tmem + static_cast<uint32_t>(kcol),
                     make_sdesc_sw128(bv + ks * 2048, 8192, 1024), idesc_o, ks > 0 ? 1u : 0u);
      }
      umma_commit(bar_o);
    }
  } else {
    // ---- softmax: warp w owns TMEM lanes / query rows [32(w%4), +32) and key half w/4
    const int q = static_cast<int>(warp & 3u), kh = static_cast<int>(warp >> 2);
    const int half = Nk / 2;
    const int c0 = kh * half;
    const uint32_t lane_base = tmem + ((static_cast<uint32_t>(q) * 32u) << 16);
    const int rloc = q * 32 + static_cast<int>(lane);
    mbar_wait(bar_s, 0);
    tc_fence_after();
    const int valid = g.N;  // keys >= N are masked
    float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
    auto max_chunk = [&](int c, const float* v) {
      if (c + 16 <= valid) {
#pragma unroll
        for (int i = 0; i < 16; ++i) m4[i & 3] = fmaxf(m4[i & 3], v[i]);
      } else {
#pragma unroll
        for (int i = 0; i < 16; ++i)
          if (c + i < valid) m4[i & 3] = fmaxf(m4[i & 3], v[i]);
      }
    };
    {
      int c = c0;
      for (; c + 64 <= c0 + half; c += 64) {
        float v0[16], v1[16], v2[16], v3[16];
        tmem_ld16x4(lane_base + c, lane_base + c + 16, lane_base + c + 32, lane_base + c + 48, v0,
                    v1, v2, v3);
        max_chunk(c, v0);
        max_chunk(c + 16, v1);
        max_chunk(c + 32, v2);
        max_chunk(c + 48, v3);
      }
      for (; c < c0 + half; c += 16) {
        float v[16];
        tmem_ld16(lane_base + c, v);
        max_chunk(c, v);
      }
    }
    red[kh * 128 + rloc] = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3]));
    named_bar(1, 256);
    const float m = fmaxf(red[rloc], red[128 + rloc]);
    const float ms = m * g.scale_log2;
    float l4[4] = {0.f, 0.f, 0.f, 0.f};
    auto p_chunk = [&](int c, const float* v) {
      uint32_t pk[8];
      if (c + 16 <= valid) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float p0 = ex2(fmaf(v[2 * i], g.scale_log2, -ms));
          const float p1 = ex2(fmaf(v[2 * i + 1], g.scale_log2, -ms));
          l4[i & 3] += p0 + p1;
          pk[i] = pack_bf16x2(p0, p1);
        }
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float p0 = (c + 2 * i < valid) ? ex2(fmaf(v[2 * i], g.scale_log2, -ms)) : 0.f;
          const float p1 = (c + 2 * i + 1 < valid) ? ex2(fmaf(v[2 * i + 1], g.scale_log2, -ms)) : 0.f;
          l4[i & 3] += p0 + p1;
          pk[i] = pack_bf16x2(p0, p1);
        }
      }
      // P columns [c0 + (c - c0)/2, +8) lie inside this warp's own, already-read S columns
      tmem_st8(lane_base + c0 + (c - c0) / 2, pk);
    };
    {
      int c = c0;
      for (; c + 32 <= c0 + half; c += 32) {
        float v0[16], v1[16];
        tmem_ld16x2(lane_base + c, lane_base + c + 16, v0, v1);
        p_chunk(c, v0);
        p_chunk(c + 16, v1);
      }
      for (; c < c0 + half; c += 16) {
        float v[16];
        tmem_ld16(lane_base + c, v);
        p_chunk(c, v);
      }
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(bar_p);
    red[256 + kh * 128 + rloc] = (l4[0] + l4[1]) + (l4[2] + l4[3]);
    named_bar(1, 256);
    const float l = red[256 + rloc] + red[256 + 128 + rloc];
    // ---- epilogue: O / l -> bf16 att (32 of the 64 head columns per warp)
    mbar_wait(bar_o, 0);
    tc_fence_after();
    float o[32];
    const int row = q0 + rloc;
    const float inv = 1.0f / l;
    tmem_ld32(lane_base + kOCol + kh * 32, o);
    if (row < g.N) {
      __nv_bfloat16* orow = out + (static_cast<int64_t>(row_seq) + row) * g.ld_o + h * 64 + kh * 32;
      uint4* dst = reinterpret_cast<uint4*>(orow);
#pragma unroll
      for (int j = 0; j < 4; ++j)
        dst[j] = make_uint4(pack_bf16x2(o[8 * j] * inv, o[8 * j + 1] * inv),
                            pack_bf16x2(o[8 * j + 2] * inv, o[8 * j + 3] * inv),
                            pack_bf16x2(o[8 * j + 4] * inv, o[8 * j + 5] * inv),
                            pack_bf16x2(o[8 * j + 6] * inv, o[8 * j + 7] * inv));
      if (kh == 0) lse[(static_cast<int64_t>(b) * g.H + h) * g.N + row] = ms + log2f(l);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 8) tmem_dealloc(tmem, kTmemCols);
}

// ======================================================================= backward
// Two kernels, each output element owned by one CTA (no atomics, bit-reproducible):
//   dq kernel   (CTA per 128-query tile):  S = Q K^T, dP = dO V^T (TMEM),
//               dS = P * (dP - D) * scale with P = exp2(S*scale*log2e - lse) -> bf16 in TMEM,
//               dQ = dS K (A from TMEM)
//   dkdv kernel (CTA per 128-key tile):    S^T = K Q^T, dP^T = V dO^T (TMEM),
//               P^T, dS^T -> bf16 in TMEM, dV = P^T dO, dK = dS^T Q (A from TMEM)
// (ref:proj/core/src/layers.cpp:185-208; softmax VJP ops.cpp:206-225.)
// TMEM: S at [0, 256), dP at [256, 512); the packed bf16 products overwrite the low half of
// each warp's own, already-read columns; accumulators live in columns no one reads any more.
constexpr int kBwdThreads = 288;  // warps 0-7 elementwise, warp 8 TMA + MMA

struct BwdGeom {
  int B, N, H, Nk;
  int64_t ld_o;       // d_out / dqkv column pitch helpers
  int64_t ld_qkv;
  float scale, scale_log2;
};

// dS (or P^T / dS^T) packed column for key/query column c of the warp's half [c0, c0+half)
__device__ __forceinline__ int packed_col(int c, int c0) { return c0 + (c - c0) / 2; }
__device__ __forceinline__ int ts_acol(int ks, int half) {
  return ks * 16 < half ? ks * 8 : half + (ks * 16 - half) / 2;
}

// ------------------------------------------------------------- persistent backward
// Same math as attn_bwd_dq_tc_kernel / attn_bwd_dkdv_tc_kernel, but one CTA per SM loops
// over work items (tile, head, sequence) and double-buffers the TMA loads: item i+1's
// operands stream in while item i is being computed. Per-item barrier phases are i & 1.
struct BwdItems {
  int ntile;  // tiles per (sequence, head)
  int nitems;
};

__device__ __forceinline__ void item_coords(int item, int ntile, int H, int& tile, int& h,
                                            int& b) {
  tile = item % ntile;
  const int bh = item / ntile;
  h = bh % H;
  b = bh / H;
}

__global__ void __launch_bounds__(kBwdThreads, 1)
    attn_bwd_dq_tc_persistent(const __grid_constant__ CUtensorMap tm_q128,
                              const __grid_constant__ CUtensorMap tm_kv,
                              const __grid_constant__ CUtensorMap tm_do128,
                              const float* __restrict__ lse, const float* __restrict__ Dg,
                              __nv_bfloat16* __restrict__ dqkv, BwdGeom g, BwdItems it) {
  pdl_trigger();

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  constexpr int kBuf = (256 + 2 * 256) * 128;  // Q tile | dO tile | K | V
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 2 * kBuf);
  uint64_t* bar_load = bars;  // [2]
  uint64_t* bar_s = bars + 2;
  uint64_t* bar_p = bars + 3;
  uint64_t* bar_o = bars + 4;
  uint64_t* bar_e = bars + 5;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 6);
  const uint32_t warp = warp_id(), lane = lane_id();
  const int Nk = g.Nk, half = Nk / 2;
  const int d = g.H * 64;
  if (warp == 8) {
    if (lane == 0) {
      tma_prefetch_desc(&tm_q128);
      tma_prefetch_desc(&tm_kv);
      tma_prefetch_desc(&tm_do128);
      mbar_init(&bar_load[0], 1);
      mbar_init(&bar_load[1], 1);
      mbar_init(bar_s, 1);
      mbar_init(bar_p, 8);
      mbar_init(bar_o, 1);
      mbar_init(bar_e, 8);
      fence_barrier_init();
    }
    tmem_alloc(tmem_slot, 512);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();
  if (warp == 8) {
    if (lane == 0) {
      auto issue_load = [&](int item, int buf) {
        int tile, h, b;
        item_coords(item, it.ntile, g.H, tile, h, b);
        uint8_t* base = smem + buf * kBuf;
        const int row_seq = b * g.N;
        mbar_arrive_expect_tx(&bar_load[buf], (256 + 2 * Nk) * 128);
        tma_load_2d(base, &tm_q128, &bar_load[buf], h * 64, row_seq + tile * 128);
        tma_load_2d(base + 128 * 128, &tm_do128, &bar_load[buf], h * 64, row_seq + tile * 128);
        tma_load_2d(base + 256 * 128, &tm_kv, &bar_load[buf], d + h * 64, row_seq);
        tma_load_2d(base + 512 * 128, &tm_kv, &bar_load[buf], 2 * d + h * 64, row_seq);
      };
      const uint32_t idesc_s = make_idesc_bf16(128, static_cast<uint32_t>(Nk), false, false);
      const uint32_t idesc_o = make_idesc_bf16(128, 64, false, true);
      int k = 0;
      if (static_cast<int>(blockIdx.x) < it.nitems) issue_load(blockIdx.x, 0);
      for (int item = blockIdx.x; item < it.nitems; item += gridDim.x, ++k) {
        const int buf = k & 1;
        if (item + static_cast<int>(gridDim.x) < it.nitems) issue_load(item + gridDim.x, buf ^ 1);
        mbar_wait(&bar_load[buf], (k >> 1) & 1);
        if (k > 0) mbar_wait(bar_e, (k - 1) & 1);  // previous epilogue done with TMEM
        tc_fence_after();
        const uint32_t base = smem_u32(smem + buf * kBuf);
        const uint32_t aq = base, ao = base + 128 * 128, bk = base + 256 * 128,
                       bv = base + 512 * 128;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          umma_bf16(tmem, make_sdesc_sw128(aq + kk * 32, 16, 1024),
                    make_sdesc_sw128(bk + kk * 32, 16, 1024), idesc_s, kk > 0 ? 1u : 0u);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          umma_bf16(tmem + 256, make_sdesc_sw128(ao + kk * 32, 16, 1024),
                    make_sdesc_sw128(bv + kk * 32, 16, 1024), idesc_s, kk > 0 ? 1u : 0u);
        umma_commit(bar_s);
        mbar_wait(bar_p, k & 1);
        tc_fence_after();
        for (int ks = 0; ks < Nk / 16; ++ks)
          umma_ts_bf16(tmem + 256, tmem + static_cast<uint32_t>(ts_acol(ks, half)),
                       make_sdesc_sw128(bk + ks * 2048, 8192, 1024), idesc_o, ks > 0 ? 1u : 0u);
        umma_commit(bar_o);
        mbar_wait(bar_o, k & 1);  // smem buffer free for the load after next
      }
    }
  } else {
    const int q = static_cast<int>(warp & 3u), kh = static_cast<int>(warp >> 2);
    const int c0 = kh * half;
    const uint32_t lane_base = tmem + ((static_cast<uint32_t>(q) * 32u) << 16);
    int k = 0;
    for (int item = blockIdx.x; item < it.nitems; item += gridDim.x, ++k) {
      int tile, h, b;
      item_coords(item, it.ntile, g.H, tile, h, b);
      const int row_seq = b * g.N;
      const int row = tile * 128 + q * 32 + static_cast<int>(lane);
      const bool row_ok = row < g.N;
      const int64_t hb = (static_cast<int64_t>(b) * g.H + h) * g.N;
      const float lr = row_ok ? lse[hb + row] : 0.f;
      const float dr = row_ok ? Dg[hb + row] : 0.f;
      mbar_wait(bar_s, k & 1);
      tc_fence_after();
      const int valid = g.N;
      const float nds = -dr * g.scale;  // dS = P * (dP*scale - D*scale)
      auto ds_chunk = [&](int c, const float* s, const float* dp) {
        uint32_t pk[8];
        if (c + 16 <= valid) {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float p0 = ex2(fmaf(s[2 * i], g.scale_log2, -lr));
            const float p1 = ex2(fmaf(s[2 * i + 1], g.scale_log2, -lr));
            pk[i] = pack_bf16x2(p0 * fmaf(dp[2 * i], g.scale, nds),
                                p1 * fmaf(dp[2 * i + 1], g.scale, nds));
          }
        } else {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int k0 = c + 2 * i;
            const float p0 = k0 < valid ? ex2(fmaf(s[2 * i], g.scale_log2, -lr)) : 0.f;
            const float p1 = k0 + 1 < valid ? ex2(fmaf(s[2 * i + 1], g.scale_log2, -lr)) : 0.f;
            pk[i] = pack_bf16x2(p0 * fmaf(dp[2 * i], g.scale, nds),
                                p1 * fmaf(dp[2 * i + 1], g.scale, nds));
          }
        }
        tmem_st8(lane_base + packed_col(c, c0), pk);
      };
      int c = c0;
      for (; c + 32 <= c0 + half; c += 32) {
        float s0[16], d0[16], s1[16], d1[16];
        tmem_ld16x4(lane_base + c, lane_base + 256 + c, lane_base + c + 16,
                    lane_base + 256 + c + 16, s0, d0, s1, d1);
        ds_chunk(c, s0, d0);
        ds_chunk(c + 16, s1, d1);
      }
      for (; c < c0 + half; c += 16) {
        float s0[16], d0[16];
        tmem_ld16x2(lane_base + c, lane_base + 256 + c, s0, d0);
        ds_chunk(c, s0, d0);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar_p);
      mbar_wait(bar_o, k & 1);
      tc_fence_after();
      float o[32];
      tmem_ld32(lane_base + 256 + kh * 32, o);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar_e);
      if (row_ok) {
        uint4* dst = reinterpret_cast<uint4*>(
            dqkv + (static_cast<int64_t>(row_seq) + row) * g.ld_qkv + h * 64 + kh * 32);
#pragma unroll
        for (int j = 0; j < 4; ++j)
          dst[j] = make_uint4(pack_bf16x2(o[8 * j], o[8 * j + 1]),
                              pack_bf16x2(o[8 * j + 2], o[8 * j + 3]),
                              pack_bf16x2(o[8 * j + 4], o[8 * j + 5]),
                              pack_bf16x2(o[8 * j + 6], o[8 * j + 7]));
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 8) tmem_dealloc(tmem, 512);
}

__global__ void __launch_bounds__(kBwdThreads, 1)
    attn_bwd_dkdv_tc_persistent(const __grid_constant__ CUtensorMap tm_kv128,
                                const __grid_constant__ CUtensorMap tm_qNk,
                                const __grid_constant__ CUtensorMap tm_doNk,
                                const float* __restrict__ lse, const float* __restrict__ Dg,
                                __nv_bfloat16* __restrict__ dqkv, BwdGeom g, BwdItems it) {
  pdl_trigger();

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  constexpr int kBuf = (256 + 2 * 256) * 128;  // K tile | V tile | Q | dO
  float* sLD = reinterpret_cast<float*>(smem + 2 * kBuf);  // [2 bufs][lse 256 | D 256]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sLD + 2 * 512);
  uint64_t* bar_load = bars;  // [2]
  uint64_t* bar_s = bars + 2;
  uint64_t* bar_p = bars + 3;
  uint64_t* bar_o = bars + 4;
  uint64_t* bar_e = bars + 5;
  uint64_t* bar_ld = bars + 6;  // [2] lse/D staged by the elementwise warps
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 8);
  const uint32_t warp = warp_id(), lane = lane_id();
  const int Nq = g.Nk, half = Nq / 2;
  const int d = g.H * 64;
  if (warp == 8) {
    if (lane == 0) {
      tma_prefetch_desc(&tm_kv128);
      tma_prefetch_desc(&tm_qNk);
      tma_prefetch_desc(&tm_doNk);
      mbar_init(&bar_load[0], 1);
      mbar_init(&bar_load[1], 1);
      mbar_init(bar_s, 1);
      mbar_init(bar_p, 8);
      mbar_init(bar_o, 1);
      mbar_init(bar_e, 8);
      fence_barrier_init();
    }
    tmem_alloc(tmem_slot, 512);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();
  if (warp == 8) {
    if (lane == 0) {
      auto issue_load = [&](int item, int buf) {
        int tile, h, b;
        item_coords(item, it.ntile, g.H, tile, h, b);
        uint8_t* base = smem + buf * kBuf;
        const int row_seq = b * g.N;
        mbar_arrive_expect_tx(&bar_load[buf], (256 + 2 * Nq) * 128);
        tma_load_2d(base, &tm_kv128, &bar_load[buf], d + h * 64, row_seq + tile * 128);
        tma_load_2d(base + 128 * 128, &tm_kv128, &bar_load[buf], 2 * d + h * 64,
                    row_seq + tile * 128);
        tma_load_2d(base + 256 * 128, &tm_qNk, &bar_load[buf], h * 64, row_seq);
        tma_load_2d(base + 512 * 128, &tm_doNk, &bar_load[buf], h * 64, row_seq);
      };
      const uint32_t idesc_s = make_idesc_bf16(128, static_cast<uint32_t>(Nq), false, false);
      const uint32_t idesc_o = make_idesc_bf16(128, 64, false, true);
      int k = 0;
      if (static_cast<int>(blockIdx.x) < it.nitems) issue_load(blockIdx.x, 0);
      for (int item = blockIdx.x; item < it.nitems; item += gridDim.x, ++k) {
        const int buf = k & 1;
        if (item + static_cast<int>(gridDim.x) < it.nitems) issue_load(item + gridDim.x, buf ^ 1);
        mbar_wait(&bar_load[buf], (k >> 1) & 1);
        if (k > 0) mbar_wait(bar_e, (k - 1) & 1);
        tc_fence_after();
        const uint32_t base = smem_u32(smem + buf * kBuf);
        const uint32_t ak = base, av = base + 128 * 128, bq = base + 256 * 128,
                       bo = base + 512 * 128;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          umma_bf16(tmem, make_sdesc_sw128(ak + kk * 32, 16, 1024),
                    make_sdesc_sw128(bq + kk * 32, 16, 1024), idesc_s, kk > 0 ? 1u : 0u);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          umma_bf16(tmem + 256, make_sdesc_sw128(av + kk * 32, 16, 1024),
                    make_sdesc_sw128(bo + kk * 32, 16, 1024), idesc_s, kk > 0 ? 1u : 0u);
        umma_commit(bar_s);
        mbar_wait(bar_p, k & 1);
        tc_fence_after();
        for (int ks = 0; ks < Nq / 16; ++ks) {
          const uint32_t ac = static_cast<uint32_t>(ts_acol(ks, half));
          umma_ts_bf16(tmem + 192, tmem + ac, make_sdesc_sw128(bo + ks * 2048, 8192, 1024),
                       idesc_o, ks > 0 ? 1u : 0u);
          umma_ts_bf16(tmem + 448, tmem + 256 + ac, make_sdesc_sw128(bq + ks * 2048, 8192, 1024),
                       idesc_o, ks > 0 ? 1u : 0u);
        }
        umma_commit(bar_o);
        mbar_wait(bar_o, k & 1);
      }
    }
  } else {
    const int qd = static_cast<int>(warp & 3u), qh = static_cast<int>(warp >> 2);
    const int c0 = qh * half;
    const uint32_t lane_base = tmem + ((static_cast<uint32_t>(qd) * 32u) << 16);
    int k = 0;
    for (int item = blockIdx.x; item < it.nitems; item += gridDim.x, ++k) {
      int tile, h, b;
      item_coords(item, it.ntile, g.H, tile, h, b);
      const int row_seq = b * g.N;
      const int64_t hb = (static_cast<int64_t>(b) * g.H + h) * g.N;
      float* sL = sLD + (k & 1) * 512;
      float* sD = sL + 256;
      for (int i = threadIdx.x; i < Nq; i += 256) {  // -lse and -D*scale per query
        sL[i] = i < g.N ? -lse[hb + i] : -INFINITY;
        sD[i] = i < g.N ? -Dg[hb + i] * g.scale : 0.f;
      }
      named_bar(2, 256);
      const int key = tile * 128 + qd * 32 + static_cast<int>(lane);
      mbar_wait(bar_s, k & 1);
      tc_fence_after();
      auto pds_chunk = [&](int c, const float* s, const float* dp) {
        uint32_t pp[8], pd[8];
        const float4* l4 = reinterpret_cast<const float4*>(sL + c);
        const float4* d4 = reinterpret_cast<const float4*>(sD + c);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float4 nl = l4[j], nd = d4[j];
          const float la[4] = {nl.x, nl.y, nl.z, nl.w}, da[4] = {nd.x, nd.y, nd.z, nd.w};
#pragma unroll
          for (int t = 0; t < 2; ++t) {
            const int e = 4 * j + 2 * t;  // masked queries carry -lse = -inf -> p = 0
            const float p0 = ex2(fmaf(s[e], g.scale_log2, la[2 * t]));
            const float p1 = ex2(fmaf(s[e + 1], g.scale_log2, la[2 * t + 1]));
            pp[2 * j + t] = pack_bf16x2(p0, p1);
            pd[2 * j + t] = pack_bf16x2(p0 * fmaf(dp[e], g.scale, da[2 * t]),
                                        p1 * fmaf(dp[e + 1], g.scale, da[2 * t + 1]));
          }
        }
        tmem_st8(lane_base + packed_col(c, c0), pp);
        tmem_st8(lane_base + 256 + packed_col(c, c0), pd);
      };
      int c = c0;
      for (; c + 32 <= c0 + half; c += 32) {
        float s0[16], d0[16], s1[16], d1[16];
        tmem_ld16x4(lane_base + c, lane_base + 256 + c, lane_base + c + 16,
                    lane_base + 256 + c + 16, s0, d0, s1, d1);
        pds_chunk(c, s0, d0);
        pds_chunk(c + 16, s1, d1);
      }
      for (; c < c0 + half; c += 16) {
        float s0[16], d0[16];
        tmem_ld16x2(lane_base + c, lane_base + 256 + c, s0, d0);
        pds_chunk(c, s0, d0);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar_p);
      mbar_wait(bar_o, k & 1);
      tc_fence_after();
      float o[32], o2[32];
      tmem_ld32(lane_base + 448 + qh * 32, o);   // dK
      tmem_ld32(lane_base + 192 + qh * 32, o2);  // dV
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar_e);
      if (key < g.N) {
        __nv_bfloat16* base =
            dqkv + (static_cast<int64_t>(row_seq) + key) * g.ld_qkv + h * 64 + qh * 32;
        uint4* dk = reinterpret_cast<uint4*>(base + d);
        uint4* dv = reinterpret_cast<uint4*>(base + 2 * d);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          dk[j] = make_uint4(pack_bf16x2(o[8 * j], o[8 * j + 1]), pack_bf16x2(o[8 * j + 2], o[8 * j + 3]),
                             pack_bf16x2(o[8 * j + 4], o[8 * j + 5]),
                             pack_bf16x2(o[8 * j + 6], o[8 * j + 7]));
          dv[j] = make_uint4(pack_bf16x2(o2[8 * j], o2[8 * j + 1]),
                             pack_bf16x2(o2[8 * j + 2], o2[8 * j + 3]),
                             pack_bf16x2(o2[8 * j + 4], o2[8 * j + 5]),
                             pack_bf16x2(o2[8 * j + 6], o2[8 * j + 7]));
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 8) tmem_dealloc(tmem, 512);
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                             const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                             const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeFn encode_fn() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  });
  return fn;
}

static int make_map(CUtensorMap* m, const void* base, int64_t rows, int64_t cols, uint32_t box_rows) {
  EncodeFn fn = encode_fn();
  if (!fn) return RP_ERR_CUDA;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(cols) * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t es[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS
             ? RP_OK
             : RP_ERR_CUDA;
}

}  // namespace attn_tc
}  // namespace rp

using namespace rp;

// Returns RP_ERR_CONFIG (without launching) when the shape is outside the tcgen05 path;
// the caller then uses the mma.sync kernel.
int rp_attention_fwd_tc(const uint16_t* qkv, int64_t S, int64_t N, int64_t H, uint16_t* out,
                        float* lse, cudaStream_t stream) {
  using namespace attn_tc;
  if (N > 256 || N < 1) return RP_ERR_CONFIG;
  Geom g;
  g.B = static_cast<int>(S);
  g.N = static_cast<int>(N);
  g.H = static_cast<int>(H);
  g.Nk = static_cast<int>((N + 31) / 32 * 32);
  g.ld_o = H * 64;
  g.scale_log2 = (1.0f / 8.0f) * 1.4426950408889634f;
  const int64_t T = S * N, cols = 3 * H * 64;
  CUtensorMap mq, mkv;
  if (make_map(&mq, qkv, T, cols, 128) || make_map(&mkv, qkv, T, cols, static_cast<uint32_t>(g.Nk)))
    return rp_fail(RP_ERR_CUDA, "attention_tc: tensor map encode failed");
  const int smem = 1024 + (128 + 2 * 256) * 128 + 4 * 128 * 4 + 64;
  static std::once_flag once;
  std::call_once(once, [smem] {
    cudaFuncSetAttribute(attn_fwd_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  });
  dim3 grid(static_cast<unsigned>((N + 127) / 128), static_cast<unsigned>(H),
            static_cast<unsigned>(S));
  launch_k(attn_fwd_tc_kernel, dim3(grid), dim3(kThreads), smem, stream, 
      mq, mkv, reinterpret_cast<__nv_bfloat16*>(out), lse, g);
  return rp_check_launch("attention_fwd_tc");
}

// Backward on the tcgen05 path (N <= 256). D = rowsum(dO * O) must already be in `Dg`.
int rp_attention_bwd_tc(const uint16_t* qkv, const uint16_t* dout, const float* lse,
                        const float* Dg, int64_t S, int64_t N, int64_t H, uint16_t* dqkv,
                        cudaStream_t stream) {
  using namespace attn_tc;
  if (N > 256 || N < 1) return RP_ERR_CONFIG;
  BwdGeom g;
  g.B = static_cast<int>(S);
  g.N = static_cast<int>(N);
  g.H = static_cast<int>(H);
  g.Nk = static_cast<int>((N + 31) / 32 * 32);
  g.ld_o = H * 64;
  g.ld_qkv = 3 * H * 64;
  g.scale = 1.0f / 8.0f;
  g.scale_log2 = g.scale * 1.4426950408889634f;
  const int64_t T = S * N;
  CUtensorMap q128, kvNk, do128, kv128, qNk, doNk;
  if (make_map(&q128, qkv, T, 3 * H * 64, 128) ||
      make_map(&kvNk, qkv, T, 3 * H * 64, static_cast<uint32_t>(g.Nk)) ||
      make_map(&do128, dout, T, H * 64, 128) || make_map(&kv128, qkv, T, 3 * H * 64, 128) ||
      make_map(&qNk, qkv, T, 3 * H * 64, static_cast<uint32_t>(g.Nk)) ||
      make_map(&doNk, dout, T, H * 64, static_cast<uint32_t>(g.Nk)))
    return rp_fail(RP_ERR_CUDA, "attention_bwd_tc: tensor map encode failed");
  const int smem_dq = 1024 + 2 * (256 + 2 * 256) * 128 + 128;
  const int smem_kv = 1024 + 2 * (256 + 2 * 256) * 128 + 2 * 512 * 4 + 128;
  static std::once_flag once;
  static int nsm = 148;
  std::call_once(once, [smem_dq, smem_kv] {
    cudaFuncSetAttribute(attn_bwd_dq_tc_persistent, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         smem_dq);
    cudaFuncSetAttribute(attn_bwd_dkdv_tc_persistent,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem_kv);
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  });
  BwdItems items;
  items.ntile = static_cast<int>((N + 127) / 128);
  items.nitems = static_cast<int>(S * H) * items.ntile;
  const unsigned grid = static_cast<unsigned>(items.nitems < nsm ? items.nitems : nsm);
  launch_k(attn_bwd_dkdv_tc_persistent, dim3(grid), dim3(kBwdThreads), smem_kv, stream, 
      kv128, qNk, doNk, lse, Dg, reinterpret_cast<__nv_bfloat16*>(dqkv), g, items);
  launch_k(attn_bwd_dq_tc_persistent, dim3(grid), dim3(kBwdThreads), smem_dq, stream, 
      q128, kvNk, do128, lse, Dg, reinterpret_cast<__nv_bfloat16*>(dqkv), g, items);
  return rp_check_launch("attention_bwd_tc");
}
