// tcgen05 attention backward for short sequences (N <= 256, head_dim 64).
//
// ref:proj/core/src/layers.cpp:185-208 (per head: dA = dO V^T, dV = A^T dO,
// dS = softmax_vjp(A, dA) / sqrt(hd), dQ = dS K, dK = dS^T Q; softmax VJP ops.cpp:206-225),
// recomputing the probabilities from the forward's log2-domain LSE instead of storing them.
// Two kernels, each output element owned by exactly one CTA (no atomics, bit-reproducible):
//
//   attn_bwd_dq_tc    item = (128-query tile, head, sequence); first D = rowsum(dO * O)
//                     for its rows (written out for the dK/dV kernel), then per 64-key chunk
//                       S = Q K_c^T, dP = dO V_c^T                 (TMEM, M = 128, N = 64)
//                       dS = P * (dP - D) * scale, P = exp2(S * scale * log2e - lse)
//                       dQ += dS K_c      (A = dS re-packed to bf16 in TMEM)
//   attn_bwd_dkdv_tc  item = (128-key tile, head, sequence); per 64-query chunk
//                       S^T = K Q_c^T, dP^T = V dO_c^T
//                       P^T, dS^T (bf16, TMEM);  dV += P^T dO_c,  dK += dS^T Q_c
//
// Each CTA needs 256 TMEM columns (S | dP | one or two 64-column accumulators) and ~100 KB
// of smem, so two CTAs share an SM: one's elementwise phase overlaps the other's MMAs and
// loads. Both kernels are persistent over their items (grid = 2 x SMs). Chunk widths are
// trimmed to the padded sequence length (multiple of 16), so no MMA reads rows the TMA did
// not write; keys / queries past N are masked explicitly (P = dS = 0).
#include "attn_common.cuh"
#include "launch.h"

namespace rp {
namespace attn_tc {

constexpr int kBwdWarps = 9;  // warps 0-7 elementwise (lane quarter w%4, column half w/4), 8 TMA+MMA
constexpr int kBwdThreads = kBwdWarps * 32;
constexpr int kBwdSmem = (2 * 128 + 2 * 256) * 128;  // two 128-row + two 256-row operand tiles

struct BwdGeom {
  int B, N, H, Nk;    // sequences, tokens, heads, N rounded up to 16
  int64_t ld_o;       // row pitch of O / dO (H * 64)
  int64_t ld_qkv;     // row pitch of qkv / dqkv (3 H * 64)
  float scale, scale_log2;
};

struct BwdPlan {
  int ntile;   // 128-row tiles per (sequence, head)
  int nitems;  // ntile * B * H
};

// Optional timeline trace of CTA 0 (diagnostics): slot e of chunk u at g_trace[u * 8 + e].
__device__ long long g_trace[8 * 64];
__device__ int g_trace_on;
__device__ __forceinline__ void trace(int u, int e) {
  if (g_trace_on && blockIdx.x == 0 && u < 64) g_trace[u * 8 + e] = clock64();
}

__device__ __forceinline__ void item_coords(int item, int ntile, int H, int& tile, int& h,
                                            int& b) {
  tile = item % ntile;
  const int bh = item / ntile;
  h = bh % H;
  b = bh / H;
}

// packed bf16 column of the A operand for K-step ks (16 columns) of a 64-column chunk whose
// halves [0, 32) / [32, 64) were packed into their own first 16 columns
__device__ __forceinline__ uint32_t chunk_acol(int ks) {
  return static_cast<uint32_t>((ks >> 1) * 32 + (ks & 1) * 8);
}

__device__ __forceinline__ void store_row32_bf16(__nv_bfloat16* dst, const float* o) {
  uint4* d4 = reinterpret_cast<uint4*>(dst);
#pragma unroll
  for (int j = 0; j < 4; ++j)
    d4[j] = make_uint4(pack_bf16x2(o[8 * j], o[8 * j + 1]), pack_bf16x2(o[8 * j + 2], o[8 * j + 3]),
                       pack_bf16x2(o[8 * j + 4], o[8 * j + 5]),
                       pack_bf16x2(o[8 * j + 6], o[8 * j + 7]));
}

// ------------------------------------------------------------------------------ dQ (+ D)
__global__ void __launch_bounds__(kBwdThreads, 2)
    attn_bwd_dq_tc(const __grid_constant__ CUtensorMap tm_q128,
                   const __grid_constant__ CUtensorMap tm_do128,
                   const __grid_constant__ CUtensorMap tm_kvNk,
                   const __nv_bfloat16* __restrict__ O, const float* __restrict__ lse,
                   float* __restrict__ Dg, __nv_bfloat16* __restrict__ dqkv, BwdGeom g,
                   BwdPlan pl) {
  pdl_trigger();

  __shared__ float red[2][128];
  __shared__ __align__(8) uint64_t bars[5];
  __shared__ uint32_t tmem_slot;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sQ = smem;                // 128 rows
  uint8_t* sDO = smem + 16384;       // 128 rows
  uint8_t* sK = smem + 32768;        // Nk rows (<= 256)
  uint8_t* sV = smem + 65536;        // Nk rows
  uint64_t* bar_load = bars;
  uint64_t* bar_s = bars + 1;  // S, dP of a chunk ready
  uint64_t* bar_p = bars + 2;  // dS of a chunk in TMEM (8 warps)
  uint64_t* bar_o = bars + 3;  // dQ of the item complete
  uint64_t* bar_e = bars + 4;  // dQ read out of TMEM (8 warps)

  const uint32_t warp = warp_id(), lane = lane_id();
  if (warp == 8) {
    if (lane == 0) {
      tma_prefetch_desc(&tm_q128);
      tma_prefetch_desc(&tm_do128);
      tma_prefetch_desc(&tm_kvNk);
      mbar_init(bar_load, 1);
      mbar_init(bar_s, 1);
      mbar_init(bar_p, 8);
      mbar_init(bar_o, 1);
      mbar_init(bar_e, 8);
      fence_barrier_init();
    }
    tmem_alloc(&tmem_slot, 256);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;
  pdl_wait();
  const int Nk = g.Nk, d = g.H * 64;
  const int nch = (Nk + 63) / 64;

  if (warp == 8) {
    if (lane == 0) {
      const uint32_t aq = smem_u32(sQ), ado = smem_u32(sDO), bk = smem_u32(sK), bv = smem_u32(sV);
      auto issue_load = [&](int item) {
        int tile, h, b;
        item_coords(item, pl.ntile, g.H, tile, h, b);
        const int row_seq = b * g.N;
        mbar_arrive_expect_tx(bar_load, (256 + 2 * Nk) * 128);
        tma_load_2d(sQ, &tm_q128, bar_load, h * 64, row_seq + tile * 128);
        tma_load_2d(sDO, &tm_do128, bar_load, h * 64, row_seq + tile * 128);
        tma_load_2d(sK, &tm_kvNk, bar_load, d + h * 64, row_seq);
        tma_load_2d(sV, &tm_kvNk, bar_load, 2 * d + h * 64, row_seq);
      };
      const uint32_t idesc_dq = make_idesc_bf16(128, 64, false, true);
      int k = 0, u = 0;
      if (static_cast<int>(blockIdx.x) < pl.nitems) issue_load(blockIdx.x);
      for (int item = blockIdx.x; item < pl.nitems; item += gridDim.x, ++k) {
        mbar_wait(bar_load, k & 1);
        tc_fence_after();
        for (int c = 0; c < nch; ++c, ++u) {
          const int w = min(64, Nk - 64 * c);
          const uint32_t idesc_s = make_idesc_bf16(128, static_cast<uint32_t>(w), false, false);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            umma_bf16(tmem, make_sdesc_sw128(aq + kk * 32, 16, 1024),
                      make_sdesc_sw128(bk + 64 * c * 128 + kk * 32, 16, 1024), idesc_s,
                      kk > 0 ? 1u : 0u);
            umma_bf16(tmem + 64, make_sdesc_sw128(ado + kk * 32, 16, 1024),
                      make_sdesc_sw128(bv + 64 * c * 128 + kk * 32, 16, 1024), idesc_s,
                      kk > 0 ? 1u : 0u);
          }
          umma_commit(bar_s);
          if (c == 0 && k > 0) mbar_wait(bar_e, (k - 1) & 1);  // previous dQ read out
          mbar_wait(bar_p, u & 1);
          tc_fence_after();
          for (int ks = 0; ks < w / 16; ++ks)
            umma_ts_bf16(tmem + 128, tmem + chunk_acol(ks),
                         make_sdesc_sw128(bk + (64 * c + 16 * ks) * 128, 8192, 1024), idesc_dq,
                         (c > 0 || ks > 0) ? 1u : 0u);
        }
        umma_commit(bar_o);
        mbar_wait(bar_o, k & 1);  // every MMA of this item retired: smem reusable
        const int nxt = item + static_cast<int>(gridDim.x);
        if (nxt < pl.nitems) issue_load(nxt);
      }
    }
  } else {
    const int q = static_cast<int>(warp & 3u), kh = static_cast<int>(warp >> 2);
    const uint32_t lq = (static_cast<uint32_t>(q) * 32u) << 16;
    const int rloc = q * 32 + static_cast<int>(lane);
    int k = 0, u = 0;
    for (int item = blockIdx.x; item < pl.nitems; item += gridDim.x, ++k) {
      int tile, h, b;
      item_coords(item, pl.ntile, g.H, tile, h, b);
      const int row = tile * 128 + rloc;
      const bool row_ok = row < g.N;
      const bool active = tile * 128 + q * 32 < g.N;
      const int64_t grow = static_cast<int64_t>(b) * g.N + row;
      const int64_t hb = (static_cast<int64_t>(b) * g.H + h) * g.N;
      const float lr = row_ok ? lse[hb + row] : 0.f;
      // ---- D = rowsum(dO * O) over this warp's 32 head columns, then across the pair
      mbar_wait(bar_load, k & 1);
      float dpart = 0.f;
      if (row_ok) {
        const uint4* o4 = reinterpret_cast<const uint4*>(O + grow * g.ld_o + h * 64 + kh * 32);
        const uint8_t* drow = sDO + rloc * 128;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const uint4 ov = __ldg(o4 + c);
          const int cc = kh * 4 + c;
          const uint4 dv = *reinterpret_cast<const uint4*>(drow + ((cc ^ (rloc & 7)) << 4));
          const uint32_t ow[4] = {ov.x, ov.y, ov.z, ov.w}, dw[4] = {dv.x, dv.y, dv.z, dv.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 a = unpack_bf16x2(ow[e]), bb = unpack_bf16x2(dw[e]);
            dpart = fmaf(a.x, bb.x, dpart);
            dpart = fmaf(a.y, bb.y, dpart);
          }
        }
      }
      red[kh][rloc] = dpart;
      named_bar(1, 256);
      const float D = red[0][rloc] + red[1][rloc];
      if (kh == 0 && row_ok) Dg[hb + row] = D;
      const float nds = -D * g.scale;
      for (int c = 0; c < nch; ++c, ++u) {
        const int w = min(64, Nk - 64 * c);
        mbar_wait(bar_s, u & 1);
        tc_fence_after();
        if (active && 32 * kh < w) {
          const uint32_t ts = tmem + lq + static_cast<uint32_t>(32 * kh);
          // two 16-key halves; half hh is packed to columns [8 hh, 8 hh + 8) of this warp's
          // 32, which it (half 0) or the earlier half (half 1) has already read
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const int key0 = 64 * c + 32 * kh + 16 * hh;
            if (key0 - 64 * c >= w) break;
            float s[16], dp[16];
            tmem_ld16x2(ts + 16 * hh, ts + 64 + 16 * hh, s, dp);
            uint32_t pk[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              const int key = key0 + 2 * e;
              const float p0 = key < g.N ? ex2(fmaf(s[2 * e], g.scale_log2, -lr)) : 0.f;
              const float p1 = key + 1 < g.N ? ex2(fmaf(s[2 * e + 1], g.scale_log2, -lr)) : 0.f;
              const float d0 = key < g.N ? p0 * fmaf(dp[2 * e], g.scale, nds) : 0.f;
              const float d1 = key + 1 < g.N ? p1 * fmaf(dp[2 * e + 1], g.scale, nds) : 0.f;
              pk[e] = pack_bf16x2(d0, d1);
            }
            tmem_st8(ts + 8 * hh, pk);
          }
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(bar_p);
      }
      // ---- dQ epilogue
      mbar_wait(bar_o, k & 1);
      tc_fence_after();
      float o[32];
      if (active) tmem_ld32(tmem + lq + 128 + static_cast<uint32_t>(32 * kh), o);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar_e);
      if (row_ok) store_row32_bf16(dqkv + grow * g.ld_qkv + h * 64 + kh * 32, o);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 8) tmem_dealloc(tmem, 256);
}

// ---------------------------------------------------------------------------- dK, dV
__global__ void __launch_bounds__(kBwdThreads, 2)
    attn_bwd_dkdv_tc(const __grid_constant__ CUtensorMap tm_kv128,
                     const __grid_constant__ CUtensorMap tm_qNk,
                     const __grid_constant__ CUtensorMap tm_doNk,
                     const float* __restrict__ lse, const float* __restrict__ Dg,
                     __nv_bfloat16* __restrict__ dqkv, BwdGeom g, BwdPlan pl) {
  pdl_trigger();

  __shared__ float sL[256], sD[256];  // -lse and -D * scale per query (-inf / 0 past N)
  __shared__ __align__(8) uint64_t bars[5];
  __shared__ uint32_t tmem_slot;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sK = smem;            // 128 rows
  uint8_t* sV = smem + 16384;    // 128 rows
  uint8_t* sQ = smem + 32768;    // Nk rows (<= 256)
  uint8_t* sDO = smem + 65536;   // Nk rows
  uint64_t* bar_load = bars;
  uint64_t* bar_s = bars + 1;
  uint64_t* bar_p = bars + 2;
  uint64_t* bar_o = bars + 3;
  uint64_t* bar_e = bars + 4;

  const uint32_t warp = warp_id(), lane = lane_id();
  if (warp == 8) {
    if (lane == 0) {
      tma_prefetch_desc(&tm_kv128);
      tma_prefetch_desc(&tm_qNk);
      tma_prefetch_desc(&tm_doNk);
      mbar_init(bar_load, 1);
      mbar_init(bar_s, 1);
      mbar_init(bar_p, 8);
      mbar_init(bar_o, 1);
      mbar_init(bar_e, 8);
      fence_barrier_init();
    }
    tmem_alloc(&tmem_slot, 256);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;
  pdl_wait();
  const int Nq = g.Nk, d = g.H * 64;
  const int nch = (Nq + 63) / 64;

  if (warp == 8) {
    if (lane == 0) {
      const uint32_t ak = smem_u32(sK), av = smem_u32(sV), bq = smem_u32(sQ), bdo = smem_u32(sDO);
      auto issue_load = [&](int item) {
        int tile, h, b;
        item_coords(item, pl.ntile, g.H, tile, h, b);
        const int row_seq = b * g.N;
        mbar_arrive_expect_tx(bar_load, (256 + 2 * Nq) * 128);
        tma_load_2d(sK, &tm_kv128, bar_load, d + h * 64, row_seq + tile * 128);
        tma_load_2d(sV, &tm_kv128, bar_load, 2 * d + h * 64, row_seq + tile * 128);
        tma_load_2d(sQ, &tm_qNk, bar_load, h * 64, row_seq);
        tma_load_2d(sDO, &tm_doNk, bar_load, h * 64, row_seq);
      };
      const uint32_t idesc_o = make_idesc_bf16(128, 64, false, true);
      int k = 0, u = 0;
      if (static_cast<int>(blockIdx.x) < pl.nitems) issue_load(blockIdx.x);
      for (int item = blockIdx.x; item < pl.nitems; item += gridDim.x, ++k) {
        mbar_wait(bar_load, k & 1);
        tc_fence_after();
        for (int c = 0; c < nch; ++c, ++u) {
          const int w = min(64, Nq - 64 * c);
          const uint32_t idesc_s = make_idesc_bf16(128, static_cast<uint32_t>(w), false, false);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            umma_bf16(tmem, make_sdesc_sw128(ak + kk * 32, 16, 1024),
                      make_sdesc_sw128(bq + 64 * c * 128 + kk * 32, 16, 1024), idesc_s,
                      kk > 0 ? 1u : 0u);
            umma_bf16(tmem + 64, make_sdesc_sw128(av + kk * 32, 16, 1024),
                      make_sdesc_sw128(bdo + 64 * c * 128 + kk * 32, 16, 1024), idesc_s,
                      kk > 0 ? 1u : 0u);
          }
          umma_commit(bar_s);
          trace(u, 0);
          if (c == 0 && k > 0) mbar_wait(bar_e, (k - 1) & 1);  // previous dK / dV read out
          mbar_wait(bar_p, u & 1);
          trace(u, 1);
          tc_fence_after();
          for (int ks = 0; ks < w / 16; ++ks) {
            const uint32_t row16 = static_cast<uint32_t>((64 * c + 16 * ks) * 128);
            const uint32_t acc = (c > 0 || ks > 0) ? 1u : 0u;
            umma_ts_bf16(tmem + 128, tmem + chunk_acol(ks),
                         make_sdesc_sw128(bdo + row16, 8192, 1024), idesc_o, acc);  // dV
            umma_ts_bf16(tmem + 192, tmem + 64 + chunk_acol(ks),
                         make_sdesc_sw128(bq + row16, 8192, 1024), idesc_o, acc);   // dK
          }
        }
        umma_commit(bar_o);
        mbar_wait(bar_o, k & 1);
        const int nxt = item + static_cast<int>(gridDim.x);
        if (nxt < pl.nitems) issue_load(nxt);
      }
    }
  } else {
    const int q = static_cast<int>(warp & 3u), kh = static_cast<int>(warp >> 2);
    const uint32_t lq = (static_cast<uint32_t>(q) * 32u) << 16;
    const int rloc = q * 32 + static_cast<int>(lane);
    int k = 0, u = 0;
    for (int item = blockIdx.x; item < pl.nitems; item += gridDim.x, ++k) {
      int tile, h, b;
      item_coords(item, pl.ntile, g.H, tile, h, b);
      const int key = tile * 128 + rloc;
      const bool active = tile * 128 + q * 32 < g.N;
      const int64_t hb = (static_cast<int64_t>(b) * g.H + h) * g.N;
      for (int i = static_cast<int>(threadIdx.x); i < 256; i += 256) {
        sL[i] = i < g.N ? -lse[hb + i] : -INFINITY;
        sD[i] = i < g.N ? -Dg[hb + i] * g.scale : 0.f;
      }
      named_bar(1, 256);
      for (int c = 0; c < nch; ++c, ++u) {
        const int w = min(64, Nq - 64 * c);
        mbar_wait(bar_s, u & 1);
        if (threadIdx.x == 0) trace(u, 2);
        tc_fence_after();
        if (active && 32 * kh < w) {
          const uint32_t ts = tmem + lq + static_cast<uint32_t>(32 * kh);
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const int q0 = 64 * c + 32 * kh + 16 * hh;
            if (q0 - 64 * c >= w) break;
            float s[16], dp[16];
            tmem_ld16x2(ts + 16 * hh, ts + 64 + 16 * hh, s, dp);
            uint32_t pp[8], pd[8];
            const float4* l4 = reinterpret_cast<const float4*>(sL + q0);
            const float4* d4 = reinterpret_cast<const float4*>(sD + q0);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const float4 nl = l4[j], nd = d4[j];
              const float la[4] = {nl.x, nl.y, nl.z, nl.w}, da[4] = {nd.x, nd.y, nd.z, nd.w};
#pragma unroll
              for (int t = 0; t < 2; ++t) {
                const int e = 4 * j + 2 * t;
                const bool v0 = q0 + e < g.N, v1 = q0 + e + 1 < g.N;
                const float p0 = v0 ? ex2(fmaf(s[e], g.scale_log2, la[2 * t])) : 0.f;
                const float p1 = v1 ? ex2(fmaf(s[e + 1], g.scale_log2, la[2 * t + 1])) : 0.f;
                pp[2 * j + t] = pack_bf16x2(p0, p1);
                pd[2 * j + t] =
                    pack_bf16x2(v0 ? p0 * fmaf(dp[e], g.scale, da[2 * t]) : 0.f,
                                v1 ? p1 * fmaf(dp[e + 1], g.scale, da[2 * t + 1]) : 0.f);
              }
            }
            tmem_st8(ts + 8 * hh, pp);       // P^T over this warp's own, read S^T columns
            tmem_st8(ts + 64 + 8 * hh, pd);  // dS^T over its own dP^T columns
          }
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        }
        tc_fence_before();
        __syncwarp();
        if (threadIdx.x == 0) trace(u, 3);
        if (lane == 0) mbar_arrive(bar_p);
      }
      mbar_wait(bar_o, k & 1);
      tc_fence_after();
      __nv_bfloat16* base =
          dqkv + (static_cast<int64_t>(b) * g.N + key) * g.ld_qkv + h * 64 + kh * 32;
      float o[32];
      if (active) tmem_ld32(tmem + lq + 128 + static_cast<uint32_t>(32 * kh), o);
      if (key < g.N) store_row32_bf16(base + 2 * d, o);  // dV
      if (active) tmem_ld32(tmem + lq + 192 + static_cast<uint32_t>(32 * kh), o);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar_e);
      if (key < g.N) store_row32_bf16(base + d, o);  // dK
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 8) tmem_dealloc(tmem, 256);
}

}  // namespace attn_tc
}  // namespace rp

using namespace rp;

extern "C" int rp_attn_trace(int on, long long* out512) {
  if (out512) cudaMemcpyFromSymbol(out512, attn_tc::g_trace, sizeof(long long) * 512);
  cudaMemcpyToSymbol(attn_tc::g_trace_on, &on, sizeof(int));
  return rp_check_launch("attn_trace");
}

// Backward on the tcgen05 path (N <= 256): dQ (and D = rowsum(dO * O) into `Dg`), then
// dK / dV. Returns RP_ERR_CONFIG without launching when the shape is outside this path.
int rp_attention_bwd_tc(const uint16_t* qkv, const uint16_t* out, const uint16_t* dout,
                        const float* lse, float* Dg, int64_t S, int64_t N, int64_t H,
                        uint16_t* dqkv, cudaStream_t stream) {
  using namespace attn_tc;
  if (N > 256 || N < 1) return RP_ERR_CONFIG;
  BwdGeom g;
  g.B = static_cast<int>(S);
  g.N = static_cast<int>(N);
  g.H = static_cast<int>(H);
  g.Nk = static_cast<int>((N + 15) / 16 * 16);
  g.ld_o = H * 64;
  g.ld_qkv = 3 * H * 64;
  g.scale = 1.0f / 8.0f;
  g.scale_log2 = g.scale * 1.4426950408889634f;
  const int64_t T = S * N;
  CUtensorMap q128, do128, kvNk, kv128, qNk, doNk;
  if (make_map(&q128, qkv, T, 3 * H * 64, 128) || make_map(&do128, dout, T, H * 64, 128) ||
      make_map(&kvNk, qkv, T, 3 * H * 64, static_cast<uint32_t>(g.Nk)) ||
      make_map(&kv128, qkv, T, 3 * H * 64, 128) ||
      make_map(&qNk, qkv, T, 3 * H * 64, static_cast<uint32_t>(g.Nk)) ||
      make_map(&doNk, dout, T, H * 64, static_cast<uint32_t>(g.Nk)))
    return rp_fail(RP_ERR_CUDA, "attention_bwd_tc: tensor map encode failed");
  const int smem = 1024 + kBwdSmem;
  static std::once_flag once;
  static int nsm = 148;
  std::call_once(once, [smem] {
    cudaFuncSetAttribute(attn_bwd_dq_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(attn_bwd_dkdv_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  });
  BwdPlan pl;
  pl.ntile = static_cast<int>((N + 127) / 128);
  pl.nitems = static_cast<int>(S * H) * pl.ntile;
  const unsigned grid = static_cast<unsigned>(pl.nitems < 2 * nsm ? pl.nitems : 2 * nsm);
  launch_k(attn_bwd_dq_tc, dim3(grid), dim3(kBwdThreads), smem, stream, q128, do128, kvNk,
           reinterpret_cast<const __nv_bfloat16*>(out), lse, Dg,
           reinterpret_cast<__nv_bfloat16*>(dqkv), g, pl);
  launch_k(attn_bwd_dkdv_tc, dim3(grid), dim3(kBwdThreads), smem, stream, kv128, qNk, doNk, lse,
           static_cast<const float*>(Dg), reinterpret_cast<__nv_bfloat16*>(dqkv), g, pl);
  return rp_check_launch("attention_bwd_tc");
}
