// tcgen05 attention backward (head_dim 64, N <= 768: keys / queries streamed in 64-row chunks).
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

#include <cstring>

namespace rp {
namespace attn_tc {


struct BwdGeom {
  int B, N, H, Nk;    // sequences, tokens, heads, N rounded up to 16
  int hd;             // head dim (64, or 72..128 on the wide variant)
  int64_t ld_o;       // row pitch of O / dO (H * hd)
  int64_t ld_qkv;     // row pitch of qkv / dqkv (3 H * hd)
  float scale, scale_log2;
};

struct BwdPlan {
  int ntile;   // 128-row tiles per (sequence, head)
  int nitems;  // ntile * B * H
};

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

// ------------------------------------------------------------------ the kernel (two passes)
// 288 threads: warps 0-7 elementwise (TMEM lane quarter w%4, column half w/4 of a 64-wide
// chunk), warp 8 TMA + MMA issue (one thread). TMEM: S [0, 64), dP [64, 128), accumulators
// from 128 (HP = 64: two 64-column ones in 256 columns, ~100 KB of smem, so two CTAs share an
// SM and one's elementwise phase overlaps the other's MMAs; HP = 128: head dims 72..128, two
// round16(hd)-column accumulators at 128 and 256 of 512 columns, ~193 KB, one CTA per SM).
// Operands (bf16, K-major SW128 atoms of 64 columns; HP = 128 stores each operand as two
// atom planes [atom][rows][128 B], the second loaded by a box of hd - 64 columns whose
// untouched tail stays zero -- tools/probe/tma_narrow_box.cu shows the narrow box landing in
// the same swizzled 128-byte rows):
//   tile  A | B   128 rows of the item (DQ: Q | dO, DKDV: K | V), double-buffered per item
//                 so the next item's tile streams in during the current one
//   chunk C | D   64 rows of the streamed side (DQ: K | V, DKDV: Q | dO), a 2-slot ring
//                 that runs ahead across item boundaries; any N up to 1024
// MMA1: S = A C_c^T, dP = B D_c^T (N = chunk width, K = hd in 16-column steps); MMA2: DQ
// dQ += dS C_c; DKDV dV += P^T D_c, dK += dS^T C_c (A operands re-packed to bf16 in TMEM;
// B operands MN-major over the chunk's atom planes, plane stride 64 rows x 128 B = LBO).
// Two MMA issuers (one thread each; an MMA costs its issuing thread ~120 cycles, so one issuer
// serialised the chunk's 12-22 MMAs): warp 8 issues S and the accumulation that reads the S
// columns (DQ dQ += dS K_c, DKDV dV += P^T dO_c) and the TMA loads; warp 9 issues dP and the
// one that reads the dP columns (DKDV dK += dS^T Q_c). Each owns its TMEM columns, so the
// in-order retirement of one thread's MMAs is the only ordering either needs.
constexpr int kBwdWarps = 10;
constexpr int kBwdThreads = kBwdWarps * 32;
template <int HP>
struct BwdCfg {
  static constexpr int kAtoms = HP / 64;
  static constexpr int kTileBytes = 2 * 128 * 128 * kAtoms;  // A | B
  static constexpr int kChunkBytes = 2 * 64 * 128 * kAtoms;  // C_c | D_c
  static constexpr int kSmem = 2 * kTileBytes + 2 * kChunkBytes;
  static constexpr int kTmemCols = HP == 64 ? 256 : 512;
  static constexpr int kAcc1 = HP == 64 ? 192 : 256;  // second accumulator (DKDV dK)
};
constexpr int kBwdSmem = BwdCfg<64>::kSmem;

// TMA maps of one operand: box {64, rows} over the first 64 head columns and, for head dims
// above 64, box {hd - 64, rows} over the rest
struct OpMaps {
  CUtensorMap lo, hi;
};

template <bool DQ, int HP>
__global__ void __launch_bounds__(kBwdThreads, HP == 64 ? 2 : 1)
    attn_bwd_tc(const __grid_constant__ OpMaps tm_a, const __grid_constant__ OpMaps tm_b,
                const __grid_constant__ OpMaps tm_c, const __grid_constant__ OpMaps tm_d,
                const __nv_bfloat16* __restrict__ O, const float* __restrict__ lse,
                float* __restrict__ Dg, __nv_bfloat16* __restrict__ dqkv, BwdGeom g, BwdPlan pl,
                __nv_bfloat16* __restrict__ dSt) {
  using Cfg = BwdCfg<HP>;
  constexpr int kTileBytes = Cfg::kTileBytes, kChunkBytes = Cfg::kChunkBytes;
  constexpr uint32_t kTilePlane = 128 * 128, kChunkPlane = 64 * 128;  // one atom plane
  pdl_trigger();

  __shared__ float red[2][128];                // DQ: D partials [column half][row]
  __shared__ __align__(16) float sL[1024];     // DKDV: -lse per query of the item
  __shared__ __align__(16) float sD[1024];     //       -D * scale
  __shared__ __align__(8) uint64_t bars[12];
  __shared__ uint32_t tmem_slot;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* tiles = smem;                     // [2][A | B]
  uint8_t* ring = smem + 2 * kTileBytes;     // [2][C_c | D_c]
  uint64_t* tile_full = bars;       // [2]
  uint64_t* tile_free = bars + 2;   // [2] the item's last MMA retired
  uint64_t* ring_full = bars + 4;   // [2]
  uint64_t* ring_free = bars + 6;   // [2] the chunk's accumulation MMAs retired
  uint64_t* bar_s = bars + 8;       // S, dP of a chunk ready
  uint64_t* bar_p = bars + 9;       // bf16 operands of a chunk in TMEM (8 warps)
  uint64_t* bar_o = bars + 10;      // the item's accumulators complete
  uint64_t* bar_e = bars + 11;      // accumulators read out (8 warps)

  const uint32_t warp = warp_id(), lane = lane_id();
  const int hd = HP == 64 ? 64 : g.hd;
  if constexpr (HP > 64) {
    // the second atom plane's columns past hd are never written by the TMA: zero them once
    for (int i = static_cast<int>(threadIdx.x) * 16; i < Cfg::kSmem; i += kBwdThreads * 16)
      *reinterpret_cast<uint4*>(smem + i) = make_uint4(0, 0, 0, 0);
    fence_proxy_async_smem();
  }
  if (warp == 8) {
    if (lane == 0) {
      tma_prefetch_desc(&tm_a.lo);
      tma_prefetch_desc(&tm_b.lo);
      tma_prefetch_desc(&tm_c.lo);
      tma_prefetch_desc(&tm_d.lo);
      for (int i = 0; i < 2; ++i) {
        mbar_init(&tile_full[i], 1);
        mbar_init(&tile_free[i], 2);
        mbar_init(&ring_full[i], 1);
        mbar_init(&ring_free[i], 2);
      }
      mbar_init(bar_s, 2);
      mbar_init(bar_p, 8);
      mbar_init(bar_o, 2);
      mbar_init(bar_e, 8);
      fence_barrier_init();
    }
    tmem_alloc(&tmem_slot, Cfg::kTmemCols);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;
  pdl_wait();
  const int Nk = g.Nk, d = g.H * hd;
  const int nch = (Nk + 63) / 64;
  const int K = pl.nitems > static_cast<int>(blockIdx.x)
                    ? (pl.nitems - static_cast<int>(blockIdx.x) + static_cast<int>(gridDim.x) - 1) /
                          static_cast<int>(gridDim.x)
                    : 0;
  auto item_of = [&](int k) { return static_cast<int>(blockIdx.x) + k * static_cast<int>(gridDim.x); };
  // column offsets of the four operands in qkv / d_out (DQ: A=Q, B=dO, C=K, D=V;
  // DKDV: A=K, B=V, C=Q, D=dO)
  const int ca = DQ ? 0 : d, cb = DQ ? 0 : 2 * d, cc = DQ ? d : 0, cd = DQ ? 2 * d : 0;

  if (warp >= 8) {
    if (lane == 0) {
      const bool ia = warp == 8;  // issuer A (S, its accumulation, TMA) or B (dP, dK)
      // one operand block of `plane`-byte atom planes: box {64} then, above 64, {hd - 64}
      auto load_op = [&](uint8_t* dst, const OpMaps& m, uint64_t* bar, int col, int row,
                         uint32_t plane) {
        tma_load_2d(dst, &m.lo, bar, col, row);
        if constexpr (HP > 64) tma_load_2d(dst + plane, &m.hi, bar, col + 64, row);
      };
      auto load_tile = [&](int k) {
        int tile, h, b;
        item_coords(item_of(k), pl.ntile, g.H, tile, h, b);
        const int row = b * g.N + tile * 128;
        uint8_t* dst = tiles + (k & 1) * kTileBytes;
        uint64_t* bar = &tile_full[k & 1];
        mbar_arrive_expect_tx(bar, static_cast<uint32_t>(2 * 128 * hd * 2));
        load_op(dst, tm_a, bar, ca + h * hd, row, kTilePlane);
        load_op(dst + kTileBytes / 2, tm_b, bar, cb + h * hd, row, kTilePlane);
      };
      auto load_chunk = [&](int idx) {  // flat chunk index over (item, chunk)
        const int k = idx / nch, c = idx % nch;
        int tile, h, b;
        item_coords(item_of(k), pl.ntile, g.H, tile, h, b);
        const int row = b * g.N + 64 * c;
        uint8_t* dst = ring + (idx & 1) * kChunkBytes;
        uint64_t* bar = &ring_full[idx & 1];
        mbar_arrive_expect_tx(bar, static_cast<uint32_t>(2 * 64 * hd * 2));
        load_op(dst, tm_c, bar, cc + h * hd, row, kChunkPlane);
        load_op(dst + kChunkBytes / 2, tm_d, bar, cd + h * hd, row, kChunkPlane);
      };
      const int nacc = (hd + 15) / 16 * 16, nks = nacc / 16;
      const uint32_t idesc_o = make_idesc_bf16(128, static_cast<uint32_t>(nacc), false, true);
      const int total = K * nch;
      if (ia && K > 0) {
        load_tile(0);
        load_chunk(0);
      }
      int u = 0;
      for (int k = 0; k < K; ++k) {
        if (ia && k + 1 < K) {  // the next item's tile streams in during this one
          if (k >= 1) mbar_wait(&tile_free[(k + 1) & 1], ((k - 1) >> 1) & 1);
          load_tile(k + 1);
        }
        mbar_wait(&tile_full[k & 1], (k >> 1) & 1);
        const uint32_t ta = smem_u32(tiles + (k & 1) * kTileBytes), tb = ta + kTileBytes / 2;
        for (int c = 0; c < nch; ++c, ++u) {
          const int w = min(64, Nk - 64 * c);
          mbar_wait(&ring_full[u & 1], (u >> 1) & 1);
          tc_fence_after();
          const uint32_t rc = smem_u32(ring + (u & 1) * kChunkBytes), rd = rc + kChunkBytes / 2;
          const uint32_t idesc_s = make_idesc_bf16(128, static_cast<uint32_t>(w), false, false);
          for (int kk = 0; kk < nks; ++kk) {
            const uint32_t ka = static_cast<uint32_t>(kk >> 2) * kTilePlane + (kk & 3) * 32;
            const uint32_t kc = static_cast<uint32_t>(kk >> 2) * kChunkPlane + (kk & 3) * 32;
            if (ia)  // S = A C_c^T
              umma_bf16(tmem, make_sdesc_sw128(ta + ka, 16, 1024),
                        make_sdesc_sw128(rc + kc, 16, 1024), idesc_s, kk > 0 ? 1u : 0u);
            else     // dP = B D_c^T
              umma_bf16(tmem + 64, make_sdesc_sw128(tb + ka, 16, 1024),
                        make_sdesc_sw128(rd + kc, 16, 1024), idesc_s, kk > 0 ? 1u : 0u);
          }
          umma_commit(bar_s);
          if (ia && u + 1 < total) {  // next chunk into the other ring slot once its MMAs retired
            if (u >= 1) mbar_wait(&ring_free[(u + 1) & 1], ((u - 1) >> 1) & 1);
            load_chunk(u + 1);
          }
          if (c == 0 && k > 0) mbar_wait(bar_e, (k - 1) & 1);  // previous accumulators read out
          mbar_wait(bar_p, u & 1);
          tc_fence_after();
          for (int ks = 0; ks < w / 16; ++ks) {
            const uint32_t row16 = static_cast<uint32_t>(16 * ks * 128);
            const uint32_t acc = (c > 0 || ks > 0) ? 1u : 0u;
            if constexpr (DQ) {
              if (ia)
                umma_ts_bf16(tmem + 128, tmem + chunk_acol(ks),
                             make_sdesc_sw128(rc + row16, kChunkPlane, 1024), idesc_o, acc);  // dQ += dS K_c
            } else {
              if (ia)
                umma_ts_bf16(tmem + 128, tmem + chunk_acol(ks),
                             make_sdesc_sw128(rd + row16, kChunkPlane, 1024), idesc_o, acc);  // dV += P^T dO_c
              else
                umma_ts_bf16(tmem + Cfg::kAcc1, tmem + 64 + chunk_acol(ks),
                             make_sdesc_sw128(rc + row16, kChunkPlane, 1024), idesc_o, acc);  // dK += dS^T Q_c
            }
          }
          umma_commit(&ring_free[u & 1]);
        }
        umma_commit(bar_o);
        umma_commit(&tile_free[k & 1]);
      }
    }
  } else {
    const int q = static_cast<int>(warp & 3u), kh = static_cast<int>(warp >> 2);
    const uint32_t lq = (static_cast<uint32_t>(q) * 32u) << 16;
    const int rloc = q * 32 + static_cast<int>(lane);
    const uint32_t ts = tmem + lq + static_cast<uint32_t>(32 * kh);
    // per-item global inputs of the NEXT item, loaded into registers under the current
    // item's last chunk and epilogue (their latency was exposed at every item start):
    // DQ: this lane's query row of O (its head-column part) and its LSE; DKDV: this thread's
    // slots of the item's -lse / -D scale rows (published to sL / sD at the item start)
    constexpr int kOq = (HP / 64) * 4;
    uint4 o_nx[kOq];
    float lr_nx = 0.f, sl_nx[4], sd_nx[4];
    auto prefetch = [&](int kn) {
      int tile_n, h_n, b_n;
      item_coords(item_of(kn), pl.ntile, g.H, tile_n, h_n, b_n);
      const int64_t hb_n = (static_cast<int64_t>(b_n) * g.H + h_n) * g.N;
      if constexpr (DQ) {
        const int row_n = tile_n * 128 + rloc;
        const int64_t grow_n = static_cast<int64_t>(b_n) * g.N + row_n;
        lr_nx = row_n < g.N ? __ldg(lse + hb_n + row_n) : 0.f;
#pragma unroll
        for (int a = 0; a < HP / 64; ++a)
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const int col = 64 * a + 32 * kh + 8 * c;
            o_nx[4 * a + c] = row_n < g.N && col < hd
                                  ? __ldg(reinterpret_cast<const uint4*>(O + grow_n * g.ld_o + h_n * hd + col))
                                  : make_uint4(0, 0, 0, 0);
          }
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int i = static_cast<int>(threadIdx.x) + 256 * j;
          sl_nx[j] = i < g.N ? -__ldg(lse + hb_n + i) : -INFINITY;
          sd_nx[j] = i < g.N ? -__ldg(Dg + hb_n + i) * g.scale : 0.f;
        }
      }
    };
    if (K > 0) prefetch(0);
    int u = 0;
    for (int k = 0; k < K; ++k) {
      int tile, h, b;
      item_coords(item_of(k), pl.ntile, g.H, tile, h, b);
      const int row = tile * 128 + rloc;  // query (DQ) or key (DKDV) of this lane
      const bool active = tile * 128 + q * 32 < g.N;
      const int64_t hb = (static_cast<int64_t>(b) * g.H + h) * g.N;
      const int64_t grow = static_cast<int64_t>(b) * g.N + row;
      // dS^T row of this lane's key (fused backward): written for keys < Nk, zero past N
      __nv_bfloat16* ds_row =
          (!DQ && dSt != nullptr && row < Nk)
              ? dSt + ((static_cast<int64_t>(b) * g.H + h) * Nk + row) * Nk
              : nullptr;
      float lr = 0.f, nds = 0.f;
      if constexpr (DQ) {
        // ---- D = rowsum(dO * O) for this lane's query (dO from the smem tile, O global):
        // warp half kh covers head columns [32 kh, 32 kh + 32) of each 64-column atom plane
        lr = lr_nx;
        mbar_wait(&tile_full[k & 1], (k >> 1) & 1);
        float dpart = 0.f;
        if (row < g.N) {
#pragma unroll
          for (int a = 0; a < HP / 64; ++a) {
            const uint8_t* drow =
                tiles + (k & 1) * kTileBytes + kTileBytes / 2 + a * kTilePlane + rloc * 128;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              const int col = 64 * a + 32 * kh + 8 * c;  // head column of this 16-byte chunk
              if (col >= hd) break;
              const uint4 ov = o_nx[4 * a + c];
              const int ch = kh * 4 + c;
              const uint4 dv = *reinterpret_cast<const uint4*>(drow + ((ch ^ (rloc & 7)) << 4));
              const uint32_t ow[4] = {ov.x, ov.y, ov.z, ov.w}, dw[4] = {dv.x, dv.y, dv.z, dv.w};
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const float2 x = unpack_bf16x2(ow[e]), y = unpack_bf16x2(dw[e]);
                dpart = fmaf(x.x, y.x, dpart);
                dpart = fmaf(x.y, y.y, dpart);
              }
            }
          }
        }
        if (k > 0) named_bar(1, 256);  // previous item's red[] read (as sL / sD below)
        red[kh][rloc] = dpart;
        named_bar(1, 256);
        const float D = red[0][rloc] + red[1][rloc];
        if (kh == 0 && row < g.N) Dg[hb + row] = D;
        nds = -D * g.scale;
      } else {
        // (ordered after every warp's reads of the previous item's sL / sD by the bar_p ->
        // MMA -> bar_o chain already; the barrier states it where racecheck can see it)
        if (k > 0) named_bar(1, 256);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int i = static_cast<int>(threadIdx.x) + 256 * j;
          if (i < Nk) {
            sL[i] = sl_nx[j];
            sD[i] = sd_nx[j];
          }
        }
        named_bar(1, 256);
      }
      for (int c = 0; c < nch; ++c, ++u) {
        const int w = min(64, Nk - 64 * c);
        mbar_wait(bar_s, u & 1);
        tc_fence_after();
        if (active && 32 * kh < w) {
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const int col0 = 64 * c + 32 * kh + 16 * hh;  // key (DQ) / query (DKDV) index
            if (col0 - 64 * c >= w) break;
            float s[16], dp[16];
            tmem_ld16x2(ts + 16 * hh, ts + 64 + 16 * hh, s, dp);
            if constexpr (DQ) {
              uint32_t pk[8];
#pragma unroll
              for (int e = 0; e < 8; ++e) {
                const int key = col0 + 2 * e;
                const float p0 = key < g.N ? ex2(fmaf(s[2 * e], g.scale_log2, -lr)) : 0.f;
                const float p1 = key + 1 < g.N ? ex2(fmaf(s[2 * e + 1], g.scale_log2, -lr)) : 0.f;
                const float d0 = key < g.N ? p0 * fmaf(dp[2 * e], g.scale, nds) : 0.f;
                const float d1 = key + 1 < g.N ? p1 * fmaf(dp[2 * e + 1], g.scale, nds) : 0.f;
                pk[e] = pack_bf16x2(d0, d1);
              }
              tmem_st8(ts + 8 * hh, pk);  // dS over this warp's own, already-read S columns
            } else {
              uint32_t pp[8], pd[8];
              const float4* l4 = reinterpret_cast<const float4*>(sL + col0);
              const float4* d4 = reinterpret_cast<const float4*>(sD + col0);
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                const float4 nl = l4[j], nd = d4[j];
                const float la[4] = {nl.x, nl.y, nl.z, nl.w}, da[4] = {nd.x, nd.y, nd.z, nd.w};
#pragma unroll
                for (int t = 0; t < 2; ++t) {
                  const int e = 4 * j + 2 * t;
                  const bool v0 = col0 + e < g.N, v1 = col0 + e + 1 < g.N;
                  const float p0 = v0 ? ex2(fmaf(s[e], g.scale_log2, la[2 * t])) : 0.f;
                  const float p1 = v1 ? ex2(fmaf(s[e + 1], g.scale_log2, la[2 * t + 1])) : 0.f;
                  pp[2 * j + t] = pack_bf16x2(p0, p1);
                  pd[2 * j + t] =
                      pack_bf16x2(v0 ? p0 * fmaf(dp[e], g.scale, da[2 * t]) : 0.f,
                                  v1 ? p1 * fmaf(dp[e + 1], g.scale, da[2 * t + 1]) : 0.f);
                }
              }
              tmem_st8(ts + 8 * hh, pp);       // P^T over own, already-read S^T columns
              tmem_st8(ts + 64 + 8 * hh, pd);  // dS^T over own dP^T columns
              if (ds_row != nullptr) {  // dS^T (this key, 16 queries) for the dQ pass
                const bool kv = row < g.N;
                uint4* dst4 = reinterpret_cast<uint4*>(ds_row + col0);
                // streaming stores: dS^T is consumed by the next kernel, keep L2 for the
                // operands this pass re-reads
                __stcs(dst4, kv ? make_uint4(pd[0], pd[1], pd[2], pd[3]) : make_uint4(0u, 0u, 0u, 0u));
                __stcs(dst4 + 1, kv ? make_uint4(pd[4], pd[5], pd[6], pd[7]) : make_uint4(0u, 0u, 0u, 0u));
              }
            }
          }
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(bar_p);
      }
      if (k + 1 < K) prefetch(k + 1);
      // ---- epilogue: warp half kh stores head columns [kh HP / 2, (kh + 1) HP / 2) < hd
      mbar_wait(bar_o, k & 1);
      tc_fence_after();
      constexpr int kHalf = HP / 2;
      float o[kHalf];
      const int c0 = kh * kHalf;
      __nv_bfloat16* dst = dqkv + grow * g.ld_qkv + h * hd + c0;
      auto ld_acc = [&](uint32_t col) {
        if (active)
#pragma unroll
          for (int j = 0; j < kHalf / 32; ++j)
            tmem_ld32(tmem + lq + col + static_cast<uint32_t>(c0 + 32 * j), o + 32 * j);
      };
      auto st_acc = [&](__nv_bfloat16* p) {
        if (row < g.N)
#pragma unroll
          for (int j = 0; j < kHalf / 8; ++j)
            if (c0 + 8 * j < hd)
              reinterpret_cast<uint4*>(p)[j] =
                  make_uint4(pack_bf16x2(o[8 * j], o[8 * j + 1]), pack_bf16x2(o[8 * j + 2], o[8 * j + 3]),
                             pack_bf16x2(o[8 * j + 4], o[8 * j + 5]),
                             pack_bf16x2(o[8 * j + 6], o[8 * j + 7]));
      };
      if constexpr (DQ) {
        ld_acc(128);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(bar_e);
        st_acc(dst);
      } else {
        ld_acc(128);
        st_acc(dst + 2 * d);  // dV
        ld_acc(Cfg::kAcc1);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(bar_e);
        st_acc(dst + d);  // dK
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 8) tmem_dealloc(tmem, Cfg::kTmemCols);  // (warp 9 idles at the barrier)
}

// ------------------------------------------------------------------ D and dQ for the fused path
// D[b][h][n] = rowsum(dO * O) (softmax VJP dot, ops.cpp:219-220): 8 threads per (row, head),
// 16 B each, so a warp reads 4 heads' contiguous 512 B of a row; 3-step shuffle reduction.
__global__ void __launch_bounds__(256)
    attn_d_kernel(const __nv_bfloat16* __restrict__ O, const __nv_bfloat16* __restrict__ dO,
                  float* __restrict__ Dg, int64_t rows, int N, int H) {
  pdl_trigger();
  pdl_wait();
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int64_t rh = i >> 3;  // (row, head) pair, head fastest
  const bool ok = rh < rows * H;
  float acc = 0.f;
  if (ok) {
    const uint4 a = __ldg(reinterpret_cast<const uint4*>(O) + i);
    const uint4 c = __ldg(reinterpret_cast<const uint4*>(dO) + i);
    const uint32_t av[4] = {a.x, a.y, a.z, a.w}, cv[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float2 fa = unpack_bf16x2(av[k]), fc = unpack_bf16x2(cv[k]);
      acc = fmaf(fa.x, fc.x, acc);
      acc = fmaf(fa.y, fc.y, acc);
    }
  }
  acc += __shfl_xor_sync(0xffffffffu, acc, 1);
  acc += __shfl_xor_sync(0xffffffffu, acc, 2);
  acc += __shfl_xor_sync(0xffffffffu, acc, 4);
  if (ok && (i & 7) == 0) {
    const int h = static_cast<int>(rh % H);
    const int64_t row = rh / H, b = row / N, n = row % N;
    Dg[(b * H + h) * N + n] = acc;
  }
}

// dQ = dS K per (128-query tile, head, sequence) from the dS^T rows the dK/dV pass wrote
// (dSt [S*H][Nk keys][Nk queries] bf16): D[M = queries][N = 64] += A . B over 64-key chunks
// with A = dS (stored [keys][queries]: MN-major) and B = K_c ([keys][64]: MN-major), the
// wgrad operand layout of the GEMM. Warp 0: TMA, warp 1: MMA (one thread), warps 2-5:
// TMEM -> bf16 -> dqkv. Accumulators double-buffered in TMEM (2 x 64 columns).
constexpr int kDqStages = 4;
constexpr int kDqStage = 16384 + 8192;  // A (2 boxes of 64 keys x 64 queries) | B (64 x 64)
__global__ void __launch_bounds__(192, 2)
    attn_dq_tc(const __grid_constant__ CUtensorMap tm_ds, const __grid_constant__ CUtensorMap tm_k,
               __nv_bfloat16* __restrict__ dqkv, BwdGeom g, BwdPlan pl) {
  pdl_trigger();
  __shared__ __align__(8) uint64_t bars[2 * kDqStages + 4];
  __shared__ uint32_t tmem_slot;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint64_t* full = bars;
  uint64_t* empty = bars + kDqStages;
  uint64_t* tfull = bars + 2 * kDqStages;
  uint64_t* tempty = bars + 2 * kDqStages + 2;
  const uint32_t warp = warp_id(), lane = lane_id();
  if (warp == 0) {
    if (lane == 0) {
      tma_prefetch_desc(&tm_ds);
      tma_prefetch_desc(&tm_k);
      for (int i = 0; i < kDqStages; ++i) {
        mbar_init(&full[i], 1);
        mbar_init(&empty[i], 1);
      }
      for (int i = 0; i < 2; ++i) {
        mbar_init(&tfull[i], 1);
        mbar_init(&tempty[i], 4);
      }
      fence_barrier_init();
    }
    tmem_alloc(&tmem_slot, 128);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;
  pdl_wait();
  const int Nk = g.Nk, nch = (Nk + 63) / 64, d = g.H * 64;
  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int item = blockIdx.x; item < pl.nitems; item += gridDim.x) {
        int tile, h, b;
        item_coords(item, pl.ntile, g.H, tile, h, b);
        const int bh = b * g.H + h;
        for (int c = 0; c < nch; ++c) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* a = smem + stage * kDqStage;
          const int krow = bh * Nk + 64 * c;  // dS^T rows of this chunk's keys
          tma_load_2d(a, &tm_ds, &full[stage], tile * 128, krow);
          tma_load_2d(a + 8192, &tm_ds, &full[stage], tile * 128 + 64, krow);
          tma_load_2d(a + 16384, &tm_k, &full[stage], d + h * 64, b * g.N + 64 * c);
          mbar_arrive_expect_tx(&full[stage], kDqStage);
          if (++stage == kDqStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = make_idesc_bf16(128, 64, true, true);
      int stage = 0, acc = 0;
      uint32_t phase = 0, acc_phase = 0;
      for (int item = blockIdx.x; item < pl.nitems; item += gridDim.x) {
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t td = tmem + static_cast<uint32_t>(acc * 64);
        for (int c = 0; c < nch; ++c) {
          const int w = min(64, Nk - 64 * c);  // keys of this chunk (multiple of 16)
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(smem + stage * kDqStage), b_addr = a_addr + 16384u;
          for (int kk = 0; kk < w / 16; ++kk)
            umma_bf16(td, make_sdesc_sw128(a_addr + kk * 2048, 8192, 1024),
                      make_sdesc_sw128(b_addr + kk * 2048, 8192, 1024), idesc,
                      (c > 0 || kk > 0) ? 1u : 0u);
          umma_commit(&empty[stage]);
          if (++stage == kDqStages) {
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
    const int q = static_cast<int>(warp & 3u);  // TMEM lane quarter of warps 2..5
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int item = blockIdx.x; item < pl.nitems; item += gridDim.x) {
      int tile, h, b;
      item_coords(item, pl.ntile, g.H, tile, h, b);
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      float o[64];
      const uint32_t ta = tmem + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(acc * 64);
      tmem_ld32(ta, o);
      tmem_ld32(ta + 32, o + 32);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      const int row = tile * 128 + q * 32 + static_cast<int>(lane);
      if (row < g.N) {
        __nv_bfloat16* dst = dqkv + (static_cast<int64_t>(b) * g.N + row) * g.ld_qkv + h * 64;
        store_row32_bf16(dst, o);
        store_row32_bf16(dst + 32, o + 32);
      }
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc(tmem, 128);
}

}  // namespace attn_tc
}  // namespace rp

using namespace rp;

// Backward on the tcgen05 path (head_dim 64). Returns RP_ERR_CONFIG without launching when
// the shape is outside this path.
//   dSt == nullptr: two passes -- dQ (and D = rowsum(dO * O) into `Dg`), then dK / dV.
//   dSt != nullptr: D first (attn_d_kernel), then ONE pass over (key tile, query chunk)
//     computing dK / dV and writing dS^T (bf16, [S*H][Nk][Nk]) on the way, then dQ = dS K
//     as a streamed MMA over dS^T (attn_dq_tc) -- S and dP are formed once instead of twice.
int rp_attention_bwd_fused_tc(const uint16_t* qkv, const uint16_t* dout, const float* lse,
                              const float* Dg, float* scratch, int64_t S, int64_t N, int64_t H,
                              uint16_t* dqkv, cudaStream_t stream);

int rp_attention_bwd_tc(const uint16_t* qkv, const uint16_t* out, const uint16_t* dout,
                        const float* lse, float* Dg, int64_t S, int64_t N, int64_t H,
                        uint16_t* dqkv, cudaStream_t stream, uint16_t* dSt, int d_ready,
                        int fused) {
  using namespace attn_tc;
  if (N > 1024 || N < 1) return RP_ERR_CONFIG;
  BwdGeom g;
  g.B = static_cast<int>(S);
  g.N = static_cast<int>(N);
  g.H = static_cast<int>(H);
  g.Nk = static_cast<int>((N + 15) / 16 * 16);
  g.hd = 64;
  g.ld_o = H * 64;
  g.ld_qkv = 3 * H * 64;
  g.scale = 1.0f / 8.0f;
  g.scale_log2 = g.scale * 1.4426950408889634f;
  const int64_t T = S * N;
  OpMaps q128, do128, k128, q64, do64, k64;
  std::memset(&q128, 0, sizeof(OpMaps));
  std::memset(&do128, 0, sizeof(OpMaps));
  std::memset(&k128, 0, sizeof(OpMaps));
  std::memset(&q64, 0, sizeof(OpMaps));
  std::memset(&do64, 0, sizeof(OpMaps));
  std::memset(&k64, 0, sizeof(OpMaps));
  if (make_map(&q128.lo, qkv, T, 3 * H * 64, 128) || make_map(&do128.lo, dout, T, H * 64, 128) ||
      make_map(&k128.lo, qkv, T, 3 * H * 64, 128) || make_map(&q64.lo, qkv, T, 3 * H * 64, 64) ||
      make_map(&do64.lo, dout, T, H * 64, 64) || make_map(&k64.lo, qkv, T, 3 * H * 64, 64))
    return rp_fail(RP_ERR_CUDA, "attention_bwd_tc: tensor map encode failed");
  const int smem = 1024 + kBwdSmem;
  const int smem_dq = 1024 + kDqStages * kDqStage;
  static std::once_flag once;
  static int nsm = 148;
  std::call_once(once, [smem, smem_dq] {
    cudaFuncSetAttribute(attn_bwd_tc<true, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(attn_bwd_tc<false, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(attn_dq_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_dq);
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  });
  BwdPlan pl;
  pl.ntile = static_cast<int>((N + 127) / 128);
  pl.nitems = static_cast<int>(S * H) * pl.ntile;
  const unsigned grid = static_cast<unsigned>(pl.nitems < 2 * nsm ? pl.nitems : 2 * nsm);
  if (dSt != nullptr && fused && N <= 208) {
    // single pass (attention_bwd_fused.cu); the dS^T region is its dQ scratch
    if (!d_ready) {
      const int64_t n = T * H * 8;
      launch_k(attn_d_kernel, dim3(static_cast<unsigned>((n + 255) / 256)), dim3(256), 0, stream,
               reinterpret_cast<const __nv_bfloat16*>(out),
               reinterpret_cast<const __nv_bfloat16*>(dout), Dg, T, g.N, g.H);
    }
    const int rc = rp_attention_bwd_fused_tc(qkv, dout, lse, Dg, reinterpret_cast<float*>(dSt), S, N,
                                             H, dqkv, stream);
    if (rc != RP_ERR_CONFIG) return rc;
  }
  if (dSt != nullptr) {
    CUtensorMap ds;
    if (make_map(&ds, dSt, S * H * g.Nk, g.Nk, 64))
      return rp_fail(RP_ERR_CUDA, "attention_bwd_tc: tensor map encode failed");
    if (!d_ready) {  // D = rowsum(dO * O), unless the d_att GEMM already produced it
      const int64_t n = T * H * 8;
      launch_k(attn_d_kernel, dim3(static_cast<unsigned>((n + 255) / 256)), dim3(256), 0, stream,
               reinterpret_cast<const __nv_bfloat16*>(out),
               reinterpret_cast<const __nv_bfloat16*>(dout), Dg, T, g.N, g.H);
    }
    launch_k(attn_bwd_tc<false, 64>, dim3(grid), dim3(kBwdThreads), smem, stream, k128, k128, q64,
             do64, reinterpret_cast<const __nv_bfloat16*>(out), lse, Dg,
             reinterpret_cast<__nv_bfloat16*>(dqkv), g, pl, reinterpret_cast<__nv_bfloat16*>(dSt));
    launch_k(attn_dq_tc, dim3(grid), dim3(192), smem_dq, stream, ds, k64.lo,
             reinterpret_cast<__nv_bfloat16*>(dqkv), g, pl);
    return rp_check_launch("attention_bwd_tc");
  }
  // dQ (+ D): tiles Q | dO, chunks K | V (qkv maps; the dO map for the dO tile)
  launch_k(attn_bwd_tc<true, 64>, dim3(grid), dim3(kBwdThreads), smem, stream, q128, do128, k64, k64,
           reinterpret_cast<const __nv_bfloat16*>(out), lse, Dg,
           reinterpret_cast<__nv_bfloat16*>(dqkv), g, pl, static_cast<__nv_bfloat16*>(nullptr));
  // dK, dV: tiles K | V, chunks Q | dO
  launch_k(attn_bwd_tc<false, 64>, dim3(grid), dim3(kBwdThreads), smem, stream, k128, k128, q64, do64,
           reinterpret_cast<const __nv_bfloat16*>(out), lse, Dg,
           reinterpret_cast<__nv_bfloat16*>(dqkv), g, pl, static_cast<__nv_bfloat16*>(nullptr));
  return rp_check_launch("attention_bwd_tc");
}

// Two-pass tcgen05 backward for head dims 72..128 (multiples of 8; e.g. the G48 config's
// 104): dQ (+ D) then dK / dV, operands as two 64-column atom planes. RP_ERR_CONFIG without
// launching outside that range.
int rp_attention_bwd_tc_wide(const uint16_t* qkv, const uint16_t* out, const uint16_t* dout,
                             const float* lse, float* Dg, int64_t S, int64_t N, int64_t H,
                             int64_t hd, uint16_t* dqkv, cudaStream_t stream) {
  using namespace attn_tc;
  if (N > 1024 || N < 1 || hd <= 64 || hd > 128 || hd % 8) return RP_ERR_CONFIG;
  BwdGeom g;
  g.B = static_cast<int>(S);
  g.N = static_cast<int>(N);
  g.H = static_cast<int>(H);
  g.Nk = static_cast<int>((N + 15) / 16 * 16);
  g.hd = static_cast<int>(hd);
  g.ld_o = H * hd;
  g.ld_qkv = 3 * H * hd;
  g.scale = 1.0f / sqrtf(static_cast<float>(hd));
  g.scale_log2 = g.scale * 1.4426950408889634f;
  const int64_t T = S * N;
  const uint32_t hi = static_cast<uint32_t>(hd - 64);
  OpMaps qkv128, do128, qkv64, do64;
  if (make_map(&qkv128.lo, qkv, T, 3 * H * hd, 128) || make_map(&qkv128.hi, qkv, T, 3 * H * hd, 128, hi) ||
      make_map(&do128.lo, dout, T, H * hd, 128) || make_map(&do128.hi, dout, T, H * hd, 128, hi) ||
      make_map(&qkv64.lo, qkv, T, 3 * H * hd, 64) || make_map(&qkv64.hi, qkv, T, 3 * H * hd, 64, hi) ||
      make_map(&do64.lo, dout, T, H * hd, 64) || make_map(&do64.hi, dout, T, H * hd, 64, hi))
    return rp_fail(RP_ERR_CUDA, "attention_bwd_tc_wide: tensor map encode failed");
  const int smem = 1024 + BwdCfg<128>::kSmem;
  static std::once_flag once;
  static int nsm = 148;
  std::call_once(once, [smem] {
    cudaFuncSetAttribute(attn_bwd_tc<true, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(attn_bwd_tc<false, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  });
  BwdPlan pl;
  pl.ntile = static_cast<int>((N + 127) / 128);
  pl.nitems = static_cast<int>(S * H) * pl.ntile;
  const unsigned grid = static_cast<unsigned>(pl.nitems < nsm ? pl.nitems : nsm);
  // dQ (+ D): tiles Q | dO, chunks K | V
  launch_k(attn_bwd_tc<true, 128>, dim3(grid), dim3(kBwdThreads), smem, stream, qkv128, do128,
           qkv64, qkv64, reinterpret_cast<const __nv_bfloat16*>(out), lse, Dg,
           reinterpret_cast<__nv_bfloat16*>(dqkv), g, pl, static_cast<__nv_bfloat16*>(nullptr));
  // dK, dV: tiles K | V, chunks Q | dO
  launch_k(attn_bwd_tc<false, 128>, dim3(grid), dim3(kBwdThreads), smem, stream, qkv128, qkv128,
           qkv64, do64, reinterpret_cast<const __nv_bfloat16*>(out), lse, Dg,
           reinterpret_cast<__nv_bfloat16*>(dqkv), g, pl, static_cast<__nv_bfloat16*>(nullptr));
  return rp_check_launch("attention_bwd_tc_wide");
}
