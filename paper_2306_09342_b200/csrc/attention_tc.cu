// tcgen05 attention forward (head_dim 64): single-pass kernel for N <= 224, two-pass for N <= 512.
//
// Same contract as the mma.sync kernels in attention.cu (ref:proj/core/src/layers.cpp:150-166
// forward: scores = (q k^T) * 1/sqrt(hd), row softmax, probs . v; layers.cpp:185-208
// backward), with the products on the 5th-gen tensor cores, accumulators in TMEM, operands
// staged by TMA, and the softmax / softmax-VJP elementwise work done by warps reading and
// writing TMEM directly (P and dS are re-packed to bf16 in TMEM and fed back to the tensor
// core as the A operand). Keys beyond N (the next sequence's rows, or TMA zero fill past the
// end) are masked to -inf. See each kernel for its pipeline.
#include "attn_common.cuh"
#include "launch.h"

#include <cstring>

namespace rp {
namespace attn_tc {

// ------------------------------------------------------------- persistent forward
// One CTA per SM loops over work items = (sequence, head); an item has ntile = ceil(N/128)
// query tiles of 128 rows that share one K/V load. Sixteen softmax warps work on one tile at
// a time (warp w: TMEM lane quarter w%4 = 32 query rows, key quarter w/4 = up to 64 keys held
// in registers), while the MMA warp computes the next tile's S into the other TMEM buffer:
//   S(j)  = Q K^T        -> TMEM S buffer j%2 (Nk columns, Nk = N rounded up to 16)
//   softmax(j)           exact: the whole key row is in TMEM; one read, a 4-way max
//                        exchange through smem, p = exp2(s*scale*log2e - m), bf16 P packed
//                        to columns [0, Nk/2) of the same buffer
//   O(j)  = P V          A = P from TMEM, B = V (smem, MN-major)
//   epilogue(j)          O / l -> bf16 att, log2-domain LSE; done after softmax(j+1) has
//                        been handed to the MMA warp, so the PV latency is hidden
// Operands are double-buffered in smem (item i+1 streams in while item i is computed).
// With Nk <= 224 the O accumulator has its own TMEM columns [448, 512) and S(j+2) can be
// issued as soon as PV(j) is; for longer rows O lives in the S buffer at [192, 256) and
// S(j+2) waits for epilogue(j). Query row quarters past N skip the softmax.
constexpr int kFwdWarps = 17;  // warps 0-15 softmax / epilogue, warp 16 TMA + MMA issue
constexpr int kFwdThreads = kFwdWarps * 32;
constexpr int kFwdBuf = 3 * 256 * 128;  // Q (2 x 128 rows) | K (<= 256 rows) | V

struct FwdPlan {
  int ntile, nitems;
  int sb;    // TMEM column stride between the two S buffers
  int ocol;  // O accumulator column: absolute (o_sep) or relative to its S buffer
  int o_sep;
};

__global__ void __launch_bounds__(kFwdThreads, 1)
    attn_fwd_tc_persistent(const __grid_constant__ CUtensorMap tm_q,
                           const __grid_constant__ CUtensorMap tm_kv,
                           __nv_bfloat16* __restrict__ out, float* __restrict__ lse, Geom g,
                           FwdPlan pl) {
  pdl_trigger();

  __shared__ float red_max[2][4][128];  // [tile parity][key quarter][row]
  __shared__ float red_sum[2][4][128];
  __shared__ __align__(8) uint64_t bars[14];
  __shared__ uint32_t tmem_slot;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint64_t* bar_load = bars;      // [2] per smem buffer: TMA bytes landed
  uint64_t* bar_free = bars + 2;  // [2] per smem buffer: last PV reading it retired
  uint64_t* bar_s = bars + 4;     // [2] per S buffer: S ready
  uint64_t* bar_p = bars + 6;     // [2] per S buffer: P in TMEM (16 warps)
  uint64_t* bar_o = bars + 8;     // [2] per tile parity: O ready
  uint64_t* bar_e = bars + 10;    // [2] per tile parity: O read out (16 warps)

  const uint32_t warp = warp_id(), lane = lane_id();
  const int Nk = g.Nk, ntile = pl.ntile, nitems = pl.nitems;
  if (warp == 16) {
    if (lane == 0) {
      tma_prefetch_desc(&tm_q);
      tma_prefetch_desc(&tm_kv);
      for (int i = 0; i < 2; ++i) {
        mbar_init(&bar_load[i], 1);
        mbar_init(&bar_free[i], 1);
        mbar_init(&bar_s[i], 1);
        mbar_init(&bar_p[i], 16);
        mbar_init(&bar_o[i], 1);
        mbar_init(&bar_e[i], 16);
      }
      fence_barrier_init();
    }
    tmem_alloc(&tmem_slot, 512);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;
  pdl_wait();
  const int d = g.H * 64;
  const int K = nitems > static_cast<int>(blockIdx.x)
                    ? (nitems - static_cast<int>(blockIdx.x) + static_cast<int>(gridDim.x) - 1) /
                          static_cast<int>(gridDim.x)
                    : 0;
  const int J = K * ntile;  // tiles of this CTA
  auto item_of = [&](int k) { return static_cast<int>(blockIdx.x) + k * static_cast<int>(gridDim.x); };
  auto sbuf = [&](int j) { return tmem + static_cast<uint32_t>((j & 1) * pl.sb); };
  auto ocol = [&](int j) {
    return pl.o_sep ? tmem + static_cast<uint32_t>(pl.ocol) : sbuf(j) + static_cast<uint32_t>(pl.ocol);
  };

  if (warp == 16) {
    if (lane == 0) {
      auto issue_load = [&](int k) {
        const int item = item_of(k), buf = k & 1;
        const int h = item % g.H, b = item / g.H;
        const int row_seq = b * g.N;
        uint8_t* base = smem + buf * kFwdBuf;
        mbar_arrive_expect_tx(&bar_load[buf], (ntile * 128 + 2 * Nk) * 128);
        for (int t = 0; t < ntile; ++t)
          tma_load_2d(base + t * 16384, &tm_q, &bar_load[buf], h * 64, row_seq + t * 128);
        tma_load_2d(base + 32768, &tm_kv, &bar_load[buf], d + h * 64, row_seq);
        tma_load_2d(base + 65536, &tm_kv, &bar_load[buf], 2 * d + h * 64, row_seq);
      };
      auto ready = [](const uint64_t* bar, uint32_t parity) { return mbar_test(bar, parity); };
      const uint32_t idesc_s = make_idesc_bf16(128, static_cast<uint32_t>(Nk), false, false);
      const uint32_t idesc_o = make_idesc_bf16(128, 64, false, true);
      int jS = 0, jP = 0, kL = 0;
      while (jP < J) {
        // next item's operands into the smem buffer its predecessor-but-one has released
        if (kL < K && (kL < 2 || ready(&bar_free[kL & 1], ((kL - 2) >> 1) & 1))) {
          issue_load(kL);
          ++kL;
        }
        // S(jS): operands landed, S buffer free (PV(jS-2) issued, or its O read out)
        if (jS < J && jS < jP + 2) {
          const int k = jS / ntile, t = jS % ntile;
          const bool buf_ok = jS < 2 || (pl.o_sep ? true : ready(&bar_e[jS & 1], ((jS - 2) >> 1) & 1));
          if (k < kL && buf_ok && ready(&bar_load[k & 1], (k >> 1) & 1)) {
            tc_fence_after();
            const uint32_t base = smem_u32(smem + (k & 1) * kFwdBuf);
            const uint32_t aq = base + static_cast<uint32_t>(t) * 16384u, bk = base + 32768u;
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              umma_bf16(sbuf(jS), make_sdesc_sw128(aq + kk * 32, 16, 1024),
                        make_sdesc_sw128(bk + kk * 32, 16, 1024), idesc_s, kk > 0 ? 1u : 0u);
            umma_commit(&bar_s[jS & 1]);
            ++jS;
          }
        }
        // PV(jP): P written, and (shared O) the previous tile's O read out
        if (jP < jS && ready(&bar_p[jP & 1], (jP >> 1) & 1) &&
            (!pl.o_sep || jP == 0 || ready(&bar_e[(jP - 1) & 1], ((jP - 1) >> 1) & 1))) {
          tc_fence_after();
          const int k = jP / ntile;
          const uint32_t bv = smem_u32(smem + (k & 1) * kFwdBuf) + 65536u;
          const uint32_t sb = sbuf(jP), od = ocol(jP);
          for (int c = 0; c < Nk / 16; ++c)
            umma_ts_bf16(od, sb + static_cast<uint32_t>(c * 8),
                         make_sdesc_sw128(bv + c * 2048, 8192, 1024), idesc_o, c > 0 ? 1u : 0u);
          umma_commit(&bar_o[jP & 1]);
          if (jP % ntile == ntile - 1) umma_commit(&bar_free[k & 1]);
          ++jP;
        }
      }
    }
  } else {
    // ---- softmax / epilogue: warp w owns TMEM lane quarter q = w%4 and key quarter cq = w/4
    const int q = static_cast<int>(warp & 3u), cq = static_cast<int>(warp >> 2);
    const int nch = Nk / 16;
    const int ch0 = cq * nch / 4, ch1 = (cq + 1) * nch / 4;  // this warp's 16-key chunks
    const int c0 = ch0 * 16;
    const uint32_t lq = (static_cast<uint32_t>(q) * 32u) << 16;
    const int rloc = q * 32 + static_cast<int>(lane);
    const int valid = g.N;
    auto epilogue = [&](int j, float ms) {
      const int k = j / ntile, t = j % ntile;
      const int item = item_of(k);
      const int h = item % g.H, b = item / g.H;
      const int row = t * 128 + rloc;
      const bool active = t * 128 + q * 32 < g.N;
      mbar_wait(&bar_o[j & 1], (j >> 1) & 1);
      tc_fence_after();
      float o[16];
      if (active) tmem_ld16(ocol(j) + lq + static_cast<uint32_t>(cq * 16), o);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar_e[j & 1]);
      if (row < g.N) {
        const float* rs = &red_sum[j & 1][0][rloc];
        const float l = (rs[0] + rs[128]) + (rs[256] + rs[384]);
        const float inv = 1.0f / l;
        uint4* dst = reinterpret_cast<uint4*>(
            out + (static_cast<int64_t>(b) * g.N + row) * g.ld_o + h * 64 + cq * 16);
        dst[0] = make_uint4(pack_bf16x2(o[0] * inv, o[1] * inv), pack_bf16x2(o[2] * inv, o[3] * inv),
                            pack_bf16x2(o[4] * inv, o[5] * inv), pack_bf16x2(o[6] * inv, o[7] * inv));
        dst[1] = make_uint4(pack_bf16x2(o[8] * inv, o[9] * inv),
                            pack_bf16x2(o[10] * inv, o[11] * inv),
                            pack_bf16x2(o[12] * inv, o[13] * inv),
                            pack_bf16x2(o[14] * inv, o[15] * inv));
        if (cq == 0) lse[(static_cast<int64_t>(b) * g.H + h) * g.N + row] = ms + log2f(l);
      }
    };
    float ms_prev = 0.f;
    for (int j = 0; j < J; ++j) {
      const int t = j % ntile;
      const bool active = t * 128 + q * 32 < g.N;  // some row of this quarter is a real query
      const uint32_t sb = sbuf(j) + lq;
      mbar_wait(&bar_s[j & 1], (j >> 1) & 1);
      tc_fence_after();
      float v[64];
      float mx = -INFINITY;
      if (active) {
        tmem_ld16x4(sb + c0, sb + c0 + 16, sb + c0 + 32, sb + c0 + 48, v, v + 16, v + 32, v + 48);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int ch = ch0 + i;
          if (ch < ch1) {
            if (ch * 16 + 16 <= valid) {
#pragma unroll
              for (int e = 0; e < 16; ++e) mx = fmaxf(mx, v[16 * i + e]);
            } else {
#pragma unroll
              for (int e = 0; e < 16; ++e)
                if (ch * 16 + e < valid) mx = fmaxf(mx, v[16 * i + e]);
            }
          }
        }
      }
      red_max[j & 1][cq][rloc] = mx;
      // the four warps of this lane quarter have read their S columns: P may now overwrite
      // [0, Nk/2) of these lanes (only they exchange maxima and sums for these rows)
      named_bar(1 + q, 128);
      const float* rm = &red_max[j & 1][0][rloc];
      const float ms = fmaxf(fmaxf(rm[0], rm[128]), fmaxf(rm[256], rm[384])) * g.scale_log2;
      float l = 0.f;
      if (active) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int ch = ch0 + i;
          if (ch < ch1) {
            uint32_t pk[8];
            if (ch * 16 + 16 <= valid) {
#pragma unroll
              for (int e = 0; e < 8; ++e) {
                const float p0 = ex2(fmaf(v[16 * i + 2 * e], g.scale_log2, -ms));
                const float p1 = ex2(fmaf(v[16 * i + 2 * e + 1], g.scale_log2, -ms));
                l += p0 + p1;
                pk[e] = pack_bf16x2(p0, p1);
              }
            } else {
#pragma unroll
              for (int e = 0; e < 8; ++e) {
                const int key = ch * 16 + 2 * e;
                const float p0 = key < valid ? ex2(fmaf(v[16 * i + 2 * e], g.scale_log2, -ms)) : 0.f;
                const float p1 =
                    key + 1 < valid ? ex2(fmaf(v[16 * i + 2 * e + 1], g.scale_log2, -ms)) : 0.f;
                l += p0 + p1;
                pk[e] = pack_bf16x2(p0, p1);
              }
            }
            tmem_st8(sb + static_cast<uint32_t>(ch * 8), pk);
          }
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar_p[j & 1]);
      red_sum[j & 1][cq][rloc] = l;
      if (j > 0) epilogue(j - 1, ms_prev);  // its sums were published before this barrier
      ms_prev = ms;
    }
    if (J > 0) {
      named_bar(1 + q, 128);  // last tile's sums
      epilogue(J - 1, ms_prev);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 16) tmem_dealloc(tmem, 512);
}

// ------------------------------------------------------------- ping-pong forward (N <= 256)
// The persistent kernel above runs its 16 softmax warps in lockstep on one tile: all of them
// sit in the row-max pass, the max exchange or the O epilogue at the same time, so the MUFU
// pipe (the exp2 floor: 16 / clock / SM, measured, tools/tmem_mufu_bench.cu) idles for most
// of every tile. Here the softmax warps form TWO groups that own alternate tiles (group g:
// tiles j = g, g + 2, ...), each warp a TMEM lane quarter q = w % 4 (its SM sub-partition)
// and a key half; while one group exchanges maxima or drains O, the other group's exp2
// stream keeps the MUFU busy. Per tile and warp:
//   pass 1   row max over the warp's key half, read from S in TMEM (16-column loads)
//   xchg     max with the partner warp of the same quarter and group (named barrier, 64)
//   pass 2   S re-read, p = exp2(s scale log2e - m), bf16 P packed IN the warp's own S
//            columns (half 0: chunk c -> column 8c; half 1: 16 cs + 8 (c - cs)), row sums
//   PV       issued by the MMA warp once the group's 8 warps arrived; O accumulates at
//            column ocol of the tile's own S buffer (free once P is packed)
//   epilogue O / l (sums exchanged the same way) -> bf16 att, log2-domain LSE
// S is double-buffered (buffer j % 2 at column 256 (j % 2)); S(j + 2) waits for
// epilogue(j). Works for N <= 256 (the persistent kernel stops at 224).
// Warp 16 issues the loads and S = Q K^T, warps 17 and 18 the P V products (a PV then never
// waits behind an S issue). One N = 64 MMA costs its issuing thread ~120 cycles whatever N
// (tools/umma_bench.cu), so with Nk <= 208 ("split" plan) the P V product is split by key
// half into two accumulators issued by the two warps in parallel (7 + 6 MMAs instead of 13
// in a row) and summed in the epilogue: key half 1 packs its P into the free tail columns
// [p1, 256) of the S buffer (never S columns, so no race with half 0's reads), which leaves
// the whole middle of the buffer dead once both halves are packed: O_a and O_b at oa and
// oa + 64. Otherwise (one accumulator at ocol) warp 17 issues every P V.
// (Splitting the PV issue per GROUP over two warps measured slower.)
constexpr int kPPThreads = kFwdThreads + 64;
struct PPPlan {
  int ntile, nitems;
  int cs;    // 16-key chunks in key half 0 (the rest are half 1's)
  int ocol;  // O accumulator column inside each S buffer (O_a with split)
  int split; // two P V accumulators (O_a at ocol, O_b at ocol + 64), half 1's P at p1
  int p1;    // split: first TMEM column of key half 1's packed P
  unsigned long long* trace;  // optional clock64 trace of CTA 0's first kTraceTiles tiles
};
constexpr int kTraceTiles = 64;
#define PP_TRACE(j, slot)                                                                   \
  do {                                                                                      \
    if (pl.trace && blockIdx.x == 0 && (j) < kTraceTiles)                                  \
      pl.trace[(j) * 12 + (slot)] = static_cast<unsigned long long>(clock64());            \
  } while (0)

__device__ __forceinline__ uint32_t pp_pcol(int c, int cs, int p1) {
  return static_cast<uint32_t>(c < cs ? 8 * c : p1 + 8 * (c - cs));
}

__global__ void __launch_bounds__(kPPThreads, 1)
    attn_fwd_tc_pp(const __grid_constant__ CUtensorMap tm_q,
                   const __grid_constant__ CUtensorMap tm_kv, __nv_bfloat16* __restrict__ out,
                   float* __restrict__ lse, Geom g, PPPlan pl) {
  pdl_trigger();

  __shared__ float red_max[2][2][128];  // [group][key half][row]
  __shared__ float red_sum[2][2][128];
  __shared__ __align__(8) uint64_t bars[12];
  __shared__ uint32_t tmem_slot;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint64_t* bar_load = bars;      // [2] per smem buffer: TMA bytes landed
  uint64_t* bar_free = bars + 2;  // [2] per smem buffer: every tile's epilogue done with it
  uint64_t* bar_s = bars + 4;     // [2] per S buffer: S ready
  uint64_t* bar_p = bars + 6;     // [2] per S buffer: P in TMEM (8 warps of the group)
  uint64_t* bar_o = bars + 8;     // [2] per S buffer: O ready
  uint64_t* bar_e = bars + 10;    // [2] per S buffer: O read out (8 warps)

  const uint32_t warp = warp_id(), lane = lane_id();
  const int Nk = g.Nk, ntile = pl.ntile, nitems = pl.nitems, nch = g.Nk / 16, cs = pl.cs;
  const int p1 = pl.split ? pl.p1 : 16 * cs;  // half 1's P: tail columns, or its own S columns
  if (warp == 16) {
    if (lane == 0) {
      tma_prefetch_desc(&tm_q);
      tma_prefetch_desc(&tm_kv);
      for (int i = 0; i < 2; ++i) {
        mbar_init(&bar_load[i], 1);
        mbar_init(&bar_free[i], static_cast<uint32_t>(8 * pl.ntile));
        mbar_init(&bar_s[i], 1);
        mbar_init(&bar_p[i], 8);
        mbar_init(&bar_o[i], pl.split ? 2 : 1);
        mbar_init(&bar_e[i], 8);
      }
      fence_barrier_init();
    }
    tmem_alloc(&tmem_slot, 512);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;
  pdl_wait();
  const int d = g.H * 64;
  const int K = nitems > static_cast<int>(blockIdx.x)
                    ? (nitems - static_cast<int>(blockIdx.x) + static_cast<int>(gridDim.x) - 1) /
                          static_cast<int>(gridDim.x)
                    : 0;
  const int J = K * ntile;
  auto item_of = [&](int k) { return static_cast<int>(blockIdx.x) + k * static_cast<int>(gridDim.x); };
  auto sbuf = [&](int j) { return tmem + static_cast<uint32_t>((j & 1) * 256); };

  if (warp == 16) {
    if (lane == 0) {
      auto issue_load = [&](int k) {
        const int item = item_of(k), buf = k & 1;
        const int h = item % g.H, b = item / g.H;
        const int row_seq = b * g.N;
        uint8_t* base = smem + buf * kFwdBuf;
        mbar_arrive_expect_tx(&bar_load[buf], (ntile * 128 + 2 * Nk) * 128);
        for (int t = 0; t < ntile; ++t)
          tma_load_2d(base + t * 16384, &tm_q, &bar_load[buf], h * 64, row_seq + t * 128);
        tma_load_2d(base + 32768, &tm_kv, &bar_load[buf], d + h * 64, row_seq);
        tma_load_2d(base + 65536, &tm_kv, &bar_load[buf], 2 * d + h * 64, row_seq);
      };
      auto ready = [](const uint64_t* bar, uint32_t parity) { return mbar_test(bar, parity); };
      const uint32_t idesc_s = make_idesc_bf16(128, static_cast<uint32_t>(Nk), false, false);
      int jS = 0, kL = 0;
      while (jS < J) {
        if (kL < K && (kL < 2 || ready(&bar_free[kL & 1], ((kL - 2) >> 1) & 1))) {
          issue_load(kL);
          ++kL;
        }
        // S(jS): operands landed and the S buffer's previous tile (jS - 2) drained
        {
          const int k = jS / ntile, t = jS % ntile;
          const bool buf_ok = jS < 2 || ready(&bar_e[jS & 1], ((jS - 2) >> 1) & 1);
          if (k < kL && buf_ok && ready(&bar_load[k & 1], (k >> 1) & 1)) {
            tc_fence_after();
            const uint32_t base = smem_u32(smem + (k & 1) * kFwdBuf);
            const uint32_t aq = base + static_cast<uint32_t>(t) * 16384u, bk = base + 32768u;
            PP_TRACE(jS, 0);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              umma_bf16(sbuf(jS), make_sdesc_sw128(aq + kk * 32, 16, 1024),
                        make_sdesc_sw128(bk + kk * 32, 16, 1024), idesc_s, kk > 0 ? 1u : 0u);
            umma_commit(&bar_s[jS & 1]);
            PP_TRACE(jS, 1);
            ++jS;
          }
        }
      }
    }
  } else if (warp == 17 || warp == 18) {
    // P V issuers (both groups' tiles in order), so a PV never waits behind an S issue:
    // warp 17 key half 0 into O_a (all keys without the split), warp 18 key half 1 into O_b
    const bool hb = warp == 18;
    if (lane == 0 && (pl.split || !hb)) {
      const uint32_t idesc_o = make_idesc_bf16(128, 64, false, true);
      const int c0 = hb ? cs : 0, c1 = pl.split && !hb ? cs : nch;
      const uint32_t ocol = static_cast<uint32_t>(pl.ocol + (hb ? 64 : 0));
      for (int jP = 0; jP < J; ++jP) {
        mbar_wait(&bar_p[jP & 1], (jP >> 1) & 1);
        tc_fence_after();
        const int k = jP / ntile;
        const uint32_t bv = smem_u32(smem + (k & 1) * kFwdBuf) + 65536u;
        const uint32_t sb = sbuf(jP), od = sb + ocol;
        if (!hb) PP_TRACE(jP, 2);
        for (int c = c0; c < c1; ++c)
          umma_ts_bf16(od, sb + pp_pcol(c, cs, p1), make_sdesc_sw128(bv + c * 2048, 8192, 1024),
                       idesc_o, c > c0 ? 1u : 0u);
        umma_commit(&bar_o[jP & 1]);
        if (!hb) PP_TRACE(jP, 3);
      }
    }
  } else {
    const int q = static_cast<int>(warp & 3u), r = static_cast<int>(warp >> 2);
    const int grp = r >> 1, half = r & 1;
    const int ch0 = half ? cs : 0, ch1 = half ? nch : cs;
    const uint32_t lq = (static_cast<uint32_t>(q) * 32u) << 16;
    const int rloc = q * 32 + static_cast<int>(lane);
    const int valid = g.N;
    const int bar_id = 1 + grp * 4 + q;
    for (int j = grp; j < J; j += 2) {
      const int k = j / ntile, t = j % ntile;
      const bool active = t * 128 + q * 32 < g.N;
      const uint32_t sb = sbuf(j) + lq;
      const bool tr = q == 0 && half == 0 && lane == 0;
      if (tr) PP_TRACE(j, 4);
      mbar_wait(&bar_s[j & 1], (j >> 1) & 1);
      tc_fence_after();
      if (tr) PP_TRACE(j, 5);
      // ---- pass 1: row max over this warp's key half, two chunks per TMEM wait (four would
      // need > 96 registers: with 18 warps, five share an SM sub-partition's 16 K registers)
      float m0 = -INFINITY, m1 = -INFINITY;
      if (active) {
        for (int c = ch0; c < ch1; c += 2) {
          const uint32_t a0 = sb + static_cast<uint32_t>(c * 16);
          float va[16], vb[16];
          if (c + 1 < ch1) {
            tmem_ld16x2(a0, a0 + 16, va, vb);
          } else {
            tmem_ld16(a0, va);
#pragma unroll
            for (int e = 0; e < 16; ++e) vb[e] = -INFINITY;
          }
          if ((c + 2) * 16 <= valid) {
#pragma unroll
            for (int e = 0; e < 16; e += 2) {
              m0 = fmaxf(m0, fmaxf(va[e], va[e + 1]));
              m1 = fmaxf(m1, fmaxf(vb[e], vb[e + 1]));
            }
          } else {
#pragma unroll
            for (int e = 0; e < 16; ++e) {
              if (c * 16 + e < valid) m0 = fmaxf(m0, va[e]);
              if (c * 16 + 16 + e < valid && c + 1 < ch1) m1 = fmaxf(m1, vb[e]);
            }
          }
        }
      }
      red_max[grp][half][rloc] = fmaxf(m0, m1);
      if (tr) PP_TRACE(j, 6);
      named_bar(bar_id, 64);
      if (tr) PP_TRACE(j, 7);
      const float ms = fmaxf(red_max[grp][0][rloc], red_max[grp][1][rloc]) * g.scale_log2;
      // ---- pass 2: p = exp2(s * scale - m), packed bf16 P in this warp's own S columns
      // (a chunk's P lands on columns already read)
      float l0 = 0.f, l1 = 0.f;
      auto expchunk = [&](const float* a, int cc) {
        uint32_t pk[8];
        if (cc * 16 + 16 <= valid) {
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const float p0 = ex2(fmaf(a[2 * e], g.scale_log2, -ms));
            const float p1 = ex2(fmaf(a[2 * e + 1], g.scale_log2, -ms));
            l0 += p0;
            l1 += p1;
            pk[e] = pack_bf16x2(p0, p1);
          }
        } else {
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const int key = cc * 16 + 2 * e;
            const float p0 = key < valid ? ex2(fmaf(a[2 * e], g.scale_log2, -ms)) : 0.f;
            const float p1 = key + 1 < valid ? ex2(fmaf(a[2 * e + 1], g.scale_log2, -ms)) : 0.f;
            l0 += p0;
            l1 += p1;
            pk[e] = pack_bf16x2(p0, p1);
          }
        }
        tmem_st8(sb + pp_pcol(cc, cs, p1), pk);
      };
      if (active) {
        for (int c = ch0; c < ch1; c += 2) {
          const uint32_t a0 = sb + static_cast<uint32_t>(c * 16);
          if (c + 1 < ch1) {
            float va[16], vb[16];
            tmem_ld16x2(a0, a0 + 16, va, vb);
            expchunk(va, c);
            expchunk(vb, c + 1);
          } else {
            float va[16];
            tmem_ld16(a0, va);
            expchunk(va, c);
          }
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar_p[j & 1]);
      if (tr) PP_TRACE(j, 8);
      red_sum[grp][half][rloc] = l0 + l1;
      named_bar(bar_id, 64);
      const float l = red_sum[grp][0][rloc] + red_sum[grp][1][rloc];
      // ---- epilogue: O / l -> att (this warp's 32 of the 64 head columns), LSE; the
      // reciprocal and log (MUFU) are taken before waiting for O
      const int item = item_of(k);
      const int h = item % g.H, b = item / g.H;
      const int row = t * 128 + rloc;
      const float inv = 1.0f / l;
      const float lse_v = ms + log2f(l);
      mbar_wait(&bar_o[j & 1], (j >> 1) & 1);
      tc_fence_after();
      if (tr) PP_TRACE(j, 9);
      float o[32];
      if (active) {
        const uint32_t oa = sbuf(j) + lq + static_cast<uint32_t>(pl.ocol + half * 32);
        tmem_ld16x2(oa, oa + 16, o, o + 16);
        if (pl.split) {  // + O_b, summed in a fixed order
          float ob[32];
          tmem_ld16x2(oa + 64, oa + 80, ob, ob + 16);
#pragma unroll
          for (int e = 0; e < 32; ++e) o[e] += ob[e];
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar_e[j & 1]);
      // O / l staged through the tile's own Q slot in smem (dead since S(j); 128 rows x 128 B,
      // 16-byte chunks XOR-swizzled by row so the row-per-lane writes are conflict free), then
      // written back as whole 128-byte rows (8 lanes per row): coalesced, where a direct
      // row-per-lane store scatters each warp instruction over 32 lines. The item's smem
      // buffer is released (bar_free) by these warps once the staging is read back.
      const uint32_t stg = smem_u32(smem + (k & 1) * kFwdBuf + t * 16384);
      if (active) {
        const uint32_t rbase = stg + static_cast<uint32_t>(rloc) * 128u;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t ch = static_cast<uint32_t>((half * 4 + u) ^ (rloc & 7));
          sts128_a(rbase + ch * 16u,
                 make_uint4(pack_bf16x2(o[8 * u] * inv, o[8 * u + 1] * inv),
                            pack_bf16x2(o[8 * u + 2] * inv, o[8 * u + 3] * inv),
                            pack_bf16x2(o[8 * u + 4] * inv, o[8 * u + 5] * inv),
                            pack_bf16x2(o[8 * u + 6] * inv, o[8 * u + 7] * inv)));
        }
      }
      if (row < g.N && half == 0) lse[(static_cast<int64_t>(b) * g.H + h) * g.N + row] = lse_v;
      named_bar(bar_id, 64);  // both halves of these 32 rows staged
      if (active) {
#pragma unroll
        for (int it = 0; it < 4; ++it) {
          const int rl = q * 32 + half * 16 + it * 4 + static_cast<int>(lane >> 3);
          const int ch = static_cast<int>(lane & 7);
          const int grow = t * 128 + rl;
          const uint4 x = lds128_a(stg + static_cast<uint32_t>(rl) * 128u +
                                 static_cast<uint32_t>((ch ^ (rl & 7)) * 16));
          if (grow < g.N)
            *reinterpret_cast<uint4*>(out + (static_cast<int64_t>(b) * g.N + grow) * g.ld_o +
                                      h * 64 + ch * 8) = x;
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar_free[k & 1]);
      if (tr) PP_TRACE(j, 10);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 16) tmem_dealloc(tmem, 512);
}

// ------------------------------------------------------------- long-sequence forward
// 224 < N <= 512 (the Rev-RoBERTa shape): the key row no longer fits next to its O in one
// TMEM buffer, so each 128-query tile makes two passes over 128-key blocks:
//   pass 1   S_j = Q K_j^T, row max only (FMNMX, no exponentials)
//   pass 2   S_j again, p = exp2(s * scale * log2e - m), row sums, bf16 P packed over the
//            block's own S columns, O += P V_j (one O accumulator, no rescaling needed)
// An item is (sequence, head, group of up to pl.group query tiles); its K and V (<= 512
// rows each) are resident in smem for the whole group, Q tiles are double-buffered. Sixteen
// elementwise warps (TMEM lane quarter w%4, 32-key column quarter w/4 of a block) and one
// TMA + MMA warp; S is double-buffered in TMEM so the next block's S is computed while the
// current one is processed.
// HP = 128 (head dims 72..128, N <= 256): every operand is two 64-column atom planes, the
// second loaded by a TMA box of hd - 64 columns whose untouched tail stays zero (as in the
// wide backward), S = Q K^T takes round16(hd) / 16 K steps and O has round16(hd) columns.
constexpr int kLongKV = 2 * 512 * 128;  // K | V, up to 512 rows each (HP = 64)
template <int HP>
struct LongCfg {
  static constexpr int kAtoms = HP / 64;
  static constexpr int kMaxRows = HP == 64 ? 512 : 256;        // resident keys
  static constexpr int kPlaneKV = kMaxRows * 128;               // one atom plane of K or V
  static constexpr int kKV = 2 * kAtoms * kPlaneKV;             // K | V
  static constexpr int kQTile = 128 * 128 * kAtoms;             // one Q tile
  static constexpr int kSmem = kKV + 2 * kQTile;
};

struct LongPlan {
  int nitems, ntile, ngroup;  // items = S * H * ngroup; ntile query tiles per sequence
  int group;                  // query tiles per item (K, V loaded once per item)
  int nkb;                    // 128-key blocks
  int hd;                     // head dim (64 on HP = 64)
};

struct LongMaps {
  CUtensorMap lo, hi;  // qkv boxes of {64, 128} and (HP = 128) {hd - 64, 128}
};

template <int HP>
__global__ void __launch_bounds__(kFwdThreads, 1)
    attn_fwd_tc_long(const __grid_constant__ LongMaps tm, __nv_bfloat16* __restrict__ out,
                     float* __restrict__ lse, Geom g, LongPlan pl) {
  using Cfg = LongCfg<HP>;
  pdl_trigger();

  __shared__ float red_max[4][128];
  __shared__ float red_sum[4][128];
  __shared__ __align__(8) uint64_t bars[16];
  __shared__ uint32_t tmem_slot;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sK = smem;                                 // [atom][kMaxRows rows]
  uint8_t* sV = smem + Cfg::kAtoms * Cfg::kPlaneKV;   // [atom][kMaxRows rows]
  uint8_t* sQ = smem + Cfg::kKV;                      // [2][atom][128 rows]
  uint64_t* kv_full = bars + 12;            // [4] K, V rows of 128-key block j of the item landed
  uint64_t* kv_free = bars + 1;             // the item's last MMA retired
  uint64_t* q_full = bars + 2;              // [2]
  uint64_t* q_free = bars + 4;              // [2] the tile's last S MMA retired
  uint64_t* bar_s = bars + 6;               // [2] per S buffer
  uint64_t* bar_p = bars + 8;               // [2] per S buffer: consumed (16 warps)
  uint64_t* bar_o = bars + 10;              // O of the tile complete
  uint64_t* bar_e = bars + 11;              // O read out (16 warps)

  const uint32_t warp = warp_id(), lane = lane_id();
  const int Nk = g.Nk, nkb = pl.nkb;
  const int hd = HP == 64 ? 64 : pl.hd;
  if constexpr (HP > 64) {
    // the second atom plane's columns past hd are never written by the TMA: zero them once
    for (int i = static_cast<int>(threadIdx.x) * 16; i < Cfg::kSmem; i += kFwdThreads * 16)
      *reinterpret_cast<uint4*>(smem + i) = make_uint4(0, 0, 0, 0);
    fence_proxy_async_smem();
  }
  if (warp == 16) {
    if (lane == 0) {
      tma_prefetch_desc(&tm.lo);
      for (int j = 0; j < 4; ++j) mbar_init(&kv_full[j], 1);
      mbar_init(kv_free, 1);
      for (int i = 0; i < 2; ++i) {
        mbar_init(&q_full[i], 1);
        mbar_init(&q_free[i], 1);
        mbar_init(&bar_s[i], 1);
        mbar_init(&bar_p[i], 16);
      }
      mbar_init(bar_o, 1);
      mbar_init(bar_e, 16);
      fence_barrier_init();
    }
    tmem_alloc(&tmem_slot, 512);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;
  pdl_wait();
  const int d = g.H * hd;
  const int K = pl.nitems > static_cast<int>(blockIdx.x)
                    ? (pl.nitems - static_cast<int>(blockIdx.x) + static_cast<int>(gridDim.x) - 1) /
                          static_cast<int>(gridDim.x)
                    : 0;
  auto coords = [&](int k, int& b, int& h, int& t0, int& nt) {
    const int item = static_cast<int>(blockIdx.x) + k * static_cast<int>(gridDim.x);
    const int grp = item % pl.ngroup, bh = item / pl.ngroup;
    h = bh % g.H;
    b = bh / g.H;
    t0 = grp * pl.group;
    nt = min(pl.group, pl.ntile - t0);
  };
  const uint32_t ocol = tmem + 256u;

  if (warp == 16) {
    if (lane == 0) {
      const int nacc = (hd + 15) / 16 * 16, nks = nacc / 16;
      const uint32_t idesc_o = make_idesc_bf16(128, static_cast<uint32_t>(nacc), false, true);
      // flat unit sequence: per item, per tile, pass 1 blocks then pass 2 blocks
      int u = 0, tt = 0;  // unit and global tile counters
      // 128 rows of one operand at head column col: atom planes `plane` bytes apart
      auto load_rows = [&](uint8_t* dst, uint64_t* bar, int col, int row, int plane) {
        tma_load_2d(dst, &tm.lo, bar, col, row);
        if constexpr (HP > 64) tma_load_2d(dst + plane, &tm.hi, bar, col + 64, row);
      };
      auto load_q = [&](int k, int t, int slot) {
        int b, h, t0, nt;
        coords(k, b, h, t0, nt);
        mbar_arrive_expect_tx(&q_full[slot], static_cast<uint32_t>(128 * hd * 2));
        load_rows(sQ + slot * Cfg::kQTile, &q_full[slot], h * hd, b * g.N + (t0 + t) * 128, 16384);
      };
      auto load_kv = [&](int k) {
        int b, h, t0, nt;
        coords(k, b, h, t0, nt);
        // per 128-key block, so the item's first S waits for its first block only (the rest
        // of K and V lands under it)
        for (int j = 0; j < nkb; ++j) {  // 128-row boxes (a TMA box is at most 256 rows)
          mbar_arrive_expect_tx(&kv_full[j], static_cast<uint32_t>(2 * 128 * hd * 2));
          load_rows(sK + j * 16384, &kv_full[j], d + h * hd, b * g.N + 128 * j, Cfg::kPlaneKV);
          load_rows(sV + j * 16384, &kv_full[j], 2 * d + h * hd, b * g.N + 128 * j, Cfg::kPlaneKV);
        }
      };
      if (K > 0) {
        load_kv(0);
        load_q(0, 0, 0);
      }
      for (int k = 0; k < K; ++k) {
        int b, h, t0, nt;
        coords(k, b, h, t0, nt);
        if (k > 0) {
          mbar_wait(kv_free, (k - 1) & 1);  // every MMA of item k-1 retired
          load_kv(k);
        }
        for (int t = 0; t < nt; ++t, ++tt) {
          // next tile's Q (this item's next tile or the next item's first one)
          {
            int nk = k, ntl = t + 1;
            if (ntl >= nt) { nk = k + 1; ntl = 0; }
            if (nk < K) {
              if (tt >= 1) mbar_wait(&q_free[(tt + 1) & 1], ((tt - 1) >> 1) & 1);
              load_q(nk, ntl, (tt + 1) & 1);
            }
          }
          mbar_wait(&q_full[tt & 1], (tt >> 1) & 1);
          const uint32_t aq = smem_u32(sQ + (tt & 1) * Cfg::kQTile);
          // the tile's units: nkb pass-1 blocks then nkb pass-2 blocks. S of unit i + 1 is
          // issued before the P V of unit i, so the elementwise warps' next block overlaps
          // the P V products (S is double-buffered; the P V of unit i - 1, which reads the
          // buffer S(i + 1) overwrites, was issued earlier and MMAs retire in order)
          const int U = 2 * nkb, ubase = u;
          auto issue_s = [&](int i) {
            const int gu = ubase + i, j = i % nkb;
            const int w = min(128, Nk - 128 * j);
            if (t == 0 && i < nkb) mbar_wait(&kv_full[j], k & 1);  // the item's K, V block j
            if (gu >= 2) mbar_wait(&bar_p[gu & 1], ((gu - 2) >> 1) & 1);  // buffer consumed
            tc_fence_after();
            const uint32_t sb = tmem + static_cast<uint32_t>((gu & 1) * 128);
            const uint32_t bk = smem_u32(sK) + static_cast<uint32_t>(128 * j * 128);
            const uint32_t idesc_s = make_idesc_bf16(128, static_cast<uint32_t>(w), false, false);
            for (int kk = 0; kk < nks; ++kk)
              umma_bf16(sb, make_sdesc_sw128(aq + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
                        make_sdesc_sw128(bk + (kk >> 2) * Cfg::kPlaneKV + (kk & 3) * 32, 16, 1024),
                        idesc_s, kk > 0 ? 1u : 0u);
            umma_commit(&bar_s[gu & 1]);
            if (i == U - 1) umma_commit(&q_free[tt & 1]);
          };
          issue_s(0);
          for (int i = 0; i < U; ++i) {
            if (i + 1 < U) issue_s(i + 1);
            if (i >= nkb) {  // pass 2: O += P V_j
              const int gu = ubase + i, j = i - nkb;
              const int w = min(128, Nk - 128 * j);
              if (j == 0 && tt > 0) mbar_wait(bar_e, (tt - 1) & 1);  // previous O read out
              mbar_wait(&bar_p[gu & 1], (gu >> 1) & 1);
              tc_fence_after();
              const uint32_t sb = tmem + static_cast<uint32_t>((gu & 1) * 128);
              const uint32_t bv = smem_u32(sV) + static_cast<uint32_t>(128 * j * 128);
              for (int ks = 0; ks < w / 16; ++ks)
                umma_ts_bf16(ocol, sb + static_cast<uint32_t>((ks >> 1) * 32 + (ks & 1) * 8),
                             make_sdesc_sw128(bv + ks * 2048, HP == 64 ? 8192 : Cfg::kPlaneKV, 1024),
                             idesc_o, (j > 0 || ks > 0) ? 1u : 0u);
              if (j == nkb - 1) umma_commit(bar_o);
            }
          }
          u += U;
        }
        umma_commit(kv_free);
      }
    }
  } else {
    const int q = static_cast<int>(warp & 3u), cq = static_cast<int>(warp >> 2);
    const uint32_t lq = (static_cast<uint32_t>(q) * 32u) << 16;
    const int rloc = q * 32 + static_cast<int>(lane);
    int u = 0, tt = 0;
    for (int k = 0; k < K; ++k) {
      int b, h, t0, nt;
      coords(k, b, h, t0, nt);
      for (int t = 0; t < nt; ++t, ++tt) {
        const int tile = t0 + t;
        const bool active = tile * 128 + q * 32 < g.N;
        float mx = -INFINITY;
        for (int j = 0; j < nkb; ++j, ++u) {  // ---- pass 1: row max
          const int c0 = 128 * j + 32 * cq;
          mbar_wait(&bar_s[u & 1], (u >> 1) & 1);
          tc_fence_after();
          if (active && c0 < Nk) {
            float v[32];
            tmem_ld32(tmem + static_cast<uint32_t>((u & 1) * 128 + 32 * cq) + lq, v);
#pragma unroll
            for (int e = 0; e < 32; ++e)
              if (c0 + e < g.N) mx = fmaxf(mx, v[e]);
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&bar_p[u & 1]);
        }
        red_max[cq][rloc] = mx;
        named_bar(1 + q, 128);  // only the four warps of a lane quarter share rows
        const float ms =
            fmaxf(fmaxf(red_max[0][rloc], red_max[1][rloc]), fmaxf(red_max[2][rloc], red_max[3][rloc])) *
            g.scale_log2;
        float l = 0.f;
        for (int j = 0; j < nkb; ++j, ++u) {  // ---- pass 2: exp, sums, P
          const int c0 = 128 * j + 32 * cq;
          mbar_wait(&bar_s[u & 1], (u >> 1) & 1);
          tc_fence_after();
          if (active && c0 < Nk) {
            const uint32_t sb = tmem + static_cast<uint32_t>((u & 1) * 128 + 32 * cq) + lq;
            float v[32];
            tmem_ld32(sb, v);
            uint32_t pk[16];
#pragma unroll
            for (int e = 0; e < 16; ++e) {
              const int key = c0 + 2 * e;
              const float p0 = key < g.N ? ex2(fmaf(v[2 * e], g.scale_log2, -ms)) : 0.f;
              const float p1 = key + 1 < g.N ? ex2(fmaf(v[2 * e + 1], g.scale_log2, -ms)) : 0.f;
              l += p0 + p1;
              pk[e] = pack_bf16x2(p0, p1);
            }
            tmem_st8(sb, pk);          // P over this warp's own, already-read S columns
            tmem_st8(sb + 8, pk + 8);
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&bar_p[u & 1]);
        }
        red_sum[cq][rloc] = l;
        named_bar(1 + q, 128);
        const float lt = (red_sum[0][rloc] + red_sum[1][rloc]) + (red_sum[2][rloc] + red_sum[3][rloc]);
        // ---- epilogue: O / l (HP / 4 of the head columns per warp, those < hd stored), LSE
        mbar_wait(bar_o, tt & 1);
        tc_fence_after();
        constexpr int kQ = HP / 4;
        float o[kQ];
        if (active) {
          if constexpr (kQ == 16)
            tmem_ld16(ocol + lq + static_cast<uint32_t>(cq * kQ), o);
          else
            tmem_ld32(ocol + lq + static_cast<uint32_t>(cq * kQ), o);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(bar_e);
        const int row = tile * 128 + rloc;
        if (row < g.N) {
          const float inv = 1.0f / lt;
          uint4* dst = reinterpret_cast<uint4*>(
              out + (static_cast<int64_t>(b) * g.N + row) * g.ld_o + h * hd + cq * kQ);
#pragma unroll
          for (int j = 0; j < kQ / 8; ++j)
            if (cq * kQ + 8 * j < hd)
              dst[j] = make_uint4(pack_bf16x2(o[8 * j] * inv, o[8 * j + 1] * inv),
                                  pack_bf16x2(o[8 * j + 2] * inv, o[8 * j + 3] * inv),
                                  pack_bf16x2(o[8 * j + 4] * inv, o[8 * j + 5] * inv),
                                  pack_bf16x2(o[8 * j + 6] * inv, o[8 * j + 7] * inv));
          if (cq == 0) lse[(static_cast<int64_t>(b) * g.H + h) * g.N + row] = ms + log2f(lt);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 16) tmem_dealloc(tmem, 512);
}

}  // namespace attn_tc
}  // namespace rp

using namespace rp;

// Returns RP_ERR_CONFIG (without launching) when the shape is outside the tcgen05 path;
// the caller then uses the mma.sync kernel.
int rp_attention_fwd_tc(const uint16_t* qkv, int64_t S, int64_t N, int64_t H, uint16_t* out,
                        float* lse, cudaStream_t stream) {
  using namespace attn_tc;
  if (N > 512 || N < 1) return RP_ERR_CONFIG;
  Geom g;
  g.B = static_cast<int>(S);
  g.N = static_cast<int>(N);
  g.H = static_cast<int>(H);
  g.Nk = static_cast<int>((N + 15) / 16 * 16);
  g.ld_o = H * 64;
  g.scale_log2 = (1.0f / 8.0f) * 1.4426950408889634f;
  const int64_t T = S * N, cols = 3 * H * 64;
  CUtensorMap mq, mkv;
  if (g.Nk > 256 || (g.Nk > 224 && rp_attn_fwd_variant() != 0)) {
    // two-pass kernel with K / V resident per (sequence, head) group
    LongMaps lm;
    std::memset(&lm, 0, sizeof(lm));
    if (make_map(&lm.lo, qkv, T, cols, 128))
      return rp_fail(RP_ERR_CUDA, "attention_tc: tensor map encode failed");
    const int smem = 1024 + LongCfg<64>::kSmem;
    static std::once_flag once_l;
    static int nsm_l = 148;
    std::call_once(once_l, [smem] {
      cudaFuncSetAttribute(attn_fwd_tc_long<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&nsm_l, cudaDevAttrMultiProcessorCount, dev);
    });
    LongPlan pl;
    pl.ntile = static_cast<int>((N + 127) / 128);
    // all of a sequence's query tiles per item (K, V loaded once), except at N = 512 with
    // too few (sequence, head) pairs to balance 148 SMs, where pairs of tiles do better
    // (measured, tools/attn_fwd_ab.py: 64 x 512 x 12 heads 234 us vs 243 us; 256 x 512:
    // 819 vs 873 us; 64 x 300: 132 vs 163 us)
    pl.group = (pl.ntile == 4 && S * H < 8 * nsm_l) ? 2 : pl.ntile;
    pl.ngroup = (pl.ntile + pl.group - 1) / pl.group;
    pl.nitems = static_cast<int>(S * H) * pl.ngroup;
    pl.nkb = static_cast<int>((N + 127) / 128);
    pl.hd = 64;
    const unsigned grid = static_cast<unsigned>(pl.nitems < nsm_l ? pl.nitems : nsm_l);
    launch_k(attn_fwd_tc_long<64>, dim3(grid), dim3(kFwdThreads), smem, stream, lm,
             reinterpret_cast<__nv_bfloat16*>(out), lse, g, pl);
    return rp_check_launch("attention_fwd_tc_long");
  }
  if (make_map(&mq, qkv, T, cols, 128) || make_map(&mkv, qkv, T, cols, static_cast<uint32_t>(g.Nk)))
    return rp_fail(RP_ERR_CUDA, "attention_tc: tensor map encode failed");
  const int smem = 1024 + 2 * kFwdBuf;
  const int smem_pp = smem;
  // ping-pong softmax groups by default (256 x 197 x 12: 113.4 vs 113.5 us; x 16 heads:
  // 134.3 vs 144.7; 64 x 128: 19.0 vs 21.0), except 208 < Nk <= 224 where the lockstep
  // kernel measured faster (128 x 224: 64.5 vs 70.1 us) (tools/attn_fwd_ab.py)
  const bool pp = g.Nk > 224 || (rp_attn_fwd_variant() != 1 && g.Nk <= 208);
  if (pp) {
    static std::once_flag once_pp;
    static int nsm_pp = 148;
    std::call_once(once_pp, [smem_pp] {
      cudaFuncSetAttribute(attn_fwd_tc_pp, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_pp);
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&nsm_pp, cudaDevAttrMultiProcessorCount, dev);
    });
    PPPlan pp;
    pp.ntile = static_cast<int>((N + 127) / 128);
    pp.nitems = static_cast<int>(S * H);
    const int nch = g.Nk / 16;
    pp.cs = (nch + 1) / 2;
    pp.p1 = 256 - 8 * (nch - pp.cs);
    const int oa = (8 * pp.cs + 31) / 32 * 32;
    // split P V: half 1's P in the tail [p1, 256) beyond every S column, O_a | O_b in the
    // columns dead once both halves are packed (Nk <= 208 at 256 columns per S buffer)
    pp.split = rp_attn_fwd_variant() == 0 && nch >= 2 && pp.p1 >= g.Nk && oa + 128 <= pp.p1;
    pp.ocol = pp.split ? oa : (8 * (nch + pp.cs) + 15) / 16 * 16;
    pp.trace = rp_attn_trace_buffer();
    const unsigned grid = static_cast<unsigned>(pp.nitems < nsm_pp ? pp.nitems : nsm_pp);
    launch_k(attn_fwd_tc_pp, dim3(grid), dim3(kPPThreads), smem_pp, stream, mq, mkv,
             reinterpret_cast<__nv_bfloat16*>(out), lse, g, pp);
    return rp_check_launch("attention_fwd_tc_pp");
  }
  if (g.Nk > 224) return RP_ERR_CONFIG;  // the lockstep kernel's TMEM plan stops at 224
  static std::once_flag once;
  static int nsm = 148;
  std::call_once(once, [smem] {
    cudaFuncSetAttribute(attn_fwd_tc_persistent, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         smem);
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  });
  FwdPlan pl;
  pl.ntile = static_cast<int>((N + 127) / 128);
  pl.nitems = static_cast<int>(S * H);
  pl.o_sep = 2 * g.Nk + 64 <= 512;
  pl.sb = pl.o_sep ? g.Nk : 256;
  pl.ocol = pl.o_sep ? 448 : 192;
  const unsigned grid = static_cast<unsigned>(pl.nitems < nsm ? pl.nitems : nsm);
  launch_k(attn_fwd_tc_persistent, dim3(grid), dim3(kFwdThreads), smem, stream, mq, mkv,
           reinterpret_cast<__nv_bfloat16*>(out), lse, g, pl);
  return rp_check_launch("attention_fwd_tc");
}

// tcgen05 forward for head dims 72..128 (multiples of 8; G48's 104) at N <= 256: the
// two-pass kernel with K / V resident per item, operands as two 64-column atom planes.
// RP_ERR_CONFIG without launching outside that range.
int rp_attention_fwd_tc_wide(const uint16_t* qkv, int64_t S, int64_t N, int64_t H, int64_t hd,
                             uint16_t* out, float* lse, cudaStream_t stream) {
  using namespace attn_tc;
  if (N > 256 || N < 1 || hd <= 64 || hd > 128 || hd % 8) return RP_ERR_CONFIG;
  Geom g;
  g.B = static_cast<int>(S);
  g.N = static_cast<int>(N);
  g.H = static_cast<int>(H);
  g.Nk = static_cast<int>((N + 15) / 16 * 16);
  g.ld_o = H * hd;
  g.scale_log2 = (1.0f / sqrtf(static_cast<float>(hd))) * 1.4426950408889634f;
  const int64_t T = S * N, cols = 3 * H * hd;
  LongMaps lm;
  if (make_map(&lm.lo, qkv, T, cols, 128) ||
      make_map(&lm.hi, qkv, T, cols, 128, static_cast<uint32_t>(hd - 64)))
    return rp_fail(RP_ERR_CUDA, "attention_tc_wide: tensor map encode failed");
  const int smem = 1024 + LongCfg<128>::kSmem;
  static std::once_flag once;
  static int nsm = 148;
  std::call_once(once, [smem] {
    cudaFuncSetAttribute(attn_fwd_tc_long<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  });
  LongPlan pl;
  pl.ntile = static_cast<int>((N + 127) / 128);
  pl.group = pl.ntile;
  pl.ngroup = 1;
  pl.nitems = static_cast<int>(S * H);
  pl.nkb = static_cast<int>((N + 127) / 128);
  pl.hd = static_cast<int>(hd);
  const unsigned grid = static_cast<unsigned>(pl.nitems < nsm ? pl.nitems : nsm);
  launch_k(attn_fwd_tc_long<128>, dim3(grid), dim3(kFwdThreads), smem, stream, lm,
           reinterpret_cast<__nv_bfloat16*>(out), lse, g, pl);
  return rp_check_launch("attention_fwd_tc_wide");
}

