// Single-pass tcgen05 attention backward for head_dim 64, N <= 208 (the ViT shapes).
//
// ref:proj/core/src/layers.cpp:185-208 (per head: dA = dO V^T, dV = A^T dO,
// dS = softmax_vjp(A, dA) / sqrt(hd), dQ = dS K, dK = dS^T Q; softmax VJP ops.cpp:206-225),
// with the probabilities recomputed from the forward's log2-domain LSE and D = rowsum(dO * O)
// taken from the d_att GEMM's RP_EPI_ROWDOT epilogue (or attn_d_kernel).
//
// One persistent CTA per SM; an item is (sequence, head, 128-key tile kt), the key tiles of a
// (sequence, head) pair are consecutive items of the same CTA, so the pair's Q and dO are
// loaded once. Per item, in TMEM (lanes = the tile's 128 keys, 512 columns):
//   MMA1   S^T  = K_kt Q^T   -> [0, Nk)          N = Nk (all queries in one instruction per
//          dP^T = V_kt dO^T  -> [256, 256 + Nk)  K-step; two issuing warps, one product each)
//   EW     16 warps (TMEM lane quarter w%4, 16-query chunks c = w/4 mod 4) read S^T, dP^T:
//            P^T  = exp2(S^T scale log2e - lse_q)          bf16, packed into [0, 128)
//                                                          (p_col; A operand of dV)
//            dS^T = P^T (dP^T - D_q) scale                 bf16, to shared memory, 8-key x
//                                                          64-query SW128 atoms: the K-major
//                                                          A of dK and the MN-major A of dQ
//   MMA2   dV  = P^T dO        (A TMEM, p_col)   -> [128, 192)   warp 17
//          dK  = dS^T Q        (A smem K-major)  -> [224, 288)   warp 18
//          dQ0 = dS[q<128] K_kt (A smem MN-major)-> [288, 352)   warp 19
//          dQ1 = dS[q>=128] K_kt                 -> [352, 416)   warp 16 (Nk > 128)
//          (over consumed S^T / dP^T columns; P^T, the A of dV, stays in [0, 128))
//          four issuing warps on four SM sub-partitions: every product has N = 64, and one
//          thread issues at most one such MMA per ~120 cycles (tools/umma2sm_bench.cu)
//   EPI    the same 16 warps drain dV, dK and dQ into bf16 SW128 staging tiles (the dS^T
//          region, consumed by then) that warp 19 writes out with bulk tensor stores. The first
//          key tile's dQ partials wait for the second: dQ0 parked in TMEM columns the pair's
//          later MMAs never touch, dQ1 (fp32) in a per-CTA scratch slot (L2-resident); the
//          last key tile adds them (fixed order partial_0 + partial_1: deterministic).
// No dS leaves the SM (the previous path wrote dS^T, 2 N^2 bytes per head, and read it back
// in a second kernel). Each output element is written by one thread of one CTA.
#include "attn_common.cuh"
#include "launch.h"

namespace rp {
namespace attn_fb {
using namespace attn_tc;

__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, uint32_t src, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(c0), "r"(c1), "r"(c2), "r"(src)
      : "memory");
}

__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, uint32_t src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1), "r"(src)
               : "memory");
}

// fp32 [rows][64] scratch: boxes of 32 columns x 128 rows, SWIZZLE_128B
inline int make_map_scratch(CUtensorMap* m, const float* base, int64_t rows) {
  EncodeFn fn = encode_fn();
  if (!fn) return RP_ERR_CUDA;
  cuuint64_t dims[2] = {64, static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {256};
  cuuint32_t box[2] = {32, 128};
  cuuint32_t es[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS
             ? RP_OK
             : RP_ERR_CUDA;
}

// bf16 [S][N][cols] view of a [S N][ld] row-major matrix: boxes of 64 columns x 128 rows,
// SWIZZLE_128B; rows past N (the next sequence) are out of bounds, so stores clip there
inline int make_map_seq(CUtensorMap* m, const void* base, int64_t S, int64_t N, int64_t cols,
                        int64_t ld) {
  EncodeFn fn = encode_fn();
  if (!fn) return RP_ERR_CUDA;
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(N),
                        static_cast<cuuint64_t>(S)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(ld) * 2, static_cast<cuuint64_t>(N * ld) * 2};
  cuuint32_t box[3] = {64, 128, 1};
  cuuint32_t es[3] = {1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS
             ? RP_OK
             : RP_ERR_CUDA;
}

constexpr int kEwWarps = 16;

// TMEM column of the packed bf16 P^T of 16-query chunk c (8 columns). Warp cg converts
// chunks cg, cg + 4, cg + 8, cg + 12 in that order and packs them into the S^T columns of
// its own first two chunks (cg and cg + 4), which it has already read: race-free, and P^T
// occupies only [0, 128), leaving [128, 256) whole for accumulators.
__device__ __forceinline__ uint32_t p_col(int c) {
  return static_cast<uint32_t>(16 * (c & 3) + 64 * (c >> 3) + 8 * ((c >> 2) & 1));
}
constexpr int kFbThreads = (kEwWarps + 4) * 32;  // + TMA/dQ1, S^T/dV, dP^T/dK, dQ0
constexpr int kMaxNk = 208;

struct FbGeom {
  int B, N, H, Nk, ntile, npairs;
  int qd_bytes;   // one of Q / dO for a pair: Nk rows x 128 B
  int ds_bytes;   // dS^T staging: 2 * ntile chunks of 128 keys x 64 queries
  int64_t ld_qkv, ld_o;
  float scale, scale_log2;
  unsigned long long* trace;  // optional clock64 trace of CTA 0's first kFbTrace items
};
constexpr int kFbTrace = 32;
#define FB_TRACE(i, slot)                                                                  \
  do {                                                                                     \
    if (g.trace && blockIdx.x == 0 && (i) < kFbTrace && lane == 0)                         \
      g.trace[(i) * 24 + (slot)] = static_cast<unsigned long long>(clock64());             \
  } while (0)

// smem layout (from the 1024-aligned base): QD[2] = (Q | dO) per pair buffer, K[2], V, DS
__host__ __device__ inline int fb_off_k(const FbGeom& g) { return 4 * g.qd_bytes; }
__host__ __device__ inline int fb_off_v(const FbGeom& g) { return 4 * g.qd_bytes + 32768; }
__host__ __device__ inline int fb_off_ds(const FbGeom& g) { return 4 * g.qd_bytes + 49152; }
__host__ __device__ inline int fb_smem(const FbGeom& g) { return fb_off_ds(g) + g.ds_bytes + 1024; }

__global__ void __launch_bounds__(kFbThreads, 1)
    attn_bwd_fused_tc(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                      const __grid_constant__ CUtensorMap tm_do,
                      const __grid_constant__ CUtensorMap tm_dqkv,
                      const __grid_constant__ CUtensorMap tm_scr, const float* __restrict__ lse,
                      const float* __restrict__ Dg, float* __restrict__ dq_scratch, FbGeom g) {
  pdl_trigger();

  __shared__ __align__(16) float sL[2][kMaxNk];  // -lse (log2 domain) per query, -inf past N
  __shared__ __align__(16) float sD[2][kMaxNk];  // -D * scale per query, 0 past N (per pair)
  __shared__ __align__(8) uint64_t bars[16];
  __shared__ uint32_t tmem_slot;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint64_t* qd_full = bars;      // [2] Q | dO of a pair landed
  uint64_t* k_full = bars + 2;   // [2] K of an item landed
  uint64_t* v_full = bars + 4;   //     V of an item landed
  uint64_t* bar_s = bars + 5;    //     S^T and dP^T in TMEM (2 issuers)
  uint64_t* bar_ew = bars + 6;   //     P^T in TMEM, dS^T in smem (16 warps)
  uint64_t* bar_m2 = bars + 7;   //     dV, dK, dQ accumulated (3 or 4 issuers)
  uint64_t* bar_epi = bars + 8;  //     accumulators drained, TMEM free (16 warps)
  uint64_t* bar_stg = bars + 9;  //     outputs staged in the dS^T region (16 warps)
  uint64_t* bar_scr = bars + 10;    //  a first key tile's dQ1 partial is in global memory
  uint64_t* bar_sfree = bars + 11;  // [4] staging tile t (= dS^T 64-query chunk t) read out

  const uint32_t warp = warp_id(), lane = lane_id();
  const int Nk = g.Nk, nch = Nk / 16, ntile = g.ntile;
  const int ngrp = (nch + 3) / 4;  // 64-query dS^T chunks = staging tiles released per item
  const bool two = Nk > 128;
  if (warp == 16) {
    if (lane == 0) {
      tma_prefetch_desc(&tm_q);
      tma_prefetch_desc(&tm_k);
      tma_prefetch_desc(&tm_do);
      tma_prefetch_desc(&tm_dqkv);
      tma_prefetch_desc(&tm_scr);
      for (int i = 0; i < 2; ++i) {
        mbar_init(&qd_full[i], 1);
        mbar_init(&k_full[i], 1);
      }
      mbar_init(v_full, 1);
      mbar_init(bar_s, 2);
      mbar_init(bar_ew, kEwWarps);
      mbar_init(bar_m2, two ? 4 : 3);
      mbar_init(bar_epi, kEwWarps);
      mbar_init(bar_stg, kEwWarps);
      for (int t = 0; t < 4; ++t) mbar_init(&bar_sfree[t], 1);
      mbar_init(bar_scr, 1);
      fence_barrier_init();
    }
    tmem_alloc(&tmem_slot, 512);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;
  pdl_wait();

  const int cta = static_cast<int>(blockIdx.x), ncta = static_cast<int>(gridDim.x);
  const int npc = g.npairs > cta ? (g.npairs - cta + ncta - 1) / ncta : 0;  // pairs of this CTA
  const int nI = npc * ntile;
  const int d = g.H * 64;
  const uint32_t sbase = smem_u32(smem);
  const uint32_t s_k = sbase + static_cast<uint32_t>(fb_off_k(g));
  const uint32_t s_v = sbase + static_cast<uint32_t>(fb_off_v(g));
  const uint32_t s_ds = sbase + static_cast<uint32_t>(fb_off_ds(g));
  auto s_q = [&](int j) { return sbase + static_cast<uint32_t>((j & 1) * 2 * g.qd_bytes); };
  auto s_do = [&](int j) { return s_q(j) + static_cast<uint32_t>(g.qd_bytes); };
  auto pair_of = [&](int j) { return cta + j * ncta; };
  const uint32_t is0 = lane == 0 ? 1u : 0u;
  // dQ K-steps of key tile kt: its keys below Nk, in 16-key steps
  auto dq_steps = [&](int kt) { return min(8, (Nk - kt * 128 + 15) / 16); };

  if (warp >= kEwWarps) {
    const int role = static_cast<int>(warp) - kEwWarps;  // 0 TMA + dQ1, 1 S^T + dV, 2 dP^T + dK, 3 dQ0
    const uint32_t idesc_s = make_idesc_bf16(128, static_cast<uint32_t>(Nk), false, false);
    const uint32_t idesc_kv = make_idesc_bf16(128, 64, false, true);   // dV (TS), dK (SS)
    const uint32_t idesc_q = make_idesc_bf16(128, 64, true, true);     // dQ (A MN-major)
    if (role == 0) {
      auto load_qd = [&](int j) {
        const int p = pair_of(j);
        const int row = (p / g.H) * g.N, h = p % g.H;
        if (lane == 0) {
          mbar_arrive_expect_tx(&qd_full[j & 1], 2u * static_cast<uint32_t>(g.qd_bytes));
          tma_load_2d(smem + (j & 1) * 2 * g.qd_bytes, &tm_q, &qd_full[j & 1], h * 64, row);
          tma_load_2d(smem + (j & 1) * 2 * g.qd_bytes + g.qd_bytes, &tm_do, &qd_full[j & 1], h * 64,
                      row);
        }
      };
      auto load_kv = [&](int i) {
        const int j = i / ntile, kt = i % ntile, p = pair_of(j);
        const int row = (p / g.H) * g.N + kt * 128, h = p % g.H;
        if (lane == 0) {
          mbar_arrive_expect_tx(&k_full[i & 1], 16384u);
          tma_load_2d(smem + fb_off_k(g) + (i & 1) * 16384, &tm_k, &k_full[i & 1], d + h * 64, row);
          mbar_arrive_expect_tx(v_full, 16384u);
          tma_load_2d(smem + fb_off_v(g), &tm_k, v_full, 2 * d + h * 64, row);
        }
      };
      if (nI > 0) {
        load_qd(0);
        load_kv(0);
      }
      for (int i = 0; i < nI; ++i) {
        const int j = i / ntile, kt = i % ntile;
        mbar_wait(bar_s, static_cast<uint32_t>(i & 1));  // MMA1(i) done: V and K[(i+1)&1] free
        FB_TRACE(i, 14);
        if (kt == 0 && j + 1 < npc) load_qd(j + 1);       // one pair ahead
        if (i + 1 < nI) load_kv(i + 1);
        FB_TRACE(i, 15);
        __syncwarp();
        if (two) {  // dQ1 = dS[q >= 128] K_kt
          mbar_wait(bar_ew, static_cast<uint32_t>(i & 1));
          tc_fence_after();
          const uint32_t kb = s_k + static_cast<uint32_t>((i & 1) * 16384);
          const int ns = dq_steps(kt);
          for (int ks = 0; ks < ns; ++ks)
            umma_bf16_pred(tmem + 352u,
                           make_sdesc_sw128(s_ds + 2u * 16384u + static_cast<uint32_t>(ks) * 2048u, 16384, 1024),
                           make_sdesc_sw128(kb + static_cast<uint32_t>(ks) * 2048u, 8192, 1024), idesc_q,
                           ks > 0 ? 1u : 0u, is0);
          umma_commit_pred(bar_m2, is0);
          FB_TRACE(i, 10);
          __syncwarp();
        }
      }
    } else if (role == 1 || role == 2) {
      for (int i = 0; i < nI; ++i) {
        const int j = i / ntile;
        if (role == 1) FB_TRACE(i, 0);
        if (i > 0) mbar_wait(bar_epi, static_cast<uint32_t>((i - 1) & 1));  // TMEM drained
        mbar_wait(&qd_full[j & 1], static_cast<uint32_t>((j >> 1) & 1));
        if (role == 1)
          mbar_wait(&k_full[i & 1], static_cast<uint32_t>((i >> 1) & 1));
        else
          mbar_wait(v_full, static_cast<uint32_t>(i & 1));
        tc_fence_after();
        if (role == 1) FB_TRACE(i, 1);
        // MMA1: S^T = K Q^T (role 1) or dP^T = V dO^T (role 2), K = 64 in four steps
        const uint32_t a = role == 1 ? s_k + static_cast<uint32_t>((i & 1) * 16384) : s_v;
        const uint32_t b = role == 1 ? s_q(j) : s_do(j);
        const uint32_t dcol = role == 1 ? 0u : 256u;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          umma_bf16_pred(tmem + dcol, make_sdesc_sw128(a + kk * 32, 16, 1024),
                         make_sdesc_sw128(b + kk * 32, 16, 1024), idesc_s, kk > 0 ? 1u : 0u, is0);
        umma_commit_pred(bar_s, is0);
        if (role == 1) FB_TRACE(i, 2);
        __syncwarp();
        // MMA2 once the elementwise warps have published P^T / dS^T
        mbar_wait(bar_ew, static_cast<uint32_t>(i & 1));
        tc_fence_after();
        if (role == 1) FB_TRACE(i, 6);
        if (role == 1) {  // dV += P^T dO   (A = P^T from TMEM, chunk c packed at column 16c)
          const uint32_t bo = s_do(j);
          for (int c = 0; c < nch; ++c)
            umma_ts_bf16_pred(tmem + 128u, tmem + p_col(c),
                              make_sdesc_sw128(bo + static_cast<uint32_t>(c) * 2048u, 8192, 1024),
                              idesc_kv, c > 0 ? 1u : 0u, is0);
        } else {  // dK += dS^T Q   (A = dS^T from smem, K-major)
          const uint32_t bq = s_q(j);
          for (int c = 0; c < nch; ++c)
            umma_bf16_pred(tmem + 224u,
                           make_sdesc_sw128(s_ds + static_cast<uint32_t>(c >> 2) * 16384u +
                                                static_cast<uint32_t>(c & 3) * 32u,
                                            16, 1024),
                           make_sdesc_sw128(bq + static_cast<uint32_t>(c) * 2048u, 8192, 1024),
                           idesc_kv, c > 0 ? 1u : 0u, is0);
        }
        umma_commit_pred(bar_m2, is0);
        FB_TRACE(i, role == 1 ? 7 : 8);
        __syncwarp();
      }
    } else {  // role 3: dQ0 = dS[q < 128] K_kt
      for (int i = 0; i < nI; ++i) {
        const int kt = i % ntile;
        mbar_wait(bar_ew, static_cast<uint32_t>(i & 1));
        tc_fence_after();
        const uint32_t kb = s_k + static_cast<uint32_t>((i & 1) * 16384);
        const int ns = dq_steps(kt);
        for (int ks = 0; ks < ns; ++ks)
          umma_bf16_pred(tmem + 288u,
                         make_sdesc_sw128(s_ds + static_cast<uint32_t>(ks) * 2048u, 16384, 1024),
                         make_sdesc_sw128(kb + static_cast<uint32_t>(ks) * 2048u, 8192, 1024), idesc_q,
                         ks > 0 ? 1u : 0u, is0);
        umma_commit_pred(bar_m2, is0);
        FB_TRACE(i, 9);
        __syncwarp();
        // the epilogue's bulk stores: bf16 dV, dK (and dQ on the last key tile) into d_qkv,
        // rows past N clipped by the [S][N][cols] map; the first key tile's dQ1 partial (fp32,
        // two 32-column halves) into this CTA's scratch slot
        const int j = i / ntile, p = pair_of(j), b = p / g.H, h = p % g.H;
        mbar_wait(bar_stg, static_cast<uint32_t>(i & 1));
        if (lane == 0) {
          // one bulk group per staging tile, released one by one: the next item's dS^T
          // writes (64-query chunk t = staging tile t, in order) wait only for their tile
          tma_store_3d(&tm_dqkv, s_ds, 2 * d + h * 64, kt * 128, b);
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          tma_store_3d(&tm_dqkv, s_ds + 16384u, d + h * 64, kt * 128, b);
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          if (kt == ntile - 1) {
            tma_store_3d(&tm_dqkv, s_ds + 32768u, h * 64, 0, b);
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            if (two) tma_store_3d(&tm_dqkv, s_ds + 49152u, h * 64, 128, b);
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          } else {
            tma_store_2d(&tm_scr, s_ds + 32768u, 0, cta * 128);
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            tma_store_2d(&tm_scr, s_ds + 49152u, 32, cta * 128);
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
          // (only the tiles some 64-query chunk of dS^T will rewrite are released: every
          // arrival has a waiter)
          asm volatile("cp.async.bulk.wait_group.read 3;" ::: "memory");
          mbar_arrive(&bar_sfree[0]);
          asm volatile("cp.async.bulk.wait_group.read 2;" ::: "memory");
          if (ngrp > 1) mbar_arrive(&bar_sfree[1]);
          asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
          if (ngrp > 2) mbar_arrive(&bar_sfree[2]);
          asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          if (ngrp > 3) mbar_arrive(&bar_sfree[3]);
          if (kt != ntile - 1) {  // the partial must be in global memory before it is read
            asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
            asm volatile("fence.proxy.async.global;" ::: "memory");
            mbar_arrive(bar_scr);
          }
        }
        __syncwarp();
      }
      if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
  } else {
    // ------------------------------------------------ elementwise + epilogue warps
    const int q = static_cast<int>(warp & 3u), cg = static_cast<int>(warp >> 2);
    const uint32_t lq = (static_cast<uint32_t>(q) * 32u) << 16;
    const int kl = q * 32 + static_cast<int>(lane);  // key (lane) within the tile
    // dS^T smem row of this lane's key: chunk stride 16 KB, 8-key group kl/8, row kl%8
    const uint32_t ds_row = s_ds + static_cast<uint32_t>(kl >> 3) * 1024u +
                            static_cast<uint32_t>(kl & 7) * 128u;
    const uint32_t sw = static_cast<uint32_t>(kl & 7);
    // output staging (reuses the dS^T region once MMA2 has consumed it): four 128-row x 64-
    // column bf16 tiles (dV, dK, dQ0, dQ1) in the SW128 layout, one bulk tensor store each;
    // this warp writes rows kl, 16-byte units 2 cg, 2 cg + 1
    const uint32_t srow = s_ds + static_cast<uint32_t>(kl) * 128u;
    const uint32_t su0 = ((2u * static_cast<uint32_t>(cg)) ^ sw) << 4;
    const uint32_t su1 = ((2u * static_cast<uint32_t>(cg) + 1u) ^ sw) << 4;
    // dQ partials of the first key tile: dQ0 parked in TMEM columns no later MMA of the pair
    // writes ([208, 224) and [464, 512): S^T / dP^T use [0, Nk) and [256, 256 + Nk), Nk <=
    // 208; the accumulators avoid them), this warp's 16 columns at `park`; dQ1 through the
    // CTA's fp32 scratch slot
    // [128 rows][64] (bulk store from staging, read back row-wise)
    const uint32_t park = cg < 3 ? 464u + 16u * static_cast<uint32_t>(cg) : 208u;
    const float4* scr_row = reinterpret_cast<const float4*>(dq_scratch + (static_cast<int64_t>(cta) * 128 + kl) * 64) +
                            4 * cg;
    auto load_lse = [&](int j, int buf) {  // the pair's -lse and -D * scale, per query
      const int p = pair_of(j);
      const int64_t hb = (static_cast<int64_t>(p / g.H) * g.H + p % g.H) * g.N;
      for (int t = static_cast<int>(threadIdx.x); t < Nk; t += kEwWarps * 32) {
        sL[buf][t] = t < g.N ? -lse[hb + t] : -INFINITY;
        sD[buf][t] = t < g.N ? -Dg[hb + t] * g.scale : 0.f;
      }
    };
    // fp32 staging of the dQ1 partial: two 128-row x 32-column SW128 tiles at 32 / 48 KB
    auto stage16f = [&](const float* v) {
      const uint32_t base = s_ds + 32768u + static_cast<uint32_t>(cg >> 1) * 16384u +
                            static_cast<uint32_t>(kl) * 128u;
#pragma unroll
      for (int u = 0; u < 4; ++u)
        sts128_a(base + (((static_cast<uint32_t>((cg & 1) * 4 + u)) ^ sw) << 4),
                 make_uint4(__float_as_uint(v[4 * u]), __float_as_uint(v[4 * u + 1]),
                            __float_as_uint(v[4 * u + 2]), __float_as_uint(v[4 * u + 3])));
    };
    auto stage16 = [&](uint32_t tile, const float* v) {
      const uint32_t base = srow + tile * 16384u;
      sts128_a(base + su0, make_uint4(pack_bf16x2(v[0], v[1]), pack_bf16x2(v[2], v[3]),
                                      pack_bf16x2(v[4], v[5]), pack_bf16x2(v[6], v[7])));
      sts128_a(base + su1, make_uint4(pack_bf16x2(v[8], v[9]), pack_bf16x2(v[10], v[11]),
                                      pack_bf16x2(v[12], v[13]), pack_bf16x2(v[14], v[15])));
    };
    if (nI > 0) load_lse(0, 0);
    for (int i = 0; i < nI; ++i) {
      const int j = i / ntile, kt = i % ntile, p = pair_of(j);
      const int b = p / g.H, h = p % g.H;
      const bool last = kt == ntile - 1;
      const float* L = sL[j & 1];
      const float* Dd = sD[j & 1];
      if (kt == 0) named_bar(1, kEwWarps * 32);  // the pair's sL / sD complete
      const bool kvalid = kt * 128 + kl < g.N;
      mbar_wait(bar_s, static_cast<uint32_t>(i & 1));
      tc_fence_after();
      if (warp == 0) FB_TRACE(i, 3);
      if (warp == 0) FB_TRACE(i, 20);
      for (int c = cg; c < nch; c += 4) {
        float s[16], dp[16];
        tmem_ld16x2(tmem + lq + static_cast<uint32_t>(16 * c), tmem + lq + 256u + static_cast<uint32_t>(16 * c),
                    s, dp);
        const float4* l4 = reinterpret_cast<const float4*>(L + 16 * c);
        const float4* d4 = reinterpret_cast<const float4*>(Dd + 16 * c);
        uint32_t pp[8], pd[8];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const float4 nl = l4[u], nd = d4[u];
          const float la[4] = {nl.x, nl.y, nl.z, nl.w}, da[4] = {nd.x, nd.y, nd.z, nd.w};
#pragma unroll
          for (int t = 0; t < 2; ++t) {
            const int e = 4 * u + 2 * t;
            float p0 = ex2(fmaf(s[e], g.scale_log2, la[2 * t]));
            float p1 = ex2(fmaf(s[e + 1], g.scale_log2, la[2 * t + 1]));
            float d0 = p0 * fmaf(dp[e], g.scale, da[2 * t]);
            float d1 = p1 * fmaf(dp[e + 1], g.scale, da[2 * t + 1]);
            if (!kvalid) p0 = p1 = d0 = d1 = 0.f;
            pp[2 * u + t] = pack_bf16x2(p0, p1);
            pd[2 * u + t] = pack_bf16x2(d0, d1);
          }
        }
        tmem_st8(tmem + lq + p_col(c), pp);  // over S^T columns this warp has read
        // dS^T (16 queries = two 16-byte units of the 64-query chunk c/4) into the atom row,
        // once item i-1's output store has read that staging tile
        if (i > 0) mbar_wait(&bar_sfree[c >> 2], static_cast<uint32_t>((i - 1) & 1));
        const uint32_t row = ds_row + static_cast<uint32_t>(c >> 2) * 16384u;
        const uint32_t u0 = static_cast<uint32_t>((c & 3) * 2);
        sts128_a(row + ((u0 ^ sw) << 4), make_uint4(pd[0], pd[1], pd[2], pd[3]));
        sts128_a(row + (((u0 + 1) ^ sw) << 4), make_uint4(pd[4], pd[5], pd[6], pd[7]));
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      fence_proxy_async_smem();  // dS^T is read by the tensor core (async proxy)
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar_ew);
      if (warp == 0) FB_TRACE(i, 4);
      if (warp == 15) FB_TRACE(i, 5);
      // under MMA2: the next pair's -lse / -D, and the first key tile's dQ partial
      if (last && j + 1 < npc) load_lse(j + 1, (j + 1) & 1);
      float4 part[4];  // the dQ1 partial of this pair's first key tile (rows 128 + kl)
      const bool add_part = ntile == 2 && kt == 1;
      if (add_part) {  // written by the bulk store (async proxy): L1-bypassing loads
        mbar_wait(bar_scr, static_cast<uint32_t>(j & 1));
#pragma unroll
        for (int e = 0; e < 4; ++e)
          part[e] = 128 + kl < Nk ? __ldcg(scr_row + e) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
      // ---- epilogue: 16 columns of each accumulator per warp
      mbar_wait(bar_m2, static_cast<uint32_t>(i & 1));
      tc_fence_after();
      if (warp == 0) FB_TRACE(i, 11);
      {
        float v[16], k[16];
        tmem_ld16x2(tmem + lq + 128u + static_cast<uint32_t>(16 * cg),
                    tmem + lq + 224u + static_cast<uint32_t>(16 * cg), v, k);
        stage16(0, v);
        stage16(1, k);
      }
      float q0[16], q1[16];
      tmem_ld16x2(tmem + lq + 288u + static_cast<uint32_t>(16 * cg),
                  tmem + lq + 352u + static_cast<uint32_t>(16 * cg), q0, q1);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar_epi);
      if (warp == 0) FB_TRACE(i, 12);
      if (warp == 0) FB_TRACE(i, 16);
      if (ntile == 2 && kt == 0) {  // first key tile: park dQ0, stage the fp32 dQ1 partial
        uint32_t pq[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) pq[e] = __float_as_uint(q0[e]);
        tmem_st16(tmem + lq + park, pq);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        stage16f(q1);
      } else {
        if (add_part) {  // partial_0 + partial_1, in this order
          float p0[16];
          tmem_ld16(tmem + lq + park, p0);
#pragma unroll
          for (int e = 0; e < 16; ++e) q0[e] = p0[e] + q0[e];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            q1[4 * e] = part[e].x + q1[4 * e];
            q1[4 * e + 1] = part[e].y + q1[4 * e + 1];
            q1[4 * e + 2] = part[e].z + q1[4 * e + 2];
            q1[4 * e + 3] = part[e].w + q1[4 * e + 3];
          }
        }
        stage16(2, q0);
        stage16(3, q1);
      }
      if (warp == 0) FB_TRACE(i, 17);
      fence_proxy_async_smem();  // staged tiles are read by the bulk stores (async proxy)
      __syncwarp();
      if (lane == 0) mbar_arrive(bar_stg);
      if (warp == 0) FB_TRACE(i, 18);
      if (warp == 0) FB_TRACE(i, 13);
    }
    // observe the last item's staging releases too (every arrival gets a wait; the stores
    // have read their tiles before the CTA's shared memory goes away)
    if (nI > 0)
      for (int t = 0; t < ngrp; ++t) mbar_wait(&bar_sfree[t], static_cast<uint32_t>((nI - 1) & 1));
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 16) tmem_dealloc(tmem, 512);
}

}  // namespace attn_fb
}  // namespace rp

using namespace rp;

unsigned long long* rp_attn_trace_buffer();

// Returns RP_ERR_CONFIG (nothing launched) when the shape is outside this kernel
// (head_dim 64 is the caller's check; N <= 208 here). `Dg` holds D = rowsum(dO * O) per
// (sequence, head, query); `scratch` >= min(S H, #SMs) * 128 * 64 floats when N > 128.
int rp_attention_bwd_fused_tc(const uint16_t* qkv, const uint16_t* dout, const float* lse,
                              const float* Dg, float* scratch, int64_t S, int64_t N, int64_t H,
                              uint16_t* dqkv, cudaStream_t stream) {
  using namespace attn_fb;
  if (N < 1 || N > kMaxNk) return RP_ERR_CONFIG;
  FbGeom g;
  g.B = static_cast<int>(S);
  g.N = static_cast<int>(N);
  g.H = static_cast<int>(H);
  g.Nk = static_cast<int>((N + 15) / 16 * 16);
  g.ntile = (g.Nk + 127) / 128;
  g.npairs = static_cast<int>(S * H);
  g.qd_bytes = g.Nk * 128;
  g.ds_bytes = 65536;  // 2 ntile 64-query chunks (dQ reads whole 128-query M tiles) and the
                       // 16 warps' 4 KB output staging slots
  g.ld_qkv = 3 * H * 64;
  g.ld_o = H * 64;
  g.scale = 1.0f / 8.0f;
  g.scale_log2 = g.scale * 1.4426950408889634f;
  g.trace = rp_attn_trace_buffer();
  const int smem = fb_smem(g);
  static int max_optin = 0, nsm = 148;
  static std::once_flag once;
  std::call_once(once, [] {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(attn_bwd_fused_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, max_optin - 4096);
  });
  if (smem > max_optin - 4096) return RP_ERR_CONFIG;
  const int64_t T = S * N;
  const unsigned grid = static_cast<unsigned>(g.npairs < nsm ? g.npairs : nsm);
  CUtensorMap mq, mk, mdo, mdq, msc;
  if (make_map(&mq, qkv, T, 3 * H * 64, static_cast<uint32_t>(g.Nk)) ||
      make_map(&mk, qkv, T, 3 * H * 64, 128) ||
      make_map(&mdo, dout, T, H * 64, static_cast<uint32_t>(g.Nk)) ||
      make_map_seq(&mdq, dqkv, S, N, 3 * H * 64, 3 * H * 64) ||
      make_map_scratch(&msc, scratch, static_cast<int64_t>(grid) * 128))
    return rp_fail(RP_ERR_CUDA, "attention_bwd_fused: tensor map encode failed");
  launch_k(attn_bwd_fused_tc, dim3(grid), dim3(kFbThreads), static_cast<size_t>(smem), stream, mq, mk,
           mdo, mdq, msc, lse, Dg, scratch, g);
  return rp_check_launch("attention_bwd_fused");
}
