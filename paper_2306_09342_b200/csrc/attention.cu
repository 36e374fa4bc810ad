// Fused multi-head self-attention forward / backward on warp-level mma.sync, any head_dim
// that is a multiple of 8 up to 128 (tiles padded to HDP = 32, 64 or 128 columns, zero-filled).
//
// Replaces the per-(batch, head, window) loop of ref:proj/core/src/layers.cpp:150-166
// (gather_block x3, matmul_nt, scale, row_softmax, probs_store, matmul, scatter_block)
// and of layers.cpp:185-208 (its VJP). The reference caches the full probability tensor
// [B,H,nW,W,W] (layers.hpp:60); here only the per-row log-sum-exp is kept and P is
// recomputed in the backward (flash-attention style), and the head split / merge
// copies (gather/scatter/slice_last/concat_last) disappear: heads are read straight out
// of the packed qkv buffer [T, 3d] (q | k | v, head i at columns i*64, as
// layers.cpp:144-146,155) and dq | dk | dv are written straight into d_qkv [T, 3d]
// (layers.cpp:210 concat_last).
//
// Scale is applied after Q.K^T as in layers.cpp:159; windows (layers.cpp:119-122) are
// handled by treating each window as its own sequence (window == N is full attention).
//
// Backward is split into a dK/dV kernel (CTA per key tile, loops over all queries) and
// a dQ kernel (CTA per query tile, loops over all keys): every output element is owned
// by exactly one warp, so there are no atomics and the result is bit-reproducible.
//
// Tensor-core path: warp-level mma.sync m16n8k16 (bf16 in, fp32 accumulate).
#include "../../include/revprop_b200.h"
#include "kernels.h"
#include "ptx.cuh"
#include "attn_common.cuh"
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <utility>
#include <vector>

#include "launch.h"

namespace rp {

constexpr int kTile = 64;        // query / key rows per CTA tile

// smem tiles hold HDP bf16 per row (HDP = padded head dim, 32, 64 or 128): 16-byte chunk c
// of row r at r*2*HDP + (c with its low 3 bits XOR r&7) -> ldmatrix is bank-conflict free.
// 32-column rows (64 B) hold 4 chunks: XOR with (r/2)&3 keeps the 8 rows of one ldmatrix
// phase on distinct bank groups (two rows share a 128-byte line).
template <int HDP>
__device__ __forceinline__ uint32_t swz(int r, int c) {
  if constexpr (HDP == 32) return static_cast<uint32_t>(r * 64 + (((c ^ (r >> 1)) & 3) << 4));
  return static_cast<uint32_t>(r * HDP * 2 + (((c & ~7) | ((c ^ r) & 7)) << 4));
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, int bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
}

// Copy `rows` rows of one head (hd bf16) into a swizzled smem tile of HDP columns; rows >=
// valid and columns >= hd are zero.
template <int HDP>
__device__ __forceinline__ void load_rows(uint8_t* s, const __nv_bfloat16* g, int64_t ld, int rows,
                                          int valid, int hd) {
  const uint32_t sb = smem_u32(s);
  constexpr int CH = HDP / 8;
  for (int i = threadIdx.x; i < rows * CH; i += blockDim.x) {
    const int r = i / CH, c = i % CH;
    const bool ok = r < valid && c * 8 < hd;
    const __nv_bfloat16* src = ok ? g + static_cast<int64_t>(r) * ld + c * 8 : g;
    cp_async16(sb + swz<HDP>(r, c), src, ok ? 16 : 0);
  }
}

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t* r) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t* r) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
__device__ __forceinline__ void mma16816(float* c, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// A fragment (16 rows x 16 k) from a row-major swizzled tile: rows r0.., k-chunk pair kc.
template <int HDP>
__device__ __forceinline__ void load_a(uint32_t base, int r0, int kc, uint32_t* a) {
  const int l = threadIdx.x & 31;
  ldsm_x4(base + swz<HDP>(r0 + (l & 15), kc + (l >> 4)), a);
}
// B fragments for two n8 tiles (n0..n0+15) x k16 from a tile stored [n][k] (no transpose).
template <int HDP>
__device__ __forceinline__ void load_b_nk(uint32_t base, int n0, int kc, uint32_t* b) {
  const int l = threadIdx.x & 31;
  ldsm_x4(base + swz<HDP>(n0 + (l & 7) + ((l >> 4) << 3), kc + ((l >> 3) & 1)), b);
}
// B fragments for two n8 tiles (column chunks nc, nc+1) x k16 (rows k0..) from [k][n].
template <int HDP>
__device__ __forceinline__ void load_b_kn(uint32_t base, int k0, int nc, uint32_t* b) {
  const int l = threadIdx.x & 31;
  ldsm_x4_t(base + swz<HDP>(k0 + (l & 15), nc + (l >> 4)), b);
}

// S(16 x 64) = A(16 x HDP, regs) . B^T where B tile [64 n][HDP k] in smem rows nb..nb+63;
// n16 blocks at or beyond `valid` rows of B are skipped (their S entries stay 0 and are
// masked by the caller).
template <int HDP>
__device__ __forceinline__ void mm_abt(const uint32_t (*a)[4], uint32_t bbase, int nb,
                                       float (*s)[4], int valid = 64) {
#pragma unroll
  for (int i = 0; i < 8; ++i) s[i][0] = s[i][1] = s[i][2] = s[i][3] = 0.f;
#pragma unroll
  for (int ks = 0; ks < HDP / 16; ++ks) {
#pragma unroll
    for (int np = 0; np < 4; ++np) {
      if (16 * np >= valid) break;
      uint32_t b[4];
      load_b_nk<HDP>(bbase, nb + 16 * np, 2 * ks, b);
      mma16816(s[2 * np], a[ks], b[0], b[1]);
      mma16816(s[2 * np + 1], a[ks], b[2], b[3]);
    }
  }
}

// acc(16 x HDP) += P(16 x 64 k, C-fragment layout) . B where B tile [64 k][HDP n] rows kb..;
// k16 steps at or beyond `valid` are skipped (P is zero there).
template <int HDP>
__device__ __forceinline__ void mm_pb(const float (*p)[4], uint32_t bbase, int kb,
                                      float (*acc)[4], int valid = 64) {
#pragma unroll
  for (int ks = 0; ks < 4; ++ks) {
    if (16 * ks >= valid) break;
    uint32_t a[4];
    a[0] = pack_bf16x2(p[2 * ks][0], p[2 * ks][1]);
    a[1] = pack_bf16x2(p[2 * ks][2], p[2 * ks][3]);
    a[2] = pack_bf16x2(p[2 * ks + 1][0], p[2 * ks + 1][1]);
    a[3] = pack_bf16x2(p[2 * ks + 1][2], p[2 * ks + 1][3]);
#pragma unroll
    for (int np = 0; np < HDP / 16; ++np) {
      uint32_t b[4];
      load_b_kn<HDP>(bbase, kb + 16 * ks, 2 * np, b);
      mma16816(acc[2 * np], a, b[0], b[1]);
      mma16816(acc[2 * np + 1], a, b[2], b[3]);
    }
  }
}

struct AttnGeom {
  int B, N, H;        // sequences, tokens per sequence, heads
  int hd;             // head dim (multiple of 8, <= the kernel's HDP)
  int64_t ld_qkv;     // row pitch of qkv / d_qkv (3*H*hd)
  int64_t ld_o;       // row pitch of out / d_out (H*hd)
  float scale;        // 1/sqrt(hd)
  float scale_log2;   // scale * log2(e)
};

// bf16 pair store of a C-fragment column pair, only inside the real head columns
__device__ __forceinline__ void store_pair(__nv_bfloat16* row, int col, int hd, float a, float b) {
  if (col < hd) *reinterpret_cast<uint32_t*>(row + col) = pack_bf16x2(a, b);
}

// ------------------------------------------------------------------------ forward
// One 64-query tile of one (sequence b, head h) against all keys: Q tile, K and V
// [npad rows] already in smem (swizzled); writes out rows and the log2-domain LSE.
template <int HDP>
__device__ __forceinline__ void fwd_tile(uint32_t bQ, uint32_t bK, uint32_t bV, int npad, int q0,
                                         int h, int b, int hd, const AttnGeom& g,
                                         __nv_bfloat16* __restrict__ out,
                                         float* __restrict__ lse) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (q0 + warp * 16 >= g.N) return;  // all 16 rows of this warp are padding
  const int gq = lane >> 2, tq = lane & 3;
  uint32_t qa[HDP / 16][4];
#pragma unroll
  for (int ks = 0; ks < HDP / 16; ++ks) load_a<HDP>(bQ, warp * 16, 2 * ks, qa[ks]);

  float m[2] = {-INFINITY, -INFINITY}, l[2] = {0.f, 0.f};
  float o[HDP / 8][4];
#pragma unroll
  for (int i = 0; i < HDP / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;

  for (int kt = 0; kt < npad; kt += kTile) {
    float s[8][4];
    const int valid = g.N - kt;
    mm_abt<HDP>(qa, bK, kt, s, valid);
    float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int col = kt + nt * 8 + 2 * tq + (e & 1);
        const float v = col < g.N ? s[nt][e] * g.scale_log2 : -INFINITY;
        s[nt][e] = v;
        mx[e >> 1] = fmaxf(mx[e >> 1], v);
      }
    }
    float corr[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 1));
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 2));
      const float nm = fmaxf(m[r], mx[r]);
      corr[r] = exp2f(m[r] - nm);
      m[r] = nm;
      l[r] *= corr[r];
    }
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float p = exp2f(s[nt][e] - m[e >> 1]);
        s[nt][e] = p;
        l[e >> 1] += p;
      }
    }
#pragma unroll
    for (int nt = 0; nt < HDP / 8; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) o[nt][e] *= corr[e >> 1];
    mm_pb<HDP>(s, bV, kt, o, valid);
  }
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    l[r] += __shfl_xor_sync(0xffffffffu, l[r], 1);
    l[r] += __shfl_xor_sync(0xffffffffu, l[r], 2);
  }
  const int rowa = q0 + warp * 16 + gq;
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int row = rowa + 8 * r;
    if (row < g.N) {
      const float inv = 1.0f / l[r];
      __nv_bfloat16* orow = out + (static_cast<int64_t>(b) * g.N + row) * g.ld_o + h * hd;
#pragma unroll
      for (int nt = 0; nt < HDP / 8; ++nt)
        store_pair(orow, nt * 8 + 2 * tq, hd, o[nt][2 * r] * inv, o[nt][2 * r + 1] * inv);
      if (tq == 0)
        lse[(static_cast<int64_t>(b) * g.H + h) * g.N + row] = m[r] + log2f(l[r]);
    }
  }
}


// grid (ceil(N/64), H, B); block 128 (4 warps x 16 query rows)
// smem: Q tile [64][64] | K [Npad][64] | V [Npad][64]
template <int HDP>
__global__ void __launch_bounds__(128)
    attn_fwd_kernel(const __nv_bfloat16* __restrict__ qkv, __nv_bfloat16* __restrict__ out,
                    float* __restrict__ lse, AttnGeom g) {
  constexpr int kRowBytes = HDP * 2;
  pdl_trigger();
  pdl_wait();

  extern __shared__ __align__(128) uint8_t sm[];
  const int npad = (g.N + kTile - 1) / kTile * kTile;
  uint8_t* sQ = sm;
  uint8_t* sK = sQ + kTile * kRowBytes;
  uint8_t* sV = sK + npad * kRowBytes;
  const int q0 = blockIdx.x * kTile, h = blockIdx.y, b = blockIdx.z;
  const int hd = g.hd;
  const __nv_bfloat16* base = qkv + static_cast<int64_t>(b) * g.N * g.ld_qkv + h * hd;
  load_rows<HDP>(sQ, base + static_cast<int64_t>(q0) * g.ld_qkv, g.ld_qkv, kTile, g.N - q0, hd);
  load_rows<HDP>(sK, base + g.H * hd, g.ld_qkv, npad, g.N, hd);
  load_rows<HDP>(sV, base + 2 * g.H * hd, g.ld_qkv, npad, g.N, hd);
  cp_async_wait_all();
  __syncthreads();
  fwd_tile<HDP>(smem_u32(sQ), smem_u32(sK), smem_u32(sV), npad, q0, h, b, hd, g, out, lse);
}

// Short sequences (windows of N <= 64 tokens, e.g. Swin's 49): a persistent CTA walks
// (sequence, head) items with the next item's Q / K / V tiles streaming into the other
// half of a double buffer (cp.async groups) while the current one computes -- one item's
// loads alone cannot keep enough bytes in flight to cover HBM latency.
template <int HDP>
__global__ void __launch_bounds__(128)
    attn_fwd_small_kernel(const __nv_bfloat16* __restrict__ qkv, __nv_bfloat16* __restrict__ out,
                          float* __restrict__ lse, AttnGeom g) {
  constexpr int kRowBytes = HDP * 2, kBuf = 3 * kTile * kRowBytes;
  pdl_trigger();
  pdl_wait();

  extern __shared__ __align__(128) uint8_t sm[];
  const int total = g.B * g.H, hd = g.hd;
  auto prefetch = [&](int item, int slot) {
    const int h = item % g.H, b = item / g.H;
    const __nv_bfloat16* base = qkv + static_cast<int64_t>(b) * g.N * g.ld_qkv + h * hd;
    uint8_t* buf = sm + slot * kBuf;
    load_rows<HDP>(buf, base, g.ld_qkv, kTile, g.N, hd);
    load_rows<HDP>(buf + kTile * kRowBytes, base + g.H * hd, g.ld_qkv, kTile, g.N, hd);
    load_rows<HDP>(buf + 2 * kTile * kRowBytes, base + 2 * g.H * hd, g.ld_qkv, kTile, g.N, hd);
  };
  int item = blockIdx.x;
  if (item < total) prefetch(item, 0);
  asm volatile("cp.async.commit_group;" ::: "memory");
  for (int k = 0; item < total; ++k, item += gridDim.x) {
    const int next = item + gridDim.x;
    if (next < total) prefetch(next, (k + 1) & 1);
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 1;" ::: "memory");
    __syncthreads();
    const uint32_t b0 = smem_u32(sm + (k & 1) * kBuf);
    fwd_tile<HDP>(b0, b0 + kTile * kRowBytes, b0 + 2 * kTile * kRowBytes, kTile, 0,
                  item % g.H, item / g.H, hd, g, out, lse);
    __syncthreads();  // this buffer is refilled by the prefetch two items ahead
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
}

// D[b][h][n] = sum_c dO[row][h*64+c] * O[row][h*64+c]   (softmax VJP dot, ops.cpp:219-220)
__global__ void attn_bwd_dot_kernel(const __nv_bfloat16* __restrict__ out,
                                    const __nv_bfloat16* __restrict__ dout,
                                    float* __restrict__ D, AttnGeom g) {
  pdl_trigger();
  pdl_wait();

  const int64_t total = static_cast<int64_t>(g.B) * g.N * g.H;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int h = static_cast<int>(i % g.H);
    const int64_t row = i / g.H;  // b*N + n
    const uint4* o = reinterpret_cast<const uint4*>(out + row * g.ld_o + h * g.hd);
    const uint4* d = reinterpret_cast<const uint4*>(dout + row * g.ld_o + h * g.hd);
    float acc = 0.f;
    for (int j = 0; j < g.hd / 8; ++j) {
      const uint4 a = o[j], c = d[j];
      const uint32_t av[4] = {a.x, a.y, a.z, a.w}, cv[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float2 fa = unpack_bf16x2(av[k]), fc = unpack_bf16x2(cv[k]);
        acc += fa.x * fc.x + fa.y * fc.y;
      }
    }
    const int64_t b = row / g.N, n = row % g.N;
    D[(b * g.H + h) * g.N + n] = acc;
  }
}

// ------------------------------------------------------------------------ dK, dV
// grid (ceil(N/64), H, B): CTA owns 64 keys; loops over all query tiles.
// smem: K tile | V tile | Q [Npad] | dO [Npad] | lse [Npad] | D [Npad]
template <int HDP>
__global__ void __launch_bounds__(128)
    attn_bwd_dkdv_kernel(const __nv_bfloat16* __restrict__ qkv,
                         const __nv_bfloat16* __restrict__ dout, const float* __restrict__ lse,
                         const float* __restrict__ Dg, __nv_bfloat16* __restrict__ dqkv,
                         AttnGeom g) {
  pdl_trigger();
  pdl_wait();

  constexpr int kRowBytes = HDP * 2;
  extern __shared__ __align__(128) uint8_t sm[];
  const int npad = (g.N + kTile - 1) / kTile * kTile;
  uint8_t* sK = sm;
  uint8_t* sV = sK + kTile * kRowBytes;
  uint8_t* sQ = sV + kTile * kRowBytes;
  uint8_t* sO = sQ + npad * kRowBytes;
  float* sL = reinterpret_cast<float*>(sO + npad * kRowBytes);
  float* sD = sL + npad;
  const int k0 = blockIdx.x * kTile, h = blockIdx.y, b = blockIdx.z;
  const int hd = g.hd;
  const __nv_bfloat16* base = qkv + static_cast<int64_t>(b) * g.N * g.ld_qkv + h * hd;
  load_rows<HDP>(sK, base + static_cast<int64_t>(k0) * g.ld_qkv + g.H * hd, g.ld_qkv, kTile,
                 g.N - k0, hd);
  load_rows<HDP>(sV, base + static_cast<int64_t>(k0) * g.ld_qkv + 2 * g.H * hd, g.ld_qkv, kTile,
                 g.N - k0, hd);
  load_rows<HDP>(sQ, base, g.ld_qkv, npad, g.N, hd);
  load_rows<HDP>(sO, dout + static_cast<int64_t>(b) * g.N * g.ld_o + h * hd, g.ld_o, npad, g.N, hd);
  const float* lrow = lse + (static_cast<int64_t>(b) * g.H + h) * g.N;
  const float* drow = Dg + (static_cast<int64_t>(b) * g.H + h) * g.N;
  for (int i = threadIdx.x; i < npad; i += blockDim.x) {
    sL[i] = i < g.N ? lrow[i] : 0.f;
    sD[i] = i < g.N ? drow[i] : 0.f;
  }
  cp_async_wait_all();
  __syncthreads();

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (k0 + warp * 16 >= g.N) return;  // padding keys only
  const int tq = lane & 3, gq = lane >> 2;
  const uint32_t bK = smem_u32(sK), bV = smem_u32(sV), bQ = smem_u32(sQ), bO = smem_u32(sO);
  uint32_t ka[HDP / 16][4], va[HDP / 16][4];
#pragma unroll
  for (int ks = 0; ks < HDP / 16; ++ks) {
    load_a<HDP>(bK, warp * 16, 2 * ks, ka[ks]);
    load_a<HDP>(bV, warp * 16, 2 * ks, va[ks]);
  }
  float dk[HDP / 8][4], dv[HDP / 8][4];
#pragma unroll
  for (int i = 0; i < HDP / 8; ++i)
#pragma unroll
    for (int e = 0; e < 4; ++e) dk[i][e] = dv[i][e] = 0.f;

  for (int qt = 0; qt < npad; qt += kTile) {
    float st[8][4], dpt[8][4];
    const int valid = g.N - qt;
    mm_abt<HDP>(ka, bQ, qt, st, valid);   // S^T [16 keys][64 queries]
    mm_abt<HDP>(va, bO, qt, dpt, valid);  // dP^T = V . dO^T
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int q = qt + nt * 8 + 2 * tq + (e & 1);
        const float p = q < g.N ? exp2f(st[nt][e] * g.scale_log2 - sL[q]) : 0.f;
        st[nt][e] = p;
        dpt[nt][e] = p * (dpt[nt][e] - sD[q]) * g.scale;
      }
    }
    mm_pb<HDP>(st, bO, qt, dv, valid);   // dV += P^T . dO
    mm_pb<HDP>(dpt, bQ, qt, dk, valid);  // dK += dS^T . Q
  }
  const int rowa = k0 + warp * 16 + gq;
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int row = rowa + 8 * r;
    if (row < g.N) {
      __nv_bfloat16* drow_k =
          dqkv + (static_cast<int64_t>(b) * g.N + row) * g.ld_qkv + g.H * hd + h * hd;
      __nv_bfloat16* drow_v = drow_k + g.H * hd;
#pragma unroll
      for (int nt = 0; nt < HDP / 8; ++nt) {
        store_pair(drow_k, nt * 8 + 2 * tq, hd, dk[nt][2 * r], dk[nt][2 * r + 1]);
        store_pair(drow_v, nt * 8 + 2 * tq, hd, dv[nt][2 * r], dv[nt][2 * r + 1]);
      }
    }
  }
  (void)gq;
}

// ------------------------------------------------------------------------ dQ
// grid (ceil(N/64), H, B): CTA owns 64 queries; loops over all key tiles.
// smem: Q tile | dO tile | K [Npad] | V [Npad]
template <int HDP>
__global__ void __launch_bounds__(128)
    attn_bwd_dq_kernel(const __nv_bfloat16* __restrict__ qkv,
                       const __nv_bfloat16* __restrict__ dout, const float* __restrict__ lse,
                       const float* __restrict__ Dg, __nv_bfloat16* __restrict__ dqkv,
                       AttnGeom g) {
  pdl_trigger();
  pdl_wait();

  constexpr int kRowBytes = HDP * 2;
  extern __shared__ __align__(128) uint8_t sm[];
  const int npad = (g.N + kTile - 1) / kTile * kTile;
  uint8_t* sQ = sm;
  uint8_t* sO = sQ + kTile * kRowBytes;
  uint8_t* sK = sO + kTile * kRowBytes;
  uint8_t* sV = sK + npad * kRowBytes;
  const int q0 = blockIdx.x * kTile, h = blockIdx.y, b = blockIdx.z;
  const int hd = g.hd;
  const __nv_bfloat16* base = qkv + static_cast<int64_t>(b) * g.N * g.ld_qkv + h * hd;
  load_rows<HDP>(sQ, base + static_cast<int64_t>(q0) * g.ld_qkv, g.ld_qkv, kTile, g.N - q0, hd);
  load_rows<HDP>(sO, dout + (static_cast<int64_t>(b) * g.N + q0) * g.ld_o + h * hd, g.ld_o, kTile,
                 g.N - q0, hd);
  load_rows<HDP>(sK, base + g.H * hd, g.ld_qkv, npad, g.N, hd);
  load_rows<HDP>(sV, base + 2 * g.H * hd, g.ld_qkv, npad, g.N, hd);
  cp_async_wait_all();
  __syncthreads();

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (q0 + warp * 16 >= g.N) return;  // padding queries only
  const int tq = lane & 3, gq = lane >> 2;
  const uint32_t bQ = smem_u32(sQ), bO = smem_u32(sO), bK = smem_u32(sK), bV = smem_u32(sV);
  uint32_t qa[HDP / 16][4], oa[HDP / 16][4];
#pragma unroll
  for (int ks = 0; ks < HDP / 16; ++ks) {
    load_a<HDP>(bQ, warp * 16, 2 * ks, qa[ks]);
    load_a<HDP>(bO, warp * 16, 2 * ks, oa[ks]);
  }
  const int rowa = q0 + warp * 16 + gq;
  float lr[2], dr[2];
  const int64_t hb = (static_cast<int64_t>(b) * g.H + h) * g.N;
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int row = rowa + 8 * r;
    lr[r] = row < g.N ? lse[hb + row] : 0.f;
    dr[r] = row < g.N ? Dg[hb + row] : 0.f;
  }
  float dq[HDP / 8][4];
#pragma unroll
  for (int i = 0; i < HDP / 8; ++i) dq[i][0] = dq[i][1] = dq[i][2] = dq[i][3] = 0.f;

  for (int kt = 0; kt < npad; kt += kTile) {
    float s[8][4], dp[8][4];
    const int valid = g.N - kt;
    mm_abt<HDP>(qa, bK, kt, s, valid);
    mm_abt<HDP>(oa, bV, kt, dp, valid);
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int kc = kt + nt * 8 + 2 * tq + (e & 1);
        const float p = kc < g.N ? exp2f(s[nt][e] * g.scale_log2 - lr[e >> 1]) : 0.f;
        s[nt][e] = p * (dp[nt][e] - dr[e >> 1]) * g.scale;
      }
    }
    mm_pb<HDP>(s, bK, kt, dq, valid);  // dQ += dS . K
  }
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int row = rowa + 8 * r;
    if (row < g.N) {
      __nv_bfloat16* drow = dqkv + (static_cast<int64_t>(b) * g.N + row) * g.ld_qkv + h * hd;
#pragma unroll
      for (int nt = 0; nt < HDP / 8; ++nt)
        store_pair(drow, nt * 8 + 2 * tq, hd, dq[nt][2 * r], dq[nt][2 * r + 1]);
    }
  }
}

// ------------------------------------------------------------ short windows (N <= 64)
// Swin's 49-token windows: every (window, head) item is ONE 64-row tile, so the online
// softmax (rescaling), the per-element exp2f range handling and the per-tile loop bounds of
// the general kernels are pure instruction overhead -- the general kernels run
// instruction-issue-bound here (ncu: 69 % issue slots busy, ~1000 instructions per warp and
// item, profiles/round2_window_attention.md). These kernels are persistent (a CTA walks
// items with the next item's tiles landing in the other half of a double buffer), stage
// the tiles by TMA when head_dim is 32 or 64 (one thread issues 3-4 box loads per item; the
// SW64 / SW128 smem swizzle is the one swz<> describes), else by cp.async, compute every
// 16 x 64 tile over all 64 key columns (no per-tile bounds) and mask only the boundary
// key tile, and use ex2.approx directly.
__device__ __forceinline__ float ex2a(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ void stsm_x4(uint32_t addr, uint32_t r0, uint32_t r1, uint32_t r2,
                                        uint32_t r3) {
  asm volatile("stmatrix.sync.aligned.m8n8.x4.shared.b16 [%0], {%1,%2,%3,%4};" ::"r"(addr),
               "r"(r0), "r"(r1), "r"(r2), "r"(r3)
               : "memory");
}
__device__ __forceinline__ void zero_smem(uint8_t* p, int bytes) {
  for (int i = threadIdx.x * 16; i < bytes; i += blockDim.x * 16)
    *reinterpret_cast<uint4*>(p + i) = make_uint4(0, 0, 0, 0);
}
// c = a . b with a zero accumulator (no register zeroing before the first k step)
__device__ __forceinline__ void mma16816_z(float* c, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%10,%10,%10,%10};"
      : "=f"(c[0]), "=f"(c[1]), "=f"(c[2]), "=f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1), "f"(0.f));
}
// S(16 x 64) = A(16 x HDP) . B^T over all 64 rows of the B tile
template <int HDP>
__device__ __forceinline__ void mm_abt64(const uint32_t (*a)[4], uint32_t bbase, float (*s)[4]) {
#pragma unroll
  for (int ks = 0; ks < HDP / 16; ++ks)
#pragma unroll
    for (int np = 0; np < 4; ++np) {
      uint32_t b[4];
      load_b_nk<HDP>(bbase, 16 * np, 2 * ks, b);
      if (ks == 0) {
        mma16816_z(s[2 * np], a[0], b[0], b[1]);
        mma16816_z(s[2 * np + 1], a[0], b[2], b[3]);
      } else {
        mma16816(s[2 * np], a[ks], b[0], b[1]);
        mma16816(s[2 * np + 1], a[ks], b[2], b[3]);
      }
    }
}
// acc(16 x HDP) = P(16 x 64, C-fragment layout) . B over all 64 rows of the B tile [k][n]
template <int HDP>
__device__ __forceinline__ void mm_pb64(const float (*p)[4], uint32_t bbase, float (*acc)[4]) {
#pragma unroll
  for (int ks = 0; ks < 4; ++ks) {
    uint32_t a[4];
    a[0] = pack_bf16x2(p[2 * ks][0], p[2 * ks][1]);
    a[1] = pack_bf16x2(p[2 * ks][2], p[2 * ks][3]);
    a[2] = pack_bf16x2(p[2 * ks + 1][0], p[2 * ks + 1][1]);
    a[3] = pack_bf16x2(p[2 * ks + 1][2], p[2 * ks + 1][3]);
#pragma unroll
    for (int np = 0; np < HDP / 16; ++np) {
      uint32_t b[4];
      load_b_kn<HDP>(bbase, 16 * ks, 2 * np, b);
      if (ks == 0) {
        mma16816_z(acc[2 * np], a, b[0], b[1]);
        mma16816_z(acc[2 * np + 1], a, b[2], b[3]);
      } else {
        mma16816(acc[2 * np], a, b[0], b[1]);
        mma16816(acc[2 * np + 1], a, b[2], b[3]);
      }
    }
  }
}

// cp.async staging (head_dim without a TMA box): rows [0, N) of q, k, v (qkv column blocks
// m * H * hd, row pitch ldq) and, with NM = 4, dO (row pitch ldo). Chunks beyond hd and
// rows beyond N are never written (zeroed once at kernel start). Slot j of a row = (matrix
// j / (HDP/8), chunk j % (HDP/8)): compile-time divisions only.
template <int HDP, int NM>
__device__ __forceinline__ void win_load(uint8_t* buf, const __nv_bfloat16* qb, int64_t mstride,
                                         int64_t ldq, const __nv_bfloat16* ob, int64_t ldo,
                                         int N, int hd) {
  constexpr int CH = HDP / 8, SL = NM * CH, kTileBytes = kTile * HDP * 2;
  const uint32_t sb = smem_u32(buf);
  const int chv = hd / 8;
  for (int i = threadIdx.x; i < N * SL; i += blockDim.x) {
    const int r = i / SL, j = i % SL, m = j / CH, c = j % CH;
    if (c < chv) {
      const __nv_bfloat16* src = (NM == 4 && m == 3) ? ob + r * ldo : qb + m * mstride + r * ldq;
      cp_async16(sb + m * kTileBytes + swz<HDP>(r, c), src + c * 8, 16);
    }
  }
}

// Mask keys >= N of a score fragment (only n8 tiles reaching past N; uniform branches).
__device__ __forceinline__ void mask_cols(float (*s)[4], int N, int tq, float fill) {
#pragma unroll
  for (int nt = 0; nt < 8; ++nt) {
    if (nt * 8 + 8 > N) {
      const int c0 = nt * 8 + 2 * tq;
      if (c0 >= N) s[nt][0] = s[nt][2] = fill;
      if (c0 + 1 >= N) s[nt][1] = s[nt][3] = fill;
    }
  }
}

// TMA maps of one window item: q | k | v boxes of {hd, N} out of qkv [T][3 H hd], dO boxes
// out of dout [T][H hd]
struct WinMaps {
  CUtensorMap qkv, dout;
};

// grid = min(items, SMs x resident CTAs); block 128 (4 warps x 16 query rows)
// NW > 0: the window length as a compile-time constant (Swin's 7 x 7 = 49): masks, loop
// bounds and row offsets fold; NW = 0 reads it from g.N. With TMA the head dim is HDP.
template <int HDP, bool TMA, int NW>
__global__ void __launch_bounds__(128)
    attn_fwd_win_kernel(const __grid_constant__ WinMaps maps,
                        const __nv_bfloat16* __restrict__ qkv, __nv_bfloat16* __restrict__ out,
                        float* __restrict__ lse, AttnGeom g) {
  constexpr int kT = kTile * HDP * 2, kBuf = 3 * kT;
  pdl_trigger();
  extern __shared__ uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) &
                                           ~static_cast<uintptr_t>(1023));
  __shared__ __align__(8) uint64_t bar[2];
  zero_smem(sm, 2 * kBuf);
  if (TMA && threadIdx.x == 0) {
    tma_prefetch_desc(&maps.qkv);
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_barrier_init();
  }
  fence_proxy_async_smem();  // the zero fill is visible to the TMA writes around it
  __syncthreads();
  pdl_wait();
  const int total = g.B * g.H, hd = TMA ? HDP : g.hd, N = NW ? NW : g.N;
  auto prefetch = [&](int item, int slot) {
    const int h = item % g.H, b = item / g.H;
    uint8_t* buf = sm + slot * kBuf;
    if constexpr (TMA) {
      if (threadIdx.x == 0) {
        mbar_arrive_expect_tx(&bar[slot], static_cast<uint32_t>(3 * N * hd * 2));
#pragma unroll
        for (int m = 0; m < 3; ++m)
          tma_load_2d(buf + m * kT, &maps.qkv, &bar[slot], (m * g.H + h) * hd, b * N);
      }
    } else {
      const __nv_bfloat16* base = qkv + static_cast<int64_t>(b) * N * g.ld_qkv + h * hd;
      win_load<HDP, 3>(buf, base, g.H * hd, g.ld_qkv, nullptr, 0, N, hd);
    }
  };
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, gq = lane >> 2, tq = lane & 3;
  int item = blockIdx.x;
  if (item < total) prefetch(item, 0);
  if (!TMA) asm volatile("cp.async.commit_group;" ::: "memory");
  for (int k = 0; item < total; ++k, item += gridDim.x) {
    const int next = item + gridDim.x;
    if (next < total) prefetch(next, (k + 1) & 1);
    if constexpr (TMA) {
      mbar_wait(&bar[k & 1], (k >> 1) & 1);
    } else {
      asm volatile("cp.async.commit_group;\ncp.async.wait_group 1;" ::: "memory");
      __syncthreads();
    }
    if (warp * 16 < N) {
      const uint32_t bQ = smem_u32(sm + (k & 1) * kBuf), bK = bQ + kT, bV = bQ + 2 * kT;
      uint32_t qa[HDP / 16][4];
#pragma unroll
      for (int ks = 0; ks < HDP / 16; ++ks) load_a<HDP>(bQ, warp * 16, 2 * ks, qa[ks]);
      float s[8][4];
      mm_abt64<HDP>(qa, bK, s);
      mask_cols(s, N, tq, -INFINITY);
      float mx[2];
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        float m = -INFINITY;
#pragma unroll
        for (int nt = 0; nt < 8; ++nt) m = fmaxf(m, fmaxf(s[nt][2 * r], s[nt][2 * r + 1]));
        m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 1));
        m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 2));
        mx[r] = m * g.scale_log2;
      }
      float l[2] = {0.f, 0.f};
#pragma unroll
      for (int nt = 0; nt < 8; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float p = ex2a(fmaf(s[nt][e], g.scale_log2, -mx[e >> 1]));
          s[nt][e] = p;
          l[e >> 1] += p;
        }
      float o[HDP / 8][4];
      mm_pb64<HDP>(s, bV, o);
      const int h = item % g.H, b = item / g.H;
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        l[r] += __shfl_xor_sync(0xffffffffu, l[r], 1);
        l[r] += __shfl_xor_sync(0xffffffffu, l[r], 2);
        const int row = warp * 16 + gq + 8 * r;
        if (row < N) {
          const float inv = __fdividef(1.0f, l[r]);
          __nv_bfloat16* orow = out + (static_cast<int64_t>(b) * N + row) * g.ld_o + h * hd;
#pragma unroll
          for (int nt = 0; nt < HDP / 8; ++nt)
            store_pair(orow, nt * 8 + 2 * tq, hd, o[nt][2 * r] * inv, o[nt][2 * r + 1] * inv);
          if (tq == 0) lse[(static_cast<int64_t>(b) * g.H + h) * N + row] = mx[r] + __log2f(l[r]);
        }
      }
    }
    __syncthreads();  // this buffer is refilled by the prefetch two items ahead
  }
  if (!TMA) asm volatile("cp.async.wait_group 0;" ::: "memory");
}

// Fused backward of one (window, head) item per pass, no D pre-pass and no O read:
//   phase A (warp w = queries 16w..): S = Q K^T, dP = dO V^T, P = exp2(S scale - lse),
//     D = rowsum(P * dP) (the softmax VJP's sum as ref:proj/core/src/ops.cpp:219-220 forms
//     it from the cached probabilities), dS' = P (dP - D), dQ = scale (dS' K); P and dS'
//     -> smem (bf16, stmatrix)
//   phase B (warp w = keys 16w..): dV = P^T dO, dK = scale (dS'^T Q) (ldmatrix.trans)
// (the softmax scale is applied once per output element instead of per score)
// Every output element is written by one warp: no atomics, bit-reproducible.
template <int HDP, bool TMA, int NW>
__global__ void __launch_bounds__(128)
    attn_bwd_win_kernel(const __grid_constant__ WinMaps maps,
                        const __nv_bfloat16* __restrict__ qkv,
                        const __nv_bfloat16* __restrict__ dout, const float* __restrict__ lse,
                        __nv_bfloat16* __restrict__ dqkv, AttnGeom g) {
  // Q K V dO (every tile 1024-byte aligned, as the TMA swizzle requires); the LSE of the
  // next item is loaded into registers one item ahead
  constexpr int kT = kTile * HDP * 2, kBuf = 4 * kT;
  constexpr int kPS = kTile * 64 * 2;                              // P or dS, bf16 [64][64]
  pdl_trigger();
  extern __shared__ uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) &
                                           ~static_cast<uintptr_t>(1023));
  __shared__ __align__(8) uint64_t bar[2];
  zero_smem(sm, 2 * kBuf + 2 * kPS);
  if (TMA && threadIdx.x == 0) {
    tma_prefetch_desc(&maps.qkv);
    tma_prefetch_desc(&maps.dout);
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_barrier_init();
  }
  fence_proxy_async_smem();
  __syncthreads();
  pdl_wait();
  const int total = g.B * g.H, hd = TMA ? HDP : g.hd, N = NW ? NW : g.N;
  auto prefetch = [&](int item, int slot) {
    const int h = item % g.H, b = item / g.H;
    uint8_t* buf = sm + slot * kBuf;
    if constexpr (TMA) {
      if (threadIdx.x == 0) {
        mbar_arrive_expect_tx(&bar[slot], static_cast<uint32_t>(4 * N * hd * 2));
#pragma unroll
        for (int m = 0; m < 3; ++m)
          tma_load_2d(buf + m * kT, &maps.qkv, &bar[slot], (m * g.H + h) * hd, b * N);
        tma_load_2d(buf + 3 * kT, &maps.dout, &bar[slot], h * hd, b * N);
      }
    } else {
      const __nv_bfloat16* base = qkv + static_cast<int64_t>(b) * N * g.ld_qkv + h * hd;
      win_load<HDP, 4>(buf, base, g.H * hd, g.ld_qkv,
                       dout + static_cast<int64_t>(b) * N * g.ld_o + h * hd, g.ld_o, N, hd);
    }
  };
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, gq = lane >> 2, tq = lane & 3;
  const uint32_t bP = smem_u32(sm + 2 * kBuf), bS = bP + kPS;
  // this thread's two query rows' LSE ([B][H][N]: item = b H + h); padded rows: P = 0
  auto load_lse = [&](int it, float* v) {
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int row = warp * 16 + gq + 8 * r;
      v[r] = it < total && row < N ? __ldg(lse + static_cast<int64_t>(it) * N + row) : INFINITY;
    }
  };
  int item = blockIdx.x;
  float lse_next[2];
  load_lse(item, lse_next);
  if (item < total) prefetch(item, 0);
  if (!TMA) asm volatile("cp.async.commit_group;" ::: "memory");
  for (int k = 0; item < total; ++k, item += gridDim.x) {
    const int next = item + gridDim.x;
    if (next < total) prefetch(next, (k + 1) & 1);
    if constexpr (TMA) {
      mbar_wait(&bar[k & 1], (k >> 1) & 1);
    } else {
      asm volatile("cp.async.commit_group;\ncp.async.wait_group 1;" ::: "memory");
      __syncthreads();
    }
    uint8_t* buf = sm + (k & 1) * kBuf;
    const uint32_t bQ = smem_u32(buf), bK = bQ + kT, bV = bQ + 2 * kT, bO = bQ + 3 * kT;
    const float lr[2] = {lse_next[0], lse_next[1]};
    load_lse(next, lse_next);
    const int h = item % g.H, b = item / g.H;
    const int64_t row0 = static_cast<int64_t>(b) * N;
    // ---- phase A: warp w owns queries [16w, 16w + 16)
    if (warp * 16 < N) {
      float s[8][4], dp[8][4];
      {
        uint32_t qa[HDP / 16][4], oa[HDP / 16][4];
#pragma unroll
        for (int ks = 0; ks < HDP / 16; ++ks) {
          load_a<HDP>(bQ, warp * 16, 2 * ks, qa[ks]);
          load_a<HDP>(bO, warp * 16, 2 * ks, oa[ks]);
        }
        mm_abt64<HDP>(qa, bK, s);
        mm_abt64<HDP>(oa, bV, dp);
      }
      mask_cols(s, N, tq, -INFINITY);
      float dsum[2] = {0.f, 0.f};
#pragma unroll
      for (int nt = 0; nt < 8; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float p = ex2a(fmaf(s[nt][e], g.scale_log2, -lr[e >> 1]));
          s[nt][e] = p;
          dsum[e >> 1] = fmaf(p, dp[nt][e], dsum[e >> 1]);
        }
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        dsum[r] += __shfl_xor_sync(0xffffffffu, dsum[r], 1);
        dsum[r] += __shfl_xor_sync(0xffffffffu, dsum[r], 2);
      }
#pragma unroll
      for (int nt = 0; nt < 8; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e) dp[nt][e] = s[nt][e] * (dp[nt][e] - dsum[e >> 1]);
      // P and dS (bf16) to smem as [query][key] 64 x 64 tiles, one stmatrix per 16 x 16 block
#pragma unroll
      for (int np = 0; np < 4; ++np) {
        const uint32_t off =
            swz<64>(warp * 16 + (lane & 7) + ((lane >> 3) & 1) * 8, 2 * np + (lane >> 4));
        stsm_x4(bP + off, pack_bf16x2(s[2 * np][0], s[2 * np][1]),
                pack_bf16x2(s[2 * np][2], s[2 * np][3]),
                pack_bf16x2(s[2 * np + 1][0], s[2 * np + 1][1]),
                pack_bf16x2(s[2 * np + 1][2], s[2 * np + 1][3]));
        stsm_x4(bS + off, pack_bf16x2(dp[2 * np][0], dp[2 * np][1]),
                pack_bf16x2(dp[2 * np][2], dp[2 * np][3]),
                pack_bf16x2(dp[2 * np + 1][0], dp[2 * np + 1][1]),
                pack_bf16x2(dp[2 * np + 1][2], dp[2 * np + 1][3]));
      }
      float dq[HDP / 8][4];
      mm_pb64<HDP>(dp, bK, dq);  // dQ = scale (dS' K)
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int row = warp * 16 + gq + 8 * r;
        if (row < N) {
          __nv_bfloat16* drow = dqkv + (row0 + row) * g.ld_qkv + h * hd;
#pragma unroll
          for (int nt = 0; nt < HDP / 8; ++nt)
            store_pair(drow, nt * 8 + 2 * tq, hd, dq[nt][2 * r] * g.scale,
                       dq[nt][2 * r + 1] * g.scale);
        }
      }
    }
    __syncthreads();
    // ---- phase B: warp w owns keys [16w, 16w + 16): dV = P^T dO, dK = dS^T Q
    if (warp * 16 < N) {
      float dk[HDP / 8][4], dv[HDP / 8][4];
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        // A = P^T (16 keys x 16 queries): transposed 8 x 8 blocks of P rows 16 ks..
        const uint32_t off =
            swz<64>(16 * ks + (lane & 7) + ((lane >> 4) << 3), 2 * warp + ((lane >> 3) & 1));
        uint32_t pa[4], sa[4];
        ldsm_x4_t(bP + off, pa);
        ldsm_x4_t(bS + off, sa);
#pragma unroll
        for (int np = 0; np < HDP / 16; ++np) {
          uint32_t bo[4], bq[4];
          load_b_kn<HDP>(bO, 16 * ks, 2 * np, bo);
          load_b_kn<HDP>(bQ, 16 * ks, 2 * np, bq);
          if (ks == 0) {
            mma16816_z(dv[2 * np], pa, bo[0], bo[1]);
            mma16816_z(dv[2 * np + 1], pa, bo[2], bo[3]);
            mma16816_z(dk[2 * np], sa, bq[0], bq[1]);
            mma16816_z(dk[2 * np + 1], sa, bq[2], bq[3]);
          } else {
            mma16816(dv[2 * np], pa, bo[0], bo[1]);
            mma16816(dv[2 * np + 1], pa, bo[2], bo[3]);
            mma16816(dk[2 * np], sa, bq[0], bq[1]);
            mma16816(dk[2 * np + 1], sa, bq[2], bq[3]);
          }
        }
      }
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int row = warp * 16 + gq + 8 * r;
        if (row < N) {
          __nv_bfloat16* drow_k = dqkv + (row0 + row) * g.ld_qkv + g.H * hd + h * hd;
          __nv_bfloat16* drow_v = drow_k + g.H * hd;
#pragma unroll
          for (int nt = 0; nt < HDP / 8; ++nt) {
            store_pair(drow_k, nt * 8 + 2 * tq, hd, dk[nt][2 * r] * g.scale,
                       dk[nt][2 * r + 1] * g.scale);
            store_pair(drow_v, nt * 8 + 2 * tq, hd, dv[nt][2 * r], dv[nt][2 * r + 1]);
          }
        }
      }
    }
    __syncthreads();  // P / dS and this buffer are rewritten by the next items
  }
  if (!TMA) asm volatile("cp.async.wait_group 0;" ::: "memory");
}

static AttnGeom make_geom(int64_t B, int64_t N, int64_t H, int64_t hd) {
  AttnGeom g;
  g.B = static_cast<int>(B);
  g.N = static_cast<int>(N);
  g.H = static_cast<int>(H);
  g.hd = static_cast<int>(hd);
  g.ld_qkv = 3 * H * hd;
  g.ld_o = H * hd;
  g.scale = 1.0f / sqrtf(static_cast<float>(hd));
  g.scale_log2 = g.scale * 1.4426950408889634f;
  return g;
}

static int set_smem_attr(const void* fn, int bytes) {
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) == cudaSuccess)
    return RP_OK;
  cudaGetLastError();  // not sticky: do not leak it into the next launch check
  return rp_fail(RP_ERR_SHAPE, "attention: sequence too long for the shared-memory tile");
}

}  // namespace rp

using namespace rp;

static int attn_check(int64_t B, int64_t N, int64_t H, int64_t hd) {
  if (B <= 0 || N <= 0 || H <= 0) return rp_fail(RP_ERR_SHAPE, "attention: empty shape");
  if (hd < 8 || hd > 128 || hd % 8)
    return rp_fail(RP_ERR_SHAPE, "attention: head_dim must be a multiple of 8 in [8, 128]");
  // tcgen05 (head_dim 64): forward up to 512 keys, backward up to 768; mma.sync keeps K and
  // V resident in smem: 768 keys at head_dim <= 64, 384 above
  const int64_t nmax = hd <= 64 ? 768 : 384;
  if (N > nmax) return rp_fail(RP_ERR_SHAPE, "attention: sequence (window) too long for head_dim");
  return RP_OK;
}

// qkv [B*N, 3*H*hd] bf16 -> out [B*N, H*hd] bf16, lse [B][H][N] (log2 domain).
// B here is the number of independent sequences (batch x windows).
int rp_attention_fwd_tc(const uint16_t* qkv, int64_t S, int64_t N, int64_t H, uint16_t* out,
                        float* lse, cudaStream_t stream);
int rp_attention_bwd_tc(const uint16_t* qkv, const uint16_t* out, const uint16_t* dout,
                        const float* lse, float* Dg, int64_t S, int64_t N, int64_t H,
                        uint16_t* dqkv, cudaStream_t stream, uint16_t* dSt, int d_ready,
                        int fused);
int rp_attention_fwd_tc_wide(const uint16_t* qkv, int64_t S, int64_t N, int64_t H, int64_t hd,
                             uint16_t* out, float* lse, cudaStream_t stream);
int rp_attention_bwd_tc_wide(const uint16_t* qkv, const uint16_t* out, const uint16_t* dout,
                             const float* lse, float* Dg, int64_t S, int64_t N, int64_t H,
                             int64_t hd, uint16_t* dqkv, cudaStream_t stream);
// 0 = tcgen05 where it applies (head_dim 64): backward in one fused pass for N <= 208
// (attention_bwd_fused.cu), above that one dK/dV pass + dQ from the stored dS^T;
// 1 = mma.sync only; 2 = tcgen05 with the two-pass (dQ pass, dK/dV pass) backward that
// keeps no dS; 3 = tcgen05 with the dS^T round trip at every N <= 256 (the previous default)
static int g_attn_impl = 0;

// clock64 trace of the ping-pong forward's CTA 0 (tools/attn_fwd_trace.py): on when set
static unsigned long long* g_attn_trace = nullptr;
unsigned long long* rp_attn_trace_buffer() { return g_attn_trace; }
extern "C" int rp_set_attention_trace(void* device_buffer) {
  g_attn_trace = static_cast<unsigned long long*>(device_buffer);
  return RP_OK;
}

// forward kernel variant for N <= 256 (A/B): 0 ping-pong softmax groups (attn_fwd_tc_pp)
// with the P V product split over two issuers where the TMEM plan allows (Nk <= 208),
// 1 the lockstep persistent kernel (N <= 224), 2 ping-pong with one P V issuer
static int g_attn_fwd_variant = 0;
int rp_attn_fwd_variant() { return g_attn_fwd_variant; }
extern "C" int rp_set_attention_fwd_variant(int v) {
  if (v < 0 || v > 2)
    return rp_fail(RP_ERR_CONFIG, "attention forward variant must be 0, 1 or 2");
  g_attn_fwd_variant = v;
  return RP_OK;
}

// Process-global switch, read when a step is enqueued: engines must drop their captured
// graphs (rp_engine_invalidate_graphs) after changing it, or the graphs keep the old kernels.
extern "C" int rp_set_attention_impl(int impl) {
  if (impl < 0 || impl > 3) return rp_fail(RP_ERR_CONFIG, "attention impl must be 0, 1, 2 or 3");
  g_attn_impl = impl;
  return RP_OK;
}

// window kernels for N <= 64 (A/B switch): 0 the single-tile fused kernels
// (attn_fwd_win_kernel / attn_bwd_win_kernel), 1 the general mma.sync kernels
static int g_attn_win_variant = 0;
extern "C" int rp_set_attention_window_variant(int v) {
  if (v < 0 || v > 1) return rp_fail(RP_ERR_CONFIG, "attention window variant must be 0 or 1");
  g_attn_win_variant = v;
  return RP_OK;
}

// TMA staging for the window kernels: head_dim 32 (64-byte rows, SW64) or 64 (SW128)
static bool win_tma(int64_t hd) { return hd == 32 || hd == 64; }
static int win_maps(WinMaps* m, const uint16_t* qkv, const uint16_t* dout, int64_t B, int64_t N,
                    int64_t H, int64_t hd) {
  attn_tc::EncodeFn fn = attn_tc::encode_fn();
  if (!fn) return RP_ERR_CUDA;
  std::memset(m, 0, sizeof(*m));
  const CUtensorMapSwizzle sw = hd == 32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B;
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(hd), static_cast<cuuint32_t>(N)};
  const cuuint32_t es[2] = {1, 1};
  auto map2d = [&](CUtensorMap* t, const void* base, int64_t cols) {
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(B * N)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(cols) * 2};
    return static_cast<int>(fn(t, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base),
                               dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
  };
  char msg[96];
  int e;
  if ((e = map2d(&m->qkv, qkv, 3 * H * hd))) {
    std::snprintf(msg, sizeof(msg), "attention window: qkv tensor map (CUresult %d)", e);
    return rp_fail(RP_ERR_CUDA, msg);
  }
  if (dout && (e = map2d(&m->dout, dout, H * hd))) {
    std::snprintf(msg, sizeof(msg), "attention window: dout tensor map (CUresult %d)", e);
    return rp_fail(RP_ERR_CUDA, msg);
  }
  return RP_OK;
}

// persistent grid: items capped at SMs x resident CTAs of `fn` (cached per kernel)
static int64_t persistent_grid(const void* fn, int smem, int64_t items) {
  static std::mutex mu;
  static std::vector<std::pair<const void*, int>> cache;
  int occ = 0;
  {
    std::lock_guard<std::mutex> lk(mu);
    for (auto& e : cache)
      if (e.first == fn) occ = e.second;
    if (!occ) {
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, 128, smem);
      if (occ < 1) occ = 1;
      cache.emplace_back(fn, occ);
    }
  }
  int nsm = 148, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  return std::min<int64_t>(items, static_cast<int64_t>(nsm) * occ);
}

template <int HDP>
static int attn_fwd_mma(const uint16_t* qkv, int64_t B, int64_t N, int64_t H, int64_t hd,
                        uint16_t* out, float* lse, cudaStream_t stream) {
  const AttnGeom g = make_geom(B, N, H, hd);
  if (N <= kTile && g_attn_win_variant == 0) {
    const int smem = 1024 + 2 * 3 * kTile * HDP * 2;
    WinMaps maps;
    std::memset(&maps, 0, sizeof(maps));
    const bool tma = win_tma(hd);
    int rc;
    if (tma && (rc = win_maps(&maps, qkv, nullptr, B, N, H, hd))) return rc;
    auto go = [&](auto kernel) {
      const void* fn = reinterpret_cast<const void*>(kernel);
      int e = set_smem_attr(fn, smem);
      if (e) return e;
      const unsigned grid = static_cast<unsigned>(persistent_grid(fn, smem, B * H));
      launch_k(kernel, dim3(grid), dim3(128), smem, stream, maps,
               reinterpret_cast<const __nv_bfloat16*>(qkv),
               reinterpret_cast<__nv_bfloat16*>(out), lse, g);
      return 0;
    };
    if ((rc = !tma ? go(attn_fwd_win_kernel<HDP, false, 0>)
              : N == 49 ? go(attn_fwd_win_kernel<HDP, true, 49>)
                        : go(attn_fwd_win_kernel<HDP, true, 0>)))
      return rc;
    return rp_check_launch("attention_fwd_window");
  }
  if (N <= kTile && B * H >= 4 * 148) {  // many short windows: persistent, double-buffered
    const int smem = 2 * 3 * kTile * HDP * 2;
    int rc;
    if ((rc = set_smem_attr(reinterpret_cast<const void*>(attn_fwd_small_kernel<HDP>), smem)))
      return rc;
    static int per_sm[3] = {0, 0, 0};
    int& occ = per_sm[HDP == 32 ? 0 : HDP == 64 ? 1 : 2];
    if (!occ) {
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, attn_fwd_small_kernel<HDP>, 128, smem);
      if (occ < 1) occ = 1;
    }
    int nsm = 148, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const int64_t items = B * H;
    const int64_t grid = std::min<int64_t>(items, static_cast<int64_t>(nsm) * occ);
    launch_k(attn_fwd_small_kernel<HDP>, dim3(static_cast<unsigned>(grid)), dim3(128), smem,
             stream, reinterpret_cast<const __nv_bfloat16*>(qkv),
             reinterpret_cast<__nv_bfloat16*>(out), lse, g);
    return rp_check_launch("attention_fwd");
  }
  const int npad = static_cast<int>((N + kTile - 1) / kTile * kTile);
  const int smem = (kTile + 2 * npad) * HDP * 2;
  int rc;
  if ((rc = set_smem_attr(reinterpret_cast<const void*>(attn_fwd_kernel<HDP>), smem))) return rc;
  dim3 grid(static_cast<unsigned>((N + kTile - 1) / kTile), static_cast<unsigned>(H),
            static_cast<unsigned>(B));
  launch_k(attn_fwd_kernel<HDP>, grid, dim3(128), smem, stream,
           reinterpret_cast<const __nv_bfloat16*>(qkv), reinterpret_cast<__nv_bfloat16*>(out), lse,
           g);
  return rp_check_launch("attention_fwd");
}

extern "C" int rp_attention_fwd(const uint16_t* qkv, int64_t B, int64_t N, int64_t H,
                                int64_t head_dim, uint16_t* out, float* lse,
                                rp_stream_t stream) {
  int rc = attn_check(B, N, H, head_dim);
  if (rc) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (g_attn_impl != 1 && head_dim == 64 && N <= 512) {
    rc = rp_attention_fwd_tc(qkv, B, N, H, out, lse, s);
    if (rc != RP_ERR_CONFIG) return rc;
  }
  if (g_attn_impl != 1 && head_dim > 64 && N > kTile) {  // G48's 104: tcgen05 at N <= 256
    rc = rp_attention_fwd_tc_wide(qkv, B, N, H, head_dim, out, lse, s);
    if (rc != RP_ERR_CONFIG) return rc;
  }
  if (head_dim <= 32) return attn_fwd_mma<32>(qkv, B, N, H, head_dim, out, lse, s);
  return head_dim <= 64 ? attn_fwd_mma<64>(qkv, B, N, H, head_dim, out, lse, s)
                        : attn_fwd_mma<128>(qkv, B, N, H, head_dim, out, lse, s);
}

// D (B N H floats), then -- for the tcgen05 backward at N <= kFusedBwdMaxN -- dS^T of every
// (sequence, head) as bf16 [B H][Nk][Nk] (Nk = N rounded up to 16), 64-float aligned
constexpr int64_t kFusedBwdMaxN = 256;
static int64_t attn_ds_offset(int64_t B, int64_t N, int64_t H) { return (B * N * H + 63) / 64 * 64; }
extern "C" int64_t rp_attention_bwd_workspace_floats(int64_t B, int64_t N, int64_t H) {
  const int64_t nk = (N + 15) / 16 * 16;
  if (N > kFusedBwdMaxN) return B * N * H;
  return attn_ds_offset(B, N, H) + (B * H * nk * nk + 1) / 2;
}

template <int HDP>
static int attn_bwd_mma(const uint16_t* qkv, const uint16_t* out, const float* lse,
                        const uint16_t* dout, int64_t B, int64_t N, int64_t H, int64_t hd,
                        uint16_t* dqkv, float* workspace, cudaStream_t s) {
  const AttnGeom g = make_geom(B, N, H, hd);
  if (N <= kTile && g_attn_win_variant == 0) {
    const int smem = 1024 + 2 * 4 * kTile * HDP * 2 + 2 * kTile * 64 * 2;
    WinMaps maps;
    std::memset(&maps, 0, sizeof(maps));
    const bool tma = win_tma(hd);
    int rc;
    if (tma && (rc = win_maps(&maps, qkv, dout, B, N, H, hd))) return rc;
    auto go = [&](auto kernel) {
      const void* fn = reinterpret_cast<const void*>(kernel);
      int e = set_smem_attr(fn, smem);
      if (e) return e;
      const unsigned grid = static_cast<unsigned>(persistent_grid(fn, smem, B * H));
      launch_k(kernel, dim3(grid), dim3(128), smem, s, maps,
               reinterpret_cast<const __nv_bfloat16*>(qkv),
               reinterpret_cast<const __nv_bfloat16*>(dout), lse,
               reinterpret_cast<__nv_bfloat16*>(dqkv), g);
      return 0;
    };
    if ((rc = !tma ? go(attn_bwd_win_kernel<HDP, false, 0>)
              : N == 49 ? go(attn_bwd_win_kernel<HDP, true, 49>)
                        : go(attn_bwd_win_kernel<HDP, true, 0>)))
      return rc;
    return rp_check_launch("attention_bwd_window");
  }
  const int64_t total = B * N * H;
  int blocks = static_cast<int>((total + 255) / 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  launch_k(attn_bwd_dot_kernel, dim3(blocks), dim3(256), 0, s,
           reinterpret_cast<const __nv_bfloat16*>(out),
           reinterpret_cast<const __nv_bfloat16*>(dout), workspace, g);
  const int npad = static_cast<int>((N + kTile - 1) / kTile * kTile);
  const int rb = HDP * 2;
  const int smem_kv = 2 * kTile * rb + 2 * npad * rb + 2 * npad * 4;
  const int smem_q = 2 * kTile * rb + 2 * npad * rb;
  int rc;
  if ((rc = set_smem_attr(reinterpret_cast<const void*>(attn_bwd_dkdv_kernel<HDP>), smem_kv)))
    return rc;
  if ((rc = set_smem_attr(reinterpret_cast<const void*>(attn_bwd_dq_kernel<HDP>), smem_q)))
    return rc;
  dim3 grid(static_cast<unsigned>((N + kTile - 1) / kTile), static_cast<unsigned>(H),
            static_cast<unsigned>(B));
  launch_k(attn_bwd_dkdv_kernel<HDP>, dim3(grid), dim3(128), smem_kv, s,
           reinterpret_cast<const __nv_bfloat16*>(qkv), reinterpret_cast<const __nv_bfloat16*>(dout),
           lse, workspace, reinterpret_cast<__nv_bfloat16*>(dqkv), g);
  launch_k(attn_bwd_dq_kernel<HDP>, dim3(grid), dim3(128), smem_q, s,
           reinterpret_cast<const __nv_bfloat16*>(qkv), reinterpret_cast<const __nv_bfloat16*>(dout),
           lse, workspace, reinterpret_cast<__nv_bfloat16*>(dqkv), g);
  return rp_check_launch("attention_bwd");
}

// d_out [B*N, H*hd] -> d_qkv [B*N, 3*H*hd]; workspace: B*N*H floats.
extern "C" int rp_attention_bwd_ex(const uint16_t* qkv, const uint16_t* out, const float* lse,
                                   const uint16_t* dout, int64_t B, int64_t N, int64_t H,
                                   int64_t head_dim, uint16_t* dqkv, float* workspace,
                                   int d_ready, rp_stream_t stream) {
  int rc = attn_check(B, N, H, head_dim);
  if (rc) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (g_attn_impl != 1 && head_dim == 64) {  // tcgen05 path computes D itself
    // dS^T storage pays off while it is small next to the dQ pass it replaces (measured:
    // 495 -> 450 us at N = 197, a loss at N = 512)
    uint16_t* dst = (g_attn_impl == 0 || g_attn_impl == 3) && N <= kFusedBwdMaxN
                        ? reinterpret_cast<uint16_t*>(workspace + attn_ds_offset(B, N, H))
                        : nullptr;
    rc = rp_attention_bwd_tc(qkv, out, dout, lse, workspace, B, N, H, dqkv, s, dst, d_ready,
                             g_attn_impl == 0);
    if (rc != RP_ERR_CONFIG) return rc;
  }
  // head dims 72..128 (G48's 104) above the window range: two-pass tcgen05, D in-kernel
  if (g_attn_impl != 1 && head_dim > 64 && N > kTile) {
    rc = rp_attention_bwd_tc_wide(qkv, out, dout, lse, workspace, B, N, H, head_dim, dqkv, s);
    if (rc != RP_ERR_CONFIG) return rc;
  }
  if (head_dim <= 32)
    return attn_bwd_mma<32>(qkv, out, lse, dout, B, N, H, head_dim, dqkv, workspace, s);
  return head_dim <= 64
             ? attn_bwd_mma<64>(qkv, out, lse, dout, B, N, H, head_dim, dqkv, workspace, s)
             : attn_bwd_mma<128>(qkv, out, lse, dout, B, N, H, head_dim, dqkv, workspace, s);
}

// d_out [B*N, H*hd] -> d_qkv [B*N, 3*H*hd]; workspace: rp_attention_bwd_workspace_floats.
extern "C" int rp_attention_bwd(const uint16_t* qkv, const uint16_t* out, const float* lse,
                                const uint16_t* dout, int64_t B, int64_t N, int64_t H,
                                int64_t head_dim, uint16_t* dqkv, float* workspace,
                                rp_stream_t stream) {
  return rp_attention_bwd_ex(qkv, out, lse, dout, B, N, H, head_dim, dqkv, workspace, 0, stream);
}
