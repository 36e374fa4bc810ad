// LayerNorm forward / backward and deterministic column reductions (HBM-bound kernels).
//
// Forward follows ref:proj/core/src/ops.cpp:264-304 (two-pass mean, population variance,
// inv_std = 1/sqrt(var + eps), y = x_hat*gamma + beta) but keeps (mean, rstd) per row
// instead of materialising x_hat: x_hat is recomputed from the fp32 residual stream in
// the backward, which saves a [T,d] write+read per LayerNorm.
// Backward follows ref:proj/core/src/ops.cpp:306-345
//   g = dy*gamma; dx = (g - mean(g) - x_hat*mean(g*x_hat)) * inv_std
//   dgamma = sum_rows dy*x_hat, dbeta = sum_rows dy
// with the reversible coupling's cotangent add fused in (dx_total = dres + dx,
// SPEC.md:234) and a bf16 copy of dx_total emitted for the next GEMM.
// All reductions have a fixed association order that depends only on the problem shape,
// never on the launch or stream co-residency, so results are bit-reproducible.
#include <mutex>

#include "../../include/revprop_b200.h"
#include "kernels.h"
#include "ptx.cuh"
#include "launch.h"

namespace rp {

constexpr int kLnWarps = 8;        // rows per CTA in the forward
// Rows per dgamma / dbeta partial. Wide rows (the single-pass backward's per-CTA shared
// memory, 8 warps x 3 x cols floats, leaves one or two CTAs per SM) and narrow rows (eight
// CTAs per SM): the partials make exactly one wave on 148 SMs (a fixed 64 left G48, 12.6k rows
// x 1664 columns at 160 KB per CTA, with 197 partials = 1.33 waves: 132 -> 100 us; RevViT-L
// 181 -> 171 us; Rev-Swin-B stage 1, 401k x 128: 182 -> 172 us). In between (three to seven
// CTAs per SM) the short CTAs of a fixed 64 rows balance better (RevViT-B: 133 us vs 149 us
// one-wave). Multiples of the 8 row warps; set by (rows, cols) alone, so results do not
// depend on the device.
static int64_t ln_bwd_rows_per_part(int64_t rows, int64_t cols) {
  const int64_t smem = static_cast<int64_t>(kLnWarps) * 3 * cols * 4;
  int64_t per_sm = (227 * 1024) / (smem > 0 ? smem : 1);
  if (per_sm > 2 && per_sm < 8) return 64;
  per_sm = per_sm < 1 ? 1 : (per_sm > 8 ? 8 : per_sm);
  const int64_t slots = 148 * per_sm;
  int64_t rpp = (rows + slots - 1) / slots;
  rpp = (rpp + kLnWarps - 1) / kLnWarps * kLnWarps;
  return rpp < kLnWarps ? kLnWarps : rpp;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// One warp per row; lane l owns float4 columns {l, l+32, ...}.
template <int V>
__global__ void __launch_bounds__(kLnWarps * 32)
    ln_fwd_kernel(const float* __restrict__ x, const float* __restrict__ gamma,
                  const float* __restrict__ beta, int64_t rows, int cols, float eps,
                  __nv_bfloat16* __restrict__ y, float* __restrict__ mean_out,
                  float* __restrict__ rstd_out) {
  pdl_trigger();
  pdl_wait();

  const int lane = threadIdx.x & 31;
  const int64_t row = static_cast<int64_t>(blockIdx.x) * kLnWarps + (threadIdx.x >> 5);
  if (row >= rows) return;
  const int c4 = cols >> 2;
  const float4* xr = reinterpret_cast<const float4*>(x + row * cols);
  float4 v[V];
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < V; ++i) {
    const int c = lane + 32 * i;
    v[i] = c < c4 ? xr[c] : make_float4(0.f, 0.f, 0.f, 0.f);
    s += (v[i].x + v[i].y) + (v[i].z + v[i].w);
  }
  const float mean = warp_sum(s) / static_cast<float>(cols);
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < V; ++i) {
    const int c = lane + 32 * i;
    if (c < c4) {
      const float a = v[i].x - mean, b = v[i].y - mean, cc = v[i].z - mean, d = v[i].w - mean;
      q += (a * a + b * b) + (cc * cc + d * d);
    }
  }
  const float var = warp_sum(q) / static_cast<float>(cols);
  const float rstd = 1.0f / sqrtf(var + eps);
  uint2* yr = reinterpret_cast<uint2*>(y + row * cols);
  const float4* g4 = reinterpret_cast<const float4*>(gamma);
  const float4* b4 = reinterpret_cast<const float4*>(beta);
#pragma unroll
  for (int i = 0; i < V; ++i) {
    const int c = lane + 32 * i;
    if (c < c4) {
      const float4 g = g4[c], b = b4[c];
      const float o0 = (v[i].x - mean) * rstd * g.x + b.x;
      const float o1 = (v[i].y - mean) * rstd * g.y + b.y;
      const float o2 = (v[i].z - mean) * rstd * g.z + b.z;
      const float o3 = (v[i].w - mean) * rstd * g.w + b.w;
      yr[c] = make_uint2(pack_bf16x2(o0, o1), pack_bf16x2(o2, o3));
    }
  }
  if (lane == 0) {
    mean_out[row] = mean;
    rstd_out[row] = rstd;
  }
}

// Backward, row part: one warp per row, all loads issued before the reductions, no
// column accumulators (keeps ~60 registers -> full occupancy; the kernel is HBM-bound).
template <int V>
__global__ void __launch_bounds__(kLnWarps * 32)
    ln_bwd_dx_kernel(const float* __restrict__ x, const float* __restrict__ mean_in,
                     const float* __restrict__ rstd_in, const float* __restrict__ gamma,
                     const __nv_bfloat16* __restrict__ dy, const float* dres, int64_t rows,
                     int cols, float* dx, __nv_bfloat16* __restrict__ dx_bf16) {
  pdl_trigger();
  pdl_wait();

  const int lane = threadIdx.x & 31;
  const int64_t row = static_cast<int64_t>(blockIdx.x) * kLnWarps + (threadIdx.x >> 5);
  if (row >= rows) return;
  const int c4 = cols >> 2;
  const float4* g4 = reinterpret_cast<const float4*>(gamma);
  const float4* xr = reinterpret_cast<const float4*>(x + row * cols);
  const uint2* dyr = reinterpret_cast<const uint2*>(dy + row * cols);
  const float4* drr = dres ? reinterpret_cast<const float4*>(dres + row * cols) : nullptr;
  float4 xv[V], rv[V];
  uint2 dv[V];
#pragma unroll
  for (int i = 0; i < V; ++i) {
    const int c = lane + 32 * i;
    if (c < c4) {
      xv[i] = xr[c];
      dv[i] = dyr[c];
      rv[i] = drr ? drr[c] : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
  const float mean = mean_in[row], rstd = rstd_in[row];
  float sg = 0.f, sgh = 0.f;
  float4 h[V], g[V];
#pragma unroll
  for (int i = 0; i < V; ++i) {
    const int c = lane + 32 * i;
    if (c < c4) {
      const float2 d01 = unpack_bf16x2(dv[i].x), d23 = unpack_bf16x2(dv[i].y);
      const float4 gm = g4[c];
      h[i] = make_float4((xv[i].x - mean) * rstd, (xv[i].y - mean) * rstd,
                         (xv[i].z - mean) * rstd, (xv[i].w - mean) * rstd);
      g[i] = make_float4(d01.x * gm.x, d01.y * gm.y, d23.x * gm.z, d23.y * gm.w);
      sg += (g[i].x + g[i].y) + (g[i].z + g[i].w);
      sgh += (g[i].x * h[i].x + g[i].y * h[i].y) + (g[i].z * h[i].z + g[i].w * h[i].w);
    }
  }
  const float inv_n = 1.0f / static_cast<float>(cols);
  const float gm = warp_sum(sg) * inv_n;
  const float ghm = warp_sum(sgh) * inv_n;
  float4* dxr = reinterpret_cast<float4*>(dx + row * cols);
  uint2* dxb = dx_bf16 ? reinterpret_cast<uint2*>(dx_bf16 + row * cols) : nullptr;
#pragma unroll
  for (int i = 0; i < V; ++i) {
    const int c = lane + 32 * i;
    if (c < c4) {
      float4 o;
      o.x = (g[i].x - gm - h[i].x * ghm) * rstd + rv[i].x;
      o.y = (g[i].y - gm - h[i].y * ghm) * rstd + rv[i].y;
      o.z = (g[i].z - gm - h[i].z * ghm) * rstd + rv[i].z;
      o.w = (g[i].w - gm - h[i].w * ghm) * rstd + rv[i].w;
      dxr[c] = o;
      if (dxb) dxb[c] = make_uint2(pack_bf16x2(o.x, o.y), pack_bf16x2(o.z, o.w));
    }
  }
}

// Backward, single pass: dx (and its bf16 copy) plus the column sums dgamma = sum dy*x_hat,
// dbeta = sum dy and, optionally, sum dx (the next block's MLP output-bias gradient, which
// is the column sum of exactly this cotangent). One warp per row, all loads issued before
// the row reductions; each warp accumulates its rows' column sums in its own shared-memory
// rows (read-modify-write, the warp's rows in order), and the CTA combines its 8 warps in
// warp order -> part[blk][NACC][cols]. Fixed association order, no atomics, one read of x,
// dy and dres.
// RPP: rows per partial when fixed at compile time (64: the row loop unrolls, which narrow
// rows need for loads in flight), 0 = the runtime `rpp`
template <int V, int NACC, int RPP = 64>
__global__ void __launch_bounds__(kLnWarps * 32)
    ln_bwd_1pass_kernel(const float* __restrict__ x, const float* __restrict__ mean_in,
                        const float* __restrict__ rstd_in, const float* __restrict__ gamma,
                        const __nv_bfloat16* __restrict__ dy, const float* dres, int64_t rows,
                        int cols, int rpp, float* dx, __nv_bfloat16* __restrict__ dx_bf16,
                        float* __restrict__ part) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ float4 acc4[];  // [warp][NACC][cols/4]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c4 = cols >> 2;
  float4* my = acc4 + static_cast<int64_t>(warp) * NACC * c4;
  for (int i = lane; i < NACC * c4; i += 32) my[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  __syncwarp();  // when cols/4 is not a multiple of 32, another lane zeroed this lane's slots
  const float4* g4 = reinterpret_cast<const float4*>(gamma);
  const float inv_n = 1.0f / static_cast<float>(cols);
  if (RPP) rpp = RPP;
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * rpp;
  for (int rr = warp; rr < rpp; rr += kLnWarps) {
    const int64_t row = r0 + rr;
    if (row >= rows) break;
    const float4* xr = reinterpret_cast<const float4*>(x + row * cols);
    const uint2* dyr = reinterpret_cast<const uint2*>(dy + row * cols);
    const float4* drr = dres ? reinterpret_cast<const float4*>(dres + row * cols) : nullptr;
    float4 xv[V], rv[V];
    uint2 dv[V];
#pragma unroll
    for (int i = 0; i < V; ++i) {
      const int c = lane + 32 * i;
      if (c < c4) {
        xv[i] = xr[c];
        dv[i] = dyr[c];
        rv[i] = drr ? drr[c] : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
    const float mean = mean_in[row], rstd = rstd_in[row];
    float sg = 0.f, sgh = 0.f;
#pragma unroll
    for (int i = 0; i < V; ++i) {
      const int c = lane + 32 * i;
      if (c < c4) {
        const float2 d01 = unpack_bf16x2(dv[i].x), d23 = unpack_bf16x2(dv[i].y);
        const float4 gm = g4[c];
        xv[i] = make_float4((xv[i].x - mean) * rstd, (xv[i].y - mean) * rstd,
                            (xv[i].z - mean) * rstd, (xv[i].w - mean) * rstd);  // x_hat
        const float gx = d01.x * gm.x, gy = d01.y * gm.y, gz = d23.x * gm.z, gw = d23.y * gm.w;
        sg += (gx + gy) + (gz + gw);
        sgh += (gx * xv[i].x + gy * xv[i].y) + (gz * xv[i].z + gw * xv[i].w);
      }
    }
    const float gmn = warp_sum(sg) * inv_n;
    const float ghm = warp_sum(sgh) * inv_n;
    float4* dxr = reinterpret_cast<float4*>(dx + row * cols);
    uint2* dxb = dx_bf16 ? reinterpret_cast<uint2*>(dx_bf16 + row * cols) : nullptr;
#pragma unroll
    for (int i = 0; i < V; ++i) {
      const int c = lane + 32 * i;
      if (c < c4) {
        const float2 d01 = unpack_bf16x2(dv[i].x), d23 = unpack_bf16x2(dv[i].y);
        const float4 gm = g4[c];
        const float4 h = xv[i];
        float4 o;
        o.x = (d01.x * gm.x - gmn - h.x * ghm) * rstd + rv[i].x;
        o.y = (d01.y * gm.y - gmn - h.y * ghm) * rstd + rv[i].y;
        o.z = (d23.x * gm.z - gmn - h.z * ghm) * rstd + rv[i].z;
        o.w = (d23.y * gm.w - gmn - h.w * ghm) * rstd + rv[i].w;
        dxr[c] = o;
        if (dxb) dxb[c] = make_uint2(pack_bf16x2(o.x, o.y), pack_bf16x2(o.z, o.w));
        float4 a = my[c];
        a.x += d01.x * h.x; a.y += d01.y * h.y; a.z += d23.x * h.z; a.w += d23.y * h.w;
        my[c] = a;
        float4 bb = my[c4 + c];
        bb.x += d01.x; bb.y += d01.y; bb.z += d23.x; bb.w += d23.y;
        my[c4 + c] = bb;
        if constexpr (NACC == 3) {
          float4 cc = my[2 * c4 + c];
          cc.x += o.x; cc.y += o.y; cc.z += o.z; cc.w += o.w;
          my[2 * c4 + c] = cc;
        }
      }
    }
  }
  __syncthreads();
  // combine the warps' rows in warp order
  float4* out = reinterpret_cast<float4*>(part + static_cast<int64_t>(blockIdx.x) * NACC * cols);
  for (int i = threadIdx.x; i < NACC * c4; i += blockDim.x) {
    float4 t = acc4[i];
    for (int w = 1; w < kLnWarps; ++w) {
      const float4 u = acc4[static_cast<int64_t>(w) * NACC * c4 + i];
      t.x += u.x; t.y += u.y; t.z += u.z; t.w += u.w;
    }
    out[i] = t;
  }
}

// Backward, column part (stage 1): CTA (rb, cb) sums dgamma = dy*x_hat and dbeta = dy
// over rows [rb*RPB, (rb+1)*RPB) in row order for 4*256 columns -> part[rb][2][cols].
__global__ void __launch_bounds__(256)
    ln_bwd_dgb_partial_kernel(const float* __restrict__ x, const float* __restrict__ mean_in,
                              const float* __restrict__ rstd_in,
                              const __nv_bfloat16* __restrict__ dy, int64_t rows, int cols,
                              int rpb, float* __restrict__ part) {
  pdl_trigger();
  pdl_wait();

  const int c = (blockIdx.y * 256 + threadIdx.x) * 4;
  if (c >= cols) return;
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * rpb;
  int64_t r1 = r0 + rpb;
  if (r1 > rows) r1 = rows;
  float4 ag = make_float4(0.f, 0.f, 0.f, 0.f), ab = ag;
  // rows in order; 4 rows' loads in flight per iteration (same association order)
  int64_t r = r0;
  for (; r + 4 <= r1; r += 4) {
    float4 xv[4];
    uint2 dv[4];
    float m[4], s[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      xv[j] = *reinterpret_cast<const float4*>(x + (r + j) * cols + c);
      dv[j] = *reinterpret_cast<const uint2*>(dy + (r + j) * cols + c);
      m[j] = mean_in[r + j];
      s[j] = rstd_in[r + j];
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 d01 = unpack_bf16x2(dv[j].x), d23 = unpack_bf16x2(dv[j].y);
      ag.x += d01.x * ((xv[j].x - m[j]) * s[j]);
      ag.y += d01.y * ((xv[j].y - m[j]) * s[j]);
      ag.z += d23.x * ((xv[j].z - m[j]) * s[j]);
      ag.w += d23.y * ((xv[j].w - m[j]) * s[j]);
      ab.x += d01.x;
      ab.y += d01.y;
      ab.z += d23.x;
      ab.w += d23.y;
    }
  }
  for (; r < r1; ++r) {
    const float4 xv = *reinterpret_cast<const float4*>(x + r * cols + c);
    const uint2 dv = *reinterpret_cast<const uint2*>(dy + r * cols + c);
    const float m = mean_in[r], s = rstd_in[r];
    const float2 d01 = unpack_bf16x2(dv.x), d23 = unpack_bf16x2(dv.y);
    ag.x += d01.x * ((xv.x - m) * s);
    ag.y += d01.y * ((xv.y - m) * s);
    ag.z += d23.x * ((xv.z - m) * s);
    ag.w += d23.y * ((xv.w - m) * s);
    ab.x += d01.x;
    ab.y += d01.y;
    ab.z += d23.x;
    ab.w += d23.y;
  }
  float* p = part + static_cast<int64_t>(blockIdx.x) * 2 * cols;
  *reinterpret_cast<float4*>(p + c) = ag;
  *reinterpret_cast<float4*>(p + cols + c) = ab;
}

// Stage 1 of a deterministic column sum over a [rows, cols] matrix (fp32 or bf16):
// CTA (rb, cb) sums rows [rb*RPB, (rb+1)*RPB) for 4*256 columns, sequentially in row order.
template <typename T>
__global__ void __launch_bounds__(256)
    colsum_partial_kernel(const T* __restrict__ in, int64_t rows, int cols, int rpb,
                          float* __restrict__ part) {
  pdl_trigger();
  pdl_wait();

  const int c = (blockIdx.y * 256 + threadIdx.x) * 4;
  if (c >= cols) return;
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * rpb;
  int64_t r1 = r0 + rpb;
  if (r1 > rows) r1 = rows;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int64_t r = r0; r < r1; ++r) {
    float4 v;
    if constexpr (sizeof(T) == 4) {
      v = *reinterpret_cast<const float4*>(reinterpret_cast<const float*>(in) + r * cols + c);
    } else {
      const uint2 u = *reinterpret_cast<const uint2*>(
          reinterpret_cast<const __nv_bfloat16*>(in) + r * cols + c);
      const float2 a = unpack_bf16x2(u.x), b = unpack_bf16x2(u.y);
      v = make_float4(a.x, a.y, b.x, b.y);
    }
    acc.x += v.x;
    acc.y += v.y;
    acc.z += v.z;
    acc.w += v.w;
  }
  *reinterpret_cast<float4*>(part + static_cast<int64_t>(blockIdx.x) * cols + c) = acc;
}

// Stage 2: out[c] (+)= sum_p part[p][c] in a fixed order. CTA = 32 warps x 32 columns;
// warp w owns parts {w, w+32, ...} with 2 interleaved accumulators; combined in order.
// (8 accumulators measured slower: the compiler reuses the load registers and serialises.)
constexpr int kFinWarps = 32;
__global__ void __launch_bounds__(kFinWarps * 32)
    colsum_final_kernel(const float* __restrict__ part, int64_t nparts, int cols, int64_t ld,
                        float* __restrict__ out, int accumulate) {
  pdl_trigger();
  pdl_wait();

  __shared__ float red[kFinWarps][33];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + lane;
  float a0 = 0.f, a1 = 0.f;
  if (c < cols) {
    int64_t p = warp;
    for (; p + kFinWarps < nparts; p += 2 * kFinWarps) {
      a0 += part[p * ld + c];
      a1 += part[(p + kFinWarps) * ld + c];
    }
    for (; p < nparts; p += kFinWarps) a0 += part[p * ld + c];
  }
  red[warp][lane] = a0 + a1;
  __syncthreads();
  if (warp == 0 && c < cols) {
    float s = red[0][lane];
    for (int w = 1; w < kFinWarps; ++w) s += red[w][lane];
    out[c] = accumulate ? out[c] + s : s;
  }
}

// Column sums over many parts in ONE launch: a cluster of kClu CTAs per 32 columns, CTA r of
// the cluster summing the r-th contiguous slice of the parts (16 warps, each warp every 16th
// part of the slice, 8 loads in flight), then the leader CTA adding the kClu slice sums from
// the other CTAs' shared memory in rank order. The association order depends only on
// (nparts, cols), so results are bit-reproducible. Replaces a slice-sum launch writing the
// slice sums back to global + a finalising launch (two launches and a dependent global round
// trip per reduction; 8.5 us -> see DESIGN.md section 9).
constexpr int kClu = 8;
constexpr int kCluWarps = 16;
__global__ void __cluster_dims__(1, kClu, 1) __launch_bounds__(kCluWarps * 32)
    colsum_cluster_kernel(const float* __restrict__ part, int64_t nparts, int cols, int64_t ld,
                          float* __restrict__ out, int accumulate) {
  pdl_trigger();
  pdl_wait();

  __shared__ float red[kCluWarps][33];
  __shared__ float slice_sum[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + lane;
  const uint32_t rank = cluster_ctarank();
  const int64_t per = (nparts + kClu - 1) / kClu;
  const int64_t p_end = min(nparts, (rank + 1) * per);
  float a0 = 0.f, a1 = 0.f;
  if (c < cols) {
    int64_t p = rank * per + warp;
    for (; p + 7 * kCluWarps < p_end; p += 8 * kCluWarps) {
      float v[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = __ldcg(part + (p + i * kCluWarps) * ld + c);
      a0 += (v[0] + v[2]) + (v[4] + v[6]);
      a1 += (v[1] + v[3]) + (v[5] + v[7]);
    }
    for (; p < p_end; p += kCluWarps) a0 += __ldcg(part + p * ld + c);
  }
  red[warp][lane] = a0 + a1;
  __syncthreads();
  if (warp == 0) {
    float t = red[0][lane];
#pragma unroll
    for (int w = 1; w < kCluWarps; ++w) t += red[w][lane];
    slice_sum[lane] = t;
  }
  cluster_sync_all();
  if (rank == 0 && warp == 0 && c < cols) {
    const uint32_t local = smem_u32(&slice_sum[lane]);
    float s = 0.f;
#pragma unroll
    for (uint32_t r = 0; r < kClu; ++r) {
      float v;
      asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(mapa_shared(local, r)) : "memory");
      s += v;
    }
    out[c] = accumulate ? out[c] + s : s;
  }
  cluster_sync_all();  // the leader's remote reads complete before any CTA exits
}

static void colsum_final(cudaStream_t s, float* part, int64_t nparts, int cols, int64_t ld,
                         float* out, int accumulate) {
  const unsigned gb = static_cast<unsigned>((cols + 31) / 32);
  if (nparts > 2 * kClu * kCluWarps) {
    launch_k(colsum_cluster_kernel, dim3(gb, kClu), dim3(kCluWarps * 32), 0, s,
             static_cast<const float*>(part), nparts, cols, ld, out, accumulate);
    return;
  }
  launch_k(colsum_final_kernel, dim3(gb), dim3(kFinWarps * 32), 0, s, part, nparts, cols, ld, out,
           accumulate);
}

template <int V>
static void launch_ln_fwd(const float* x, const float* g, const float* b, int64_t rows,
                          int cols, float eps, __nv_bfloat16* y, float* mean, float* rstd,
                          cudaStream_t s) {
  const int64_t blocks = (rows + kLnWarps - 1) / kLnWarps;
  launch_k(ln_fwd_kernel<V>, dim3(static_cast<unsigned>(blocks)), dim3(kLnWarps * 32), 0, s, x, g, b, rows, cols,
                                                                           eps, y, mean, rstd);
}

template <int V>
static void launch_ln_bwd_1pass(const float* x, const float* mean, const float* rstd,
                                const float* gamma, const __nv_bfloat16* dy, const float* dres,
                                int64_t rows, int cols, float* dx, __nv_bfloat16* dxb,
                                float* part, int nacc, cudaStream_t s) {
  const int64_t rpp = ln_bwd_rows_per_part(rows, cols);
  const int64_t blocks = (rows + rpp - 1) / rpp;
  const int smem = kLnWarps * nacc * cols * static_cast<int>(sizeof(float));
  static std::once_flag once;  // (the four instantiations share one function-pointer type)
  std::call_once(once, [] {
    constexpr int a3 = kLnWarps * 3 * 2048 * 4, a2 = kLnWarps * 2 * 2048 * 4;
    cudaFuncSetAttribute(ln_bwd_1pass_kernel<V, 3, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize, a3);
    cudaFuncSetAttribute(ln_bwd_1pass_kernel<V, 3, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, a3);
    cudaFuncSetAttribute(ln_bwd_1pass_kernel<V, 2, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize, a2);
    cudaFuncSetAttribute(ln_bwd_1pass_kernel<V, 2, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, a2);
  });
  auto go = [&](auto kernel, int) {
    launch_k(kernel, dim3(static_cast<unsigned>(blocks)), dim3(kLnWarps * 32), smem, s, x, mean,
             rstd, gamma, dy, dres, rows, cols, static_cast<int>(rpp), dx, dxb, part);
  };
  if (nacc == 3)
    rpp == 64 ? go(ln_bwd_1pass_kernel<V, 3, 64>, 3) : go(ln_bwd_1pass_kernel<V, 3, 0>, 3);
  else
    rpp == 64 ? go(ln_bwd_1pass_kernel<V, 2, 64>, 2) : go(ln_bwd_1pass_kernel<V, 2, 0>, 2);
}

template <int V>
static void launch_ln_bwd(const float* x, const float* mean, const float* rstd,
                          const float* gamma, const __nv_bfloat16* dy, const float* dres,
                          int64_t rows, int cols, float* dx, __nv_bfloat16* dxb, cudaStream_t s) {
  const int64_t blocks = (rows + kLnWarps - 1) / kLnWarps;
  launch_k(ln_bwd_dx_kernel<V>, dim3(static_cast<unsigned>(blocks)), dim3(kLnWarps * 32), 0, s, 
      x, mean, rstd, gamma, dy, dres, rows, cols, dx, dxb);
}

}  // namespace rp

using namespace rp;

int64_t rp_ln_bwd_num_parts(int64_t rows, int64_t cols) {
  const int64_t rpp = ln_bwd_rows_per_part(rows, cols);
  return (rows + rpp - 1) / rpp;
}

#define RP_LN_DISPATCH(FN, ...)                      \
  do {                                               \
    const int v = (cols / 4 + 31) / 32;              \
    if (v <= 2)                                      \
      FN<2>(__VA_ARGS__);                            \
    else if (v <= 4)                                 \
      FN<4>(__VA_ARGS__);                            \
    else if (v <= 6)                                 \
      FN<6>(__VA_ARGS__);                            \
    else if (v <= 8)                                 \
      FN<8>(__VA_ARGS__);                            \
    else if (v <= 13)                                \
      FN<13>(__VA_ARGS__);                           \
    else if (v <= 16)                                \
      FN<16>(__VA_ARGS__);                           \
    else                                             \
      return rp_fail(RP_ERR_SHAPE, "layer_norm: width > 2048 unsupported"); \
  } while (0)

extern "C" int rp_layer_norm_fwd(const float* x, const float* gamma, const float* beta,
                                 int64_t rows, int64_t cols, double eps, uint16_t* y,
                                 float* mean, float* rstd, rp_stream_t stream) {
  if (rows <= 0 || cols <= 0 || cols % 4) return rp_fail(RP_ERR_SHAPE, "layer_norm: cols % 4");
  if (!(eps > 0.0)) return rp_fail(RP_ERR_SHAPE, "layer_norm: eps must be positive");
  RP_LN_DISPATCH(launch_ln_fwd, x, gamma, beta, rows, static_cast<int>(cols),
                 static_cast<float>(eps), reinterpret_cast<__nv_bfloat16*>(y), mean, rstd,
                 static_cast<cudaStream_t>(stream));
  return rp_check_launch("layer_norm_fwd");
}

static int g_ln_bwd_impl = 1;  // 1 = single pass (fused column sums), 0 = row kernel + column kernels

extern "C" int rp_set_ln_bwd_impl(int impl) {
  g_ln_bwd_impl = impl;
  return RP_OK;
}

extern "C" int rp_layer_norm_bwd_ex(const float* x, const float* mean, const float* rstd,
                                    const float* gamma, const uint16_t* dy, const float* dres,
                                    int64_t rows, int64_t cols, float* dx, uint16_t* dx_bf16,
                                    float* dgamma, float* dbeta, float* dx_colsum,
                                    float* workspace, int accumulate, rp_stream_t stream) {
  if (rows <= 0 || cols <= 0 || cols % 4) return rp_fail(RP_ERR_SHAPE, "layer_norm_vjp: cols % 4");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const __nv_bfloat16* dyb = reinterpret_cast<const __nv_bfloat16*>(dy);
  const int64_t nparts = rp_ln_bwd_num_parts(rows, cols);
  const unsigned gb = static_cast<unsigned>((cols + 31) / 32);
  if ((dgamma || dbeta || dx_colsum) && (g_ln_bwd_impl == 1 || dx_colsum) && cols <= 2048) {
    const int nacc = dx_colsum ? 3 : 2;
    RP_LN_DISPATCH(launch_ln_bwd_1pass, x, mean, rstd, gamma, dyb, dres, rows,
                   static_cast<int>(cols), dx, reinterpret_cast<__nv_bfloat16*>(dx_bf16),
                   workspace, nacc, s);
    const int64_t ld = nacc * cols;
    if (dgamma && dbeta == dgamma + cols) {
      colsum_final(s, workspace, nparts, static_cast<int>(2 * cols), ld, dgamma, accumulate);
    } else {
      if (dgamma)
        colsum_final(s, workspace, nparts, static_cast<int>(cols), ld, dgamma, accumulate);
      if (dbeta)
        colsum_final(s, workspace + cols, nparts, static_cast<int>(cols), ld, dbeta, accumulate);
    }
    if (dx_colsum)
      colsum_final(s, workspace + 2 * cols, nparts, static_cast<int>(cols), ld, dx_colsum, 0);
    return rp_check_launch("layer_norm_bwd");
  }
  if (dgamma || dbeta) {  // column partials first (reads x, dy before dx may alias dres)
    dim3 grid(static_cast<unsigned>(nparts), static_cast<unsigned>((cols / 4 + 255) / 256));
    launch_k(ln_bwd_dgb_partial_kernel, grid, dim3(256), 0, s, x, mean, rstd, dyb, rows,
             static_cast<int>(cols), static_cast<int>(ln_bwd_rows_per_part(rows, cols)), workspace);
    if (dgamma && dbeta == dgamma + cols) {  // adjacent in the flat grad buffer: one launch
      colsum_final(s, workspace, nparts, static_cast<int>(2 * cols), 2 * cols, dgamma, accumulate);
    } else {
      if (dgamma)
        colsum_final(s, workspace, nparts, static_cast<int>(cols), 2 * cols, dgamma, accumulate);
      if (dbeta)
        colsum_final(s, workspace + cols, nparts, static_cast<int>(cols), 2 * cols, dbeta,
                     accumulate);
    }
  }
  RP_LN_DISPATCH(launch_ln_bwd, x, mean, rstd, gamma, dyb, dres, rows, static_cast<int>(cols), dx,
                 reinterpret_cast<__nv_bfloat16*>(dx_bf16), s);
  return rp_check_launch("layer_norm_bwd");
}

extern "C" int rp_layer_norm_bwd(const float* x, const float* mean, const float* rstd,
                                 const float* gamma, const uint16_t* dy, const float* dres,
                                 int64_t rows, int64_t cols, float* dx, uint16_t* dx_bf16,
                                 float* dgamma, float* dbeta, float* workspace,
                                 int accumulate, rp_stream_t stream) {
  return rp_layer_norm_bwd_ex(x, mean, rstd, gamma, dy, dres, rows, cols, dx, dx_bf16, dgamma,
                              dbeta, nullptr, workspace, accumulate, stream);
}

extern "C" int64_t rp_layer_norm_bwd_workspace_floats(int64_t rows, int64_t cols) {
  return rp_ln_bwd_num_parts(rows, cols) * 3 * cols;
}

extern "C" int rp_colsum_parts(float* part, int64_t nparts, int64_t cols, float* out,
                               int accumulate, rp_stream_t stream) {
  if (nparts <= 0 || cols <= 0) return rp_fail(RP_ERR_SHAPE, "colsum_parts: empty");
  colsum_final(static_cast<cudaStream_t>(stream), part, nparts, static_cast<int>(cols), cols, out,
               accumulate);
  return rp_check_launch("colsum_parts");
}

// column sum of a [rows, cols] matrix: out[c] (+)= sum_r in[r][c]
// (ref:proj/core/src/layers.cpp:38-52 col_sum, used for the MLP bias grads)
static const int kColRpb = 128;
extern "C" int64_t rp_colsum_workspace_floats(int64_t rows, int64_t cols) {
  return ((rows + kColRpb - 1) / kColRpb) * cols;
}

extern "C" int rp_colsum(const void* in, int in_is_bf16, int64_t rows, int64_t cols, float* out,
                         float* workspace, int accumulate, rp_stream_t stream) {
  if (rows <= 0 || cols <= 0 || cols % 4) return rp_fail(RP_ERR_SHAPE, "col_sum: cols % 4");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t nparts = (rows + kColRpb - 1) / kColRpb;
  dim3 grid(static_cast<unsigned>(nparts), static_cast<unsigned>((cols / 4 + 255) / 256));
  if (in_is_bf16)
    launch_k(colsum_partial_kernel<__nv_bfloat16>, dim3(grid), dim3(256), 0, s, 
        static_cast<const __nv_bfloat16*>(in), rows, static_cast<int>(cols), kColRpb, workspace);
  else
    launch_k(colsum_partial_kernel<float>, dim3(grid), dim3(256), 0, s, static_cast<const float*>(in), rows,
                                                      static_cast<int>(cols), kColRpb,
                                                      workspace);
  colsum_final(s, workspace, nparts, static_cast<int>(cols), cols, out, accumulate);
  return rp_check_launch("col_sum");
}
