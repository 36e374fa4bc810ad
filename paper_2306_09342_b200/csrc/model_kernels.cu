// Model glue kernels of the isotropic reversible model:
// parameter init (counter RNG of ref:proj/core/include/revprop/rng.hpp:13-71), fp32->bf16
// weight shadow, SGD, the head (fuse-average, mean-pool, logits, cross-entropy and their
// VJPs) and small element-wise helpers. All are HBM- or launch-bound; none sits on the
// tensor-core critical path. Every reduction has a fixed order (no atomics).
#include "../../include/revprop_b200.h"
#include "kernels.h"
#include "model_kernels.h"
#include "ptx.cuh"
#include "launch.h"

namespace rp {

// ------------------------------------------------------------- counter RNG (rng.hpp)
__host__ __device__ __forceinline__ uint64_t rng_mix(uint64_t z) {
  z ^= z >> 33;
  z *= 0xff51afd7ed558ccdULL;
  z ^= z >> 33;
  z *= 0xc4ceb9fe1a85ec53ULL;
  z ^= z >> 33;
  return z;
}
// Rng(seed, stream).next_u64() at `counter` (rng.hpp:27-33)
__host__ __device__ __forceinline__ uint64_t rng_u64(uint64_t seed, uint64_t stream,
                                                     uint64_t counter) {
  uint64_t h = rng_mix(seed ^ 0x9e3779b97f4a7c15ULL);
  h = rng_mix(h ^ (stream * 0xbf58476d1ce4e5b9ULL + 0x94d049bb133111ebULL));
  h = rng_mix(h ^ (counter * 0x2545f4914f6cdd1dULL + 0xd6e8feb86659fd93ULL));
  return h;
}
// next_normal at counters (c, c+1) (rng.hpp:38-42)
__device__ __forceinline__ double rng_normal(uint64_t seed, uint64_t stream, uint64_t c) {
  const double u1 = static_cast<double>((rng_u64(seed, stream, c) >> 11) + 1) * 0x1.0p-53;
  const double u2 = static_cast<double>(rng_u64(seed, stream, c + 1) >> 11) * 0x1.0p-53;
  return sqrt(-2.0 * log(u1)) * cos(2.0 * 3.14159265358979323846 * u2);
}

// Parameter element e of flat tensor j: Rng(seed, (1<<56)|(j<<32)|e).next_trunc_normal(sigma)
// (trunc normal at +-2 sigma, rng.hpp:45-50); kinds: 0 trunc-normal, 1 zeros, 2 ones.
__global__ void init_tensor_kernel(float* __restrict__ p, int64_t n, uint64_t seed,
                                   uint64_t tensor_idx, int kind, double sigma) {
  pdl_trigger();
  pdl_wait();

  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float v;
    if (kind == 1) {
      v = 0.f;
    } else if (kind == 2) {
      v = 1.f;
    } else {
      const uint64_t stream = (1ull << 56) | (tensor_idx << 32) | static_cast<uint64_t>(e);
      double z = 0.0;
      for (uint64_t c = 0;; c += 2) {
        z = rng_normal(seed, stream, c);
        if (z >= -2.0 && z <= 2.0) break;
      }
      v = static_cast<float>(z * sigma);
    }
    p[e] = v;
  }
}

// Synthetic input element e: Rng(seed, (2<<56)|e).next_normal(), stored as bf16.
__global__ void init_inputs_kernel(__nv_bfloat16* __restrict__ x, int64_t n, uint64_t seed) {
  pdl_trigger();
  pdl_wait();

  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint64_t stream = (2ull << 56) | static_cast<uint64_t>(e);
    x[e] = __float2bfloat16_rn(static_cast<float>(rng_normal(seed, stream, 0)));
  }
}

__global__ void f32_to_bf16_kernel(const float* __restrict__ in, __nv_bfloat16* __restrict__ out,
                                   int64_t n) {
  pdl_trigger();
  pdl_wait();

  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = __float2bfloat16_rn(in[i]);
}

// SGD: theta <- theta - lr * scale * g, fp32 master + bf16 shadow.
// lr is read from device memory so a captured CUDA graph can change it between steps.
__global__ void sgd_kernel(float* __restrict__ p, const float* __restrict__ g,
                           __nv_bfloat16* __restrict__ pb, int64_t n,
                           const float* __restrict__ lr, float scale) {
  pdl_trigger();
  pdl_wait();

  // explicit roundings (no FMA contraction): p - (lr * scale) * g exactly as the fp32
  // formula reads, so the update is bit-reproducible on the host
  const float step = __fmul_rn(lr[0], scale);
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const float v = __fsub_rn(p[i], __fmul_rn(step, g[i]));
    p[i] = v;
    pb[i] = __float2bfloat16_rn(v);
  }
}

// The same update on 4 consecutive parameters per thread and iteration (16-byte p / g
// accesses, one 8-byte bf16 store): the scalar loop's 4- and 2-byte accesses reached 78 % of
// HBM bandwidth at G48's 33 M parameters per block. p, g 16-byte and pb 8-byte aligned;
// n4 = n / 4 (the tail, n % 4, runs in the scalar kernel).
__global__ void sgd4_kernel(float4* __restrict__ p, const float4* __restrict__ g,
                            uint2* __restrict__ pb, int64_t n4, const float* __restrict__ lr,
                            float scale) {
  pdl_trigger();
  pdl_wait();
  const float step = __fmul_rn(lr[0], scale);
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n4;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const float4 pv = p[i], gv = g[i];
    float4 v;
    v.x = __fsub_rn(pv.x, __fmul_rn(step, gv.x));
    v.y = __fsub_rn(pv.y, __fmul_rn(step, gv.y));
    v.z = __fsub_rn(pv.z, __fmul_rn(step, gv.z));
    v.w = __fsub_rn(pv.w, __fmul_rn(step, gv.w));
    p[i] = v;
    const __nv_bfloat162 lo = __floats2bfloat162_rn(v.x, v.y), hi = __floats2bfloat162_rn(v.z, v.w);
    pb[i] = make_uint2(*reinterpret_cast<const uint32_t*>(&lo), *reinterpret_cast<const uint32_t*>(&hi));
  }
}

// AdamW (decoupled weight decay), bias-corrected with the device step counter t.
__global__ void adamw_kernel(float* __restrict__ p, const float* __restrict__ g,
                             __nv_bfloat16* __restrict__ pb, float* __restrict__ m,
                             float* __restrict__ v, int64_t n, const float* __restrict__ lr,
                             const float* __restrict__ t, float b1, float b2, float eps,
                             float wd, float scale) {
  pdl_trigger();
  pdl_wait();
  const float step = lr[0];
  const float tt = t[0];
  // torch.optim.AdamW's order of operations (decay first, then the bias-corrected step):
  // p *= 1 - lr wd; p -= (lr / bc1) m / (sqrt(v) / sqrt(bc2) + eps)
  const float bc1 = 1.0f - powf(b1, tt), bc2s = sqrtf(1.0f - powf(b2, tt));
  const float step_size = step / bc1, decay = 1.0f - step * wd;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const float gi = g[i] * scale;
    const float mi = b1 * m[i] + (1.0f - b1) * gi;
    const float vi = b2 * v[i] + (1.0f - b2) * gi * gi;
    m[i] = mi;
    v[i] = vi;
    const float pv = p[i] * decay - step_size * (mi / (sqrtf(vi) / bc2s + eps));
    p[i] = pv;
    pb[i] = __float2bfloat16_rn(pv);
  }
}

__global__ void add_scalar_kernel(float* x, float a) {
  pdl_trigger();
  pdl_wait();
  x[0] += a;
}

// fuse(average) + mean_tokens (layers.cpp:276-280 -> ops.cpp:408-427):
// pooled[b][c] = (sum_n (o1 + o2) * 0.5) * (1/N), summed in token order.
__global__ void pool_kernel(const float* __restrict__ o1, const float* __restrict__ o2,
                            int64_t B, int64_t N, int64_t d, float* __restrict__ pooled) {
  pdl_trigger();
  pdl_wait();

  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= B * d) return;
  const int64_t b = i / d, c = i % d;
  const float* p1 = o1 + b * N * d + c;
  const float* p2 = o2 + b * N * d + c;
  float s = 0.f;
  for (int64_t n = 0; n < N; ++n) s += (p1[n * d] + p2[n * d]) * 0.5f;
  pooled[i] = s * (1.0f / static_cast<float>(N));
}

// C[M,N] = sum_k A(m,k) B(k,n); A(m,k) = A[m*sam + k*sak], B(k,n) = B[k*sbk + n*sbn].
// fp32 GEMM for the small head products (C = 1000 is not a tensor-core tile multiple):
// 32 x 32 output tile per CTA (enough CTAs to fill the GPU at M = 256), 256 threads, 2 x 2
// outputs per thread in registers, 32-deep k slices staged through smem (any strides, so
// transposed operands need no copy). Fixed k order: deterministic.
__global__ void __launch_bounds__(256)
    simt_gemm_kernel(int64_t M, int64_t N, int64_t K, const float* __restrict__ A, int64_t sam,
                     int64_t sak, const float* __restrict__ Bm, int64_t sbk, int64_t sbn,
                     float* __restrict__ Cm, int64_t ldc) {
  pdl_trigger();
  pdl_wait();

  __shared__ float as[32][32 + 1], bs[32][32 + 1];  // [k][m], [k][n]
  const int tid = threadIdx.x;
  const int tm = (tid >> 4) * 2, tn = (tid & 15) * 2;
  const int64_t m0 = static_cast<int64_t>(blockIdx.y) * 32, n0 = static_cast<int64_t>(blockIdx.x) * 32;
  float acc[2][2] = {};
  // the next k slice is fetched into registers while the current one is multiplied
  float ra[4], rb[4];
  auto fetch = [&](int64_t k0) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int i = tid + 256 * j;
      const int kk = i & 31, mm = i >> 5;  // A: consecutive threads walk k
      const int64_t gm = m0 + mm, gk = k0 + kk;
      ra[j] = (gm < M && gk < K) ? A[gm * sam + gk * sak] : 0.f;
      const int nn = i & 31, kb = i >> 5;  // B: consecutive threads walk n
      const int64_t gn = n0 + nn, gkb = k0 + kb;
      rb[j] = (gkb < K && gn < N) ? Bm[gkb * sbk + gn * sbn] : 0.f;
    }
  };
  fetch(0);
  for (int64_t k0 = 0; k0 < K; k0 += 32) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int i = tid + 256 * j;
      as[i & 31][i >> 5] = ra[j];
      bs[i >> 5][i & 31] = rb[j];
    }
    __syncthreads();
    if (k0 + 32 < K) fetch(k0 + 32);
#pragma unroll 8
    for (int k = 0; k < 32; ++k) {
      const float a0 = as[k][tm], a1 = as[k][tm + 1], b0 = bs[k][tn], b1 = bs[k][tn + 1];
      acc[0][0] = fmaf(a0, b0, acc[0][0]);
      acc[0][1] = fmaf(a0, b1, acc[0][1]);
      acc[1][0] = fmaf(a1, b0, acc[1][0]);
      acc[1][1] = fmaf(a1, b1, acc[1][1]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int64_t m = m0 + tm + i, n = n0 + tn + j;
      if (m < M && n < N) Cm[m * ldc + n] = acc[i][j];
    }
}

// Mean cross-entropy, log-sum-exp stabilised. One warp per row:
// d_logits = (softmax - onehot) / B; row_loss[b] = lse - logit[label].
__global__ void ce_kernel(const float* __restrict__ logits, const int32_t* __restrict__ labels,
                          int64_t B, int64_t C, float* __restrict__ d_logits,
                          float* __restrict__ row_loss) {
  pdl_trigger();
  pdl_wait();

  const int64_t b = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (b >= B) return;
  const float* lr = logits + b * C;
  float mx = -INFINITY;
  for (int64_t c = lane; c < C; c += 32) mx = fmaxf(mx, lr[c]);
#pragma unroll
  for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  float s = 0.f;
  for (int64_t c = lane; c < C; c += 32) s += expf(lr[c] - mx);
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  const float lse = mx + logf(s);
  const int32_t y = labels[b];
  const float invB = 1.0f / static_cast<float>(B);
  for (int64_t c = lane; c < C; c += 32) {
    const float p = expf(lr[c] - lse);
    d_logits[b * C + c] = (p - (c == y ? 1.f : 0.f)) * invB;
  }
  if (lane == 0) row_loss[b] = lse - lr[y];
}

// loss = (1/B) sum_b row_loss[b], fixed order, optionally * 1/world for DP averaging
__global__ void loss_reduce_kernel(const float* __restrict__ row_loss, int64_t B,
                                   float* __restrict__ loss) {
  pdl_trigger();
  pdl_wait();

  __shared__ float red[256];
  float s = 0.f;
  for (int64_t i = threadIdx.x; i < B; i += blockDim.x) s += row_loss[i];
  red[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.f;
    for (int i = 0; i < static_cast<int>(blockDim.x); ++i) t += red[i];
    loss[0] = t / static_cast<float>(B);
  }
}

// spread_tokens + fuse_vjp(average) (ops.cpp:429-447, layers.cpp:289-293):
// d_o1 = d_o2 = (d_pooled[b] * (1/N)) * 0.5, written fp32 (both) + bf16 (both).
__global__ void spread_kernel(const float* __restrict__ d_pooled, int64_t B, int64_t N,
                              int64_t d, float* __restrict__ d1, float* __restrict__ d2,
                              __nv_bfloat16* __restrict__ d1b, __nv_bfloat16* __restrict__ d2b) {
  pdl_trigger();
  pdl_wait();

  // 4 consecutive columns per thread (d % 4 == 0): float4 / 2 x bf16x2 stores
  const int64_t total4 = B * N * d / 4;
  const float scale = 0.5f / static_cast<float>(N);
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total4;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t e = 4 * i, c = e % d, b = e / (N * d);
    const float4 p = *reinterpret_cast<const float4*>(d_pooled + b * d + c);
    const float4 v = make_float4(p.x * scale, p.y * scale, p.z * scale, p.w * scale);
    reinterpret_cast<float4*>(d1)[i] = v;
    reinterpret_cast<float4*>(d2)[i] = v;
    const uint2 vb = make_uint2(pack_bf16x2(v.x, v.y), pack_bf16x2(v.z, v.w));
    reinterpret_cast<uint2*>(d1b)[i] = vb;
    reinterpret_cast<uint2*>(d2b)[i] = vb;
  }
}

// out = bf16(a + b)  (embedding cotangent: e feeds both halves of the coupled pair)
__global__ void add_to_bf16_kernel(const float* __restrict__ a, const float* __restrict__ b,
                                   __nv_bfloat16* __restrict__ out, int64_t n) {
  pdl_trigger();
  pdl_wait();

  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = __float2bfloat16_rn(a[i] + b[i]);
}

// out = a + sign * b (fp32): the coupling add / subtract of the standalone revcore entry
// points (ref:proj/core/src/ops.cpp:96-106 add / sub)
__global__ void axpy_sign_kernel(const float* __restrict__ a, const float* __restrict__ b,
                                 float sign, float* __restrict__ out, int64_t n) {
  pdl_trigger();
  pdl_wait();
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = __fadd_rn(a[i], sign * b[i]);
}

// SGD on caller-owned fp32 parameters with a host learning rate, same
// rounding as sgd_kernel: p - lr * g, no contraction
__global__ void sgd_value_kernel(float* __restrict__ p, const float* __restrict__ g, int64_t n,
                                 float lr) {
  pdl_trigger();
  pdl_wait();
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    p[i] = __fsub_rn(p[i], __fmul_rn(lr, g[i]));
}

// fuse(average) of a stage output (layers.cpp:277-279: ops::scale(ops::add(i1, i2), 0.5)),
// written bf16 as the patch_merge GEMM operand
__global__ void fuse_avg_kernel(const float* __restrict__ o1, const float* __restrict__ o2,
                                int64_t n4, __nv_bfloat16* __restrict__ out) {
  pdl_trigger();
  pdl_wait();

  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n4;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const float4 a = reinterpret_cast<const float4*>(o1)[i];
    const float4 b = reinterpret_cast<const float4*>(o2)[i];
    reinterpret_cast<uint2*>(out)[i] =
        make_uint2(pack_bf16x2((a.x + b.x) * 0.5f, (a.y + b.y) * 0.5f),
                   pack_bf16x2((a.z + b.z) * 0.5f, (a.w + b.w) * 0.5f));
  }
}

// concat_last(o1, o2) (ops.cpp:366-391) for the mlp fusion: out [rows, 2d] bf16
__global__ void concat_kernel(const float* __restrict__ o1, const float* __restrict__ o2,
                              int64_t rows, int64_t d, __nv_bfloat16* __restrict__ out) {
  pdl_trigger();
  pdl_wait();

  const int64_t d4 = d / 4, total = rows * 2 * d4;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / (2 * d4), c = i % (2 * d4);
    const float* src = c < d4 ? o1 : o2;
    const float4 v = reinterpret_cast<const float4*>(src + r * d)[c < d4 ? c : c - d4];
    reinterpret_cast<uint2*>(out)[i] = make_uint2(pack_bf16x2(v.x, v.y), pack_bf16x2(v.z, v.w));
  }
}

// fuse_vjp(average) (layers.cpp:289-292): d_i1 = d_i2 = d_y * 0.5; d1 holds d_y on entry
__global__ void halve_dup_kernel(float* __restrict__ d1, int64_t n4, float* __restrict__ d2,
                                 __nv_bfloat16* __restrict__ d1b,
                                 __nv_bfloat16* __restrict__ d2b) {
  pdl_trigger();
  pdl_wait();

  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n4;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float4 v = reinterpret_cast<float4*>(d1)[i];
    v = make_float4(v.x * 0.5f, v.y * 0.5f, v.z * 0.5f, v.w * 0.5f);
    reinterpret_cast<float4*>(d1)[i] = v;
    reinterpret_cast<float4*>(d2)[i] = v;
    const uint2 vb = make_uint2(pack_bf16x2(v.x, v.y), pack_bf16x2(v.z, v.w));
    reinterpret_cast<uint2*>(d1b)[i] = vb;
    reinterpret_cast<uint2*>(d2b)[i] = vb;
  }
}

// x *= s (fp32 and its bf16 shadow): the verify command's fault-injection hook
__global__ void scale_pair_kernel(float* __restrict__ x, __nv_bfloat16* __restrict__ xb,
                                  int64_t n, float s) {
  pdl_trigger();
  pdl_wait();

  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const float v = x[i] * s;
    x[i] = v;
    xb[i] = __float2bfloat16_rn(v);
  }
}

static inline unsigned grid_for(int64_t n, int threads = 256, int cap = 148 * 16) {
  int64_t g = (n + threads - 1) / threads;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return static_cast<unsigned>(g);
}

}  // namespace rp

using namespace rp;

uint64_t rp_rng_u64_host(uint64_t seed, uint64_t stream, uint64_t counter) {
  return rng_u64(seed, stream, counter);
}

int rpk_init_tensor(float* p, int64_t n, uint64_t seed, uint64_t tensor_idx, int kind,
                    double sigma, cudaStream_t s) {
  launch_k(init_tensor_kernel, dim3(grid_for(n)), dim3(256), 0, s, p, n, seed, tensor_idx, kind, sigma);
  return rp_check_launch("init_tensor");
}
int rpk_init_inputs(uint16_t* x, int64_t n, uint64_t seed, cudaStream_t s) {
  launch_k(init_inputs_kernel, dim3(grid_for(n)), dim3(256), 0, s, reinterpret_cast<__nv_bfloat16*>(x), n, seed);
  return rp_check_launch("init_inputs");
}
int rpk_f32_to_bf16(const float* in, uint16_t* out, int64_t n, cudaStream_t s) {
  launch_k(f32_to_bf16_kernel, dim3(grid_for(n)), dim3(256), 0, s, in, reinterpret_cast<__nv_bfloat16*>(out), n);
  return rp_check_launch("f32_to_bf16");
}
int rpk_sgd(float* p, const float* g, uint16_t* pb, int64_t n, const float* lr, float scale,
            cudaStream_t s) {
  const bool vec = ((reinterpret_cast<uintptr_t>(p) | reinterpret_cast<uintptr_t>(g)) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(pb) & 7) == 0;
  const int64_t n4 = vec ? n / 4 : 0;
  if (n4 > 0)
    launch_k(sgd4_kernel, dim3(grid_for(n4)), dim3(256), 0, s, reinterpret_cast<float4*>(p),
             reinterpret_cast<const float4*>(g), reinterpret_cast<uint2*>(pb), n4, lr, scale);
  if (n - 4 * n4 > 0)
    launch_k(sgd_kernel, dim3(grid_for(n - 4 * n4)), dim3(256), 0, s, p + 4 * n4, g + 4 * n4,
             reinterpret_cast<__nv_bfloat16*>(pb) + 4 * n4, n - 4 * n4, lr, scale);
  return rp_check_launch("sgd");
}
int rpk_adamw(float* p, const float* g, uint16_t* pb, float* m, float* v, int64_t n,
              const float* lr, const float* t, float b1, float b2, float eps, float wd,
              float scale, cudaStream_t s) {
  launch_k(adamw_kernel, dim3(grid_for(n)), dim3(256), 0, s, p, g,
           reinterpret_cast<__nv_bfloat16*>(pb), m, v, n, lr, t, b1, b2, eps, wd, scale);
  return rp_check_launch("adamw");
}
int rpk_add_scalar(float* x, float a, cudaStream_t s) {
  launch_k(add_scalar_kernel, dim3(1), dim3(1), 0, s, x, a);
  return rp_check_launch("add_scalar");
}
int rpk_pool(const float* o1, const float* o2, int64_t B, int64_t N, int64_t d, float* pooled,
             cudaStream_t s) {
  launch_k(pool_kernel, dim3(static_cast<unsigned>((B * d + 255) / 256)), dim3(256), 0, s, o1, o2, B, N, d, pooled);
  return rp_check_launch("pool");
}
int rpk_simt_gemm(int64_t M, int64_t N, int64_t K, const float* A, int64_t sam, int64_t sak,
                  const float* B, int64_t sbk, int64_t sbn, float* C, int64_t ldc,
                  cudaStream_t s) {
  dim3 grid(static_cast<unsigned>((N + 31) / 32), static_cast<unsigned>((M + 31) / 32));
  launch_k(simt_gemm_kernel, dim3(grid), dim3(256), 0, s, M, N, K, A, sam, sak, B, sbk, sbn, C, ldc);
  return rp_check_launch("simt_gemm");
}
int rpk_cross_entropy(const float* logits, const int32_t* labels, int64_t B, int64_t C,
                      float* d_logits, float* row_loss, float* loss, cudaStream_t s) {
  launch_k(ce_kernel, dim3(static_cast<unsigned>((B + 7) / 8)), dim3(256), 0, s, logits, labels, B, C, d_logits,
                                                              row_loss);
  launch_k(loss_reduce_kernel, dim3(1), dim3(256), 0, s, row_loss, B, loss);
  return rp_check_launch("cross_entropy");
}
int rpk_spread(const float* d_pooled, int64_t B, int64_t N, int64_t d, float* d1, float* d2,
               uint16_t* d1b, uint16_t* d2b, cudaStream_t s) {
  launch_k(spread_kernel, dim3(grid_for(B * N * d / 4)), dim3(256), 0, s, d_pooled, B, N, d, d1, d2,
                                                    reinterpret_cast<__nv_bfloat16*>(d1b),
                                                    reinterpret_cast<__nv_bfloat16*>(d2b));
  return rp_check_launch("spread");
}
int rpk_add_to_bf16(const float* a, const float* b, uint16_t* out, int64_t n, cudaStream_t s) {
  launch_k(add_to_bf16_kernel, dim3(grid_for(n)), dim3(256), 0, s, a, b, reinterpret_cast<__nv_bfloat16*>(out), n);
  return rp_check_launch("add_to_bf16");
}
int rpk_axpy_sign(const float* a, const float* b, float sign, float* out, int64_t n,
                  cudaStream_t s) {
  launch_k(axpy_sign_kernel, dim3(grid_for(n)), dim3(256), 0, s, a, b, sign, out, n);
  return rp_check_launch("axpy_sign");
}
int rpk_sgd_value(float* p, const float* g, int64_t n, float lr, cudaStream_t s) {
  launch_k(sgd_value_kernel, dim3(grid_for(n)), dim3(256), 0, s, p, g, n, lr);
  return rp_check_launch("sgd_value");
}
int rpk_fuse_avg_bf16(const float* o1, const float* o2, int64_t n, uint16_t* out, cudaStream_t s) {
  launch_k(fuse_avg_kernel, dim3(grid_for(n / 4)), dim3(256), 0, s, o1, o2, n / 4,
           reinterpret_cast<__nv_bfloat16*>(out));
  return rp_check_launch("fuse_avg");
}
int rpk_concat_bf16(const float* o1, const float* o2, int64_t rows, int64_t d, uint16_t* out,
                    cudaStream_t s) {
  launch_k(concat_kernel, dim3(grid_for(rows * d / 2)), dim3(256), 0, s, o1, o2, rows, d,
           reinterpret_cast<__nv_bfloat16*>(out));
  return rp_check_launch("concat");
}
int rpk_halve_dup(float* d1, int64_t n, float* d2, uint16_t* d1b, uint16_t* d2b, cudaStream_t s) {
  launch_k(halve_dup_kernel, dim3(grid_for(n / 4)), dim3(256), 0, s, d1, n / 4, d2,
           reinterpret_cast<__nv_bfloat16*>(d1b), reinterpret_cast<__nv_bfloat16*>(d2b));
  return rp_check_launch("halve_dup");
}
int rpk_scale_pair(float* x, uint16_t* xb, int64_t n, float s, cudaStream_t st) {
  launch_k(scale_pair_kernel, dim3(grid_for(n)), dim3(256), 0, st, x,
           reinterpret_cast<__nv_bfloat16*>(xb), n, s);
  return rp_check_launch("scale_pair");
}
