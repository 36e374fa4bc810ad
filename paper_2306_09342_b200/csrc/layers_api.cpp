// The reference's layer / revcore / optimizer API as pure functions over CALLER-owned device
// tensors (no engine): ref:proj/core/include/revprop/layers.hpp:82-138
// (attention_forward / attention_vjp / mlp_forward / mlp_vjp with their caches), SPEC.md:
// 213-239 (rev_forward / rev_inverse / rev_backward_local) and SPEC.md:387-395 (sgd_update).
// The C++ wrapper in include/revprop_b200.hpp gives them the reference's names and types.
//
// Same kernels as the engine's hot path (tcgen05 GEMMs with fused epilogues, the attention
// kernels, LayerNorm), composed per call: weights arrive fp32 in the reference's [in, out]
// layout and are shadowed to bf16 once per forward (kept in the cache for the VJP, which
// is the reference's contract: the VJP takes the forward's cache). The cache owns device
// buffers (value semantics, like the reference's AttentionCache / MlpCache); temporaries are
// stream-ordered allocations (cudaMallocAsync) on the caller's stream.
#include <cuda_runtime.h>

#include <algorithm>
#include <string>
#include <vector>

#include "../../include/revprop_b200.h"
#include "kernels.h"
#include "model_kernels.h"

struct RpLayerCache {
  int kind = 0;  // 1 attention (F), 2 MLP (G)
  int64_t T = 0, N = 0, d = 0, h = 0, H = 0, W = 0;
  cudaStream_t stream = nullptr;
  std::vector<void*> bufs;
  // attention: x (fp32), mean / rstd, h (bf16 LN output), qkv, att (bf16), lse, w_qkv / w_out
  // bf16 shadows. MLP: x, mean / rstd, h, a = gelu(u), slope = gelu'(u) (bf16), w1 / w2 bf16.
  float *x = nullptr, *mean = nullptr, *rstd = nullptr, *lse = nullptr;
  uint16_t *hb = nullptr, *qkv = nullptr, *att = nullptr, *a = nullptr, *slope = nullptr,
           *w0 = nullptr, *w1 = nullptr;
  int64_t bytes = 0;
};

namespace {

constexpr int kSms = 148;

int cuda_ok(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return RP_OK;
  cudaGetLastError();
  const std::string m = std::string(what) + ": " + cudaGetErrorString(e);
  return rp_fail(e == cudaErrorMemoryAllocation ? RP_ERR_BUDGET : RP_ERR_CUDA, m.c_str());
}

#define RP_TRY(x)                 \
  do {                            \
    int rc_ = (x);                \
    if (rc_ != RP_OK) return rc_; \
  } while (0)

template <class T>
int cache_alloc(RpLayerCache* c, T** p, int64_t n) {
  void* q = nullptr;
  const size_t bytes = static_cast<size_t>(std::max<int64_t>(n, 1)) * sizeof(T);
  RP_TRY(cuda_ok(cudaMallocAsync(&q, bytes, c->stream), "layer cache allocation"));
  c->bufs.push_back(q);
  c->bytes += static_cast<int64_t>(bytes);
  *p = static_cast<T*>(q);
  return RP_OK;
}

// stream-ordered scratch freed when the scope ends (after the work using it is enqueued)
struct Scratch {
  cudaStream_t s;
  std::vector<void*> p;
  explicit Scratch(cudaStream_t st) : s(st) {}
  ~Scratch() {
    for (void* q : p) cudaFreeAsync(q, s);
  }
  template <class T>
  int get(T** out, int64_t n) {
    void* q = nullptr;
    RP_TRY(cuda_ok(cudaMallocAsync(&q, static_cast<size_t>(std::max<int64_t>(n, 1)) * sizeof(T), s),
                   "scratch allocation"));
    p.push_back(q);
    *out = static_cast<T*>(q);
    return RP_OK;
  }
};

int gemm_bn(int64_t N) { return (N % 256 != 0 && N < 512) ? 128 : 512; }

// split-K count for the wgrad GEMMs (K = T rows): enough units to fill the SMs
int wgrad_splits(int64_t M, int64_t N, int64_t K) {
  const int bn = gemm_bn(N);
  const bool pair = bn == 512;
  const int tm = pair ? 256 : 128, tn = pair ? 256 : bn, slots = pair ? kSms / 2 : kSms;
  const int64_t tiles = ((M + tm - 1) / tm) * ((N + tn - 1) / tn), kb = (K + 63) / 64;
  int best = 1;
  double best_eff = 0.0;
  for (int s = 1; s <= 64 && kb / s >= 8; ++s) {
    const int64_t units = tiles * s;
    const double waves = static_cast<double>((units + slots - 1) / slots);
    const double eff = static_cast<double>(units) / (waves * slots) - 0.004 * s;
    if (eff > best_eff + 1e-9) {
      best_eff = eff;
      best = s;
    }
  }
  return best;
}

struct G {
  const uint16_t* A;
  int64_t lda;
  int a_mn;
  const uint16_t* B;
  int64_t ldb;
  int b_mn;
  int64_t M, N, K;
  int epi;
  void* out;
  int64_t ldo;
};

int gemm(const G& g, cudaStream_t s, Scratch& sc, const void* aux = nullptr,
         const float* bias = nullptr, float sign = 1.f, void* out2 = nullptr,
         float* colsum = nullptr) {
  RpGemmDesc d{};
  d.A = g.A;
  d.lda = g.lda;
  d.a_mn = g.a_mn;
  d.B = g.B;
  d.ldb = g.ldb;
  d.b_mn = g.b_mn;
  d.M = g.M;
  d.N = g.N;
  d.K = g.K;
  d.epi = g.epi;
  d.out = g.out;
  d.ldo = g.ldo;
  d.out2 = out2;
  d.ldo2 = g.ldo;
  d.aux = aux;
  d.ldaux = g.ldo;
  d.bias = bias;
  d.sign = sign;
  d.splits = 1;
  d.bn = gemm_bn(g.N);
  d.colsum_part = colsum;
  if (g.epi == RP_EPI_F32 && g.a_mn == 1 && g.b_mn == 1) {  // wgrad: split K = rows
    d.splits = wgrad_splits(g.M, g.N, g.K);
    if (d.splits > 1) RP_TRY(sc.get(&d.workspace, static_cast<int64_t>(d.splits) * g.M * g.N));
  }
  return rp_gemm(&d, s);
}

int to_bf16(const float* in, int64_t n, uint16_t* out, cudaStream_t s) {
  return rpk_f32_to_bf16(in, out, n, s);
}

int check_rows(int64_t B, int64_t N, int64_t d) {
  if (B < 1 || N < 1) return rp_fail(RP_ERR_SHAPE, "layer: batch and tokens must be >= 1");
  if (d < 64 || d % 64) return rp_fail(RP_ERR_SHAPE, "layer: width must be a multiple of 64");
  return RP_OK;
}

int attn_geom(const RpAttentionParamsDev* p, int64_t N, int64_t* W, int64_t* hd) {
  if (!p || !p->w_qkv || !p->w_out || !p->ln_gamma || !p->ln_beta)
    return rp_fail(RP_ERR_CONTRACT, "attention: null parameter");
  if (p->heads < 1 || p->width % p->heads)
    return rp_fail(RP_ERR_SHAPE, "attention: width not divisible by heads");  // layers.cpp:139
  *hd = p->width / p->heads;
  if (*hd % 8 || *hd > 128) return rp_fail(RP_ERR_SHAPE, "attention: head_dim must be a multiple of 8, <= 128");
  *W = p->window > 0 ? p->window : N;
  if (N % *W) return rp_fail(RP_ERR_SHAPE, "attention: sequence length not divisible by window");
  return RP_OK;
}

}  // namespace

// ---------------------------------------------------------------- attention (F)
extern "C" int rp_attention_forward(const RpAttentionParamsDev* p, const float* x, int64_t batch,
                                    int64_t tokens, float* y, RpLayerCache** cache,
                                    rp_stream_t stream) {
  if (!x || !y) return rp_fail(RP_ERR_CONTRACT, "attention_forward: null tensor");
  int64_t W = 0, hd = 0;
  RP_TRY(attn_geom(p, tokens, &W, &hd));
  const int64_t d = p->width, T = batch * tokens, H = p->heads;
  RP_TRY(check_rows(batch, tokens, d));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  RpLayerCache* c = new RpLayerCache();
  c->kind = 1;
  c->T = T;
  c->N = tokens;
  c->d = d;
  c->H = H;
  c->W = W;
  c->stream = s;
  auto fail = [&](int rc) {
    rp_layer_cache_destroy(c);
    return rc;
  };
  int rc;
  if ((rc = cache_alloc(c, &c->x, T * d)) || (rc = cache_alloc(c, &c->mean, T)) ||
      (rc = cache_alloc(c, &c->rstd, T)) || (rc = cache_alloc(c, &c->hb, T * d)) ||
      (rc = cache_alloc(c, &c->qkv, 3 * T * d)) || (rc = cache_alloc(c, &c->att, T * d)) ||
      (rc = cache_alloc(c, &c->lse, T * H)) || (rc = cache_alloc(c, &c->w0, 3 * d * d)) ||
      (rc = cache_alloc(c, &c->w1, d * d)))
    return fail(rc);
  Scratch sc(s);
  if ((rc = cuda_ok(cudaMemcpyAsync(c->x, x, static_cast<size_t>(T * d) * 4,
                                    cudaMemcpyDeviceToDevice, s), "copy x")) ||
      (rc = to_bf16(p->w_qkv, 3 * d * d, c->w0, s)) || (rc = to_bf16(p->w_out, d * d, c->w1, s)) ||
      // h = LN(x) (ops.cpp:264-304), qkv = h W_qkv (layers.cpp:144-146)
      (rc = rp_layer_norm_fwd(x, p->ln_gamma, p->ln_beta, T, d, 1e-5, c->hb, c->mean, c->rstd, s)) ||
      (rc = gemm({c->hb, d, 0, c->w0, 3 * d, 1, T, 3 * d, d, RP_EPI_BF16, c->qkv, 3 * d}, s, sc)) ||
      // per (sequence, head, window) softmax(q k^T / sqrt(hd)) v (layers.cpp:150-166)
      (rc = rp_attention_fwd(c->qkv, T / W, W, H, hd, c->att, c->lse, s)) ||
      // y = att W_out (layers.cpp:167), no residual
      (rc = gemm({c->att, d, 0, c->w1, d, 1, T, d, d, RP_EPI_F32, y, d}, s, sc)))
    return fail(rc);
  if (cache)
    *cache = c;
  else
    rp_layer_cache_destroy(c);
  return rp_check_launch("attention_forward");
}

extern "C" int rp_attention_vjp(const RpLayerCache* c, const RpAttentionParamsDev* p,
                                const float* d_y, float* d_x, const RpAttentionGradsDev* gr,
                                rp_stream_t stream) {
  if (!c || c->kind != 1)
    return rp_fail(RP_ERR_CONTRACT, "attention_vjp: cache was not produced by attention_forward");
  if (!d_y || !d_x || !gr) return rp_fail(RP_ERR_CONTRACT, "attention_vjp: null tensor");
  int64_t W = 0, hd = 0;
  RP_TRY(attn_geom(p, c->N, &W, &hd));
  if (p->width != c->d || p->heads != c->H || W != c->W)
    return rp_fail(RP_ERR_CONTRACT, "attention_vjp: parameters do not match the cache");
  const int64_t T = c->T, d = c->d, H = c->H;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Scratch sc(s);
  uint16_t *dyb = nullptr, *datt = nullptr, *dqkv = nullptr, *dh = nullptr;
  float *aws = nullptr, *lnws = nullptr;
  RP_TRY(sc.get(&dyb, T * d));
  RP_TRY(sc.get(&datt, T * d));
  RP_TRY(sc.get(&dqkv, 3 * T * d));
  RP_TRY(sc.get(&dh, T * d));
  RP_TRY(sc.get(&aws, rp_attention_bwd_workspace_floats(T / W, W, H)));
  RP_TRY(sc.get(&lnws, rp_layer_norm_bwd_workspace_floats(T, d)));
  RP_TRY(to_bf16(d_y, T * d, dyb, s));
  // d_att = d_y W_out^T, dW_out = att^T d_y (layers.cpp:176-183)
  RP_TRY(gemm({dyb, d, 0, c->w1, d, 0, T, d, d, RP_EPI_BF16, datt, d}, s, sc));
  if (gr->d_w_out)
    RP_TRY(gemm({c->att, d, 1, dyb, d, 1, d, d, T, RP_EPI_F32, gr->d_w_out, d}, s, sc));
  // per head: dV, dS = softmax_vjp / sqrt(hd), dQ, dK (layers.cpp:185-208)
  RP_TRY(rp_attention_bwd(c->qkv, c->att, c->lse, datt, T / W, W, H, hd, dqkv, aws, s));
  // dW_qkv = h^T d_qkv, d_h = d_qkv W_qkv^T (layers.cpp:209-214), then the LN VJP
  if (gr->d_w_qkv)
    RP_TRY(gemm({c->hb, d, 1, dqkv, 3 * d, 1, d, 3 * d, T, RP_EPI_F32, gr->d_w_qkv, 3 * d}, s, sc));
  RP_TRY(gemm({dqkv, 3 * d, 0, c->w0, 3 * d, 0, T, d, 3 * d, RP_EPI_BF16, dh, d}, s, sc));
  RP_TRY(rp_layer_norm_bwd(c->x, c->mean, c->rstd, p->ln_gamma, dh, nullptr, T, d, d_x, nullptr,
                           gr->d_ln_gamma, gr->d_ln_beta, lnws, 0, s));
  return rp_check_launch("attention_vjp");
}

// ---------------------------------------------------------------- MLP (G)
namespace {
int mlp_check(const RpMlpParamsDev* p) {
  if (!p || !p->w1 || !p->b1 || !p->w2 || !p->b2 || !p->ln_gamma || !p->ln_beta)
    return rp_fail(RP_ERR_CONTRACT, "mlp: null parameter");
  if (p->hidden < 64 || p->hidden % 64)
    return rp_fail(RP_ERR_SHAPE, "mlp: hidden width must be a multiple of 64");
  return RP_OK;
}
}  // namespace

extern "C" int rp_mlp_forward(const RpMlpParamsDev* p, const float* x, int64_t batch,
                              int64_t tokens, float* y, RpLayerCache** cache, rp_stream_t stream) {
  if (!x || !y) return rp_fail(RP_ERR_CONTRACT, "mlp_forward: null tensor");
  RP_TRY(mlp_check(p));
  const int64_t d = p->width, h = p->hidden, T = batch * tokens;
  RP_TRY(check_rows(batch, tokens, d));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  RpLayerCache* c = new RpLayerCache();
  c->kind = 2;
  c->T = T;
  c->N = tokens;
  c->d = d;
  c->h = h;
  c->stream = s;
  auto fail = [&](int rc) {
    rp_layer_cache_destroy(c);
    return rc;
  };
  int rc;
  if ((rc = cache_alloc(c, &c->x, T * d)) || (rc = cache_alloc(c, &c->mean, T)) ||
      (rc = cache_alloc(c, &c->rstd, T)) || (rc = cache_alloc(c, &c->hb, T * d)) ||
      (rc = cache_alloc(c, &c->a, T * h)) || (rc = cache_alloc(c, &c->slope, T * h)) ||
      (rc = cache_alloc(c, &c->w0, d * h)) || (rc = cache_alloc(c, &c->w1, h * d)))
    return fail(rc);
  Scratch sc(s);
  if ((rc = cuda_ok(cudaMemcpyAsync(c->x, x, static_cast<size_t>(T * d) * 4,
                                    cudaMemcpyDeviceToDevice, s), "copy x")) ||
      (rc = to_bf16(p->w1, d * h, c->w0, s)) || (rc = to_bf16(p->w2, h * d, c->w1, s)) ||
      (rc = rp_layer_norm_fwd(x, p->ln_gamma, p->ln_beta, T, d, 1e-5, c->hb, c->mean, c->rstd, s)) ||
      // a = gelu(h W1 + b1) and gelu'(u) for the VJP (layers.cpp:226-233)
      (rc = gemm({c->hb, d, 0, c->w0, h, 1, T, h, d, RP_EPI_BIAS_GELU_SLOPE, c->a, h}, s, sc,
                 nullptr, p->b1, 1.f, c->slope)) ||
      // y = a W2 + b2 (layers.cpp:234-236): the residual epilogue onto a zeroed output
      (rc = cuda_ok(cudaMemsetAsync(y, 0, static_cast<size_t>(T * d) * 4, s), "memset")) ||
      (rc = gemm({c->a, h, 0, c->w1, d, 1, T, d, h, RP_EPI_RESID, y, d}, s, sc, y, p->b2, 1.f)))
    return fail(rc);
  if (cache)
    *cache = c;
  else
    rp_layer_cache_destroy(c);
  return rp_check_launch("mlp_forward");
}

extern "C" int rp_mlp_vjp(const RpLayerCache* c, const RpMlpParamsDev* p, const float* d_y,
                          float* d_x, const RpMlpGradsDev* gr, rp_stream_t stream) {
  if (!c || c->kind != 2)
    return rp_fail(RP_ERR_CONTRACT, "mlp_vjp: cache was not produced by mlp_forward");
  if (!d_y || !d_x || !gr) return rp_fail(RP_ERR_CONTRACT, "mlp_vjp: null tensor");
  RP_TRY(mlp_check(p));
  if (p->width != c->d || p->hidden != c->h)
    return rp_fail(RP_ERR_CONTRACT, "mlp_vjp: parameters do not match the cache");
  const int64_t T = c->T, d = c->d, h = c->h;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Scratch sc(s);
  uint16_t *dyb = nullptr, *du = nullptr, *dh = nullptr;
  float *colws = nullptr, *lnws = nullptr, *cparts = nullptr;
  RP_TRY(sc.get(&dyb, T * d));
  RP_TRY(sc.get(&du, T * h));
  RP_TRY(sc.get(&dh, T * d));
  RP_TRY(sc.get(&colws, rp_colsum_workspace_floats(T, d)));
  RP_TRY(sc.get(&cparts, ((T + 31) / 32) * h));
  RP_TRY(sc.get(&lnws, rp_layer_norm_bwd_workspace_floats(T, d)));
  RP_TRY(to_bf16(d_y, T * d, dyb, s));
  // d_b2 = col_sum(d_y) (layers.cpp:38-52, 247)
  if (gr->d_b2) RP_TRY(rp_colsum(d_y, 0, T, d, gr->d_b2, colws, 0, s));
  // d_u = (d_y W2^T) * gelu'(u) with per-32-row column sums of d_u -> d_b1 (layers.cpp:248-252)
  RP_TRY(gemm({dyb, d, 0, c->w1, d, 0, T, h, d, RP_EPI_MUL, du, h}, s, sc, c->slope, nullptr, 1.f,
              nullptr, cparts));
  if (gr->d_b1) RP_TRY(rp_colsum_parts(cparts, (T + 31) / 32, h, gr->d_b1, 0, s));
  // dW2 = a^T d_y, dW1 = h^T d_u, d_h = d_u W1^T (layers.cpp:246-256)
  if (gr->d_w2) RP_TRY(gemm({c->a, h, 1, dyb, d, 1, h, d, T, RP_EPI_F32, gr->d_w2, d}, s, sc));
  if (gr->d_w1) RP_TRY(gemm({c->hb, d, 1, du, h, 1, d, h, T, RP_EPI_F32, gr->d_w1, h}, s, sc));
  RP_TRY(gemm({du, h, 0, c->w0, h, 0, T, d, h, RP_EPI_BF16, dh, d}, s, sc));
  RP_TRY(rp_layer_norm_bwd(c->x, c->mean, c->rstd, p->ln_gamma, dh, nullptr, T, d, d_x, nullptr,
                           gr->d_ln_gamma, gr->d_ln_beta, lnws, 0, s));
  return rp_check_launch("mlp_vjp");
}

extern "C" int64_t rp_layer_cache_bytes(const RpLayerCache* c) { return c ? c->bytes : -1; }

extern "C" int rp_layer_cache_destroy(RpLayerCache* c) {
  if (!c) return RP_OK;
  for (void* q : c->bufs) cudaFreeAsync(q, c->stream);
  delete c;
  return RP_OK;
}

// ---------------------------------------------------------------- revcore
namespace {
int block_check(const RpRevBlockDev* b, int64_t batch, int64_t tokens) {
  if (!b) return rp_fail(RP_ERR_CONTRACT, "rev block: null block");
  if (b->f.width != b->g.width)
    return rp_fail(RP_ERR_SHAPE, "rev block: F and G disagree on the model width");
  return check_rows(batch, tokens, b->f.width);
}
}  // namespace

// o2 = i2 + F(i1); o1 = i1 + G(o2); stores nothing
extern "C" int rp_rev_forward(const RpRevBlockDev* b, int64_t batch, int64_t tokens,
                              const float* i1, const float* i2, float* o1, float* o2,
                              rp_stream_t stream) {
  RP_TRY(block_check(b, batch, tokens));
  if (!i1 || !i2 || !o1 || !o2) return rp_fail(RP_ERR_CONTRACT, "rev_forward: null tensor");
  const int64_t n = batch * tokens * b->f.width;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Scratch sc(s);
  float* y = nullptr;
  RP_TRY(sc.get(&y, n));
  RP_TRY(rp_attention_forward(&b->f, i1, batch, tokens, y, nullptr, stream));
  RP_TRY(rpk_axpy_sign(i2, y, 1.f, o2, n, s));
  RP_TRY(rp_mlp_forward(&b->g, o2, batch, tokens, y, nullptr, stream));
  return rpk_axpy_sign(i1, y, 1.f, o1, n, s);
}

// i1 = o1 - G(o2); i2 = o2 - F(i1): one F and one G evaluation
extern "C" int rp_rev_inverse(const RpRevBlockDev* b, int64_t batch, int64_t tokens,
                              const float* o1, const float* o2, float* i1, float* i2,
                              rp_stream_t stream) {
  RP_TRY(block_check(b, batch, tokens));
  if (!i1 || !i2 || !o1 || !o2) return rp_fail(RP_ERR_CONTRACT, "rev_inverse: null tensor");
  const int64_t n = batch * tokens * b->f.width;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Scratch sc(s);
  float* y = nullptr;
  RP_TRY(sc.get(&y, n));
  RP_TRY(rp_mlp_forward(&b->g, o2, batch, tokens, y, nullptr, stream));
  RP_TRY(rpk_axpy_sign(o1, y, -1.f, i1, n, s));
  RP_TRY(rp_attention_forward(&b->f, i1, batch, tokens, y, nullptr, stream));
  return rpk_axpy_sign(o2, y, -1.f, i2, n, s);
}

// Fused recompute + VJP: recompute (i1, i2) caching F/G once; then
// d_i2 = d_o2 + VJP_G(d_o1), d_i1 = d_o1 + VJP_F(d_i2) -- G path before F path;
// caches die on return.
extern "C" int rp_rev_backward_local(const RpRevBlockDev* b, int64_t batch, int64_t tokens,
                                     const float* o1, const float* o2, const float* d_o1,
                                     const float* d_o2, float* i1, float* i2, float* d_i1,
                                     float* d_i2, const RpRevBlockGradsDev* gr,
                                     rp_stream_t stream) {
  RP_TRY(block_check(b, batch, tokens));
  if (!o1 || !o2 || !d_o1 || !d_o2 || !i1 || !i2 || !d_i1 || !d_i2 || !gr)
    return rp_fail(RP_ERR_CONTRACT, "rev_backward_local: null tensor");
  const int64_t n = batch * tokens * b->f.width;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Scratch sc(s);
  float *y = nullptr, *dx = nullptr;
  RP_TRY(sc.get(&y, n));
  RP_TRY(sc.get(&dx, n));
  RpLayerCache *cg = nullptr, *cf = nullptr;
  int rc = rp_mlp_forward(&b->g, o2, batch, tokens, y, &cg, stream);
  if (rc == RP_OK) rc = rpk_axpy_sign(o1, y, -1.f, i1, n, s);
  if (rc == RP_OK) rc = rp_attention_forward(&b->f, i1, batch, tokens, y, &cf, stream);
  if (rc == RP_OK) rc = rpk_axpy_sign(o2, y, -1.f, i2, n, s);
  if (rc == RP_OK) rc = rp_mlp_vjp(cg, &b->g, d_o1, dx, &gr->d_g, stream);
  if (rc == RP_OK) rc = rpk_axpy_sign(d_o2, dx, 1.f, d_i2, n, s);
  if (rc == RP_OK) rc = rp_attention_vjp(cf, &b->f, d_i2, dx, &gr->d_f, stream);
  if (rc == RP_OK) rc = rpk_axpy_sign(d_o1, dx, 1.f, d_i1, n, s);
  rp_layer_cache_destroy(cg);
  rp_layer_cache_destroy(cf);
  return rc;
}

// theta <- theta - lr * g, fp32 with no contraction: bit-identical to the
// host's p - lr * g
extern "C" int rp_sgd_update(float* params, const float* grads, int64_t n, float lr,
                             rp_stream_t stream) {
  if (n < 0 || (n > 0 && (!params || !grads)))
    return rp_fail(RP_ERR_CONTRACT, "sgd_update: missing grads");
  if (n == 0) return RP_OK;
  return rpk_sgd_value(params, grads, n, lr, static_cast<cudaStream_t>(stream));
}
