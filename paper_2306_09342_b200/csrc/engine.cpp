// The reversible training engine (host C++ over the sm_100a kernels).
//
// Implements the SPEC's engines module on one B200, for the isotropic model and the
// hierarchical (Rev-Swin-style) one -- stages of blocks joined by fuse + patch_merge
// boundaries (ref:proj/core/src/layers.cpp:261-303):
//   step_reprop  forward storing only the stage boundary, backward
//                                     block L..1 with fused recompute + VJP, one lane
//   step_pareprop  the same work split over two CUDA streams: lane R
//                                     recomputes block i-1 while lane G runs block i's VJP
//   sgd_update  per-bucket, overlapped with the backward
// plus data parallelism over the GPUs of one box: one fp32 gradient bucket per block,
// ncclAllReduce'd on a comm stream as soon as lane G finishes that block.
//
// Memory is a static arena sized at creation; the step never allocates (the paper's
// "synchronous memory freeing" pitfall, §3.3, cannot occur). The coupled residual
// stream and all cotangents are fp32; GEMM operands are bf16 shadows.
//
// Buffer rotation, per stage (stage-local block j maps X_j -> X_{j+1}; X_0 = (e, e) is the
// stored stage input): X_j.i1 lives in the stage's buf1[j % 2], X_j.i2 in buf2[j % 3]
// (j >= 1), so the stage output X_L stays intact for the backward.
// Block caches live in slot[b % 2] with b the GLOBAL block index (slots are shared by all
// stages, sized for the largest). R(b) writes buf1[j%2], buf2[j%3], slot[b%2]: exactly what
// VJP(b+2) reads, so R(b) waits on G_done[b+2] -- the capacity-1 rendezvous of
// SPEC.md:381/415/420 (R at most one block ahead, <= 2 blocks of caches live), applied
// across stage boundaries too.
// Every kernel's arithmetic is independent of grid size and stream co-residency, so
// PaReprop reproduces Reprop bit for bit.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/revprop_b200.h"
#include "kernels.h"
#include "model_kernels.h"

namespace {

constexpr int kSms = 148;

struct Slot {
  uint16_t *hF = nullptr, *qkv = nullptr, *att = nullptr, *hG = nullptr, *u = nullptr,
           *a = nullptr;
  float *lse = nullptr, *meanF = nullptr, *rstdF = nullptr, *meanG = nullptr, *rstdG = nullptr;
};

struct BlockPlans {
  // lane R (recompute) -- also used by the forward with +1 residual sign
  RpGemmPlan *r_w1 = nullptr, *r_w2 = nullptr, *r_qkv = nullptr, *r_proj = nullptr;
  RpGemmPlan *f_qkv = nullptr, *f_proj = nullptr, *f_w1 = nullptr, *f_w2 = nullptr;
  // lane G (VJP)
  RpGemmPlan *g_dw2 = nullptr, *g_ww2 = nullptr, *g_ww1 = nullptr, *g_dw1 = nullptr,
             *g_dproj = nullptr, *g_wproj = nullptr, *g_wqkv = nullptr, *g_dqkv = nullptr;
};

// GEMM tiling used by the engine: CTA-pair (cta_group::2) 256 x 256 tiles.
constexpr int kGemmBn = 512;

// Narrow outputs (the Rev-Swin stages of width 128 / 384) waste a large part of a 256-wide
// CTA-pair tile; they run on single-CTA 128 x 128 tiles instead.
int gemm_bn(int64_t N) { return (N % 256 != 0 && N < 512) ? 128 : kGemmBn; }

// Split-K count for a weight-gradient GEMM: minimise (waves of work units) x (k-blocks per
// split) x (time per k-block per tile) + the extra HBM traffic splitting costs (s fp32
// partial tiles written instead of one, then read back and reduced: 2 s M N 4 bytes).
// Counting only wave efficiency picked 10 splits for G48's QKV wgrad (1664 x 4992, K =
// 12608): ~300 MB of partials + a 55 us reduction to save 4 % of a 165 us GEMM.
int pick_splits(int64_t M, int64_t N, int64_t K, int bn) {
  const bool pair = bn == 512;
  const int tm = pair ? 256 : 128, tn = pair ? 256 : bn;
  const int slots = pair ? kSms / 2 : kSms;
  const int64_t tiles = ((M + tm - 1) / tm) * ((N + tn - 1) / tn);
  const int64_t kb = (K + 63) / 64;
  // ~0.42 us per 64-deep k-block of a 128 x 256 tile per SM (or 256 x 256 per CTA pair) at
  // ~10 TFLOP/s per SM; ~6 TB/s of HBM for the partials
  const double t_kb = 0.42e-6 * (pair ? 1.0 : static_cast<double>(tn) / 256.0);
  const double t_byte = 1.0 / 6.0e12;
  int best = 1;
  double best_t = 0.0;
  for (int s = 1; s <= 64; ++s) {
    if (s > 1 && kb / s < 8) break;  // keep >= 8 k-blocks per split
    const int64_t units = tiles * s;
    const double waves = static_cast<double>((units + slots - 1) / slots);
    const double t = waves * static_cast<double>((kb + s - 1) / s) * t_kb +
                     (s > 1 ? 2.0 * s * static_cast<double>(M) * static_cast<double>(N) * 4.0 * t_byte : 0.0);
    if (s == 1 || t < best_t * (1.0 - 1e-6)) {
      best_t = t;
      best = s;
    }
  }
  return best;
}

}  // namespace

// One stage of blocks (an isotropic model has one). Geometry, the stored stage input e
// (i1 = i2 = e), the rotating X buffers, and the boundary that follows it.
struct RpStage {
  int64_t L = 0, first = 0;                   // blocks, global index of the first block
  int64_t N = 0, d = 0, h = 0, H = 0, W = 0;  // tokens, width, hidden, heads, window
  int64_t T = 0, block_size = 0;              // rows (batch x tokens), params per block
  float* e = nullptr;
  float* buf1[2] = {nullptr, nullptr};
  float* buf2[3] = {nullptr, nullptr, nullptr};
  int64_t stash_off = 0;  // Vanilla stash offset of X_1 (floats)
  // ledger quantities (bytes): block footprint, caches alone (Vanilla),
  // stored stage input + output, Vanilla stash
  int64_t led_block = 0, led_cache = 0, led_store = 0, led_stash = 0;
  // boundary after this stage (ref layers.hpp:144-149): merge_w [(r d), d_next] then
  // fusion_w [2d, d] (mlp fusion); -1 for the last stage
  int64_t bnd_tix = -1, bnd_size = 0;
  RpGemmPlan *b_fuse = nullptr, *b_merge = nullptr, *b_dmerge = nullptr, *b_wmerge = nullptr,
             *b_dfuse1 = nullptr, *b_dfuse2 = nullptr, *b_wfuse = nullptr;
};

struct RpEngine {
  RpModelConfig cfg{};
  // B, in, C; L = total blocks; T = B * N input rows (stage 0)
  int64_t B = 0, N = 0, in = 0, C = 0, L = 0, T = 0;
  int64_t P = 0;
  std::vector<RpStage> st;
  std::vector<int> stage_of;        // global block -> stage
  std::vector<int64_t> blk_tix;     // global block -> tensor index of its w_qkv
  int64_t head_tix = 0;
  int64_t r = 2;                    // tokens merged per boundary group
  int fusion = 0;                   // 0 average, 1 mlp (BoundaryParams.fusion_kind)
  std::vector<int64_t> t_off, t_numel;  // flat tensor table
  std::vector<int> t_kind;              // init kind: 0 weight, 1 zero (bias, beta), 2 one
  int dev = 0;
  cudaStream_t sG = nullptr, sR = nullptr, sC = nullptr;
  // input pipelining (rp_engine_prefetch_batch): copy stream, staging buffers, events
  cudaStream_t sX = nullptr;
  uint16_t* in_stage = nullptr;
  int32_t* lab_stage = nullptr;
  cudaEvent_t evStaged = nullptr, evStageFree = nullptr, evLoss = nullptr;
  bool staged = false;
  std::vector<cudaEvent_t> evR, evG;
  cudaEvent_t evFwd = nullptr, evCommDone = nullptr, evRDone = nullptr, evEmbed = nullptr,
              evLogits = nullptr;
  std::vector<cudaEvent_t> ts;  // timing events for the slot log (eager, instrumented)
  bool instrument = false;
  // parameters
  float *params = nullptr, *grads = nullptr, *lr = nullptr, *lr_apply = nullptr;
  uint16_t* pb = nullptr;
  // data
  uint16_t* inputs = nullptr;
  int32_t* labels = nullptr;
  // activations
  float* e = nullptr;
  float* buf1[2] = {nullptr, nullptr};
  float* buf2[3] = {nullptr, nullptr, nullptr};
  Slot slot[2];
  // lane G temporaries
  float *d1 = nullptr, *d2 = nullptr;
  uint16_t *d1b = nullptr, *d2b = nullptr, *du = nullptr, *dh = nullptr, *datt = nullptr,
           *dqkv = nullptr, *deb = nullptr;
  // boundary recompute (fused stage output, bf16 [T, d]; mlp: concat [T, 2d]) and its events
  uint16_t *fb = nullptr, *cb = nullptr;
  std::vector<cudaEvent_t> evBnd, evFuse;
  float *ln_ws = nullptr, *col_ws = nullptr, *split_ws = nullptr, *attn_ws = nullptr;
  // head
  float *pooled = nullptr, *logits = nullptr, *dlogits = nullptr, *row_loss = nullptr,
        *loss = nullptr, *dpooled = nullptr;
  std::vector<BlockPlans> plans;
  RpGemmPlan *p_embed = nullptr, *p_embed_w = nullptr;
  std::vector<RpGemmPlan*> all_plans;
  // graphs: index by mode (1 reprop, 2 pareprop)
  cudaGraphExec_t graph[3] = {nullptr, nullptr, nullptr};  // by mode: 0 vanilla, 1, 2
  // NCCL
  ncclComm_t comm = nullptr;
  int world = 1, rank = 0;
  int r_ctas = 0, g_ctas = 0;  // PaReprop SM partition (0 = all)
  std::vector<void*> allocs;
  // live GEMM profiling (eager steps only)
  bool prof = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> prof_ev;
  std::vector<double> prof_flops;
  size_t prof_used = 0;
  int64_t graph_kernels[3] = {0, 0, 0};
  // Vanilla engine: every block's input pair is stored in the forward
  float *stash1 = nullptr, *stash2 = nullptr;  // per stage: X_1..X_L, [L][T*d] each
  bool vanilla_ready = false, vmode = false;
  std::vector<RpGemmPlan*> vf_proj, vf_w2;
  // optimizer: 0 SGD, 1 AdamW
  int optimizer = 0;
  float beta1 = 0.9f, beta2 = 0.999f, eps = 1e-8f, wd = 0.f;
  float *adam_m = nullptr, *adam_v = nullptr, *step_t = nullptr;
  int fault = 0;  // test hook: 1 = corrupt every block's F-path VJP
  // caller-stream ordering of the block / layer entry points: work the caller enqueued on
  // `caller` (default: the legacy default stream) before the call is complete before the
  // engine reads the caller's device pointers
  cudaStream_t caller = nullptr;
  cudaEvent_t evCaller = nullptr;
  // recompute trace (eager steps): every block's input pair as the forward saw it and as
  // lane R reconstructed it, [sum_b 2 T_s d_s] floats each, block b at trace_off[b]
  float *trace_fwd = nullptr, *trace_rec = nullptr;
  std::vector<int64_t> trace_off;
  // arena bookkeeping (bytes actually allocated, by category) and the live ledger replay of
  // the last enqueued step's schedule (ref ledger.hpp:18-104)
  int64_t arena_bytes[3] = {0, 0, 0};  // 0 other, 1 activations, 2 params / grads / state
  int64_t led_live = 0, led_peak = 0, led_events = 0, blocks_processed = 0, led_fixed = 0;
  std::vector<int64_t> led_held;  // per block: bytes charged and not yet released
  int led_error = 0;
  // last step: timing events around it on the engine stream, whether it was instrumented
  cudaEvent_t evStepBeg = nullptr, evStepEnd = nullptr;
  bool step_timed = false, step_instrumented = false;
  int last_mode = -1;
  // ledger results of the last enqueue of each mode (a graph replay re-runs that schedule)
  int64_t led_peak_m[3] = {0, 0, 0}, led_events_m[3] = {0, 0, 0}, blocks_m[3] = {0, 0, 0};
  // gradient buckets (offset, floats) by owner, from the shared bucket plan
  std::pair<int64_t, int64_t> bk_head{0, 0}, bk_embed{0, 0};
  std::vector<std::pair<int64_t, int64_t>> bk_block, bk_bnd;
  int comm_reserve = 0;  // SMs kept free of GEMM CTAs for the NCCL kernels (world > 1)
  float quantum = 0.f;   // exact-coupling grid 2^-bits of the residual stream (0 = off)
  // diagnostic schedule flags (rp_engine_set_diag; timing experiments only, results are
  // garbage): 1 lanes R and G free-running (no rendezvous events), 2 skip lane G's kernels,
  // 4 skip lane R's kernels
  int diag = 0;
};

namespace {

#define RP_TRY(x)                 \
  do {                            \
    int rc_ = (x);                \
    if (rc_ != RP_OK) return rc_; \
  } while (0)

int cuda_ok(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return RP_OK;
  std::string m = std::string(what) + ": " + cudaGetErrorString(e);
  return rp_fail(RP_ERR_CUDA, m.c_str());
}

// cat: 0 workspace / other, 1 activation storage (what the ledger accounts), 2 parameters,
// gradients and optimizer state
template <class T>
int dalloc(RpEngine* g, T** p, int64_t count, int cat = 0) {
  void* q = nullptr;
  const size_t bytes = static_cast<size_t>(count > 0 ? count : 1) * sizeof(T);
  cudaError_t e = cudaMalloc(&q, bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();  // not sticky: do not leak it into the next launch check
    std::string m = "device allocation of " + std::to_string(bytes) + " bytes failed: " +
                    cudaGetErrorString(e);
    return rp_fail(RP_ERR_BUDGET, m.c_str());
  }
  g->allocs.push_back(q);
  g->arena_bytes[cat] += static_cast<int64_t>(bytes);
  *p = static_cast<T*>(q);
  return RP_OK;
}

// The block / layer entry points read caller device pointers on the engine stream: order
// them after everything the caller enqueued on its stream (default: the legacy stream,
// torch's default) before the call.
int wait_caller(RpEngine* g) {
  cudaStream_t cs = g->caller ? g->caller : cudaStreamLegacy;
  RP_TRY(cuda_ok(cudaEventRecord(g->evCaller, cs), "record caller stream"));
  return cuda_ok(cudaStreamWaitEvent(g->sG, g->evCaller, 0), "wait caller stream");
}

// tensor index helpers (flat order, SPEC.md:279-282 Model fields)
enum BlockTensor { kWqkv = 0, kWout, kLnFg, kLnFb, kW1, kB1, kW2, kB2, kLnGg, kLnGb, kPerBlock };
inline int64_t tix_block(const RpEngine* g, int64_t b, int t) {
  return g->blk_tix[static_cast<size_t>(b)] + t;
}
inline RpStage& stage_of(RpEngine* g, int64_t b) {
  return g->st[static_cast<size_t>(g->stage_of[static_cast<size_t>(b)])];
}

struct GemmArgs {
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
  void* out2 = nullptr;
  const void* aux = nullptr;
  int64_t ldaux = 0;
  const float* bias = nullptr;
  float sign = 1.f;
  int splits = 1;
  float* ws = nullptr;
  float* colsum_part = nullptr;
  float* rowdot = nullptr;
  int64_t rd_seq = 0;
  float quantum = 0.f;  // exact-coupling grid of a residual-stream output
};

// the tcgen05 attention backward with the stored dS^T (head_dim 64, <= 256 tokens per
// window) takes D = rowsum(dO * O) from the d_att GEMM's ROWDOT epilogue
inline bool fused_attn_bwd(const RpStage& St) { return St.d / St.H == 64 && St.W <= 256; }

int mk_plan(RpEngine* g, const GemmArgs& a, RpGemmPlan** out) {
  RpGemmDesc d{};
  d.A = a.A;
  d.lda = a.lda;
  d.a_mn = a.a_mn;
  d.B = a.B;
  d.ldb = a.ldb;
  d.b_mn = a.b_mn;
  d.M = a.M;
  d.N = a.N;
  d.K = a.K;
  d.epi = a.epi;
  d.out = a.out;
  d.ldo = a.ldo;
  d.out2 = a.out2;
  d.ldo2 = a.ldo;
  d.aux = a.aux;
  d.ldaux = a.ldaux ? a.ldaux : a.ldo;
  d.bias = a.bias;
  d.sign = a.sign;
  d.splits = a.splits;
  d.workspace = a.ws;
  d.colsum_part = a.colsum_part;
  d.rowdot = a.rowdot;
  d.rd_seq = a.rd_seq;
  d.quantum = a.quantum;
  d.max_ctas = 0;
  d.bn = gemm_bn(a.N);
  int rc = rp_gemm_plan_create(&d, out);
  if (rc != RP_OK) return rp_fail(rc, "engine: gemm plan creation failed");
  g->all_plans.push_back(*out);
  return RP_OK;
}

const uint16_t* wb(const RpEngine* g, int64_t tix) { return g->pb + g->t_off[tix]; }
const float* wf(const RpEngine* g, int64_t tix) { return g->params + g->t_off[tix]; }
float* gr(const RpEngine* g, int64_t tix) { return g->grads + g->t_off[tix]; }

// X_j storage (stage-local j): rotating buffers for Reprop / PaReprop, the stash for Vanilla.
float* X1(RpEngine* g, const RpStage& S, int64_t j) {
  if (j == 0) return S.e;
  return g->vmode ? g->stash1 + S.stash_off + (j - 1) * S.T * S.d : S.buf1[j % 2];
}
float* X2(RpEngine* g, const RpStage& S, int64_t j) {
  if (j == 0) return S.e;
  return g->vmode ? g->stash2 + S.stash_off + (j - 1) * S.T * S.d : S.buf2[j % 3];
}

int build_plans(RpEngine* g) {
  g->plans.resize(static_cast<size_t>(g->L));
  for (size_t si = 0; si < g->st.size(); ++si) {
    RpStage& St = g->st[si];
    const int64_t T = St.T, d = St.d, h = St.h;
    const int s_qkv = pick_splits(d, 3 * d, T, gemm_bn(3 * d)),
              s_proj = pick_splits(d, d, T, gemm_bn(d)), s_w1 = pick_splits(d, h, T, gemm_bn(h)),
              s_w2 = pick_splits(h, d, T, gemm_bn(d));
    for (int64_t j = 0; j < St.L; ++j) {
      const int64_t b = St.first + j;
      BlockPlans& p = g->plans[static_cast<size_t>(b)];
      Slot& S = g->slot[b % 2];
      Slot& F = g->slot[0];  // forward temporaries
      const uint16_t *Wqkv = wb(g, tix_block(g, b, kWqkv)), *Wout = wb(g, tix_block(g, b, kWout)),
                     *W1 = wb(g, tix_block(g, b, kW1)), *W2 = wb(g, tix_block(g, b, kW2));
      const float *b1 = wf(g, tix_block(g, b, kB1)), *b2 = wf(g, tix_block(g, b, kB2));
      // ---- forward (stores nothing)
      RP_TRY(mk_plan(g, {F.hF, d, 0, Wqkv, 3 * d, 1, T, 3 * d, d, RP_EPI_BF16, F.qkv, 3 * d},
                     &p.f_qkv));
      {
        GemmArgs a{F.att, d, 0, Wout, d, 1, T, d, d, RP_EPI_RESID, X2(g, St, j + 1), d};
        a.aux = X2(g, St, j);
        a.quantum = g->quantum;
        RP_TRY(mk_plan(g, a, &p.f_proj));
      }
      {
        GemmArgs a{F.hF, d, 0, W1, h, 1, T, h, d, RP_EPI_BIAS_GELU, F.a, h};
        a.bias = b1;
        RP_TRY(mk_plan(g, a, &p.f_w1));
      }
      {
        GemmArgs a{F.a, h, 0, W2, d, 1, T, d, h, RP_EPI_RESID, X1(g, St, j + 1), d};
        a.aux = X1(g, St, j);
        a.bias = b2;
        a.quantum = g->quantum;
        RP_TRY(mk_plan(g, a, &p.f_w2));
      }
      // ---- lane R: inverse with caches
      {  // keeps gelu'(u) (not u) for the MLP dgrad: slot.u holds the slope
        GemmArgs a{S.hG, d, 0, W1, h, 1, T, h, d, RP_EPI_BIAS_GELU_SLOPE, S.a, h};
        a.out2 = S.u;
        a.bias = b1;
        RP_TRY(mk_plan(g, a, &p.r_w1));
      }
      RP_TRY(mk_plan(g, {S.hF, d, 0, Wqkv, 3 * d, 1, T, 3 * d, d, RP_EPI_BF16, S.qkv, 3 * d},
                     &p.r_qkv));
      if (j > 0) {
        GemmArgs a{S.a, h, 0, W2, d, 1, T, d, h, RP_EPI_RESID, X1(g, St, j), d};
        a.aux = X1(g, St, j + 1);
        a.bias = b2;
        a.sign = -1.f;
        a.quantum = g->quantum;
        RP_TRY(mk_plan(g, a, &p.r_w2));
        GemmArgs c{S.att, d, 0, Wout, d, 1, T, d, d, RP_EPI_RESID, X2(g, St, j), d};
        c.aux = X2(g, St, j + 1);
        c.sign = -1.f;
        c.quantum = g->quantum;
        RP_TRY(mk_plan(g, c, &p.r_proj));
      }
      // ---- lane G: VJPs (layers.cpp:171-220, 241-259)
      {
        GemmArgs a{g->d1b, d, 0, W2, d, 0, T, h, d, RP_EPI_MUL, g->du, h};
        a.aux = S.u;
        a.colsum_part = g->col_ws;        // + per-32-row column sums of d_u (-> db1)
        RP_TRY(mk_plan(g, a, &p.g_dw2));  // d_u = gelu'(u) * (d_o1 . W2^T)
      }
      {
        GemmArgs a{S.a, h, 1, g->d1b, d, 1, h, d, T, RP_EPI_F32, gr(g, tix_block(g, b, kW2)), d};
        a.splits = s_w2;
        a.ws = g->split_ws;
        RP_TRY(mk_plan(g, a, &p.g_ww2));  // dW2 = a^T d_o1
      }
      {
        GemmArgs a{S.hG, d, 1, g->du, h, 1, d, h, T, RP_EPI_F32, gr(g, tix_block(g, b, kW1)), h};
        a.splits = s_w1;
        a.ws = g->split_ws;
        RP_TRY(mk_plan(g, a, &p.g_ww1));  // dW1 = hG^T d_u
      }
      RP_TRY(mk_plan(g, {g->du, h, 0, W1, h, 0, T, d, h, RP_EPI_BF16, g->dh, d}, &p.g_dw1));
      if (fused_attn_bwd(St)) {  // d_att GEMM also emits D = rowsum(d_att * att) per head
        GemmArgs a{g->d2b, d, 0, Wout, d, 0, T, d, d, RP_EPI_ROWDOT, g->datt, d};
        a.aux = S.att;
        a.rowdot = g->attn_ws;
        a.rd_seq = St.W;
        RP_TRY(mk_plan(g, a, &p.g_dproj));
      } else {
        RP_TRY(mk_plan(g, {g->d2b, d, 0, Wout, d, 0, T, d, d, RP_EPI_BF16, g->datt, d}, &p.g_dproj));
      }
      {
        GemmArgs a{S.att, d, 1, g->d2b, d, 1, d, d, T, RP_EPI_F32, gr(g, tix_block(g, b, kWout)), d};
        a.splits = s_proj;
        a.ws = g->split_ws;
        RP_TRY(mk_plan(g, a, &p.g_wproj));
      }
      {
        GemmArgs a{S.hF, d, 1, g->dqkv, 3 * d, 1, d, 3 * d, T, RP_EPI_F32,
                   gr(g, tix_block(g, b, kWqkv)), 3 * d};
        a.splits = s_qkv;
        a.ws = g->split_ws;
        RP_TRY(mk_plan(g, a, &p.g_wqkv));
      }
      RP_TRY(mk_plan(g, {g->dqkv, 3 * d, 0, Wqkv, 3 * d, 0, T, d, 3 * d, RP_EPI_BF16, g->dh, d},
                     &p.g_dqkv));
    }
    // ---- boundary after this stage (layers.cpp:261-303): f = fuse(o1, o2) (bf16, recomputed
    // from the stored stage output in the backward), e_next = group_r(f) . merge_w (fp32)
    if (St.bnd_tix >= 0) {
      const RpStage& Nx = g->st[si + 1];
      const int64_t rd = g->r * d, dn = Nx.d, Tn = Nx.T;
      const uint16_t* Mw = wb(g, St.bnd_tix);
      if (g->fusion == 1)  // f = concat(o1, o2) . fusion_w
        RP_TRY(mk_plan(g, {g->cb, 2 * d, 0, wb(g, St.bnd_tix + 1), d, 1, T, d, 2 * d, RP_EPI_BF16,
                           g->fb, d},
                       &St.b_fuse));
      {
        GemmArgs a{g->fb, rd, 0, Mw, dn, 1, Tn, dn, rd, RP_EPI_F32, Nx.e, dn};
        a.quantum = g->quantum;  // the next stage's input starts on the grid
        RP_TRY(mk_plan(g, a, &St.b_merge));
      }
      // d_f = d_y . merge_w^T  ([Tn, r d] == [T, d] row-major): fp32 into d1 (average
      // fusion: d_i1 = d_i2 = d_f / 2 next), bf16 into datt (mlp: the operand of two GEMMs)
      if (g->fusion == 1)
        RP_TRY(mk_plan(g, {g->deb, dn, 0, Mw, dn, 0, Tn, rd, dn, RP_EPI_BF16, g->datt, rd},
                       &St.b_dmerge));
      else
        RP_TRY(mk_plan(g, {g->deb, dn, 0, Mw, dn, 0, Tn, rd, dn, RP_EPI_F32, g->d1, rd},
                       &St.b_dmerge));
      {  // d_merge_w = group_r(f)^T . d_y
        GemmArgs a{g->fb, rd, 1, g->deb, dn, 1, rd, dn, Tn, RP_EPI_F32, gr(g, St.bnd_tix), dn};
        a.splits = pick_splits(rd, dn, Tn, gemm_bn(dn));
        a.ws = g->split_ws;
        RP_TRY(mk_plan(g, a, &St.b_wmerge));
      }
      if (g->fusion == 1) {
        // d_i1 = d_f . fusion_w[0:d]^T, d_i2 = d_f . fusion_w[d:2d]^T (fp32), d_f bf16 in datt
        const uint16_t* Fw = wb(g, St.bnd_tix + 1);
        RP_TRY(mk_plan(g, {g->datt, d, 0, Fw, d, 0, T, d, d, RP_EPI_F32, g->d1, d}, &St.b_dfuse1));
        RP_TRY(mk_plan(g, {g->datt, d, 0, Fw + d * d, d, 0, T, d, d, RP_EPI_F32, g->d2, d},
                       &St.b_dfuse2));
        GemmArgs a{g->cb, 2 * d, 1, g->datt, d, 1, 2 * d, d, T, RP_EPI_F32,
                   gr(g, St.bnd_tix + 1), d};
        a.splits = pick_splits(2 * d, d, T, gemm_bn(d));
        a.ws = g->split_ws;
        RP_TRY(mk_plan(g, a, &St.b_wfuse));  // d_fusion_w = concat^T . d_f
      }
    }
  }
  // embedding: e = x . embed_w ; d_embed_w = x^T . (d_i1 + d_i2)
  const RpStage& S0 = g->st[0];
  {
    GemmArgs a{g->inputs, g->in, 0, wb(g, 0), S0.d, 1, g->T, S0.d, g->in, RP_EPI_F32, S0.e, S0.d};
    a.quantum = g->quantum;  // the residual stream starts on the exact-coupling grid
    RP_TRY(mk_plan(g, a, &g->p_embed));
  }
  {
    GemmArgs a{g->inputs, g->in, 1, g->deb, S0.d, 1, g->in, S0.d, g->T, RP_EPI_F32, gr(g, 0), S0.d};
    a.splits = pick_splits(g->in, S0.d, g->T, gemm_bn(S0.d));
    a.ws = g->split_ws;
    RP_TRY(mk_plan(g, a, &g->p_embed_w));
  }
  return RP_OK;
}

// GEMM timing (live roofline): when g->prof is set, every plan launch is bracketed by
// CUDA events on its own stream; rp_engine_gemm_profile() sums durations and FLOPs.
struct GemmProf {
  cudaEvent_t a, b;
  double flops;
};
thread_local RpEngine* t_prof_engine = nullptr;

int launch(RpGemmPlan* p, cudaStream_t s);

int launch(RpGemmPlan* p, cudaStream_t s) {
  RpEngine* g = t_prof_engine;
  if (!g || !g->prof) return rp_gemm_plan_launch(p, s);
  if (g->prof_used == g->prof_ev.size()) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    g->prof_ev.push_back({a, b});
    g->prof_flops.push_back(0.0);
  }
  auto& ev = g->prof_ev[g->prof_used];
  int64_t M, N, K;
  rp_gemm_plan_shape(p, &M, &N, &K);
  g->prof_flops[g->prof_used] = 2.0 * static_cast<double>(M) * N * K;
  ++g->prof_used;
  cudaEventRecord(ev.first, s);
  const int rc = rp_gemm_plan_launch(p, s);
  cudaEventRecord(ev.second, s);
  return rc;
}

int ln_fwd(RpEngine* g, const RpStage& St, const float* x, int64_t tg, int64_t tb, uint16_t* y,
           float* mean, float* rstd, cudaStream_t s) {
  return rp_layer_norm_fwd(x, wf(g, tg), wf(g, tb), St.T, St.d, 1e-5, y, mean, rstd, s);
}

int attn_fwd(const RpStage& St, const uint16_t* qkv, uint16_t* att, float* lse, cudaStream_t s) {
  return rp_attention_fwd(qkv, St.T / St.W, St.W, St.H, St.d / St.H, att, lse, s);
}

void mark(RpEngine* g, int lane, int64_t b, int which, cudaStream_t s) {
  if (!g->instrument) return;
  cudaEventRecord(g->ts[static_cast<size_t>(((lane * g->L) + b) * 2 + which)], s);
}

// f = fuse(o1, o2) of stage St's output into g->fb (bf16): average (layers.cpp:277-279) or
// concat . fusion_w (layers.cpp:283-286). Used by the forward and, from the stored stage
// output, by the backward.
int boundary_fuse(RpEngine* g, RpStage& St, cudaStream_t s) {
  const float *o1 = X1(g, St, St.L), *o2 = X2(g, St, St.L);
  if (g->fusion == 1) {
    RP_TRY(rpk_concat_bf16(o1, o2, St.T, St.d, g->cb, s));
    return launch(St.b_fuse, s);
  }
  return rpk_fuse_avg_bf16(o1, o2, St.T * St.d, g->fb, s);
}

// ---- live ledger (SPEC.md:346-349 ledger_track; ref ledger.hpp:18-104): the step's
// enqueue replays each activation buffer's lifetime as charge / release events, in the
// order the schedule's dependencies allow them on the device (a block's footprint lives
// from its recompute (lane R) until its VJP (lane G) is done; under PaReprop R(b) may only
// start once G(b+2) is done, the capacity-1 rendezvous). A release larger than the live
// total is the reference's AccountingError.
void led_charge(RpEngine* g, int64_t bytes) {
  g->led_live += bytes;
  g->led_peak = std::max(g->led_peak, g->led_live);
  ++g->led_events;
}
void led_release(RpEngine* g, int64_t bytes) {
  ++g->led_events;
  if (bytes > g->led_live) {
    g->led_error = 1;
    g->led_live = 0;
    return;
  }
  g->led_live -= bytes;
}
void led_release_block(RpEngine* g, int64_t b) {
  if (b < 0 || b >= g->L) return;
  int64_t& h = g->led_held[static_cast<size_t>(b)];
  if (h) led_release(g, h);
  h = 0;
}
void led_charge_block(RpEngine* g, int64_t b, int64_t bytes) {
  led_charge(g, bytes);
  g->led_held[static_cast<size_t>(b)] += bytes;
}

// recompute trace: block b's input pair into trace buffer `dst` (eager steps only)
int trace_pair(RpEngine* g, float* dst, int64_t b, cudaStream_t s) {
  if (!dst) return RP_OK;
  RpStage& St = stage_of(g, b);
  const int64_t j = b - St.first, n = St.T * St.d;
  float* o = dst + g->trace_off[static_cast<size_t>(b)];
  RP_TRY(cuda_ok(cudaMemcpyAsync(o, X1(g, St, j), static_cast<size_t>(n) * 4,
                                 cudaMemcpyDeviceToDevice, s), "trace"));
  return cuda_ok(cudaMemcpyAsync(o + n, X2(g, St, j), static_cast<size_t>(n) * 4,
                                 cudaMemcpyDeviceToDevice, s), "trace");
}

int forward(RpEngine* g, cudaStream_t s) {
  RP_TRY(launch(g->p_embed, s));
  Slot& F = g->slot[0];
  for (RpStage& St : g->st) {
    led_charge(g, g->vmode ? St.led_stash : St.led_store);  // stored stage boundaries
    for (int64_t j = 0; j < St.L; ++j) {
      const int64_t b = St.first + j;
      BlockPlans& p = g->plans[static_cast<size_t>(b)];
      RP_TRY(trace_pair(g, g->trace_fwd, b, s));
      RP_TRY(ln_fwd(g, St, X1(g, St, j), tix_block(g, b, kLnFg), tix_block(g, b, kLnFb), F.hF,
                    F.meanF, F.rstdF, s));
      RP_TRY(launch(p.f_qkv, s));
      RP_TRY(attn_fwd(St, F.qkv, F.att, F.lse, s));
      RP_TRY(launch(g->vmode ? g->vf_proj[static_cast<size_t>(b)] : p.f_proj, s));  // o2 = i2 + F(i1)
      RP_TRY(ln_fwd(g, St, X2(g, St, j + 1), tix_block(g, b, kLnGg), tix_block(g, b, kLnGb), F.hF,
                    F.meanF, F.rstdF, s));
      RP_TRY(launch(p.f_w1, s));
      RP_TRY(launch(g->vmode ? g->vf_w2[static_cast<size_t>(b)] : p.f_w2, s));  // o1 = i1 + G(o2)
    }
    if (St.bnd_tix >= 0) {  // fuse -> patch_merge -> duplicate
      RP_TRY(boundary_fuse(g, St, s));
      RP_TRY(launch(St.b_merge, s));
    }
  }
  return RP_OK;
}

int head(RpEngine* g, cudaStream_t s) {
  RpStage& Ls = g->st.back();
  const int64_t B = g->B, d = Ls.d, C = g->C;
  const float* hw = wf(g, g->head_tix);
  RP_TRY(rpk_pool(X1(g, Ls, Ls.L), X2(g, Ls, Ls.L), B, Ls.N, d, g->pooled, s));
  RP_TRY(rpk_simt_gemm(B, C, d, g->pooled, d, 1, hw, C, 1, g->logits, C, s));
  RP_TRY(rpk_cross_entropy(g->logits, g->labels, B, C, g->dlogits, g->row_loss, g->loss, s));
  // the head weight gradient goes to the comm stream (ahead of the head bucket's optimizer
  // step there), in parallel with d_pooled and the spread on the engine stream
  RP_TRY(cuda_ok(cudaEventRecord(g->evLogits, s), "record"));
  RP_TRY(cuda_ok(cudaStreamWaitEvent(g->sC, g->evLogits, 0), "wait"));
  RP_TRY(rpk_simt_gemm(d, C, B, g->pooled, 1, d, g->dlogits, C, 1, gr(g, g->head_tix), C, g->sC));
  RP_TRY(rpk_simt_gemm(B, d, C, g->dlogits, C, 1, hw, 1, C, g->dpooled, d, s));
  RP_TRY(rpk_spread(g->dpooled, B, Ls.N, d, g->d1, g->d2, g->d1b, g->d2b, s));
  return RP_OK;
}

// Lane R halves: G recomputes the MLP caches from X2_{j+1} (= o2) and, unless j == 0, the
// input i1 = o1 - G(o2); F recomputes the attention caches from X1_j (= i1) and, unless
// j == 0, i2 = o2 - F(i1). `inverse` = false keeps only the caches (the layer VJP entries).
int recompute_g(RpEngine* g, int64_t b, cudaStream_t s, bool inverse) {
  BlockPlans& p = g->plans[static_cast<size_t>(b)];
  RpStage& St = stage_of(g, b);
  const int64_t j = b - St.first;
  Slot& S = g->slot[b % 2];
  RP_TRY(ln_fwd(g, St, X2(g, St, j + 1), tix_block(g, b, kLnGg), tix_block(g, b, kLnGb), S.hG,
                S.meanG, S.rstdG, s));
  RP_TRY(launch(p.r_w1, s));
  if (inverse && j > 0 && !g->vmode) RP_TRY(launch(p.r_w2, s));  // i1 = o1 - G(o2)
  return RP_OK;
}
int recompute_f(RpEngine* g, int64_t b, cudaStream_t s, bool inverse) {
  BlockPlans& p = g->plans[static_cast<size_t>(b)];
  RpStage& St = stage_of(g, b);
  const int64_t j = b - St.first;
  Slot& S = g->slot[b % 2];
  RP_TRY(ln_fwd(g, St, X1(g, St, j), tix_block(g, b, kLnFg), tix_block(g, b, kLnFb), S.hF, S.meanF,
                S.rstdF, s));
  RP_TRY(launch(p.r_qkv, s));
  RP_TRY(attn_fwd(St, S.qkv, S.att, S.lse, s));
  if (inverse && j > 0 && !g->vmode) RP_TRY(launch(p.r_proj, s));  // i2 = o2 - F(i1)
  return RP_OK;
}

// Lane R: recompute block b's input and caches from its output X_{j+1}.
int lane_r(RpEngine* g, int64_t b, cudaStream_t s) {
  mark(g, 0, b, 0, s);
  RP_TRY(recompute_g(g, b, s, true));
  RP_TRY(recompute_f(g, b, s, true));
  RP_TRY(trace_pair(g, g->trace_rec, b, s));
  mark(g, 0, b, 1, s);
  return RP_OK;
}

// Lane G halves (layers.cpp:241-259 and 171-220). vjp_g: MLP VJP of d_o1 (d1 / d1b), adds
// LN_G^T(d_hG) to d2 in place (d_o2t = d_o2 + VJP_G(d_o1)). vjp_f: attention VJP of d_o2t
// (d2b), adds LN_F^T(d_hF) to d1 in place (d_i1 = d_o1 + VJP_F(d_o2t)).
// own_b2: this block's MLP output-bias grad from its incoming d_o1 (a column-sum pass); in
// a stage only the top block needs it, every other block's b2 grad is produced by the
// block above in the same pass that writes its d_o1 (next_b2, the F-path LN backward).
int vjp_g(RpEngine* g, int64_t b, cudaStream_t s, bool own_b2) {
  BlockPlans& p = g->plans[static_cast<size_t>(b)];
  RpStage& St = stage_of(g, b);
  const int64_t j = b - St.first;
  Slot& S = g->slot[b % 2];
  const int64_t T = St.T, d = St.d, h = St.h;
  // (the own-b2 column sum runs first: the d_u GEMM below writes its partials to col_ws)
  if (own_b2) RP_TRY(rp_colsum(g->d1, 0, T, d, gr(g, tix_block(g, b, kB2)), g->col_ws, 0, s));
  RP_TRY(launch(p.g_dw2, s));
  RP_TRY(launch(p.g_ww2, s));
  RP_TRY(launch(p.g_ww1, s));
  // db1 = colsum(d_u): per-32-row partials come out of the d_u GEMM's epilogue (fp32)
  RP_TRY(rp_colsum_parts(g->col_ws, (T + 31) / 32, h, gr(g, tix_block(g, b, kB1)), 0, s));
  RP_TRY(launch(p.g_dw1, s));
  // d_o2t = d_o2 + LN_G^T(d_hG)   (in place in d2 / d2b)
  return rp_layer_norm_bwd(X2(g, St, j + 1), S.meanG, S.rstdG, wf(g, tix_block(g, b, kLnGg)),
                           g->dh, g->d2, T, d, g->d2, g->d2b, gr(g, tix_block(g, b, kLnGg)),
                           gr(g, tix_block(g, b, kLnGb)), g->ln_ws, 0, s);
}
int vjp_f(RpEngine* g, int64_t b, cudaStream_t s, bool next_b2) {
  BlockPlans& p = g->plans[static_cast<size_t>(b)];
  RpStage& St = stage_of(g, b);
  const int64_t j = b - St.first;
  Slot& S = g->slot[b % 2];
  const int64_t T = St.T, d = St.d;
  RP_TRY(launch(p.g_dproj, s));
  RP_TRY(launch(p.g_wproj, s));
  RP_TRY(rp_attention_bwd_ex(S.qkv, S.att, S.lse, g->datt, T / St.W, St.W, St.H, d / St.H,
                             g->dqkv, g->attn_ws, fused_attn_bwd(St) ? 1 : 0, s));
  RP_TRY(launch(p.g_wqkv, s));
  RP_TRY(launch(p.g_dqkv, s));
  // d_i1 = d_o1 + LN_F^T(d_hF)    (in place in d1 / d1b); d_i2 = d_o2t (already in d2)
  return rp_layer_norm_bwd_ex(X1(g, St, j), S.meanF, S.rstdF, wf(g, tix_block(g, b, kLnFg)),
                              g->dh, g->d1, T, d, g->d1, g->d1b, gr(g, tix_block(g, b, kLnFg)),
                              gr(g, tix_block(g, b, kLnFb)),
                              next_b2 ? gr(g, tix_block(g, b - 1, kB2)) : nullptr, g->ln_ws, 0, s);
}

// Lane G: the VJP half of rev_backward_local, G-path before F-path.
int lane_g(RpEngine* g, int64_t b, cudaStream_t s, bool own_b2, bool next_b2) {
  const RpStage& St = stage_of(g, b);
  mark(g, 1, b, 0, s);
  RP_TRY(vjp_g(g, b, s, own_b2));
  RP_TRY(vjp_f(g, b, s, next_b2));
  if (g->fault == 1) RP_TRY(rpk_scale_pair(g->d1, g->d1b, St.T * St.d, 1.5f, s));  // injected fault
  mark(g, 1, b, 1, s);
  return RP_OK;
}

// bucket b (block params) -> allreduce (DP) -> SGD, on the comm stream
int bucket_update(RpEngine* g, int64_t off, int64_t n, cudaStream_t s) {
  if (g->comm) {
    ncclResult_t r = ncclAllReduce(g->grads + off, g->grads + off, static_cast<size_t>(n),
                                   ncclFloat32, ncclSum, g->comm, s);
    if (r != ncclSuccess) return rp_fail(RP_ERR_SCHEDULER, ncclGetErrorString(r));
  }
  if (g->optimizer == 1)
    return rpk_adamw(g->params + off, g->grads + off, g->pb + off, g->adam_m + off,
                     g->adam_v + off, n, g->lr, g->step_t, g->beta1, g->beta2, g->eps, g->wd,
                     1.0f / static_cast<float>(g->world), s);
  return rpk_sgd(g->params + off, g->grads + off, g->pb + off, n, g->lr,
                 1.0f / static_cast<float>(g->world), s);
}

// Backward through the boundary after stage St (layers.cpp:269-303), on lane G, entered with
// the next stage's input cotangents in d1/d2 (fp32): d_y = d_i1 + d_i2 (both halves of the
// next stage's input are y), then patch_merge_vjp and fuse_vjp leave stage St's output
// cotangents in d1/d2 (+ bf16 shadows). g->fb (and cb) hold fuse(St's output), recomputed
// by boundary_fuse before this runs (evFuse[s] when it ran on lane R).
int boundary_vjp(RpEngine* g, RpStage& St, cudaStream_t s) {
  const RpStage& Nx = g->st[static_cast<size_t>(&St - g->st.data()) + 1];
  RP_TRY(rpk_add_to_bf16(g->d1, g->d2, g->deb, Nx.T * Nx.d, s));
  RP_TRY(launch(St.b_wmerge, s));
  RP_TRY(launch(St.b_dmerge, s));
  const int64_t n = St.T * St.d;
  if (g->fusion == 1) {
    RP_TRY(launch(St.b_wfuse, s));
    RP_TRY(launch(St.b_dfuse1, s));
    RP_TRY(launch(St.b_dfuse2, s));
    RP_TRY(rpk_f32_to_bf16(g->d1, g->d1b, n, s));
    return rpk_f32_to_bf16(g->d2, g->d2b, n, s);
  }
  return rpk_halve_dup(g->d1, n, g->d2, g->d1b, g->d2b, s);  // d_i1 = d_i2 = d_f / 2
}

int enqueue_step_impl(RpEngine* g, int mode);

int enqueue_step(RpEngine* g, int mode) {
  g->vmode = mode == 0;
  // the live GEMM profiler looks its engine up through t_prof_engine while this step is
  // enqueued -- and only then: outside a step (block / layer entry points, other engines)
  // it must not point at an engine that may since have been destroyed
  t_prof_engine = g;
  g->prof_used = 0;
  const int rc = enqueue_step_impl(g, mode == 0 ? 1 : mode);
  t_prof_engine = nullptr;
  g->vmode = false;
  if (rc == RP_OK) {
    g->led_peak_m[mode] = g->led_peak;
    g->led_events_m[mode] = g->led_events;
    g->blocks_m[mode] = g->blocks_processed;
  }
  return rc;
}

int enqueue_step_impl(RpEngine* g, int mode) {
  cudaStream_t sG = g->sG, sR = g->sR, sC = g->sC;
  g->led_live = g->led_peak = g->led_events = g->blocks_processed = 0;
  g->led_error = 0;
  g->led_held.assign(static_cast<size_t>(g->L), 0);
  led_charge(g, g->led_fixed);  // cotangent pair + lane-G temporaries
  if (g->optimizer == 1) RP_TRY(rpk_add_scalar(g->step_t, 1.0f, sG));
  RP_TRY(forward(g, sG));
  RP_TRY(head(g, sG));
  RP_TRY(cuda_ok(cudaEventRecord(g->evFwd, sG), "record"));
  // the head bucket can go as soon as the head backward is done
  RP_TRY(cuda_ok(cudaStreamWaitEvent(sC, g->evFwd, 0), "wait"));
  RP_TRY(bucket_update(g, g->bk_head.first, g->bk_head.second, sC));
  if (mode == 2) RP_TRY(cuda_ok(cudaStreamWaitEvent(sR, g->evFwd, 0), "wait"));
  for (size_t si = g->st.size(); si-- > 0;) {
    RpStage& St = g->st[si];
    for (int64_t j = St.L - 1; j >= 0; --j) {
      const int64_t b = St.first + j;
      const bool top = j == St.L - 1, next_b2 = j > 0;
      // ledger: the footprint lane R is about to fill replaces the one whose VJP it waits
      // for (b + 2 under PaReprop, b + 1 in one lane); Vanilla only recomputes caches
      led_release_block(g, b + (mode == 2 ? 2 : 1));
      led_charge_block(g, b, g->vmode ? St.led_cache : St.led_block);
      ++g->blocks_processed;
      const bool free_lanes = (g->diag & 1) != 0;
      if (mode == 2) {
        if (b + 2 <= g->L - 1 && !free_lanes)
          RP_TRY(cuda_ok(cudaStreamWaitEvent(sR, g->evG[static_cast<size_t>(b + 2)], 0), "wait"));
        if (!(g->diag & 4)) RP_TRY(lane_r(g, b, sR));
        RP_TRY(cuda_ok(cudaEventRecord(g->evR[static_cast<size_t>(b)], sR), "record"));
        if (!free_lanes)
          RP_TRY(cuda_ok(cudaStreamWaitEvent(sG, g->evR[static_cast<size_t>(b)], 0), "wait"));
      } else if (!(g->diag & 4)) {
        RP_TRY(lane_r(g, b, sG));
      }
      if (!(g->diag & 2)) RP_TRY(lane_g(g, b, sG, top, next_b2));
      RP_TRY(cuda_ok(cudaEventRecord(g->evG[static_cast<size_t>(b)], sG), "record"));
      RP_TRY(cuda_ok(cudaStreamWaitEvent(sC, g->evG[static_cast<size_t>(b)], 0), "wait"));
      RP_TRY(bucket_update(g, g->bk_block[static_cast<size_t>(b)].first,
                           g->bk_block[static_cast<size_t>(b)].second, sC));
    }
    if (si == 0) break;
    // boundary between stage si-1 and si: recompute fuse(stage si-1 output) -- on lane R
    // under PaReprop (after lane G has finished the previous boundary's use of fb / cb) --
    // then the boundary VJP on lane G.
    RpStage& Pv = g->st[si - 1];
    if (mode == 2) {
      if (si + 1 < g->st.size())
        RP_TRY(cuda_ok(cudaStreamWaitEvent(sR, g->evBnd[si], 0), "wait"));
      RP_TRY(boundary_fuse(g, Pv, sR));
      RP_TRY(cuda_ok(cudaEventRecord(g->evFuse[si - 1], sR), "record"));
      RP_TRY(cuda_ok(cudaStreamWaitEvent(sG, g->evFuse[si - 1], 0), "wait"));
    } else {
      RP_TRY(boundary_fuse(g, Pv, sG));
    }
    RP_TRY(boundary_vjp(g, Pv, sG));
    RP_TRY(cuda_ok(cudaEventRecord(g->evBnd[si - 1], sG), "record"));
    RP_TRY(cuda_ok(cudaStreamWaitEvent(sC, g->evBnd[si - 1], 0), "wait"));
    RP_TRY(bucket_update(g, g->bk_bnd[si - 1].first, g->bk_bnd[si - 1].second, sC));
  }
  if (mode == 2) RP_TRY(cuda_ok(cudaEventRecord(g->evRDone, sR), "record"));
  for (int64_t b = 0; b < g->L; ++b) led_release_block(g, b);
  for (const RpStage& St : g->st) led_release(g, g->vmode ? St.led_stash : St.led_store);
  led_release(g, g->led_fixed);
  if (g->led_error || g->led_live != 0)
    return rp_fail(RP_ERR_ACCOUNTING, "ledger: activation bytes released twice or never");
  // embedding backward: e fed both halves -> d_e = d_i1 + d_i2
  const RpStage& S0 = g->st[0];
  RP_TRY(rpk_add_to_bf16(g->d1, g->d2, g->deb, S0.T * S0.d, sG));
  RP_TRY(launch(g->p_embed_w, sG));
  RP_TRY(cuda_ok(cudaEventRecord(g->evEmbed, sG), "record"));
  RP_TRY(cuda_ok(cudaStreamWaitEvent(sC, g->evEmbed, 0), "wait"));
  RP_TRY(bucket_update(g, g->bk_embed.first, g->bk_embed.second, sC));
  if (g->comm) {
    ncclResult_t r = ncclAllReduce(g->loss, g->loss, 1, ncclFloat32, ncclAvg, g->comm, sC);
    if (r != ncclSuccess) return rp_fail(RP_ERR_SCHEDULER, ncclGetErrorString(r));
  }
  RP_TRY(cuda_ok(cudaEventRecord(g->evCommDone, sC), "record"));
  RP_TRY(cuda_ok(cudaStreamWaitEvent(sG, g->evCommDone, 0), "wait"));
  if (mode == 2) RP_TRY(cuda_ok(cudaStreamWaitEvent(sG, g->evRDone, 0), "wait"));
  return rp_check_launch("engine step");
}

void set_partition(RpEngine* g, int mode) {
  int r = (mode == 2) ? g->r_ctas : 0;
  int gg = (mode == 2) ? g->g_ctas : 0;
  // data parallel: the backward's persistent GEMM grids leave comm_reserve SMs to the NCCL
  // kernels of the bucket all-reduces, so those start at once instead of waiting for a
  // whole GEMM to drain (the all-reduce then overlaps the backward)
  if (g->comm_reserve > 0) {
    const int cap = kSms - g->comm_reserve;
    r = r > 0 ? std::min(r, cap) : cap;
    gg = gg > 0 ? std::min(gg, cap) : cap;
  }
  for (auto& p : g->plans) {
    for (RpGemmPlan* q : {p.r_w1, p.r_w2, p.r_qkv, p.r_proj})
      if (q) rp_gemm_plan_set_max_ctas(q, r);
    for (RpGemmPlan* q : {p.g_dw2, p.g_ww2, p.g_ww1, p.g_dw1, p.g_dproj, p.g_wproj, p.g_wqkv,
                          p.g_dqkv})
      if (q) rp_gemm_plan_set_max_ctas(q, gg);
  }
}

}  // namespace

// Stage geometry from the config (validated); no allocation. An isotropic model is one stage.
namespace {
int stage_geoms(const RpModelConfig* c, std::vector<RpStage>* out) {
  out->clear();
  if (c->depth < 1 || c->width < 16 || c->heads < 1 || c->hidden < 16 || c->seq_len < 1 ||
      c->in_dim < 8 || c->num_classes < 1 || c->batch < 1)
    return rp_fail(RP_ERR_CONFIG, "engine_create: invalid model config");
  if (c->in_dim % 16) return rp_fail(RP_ERR_CONFIG, "engine_create: in_dim must be a multiple of 16");
  const bool hier = c->stages >= 2;
  const int64_t S = hier ? c->stages : 1;
  if (S > 8) return rp_fail(RP_ERR_CONFIG, "engine_create: at most 8 stages");
  if (hier) {
    int64_t tot = 0;
    for (int64_t s = 0; s < S; ++s) tot += c->stage_depth[s];
    if (tot != c->depth || c->stage_width[0] != c->width || c->stage_heads[0] != c->heads)
      return rp_fail(RP_ERR_CONFIG,
                     "engine_create: hierarchical config needs depth = sum(stage_depth), "
                     "width = stage_width[0], heads = stage_heads[0]");
    if (c->hidden % c->width)
      return rp_fail(RP_ERR_CONFIG, "engine_create: hidden must be a multiple of width (MLP ratio)");
    if (c->reduction < 1) return rp_fail(RP_ERR_CONFIG, "engine_create: reduction must be >= 1");
    if (c->fusion != 0 && c->fusion != 1)
      return rp_fail(RP_ERR_CONFIG, "engine_create: fusion must be 0 (average) or 1 (mlp)");
  }
  int64_t n = c->seq_len, first = 0;
  for (int64_t s = 0; s < S; ++s) {
    RpStage St;
    if (s > 0) {
      if (n % c->reduction)
        return rp_fail(RP_ERR_SHAPE, "group_tokens: token count not divisible by r");
      n /= c->reduction;
    }
    St.L = hier ? c->stage_depth[s] : c->depth;
    St.d = hier ? c->stage_width[s] : c->width;
    St.H = hier ? c->stage_heads[s] : c->heads;
    St.h = hier ? St.d * (c->hidden / c->width) : c->hidden;
    St.N = n;
    St.first = first;
    St.T = c->batch * n;
    if (St.L < 1 || St.d < 16 || St.H < 1 || St.d % St.H || (St.d / St.H) % 8 || St.d / St.H > 128)
      return rp_fail(RP_ERR_CONFIG,
                     "engine_create: invalid stage (head_dim = width/heads must be a multiple of "
                     "8, at most 128)");
    if (St.d % 64 || St.h % 64)  // the GEMM epilogue works in 64-column chunks
      return rp_fail(RP_ERR_CONFIG, "engine_create: width/hidden must be multiples of 64");
    // hierarchical stages attend in windows of min(window, tokens) (the last stages of a
    // Swin-style model are a single window); the isotropic model keeps the reference's
    // rule that the window must divide the sequence (layers.cpp:118-120)
    St.W = c->window > 0 ? (hier ? std::min(c->window, n) : c->window) : n;
    if (n % St.W)
      return rp_fail(RP_ERR_SHAPE, "attention: sequence length not divisible by window");
    St.block_size = 4 * St.d * St.d + 2 * St.d * St.h + St.h + 5 * St.d;
    first += St.L;
    out->push_back(St);
  }
  return RP_OK;
}

// The data-parallel gradient buckets (one all-reduce each) in the order the step issues
// them: the head, then per stage from the last, its blocks from the top down, then the
// boundary below that stage, and the embedding last. Offsets into the flat parameter /
// gradient vector (order of include/revprop_b200.h). kind: 0 embed, 1 block, 2 boundary,
// 3 head; index: block / stage index.
struct Bucket {
  int64_t off, n;
  int kind;
  int64_t index;
};
void bucket_plan(const RpModelConfig* c, const std::vector<RpStage>& st, std::vector<Bucket>* out) {
  const int64_t r = c->stages >= 2 ? c->reduction : 2;
  const int fusion = c->stages >= 2 ? c->fusion : 0;
  std::vector<int64_t> blk_off, bnd_off, bnd_n;
  int64_t off = c->in_dim * st[0].d;  // embed_w first
  for (size_t s = 0; s < st.size(); ++s) {
    for (int64_t j = 0; j < st[s].L; ++j) {
      blk_off.push_back(off);
      off += st[s].block_size;
    }
    if (s + 1 < st.size()) {
      const int64_t n = r * st[s].d * st[s + 1].d + (fusion == 1 ? 2 * st[s].d * st[s].d : 0);
      bnd_off.push_back(off);
      bnd_n.push_back(n);
      off += n;
    }
  }
  out->clear();
  out->push_back({off, st.back().d * c->num_classes, 3, 0});
  for (size_t s = st.size(); s-- > 0;) {
    for (int64_t j = st[s].L - 1; j >= 0; --j) {
      const int64_t b = st[s].first + j;
      out->push_back({blk_off[static_cast<size_t>(b)], st[s].block_size, 1, b});
    }
    if (s > 0) out->push_back({bnd_off[s - 1], bnd_n[s - 1], 2, static_cast<int64_t>(s - 1)});
  }
  out->push_back({0, c->in_dim * st[0].d, 0, 0});
}
}  // namespace

// The gradient buckets of a model config (no device needed): offsets / sizes (floats) in
// all-reduce order, kinds (0 embed, 1 block, 2 boundary, 3 head). Returns the count, or a
// negative status when `cap` is too small.
extern "C" int rp_model_bucket_plan(const RpModelConfig* c, int64_t* offsets, int64_t* sizes,
                                    int* kinds, int64_t cap) {
  if (!c) return -rp_fail(RP_ERR_CONTRACT, "null config");
  std::vector<RpStage> st;
  const int rc = stage_geoms(c, &st);
  if (rc != RP_OK) return -rc;
  std::vector<Bucket> bk;
  bucket_plan(c, st, &bk);
  if (cap < static_cast<int64_t>(bk.size()))
    return -rp_fail(RP_ERR_SHAPE, "bucket plan capacity too small");
  for (size_t i = 0; i < bk.size(); ++i) {
    if (offsets) offsets[i] = bk[i].off;
    if (sizes) sizes[i] = bk[i].n;
    if (kinds) kinds[i] = bk[i].kind;
  }
  return static_cast<int>(bk.size());
}

// ---------------------------------------------------------------- activation ledger
// Bytes of activation storage each engine keeps live at its peak (SPEC.md:346-349
// MemoryLedger semantics, ref:proj/core/include/revprop/ledger.hpp:18-62), from the
// arena plan of this engine: stored stage boundaries, per-block recompute footprint,
// cotangents and lane-G temporaries. Parameters, gradients and split-K / reduction
// workspaces are excluded (they do not scale with depth or batch in the same way).
//   mode 0 vanilla   stores every block's input pair + one block's caches
//   mode 1 reprop    every stage's input + output + one block footprint
//   mode 2 pareprop  reprop + one more block footprint (rendezvous depth 1)
// Per-block quantities are the largest over the stages (the slots are shared).
namespace {
// one stage's ledger quantities (bytes)
struct StageLedger {
  int64_t block, cache, store, stash;
};
StageLedger stage_ledger(const RpStage& S) {
  const int64_t T = S.T, d = S.d, h = S.h, H = S.H;
  const int64_t pair = 2 * T * d * 4;  // one coupled (i1, i2) fp32 pair
  // block footprint: recomputed input pair + F caches (hF, qkv, att: bf16; lse, LN stats)
  // + G caches (hG, slope, a: bf16; LN stats)
  const int64_t cache_f = T * d * 2 + T * 3 * d * 2 + T * d * 2 + T * H * 4 + 2 * T * 4;
  const int64_t cache_g = T * d * 2 + 2 * T * h * 2 + 2 * T * 4;
  StageLedger r;
  r.cache = cache_f + cache_g;
  r.block = pair + r.cache;
  r.store = T * d * 4 /* stage input e, shared by i1 = i2 */ + pair /* stage output */;
  r.stash = T * d * 4 + S.L * pair;  // Vanilla: e + every block's output pair
  return r;
}
struct LedgerTerms {
  int64_t block = 0, cache = 0, stages = 0, stash = 0, fixed = 0;
};
LedgerTerms ledger_terms(const std::vector<RpStage>& st, int fusion) {
  LedgerTerms t;
  int64_t cot = 0, temps = 0;
  for (const RpStage& S : st) {
    const StageLedger l = stage_ledger(S);
    const int64_t T = S.T, d = S.d, h = S.h;
    t.block = std::max(t.block, l.block);
    t.cache = std::max(t.cache, l.cache);
    cot = std::max(cot, 2 * T * d * 4 + 2 * T * d * 2);                               // d_out pair
    temps = std::max(temps, T * h * 2 + 2 * T * d * 2 + T * 3 * d * 2 + T * d * 2);  // du,dh,datt,dqkv,de
    t.stages += l.store;
    t.stash += l.stash;
  }
  if (st.size() > 1) {  // boundary recompute buffers (fused output, mlp concat)
    int64_t fb = 0;
    for (size_t s = 0; s + 1 < st.size(); ++s)
      fb = std::max(fb, st[s].T * st[s].d * 2 * (fusion == 1 ? 3 : 1));
    temps += fb;
  }
  t.fixed = cot + temps;
  return t;
}
}  // namespace

extern "C" int rp_activation_bytes(const RpModelConfig* c, int mode, int64_t* out_peak,
                                   int64_t* out_block_footprint) {
  if (!c || !out_peak) return rp_fail(RP_ERR_CONTRACT, "null argument");
  if (mode < 0 || mode > 2) return rp_fail(RP_ERR_CONFIG, "mode must be 0, 1 or 2");
  std::vector<RpStage> st;
  RP_TRY(stage_geoms(c, &st));
  const LedgerTerms t = ledger_terms(st, c->fusion);
  int64_t peak = 0;
  if (mode == 0)
    peak = t.stash + t.cache + t.fixed;
  else
    peak = t.stages + (mode == 2 ? 2 : 1) * t.block + t.fixed;
  *out_peak = peak;
  if (out_block_footprint) *out_block_footprint = t.block;
  return RP_OK;
}

extern "C" int rp_engine_create(const RpModelConfig* c, RpEngine** out) {
  if (!c || !out) return rp_fail(RP_ERR_CONTRACT, "engine_create: null argument");
  *out = nullptr;
  std::vector<RpStage> geo;
  RP_TRY(stage_geoms(c, &geo));
  RpEngine* g = new RpEngine();
  g->cfg = *c;
  g->st = geo;
  g->B = c->batch;
  g->N = c->seq_len;
  g->in = c->in_dim;
  g->C = c->num_classes;
  g->L = c->depth;
  g->T = g->B * g->N;
  g->r = c->stages >= 2 ? c->reduction : 2;
  g->fusion = c->stages >= 2 ? c->fusion : 0;
  g->dev = c->device;
  auto fail = [&](int rc) {
    rp_engine_destroy(g);
    return rc;
  };
  if (cudaSetDevice(g->dev) != cudaSuccess) return fail(rp_fail(RP_ERR_CUDA, "cudaSetDevice failed"));
  // flat tensor table: embed_w | stage blocks | boundary | ... | head_w
  auto add = [&](int64_t n, int kind) {
    const int64_t off = g->t_off.empty() ? 0 : g->t_off.back() + g->t_numel.back();
    g->t_off.push_back(off);
    g->t_numel.push_back(n);
    g->t_kind.push_back(kind);
  };
  add(g->in * g->st[0].d, 0);
  for (size_t s = 0; s < g->st.size(); ++s) {
    RpStage& St = g->st[s];
    const int64_t d = St.d, h = St.h;
    for (int64_t j = 0; j < St.L; ++j) {
      g->blk_tix.push_back(static_cast<int64_t>(g->t_off.size()));
      g->stage_of.push_back(static_cast<int>(s));
      add(d * 3 * d, 0);  // w_qkv
      add(d * d, 0);      // w_out
      add(d, 2);          // lnF gamma
      add(d, 1);          // lnF beta
      add(d * h, 0);      // w1
      add(h, 1);          // b1
      add(h * d, 0);      // w2
      add(d, 1);          // b2
      add(d, 2);          // lnG gamma
      add(d, 1);          // lnG beta
    }
    if (s + 1 < g->st.size()) {
      St.bnd_tix = static_cast<int64_t>(g->t_off.size());
      add(g->r * d * g->st[s + 1].d, 0);    // merge_w
      if (g->fusion == 1) add(2 * d * d, 0);  // fusion_w
      St.bnd_size = g->r * d * g->st[s + 1].d + (g->fusion == 1 ? 2 * d * d : 0);
    }
  }
  g->head_tix = static_cast<int64_t>(g->t_off.size());
  add(g->st.back().d * g->C, 0);
  g->P = g->t_off.back() + g->t_numel.back();
  {
    std::vector<Bucket> bk;
    bucket_plan(c, g->st, &bk);
    g->bk_block.resize(static_cast<size_t>(g->L));
    g->bk_bnd.resize(g->st.size());
    int64_t covered = 0;
    for (const Bucket& k : bk) {
      const std::pair<int64_t, int64_t> v{k.off, k.n};
      covered += k.n;
      if (k.kind == 0) g->bk_embed = v;
      if (k.kind == 1) g->bk_block[static_cast<size_t>(k.index)] = v;
      if (k.kind == 2) g->bk_bnd[static_cast<size_t>(k.index)] = v;
      if (k.kind == 3) g->bk_head = v;
    }
    // the plan must tile the tensor table exactly (every parameter in one bucket)
    bool ok = covered == g->P && g->bk_head.first == g->t_off[static_cast<size_t>(g->head_tix)];
    for (int64_t b = 0; b < g->L; ++b)
      ok = ok && g->bk_block[static_cast<size_t>(b)].first ==
                     g->t_off[static_cast<size_t>(tix_block(g, b, 0))];
    for (size_t si = 0; si + 1 < g->st.size(); ++si)
      ok = ok && g->bk_bnd[si].first == g->t_off[static_cast<size_t>(g->st[si].bnd_tix)];
    if (!ok) {
      rp_engine_destroy(g);
      return rp_fail(RP_ERR_CONTRACT, "engine_create: bucket plan does not tile the parameters");
    }
  }
  {
    const LedgerTerms lt = ledger_terms(g->st, g->fusion);
    g->led_fixed = lt.fixed;
    for (RpStage& St : g->st) {
      const StageLedger l = stage_ledger(St);
      St.led_block = l.block;
      St.led_cache = l.cache;
      St.led_store = l.store;
      St.led_stash = l.stash;
    }
    int64_t off = 0;
    for (int64_t b = 0; b < g->L; ++b) {
      g->trace_off.push_back(off);
      const RpStage& St = stage_of(g, b);
      off += 2 * St.T * St.d;
    }
    g->trace_off.push_back(off);  // total
  }
  int rc = RP_OK;
  // Lane G (the critical path) and the comm / optimizer stream get the highest stream
  // priority, lane R the lowest: the block scheduler then fills idle SMs and kernel tails
  // with recompute work instead of letting it compete with the gradient lane, and a
  // bucket's all-reduce (a few CTAs, latency-critical) is not queued behind the lanes' work.
  int prio_lo = 0, prio_hi = 0;
  cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
  const bool use_prio = c->lane_priority != 0;
  if ((rc = cuda_ok(cudaStreamCreateWithPriority(&g->sG, cudaStreamNonBlocking,
                                                 use_prio ? prio_hi : 0),
                    "stream")) ||
      (rc = cuda_ok(cudaStreamCreateWithPriority(&g->sR, cudaStreamNonBlocking,
                                                 use_prio ? prio_lo : 0),
                    "stream")) ||
      (rc = cuda_ok(cudaStreamCreateWithPriority(&g->sC, cudaStreamNonBlocking,
                                                 use_prio ? prio_hi : 0),
                    "stream")))
    return fail(rc);
  g->evR.resize(static_cast<size_t>(g->L));
  g->evG.resize(static_cast<size_t>(g->L));
  g->evBnd.resize(g->st.size());
  g->evFuse.resize(g->st.size());
  for (auto* v : {&g->evR, &g->evG, &g->evBnd, &g->evFuse})
    for (auto& e : *v) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  for (cudaEvent_t* e : {&g->evFwd, &g->evCommDone, &g->evRDone, &g->evEmbed, &g->evLogits,
                         &g->evCaller})
    cudaEventCreateWithFlags(e, cudaEventDisableTiming);
  cudaEventCreate(&g->evStepBeg);
  cudaEventCreate(&g->evStepEnd);
  g->ts.resize(static_cast<size_t>(4 * g->L));
  for (auto& e : g->ts) cudaEventCreate(&e);
  // arena: per-block buffers sized for the largest stage (shared by all stages)
  int64_t Td = 0, Th = 0, TH = 0, Tmax = 0, ln_ws = 0, attn_ws = 0, col_ws = 0, split_ws = 0;
  int64_t fb = 0;
  auto splits_ws = [&](int64_t m, int64_t n, int64_t k) {
    const int sp = pick_splits(m, n, k, gemm_bn(n));
    if (sp > 1) split_ws = std::max<int64_t>(split_ws, sp * m * n);
  };
  for (size_t s = 0; s < g->st.size(); ++s) {
    const RpStage& St = g->st[s];
    const int64_t T = St.T, d = St.d, h = St.h;
    Td = std::max(Td, T * d);
    Th = std::max(Th, T * h);
    TH = std::max(TH, T * St.H);
    Tmax = std::max(Tmax, T);
    ln_ws = std::max(ln_ws, rp_layer_norm_bwd_workspace_floats(T, d));
    attn_ws = std::max(attn_ws, rp_attention_bwd_workspace_floats(T / St.W, St.W, St.H));
    col_ws = std::max(col_ws, rp_colsum_workspace_floats(T, h > d ? h : d));
    col_ws = std::max(col_ws, ((T + 31) / 32) * h);  // d_u epilogue partials
    for (auto mn : {std::pair<int64_t, int64_t>{d, 3 * d}, {d, d}, {d, h}, {h, d}}) splits_ws(mn.first, mn.second, T);
    if (s + 1 < g->st.size()) {
      const RpStage& Nx = g->st[s + 1];
      splits_ws(g->r * d, Nx.d, Nx.T);
      if (g->fusion == 1) splits_ws(2 * d, d, T);
      fb = std::max(fb, T * d);
    }
  }
  splits_ws(g->in, g->st[0].d, g->T);
  if ((rc = dalloc(g, &g->params, g->P, 2)) || (rc = dalloc(g, &g->grads, g->P, 2)) ||
      (rc = dalloc(g, &g->pb, g->P, 2)) || (rc = dalloc(g, &g->lr, 1)) ||
      (rc = dalloc(g, &g->lr_apply, 1)) ||
      (rc = dalloc(g, &g->inputs, g->T * g->in)) || (rc = dalloc(g, &g->labels, g->B)))
    return fail(rc);
  for (RpStage& St : g->st) {
    const int64_t n = St.T * St.d;
    if ((rc = dalloc(g, &St.e, n, 1)) || (rc = dalloc(g, &St.buf1[0], n, 1)) ||
        (rc = dalloc(g, &St.buf1[1], n, 1)) || (rc = dalloc(g, &St.buf2[0], n, 1)) ||
        (rc = dalloc(g, &St.buf2[1], n, 1)) || (rc = dalloc(g, &St.buf2[2], n, 1)))
      return fail(rc);
  }
  for (Slot& S : g->slot) {
    if ((rc = dalloc(g, &S.hF, Td, 1)) || (rc = dalloc(g, &S.qkv, 3 * Td, 1)) ||
        (rc = dalloc(g, &S.att, Td, 1)) || (rc = dalloc(g, &S.hG, Td, 1)) ||
        (rc = dalloc(g, &S.u, Th, 1)) || (rc = dalloc(g, &S.a, Th, 1)) ||
        (rc = dalloc(g, &S.lse, TH, 1)) || (rc = dalloc(g, &S.meanF, Tmax, 1)) ||
        (rc = dalloc(g, &S.rstdF, Tmax, 1)) || (rc = dalloc(g, &S.meanG, Tmax, 1)) ||
        (rc = dalloc(g, &S.rstdG, Tmax, 1)))
      return fail(rc);
  }
  if ((rc = dalloc(g, &g->d1, Td, 1)) || (rc = dalloc(g, &g->d2, Td, 1)) ||
      (rc = dalloc(g, &g->d1b, Td, 1)) || (rc = dalloc(g, &g->d2b, Td, 1)) ||
      (rc = dalloc(g, &g->du, Th, 1)) || (rc = dalloc(g, &g->dh, Td, 1)) ||
      (rc = dalloc(g, &g->datt, Td, 1)) || (rc = dalloc(g, &g->dqkv, 3 * Td, 1)) ||
      (rc = dalloc(g, &g->deb, Td, 1)) || (rc = dalloc(g, &g->ln_ws, ln_ws)) ||
      (rc = dalloc(g, &g->col_ws, col_ws)) || (rc = dalloc(g, &g->split_ws, split_ws)) ||
      (rc = dalloc(g, &g->attn_ws, attn_ws)) ||
      (rc = dalloc(g, &g->pooled, g->B * g->st.back().d)) ||
      (rc = dalloc(g, &g->logits, g->B * g->C)) || (rc = dalloc(g, &g->dlogits, g->B * g->C)) ||
      (rc = dalloc(g, &g->row_loss, g->B)) || (rc = dalloc(g, &g->loss, 1)) ||
      (rc = dalloc(g, &g->dpooled, g->B * g->st.back().d)))
    return fail(rc);
  if (fb > 0 && ((rc = dalloc(g, &g->fb, fb, 1)) ||
                 (g->fusion == 1 && (rc = dalloc(g, &g->cb, 2 * fb, 1)))))
    return fail(rc);
  {
    const int bits = c->exact_coupling_bits == 0 ? 17 : c->exact_coupling_bits;
    if (bits > 0 && bits > 60) return fail(rp_fail(RP_ERR_CONFIG, "exact_coupling_bits too large"));
    g->quantum = bits > 0 ? std::ldexp(1.0f, -bits) : 0.f;
  }
  if ((rc = build_plans(g))) return fail(rc);
  g->optimizer = c->optimizer;
  if (c->optimizer == 1) {
    g->beta1 = c->beta1;
    g->beta2 = c->beta2;
    g->eps = c->adam_eps;
    g->wd = c->weight_decay;
    if ((rc = dalloc(g, &g->adam_m, g->P, 2)) || (rc = dalloc(g, &g->adam_v, g->P, 2)) ||
        (rc = dalloc(g, &g->step_t, 1)))
      return fail(rc);
    cudaMemset(g->adam_m, 0, static_cast<size_t>(g->P) * 4);
    cudaMemset(g->adam_v, 0, static_cast<size_t>(g->P) * 4);
    cudaMemset(g->step_t, 0, 4);
  } else if (c->optimizer != 0) {
    return fail(rp_fail(RP_ERR_CONFIG, "optimizer must be 0 (SGD) or 1 (AdamW)"));
  }
  // default PaReprop SM partition: recompute : VJP work is ~1 : 2
  g->r_ctas = c->r_ctas > 0 ? c->r_ctas : 0;
  g->g_ctas = c->g_ctas > 0 ? c->g_ctas : 0;
  // initial parameters + synthetic batch from the counter RNG
  if ((rc = rp_engine_init_params(g, c->seed)) || (rc = rp_engine_synthetic_batch(g, c->seed)))
    return fail(rc);
  const float lr0 = 0.f;
  cudaMemcpy(g->lr, &lr0, sizeof(float), cudaMemcpyHostToDevice);
  cudaMemset(g->grads, 0, static_cast<size_t>(g->P) * sizeof(float));
  if ((rc = cuda_ok(cudaDeviceSynchronize(), "engine_create"))) return fail(rc);
  *out = g;
  return RP_OK;
}

extern "C" void rp_engine_destroy(RpEngine* g) {
  if (!g) return;
  cudaDeviceSynchronize();
  for (auto& x : g->graph)
    if (x) cudaGraphExecDestroy(x);
  for (RpGemmPlan* p : g->all_plans) rp_gemm_plan_destroy(p);
  for (void* p : g->allocs) cudaFree(p);
  for (auto* v : {&g->evR, &g->evG, &g->ts, &g->evBnd, &g->evFuse})
    for (auto& e : *v)
      if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : {g->evFwd, g->evCommDone, g->evRDone, g->evEmbed, g->evLogits,
                        g->evCaller, g->evStepBeg, g->evStepEnd})
    if (e) cudaEventDestroy(e);
  for (cudaStream_t s : {g->sG, g->sR, g->sC, g->sX})
    if (s) cudaStreamDestroy(s);
  for (cudaEvent_t e : {g->evStaged, g->evStageFree, g->evLoss})
    if (e) cudaEventDestroy(e);
  if (g->comm) ncclCommDestroy(g->comm);
  delete g;
}

extern "C" int64_t rp_engine_param_count(const RpEngine* g) { return g ? g->P : -1; }

extern "C" int rp_engine_tensor_table(const RpEngine* g, int64_t* offsets, int64_t* numels,
                                      int64_t cap) {
  if (!g) return rp_fail(RP_ERR_CONTRACT, "null engine");
  const int64_t n = static_cast<int64_t>(g->t_off.size());
  if (cap < n) return rp_fail(RP_ERR_SHAPE, "tensor table capacity too small");
  for (int64_t i = 0; i < n; ++i) {
    offsets[i] = g->t_off[static_cast<size_t>(i)];
    numels[i] = g->t_numel[static_cast<size_t>(i)];
  }
  return static_cast<int>(n);
}

extern "C" int rp_engine_init_params(RpEngine* g, uint64_t seed) {
  if (!g) return rp_fail(RP_ERR_CONTRACT, "null engine");
  // weights trunc-normal(0.02), biases zero; LayerNorm gamma = 1, beta = 0.
  for (size_t j = 0; j < g->t_off.size(); ++j) {
    const int kind = g->t_kind[j];
    RP_TRY(rpk_init_tensor(g->params + g->t_off[j], g->t_numel[j], seed, j, kind, 0.02, g->sG));
  }
  RP_TRY(rpk_f32_to_bf16(g->params, g->pb, g->P, g->sG));
  return cuda_ok(cudaStreamSynchronize(g->sG), "init_params");
}

extern "C" int rp_engine_synthetic_batch(RpEngine* g, uint64_t seed) {
  if (!g) return rp_fail(RP_ERR_CONTRACT, "null engine");
  RP_TRY(rpk_init_inputs(g->inputs, g->T * g->in, seed, g->sG));
  std::vector<int32_t> lab(static_cast<size_t>(g->B));
  // labels: Rng(seed, 3<<56).next_int(0, C) in batch order (rng.hpp:53-57)
  for (int64_t b = 0; b < g->B; ++b)
    lab[static_cast<size_t>(b)] = static_cast<int32_t>(
        rp_rng_u64_host(seed, 3ull << 56, static_cast<uint64_t>(b)) % static_cast<uint64_t>(g->C));
  RP_TRY(cuda_ok(cudaMemcpyAsync(g->labels, lab.data(), lab.size() * sizeof(int32_t),
                                 cudaMemcpyHostToDevice, g->sG),
                 "labels"));
  return cuda_ok(cudaStreamSynchronize(g->sG), "synthetic_batch");
}

extern "C" int rp_engine_set_params(RpEngine* g, const float* host) {
  if (!g || !host) return rp_fail(RP_ERR_CONTRACT, "null argument");
  RP_TRY(cuda_ok(cudaMemcpyAsync(g->params, host, static_cast<size_t>(g->P) * 4,
                                 cudaMemcpyHostToDevice, g->sG),
                 "set_params"));
  RP_TRY(rpk_f32_to_bf16(g->params, g->pb, g->P, g->sG));
  return cuda_ok(cudaStreamSynchronize(g->sG), "set_params");
}

extern "C" int rp_engine_get_params(RpEngine* g, float* host) {
  if (!g || !host) return rp_fail(RP_ERR_CONTRACT, "null argument");
  // ordered after the engine's pending work (its streams are non-blocking: a plain
  // cudaMemcpy on the legacy stream would not wait for an in-flight step)
  RP_TRY(cuda_ok(cudaMemcpyAsync(host, g->params, static_cast<size_t>(g->P) * 4,
                                 cudaMemcpyDeviceToHost, g->sG),
                 "get_params"));
  return rp_engine_sync(g);
}

// The gradient of the mean loss over the global batch: after a data-parallel step the
// buffer holds the all-reduced SUM of the ranks' gradients (the optimizer folds 1 / world
// into its step), so the host copy is scaled by 1 / world.
extern "C" int rp_engine_get_grads(RpEngine* g, float* host) {
  if (!g || !host) return rp_fail(RP_ERR_CONTRACT, "null argument");
  RP_TRY(cuda_ok(cudaMemcpyAsync(host, g->grads, static_cast<size_t>(g->P) * 4,
                                 cudaMemcpyDeviceToHost, g->sG),
                 "get_grads"));
  RP_TRY(rp_engine_sync(g));
  if (g->world > 1) {
    const float inv = 1.0f / static_cast<float>(g->world);
    for (int64_t i = 0; i < g->P; ++i) host[i] *= inv;
  }
  return RP_OK;
}

// inputs: bf16 [B, N, in_dim] (host, ideally pinned), labels int32 [B]; async on the
// engine's stream (the next step is ordered after it).
extern "C" int rp_engine_set_batch(RpEngine* g, const uint16_t* inputs, const int32_t* labels) {
  if (!g || !inputs || !labels) return rp_fail(RP_ERR_CONTRACT, "null argument");
  RP_TRY(cuda_ok(cudaMemcpyAsync(g->inputs, inputs, static_cast<size_t>(g->T * g->in) * 2,
                                 cudaMemcpyHostToDevice, g->sG),
                 "set_batch inputs"));
  return cuda_ok(cudaMemcpyAsync(g->labels, labels, static_cast<size_t>(g->B) * 4,
                                 cudaMemcpyHostToDevice, g->sG),
                 "set_batch labels");
}

// Pipelined input: the host -> device copy of the NEXT step's batch runs on a copy stream
// while the current step computes; the next rp_engine_step waits for it and moves it into
// the step's input buffers (a device-to-device copy on the engine stream, outside the
// captured graph). Host buffers should be pinned and stay valid until that step starts.
extern "C" int rp_engine_prefetch_batch(RpEngine* g, const uint16_t* inputs, const int32_t* labels) {
  if (!g || !inputs || !labels) return rp_fail(RP_ERR_CONTRACT, "null argument");
  if (!g->sX) {
    RP_TRY(cuda_ok(cudaStreamCreateWithFlags(&g->sX, cudaStreamNonBlocking), "stream"));
    for (cudaEvent_t* e : {&g->evStaged, &g->evStageFree})
      RP_TRY(cuda_ok(cudaEventCreateWithFlags(e, cudaEventDisableTiming), "event"));
    // (evLoss belongs to read_loss_async: created there on first use, never replaced here,
    // so a recorded loss read-back is not lost)
    RP_TRY(dalloc(g, &g->in_stage, g->T * g->in));
    RP_TRY(dalloc(g, &g->lab_stage, g->B));
  }
  // the staging buffers are free once the previous staged batch has been moved out
  RP_TRY(cuda_ok(cudaStreamWaitEvent(g->sX, g->evStageFree, 0), "wait"));
  RP_TRY(cuda_ok(cudaMemcpyAsync(g->in_stage, inputs, static_cast<size_t>(g->T * g->in) * 2,
                                 cudaMemcpyHostToDevice, g->sX),
                 "prefetch inputs"));
  RP_TRY(cuda_ok(cudaMemcpyAsync(g->lab_stage, labels, static_cast<size_t>(g->B) * 4,
                                 cudaMemcpyHostToDevice, g->sX),
                 "prefetch labels"));
  RP_TRY(cuda_ok(cudaEventRecord(g->evStaged, g->sX), "record"));
  g->staged = true;
  return RP_OK;
}

// Asynchronous loss read-back: device -> host copy of the last enqueued step's loss into
// `loss` (pinned) on the engine stream; rp_engine_wait_loss blocks until it has landed.
extern "C" int rp_engine_read_loss_async(RpEngine* g, float* loss) {
  if (!g || !loss) return rp_fail(RP_ERR_CONTRACT, "null argument");
  if (!g->evLoss) RP_TRY(cuda_ok(cudaEventCreateWithFlags(&g->evLoss, cudaEventDisableTiming), "event"));
  RP_TRY(cuda_ok(cudaMemcpyAsync(loss, g->loss, sizeof(float), cudaMemcpyDeviceToHost, g->sG),
                 "read_loss_async"));
  return cuda_ok(cudaEventRecord(g->evLoss, g->sG), "record");
}

extern "C" int rp_engine_wait_loss(RpEngine* g) {
  if (!g) return rp_fail(RP_ERR_CONTRACT, "null engine");
  if (!g->evLoss) return RP_OK;
  return cuda_ok(cudaEventSynchronize(g->evLoss), "wait_loss");
}

extern "C" int rp_engine_set_batch_device(RpEngine* g, const uint16_t* inputs,
                                          const int32_t* labels) {
  if (!g || !inputs || !labels) return rp_fail(RP_ERR_CONTRACT, "null argument");
  RP_TRY(wait_caller(g));
  RP_TRY(cuda_ok(cudaMemcpyAsync(g->inputs, inputs, static_cast<size_t>(g->T * g->in) * 2,
                                 cudaMemcpyDeviceToDevice, g->sG),
                 "set_batch inputs"));
  return cuda_ok(cudaMemcpyAsync(g->labels, labels, static_cast<size_t>(g->B) * 4,
                                 cudaMemcpyDeviceToDevice, g->sG),
                 "set_batch labels");
}

extern "C" int rp_engine_set_lr(RpEngine* g, float lr) {
  if (!g) return rp_fail(RP_ERR_CONTRACT, "null engine");
  return cuda_ok(cudaMemcpyAsync(g->lr, &lr, sizeof(float), cudaMemcpyHostToDevice, g->sG),
                 "set_lr");
}

// Allocates the Vanilla stash (every block's input pair, 2 L T d fp32) and its forward
// plans; afterwards rp_engine_step(engine, 0, ...) runs store-everything training.
extern "C" int rp_engine_enable_vanilla(RpEngine* g) {
  if (!g) return rp_fail(RP_ERR_CONTRACT, "null engine");
  if (g->vanilla_ready) return RP_OK;
  int64_t n = 0;
  for (RpStage& St : g->st) {
    St.stash_off = n;
    n += St.L * St.T * St.d;
  }
  RP_TRY(dalloc(g, &g->stash1, n, 1));
  RP_TRY(dalloc(g, &g->stash2, n, 1));
  Slot& F = g->slot[0];
  g->vmode = true;
  g->vf_proj.resize(static_cast<size_t>(g->L));
  g->vf_w2.resize(static_cast<size_t>(g->L));
  for (int64_t b = 0; b < g->L; ++b) {
    RpStage& St = stage_of(g, b);
    const int64_t T = St.T, d = St.d, h = St.h, j = b - St.first;
    GemmArgs a{F.att, d, 0, wb(g, tix_block(g, b, kWout)), d, 1, T, d, d, RP_EPI_RESID,
               X2(g, St, j + 1), d};
    a.aux = X2(g, St, j);
    a.quantum = g->quantum;
    int rc = mk_plan(g, a, &g->vf_proj[static_cast<size_t>(b)]);
    if (rc == RP_OK) {
      GemmArgs c{F.a, h, 0, wb(g, tix_block(g, b, kW2)), d, 1, T, d, h, RP_EPI_RESID,
                 X1(g, St, j + 1), d};
      c.aux = X1(g, St, j);
      c.bias = wf(g, tix_block(g, b, kB2));
      c.quantum = g->quantum;
      rc = mk_plan(g, c, &g->vf_w2[static_cast<size_t>(b)]);
    }
    if (rc != RP_OK) {
      g->vmode = false;
      return rc;
    }
  }
  // the boundary merge GEMMs read fuse(stage output) computed from the stash in vmode and
  // write the next stage's e, which is not stashed: the same plans serve both modes
  g->vmode = false;
  g->vanilla_ready = true;
  return RP_OK;
}

// Test hook for the verify command ("deliberately corrupted VJP"): kind 1
// scales every block's propagated F-path cotangent by 1.5; kind 0 restores the true VJP.
extern "C" int rp_engine_inject_fault(RpEngine* g, int kind) {
  if (!g) return rp_fail(RP_ERR_CONTRACT, "null engine");
  if (kind < 0 || kind > 1) return rp_fail(RP_ERR_CONFIG, "inject_fault: kind must be 0 or 1");
  g->fault = kind;
  return rp_engine_invalidate_graphs(g);
}

// Drop captured graphs (e.g. after toggling rp_set_pdl); the next step recaptures.
extern "C" int rp_engine_invalidate_graphs(RpEngine* g) {
  if (!g) return rp_fail(RP_ERR_CONTRACT, "null engine");
  RP_TRY(cuda_ok(cudaStreamSynchronize(g->sG), "sync"));
  for (auto& x : g->graph)
    if (x) {
      cudaGraphExecDestroy(x);
      x = nullptr;
    }
  return RP_OK;
}

extern "C" int rp_engine_set_partition(RpEngine* g, int r_ctas, int g_ctas) {
  if (!g) return rp_fail(RP_ERR_CONTRACT, "null engine");
  g->r_ctas = r_ctas;
  g->g_ctas = g_ctas;
  if (g->graph[2]) {
    cudaGraphExecDestroy(g->graph[2]);
    g->graph[2] = nullptr;
  }
  return RP_OK;
}

// mode: 1 = Reprop, 2 = PaReprop. use_graph: capture once, then replay.
// The step is asynchronous on the engine stream; rp_engine_sync / read_loss wait for it.
extern "C" int rp_engine_step(RpEngine* g, int mode, int use_graph) {
  if (!g) return rp_fail(RP_ERR_CONTRACT, "null engine");
  if (mode < 0 || mode > 2)
    return rp_fail(RP_ERR_CONFIG, "step: mode must be 0 (vanilla), 1 (reprop) or 2 (pareprop)");
  if (mode == 0 && !g->vanilla_ready)
    return rp_fail(RP_ERR_CONTRACT, "step: vanilla mode needs rp_engine_enable_vanilla()");
  set_partition(g, mode);
  if (g->staged) {  // the batch prefetched by rp_engine_prefetch_batch becomes this step's
    RP_TRY(cuda_ok(cudaStreamWaitEvent(g->sG, g->evStaged, 0), "wait staged batch"));
    RP_TRY(cuda_ok(cudaMemcpyAsync(g->inputs, g->in_stage, static_cast<size_t>(g->T * g->in) * 2,
                                   cudaMemcpyDeviceToDevice, g->sG),
                   "stage -> inputs"));
    RP_TRY(cuda_ok(cudaMemcpyAsync(g->labels, g->lab_stage, static_cast<size_t>(g->B) * 4,
                                   cudaMemcpyDeviceToDevice, g->sG),
                   "stage -> labels"));
    RP_TRY(cuda_ok(cudaEventRecord(g->evStageFree, g->sG), "record"));
    g->staged = false;
  }
  const bool eager = !use_graph || g->instrument || g->trace_fwd || g->trace_rec;
  g->last_mode = mode;
  g->step_instrumented = g->instrument && eager;
  RP_TRY(cuda_ok(cudaEventRecord(g->evStepBeg, g->sG), "record"));
  g->step_timed = true;
  if (eager) {
    RP_TRY(enqueue_step(g, mode));
    return cuda_ok(cudaEventRecord(g->evStepEnd, g->sG), "record");
  }
  if (!g->graph[mode]) {
    cudaGraph_t graph = nullptr;
    RP_TRY(cuda_ok(cudaStreamBeginCapture(g->sG, cudaStreamCaptureModeThreadLocal), "capture"));
    const int rc = enqueue_step(g, mode);
    const cudaError_t e = cudaStreamEndCapture(g->sG, &graph);
    if (rc != RP_OK) return rc;
    RP_TRY(cuda_ok(e, "end capture"));
    RP_TRY(cuda_ok(cudaGraphInstantiate(&g->graph[mode], graph, 0), "graph instantiate"));
    size_t nn = 0;
    cudaGraphGetNodes(graph, nullptr, &nn);
    std::vector<cudaGraphNode_t> nodes(nn);
    cudaGraphGetNodes(graph, nodes.data(), &nn);
    int64_t kernels = 0;
    for (auto nd : nodes) {
      cudaGraphNodeType t;
      cudaGraphNodeGetType(nd, &t);
      if (t == cudaGraphNodeTypeKernel) ++kernels;
    }
    g->graph_kernels[mode] = kernels;
    cudaGraphDestroy(graph);
  }
  RP_TRY(cuda_ok(cudaGraphLaunch(g->graph[mode], g->sG), "graph launch"));
  return cuda_ok(cudaEventRecord(g->evStepEnd, g->sG), "record");
}

extern "C" int rp_engine_sync(RpEngine* g) {
  if (!g) return rp_fail(RP_ERR_CONTRACT, "null engine");
  const cudaError_t e = cudaStreamSynchronize(g->sG);
  if (e != cudaSuccess) {
    std::string m = std::string("pipeline lane failed: ") + cudaGetErrorString(e);
    return rp_fail(RP_ERR_SCHEDULER, m.c_str());
  }
  return RP_OK;
}

extern "C" int rp_engine_read_loss(RpEngine* g, float* loss) {
  if (!g || !loss) return rp_fail(RP_ERR_CONTRACT, "null argument");
  RP_TRY(cuda_ok(cudaMemcpyAsync(loss, g->loss, sizeof(float), cudaMemcpyDeviceToHost, g->sG),
                 "read_loss"));
  return rp_engine_sync(g);
}

// Kernel launches per captured step (counted from the CUDA graph's kernel nodes).
extern "C" int64_t rp_engine_graph_kernels(const RpEngine* g, int mode) {
  return (g && mode >= 0 && mode <= 2) ? g->graph_kernels[mode] : -1;
}

// Runs one eager step with every tcgen05 GEMM launch bracketed by CUDA events on its own
// stream; returns the summed GEMM time (ms), FLOPs and launch count of that step.
extern "C" int rp_engine_gemm_profile(RpEngine* g, int mode, double* ms, double* flops,
                                      int64_t* launches) {
  if (!g) return rp_fail(RP_ERR_CONTRACT, "null engine");
  set_partition(g, mode);
  g->prof = true;
  const int rc = enqueue_step(g, mode);
  g->prof = false;
  RP_TRY(rc);
  RP_TRY(rp_engine_sync(g));
  double t = 0.0, f = 0.0;
  for (size_t i = 0; i < g->prof_used; ++i) {
    float x = 0.f;
    cudaEventElapsedTime(&x, g->prof_ev[i].first, g->prof_ev[i].second);
    t += x;
    f += g->prof_flops[i];
  }
  if (ms) *ms = t;
  if (flops) *flops = f;
  if (launches) *launches = static_cast<int64_t>(g->prof_used);
  return RP_OK;
}

extern "C" void* rp_engine_stream(RpEngine* g) { return g ? static_cast<void*>(g->sG) : nullptr; }

// Instrumented slot log (eager mode): per lane (0 = R, 1 = G) and block, start/end in ms
// relative to the first R slot. out: [2][L][2] floats.
extern "C" int rp_engine_set_instrument(RpEngine* g, int on) {
  if (!g) return rp_fail(RP_ERR_CONTRACT, "null engine");
  g->instrument = on != 0;
  return RP_OK;
}

extern "C" int rp_engine_slot_log(RpEngine* g, float* out) {
  if (!g || !out) return rp_fail(RP_ERR_CONTRACT, "null argument");
  RP_TRY(rp_engine_sync(g));
  cudaEvent_t ref = g->ts[static_cast<size_t>((0 * g->L + (g->L - 1)) * 2)];
  for (int lane = 0; lane < 2; ++lane)
    for (int64_t b = 0; b < g->L; ++b)
      for (int w = 0; w < 2; ++w) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ref, g->ts[static_cast<size_t>(((lane * g->L) + b) * 2 + w)]);
        out[(lane * g->L + b) * 2 + w] = ms;
      }
  return RP_OK;
}

// ---------------------------------------------------------------- data parallel (NCCL)
extern "C" int rp_nccl_unique_id(uint8_t* out128) {
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return rp_fail(RP_ERR_CUDA, ncclGetErrorString(r));
  std::memcpy(out128, id.internal, NCCL_UNIQUE_ID_BYTES);
  return RP_OK;
}

extern "C" int rp_engine_comm_init(RpEngine* g, const uint8_t* id128, int world, int rank) {
  if (!g || !id128) return rp_fail(RP_ERR_CONTRACT, "null argument");
  if (world < 1 || rank < 0 || rank >= world) return rp_fail(RP_ERR_CONFIG, "bad world/rank");
  // world == 1 also builds a (single-rank) communicator: the NCCL path of the step --
  // per-block bucket all-reduce on the comm stream inside the captured graph -- then runs
  // and is testable on one GPU
  if (g->comm) return rp_fail(RP_ERR_CONTRACT, "comm_init: communicator already initialised");
  ncclUniqueId id;
  std::memcpy(id.internal, id128, NCCL_UNIQUE_ID_BYTES);
  cudaSetDevice(g->dev);
  // Deterministic all-reduce: one algorithm and protocol for every bucket size (the
  // ring's reduction order is then fixed, so results repeat run to run and PaReprop equals
  // Reprop bit for bit at any world size). Caller settings win (setenv does not overwrite);
  // they must be in place before the process's first NCCL communicator is created.
  setenv("NCCL_ALGO", "Ring", 0);
  setenv("NCCL_PROTO", "Simple", 0);
  // a bounded number of NCCL CTAs, and as many SMs kept free of backward GEMM CTAs
  const int ctas = g->cfg.comm_ctas > 0 ? g->cfg.comm_ctas : 4;
  ncclConfig_t nc = NCCL_CONFIG_INITIALIZER;
  nc.blocking = 1;
  nc.minCTAs = std::min(2, ctas);
  nc.maxCTAs = ctas;
  ncclResult_t r = ncclCommInitRankConfig(&g->comm, world, id, rank, &nc);
  if (r != ncclSuccess) return rp_fail(RP_ERR_CUDA, ncclGetErrorString(r));
  g->world = world;
  g->rank = rank;
  g->comm_reserve = world > 1 ? (ctas + 1) / 2 * 2 : 0;  // whole CTA pairs
  for (auto& x : g->graph)
    if (x) {
      cudaGraphExecDestroy(x);
      x = nullptr;
    }
  return RP_OK;
}

// ---------------------------------------------------------------- block-level entry points
// (revcore on device pointers owned by the caller; params are the engine's block b)
// rev_forward: (i1, i2) -> (o1, o2), fp32 [T_s, d_s] of block b's stage
extern "C" int rp_engine_rev_forward(RpEngine* g, int64_t b, const float* i1, const float* i2,
                                     float* o1, float* o2) {
  if (!g || b < 0 || b >= g->L) return rp_fail(RP_ERR_CONTRACT, "bad engine/block");
  RP_TRY(wait_caller(g));
  cudaStream_t s = g->sG;
  RpStage& St = stage_of(g, b);
  const int64_t j = b - St.first;
  const size_t bytes = static_cast<size_t>(St.T * St.d) * 4;
  // stage the pair into X_j (b's input slots) so the forward plans can be reused
  RP_TRY(cuda_ok(cudaMemcpyAsync(X1(g, St, j), i1, bytes, cudaMemcpyDeviceToDevice, s), "copy"));
  if (j > 0) RP_TRY(cuda_ok(cudaMemcpyAsync(X2(g, St, j), i2, bytes, cudaMemcpyDeviceToDevice, s), "copy"));
  else if (i1 != i2) return rp_fail(RP_ERR_CONTRACT, "a stage's first block input is the duplicated stage input (i1 == i2)");
  BlockPlans& p = g->plans[static_cast<size_t>(b)];
  Slot& F = g->slot[0];
  RP_TRY(ln_fwd(g, St, X1(g, St, j), tix_block(g, b, kLnFg), tix_block(g, b, kLnFb), F.hF, F.meanF,
                F.rstdF, s));
  RP_TRY(launch(p.f_qkv, s));
  RP_TRY(attn_fwd(St, F.qkv, F.att, F.lse, s));
  RP_TRY(launch(p.f_proj, s));
  RP_TRY(ln_fwd(g, St, X2(g, St, j + 1), tix_block(g, b, kLnGg), tix_block(g, b, kLnGb), F.hF,
                F.meanF, F.rstdF, s));
  RP_TRY(launch(p.f_w1, s));
  RP_TRY(launch(p.f_w2, s));
  RP_TRY(cuda_ok(cudaMemcpyAsync(o1, X1(g, St, j + 1), bytes, cudaMemcpyDeviceToDevice, s), "copy"));
  RP_TRY(cuda_ok(cudaMemcpyAsync(o2, X2(g, St, j + 1), bytes, cudaMemcpyDeviceToDevice, s), "copy"));
  return rp_engine_sync(g);
}

// rev_backward_local for a block that is not its stage's first:
// (o1, o2, d_o1, d_o2) -> (i1, i2, d_i1, d_i2) + the block's grads in the engine grad buffer.
extern "C" int rp_engine_rev_backward_local(RpEngine* g, int64_t b, const float* o1,
                                            const float* o2, const float* d_o1,
                                            const float* d_o2, float* i1, float* i2,
                                            float* d_i1, float* d_i2) {
  if (!g || b < 1 || b >= g->L) return rp_fail(RP_ERR_CONTRACT, "bad engine/block (b >= 1)");
  RpStage& St = stage_of(g, b);
  const int64_t j = b - St.first;
  if (j < 1) return rp_fail(RP_ERR_CONTRACT, "rev_backward_local: block is its stage's first");
  RP_TRY(wait_caller(g));
  cudaStream_t s = g->sG;
  const int64_t n = St.T * St.d;
  const size_t bytes = static_cast<size_t>(n) * 4;
  RP_TRY(cuda_ok(cudaMemcpyAsync(X1(g, St, j + 1), o1, bytes, cudaMemcpyDeviceToDevice, s), "copy"));
  RP_TRY(cuda_ok(cudaMemcpyAsync(X2(g, St, j + 1), o2, bytes, cudaMemcpyDeviceToDevice, s), "copy"));
  RP_TRY(cuda_ok(cudaMemcpyAsync(g->d1, d_o1, bytes, cudaMemcpyDeviceToDevice, s), "copy"));
  RP_TRY(cuda_ok(cudaMemcpyAsync(g->d2, d_o2, bytes, cudaMemcpyDeviceToDevice, s), "copy"));
  RP_TRY(rpk_f32_to_bf16(g->d1, g->d1b, n, s));
  RP_TRY(rpk_f32_to_bf16(g->d2, g->d2b, n, s));
  set_partition(g, 1);
  RP_TRY(lane_r(g, b, s));
  RP_TRY(lane_g(g, b, s, true, false));
  RP_TRY(cuda_ok(cudaMemcpyAsync(i1, X1(g, St, j), bytes, cudaMemcpyDeviceToDevice, s), "copy"));
  RP_TRY(cuda_ok(cudaMemcpyAsync(i2, X2(g, St, j), bytes, cudaMemcpyDeviceToDevice, s), "copy"));
  RP_TRY(cuda_ok(cudaMemcpyAsync(d_i1, g->d1, bytes, cudaMemcpyDeviceToDevice, s), "copy"));
  RP_TRY(cuda_ok(cudaMemcpyAsync(d_i2, g->d2, bytes, cudaMemcpyDeviceToDevice, s), "copy"));
  return rp_engine_sync(g);
}

// rev_inverse for a block that is not its stage's first:
// (o1, o2) -> (i1, i2) = (o1 - G(o2), o2 - F(i1)); one F and one G evaluation.
extern "C" int rp_engine_rev_inverse(RpEngine* g, int64_t b, const float* o1, const float* o2,
                                     float* i1, float* i2) {
  if (!g || b < 1 || b >= g->L) return rp_fail(RP_ERR_CONTRACT, "bad engine/block (b >= 1)");
  RpStage& St = stage_of(g, b);
  const int64_t j = b - St.first;
  if (j < 1) return rp_fail(RP_ERR_CONTRACT, "rev_inverse: block is its stage's first");
  RP_TRY(wait_caller(g));
  cudaStream_t s = g->sG;
  const size_t bytes = static_cast<size_t>(St.T * St.d) * 4;
  RP_TRY(cuda_ok(cudaMemcpyAsync(X1(g, St, j + 1), o1, bytes, cudaMemcpyDeviceToDevice, s), "copy"));
  RP_TRY(cuda_ok(cudaMemcpyAsync(X2(g, St, j + 1), o2, bytes, cudaMemcpyDeviceToDevice, s), "copy"));
  set_partition(g, 1);
  RP_TRY(lane_r(g, b, s));
  RP_TRY(cuda_ok(cudaMemcpyAsync(i1, X1(g, St, j), bytes, cudaMemcpyDeviceToDevice, s), "copy"));
  RP_TRY(cuda_ok(cudaMemcpyAsync(i2, X2(g, St, j), bytes, cudaMemcpyDeviceToDevice, s), "copy"));
  return rp_engine_sync(g);
}

// Stage boundary after stage `stage` (hierarchical models; ref:proj/core/src/layers.cpp:261-303):
// forward  y = patch_merge(fuse(o1, o2)) -> fp32 [T_{s+1}, d_{s+1}] (the next stage's input);
// backward given the next stage's input cotangents (d_i1, d_i2, fp32): the stage output's
// cotangents (d_o1, d_o2) and the boundary's parameter grads in the engine grad buffer.
extern "C" int rp_engine_boundary_forward(RpEngine* g, int64_t stage, const float* o1,
                                          const float* o2, float* y) {
  if (!g || stage < 0 || stage + 1 >= static_cast<int64_t>(g->st.size()))
    return rp_fail(RP_ERR_CONTRACT, "boundary_forward: no boundary after this stage");
  RpStage& St = g->st[static_cast<size_t>(stage)];
  const RpStage& Nx = g->st[static_cast<size_t>(stage) + 1];
  RP_TRY(wait_caller(g));
  cudaStream_t s = g->sG;
  const size_t bytes = static_cast<size_t>(St.T * St.d) * 4;
  RP_TRY(cuda_ok(cudaMemcpyAsync(X1(g, St, St.L), o1, bytes, cudaMemcpyDeviceToDevice, s), "copy"));
  RP_TRY(cuda_ok(cudaMemcpyAsync(X2(g, St, St.L), o2, bytes, cudaMemcpyDeviceToDevice, s), "copy"));
  RP_TRY(boundary_fuse(g, St, s));
  RP_TRY(launch(St.b_merge, s));
  RP_TRY(cuda_ok(cudaMemcpyAsync(y, Nx.e, static_cast<size_t>(Nx.T * Nx.d) * 4,
                                 cudaMemcpyDeviceToDevice, s),
                 "copy"));
  return rp_engine_sync(g);
}

extern "C" int rp_engine_boundary_vjp(RpEngine* g, int64_t stage, const float* o1,
                                      const float* o2, const float* d_i1, const float* d_i2,
                                      float* d_o1, float* d_o2) {
  if (!g || stage < 0 || stage + 1 >= static_cast<int64_t>(g->st.size()))
    return rp_fail(RP_ERR_CONTRACT, "boundary_vjp: no boundary after this stage");
  RpStage& St = g->st[static_cast<size_t>(stage)];
  const RpStage& Nx = g->st[static_cast<size_t>(stage) + 1];
  RP_TRY(wait_caller(g));
  cudaStream_t s = g->sG;
  const size_t bytes = static_cast<size_t>(St.T * St.d) * 4;
  const size_t nbytes = static_cast<size_t>(Nx.T * Nx.d) * 4;
  RP_TRY(cuda_ok(cudaMemcpyAsync(X1(g, St, St.L), o1, bytes, cudaMemcpyDeviceToDevice, s), "copy"));
  RP_TRY(cuda_ok(cudaMemcpyAsync(X2(g, St, St.L), o2, bytes, cudaMemcpyDeviceToDevice, s), "copy"));
  RP_TRY(cuda_ok(cudaMemcpyAsync(g->d1, d_i1, nbytes, cudaMemcpyDeviceToDevice, s), "copy"));
  RP_TRY(cuda_ok(cudaMemcpyAsync(g->d2, d_i2, nbytes, cudaMemcpyDeviceToDevice, s), "copy"));
  set_partition(g, 1);
  RP_TRY(boundary_fuse(g, St, s));
  RP_TRY(boundary_vjp(g, St, s));
  RP_TRY(cuda_ok(cudaMemcpyAsync(d_o1, g->d1, bytes, cudaMemcpyDeviceToDevice, s), "copy"));
  RP_TRY(cuda_ok(cudaMemcpyAsync(d_o2, g->d2, bytes, cudaMemcpyDeviceToDevice, s), "copy"));
  return rp_engine_sync(g);
}

// ---------------------------------------------------------------- layer-level entry points
// The reference's F / G layer API (ref:proj/core/include/revprop/layers.hpp:82-138) on
// block b's parameters, device pointers fp32 [T_s, d_s]; VJP parameter grads land in the
// engine's gradient buffer (block b's slices), the input cotangent in d_x.
namespace {
int layer_check(RpEngine* g, int64_t b) {
  if (!g || b < 0 || b >= g->L) return rp_fail(RP_ERR_CONTRACT, "bad engine/block");
  return RP_OK;
}
}  // namespace

// attention_forward (layers.cpp:134-169): y = Proj(MHSA(LN(x))), no residual
extern "C" int rp_engine_attention_forward(RpEngine* g, int64_t b, const float* x, float* y) {
  RP_TRY(layer_check(g, b));
  RP_TRY(wait_caller(g));
  RpStage& St = stage_of(g, b);
  BlockPlans& p = g->plans[static_cast<size_t>(b)];
  Slot& F = g->slot[0];
  cudaStream_t s = g->sG;
  set_partition(g, 1);
  RP_TRY(ln_fwd(g, St, x, tix_block(g, b, kLnFg), tix_block(g, b, kLnFb), F.hF, F.meanF, F.rstdF, s));
  RP_TRY(launch(p.f_qkv, s));
  RP_TRY(attn_fwd(St, F.qkv, F.att, F.lse, s));
  RpGemmDesc dsc{};
  dsc.A = F.att;
  dsc.lda = St.d;
  dsc.B = wb(g, tix_block(g, b, kWout));
  dsc.ldb = St.d;
  dsc.b_mn = 1;
  dsc.M = St.T;
  dsc.N = St.d;
  dsc.K = St.d;
  dsc.epi = RP_EPI_F32;
  dsc.out = y;
  dsc.ldo = St.d;
  dsc.splits = 1;
  dsc.bn = gemm_bn(dsc.N);
  RP_TRY(rp_gemm(&dsc, s));
  return rp_engine_sync(g);
}

// mlp_forward (layers.cpp:222-239): y = W2 gelu(W1 LN(x) + b1) + b2, no residual
extern "C" int rp_engine_mlp_forward(RpEngine* g, int64_t b, const float* x, float* y) {
  RP_TRY(layer_check(g, b));
  RP_TRY(wait_caller(g));
  RpStage& St = stage_of(g, b);
  BlockPlans& p = g->plans[static_cast<size_t>(b)];
  Slot& F = g->slot[0];
  cudaStream_t s = g->sG;
  set_partition(g, 1);
  RP_TRY(ln_fwd(g, St, x, tix_block(g, b, kLnGg), tix_block(g, b, kLnGb), F.hF, F.meanF, F.rstdF, s));
  RP_TRY(launch(p.f_w1, s));  // F.a = gelu(hG W1 + b1)
  RP_TRY(cuda_ok(cudaMemsetAsync(y, 0, static_cast<size_t>(St.T * St.d) * 4, s), "memset"));
  RpGemmDesc dsc{};
  dsc.A = F.a;
  dsc.lda = St.h;
  dsc.B = wb(g, tix_block(g, b, kW2));
  dsc.ldb = St.d;
  dsc.b_mn = 1;
  dsc.M = St.T;
  dsc.N = St.d;
  dsc.K = St.h;
  dsc.epi = RP_EPI_RESID;  // y = 0 + (a W2 + b2)
  dsc.out = y;
  dsc.ldo = St.d;
  dsc.aux = y;
  dsc.ldaux = St.d;
  dsc.bias = wf(g, tix_block(g, b, kB2));
  dsc.sign = 1.f;
  dsc.splits = 1;
  dsc.bn = gemm_bn(dsc.N);
  RP_TRY(rp_gemm(&dsc, s));
  return rp_engine_sync(g);
}

// attention_vjp (layers.cpp:171-220): d_x and the F parameter grads of d_y, caches
// recomputed from x
extern "C" int rp_engine_attention_vjp(RpEngine* g, int64_t b, const float* x, const float* d_y,
                                       float* d_x) {
  RP_TRY(layer_check(g, b));
  RP_TRY(wait_caller(g));
  RpStage& St = stage_of(g, b);
  const int64_t j = b - St.first, n = St.T * St.d;
  cudaStream_t s = g->sG;
  set_partition(g, 1);
  const size_t bytes = static_cast<size_t>(n) * 4;
  RP_TRY(cuda_ok(cudaMemcpyAsync(X1(g, St, j), x, bytes, cudaMemcpyDeviceToDevice, s), "copy"));
  RP_TRY(cuda_ok(cudaMemcpyAsync(g->d2, d_y, bytes, cudaMemcpyDeviceToDevice, s), "copy"));
  RP_TRY(rpk_f32_to_bf16(g->d2, g->d2b, n, s));
  RP_TRY(cuda_ok(cudaMemsetAsync(g->d1, 0, bytes, s), "memset"));  // no residual cotangent
  RP_TRY(recompute_f(g, b, s, false));
  RP_TRY(vjp_f(g, b, s, false));
  RP_TRY(cuda_ok(cudaMemcpyAsync(d_x, g->d1, bytes, cudaMemcpyDeviceToDevice, s), "copy"));
  return rp_engine_sync(g);
}

// mlp_vjp (layers.cpp:241-259): d_x and the G parameter grads of d_y, caches recomputed
// from x
extern "C" int rp_engine_mlp_vjp(RpEngine* g, int64_t b, const float* x, const float* d_y,
                                 float* d_x) {
  RP_TRY(layer_check(g, b));
  RP_TRY(wait_caller(g));
  RpStage& St = stage_of(g, b);
  const int64_t j = b - St.first, n = St.T * St.d;
  cudaStream_t s = g->sG;
  set_partition(g, 1);
  const size_t bytes = static_cast<size_t>(n) * 4;
  RP_TRY(cuda_ok(cudaMemcpyAsync(X2(g, St, j + 1), x, bytes, cudaMemcpyDeviceToDevice, s), "copy"));
  RP_TRY(cuda_ok(cudaMemcpyAsync(g->d1, d_y, bytes, cudaMemcpyDeviceToDevice, s), "copy"));
  RP_TRY(rpk_f32_to_bf16(g->d1, g->d1b, n, s));
  RP_TRY(cuda_ok(cudaMemsetAsync(g->d2, 0, bytes, s), "memset"));  // no residual cotangent
  RP_TRY(recompute_g(g, b, s, false));
  RP_TRY(vjp_g(g, b, s, true));
  RP_TRY(cuda_ok(cudaMemcpyAsync(d_x, g->d2, bytes, cudaMemcpyDeviceToDevice, s), "copy"));
  return rp_engine_sync(g);
}

// ---------------------------------------------------------------- stream contract, trace, stats
extern "C" int rp_engine_set_caller_stream(RpEngine* g, rp_stream_t stream) {
  if (!g) return rp_fail(RP_ERR_CONTRACT, "null engine");
  g->caller = static_cast<cudaStream_t>(stream);
  return RP_OK;
}

extern "C" int64_t rp_engine_trace_floats(const RpEngine* g) {
  return g ? g->trace_off.back() : -1;
}

extern "C" int rp_engine_set_trace(RpEngine* g, float* fwd, float* rec) {
  if (!g) return rp_fail(RP_ERR_CONTRACT, "null engine");
  g->trace_fwd = fwd;
  g->trace_rec = rec;
  return RP_OK;
}

// StepStats of the last step: waits for it. wall_ns: device time between
// events recorded on the engine stream before and after the step; lane_busy_ns: sum of the
// lane's block slots (instrumented steps only, else -1); ledger peak / events and
// blocks_processed from the step's schedule; arena bytes as allocated.
extern "C" int rp_engine_step_stats(RpEngine* g, RpStepStats* out) {
  if (!g || !out) return rp_fail(RP_ERR_CONTRACT, "null argument");
  if (!g->step_timed) return rp_fail(RP_ERR_CONTRACT, "step_stats: no step has run");
  RP_TRY(rp_engine_sync(g));
  std::memset(out, 0, sizeof(*out));
  RP_TRY(cuda_ok(cudaMemcpy(&out->loss, g->loss, sizeof(float), cudaMemcpyDeviceToHost), "loss"));
  float ms = 0.f;
  RP_TRY(cuda_ok(cudaEventElapsedTime(&ms, g->evStepBeg, g->evStepEnd), "elapsed"));
  out->wall_ns = static_cast<int64_t>(static_cast<double>(ms) * 1e6);
  const int m = g->last_mode;
  out->mode = m;
  out->peak_activation_bytes = g->led_peak_m[m];
  out->ledger_events = g->led_events_m[m];
  out->blocks_processed = g->blocks_m[m];
  out->lane_busy_ns[0] = out->lane_busy_ns[1] = -1;
  if (g->step_instrumented) {
    for (int lane = 0; lane < 2; ++lane) {
      double busy = 0.0;
      for (int64_t b = 0; b < g->L; ++b) {
        float x = 0.f;
        cudaEventElapsedTime(&x, g->ts[static_cast<size_t>(((lane * g->L) + b) * 2)],
                             g->ts[static_cast<size_t>(((lane * g->L) + b) * 2 + 1)]);
        busy += x;
      }
      out->lane_busy_ns[lane] = static_cast<int64_t>(busy * 1e6);
    }
  }
  out->arena_activation_bytes = g->arena_bytes[1];
  out->arena_param_bytes = g->arena_bytes[2];
  out->arena_total_bytes = g->arena_bytes[0] + g->arena_bytes[1] + g->arena_bytes[2];
  return RP_OK;
}

// sgd_update(model, grads, lr) as a separate call: theta <- theta - lr * g
// over every parameter, with `host_grads` (the mean gradient, e.g. a GradStore the caller
// holds) or, when NULL, the last step's all-reduced gradient (1/world folded in). Refreshes
// the bf16 GEMM shadow. The in-step optimizer (rp_engine_set_lr) is the fused alternative.
extern "C" int rp_engine_sgd_update(RpEngine* g, const float* host_grads, float lr) {
  if (!g) return rp_fail(RP_ERR_CONTRACT, "null engine");
  float scale = 1.0f / static_cast<float>(g->world);
  if (host_grads) {
    RP_TRY(cuda_ok(cudaMemcpyAsync(g->grads, host_grads, static_cast<size_t>(g->P) * 4,
                                   cudaMemcpyHostToDevice, g->sG), "sgd_update grads"));
    scale = 1.0f;
  }
  RP_TRY(cuda_ok(cudaMemcpyAsync(g->lr_apply, &lr, sizeof(float), cudaMemcpyHostToDevice, g->sG),
                 "sgd_update lr"));
  RP_TRY(rpk_sgd(g->params, g->grads, g->pb, g->P, g->lr_apply, scale, g->sG));
  return rp_engine_sync(g);
}

// Timing experiments only (the step's results are garbage while set): flags 1 = lanes R and G
// free-running in PaReprop (no rendezvous: the upper bound of what overlapping them can
// gain), 2 = skip lane G, 4 = skip lane R. 0 restores the real schedule.
extern "C" int rp_engine_set_diag(RpEngine* g, int flags) {
  if (!g) return rp_fail(RP_ERR_CONTRACT, "null engine");
  if (flags < 0 || flags > 7) return rp_fail(RP_ERR_CONFIG, "diag flags must be in [0, 7]");
  g->diag = flags;
  return rp_engine_invalidate_graphs(g);
}
