/*
 * revprop_b200.h -- C ABI of the B200-native PaReprop training engine.
 *
 * Every entry point takes plain device/host pointers, int64 sizes and an opaque CUDA
 * stream (void*), and returns an int status. Status codes map one-to-one onto the
 * reference's exception hierarchy (ref:proj/core/include/revprop/errors.hpp:9-48):
 *
 *   RP_OK              0
 *   RP_ERR_SHAPE       1  -> revprop::ShapeError       (errors.hpp:15-18)
 *   RP_ERR_CONTRACT    2  -> revprop::ContractError    (errors.hpp:21-24)
 *   RP_ERR_CONFIG      3  -> revprop::ConfigError      (errors.hpp:27-30)
 *   RP_ERR_BUDGET      4  -> revprop::BudgetError      (errors.hpp:33-36)
 *   RP_ERR_SCHEDULER   5  -> revprop::SchedulerError   (errors.hpp:39-42)
 *   RP_ERR_ACCOUNTING  6  -> revprop::AccountingError  (errors.hpp:45-48)
 *   RP_ERR_CUDA        7  -> revprop::Error (device / driver failure)
 *
 * rp_last_error() returns a thread-local human-readable message for the last failure.
 * The caller owns every buffer; launchers never allocate. Matrices are row-major.
 * bf16 buffers are passed as uint16_t* (raw bf16 bit patterns).
 */
#ifndef REVPROP_B200_H_
#define REVPROP_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef void* rp_stream_t; /* cudaStream_t */

enum {
  RP_OK = 0,
  RP_ERR_SHAPE = 1,
  RP_ERR_CONTRACT = 2,
  RP_ERR_CONFIG = 3,
  RP_ERR_BUDGET = 4,
  RP_ERR_SCHEDULER = 5,
  RP_ERR_ACCOUNTING = 6,
  RP_ERR_CUDA = 7
};

const char* rp_last_error(void);
/* Programmatic dependent launch between consecutive kernels: 1 on, 0 (default) off. */
int rp_set_pdl(int on);
/* Library build / device information: writes "sm_100a ..." into buf. */
int rp_version(char* buf, int len);

/* ------------------------------------------------------------------ GEMM (tcgen05)
 * C[M,N] = sum_k A[m,k] B[k,n], bf16 in, fp32 accumulate (TMEM), fused epilogue.
 * Replaces ref:proj/core/src/ops.cpp:130-180 (matmul / matmul_tn / matmul_nt /
 * matmul_vjp) plus the bias/GELU/residual element-wise ops that follow them in
 * ref:proj/core/src/layers.cpp:208-259 (add_rowvec, gelu, gelu_vjp) and
 * ref:proj/core/src/ops.cpp:96-106 (the coupling add / sub).
 *   a_mn = 0: A stored [M][K] (pitch lda);  a_mn = 1: A stored [K][M]
 *   b_mn = 0: B stored [N][K] (pitch ldb);  b_mn = 1: B stored [K][N]
 */
enum {
  RP_EPI_BF16 = 0,      /* out(bf16) = acc                                        */
  RP_EPI_F32 = 1,       /* out(f32)  = acc  (split-K allowed: workspace [S][M][N]) */
  RP_EPI_BIAS_GELU = 2, /* u = acc + bias; out(bf16) = gelu(u); out2(bf16) = u    */
  RP_EPI_RESID = 3,     /* out(f32) = aux(f32) + sign * (acc + bias)              */
  RP_EPI_GELU_BWD = 4,  /* out(bf16) = acc * gelu'(aux(bf16) u)                   */
  RP_EPI_BIAS_GELU_SLOPE = 5, /* u = acc + bias; out(bf16) = gelu(u); out2(bf16) = gelu'(u) */
  RP_EPI_MUL = 6,       /* out(bf16) = acc * aux(bf16)  (MLP dgrad with the saved slope) */
  RP_EPI_ROWDOT = 7     /* out(bf16) = acc; and per 64-column head h of row r = s*rd_seq + t:
                           rowdot[(s*H + h)*rd_seq + t] = sum_c bf16(acc) aux(bf16), H = N/64
                           (the attention-backward D = rowsum(dO * O) from the d_att GEMM) */
};

typedef struct RpGemmDesc {
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
  void* out2; /* optional */
  int64_t ldo2;
  const void* aux; /* residual (f32) or u (bf16) */
  int64_t ldaux;
  const float* bias; /* optional, length N */
  float sign;
  int splits;       /* split-K count (RP_EPI_F32 only) */
  float* workspace; /* splits*M*N floats when splits > 1 */
  int max_ctas;     /* 0 = one CTA per SM */
  int bn;           /* tile N: 256 (default) or 128 */
  float* colsum_part; /* optional (RP_EPI_MUL / RP_EPI_GELU_BWD): column sums of the fp32
                         epilogue output per 32-row group, [ceil(M/32)][N]; reduce them with
                         rp_colsum_parts (the MLP hidden-bias gradient, layers.cpp:38-52) */
  float* rowdot;    /* RP_EPI_ROWDOT output */
  int64_t rd_seq;   /* RP_EPI_ROWDOT: rows per sequence (tokens per attention window) */
  float quantum;    /* RP_EPI_RESID / RP_EPI_F32 (no split-K): round acc (+ bias) to a multiple of
                       this power of two before the store / residual add (0 = off). With the
                       residual on the same grid the coupling's fp32 add and subtract are exact
                       (see RpModelConfig.exact_coupling_bits). */
} RpGemmDesc;

typedef struct RpGemmPlan RpGemmPlan;
int rp_gemm_plan_create(const RpGemmDesc* desc, RpGemmPlan** plan);
int rp_gemm_plan_launch(const RpGemmPlan* plan, rp_stream_t stream);
int rp_gemm_plan_set_max_ctas(RpGemmPlan* plan, int max_ctas);
void rp_gemm_plan_destroy(RpGemmPlan* plan);
int rp_gemm_plan_shape(const RpGemmPlan* plan, int64_t* M, int64_t* N, int64_t* K);
int rp_gemm(const RpGemmDesc* desc, rp_stream_t stream);
/* MMA issue form of the GEMM kernels (A/B switch, process-global, read at launch; captured
 * graphs keep theirs): 1 (default) the issuing warp stays converged and issues predicated on
 * one lane, 0 a single diverged lane issues. Same MMAs in the same order: bit-identical. */
int rp_set_mma_issue(int mode);
/* Instrumentation (tools/gemm_trace.py): a device buffer of 64 x 8 uint64 receives clock64
 * stamps of the CTA-pair GEMM's cluster 0 (per tile: accumulator wait / acquire / operand
 * wait cycles / last MMA; epilogue start / end). NULL turns it off. */
int rp_set_gemm_trace(void* device_buffer);

/* ------------------------------------------------------------------ LayerNorm / reductions
 * rp_layer_norm_fwd: ref:proj/core/src/ops.cpp:264-304 (y = x_hat*gamma + beta, two-pass
 *   population variance). x fp32 [rows, cols] -> y bf16, per-row mean / rstd (fp32).
 * rp_layer_norm_bwd: ref:proj/core/src/ops.cpp:306-345, fused with the coupling's cotangent
 *   add: dx = dres + LN^T(dy) (fp32, optional bf16 copy); dgamma/dbeta (+)= deterministic
 *   column sums. workspace: rp_layer_norm_bwd_workspace_floats(rows, cols) floats.
 * rp_colsum: ref:proj/core/src/layers.cpp:38-52 (col_sum, the MLP bias grads).
 */
int rp_layer_norm_fwd(const float* x, const float* gamma, const float* beta, int64_t rows,
                      int64_t cols, double eps, uint16_t* y, float* mean, float* rstd,
                      rp_stream_t stream);
int rp_layer_norm_bwd(const float* x, const float* mean, const float* rstd, const float* gamma,
                      const uint16_t* dy, const float* dres, int64_t rows, int64_t cols,
                      float* dx, uint16_t* dx_bf16, float* dgamma, float* dbeta,
                      float* workspace, int accumulate, rp_stream_t stream);
/* Same, plus (dx_colsum != NULL) dx_colsum[c] = sum_r dx[r][c] of the produced cotangent: the
 * next reversible block's MLP output-bias gradient (ref:proj/core/src/layers.cpp:38-52
 * col_sum over the same d_o1), computed in the same single pass over x, dy and dres. */
int rp_layer_norm_bwd_ex(const float* x, const float* mean, const float* rstd, const float* gamma,
                         const uint16_t* dy, const float* dres, int64_t rows, int64_t cols,
                         float* dx, uint16_t* dx_bf16, float* dgamma, float* dbeta,
                         float* dx_colsum, float* workspace, int accumulate, rp_stream_t stream);
/* 1 (default): single-pass backward; 0: row kernel + separate column-sum pass (A/B only). */
int rp_set_ln_bwd_impl(int impl);
int64_t rp_layer_norm_bwd_workspace_floats(int64_t rows, int64_t cols);
int rp_colsum(const void* in, int in_is_bf16, int64_t rows, int64_t cols, float* out,
              float* workspace, int accumulate, rp_stream_t stream);
/* out[c] (+)= sum_p part[p][c] in a fixed order (second stage of a column sum). */
/* out[c] (+)= sum_p part[p][c] in a fixed order; `part` is scratch afterwards (many parts
 * are reduced in place in slices first) */
int rp_colsum_parts(float* part, int64_t nparts, int64_t cols, float* out, int accumulate,
                    rp_stream_t stream);
int64_t rp_colsum_workspace_floats(int64_t rows, int64_t cols);

/* ------------------------------------------------------------------ attention (head_dim 64)
 * Replaces the per-(batch, head, window) loops of ref:proj/core/src/layers.cpp:150-166
 * (forward) and :185-208 (VJP). qkv [S*N, 3*H*64] bf16 (q | k | v, head i at column i*64,
 * layers.cpp:144-146), S independent sequences (batch x windows) of N tokens.
 * lse: [S][H][N] fp32 (log2 domain), kept instead of the probability tensor.
 * N <= 768. tcgen05 kernels: forward N <= 512 (single pass N <= 224, two-pass above),
 * backward N <= 768 (keys / queries streamed in 64-row chunks); mma.sync forward above 512.
 */
int rp_attention_fwd(const uint16_t* qkv, int64_t S, int64_t N, int64_t H, int64_t head_dim,
                     uint16_t* out, float* lse, rp_stream_t stream);
int rp_attention_bwd(const uint16_t* qkv, const uint16_t* out, const float* lse,
                     const uint16_t* dout, int64_t S, int64_t N, int64_t H, int64_t head_dim,
                     uint16_t* dqkv, float* workspace, rp_stream_t stream);
/* as rp_attention_bwd; d_ready = 1: D = rowsum(dO * O) is already in workspace[0, S N H)
 * (e.g. from an RP_EPI_ROWDOT d_att GEMM) and the tcgen05 path does not recompute it */
int rp_attention_bwd_ex(const uint16_t* qkv, const uint16_t* out, const float* lse,
                        const uint16_t* dout, int64_t S, int64_t N, int64_t H, int64_t head_dim,
                        uint16_t* dqkv, float* workspace, int d_ready, rp_stream_t stream);
/* D = rowsum(dO * O) (S N H floats) and, for the tcgen05 backward, the bf16 dS^T of every
 * (sequence, head) ([S H][Nk][Nk], Nk = N rounded up to 16) */
int64_t rp_attention_bwd_workspace_floats(int64_t S, int64_t N, int64_t H);
/* 0 (default): tcgen05 kernels where they apply; backward for N <= 208 = one fused pass per
 * (sequence, head, 128-key tile) with dS kept on chip, above that one dK/dV pass that also
 * writes dS^T + a dQ = dS K pass over it; 1: warp-level mma.sync only; 2: tcgen05 with the
 * two-pass backward (dQ pass, dK/dV pass, each recomputing S and dP; no dS stored);
 * 3: tcgen05 with the dS^T round trip at every N <= 256 (the round-1 default).
 * Process-global; other values are RP_ERR_CONFIG. Captured engine graphs keep the kernels
 * they were captured with: call rp_engine_invalidate_graphs after changing it. */
int rp_set_attention_impl(int impl);
/* tcgen05 forward for N <= 256 (A/B switch, process-global like the above): 0 (default) two
 * ping-pong groups of softmax warps on alternate query tiles, the P V product split by key half
 * over two issuing warps where it fits TMEM (N <= 208); 1 the lockstep kernel (N <= 224);
 * 2 the ping-pong kernel with one P V issuer */
int rp_set_attention_fwd_variant(int variant);
/* Windows of N <= 64 tokens (Swin), any head_dim (A/B switch, process-global like the above):
 * 0 (default) single-tile persistent kernels -- the backward one fused pass per (window, head)
 * with D = rowsum(P * dP) formed in the kernel; 1 the general mma.sync kernels (D pre-pass,
 * separate dK/dV and dQ passes) */
int rp_set_attention_window_variant(int variant);
/* Instrumentation: a device buffer of 64 x 12 uint64 receives clock64 stamps of the ping-pong
 * forward's CTA 0 (per tile: S issue, PV issue, softmax phases); NULL turns it off. */
int rp_set_attention_trace(void* device_buffer);

/* ------------------------------------------------------------------ training engine
 * Isotropic reversible model and its engines:
 * step_reprop (mode 1) and step_pareprop (mode 2, two CUDA streams), SGD, optional
 * data parallelism over NCCL. Parameters are one flat fp32 vector in the order
 *   embed_w [in,d] | per block: w_qkv [d,3d], w_out [d,d], lnF_gamma [d], lnF_beta [d],
 *   w1 [d,h], b1 [h], w2 [h,d], b2 [d], lnG_gamma [d], lnG_beta [d] | head_w [d,C]
 * (weights [in, out] row-major, as ref layers.hpp:43-52, 94-103: y = x . W).
 */
typedef struct RpModelConfig {
  int64_t depth, width, heads, hidden, seq_len, in_dim, num_classes, batch;
  int64_t window;  /* tokens per attention window; 0 = full attention */
  uint64_t seed;
  int device;
  int r_ctas; /* PaReprop: max CTAs per recompute-lane GEMM (0 = all SMs) */
  int g_ctas; /* PaReprop: max CTAs per gradient-lane GEMM (0 = all SMs) */
  int lane_priority; /* 1: gradient lane high / recompute lane low stream priority */
  int optimizer;     /* 0: SGD, 1: AdamW */
  float beta1, beta2, adam_eps, weight_decay;
  /* Hierarchical (Rev-Swin-style) model, SPEC.md:276-277 / 298-306 / 325: stages >= 2 stages
   * of stage_depth[s] blocks, width stage_width[s], stage_heads[s] heads, MLP hidden
   * stage_width[s] * hidden / width, seq_len / reduction^s tokens and attention windows of
   * min(window, tokens). Stage s >= 1 starts from patch_merge(fuse(stage s-1 output))
   * duplicated into both halves (ref:proj/core/src/layers.cpp:261-303). stages 0 or 1:
   * isotropic (depth / width / heads / hidden). Requires depth = sum of stage_depth,
   * width = stage_width[0], heads = stage_heads[0]. Parameters then follow the order
   *   embed_w | stage 0 blocks | merge_w_0 [(r d_0), d_1] (, fusion_w_0 [2 d_0, d_0]) |
   *   stage 1 blocks | ... | head_w [d_last, C]. */
  int64_t stages;
  int64_t stage_depth[8], stage_width[8], stage_heads[8];
  int64_t reduction; /* r: tokens merged per boundary group (2 sequences, 4 2-D grids) */
  int fusion;        /* BoundaryParams.fusion_kind: 0 average, 1 mlp */
  /* Data parallel (rp_engine_comm_init): NCCL CTAs per all-reduce (ncclConfig_t maxCTAs;
   * 0 = 4). With world > 1 the backward GEMMs leave as many SMs (rounded up to CTA pairs)
   * free for them, so bucket all-reduces overlap the backward instead of queueing behind
   * the persistent GEMM grids. */
  int comm_ctas;
  /* Exact coupling (0 = default 17; -1 = off): F's and G's outputs (and the embedding /
   * patch-merge outputs that start a stage) are rounded to multiples of 2^-bits in their
   * GEMM epilogues, so every residual-stream value is on that grid and the fp32
   * o2 = i2 + F(i1), o1 = i1 + G(o2) and the inverse's subtractions are exact while
   * |X| < 2^(24 - bits) (128 at 17). The inverse then reconstructs every block input bit
   * for bit at any depth (the recompute sees the forward's exact inputs, so its bf16 GEMM
   * operands round identically), instead of compounding fp32 round-trip error through the
   * bf16 roundings. Cost: one rounding of at most 2^-(bits+1) per coupling add. */
  int exact_coupling_bits;
} RpModelConfig;

/* Ledger-predicted peak activation bytes of an engine (mode 0 vanilla, 1 reprop,
 * 2 pareprop) and the per-block footprint, from the config alone (no device needed). */
int rp_activation_bytes(const RpModelConfig* cfg, int mode, int64_t* peak_bytes,
                        int64_t* block_footprint_bytes);

typedef struct RpEngine RpEngine;
int rp_engine_create(const RpModelConfig* cfg, RpEngine** engine);
void rp_engine_destroy(RpEngine* engine);
int64_t rp_engine_param_count(const RpEngine* engine);
int rp_engine_tensor_table(const RpEngine* engine, int64_t* offsets, int64_t* numels,
                           int64_t capacity);
int rp_engine_init_params(RpEngine* engine, uint64_t seed);
int rp_engine_synthetic_batch(RpEngine* engine, uint64_t seed);
int rp_engine_set_params(RpEngine* engine, const float* host_params);
int rp_engine_get_params(RpEngine* engine, float* host_params);
int rp_engine_get_grads(RpEngine* engine, float* host_grads);
int rp_engine_set_batch(RpEngine* engine, const uint16_t* host_inputs_bf16,
                        const int32_t* host_labels);
int rp_engine_set_batch_device(RpEngine* engine, const uint16_t* inputs_bf16,
                               const int32_t* labels);
/* Pipelined input: H2D copy of the next step's batch on a copy stream, overlapping the
 * current step; the next rp_engine_step consumes it. Host buffers pinned, valid until then. */
int rp_engine_prefetch_batch(RpEngine* engine, const uint16_t* host_inputs_bf16,
                             const int32_t* host_labels);
/* Asynchronous D2H of the last enqueued step's loss into pinned `loss`; rp_engine_wait_loss
 * blocks until it has landed. */
int rp_engine_read_loss_async(RpEngine* engine, float* loss);
int rp_engine_wait_loss(RpEngine* engine);
int rp_engine_set_lr(RpEngine* engine, float lr);
/* sgd_update as its own call: params -= lr * grads over the whole model, with
 * host_grads (the mean gradient, flat, engine order) or NULL = the last step's gradient.
 * Bit-identical to fp32 p - lr * g; refreshes the bf16 shadow. */
int rp_engine_sgd_update(RpEngine* engine, const float* host_grads, float lr);
int rp_engine_set_partition(RpEngine* engine, int r_ctas, int g_ctas);
int rp_engine_invalidate_graphs(RpEngine* engine);
/* Test hook of the verify command: kind 1 corrupts every block's F-path VJP
 * (propagated cotangent x 1.5), kind 0 restores it. */
int rp_engine_inject_fault(RpEngine* engine, int kind);
int rp_engine_enable_vanilla(RpEngine* engine);
/* mode: 0 vanilla (needs rp_engine_enable_vanilla), 1 reprop, 2 pareprop */
int rp_engine_step(RpEngine* engine, int mode, int use_graph);
int rp_engine_sync(RpEngine* engine);
int rp_engine_read_loss(RpEngine* engine, float* loss);
void* rp_engine_stream(RpEngine* engine);
int64_t rp_engine_graph_kernels(const RpEngine* engine, int mode);
int rp_engine_gemm_profile(RpEngine* engine, int mode, double* ms, double* flops,
                           int64_t* launches);
int rp_engine_set_instrument(RpEngine* engine, int on);
int rp_engine_slot_log(RpEngine* engine, float* out);

/* StepStats of the last step (the reference's MemoryLedger semantics,
 * ref:proj/core/include/revprop/ledger.hpp:18-104). Blocks until that step is done.
 *   wall_ns                device time of the step (events on the engine stream around it)
 *   peak_activation_bytes  peak of the live ledger: the step's enqueue replays every
 *                          activation buffer's lifetime as charge / release events in the
 *                          order the schedule allows on the device; equals
 *                          rp_activation_bytes() for isotropic models, <= it for
 *                          hierarchical ones (per-stage footprints); a release below zero
 *                          fails the step with RP_ERR_ACCOUNTING (AccountingError)
 *   lane_busy_ns[2]        lane R / lane G busy time, instrumented steps only (else -1)
 *   blocks_processed       reversible blocks run through the backward (== depth)
 *   arena_*_bytes          device bytes the engine actually allocated: activation storage
 *                          (what the ledger accounts), parameters / grads / optimizer
 *                          state, and everything (incl. workspaces) */
typedef struct RpStepStats {
  float loss;
  int mode;
  int64_t wall_ns;
  int64_t peak_activation_bytes;
  int64_t lane_busy_ns[2];
  int64_t blocks_processed;
  int64_t ledger_events;
  int64_t arena_activation_bytes;
  int64_t arena_param_bytes;
  int64_t arena_total_bytes;
} RpStepStats;
int rp_engine_step_stats(RpEngine* engine, RpStepStats* out);

/* Stream contract of the block / layer entry points below (rp_engine_rev_*,
 * rp_engine_boundary_*, rp_engine_attention_* / mlp_*, rp_engine_set_batch_device): they
 * read caller-owned device pointers on the engine's own (non-blocking) stream after waiting
 * for an event recorded on the caller's stream at entry, so everything the caller enqueued
 * on that stream before the call is visible. Default caller stream: the legacy default
 * stream (torch's default stream); set another with rp_engine_set_caller_stream. They return
 * after their results are complete (host-synchronous). */
int rp_engine_set_caller_stream(RpEngine* engine, rp_stream_t stream);

/* Recompute trace (test instrumentation): when set, eager steps copy every block's input
 * pair (i1 | i2, fp32 [T_s d_s] each) as the forward saw it into `fwd` and as lane R
 * reconstructed it in the backward into `rec` (the stage's first block: its stored input).
 * Buffers: rp_engine_trace_floats() floats each, device memory; block b at the sum over
 * earlier blocks of 2 T_s d_s. NULL turns it off. Traced steps never use the CUDA graph. */
int64_t rp_engine_trace_floats(const RpEngine* engine);
/* Timing experiments only -- a step's numbers are garbage while flags != 0: 1 runs PaReprop's
 * lanes R and G free (no rendezvous events; the upper bound of the overlap gain), 2 skips
 * lane G's kernels, 4 skips lane R's. 0 restores the real schedule. */
int rp_engine_set_diag(RpEngine* engine, int flags);
int rp_engine_set_trace(RpEngine* engine, float* fwd, float* rec);
/* Data parallelism over NCCL: one fp32 all-reduce (sum) per gradient
 * bucket on the engine's comm stream as soon as lane G finishes the bucket's owner, the
 * optimizer step of that bucket right after with 1/world folded in. The communicator is
 * created with ncclCommInitRankConfig (maxCTAs = comm_ctas); NCCL_ALGO=Ring and
 * NCCL_PROTO=Simple are set unless the caller set them (deterministic reduction order).
 * world == 1 builds a single-rank communicator (the same code path on one GPU).
 * rp_engine_get_grads then returns the MEAN of the ranks' gradients. */
int rp_nccl_unique_id(uint8_t* out128);
int rp_engine_comm_init(RpEngine* engine, const uint8_t* id128, int world, int rank);
/* The gradient buckets of a config in all-reduce order (no device needed): offsets / sizes
 * in floats into the flat parameter vector, kinds 0 embed, 1 block, 2 boundary, 3 head.
 * Returns the bucket count (negative status if cap is too small). */
int rp_model_bucket_plan(const RpModelConfig* cfg, int64_t* offsets, int64_t* sizes, int* kinds,
                         int64_t cap);
int rp_engine_rev_forward(RpEngine* engine, int64_t block, const float* i1, const float* i2,
                          float* o1, float* o2);
int rp_engine_rev_backward_local(RpEngine* engine, int64_t block, const float* o1,
                                 const float* o2, const float* d_o1, const float* d_o2,
                                 float* i1, float* i2, float* d_i1, float* d_i2);
/* rev_inverse for a block that is not its stage's first: (o1, o2) ->
 * (i1, i2) = (o1 - G(o2), o2 - F(i1)), fp32 [T_s, d_s] device pointers. */
int rp_engine_rev_inverse(RpEngine* engine, int64_t block, const float* o1, const float* o2,
                          float* i1, float* i2);
/* Hierarchical models: the stage boundary after `stage` (ref:proj/core/src/layers.cpp:261-303).
 * forward: y = patch_merge(fuse(o1, o2)), fp32 [T_{s+1}, d_{s+1}];
 * vjp: from the next stage's input cotangents (d_i1, d_i2) to the stage output's (d_o1,
 * d_o2); merge_w / fusion_w grads land in the engine's gradient buffer. */
int rp_engine_boundary_forward(RpEngine* engine, int64_t stage, const float* o1,
                               const float* o2, float* y);
int rp_engine_boundary_vjp(RpEngine* engine, int64_t stage, const float* o1, const float* o2,
                           const float* d_i1, const float* d_i2, float* d_o1, float* d_o2);
/* The reference's layer API on block `block`'s parameters (ref:proj/core/include/revprop/
 * layers.hpp:82-138), fp32 [T_s, d_s] device pointers, no residual inside:
 * attention_forward y = Proj(MHSA(LN_F(x))); mlp_forward y = W2 gelu(W1 LN_G(x) + b1) + b2;
 * the VJPs recompute their caches from x, write d_x and the layer's parameter grads into
 * the engine's gradient buffer. */
int rp_engine_attention_forward(RpEngine* engine, int64_t block, const float* x, float* y);
int rp_engine_mlp_forward(RpEngine* engine, int64_t block, const float* x, float* y);
int rp_engine_attention_vjp(RpEngine* engine, int64_t block, const float* x, const float* d_y,
                            float* d_x);
int rp_engine_mlp_vjp(RpEngine* engine, int64_t block, const float* x, const float* d_y,
                      float* d_x);

/* ------------------------------------------------------------------ reference layer API
 * The reference's pure layer / revcore / optimizer functions over CALLER-owned device
 * tensors, no engine (include/revprop_b200.hpp wraps them in the reference's names and
 * types). fp32 device pointers in the reference's layouts: activations [batch, tokens, width]
 * row-major, weights [in, out] row-major (layers.hpp:43-52, 94-103). Work is enqueued on
 * `stream`; temporaries are stream-ordered allocations; results are complete when the
 * stream is. */
typedef struct RpAttentionParamsDev { /* AttentionParams, layers.hpp:43-52 */
  const float* w_qkv;    /* [width, 3 width], no bias */
  const float* w_out;    /* [width, width], no bias */
  const float* ln_gamma; /* [width] */
  const float* ln_beta;  /* [width] */
  int64_t width, heads;
  int64_t window;        /* tokens per attention window; 0 = full attention */
} RpAttentionParamsDev;
typedef struct RpMlpParamsDev { /* MlpParams, layers.hpp:94-103 */
  const float *w1, *b1, *w2, *b2, *ln_gamma, *ln_beta; /* [d,h] [h] [h,d] [d] [d] [d] */
  int64_t width, hidden;
} RpMlpParamsDev;
typedef struct RpAttentionGradsDev { /* AttentionGrads, layers.hpp:67-72 (NULL = skip) */
  float *d_w_qkv, *d_w_out, *d_ln_gamma, *d_ln_beta;
} RpAttentionGradsDev;
typedef struct RpMlpGradsDev { /* MlpGrads, layers.hpp:116-123 (NULL = skip) */
  float *d_w1, *d_b1, *d_w2, *d_b2, *d_ln_gamma, *d_ln_beta;
} RpMlpGradsDev;
/* AttentionCache / MlpCache (layers.hpp:54-65, 105-114): opaque, owns its device buffers
 * (the layer's input, LayerNorm statistics, bf16 operands, log-sum-exp instead of the
 * probability tensor). A VJP given the other layer's cache is RP_ERR_CONTRACT. */
typedef struct RpLayerCache RpLayerCache;
/* y = Proj(MHSA(LN(x))) (layers.hpp:82, layers.cpp:134-169); cache may be NULL */
int rp_attention_forward(const RpAttentionParamsDev* p, const float* x, int64_t batch,
                         int64_t tokens, float* y, RpLayerCache** cache, rp_stream_t stream);
/* d_x and the parameter grads of d_y (layers.hpp:89, layers.cpp:171-220) */
int rp_attention_vjp(const RpLayerCache* cache, const RpAttentionParamsDev* p, const float* d_y,
                     float* d_x, const RpAttentionGradsDev* grads, rp_stream_t stream);
/* y = W2 gelu(W1 LN(x) + b1) + b2 (layers.hpp:131, layers.cpp:222-239) */
int rp_mlp_forward(const RpMlpParamsDev* p, const float* x, int64_t batch, int64_t tokens,
                   float* y, RpLayerCache** cache, rp_stream_t stream);
/* layers.hpp:138, layers.cpp:241-259 */
int rp_mlp_vjp(const RpLayerCache* cache, const RpMlpParamsDev* p, const float* d_y, float* d_x,
               const RpMlpGradsDev* grads, rp_stream_t stream);
int64_t rp_layer_cache_bytes(const RpLayerCache* cache);
int rp_layer_cache_destroy(RpLayerCache* cache);

typedef struct RpRevBlockDev { RpAttentionParamsDev f; RpMlpParamsDev g; } RpRevBlockDev;
typedef struct RpRevBlockGradsDev { RpAttentionGradsDev d_f; RpMlpGradsDev d_g; } RpRevBlockGradsDev;
/* o2 = i2 + F(i1), o1 = i1 + G(o2) */
int rp_rev_forward(const RpRevBlockDev* block, int64_t batch, int64_t tokens, const float* i1,
                   const float* i2, float* o1, float* o2, rp_stream_t stream);
/* i1 = o1 - G(o2), i2 = o2 - F(i1) */
int rp_rev_inverse(const RpRevBlockDev* block, int64_t batch, int64_t tokens, const float* o1,
                   const float* o2, float* i1, float* i2, rp_stream_t stream);
/* recomputed inputs, input cotangents and the block's parameter grads */
int rp_rev_backward_local(const RpRevBlockDev* block, int64_t batch, int64_t tokens,
                          const float* o1, const float* o2, const float* d_o1, const float* d_o2,
                          float* i1, float* i2, float* d_i1, float* d_i2,
                          const RpRevBlockGradsDev* grads, rp_stream_t stream);
/* params <- params - lr * grads (fp32, bit-identical to the host formula) */
int rp_sgd_update(float* params, const float* grads, int64_t n, float lr, rp_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* REVPROP_B200_H_ */
