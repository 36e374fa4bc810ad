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
  RP_EPI_GELU_BWD = 4   /* out(bf16) = acc * gelu'(aux(bf16) u)                   */
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
} RpGemmDesc;

typedef struct RpGemmPlan RpGemmPlan;
int rp_gemm_plan_create(const RpGemmDesc* desc, RpGemmPlan** plan);
int rp_gemm_plan_launch(const RpGemmPlan* plan, rp_stream_t stream);
int rp_gemm_plan_set_max_ctas(RpGemmPlan* plan, int max_ctas);
void rp_gemm_plan_destroy(RpGemmPlan* plan);
int rp_gemm(const RpGemmDesc* desc, rp_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* REVPROP_B200_H_ */
