#pragma once
#include "../../include/revprop_b200.h"

namespace rp {
// Device-side view of an RpGemmDesc epilogue (plain POD, passed by value to the kernel).
struct GemmEpi {
  void* out;
  int64_t ldo;
  void* out2;
  int64_t ldo2;
  const void* aux;
  int64_t ldaux;
  const float* bias;
  float sign;
  int64_t split_stride;
  float* colsum;  // optional: per-32-row column partials [ceil(M/32)][ldcs] of the fp32 output
  int64_t ldcs;
  float* rowdot;   // RP_EPI_ROWDOT: per-(row, 64-column head) dot of the bf16 output with aux
  int64_t rd_seq;  // rows per sequence
  int64_t rd_heads;
  // RP_EPI_RESID / RP_EPI_F32: round the GEMM result (+ bias) to a multiple of quant (a power
  // of two; 0 = off) before it is stored / added to the residual: the exact-coupling grid
  float quant, inv_quant;
};
}  // namespace rp
