// Host launchers of the model-glue kernels (model_kernels.cu); internal to the library.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

uint64_t rp_rng_u64_host(uint64_t seed, uint64_t stream, uint64_t counter);
int rpk_init_tensor(float* p, int64_t n, uint64_t seed, uint64_t tensor_idx, int kind,
                    double sigma, cudaStream_t s);
int rpk_init_inputs(uint16_t* x, int64_t n, uint64_t seed, cudaStream_t s);
int rpk_f32_to_bf16(const float* in, uint16_t* out, int64_t n, cudaStream_t s);
int rpk_sgd(float* p, const float* g, uint16_t* pb, int64_t n, const float* lr, float scale,
            cudaStream_t s);
int rpk_pool(const float* o1, const float* o2, int64_t B, int64_t N, int64_t d, float* pooled,
             cudaStream_t s);
int rpk_simt_gemm(int64_t M, int64_t N, int64_t K, const float* A, int64_t sam, int64_t sak,
                  const float* B, int64_t sbk, int64_t sbn, float* C, int64_t ldc,
                  cudaStream_t s);
int rpk_cross_entropy(const float* logits, const int32_t* labels, int64_t B, int64_t C,
                      float* d_logits, float* row_loss, float* loss, cudaStream_t s);
int rpk_spread(const float* d_pooled, int64_t B, int64_t N, int64_t d, float* d1, float* d2,
               uint16_t* d1b, uint16_t* d2b, cudaStream_t s);
int rpk_add_to_bf16(const float* a, const float* b, uint16_t* out, int64_t n, cudaStream_t s);
int rpk_adamw(float* p, const float* g, uint16_t* pb, float* m, float* v, int64_t n,
              const float* lr, const float* t, float b1, float b2, float eps, float wd,
              float scale, cudaStream_t s);
int rpk_add_scalar(float* x, float a, cudaStream_t s);
// stage boundary (layers.cpp:276-303)
int rpk_fuse_avg_bf16(const float* o1, const float* o2, int64_t n, uint16_t* out, cudaStream_t s);
int rpk_concat_bf16(const float* o1, const float* o2, int64_t rows, int64_t d, uint16_t* out,
                    cudaStream_t s);
int rpk_halve_dup(float* d1, int64_t n, float* d2, uint16_t* d1b, uint16_t* d2b, cudaStream_t s);
int rpk_scale_pair(float* x, uint16_t* xb, int64_t n, float s, cudaStream_t st);
// standalone revcore / optimizer entry points (layers_api.cpp)
int rpk_axpy_sign(const float* a, const float* b, float sign, float* out, int64_t n,
                  cudaStream_t s);
int rpk_sgd_value(float* p, const float* g, int64_t n, float lr, cudaStream_t s);
