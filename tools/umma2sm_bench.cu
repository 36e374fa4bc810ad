// Microbenchmark: tcgen05.mma.cta_group::2 (M = 256, N = 256, K = 16, SS) issue rate with
// one or two issuing warps in the leader CTA (each into its own 256-column accumulator), with
// and without a concurrent bulk-copy stream into both CTAs' shared memory (the TMA operand
// writes a GEMM pipeline does at the same time). Answers: is the CTA-pair GEMM main loop
// bound by the single issuer (~172 cycles per MMA, tools/umma_bench.cu) or by shared-memory
// bandwidth (operand reads + TMA writes)?
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2306_09342_b200/csrc \
//        tools/umma2sm_bench.cu -o tools/umma2sm_bench && ./tools/umma2sm_bench
#include <cstdio>

#include "ptx.cuh"

using namespace rp;

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}

constexpr int kOpBytes = 65536;   // A (4 x 16 KB k16 steps... 64 rows of SW128) | B
constexpr int kCopyBytes = 65536; // bulk-copy landing zone (2 x 32 KB)

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    bench2(int n, int issuers, int ncopy, const uint8_t* __restrict__ gsrc, long long* out, int N,
           int cg1) {
  extern __shared__ uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) &
                                           ~static_cast<uintptr_t>(1023));
  __shared__ __align__(8) uint64_t bars[4];
  __shared__ uint32_t slot;
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  for (int i = threadIdx.x; i < kOpBytes / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) mbar_init(&bars[i], 1);
    fence_barrier_init();
  }
  fence_proxy_async_smem();
  cluster_sync_all();
  if (warp == 1) tmem_alloc_2sm(&slot, 512);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = slot;
  long long t_mma = 0, t_copy = 0;
  if (warp < 2 && static_cast<int>(warp) < issuers && rank == 0) {
    const uint32_t idesc = make_idesc_bf16(cg1 ? 128 : 256, static_cast<uint32_t>(N), false, false);
    const uint32_t a = smem_u32(sm), b = smem_u32(sm + 32768);
    uint64_t ad[4], bd[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      ad[j] = make_sdesc_sw128(a + j * 32, 16, 1024);
      bd[j] = make_sdesc_sw128(b + j * 32, 16, 1024);
    }
    const uint32_t d = tmem + warp * 256u;
    const uint32_t is0 = lane == 0 ? 1u : 0u;
    __syncwarp();
    const long long t0 = clock64();
    for (int i = 0; i < n; i += 8) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (cg1)
          umma_bf16_pred(d, ad[j & 3], bd[j & 3], idesc, 1u, is0);
        else
          umma_bf16_2sm_pred(d, ad[j & 3], bd[j & 3], idesc, 1u, is0);
      }
    }
    if (cg1)
      umma_commit_pred(&bars[warp], is0);
    else
      umma_commit_2sm_mc_pred(&bars[warp], 0x3, is0);
    __syncwarp();
    mbar_wait(&bars[warp], 0);
    t_mma = clock64() - t0;
  } else if (warp == 3 && ncopy > 0) {
    // bulk copies from a small (L2-resident) global buffer, 16 KB each, 2 in flight
    uint64_t* cb = &bars[2];
    if (lane == 0) {
      const long long t0 = clock64();
      const uint32_t dst = smem_u32(sm + kOpBytes);
      for (int i = 0; i < ncopy; ++i) {
        const int s = i & 1;
        if (i >= 2) mbar_wait(&cb[s], ((i - 2) >> 1) & 1);
        mbar_arrive_expect_tx(&cb[s], 16384);
        bulk_g2s(dst + s * 32768, gsrc + (static_cast<size_t>(blockIdx.x) * 2 + s) * 16384, 16384,
                 smem_u32(&cb[s]));
      }
      for (int i = ncopy - 2 > 0 ? ncopy - 2 : 0; i < ncopy; ++i)
        mbar_wait(&cb[i & 1], (i >> 1) & 1);
      t_copy = clock64() - t0;
    }
  }
  if (rank == 0 && lane == 0 && warp == 0) out[blockIdx.x * 2 + 0] = t_mma;
  if (lane == 0 && warp == 3) out[blockIdx.x * 2 + 1] = t_copy;
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  if (warp == 1) tmem_dealloc_2sm(tmem, 512);
}

int main() {
  const int maxgrid = 148;
  long long* d;
  cudaMalloc(&d, maxgrid * 2 * sizeof(long long));
  uint8_t* g;
  cudaMalloc(&g, maxgrid * 2 * 16384);
  cudaMemset(g, 0, maxgrid * 2 * 16384);
  const int smem = kOpBytes + kCopyBytes + 1024;
  cudaFuncSetAttribute(bench2, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  printf("cg1 grid issuers   N     n  ncopy   mma_cyc  cyc/mma  copy_cyc  copyB/cyc/SM\n");
  for (int cg1 : {0, 1})
    for (int N : {64, 128, 256})
      for (int issuers : {1, 2})
        for (int ncopy : {0, 1024}) {
          const int grid = 148;
          const int n = 1024;
          for (int rep = 0; rep < 2; ++rep) {
            cudaMemset(d, 0, maxgrid * 2 * sizeof(long long));
            bench2<<<grid, 128, smem>>>(n, issuers, ncopy, g, d, N, cg1);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) {
              printf("error %s\n", cudaGetErrorString(e));
              return 1;
            }
          }
          long long h[2 * maxgrid];
          cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
          const double per = static_cast<double>(h[0]) / n / issuers;
          const double cb = h[1] > 0 ? 16384.0 * ncopy / h[1] : 0.0;
          printf("%3d %4d %7d %3d %5d %6d %9lld  %7.1f %9lld  %12.1f\n", cg1, grid, issuers, N, n, ncopy,
                 h[0], per, h[1], cb);
        }
  return 0;
}
