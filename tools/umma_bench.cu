// Microbenchmark: tcgen05.mma (kind::f16, cta_group::1, M = 128, K = 16) issue-to-completion
// cost per instruction as a function of N, operand source (SS: A and B in smem; TS: A in
// TMEM) and the number of independent accumulator chains. One CTA on one SM; cycles from the
// first issue to the commit's mbarrier completion, divided by the number of MMAs.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2306_09342_b200/csrc \
//        tools/umma_bench.cu -o tools/umma_bench && ./tools/umma_bench
#include <cstdio>

#include "ptx.cuh"

using namespace rp;

__device__ __forceinline__ void umma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc,
                                        uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}

__global__ void bench(int M, int N, int ts, int chains, int n, int variant, long long* out, int issuers) {
  extern __shared__ uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) &
                                           ~static_cast<uintptr_t>(1023));
  __shared__ __align__(8) uint64_t bars[4];
  __shared__ uint32_t slot;
  const uint32_t warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) mbar_init(&bars[i], 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(&slot, 512);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  // variant bit 0: whole warp 0 runs the loop, one elected lane issues (warp-uniform
  // control flow); bit 1: 8 MMAs per iteration with compile-time-constant operand offsets
  if ((variant & 4) && static_cast<int>(warp) < issuers) {
    // warp-convergent issue: all 32 lanes run the loop, elect.sync picks the issuing lane
    // (the CUTLASS / DeepGEMM pattern), descriptors precomputed outside the loop
    uint64_t& bar = bars[warp];
    const uint32_t idesc = make_idesc_bf16(static_cast<uint32_t>(M), static_cast<uint32_t>(N), false, false);
    const uint32_t a = smem_u32(sm), b = smem_u32(sm + 32768);
    uint64_t ad[4], bd[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      ad[j] = make_sdesc_sw128(a + j * 32, 16, 1024);
      bd[j] = make_sdesc_sw128(b + j * 32, 16, 1024);
    }
    for (int rep = 0; rep < 2; ++rep) {
      __syncwarp();
      const long long t0 = clock64();
      for (int i = 0; i < n; i += 8) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint32_t d = tmem + static_cast<uint32_t>((j % chains) * N);
          if (variant & 8) {  // converged warp, predicate from a precomputed leader flag
            const uint32_t leader = (threadIdx.x & 31) == 0;
            asm volatile(
                "{\n\t.reg .pred e;\n\tsetp.ne.b32 e, %4, 0;\n\t"
                "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;\n\t}" ::"r"(d),
                "l"(ad[j & 3]), "l"(bd[j & 3]), "r"(idesc), "r"(leader)
                : "memory");
          } else if (variant & 16) {  // elect once, 1 divergent lane issues the block
            if (j == 0 && (threadIdx.x & 31) == 0) {
#pragma unroll
              for (int jj = 0; jj < 8; ++jj)
                asm volatile("tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;" ::"r"(
                                 tmem + static_cast<uint32_t>((jj % chains) * N)),
                             "l"(ad[jj & 3]), "l"(bd[jj & 3]), "r"(idesc)
                             : "memory");
            }
          } else if (ts)
            asm volatile(
                "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, 1;\n\t}" ::"r"(d),
                "r"(tmem + 256u + static_cast<uint32_t>((j & 3) * 8)), "l"(bd[j & 3]), "r"(idesc)
                : "memory");
          else
            asm volatile(
                "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;\n\t}" ::"r"(d),
                "l"(ad[j & 3]), "l"(bd[j & 3]), "r"(idesc)
                : "memory");
        }
      }
      if ((threadIdx.x & 31) == 0) umma_commit(&bar);
      __syncwarp();
      const long long t1 = clock64();
      mbar_wait(&bar, rep & 1);
      const long long t2 = clock64();
      if (rep == 1 && (threadIdx.x & 31) == 0 && warp == 0) {
        out[0] = t1 - t0;
        out[1] = t2 - t0;
      }
    }
  } else if (static_cast<int>(warp) < issuers && (threadIdx.x & 31) == 0) {
    uint64_t& bar = bars[warp];
    const uint32_t idesc = make_idesc_bf16(static_cast<uint32_t>(M), static_cast<uint32_t>(N), false, false);
    const uint32_t a = smem_u32(sm), b = smem_u32(sm + 32768);
    const bool issuer = (threadIdx.x & 31) == 0;
    for (int rep = 0; rep < 2; ++rep) {  // rep 0 warms up
      const long long t0 = clock64();
      if (variant & 2) {
        for (int i = 0; i < n; i += 8) {
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const uint32_t d = tmem + static_cast<uint32_t>(warp * 64 + (j % chains) * N);
            const uint64_t bd = make_sdesc_sw128(b + (j & 3) * 32, 16, 1024);
            if (issuer) {
              if (ts)
                umma_ts(d, tmem + 256u + static_cast<uint32_t>((j & 3) * 8), bd, idesc, 1u);
              else
                umma_bf16(d, make_sdesc_sw128(a + (j & 3) * 32, 16, 1024), bd, idesc, 1u);
            }
            if (variant & 1) __syncwarp();
          }
        }
      } else {
        for (int i = 0; i < n; ++i) {
          const int c = i % chains;
          const uint32_t d = tmem + static_cast<uint32_t>(c * N);
          const uint64_t bd = make_sdesc_sw128(b + (i & 3) * 32, 16, 1024);
          if (issuer) {
            if (ts)
              umma_ts(d, tmem + 256u + static_cast<uint32_t>((i & 3) * 8), bd, idesc, i >= chains);
            else
              umma_bf16(d, make_sdesc_sw128(a + (i & 3) * 32, 16, 1024), bd, idesc, i >= chains);
          }
          if (variant & 1) __syncwarp();
        }
      }
      if (issuer) umma_commit(&bar);
      const long long t1 = clock64();
      mbar_wait(&bar, rep & 1);
      const long long t2 = clock64();
      if (rep == 1 && issuer && warp == 0) {
        out[0] = t1 - t0;
        out[1] = t2 - t0;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc(tmem, 512);
}


// Two (or four) warps take turns issuing MMAs into ONE accumulator: warp w issues MMA i when
// i % nw == w, after the previous issuer's hand-off (named barrier); the accumulation order
// is the issue order, so the result is deterministic.
__global__ void bench_alt(int N, int n, int nw, long long* out) {
  extern __shared__ uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) &
                                           ~static_cast<uintptr_t>(1023));
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t slot;
  __shared__ volatile int turn;
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
    turn = 0;
  }
  if (warp == 0) tmem_alloc(&slot, 512);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t idesc = make_idesc_bf16(128u, static_cast<uint32_t>(N), false, false);
  const uint32_t a = smem_u32(sm), b = smem_u32(sm + 32768);
  uint64_t ad[4], bd[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    ad[j] = make_sdesc_sw128(a + j * 32, 16, 1024);
    bd[j] = make_sdesc_sw128(b + j * 32, 16, 1024);
  }
  long long t0 = 0;
  if (static_cast<int>(warp) < nw) {
    __syncwarp();
    t0 = clock64();
    for (int i = static_cast<int>(warp); i < n; i += nw) {
      if (lane == 0) {
        while (turn != i) {
        }
        asm volatile("tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;" ::"r"(tmem),
                     "l"(ad[i & 3]), "l"(bd[i & 3]), "r"(idesc)
                     : "memory");
        turn = i + 1;
      }
      __syncwarp();
    }
    if (lane == 0 && static_cast<int>(warp) == (n - 1) % nw) umma_commit(&bar);
  }
  if (warp == 0) {
    mbar_wait(&bar, 0);
    if (lane == 0) out[0] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc(tmem, 512);
}
int main() {
  long long* d;
  cudaMalloc(&d, 16);
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 1024);
  // cycles per MMA as a function of the number of MMAs n: a fixed start-up / completion
  // cost shows up as cyc/mma falling with n; the slope between two n is the true rate
  printf("variant issuers  N chains     n  issue_cyc  total_cyc  cyc/mma\n");
  for (int variant : {2, 12})
    for (int N : {64, 128, 256})
      for (int issuers : {1, 2, 4})
        for (int n : {64, 256, 1024, 4096}) {
          if (issuers * N > 512) continue;
          bench<<<1, 128, 65536 + 1024>>>(128, N, 0, 1, n, variant, d, issuers);
          long long h[2];
          cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
          cudaError_t e = cudaGetLastError();
          if (e != cudaSuccess) {
            printf("error %s\n", cudaGetErrorString(e));
            return 1;
          }
          printf("%7d %7d %3d %6d %5d  %9lld  %9lld  %7.1f\n", variant, issuers, N, 1, n, h[0], h[1],
                 static_cast<double>(h[1]) / n);
        }
  return 0;
}
