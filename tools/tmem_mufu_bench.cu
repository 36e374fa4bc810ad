// Microbenchmarks for the attention kernels' elementwise floors on one SM (and the chip):
//   (1) tcgen05.ld 32x32b.x32 throughput from TMEM into registers, W warps (warp w reads lane
//       quarter w % 4), bytes / clock / SM
//   (2) MUFU.EX2 throughput, W warps of independent chains, ex2 / clock / SM
//   (3) FFMA throughput for reference
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tmem_mufu_bench tools/tmem_mufu_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32, 1) tmem_ld_bench(int iters, float* out, long long* cyc) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t base = slot + ((static_cast<uint32_t>(warp & 3) * 32u) << 16);
  const uint32_t colofs = static_cast<uint32_t>((warp >> 2) * 32) % 512;
  float acc = 0.f;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(base + ((colofs + static_cast<uint32_t>(it * 32)) & 511u)));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) acc += __uint_as_float(r[i]);
  }
  long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(slot), "r"(512));
}

// 8 independent ex2 chains per thread
template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32, 1) mufu_bench(int iters, float* out, long long* cyc) {
  float x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = 0.001f * (threadIdx.x + i);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float y;
      asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x[i]));
      x[i] = y * -0.5f;
    }
  }
  long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int W>
void run(int nblocks) {
  float* out;
  long long* cyc;
  cudaMalloc(&out, sizeof(float) * nblocks * W * 32);
  cudaMalloc(&cyc, sizeof(long long) * nblocks);
  const int iters = 4096;
  long long hc = 0;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  tmem_ld_bench<W><<<nblocks, W * 32>>>(16, out, cyc);
  cudaEventRecord(a);
  tmem_ld_bench<W><<<nblocks, W * 32>>>(iters, out, cyc);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  cudaMemcpy(&hc, cyc, sizeof(long long), cudaMemcpyDeviceToHost);
  const double bytes_sm = double(W) * 32 * 32 * 4 * iters;
  printf("tmem_ld x32  warps %2d blocks %3d: %.1f B/clk/SM (clock64), chip %.1f TB/s, %s\n", W, nblocks,
         bytes_sm / double(hc), bytes_sm * nblocks / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  mufu_bench<W><<<nblocks, W * 32>>>(16, out, cyc);
  cudaEventRecord(a);
  mufu_bench<W><<<nblocks, W * 32>>>(iters, out, cyc);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  cudaMemcpy(&hc, cyc, sizeof(long long), cudaMemcpyDeviceToHost);
  const double ex_sm = double(W) * 32 * 8 * iters;
  printf("mufu ex2     warps %2d blocks %3d: %.2f ex2/clk/SM (clock64), chip %.2f Tex2/s\n", W, nblocks,
         ex_sm / double(hc), ex_sm * nblocks / (ms * 1e-3) / 1e12);
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  run<4>(1);
  run<8>(1);
  run<16>(1);
  run<16>(148);
  run<32>(148);
  return 0;
}
