// Probe: smem layout of a SWIZZLE_128B TMA box whose inner dimension (40 bf16 = 80 B) is
// narrower than the 128-byte swizzle span. Prints, per smem row of 128 B, which source
// columns landed in which 16-byte chunk (or '-' for untouched zero bytes).
//   nvcc -gencode arch=compute_100a,code=sm_100a -I paper_2306_09342_b200/csrc \
//        tools/probe/tma_narrow_box.cu -o tools/probe/tma_narrow_box -lcuda
#include <cuda.h>
#include <cstdio>

#include "ptx.cuh"
using namespace rp;
typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                             const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                             const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__global__ void k(const __grid_constant__ CUtensorMap m, uint16_t* out) {
  __shared__ __align__(1024) uint16_t buf[16 * 64];
  __shared__ __align__(8) uint64_t bar;
  for (int i = threadIdx.x; i < 16 * 64; i += blockDim.x) buf[i] = 0xffff;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  fence_proxy_async_smem();
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(&bar, 16 * 40 * 2);
    tma_load_2d(buf, &m, &bar, 64, 0);
  }
  mbar_wait(&bar, 0);
  for (int i = threadIdx.x; i < 16 * 64; i += blockDim.x) out[i] = buf[i];
}

int main() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  EncodeFn fn = reinterpret_cast<EncodeFn>(p);
  const int R = 16, C = 312;  // 3 heads x 104
  uint16_t h[R * C];
  for (int r = 0; r < R; ++r)
    for (int c = 0; c < C; ++c) h[r * C + c] = static_cast<uint16_t>(r * 1000 + c);
  uint16_t *d, *o;
  cudaMalloc(&d, sizeof(h));
  cudaMalloc(&o, 16 * 64 * 2);
  cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
  CUtensorMap m;
  cuuint64_t dims[2] = {C, R};
  cuuint64_t strides[1] = {C * 2};
  cuuint32_t box[2] = {40, 16}, es[2] = {1, 1};
  CUresult r = fn(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  k<<<1, 128>>>(m, o);
  printf("kernel %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  uint16_t ho[16 * 64];
  cudaMemcpy(ho, o, sizeof(ho), cudaMemcpyDeviceToHost);
  for (int row = 0; row < 16; ++row) {
    printf("smem row %2d:", row);
    for (int ch = 0; ch < 8; ++ch) {
      const uint16_t v = ho[row * 64 + ch * 8];
      if (v == 0xffff) printf("    -    ");
      else printf(" r%2d c%3d", v / 1000, v % 1000);
    }
    printf("\n");
  }
  return 0;
}
