// Probe: which parameters does cuTensorMapEncodeTiled accept for a rank-1 fp32 map?
//   nvcc -gencode arch=compute_100a,code=sm_100a tools/probe/tmap1d.cu -o tools/probe/tmap1d
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                             const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                             const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  EncodeFn fn = reinterpret_cast<EncodeFn>(p);
  float* d;
  cudaMalloc(&d, 401408 * 4);
  CUtensorMap m;
  cuuint64_t dims[2] = {401408, 1};
  cuuint64_t strides[1] = {401408 * 4};
  cuuint32_t es[2] = {1, 1};
  for (int rank : {1, 2})
    for (cuuint32_t box0 : {52u, 64u, 56u})
      for (int prom : {0, 1}) {
        cuuint32_t box[2] = {box0, 1};
        CUresult r = fn(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, rank, d, dims, rank == 1 ? nullptr : strides,
                        box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        prom ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_NONE,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        printf("rank %d box %u prom %d -> %d\n", rank, box0, prom, (int)r);
      }
  return 0;
}
