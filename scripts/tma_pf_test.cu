// Standalone check of a 2-D TMA L2 prefetch of a tableau column (experiment for k_lookahead).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstring>
__global__ void k(const __grid_constant__ CUtensorMap tm, int x, int rows, int mode) {
  if (threadIdx.x == 0) {
    for (int y = 0; y < rows; y += 256) {
      if (mode == 0)
        asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(
                         reinterpret_cast<uint64_t>(&tm)), "r"(x), "r"(y) : "memory");
      else
        asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global [%0, {%1, %2}];" ::"l"(
                         reinterpret_cast<uint64_t>(&tm)), "r"(x), "r"(y) : "memory");
    }
  }
}
int main() {
  using encode_t = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  printf("entry %d\n", (int)cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  encode_t encode = (encode_t)fn;
  const long long ld = 16016; const int rows = 8001;
  double* T; cudaMalloc(&T, sizeof(double) * ld * rows);
  for (int box0 : {2, 4, 16}) for (int x : {0, 1, 7, 16014, 16015}) for (int mode : {0, 1}) {
    CUtensorMap tm;
    const cuuint64_t dims[2] = {(cuuint64_t)ld, (cuuint64_t)rows};
    const cuuint64_t strides[1] = {(cuuint64_t)ld * 8};
    const cuuint32_t box[2] = {(cuuint32_t)box0, 256};
    const cuuint32_t es[2] = {1, 1};
    CUresult r = encode(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, T, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    k<<<1, 32>>>(tm, x, rows, mode);
    cudaError_t e = cudaDeviceSynchronize();
    printf("box0 %d x %d mode %d: encode %d launch %s\n", box0, x, mode, (int)r, cudaGetErrorString(e));
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
