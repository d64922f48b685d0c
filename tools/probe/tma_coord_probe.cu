// Probe: does a TMA 2D tensor store accept a box whose first element is not
// 16-B aligned in global memory (start coordinate odd, fp64), and boxes
// clipped at small dims?  Each case runs in its own process (an illegal
// instruction poisons the context).  Development aid for capi.cu make_soa_tmaps.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>

__global__ void store_kernel(const __grid_constant__ CUtensorMap m, int c0, int c1) {
  extern __shared__ __align__(1024) double s[];
  for (int i = threadIdx.x; i < 256 * 4; i += blockDim.x) s[i] = 1000.0 + i;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                     reinterpret_cast<uint64_t>(&m)),
                 "r"(static_cast<uint32_t>(__cvta_generic_to_shared(s))), "r"(c0), "r"(c1)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  // args: base_off(doubles) dim0 rows stride_doubles c0
  const int base_off = atoi(argv[1]);
  const unsigned long long dim0 = strtoull(argv[2], 0, 10);
  const int rows = atoi(argv[3]);
  const unsigned long long stride = strtoull(argv[4], 0, 10);
  const int c0 = atoi(argv[5]);
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  EncodeTiledFn enc = reinterpret_cast<EncodeTiledFn>(p);
  double* d = nullptr;
  cudaMalloc(&d, 1 << 24);
  cudaMemset(d, 0, 1 << 24);
  CUtensorMap m;
  memset(&m, 0, sizeof m);
  const cuuint64_t dims[2] = {dim0, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {stride * 8};
  const cuuint32_t box[2] = {256, (cuuint32_t)rows};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, d + base_off, dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode=%d ", (int)r);
  cudaFuncSetAttribute(store_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 256 * 4 * 8);
  store_kernel<<<1, 128, 256 * 4 * 8>>>(m, c0, 0);
  cudaError_t e = cudaDeviceSynchronize();
  printf("launch=%s ", cudaGetErrorString(e));
  if (e == cudaSuccess) {
    double h[8];
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    printf("d[0..7]=");
    for (int i = 0; i < 8; ++i) printf("%g ", h[i]);
  }
  printf("\n");
  return 0;
}
