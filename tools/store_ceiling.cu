// tools/store_ceiling.cu -- write-bandwidth ceilings for the Boys output
// pattern (development aid, no Boys arithmetic).  configs[1] traffic: read
// 8 B of x, write 8*(k+1) B of F per x, k = 32, n = 1e8 (26.4 GB written).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/store_ceiling tools/store_ceiling.cu
// Each variant is CUDA-event timed, best of 5 after one warm-up.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdint>
#include <cstring>

#define CK(x)                                                                       \
  do {                                                                              \
    cudaError_t e_ = (x);                                                           \
    if (e_ != cudaSuccess) {                                                        \
      std::printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));        \
      return 1;                                                                     \
    }                                                                               \
  } while (0)

constexpr int R = 33;

// Pure write, 16 B per thread store, grid-stride.
__global__ void fill_v2(double2* out, size_t n2) {
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n2; i += stride)
    __stcs(out + i, make_double2(1.0, 2.0));
}

// Pure write, 32 B per thread store (256-bit st.global, sm_100).
__global__ void fill_v4(double* out, size_t n4) {
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += stride) {
    double* p = out + 4 * i;
    asm volatile("st.global.cs.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(1.0), "d"(2.0), "d"(3.0),
                 "d"(4.0)
                 : "memory");
  }
}

// SoA pattern through LSU: a warp per 32-x tile, R rows of 256 B.
__global__ void soa_lsu(const double* xs, size_t n, double* out) {
  const size_t ntiles = n / 32;
  const size_t warps = size_t(gridDim.x) * (blockDim.x / 32);
  const int lane = threadIdx.x & 31;
  for (size_t t = size_t(blockIdx.x) * (blockDim.x / 32) + threadIdx.x / 32; t < ntiles; t += warps) {
    const size_t i = t * 32 + lane;
    const double x = __ldcs(xs + i);
#pragma unroll
    for (int l = 0; l < R; ++l) __stcs(out + size_t(l) * n + i, x * (l + 1));
  }
}

// AoS pattern through LSU: each warp writes its tile's 32*R contiguous doubles.
__global__ void aos_lsu(const double* xs, size_t n, double* out) {
  const size_t ntiles = n / 32;
  const size_t warps = size_t(gridDim.x) * (blockDim.x / 32);
  const int lane = threadIdx.x & 31;
  for (size_t t = size_t(blockIdx.x) * (blockDim.x / 32) + threadIdx.x / 32; t < ntiles; t += warps) {
    const double x = __ldcs(xs + t * 32 + lane);
    double* base = out + t * 32 * R;
#pragma unroll
    for (int l = 0; l < R; ++l) __stcs(base + l * 32 + lane, x * (l + 1));
  }
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// SoA pattern through the TMA engine: 128-x block tile staged in smem, one 2D
// tensor store per tile; NB stage buffers so the next tile's smem writes do not
// wait for the previous store's reads.
template <int NB>
__global__ void __launch_bounds__(128) soa_tma(const __grid_constant__ CUtensorMap tm, const double* xs,
                                               size_t n) {
  extern __shared__ __align__(128) double stage[];
  const size_t ntiles = n / 128;
  int buf = 0;
  for (size_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    double* s = stage + buf * 128 * R;
    if (threadIdx.x == 0)
      asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(NB - 1) : "memory");
    __syncthreads();
    const double x = __ldcs(xs + t * 128 + threadIdx.x);
#pragma unroll
    for (int l = 0; l < R; ++l) s[l * 128 + threadIdx.x] = x * (l + 1);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      asm volatile(
          "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(&tm),
          "r"(int(t * 128)), "r"(0), "r"(smem_u32(s))
          : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    buf = (buf + 1) % NB;
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// Pure write through the TMA engine: 1D bulk stores of `chunk` bytes from an
// uninitialised smem buffer (content irrelevant), NB in flight per block.
__global__ void bulk_fill(char* out, size_t bytes, uint32_t chunk, int nb) {
  extern __shared__ __align__(128) char sb[];
  if (threadIdx.x != 0) return;
  const size_t nch = bytes / chunk;
  int inflight = 0;
  for (size_t c = blockIdx.x; c < nch; c += gridDim.x) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(out + c * chunk),
                 "r"(smem_u32(sb)), "r"(chunk)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    if (++inflight >= nb) {
      asm volatile("cp.async.bulk.wait_group.read 4;" ::: "memory");
      inflight = 4;
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <class F>
float best_ms(F launch) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  launch();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return best;
}

int main() {
  const size_t n = 100000000;
  const double wbytes = double(n) * R * 8, rbytes = double(n) * 8;
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  double *xs, *out;
  CK(cudaMalloc(&xs, n * 8));
  CK(cudaMalloc(&out, n * R * 8));
  CK(cudaMemset(xs, 0, n * 8));
  auto report = [&](const char* name, float ms, double bytes) {
    std::printf("{\"variant\": \"%s\", \"ms\": %.4f, \"gbs\": %.1f}\n", name, ms, bytes / (ms * 1e-3) / 1e9);
    std::fflush(stdout);
  };
  for (int bps : {4, 8, 16}) {
    char nm[64];
    std::snprintf(nm, sizeof nm, "fill_v2 bps=%d", bps);
    report(nm, best_ms([&] { fill_v2<<<sms * bps, 256>>>(reinterpret_cast<double2*>(out), n * R / 2); }), wbytes);
    std::snprintf(nm, sizeof nm, "fill_v4 bps=%d", bps);
    report(nm, best_ms([&] { fill_v4<<<sms * bps, 256>>>(out, n * R / 4); }), wbytes);
    std::snprintf(nm, sizeof nm, "soa_lsu bps=%d", bps);
    report(nm, best_ms([&] { soa_lsu<<<sms * bps, 256>>>(xs, n, out); }), wbytes + rbytes);
    std::snprintf(nm, sizeof nm, "aos_lsu bps=%d", bps);
    report(nm, best_ms([&] { aos_lsu<<<sms * bps, 256>>>(xs, n, out); }), wbytes + rbytes);
  }
  CK(cudaGetLastError());
  for (uint32_t chunk : {4096u, 16384u, 33792u}) {
    for (int bps : {1, 2, 4}) {
      CK(cudaFuncSetAttribute(bulk_fill, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
      char nm[64];
      std::snprintf(nm, sizeof nm, "bulk_fill chunk=%u bps=%d", chunk, bps);
      const size_t bytes = size_t(wbytes) / chunk * chunk;
      report(nm, best_ms([&] { bulk_fill<<<sms * bps, 32, chunk>>>(reinterpret_cast<char*>(out), bytes, chunk, 8); }),
             double(bytes));
    }
  }
  CK(cudaGetLastError());
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
  CUtensorMap tm;
  const cuuint64_t dims[2] = {n, R};
  const cuuint64_t strides[1] = {n * 8};
  const cuuint32_t box[2] = {128, R};
  const cuuint32_t es[2] = {1, 1};
  if (reinterpret_cast<EncodeTiledFn>(p)(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, out, dims, strides, box, es,
                                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                         CU_TENSOR_MAP_L2_PROMOTION_NONE,
                                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
    std::printf("encode failed\n");
    return 1;
  }
  const int smem1 = 128 * R * 8;
  CK(cudaFuncSetAttribute(soa_tma<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem1));
  CK(cudaFuncSetAttribute(soa_tma<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * smem1));
  for (int bps : {2, 4, 6}) {
    char nm[64];
    std::snprintf(nm, sizeof nm, "soa_tma nb=1 bps=%d", bps);
    report(nm, best_ms([&] { soa_tma<1><<<sms * bps, 128, smem1>>>(tm, xs, n); }), wbytes + rbytes);
    if (bps <= 3 || 2 * smem1 * bps <= 220 * 1024) {
      std::snprintf(nm, sizeof nm, "soa_tma nb=2 bps=%d", bps);
      report(nm, best_ms([&] { soa_tma<2><<<sms * bps, 128, 2 * smem1>>>(tm, xs, n); }), wbytes + rbytes);
    }
  }
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  return 0;
}
