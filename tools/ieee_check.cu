// tools/ieee_check.cu -- div_rn_fast / sqrt_rn_fast (boys_device.cuh) against
// the compiled __ddiv_rn / __dsqrt_rn, bit for bit, over in_bc_fast_range:
// 2^31 log-uniform x in [2^-971, 2^1022), 2^31 uniform x in [0, 200], the ulp
// neighbourhoods of 2^24 perfect squares, and the range ends.  Checks 0.5/x,
// sqrt(x) and (sqrt(pi)/2)/sqrt(x).  Prints the mismatch count (expected 0).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -diag-suppress 1886 \
//        -Ipaper_2512_10059_b200/csrc -o build/ieee_check tools/ieee_check.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "boys_device.cuh"

__device__ unsigned long long g_checked = 0, g_bad = 0;
__device__ double g_first = 0;

__device__ void check(double x) {
  if (!boysfn_dev::in_bc_fast_range(x)) return;
  const double c = boysfn_dev::kExpC[13];
  const double s = boysfn_dev::sqrt_rn_fast(x);
  const bool ok = __double_as_longlong(boysfn_dev::div_rn_fast(0.5, x)) == __double_as_longlong(__ddiv_rn(0.5, x)) &&
                  __double_as_longlong(s) == __double_as_longlong(__dsqrt_rn(x)) &&
                  __double_as_longlong(boysfn_dev::div_rn_fast(c, s)) ==
                      __double_as_longlong(__ddiv_rn(c, __dsqrt_rn(x)));
  if (!ok && atomicAdd(&g_bad, 1ull) == 0) g_first = x;
}

__device__ unsigned long long mix(unsigned long long z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void sweep(unsigned long long n, unsigned long long seed, int mode) {
  unsigned long long cnt = 0;
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const double u = (mix(seed + (i + 1) * 0x9E3779B97F4A7C15ull) >> 11) * 0x1.0p-53;
    double x;
    if (mode == 0) x = exp2(-971.0 + 1993.0 * u);  // log-uniform over the fast range
    else if (mode == 1) x = 200.0 * u;
    else {  // perfect squares m^2 and their +-3 ulp neighbours
      const double m = static_cast<double>((i >> 3) + 1);
      x = m * m;
      for (int d = static_cast<int>(i & 7) - 3; d != 0; d += d < 0 ? 1 : -1) x = nextafter(x, d < 0 ? 0.0 : 1e308);
    }
    check(x);
    ++cnt;
  }
  atomicAdd(&g_checked, cnt);
}

__global__ void ends() {
  const double v[] = {0x1p-971, 0x1.0000000000001p-971, 0x1.fffffffffffffp1021, 0x1p1021, 11.899848152108484,
                      28.98933773882074, 28.989337738820744, 1.0, 4.0, 2.0, 3.0, 0x1.fffffffffffffp-1};
  for (double x : v) check(x);
}

int main() {
  sweep<<<148 * 8, 256>>>(1ull << 31, 11, 0);
  sweep<<<148 * 8, 256>>>(1ull << 31, 12, 1);
  sweep<<<148 * 8, 256>>>(1ull << 27, 13, 2);
  ends<<<1, 1>>>();
  const cudaError_t e = cudaDeviceSynchronize();
  unsigned long long checked = 0, bad = 0;
  double first = 0;
  cudaMemcpyFromSymbol(&checked, g_checked, sizeof checked);
  cudaMemcpyFromSymbol(&bad, g_bad, sizeof bad);
  cudaMemcpyFromSymbol(&first, g_first, sizeof first);
  std::printf("{\"ieee_check\": \"%s\", \"checked\": %llu, \"mismatches\": %llu, \"first_x\": %.17g}\n",
              cudaGetErrorString(e), checked, bad, first);
  return (e == cudaSuccess && bad == 0) ? 0 : 1;
}
