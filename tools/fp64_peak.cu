// tools/fp64_peak.cu -- DFMA throughput microbenchmark (the FP64 roofline
// denominator; MEASURED_PEAKS.json has no FP64 figure).  8 independent FMA
// chains per thread, 8 resident 256-thread blocks per SM, CUDA-event timed.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/fp64_peak tools/fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_loop(double* out, int iters, double a, double b) {
  double v[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) v[j] = threadIdx.x * 1e-3 + j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = fma(v[j], a, b);
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += v[j];
  if (s == 12345.678) out[0] = s;  // keep the chains live
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 8);
  const int iters = 1 << 16, threads = 256, blocks = sms * 8;
  dfma_loop<<<blocks, threads>>>(out, 1024, 0.999999, 1e-9);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    dfma_loop<<<blocks, threads>>>(out, iters, 0.999999, 1e-9);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  const double fmas = double(blocks) * threads * iters * 8;
  std::printf("{\"fp64_tflops\": %.2f, \"dfma_per_s\": %.4e, \"sms\": %d, \"ms\": %.3f}\n", 2 * fmas / (best * 1e-3) / 1e12,
              fmas / (best * 1e-3), sms, best);
  return 0;
}
