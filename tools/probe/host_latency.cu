// host_latency.cu -- per-call latency of boysfn_eval_host on small batches
// against bare CUDA launch+sync round trips (development aid).
//   nvcc -O2 -gencode arch=compute_100a,code=sm_100a tools/probe/host_latency.cu \
//        -Iinclude -Lpaper_2512_10059_b200/_lib -lboysfn_b200 -o tools/probe/host_latency
#include <chrono>
#include <cstdio>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>
#include "boysfn_b200.h"

__global__ void empty_kernel() {}

template <class F>
double median_us(F f, int reps) {
  std::vector<double> t(reps);
  for (int i = 0; i < reps; ++i) {
    auto a = std::chrono::steady_clock::now();
    f();
    auto b = std::chrono::steady_clock::now();
    t[i] = std::chrono::duration<double, std::micro>(b - a).count();
  }
  std::sort(t.begin(), t.end());
  return t[reps / 2];
}

int main() {
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  unsigned long long* d;
  cudaMalloc(&d, 64);
  empty_kernel<<<1, 32, 0, s>>>();
  cudaStreamSynchronize(s);
  printf("empty launch + sync          %7.2f us\n", median_us([&] { empty_kernel<<<1, 32, 0, s>>>(); cudaStreamSynchronize(s); }, 2000));
  printf("memset + launch + sync       %7.2f us\n", median_us([&] { cudaMemsetAsync(d, 0, 8, s); empty_kernel<<<1, 32, 0, s>>>(); cudaStreamSynchronize(s); }, 2000));
  printf("148 blocks launch + sync     %7.2f us\n", median_us([&] { empty_kernel<<<148 * 8, 128, 0, s>>>(); cudaStreamSynchronize(s); }, 2000));
  boysfn_tables_t t;
  if (boysfn_tables_embedded(&t) != 0) { printf("tables failed\n"); return 1; }
  for (int k : {0, 8, 32}) {
    for (size_t n : {size_t(1), size_t(100), size_t(1000), size_t(3000), size_t(10000), size_t(30000), size_t(100000)}) {
      std::vector<double> x(n, 3.5), out(n * (k + 1));
      size_t fb = 0;
      boysfn_eval_host(t, x.data(), n, k, out.data(), out.size(), BOYSFN_LAYOUT_AOS, n, &fb);
      double us = median_us([&] { boysfn_eval_host(t, x.data(), n, k, out.data(), out.size(), BOYSFN_LAYOUT_AOS, n, &fb); }, n < 1000 ? 2000 : 200);
      printf("boysfn_eval_host k=%2d n=%6zu values=%8zu %8.2f us %6.2f GB/s\n", k, n, n * (k + 1), us, n * (k + 1) * 8e-3 / us);
    }
  }
  return 0;
}
