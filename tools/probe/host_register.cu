// host_register.cu -- cudaHostRegister / Unregister cost on fresh pageable
// memory, and D2H into it (development aid): could the pageable host path DMA
// straight into the caller's buffer by page-locking it chunk by chunk?
//   nvcc -O2 -gencode arch=compute_100a,code=sm_100a tools/probe/host_register.cu -o tools/probe/host_register
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>

static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }

int main() {
  const size_t sizes[] = {size_t(64) << 20, size_t(256) << 20, size_t(1) << 30};
  void* dbuf;
  cudaMalloc(&dbuf, size_t(1) << 30);
  cudaMemset(dbuf, 1, size_t(1) << 30);
  for (size_t bytes : sizes) {
    for (int rep = 0; rep < 2; ++rep) {
      char* h = static_cast<char*>(std::malloc(bytes));
      std::memset(h, 0, bytes);  // first touch
      double t0 = now();
      cudaError_t e = cudaHostRegister(h, bytes, cudaHostRegisterDefault);
      double t1 = now();
      cudaMemcpy(h, dbuf, bytes, cudaMemcpyDeviceToHost);
      double t2 = now();
      cudaHostUnregister(h);
      double t3 = now();
      cudaMemcpy(h, dbuf, bytes, cudaMemcpyDeviceToHost);  // pageable (driver-staged)
      double t4 = now();
      std::printf("%5zu MB: register %7.2f ms (%6.1f GB/s) D2H registered %6.1f GB/s  unregister %6.2f ms (%6.1f GB/s)  D2H pageable %5.1f GB/s  rc=%d\n",
                  bytes >> 20, (t1 - t0) * 1e3, bytes / (t1 - t0) / 1e9, bytes / (t2 - t1) / 1e9, (t3 - t2) * 1e3,
                  bytes / (t3 - t2) / 1e9, bytes / (t4 - t3) / 1e9, static_cast<int>(e));
      std::free(h);
    }
  }
  return 0;
}
