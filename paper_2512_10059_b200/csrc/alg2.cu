// alg2.cu -- C ABI of Algorithm 2 (the paper's fused Boys benchmark,
// PAPER.md:353-390) and its kernel instantiations:
//     z_i = sum_{l=0..k} c_l sum_j F_l(x_i + x_j) y_j.
// Pipeline (one stream, stream-ordered scratch): CUB radix sort of x with the
// original index -> gather (x, e^{-x}, y) in sorted order -> the fused pair
// kernel over (i-block, j-segment) items (alg2_device.cuh) -> sum of the
// segments' partial sums, scattered back to the caller's order.
#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <utility>

#include "alg2_device.cuh"
#include "capi_internal.h"
#include "variant_degrees.h"

namespace boysfn_dev {
namespace {

template <int K, int V>
const void* alg2_entry() {
  constexpr int NA = VariantDegrees<K, V>::NA, MA = VariantDegrees<K, V>::MA;
  constexpr int NB = VariantDegrees<K, V>::NB, MB = VariantDegrees<K, V>::MB;
  return reinterpret_cast<const void*>(&boys_alg2_kernel<K, NA, MA, NB, MB>);
}

template <size_t... Ks>
const void* alg2_lookup(int k, int v, std::index_sequence<Ks...>) {
  static const void* const table[3][sizeof...(Ks)] = {
      {alg2_entry<static_cast<int>(Ks), kVariantEmbedded>()...},
      {alg2_entry<static_cast<int>(Ks), kVariantPadded>()...},
      {alg2_entry<static_cast<int>(Ks), kVariantCompact>()...}};
  return table[v][k];
}

__global__ void iota_kernel(unsigned* idx, size_t n) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
    idx[i] = static_cast<unsigned>(i);
}

__global__ void gather_kernel(const unsigned* perm, const double* xs_sorted, const double* y, double* es,
                              double* ys, size_t n) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
    es[i] = exp(-xs_sorted[i]);
    ys[i] = y[perm[i]];
  }
}

// z[perm[i]] = sum over j-segments of the partial sums, in segment order.
__global__ void scatter_kernel(const unsigned* perm, const double* partial, int nseg, double* z, size_t n) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
    double s = partial[i];
    for (int g = 1; g < nseg; ++g) s += partial[static_cast<size_t>(g) * n + i];
    z[perm[i]] = s;
  }
}

}  // namespace
}  // namespace boysfn_dev

BOYSFN_API int boysfn_alg2_device(boysfn_tables_t t, const double* d_x, const double* d_y, size_t n, int k,
                                  const double* c, double* d_z, void* stream_) {
  using namespace boysfn_dev;
  using boysfn_internal::fail;
  if (t == nullptr || c == nullptr) return fail(BOYSFN_ERR_ARG, "null argument");
  if (k < 0 || k > t->k_max) return fail(BOYSFN_ERR_RANGE, "boys_batch: k out of range for this table set");
  if (k > kKernelKmax) return fail(BOYSFN_ERR_UNSUPPORTED, "device kernels evaluate k <= 32");
  if (!t->degree_ok[k]) return fail(BOYSFN_ERR_UNSUPPORTED, "table degree exceeds the device image (max 23)");
  if (n == 0) return BOYSFN_OK;
  if (n >= (size_t(1) << 32)) return fail(BOYSFN_ERR_UNSUPPORTED, "Algorithm 2 takes n < 2^32");
  if (d_x == nullptr || d_y == nullptr || d_z == nullptr) return fail(BOYSFN_ERR_ARG, "null buffer");
  cudaStream_t s = static_cast<cudaStream_t>(stream_);
  int dev = 0, sms = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const unsigned grid1 = static_cast<unsigned>(std::min<size_t>((n + 255) / 256, size_t(sms) * 8));

  // Work decomposition of the pair kernel: i-blocks x j-segments, about 16
  // items per resident block so the last wave is short; segments are whole
  // shared-memory tiles.
  const void* pair_fn = alg2_lookup(k, t->variant[k], std::make_index_sequence<kKernelKmax + 1>{});
  int bps = 0;
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, pair_fn, kAlg2Threads, 0));
  const size_t slots = size_t(sms) * std::max(bps, 1);
  const size_t nib = (n + kAlg2Threads - 1) / kAlg2Threads;
  const size_t tiles = (n + kAlg2TileJ - 1) / kAlg2TileJ;
  const int nseg = static_cast<int>(std::min<size_t>({32, tiles, std::max<size_t>(1, (16 * slots + nib - 1) / nib)}));
  const size_t seg_len = (tiles + nseg - 1) / nseg * kAlg2TileJ;

  // scratch: sorted x, e, y (doubles), partial sums (nseg x n), index in/out
  // (u32), item counter, CUB temp
  size_t cub_bytes = 0;
  CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, cub_bytes, static_cast<const double*>(nullptr),
                                           static_cast<double*>(nullptr), static_cast<const unsigned*>(nullptr),
                                           static_cast<unsigned*>(nullptr), n, 0, 64, s));
  const size_t dbl = ((n * sizeof(double) + 255) / 256) * 256, u32 = ((n * sizeof(unsigned) + 255) / 256) * 256;
  const size_t part = ((size_t(nseg) * n * sizeof(double) + 255) / 256) * 256;
  char* scratch = nullptr;
  CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&scratch), 3 * dbl + part + 2 * u32 + 256 + cub_bytes, s));
  double* xs = reinterpret_cast<double*>(scratch);
  double* es = reinterpret_cast<double*>(scratch + dbl);
  double* ys = reinterpret_cast<double*>(scratch + 2 * dbl);
  double* partial = reinterpret_cast<double*>(scratch + 3 * dbl);
  unsigned* idx = reinterpret_cast<unsigned*>(scratch + 3 * dbl + part);
  unsigned* perm = reinterpret_cast<unsigned*>(scratch + 3 * dbl + part + u32);
  unsigned long long* counter = reinterpret_cast<unsigned long long*>(scratch + 3 * dbl + part + 2 * u32);
  void* cub_tmp = scratch + 3 * dbl + part + 2 * u32 + 256;

  int status = BOYSFN_OK;
  iota_kernel<<<grid1, 256, 0, s>>>(idx, n);
  cudaError_t e = cub::DeviceRadixSort::SortPairs(cub_tmp, cub_bytes, d_x, xs, idx, perm, n, 0, 64, s);
  if (e == cudaSuccess) {
    gather_kernel<<<grid1, 256, 0, s>>>(perm, xs, d_y, es, ys, n);
    Alg2Coef coef{};
    for (int l = 0; l <= k; ++l) coef.c[l] = c[l];
    EvalParams p = t->params[k];
    size_t seg = seg_len;
    int ns = nseg;
    void* args[] = {&p, &coef, &xs, &es, &ys, &n, &ns, &seg, &counter, &partial};
    const unsigned grid2 = static_cast<unsigned>(std::min<size_t>(slots, nib * nseg));
    e = cudaMemsetAsync(counter, 0, sizeof(unsigned long long), s);
    if (e == cudaSuccess) e = cudaLaunchKernel(pair_fn, dim3(grid2), dim3(kAlg2Threads), args, 0, s);
    if (e == cudaSuccess) scatter_kernel<<<grid1, 256, 0, s>>>(perm, partial, nseg, d_z, n);
  }
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) status = boysfn_internal::cuda_fail(e, "boysfn_alg2_device");
  cudaFreeAsync(scratch, s);
  for (int i = 0; i < 4; ++i) boysfn_internal::count_launch();  // iota, gather, pairs, scatter (CUB's sort not counted)
  return status;
}
