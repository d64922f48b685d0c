// verify.cu -- verify_tables on the GPU (reference: verify.cpp:12-63,
// verify.hpp:12-35): sample each region with
// the reference's generator (std::mt19937_64(seed), u = (rng() >> 11) * 2^-53,
// verify.cpp:23-30), evaluate the extended-precision oracle for F_0..F_kmax
// and every order k = 0..k_max of the evaluator under test, and report the
// per-(k, region) maximum absolute error with the reference's worst-case
// bookkeeping (strict '>' in loop order region, sample, k, l).
//
// The oracle runs on the device in double-double arithmetic (~106-bit
// significand): the reference's series (reference.cpp:10-23) with the same
// truncation length reference_terms_for(0, x) (reference.cpp:46-54, verify.cpp:35,
// computed on the host exactly as there), e^{-x} by range reduction and a
// Taylor series, the downward recurrence (reference.cpp:25-35) in double-double,
// and one rounding to double (verify.cpp:38).  The reference uses MPFR at
// 62 digits; after rounding to double the two agree except at ties (tested
// against the binary128 oracle, tests/test_gpu_verify.py).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <random>
#include <stdexcept>
#include <vector>

#include "boys_launch.h"
#include "capi_internal.h"
#include "dd_math.cuh"

namespace {

using namespace boysfn_dd;

// F_0..F_kmax at each sample, rounded to double: oracle[i*(kmax+1) + l].
__global__ void dd_oracle_kernel(const double* __restrict__ xs, const int* __restrict__ terms, size_t n, int kmax,
                                 double* __restrict__ oracle) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
    const double x = xs[i];
    const int L = terms[i];
    // series at order kmax (reference.cpp:10-23)
    dd term = dd_div_d(dd{1.0, 0.0}, kmax + 0.5);
    dd sum = term;
    for (int l = 1; l <= L; ++l) {
      term = dd_div_d(dd_mul_d(term, x), kmax + l + 0.5);
      sum = dd_add(sum, term);
    }
    const dd e = dd_exp_neg(x);
    dd f = dd_mul(dd_mul_d(e, 0.5), sum);
    double* row = oracle + i * static_cast<size_t>(kmax + 1);
    row[kmax] = f.hi + f.lo;
    // downward recurrence in extended precision (reference.cpp:30-34)
    for (int l = kmax - 1; l >= 0; --l) {
      f = dd_div_d(dd_add(dd_mul_d(f, 2.0 * x), e), 2.0 * l + 1.0);
      row[l] = f.hi + f.lo;
    }
  }
}

// Max |F_l - oracle_l| over l <= k per sample, folded into per-region maxima
// (positive doubles compare like their uint64 bit patterns).
__global__ void compare_kernel(const double* __restrict__ got, const double* __restrict__ oracle, size_t n,
                               int spr, int k, int kmax, unsigned long long* __restrict__ region_max) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
    double m = 0.0;
    for (int l = 0; l <= k; ++l)
      m = fmax(m, fabs(got[i * (k + 1) + l] - oracle[i * static_cast<size_t>(kmax + 1) + l]));
    atomicMax(region_max + i / spr, static_cast<unsigned long long>(__double_as_longlong(m)));
  }
}

// First (sample, l) in loop order whose error equals the global maximum.
__global__ void locate_kernel(const double* __restrict__ got, const double* __restrict__ oracle, size_t n, int k,
                              int kmax, double target, unsigned long long* __restrict__ first) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
    for (int l = 0; l <= k; ++l)
      if (fabs(got[i * (k + 1) + l] - oracle[i * static_cast<size_t>(kmax + 1) + l]) == target) {
        atomicMin(first, static_cast<unsigned long long>(i));
        break;
      }
}

// reference_terms_for (reference.cpp:46-54); -1 where the reference throws.
int terms_for(int k, double x, double rel_target) {
  if (x <= 0) return 150;
  const double log_target = std::log(rel_target);
  for (int L = 150; L <= 20000; L += 25) {
    const double s = k + L + 1.5;
    if (s * std::log(x) - std::lgamma(s) <= log_target) return L;
  }
  return -1;
}

}  // namespace

BOYSFN_API int boysfn_verify_tables(boysfn_tables_t t, int samples_per_region, double xmax, uint64_t seed,
                                    boysfn_verify_report* rep) {
  using boysfn_internal::fail;
  if (t == nullptr || rep == nullptr || rep->per_k == nullptr) return fail(BOYSFN_ERR_ARG, "null argument");
  // verify.cpp:14-18 (validate_tables, recorded when the handle was built)
  if (t->valid_status != BOYSFN_OK) return fail(t->valid_status, t->valid_msg);
  if (samples_per_region < 1)
    return fail(BOYSFN_ERR_INVALID, "verify_tables: need at least one sample per region");
  if (xmax <= t->x1) return fail(BOYSFN_ERR_INVALID, "verify_tables: xmax must exceed x1");
  const int kmax = t->k_max;
  const size_t spr = static_cast<size_t>(samples_per_region), n = 3 * spr;

  // samples exactly as verify.cpp:23-33 draws them, with their series lengths
  std::vector<double> xs(n);
  std::vector<int> terms(n);
  {
    std::mt19937_64 rng(seed);
    const double lo[3] = {0.0, t->x0, t->x1};
    const double hi[3] = {t->x0, t->x1, xmax};
    for (int r = 0; r < 3; ++r)
      for (size_t s = 0; s < spr; ++s) {
        const double u = static_cast<double>(rng() >> 11) * 0x1.0p-53;
        const double x = lo[r] + (hi[r] - lo[r]) * u;
        const int L = terms_for(0, x, 1e-30);
        if (L < 0) return fail(BOYSFN_ERR_INVALID, "reference_terms_for: no L below cap reaches target");
        xs[r * spr + s] = x;
        terms[r * spr + s] = L;
      }
  }

  cudaStream_t s = nullptr;
  double *d_x = nullptr, *d_oracle = nullptr, *d_got = nullptr;
  int* d_terms = nullptr;
  unsigned long long *d_max = nullptr, *d_first = nullptr;
  auto release = [&]() {
    cudaFree(d_x);
    cudaFree(d_oracle);
    cudaFree(d_got);
    cudaFree(d_terms);
    cudaFree(d_max);
    cudaFree(d_first);
  };
  auto cuda_ok = [&](cudaError_t e, const char* where) {
    if (e == cudaSuccess) return true;
    boysfn_internal::cuda_fail(e, where);
    return false;
  };
  int status = BOYSFN_OK;
  const size_t kk = static_cast<size_t>(kmax) + 1;
  std::vector<unsigned long long> maxima(kk * 3, 0);
  do {
    if (!cuda_ok(cudaMalloc(&d_x, n * sizeof(double)), "cudaMalloc") ||
        !cuda_ok(cudaMalloc(&d_terms, n * sizeof(int)), "cudaMalloc") ||
        !cuda_ok(cudaMalloc(&d_oracle, n * kk * sizeof(double)), "cudaMalloc") ||
        !cuda_ok(cudaMalloc(&d_got, n * kk * sizeof(double)), "cudaMalloc") ||
        !cuda_ok(cudaMalloc(&d_max, kk * 3 * sizeof(unsigned long long)), "cudaMalloc") ||
        !cuda_ok(cudaMalloc(&d_first, sizeof(unsigned long long)), "cudaMalloc")) {
      status = BOYSFN_ERR_CUDA;
      break;
    }
    cudaMemcpy(d_x, xs.data(), n * sizeof(double), cudaMemcpyHostToDevice);
    cudaMemcpy(d_terms, terms.data(), n * sizeof(int), cudaMemcpyHostToDevice);
    cudaMemset(d_max, 0, kk * 3 * sizeof(unsigned long long));
    const unsigned grid = static_cast<unsigned>(std::min<size_t>((n + 127) / 128, 148 * 16));
    dd_oracle_kernel<<<grid, 128, 0, s>>>(d_x, d_terms, n, kmax, d_oracle);
    boysfn_internal::count_launch();
    for (int k = 0; k <= kmax && status == BOYSFN_OK; ++k) {
      status = boysfn_eval_device(t, d_x, n, k, d_got, n * (k + 1), BOYSFN_LAYOUT_AOS, 0, s, nullptr);
      if (status) break;
      compare_kernel<<<grid, 128, 0, s>>>(d_got, d_oracle, n, samples_per_region, k, kmax, d_max + 3 * k);
      boysfn_internal::count_launch();
    }
    if (status) break;
    if (!cuda_ok(cudaMemcpy(maxima.data(), d_max, kk * 3 * sizeof(unsigned long long), cudaMemcpyDeviceToHost),
                 "cudaMemcpy"))
      status = BOYSFN_ERR_CUDA;
  } while (false);

  if (status == BOYSFN_OK) {
    rep->max_err = 0;
    rep->worst_x = 0;
    rep->worst_k = 0;
    rep->worst_region = '-';
    for (int r = 0; r < 3; ++r) rep->max_err_region[r] = 0;
    for (size_t k = 0; k < kk; ++k)
      for (int r = 0; r < 3; ++r) {
        double v;
        std::memcpy(&v, &maxima[3 * k + r], sizeof v);
        rep->per_k[3 * k + r] = v;
        rep->max_err_region[r] = std::max(rep->max_err_region[r], v);
        rep->max_err = std::max(rep->max_err, v);
      }
    // the reference records the first (region, sample, k, l) reaching the
    // maximum: scan orders in loop order for the smallest sample index
    if (rep->max_err > 0) {
      unsigned long long best = ~0ull;
      int best_k = -1;
      for (int k = 0; k <= kmax && status == BOYSFN_OK; ++k) {
        bool has = false;
        for (int r = 0; r < 3; ++r) has |= rep->per_k[3 * k + r] == rep->max_err;
        if (!has) continue;
        status = boysfn_eval_device(t, d_x, n, k, d_got, n * (k + 1), BOYSFN_LAYOUT_AOS, 0, s, nullptr);
        if (status) break;
        cudaMemset(d_first, 0xFF, sizeof(unsigned long long));
        const unsigned grid = static_cast<unsigned>(std::min<size_t>((n + 127) / 128, 148 * 16));
        locate_kernel<<<grid, 128, 0, s>>>(d_got, d_oracle, n, k, kmax, rep->max_err, d_first);
        boysfn_internal::count_launch();
        unsigned long long first = ~0ull;
        cudaMemcpy(&first, d_first, sizeof first, cudaMemcpyDeviceToHost);
        if (first < best) {  // a smaller sample index wins; equal index keeps the smaller k
          best = first;
          best_k = k;
        }
      }
      if (status == BOYSFN_OK && best != ~0ull) {
        rep->worst_x = xs[best];
        rep->worst_k = best_k;
        rep->worst_region = static_cast<char>('A' + best / spr);
      }
    }
    if (status == BOYSFN_OK)
      if (cudaError_t e = cudaDeviceSynchronize()) status = boysfn_internal::cuda_fail(e, "boysfn_verify_tables");
  }
  release();
  return status;
}
