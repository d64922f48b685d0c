// gen_scan.cu -- the coefficient generator's error scan on the B200 (SURVEY.md
// section 8(f) rank 4; reference: remez.cpp:33-108, the ErrorCurve grid scan of
// the weighted Remez error rho (f - p/q)).
//
// One thread per abscissa evaluates, in double-double:
//   f(x) = F_k(x) by the reference's equal-sign series (reference.cpp:10-23),
//          summed until the terms fall below 1e-34 of the sum (x <= ~60 in the
//          generation domain, so a few hundred terms at most);
//   r(x) = p(x)/q(x) by Horner with double-double coefficients;
//   rho(x) = 1 (region B, r_B) or rho_A,k(x) = max_l prod_{n=l}^{k-1} x/(n+1/2)
//            (Eq. 18, regions.cpp:74-85; region A, r_A[k]) in double;
// and writes e(x) = rho (f - r) rounded to double.  e is ~eps_tol (5e-14) in
// magnitude while f and r are O(1), so double-double leaves ~16 correct digits
// in e where the Remez exchange needs 3.
#include <cuda_runtime.h>

#include <algorithm>

#include "capi_internal.h"
#include "dd_math.cuh"

namespace {

using namespace boysfn_dd;

constexpr int kMaxGenCoef = 65;  // degree <= 64

struct GenRational {
  dd num[kMaxGenCoef];
  dd den[kMaxGenCoef];
  int n, m;
};

__device__ dd boys_series_dd(int k, double x) {
  dd term = dd_div_d(dd{1.0, 0.0}, k + 0.5);
  dd sum = term;
  for (int l = 1; l < 20000; ++l) {
    term = dd_div_d(dd_mul_d(term, x), k + l + 0.5);
    sum = dd_add(sum, term);
    if (l > x && term.hi < 1e-34 * sum.hi) break;
  }
  return dd_mul(dd_mul_d(dd_exp_neg(x), 0.5), sum);
}

__device__ dd horner_dd(const dd* c, int deg, double x) {
  dd acc = c[deg];
  for (int i = deg - 1; i >= 0; --i) acc = dd_add(dd_mul_d(acc, x), c[i]);
  return acc;
}

__device__ double rho_A(int k, double x) {
  double prod = 1.0, best = 1.0;
  for (int l = k - 1; l >= 0; --l) {
    prod = prod * x / (l + 0.5);
    best = fmax(best, prod);
  }
  return best;
}

__global__ void gen_error_kernel(const __grid_constant__ GenRational R, int k, int weight,
                                 const double* __restrict__ xs, size_t n, double* __restrict__ err) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
    const double x = xs[i];
    const dd f = boys_series_dd(k, x);
    const dd r = dd_div(horner_dd(R.num, R.n, x), horner_dd(R.den, R.m, x));
    const dd d = dd_sub(f, r);
    const double w = weight == 1 ? rho_A(k, x) : 1.0;
    err[i] = w * (d.hi + d.lo);
  }
}

__global__ void gen_boys_kernel(int k, const double* __restrict__ xs, size_t n, double* __restrict__ hi,
                                double* __restrict__ lo) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
    const dd f = boys_series_dd(k, xs[i]);
    hi[i] = f.hi;
    lo[i] = f.lo;
  }
}

// Per host thread: a private stream and device buffers grown on demand, so
// generator threads scanning concurrently neither allocate per call (cudaFree
// synchronises the device) nor serialise on the legacy default stream.
struct ScanScratch {
  cudaStream_t stream = nullptr;
  double* d[3] = {nullptr, nullptr, nullptr};
  size_t cap = 0;
  int device = -1;
  ~ScanScratch() {
    for (double* p : d) cudaFree(p);
    if (stream) cudaStreamDestroy(stream);
  }
};

int scratch_for(size_t n, ScanScratch** out) {
  thread_local ScanScratch s;
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  if (s.device != dev) {  // first use on this thread, or the thread switched devices
    for (double*& p : s.d) {
      cudaFree(p);
      p = nullptr;
    }
    s.cap = 0;
    if (s.stream) cudaStreamDestroy(s.stream);
    s.stream = nullptr;
    CUDA_TRY(cudaStreamCreateWithFlags(&s.stream, cudaStreamNonBlocking));
    s.device = dev;
  }
  if (n > s.cap) {
    for (double*& p : s.d) {
      cudaFree(p);
      p = nullptr;
      CUDA_TRY(cudaMalloc(&p, n * sizeof(double)));
    }
    s.cap = n;
  }
  *out = &s;
  return BOYSFN_OK;
}

}  // namespace

BOYSFN_API int boysfn_gen_error_scan(int k, const double* num_hi, const double* num_lo, int n, const double* den_hi,
                                     const double* den_lo, int m, int weight, const double* xs, size_t npts,
                                     double* err) {
  using boysfn_internal::fail;
  if (k < 0 || k > 64) return fail(BOYSFN_ERR_ARG, "gen_error_scan: k must lie in [0, 64]");
  if (n < 0 || m < 0 || n >= kMaxGenCoef || m >= kMaxGenCoef)
    return fail(BOYSFN_ERR_ARG, "gen_error_scan: degrees must lie in [0, 64]");
  if (weight != 0 && weight != 1) return fail(BOYSFN_ERR_ARG, "gen_error_scan: weight must be 0 (one) or 1 (rho_A)");
  if (npts == 0) return BOYSFN_OK;
  if (!num_hi || !num_lo || !den_hi || !den_lo || !xs || !err) return fail(BOYSFN_ERR_ARG, "null argument");
  GenRational R{};
  R.n = n;
  R.m = m;
  for (int i = 0; i <= n; ++i) R.num[i] = dd{num_hi[i], num_lo[i]};
  for (int i = 0; i <= m; ++i) R.den[i] = dd{den_hi[i], den_lo[i]};
  ScanScratch* S = nullptr;
  if (int st = scratch_for(npts, &S)) return st;
  CUDA_TRY(cudaMemcpyAsync(S->d[0], xs, npts * sizeof(double), cudaMemcpyHostToDevice, S->stream));
  const unsigned grid = static_cast<unsigned>(std::min<size_t>((npts + 255) / 256, 148 * 16));
  gen_error_kernel<<<grid, 256, 0, S->stream>>>(R, k, weight, S->d[0], npts, S->d[1]);
  CUDA_TRY(cudaGetLastError());
  boysfn_internal::count_launch();
  CUDA_TRY(cudaMemcpyAsync(err, S->d[1], npts * sizeof(double), cudaMemcpyDeviceToHost, S->stream));
  CUDA_TRY(cudaStreamSynchronize(S->stream));
  return BOYSFN_OK;
}

BOYSFN_API int boysfn_gen_boys_dd(int k, const double* xs, size_t npts, double* hi, double* lo) {
  using boysfn_internal::fail;
  if (k < 0 || k > 64) return fail(BOYSFN_ERR_ARG, "gen_boys_dd: k must lie in [0, 64]");
  if (npts == 0) return BOYSFN_OK;
  if (!xs || !hi || !lo) return fail(BOYSFN_ERR_ARG, "null argument");
  ScanScratch* S = nullptr;
  if (int st = scratch_for(npts, &S)) return st;
  CUDA_TRY(cudaMemcpyAsync(S->d[0], xs, npts * sizeof(double), cudaMemcpyHostToDevice, S->stream));
  const unsigned grid = static_cast<unsigned>(std::min<size_t>((npts + 255) / 256, 148 * 16));
  gen_boys_kernel<<<grid, 256, 0, S->stream>>>(k, S->d[0], npts, S->d[1], S->d[2]);
  CUDA_TRY(cudaGetLastError());
  boysfn_internal::count_launch();
  CUDA_TRY(cudaMemcpyAsync(hi, S->d[1], npts * sizeof(double), cudaMemcpyDeviceToHost, S->stream));
  CUDA_TRY(cudaMemcpyAsync(lo, S->d[2], npts * sizeof(double), cudaMemcpyDeviceToHost, S->stream));
  CUDA_TRY(cudaStreamSynchronize(S->stream));
  return BOYSFN_OK;
}
