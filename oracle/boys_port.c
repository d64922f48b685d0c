/*
 * oracle/boys_port.c -- TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * A plain-C restatement of the reference hot path, Algorithm 1 of
 * arXiv 2512.10059 as implemented in /root/reference/proj/core/src/eval.cpp.
 * It performs the same double-precision operations in the same order as the
 * reference so that, compiled with -O2 -ffp-contract=off (the reference is
 * built -O2 without -march, hence without FMA: proj/CMakeLists.txt:6-8,
 * core/CMakeLists.txt:32), it is bit-identical to the reference.  That claim is
 * pinned by tests/test_oracle.py against the compiled reference (oracle/_ref)
 * and against the committed golden vectors in tests/golden/.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * arm may load this file's library.  The CUDA product path never calls it.
 */
#define _GNU_SOURCE  /* exp10 */
#include "boys_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* sqrt(pi)/2, correctly rounded -- eval.cpp:11 */
static const double kHalfSqrtPiOracle = 0.88622692545275801364908374167057;

/* check_input -- eval.cpp:13-18: x checked before k. */
static int port_check_input(double x, int k, const oracle_tables* t) {
  if (!isfinite(x) || x < 0) return ORACLE_ERR_DOMAIN;
  if (k < 0 || k > t->k_max) return ORACLE_ERR_RANGE;
  return ORACLE_OK;
}

/* classify_region -- eval.cpp:22-26 (half-open: boundary doubles go right). */
int oracle_classify_region(double x, const oracle_tables* t) {
  if (x < t->x0) return ORACLE_REGION_A;
  if (x < t->x1) return ORACLE_REGION_B;
  return ORACLE_REGION_C;
}

/* eval_rational -- eval.cpp:28-36: Horner from the top of ascending storage,
 * separate multiply and add (no contraction), one division. */
double oracle_eval_rational(const oracle_rational* r, double x) {
  double num = r->numer[r->n];
  for (int i = r->n; i-- > 0;) num = num * x + r->numer[i];
  double den = r->denom[r->m];
  for (int i = r->m; i-- > 0;) den = den * x + r->denom[i];
  return num / den;
}

/* downward_recursion -- eval.cpp:38-47. */
static void port_downward(double seed, double x, int k, double* out) {
  out[k] = seed;
  if (k == 0) return;
  const double e = exp(-x);
  const double twox = 2.0 * x;
  for (int l = k - 1; l >= 0; --l) out[l] = (twox * out[l + 1] + e) / (2 * l + 1);
}

/* upward_recursion -- eval.cpp:49-57 (exp evaluated even for k == 0). */
static void port_upward(double seed, double x, int k, double* out) {
  out[0] = seed;
  const double e = exp(-x);
  const double twox = 2.0 * x;
  for (int l = 0; l < k; ++l) out[l + 1] = ((2 * l + 1) * out[l] - e) / twox;
}

/* boys_batch_region -- eval.cpp:59-81 (region forced; test seam). */
int oracle_boys_batch_region(double x, int k, const oracle_tables* t, int region,
                             double* out) {
  int st = port_check_input(x, k, t);
  if (st != ORACLE_OK) return st;
  switch (region) {
    case ORACLE_REGION_A:
      port_downward(oracle_eval_rational(&t->r_A[k], x), x, k, out);
      break;
    case ORACLE_REGION_B:
      if (!(x > 0)) return ORACLE_ERR_DOMAIN; /* upward_recursion precondition, eval.cpp:50 */
      port_upward(oracle_eval_rational(&t->r_B, x), x, k, out);
      break;
    default: {
      out[0] = kHalfSqrtPiOracle / sqrt(x);
      const double inv2x = 0.5 / x;
      for (int l = 0; l < k; ++l) out[l + 1] = (2 * l + 1) * inv2x * out[l];
      break;
    }
  }
  return ORACLE_OK;
}

/* boys_batch -- eval.cpp:83-86. */
int oracle_boys_batch(double x, int k, const oracle_tables* t, double* out) {
  int st = port_check_input(x, k, t);
  if (st != ORACLE_OK) return st;
  return oracle_boys_batch_region(x, k, t, oracle_classify_region(x, t), out);
}

/* boys_batch_many -- eval.cpp:88-96.  Rows before the first bad x are written,
 * later rows are untouched; *first_bad receives the offending index. */
int oracle_boys_batch_many(const double* xs, size_t n, int k, const oracle_tables* t,
                           double* out, size_t out_len, size_t* first_bad) {
  if (out_len != n * ((size_t)k + 1)) return ORACLE_ERR_SIZE;
  const size_t row = (size_t)k + 1;
  for (size_t i = 0; i < n; ++i) {
    int st = oracle_boys_batch(xs[i], k, t, out + i * row);
    if (st != ORACLE_OK) {
      if (first_bad) *first_bad = i;
      return st;
    }
  }
  return ORACLE_OK;
}

/* ---- multi-threaded driver for the CPU baseline (disjoint spans; the path is
 * reentrant).  Threads are the only addition to the reference. */
typedef struct {
  const double* xs;
  size_t n;
  int k;
  const oracle_tables* t;
  double* out;
  int status;
  size_t bad;
} port_job;

static void* port_worker(void* arg) {
  port_job* j = (port_job*)arg;
  j->status = oracle_boys_batch_many(j->xs, j->n, j->k, j->t, j->out,
                                     j->n * ((size_t)j->k + 1), &j->bad);
  return NULL;
}

int oracle_boys_batch_many_mt(const double* xs, size_t n, int k, const oracle_tables* t,
                              double* out, int nthreads) {
  if (nthreads < 1) nthreads = 1;
  if ((size_t)nthreads > n) nthreads = n ? (int)n : 1;
  pthread_t* th = (pthread_t*)calloc((size_t)nthreads, sizeof(pthread_t));
  port_job* jobs = (port_job*)calloc((size_t)nthreads, sizeof(port_job));
  const size_t row = (size_t)k + 1;
  size_t begin = 0;
  for (int w = 0; w < nthreads; ++w) {
    size_t cnt = n / nthreads + ((size_t)w < n % nthreads ? 1 : 0);
    jobs[w] = (port_job){xs + begin, cnt, k, t, out + begin * row, 0, 0};
    pthread_create(&th[w], NULL, port_worker, &jobs[w]);
    begin += cnt;
  }
  int st = ORACLE_OK;
  for (int w = 0; w < nthreads; ++w) {
    pthread_join(th[w], NULL);
    if (st == ORACLE_OK && jobs[w].status != ORACLE_OK) st = jobs[w].status;
  }
  free(th);
  free(jobs);
  return st;
}

/* ---- Full-batch parity check (test infrastructure): every row of a device
 * output against this restatement, computed on the fly per thread (no host
 * copy of the reference output).  Records the max |gpu - ref|, the number of
 * values above tol, and the number of region-C values (x >= x1) that differ
 * in any bit.  layout 0: AoS out[i*(k+1)+l]; 1: SoA out[l*ld+i]. */
typedef struct {
  const double* xs;
  const double* out;
  size_t i0, i1, ld;
  int k, soa;
  double tol;
  const oracle_tables* t;
  double max_dev;
  size_t over_tol, c_mismatch, c_values;
  int status;
} cmp_job;

static void* cmp_worker(void* arg) {
  cmp_job* j = (cmp_job*)arg;
  double F[130];
  const size_t row = (size_t)j->k + 1;
  for (size_t i = j->i0; i < j->i1; ++i) {
    if (oracle_boys_batch(j->xs[i], j->k, j->t, F) != ORACLE_OK) {
      j->status = ORACLE_ERR_DOMAIN;
      return NULL;
    }
    const int inC = !(j->xs[i] < j->t->x1);
    for (size_t l = 0; l < row; ++l) {
      const double g = j->soa ? j->out[l * j->ld + i] : j->out[i * row + l];
      const double d = fabs(g - F[l]);
      if (d > j->max_dev) j->max_dev = d;
      if (d > j->tol) ++j->over_tol;
      if (inC) {
        ++j->c_values;
        if (memcmp(&g, &F[l], sizeof g) != 0) ++j->c_mismatch;
      }
    }
  }
  return NULL;
}

int oracle_compare_output(const double* xs, size_t n, int k, const oracle_tables* t, const double* out, int soa,
                          size_t ld, double tol, int nthreads, double* max_dev, size_t* over_tol, size_t* c_mismatch,
                          size_t* c_values) {
  if (nthreads < 1) nthreads = 1;
  if ((size_t)nthreads > n) nthreads = n ? (int)n : 1;
  if (k < 0 || k > 128) return ORACLE_ERR_RANGE;
  pthread_t* th = (pthread_t*)calloc((size_t)nthreads, sizeof(pthread_t));
  cmp_job* jobs = (cmp_job*)calloc((size_t)nthreads, sizeof(cmp_job));
  size_t begin = 0;
  for (int w = 0; w < nthreads; ++w) {
    const size_t cnt = n / nthreads + ((size_t)w < n % nthreads ? 1 : 0);
    jobs[w] = (cmp_job){xs, out, begin, begin + cnt, ld, k, soa, tol, t, 0.0, 0, 0, 0, ORACLE_OK};
    pthread_create(&th[w], NULL, cmp_worker, &jobs[w]);
    begin += cnt;
  }
  int st = ORACLE_OK;
  *max_dev = 0.0;
  *over_tol = *c_mismatch = *c_values = 0;
  for (int w = 0; w < nthreads; ++w) {
    pthread_join(th[w], NULL);
    if (st == ORACLE_OK && jobs[w].status != ORACLE_OK) st = jobs[w].status;
    if (jobs[w].max_dev > *max_dev) *max_dev = jobs[w].max_dev;
    *over_tol += jobs[w].over_tol;
    *c_mismatch += jobs[w].c_mismatch;
    *c_values += jobs[w].c_values;
  }
  free(th);
  free(jobs);
  return st;
}

/* ---- Algorithm 2 direct summation (the benchmark's correctness
 * oracle): z_i = sum_j y_j sum_l c_l F_l(x_i + x_j) with every F from the
 * reference restatement above; zabs_i = sum_j |y_j sum_l c_l F_l| scales the
 * relative tolerance.  Rows are split over threads. */
typedef struct {
  const double *x, *y, *c;
  size_t n, i0, i1;
  int k;
  const oracle_tables* t;
  double *z, *zabs;
  int status;
} alg2_job;

static void* alg2_worker(void* arg) {
  alg2_job* j = (alg2_job*)arg;
  double F[130];
  for (size_t i = j->i0; i < j->i1; ++i) {
    double z = 0, za = 0;
    for (size_t jj = 0; jj < j->n; ++jj) {
      if (oracle_boys_batch(j->x[i] + j->x[jj], j->k, j->t, F) != ORACLE_OK) {
        j->status = ORACLE_ERR_DOMAIN;
        return NULL;
      }
      double w = 0;
      for (int l = 0; l <= j->k; ++l) w += j->c[l] * F[l];
      z += j->y[jj] * w;
      za += fabs(j->y[jj] * w);
    }
    j->z[i] = z;
    if (j->zabs) j->zabs[i] = za;
  }
  return NULL;
}

int oracle_alg2_direct(const double* x, const double* y, size_t n, int k, const double* c,
                       const oracle_tables* t, double* z, double* zabs, int nthreads) {
  if (k < 0 || k > t->k_max || k >= 130) return ORACLE_ERR_RANGE;
  if (nthreads < 1) nthreads = 1;
  if ((size_t)nthreads > n) nthreads = n ? (int)n : 1;
  pthread_t* th = (pthread_t*)calloc((size_t)nthreads, sizeof(pthread_t));
  alg2_job* jobs = (alg2_job*)calloc((size_t)nthreads, sizeof(alg2_job));
  size_t begin = 0;
  for (int w = 0; w < nthreads; ++w) {
    const size_t cnt = n / nthreads + ((size_t)w < n % nthreads ? 1 : 0);
    jobs[w] = (alg2_job){x, y, c, n, begin, begin + cnt, k, t, z, zabs, 0};
    pthread_create(&th[w], NULL, alg2_worker, &jobs[w]);
    begin += cnt;
  }
  int st = ORACLE_OK;
  for (int w = 0; w < nthreads; ++w) {
    pthread_join(th[w], NULL);
    if (jobs[w].status != ORACLE_OK) st = jobs[w].status;
  }
  free(th);
  free(jobs);
  return st;
}

/* ---- the sampling of verify_tables (verify.cpp:23-33): std::mt19937_64(seed)
 * restated from the C++ standard ([rand.eng.mers], [rand.predef]: w=64, n=312,
 * m=156, r=31, a=0xB5026F5AA96619E9, tempering u=29 d=0x5555555555555555 s=17
 * b=0x71D67FFFEDA60000 t=37 c=0xFFF7EEE000000000 l=43, f=6364136223846793005),
 * x = lo + (hi - lo) * ((rng() >> 11) * 2^-53) per region in order A, B, C. */
typedef struct {
  uint64_t mt[312];
  int idx;
} mt64;

static void mt64_seed(mt64* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->idx = 312;
}

static uint64_t mt64_next(mt64* g) {
  if (g->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      const uint64_t y = (g->mt[i] & 0xFFFFFFFF80000000ULL) | (g->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
      g->mt[i] = g->mt[(i + 156) % 312] ^ (y >> 1) ^ ((y & 1) ? 0xB5026F5AA96619E9ULL : 0);
    }
    g->idx = 0;
  }
  uint64_t y = g->mt[g->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

uint64_t oracle_mt64_nth(uint64_t seed, size_t nth) {
  mt64 g;
  mt64_seed(&g, seed);
  uint64_t v = 0;
  for (size_t i = 0; i < nth; ++i) v = mt64_next(&g);
  return v;
}

void oracle_verify_samples(double x0, double x1, double xmax, size_t per_region, uint64_t seed, double* xs) {
  mt64 g;
  mt64_seed(&g, seed);
  const double lo[3] = {0.0, x0, x1}, hi[3] = {x0, x1, xmax};
  for (int r = 0; r < 3; ++r)
    for (size_t s = 0; s < per_region; ++s) {
      const double u = (double)(mt64_next(&g) >> 11) * 0x1.0p-53;
      xs[r * per_region + s] = lo[r] + (hi[r] - lo[r]) * u;
    }
}

/* ---- synthetic workload generator shared with the device generator
 * (paper_2512_10059_b200/csrc/boys_kernels.cu: gen_uniform_kernel).  splitmix64
 * keyed by the global index, so shards of any size reproduce one stream. */
static uint64_t splitmix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

void oracle_gen_uniform(double* x, size_t n, uint64_t seed, uint64_t offset, double lo,
                        double hi) {
  const double span = hi - lo;
  for (size_t i = 0; i < n; ++i) {
    const uint64_t z = splitmix64(seed + (offset + i + 1) * 0x9E3779B97F4A7C15ULL);
    const double u = (double)(z >> 11) * 0x1.0p-53;
    x[i] = lo + span * u; /* -ffp-contract=off: mul and add rounded separately */
  }
}

/* The log-uniform stream of boysfn_generate_loguniform: 10^(lo + span*u) with
 * the same u; host exp10 (glibc) may differ from the device's by an ulp, so
 * this is the same law, not the same doubles (the reference arm's input). */
void oracle_gen_loguniform(double* x, size_t n, uint64_t seed, uint64_t offset, double lo, double hi) {
  const double span = hi - lo;
  for (size_t i = 0; i < n; ++i) {
    const uint64_t z = splitmix64(seed + (offset + i + 1) * 0x9E3779B97F4A7C15ULL);
    x[i] = exp10(lo + span * ((double)(z >> 11) * 0x1.0p-53));
  }
}

/* The configs[2] boundary-stress stream of boysfn_generate_boundary
 * (capi.cu: gen_boundary_kernel), operation for operation; only mode 1's
 * exp10 can differ from the device's by an ulp. */
void oracle_gen_boundary(double* x, size_t n, uint64_t seed, uint64_t offset, double x0, double x1) {
  for (size_t i = 0; i < n; ++i) {
    const uint64_t z = splitmix64(seed + (offset + i + 1) * 0x9E3779B97F4A7C15ULL);
    const uint64_t w = splitmix64(z ^ 0xD1B54A32D192ED03ULL);
    const int which = (int)(z % 3), mode = (int)((z >> 8) % 3);
    const double u = (double)(w >> 11) * 0x1.0p-53;
    const double b = which == 0 ? 0.0 : which == 1 ? x0 : x1;
    double v;
    if (mode == 0) {
      const long long j = (long long)((w >> 20) % 129) - 64;
      if (b == 0.0) {
        v = (double)(j < 0 ? -j : j) * 4.9406564584124654e-324;
      } else {
        uint64_t bits;
        memcpy(&bits, &b, sizeof bits);
        bits += (uint64_t)j;
        memcpy(&v, &bits, sizeof v);
      }
    } else if (mode == 1) {
      /* the device contracts 1 + 14u into one fma (nvcc's default) */
      const double off = exp10(-fma(14.0, u, 1.0));
      v = ((w >> 10) & 1) ? b + off : b - off;
    } else {
      v = b + (2.0 * u - 1.0);
    }
    x[i] = fabs(v);
  }
}
