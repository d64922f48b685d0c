/*
 * oracle/boys_hp.c -- TEST INFRASTRUCTURE ONLY (the accuracy checker).
 *
 * Extended-precision Boys oracle, a restatement of the reference's
 * multiprecision oracle /root/reference/proj/core/src/reference.cpp in
 * IEEE binary128 (__float128, libquadmath; 113-bit significand, ~34 digits).
 * The reference uses Boost.Multiprecision mpfr_float at 50+12 digits
 * (highprec.hpp:10-13), which cannot be built here (no Boost/MPFR headers);
 * binary128 is ample for a 5e-14 absolute gate on values <= 1: every path below
 * keeps a relative error under ~1e-30 before the final rounding to double.
 *
 *  - series (reference.cpp:10-23, Eq. 21): term_0 = 1/(k+1/2),
 *    term_l = term_{l-1} * x / (k+l+1/2), F_k = e^{-x}/2 * sum.
 *  - batch (reference.cpp:25-35): F_kmax from the series, then the downward
 *    recurrence F_l = (2x F_{l+1} + e^{-x})/(2l+1) carried in extended precision.
 *  - series length (reference.cpp:46-54, reference_terms_for): smallest
 *    multiple-of-25 L >= 150 whose bound x^{k+L+3/2}/Gamma(k+L+3/2) <= rel.
 *    The reference throws above x ~ 7331 (cap L <= 20000); there, and for any
 *    x >= max(kClosedFormX, kmax + 12), F_kmax comes from the closed form
 *    F_k(x) = [Gamma(k+1/2) - Gamma(k+1/2, x)] / (2 x^{k+1/2}),
 *    with Gamma(a, x) by the modified-Lentz continued fraction the reference
 *    uses for erfc (highprec.cpp:95-117).  tests/test_oracle.py checks that the
 *    two forms agree on their overlap and that both match mpmath at 40 digits.
 *
 * Results are rounded to double once (verify.cpp:38), so the error convention
 * of the tests is the reference's: |double - double(oracle)|.
 */
#include <math.h>
#include <pthread.h>
#include <quadmath.h>
#include <stdlib.h>

#include "boys_oracle.h"

typedef __float128 q_t;

/* Above this x the closed form is used (cheaper; the series needs ~x terms). */
static const double kClosedFormX = 60.0;

/* reference_terms_for -- reference.cpp:46-54 (double-precision lgamma sizing). */
int oracle_hp_terms_for(int k, double x, double rel_target) {
  if (x <= 0) return 150;
  const double log_target = log(rel_target);
  for (int L = 150; L <= 20000; L += 25) {
    const double s = k + L + 1.5;
    if (s * log(x) - lgamma(s) <= log_target) return L;
  }
  return -1; /* the reference throws std::runtime_error here */
}

/* truncation_bound -- reference.cpp:37-44: x^(k+L+3/2) / Gamma(k+L+3/2). */
double oracle_hp_truncation_bound(int k, double x, int L) {
  if (x == 0) return 0.0;
  const q_t s = (q_t)k + L + 1.5Q;
  return (double)expq(s * logq((q_t)x) - lgammaq(s));
}

/* boys_reference -- reference.cpp:10-23 (the series, all terms positive). */
static q_t hp_series_q(int k, q_t x, int L) {
  q_t term = 1.0Q / ((q_t)k + 0.5Q);
  q_t sum = term;
  for (int l = 1; l <= L; ++l) {
    term *= x;
    term /= ((q_t)k + l + 0.5Q);
    sum += term;
  }
  return expq(-x) / 2 * sum;
}

double oracle_hp_series(int k, double x, int L) { return (double)hp_series_q(k, (q_t)x, L); }

/* Gamma(k + 1/2) = sqrt(pi) * prod_{i=1..k} (i - 1/2) -- highprec.cpp:69-75. */
static q_t hp_gamma_half(int k) {
  q_t v = sqrtq(M_PIq);
  for (int i = 1; i <= k; ++i) v *= ((q_t)i - 0.5Q);
  return v;
}

/* Gamma(a, z) by modified Lentz -- the scheme of highprec.cpp:95-117. */
static q_t hp_upper_gamma_cf(q_t a, q_t z) {
  const q_t eps = 1e-33Q;
  const q_t fpmin = 1e-4000Q;
  q_t b = z + 1 - a;
  q_t c = 1 / fpmin;
  q_t d = 1 / b;
  q_t h = d;
  for (int i = 1; i < 100000; ++i) {
    const q_t an = -(q_t)i * ((q_t)i - a);
    b += 2;
    d = an * d + b;
    if (fabsq(d) < fpmin) d = fpmin;
    c = b + an / c;
    if (fabsq(c) < fpmin) c = fpmin;
    d = 1 / d;
    const q_t del = d * c;
    h *= del;
    if (fabsq(del - 1) <= eps) break;
  }
  return expq(-z + a * logq(z)) * h;
}

static q_t hp_closed_form_q(int k, q_t x) {
  const q_t a = (q_t)k + 0.5Q;
  const q_t lower = hp_gamma_half(k) - hp_upper_gamma_cf(a, x);
  return lower / (2 * expq(a * logq(x)));
}

double oracle_hp_closed_form(int k, double x) { return (double)hp_closed_form_q(k, (q_t)x); }

/* boys_reference_batch -- reference.cpp:25-35, rounded to double. */
int oracle_hp_boys_batch(int kmax, double xd, double* out) {
  if (kmax < 0 || !(xd >= 0) || isinf(xd)) return ORACLE_ERR_DOMAIN;
  if (xd == 0) {
    for (int l = 0; l <= kmax; ++l) out[l] = (double)(1.0Q / (2 * l + 1));
    return ORACLE_OK;
  }
  const q_t x = (q_t)xd;
  q_t fk;
  /* The continued fraction for Gamma(a, x) needs x comfortably above a + 1. */
  if (xd < kClosedFormX || xd < kmax + 12.0) {
    /* verify.cpp:35 sizes L at k = 0 (conservative); 1e-30 target as there. */
    const int L = oracle_hp_terms_for(0, xd, 1e-30);
    if (L < 0) return ORACLE_ERR_RANGE;
    fk = hp_series_q(kmax, x, L);
  } else {
    fk = hp_closed_form_q(kmax, x);
  }
  q_t vals[130];
  if (kmax >= 130) return ORACLE_ERR_RANGE;
  vals[kmax] = fk;
  const q_t e = expq(-x);
  for (int l = kmax - 1; l >= 0; --l) vals[l] = (2 * x * vals[l + 1] + e) / (2 * l + 1);
  for (int l = 0; l <= kmax; ++l) out[l] = (double)vals[l];
  return ORACLE_OK;
}

typedef struct {
  int kmax;
  const double* xs;
  size_t n;
  double* out;
  int status;
} hp_job;

static void* hp_worker(void* arg) {
  hp_job* j = (hp_job*)arg;
  for (size_t i = 0; i < j->n; ++i) {
    int st = oracle_hp_boys_batch(j->kmax, j->xs[i], j->out + i * (size_t)(j->kmax + 1));
    if (st != ORACLE_OK) j->status = st;
  }
  return NULL;
}

int oracle_hp_boys_batch_many(int kmax, const double* xs, size_t n, double* out, int nthreads) {
  if (nthreads < 1) nthreads = 1;
  if ((size_t)nthreads > n) nthreads = n ? (int)n : 1;
  pthread_t* th = (pthread_t*)calloc((size_t)nthreads, sizeof(pthread_t));
  hp_job* jobs = (hp_job*)calloc((size_t)nthreads, sizeof(hp_job));
  size_t begin = 0;
  for (int w = 0; w < nthreads; ++w) {
    size_t cnt = n / nthreads + ((size_t)w < n % nthreads ? 1 : 0);
    jobs[w] = (hp_job){kmax, xs + begin, cnt, out + begin * (size_t)(kmax + 1), 0};
    pthread_create(&th[w], NULL, hp_worker, &jobs[w]);
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
