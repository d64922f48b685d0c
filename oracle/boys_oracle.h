/*
 * oracle/boys_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * C interface of the CPU oracle: a bit-faithful restatement of the reference's
 * Algorithm 1 (boys_port.c, following /root/reference/proj/core/src/eval.cpp)
 * and an extended-precision Boys oracle (boys_hp.c, following
 * /root/reference/proj/core/src/reference.cpp).  Loaded by tests/ and bench.py's
 * CPU baseline only; the CUDA product never links it.
 */
#ifndef BOYS_ORACLE_H
#define BOYS_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  ORACLE_OK = 0,
  ORACLE_ERR_SIZE = 1,   /* std::invalid_argument, eval.cpp:90-91 */
  ORACLE_ERR_DOMAIN = 2, /* std::domain_error, eval.cpp:14-15 */
  ORACLE_ERR_RANGE = 3   /* std::out_of_range, eval.cpp:16-17 */
};

enum { ORACLE_REGION_A = 0, ORACLE_REGION_B = 1, ORACLE_REGION_C = 2 };

/* Mirrors RationalApproximant (tables.hpp:12-17): ascending degree, monic q. */
typedef struct {
  int n, m;
  const double* numer; /* n+1 */
  const double* denom; /* m+1 */
} oracle_rational;

/* Mirrors CoefficientTableSet (tables.hpp:21-28). */
typedef struct {
  double x0, x1;
  int k_max;
  double eps_tol;
  oracle_rational r_B;
  const oracle_rational* r_A; /* k_max+1 */
} oracle_tables;

/* ---- Algorithm 1 restatement (boys_port.c) ---- */
int oracle_classify_region(double x, const oracle_tables* t);
double oracle_eval_rational(const oracle_rational* r, double x);
int oracle_boys_batch_region(double x, int k, const oracle_tables* t, int region, double* out);
int oracle_boys_batch(double x, int k, const oracle_tables* t, double* out);
int oracle_boys_batch_many(const double* xs, size_t n, int k, const oracle_tables* t,
                           double* out, size_t out_len, size_t* first_bad);
int oracle_boys_batch_many_mt(const double* xs, size_t n, int k, const oracle_tables* t,
                              double* out, int nthreads);
void oracle_gen_uniform(double* x, size_t n, uint64_t seed, uint64_t offset, double lo,
                        double hi);
void oracle_gen_loguniform(double* x, size_t n, uint64_t seed, uint64_t offset, double lo, double hi);
void oracle_gen_boundary(double* x, size_t n, uint64_t seed, uint64_t offset, double x0, double x1);
/* Every value of a device output (AoS: soa = 0; SoA: soa = 1, row stride ld)
 * against the restatement, threaded, reference rows computed on the fly. */
int oracle_compare_output(const double* xs, size_t n, int k, const oracle_tables* t, const double* out, int soa,
                          size_t ld, double tol, int nthreads, double* max_dev, size_t* over_tol, size_t* c_mismatch,
                          size_t* c_values);
/* verify_tables' sampling (verify.cpp:23-33) and its std::mt19937_64. */
uint64_t oracle_mt64_nth(uint64_t seed, size_t nth);
void oracle_verify_samples(double x0, double x1, double xmax, size_t per_region, uint64_t seed, double* xs);
/* Algorithm 2 by direct summation. */
int oracle_alg2_direct(const double* x, const double* y, size_t n, int k, const double* c,
                       const oracle_tables* t, double* z, double* zabs, int nthreads);

/* ---- extended-precision oracle (boys_hp.c) ---- */
/* F_0..F_kmax at x, rounded to double (verify.cpp:38 convention). */
int oracle_hp_boys_batch(int kmax, double x, double* out);
/* Same, batched and threaded; returns 0 on success. */
int oracle_hp_boys_batch_many(int kmax, const double* xs, size_t n, double* out, int nthreads);
/* Series restatement alone (reference.cpp:10-23) at truncation index L. */
double oracle_hp_series(int k, double x, int L);
/* Closed form via the upper incomplete gamma continued fraction. */
double oracle_hp_closed_form(int k, double x);
/* reference_terms_for (reference.cpp:46-54); -1 where the reference throws. */
int oracle_hp_terms_for(int k, double x, double rel_target);
/* truncation_bound (reference.cpp:37-44), as a double. */
double oracle_hp_truncation_bound(int k, double x, int L);

#ifdef __cplusplus
}
#endif
#endif
