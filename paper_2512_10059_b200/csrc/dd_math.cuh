// dd_math.cuh -- double-double (~106-bit significand) device arithmetic for
// the extended-precision oracles: verify_tables (verify.cu) and the
// generator's error scan (gen_scan.cu).  Error-free transformations by FMA;
// e^{-x} by ln 2 range reduction and a 30-term Taylor series.
#pragma once

namespace boysfn_dd {

struct dd {
  double hi, lo;
};

__device__ __forceinline__ dd two_sum(double a, double b) {
  const double s = a + b;
  const double bb = s - a;
  return {s, (a - (s - bb)) + (b - bb)};
}
__device__ __forceinline__ dd quick_two_sum(double a, double b) {
  const double s = a + b;
  return {s, b - (s - a)};
}
__device__ __forceinline__ dd dd_add(dd a, dd b) {
  dd s = two_sum(a.hi, b.hi);
  const dd t = two_sum(a.lo, b.lo);
  s.lo += t.hi;
  s = quick_two_sum(s.hi, s.lo);
  s.lo += t.lo;
  return quick_two_sum(s.hi, s.lo);
}
__device__ __forceinline__ dd dd_mul_d(dd a, double b) {
  const double p = a.hi * b;
  double e = __fma_rn(a.hi, b, -p);
  e = __fma_rn(a.lo, b, e);
  return quick_two_sum(p, e);
}
__device__ __forceinline__ dd dd_mul(dd a, dd b) {
  const double p = a.hi * b.hi;
  double e = __fma_rn(a.hi, b.hi, -p);
  e = __fma_rn(a.hi, b.lo, e);
  e = __fma_rn(a.lo, b.hi, e);
  return quick_two_sum(p, e);
}
__device__ __forceinline__ dd dd_div_d(dd a, double b) {
  const double q1 = a.hi / b;
  dd r = dd_add(a, dd_mul_d(dd{q1, 0.0}, -b));
  const double q2 = r.hi / b;
  r = dd_add(r, dd_mul_d(dd{q2, 0.0}, -b));
  const double q3 = r.hi / b;
  const dd q = quick_two_sum(q1, q2);
  return dd_add(q, dd{q3, 0.0});
}

// e^{-x} in double-double, 0 <= x <= ~700.
static __device__ dd dd_exp_neg(double x) {
  const dd ln2{0.6931471805599453, 2.3190468138462996e-17};
  const double n = rint(x / ln2.hi);
  // r = x - n ln2, exactly enough in dd
  dd r = dd_add(dd{x, 0.0}, dd_mul_d(ln2, -n));
  r = dd{-r.hi, -r.lo};  // exponent of the reduced factor: -(x - n ln2)
  // Taylor series of e^r, |r| <= 0.35: 30 terms < 1e-40
  dd term{1.0, 0.0}, sum{1.0, 0.0};
  for (int j = 1; j <= 30; ++j) {
    term = dd_div_d(dd_mul(term, r), static_cast<double>(j));
    sum = dd_add(sum, term);
  }
  const double s = ldexp(1.0, -static_cast<int>(n));  // exact power of two
  return {sum.hi * s, sum.lo * s};
}

__device__ __forceinline__ dd dd_neg(dd a) { return {-a.hi, -a.lo}; }
__device__ __forceinline__ dd dd_sub(dd a, dd b) { return dd_add(a, dd_neg(b)); }
// a / b, three quotient digits
__device__ __forceinline__ dd dd_div(dd a, dd b) {
  const double q1 = a.hi / b.hi;
  dd r = dd_sub(a, dd_mul_d(b, q1));
  const double q2 = r.hi / b.hi;
  r = dd_sub(r, dd_mul_d(b, q2));
  const double q3 = r.hi / b.hi;
  return dd_add(quick_two_sum(q1, q2), dd{q3, 0.0});
}

}  // namespace boysfn_dd
