// highprec.hpp -- extended-precision substrate of the native generator.
// Mirrors the reference's boysfn/highprec.hpp (highprec.hpp:1-41) with
// hp::Real = __float128 (IEEE binary128, 113-bit significand, ~34 digits; the
// paper's own generator used quadruple precision) instead of a 50+12-digit
// MPFR float: Boost.Multiprecision and the MPFR headers are not available to
// this build.  The Python generator (paper_2512_10059_b200/gen) runs the same
// algorithms at the reference's 50+12 digits in mpmath.
#pragma once

#include <quadmath.h>

namespace boysfn::hp {

using Real = __float128;

// Working digits + guard digits = the binary128 significand (~34 digits).
inline constexpr int kDefaultDigits10 = 22;
inline constexpr int kGuardDigits10 = 12;

void set_working_digits(int digits10);  // 16 .. 22
int working_digits();

Real pow10(int e);  // 10^e
const Real& sqrt_pi();
Real exp(const Real& x);
Real gamma_half(int k);                  // Gamma(k + 1/2)
Real erf(const Real& x);                 // x >= 0
Real erfc(const Real& x);                // x >= 0
Real upper_gamma_half(int k, const Real& x);  // Gamma(k + 1/2, x), x >= 0

inline Real abs(const Real& x) { return fabsq(x); }
inline Real sqrt(const Real& x) { return sqrtq(x); }
inline Real log(const Real& x) { return logq(x); }
inline Real pow(const Real& x, const Real& y) { return powq(x, y); }

}  // namespace boysfn::hp
