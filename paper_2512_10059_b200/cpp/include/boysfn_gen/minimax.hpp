// boysfn_gen/minimax.hpp -- the native coefficient generator: the region
// partition of arXiv 2512.10059 (Eqs. 12, 18, 20), a weighted rational
// minimax exchange (the paper's Fig. 1, Steps 1-6) and the Walsh-table degree
// search (Sec. II.D), in binary128 (the paper's own generator used quadruple
// precision), with the extremum search optionally on the B200
// (boysfn_gen_error_scan).  The same specified algorithms as the reference's
// generator library (regions/remez/highprec); a 50-digit mpmath version of
// them lives in paper_2512_10059_b200/gen/ and is used to cross-check this one.
#pragma once

#include <cstdint>
#include <functional>
#include <optional>
#include <tuple>
#include <vector>

#include <quadmath.h>

namespace boysfn::gen {

using real = __float128;
using rvec = std::vector<real>;

// Working digits (plus a fixed 12 guard digits; 22 + 12 fill binary128).  The
// solver's tolerances are powers of ten of these, as specified.
inline constexpr int kGuard = 12;
void set_digits(int working_digits);  // 16 .. 22
int digits();
real ten_to(int e);

// ---- special functions (x >= 0) ----
real gamma_half(int k);                       // Gamma(k + 1/2)
real erf_pos(real x);
real erfc_pos(real x);
real upper_gamma_half(int k, real x);         // Gamma(k + 1/2, x)
real boys_series(int k, real x, int terms);   // F_k by the equal-sign series (Eq. 21)
int series_terms(int k, double x, double rel);  // terms for an Eq. 22 bound <= rel (multiple of 25, >= 150)
real series_bound(int k, real x, int terms);  // Eq. 22
real recurrence_weight(int k, real x);        // rho_A,k (Eq. 18)

struct Partition {
  real x0, x1;
};
Partition partition(int k_max, real eps_tol);  // x0 (Eq. 20), x1 (Eq. 12, safeguarded Newton)

// ---- polynomials (ascending coefficients) ----
real horner(const rvec& c, real x);
rvec trim_top(const rvec& c, real rel);          // drop top coefficients below rel * max|c|
int sturm_count(const rvec& c, real a, real b);  // distinct real roots in (a, b]
rvec newton_to_monomial(const rvec& xs, const rvec& ys);
std::vector<int> leja_sequence(const rvec& xs);

// ---- symmetric eigenproblem (cyclic Jacobi) ----
void jacobi(std::vector<rvec> a, rvec& values, std::vector<rvec>& vectors);  // vectors[j] <-> values[j]

// ---- minimax ----
struct Rational {
  rvec num, den;
  real operator()(real x) const { return horner(num, x) / horner(den, x); }
};

// f and weight w on [a, b]; boys_k >= 0 names f = F_k and w = 1 (weight_kind
// 0) or rho_A,k (1), which lets the GPU scan evaluate the error itself.
struct Target {
  std::function<real(real)> f;
  std::function<real(real)> w;  // empty: 1
  int boys_k = -1;
  int weight_kind = 0;
};

struct FitOptions {
  int n = 0, m = 0;
  real conv = 0;         // stop when sup - |E| <= conv
  real abort_level = 0;  // Step 6: give up when every new node's error exceeds it (<= 0: never)
  std::uint64_t seed = 1;
  int max_iterations = 200, max_restarts = 100;
  int grid = 0;          // CPU scan grid; 0: 64 (n+m+2)
  bool gpu = false;      // GPU scan (needs Target::boys_k >= 0)
  int gpu_grid = 1 << 16, gpu_zoom = 2048;
};

enum class Outcome { converged, infeasible, iteration_limit, restart_limit };

struct Fit {
  Outcome outcome = Outcome::iteration_limit;
  Rational r;             // monic denominator on convergence
  real sup = 0;           // weighted sup error
  real level = 0;         // signed levelled error E of the last solve
  real lower_bound = 0;   // Step-6 certificate
  int iterations = 0, restarts = 0;
  rvec alternants;
  std::vector<std::pair<real, real>> history;  // (|E|, sup) per accepted iteration
};

Fit fit(const Target& t, real a, real b, const FitOptions& o);

struct DegreeChoice {
  bool ok = false;
  int n = 0, m = 0;
  Rational r;
  real sup = 0;
  int cells = 0;
  std::vector<std::tuple<int, int, real, Rational>> runners_up;  // the winning diagonal, best first
};

// Walsh table by anti-diagonals n + m = 0, 1, ...: the first diagonal with a
// cell meeting eps_tol wins, ties by the smaller sup error; cells pruned by the
// Step-6 abort at eps_tol.
DegreeChoice choose_degrees(const Target& t, real a, real b, real eps_tol, int max_degree, std::uint64_t seed,
                            bool gpu);

}  // namespace boysfn::gen
