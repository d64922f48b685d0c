// gen_hp.cpp -- binary128 restatement of highprec.cpp, reference.cpp,
// polynomial.cpp, linalg.cpp and regions.cpp of the reference generator
// (file:line cited per function).  Same algorithms; precision-dependent
// tolerances follow working_digits() + kGuardDigits10 as in the reference.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <sstream>
#include <stdexcept>
#include <string>

#include "boysfn/highprec.hpp"
#include "boysfn/linalg.hpp"
#include "boysfn/polynomial.hpp"
#include "boysfn/reference.hpp"
#include "boysfn/regions.hpp"

namespace boysfn {
namespace hp {
namespace {
std::atomic<int> g_digits{kDefaultDigits10};
Real series_eps() { return pow10(-(working_digits() + kGuardDigits10 - 2)); }  // highprec.cpp:28-32
}  // namespace

void set_working_digits(int d) {  // highprec.cpp:36-41 (capped by the binary128 significand)
  if (d < 16 || d > kDefaultDigits10)
    throw std::invalid_argument("working precision must lie in [16, 22] digits for binary128");
  g_digits.store(d);
}
int working_digits() { return g_digits.load(); }

Real pow10(int e) {
  Real r = 1, b = 10;
  unsigned u = static_cast<unsigned>(e < 0 ? -e : e);
  while (u) {
    if (u & 1) r *= b;
    b *= b;
    u >>= 1;
  }
  return e < 0 ? 1 / r : r;
}

const Real& sqrt_pi() {
  static const Real v = sqrtq(M_PIq);
  return v;
}

Real exp(const Real& x) {
  if (!finiteq(x)) throw std::domain_error("hp::exp: non-finite argument");
  const Real r = expq(x);
  if (!finiteq(r)) throw std::overflow_error("hp::exp: result overflows exponent range");
  return r;
}

Real gamma_half(int k) {  // highprec.cpp:62-68
  if (k < 0) throw std::domain_error("hp::gamma_half: k must be non-negative");
  Real v = sqrt_pi();
  for (int i = 1; i <= k; ++i) v *= (Real(i) - Real(0.5));
  return v;
}

namespace {
Real erf_series(const Real& x) {  // highprec.cpp:75-89
  const Real eps = series_eps(), xx = x * x;
  Real u = x, sum = x;
  for (int n = 1; n < 100000; ++n) {
    u *= -xx;
    u /= n;
    const Real term = u / (2 * n + 1);
    sum += term;
    if (fabsq(term) <= fabsq(sum) * eps) break;
  }
  return 2 * sum / sqrt_pi();
}

Real upper_gamma_cf(const Real& a, const Real& z) {  // highprec.cpp:95-117 (modified Lentz)
  const Real eps = series_eps();
  const Real fpmin = pow10(-4000);  // far below any term; binary128 reaches ~1e-4965
  Real b = z + 1 - a, c = 1 / fpmin, d = 1 / b, h = d;
  for (int i = 1; i < 100000; ++i) {
    const Real an = -Real(i) * (Real(i) - a);
    b += 2;
    d = an * d + b;
    if (fabsq(d) < fpmin) d = fpmin;
    c = b + an / c;
    if (fabsq(c) < fpmin) c = fpmin;
    d = 1 / d;
    const Real del = d * c;
    h *= del;
    if (fabsq(del - 1) <= eps) break;
  }
  return exp(-z + a * logq(z)) * h;
}
}  // namespace

Real erf(const Real& x) {
  if (x < 0) throw std::domain_error("hp::erf: negative argument unsupported");
  return x < 2 ? erf_series(x) : 1 - erfc(x);
}

Real erfc(const Real& x) {
  if (x < 0) throw std::domain_error("hp::erfc: negative argument unsupported");
  return x < 2 ? 1 - erf_series(x) : upper_gamma_cf(Real(0.5), x * x) / sqrt_pi();
}

Real upper_gamma_half(int k, const Real& x) {  // highprec.cpp:133-151
  if (k < 0) throw std::domain_error("hp::upper_gamma_half: k must be non-negative");
  if (x < 0) throw std::domain_error("hp::upper_gamma_half: x must be non-negative");
  if (x == 0) return gamma_half(k);
  Real g = sqrt_pi() * erfc(sqrtq(x));
  if (k == 0) return g;
  const Real e = exp(-x);
  Real xpow = sqrtq(x);
  for (int j = 0; j < k; ++j) {
    g = (Real(j) + Real(0.5)) * g + xpow * e;
    xpow *= x;
  }
  return g;
}
}  // namespace hp

using hp::Real;

// ------------------------------------------------------------ reference --
Real boys_reference(int k, const Real& x, const ReferenceConfig& cfg) {  // reference.cpp:10-23
  if (k < 0) throw std::domain_error("boys_reference: k must be non-negative");
  if (x < 0) throw std::domain_error("boys_reference: x must be non-negative");
  if (cfg.truncation_terms < 1) throw std::invalid_argument("boys_reference: truncation_terms must be >= 1");
  Real term = 1 / (Real(k) + Real(0.5)), sum = term;
  for (int l = 1; l <= cfg.truncation_terms; ++l) {
    term *= x;
    term /= (Real(k + l) + Real(0.5));
    sum += term;
  }
  return hp::exp(-x) / 2 * sum;
}

std::vector<Real> boys_reference_batch(int kmax, const Real& x, const ReferenceConfig& cfg) {  // :25-35
  std::vector<Real> v(static_cast<size_t>(kmax) + 1);
  v[kmax] = boys_reference(kmax, x, cfg);
  if (kmax == 0) return v;
  const Real e = hp::exp(-x);
  for (int l = kmax - 1; l >= 0; --l) v[l] = (2 * x * v[l + 1] + e) / (2 * l + 1);
  return v;
}

Real truncation_bound(int k, const Real& x, int L) {  // reference.cpp:37-44
  if (k < 0 || L < 0) throw std::domain_error("truncation_bound: k, L must be non-negative");
  if (x < 0) throw std::domain_error("truncation_bound: x must be non-negative");
  if (x == 0) return 0;
  return powq(x, Real(k) + L + Real(1.5)) / hp::gamma_half(k + L + 1);
}

int reference_terms_for(int k, double x, double rel_target) {  // reference.cpp:46-54
  if (x <= 0) return 150;
  const double lt = std::log(rel_target);
  for (int L = 150; L <= 20000; L += 25) {
    const double s = k + L + 1.5;
    if (s * std::log(x) - std::lgamma(s) <= lt) return L;
  }
  throw std::runtime_error("reference_terms_for: no L below cap reaches target");
}

// ----------------------------------------------------------- polynomial --
Real poly_eval(const Poly& p, const Real& x) {  // polynomial.cpp:9-14
  if (p.empty()) return 0;
  Real acc = p.back();
  for (auto it = p.rbegin() + 1; it != p.rend(); ++it) acc = acc * x + *it;
  return acc;
}

Poly poly_derivative(const Poly& p) {
  if (p.size() <= 1) return Poly{Real(0)};
  Poly d(p.size() - 1);
  for (size_t i = 1; i < p.size(); ++i) d[i - 1] = Real(static_cast<double>(i)) * p[i];
  return d;
}

Poly poly_trim(const Poly& p, const Real& rel_tol) {  // polynomial.cpp:23-32
  Real maxc = 0;
  for (const auto& c : p) maxc = std::max(maxc, fabsq(c));
  if (maxc == 0) return Poly{Real(0)};
  const Real cut = maxc * rel_tol;
  size_t n = p.size();
  while (n > 1 && fabsq(p[n - 1]) <= cut) --n;
  return Poly(p.begin(), p.begin() + static_cast<long>(n));
}

int poly_degree(const Poly& p) {
  for (size_t i = p.size(); i-- > 0;)
    if (p[i] != 0) return static_cast<int>(i);
  return 0;
}

namespace {
Poly poly_rem(Poly u, const Poly& v) {  // polynomial.cpp:43-62
  const int dv = static_cast<int>(v.size()) - 1;
  while (static_cast<int>(u.size()) - 1 >= dv && !(u.size() == 1 && u[0] == 0)) {
    const int du = static_cast<int>(u.size()) - 1;
    const Real q = u.back() / v.back();
    for (int i = 0; i <= dv; ++i) u[du - dv + i] -= q * v[i];
    u.pop_back();
    while (u.size() > 1 && u.back() == 0) u.pop_back();
    Real maxc = 0;
    for (const auto& c : u) maxc = std::max(maxc, fabsq(c));
    if (maxc == 0) return Poly{Real(0)};
  }
  return u;
}

void normalize_scale(Poly& p) {
  Real maxc = 0;
  for (const auto& c : p) maxc = std::max(maxc, fabsq(c));
  if (maxc == 0) return;
  for (auto& c : p) c /= maxc;
}

int sign_variations(const std::vector<Poly>& chain, const Real& x, const Real& tiny) {
  int count = 0, prev = 0;
  for (const auto& q : chain) {
    const Real v = poly_eval(q, x);
    const int s = v > tiny ? 1 : (v < -tiny ? -1 : 0);
    if (s == 0) continue;
    if (prev != 0 && s != prev) ++count;
    prev = s;
  }
  return count;
}
}  // namespace

int sturm_root_count(const Poly& p, const Real& a, const Real& b) {  // polynomial.cpp:88-115
  if (a > b) throw std::invalid_argument("sturm_root_count: a > b");
  const int d = hp::working_digits() + hp::kGuardDigits10;
  const Real trim_tol = hp::pow10(-(d - 6));
  Poly p0 = poly_trim(p, trim_tol);
  if (p0.size() == 1 && p0[0] == 0) throw std::invalid_argument("sturm_root_count: zero polynomial");
  if (p0.size() == 1) return 0;
  std::vector<Poly> chain;
  normalize_scale(p0);
  chain.push_back(p0);
  Poly p1 = poly_derivative(p0);
  normalize_scale(p1);
  chain.push_back(p1);
  while (chain.back().size() > 1) {
    Poly r = poly_trim(poly_rem(chain[chain.size() - 2], chain.back()), trim_tol);
    if (r.size() == 1 && r[0] == 0) break;
    for (auto& c : r) c = -c;
    normalize_scale(r);
    chain.push_back(std::move(r));
  }
  const Real tiny = hp::pow10(-(d - 8));
  return sign_variations(chain, a, tiny) - sign_variations(chain, b, tiny);
}

Poly newton_interpolate(const std::vector<Real>& xs, const std::vector<Real>& ys) {  // :117-141
  const size_t n = xs.size();
  if (n == 0 || ys.size() != n) throw std::invalid_argument("newton_interpolate: size mismatch");
  std::vector<Real> c = ys;
  for (size_t j = 1; j < n; ++j)
    for (size_t i = n - 1; i >= j; --i) {
      c[i] = (c[i] - c[i - 1]) / (xs[i] - xs[i - j]);
      if (i == j) break;
    }
  Poly result{c[0]}, basis{Real(1)};
  for (size_t i = 1; i < n; ++i) {
    Poly next(basis.size() + 1, Real(0));
    for (size_t j = 0; j < basis.size(); ++j) {
      next[j + 1] += basis[j];
      next[j] -= basis[j] * xs[i - 1];
    }
    basis = std::move(next);
    if (result.size() < basis.size()) result.resize(basis.size(), Real(0));
    for (size_t j = 0; j < basis.size(); ++j) result[j] += c[i] * basis[j];
  }
  return result;
}

std::vector<int> leja_order(const std::vector<Real>& xs) {  // polynomial.cpp:143-164
  const int n = static_cast<int>(xs.size());
  std::vector<int> order;
  std::vector<bool> used(n, false);
  int first = 0;
  for (int i = 1; i < n; ++i)
    if (fabsq(xs[i]) > fabsq(xs[first])) first = i;
  order.push_back(first);
  used[first] = true;
  std::vector<Real> logdist(n, Real(0));
  for (int step = 1; step < n; ++step) {
    int best = -1;
    for (int i = 0; i < n; ++i) {
      if (used[i]) continue;
      logdist[i] += logq(fabsq(xs[i] - xs[order.back()]));
      if (best < 0 || logdist[i] > logdist[best]) best = i;
    }
    order.push_back(best);
    used[best] = true;
  }
  return order;
}

// --------------------------------------------------------------- linalg --
SymmetricEigenResult jacobi_eigensolve(std::vector<std::vector<Real>> a, int max_sweeps) {  // linalg.cpp:9-71
  const int d = static_cast<int>(a.size());
  for (const auto& row : a)
    if (static_cast<int>(row.size()) != d) throw std::invalid_argument("jacobi_eigensolve: matrix not square");
  std::vector<std::vector<Real>> v(d, std::vector<Real>(d, Real(0)));
  for (int i = 0; i < d; ++i) v[i][i] = 1;
  Real norm = 0;
  for (int i = 0; i < d; ++i)
    for (int j = 0; j < d; ++j) norm += a[i][j] * a[i][j];
  norm = sqrtq(norm);
  const Real stop = norm * hp::pow10(-(hp::working_digits() + hp::kGuardDigits10 - 4));
  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    Real off = 0;
    for (int p = 0; p < d; ++p)
      for (int q = p + 1; q < d; ++q) off += a[p][q] * a[p][q];
    if (sqrtq(2 * off) <= stop) break;
    for (int p = 0; p < d; ++p)
      for (int q = p + 1; q < d; ++q) {
        if (fabsq(a[p][q]) <= stop / (d * d)) continue;
        const Real theta = (a[q][q] - a[p][p]) / (2 * a[p][q]);
        Real t = 1 / (fabsq(theta) + sqrtq(theta * theta + 1));
        if (theta < 0) t = -t;
        const Real c = 1 / sqrtq(t * t + 1), s = t * c, tau = s / (1 + c);
        const Real apq = a[p][q];
        a[p][p] -= t * apq;
        a[q][q] += t * apq;
        a[p][q] = a[q][p] = 0;
        for (int i = 0; i < d; ++i) {
          if (i != p && i != q) {
            const Real aip = a[i][p], aiq = a[i][q];
            a[i][p] = a[p][i] = aip - s * (aiq + tau * aip);
            a[i][q] = a[q][i] = aiq + s * (aip - tau * aiq);
          }
          const Real vip = v[i][p], viq = v[i][q];
          v[i][p] = vip - s * (viq + tau * vip);
          v[i][q] = viq + s * (vip - tau * viq);
        }
      }
  }
  SymmetricEigenResult r;
  r.values.resize(d);
  r.vectors.assign(d, std::vector<Real>(d));
  for (int j = 0; j < d; ++j) {
    r.values[j] = a[j][j];
    for (int i = 0; i < d; ++i) r.vectors[j][i] = v[i][j];
  }
  return r;
}

// -------------------------------------------------------------- regions --
Real compute_x0(int k_max) {  // regions.cpp:10-17
  if (k_max < 1) throw std::domain_error("compute_x0: k_max must be >= 1");
  const Real prod = hp::gamma_half(k_max) / hp::sqrt_pi();
  Real x0 = powq(prod, Real(1) / k_max);
  return x0 < 1 ? Real(1) : x0;
}

namespace {
Real asymptotic_error(int k_max, const Real& x) {
  return hp::upper_gamma_half(k_max, x) / (2 * powq(x, Real(k_max) + Real(0.5)));
}
}  // namespace

Real compute_x1(int k_max, const Real& eps_tol) {  // regions.cpp:28-72
  if (k_max < 0) throw std::domain_error("compute_x1: k_max must be non-negative");
  if (!(eps_tol > 0 && eps_tol < 1)) throw std::domain_error("compute_x1: eps_tol must lie in (0, 1)");
  std::ostringstream trace;
  const Real s = Real(k_max) + Real(0.5);
  Real hi = Real(k_max) + 35, lo = hi;
  if (asymptotic_error(k_max, hi) > eps_tol) {
    while (asymptotic_error(k_max, hi) > eps_tol) {
      lo = hi;
      hi *= 2;
      if (hi > Real(k_max) + 100000) throw std::runtime_error("compute_x1: failed to bracket root (right)");
    }
  } else {
    while (asymptotic_error(k_max, lo) <= eps_tol) {
      hi = lo;
      lo *= Real(0.5);
      if (lo < Real(1) / 1048576) throw std::runtime_error("compute_x1: failed to bracket root (left)");
    }
  }
  Real x = (lo + hi) / 2;
  // residual target eps*1e-21 as in the reference, floored at the binary128
  // resolution of the residual itself
  const Real tol = std::max(eps_tol * hp::pow10(-21), eps_tol * hp::pow10(-(hp::working_digits() + 8)));
  for (int iter = 0; iter < 500; ++iter) {
    const Real err = asymptotic_error(k_max, x), h = err - eps_tol;
    trace << "iter " << iter << " x=" << static_cast<double>(x) << " h/eps=" << static_cast<double>(h / eps_tol) << "\n";
    if (fabsq(h) <= tol) return x;
    if (h > 0)
      lo = x;
    else
      hi = x;
    const Real hprime = -hp::exp(-x) / (2 * x) - s * err / x;
    Real next = x - h / hprime;
    if (!(next > lo && next < hi)) next = (lo + hi) / 2;
    if (next == x) return x;  // converged to the last representable step
    x = next;
  }
  throw std::runtime_error("compute_x1: Newton did not converge; trace:\n" + trace.str());
}

Real weight_rho_A(int k, const Real& x) {  // regions.cpp:74-85
  if (k < 0) throw std::domain_error("weight_rho_A: k must be non-negative");
  if (x < 0) throw std::domain_error("weight_rho_A: x must be non-negative");
  Real prod = 1, best = 1;
  for (int l = k - 1; l >= 0; --l) {
    prod *= x;
    prod /= (Real(l) + Real(0.5));
    if (prod > best) best = prod;
  }
  return best;
}

RegionPartition make_partition(int k_max, double eps_tol) {
  RegionPartition p;
  p.k_max = k_max;
  p.eps_tol = eps_tol;
  p.x0 = static_cast<double>(compute_x0(k_max));
  p.x1 = static_cast<double>(compute_x1(k_max, Real(eps_tol)));
  return p;
}

}  // namespace boysfn
