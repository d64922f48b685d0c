// special.cpp -- binary128 numerics of the native generator: Gamma(k + 1/2)
// and the upper incomplete gamma at half-integer order, erf/erfc, the Boys
// series and its truncation bound, the region partition, polynomial helpers
// (Horner, Sturm chains, Newton interpolation, Leja order) and a cyclic
// Jacobi eigensolver.  See boysfn_gen/minimax.hpp.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <stdexcept>
#include <string>

#include "boysfn_gen/minimax.hpp"

namespace boysfn::gen {

namespace {
std::atomic<int> g_digits{22};
// 10^-(working + guard - slack): the precision-relative thresholds
real rel_tol(int slack) { return ten_to(-(digits() + kGuard - slack)); }
real half(int j) { return real(j) - real(0.5); }  // j - 1/2
}  // namespace

void set_digits(int d) {
  if (d < 16 || d > 22) throw std::invalid_argument("working digits must lie in [16, 22] for binary128");
  g_digits = d;
}
int digits() { return g_digits; }

real ten_to(int e) {
  real p = 1, base = 10;
  for (unsigned u = static_cast<unsigned>(e < 0 ? -e : e); u; u >>= 1, base *= base)
    if (u & 1) p *= base;
  return e < 0 ? 1 / p : p;
}

// ------------------------------------------------------------- gamma & erf
real gamma_half(int k) {
  if (k < 0) throw std::domain_error("gamma_half: k must be non-negative");
  real g = sqrtq(M_PIq);
  for (int j = 1; j <= k; ++j) g *= half(j);  // Gamma(s + 1) = s Gamma(s)
  return g;
}

namespace {
// erf(x) = 2/sqrt(pi) sum_j (-x^2)^j x / (j! (2j + 1)), used below x = 2
real erf_taylor(real x) {
  const real stop = rel_tol(2), x2 = x * x;
  real power = x, total = x;
  for (int j = 1; j < 100000; ++j) {
    power = -power * x2 / j;
    const real term = power / (2 * j + 1);
    total += term;
    if (fabsq(term) <= fabsq(total) * stop) break;
  }
  return 2 * total / sqrtq(M_PIq);
}

// Gamma(a, z) = e^-z z^a / (z + 1 - a - 1 (1 - a) / (z + 3 - a - ...)), modified
// Lentz (z > 0, away from the transition region)
real gamma_upper_cf(real a, real z) {
  const real stop = rel_tol(2), tiny = ten_to(-4000);
  real b = z + 1 - a, c = 1 / tiny, d = 1 / b, f = d;
  for (int i = 1; i < 100000; ++i) {
    const real an = -real(i) * (real(i) - a);
    b += 2;
    d = an * d + b;
    if (fabsq(d) < tiny) d = tiny;
    c = b + an / c;
    if (fabsq(c) < tiny) c = tiny;
    d = 1 / d;
    const real step = d * c;
    f *= step;
    if (fabsq(step - 1) <= stop) break;
  }
  return expq(a * logq(z) - z) * f;
}
}  // namespace

real erf_pos(real x) {
  if (x < 0) throw std::domain_error("erf_pos: negative argument");
  return x < 2 ? erf_taylor(x) : 1 - erfc_pos(x);
}

real erfc_pos(real x) {
  if (x < 0) throw std::domain_error("erfc_pos: negative argument");
  return x < 2 ? 1 - erf_taylor(x) : gamma_upper_cf(real(0.5), x * x) / sqrtq(M_PIq);
}

real upper_gamma_half(int k, real x) {
  if (k < 0 || x < 0) throw std::domain_error("upper_gamma_half: k and x must be non-negative");
  if (x == 0) return gamma_half(k);
  // Gamma(1/2, x) = sqrt(pi) erfc(sqrt x), then Gamma(s + 1, x) = s Gamma(s, x) + x^s e^-x
  const real rx = sqrtq(x), ex = expq(-x);
  real g = sqrtq(M_PIq) * erfc_pos(rx), xs = rx;
  for (int j = 0; j < k; ++j, xs *= x) g = (real(j) + real(0.5)) * g + xs * ex;
  return g;
}

// --------------------------------------------------------------- Boys series
real boys_series(int k, real x, int terms) {
  if (k < 0 || x < 0) throw std::domain_error("boys_series: k and x must be non-negative");
  real t = 1 / (real(k) + real(0.5)), s = t;
  for (int l = 1; l <= terms; ++l) {
    t = t * x / (real(k + l) + real(0.5));
    s += t;
  }
  return expq(-x) / 2 * s;
}

int series_terms(int k, double x, double rel) {
  if (x <= 0) return 150;
  for (int L = 150; L <= 20000; L += 25) {
    const double s = k + L + 1.5;
    if (s * std::log(x) - std::lgamma(s) <= std::log(rel)) return L;
  }
  throw std::runtime_error("series_terms: no truncation length reaches the target");
}

real series_bound(int k, real x, int terms) {
  return x == 0 ? real(0) : powq(x, real(k + terms) + real(1.5)) / gamma_half(k + terms + 1);
}

real recurrence_weight(int k, real x) {
  // largest amplification of a seed error at order k down to order l
  real amp = 1, worst = 1;
  for (int l = k - 1; l >= 0; --l) {
    amp = amp * x / (real(l) + real(0.5));
    worst = std::max(worst, amp);
  }
  return worst;
}

// ------------------------------------------------------------------ regions
Partition partition(int k_max, real eps) {
  if (k_max < 1) throw std::domain_error("partition: k_max must be >= 1");
  if (!(eps > 0 && eps < 1)) throw std::domain_error("partition: eps_tol must lie in (0, 1)");
  Partition p;
  // x0: geometric mean of (k + 1/2), k < k_max, at least 1
  p.x0 = std::max(real(1), powq(gamma_half(k_max) / sqrtq(M_PIq), real(1) / k_max));
  // x1: Gamma(s, x)/(2 x^s) = eps with s = k_max + 1/2; bracket from k_max + 35
  const real s = real(k_max) + real(0.5);
  auto h = [&](real x) { return upper_gamma_half(k_max, x) / (2 * powq(x, s)) - eps; };
  real lo = real(k_max) + 35, hi = lo;
  if (h(hi) > 0) {
    while (h(hi) > 0) {
      lo = hi;
      hi *= 2;
      if (hi > real(k_max) + 100000) throw std::runtime_error("partition: x1 not bracketed (right)");
    }
  } else {
    while (h(lo) <= 0) {
      hi = lo;
      lo /= 2;
      if (lo < real(1) / 1048576) throw std::runtime_error("partition: x1 not bracketed (left)");
    }
  }
  real x = (lo + hi) / 2;
  const real goal = eps * ten_to(-21);
  for (int it = 0; it < 500; ++it) {
    const real hx = h(x), err = hx + eps;
    if (fabsq(hx) <= goal) {
      p.x1 = x;
      return p;
    }
    (hx > 0 ? lo : hi) = x;
    const real slope = -expq(-x) / (2 * x) - s * err / x;
    real next = x - hx / slope;
    if (!(next > lo && next < hi)) next = (lo + hi) / 2;
    if (next == x) break;
    x = next;
  }
  p.x1 = x;
  return p;
}

// -------------------------------------------------------------- polynomials
real horner(const rvec& c, real x) {
  real v = 0;
  for (auto it = c.rbegin(); it != c.rend(); ++it) v = v * x + *it;
  return v;
}

rvec trim_top(const rvec& c, real rel) {
  real big = 0;
  for (real v : c) big = std::max(big, fabsq(v));
  if (big == 0) return {real(0)};
  size_t len = c.size();
  while (len > 1 && fabsq(c[len - 1]) <= big * rel) --len;
  return rvec(c.begin(), c.begin() + static_cast<long>(len));
}

namespace {
void scale_unit(rvec& p) {  // divide by the largest |coefficient|
  real big = 0;
  for (real v : p) big = std::max(big, fabsq(v));
  if (big > 0)
    for (real& v : p) v /= big;
}

rvec remainder(rvec u, const rvec& v) {
  const size_t dv = v.size() - 1;
  while (u.size() - 1 >= dv && !(u.size() == 1 && u[0] == 0)) {
    const real q = u.back() / v.back();
    const size_t shift = u.size() - 1 - dv;
    for (size_t i = 0; i <= dv; ++i) u[shift + i] -= q * v[i];
    u.pop_back();
    while (u.size() > 1 && u.back() == 0) u.pop_back();
    real big = 0;
    for (real w : u) big = std::max(big, fabsq(w));
    if (big == 0) return {real(0)};
  }
  return u;
}

int sign_changes(const std::vector<rvec>& chain, real x, real zero) {
  int changes = 0, last = 0;
  for (const rvec& q : chain) {
    const real v = horner(q, x);
    const int sg = v > zero ? 1 : (v < -zero ? -1 : 0);
    if (sg != 0) {
      if (last != 0 && sg != last) ++changes;
      last = sg;
    }
  }
  return changes;
}
}  // namespace

int sturm_count(const rvec& c, real a, real b) {
  if (a > b) throw std::invalid_argument("sturm_count: a > b");
  const real cut = rel_tol(6);
  rvec p = trim_top(c, cut);
  if (p.size() == 1) {
    if (p[0] == 0) throw std::invalid_argument("sturm_count: zero polynomial");
    return 0;
  }
  std::vector<rvec> chain;
  scale_unit(p);
  chain.push_back(p);
  rvec d(p.size() - 1);
  for (size_t i = 1; i < p.size(); ++i) d[i - 1] = real(static_cast<double>(i)) * p[i];
  scale_unit(d);
  chain.push_back(d);
  while (chain.back().size() > 1) {
    rvec r = trim_top(remainder(chain[chain.size() - 2], chain.back()), cut);
    if (r.size() == 1 && r[0] == 0) break;
    for (real& v : r) v = -v;
    scale_unit(r);
    chain.push_back(std::move(r));
  }
  const real zero = rel_tol(8);
  return sign_changes(chain, a, zero) - sign_changes(chain, b, zero);
}

rvec newton_to_monomial(const rvec& xs, const rvec& ys) {
  const size_t n = xs.size();
  if (n == 0 || ys.size() != n) throw std::invalid_argument("newton_to_monomial: size mismatch");
  rvec dd = ys;  // divided differences, in place
  for (size_t order = 1; order < n; ++order)
    for (size_t i = n - 1; i >= order; --i) {
      dd[i] = (dd[i] - dd[i - 1]) / (xs[i] - xs[i - order]);
      if (i == order) break;
    }
  rvec out{dd[0]}, basis{real(1)};  // basis = prod_{j<i} (x - x_j)
  for (size_t i = 1; i < n; ++i) {
    rvec next(basis.size() + 1, real(0));
    for (size_t j = 0; j < basis.size(); ++j) {
      next[j + 1] += basis[j];
      next[j] -= basis[j] * xs[i - 1];
    }
    basis.swap(next);
    out.resize(std::max(out.size(), basis.size()), real(0));
    for (size_t j = 0; j < basis.size(); ++j) out[j] += dd[i] * basis[j];
  }
  return out;
}

std::vector<int> leja_sequence(const rvec& xs) {
  const int n = static_cast<int>(xs.size());
  std::vector<int> seq;
  std::vector<char> taken(n, 0);
  int start = 0;
  for (int i = 1; i < n; ++i)
    if (fabsq(xs[i]) > fabsq(xs[start])) start = i;
  seq.push_back(start);
  taken[start] = 1;
  rvec score(n, real(0));  // sum of log distances to the chosen points
  while (static_cast<int>(seq.size()) < n) {
    int pick = -1;
    for (int i = 0; i < n; ++i) {
      if (taken[i]) continue;
      score[i] += logq(fabsq(xs[i] - xs[seq.back()]));
      if (pick < 0 || score[i] > score[pick]) pick = i;
    }
    seq.push_back(pick);
    taken[pick] = 1;
  }
  return seq;
}

// ------------------------------------------------------------------ Jacobi
void jacobi(std::vector<rvec> a, rvec& values, std::vector<rvec>& vectors) {
  const int d = static_cast<int>(a.size());
  std::vector<rvec> v(d, rvec(d, real(0)));
  for (int i = 0; i < d; ++i) v[i][i] = 1;
  real frob = 0;
  for (const rvec& row : a)
    for (real e : row) frob += e * e;
  const real stop = sqrtq(frob) * rel_tol(4);
  for (int sweep = 0; sweep < 100; ++sweep) {
    real off = 0;
    for (int p = 0; p < d; ++p)
      for (int q = p + 1; q < d; ++q) off += a[p][q] * a[p][q];
    if (sqrtq(2 * off) <= stop) break;
    for (int p = 0; p < d; ++p)
      for (int q = p + 1; q < d; ++q) {
        const real apq = a[p][q];
        if (fabsq(apq) <= stop / (d * d)) continue;
        // rotation annihilating a[p][q]: t = tan(phi), the smaller root
        const real theta = (a[q][q] - a[p][p]) / (2 * apq);
        const real t = (theta < 0 ? -1 : 1) / (fabsq(theta) + sqrtq(theta * theta + 1));
        const real c = 1 / sqrtq(t * t + 1), s = t * c, tau = s / (1 + c);
        a[p][p] -= t * apq;
        a[q][q] += t * apq;
        a[p][q] = a[q][p] = 0;
        for (int i = 0; i < d; ++i) {
          if (i != p && i != q) {
            const real ip = a[i][p], iq = a[i][q];
            a[i][p] = a[p][i] = ip - s * (iq + tau * ip);
            a[i][q] = a[q][i] = iq + s * (ip - tau * iq);
          }
          const real vp = v[i][p], vq = v[i][q];
          v[i][p] = vp - s * (vq + tau * vp);
          v[i][q] = vq + s * (vp - tau * vq);
        }
      }
  }
  values.assign(d, real(0));
  vectors.assign(d, rvec(d, real(0)));
  for (int j = 0; j < d; ++j) {
    values[j] = a[j][j];
    for (int i = 0; i < d; ++i) vectors[j][i] = v[i][j];
  }
}

}  // namespace boysfn::gen
