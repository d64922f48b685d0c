// minimax.cpp -- the weighted rational minimax exchange of arXiv 2512.10059
// (Fig. 1: random nodes; the levelled fixed-node solve; pole-free selection by
// Sturm counts; convergence test; extremum exchange; the infeasibility abort)
// and the Walsh-table degree search, for the native generator.
//
// The fixed-node system rho (f - p/q)(x_i) = (-1)^i E is solved as the
// specified symmetric eigenproblem: q is expanded in polynomials orthonormal
// under the node weights |omega_i| / rho_i (omega the barycentric weights),
// which turns "p interpolates (f_i - (-1)^i E / rho_i) q_i with degree <= n"
// into A beta = lambda beta with E = +-lambda; p then follows by Newton
// interpolation on a Leja-ordered subset of the nodes.
//
// The error-curve extrema come from one of two scanners: the specified grid of
// 64 (n+m+2) points with golden-section refinement in binary128, or the B200
// (boysfn_gen_error_scan: the weighted error in double-double on a
// 65,536-point grid, each local maximum re-sampled on a 2,048-point zoom).
#include <algorithm>
#include <cmath>
#include <random>
#include <stdexcept>
#include <string>

#include "../../../../include/boysfn_b200.h"
#include "boysfn_gen/minimax.hpp"

namespace boysfn::gen {
namespace {

struct Peak {
  real x;
  real e;  // signed weighted error
};

int sgn(real v) { return (v > 0) - (v < 0); }

real weight_at(const Target& t, real x) { return t.w ? t.w(x) : real(1); }

// ------------------------------------------------------------ error scanning
class Scanner {
 public:
  Scanner(const Target& t, real a, real b, const FitOptions& o) : t_(t), a_(a), b_(b), o_(o) {
    if (o.gpu) {
      if (t.boys_k < 0) throw std::invalid_argument("GPU scan needs a Boys target (Target::boys_k)");
      return;
    }
    const int K = o.grid ? o.grid : 64 * (o.n + o.m + 2);
    for (int i = 0; i < K; ++i) {
      const real x = a + (b - a) * i / (K - 1);
      xs_.push_back(x);
      fw_.emplace_back(t.f(x), weight_at(t, x));
    }
  }

  real error(const Rational& r, real x) const {
    if (o_.gpu) return device({static_cast<double>(x)}, r)[0];
    return weight_at(t_, x) * (t_.f(x) - r(x));
  }

  std::vector<Peak> peaks(const Rational& r) const { return merged(o_.gpu ? device_peaks(r) : host_peaks(r)); }

 private:
  // grid local maxima of |e|, each refined by golden section on its two cells
  std::vector<Peak> host_peaks(const Rational& r) const {
    const size_t K = xs_.size();
    rvec e(K);
    for (size_t i = 0; i < K; ++i) e[i] = fw_[i].second * (fw_[i].first - r(xs_[i]));
    const real tol = (b_ - a_) * ten_to(-(digits() * 2 / 5));
    std::vector<Peak> out;
    for (size_t i = 0; i < K; ++i) {
      const real m = fabsq(e[i]);
      if ((i > 0 && m < fabsq(e[i - 1])) || (i + 1 < K && m < fabsq(e[i + 1]))) continue;
      const real lo = i ? xs_[i - 1] : a_, hi = i + 1 < K ? xs_[i + 1] : b_;
      Peak p{golden_argmax([&](real x) { return fabsq(error(r, x)); }, lo, hi, tol), 0};
      p.e = error(r, p.x);
      if (fabsq(p.e) < m) p = {xs_[i], e[i]};  // never worse than the grid point
      out.push_back(p);
    }
    return out;
  }

  static real golden_argmax(const std::function<real(real)>& g, real lo, real hi, real tol) {
    const real r5 = sqrtq(real(5)), big = (r5 - 1) / 2, small = (3 - r5) / 2;
    real w = hi - lo;
    if (w <= tol) return (lo + hi) / 2;
    real c = lo + small * w, d = lo + big * w, gc = g(c), gd = g(d);
    while (w > tol) {
      if (gc >= gd) {  // the maximum lies in [lo, d]
        hi = d;
        d = c;
        gd = gc;
        w = hi - lo;
        c = lo + small * w;
        gc = g(c);
      } else {  // in [c, hi]
        lo = c;
        c = d;
        gc = gd;
        w = hi - lo;
        d = lo + big * w;
        gd = g(d);
      }
    }
    return (lo + hi) / 2;
  }

  rvec device(const std::vector<double>& xs, const Rational& r) const {
    std::vector<double> nh, nl, dh, dl, err(xs.size());
    for (real c : r.num) {
      nh.push_back(static_cast<double>(c));
      nl.push_back(static_cast<double>(c - real(nh.back())));
    }
    for (real c : r.den) {
      dh.push_back(static_cast<double>(c));
      dl.push_back(static_cast<double>(c - real(dh.back())));
    }
    if (boysfn_gen_error_scan(t_.boys_k, nh.data(), nl.data(), static_cast<int>(nh.size()) - 1, dh.data(), dl.data(),
                              static_cast<int>(dh.size()) - 1, t_.weight_kind, xs.data(), xs.size(),
                              err.data()) != BOYSFN_OK)
      throw std::runtime_error(std::string("boysfn_gen_error_scan: ") + boysfn_last_error());
    return rvec(err.begin(), err.end());
  }

  std::vector<Peak> device_peaks(const Rational& r) const {
    const int G = o_.gpu_grid, Z = o_.gpu_zoom;
    const double a = static_cast<double>(a_), b = static_cast<double>(b_);
    std::vector<double> grid(G);
    for (int i = 0; i < G; ++i) grid[i] = i + 1 == G ? b : a + (b - a) * i / (G - 1);
    const rvec e = device(grid, r);
    std::vector<int> tops;
    for (int i = 0; i < G; ++i) {
      const real m = fabsq(e[i]);
      if ((i == 0 || m >= fabsq(e[i - 1])) && (i + 1 == G || m >= fabsq(e[i + 1]))) tops.push_back(i);
    }
    const size_t keep = static_cast<size_t>(64) * (o_.n + o_.m + 2);
    if (tops.size() > keep) {  // a flat or noise-level curve: keep the largest
      std::nth_element(tops.begin(), tops.begin() + static_cast<long>(keep), tops.end(),
                       [&](int u, int v) { return fabsq(e[u]) > fabsq(e[v]); });
      tops.resize(keep);
      std::sort(tops.begin(), tops.end());
    }
    std::vector<double> zoom;
    zoom.reserve(tops.size() * Z);
    for (int i : tops) {
      const double lo = grid[std::max(i - 1, 0)], hi = grid[std::min(i + 1, G - 1)];
      for (int j = 0; j < Z; ++j) zoom.push_back(lo + (hi - lo) * j / (Z - 1));
    }
    const rvec ez = device(zoom, r);
    std::vector<Peak> out;
    for (size_t q = 0; q < tops.size(); ++q) {
      const auto first = ez.begin() + static_cast<long>(q * Z);
      const auto best = std::max_element(first, first + Z, [](real u, real v) { return fabsq(u) < fabsq(v); });
      Peak p{real(zoom[static_cast<size_t>(best - ez.begin())]), *best};
      if (fabsq(p.e) < fabsq(e[tops[q]])) p = {real(grid[tops[q]]), e[tops[q]]};
      out.push_back(p);
    }
    return out;
  }

  // sorted by x; refinements that met on one extremum collapse to the larger
  std::vector<Peak> merged(std::vector<Peak> v) const {
    std::sort(v.begin(), v.end(), [](const Peak& u, const Peak& w) { return u.x < w.x; });
    const real near = (b_ - a_) * ten_to(-(digits() / 3));
    std::vector<Peak> out;
    for (const Peak& p : v) {
      if (!out.empty() && p.x - out.back().x < near) {
        if (fabsq(p.e) > fabsq(out.back().e)) out.back() = p;
      } else {
        out.push_back(p);
      }
    }
    return out;
  }

  const Target& t_;
  real a_, b_;
  FitOptions o_;
  rvec xs_;
  std::vector<std::pair<real, real>> fw_;  // f and w on the CPU grid
};

// --------------------------------------------------------- node exchange
struct Exchange {
  bool ok = false;
  rvec nodes;
  real sup = 0;       // over every located extremum
  real weakest = 0;   // smallest |e| among the chosen nodes
};

// N alternating extrema at or above |E| (condition i) including the global
// maximum (condition ii).
Exchange exchange_nodes(const std::vector<Peak>& peaks, int N, real level) {
  Exchange x;
  for (const Peak& p : peaks) x.sup = std::max(x.sup, fabsq(p.e));
  const real floor = level * (1 - ten_to(-10));
  std::vector<Peak> alt;  // sign-alternating, each run reduced to its largest member
  for (const Peak& p : peaks) {
    if (p.e == 0 || fabsq(p.e) < floor) continue;
    if (!alt.empty() && sgn(alt.back().e) == sgn(p.e)) {
      if (fabsq(p.e) > fabsq(alt.back().e)) alt.back() = p;
    } else {
      alt.push_back(p);
    }
  }
  if (static_cast<int>(alt.size()) < N) return x;
  while (static_cast<int>(alt.size()) > N) {
    if (static_cast<int>(alt.size()) == N + 1) {  // drop the weaker end
      if (fabsq(alt.front().e) <= fabsq(alt.back().e))
        alt.erase(alt.begin());
      else
        alt.pop_back();
      continue;
    }
    size_t top = 0;
    for (size_t i = 1; i < alt.size(); ++i)
      if (fabsq(alt[i].e) > fabsq(alt[top].e)) top = i;
    // remove the adjacent pair with the smallest larger-member, sparing the top
    size_t cut = alt.size();
    real cut_score = 0;
    for (size_t i = 0; i + 1 < alt.size(); ++i) {
      if (i == top || i + 1 == top) continue;
      const real score = std::max(fabsq(alt[i].e), fabsq(alt[i + 1].e));
      if (cut == alt.size() || score < cut_score) {
        cut = i;
        cut_score = score;
      }
    }
    if (cut == alt.size()) return x;
    alt.erase(alt.begin() + static_cast<long>(cut), alt.begin() + static_cast<long>(cut) + 2);
  }
  x.ok = true;
  x.weakest = fabsq(alt.front().e);
  for (const Peak& p : alt) {
    x.nodes.push_back(p.x);
    x.weakest = std::min(x.weakest, fabsq(p.e));
  }
  return x;
}

rvec random_nodes(real a, real b, int N, std::mt19937_64& rng) {
  const real w = b - a;
  rvec v(N);
  for (int attempt = 0; attempt < 1000; ++attempt) {
    for (real& x : v) x = a + w * real(static_cast<double>(rng() >> 11) * 0x1.0p-53);
    std::sort(v.begin(), v.end());
    bool apart = true;
    for (int i = 1; i < N && apart; ++i) apart = v[i] - v[i - 1] >= w * real(1e-12);
    if (apart) return v;
  }
  throw std::runtime_error("random_nodes: could not draw distinct nodes");
}

// ------------------------------------------------------ fixed-node solve
struct Levelled {
  Rational r;    // p, q (q not normalised)
  real E;        // signed levelled error
  real residual; // relative node residual
};

std::vector<Levelled> levelled_solutions(const rvec& x, const rvec& f, const rvec& w, int n, int m) {
  const int N = n + m + 2;
  rvec omega(N), mu(N);
  for (int i = 0; i < N; ++i) {
    real prod = 1;
    for (int j = 0; j < N; ++j)
      if (j != i) prod *= x[i] - x[j];
    if (prod == 0) return {};
    omega[i] = 1 / prod;  // barycentric weight; (-1)^i omega_i has one sign
    if (!(w[i] > 0)) throw std::invalid_argument("levelled_solutions: weight must be positive");
  }
  for (int i = 0; i < N; ++i) mu[i] = fabsq(omega[i]) / w[i];
  auto inner = [&](const rvec& u, const rvec& v) {
    real s = 0;
    for (int i = 0; i < N; ++i) s += mu[i] * u[i] * v[i];
    return s;
  };
  // phi_0..phi_m orthonormal under <.,.>_mu (three-term recurrence), kept as
  // node values and as monomial coefficients
  std::vector<rvec> at(m + 1, rvec(N)), mono(m + 1);
  {
    real s0 = 0;
    for (real v : mu) s0 += v;
    const real c0 = 1 / sqrtq(s0);
    at[0].assign(N, c0);
    mono[0] = {c0};
    real beta_prev = 0;
    for (int j = 0; j < m; ++j) {
      rvec u(N);
      for (int i = 0; i < N; ++i) u[i] = x[i] * at[j][i];
      const real alpha = inner(u, at[j]);
      for (int i = 0; i < N; ++i) {
        u[i] -= alpha * at[j][i];
        if (j > 0) u[i] -= beta_prev * at[j - 1][i];
      }
      const real beta = sqrtq(inner(u, u));
      if (beta == 0) return {};
      for (real& v : u) v /= beta;
      rvec um(mono[j].size() + 1, real(0));
      for (size_t c = 0; c < mono[j].size(); ++c) {
        um[c + 1] += mono[j][c];
        um[c] -= alpha * mono[j][c];
      }
      if (j > 0)
        for (size_t c = 0; c < mono[j - 1].size(); ++c) um[c] -= beta_prev * mono[j - 1][c];
      for (real& v : um) v /= beta;
      at[j + 1] = std::move(u);
      mono[j + 1] = std::move(um);
      beta_prev = beta;
    }
  }
  std::vector<rvec> A(m + 1, rvec(m + 1));
  for (int s = 0; s <= m; ++s)
    for (int t = s; t <= m; ++t) {
      real sum = 0;
      for (int i = 0; i < N; ++i) sum += omega[i] * f[i] * at[s][i] * at[t][i];
      A[s][t] = A[t][s] = sum;
    }
  rvec lam;
  std::vector<rvec> vec;
  jacobi(A, lam, vec);
  const real flip = (N - 1) % 2 == 0 ? 1 : -1;
  real scale = 0;
  for (int i = 0; i < N; ++i) scale = std::max(scale, fabsq(w[i] * f[i]));
  const real res_tol = ten_to(-(digits() - 8));
  const std::vector<int> order = leja_sequence(x);
  std::vector<Levelled> out;
  for (int j = 0; j <= m; ++j) {
    Levelled L;
    L.E = flip * lam[j];
    rvec qx(N, real(0));
    L.r.den.assign(static_cast<size_t>(m) + 1, real(0));
    for (int s = 0; s <= m; ++s) {
      for (int i = 0; i < N; ++i) qx[i] += vec[j][s] * at[s][i];
      for (size_t c = 0; c < mono[s].size(); ++c) L.r.den[c] += vec[j][s] * mono[s][c];
    }
    real qbig = 0;
    for (real v : qx) qbig = std::max(qbig, fabsq(v));
    if (!(qbig > 0)) continue;
    const real qzero = qbig * ten_to(-(digits() + kGuard - 6));
    if (std::any_of(qx.begin(), qx.end(), [&](real v) { return fabsq(v) <= qzero; })) continue;
    rvec px(n + 1), py(n + 1);
    for (int t = 0; t <= n; ++t) {
      const int i = order[t];
      px[t] = x[i];
      py[t] = (f[i] - (i % 2 ? -1 : 1) * L.E / w[i]) * qx[i];
    }
    L.r.num = newton_to_monomial(px, py);
    real worst = 0;
    for (int i = 0; i < N; ++i) {
      const real ri = horner(L.r.num, x[i]) / qx[i];
      worst = std::max(worst, fabsq(w[i] * (f[i] - ri) - (i % 2 ? -1 : 1) * L.E));
    }
    const real denom_scale = std::max(fabsq(L.E), scale);
    L.residual = worst / (denom_scale == 0 ? real(1) : denom_scale);
    if (L.residual <= res_tol) out.push_back(std::move(L));
  }
  return out;
}

// the candidate whose q has no root in [a, b] (best residual among several)
const Levelled* pole_free(const std::vector<Levelled>& cands, real a, real b) {
  const Levelled* pick = nullptr;
  const real cut = ten_to(-(digits() + kGuard - 8));
  for (const Levelled& c : cands) {
    const rvec q = trim_top(c.r.den, cut);
    if (q.size() == 1) {
      if (q[0] == 0) continue;
    } else {
      real big = 0;
      for (real v : q) big = std::max(big, fabsq(v));
      if (fabsq(horner(q, a)) <= big * cut) continue;  // a root at a itself
      if (sturm_count(q, a, b) != 0) continue;
    }
    if (pick == nullptr || c.residual < pick->residual) pick = &c;
  }
  return pick;
}

Rational monic(const Rational& r) {
  Rational m;
  m.den = trim_top(r.den, ten_to(-(digits() - 4)));
  const real lead = m.den.back();
  for (real& v : m.den) v /= lead;
  m.den.back() = 1;
  m.num = r.num;
  for (real& v : m.num) v /= lead;
  return m;
}

}  // namespace

Fit fit(const Target& t, real a, real b, const FitOptions& o) {
  if (!t.f) throw std::invalid_argument("fit: no target function");
  if (!(a < b)) throw std::invalid_argument("fit: need a < b");
  if (o.n < 0 || o.m < 0) throw std::invalid_argument("fit: degrees must be non-negative");
  const int N = o.n + o.m + 2;
  if (o.grid != 0 && o.grid < 4 * N) throw std::invalid_argument("fit: grid must hold at least 4 (n+m+2) points");
  Fit out;
  std::mt19937_64 rng(o.seed);
  const Scanner scan(t, a, b, o);
  rvec nodes = random_nodes(a, b, N, rng);
  auto restart = [&]() {
    if (out.restarts >= o.max_restarts) return false;
    ++out.restarts;
    nodes = random_nodes(a, b, N, rng);
    return true;
  };
  for (;;) {
    rvec f(N), w(N);
    for (int i = 0; i < N; ++i) {
      f[i] = t.f(nodes[i]);
      w[i] = weight_at(t, nodes[i]);
    }
    const std::vector<Levelled> cands = levelled_solutions(nodes, f, w, o.n, o.m);
    const Levelled* sel = pole_free(cands, a, b);
    if (sel == nullptr) {
      if (restart()) continue;
      out.outcome = Outcome::restart_limit;
      return out;
    }
    ++out.iterations;
    const real E = fabsq(sel->E);
    const Exchange ex = exchange_nodes(scan.peaks(sel->r), N, E);
    if (E > ex.sup * (1 + ten_to(-10))) throw std::logic_error("fit: |E| above the sup error (de la Vallee-Poussin)");
    out.history.emplace_back(E, ex.sup);
    if (ex.sup - E <= o.conv) {
      out.outcome = Outcome::converged;
      out.r = monic(sel->r);
      out.sup = ex.sup;
      out.level = sel->E;
      out.alternants = ex.ok ? ex.nodes : nodes;
      return out;
    }
    if (!ex.ok) {
      if (restart()) continue;
      out.outcome = Outcome::restart_limit;
      return out;
    }
    if (o.abort_level > 0 && ex.weakest > o.abort_level) {
      out.outcome = Outcome::infeasible;
      out.lower_bound = ex.weakest;
      out.sup = ex.sup;
      out.level = sel->E;
      return out;
    }
    if (out.iterations >= o.max_iterations) {
      out.outcome = Outcome::iteration_limit;
      out.sup = ex.sup;
      out.level = sel->E;
      return out;
    }
    nodes = ex.nodes;
  }
}

DegreeChoice choose_degrees(const Target& t, real a, real b, real eps, int max_degree, std::uint64_t seed, bool gpu) {
  if (!(eps > 0)) throw std::invalid_argument("choose_degrees: eps_tol must be positive");
  DegreeChoice best_any;
  for (int d = 0; d <= max_degree; ++d) {
    DegreeChoice diag;
    for (int n = 0; n <= d; ++n) {
      const int m = d - n;
      FitOptions o;
      o.n = n;
      o.m = m;
      o.conv = eps / 100;
      o.abort_level = eps;
      o.seed = seed + 0x9e3779b97f4a7c15ull * (static_cast<std::uint64_t>(n) * 64 + m + 1);
      o.gpu = gpu;
      const Fit c = fit(t, a, b, o);
      ++best_any.cells;
      if (c.outcome != Outcome::converged) continue;
      if (!best_any.ok || c.sup < best_any.sup) {  // best seen anywhere (reported if nothing meets eps)
        best_any.ok = true;
        best_any.n = n;
        best_any.m = m;
        best_any.r = c.r;
        best_any.sup = c.sup;
      }
      if (c.sup <= eps) diag.runners_up.emplace_back(n, m, c.sup, c.r);
    }
    if (!diag.runners_up.empty()) {
      std::stable_sort(diag.runners_up.begin(), diag.runners_up.end(),
                       [](const auto& u, const auto& v) { return std::get<2>(u) < std::get<2>(v); });
      std::tie(diag.n, diag.m, diag.sup, diag.r) = diag.runners_up.front();
      diag.ok = true;
      diag.cells = best_any.cells;
      return diag;
    }
  }
  best_any.ok = false;
  return best_any;
}

}  // namespace boysfn::gen
