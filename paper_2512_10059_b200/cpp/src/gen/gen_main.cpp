// gen_main.cpp -- `boysfn_gen`, the native table generator: the `regions` and
// `gen` subcommands SPEC.md:464-480 specifies (the reference ships no CLI),
// plus `remez` (one cell) and `selftest`.
//
//   boysfn_gen regions --kmax 32 --eps 5e-14
//   boysfn_gen gen --kmax 32 --eps 5e-14 --out tables.txt [--workers 16] [--mp] [--max-degree 24]
//   boysfn_gen remez --region A|B [--k 12] --n 8 --m 9 [--mp]
//   boysfn_gen selftest
//
// Exit codes: 0 success, 1 input error, 2 verification failure,
// 3 internal non-convergence.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <fstream>
#include <map>
#include <mutex>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "boysfn/tables.hpp"
#include "boysfn/verify.hpp"
#include "boysfn_gen/minimax.hpp"

namespace g = boysfn::gen;
using g::real;

namespace {

std::map<std::string, std::string> flags(int argc, char** argv) {
  std::map<std::string, std::string> f;
  for (int i = 2; i < argc; ++i) {
    const std::string a = argv[i];
    if (a.rfind("--", 0) != 0) throw std::invalid_argument("unexpected argument " + a);
    const bool has_value = i + 1 < argc && std::string(argv[i + 1]).rfind("--", 0) != 0;
    f[a.substr(2)] = has_value ? argv[++i] : "1";
  }
  return f;
}

double seconds_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// F_k (series long enough for 1e-36 relative) with weight 1 (region B) or
// rho_A,k (region A); named for the GPU scan
g::Target boys_target(int k, bool region_a) {
  g::Target t;
  t.f = [k](real x) {
    const double xd = static_cast<double>(x);
    return g::boys_series(k, x, xd > 0 ? g::series_terms(k, xd, 1e-36) : 150);
  };
  if (region_a) t.w = [k](real x) { return g::recurrence_weight(k, x); };
  t.boys_k = k;
  t.weight_kind = region_a ? 1 : 0;
  return t;
}

boysfn::RationalApproximant to_table(const g::Rational& r) {
  boysfn::RationalApproximant a;
  for (real c : r.num) a.numer.push_back(static_cast<double>(c));
  for (real c : r.den) a.denom.push_back(static_cast<double>(c));
  a.denom.back() = 1.0;
  return a;
}

int cmd_regions(const std::map<std::string, std::string>& f) {
  const g::Partition p = g::partition(std::stoi(f.at("kmax")), real(std::stod(f.at("eps"))));
  std::printf("x0=%.17g x1=%.17g\n", static_cast<double>(p.x0), static_cast<double>(p.x1));
  return 0;
}

int cmd_remez(const std::map<std::string, std::string>& f) {
  const int kmax = f.count("kmax") ? std::stoi(f.at("kmax")) : 32;
  const double eps = f.count("eps") ? std::stod(f.at("eps")) : 5e-14;
  const bool region_a = f.at("region") == "A";
  const int k = region_a ? std::stoi(f.at("k")) : 0;
  const g::Partition p = g::partition(kmax, real(eps));
  g::FitOptions o;
  o.n = std::stoi(f.at("n"));
  o.m = std::stoi(f.at("m"));
  o.conv = real(eps) / 100;
  o.gpu = !f.count("mp");
  const auto t0 = std::chrono::steady_clock::now();
  const g::Fit r = g::fit(boys_target(k, region_a), region_a ? real(0) : p.x0, region_a ? p.x0 : p.x1, o);
  std::printf("status=%d iterations=%d reguesses=%d alternation=%zu sup=%.6e seconds=%.2f\n",
              static_cast<int>(r.outcome), r.iterations, r.restarts,
              r.outcome == g::Outcome::converged ? r.alternants.size() : size_t(0), static_cast<double>(r.sup),
              seconds_since(t0));
  if (r.outcome != g::Outcome::converged) return 3;
  for (real c : r.r.num) std::printf("numer %.17e\n", static_cast<double>(c));
  for (real c : r.r.den) std::printf("denom %.17e\n", static_cast<double>(c));
  return 0;
}

struct Job {
  std::string name;
  int k = 0;
  bool region_a = false;
  g::DegreeChoice choice;
  double seconds = 0;
};

int cmd_gen(const std::map<std::string, std::string>& f) {
  const int kmax = std::stoi(f.at("kmax"));
  const double eps = std::stod(f.at("eps"));
  const std::string out = f.at("out");
  const int workers = f.count("workers") ? std::max(1, std::stoi(f.at("workers"))) : 1;
  const int max_degree = f.count("max-degree") ? std::stoi(f.at("max-degree")) : 24;
  const int vsamples = f.count("verify-samples") ? std::stoi(f.at("verify-samples")) : 10000;
  const bool gpu = !f.count("mp");
  const g::Partition part = g::partition(kmax, real(eps));

  std::vector<Job> jobs(kmax + 2);
  jobs[0].name = "B";
  for (int k = 0; k <= kmax; ++k) jobs[k + 1] = Job{"A[" + std::to_string(k) + "]", k, true, {}, 0};
  // the longest searches (high orders) first
  std::vector<size_t> order{0};
  for (int k = kmax; k >= 0; --k) order.push_back(static_cast<size_t>(k) + 1);
  std::atomic<size_t> next{0};
  std::mutex mu;
  std::vector<std::string> errors;
  auto work = [&] {
    for (size_t i = next++; i < order.size(); i = next++) {
      Job& j = jobs[order[i]];
      const auto t0 = std::chrono::steady_clock::now();
      try {
        j.choice = g::choose_degrees(boys_target(j.k, j.region_a), j.region_a ? real(0) : part.x0,
                                     j.region_a ? part.x0 : part.x1, real(eps), max_degree, 1, gpu);
      } catch (const std::exception& e) {
        std::lock_guard<std::mutex> lk(mu);
        errors.push_back(j.name + ": " + e.what());
      }
      j.seconds = seconds_since(t0);
    }
  };
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> pool;
  for (int i = 1; i < workers; ++i) pool.emplace_back(work);
  work();
  for (auto& th : pool) th.join();
  for (const auto& e : errors) std::fprintf(stderr, "error: %s\n", e.c_str());
  if (!errors.empty()) return 3;
  bool all = true;
  for (const Job& j : jobs) {
    std::printf("%-6s n=%2d m=%2d sup=%.4e met=%d cells=%3d %7.1fs\n", j.name.c_str(), j.choice.n, j.choice.m,
                static_cast<double>(j.choice.sup), j.choice.ok ? 1 : 0, j.choice.cells, j.seconds);
    all = all && j.choice.ok;
  }
  std::printf("generated in %.1f s\n", seconds_since(t0));
  if (!all) return 3;

  boysfn::CoefficientTableSet set;
  set.x0 = static_cast<double>(part.x0);
  set.x1 = static_cast<double>(part.x1);
  set.k_max = kmax;
  set.eps_tol = eps;
  set.r_B = to_table(jobs[0].choice.r);
  for (int k = 0; k <= kmax; ++k) set.r_A.push_back(to_table(jobs[k + 1].choice.r));
  // certify on the GPU before writing (SPEC.md: gen output passes verify);
  // an order that misses gets the next cell of its winning anti-diagonal
  std::vector<size_t> used(kmax + 1, 0);
  for (;;) {
    const boysfn::VerifyReport rep = boysfn::verify_tables(set, vsamples, 200.0, 1);
    std::printf("verify_tables: max_err %.4e at k=%d region %c\n", rep.max_err, rep.worst_k, rep.worst_region);
    if (rep.max_err <= eps) break;
    bool changed = false;
    for (const auto& e : rep.per_k) {
      const auto& alts = jobs[e.k + 1].choice.runners_up;
      if (e.max_err_a <= eps || used[e.k] + 1 >= alts.size()) continue;
      const auto& [n, m, sup, r] = alts[++used[e.k]];
      set.r_A[e.k] = to_table(r);
      std::printf("certify: r_A[%d] -> (%d,%d) sup %.3e\n", e.k, n, m, static_cast<double>(sup));
      changed = true;
    }
    if (!changed) return 2;
  }
  std::ofstream(out) << boysfn::emit_tables(set);
  return 0;
}

int cmd_selftest() {
  int failures = 0;
  auto check = [&](bool ok, const char* what) {
    std::printf("%s %s\n", ok ? "ok  " : "FAIL", what);
    failures += !ok;
  };
  const g::Partition p = g::partition(32, real(5e-14));
  char buf[64];
  std::snprintf(buf, sizeof buf, "%.17g", static_cast<double>(p.x0));
  check(std::string(buf) == "11.899848152108484", "x0(32) = 11.899848152108484");
  check(static_cast<double>(p.x1) == 28.989337738820740, "x1(32, 5e-14) = 28.989337738820740");
  check(g::partition(1, real(1e-8)).x0 == 1 && g::partition(2, real(1e-8)).x0 == 1, "x0(1) = x0(2) = 1");
  check(g::recurrence_weight(2, real(3)) == 12, "rho_A,2(3) = 12");
  g::Target sq;
  sq.f = [](real x) { return x * x; };
  g::FitOptions o;
  o.n = 1;
  o.conv = real(1e-25);
  const g::Fit r = g::fit(sq, 0, 1, o);
  check(r.outcome == g::Outcome::converged && fabsq(r.sup - real(0.125)) < real(1e-12) && r.alternants.size() == 3,
        "x^2 by (1,0) on [0,1]: sup 1/8 +- 1e-12 (SPEC acceptance 6), 3 alternation nodes");
  bool vp = true;
  for (const auto& [E, sup] : r.history) vp = vp && E <= sup * (1 + g::ten_to(-10));
  check(vp, "|E| <= sup error at every iteration (de la Vallee-Poussin)");
  check(g::sturm_count({real(-1), real(0), real(1)}, 0, 2) == 1 && g::sturm_count({real(1), real(0), real(1)}, -10, 10) == 0,
        "Sturm counts of x^2-1 on (0,2] and x^2+1 on (-10,10]");
  std::mt19937_64 mt(5489);
  for (int i = 0; i < 9999; ++i) mt();
  check(mt() == 9981545732273789042ull, "std::mt19937_64 10000th output");
  return failures ? 1 : 0;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: boysfn_gen regions|gen|remez|selftest [--flags]\n");
    return 1;
  }
  const std::string cmd = argv[1];
  try {
    const auto f = flags(argc, argv);
    if (cmd == "regions") return cmd_regions(f);
    if (cmd == "gen") return cmd_gen(f);
    if (cmd == "remez") return cmd_remez(f);
    if (cmd == "selftest") return cmd_selftest();
    std::fprintf(stderr, "unknown command %s\n", cmd.c_str());
    return 1;
  } catch (const std::out_of_range& e) {
    std::fprintf(stderr, "error: missing flag (%s)\n", e.what());
    return 1;
  } catch (const std::invalid_argument& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 3;
  }
}
