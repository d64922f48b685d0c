// gen_main.cpp -- `boysfn_gen`, the native table generator (SPEC.md:464-480:
// the `regions` and `gen` subcommands the reference specifies but does not
// ship), on the binary128 restatement of the reference's generator library
// with the extremum scan on the B200.
//
//   boysfn_gen regions --kmax 32 --eps 5e-14
//   boysfn_gen gen --kmax 32 --eps 5e-14 --out tables.txt [--workers 16] [--mp] [--max-degree 24]
//   boysfn_gen remez --region A|B --k 12 --n 8 --m 9 [--mp]
//   boysfn_gen selftest
//
// Exit codes: 0 success, 1 input error, 2 verification failure,
// 3 internal non-convergence.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "boysfn/reference.hpp"
#include "boysfn/regions.hpp"
#include "boysfn/remez.hpp"
#include "boysfn/tables.hpp"
#include "boysfn/verify.hpp"

using boysfn::hp::Real;

namespace {

std::map<std::string, std::string> parse_flags(int argc, char** argv, int first) {
  std::map<std::string, std::string> f;
  for (int i = first; i < argc; ++i) {
    std::string a = argv[i];
    if (a.rfind("--", 0) != 0) throw std::invalid_argument("unexpected argument " + a);
    if (i + 1 < argc && std::string(argv[i + 1]).rfind("--", 0) != 0)
      f[a.substr(2)] = argv[++i];
    else
      f[a.substr(2)] = "1";
  }
  return f;
}

boysfn::RealFn boys_target(int k) {
  return [k](const Real& x) {
    const double xd = static_cast<double>(x);
    boysfn::ReferenceConfig cfg;
    cfg.truncation_terms = xd > 0 ? boysfn::reference_terms_for(k, xd, 1e-36) : 150;
    return boysfn::boys_reference(k, x, cfg);
  };
}

boysfn::RealFn rho_A(int k) {
  return [k](const Real& x) { return boysfn::weight_rho_A(k, x); };
}

boysfn::RationalApproximant to_double(const boysfn::RationalHP& r) {
  boysfn::RationalApproximant a;
  for (const auto& c : r.numer) a.numer.push_back(static_cast<double>(c));
  for (const auto& c : r.denom) a.denom.push_back(static_cast<double>(c));
  a.denom.back() = 1.0;
  return a;
}

struct TableJob {
  std::string name;
  int k = 0;
  bool region_b = false;
  boysfn::WalshResult res;
  double seconds = 0;
};

void run_job(TableJob& j, const Real& a, const Real& b, const Real& eps, int max_degree, bool gpu) {
  const auto t0 = std::chrono::steady_clock::now();
  boysfn::WalshOptions opt;
  if (gpu) opt.scan = boysfn::ScanTarget{j.k, j.region_b ? 0 : 1};
  j.res = boysfn::walsh_search(boys_target(j.k), j.region_b ? boysfn::RealFn() : rho_A(j.k), a, b, eps,
                               max_degree, opt);
  j.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

int cmd_regions(const std::map<std::string, std::string>& f) {
  const int kmax = std::stoi(f.at("kmax"));
  const double eps = std::stod(f.at("eps"));
  std::printf("x0=%.17g x1=%.17g\n", static_cast<double>(boysfn::compute_x0(kmax)),
              static_cast<double>(boysfn::compute_x1(kmax, Real(eps))));
  return 0;
}

int cmd_remez(const std::map<std::string, std::string>& f) {
  const int kmax = f.count("kmax") ? std::stoi(f.at("kmax")) : 32;
  const double eps = f.count("eps") ? std::stod(f.at("eps")) : 5e-14;
  const bool region_b = f.at("region") == "B";
  const int k = region_b ? 0 : std::stoi(f.at("k"));
  const Real x0 = boysfn::compute_x0(kmax), x1 = boysfn::compute_x1(kmax, Real(eps));
  boysfn::RemezProblem p;
  p.f = boys_target(k);
  if (!region_b) p.rho = rho_A(k);
  p.a = region_b ? x0 : Real(0);
  p.b = region_b ? x1 : x0;
  p.n = std::stoi(f.at("n"));
  p.m = std::stoi(f.at("m"));
  p.eps_conv = Real(eps) / 100;
  if (!f.count("mp")) p.scan = boysfn::ScanTarget{k, region_b ? 0 : 1};
  const auto t0 = std::chrono::steady_clock::now();
  const auto r = boysfn::remez_solve(p);
  const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  std::printf("status=%d iterations=%d reguesses=%d alternation=%d sup=%.6e seconds=%.2f\n",
              static_cast<int>(r.status), r.iterations, r.reguesses, r.alternation_count,
              static_cast<double>(r.sup_error), s);
  if (r.status == boysfn::RemezStatus::Converged) {
    for (const auto& c : r.approximant.numer) std::printf("numer %.17e\n", static_cast<double>(c));
    for (const auto& c : r.approximant.denom) std::printf("denom %.17e\n", static_cast<double>(c));
  }
  return r.status == boysfn::RemezStatus::Converged ? 0 : 3;
}

int cmd_gen(const std::map<std::string, std::string>& f) {
  const int kmax = std::stoi(f.at("kmax"));
  const double eps = std::stod(f.at("eps"));
  const std::string out = f.at("out");
  const int workers = f.count("workers") ? std::stoi(f.at("workers")) : 1;
  const int max_degree = f.count("max-degree") ? std::stoi(f.at("max-degree")) : 24;
  const bool gpu = !f.count("mp");
  const int vsamples = f.count("verify-samples") ? std::stoi(f.at("verify-samples")) : 10000;
  const Real x0 = boysfn::compute_x0(kmax), x1 = boysfn::compute_x1(kmax, Real(eps));
  std::vector<TableJob> jobs(kmax + 2);
  jobs[0].name = "B";
  jobs[0].region_b = true;
  for (int k = 0; k <= kmax; ++k) {
    jobs[k + 1].name = "A[" + std::to_string(k) + "]";
    jobs[k + 1].k = k;
  }
  // largest orders first: their searches are the longest
  std::vector<int> order(jobs.size());
  for (size_t i = 0; i < order.size(); ++i) order[i] = static_cast<int>(i);
  std::sort(order.begin() + 1, order.end(), [](int u, int v) { return u > v; });
  std::atomic<size_t> next{0};
  std::mutex io;
  std::vector<std::string> errors;
  auto worker = [&] {
    for (size_t i = next.fetch_add(1); i < order.size(); i = next.fetch_add(1)) {
      TableJob& j = jobs[order[i]];
      try {
        run_job(j, j.region_b ? x0 : Real(0), j.region_b ? x1 : x0, Real(eps), max_degree, gpu);
      } catch (const std::exception& e) {
        std::lock_guard<std::mutex> lk(io);
        errors.push_back(j.name + ": " + e.what());
      }
    }
  };
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> pool;
  for (int t = 1; t < workers; ++t) pool.emplace_back(worker);
  worker();
  for (auto& t : pool) t.join();
  const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  for (const auto& e : errors) std::fprintf(stderr, "error: %s\n", e.c_str());
  if (!errors.empty()) return 3;
  bool met = true;
  for (const auto& j : jobs) {
    std::printf("%-6s n=%2d m=%2d sup=%.4e met=%d cells=%3zu %7.1fs\n", j.name.c_str(), j.res.n, j.res.m,
                static_cast<double>(j.res.sup_error), j.res.met_tolerance ? 1 : 0, j.res.cells.size(), j.seconds);
    met = met && j.res.met_tolerance;
  }
  std::printf("generated in %.1f s\n", secs);
  if (!met) return 3;
  boysfn::CoefficientTableSet set;
  set.x0 = static_cast<double>(x0);
  set.x1 = static_cast<double>(x1);
  set.k_max = kmax;
  set.eps_tol = eps;
  set.r_B = to_double(jobs[0].res.approximant);
  for (int k = 0; k <= kmax; ++k) set.r_A.push_back(to_double(jobs[k + 1].res.approximant));
  // self-certification (SPEC.md: gen output passes verify before gen reports
  // success); runner-up cells of an order's winning anti-diagonal on a miss
  std::vector<size_t> tried(kmax + 1, 0);
  for (;;) {
    const auto rep = boysfn::verify_tables(set, vsamples, 200.0, 1);
    std::printf("verify_tables: max_err %.4e at k=%d region %c\n", rep.max_err, rep.worst_k, rep.worst_region);
    if (rep.max_err <= eps) break;
    bool swapped = false;
    for (const auto& e : rep.per_k) {
      if (e.max_err_a <= eps) continue;
      const auto& alts = jobs[e.k + 1].res.alternatives;
      if (tried[e.k] + 1 < alts.size()) {
        ++tried[e.k];
        const auto& alt = alts[tried[e.k]];
        set.r_A[e.k] = to_double(alt.approximant);
        std::printf("certify: r_A[%d] -> (%d,%d) sup %.3e\n", e.k, alt.n, alt.m, static_cast<double>(alt.sup_error));
        swapped = true;
      }
    }
    if (!swapped) return 2;
  }
  std::ofstream(out) << boysfn::emit_tables(set);
  return 0;
}

int cmd_selftest() {
  int fails = 0;
  auto check = [&](bool ok, const char* what) {
    std::printf("%s %s\n", ok ? "ok  " : "FAIL", what);
    fails += ok ? 0 : 1;
  };
  char buf[64];
  std::snprintf(buf, sizeof buf, "%.17g", static_cast<double>(boysfn::compute_x0(32)));
  check(std::string(buf) == "11.899848152108484", "compute_x0(32) = 11.899848152108484");
  check(static_cast<double>(boysfn::compute_x1(32, Real(5e-14))) == 28.989337738820740,
        "compute_x1(32, 5e-14) = 28.989337738820740");
  check(boysfn::weight_rho_A(2, Real(3)) == 12, "weight_rho_A(2, 3) = 12");
  boysfn::RemezProblem p;
  p.f = [](const Real& x) { return x * x; };
  p.n = 1;
  p.m = 0;
  p.eps_conv = Real(1e-25);
  const auto r = boysfn::remez_solve(p);
  check(r.status == boysfn::RemezStatus::Converged && fabsq(r.sup_error - Real(0.125)) < Real(1e-12) &&
            r.alternation_count == 3,
        "remez x^2 by (1,0) on [0,1]: sup 1/8 +- 1e-12 (SPEC acceptance 6), 3 alternation nodes");
  check(boysfn::sturm_root_count({Real(-1), Real(0), Real(1)}, Real(0), Real(2)) == 1, "sturm x^2-1 on (0,2]");
  std::mt19937_64 g(5489);
  for (int i = 0; i < 9999; ++i) g();
  check(g() == 9981545732273789042ull, "std::mt19937_64 10000th output");
  return fails ? 1 : 0;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: boysfn_gen regions|gen|remez|selftest [--flags]\n");
    return 1;
  }
  const std::string cmd = argv[1];
  try {
    const auto f = parse_flags(argc, argv, 2);
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
