// tests/cpp/shim_test.cpp -- exercises the drop-in C++ API (boysfn/eval.hpp,
// boysfn/tables.hpp from paper_2512_10059_b200/cpp) exactly as reference code
// would call it, linked against libboysfn_b200.so.  The checker is the CPU
// oracle (oracle/boys_port.c), linked as a separate test-only library.
//
//   shim_test parse <file>   CPU only: parse_tables + emit_tables, print
//                            "OK\n<text>" or "ERR <status>\n<message>"
//   shim_test gpu            device checks; exit 0 on success
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "boys_oracle.h"
#include "boysfn/eval.hpp"
#include "boysfn/tables.hpp"
#include "boysfn/verify.hpp"

namespace {

int failures = 0;
#define CHECK(cond, ...)                                      \
  do {                                                        \
    if (!(cond)) {                                            \
      ++failures;                                             \
      std::fprintf(stderr, "FAIL %s:%d: ", __FILE__, __LINE__); \
      std::fprintf(stderr, __VA_ARGS__);                      \
      std::fprintf(stderr, "\n");                             \
    }                                                         \
  } while (0)

int cmd_parse(const char* path) {
  std::ifstream f(path, std::ios::binary);
  std::stringstream ss;
  ss << f.rdbuf();
  try {
    const std::string out = boysfn::emit_tables(boysfn::parse_tables(ss.str()));
    std::printf("OK\n%s", out.c_str());
  } catch (const boysfn::TableParseError& e) {
    std::printf("ERR 8\n%s", e.what());
  } catch (const std::invalid_argument& e) {
    std::printf("ERR 4\n%s", e.what());
  }
  return 0;
}

// Oracle view of a boysfn::CoefficientTableSet.
struct OracleTables {
  std::vector<oracle_rational> ra;
  oracle_tables t{};
  explicit OracleTables(const boysfn::CoefficientTableSet& s) {
    auto conv = [](const boysfn::RationalApproximant& r) {
      return oracle_rational{r.degree_n(), r.degree_m(), r.numer.data(), r.denom.data()};
    };
    for (const auto& r : s.r_A) ra.push_back(conv(r));
    t = oracle_tables{s.x0, s.x1, s.k_max, s.eps_tol, conv(s.r_B), ra.data()};
  }
};

double region_c_mismatch_or_dev(const std::vector<double>& xs, int k, const std::vector<double>& got,
                                const std::vector<double>& want, double x1, bool* c_exact) {
  double dev = 0;
  *c_exact = true;
  for (size_t i = 0; i < xs.size(); ++i)
    for (int l = 0; l <= k; ++l) {
      const double a = got[i * (k + 1) + l], b = want[i * (k + 1) + l];
      if (xs[i] >= x1 && std::memcmp(&a, &b, sizeof a) != 0) *c_exact = false;
      dev = std::fmax(dev, std::fabs(a - b));
    }
  return dev;
}

int cmd_gpu() {
  const auto& T = boysfn::embedded_default();
  OracleTables O(T);
  // 1) boys_batch_many over all orders vs the reference restatement
  std::vector<double> xs(10007);
  oracle_gen_uniform(xs.data(), xs.size(), 11, 0, 0.0, 45.0);
  xs[0] = 0.0;
  xs[1] = T.x0;
  xs[2] = T.x1;
  xs[3] = std::nextafter(T.x1, 0.0);
  for (int k = 0; k <= T.k_max; ++k) {
    std::vector<double> got(xs.size() * (k + 1)), want(got.size());
    boysfn::boys_batch_many(xs, k, T, got);
    size_t bad = 0;
    CHECK(oracle_boys_batch_many(xs.data(), xs.size(), k, &O.t, want.data(), want.size(), &bad) == 0, "oracle");
    bool c_exact = false;
    const double dev = region_c_mismatch_or_dev(xs, k, got, want, T.x1, &c_exact);
    CHECK(dev <= 5e-14, "k=%d max dev %g", k, dev);
    CHECK(c_exact, "k=%d region C not bit-identical", k);
  }
  // 2) the same through a copied (non-embedded) table set
  {
    boysfn::CoefficientTableSet copy = T;
    std::vector<double> a(xs.size() * 9), b(a.size());
    boysfn::boys_batch_many(xs, 8, T, a);
    boysfn::boys_batch_many(xs, 8, copy, b);
    CHECK(std::memcmp(a.data(), b.data(), a.size() * sizeof(double)) == 0, "copied table set differs");
  }
  // 3) exceptions: types, messages, partial output
  {
    std::vector<double> out(xs.size() * 5 - 1);
    try {
      boysfn::boys_batch_many(xs, 4, T, out);
      CHECK(false, "size mismatch not thrown");
    } catch (const std::invalid_argument& e) {
      CHECK(std::string(e.what()) == "boys_batch_many: output span has wrong size", "%s", e.what());
    }
  }
  {
    std::vector<double> bx(xs.begin(), xs.begin() + 300);
    bx[123] = -2.0;
    std::vector<double> out(bx.size() * 7, -7.0), want(out.size());
    size_t fb = 0;
    oracle_boys_batch_many(bx.data(), bx.size(), 6, &O.t, want.data(), want.size(), &fb);
    try {
      boysfn::boys_batch_many(bx, 6, T, out);
      CHECK(false, "domain_error not thrown");
    } catch (const std::domain_error& e) {
      CHECK(std::string(e.what()) == "boys_batch: x must be finite and non-negative", "%s", e.what());
    }
    double dev = 0;
    for (size_t i = 0; i < 123 * 7; ++i) dev = std::fmax(dev, std::fabs(out[i] - want[i]));
    CHECK(dev <= 5e-14, "rows before the bad x: dev %g", dev);
    bool untouched = true;
    for (size_t i = 123 * 7; i < out.size(); ++i) untouched &= out[i] == -7.0;
    CHECK(untouched, "rows at/after the bad x were written");
  }
  try {
    boysfn::boys_batch(1.0, 33, T);
    CHECK(false, "out_of_range not thrown");
  } catch (const std::out_of_range& e) {
    CHECK(std::string(e.what()) == "boys_batch: k out of range for this table set", "%s", e.what());
  }
  try {
    boysfn::boys_batch(NAN, 40, T);
    CHECK(false, "domain_error not thrown");
  } catch (const std::domain_error&) {
  }
  // 4) boys_batch / boys_batch_region / classify_region
  {
    const boysfn::BoysBatch b = boysfn::boys_batch(15.0, 12, T);
    CHECK(b.values.size() == 13 && b.k == 12 && b.x == 15.0, "BoysBatch shape");
    CHECK(std::fabs(b.values[12] - 1.0562165298583307e-07) <= 5e-14, "F_12(15) = %.17g", b.values[12]);
    const boysfn::BoysBatch c = boysfn::boys_batch(40.0, 0, T);
    CHECK(c.values[0] == 0.14012478040994822, "F_0(40) = %.17g", c.values[0]);
    CHECK(boysfn::classify_region(T.x0, T) == boysfn::Region::B, "x0 -> B");
    CHECK(boysfn::classify_region(std::nextafter(T.x0, 0.0), T) == boysfn::Region::A, "x0- -> A");
    CHECK(boysfn::classify_region(T.x1, T) == boysfn::Region::C, "x1 -> C");
    for (int r = 0; r < 3; ++r) {
      // each forced region at a point of its own interval's closure
      const double x = r == 0 ? T.x0 - 1e-9 : r == 1 ? T.x0 + 1e-9 : T.x1 + 1e-9;
      const auto g = boysfn::boys_batch_region(x, 20, T, static_cast<boysfn::Region>(r));
      std::vector<double> w(21);
      oracle_boys_batch_region(x, 20, &O.t, r, w.data());
      double dev = 0;
      for (int l = 0; l <= 20; ++l) dev = std::fmax(dev, std::fabs(g.values[l] - w[l]));
      CHECK(dev <= 5e-14, "forced region %d dev %g", r, dev);
    }
    try {
      boysfn::boys_batch_region(0.0, 3, T, boysfn::Region::B);
      CHECK(false, "upward at x=0 not rejected");
    } catch (const std::domain_error& e) {
      CHECK(std::string(e.what()) == "upward_recursion: x must be positive", "%s", e.what());
    }
  }
  // 5) verify_tables (verify.hpp:34-35) through the drop-in
  {
    const boysfn::VerifyReport r = boysfn::verify_tables(T, 500);
    CHECK(r.per_k.size() == 33 && r.all_within(5e-14), "verify: max_err %g", r.max_err);
    CHECK(r.worst_region == 'A' || r.worst_region == 'B' || r.worst_region == 'C', "worst region");
    try {
      boysfn::verify_tables(T, 10, 20.0);
      CHECK(false, "xmax <= x1 not rejected");
    } catch (const std::invalid_argument& e) {
      CHECK(std::string(e.what()) == "verify_tables: xmax must exceed x1", "%s", e.what());
    }
  }
  // 6) empty input
  {
    std::vector<double> none, out;
    boysfn::boys_batch_many(none, 99, T, out);  // the reference does not throw here
  }
  std::printf("%s (%d failures)\n", failures ? "FAILED" : "OK", failures);
  return failures ? 1 : 0;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc >= 3 && std::strcmp(argv[1], "parse") == 0) return cmd_parse(argv[2]);
  if (argc >= 2 && std::strcmp(argv[1], "gpu") == 0) return cmd_gpu();
  std::fprintf(stderr, "usage: shim_test parse <file> | gpu\n");
  return 2;
}
