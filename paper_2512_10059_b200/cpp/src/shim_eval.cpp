// shim_eval.cpp -- the drop-in boysfn::boys_batch_many & co.  Host-side
// validation and exception mapping only; every value is computed by the
// sm_100a kernels behind include/boysfn_b200.h.  Replaces the reference's
// eval.cpp (core/CMakeLists.txt:16) in a boysfn_core build.
#include <stdexcept>
#include <string>
#include <vector>

#include "../../../include/boysfn_b200.h"
#include "boysfn/eval.hpp"
#include "boysfn/verify.hpp"

namespace boysfn {
namespace {

// Rethrows a C-ABI status as the reference's exception type and message.
void raise(int status) {
  if (status == BOYSFN_OK) return;
  const std::string msg = boysfn_last_error();
  switch (status) {
    case BOYSFN_ERR_SIZE: throw std::invalid_argument(msg);
    case BOYSFN_ERR_DOMAIN: throw std::domain_error(msg);
    case BOYSFN_ERR_RANGE: throw std::out_of_range(msg);
    case BOYSFN_ERR_TABLES: throw std::invalid_argument(msg);
    case BOYSFN_ERR_INVALID: throw std::invalid_argument(msg);
    default: throw std::runtime_error("boysfn_b200: " + std::string(boysfn_status_string(status)) + ": " + msg);
  }
}

// A device table handle for `tables`: the process-lifetime embedded handle for
// embedded_default() itself, otherwise a short-lived handle (validation plus a
// host-side pack of the coefficients; no device allocation).
class Handle {
 public:
  explicit Handle(const CoefficientTableSet& t) {
    if (&t == &embedded_default()) {
      raise(boysfn_tables_embedded(&h_));
      return;
    }
    std::vector<boysfn_rational_desc> ra(t.r_A.size());
    auto desc = [](const RationalApproximant& r) {
      return boysfn_rational_desc{r.degree_n(), r.degree_m(), r.numer.data(), r.denom.data()};
    };
    for (size_t k = 0; k < t.r_A.size(); ++k) ra[k] = desc(t.r_A[k]);
    // eval.cpp evaluates any set it is given: only what the device image needs
    // is checked here (boysfn_tables_create); verify_tables validates first.
    if (t.k_max >= 0 && t.r_A.size() < static_cast<size_t>(t.k_max) + 1)
      throw std::invalid_argument("tables: need exactly k_max+1 region-A tables");
    const boysfn_table_desc d{t.x0, t.x1, t.k_max, t.eps_tol, desc(t.r_B), ra.data()};
    raise(boysfn_tables_create(&d, &h_));
  }
  ~Handle() { boysfn_tables_destroy(h_); }
  Handle(const Handle&) = delete;
  Handle& operator=(const Handle&) = delete;
  boysfn_tables_t get() const { return h_; }

 private:
  boysfn_tables_t h_ = nullptr;
};

}  // namespace

Region classify_region(double x, const CoefficientTableSet& tables) {
  if (x < tables.x0) return Region::A;
  if (x < tables.x1) return Region::B;
  return Region::C;
}

void boys_batch_many(std::span<const double> xs, int k, const CoefficientTableSet& tables,
                     std::span<double> out) {
  const Handle h(tables);
  raise(boysfn_eval_host(h.get(), xs.data(), xs.size(), k, out.data(), out.size(), BOYSFN_LAYOUT_AOS, 0,
                         nullptr));
}

BoysBatch boys_batch(double x, int k, const CoefficientTableSet& tables) {
  BoysBatch b;
  b.x = x;
  b.k = k;
  const Handle h(tables);
  // One-row boys_batch_many: same checks (x, then k), same messages.
  if (k < 0 || k > tables.k_max) {
    double dummy = 0;
    raise(boysfn_eval_host(h.get(), &x, 1, k, &dummy, 1 * (static_cast<size_t>(k) + 1),
                           BOYSFN_LAYOUT_AOS, 0, nullptr));
  }
  b.values.resize(static_cast<size_t>(k) + 1);
  raise(boysfn_eval_host(h.get(), &x, 1, k, b.values.data(), b.values.size(), BOYSFN_LAYOUT_AOS, 0,
                         nullptr));
  return b;
}

BoysBatch boys_batch_region(double x, int k, const CoefficientTableSet& tables, Region region) {
  BoysBatch b;
  b.x = x;
  b.k = k;
  const Handle h(tables);
  std::vector<double> v(k >= 0 ? static_cast<size_t>(k) + 1 : 1);
  raise(boysfn_eval_region_host(h.get(), x, k, static_cast<int>(region), v.data()));
  b.values = std::move(v);
  return b;
}

VerifyReport verify_tables(const CoefficientTableSet& tables, int samples_per_region, double xmax,
                           std::uint64_t seed) {
  validate_tables(tables);  // verify.cpp:14
  const Handle h(tables);
  std::vector<double> per_k((static_cast<size_t>(tables.k_max) + 1) * 3);
  boysfn_verify_report r{};
  r.per_k = per_k.data();
  raise(boysfn_verify_tables(h.get(), samples_per_region, xmax, seed, &r));
  VerifyReport rep;
  rep.per_k.resize(tables.k_max + 1);
  for (int k = 0; k <= tables.k_max; ++k)
    rep.per_k[k] = VerifyEntry{k, per_k[3 * k], per_k[3 * k + 1], per_k[3 * k + 2]};
  rep.max_err = r.max_err;
  rep.worst_x = r.worst_x;
  rep.worst_k = r.worst_k;
  rep.worst_region = r.worst_region;
  for (int i = 0; i < 3; ++i) rep.max_err_region[i] = r.max_err_region[i];
  return rep;
}

}  // namespace boysfn
