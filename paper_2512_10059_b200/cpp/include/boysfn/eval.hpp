// boysfn/eval.hpp -- drop-in replacement of the reference evaluation API,
// /root/reference/proj/core/include/boysfn/eval.hpp:1-47, backed by the
// sm_100a kernels of libboysfn_b200.so through the C ABI in
// include/boysfn_b200.h.
//
// Same names, signatures, exception types and messages as the reference:
//   std::invalid_argument  output span size mismatch        (eval.cpp:90-91)
//   std::domain_error      x negative or non-finite         (eval.cpp:14-15)
//   std::out_of_range      k outside [0, tables.k_max]      (eval.cpp:16-17)
// and the same partial-output behaviour: rows before the first bad x are
// written, later rows are untouched.  A CUDA failure throws std::runtime_error
// (the reference has no device).  The scalar helpers eval_rational,
// downward_recursion and upward_recursion of the reference (eval.hpp:22-31)
// are internal steps of the device kernel and are not exported.
#pragma once

#include <span>
#include <vector>

#include "boysfn/tables.hpp"

namespace boysfn {

// F_0(x)..F_k(x) for one argument.  Reference: eval.hpp:11-15.
struct BoysBatch {
  double x = 0;
  int k = 0;
  std::vector<double> values;
};

// [0, x0) -> A, [x0, x1) -> B, [x1, inf) -> C.  Reference: eval.hpp:17-20.
enum class Region { A, B, C };

Region classify_region(double x, const CoefficientTableSet& tables);

// One argument, evaluated on the device.  Reference: eval.hpp:37, eval.cpp:83-86.
BoysBatch boys_batch(double x, int k, const CoefficientTableSet& tables);

// Forced region (branch-agreement seam).  Reference: eval.hpp:39-41, eval.cpp:59-81.
BoysBatch boys_batch_region(double x, int k, const CoefficientTableSet& tables, Region region);

// Bulk entry: out holds xs.size()*(k+1) doubles, row-major (AoS).
// Reference: eval.hpp:43-45, eval.cpp:88-96.
void boys_batch_many(std::span<const double> xs, int k, const CoefficientTableSet& tables,
                     std::span<double> out);

}  // namespace boysfn
