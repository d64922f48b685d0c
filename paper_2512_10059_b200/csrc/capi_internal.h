// capi_internal.h -- shared by the C-ABI translation units (capi.cu, alg2.cu).
#pragma once

#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "../../include/boysfn_b200.h"
#include "boys_device.cuh"

#define BOYSFN_API extern "C" __attribute__((visibility("default")))

// Immutable device-side image of one CoefficientTableSet (boysfn_tables_t).
struct boysfn_tables_s {
  double x0 = 0, x1 = 0, eps_tol = 0;
  int k_max = 0;
  bool is_embedded = false;
  std::vector<boysfn_dev::EvalParams> params;  // one launch image per order k <= k_max
  std::vector<int> variant;                    // templated-kernel degree variant per k
  std::vector<int> degree_ok;                  // 1 if r_A[k], r_B fit the device image
  std::vector<int> deg_na, deg_ma;             // degrees of r_A[k] (generic kernel)
  int deg_nb = 0, deg_mb = 0;                  // degrees of r_B
  // validate_tables (tables.cpp:14-32) outcome, recorded at creation: the
  // evaluation paths do not need it (eval.cpp never validates), verify_tables
  // does (verify.cpp:14)
  int valid_status = 0;
  std::string valid_msg;
};

namespace boysfn_internal {
int fail(int status, const std::string& msg);         // sets boysfn_last_error()
int cuda_fail(cudaError_t e, const char* where);      // BOYSFN_ERR_CUDA
void count_launch();                                  // boysfn_kernel_launch_count()
}  // namespace boysfn_internal

#define CUDA_TRY(call)                                                   \
  do {                                                                   \
    cudaError_t e_ = (call);                                             \
    if (e_ != cudaSuccess) return boysfn_internal::cuda_fail(e_, #call); \
  } while (0)
