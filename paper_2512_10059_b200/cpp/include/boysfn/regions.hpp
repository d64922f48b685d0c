// regions.hpp -- x0 (Eq. 20), x1 (Eq. 12), rho_A,k (Eq. 18) (mirrors the
// reference's boysfn/regions.hpp).
#pragma once

#include "boysfn/highprec.hpp"

namespace boysfn {

struct RegionPartition {
  double x0 = 0;
  double x1 = 0;
  int k_max = 0;
  double eps_tol = 0;
};

hp::Real compute_x0(int k_max);
hp::Real compute_x1(int k_max, const hp::Real& eps_tol);
hp::Real weight_rho_A(int k, const hp::Real& x);
RegionPartition make_partition(int k_max, double eps_tol);

}  // namespace boysfn
