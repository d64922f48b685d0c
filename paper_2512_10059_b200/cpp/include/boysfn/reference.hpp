// reference.hpp -- the equal-sign Boys series oracle and its truncation bound
// (mirrors the reference's boysfn/reference.hpp; reference.cpp:10-54).
#pragma once

#include <vector>

#include "boysfn/highprec.hpp"

namespace boysfn {

struct ReferenceConfig {
  int truncation_terms = 150;
};

hp::Real boys_reference(int k, const hp::Real& x, const ReferenceConfig& cfg = {});
std::vector<hp::Real> boys_reference_batch(int kmax, const hp::Real& x, const ReferenceConfig& cfg = {});
hp::Real truncation_bound(int k, const hp::Real& x, int L);
int reference_terms_for(int k, double x, double rel_target = 1e-30);

}  // namespace boysfn
