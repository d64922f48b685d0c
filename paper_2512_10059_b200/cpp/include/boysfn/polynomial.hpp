// polynomial.hpp -- monomial-basis polynomials, ascending coefficients
// (mirrors the reference's boysfn/polynomial.hpp).
#pragma once

#include <vector>

#include "boysfn/highprec.hpp"

namespace boysfn {

using Poly = std::vector<hp::Real>;

hp::Real poly_eval(const Poly& p, const hp::Real& x);
Poly poly_derivative(const Poly& p);
Poly poly_trim(const Poly& p, const hp::Real& rel_tol);
int poly_degree(const Poly& p);
int sturm_root_count(const Poly& p, const hp::Real& a, const hp::Real& b);  // roots in (a, b]
Poly newton_interpolate(const std::vector<hp::Real>& xs, const std::vector<hp::Real>& ys);
std::vector<int> leja_order(const std::vector<hp::Real>& xs);

}  // namespace boysfn
