// Test tooling only (oracle/_ref build). Stand-in for Boost.Math's
// <boost/math/quadrature/gauss_kronrod.hpp>. It is NOT a Kronrod rule: it is an
// adaptive bisection with a 30-point Gauss-Legendre rule on each half,
// error estimated from one level of refinement. Only the reference's
// diagnostic paths (numeric radial transforms, 1D tail integrals) use it; the
// hot path (grids, C tables for d <= 2 spectral mode, the matvec) does not.
#pragma once

#include <cmath>
#include <limits>

#include "boost/math/quadrature/gauss.hpp"

namespace boost {
namespace math {
namespace quadrature {

template <class Real, unsigned N>
class gauss_kronrod {
  template <class F>
  static Real recurse(F& f, Real a, Real b, Real whole, unsigned depth,
                      Real tol, Real& err) {
    Real m = (a + b) / 2;
    Real left = gauss<Real, 30>::integrate(f, a, m);
    Real right = gauss<Real, 30>::integrate(f, m, b);
    Real diff = std::abs(left + right - whole);
    if (depth == 0 || diff <= tol * std::abs(left + right) || diff < 1e-300) {
      err += diff;
      return left + right;
    }
    return recurse(f, a, m, left, depth - 1, tol, err) +
           recurse(f, m, b, right, depth - 1, tol, err);
  }

 public:
  template <class F>
  static Real integrate(F f, Real a, Real b, unsigned max_depth = 15,
                        Real tol = std::sqrt(std::numeric_limits<Real>::epsilon()),
                        Real* error = nullptr, Real* pL1 = nullptr) {
    Real whole = gauss<Real, 30>::integrate(f, a, b);
    Real err = 0;
    Real v = recurse(f, a, b, whole, max_depth, tol, err);
    if (error) *error = err;
    if (pL1) *pL1 = std::abs(v);
    return v;
  }
};

}  // namespace quadrature
}  // namespace math
}  // namespace boost
