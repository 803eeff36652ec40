// Test tooling only (oracle/_ref build). Stand-in for Boost.Math's
// <boost/math/quadrature/tanh_sinh.hpp>: the published double-exponential
// rule x = tanh(pi/2 sinh t), w = (pi/2) cosh t / cosh^2(pi/2 sinh t), with the
// step halved until successive estimates agree to `tol` relative to the L1
// norm (Boost's default tolerance sqrt(eps), at most 15 refinements). Nodes
// are placed through their distance to the nearer endpoint so the endpoints
// themselves are never sampled.
#pragma once

#include <cmath>
#include <cstddef>
#include <limits>
#include <stdexcept>

namespace boost {
namespace math {
namespace quadrature {

template <class Real>
class tanh_sinh {
 public:
  explicit tanh_sinh(std::size_t max_refinements = 15,
                     Real /*min_complement*/ = Real(0))
      : max_ref_(max_refinements) {}

  template <class F>
  Real integrate(F f, Real a, Real b,
                 Real tol = std::sqrt(std::numeric_limits<Real>::epsilon()),
                 Real* error = nullptr, Real* L1 = nullptr,
                 std::size_t* levels = nullptr) const {
    if (!(b > a)) {
      if (a == b) return Real(0);
      return -integrate(f, b, a, tol, error, L1, levels);
    }
    const Real half_pi = Real(1.5707963267948966192313216916397514L);
    const Real c = (a + b) / 2, h = (b - a) / 2;
    const Real t_max = Real(6.56);  // complement below ~1e-300 past here
    // sum over t = k * step of w(t) [f(x(t)) + f(x(-t))] (t != 0) + w(0) f(c)
    auto node = [&](Real t, Real& comp, Real& w) {
      Real s = half_pi * std::sinh(t);
      Real e = std::exp(-2 * s);
      comp = 2 * e / (1 + e);  // 1 - tanh(s)
      Real ch = std::cosh(s);
      w = half_pi * std::cosh(t) / (ch * ch);
    };
    Real step = Real(1);
    Real sum = f(c) * half_pi, l1 = std::abs(sum);
    auto add_points = [&](Real t0, Real dt) {
      for (Real t = t0; t <= t_max; t += dt) {
        Real comp, w;
        node(t, comp, w);
        if (comp * h <= 0) break;
        Real xr = b - h * comp, xl = a + h * comp;
        if (!(xr < b) || !(xl > a)) break;
        Real fr = f(xr), fl = f(xl);
        sum += w * (fr + fl);
        l1 += w * (std::abs(fr) + std::abs(fl));
      }
    };
    add_points(step, step);
    Real est = sum * step * h, prev = est;
    Real err = std::numeric_limits<Real>::max();
    std::size_t k = 0;
    for (k = 1; k <= max_ref_; ++k) {
      step /= 2;
      add_points(step, 2 * step);
      est = sum * step * h;
      err = std::abs(est - prev);
      if (k >= 3 && err <= tol * l1 * step * h) break;
      prev = est;
    }
    if (error) *error = err;
    if (L1) *L1 = l1 * step * h;
    if (levels) *levels = k;
    return est;
  }

 private:
  std::size_t max_ref_;
};

}  // namespace quadrature
}  // namespace math
}  // namespace boost
