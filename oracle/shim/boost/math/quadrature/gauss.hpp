// Test tooling only (oracle/_ref build). Minimal stand-in for the Boost.Math
// header <boost/math/quadrature/gauss.hpp>, which is absent from this image.
// It restates the published N-point Gauss-Legendre rule: nodes are the roots
// of P_N (Newton iteration in long double from the Chebyshev-like initial
// guess), weights 2 / ((1 - x^2) P_N'(x)^2). Integration over [a, b] maps to
// [-1, 1] as Boost does: Q = scale * sum_i w_i (f(avg + scale x_i) +
// f(avg - scale x_i)), positive abscissae in increasing order.
#pragma once

#include <array>
#include <cmath>
#include <stdexcept>

namespace boost {
namespace math {
namespace quadrature {

template <class Real, unsigned N>
class gauss {
  static constexpr unsigned kHalf = (N + 1) / 2;

  struct Rule {
    std::array<Real, kHalf> x{};
    std::array<Real, kHalf> w{};
    Rule() {
      const long double pi = 3.141592653589793238462643383279502884L;
      for (unsigned i = 0; i < N / 2; ++i) {
        // i-th largest root, refined by Newton on P_N.
        long double z = std::cos(pi * (i + 0.75L) / (N + 0.5L));
        long double dp = 0.0L;
        for (int it = 0; it < 100; ++it) {
          long double p0 = 1.0L, p1 = z;
          for (unsigned k = 2; k <= N; ++k) {
            long double p2 = ((2.0L * k - 1.0L) * z * p1 - (k - 1.0L) * p0) / k;
            p0 = p1;
            p1 = p2;
          }
          dp = N * (z * p1 - p0) / (z * z - 1.0L);
          long double dz = p1 / dp;
          z -= dz;
          if (std::fabs(dz) < 1e-21L) break;
        }
        // recompute derivative at the converged root
        long double p0 = 1.0L, p1 = z;
        for (unsigned k = 2; k <= N; ++k) {
          long double p2 = ((2.0L * k - 1.0L) * z * p1 - (k - 1.0L) * p0) / k;
          p0 = p1;
          p1 = p2;
        }
        dp = N * (z * p1 - p0) / (z * z - 1.0L);
        // store ascending: largest root goes last
        unsigned slot = kHalf - 1 - i;
        x[slot] = static_cast<Real>(z);
        w[slot] = static_cast<Real>(2.0L / ((1.0L - z * z) * dp * dp));
      }
      if (N % 2 == 1) {
        // centre node for odd N
        long double p0 = 1.0L, p1 = 0.0L;
        for (unsigned k = 2; k <= N; ++k) {
          long double p2 = ((2.0L * k - 1.0L) * 0.0L * p1 - (k - 1.0L) * p0) / k;
          p0 = p1;
          p1 = p2;
        }
        long double dp = N * (0.0L * p1 - p0) / (0.0L - 1.0L);
        x[0] = 0;
        w[0] = static_cast<Real>(2.0L / (dp * dp));
      }
    }
  };

  static const Rule& rule() {
    static const Rule r;
    return r;
  }

 public:
  static const std::array<Real, kHalf>& abscissa() { return rule().x; }
  static const std::array<Real, kHalf>& weights() { return rule().w; }

  template <class F>
  static auto integrate(F f, Real* pL1 = nullptr) -> decltype(f(Real(0))) {
    using R = decltype(f(Real(0)));
    const Rule& r = rule();
    R result = (N % 2 == 1) ? f(Real(0)) * r.w[0] : R(0);
    Real l1 = (N % 2 == 1) ? std::abs(result) : Real(0);
    for (unsigned i = (N % 2 == 1) ? 1 : 0; i < kHalf; ++i) {
      R fp = f(r.x[i]);
      R fm = f(-r.x[i]);
      result += (fp + fm) * r.w[i];
      l1 += (std::abs(fp) + std::abs(fm)) * r.w[i];
    }
    if (pL1) *pL1 = l1;
    return result;
  }

  template <class F>
  static auto integrate(F f, Real a, Real b, Real* pL1 = nullptr)
      -> decltype(f(Real(0))) {
    // Boost only rejects NaN / infinite bounds here; b < a integrates with a
    // negative scale (a signed integral), which cell_average_2d relies on
    // when a split leaves a corner cell smaller than the pole ball.
    if (!std::isfinite(a) || !std::isfinite(b))
      throw std::domain_error("gauss: bounds not finite");
    Real avg = (a + b) * Real(0.5);
    Real scale = (b - a) * Real(0.5);
    auto u = [&](Real z) { return f(avg + scale * z); };
    auto q = integrate(u, pL1);
    if (pL1) *pL1 *= scale;
    return scale * q;
  }
};

}  // namespace quadrature
}  // namespace math
}  // namespace boost
