// Test tooling only (oracle/_ref build). Placeholder for Boost.Math's Ooura
// oscillatory integrators. The reference uses them only in diagnostic
// transforms (radial_fourier_numeric for IMQ, 1D TPS tails), none of which are
// on the matvec hot path; calling them through the shim throws.
#pragma once

#include <stdexcept>
#include <utility>

namespace boost {
namespace math {
namespace quadrature {

template <class Real>
class ooura_fourier_cos {
 public:
  explicit ooura_fourier_cos(Real = Real(0), std::size_t = 0) {}
  template <class F>
  std::pair<Real, Real> integrate(F, Real) const {
    throw std::runtime_error("ooura_fourier_cos is not available in the shim");
  }
};

template <class Real>
class ooura_fourier_sin {
 public:
  explicit ooura_fourier_sin(Real = Real(0), std::size_t = 0) {}
  template <class F>
  std::pair<Real, Real> integrate(F, Real) const {
    throw std::runtime_error("ooura_fourier_sin is not available in the shim");
  }
};

}  // namespace quadrature
}  // namespace math
}  // namespace boost
