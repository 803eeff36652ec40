// Host plan-time math of the band-limited FMM: kernel-spec grammar, closed
// form spectra and the translation spectrum C(xi_m) on the uniform
// left-endpoint grid. Everything here runs once per plan; the per-matvec hot
// path is the CUDA code in blfmm.cu and its k_*.inc.cuh fragments.
//
// Reference behaviour followed:
//   parse_kernel_spec      kernels.cpp:48-103
//   eval_kernel            kernels.cpp:131-161 (device copy: device.cuh phi_of_r2)
//   eval_fourier           kernels.cpp:190-238; d = 3 from the same
//                          (r^2+c^2)^{-beta} family
//   make_quadrature        bandlimit.cpp:269-292 (row-major tensor nodes)
//   translation_coefficients (spectral) bandlimit.cpp:388-447 with the cell
//                          averages of bandlimit.cpp:336-384 and their 3-D
//                          analogue (fold / split / corner / tensor rule).
//   eval_bandlimited (d=1) bandlimit.cpp:307-334 with the band integrals of
//                          bandlimit.cpp:61-100 (Gaussian, IMQ, MQ tail form)
//   bandlimited_radial_table bandlimit.cpp:229-262 (1027 samples, cached)
#include <algorithm>
#include <cctype>
#include <cmath>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <tuple>
#include <vector>

#include "blfmm_internal.h"

namespace blfmm_gpu {
namespace {

constexpr double kPi = 3.14159265358979323846;
constexpr double kTwoPi = 2.0 * kPi;
constexpr double kPoleBall = 1e-8;  // exclusion radius around the spectral pole

// Gauss-Legendre rule with N nodes: roots of P_N by Newton in long double.
template <int N>
class GaussLegendre {
 public:
  GaussLegendre() {
    constexpr int n = N;
    for (int i = 0; i < n / 2; ++i) {
      long double z = std::cos(3.14159265358979323846264338L * (i + 0.75L) / (n + 0.5L));
      long double deriv = 0;
      for (int it = 0; it < 100; ++it) {
        long double p_prev = 1, p = z;
        for (int k = 2; k <= n; ++k) {
          long double p_next = ((2.0L * k - 1) * z * p - (k - 1.0L) * p_prev) / k;
          p_prev = p;
          p = p_next;
        }
        deriv = n * (z * p - p_prev) / (z * z - 1);
        long double step = p / deriv;
        z -= step;
        if (std::fabs(step) < 1e-21L) break;
      }
      long double p_prev = 1, p = z;
      for (int k = 2; k <= n; ++k) {
        long double p_next = ((2.0L * k - 1) * z * p - (k - 1.0L) * p_prev) / k;
        p_prev = p;
        p = p_next;
      }
      deriv = n * (z * p - p_prev) / (z * z - 1);
      node_[n / 2 - 1 - i] = static_cast<double>(z);
      weight_[n / 2 - 1 - i] = static_cast<double>(2.0L / ((1 - z * z) * deriv * deriv));
    }
  }
  // Signed integral over [a, b] (b < a integrates with a negative scale).
  template <class F>
  double integrate(const F& f, double a, double b) const {
    double mid = 0.5 * (a + b), half = 0.5 * (b - a), acc = 0.0;
    for (int i = 0; i < N / 2; ++i)
      acc += (f(mid + half * node_[i]) + f(mid - half * node_[i])) * weight_[i];
    return half * acc;
  }
  double node(int i) const { return node_[i]; }
  double weight(int i) const { return weight_[i]; }

 private:
  double node_[N / 2];
  double weight_[N / 2];
};
using GaussLegendre30 = GaussLegendre<30>;

const GaussLegendre30& gl() {
  static const GaussLegendre30 rule;
  return rule;
}

// tanh-sinh (double exponential) rule, tolerance sqrt(eps) relative to L1;
// abscissae addressed through their endpoint complement.
template <class F>
double double_exponential(const F& f, double a, double b) {
  if (a == b) return 0.0;
  if (b < a) return -double_exponential(f, b, a);
  const double hp = 0.5 * kPi, mid = 0.5 * (a + b), half = 0.5 * (b - a);
  const double tol = 1.4901161193847656e-08;
  double h = 1.0, sum = hp * f(mid), l1 = std::abs(sum);
  auto sweep = [&](double t0, double dt) {
    for (double t = t0; t <= 6.56; t += dt) {
      double s = hp * std::sinh(t), e = std::exp(-2.0 * s);
      double comp = 2.0 * e / (1.0 + e), ch = std::cosh(s);
      double w = hp * std::cosh(t) / (ch * ch);
      double xr = b - half * comp, xl = a + half * comp;
      if (!(xr < b) || !(xl > a)) break;
      double fr = f(xr), fl = f(xl);
      sum += w * (fr + fl);
      l1 += w * (std::abs(fr) + std::abs(fl));
    }
  };
  sweep(h, h);
  double last = sum * h * half, cur = last;
  for (int level = 1; level <= 15; ++level) {
    h *= 0.5;
    sweep(h, 2.0 * h);
    cur = sum * h * half;
    if (level >= 3 && std::abs(cur - last) <= tol * l1 * h * half) break;
    last = cur;
  }
  return cur;
}

double bessel_k(double nu, double z) {
  if (z > 690.0) return 0.0;  // hard underflow, kernels.cpp:36-44
  return std::cyl_bessel_k(nu, z);
}

// Corner square [0,delta]^2 minus the pole disc, polar coordinates split on
// the diagonal (bandlimit.cpp:134-154 with x = 0).
template <class S>
double corner_square(const S& spec, double delta, double r0) {
  const auto& g = gl();
  auto wedge = [&](double t0, double t1, bool use_cos) {
    auto over_angle = [&](double th) {
      double rmax = delta / (use_cos ? std::cos(th) : std::sin(th));
      return g.integrate([&](double r) { return r * spec(r); }, r0, rmax);
    };
    return g.integrate(over_angle, t0, t1);
  };
  return wedge(0.0, 0.25 * kPi, true) + wedge(0.25 * kPi, 0.5 * kPi, false);
}

// Corner cube [0,delta]^3 minus the pole ball: 3 pyramids (largest
// coordinate) x 2 azimuth halves of one congruent piece, spherical coords.
template <class S>
double corner_cube(const S& spec, double delta, double r0) {
  const auto& g = gl();
  auto over_phi = [&](double phi) {
    double th_max = std::atan(1.0 / std::cos(phi));
    auto over_theta = [&](double th) {
      double rmax = delta / std::cos(th);
      return std::sin(th) *
             g.integrate([&](double r) { return r * r * spec(r); }, r0, rmax);
    };
    return g.integrate(over_theta, 0.0, th_max);
  };
  return 6.0 * g.integrate(over_phi, 0.0, 0.25 * kPi);
}

struct Spectrum {
  KernelSpec k;
  int d;
  double operator()(double rho) const { return fourier_value(k, rho, d); }
};

double average_1d(const KernelSpec& k, double a, double b) {
  Spectrum s{k, 1};
  auto f = [&](double xi) { return s(std::abs(xi)); };
  double lo = a, hi = b, v;
  if (lo < 0.0 && hi > 0.0) {
    v = double_exponential(f, lo, -kPoleBall) + double_exponential(f, kPoleBall, hi);
  } else {
    if (lo == 0.0) lo = kPoleBall;
    if (hi == 0.0) hi = -kPoleBall;
    v = double_exponential(f, lo, hi);
  }
  return v / (b - a);
}

// Generic-dimension cell average over prod_k [a_k, b_k] of the radial
// spectrum: fold each axis to the positive side, split an axis straddling 0,
// integrate the origin corner cube in polar/spherical coordinates with the
// pole ball excluded, and everything else with a tensor 30-point rule.
double average_nd(const KernelSpec& k, int d, double* a, double* b) {
  Spectrum s{k, d};
  for (int ax = 0; ax < d; ++ax)
    if (b[ax] <= 0.0) {
      double t = a[ax];
      a[ax] = -b[ax];
      b[ax] = -t;
    }
  double vol = 1.0;
  for (int ax = 0; ax < d; ++ax) vol *= b[ax] - a[ax];
  for (int ax = 0; ax < d; ++ax) {
    if (a[ax] < 0.0) {
      double a_lo[3], b_lo[3], a_hi[3], b_hi[3];
      for (int q = 0; q < d; ++q) a_lo[q] = a_hi[q] = a[q], b_lo[q] = b_hi[q] = b[q];
      b_lo[ax] = 0.0;
      a_hi[ax] = 0.0;
      double rest = vol / (b[ax] - a[ax]);
      double v = average_nd(k, d, a_lo, b_lo) * (-a[ax]) * rest +
                 average_nd(k, d, a_hi, b_hi) * b[ax] * rest;
      return v / vol;
    }
  }
  bool corner = true;
  for (int ax = 0; ax < d; ++ax)
    if (a[ax] != 0.0 || b[ax] != b[0]) corner = false;
  if (corner)
    return (d == 2 ? corner_square(s, b[0], kPoleBall) : corner_cube(s, b[0], kPoleBall)) / vol;
  const auto& g = gl();
  if (d == 2) {
    auto outer = [&](double x) {
      return g.integrate([&](double y) { return s(std::hypot(x, y)); }, a[1], b[1]);
    };
    return g.integrate(outer, a[0], b[0]) / vol;
  }
  auto outer = [&](double x) {
    auto middle = [&](double y) {
      return g.integrate([&](double z) { return s(std::hypot(x, y, z)); }, a[2], b[2]);
    };
    return g.integrate(middle, a[1], b[1]);
  };
  return g.integrate(outer, a[0], b[0]) / vol;
}

template <class F>
void parallel_for(long n, const F& f) {
  unsigned hw = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  if (n < 64 || hw == 1) {
    for (long i = 0; i < n; ++i) f(i);
    return;
  }
  std::vector<std::thread> pool;
  for (unsigned t = 0; t < hw; ++t)
    pool.emplace_back([&, t] {
      for (long i = t; i < n; i += hw) f(i);
    });
  for (auto& th : pool) th.join();
}

std::string lower(std::string s) {
  for (auto& c : s) c = static_cast<char>(std::tolower(static_cast<unsigned char>(c)));
  return s;
}

}  // namespace

KernelSpec parse_spec(const std::string& spec) {
  std::string s = lower(spec), name = s, param;
  if (auto colon = s.find(':'); colon != std::string::npos) {
    name = s.substr(0, colon);
    param = s.substr(colon + 1);
  }
  KernelSpec k;
  std::string key;
  if (name == "gaussian" || name == "ga") {
    k = {BLFMM_KERNEL_GAUSSIAN, 1.0};
    key = "c";
  } else if (name == "mq" || name == "multiquadric") {
    k = {BLFMM_KERNEL_MQ, 1.0};
    key = "c";
  } else if (name == "imq") {
    k = {BLFMM_KERNEL_IMQ, 1.0};
    key = "c";
  } else if (name == "tps") {
    k = {BLFMM_KERNEL_TPS, 2.0};
    key = "beta";
  } else if (name == "wendland" || name == "wendlandc2") {
    k = {BLFMM_KERNEL_WENDLAND_C2, 0.5};
    key = "eps";
  } else if (name == "wendland31") {
    k = {BLFMM_KERNEL_WENDLAND31, 0.5};
    key = "eps";
  } else {
    throw Error(BLFMM_EINVAL, "unknown kernel '" + name + "'");
  }
  if (!param.empty()) {
    auto eq = param.find('=');
    if (eq == std::string::npos)
      throw Error(BLFMM_EINVAL, "kernel parameter must be key=value, got '" + param + "'");
    std::string got = param.substr(0, eq);
    if (got != key)
      throw Error(BLFMM_EINVAL, "kernel '" + name + "' takes parameter '" + key +
                                    "', not '" + got + "'");
    std::size_t used = 0;
    double value;
    try {
      value = std::stod(param.substr(eq + 1), &used);
    } catch (const std::exception&) {
      throw Error(BLFMM_EINVAL, "bad numeric value in '" + param + "'");
    }
    if (used != param.size() - eq - 1)
      throw Error(BLFMM_EINVAL, "bad numeric value in '" + param + "'");
    if (!(value > 0.0) || !std::isfinite(value))
      throw Error(BLFMM_EINVAL, "kernel parameter must be positive");
    if (k.type == BLFMM_KERNEL_TPS &&
        (value != std::floor(value) || std::fmod(value, 2.0) != 0.0))
      throw Error(BLFMM_EINVAL, "tps beta must be a positive even integer");
    k.shape = value;
  }
  return k;
}

void require_fmm_kernel(const KernelSpec& k) {
  if (k.type != BLFMM_KERNEL_GAUSSIAN && k.type != BLFMM_KERNEL_MQ &&
      k.type != BLFMM_KERNEL_IMQ)
    throw Error(BLFMM_EDOMAIN,
                "kernel not supported by the GPU band-limited FMM (gaussian, mq, imq)");
}

void require_radial_kernel(const KernelSpec& k) {
  if (k.type < BLFMM_KERNEL_GAUSSIAN || k.type > BLFMM_KERNEL_WENDLAND31)
    throw Error(BLFMM_EINVAL, "unknown kernel type");
  if (!(k.shape > 0.0) || !std::isfinite(k.shape))
    throw Error(BLFMM_EINVAL, "kernel parameter must be positive");
  if (k.type == BLFMM_KERNEL_TPS &&
      (k.shape != std::floor(k.shape) || std::fmod(k.shape, 2.0) != 0.0))
    throw Error(BLFMM_EINVAL, "tps beta must be a positive even integer");
}

double fourier_value(const KernelSpec& k, double xi, int d) {
  if (d < 1 || d > 3) throw Error(BLFMM_EINVAL, "d must be 1, 2 or 3");
  xi = std::abs(xi);
  const double c = k.shape;
  switch (k.type) {
    case BLFMM_KERNEL_GAUSSIAN:
      return std::pow(kPi / c, 0.5 * d) * std::exp(-xi * xi / (4.0 * c));
    case BLFMM_KERNEL_IMQ:
      if (xi == 0.0) throw Error(BLFMM_EDOMAIN, "imq transform singular at xi=0");
      if (d == 1) return 2.0 * bessel_k(0.0, c * xi);
      if (d == 2) return 2.0 * kPi * std::exp(-c * xi) / xi;
      return 4.0 * kPi * c * bessel_k(1.0, c * xi) / xi;
    case BLFMM_KERNEL_MQ:
      if (xi == 0.0) throw Error(BLFMM_EDOMAIN, "mq generalized transform singular at xi=0");
      if (d == 1) return -2.0 * c * bessel_k(1.0, c * xi) / xi;
      if (d == 2) return -2.0 * kPi * (1.0 + c * xi) * std::exp(-c * xi) / (xi * xi * xi);
      return -4.0 * kPi * c * c * bessel_k(2.0, c * xi) / (xi * xi);
    default:
      throw Error(BLFMM_EDOMAIN, "no closed-form transform for this kernel");
  }
}

std::vector<double> translation_spectrum(const KernelSpec& k, double sigma,
                                         int m, int d) {
  if (!(sigma > 0.0)) throw Error(BLFMM_EINVAL, "sigma must be > 0");
  if (m < 2) throw Error(BLFMM_EINVAL, "m_per_dim must be >= 2");
  if (d < 1 || d > 3) throw Error(BLFMM_EINVAL, "d must be 1, 2 or 3");
  require_fmm_kernel(k);
  long kk = 1;
  for (int q = 0; q < d; ++q) kk *= m;
  const double dxi = 2.0 * sigma / m;
  const double scale = d == 1 ? 1.0 / kTwoPi
                              : (d == 2 ? 1.0 / (kTwoPi * kTwoPi)
                                        : 1.0 / (kTwoPi * kTwoPi * kTwoPi));
  std::vector<double> axis(m);
  for (int q = 0; q < m; ++q) axis[q] = -sigma + q * dxi;
  std::vector<double> c(kk);
  auto node_axes = [&](long node, double* v) {
    for (int q = d - 1; q >= 0; --q) {
      v[q] = axis[node % m];
      node /= m;
    }
  };
  if (k.type == BLFMM_KERNEL_GAUSSIAN) {
    // smooth spectrum: point samples
    parallel_for(kk, [&](long node) {
      double v[3];
      node_axes(node, v);
      double rho = d == 1 ? std::abs(v[0])
                          : (d == 2 ? std::hypot(v[0], v[1]) : std::hypot(v[0], v[1], v[2]));
      c[node] = scale * fourier_value(k, rho, d);
    });
    return c;
  }
  if (d == 1) {
    parallel_for(kk, [&](long node) {
      c[node] = scale * average_1d(k, axis[node], axis[node] + dxi);
    });
    return c;
  }
  // Singular spectra: cell averages. The average only depends on the folded
  // per-axis intervals (and, the spectrum being radial on cubic cells, not
  // on their order), so each distinct sorted folded triple is integrated once.
  using Cell = std::tuple<double, double, double, double, double, double>;
  std::vector<Cell> cell_of(kk);
  std::map<Cell, long> index;
  std::vector<Cell> unique;
  for (long node = 0; node < kk; ++node) {
    double v[3];
    node_axes(node, v);
    std::pair<double, double> iv[3] = {{0, 0}, {0, 0}, {0, 0}};
    for (int q = 0; q < d; ++q) {
      double a = v[q], b = v[q] + dxi;
      if (b <= 0.0) {
        double t = a;
        a = -b;
        b = -t;
      }
      iv[q] = {a, b};
    }
    std::sort(iv, iv + d);
    Cell cell{iv[0].first, iv[0].second, iv[1].first, iv[1].second, iv[2].first, iv[2].second};
    cell_of[node] = cell;
    if (index.emplace(cell, static_cast<long>(unique.size())).second) unique.push_back(cell);
  }
  std::vector<double> avg(unique.size());
  parallel_for(static_cast<long>(unique.size()), [&](long u) {
    double a[3] = {std::get<0>(unique[u]), std::get<2>(unique[u]), std::get<4>(unique[u])};
    double b[3] = {std::get<1>(unique[u]), std::get<3>(unique[u]), std::get<5>(unique[u])};
    avg[u] = average_nd(k, d, a, b);
  });
  for (long node = 0; node < kk; ++node) c[node] = scale * avg[index[cell_of[node]]];
  return c;
}

// ---------------------------------------------------------------------------
// Band-limited kernel Phi_sigma in d = 1 (bandlimit.cpp:307-334): the inverse
// transform of the spectrum restricted to |xi| < sigma. Host-side plan-time
// math for the O(N^2) band-limited and hybrid oracles (fmm.cpp:57-113).
namespace {

// Composite 8-point Gauss-Legendre over `panels` uniform panels of [a, b]
// (bandlimit.cpp:29-44: the panel count, not the rule order, is the knob).
template <class F>
double composite_gl8(const F& f, double a, double b, int panels) {
  static const GaussLegendre<8> rule;
  const double h = (b - a) / panels;
  double sum = 0.0;
  for (int p = 0; p < panels; ++p) {
    const double mid = a + (p + 0.5) * h, half = 0.5 * h;
    double acc = 0.0;
    for (int q = 0; q < 4; ++q) {
      const double dx = half * rule.node(q);
      acc += rule.weight(q) * (f(mid - dx) + f(mid + dx));
    }
    sum += acc * half;
  }
  return sum;
}

// Upper integration limit where the spectrum has decayed below ~1e-17 of its
// scale (bandlimit.cpp:48-58).
double band_cutoff(const KernelSpec& k, double sigma) {
  if (k.type == BLFMM_KERNEL_GAUSSIAN) return std::min(sigma, 12.6 * std::sqrt(k.shape) + 1.0);
  if (k.type == BLFMM_KERNEL_IMQ) return std::min(sigma, 46.0 / k.shape + 1.0);
  return sigma;
}

// Adaptive bisection with the 30-point rule on each half, stopped when one
// more level changes the half-sums by <= tol relative (MQ tail integral).
template <class F>
double adaptive_gl30(const F& f, double a, double b, double whole, int depth, double tol) {
  const double m = 0.5 * (a + b);
  const double left = gl().integrate(f, a, m), right = gl().integrate(f, m, b);
  const double both = left + right, diff = std::abs(both - whole);
  if (depth == 0 || diff <= tol * std::abs(both) || diff < 1e-300) return both;
  return adaptive_gl30(f, a, m, left, depth - 1, tol) +
         adaptive_gl30(f, m, b, right, depth - 1, tol);
}

double plain_kernel(const KernelSpec& k, double r) {  // kernels.cpp:131-161
  const double c = k.shape;
  if (k.type == BLFMM_KERNEL_GAUSSIAN) return std::exp(-c * r * r);
  const double q = std::sqrt(r * r + c * c);
  return k.type == BLFMM_KERNEL_IMQ ? 1.0 / q : q;
}

}  // namespace

double eval_bandlimited_1d(const KernelSpec& k, double sigma, double x, int refinement) {
  if (!(sigma > 0.0)) throw Error(BLFMM_EINVAL, "sigma must be positive");
  if (refinement < 1024) throw Error(BLFMM_EINVAL, "refinement below reference resolution");
  require_fmm_kernel(k);
  const double r = std::abs(x);
  const double hi = band_cutoff(k, sigma);
  auto f = [&](double xi) { return fourier_value(k, std::abs(xi), 1) * std::cos(xi * r); };
  switch (k.type) {
    case BLFMM_KERNEL_GAUSSIAN:  // bandlimit.cpp:61-68
      return composite_gl8(f, 0.0, hi, refinement) / kPi;
    case BLFMM_KERNEL_IMQ: {  // bandlimit.cpp:70-84: K_0's log singularity in a DE head panel
      const double delta = hi / refinement;
      const double head = double_exponential(f, 0.0, delta);
      const double body = refinement > 1 ? composite_gl8(f, delta, hi, refinement - 1) : 0.0;
      return (head + body) / kPi;
    }
    default: {  // MQ, bandlimit.cpp:98-113: Phi - (1/pi) int_sigma^inf Phi^ cos
      const double top = sigma + 60.0 / k.shape;
      const double whole = gl().integrate(f, sigma, top);
      return plain_kernel(k, r) - adaptive_gl30(f, sigma, top, whole, 15, 1e-13) / kPi;
    }
  }
}

std::vector<double> bandlimited_radial_table(const KernelSpec& k, double sigma, double rmax,
                                             int refinement, double* step) {
  if (!(rmax > 0.0) || !std::isfinite(rmax)) throw Error(BLFMM_EINVAL, "rmax must be > 0");
  if (!(sigma > 0.0)) throw Error(BLFMM_EINVAL, "sigma must be positive");
  if (refinement < 1024) throw Error(BLFMM_EINVAL, "refinement below reference resolution");
  require_fmm_kernel(k);
  // process-wide cache keyed like bandlimit.cpp:245-251 (clipped sigma: spectra
  // decayed to nothing by the band edge give the same table for larger sigma)
  using Key = std::tuple<int, double, double, double, int>;
  static std::mutex mu;
  static std::map<Key, std::vector<double>> cache;
  const Key key{k.type, k.shape, band_cutoff(k, sigma), rmax, refinement};
  const double h = rmax / kRadialIntervals;
  if (step) *step = h;
  {
    std::lock_guard<std::mutex> lock(mu);
    if (auto it = cache.find(key); it != cache.end()) return it->second;
  }
  std::vector<double> vals(kRadialIntervals + 3);
  parallel_for(static_cast<long>(vals.size()), [&](long i) {
    vals[i] = eval_bandlimited_1d(k, sigma, i * h, refinement);
  });
  std::lock_guard<std::mutex> lock(mu);
  return cache.emplace(key, std::move(vals)).first->second;
}

}  // namespace blfmm_gpu
