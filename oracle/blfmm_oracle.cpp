// ============================================================================
// TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT.
//
// CPU restatement of the reference's band-limited multilevel FMM matvec
// (blfmm, /root/reference/proj/core), generalised from d in {1,2} to
// d in {1,2,3}. Only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference legs load this library, and only as the
// checker or the CPU baseline. The product (paper_1606_07652_b200) never
// links or calls it.
//
// Pinning: the d <= 2 instantiation is checked against the reference itself
// (oracle/_ref/libblfmm_ref.so, compiled from the reference's own sources) and
// against the reference tests' golden values (tests/test_oracle.py). The d = 3
// instantiation has no reference counterpart; it is pinned by the method's
// defining near/far low-rank sum, which the reference satisfies in d = 2
// (tests/lowrank_split.py). Only its 3-D singular C tables rest on the
// restatement alone, checked by independent quadrature. Empty boxes are not
// allocated: every skipped term is an exact zero in the reference (x + 0*y ==
// x for finite y), so this "sparse" storage is result-identical to the
// reference's dense allocation (mlfmm.cpp:206-216, 273-282).
// ============================================================================
#include <omp.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <map>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

namespace {

using C = std::complex<double>;
constexpr double kPi = 3.14159265358979323846;
constexpr double kTwoPi = 2.0 * kPi;
constexpr double kPoleBall = 1e-8;  // bandlimit.cpp:20

enum KType { GAUSSIAN = 0, MQ = 1, IMQ = 2, TPS = 3, WENDLAND_C2 = 4, WENDLAND31 = 5 };

struct Kernel {
  int type;
  double c;
};

thread_local std::string g_err;
int g_mode = 0, g_stencil = 10;
// Optional target subset (parity checks at sizes where the full far field is
// too slow on the host): the dense leaf ids whose points are evaluated. The
// upsweep still runs over every box (all sources); couple, L2L, L2P and the
// near field run only on the selected leaves and their ancestors, with the
// same per-box arithmetic as the full sweep, so the selected targets' values
// are those of the full matvec. Empty = every leaf.
std::vector<long> g_target_leaves;

// ---------------------------------------------------------------- kernels
// eval_kernel, kernels.cpp:131-161
double eval_kernel(const Kernel& k, double r) {
  r = std::abs(r);
  double c = k.c;
  switch (k.type) {
    case GAUSSIAN:
      return std::exp(-c * r * r);
    case MQ:
      return std::sqrt(r * r + c * c);
    case IMQ:
      return 1.0 / std::sqrt(r * r + c * c);
    case TPS: {  // kernels.cpp:141-146: sign r^beta log r, 0 at r = 0
      if (r == 0.0) return 0.0;
      int beta = static_cast<int>(c);
      double sign = (1 + beta / 2) % 2 == 0 ? 1.0 : -1.0;
      double p = 1.0;  // pow_int: repeated multiplication
      for (int q = 0; q < beta; ++q) p *= r;
      return sign * p * std::log(r);
    }
    case WENDLAND_C2: {  // kernels.cpp:147-152
      double u = c * r;
      if (u >= 1.0) return 0.0;
      double v = 1.0 - u;
      return v * v * v * v * (4.0 * u + 1.0);
    }
    case WENDLAND31: {  // kernels.cpp:153-158
      double u = c * r;
      if (u >= 1.0) return 0.0;
      double v = 1.0 - u;
      return v * v * v * (3.0 * u + 1.0);
    }
  }
  throw std::domain_error("unsupported kernel type");
}

// eval_fourier, kernels.cpp:190-238, extended to d = 3 with the same
// (r^2+c^2)^{-beta} family: Gaussian (pi/c)^{3/2} e^{-xi^2/4c};
// IMQ 4 pi c K1(c xi)/xi; MQ -4 pi c^2 K2(c xi)/xi^2.
double bessel_k(double nu, double z) {  // kernels.cpp:36-44
  if (z > 690.0) return 0.0;
  return std::cyl_bessel_k(nu, z);
}

double eval_fourier(const Kernel& k, double xi, int d) {
  if (d < 1 || d > 3) throw std::invalid_argument("d must be 1, 2 or 3");
  xi = std::abs(xi);
  double c = k.c;
  switch (k.type) {
    case GAUSSIAN:
      return std::pow(kPi / c, 0.5 * d) * std::exp(-xi * xi / (4.0 * c));
    case IMQ:
      if (xi == 0.0) throw std::domain_error("imq transform singular at xi=0");
      if (d == 1) return 2.0 * bessel_k(0.0, c * xi);
      if (d == 2) return 2.0 * kPi * std::exp(-c * xi) / xi;
      return 4.0 * kPi * c * bessel_k(1.0, c * xi) / xi;
    case MQ:
      if (xi == 0.0)
        throw std::domain_error("mq generalized transform singular at xi=0");
      if (d == 1) return -2.0 * c * bessel_k(1.0, c * xi) / xi;
      if (d == 2)
        return -2.0 * kPi * (1.0 + c * xi) * std::exp(-c * xi) /
               (xi * xi * xi);
      return -4.0 * kPi * c * c * bessel_k(2.0, c * xi) / (xi * xi);
  }
  throw std::domain_error("unsupported kernel type");
}

bool singular_at_origin(const Kernel& k) { return k.type != GAUSSIAN; }

// ----------------------------------------------------------- quadrature
// 30-point Gauss-Legendre (the reference uses Boost's gauss<double,30>).
struct GL30 {
  double x[15], w[15];  // positive abscissae, ascending
  GL30() {
    const int n = 30;
    for (int i = 0; i < 15; ++i) {
      long double z = std::cos(3.14159265358979323846264338L * (i + 0.75L) / (n + 0.5L));
      long double dp = 0;
      for (int it = 0; it < 100; ++it) {
        long double p0 = 1, p1 = z;
        for (int kk = 2; kk <= n; ++kk) {
          long double p2 = ((2.0L * kk - 1) * z * p1 - (kk - 1.0L) * p0) / kk;
          p0 = p1;
          p1 = p2;
        }
        dp = n * (z * p1 - p0) / (z * z - 1);
        long double dz = p1 / dp;
        z -= dz;
        if (std::fabs(dz) < 1e-21L) break;
      }
      long double p0 = 1, p1 = z;
      for (int kk = 2; kk <= n; ++kk) {
        long double p2 = ((2.0L * kk - 1) * z * p1 - (kk - 1.0L) * p0) / kk;
        p0 = p1;
        p1 = p2;
      }
      dp = n * (z * p1 - p0) / (z * z - 1);
      x[14 - i] = static_cast<double>(z);
      w[14 - i] = static_cast<double>(2.0L / ((1 - z * z) * dp * dp));
    }
  }
  template <class F>
  double integrate(const F& f, double a, double b) const {
    double avg = (a + b) * 0.5, scale = (b - a) * 0.5;
    double r = 0.0;
    for (int i = 0; i < 15; ++i)
      r += (f(avg + scale * x[i]) + f(avg - scale * x[i])) * w[i];
    return scale * r;
  }
};
const GL30& gl30() {
  static const GL30 g;
  return g;
}

// Double-exponential (tanh-sinh) rule on [a,b], nodes placed through their
// endpoint complement; tolerance sqrt(eps) relative to L1 (Boost default).
template <class F>
double tanh_sinh(const F& f, double a, double b) {
  if (a == b) return 0.0;
  if (b < a) return -tanh_sinh(f, b, a);
  const double hp = kPi / 2, c = (a + b) / 2, h = (b - a) / 2;
  const double tol = std::sqrt(2.220446049250313e-16);
  double step = 1.0, sum = f(c) * hp, l1 = std::abs(sum);
  auto add = [&](double t0, double dt) {
    for (double t = t0; t <= 6.56; t += dt) {
      double s = hp * std::sinh(t), e = std::exp(-2 * s);
      double comp = 2 * e / (1 + e), ch = std::cosh(s);
      double w = hp * std::cosh(t) / (ch * ch);
      double xr = b - h * comp, xl = a + h * comp;
      if (!(xr < b) || !(xl > a)) break;
      double fr = f(xr), fl = f(xl);
      sum += w * (fr + fl);
      l1 += w * (std::abs(fr) + std::abs(fl));
    }
  };
  add(step, step);
  double prev = sum * step * h, est = prev;
  for (int k = 1; k <= 15; ++k) {
    step /= 2;
    add(step, 2 * step);
    est = sum * step * h;
    if (k >= 3 && std::abs(est - prev) <= tol * l1 * step * h) break;
    prev = est;
  }
  return est;
}

// corner_polar, bandlimit.cpp:134-154 (x1 = x2 = 0 as in cell_average_2d)
template <class S>
double corner_polar(const S& spec, double delta, double r0) {
  const GL30& g = gl30();
  auto sector = [&](double t0, double t1, auto rmax) {
    auto outer = [&](double th) {
      double rm = rmax(th);
      auto inner = [&](double r) { return r * spec(r); };
      return g.integrate(inner, r0, rm);
    };
    return g.integrate(outer, t0, t1);
  };
  double v = sector(0.0, 0.25 * kPi, [&](double t) { return delta / std::cos(t); });
  v += sector(0.25 * kPi, 0.5 * kPi, [&](double t) { return delta / std::sin(t); });
  return v;
}

// 3-D analogue: integral of spec(|xi|) over the corner cube [0,delta]^3 with
// the pole ball |xi| < r0 excluded. The cube splits into 3 congruent
// pyramids (largest coordinate), each into 2 congruent azimuth halves:
//   6 * int_0^{pi/4} dphi int_0^{atan(1/cos phi)} sin(th) dth
//         int_{r0}^{delta/cos th} rho^2 spec(rho) drho.
template <class S>
double corner_spherical(const S& spec, double delta, double r0) {
  const GL30& g = gl30();
  auto over_phi = [&](double phi) {
    double thmax = std::atan(1.0 / std::cos(phi));
    auto over_th = [&](double th) {
      double rm = delta / std::cos(th);
      auto inner = [&](double r) { return r * r * spec(r); };
      return std::sin(th) * g.integrate(inner, r0, rm);
    };
    return g.integrate(over_th, 0.0, thmax);
  };
  return 6.0 * g.integrate(over_phi, 0.0, 0.25 * kPi);
}

// cell_average_1d, bandlimit.cpp:336-350
double cell_average_1d(const Kernel& k, double a, double b) {
  auto f = [&](double xi) { return eval_fourier(k, std::abs(xi), 1); };
  double lo = a, hi = b, integral;
  if (lo < 0.0 && hi > 0.0) {
    integral = tanh_sinh(f, lo, -kPoleBall) + tanh_sinh(f, kPoleBall, hi);
  } else {
    if (lo == 0.0) lo = kPoleBall;
    if (hi == 0.0) hi = -kPoleBall;
    integral = tanh_sinh(f, lo, hi);
  }
  return integral / (b - a);
}

// cell_average_2d, bandlimit.cpp:355-384
double cell_average_2d(const Kernel& k, double a1, double b1, double a2,
                       double b2) {
  auto spec = [&](double rho) { return eval_fourier(k, rho, 2); };
  if (b1 <= 0.0) std::swap(a1, b1), a1 = -a1, b1 = -b1;
  if (b2 <= 0.0) std::swap(a2, b2), a2 = -a2, b2 = -b2;
  if (a1 < 0.0 || a2 < 0.0) {
    double area = (b1 - a1) * (b2 - a2);
    double v;
    if (a1 < 0.0) {
      v = cell_average_2d(k, a1, 0.0, a2, b2) * (-a1) * (b2 - a2) +
          cell_average_2d(k, 0.0, b1, a2, b2) * b1 * (b2 - a2);
    } else {
      v = cell_average_2d(k, a1, b1, a2, 0.0) * (b1 - a1) * (-a2) +
          cell_average_2d(k, a1, b1, 0.0, b2) * (b1 - a1) * b2;
    }
    return v / area;
  }
  double area = (b1 - a1) * (b2 - a2);
  if (a1 == 0.0 && a2 == 0.0 && b1 == b2)
    return corner_polar(spec, b1, kPoleBall) / area;
  const GL30& g = gl30();
  auto outer = [&](double x1) {
    auto inner = [&](double x2) { return spec(std::hypot(x1, x2)); };
    return g.integrate(inner, a2, b2);
  };
  return g.integrate(outer, a1, b1) / area;
}

// cell_average_3d: the same fold / split / corner / tensor-rule structure.
double cell_average_3d(const Kernel& k, double a[3], double b[3]) {
  auto spec = [&](double rho) { return eval_fourier(k, rho, 3); };
  for (int ax = 0; ax < 3; ++ax)
    if (b[ax] <= 0.0) std::swap(a[ax], b[ax]), a[ax] = -a[ax], b[ax] = -b[ax];
  double vol = (b[0] - a[0]) * (b[1] - a[1]) * (b[2] - a[2]);
  for (int ax = 0; ax < 3; ++ax) {
    if (a[ax] < 0.0) {
      double al[3] = {a[0], a[1], a[2]}, bl[3] = {b[0], b[1], b[2]};
      double ar[3] = {a[0], a[1], a[2]}, br[3] = {b[0], b[1], b[2]};
      bl[ax] = 0.0;
      ar[ax] = 0.0;
      double other = vol / (b[ax] - a[ax]);
      double v = cell_average_3d(k, al, bl) * (-a[ax]) * other +
                 cell_average_3d(k, ar, br) * b[ax] * other;
      return v / vol;
    }
  }
  if (a[0] == 0.0 && a[1] == 0.0 && a[2] == 0.0 && b[0] == b[1] && b[1] == b[2])
    return corner_spherical(spec, b[0], kPoleBall) / vol;
  const GL30& g = gl30();
  auto f1 = [&](double x1) {
    auto f2 = [&](double x2) {
      auto f3 = [&](double x3) { return spec(std::hypot(x1, x2, x3)); };
      return g.integrate(f3, a[2], b[2]);
    };
    return g.integrate(f2, a[1], b[1]);
  };
  return g.integrate(f1, a[0], b[0]) / vol;
}

// translation_coefficients, spectral mode, bandlimit.cpp:388-447.
// Node order is make_quadrature's row-major tensor order
// (bandlimit.cpp:279-290), extended to (m1*M + m2)*M + m3 for d = 3.
std::vector<double> c_table(const Kernel& k, double sigma, int M, int d) {
  if (!(sigma > 0.0)) throw std::invalid_argument("sigma must be positive");
  if (M < 2) throw std::invalid_argument("m_per_dim must be >= 2");
  if (d < 1 || d > 3) throw std::invalid_argument("d must be 1, 2 or 3");
  long K = 1;
  for (int i = 0; i < d; ++i) K *= M;
  double dxi = 2.0 * sigma / M;
  double inv = 1.0;
  for (int i = 0; i < d; ++i) inv /= kTwoPi;
  // bandlimit.cpp:395 computes (2pi)^{-d} as 1/(2pi)^d
  inv = d == 1 ? 1.0 / kTwoPi
               : (d == 2 ? 1.0 / (kTwoPi * kTwoPi)
                         : 1.0 / (kTwoPi * kTwoPi * kTwoPi));
  std::vector<double> ax(M);
  for (int m = 0; m < M; ++m) ax[m] = -sigma + m * dxi;
  std::vector<double> out(K);
  bool sing = singular_at_origin(k);
  if (!sing) {
#pragma omp parallel for schedule(static)
    for (long m = 0; m < K; ++m) {
      long r = m;
      double x[3] = {0, 0, 0};
      for (int i = d - 1; i >= 0; --i) {
        x[i] = ax[r % M];
        r /= M;
      }
      double rho = d == 1 ? std::abs(x[0])
                          : (d == 2 ? std::hypot(x[0], x[1])
                                    : std::hypot(x[0], x[1], x[2]));
      out[m] = inv * eval_fourier(k, rho, d);
    }
    return out;
  }
  if (d == 1) {
    for (int m = 0; m < M; ++m)
      out[m] = inv * cell_average_1d(k, ax[m], ax[m] + dxi);
  } else if (d == 2) {
#pragma omp parallel for schedule(dynamic)
    for (long m = 0; m < K; ++m) {
      double a1 = ax[m / M], a2 = ax[m % M];
      out[m] = inv * cell_average_2d(k, a1, a1 + dxi, a2, a2 + dxi);
    }
  } else {
    // Cells whose folded bounds coincide bit-for-bit are computed once.
    using Key = std::tuple<double, double, double, double, double, double>;
    std::vector<Key> keys(K);
    for (long m = 0; m < K; ++m) {
      long r = m;
      double a[3], b[3];
      for (int i = 2; i >= 0; --i) {
        a[i] = ax[r % M];
        b[i] = a[i] + dxi;
        r /= M;
      }
      for (int i = 0; i < 3; ++i)
        if (b[i] <= 0.0) std::swap(a[i], b[i]), a[i] = -a[i], b[i] = -b[i];
      keys[m] = Key{a[0], b[0], a[1], b[1], a[2], b[2]};
    }
    std::map<Key, long> uniq;
    std::vector<Key> ulist;
    for (long m = 0; m < K; ++m)
      if (uniq.emplace(keys[m], (long)ulist.size()).second) ulist.push_back(keys[m]);
    std::vector<double> uval(ulist.size());
#pragma omp parallel for schedule(dynamic)
    for (long u = 0; u < (long)ulist.size(); ++u) {
      double a[3] = {std::get<0>(ulist[u]), std::get<2>(ulist[u]), std::get<4>(ulist[u])};
      double b[3] = {std::get<1>(ulist[u]), std::get<3>(ulist[u]), std::get<5>(ulist[u])};
      uval[u] = cell_average_3d(k, a, b);
    }
    for (long m = 0; m < K; ++m) out[m] = inv * uval[uniq[keys[m]]];
  }
  return out;
}

// ------------------------------------------------------------------ tree
// BoxTree semantics of geometry.hpp:49-72 / geometry.cpp:201-321 for
// d <= 3: row-major ids ((i*n)+j)*n+k, clipped 3^d neighbor block, interaction
// list = children of the parent's neighbors minus own neighbors (levels >= 2),
// leaf binning by truncation + clamp, leaf points in ascending index order.
struct Tree {
  int d = 1, L = 2;
  double lo[3] = {0, 0, 0}, hi[3] = {1, 1, 1};
  std::vector<long> leaf_start;  // CSR over dense leaf ids
  std::vector<int> leaf_pts;
  std::vector<std::vector<char>> occ;  // [level][box] subtree has points

  long nper(int l) const { return 1L << l; }
  long count(int l) const { return 1L << (d * l); }
  double side(int l, int k) const { return (hi[k] - lo[k]) / nper(l); }
  void idx(int l, long b, long* i) const {
    long n = nper(l);
    for (int k = d - 1; k >= 0; --k) {
      i[k] = b % n;
      b /= n;
    }
  }
  long id(int l, const long* i) const {
    long n = nper(l), b = 0;
    for (int k = 0; k < d; ++k) b = b * n + i[k];
    return b;
  }
  void center(int l, long b, double* c) const {
    long i[3];
    idx(l, b, i);
    for (int k = 0; k < 3; ++k) c[k] = 0.0;
    for (int k = 0; k < d; ++k) c[k] = lo[k] + (i[k] + 0.5) * side(l, k);
  }
  long leaf_of(const double* x) const {
    long n = nper(L), i[3];
    for (int k = 0; k < d; ++k) {
      long v = static_cast<int>((x[k] - lo[k]) / side(L, k));
      i[k] = std::clamp(v, 0L, n - 1);
    }
    return id(L, i);
  }
  std::vector<long> children(int l, long b) const {
    std::vector<long> out;
    if (l >= L) return out;
    long i[3], c[3];
    idx(l, b, i);
    int nc = 1 << d;
    for (int q = 0; q < nc; ++q) {  // row-major over (di, dj, dk)
      for (int k = 0; k < d; ++k) c[k] = 2 * i[k] + ((q >> (d - 1 - k)) & 1);
      out.push_back(id(l + 1, c));
    }
    return out;
  }
  std::vector<long> neighbors(int l, long b) const {
    std::vector<long> out;
    long i[3], c[3], n = nper(l);
    idx(l, b, i);
    int tot = 1;
    for (int k = 0; k < d; ++k) tot *= 3;
    for (int q = 0; q < tot; ++q) {
      int r = q;
      bool ok = true;
      for (int k = d - 1; k >= 0; --k) {
        c[k] = i[k] + (r % 3) - 1;
        r /= 3;
        if (c[k] < 0 || c[k] >= n) ok = false;
      }
      if (ok) out.push_back(id(l, c));
    }
    std::sort(out.begin(), out.end());
    return out;
  }
  std::vector<long> interaction(int l, long b) const {
    std::vector<long> out;
    if (l < 2) return out;
    long i[3], p[3], c[3], np = nper(l) / 2;
    idx(l, b, i);
    for (int k = 0; k < d; ++k) p[k] = i[k] / 2;
    int tot = 1;
    for (int k = 0; k < d; ++k) tot *= 3;
    for (int q = 0; q < tot; ++q) {
      int r = q;
      long qq[3];
      bool ok = true;
      for (int k = d - 1; k >= 0; --k) {
        qq[k] = p[k] + (r % 3) - 1;
        r /= 3;
        if (qq[k] < 0 || qq[k] >= np) ok = false;
      }
      if (!ok) continue;
      for (int cq = 0; cq < (1 << d); ++cq) {
        bool own = true;
        for (int k = 0; k < d; ++k) {
          c[k] = 2 * qq[k] + ((cq >> (d - 1 - k)) & 1);
          if (std::abs(c[k] - i[k]) > 1) own = false;
        }
        if (own) continue;
        out.push_back(id(l, c));
      }
    }
    std::sort(out.begin(), out.end());
    return out;
  }
  long npts(long leaf) const { return leaf_start[leaf + 1] - leaf_start[leaf]; }
  const int* pts(long leaf) const { return leaf_pts.data() + leaf_start[leaf]; }
  long parent(int l, long b) const {
    long i[3];
    idx(l, b, i);
    for (int k = 0; k < d; ++k) i[k] /= 2;
    return id(l - 1, i);
  }
};

struct Problem {
  int d;
  long n;
  const double* x;  // n*d, AoS
  double lo[3], hi[3];
  Kernel k;
  double sigma;
  int M;
  int L;
};

Tree build_tree(const Problem& p, int L) {
  if (L < 2) throw std::invalid_argument("leaf_level must be >= 2");
  if (p.d * L > 24) throw std::invalid_argument("box count cap exceeded");
  Tree t;
  t.d = p.d;
  t.L = L;
  for (int k = 0; k < 3; ++k) t.lo[k] = p.lo[k], t.hi[k] = p.hi[k];
  long nb = t.count(L);
  std::vector<long> leaf(p.n);
  t.leaf_start.assign(nb + 1, 0);
  for (long i = 0; i < p.n; ++i) {
    leaf[i] = t.leaf_of(p.x + i * p.d);
    t.leaf_start[leaf[i] + 1]++;
  }
  for (long b = 0; b < nb; ++b) t.leaf_start[b + 1] += t.leaf_start[b];
  t.leaf_pts.resize(p.n);
  std::vector<long> fill(t.leaf_start.begin(), t.leaf_start.end() - 1);
  for (long i = 0; i < p.n; ++i) t.leaf_pts[fill[leaf[i]]++] = static_cast<int>(i);
  t.occ.resize(L + 1);
  for (int l = 0; l <= L; ++l) t.occ[l].assign(t.count(l), 0);
  for (long b = 0; b < nb; ++b)
    if (t.npts(b) > 0) t.occ[L][b] = 1;
  for (int l = L; l >= 1; --l)
    for (long b = 0; b < t.count(l); ++b)
      if (t.occ[l][b]) t.occ[l - 1][t.parent(l, b)] = 1;
  return t;
}

double dot(int d, const double* a, const double* b) {  // common.hpp:15-19
  double s = a[0] * b[0];
  if (d >= 2) s += a[1] * b[1];
  if (d == 3) s += a[2] * b[2];
  return s;
}
double dist(int d, const double* a, const double* b) {  // common.hpp:21-29
  double dx = a[0] - b[0];
  double s = dx * dx;
  if (d >= 2) {
    double dy = a[1] - b[1];
    s += dy * dy;
  }
  if (d == 3) {
    double dz = a[2] - b[2];
    s += dz * dz;
  }
  return std::sqrt(s);
}

struct Grid {  // make_quadrature, bandlimit.cpp:269-292
  int d, M;
  long K;
  double weight;
  std::vector<double> nodes;  // K*3
};
Grid make_grid(double sigma, int M, int d) {
  if (!(sigma > 0.0)) throw std::invalid_argument("sigma must be positive");
  if (M < 2) throw std::invalid_argument("m_per_dim must be >= 2");
  Grid g;
  g.d = d;
  g.M = M;
  g.K = 1;
  for (int i = 0; i < d; ++i) g.K *= M;
  double dxi = 2.0 * sigma / M;
  g.weight = d == 1 ? dxi : (d == 2 ? dxi * dxi : dxi * dxi * dxi);
  g.nodes.assign(g.K * 3, 0.0);
  for (long m = 0; m < g.K; ++m) {
    long r = m;
    for (int i = d - 1; i >= 0; --i) {
      g.nodes[m * 3 + i] = -sigma + (r % M) * dxi;
      r /= M;
    }
  }
  return g;
}

// Per-axis k-point Lagrange interpolation (lagrange_matrix, mlfmm.cpp:42-80):
// row r holds the weights of source nodes lo[r] .. lo[r]+k-1 at target r.
struct Interp {
  int rows = 0, cols = 0, k = 0;
  std::vector<int> lo;
  std::vector<double> w;  // rows*k
};
Interp lagrange(const std::vector<double>& src, const std::vector<double>& tgt, int k) {
  int n = static_cast<int>(src.size());
  if (k < 1 || k > n) throw std::invalid_argument("stencil size out of range");
  for (int i = 1; i < n; ++i)
    if (!(src[i] > src[i - 1])) throw std::invalid_argument("source nodes must be strictly increasing");
  Interp P;
  P.rows = static_cast<int>(tgt.size());
  P.cols = n;
  P.k = k;
  P.lo.resize(P.rows);
  P.w.resize((size_t)P.rows * k);
  for (int r = 0; r < P.rows; ++r) {
    double t = tgt[r];
    int lo = static_cast<int>(std::lower_bound(src.begin(), src.end(), t) - src.begin()) - k / 2;
    lo = std::clamp(lo, 0, n - k);
    while (lo > 0 && t - src[lo - 1] < src[lo + k - 1] - t) --lo;
    while (lo + k < n && src[lo + k] - t < t - src[lo]) ++lo;
    P.lo[r] = lo;
    for (int j = 0; j < k; ++j) {
      double w = 1.0;
      for (int l = 0; l < k; ++l) {
        if (l == j) continue;
        w *= (t - src[lo + l]) / (src[lo + j] - src[lo + l]);
      }
      P.w[(size_t)r * k + j] = w;
    }
  }
  return P;
}
std::vector<double> axis_nodes(double sigma, int M) {  // mlfmm.cpp:15-20
  std::vector<double> v(M);
  double dxi = 2.0 * sigma / M;
  for (int m = 0; m < M; ++m) v[m] = -sigma + m * dxi;
  return v;
}

// make_level_grids (mlfmm.cpp:112-142): shared mode reuses the leaf grid and
// C table at every level; scaled mode halves the band per coarsening step
// (sigma_{l-1} = sigma_l / 2, weights / 2^d), one C table per level and the
// child -> parent Lagrange transfer P[l] (grid l nodes -> grid l-1 nodes).
struct Grids {
  bool scaled = false;
  int k = 0;
  std::vector<Grid> g;                 // [0..L]
  std::vector<std::vector<double>> c;  // [0..L]
  std::vector<Interp> P;               // [3..L]
  std::vector<double> sig;             // band per level
};
Grids make_grids(const Kernel& kern, double sigma, int M, int d, int L, int mode, int stencil,
                 const double* c_in) {
  Grids G;
  G.scaled = mode == 1;
  G.k = std::min(stencil, M);
  G.g.resize(L + 1);
  G.c.resize(L + 1);
  G.sig.assign(L + 1, sigma);
  long K = 1;
  for (int i = 0; i < d; ++i) K *= M;
  double s = sigma;
  for (int l = L; l >= 2; --l) {
    G.sig[l] = s;
    G.g[l] = make_grid(s, M, d);
    if (!G.scaled && l < L) {
      G.c[l] = G.c[L];
    } else if (c_in) {  // caller tables: one per level (levels 2..L) in scaled mode
      const double* src = G.scaled ? c_in + (long)(l - 2) * K : c_in;
      G.c[l].assign(src, src + K);
    } else {
      G.c[l] = c_table(kern, s, M, d);
    }
    if (G.scaled) s = s / 2.0;
  }
  if (G.scaled) {
    G.P.resize(L + 1);
    for (int l = 3; l <= L; ++l)
      G.P[l] = lagrange(axis_nodes(G.sig[l], M), axis_nodes(G.sig[l - 1], M), G.k);
  }
  return G;
}

// Tensor application of P along every axis (interp_apply, mlfmm.cpp:146-171;
// axis 0 first) and of P^T (interp_apply_transpose, 173-197).
void interp_tensor(const Interp& P, int d, int M, const std::vector<C>& x, std::vector<C>& out,
                   bool transpose) {
  std::vector<C> cur = x, nxt(x.size());
  long K = (long)cur.size();
  for (int ax = 0; ax < d; ++ax) {
    long stride = 1;
    for (int q = ax + 1; q < d; ++q) stride *= M;
    std::fill(nxt.begin(), nxt.end(), C(0.0, 0.0));
    for (long base = 0; base < K; ++base) {
      if ((base / stride) % M != 0) continue;  // base has axis index 0
      for (int r = 0; r < P.rows; ++r)
        for (int j = 0; j < P.k; ++j) {
          const int c = P.lo[r] + j;
          const double w = P.w[(size_t)r * P.k + j];
          if (!transpose)
            nxt[base + r * stride] += w * cur[base + c * stride];
          else
            nxt[base + c * stride] += w * cur[base + r * stride];
        }
    }
    std::swap(cur, nxt);
  }
  out = std::move(cur);
}

using Level = std::vector<std::vector<C>>;  // [box] -> K coeffs (empty = 0)

struct Stats {
  long long near_pairs;
  long long far_work;
  double max_imag;
};

// Optional stage sampling for the CPU baseline: only every `stride`-th
// occupied box of each stage is processed (outputs then meaningless; the
// stage time is multiplied back by the stride).
struct Sampler {
  int stride = 1;
  double t[6] = {0, 0, 0, 0, 0, 0};  // p2m, m2m, m2l, l2l, l2p, near
};

template <class F>
double timed(F&& f) {
  auto t0 = std::chrono::steady_clock::now();
  f();
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

std::vector<long> occupied(const Tree& t, int l, int stride) {
  std::vector<long> v;
  long cnt = 0;
  for (long b = 0; b < t.count(l); ++b)
    if (t.occ[l][b] && (cnt++ % stride) == 0) v.push_back(b);
  return v;
}

// Boxes of level l that are ancestors of (or are) a selected target leaf.
std::vector<char> target_chain(const Tree& t, int l) {
  std::vector<char> on(t.count(l), g_target_leaves.empty() ? 1 : 0);
  for (long a : g_target_leaves) {
    long i[3];
    t.idx(t.L, a, i);
    for (int k = 0; k < t.d; ++k) i[k] >>= (t.L - l);
    on[t.id(l, i)] = 1;
  }
  return on;
}
std::vector<long> occupied_targets(const Tree& t, int l, int stride) {
  auto v = occupied(t, l, stride);
  if (g_target_leaves.empty()) return v;
  auto on = target_chain(t, l);
  std::vector<long> out;
  for (long b : v)
    if (on[b]) out.push_back(b);
  return out;
}

// upsweep, mlfmm.cpp:201-266 (shared grids)
std::vector<Level> upsweep(const Problem& p, const Tree& t, const Grids& G,
                           const double* w, Sampler* s) {
  int L = t.L, stride = s ? s->stride : 1;
  const Grid& g = G.g[L];
  std::vector<Level> ex(L + 1);
  for (int l = 2; l <= L; ++l) ex[l].resize(t.count(l));
  if (stride > 1)  // sampled timing: every occupied box holds (zero) data so
                   // sampled boxes read real memory for all their sources
    for (int l = 2; l <= L; ++l)
      for (long b : occupied(t, l, 1)) ex[l][b].assign(g.K, C(0.0, 0.0));
  auto leaves = occupied(t, L, stride);
  double tp = timed([&] {
#pragma omp parallel for schedule(dynamic)
    for (long q = 0; q < (long)leaves.size(); ++q) {
      long b = leaves[q];
      double xb[3];
      t.center(L, b, xb);
      auto& co = ex[L][b];
      co.assign(g.K, C(0.0, 0.0));
      const int* pj = t.pts(b);
      for (long jj = 0; jj < t.npts(b); ++jj) {
        int j = pj[jj];
        double r[3] = {0, 0, 0};
        for (int k = 0; k < p.d; ++k) r[k] = xb[k] - p.x[(long)j * p.d + k];
        for (long m = 0; m < g.K; ++m)
          co[m] += w[j] * std::polar(1.0, dot(p.d, &g.nodes[m * 3], r));
      }
    }
  });
  double tm = timed([&] {
    for (int l = L; l >= 3; --l) {
      auto parents = occupied(t, l - 1, stride);
#pragma omp parallel for schedule(dynamic)
      for (long q = 0; q < (long)parents.size(); ++q) {
        long pb = parents[q];
        double xp[3];
        t.center(l - 1, pb, xp);
        auto& out = ex[l - 1][pb];
        out.assign(g.K, C(0.0, 0.0));
        const Grid& gp = G.g[l - 1];
        std::vector<C> tmp;
        for (long c : t.children(l - 1, pb)) {
          const auto& vc = ex[l][c];
          if (vc.empty()) continue;
          double xc[3];
          t.center(l, c, xc);
          double r[3] = {0, 0, 0};
          for (int k = 0; k < p.d; ++k) r[k] = xp[k] - xc[k];
          if (!G.scaled) {
            for (long m = 0; m < g.K; ++m)
              out[m] += std::polar(1.0, dot(p.d, &gp.nodes[m * 3], r)) * vc[m];
          } else {  // mlfmm.cpp:256-261: interpolate to the parent grid, then shift
            interp_tensor(G.P[l], p.d, p.M, vc, tmp, false);
            for (long m = 0; m < g.K; ++m)
              out[m] += std::polar(1.0, dot(p.d, &gp.nodes[m * 3], r)) * tmp[m];
          }
        }
      }
    }
  });
  if (s) s->t[0] += tp * stride, s->t[1] += tm * stride;
  return ex;
}

// couple, mlfmm.cpp:268-299
std::vector<Level> couple(const Problem& p, const Tree& t, const Grids& G,
                          const std::vector<Level>& mult, Sampler* s) {
  int L = t.L, stride = s ? s->stride : 1;
  const Grid& g = G.g[L];
  std::vector<Level> loc(L + 1);
  if (stride > 1)
    for (int l = 2; l <= L; ++l) {
      loc[l].resize(t.count(l));
      for (long b : occupied(t, l, 1)) loc[l][b].assign(g.K, C(0.0, 0.0));
    }
  double tc = timed([&] {
    for (int l = 2; l <= L; ++l) {
      loc[l].resize(t.count(l));
      auto targets = occupied_targets(t, l, stride);
#pragma omp parallel for schedule(dynamic)
      for (long q = 0; q < (long)targets.size(); ++q) {
        long a = targets[q];
        double xa[3];
        t.center(l, a, xa);
        auto& out = loc[l][a];
        if (out.empty()) out.assign(g.K, C(0.0, 0.0));
        const Grid& gl = G.g[l];
        const std::vector<double>& cv = G.c[l];
        for (long b : t.interaction(l, a)) {
          const auto& vb = mult[l][b];
          if (vb.empty()) continue;
          double xb[3];
          t.center(l, b, xb);
          double r[3] = {0, 0, 0};
          for (int k = 0; k < p.d; ++k) r[k] = xa[k] - xb[k];
          for (long m = 0; m < g.K; ++m)
            out[m] += cv[m] * std::polar(1.0, dot(p.d, &gl.nodes[m * 3], r)) * vb[m];
        }
      }
    }
  });
  if (s) s->t[2] += tc * stride;
  return loc;
}

// downsweep, mlfmm.cpp:301-359
void downsweep(const Problem& p, const Tree& t, const Grids& G,
               const std::vector<Level>& locals, double* out, double* max_imag,
               Sampler* s, std::vector<Level>* acc_out = nullptr) {
  int L = t.L, stride = s ? s->stride : 1;
  const Grid& g = G.g[L];
  std::vector<Level> acc;
  double tcopy = timed([&] { acc = locals; });  // mlfmm.cpp:305
  double tl = timed([&] {
    for (int l = 2; l < L; ++l) {
      auto parents = occupied_targets(t, l, stride);
#pragma omp parallel for schedule(dynamic)
      for (long q = 0; q < (long)parents.size(); ++q) {
        long pb = parents[q];
        const auto& lp = acc[l][pb];
        if (lp.empty()) continue;
        double xp[3];
        t.center(l, pb, xp);
        const Grid& gc = G.g[l + 1];
        const double wratio = G.g[l].weight / gc.weight;  // uniform weights
        std::vector<C> tmp;
        if (G.scaled) interp_tensor(G.P[l + 1], p.d, p.M, lp, tmp, true);
        for (long c : t.children(l, pb)) {
          auto& lc = acc[l + 1][c];
          if (lc.empty()) continue;  // unoccupied child: never reaches a point
          double xc[3];
          t.center(l + 1, c, xc);
          double r[3] = {0, 0, 0};
          for (int k = 0; k < p.d; ++k) r[k] = xc[k] - xp[k];
          if (!G.scaled) {
            for (long m = 0; m < g.K; ++m)
              lc[m] += std::polar(1.0, dot(p.d, &gc.nodes[m * 3], r)) * lp[m];
          } else {  // mlfmm.cpp:331-337: anterpolate, weight ratio, shift
            for (long m = 0; m < g.K; ++m)
              lc[m] += wratio * std::polar(1.0, dot(p.d, &gc.nodes[m * 3], r)) * tmp[m];
          }
        }
      }
    }
  });
  double imag = 0.0;
  auto leaves = occupied_targets(t, L, stride);
  double tp = timed([&] {
#pragma omp parallel for schedule(dynamic) reduction(max : imag)
    for (long q = 0; q < (long)leaves.size(); ++q) {
      long a = leaves[q];
      const auto& la = acc[L][a];
      if (la.empty()) continue;
      double xa[3];
      t.center(L, a, xa);
      const int* pi = t.pts(a);
      for (long ii = 0; ii < t.npts(a); ++ii) {
        int i = pi[ii];
        double r[3] = {0, 0, 0};
        for (int k = 0; k < p.d; ++k) r[k] = p.x[(long)i * p.d + k] - xa[k];
        C v(0.0, 0.0);
        for (long m = 0; m < g.K; ++m)
          v += g.weight * std::polar(1.0, dot(p.d, &g.nodes[m * 3], r)) * la[m];
        out[i] += v.real();
        imag = std::max(imag, std::abs(v.imag()));
      }
    }
  });
  if (max_imag) *max_imag = imag;
  if (s) s->t[3] += tl * stride + tcopy, s->t[4] += tp * stride;
  if (acc_out) *acc_out = std::move(acc);
}

long long sum_il_sizes(const Tree& t, int l) {
  // sum_a |IL_l(a)| over the dense box set: the 6-block and 3-block counts
  // factor over axes (per-axis clipped sizes).
  long n = t.nper(l), np = n / 2;
  long long s6 = 1, s3 = 1;
  for (int k = 0; k < t.d; ++k) {
    long long a6 = 0, a3 = 0;
    for (long i = 0; i < n; ++i) {
      long pi = i / 2;
      long lo6 = std::max(0L, pi - 1), hi6 = std::min(np - 1, pi + 1);
      a6 += 2 * (hi6 - lo6 + 1);
      long lo3 = std::max(0L, i - 1), hi3 = std::min(n - 1, i + 1);
      a3 += hi3 - lo3 + 1;
    }
    s6 *= a6;
    s3 *= a3;
  }
  return s6 - s3;
}

// mlfmm_matvec, mlfmm.cpp:361-406
void mlfmm(const Problem& p, const Grids& G, const double* w, double* out, Stats* st,
           Sampler* s) {
  if (p.L < 2) throw std::invalid_argument("leaf_level must be >= 2");
  Tree t = build_tree(p, p.L);
  const Grid& g = G.g[p.L];
  std::fill(out, out + p.n, 0.0);
  auto mult = upsweep(p, t, G, w, s);
  auto loc = couple(p, t, G, mult, s);
  mult.clear();
  double imag = 0.0;
  downsweep(p, t, G, loc, out, &imag, s);
  loc.clear();
  int L = t.L, stride = s ? s->stride : 1;
  long long near = 0;
  auto leaves = occupied_targets(t, L, stride);
  double tn = timed([&] {
#pragma omp parallel for schedule(dynamic) reduction(+ : near)
    for (long q = 0; q < (long)leaves.size(); ++q) {
      long a = leaves[q];
      auto nb = t.neighbors(L, a);
      const int* pi = t.pts(a);
      for (long ii = 0; ii < t.npts(a); ++ii) {
        int i = pi[ii];
        double v = 0.0;
        for (long b : nb) {
          const int* pj = t.pts(b);
          for (long jj = 0; jj < t.npts(b); ++jj) {
            int j = pj[jj];
            v += w[j] * eval_kernel(p.k, dist(p.d, p.x + (long)i * p.d, p.x + (long)j * p.d));
            ++near;
          }
        }
        out[i] += v;
      }
    }
  });
  if (s) s->t[5] += tn * stride;
  if (st) {
    st->near_pairs = near;
    st->max_imag = imag;
    long long far = 2LL * p.n * g.K;
    for (int l = 2; l <= L; ++l) far += sum_il_sizes(t, l) * g.K;
    st->far_work = far;
  }
}

// fmm_matvec_single, fmm.cpp:123-213
void single_level(const Problem& p, const std::vector<double>& cv,
                  const double* w, double* out, Stats* st) {
  Tree t = build_tree(p, p.L);
  Grid g = make_grid(p.sigma, p.M, p.d);
  int lev = t.L;
  long boxes = t.count(lev);
  Level mult(boxes), local(boxes);
  for (long b = 0; b < boxes; ++b) {
    if (t.npts(b) == 0) continue;
    mult[b].assign(g.K, C(0.0, 0.0));
    double xb[3];
    t.center(lev, b, xb);
    const int* pj = t.pts(b);
    for (long jj = 0; jj < t.npts(b); ++jj) {
      int j = pj[jj];
      double r[3] = {0, 0, 0};
      for (int k = 0; k < p.d; ++k) r[k] = xb[k] - p.x[(long)j * p.d + k];
      for (long m = 0; m < g.K; ++m)
        mult[b][m] += w[j] * std::polar(1.0, dot(p.d, &g.nodes[m * 3], r));
    }
  }
  long long far_pairs = 0;
#pragma omp parallel for schedule(dynamic) reduction(+ : far_pairs)
  for (long a = 0; a < boxes; ++a) {
    if (t.npts(a) == 0) continue;
    local[a].assign(g.K, C(0.0, 0.0));
    double xa[3];
    t.center(lev, a, xa);
    long ia[3];
    t.idx(lev, a, ia);
    for (long b = 0; b < boxes; ++b) {
      long ib[3];
      t.idx(lev, b, ib);
      bool nbr = true;
      for (int k = 0; k < p.d; ++k)
        if (std::abs(ia[k] - ib[k]) > 1) nbr = false;
      if (nbr) continue;
      if (mult[b].empty()) continue;
      double xb[3];
      t.center(lev, b, xb);
      double r[3] = {0, 0, 0};
      for (int k = 0; k < p.d; ++k) r[k] = xa[k] - xb[k];
      for (long m = 0; m < g.K; ++m)
        local[a][m] += cv[m] * std::polar(1.0, dot(p.d, &g.nodes[m * 3], r)) * mult[b][m];
      ++far_pairs;
    }
  }
  double max_imag = 0.0;
  long long near_pairs = 0;
#pragma omp parallel for schedule(dynamic) reduction(+ : near_pairs) reduction(max : max_imag)
  for (long a = 0; a < boxes; ++a) {
    if (t.npts(a) == 0) continue;
    double xa[3];
    t.center(lev, a, xa);
    auto nb = t.neighbors(lev, a);
    const int* pi = t.pts(a);
    for (long ii = 0; ii < t.npts(a); ++ii) {
      int i = pi[ii];
      C acc(0.0, 0.0);
      double r[3] = {0, 0, 0};
      for (int k = 0; k < p.d; ++k) r[k] = p.x[(long)i * p.d + k] - xa[k];
      for (long m = 0; m < g.K; ++m)
        acc += g.weight * std::polar(1.0, dot(p.d, &g.nodes[m * 3], r)) * local[a][m];
      double v = acc.real();
      max_imag = std::max(max_imag, std::abs(acc.imag()));
      for (long b : nb) {
        const int* pj = t.pts(b);
        for (long jj = 0; jj < t.npts(b); ++jj) {
          int j = pj[jj];
          v += w[j] * eval_kernel(p.k, dist(p.d, p.x + (long)i * p.d, p.x + (long)j * p.d));
          ++near_pairs;
        }
      }
      out[i] = v;
    }
  }
  if (st) {
    st->near_pairs = near_pairs;
    st->far_work = 2LL * p.n * g.K + far_pairs * g.K;
    st->max_imag = max_imag;
  }
}

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::domain_error& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 9;
  }
}

Problem make_problem(int d, long n, const double* x, const double* lo,
                     const double* hi, int ktype, double shape, double sigma,
                     int M, int L) {
  if (d < 1 || d > 3) throw std::invalid_argument("d must be 1, 2 or 3");
  Problem p{};
  p.d = d;
  p.n = n;
  p.x = x;
  for (int k = 0; k < 3; ++k) {
    p.lo[k] = lo ? lo[k] : 0.0;
    p.hi[k] = hi ? hi[k] : 1.0;
  }
  p.k = Kernel{ktype, shape};
  p.sigma = sigma;
  p.M = M;
  p.L = L;
  return p;
}

}  // namespace

extern "C" {

const char* orc_last_error() { return g_err.c_str(); }

// GridMode for the following orc_mlfmm / orc_expansions calls (0 shared,
// 1 scaled) and the Lagrange stencil size (make_level_grids' stencil_k).
// In scaled mode a caller C table holds one K-entry table per level 2..L.
void orc_set_grid_mode(int mode, int stencil_k) {
  g_mode = mode;
  g_stencil = stencil_k;
}

// bench.py's CPU legs: use every host thread even when a launcher (torchrun)
// exported OMP_NUM_THREADS=1 before this library was loaded.
// Target-leaf subset for the following orc_mlfmm calls (n = 0: all leaves).
void orc_set_target_leaves(long n, const long* leaf_ids) {
  g_target_leaves.assign(leaf_ids, leaf_ids + (n > 0 ? n : 0));
}

void orc_set_num_threads(int n) {
  if (n > 0) omp_set_num_threads(n);
}
int orc_get_max_threads() { return omp_get_max_threads(); }

std::uint64_t orc_hash64(std::uint64_t x) {  // common.hpp:45-50
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

double orc_uniform01(std::uint64_t seed, std::uint64_t counter) {  // common.hpp:52-55
  std::uint64_t z = orc_hash64(seed ^ orc_hash64(counter));
  return (z >> 11) * 0x1.0p-53;
}

int orc_eval_kernel(int ktype, double shape, double r, double* out) {
  return guard([&] { *out = eval_kernel(Kernel{ktype, shape}, r); });
}

int orc_eval_fourier(int ktype, double shape, double xi, int d, double* out) {
  return guard([&] { *out = eval_fourier(Kernel{ktype, shape}, xi, d); });
}

int orc_cell_average(int ktype, double shape, int d, const double* a,
                     const double* b, double* out) {
  return guard([&] {
    Kernel k{ktype, shape};
    if (d == 1) *out = cell_average_1d(k, a[0], b[0]);
    else if (d == 2) *out = cell_average_2d(k, a[0], b[0], a[1], b[1]);
    else {
      double aa[3] = {a[0], a[1], a[2]}, bb[3] = {b[0], b[1], b[2]};
      *out = cell_average_3d(k, aa, bb);
    }
  });
}

int orc_c_table(int ktype, double shape, double sigma, int M, int d,
                double* c_out) {
  return guard([&] {
    auto c = c_table(Kernel{ktype, shape}, sigma, M, d);
    std::memcpy(c_out, c.data(), c.size() * sizeof(double));
  });
}

// Multilevel matvec for nrhs right-hand sides. w and out are [rhs][n]
// (rhs-major). c_in: optional K-entry C table (NULL = compute). stride > 1
// samples boxes per stage for timing (stage_seconds[6] receives the
// extrapolated times of p2m, m2m, m2l, l2l, l2p, near); outputs are then
// not meaningful.
int orc_mlfmm(int d, long n, const double* x, const double* lo,
              const double* hi, int ktype, double shape, double sigma, int M,
              int L, const double* c_in, int nrhs, const double* w,
              double* out, long long* near, long long* far, double* imag,
              int stride, double* stage_seconds) {
  return guard([&] {
    Problem p = make_problem(d, n, x, lo, hi, ktype, shape, sigma, M, L);
    Grids G = make_grids(p.k, sigma, M, d, L, g_mode, g_stencil, c_in);
    Sampler smp;
    smp.stride = stride > 0 ? stride : 1;
    double im = 0.0;
    for (int r = 0; r < nrhs; ++r) {
      Stats st{};
      mlfmm(p, G, w + (long)r * n, out + (long)r * n, &st, &smp);
      if (near) *near = st.near_pairs;
      if (far) *far = st.far_work;
      im = std::max(im, st.max_imag);
    }
    if (imag) *imag = im;
    if (stage_seconds)
      for (int i = 0; i < 6; ++i) stage_seconds[i] = smp.t[i];
  });
}

int orc_single(int d, long n, const double* x, const double* lo,
               const double* hi, int ktype, double shape, double sigma, int M,
               int level, const double* c_in, const double* w, double* out,
               long long* near, long long* far, double* imag) {
  return guard([&] {
    Problem p = make_problem(d, n, x, lo, hi, ktype, shape, sigma, M, level);
    if (level < 1) throw std::invalid_argument("level must be >= 1");
    long K = 1;
    for (int i = 0; i < d; ++i) K *= M;
    std::vector<double> cv = c_in ? std::vector<double>(c_in, c_in + K)
                                  : c_table(p.k, sigma, M, d);
    Stats st{};
    single_level(p, cv, w, out, &st);
    if (near) *near = st.near_pairs;
    if (far) *far = st.far_work;
    if (imag) *imag = st.max_imag;
  });
}

// direct_matvec, fmm.cpp:30-75 (plain kernel). Optional target subset.
int orc_direct(int d, long n, const double* x, int ktype, double shape,
               const double* w, long n_targets, const long* targets,
               double* out) {
  return guard([&] {
    Kernel k{ktype, shape};
    long nt = targets ? n_targets : n;
#pragma omp parallel for schedule(static)
    for (long q = 0; q < nt; ++q) {
      long i = targets ? targets[q] : q;
      double acc = 0.0;
      for (long j = 0; j < n; ++j)
        acc += w[j] * eval_kernel(k, dist(d, x + i * d, x + j * d));
      out[q] = acc;
    }
  });
}

// Stage expansions of one level in dense row-major box order,
// out[(box*K + node)*2 + {re,im}]; kind 0 multipoles (upsweep), 1 couple()
// locals, 2 locals after L2L (downsweep's working copy).
int orc_expansions(int d, long n, const double* x, const double* lo,
                   const double* hi, int ktype, double shape, double sigma,
                   int M, int L, const double* c_in, const double* w,
                   int level, int kind, double* out) {
  return guard([&] {
    Problem p = make_problem(d, n, x, lo, hi, ktype, shape, sigma, M, L);
    Tree t = build_tree(p, L);
    Grids G = make_grids(p.k, sigma, M, d, L, g_mode, g_stencil, c_in);
    const Grid& g = G.g[L];
    auto mult = upsweep(p, t, G, w, nullptr);
    std::vector<Level> src;
    if (kind == 0) {
      src = std::move(mult);
    } else {
      auto loc = couple(p, t, G, mult, nullptr);
      if (kind == 1) {
        src = std::move(loc);
      } else {
        std::vector<double> dummy(n, 0.0);
        downsweep(p, t, G, loc, dummy.data(), nullptr, nullptr, &src);
      }
    }
    long cnt = t.count(level);
    std::fill(out, out + cnt * g.K * 2, 0.0);
    for (long b = 0; b < cnt; ++b) {
      const auto& v = src[level][b];
      if (v.empty()) continue;
      for (long m = 0; m < g.K; ++m) {
        out[(b * g.K + m) * 2] = v[m].real();
        out[(b * g.K + m) * 2 + 1] = v[m].imag();
      }
    }
  });
}

// Tree lists (see ref_tree_lists in ref_capi.cpp for the layout).
int orc_tree_lists(int d, long n, const double* x, const double* lo,
                   const double* hi, int L, int level, int which, int* counts,
                   long* ids) {
  return guard([&] {
    Problem p = make_problem(d, n, x, lo, hi, 0, 1.0, 1.0, 2, L);
    Tree t = build_tree(p, L);
    long pos = 0;
    long cnt = which == 2 ? t.count(L) : t.count(level);
    for (long b = 0; b < cnt; ++b) {
      if (which == 2) {
        counts[b] = static_cast<int>(t.npts(b));
        if (ids)
          for (long q = 0; q < t.npts(b); ++q) ids[pos++] = t.pts(b)[q];
      } else {
        auto v = which == 0 ? t.neighbors(level, b) : t.interaction(level, b);
        counts[b] = static_cast<int>(v.size());
        if (ids)
          for (long q : v) ids[pos++] = q;
      }
    }
  });
}

long long orc_sum_il(int d, int L, int level) {
  Tree t;
  t.d = d;
  t.L = L;
  return sum_il_sizes(t, level);
}

}  // extern "C"
