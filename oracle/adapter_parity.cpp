// Test infrastructure: the reference library (compiled from its own sources)
// and the GPU library linked into ONE program through include/blfmm_gpu.hpp,
// the drop-in a reference maintainer would use. Runs the reference matvec and
// the GPU matvec on the reference's own PointSet / BoxTree / LevelGrids and
// prints one JSON line per case; exit code = number of failed cases.
// Built by oracle/Makefile into oracle/_ref/adapter_parity (needs a GPU to run).
#include <cmath>
#include <cstdio>
#include <string>
#include <tuple>
#include <vector>

#include "blfmm/mlfmm.hpp"
#include "blfmm_gpu.hpp"

using namespace blfmm;

static double rel_l2(const std::vector<double>& a, const std::vector<double>& b) {
  double num = 0, den = 0;
  for (size_t i = 0; i < a.size(); ++i) {
    num += (a[i] - b[i]) * (a[i] - b[i]);
    den += b[i] * b[i];
  }
  return std::sqrt(num / (den > 0 ? den : 1.0));
}

static int run_case(const char* name, const std::string& spec, int d, int n, double sigma, int m,
                    int leaf, bool single, GridMode mode = GridMode::shared, int stencil = 10) {
  PointSet ps;
  ps.d = d;
  for (int i = 0; i < n; ++i)
    ps.pts.push_back(Pt{uniform01(1001, static_cast<uint64_t>(d) * i),
                        d == 2 ? uniform01(1001, static_cast<uint64_t>(d) * i + 1) : 0.0});
  std::vector<double> w(n);
  for (int j = 0; j < n; ++j) w[j] = 2.0 * uniform01(2001, j) - 1.0;
  RadialKernel k = parse_kernel_spec(spec);
  BoxTree tree = build_tree(ps, leaf);
  SumRequest req{k, sigma, &ps, w, m};
  SumResult ref, gpu;
  if (single) {
    ref = fmm_matvec_single(req, tree);
    gpu = blfmm::gpu::fmm_matvec_single(req, tree);
  } else {
    LevelGrids grids = make_level_grids(k, sigma, m, d, leaf, mode, stencil);
    ref = mlfmm_matvec(req, tree, grids);
    gpu = blfmm::gpu::mlfmm_matvec(req, tree, grids);
    // second call reuses the cached plan (solver pattern)
    gpu = blfmm::gpu::mlfmm_matvec(req, tree, grids);
  }
  double e = rel_l2(gpu.values, ref.values);
  bool ok = e <= 1e-10 && gpu.stats.near_pairs == ref.stats.near_pairs &&
            gpu.stats.far_work == ref.stats.far_work;
  std::printf(
      "{\"case\": \"%s\", \"rel_l2\": %.3e, \"near_pairs\": [%lld, %lld], \"far_work\": [%lld, "
      "%lld], \"max_imag\": [%.6e, %.6e], \"ok\": %s}\n",
      name, e, gpu.stats.near_pairs, ref.stats.near_pairs, gpu.stats.far_work,
      ref.stats.far_work, gpu.stats.max_imag_residual, ref.stats.max_imag_residual,
      ok ? "true" : "false");
  return ok ? 0 : 1;
}

// solve_interpolation through the adapter (blfmm_solve: the Krylov loop in the
// library over the GPU plan) against the same recurrences run on the host with
// the REFERENCE's own mlfmm_matvec (solver.cpp:43-88 for CG; the reference's
// solver.cpp needs Eigen, absent here): same iterate sequence up to the
// matvec's rounding, and the GPU solution's residual under the reference
// matvec.
static int solve_case(const char* name, const std::string& spec, int n, double sigma, int m,
                      int leaf) {
  // test_solver.cpp:209-242's setting: 1-D, jittered points on [0, 32]
  PointSet ps;
  ps.d = 1;
  ps.domain.lo = Pt{0.0, 0.0};
  ps.domain.hi = Pt{32.0, 1.0};
  for (int i = 0; i < n; ++i)
    ps.pts.push_back(Pt{(i + 0.5 + 0.4 * (uniform01(3001, i) - 0.5)) * 32.0 / n, 0.0});
  std::vector<double> b(n);
  for (int j = 0; j < n; ++j)
    b[j] = std::sin(M_PI * ps.pts[j][0] / 32.0) + 0.5 * std::cos(3.0 * M_PI * ps.pts[j][0] / 32.0);
  RadialKernel k = parse_kernel_spec(spec);
  blfmm::gpu::InterpolationProblem prob;
  prob.kernel = k;
  prob.ps = &ps;
  prob.rhs = b;
  prob.backend = blfmm::gpu::Backend::mlfmm;
  prob.tol = 1e-12;
  prob.max_iter = 2000;
  prob.sigma = sigma;
  prob.m_per_dim = m;
  prob.leaf_level = leaf;
  std::vector<double> x;
  blfmm::gpu::SolveStats st;
  try {
    std::tie(x, st) = blfmm::gpu::solve_interpolation(prob);
  } catch (const std::exception& e) {
    std::printf("{\"case\": \"solve %s\", \"error\": \"%s\", \"ok\": false}\n", name, e.what());
    return 1;
  }
  // reference matvec, reference CG recurrence on the host
  BoxTree tree = build_tree(ps, leaf);
  LevelGrids grids = make_level_grids(k, sigma, m, 1, leaf, GridMode::shared, 10);
  auto apply = [&](const std::vector<double>& v) {
    SumRequest req{k, sigma, &ps, v, m};
    return mlfmm_matvec(req, tree, grids).values;
  };
  std::vector<double> xr(n, 0.0), r = b, p = b;
  double bn = 0, rr = 0;
  for (double v : b) bn += v * v;
  bn = std::sqrt(bn);
  rr = bn * bn;
  int it = 0;
  for (; it < prob.max_iter; ++it) {
    std::vector<double> ap = apply(p);
    double pap = 0;
    for (int i = 0; i < n; ++i) pap += p[i] * ap[i];
    const double alpha = rr / pap;
    for (int i = 0; i < n; ++i) {
      xr[i] += alpha * p[i];
      r[i] -= alpha * ap[i];
    }
    double rn = 0;
    for (double v : r) rn += v * v;
    if (std::sqrt(rn) / bn <= prob.tol) {
      ++it;
      break;
    }
    const double beta = rn / rr;
    rr = rn;
    for (int i = 0; i < n; ++i) p[i] = r[i] + beta * p[i];
  }
  std::vector<double> ax = apply(x);
  double res = 0;
  for (int i = 0; i < n; ++i) res += (ax[i] - b[i]) * (ax[i] - b[i]);
  res = std::sqrt(res) / bn;
  const double ex = rel_l2(x, xr);
  // (ill-conditioned cases: the reduction order shifts the iteration count slightly)
  const bool ok = st.converged && st.method == "cg" && res <= 1e-11 && ex <= 1e-8 &&
                  std::abs(st.iterations - it) <= std::max(2, it / 50);
  std::printf(
      "{\"case\": \"solve %s\", \"iterations\": [%d, %d], \"residual_ref_matvec\": %.3e, "
      "\"rel_l2_vs_ref_cg\": %.3e, \"ok\": %s}\n",
      name, st.iterations, it, res, ex, ok ? "true" : "false");
  return ok ? 0 : 1;
}

// Backend::dense through the adapter (blfmm_solve_dense: the Krylov loop on the
// matrix-free O(N^2) device kernel): the solution's residual under the matrix
// assembled with the REFERENCE's eval_kernel / dist exactly as assemble_dense
// (solver.cpp:207-240), the method the reference picks (positive_definite),
// and the N <= 8192 cap as std::length_error.
static int dense_case(const std::string& spec, int d, int n, const char* method) {
  PointSet ps;
  ps.d = d;
  for (int i = 0; i < n; ++i) {
    if (d == 1) ps.pts.push_back(Pt{(i + 0.5 + 0.3 * (uniform01(3101, i) - 0.5)) / n, 0.0});
    else ps.pts.push_back(Pt{uniform01(3102, 2 * i), uniform01(3102, 2 * i + 1)});
  }
  std::vector<double> b(n);
  for (int j = 0; j < n; ++j) b[j] = std::sin(M_PI * ps.pts[j][0]) + 0.25 * std::cos(2.0 * ps.pts[j][1]);
  RadialKernel k = parse_kernel_spec(spec);
  blfmm::gpu::InterpolationProblem prob;
  prob.kernel = k;
  prob.ps = &ps;
  prob.rhs = b;
  prob.backend = blfmm::gpu::Backend::dense;
  prob.tol = 1e-9;
  prob.max_iter = 4000;
  std::vector<double> x;
  blfmm::gpu::SolveStats st;
  try {
    std::tie(x, st) = blfmm::gpu::solve_interpolation(prob);
  } catch (const std::exception& e) {
    std::printf("{\"case\": \"dense %s\", \"error\": \"%s\", \"ok\": false}\n", spec.c_str(),
                e.what());
    return 1;
  }
  double res = 0, bn = 0;
  for (int i = 0; i < n; ++i) {
    double acc = 0;
    for (int j = 0; j < n; ++j) acc += eval_kernel(k, dist(d, ps.pts[i], ps.pts[j])) * x[j];
    res += (acc - b[i]) * (acc - b[i]);
    bn += b[i] * b[i];
  }
  res = std::sqrt(res / bn);
  const bool ok = st.converged && st.method == method && res <= 20 * prob.tol;
  std::printf("{\"case\": \"dense %s d=%d N=%d\", \"method\": \"%s\", \"iterations\": %d, "
              "\"residual_ref_matrix\": %.3e, \"ok\": %s}\n",
              spec.c_str(), d, n, st.method.c_str(), st.iterations, res, ok ? "true" : "false");
  return ok ? 0 : 1;
}

int main() {
  int fails = 0;
  fails += dense_case("tps:beta=2", 1, 200, "gmres");  // test_solver.cpp:286-303's kernel
  fails += dense_case("wendland:eps=4", 2, 400, "cg");
  fails += dense_case("imq:c=0.01", 1, 200, "cg");
  fails += dense_case("mq:c=0.05", 2, 300, "gmres");
  try {  // assemble_dense's cap (solver.cpp:211)
    PointSet big;
    big.d = 1;
    for (int i = 0; i < 8193; ++i) big.pts.push_back(Pt{i / 8193.0, 0.0});
    blfmm::gpu::InterpolationProblem prob;
    prob.kernel = parse_kernel_spec("gaussian:c=1");
    prob.ps = &big;
    prob.rhs.assign(8193, 1.0);
    prob.backend = blfmm::gpu::Backend::dense;
    blfmm::gpu::solve_interpolation(prob);
    std::printf("{\"case\": \"dense cap\", \"ok\": false}\n");
    ++fails;
  } catch (const std::length_error&) {
    std::printf("{\"case\": \"dense cap\", \"ok\": true}\n");
  }
  fails += solve_case("gaussian:c=256 band-capturing 1D N=512", "gaussian:c=256", 512, 203.0,
                      2112, 4);
  fails += solve_case("gaussian:c=256 band-capturing 1D N=1024", "gaussian:c=256", 1024, 203.0,
                      2112, 5);
  fails += run_case("P1 gaussian:c=16 2D N=4096", "gaussian:c=16", 2, 4096, M_PI, 64, 3, false);
  fails += run_case("P1b band-capturing", "gaussian:c=16", 2, 4096, 51.4, 44, 3, false);
  fails += run_case("P4-shape mq:c=0.05 2D N=16384", "mq:c=0.05", 2, 16384, M_PI, 16, 5, false);
  fails += run_case("imq:c=0.1 2D N=8192", "imq:c=0.1", 2, 8192, M_PI, 16, 4, false);
  fails += run_case("imq:c=1 1D N=1024 L=5", "imq:c=1", 1, 1024, M_PI, 64, 5, false);
  fails += run_case("single-level imq:c=1 2D", "imq:c=1", 2, 2048, M_PI, 12, 3, true);
  fails += run_case("scaled grids imq:c=1 2D stencil 10", "imq:c=1", 2, 4096, M_PI, 16, 4,
                    false, GridMode::scaled, 10);
  fails += run_case("scaled grids gaussian:c=1 1D stencil 6", "gaussian:c=1", 1, 2048, M_PI, 16,
                    6, false, GridMode::scaled, 6);
  // error mapping: mismatched grids -> std::invalid_argument
  try {
    PointSet ps;
    ps.d = 2;
    ps.pts = {Pt{0.1, 0.2}, Pt{0.3, 0.4}};
    BoxTree tree = build_tree(ps, 3);
    LevelGrids grids = make_level_grids(parse_kernel_spec("imq:c=1"), M_PI, 8, 2, 4,
                                        GridMode::shared, 10);
    SumRequest req{parse_kernel_spec("imq:c=1"), M_PI, &ps, {1.0, 2.0}, 8};
    blfmm::gpu::mlfmm_matvec(req, tree, grids);
    std::printf("{\"case\": \"error mapping\", \"ok\": false}\n");
    ++fails;
  } catch (const std::invalid_argument&) {
    std::printf("{\"case\": \"error mapping\", \"ok\": true}\n");
  }
  return fails;
}
