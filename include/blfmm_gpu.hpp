// blfmm_gpu.hpp — header-only C++ adapter: the reference library's own
// signatures (namespace blfmm, d <= 2 types of /root/reference/proj/core/include)
// implemented on the C ABI of blfmm_gpu.h, so reference callers (the Krylov
// solver, the CLI, the tests) can switch the matvec to the B200 path by
// replacing `blfmm::mlfmm_matvec(...)` with `blfmm::gpu::mlfmm_matvec(...)`.
//
// Include AFTER putting the reference headers on the include path; link with
// libblfmm_gpu.so. Mirrors:
//   SumResult mlfmm_matvec(const SumRequest&, const BoxTree&, const LevelGrids&)
//                                             core/include/blfmm/mlfmm.hpp:98-99
//   SumResult fmm_matvec_single(const SumRequest&, const BoxTree&)
//                                             core/include/blfmm/fmm.hpp:55
//   SumResult direct_matvec(const RadialKernel&, const PointSet&,
//                           const std::vector<double>&, bool, double, int)
//                                             core/include/blfmm/fmm.hpp:33-36
//   SumResult direct_matvec_hybrid(const RadialKernel&, const PointSet&,
//                                  const BoxTree&, const std::vector<double>&,
//                                  double, int)       core/include/blfmm/fmm.hpp:40-43
// Errors are rethrown as the reference's exception classes
// (std::invalid_argument, std::domain_error, blfmm::accuracy_error).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "blfmm/mlfmm.hpp"
#include "blfmm_gpu.h"

namespace blfmm {
namespace gpu {

inline void check(int code) {
  if (code == BLFMM_OK) return;
  std::string msg = blfmm_last_error();
  switch (code) {
    case BLFMM_EINVAL:
      throw std::invalid_argument(msg);
    case BLFMM_EDOMAIN:
      throw std::domain_error(msg);
    case BLFMM_EACCURACY:
      throw accuracy_error(msg, blfmm_last_error_value());
    case BLFMM_ENOMEM:
      throw std::bad_alloc();
    case BLFMM_ELENGTH:
      throw std::length_error(msg);
    default:
      throw std::runtime_error("blfmm_gpu: " + msg);
  }
}

// Plan cache: the tree + grids a caller builds once are reused across
// matvecs (the solver pattern, solver.cpp:280-293). The reference recomputes
// from req.ps on every call, so the cached plan is reused only when the FULL
// coordinate array (and the domain) equals the copy the plan was built from:
// a new PointSet at a reused address, or coordinates rewritten in place,
// rebuild the plan instead of hitting a stale one.
inline void flatten_points(const PointSet& ps, std::vector<double>& out) {
  const int d = ps.d;
  out.resize(ps.pts.size() * d + 4);
  for (std::size_t i = 0; i < ps.pts.size(); ++i)
    for (int q = 0; q < d; ++q) out[i * d + q] = ps.pts[i][q];
  const std::size_t t = ps.pts.size() * d;
  out[t] = ps.domain.lo[0];
  out[t + 1] = ps.domain.lo[1];
  out[t + 2] = ps.domain.hi[0];
  out[t + 3] = ps.domain.hi[1];
}

struct PlanHandle {
  blfmm_plan* p = nullptr;
  std::vector<double> coords;  // flattened coordinates + domain the plan was built from
  std::size_t n = 0;
  int leaf = 0, m = 0, mode = 0, stencil = 10;
  double sigma = 0.0;
  RadialKernel kernel;
  std::vector<double> c_vals;
  ~PlanHandle() {
    if (p) blfmm_plan_destroy(p);
  }
};

inline blfmm_plan* plan_for(const PointSet& ps, const BoxTree& tree, const RadialKernel& k,
                            double sigma, int m, const std::vector<double>& c_vals,
                            int mode = BLFMM_GRID_SHARED, int stencil_k = 10) {
  thread_local std::unique_ptr<PlanHandle> cache;
  thread_local std::vector<double> coords;
  flatten_points(ps, coords);
  if (cache && cache->n == ps.pts.size() && cache->coords == coords &&
      cache->leaf == tree.leaf_level &&
      cache->m == m && cache->sigma == sigma && cache->kernel.type == k.type &&
      cache->kernel.shape == k.shape && cache->c_vals == c_vals && cache->mode == mode &&
      cache->stencil == stencil_k)
    return cache->p;
  cache.reset(new PlanHandle());
  const int d = ps.d;
  blfmm_plan_desc desc;
  std::memset(&desc, 0, sizeof(desc));
  desc.d = d;
  desc.n = static_cast<long long>(ps.pts.size());
  desc.coords = coords.data();
  for (int q = 0; q < d; ++q) {
    desc.domain_lo[q] = tree.domain.lo[q];
    desc.domain_hi[q] = tree.domain.hi[q];
  }
  desc.kernel_type = static_cast<int>(k.type);  // same enumerator order
  desc.kernel_shape = k.shape;
  desc.sigma = sigma;
  desc.m_per_dim = m;
  desc.leaf_level = tree.leaf_level;
  desc.grid_mode = mode;
  desc.stencil_k = stencil_k;
  desc.nrhs = 1;
  desc.device = -1;
  desc.c_table = c_vals.data();  // the reference's own C(xi_m): bit-identical spectrum
  desc.world = 1;
  check(blfmm_plan_create(&desc, &cache->p));
  cache->coords = coords;
  cache->n = ps.pts.size();
  cache->leaf = tree.leaf_level;
  cache->m = m;
  cache->sigma = sigma;
  cache->kernel = k;
  cache->c_vals = c_vals;
  cache->mode = mode;
  cache->stencil = stencil_k;
  return cache->p;
}

inline SumResult run(blfmm_plan* p, const std::vector<double>& w, bool single) {
  SumResult res;
  res.values.assign(w.size(), 0.0);
  blfmm_stats st{};
  check(single ? blfmm_execute_single(p, w.data(), res.values.data(), &st, nullptr)
               : blfmm_execute(p, w.data(), res.values.data(), &st, nullptr));
  res.stats.near_pairs = st.near_pairs;
  res.stats.far_work = st.far_work;
  res.stats.max_imag_residual = st.max_imag_residual;
  return res;
}

// mlfmm.cpp:361-406 semantics (shared grids).
inline SumResult mlfmm_matvec(const SumRequest& req, const BoxTree& tree,
                              const LevelGrids& grids) {
  if (!req.ps) throw std::invalid_argument("request has no point set");
  const PointSet& ps = *req.ps;
  if (req.weights.size() != static_cast<std::size_t>(ps.size()))
    throw std::invalid_argument("weight count != point count");
  if (grids.d != ps.d || grids.leaf_level != tree.leaf_level)
    throw std::invalid_argument("grids incompatible with tree/points");
  const auto& g = grids.grids[tree.leaf_level];
  if (grids.mode == GridMode::scaled) {
    // the reference's own per-level C tables, levels 2..L in order
    std::vector<double> c;
    for (int l = 2; l <= tree.leaf_level; ++l)
      c.insert(c.end(), grids.factors[l].c_vals.begin(), grids.factors[l].c_vals.end());
    blfmm_plan* p = plan_for(ps, tree, grids.kernel, g.sigma, g.m_per_dim, c, BLFMM_GRID_SCALED,
                             grids.stencil_k);
    return run(p, req.weights, false);
  }
  blfmm_plan* p = plan_for(ps, tree, grids.kernel, g.sigma, g.m_per_dim,
                           grids.factors[tree.leaf_level].c_vals);
  return run(p, req.weights, false);
}

// fmm.cpp:123-213 semantics: equal to the shared-grid sweep to rounding.
inline SumResult fmm_matvec_single(const SumRequest& req, const BoxTree& tree) {
  if (!req.ps) throw std::invalid_argument("request has no point set");
  if (static_cast<int>(req.weights.size()) != req.ps->size())
    throw std::invalid_argument("weights length != point count");
  if (!(req.sigma > 0.0)) throw std::invalid_argument("sigma must be > 0");
  if (req.m_per_dim < 2) throw std::invalid_argument("m_per_dim must be >= 2");
  QuadratureGrid grid = make_quadrature(req.sigma, req.m_per_dim, req.ps->d);
  LowRankFactors f = translation_coefficients(req.kernel, grid, TranslationMode::spectral);
  blfmm_plan* p = plan_for(*req.ps, tree, req.kernel, req.sigma, req.m_per_dim, f.c_vals);
  return run(p, req.weights, true);
}

// Band-limited (leaf < 0, fmm.cpp:57-70) or hybrid (fmm.cpp:77-113) O(N^2)
// oracle on the GPU; d = 1 (std::domain_error otherwise, as the reference).
inline SumResult detail_direct_bandlimited(const RadialKernel& k, const PointSet& ps,
                                           const std::vector<double>& weights, double sigma,
                                           int refinement, int leaf) {
  const int n = ps.size();
  if (static_cast<int>(weights.size()) != n)
    throw std::invalid_argument("weights length != point count");
  std::vector<double> coords(n);
  for (int i = 0; i < n; ++i) coords[i] = ps.pts[i][0];
  const double lo[2] = {ps.domain.lo[0], ps.domain.lo[1]};
  const double hi[2] = {ps.domain.hi[0], ps.domain.hi[1]};
  SumResult res;
  res.values.assign(n, 0.0);
  check(blfmm_direct_bandlimited(ps.d, n, coords.data(), lo, hi, static_cast<int>(k.type),
                                 k.shape, weights.data(), sigma, refinement, leaf,
                                 res.values.data(), -1));
  res.stats.near_pairs = static_cast<long long>(n) * n;
  return res;
}

// fmm.cpp:77-113: original kernel in the target leaf's neighbour block,
// Phi_sigma elsewhere (include/blfmm/fmm.hpp:40-43).
inline SumResult direct_matvec_hybrid(const RadialKernel& k, const PointSet& ps,
                                      const BoxTree& tree, const std::vector<double>& weights,
                                      double sigma, int refinement = 1024) {
  if (ps.d != 1) throw std::domain_error("hybrid direct oracle is 1d only");
  return detail_direct_bandlimited(k, ps, weights, sigma, refinement, tree.leaf_level);
}

// fmm.cpp:30-75 O(N^2) sum: plain kernel, or the band-limited table oracle.
inline SumResult direct_matvec(const RadialKernel& k, const PointSet& ps,
                               const std::vector<double>& weights, bool use_bandlimited,
                               double sigma, int refinement = 1024) {
  const int n = ps.size();
  if (use_bandlimited) return detail_direct_bandlimited(k, ps, weights, sigma, refinement, -1);
  if (static_cast<int>(weights.size()) != n)
    throw std::invalid_argument("weights length != point count");
  std::vector<double> coords(static_cast<std::size_t>(n) * ps.d);
  for (int i = 0; i < n; ++i)
    for (int q = 0; q < ps.d; ++q) coords[static_cast<std::size_t>(i) * ps.d + q] = ps.pts[i][q];
  SumResult res;
  res.values.assign(n, 0.0);
  check(blfmm_direct(ps.d, n, coords.data(), static_cast<int>(k.type), k.shape, weights.data(),
                     n, nullptr, res.values.data(), -1));
  res.stats.near_pairs = static_cast<long long>(n) * n;
  return res;
}

// solve_interpolation (solver.cpp:269-300, solver.hpp:16-46) without Eigen:
// the Krylov loop runs in the library (blfmm_solve, device vectors) over the
// multilevel plan of the problem's points (Backend::mlfmm, leaf level
// lround(log2(N/32)) >= 3 unless given) or the single-level tree
// (Backend::single_fmm, lround(log2(sqrt N)) >= 2; shared grids make the
// multilevel sweep equal to the single-level sum to rounding). CG for the
// positive definite kernels (kernels.cpp:334-337), restarted GMRES otherwise.
// Backend::dense (the reference's default; Eigen assembly + a * x there) runs
// the same loops on the matrix-free O(N^2) device kernel (blfmm_solve_dense),
// for every kernel type, N <= 8192 (std::length_error beyond, as assemble_dense).
enum class Backend { dense, single_fmm, mlfmm };
struct InterpolationProblem {
  RadialKernel kernel;
  const PointSet* ps = nullptr;
  std::vector<double> rhs;
  Backend backend = Backend::mlfmm;
  double tol = 1e-10;
  int max_iter = 2000;
  double sigma = 0.0;  // <= 0: pi
  int m_per_dim = 0;   // <= 0: choose_truncation(N)
  int leaf_level = 0;  // 0: from N
};
struct SolveStats {
  int iterations = 0;
  double residual = 0.0;
  long long matvecs = 0;
  std::string method;
  bool converged = false;
};

inline std::pair<std::vector<double>, SolveStats> solve_interpolation(
    const InterpolationProblem& prob) {
  if (!prob.ps) throw std::invalid_argument("problem has no point set");
  const PointSet& ps = *prob.ps;
  const int n = ps.size();
  if (prob.rhs.size() != static_cast<std::size_t>(n))
    throw std::invalid_argument("rhs length != point count");
  if (!(prob.tol > 0.0)) throw std::invalid_argument("tol must be positive");
  // positive_definite, kernels.cpp:334-337
  const bool pd = prob.kernel.type == KernelType::Gaussian || prob.kernel.type == KernelType::IMQ ||
                  prob.kernel.type == KernelType::WendlandC2 ||
                  prob.kernel.type == KernelType::Wendland31;
  auto finish = [&](int rc, const blfmm_solve_stats& st, std::vector<double>& x) {
    SolveStats out;
    out.iterations = st.iterations;
    out.residual = st.residual;
    out.matvecs = st.matvecs;
    out.method = st.method == BLFMM_SOLVE_CG ? "cg" : "gmres";
    out.converged = st.converged != 0;
    check(rc);  // BLFMM_EACCURACY -> accuracy_error (best residual), as the reference
    return std::pair<std::vector<double>, SolveStats>{std::move(x), out};
  };
  if (prob.backend == Backend::dense) {
    std::vector<double> coords(static_cast<std::size_t>(n) * ps.d);
    for (int i = 0; i < n; ++i)
      for (int q = 0; q < ps.d; ++q) coords[static_cast<std::size_t>(i) * ps.d + q] = ps.pts[i][q];
    std::vector<double> x(n, 0.0);
    blfmm_solve_stats st{};
    const int rc = blfmm_solve_dense(ps.d, n, coords.data(), static_cast<int>(prob.kernel.type),
                                     prob.kernel.shape, pd ? BLFMM_SOLVE_CG : BLFMM_SOLVE_GMRES,
                                     prob.rhs.data(), x.data(), prob.tol, prob.max_iter, &st, -1);
    return finish(rc, st, x);
  }
  const double sigma = prob.sigma > 0.0 ? prob.sigma : 3.14159265358979323846;
  const int m = prob.m_per_dim > 0 ? prob.m_per_dim : choose_truncation(n);
  int level;
  if (prob.backend == Backend::single_fmm) {
    level = std::max(2, static_cast<int>(std::lround(std::log2(std::sqrt(static_cast<double>(n))))));
    if (prob.leaf_level > 0) level = prob.leaf_level;
  } else {
    level = std::max(3, static_cast<int>(std::lround(std::log2(static_cast<double>(n) / 32.0))));
    if (prob.leaf_level > 0) level = prob.leaf_level;
  }
  BoxTree tree = build_tree(ps, level);
  LevelGrids grids = make_level_grids(prob.kernel, sigma, m, ps.d, level, GridMode::shared, 10);
  blfmm_plan* p = plan_for(ps, tree, prob.kernel, sigma, m, grids.factors[level].c_vals);
  std::vector<double> x(n, 0.0);
  blfmm_solve_stats st{};
  const int rc = blfmm_solve(p, pd ? BLFMM_SOLVE_CG : BLFMM_SOLVE_GMRES, prob.rhs.data(),
                             x.data(), prob.tol, prob.max_iter, &st);
  return finish(rc, st, x);
}

}  // namespace gpu
}  // namespace blfmm
