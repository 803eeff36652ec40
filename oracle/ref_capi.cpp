// Test infrastructure only: a C-ABI shim around the UNMODIFIED reference
// library, compiled from the sources under /root/reference/proj/core/src by
// oracle/Makefile into oracle/_ref/libblfmm_ref.so. Used by tests/ (to pin the
// restated oracle and the GPU path against the reference itself for d <= 2)
// and by bench.py's cpu_baseline / --impl reference leg. Never linked by the
// product.
//
// Wrapped reference entry points:
//   mlfmm_matvec            core/include/blfmm/mlfmm.hpp:98-99
//   fmm_matvec_single       core/include/blfmm/fmm.hpp:55
//   direct_matvec           core/include/blfmm/fmm.hpp:33-36
//   build_tree              core/include/blfmm/geometry.hpp:72
//   make_level_grids        core/include/blfmm/mlfmm.hpp:61-63
//   translation_coefficients core/include/blfmm/bandlimit.hpp:106-108
//   upsweep / couple        core/include/blfmm/mlfmm.hpp:79-87
//   direct_matvec (band-limited) / direct_matvec_hybrid
//                           core/include/blfmm/fmm.hpp:33-43
//   eval_bandlimited        core/include/blfmm/bandlimit.hpp:56-62
#include <chrono>
#include <cstring>
#include <string>

#include "blfmm/fmm.hpp"
#include "blfmm/mlfmm.hpp"

using namespace blfmm;

namespace {

thread_local std::string g_err;
GridMode g_mode = GridMode::shared;  // ref_set_grid_mode
int g_stencil = 10;

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
  } catch (const accuracy_error& e) {
    g_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 9;
  }
}

PointSet make_ps(int d, int n, const double* x, const double* lo,
                 const double* hi) {
  PointSet ps;
  ps.d = d;
  if (lo) ps.domain.lo = Pt{lo[0], d == 2 ? lo[1] : 0.0};
  if (hi) ps.domain.hi = Pt{hi[0], d == 2 ? hi[1] : 1.0};
  ps.pts.resize(n);
  for (int i = 0; i < n; ++i)
    ps.pts[i] = Pt{x[static_cast<size_t>(i) * d], d == 2 ? x[static_cast<size_t>(i) * d + 1] : 0.0};
  return ps;
}

void put_stats(const SumStats& s, long long* near, long long* far,
               double* imag) {
  if (near) *near = s.near_pairs;
  if (far) *far = s.far_work;
  if (imag) *imag = s.max_imag_residual;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// GridMode (0 shared, 1 scaled) and stencil_k of make_level_grids for the
// following ref_mlfmm / ref_expansions / ref_level_c_tables calls.
void ref_set_grid_mode(int mode, int stencil_k) {
  g_mode = mode == 1 ? GridMode::scaled : GridMode::shared;
  g_stencil = stencil_k;
}

// LevelGrids::factors[l].c_vals for l = 2..leaf, concatenated (K each).
int ref_level_c_tables(const char* spec, double sigma, int m, int d, int leaf, double* out) {
  return guard([&] {
    LevelGrids grids = make_level_grids(parse_kernel_spec(spec), sigma, m, d, leaf, g_mode,
                                        g_stencil);
    size_t pos = 0;
    for (int l = 2; l <= leaf; ++l) {
      const auto& c = grids.factors[l].c_vals;
      std::memcpy(out + pos, c.data(), c.size() * sizeof(double));
      pos += c.size();
    }
  });
}

int ref_eval_fourier(const char* spec, double xi, int d, double* out) {
  return guard([&] { *out = eval_fourier(parse_kernel_spec(spec), xi, d).value; });
}

int ref_eval_kernel(const char* spec, double r, double* out) {
  return guard([&] { *out = eval_kernel(parse_kernel_spec(spec), r); });
}

int ref_c_table(const char* spec, double sigma, int m, int d, double* c_out) {
  return guard([&] {
    auto g = make_quadrature(sigma, m, d);
    auto f = translation_coefficients(parse_kernel_spec(spec), g,
                                      TranslationMode::spectral);
    std::memcpy(c_out, f.c_vals.data(), f.c_vals.size() * sizeof(double));
  });
}

int ref_direct(int d, int n, const double* x, const char* spec,
               const double* w, double* out, long long* near) {
  return guard([&] {
    PointSet ps = make_ps(d, n, x, nullptr, nullptr);
    std::vector<double> wv(w, w + n);
    auto r = direct_matvec(parse_kernel_spec(spec), ps, wv, false, 0.0);
    std::memcpy(out, r.values.data(), n * sizeof(double));
    if (near) *near = r.stats.near_pairs;
  });
}

// One multilevel matvec with tree + grids built inside (shared grids by
// default, the mode both production callers force: blfmm_cli.cpp:384-385,
// solver.cpp:286-287; ref_set_grid_mode selects scaled grids). When `seconds` is given it receives the wall time of
// the mlfmm_matvec call alone (tree and grids prebuilt, the
// bench_matvec.cpp:48-61 convention), best of `reps`.
int ref_mlfmm(int d, int n, const double* x, const double* lo,
              const double* hi, const char* spec, double sigma, int m,
              int leaf, const double* w, double* out, long long* near,
              long long* far, double* imag, int reps, double* seconds) {
  return guard([&] {
    PointSet ps = make_ps(d, n, x, lo, hi);
    RadialKernel k = parse_kernel_spec(spec);
    BoxTree tree = build_tree(ps, leaf);
    LevelGrids grids =
        make_level_grids(k, sigma, m, d, leaf, g_mode, g_stencil);
    SumRequest req{k, sigma, &ps, std::vector<double>(w, w + n), m};
    double best = 1e300;
    SumResult r;
    for (int rep = 0; rep < (reps > 0 ? reps : 1); ++rep) {
      auto t0 = std::chrono::steady_clock::now();
      r = mlfmm_matvec(req, tree, grids);
      auto t1 = std::chrono::steady_clock::now();
      best = std::min(best, std::chrono::duration<double>(t1 - t0).count());
    }
    if (seconds) *seconds = best;
    std::memcpy(out, r.values.data(), n * sizeof(double));
    put_stats(r.stats, near, far, imag);
  });
}

int ref_single(int d, int n, const double* x, const double* lo,
               const double* hi, const char* spec, double sigma, int m,
               int level, const double* w, double* out, long long* near,
               long long* far, double* imag) {
  return guard([&] {
    PointSet ps = make_ps(d, n, x, lo, hi);
    BoxTree tree = build_tree(ps, level);
    SumRequest req{parse_kernel_spec(spec), sigma, &ps,
                   std::vector<double>(w, w + n), m};
    auto r = fmm_matvec_single(req, tree);
    std::memcpy(out, r.values.data(), n * sizeof(double));
    put_stats(r.stats, near, far, imag);
  });
}

// Stage-level expansions in reference box-id order (row-major), dense:
// out[(box * K + node) * 2 + {0,1}]. kind 0 = upsweep multipoles,
// kind 1 = couple() locals (before L2L).
int ref_expansions(int d, int n, const double* x, const double* lo,
                   const double* hi, const char* spec, double sigma, int m,
                   int leaf, const double* w, int level, int kind,
                   double* out) {
  return guard([&] {
    PointSet ps = make_ps(d, n, x, lo, hi);
    RadialKernel k = parse_kernel_spec(spec);
    BoxTree tree = build_tree(ps, leaf);
    LevelGrids grids =
        make_level_grids(k, sigma, m, d, leaf, g_mode, g_stencil);
    auto mult = upsweep(tree, grids, ps, std::vector<double>(w, w + n));
    const LevelExpansions* src = &mult;
    LevelExpansions loc;
    if (kind == 1) {
      loc = couple(tree, grids, mult);
      src = &loc;
    }
    size_t kk = grids.grids[level].node_count();
    for (size_t b = 0; b < (*src)[level].size(); ++b)
      for (size_t q = 0; q < kk; ++q) {
        out[(b * kk + q) * 2] = (*src)[level][b].coeffs[q].real();
        out[(b * kk + q) * 2 + 1] = (*src)[level][b].coeffs[q].imag();
      }
  });
}

// Tree lists of one level, flattened: counts[box] entries each, concatenated
// in box order into `ids` (caller sizes it by the first call with ids=NULL,
// which only fills counts). which: 0 neighbors, 1 interaction, 2 leaf points.
int ref_tree_lists(int d, int n, const double* x, const double* lo,
                   const double* hi, int leaf, int level, int which,
                   int* counts, int* ids) {
  return guard([&] {
    PointSet ps = make_ps(d, n, x, lo, hi);
    BoxTree tree = build_tree(ps, leaf);
    const std::vector<std::vector<int>>& lists =
        which == 0 ? tree.neighbors[level]
                   : (which == 1 ? tree.interaction[level] : tree.leaf_points);
    size_t pos = 0;
    for (size_t b = 0; b < lists.size(); ++b) {
      counts[b] = static_cast<int>(lists[b].size());
      if (ids)
        for (int v : lists[b]) ids[pos++] = v;
    }
  });
}

// Band-limited O(N^2) oracle (use_bandlimited = true) or, leaf >= 0, the
// hybrid oracle on build_tree(ps, leaf); d = 1.
int ref_direct_bl(int d, int n, const double* x, const double* lo, const double* hi,
                  const char* spec, const double* w, double sigma, int refinement, int leaf,
                  double* out) {
  return guard([&] {
    PointSet ps = make_ps(d, n, x, lo, hi);
    std::vector<double> wv(w, w + n);
    auto k = parse_kernel_spec(spec);
    SumResult r = leaf >= 0
                      ? direct_matvec_hybrid(k, ps, build_tree(ps, leaf), wv, sigma, refinement)
                      : direct_matvec(k, ps, wv, true, sigma, refinement);
    std::memcpy(out, r.values.data(), n * sizeof(double));
  });
}

int ref_eval_bandlimited(const char* spec, double sigma, double x, int refinement,
                         double* out) {
  return guard([&] {
    *out = eval_bandlimited(parse_kernel_spec(spec), sigma, Pt{x, 0.0}, 1, refinement);
  });
}

}  // extern "C"
