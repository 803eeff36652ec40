// Krylov caller of the matvec: the iteration of solve_interpolation
// (solver.cpp:43-88 run_cg, 90-203 run_gmres, 269-300) on device vectors.
// The matvec is the plan's own blfmm_execute_device (the FMM kernels); the
// vector algebra is a handful of small kernels with deterministic two-pass
// reductions (fixed block partition, partial sums added in block order), so
// a solve is bit-reproducible. The small Hessenberg / Givens work of GMRES
// stays on the host, as in the reference.
#include <cuda_runtime.h>

#include <algorithm>
#include <functional>
#include <cmath>
#include <limits>
#include <string>
#include <vector>

#include "blfmm_internal.h"

namespace blfmm_gpu {
namespace {

constexpr int kRedThreads = 256, kRedBlocks = 592;  // 4 per SM on 148 SMs

__global__ void k_dot_partial(const double* __restrict__ a, const double* __restrict__ b,
                              long long n, double* __restrict__ part) {
  __shared__ double sh[kRedThreads];
  double s = 0.0;
  for (long long i = blockIdx.x * (long long)kRedThreads + threadIdx.x; i < n;
       i += (long long)gridDim.x * kRedThreads)
    s = fma(a[i], b[i], s);
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int o = kRedThreads / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}
__global__ void k_sum_partials(const double* __restrict__ part, int m, double* __restrict__ out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < m; ++i) s += part[i];
    *out = s;
  }
}
// y = y + alpha x  (alpha read from the host argument)
__global__ void k_axpy(double* __restrict__ y, const double* __restrict__ x, double alpha,
                       long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    y[i] = fma(alpha, x[i], y[i]);
}
// p = r + beta p
__global__ void k_xpby(double* __restrict__ p, const double* __restrict__ r, double beta,
                       long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    p[i] = r[i] + beta * p[i];
}
// y = s x
__global__ void k_scale_copy(double* __restrict__ y, const double* __restrict__ x, double s,
                             long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    y[i] = s * x[i];
}
// y = b - y
__global__ void k_bminus(double* __restrict__ y, const double* __restrict__ b, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    y[i] = b[i] - y[i];
}

void ck(cudaError_t e) {
  if (e != cudaSuccess) throw Error(BLFMM_ECUDA, cudaGetErrorString(e));
}
void ckb(int rc) {
  if (rc != BLFMM_OK) throw Error(rc, blfmm_last_error());
}

struct Vecs {
  long long n;
  cudaStream_t st;
  double* part = nullptr;  // [kRedBlocks + 1]
  std::vector<double*> bufs;
  Vecs(long long n_, cudaStream_t s) : n(n_), st(s) {
    ck(cudaMalloc(&part, sizeof(double) * (kRedBlocks + 1)));
  }
  ~Vecs() {
    cudaFree(part);
    for (double* b : bufs) cudaFree(b);
  }
  double* alloc() {
    double* p = nullptr;
    ck(cudaMalloc(&p, sizeof(double) * std::max<long long>(n, 1)));
    bufs.push_back(p);
    return p;
  }
  unsigned grid() const {
    return static_cast<unsigned>(std::min<long long>((n + 255) / 256, 148LL * 8));
  }
  double dot(const double* a, const double* b) {
    k_dot_partial<<<kRedBlocks, kRedThreads, 0, st>>>(a, b, n, part);
    k_sum_partials<<<1, 32, 0, st>>>(part, kRedBlocks, part + kRedBlocks);
    double h = 0.0;
    ck(cudaMemcpyAsync(&h, part + kRedBlocks, sizeof(double), cudaMemcpyDeviceToHost, st));
    ck(cudaStreamSynchronize(st));
    return h;
  }
  void axpy(double* y, const double* x, double a) { k_axpy<<<grid(), 256, 0, st>>>(y, x, a, n); }
  void xpby(double* p, const double* r, double b) { k_xpby<<<grid(), 256, 0, st>>>(p, r, b, n); }
  void scale(double* y, const double* x, double s) {
    k_scale_copy<<<grid(), 256, 0, st>>>(y, x, s, n);
  }
  void bminus(double* y, const double* b) { k_bminus<<<grid(), 256, 0, st>>>(y, b, n); }
};

// solver.cpp:43-88
// y = A x on device vectors, on the solve's stream: the plan's FMM matvec
// (blfmm_solve) or the dense kernel sum (blfmm_solve_dense)
using Apply = std::function<void(const double*, double*)>;

void run_cg(const Apply& apply, Vecs& v, const double* b, double* x, double tol, int max_iter,
            blfmm_solve_stats& st) {
  const long long n = v.n;
  st.method = BLFMM_SOLVE_CG;
  ck(cudaMemsetAsync(x, 0, sizeof(double) * n, v.st));
  const double bnorm = std::sqrt(v.dot(b, b));
  if (bnorm == 0.0) {
    st.converged = 1;
    return;
  }
  double* r = v.alloc();
  double* p = v.alloc();
  double* ap = v.alloc();
  ck(cudaMemcpyAsync(r, b, sizeof(double) * n, cudaMemcpyDeviceToDevice, v.st));
  ck(cudaMemcpyAsync(p, b, sizeof(double) * n, cudaMemcpyDeviceToDevice, v.st));
  double rr = v.dot(r, r);
  double best = std::sqrt(rr) / bnorm;
  for (int it = 0; it < max_iter; ++it) {
    apply(p, ap);
    ++st.matvecs;
    const double pap = v.dot(p, ap);
    if (pap <= 0.0) break;  // matrix not PD to working precision
    const double alpha = rr / pap;
    v.axpy(x, p, alpha);
    v.axpy(r, ap, -alpha);
    const double rr_new = v.dot(r, r);
    st.iterations = it + 1;
    const double rel = std::sqrt(rr_new) / bnorm;
    best = std::min(best, rel);
    if (rel <= tol) {
      st.residual = rel;
      st.converged = 1;
      return;
    }
    const double beta = rr_new / rr;
    rr = rr_new;
    v.xpby(p, r, beta);
  }
  st.residual = best;
  Error e(BLFMM_EACCURACY, "cg did not reach tolerance");
  e.achieved = best;
  throw e;
}

// solver.cpp:90-203 (restart min(max_iter, 300), modified Gram-Schmidt,
// Givens rotations, breakdown at |w| < 1e-14 beta)
void run_gmres(const Apply& apply, Vecs& v, const double* b, double* x, double tol, int max_iter,
               blfmm_solve_stats& st) {
  const long long n = v.n;
  st.method = BLFMM_SOLVE_GMRES;
  ck(cudaMemsetAsync(x, 0, sizeof(double) * n, v.st));
  const double bnorm = std::sqrt(v.dot(b, b));
  if (bnorm == 0.0) {
    st.converged = 1;
    return;
  }
  const int restart = std::min(max_iter, 300);
  double best = std::numeric_limits<double>::infinity();
  int total_it = 0;
  double* r = v.alloc();
  double* w = v.alloc();
  std::vector<double*> basis;  // V columns, allocated on first use and reused per cycle
  while (total_it < max_iter) {
    if (total_it == 0) {
      ck(cudaMemcpyAsync(r, b, sizeof(double) * n, cudaMemcpyDeviceToDevice, v.st));
    } else {
      apply(x, r);
      ++st.matvecs;
      v.bminus(r, b);
    }
    const double beta = std::sqrt(v.dot(r, r));
    if (beta / bnorm <= tol) {
      st.residual = beta / bnorm;
      st.converged = 1;
      return;
    }
    const int m = std::min(restart, max_iter - total_it);
    if (basis.empty()) basis.push_back(v.alloc());
    v.scale(basis[0], r, 1.0 / beta);
    std::vector<std::vector<double>> h;
    std::vector<double> cs, sn, g{beta};
    int k = 0;
    for (; k < m; ++k) {
      apply(basis[k], w);
      ++st.matvecs;
      h.emplace_back(k + 2, 0.0);
      for (int j = 0; j <= k; ++j) {
        const double d = v.dot(w, basis[j]);
        h[k][j] = d;
        v.axpy(w, basis[j], -d);
      }
      const double wn = std::sqrt(v.dot(w, w));
      h[k][k + 1] = wn;
      const bool breakdown = wn < 1e-14 * beta;
      if (!breakdown) {
        if ((int)basis.size() < k + 2) basis.push_back(v.alloc());
        v.scale(basis[k + 1], w, 1.0 / wn);
      }
      for (int j = 0; j < k; ++j) {
        const double t = cs[j] * h[k][j] + sn[j] * h[k][j + 1];
        h[k][j + 1] = -sn[j] * h[k][j] + cs[j] * h[k][j + 1];
        h[k][j] = t;
      }
      const double denom = std::hypot(h[k][k], h[k][k + 1]);
      cs.push_back(h[k][k] / denom);
      sn.push_back(h[k][k + 1] / denom);
      h[k][k] = denom;
      h[k][k + 1] = 0.0;
      g.push_back(-sn[k] * g[k]);
      g[k] = cs[k] * g[k];
      ++total_it;
      st.iterations = total_it;
      const double rel = std::abs(g[k + 1]) / bnorm;
      best = std::min(best, rel);
      if (rel <= tol || breakdown) {
        ++k;
        break;
      }
    }
    std::vector<double> y(k, 0.0);
    for (int j = k - 1; j >= 0; --j) {
      double s = g[j];
      for (int l = j + 1; l < k; ++l) s -= h[l][j] * y[l];
      y[j] = s / h[j][j];
    }
    for (int j = 0; j < k; ++j) v.axpy(x, basis[j], y[j]);
    apply(x, r);
    ++st.matvecs;
    v.bminus(r, b);
    const double res = std::sqrt(v.dot(r, r)) / bnorm;
    best = std::min(best, res);
    if (res <= tol) {
      st.residual = res;
      st.converged = 1;
      return;
    }
  }
  st.residual = best;
  Error e(BLFMM_EACCURACY, "gmres did not reach tolerance");
  e.achieved = best;
  throw e;
}

}  // namespace
}  // namespace blfmm_gpu

namespace blfmm_gpu {
namespace {
// the shared body of blfmm_solve / blfmm_solve_dense: device vectors, the
// Krylov loop, the best iterate back to the host even when it throws
int solve_body(long long n, const std::function<Apply(cudaStream_t)>& make_apply, int method,
               const double* b, double* x, double tol, int max_iter, blfmm_solve_stats* stats) {
  blfmm_solve_stats st{};
  int rc = BLFMM_OK;
  try {
    if (n && (!b || !x)) throw Error(BLFMM_EINVAL, "null rhs / solution");
    if (!(tol > 0.0)) throw Error(BLFMM_EINVAL, "tol must be positive");
    if (method != BLFMM_SOLVE_CG && method != BLFMM_SOLVE_GMRES)
      throw Error(BLFMM_EINVAL, "unknown Krylov method");
    cudaStream_t s = nullptr;
    ck(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    struct StreamGuard {
      cudaStream_t s;
      ~StreamGuard() { cudaStreamDestroy(s); }
    } sg{s};
    const Apply apply = make_apply(s);
    Vecs v(n, s);
    double* db = v.alloc();
    double* dx = v.alloc();
    if (n) ck(cudaMemcpyAsync(db, b, sizeof(double) * n, cudaMemcpyHostToDevice, s));
    try {
      if (method == BLFMM_SOLVE_CG) run_cg(apply, v, db, dx, tol, max_iter, st);
      else run_gmres(apply, v, db, dx, tol, max_iter, st);
    } catch (const Error&) {
      if (n) {  // the best iterate so far, as the reference's result
        cudaMemcpyAsync(x, dx, sizeof(double) * n, cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
      }
      throw;
    }
    if (n) ck(cudaMemcpyAsync(x, dx, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
    ck(cudaStreamSynchronize(s));
  } catch (const Error& e) {
    set_error(e);
    rc = e.code;
  } catch (const std::bad_alloc&) {
    set_error_message("host allocation failed");
    rc = BLFMM_ENOMEM;
  } catch (const std::exception& e) {
    set_error_message(e.what());
    rc = BLFMM_EINVAL;
  }
  if (stats) *stats = st;
  return rc;
}
}  // namespace
}  // namespace blfmm_gpu

extern "C" int blfmm_solve(blfmm_plan* plan, int method, const double* b, double* x, double tol,
                           int max_iter, blfmm_solve_stats* stats) {
  using namespace blfmm_gpu;
  blfmm_plan_info info{};
  try {
    if (!plan) throw Error(BLFMM_EINVAL, "null plan");
    ckb(blfmm_plan_get_info(plan, &info));
    if (info.nrhs != 1) throw Error(BLFMM_EINVAL, "the solver takes a one right-hand-side plan");
  } catch (const Error& e) {
    set_error(e);
    if (stats) *stats = blfmm_solve_stats{};
    return e.code;
  }
  return solve_body(
      info.n,
      [plan](cudaStream_t s) -> Apply {
        return [plan, s](const double* in, double* out) {
          ckb(blfmm_execute_device(plan, in, out, nullptr, s));
        };
      },
      method, b, x, tol, max_iter, stats);
}

// solve_interpolation, Backend::dense (solver.cpp:207-262, 269-275): the same
// Krylov loops on the dense kernel matrix A_ij = phi(|x_i - x_j|), applied
// matrix-free on the device (k_direct) instead of assembled; every
// RadialKernel type; N <= 8192 as assemble_dense (std::length_error beyond).
extern "C" int blfmm_solve_dense(int d, long long n, const double* coords, int kernel_type,
                                 double shape, int method, const double* b, double* x,
                                 double tol, int max_iter, blfmm_solve_stats* stats,
                                 int device) {
  using namespace blfmm_gpu;
  double* dcoords = nullptr;
  int prev = -1;
  try {
    if (d < 1 || d > 3) throw Error(BLFMM_EINVAL, "d must be 1, 2 or 3");
    if (n < 0) throw Error(BLFMM_EINVAL, "n must be >= 0");
    if (n > 8192) throw Error(BLFMM_ELENGTH, "dense assembly capped at N=8192");
    if (n && !coords) throw Error(BLFMM_EINVAL, "null coordinates");
    require_radial_kernel(KernelSpec{kernel_type, shape});
    if (device >= 0) {
      ck(cudaGetDevice(&prev));
      ck(cudaSetDevice(device));
    }
    if (n) {
      ck(cudaMalloc(&dcoords, sizeof(double) * n * d));
      ck(cudaMemcpy(dcoords, coords, sizeof(double) * n * d, cudaMemcpyHostToDevice));
    }
  } catch (const Error& e) {
    set_error(e);
    if (dcoords) cudaFree(dcoords);
    if (prev >= 0) cudaSetDevice(prev);
    if (stats) *stats = blfmm_solve_stats{};
    return e.code;
  }
  const int rc = solve_body(
      n,
      [=](cudaStream_t s) -> Apply {
        return [=](const double* in, double* out) {
          direct_device(d, n, dcoords, kernel_type, shape, in, out, s);
        };
      },
      method, b, x, tol, max_iter, stats);
  if (dcoords) cudaFree(dcoords);
  if (prev >= 0) cudaSetDevice(prev);
  return rc;
}
