// O(N^2) direct and band-limited direct kernels.
// Fragment of blfmm.cu (one translation unit): included inside
// namespace blfmm_gpu after the plan definition; not a standalone header.

// ---------------------------------------------------------------- direct
// O(N^2) check, fmm.cpp:30-75: targets in ascending source order, every
// operation IEEE-rounded as the reference's (so IMQ / MQ sums are bit-identical
// to direct_matvec's; the Gaussian differs only by exp()'s last bit).
__device__ __forceinline__ double phi_ref(int type, double c, double r) {
  r = fabs(r);
  const double rr = __dmul_rn(r, r);
  if (type == BLFMM_KERNEL_GAUSSIAN) return exp(__dmul_rn(__dmul_rn(-c, r), r));
  if (type == BLFMM_KERNEL_TPS) {  // kernels.cpp:141-146: sign r^beta log r, 0 at r = 0
    if (r == 0.0) return 0.0;
    const int beta = static_cast<int>(c);
    double p = 1.0;  // pow_int: repeated multiplication
    for (int q = 0; q < beta; ++q) p = __dmul_rn(p, r);
    const double sign = (1 + beta / 2) % 2 == 0 ? 1.0 : -1.0;
    return __dmul_rn(__dmul_rn(sign, p), log(r));
  }
  if (type == BLFMM_KERNEL_WENDLAND_C2 || type == BLFMM_KERNEL_WENDLAND31) {
    const double u = __dmul_rn(c, r);  // kernels.cpp:147-158
    if (u >= 1.0) return 0.0;
    const double v = __dadd_rn(1.0, -u);
    const double v3 = __dmul_rn(__dmul_rn(v, v), v);
    if (type == BLFMM_KERNEL_WENDLAND_C2)
      return __dmul_rn(__dmul_rn(v3, v), __dadd_rn(__dmul_rn(4.0, u), 1.0));
    return __dmul_rn(v3, __dadd_rn(__dmul_rn(3.0, u), 1.0));
  }
  const double q = __dsqrt_rn(__dadd_rn(rr, __dmul_rn(c, c)));
  return type == BLFMM_KERNEL_IMQ ? __ddiv_rn(1.0, q) : q;
}
constexpr int kDirectThreads = 256;
template <int D>
__global__ void __launch_bounds__(kDirectThreads)
    k_direct(const double* __restrict__ x, const double* __restrict__ lam,
             long long n, const long long* __restrict__ targets, long long nt,
             int ktype, double kc, double* __restrict__ out) {
  __shared__ double sx[kDirectThreads][D + 1];
  long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  long long i = q < nt ? (targets ? targets[q] : q) : 0;
  double xi[3] = {0, 0, 0};
  if (q < nt)
    for (int k = 0; k < D; ++k) xi[k] = x[i * D + k];
  double acc = 0.0;
  for (long long j0 = 0; j0 < n; j0 += kDirectThreads) {
    __syncthreads();
    long long j = j0 + threadIdx.x;
    if (j < n) {
      for (int k = 0; k < D; ++k) sx[threadIdx.x][k] = x[j * D + k];
      sx[threadIdx.x][D] = lam[j];
    }
    __syncthreads();
    long long rem = n - j0;
    int cnt = rem < kDirectThreads ? static_cast<int>(rem) : kDirectThreads;
    for (int u = 0; u < cnt; ++u) {
      // the reference's arithmetic operation by operation (no contraction):
      // 1-D r = x_i - x_j (fmm.cpp:43), else r = dist() = sqrt(dx^2 + dy^2)
      // (common.hpp:21-29), then eval_kernel(r) (kernels.cpp:131-161)
      const double dx = __dsub_rn(xi[0], sx[u][0]);
      double r = dx;
      if (D > 1) {
        const double dy = __dsub_rn(xi[1], sx[u][1]);
        double s2 = __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
        if (D > 2) {
          const double dz = __dsub_rn(xi[2], sx[u][2]);
          s2 = __dadd_rn(s2, __dmul_rn(dz, dz));
        }
        r = __dsqrt_rn(s2);
      }
      acc = __dadd_rn(acc, __dmul_rn(sx[u][D], phi_ref(ktype, kc, r)));
    }
  }
  if (q < nt) out[q] = acc;
}

// Band-limited O(N^2) oracles, d = 1 (fmm.cpp:57-70 and 77-113): Phi_sigma
// from the cubic-interpolated radial table (RadialTable::operator(),
// bandlimit.cpp:229-239) held in shared memory, or - HYBRID - the original
// kernel for sources in the target leaf's 3-box neighbourhood (the tree's
// leaf_of binning, geometry.cpp:254-262; 1-D neighbours are |a - b| <= 1).
// Sources are summed in ascending index order, each operation IEEE-rounded.
constexpr int kDirectBLThreads = 256;
__device__ __forceinline__ int leaf_bin(double x, double lo, double side, int nleaf) {
  const double u = __ddiv_rn(__dsub_rn(x, lo), side);
  const int i = u >= 2147483647.0 ? nleaf - 1 : (u <= -2147483648.0 ? 0 : static_cast<int>(u));
  return min(max(i, 0), nleaf - 1);
}
template <bool HYBRID>
__global__ void __launch_bounds__(kDirectBLThreads)
    k_direct_bl1(const double* __restrict__ x, const double* __restrict__ lam, long long n,
                 const double* __restrict__ tab, int ntab, double step, int ktype, double kc,
                 double lo, double side, int nleaf, double* __restrict__ out) {
  extern __shared__ double bl_dyn[];  // [ntab] table + [kDirectBLThreads][3] sources
  double* stab = bl_dyn;
  double (*src)[3] = reinterpret_cast<double (*)[3]>(bl_dyn + ntab);
  for (int t = threadIdx.x; t < ntab; t += blockDim.x) stab[t] = tab[t];
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const double xi = i < n ? x[i] : 0.0;
  const int li = HYBRID ? leaf_bin(xi, lo, side, nleaf) : 0;
  double acc = 0.0;
  for (long long j0 = 0; j0 < n; j0 += kDirectBLThreads) {
    __syncthreads();
    const long long j = j0 + threadIdx.x;
    if (j < n) {
      src[threadIdx.x][0] = x[j];
      src[threadIdx.x][1] = lam[j];
      src[threadIdx.x][2] = HYBRID ? static_cast<double>(leaf_bin(x[j], lo, side, nleaf)) : 0.0;
    }
    __syncthreads();
    const long long rem = n - j0;
    const int cnt = rem < kDirectBLThreads ? static_cast<int>(rem) : kDirectBLThreads;
    for (int u = 0; u < cnt; ++u) {
      const double r = __dsub_rn(xi, src[u][0]);
      double v;
      if (HYBRID && abs(li - static_cast<int>(src[u][2])) <= 1) {
        v = phi_ref(ktype, kc, r);
      } else {
        const double uu = __ddiv_rn(fabs(r), step);
        const int k = min(max(uu >= 2147483647.0 ? ntab : static_cast<int>(uu), 1), ntab - 3);
        const double t = __dsub_rn(uu, static_cast<double>(k));
        const double tm1 = __dsub_rn(t, 1.0), tm2 = __dsub_rn(t, 2.0), tp1 = __dadd_rn(t, 1.0);
        const double tt1 = __dsub_rn(__dmul_rn(t, t), 1.0);
        const double w0 = __ddiv_rn(__dmul_rn(__dmul_rn(-t, tm1), tm2), 6.0);
        const double w1 = __ddiv_rn(__dmul_rn(tt1, tm2), 2.0);
        const double w2 = __ddiv_rn(__dmul_rn(__dmul_rn(-t, tp1), tm2), 2.0);
        const double w3 = __ddiv_rn(__dmul_rn(t, tt1), 6.0);
        v = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(stab[k - 1], w0), __dmul_rn(stab[k], w1)),
                                __dmul_rn(stab[k + 1], w2)),
                      __dmul_rn(stab[k + 2], w3));
      }
      acc = __dadd_rn(acc, __dmul_rn(src[u][1], v));
    }
  }
  if (i < n) out[i] = acc;
}
