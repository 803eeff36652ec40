// GridMode::scaled kernels (Lagrange M2M / L2L, direct IL couple).
// Fragment of blfmm.cu (one translation unit): included inside
// namespace blfmm_gpu after the plan definition; not a standalone header.

// ====================================================== scaled grids
constexpr long long kScaledMaxK = 6400;  // two K-vectors of double2 in shared memory
// GridMode::scaled (mlfmm.cpp:112-142, 148-197, 256-261, 331-337): level l has
// its own grid (sigma_l = sigma_leaf / 2^{L-l}, same M) and C table, M2M
// interpolates a child expansion onto the parent grid with the per-axis
// k-point Lagrange matrix P_l (tensor-applied, axis 0 first) before the phase
// shift, couple sums the interaction list directly (no telescoping: the
// transfers are not exact shifts), and L2L anterpolates with P^T, scales by
// the weight ratio w_l / w_{l+1} and shifts. P is stored dense [M][M].

// One tensor pass along axis `ax` over a K-vector in shared memory:
// dst[.., r, ..] = sum_c A[r][c] src[.., c, ..] (A = P, or P^T via transpose).
template <int D>
__device__ __forceinline__ void tensor_pass(const double2* __restrict__ src,
                                            double2* __restrict__ dst,
                                            const double* __restrict__ A, bool transpose,
                                            int M, int K, int ax) {
  int stride = 1;
  for (int q = ax + 1; q < D; ++q) stride *= M;
  for (int e = threadIdx.x; e < K; e += blockDim.x) {
    const int r = (e / stride) % M;
    const int base = e - r * stride;
    double2 acc = make_double2(0.0, 0.0);
    for (int c = 0; c < M; ++c) {
      const double w = transpose ? A[c * M + r] : A[r * M + c];
      if (w == 0.0) continue;
      const double2 v = src[base + c * stride];
      acc.x = fma(w, v.x, acc.x);
      acc.y = fma(w, v.y, acc.y);
    }
    dst[e] = acc;
  }
}

// M2M (scaled): one CTA per parent p at level l-1; every child expansion is
// interpolated in shared memory (2 K-buffers) and accumulated, shifted with
// the parent grid's phases tab[k][delta][m] = e^{i xi^{l-1}_m (1/2-delta) h_l}.
template <int D>
__global__ void k_m2m_scaled(const uint32_t* __restrict__ child_key,
                             const int* __restrict__ child_start,
                             const double2* __restrict__ child_mult, long long nchild,
                             long long nparent, const double* __restrict__ P,
                             const double2* __restrict__ tab, int M, int K,
                             double2* __restrict__ parent_mult) {
  extern __shared__ double2 sbuf[];  // [2][K]
  double2* b0 = sbuf;
  double2* b1 = sbuf + K;
  const long long p = blockIdx.x;
  const int r = blockIdx.y;
  double2* out = parent_mult + ((long long)r * nparent + p) * K;
  for (int e = threadIdx.x; e < K; e += blockDim.x) out[e] = make_double2(0.0, 0.0);
  for (int c = child_start[p]; c < child_start[p + 1]; ++c) {
    const double2* vc = child_mult + ((long long)r * nchild + c) * K;
    __syncthreads();
    for (int e = threadIdx.x; e < K; e += blockDim.x) b0[e] = vc[e];
    __syncthreads();
    double2* src = b0;
    double2* dst = b1;
    for (int ax = 0; ax < D; ++ax) {
      tensor_pass<D>(src, dst, P, false, M, K, ax);
      __syncthreads();
      double2* t = src;
      src = dst;
      dst = t;
    }
    const uint32_t oct = child_key[c];
    for (int e = threadIdx.x; e < K; e += blockDim.x) {
      int mk[3];
      node_axes<D>(e, M, nullptr, mk);
      double2 ph = make_double2(1.0, 0.0);
      for (int k = 0; k < D; ++k) {
        const int delta = (oct >> (D - 1 - k)) & 1;
        const double2 q = __ldg(&tab[(k * 2 + delta) * M + mk[k]]);
        ph = k == 0 ? q : cmul(ph, q);
      }
      double2 acc = out[e];
      cmac(acc, ph, src[e]);
      out[e] = acc;
    }
  }
}

// M2M (scaled), 3-D: one CTA (256 threads) per parent; per child the three
// interpolation passes use ONE shared K-buffer: axis 0 reads the child's
// expansion straight from global memory, axis 1 computes into registers and
// writes back after a barrier, axis 2 feeds the phase shift and the
// parent's accumulators, which stay in registers (KPT = K / 256 per thread).
// Taps come from the CSR form of P (k consecutive source nodes per row).
template <int KPT, int NT>
__global__ void __launch_bounds__(NT, 2)
    k_m2m_scaled3(const uint32_t* __restrict__ child_key, const int* __restrict__ child_start,
                  const double2* __restrict__ child_mult, long long nchild, long long nparent,
                  const int* __restrict__ plo, const double* __restrict__ pw, int kst,
                  const double2* __restrict__ tab, int M, int K,
                  double2* __restrict__ parent_mult) {
  extern __shared__ double2 sb[];  // [K]
  const long long p = blockIdx.x;
  const int r = blockIdx.y;
  const int MM = M * M;
  double2 acc[KPT], tmp[KPT];
#pragma unroll
  for (int i = 0; i < KPT; ++i) acc[i] = make_double2(0.0, 0.0);
  for (int c = child_start[p]; c < child_start[p + 1]; ++c) {
    const double2* vc = child_mult + ((long long)r * nchild + c) * K;
    __syncthreads();  // previous child's axis-2 reads done
    // axis 0 (stride M^2), global -> shared
#pragma unroll
    for (int i = 0; i < KPT; ++i) {
      const int e = threadIdx.x + NT * i;
      if (e >= K) continue;
      const int r0 = e / MM, rest = e - r0 * MM;
      double2 a = make_double2(0.0, 0.0);
      const int lo = plo[r0];
      for (int j = 0; j < kst; ++j) {
        const double w = pw[r0 * kst + j];
        const double2 x = __ldg(vc + (lo + j) * MM + rest);
        a.x = fma(w, x.x, a.x);
        a.y = fma(w, x.y, a.y);
      }
      sb[e] = a;
    }
    __syncthreads();
    // axis 1 (stride M), shared -> registers -> shared
#pragma unroll
    for (int i = 0; i < KPT; ++i) {
      const int e = threadIdx.x + NT * i;
      if (e >= K) continue;
      const int r1 = (e / M) % M, base = e - r1 * M;
      double2 a = make_double2(0.0, 0.0);
      const int lo = plo[r1];
      for (int j = 0; j < kst; ++j) {
        const double w = pw[r1 * kst + j];
        const double2 x = sb[base + (lo + j) * M];
        a.x = fma(w, x.x, a.x);
        a.y = fma(w, x.y, a.y);
      }
      tmp[i] = a;
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < KPT; ++i) {
      const int e = threadIdx.x + NT * i;
      if (e < K) sb[e] = tmp[i];
    }
    __syncthreads();
    // axis 2 (stride 1) + parent-grid phase shift into the accumulators
    const uint32_t oct = child_key[c];
    const int d0 = (oct >> 2) & 1, d1 = (oct >> 1) & 1, d2 = oct & 1;
#pragma unroll
    for (int i = 0; i < KPT; ++i) {
      const int e = threadIdx.x + NT * i;
      if (e >= K) continue;
      const int r2 = e % M, base = e - r2;
      double2 a = make_double2(0.0, 0.0);
      const int lo = plo[r2];
      for (int j = 0; j < kst; ++j) {
        const double w = pw[r2 * kst + j];
        const double2 x = sb[base + lo + j];
        a.x = fma(w, x.x, a.x);
        a.y = fma(w, x.y, a.y);
      }
      const int m0 = e / MM, m1 = (e / M) % M;
      double2 ph = __ldg(&tab[(0 * 2 + d0) * M + m0]);
      ph = cmul(ph, __ldg(&tab[(1 * 2 + d1) * M + m1]));
      ph = cmul(ph, __ldg(&tab[(2 * 2 + d2) * M + r2]));
      cmac(acc[i], ph, a);
    }
  }
  double2* out = parent_mult + ((long long)r * nparent + p) * K;
#pragma unroll
  for (int i = 0; i < KPT; ++i) {
    const int e = threadIdx.x + NT * i;
    if (e < K) out[e] = acc[i];
  }
}

// L2L (scaled), 3-D: one CTA per parent; the parent's local is anterpolated
// once (P^T along each axis, CSR of the transpose: column c collects the rows
// whose stencil covers it) with one shared K-buffer, the result stays in
// registers and is shifted into every child's local.
template <int KPT, int NT>
__global__ void __launch_bounds__(NT, 2)
    k_l2l_scaled3(const int* __restrict__ child_start, const uint32_t* __restrict__ child_key,
                  const double2* __restrict__ ploc, long long nparent, double2* __restrict__ cloc,
                  long long nchild, const int* __restrict__ tr, const double* __restrict__ tw,
                  int kt, const double2* __restrict__ tab, double wratio, int M, int K) {
  extern __shared__ double2 sb[];  // [K]
  const long long p = blockIdx.x;
  const int r = blockIdx.y;
  const int MM = M * M;
  const double2* lp = ploc + ((long long)r * nparent + p) * K;
  double2 t[KPT];
  // axis 0, global -> shared
#pragma unroll
  for (int i = 0; i < KPT; ++i) {
    const int e = threadIdx.x + NT * i;
    if (e >= K) continue;
    const int c0 = e / MM, rest = e - c0 * MM;
    double2 a = make_double2(0.0, 0.0);
    for (int j = 0; j < kt; ++j) {
      const double w = tw[c0 * kt + j];
      const double2 x = __ldg(lp + tr[c0 * kt + j] * MM + rest);
      a.x = fma(w, x.x, a.x);
      a.y = fma(w, x.y, a.y);
    }
    sb[e] = a;
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < KPT; ++i) {
    const int e = threadIdx.x + NT * i;
    if (e >= K) continue;
    const int c1 = (e / M) % M, base = e - c1 * M;
    double2 a = make_double2(0.0, 0.0);
    for (int j = 0; j < kt; ++j) {
      const double w = tw[c1 * kt + j];
      const double2 x = sb[base + tr[c1 * kt + j] * M];
      a.x = fma(w, x.x, a.x);
      a.y = fma(w, x.y, a.y);
    }
    t[i] = a;
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < KPT; ++i) {
    const int e = threadIdx.x + NT * i;
    if (e < K) sb[e] = t[i];
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < KPT; ++i) {
    const int e = threadIdx.x + NT * i;
    if (e >= K) continue;
    const int c2 = e % M, base = e - c2;
    double2 a = make_double2(0.0, 0.0);
    for (int j = 0; j < kt; ++j) {
      const double w = tw[c2 * kt + j];
      const double2 x = sb[base + tr[c2 * kt + j]];
      a.x = fma(w, x.x, a.x);
      a.y = fma(w, x.y, a.y);
    }
    t[i] = make_double2(wratio * a.x, wratio * a.y);
  }
  for (int c = child_start[p]; c < child_start[p + 1]; ++c) {
    const uint32_t oct = child_key[c];
    const int d0 = (oct >> 2) & 1, d1 = (oct >> 1) & 1, d2 = oct & 1;
    double2* lc = cloc + ((long long)r * nchild + c) * K;
#pragma unroll
    for (int i = 0; i < KPT; ++i) {
      const int e = threadIdx.x + NT * i;
      if (e >= K) continue;
      const int m0 = e / MM, m1 = (e / M) % M, m2 = e % M;
      double2 q0 = __ldg(&tab[(0 * 2 + d0) * M + m0]);
      double2 q1 = __ldg(&tab[(1 * 2 + d1) * M + m1]);
      double2 q2 = __ldg(&tab[(2 * 2 + d2) * M + m2]);
      q0.y = -q0.y;
      q1.y = -q1.y;
      q2.y = -q2.y;
      const double2 ph = cmul(cmul(q0, q1), q2);
      double2 v = lc[e];
      cmac(v, ph, t[i]);
      lc[e] = v;
    }
  }
}

// couple (scaled), mlfmm.cpp:268-299 literally: one CTA per (box a at level
// l, node chunk, rhs), thread = node; IL(a) = the children of the parent's
// 3^d block (coords 2p-2 .. 2p+3) minus a's 3^d neighbourhood, phase
// e^{i xi^l (x_a - x_b)} as a product of per-axis tabs (offsets -3..3).
constexpr int kCoupleSThreads = 128;
template <int D>
__global__ void __launch_bounds__(kCoupleSThreads)
    k_couple_scaled(const uint32_t* __restrict__ key, long long nbox, int level,
                    const int* __restrict__ slotmap, const double2* __restrict__ mult,
                    const double2* __restrict__ m2l_tab, const double* __restrict__ ctab, int M,
                    int K, double2* __restrict__ loc) {
  constexpr int E = D == 1 ? 6 : (D == 2 ? 36 : 216);
  __shared__ int slot[E];
  __shared__ signed char off[E][3];
  const long long a = blockIdx.x;
  const int r = blockIdx.z;
  int ac[3] = {0, 0, 0};
  morton_decode<D>(key[a], level, ac);
  const int n = 1 << level;
  for (int t = threadIdx.x; t < E; t += blockDim.x) {
    int q[3] = {0, 0, 0}, b[3] = {0, 0, 0};
    int rr = t;
    for (int k = D - 1; k >= 0; --k) {
      q[k] = rr % 6;
      rr /= 6;
    }
    bool ok = true, own = true;
    for (int k = 0; k < D; ++k) {
      b[k] = 2 * (ac[k] >> 1) - 2 + q[k];
      ok = ok && b[k] >= 0 && b[k] < n;
      own = own && abs(b[k] - ac[k]) <= 1;
      off[t][k] = static_cast<signed char>(ac[k] - b[k]);  // x_a - x_b = off * h
    }
    slot[t] = (ok && !own) ? slotmap[rowmajor_id<D>(b, level)] : -1;
  }
  __syncthreads();
  const int e = blockIdx.y * blockDim.x + threadIdx.x;
  if (e >= K) return;
  int mk[3];
  node_axes<D>(e, M, nullptr, mk);
  double2 acc = make_double2(0.0, 0.0);
  const double2* vm = mult + (long long)r * nbox * K + e;
  for (int t = 0; t < E; ++t) {
    const int s = slot[t];
    if (s < 0) continue;
    // m2l_tab[k][o + 3][m] = e^{-i xi_m o h}; x_a - x_b = off h => o = -off
    double2 ph = make_double2(1.0, 0.0);
    for (int k = 0; k < D; ++k) {
      const double2 q = __ldg(&m2l_tab[(k * 7 + (3 - off[t][k])) * M + mk[k]]);
      ph = k == 0 ? q : cmul(ph, q);
    }
    cmac(acc, ph, vm[(long long)s * K]);
  }
  const double cm = ctab[e];
  loc[((long long)r * nbox + a) * K + e] = make_double2(cm * acc.x, cm * acc.y);
}

// couple (scaled), 3-D, separable: one CTA per (parent p at level l-1, node
// chunk, rhs), thread = node. For each child a of p,
//   sum_{b in IL(a)} = sum over the 6^3 block of p's neighbours' children
//                      (coords 2p-2 .. 2p+3) - sum over a's 3^3 neighbourhood,
// both separable with the per-axis taps T_k(o) = e^{-i xi_k o h} (o = -3..3,
// T(-o) = conj T(o)): z, y and x passes stream through registers, so a box's
// 16 B are loaded once per parent instead of once per interaction.
constexpr int kCoupleS3Threads = 128;
template <int SCMINB>
__global__ void __launch_bounds__(kCoupleS3Threads, SCMINB)
    k_couple_scaled3(const uint32_t* __restrict__ pkey, long long nparent, int level,
                     const int* __restrict__ slotmap, const double2* __restrict__ mult,
                     long long nbox, const double2* __restrict__ m2l_tab,
                     const double* __restrict__ ctab, int M, int K,
                     double2* __restrict__ loc) {
  __shared__ int voff[216];
  __shared__ int slot[216];
  const long long p = blockIdx.x;
  const int r = blockIdx.z;
  int pc[3];
  morton_decode<3>(pkey[p], level - 1, pc);
  const int n = 1 << level;
  for (int t = threadIdx.x; t < 216; t += blockDim.x) {
    const int q[3] = {t / 36, (t / 6) % 6, t % 6};
    int b[3];
    bool ok = true;
    for (int k = 0; k < 3; ++k) {
      b[k] = 2 * pc[k] - 2 + q[k];
      ok = ok && b[k] >= 0 && b[k] < n;
    }
    const int sl = ok ? slotmap[rowmajor_id<3>(b, level)] : -1;
    slot[t] = sl;
    // empty boxes read the zero expansion after the level's last box
    voff[t] = static_cast<int>(((long long)r * nbox + (sl >= 0 ? sl : 0)) * K);
    if (sl < 0) voff[t] = static_cast<int>((long long)nbox * K * gridDim.z);
  }
  __syncthreads();
  const int e = blockIdx.y * blockDim.x + threadIdx.x;
  if (e >= K) return;
  int mk[3];
  node_axes<3>(e, M, nullptr, mk);
  double2 T[3][4];  // T[k][o] = e^{-i xi_k o h}, o = 1..3 (o = 0 is an add)
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    T[k][0] = make_double2(1.0, 0.0);
#pragma unroll
    for (int o = 1; o < 4; ++o) T[k][o] = __ldg(&m2l_tab[(k * 7 + o + 3) * M + mk[k]]);
  }
  // acc += T(o) v  (o may be negative: conj)
  auto tap = [](double2& acc, const double2 (&Tk)[4], int o, const double2& v) {
    if (o == 0) {
      acc.x += v.x;
      acc.y += v.y;
      return;
    }
    const double2 q = Tk[o < 0 ? -o : o];
    const double qy = o < 0 ? -q.y : q.y;
    acc.x = fma(q.x, v.x, fma(-qy, v.y, acc.x));
    acc.y = fma(q.x, v.y, fma(qy, v.x, acc.y));
  };
  // il = S6 - NS accumulated in one chain: at the x level an |o| <= 1 slice
  // contributes T(o) (y6 - y3), an outer slice T(o) y6
  double2 il[2][2][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int c = 0; c < 2; ++c) il[a][b][c] = make_double2(0.0, 0.0);
  const double2* v = mult + e;
#pragma unroll
  for (int x = 0; x < 6; ++x) {
    double2 y6[2][2], y3[2][2];
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int c = 0; c < 2; ++c) y6[b][c] = y3[b][c] = make_double2(0.0, 0.0);
#pragma unroll
    for (int y = 0; y < 6; ++y) {
      double2 col[6];
#pragma unroll
      for (int z = 0; z < 6; ++z) col[z] = __ldg(v + voff[(x * 6 + y) * 6 + z]);
      double2 z6[2], z3[2];
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        z3[c] = make_double2(0.0, 0.0);
#pragma unroll
        for (int z = 1 + c; z <= 3 + c; ++z) tap(z3[c], T[2], z - 2 - c, col[z]);
        z6[c] = z3[c];
#pragma unroll
        for (int z = 0; z < 6; ++z)
          if (z < 1 + c || z > 3 + c) tap(z6[c], T[2], z - 2 - c, col[z]);
      }
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        const int o = y - 2 - b;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          tap(y6[b][c], T[1], o, z6[c]);
          if (o >= -1 && o <= 1) tap(y3[b][c], T[1], o, z3[c]);
        }
      }
    }
#pragma unroll
    for (int a = 0; a < 2; ++a) {
      const int o = x - 2 - a;
#pragma unroll
      for (int b = 0; b < 2; ++b)
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          double2 yv = y6[b][c];
          if (o >= -1 && o <= 1) {
            yv.x -= y3[b][c].x;
            yv.y -= y3[b][c].y;
          }
          tap(il[a][b][c], T[0], o, yv);
        }
    }
  }
  const double cm = ctab[e];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int s = slot[((2 + a) * 6 + (2 + b)) * 6 + (2 + c)];
        if (s < 0) continue;
        loc[((long long)r * nbox + s) * K + e] =
            make_double2(cm * il[a][b][c].x, cm * il[a][b][c].y);
      }
}

// L2L (scaled): one CTA per parent p at level l; its accumulated local is
// anterpolated (P^T) in shared memory, scaled by wratio and shifted into each
// child's local (child grid phases tab[k][delta][m] = e^{i xi^{l+1}_m
// (1/2 - delta) h_{l+1}}, conjugated: x_c - x_p = (delta - 1/2) h).
template <int D>
__global__ void k_l2l_scaled(const int* __restrict__ child_start,
                             const uint32_t* __restrict__ child_key,
                             const double2* __restrict__ ploc, long long nparent,
                             double2* __restrict__ cloc, long long nchild,
                             const double* __restrict__ P, const double2* __restrict__ tab,
                             double wratio, int M, int K) {
  extern __shared__ double2 sbuf[];
  double2* b0 = sbuf;
  double2* b1 = sbuf + K;
  const long long p = blockIdx.x;
  const int r = blockIdx.y;
  const double2* lp = ploc + ((long long)r * nparent + p) * K;
  for (int e = threadIdx.x; e < K; e += blockDim.x) b0[e] = lp[e];
  __syncthreads();
  double2* src = b0;
  double2* dst = b1;
  for (int ax = 0; ax < D; ++ax) {
    tensor_pass<D>(src, dst, P, true, M, K, ax);
    __syncthreads();
    double2* t = src;
    src = dst;
    dst = t;
  }
  for (int c = child_start[p]; c < child_start[p + 1]; ++c) {
    const uint32_t oct = child_key[c];
    double2* lc = cloc + ((long long)r * nchild + c) * K;
    for (int e = threadIdx.x; e < K; e += blockDim.x) {
      int mk[3];
      node_axes<D>(e, M, nullptr, mk);
      double2 ph = make_double2(1.0, 0.0);
      for (int k = 0; k < D; ++k) {
        const int delta = (oct >> (D - 1 - k)) & 1;
        double2 q = __ldg(&tab[(k * 2 + delta) * M + mk[k]]);
        q.y = -q.y;
        ph = k == 0 ? q : cmul(ph, q);
      }
      const double2 t = cmul(ph, src[e]);
      double2 v = lc[e];
      v.x = fma(wratio, t.x, v.x);
      v.y = fma(wratio, t.y, v.y);
      lc[e] = v;
    }
  }
}

// Plan-time region tables: for every parent slot p at level l-1, the level-l
// slots of the 4^d block around its children (coords 2p-1 .. 2p+2 per axis),
// -1 for empty / outside the domain. 4^d ints per parent (256 B in 3-D).
template <int D>
__global__ void k_region_slots(const uint32_t* __restrict__ parent_key, long long nparent,
                               int level, const int* __restrict__ slotmap,
                               int* __restrict__ region) {
  constexpr int E1 = D >= 2 ? 4 : 1, E2 = D == 3 ? 4 : 1, REG = 4 * E1 * E2;
  const long long gid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (gid >= nparent * REG) return;
  const long long p = gid / REG;
  const int t = static_cast<int>(gid % REG);
  int pc[3] = {0, 0, 0};
  morton_decode<D>(parent_key[p], level - 1, pc);
  const int n = 1 << level;
  int q[3] = {t / (E1 * E2), (t / E2) % E1, t % E2}, b[3];
  bool ok = true;
  for (int k = 0; k < D; ++k) {
    b[k] = 2 * pc[k] - 1 + q[k];
    ok = ok && b[k] >= 0 && b[k] < n;
  }
  region[gid] = ok ? slotmap[rowmajor_id<D>(b, level)] : -1;
}
