// Scalar L2P / near field, phase tables, FP64 DMMA helpers, generic / 2-D / large-M P2M and L2P.
// Fragment of blfmm.cu (one translation unit): included inside
// namespace blfmm_gpu after the plan definition; not a standalone header.

// ---------------------------------------------------------------- L2P
// u_i += Re sum_m w_m e^{i xi_m . (x_i - x_a)} L_a[m]  (mlfmm.cpp:342-357)
constexpr int kL2PThreads = 256;

template <int D, int kL2PBatch>
__global__ void __launch_bounds__(kL2PThreads)
    k_l2p(const uint32_t* __restrict__ leaf_key, const int* __restrict__ leaf_start,
          const double* __restrict__ x0, const double* __restrict__ x1,
          const double* __restrict__ x2, const double2* __restrict__ loc,
          const double* __restrict__ xi, int M, long long K, int L, long long n,
          long long nleaf, double lo0, double lo1, double lo2, double s0,
          double s1, double s2, double weight, double* __restrict__ far_,
          unsigned long long* __restrict__ imag_bits) {
  extern __shared__ double2 smem[];
  double2* ph = smem;  // [kL2PBatch][D][M]
  __shared__ double2 red[kL2PThreads / 32][kL2PBatch];
  const long long a = blockIdx.x;
  const int r = blockIdx.y;
  int c[3];
  morton_decode<D>(leaf_key[a], L, c);
  const double lo[3] = {lo0, lo1, lo2}, side[3] = {s0, s1, s2};
  double xa[3];
  for (int k = 0; k < D; ++k) xa[k] = lo[k] + (c[k] + 0.5) * side[k];
  const int p0 = leaf_start[a], p1 = leaf_start[a + 1];
  const double* xs[3] = {x0, x1, x2};
  const double2* la = loc + ((long long)r * nleaf + a) * K;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double imag_max = 0.0;
  for (int pb = p0; pb < p1; pb += kL2PBatch) {
    int nb = min(kL2PBatch, p1 - pb);
    __syncthreads();
    double2 part[kL2PBatch];
#pragma unroll
    for (int j = 0; j < kL2PBatch; ++j) part[j] = make_double2(0.0, 0.0);
    if (D == 1) {
      // d = 1: node = m and each point-node phase is used once: formed in
      // registers (no staged rows, any M); same operations as the staged form
      double rk[kL2PBatch];
#pragma unroll
      for (int j = 0; j < kL2PBatch; ++j) rk[j] = j < nb ? x0[pb + j] - xa[0] : 0.0;
      for (long long e = threadIdx.x; e < K; e += blockDim.x) {
        const double2 lv = la[e];
        const double xe = xi[e];
#pragma unroll
        for (int j = 0; j < kL2PBatch; ++j)
          if (j < nb) cmac(part[j], polar1(xe * rk[j]), lv);
      }
    } else {
    for (int t = threadIdx.x; t < nb * D * M; t += blockDim.x) {
      int j = t / (D * M), k = (t / M) % D, m = t % M;
      double rk = xs[k][pb + j] - xa[k];
      ph[t] = polar1(xi[m] * rk);
    }
    __syncthreads();
    for (long long e = threadIdx.x; e < K; e += blockDim.x) {
      int mk[3];
      long long t = e;
      for (int k = D - 1; k >= 0; --k) {
        mk[k] = static_cast<int>(t % M);
        t /= M;
      }
      double2 lv = la[e];
#pragma unroll
      for (int j = 0; j < kL2PBatch; ++j) {
        if (j < nb) {
          const double2* pj = ph + (size_t)j * D * M;
          double2 p = pj[mk[0]];
          if (D > 1) p = cmul(p, pj[M + mk[1]]);
          if (D > 2) p = cmul(p, pj[2 * M + mk[2]]);
          cmac(part[j], p, lv);
        }
      }
    }
    }
#pragma unroll
    for (int j = 0; j < kL2PBatch; ++j) {
      for (int off = 16; off > 0; off >>= 1) {
        part[j].x += __shfl_down_sync(0xffffffffu, part[j].x, off);
        part[j].y += __shfl_down_sync(0xffffffffu, part[j].y, off);
      }
      if (lane == 0) red[warp][j] = part[j];
    }
    __syncthreads();
    if (threadIdx.x < nb) {
      double2 s = make_double2(0.0, 0.0);
      for (int w = 0; w < kL2PThreads / 32; ++w) {
        s.x += red[w][threadIdx.x].x;
        s.y += red[w][threadIdx.x].y;
      }
      far_[(long long)r * n + pb + threadIdx.x] = weight * s.x;
      imag_max = fmax(imag_max, fabs(weight * s.y));
    }
  }
  if (threadIdx.x < kL2PBatch && imag_max > 0.0)
    atomicMax(imag_bits, static_cast<unsigned long long>(__double_as_longlong(imag_max)));
}

// ---------------------------------------------------------------- near
// u_i += sum_{b in N(a)} sum_{j in b} lambda_j phi(|x_i - x_j|)
// (mlfmm.cpp:381-396): original kernel, self term included. One CTA per
// target leaf, one thread per target, RT right-hand sides per thread.
constexpr int kNearThreads = 64;

template <int D, int RT>
__global__ void __launch_bounds__(kNearThreads)
    k_near(const uint32_t* __restrict__ leaf_key, const int* __restrict__ leaf_start,
           const int* __restrict__ slotmap, const double* __restrict__ x0,
           const double* __restrict__ x1, const double* __restrict__ x2,
           const double* __restrict__ lam, long long n, int R, int L, int ktype,
           double kc, double* __restrict__ near_) {
  const long long a = blockIdx.x;
  const int r0 = blockIdx.y * RT;
  int c[3], b[3];
  morton_decode<D>(leaf_key[a], L, c);
  const int nper = 1 << L;
  const int p0 = leaf_start[a], p1 = leaf_start[a + 1];
  int nbr[D == 1 ? 3 : (D == 2 ? 9 : 27)];
  int nn = 0;
  constexpr int tot = D == 1 ? 3 : (D == 2 ? 9 : 27);
  for (int q = 0; q < tot; ++q) {
    int rr = q;
    bool ok = true;
    for (int k = D - 1; k >= 0; --k) {
      b[k] = c[k] + rr % 3 - 1;
      rr /= 3;
      ok = ok && b[k] >= 0 && b[k] < nper;
    }
    int s = ok ? slotmap[rowmajor_id<D>(b, L)] : -1;
    if (s >= 0) nbr[nn++] = s;
  }
  for (int i = p0 + threadIdx.x; i < p1; i += blockDim.x) {
    double xi0 = x0[i], xi1 = D > 1 ? x1[i] : 0.0, xi2 = D > 2 ? x2[i] : 0.0;
    double acc[RT];
#pragma unroll
    for (int q = 0; q < RT; ++q) acc[q] = 0.0;
    for (int u = 0; u < nn; ++u) {
      int s = nbr[u];
      int j0 = leaf_start[s], j1 = leaf_start[s + 1];
      for (int j = j0; j < j1; ++j) {
        double dx = xi0 - x0[j], s2 = dx * dx;
        if (D > 1) {
          double dy = xi1 - x1[j];
          s2 = fma(dy, dy, s2);
        }
        if (D > 2) {
          double dz = xi2 - x2[j];
          s2 = fma(dz, dz, s2);
        }
        double ph = phi_of_r2(ktype, kc, s2);
#pragma unroll
        for (int q = 0; q < RT; ++q)
          if (RT == 1 || r0 + q < R) acc[q] = fma(lam[(long long)(r0 + q) * n + j], ph, acc[q]);
      }
    }
#pragma unroll
    for (int q = 0; q < RT; ++q)
      if (RT == 1 || r0 + q < R) near_[(long long)(r0 + q) * n + i] = acc[q];
  }
}

// ------------------------------------------- plan-time per-point phases
// ph[(i*D + k)*M + m] = e^{i xi_m (x_{i,k} - x_{a(i),k})} for sorted point i in
// leaf a(i). Geometry only, so it is built once per plan; L2P uses it as is,
// P2M uses its conjugate e^{i xi_m (x_a - x_i)} (sin is odd: bit-identical to
// evaluating the negated argument).
template <int D>
__global__ void k_point_phases(const uint32_t* __restrict__ leaf_key,
                               const int* __restrict__ leaf_start, long long nleaf,
                               const double* __restrict__ x0, const double* __restrict__ x1,
                               const double* __restrict__ x2, const double* __restrict__ xi,
                               int M, int L, double lo0, double lo1, double lo2, double s0,
                               double s1, double s2, double2* __restrict__ ph) {
  const long long a = blockIdx.x;
  int c[3];
  morton_decode<D>(leaf_key[a], L, c);
  const double ctr[3] = {lo0 + (c[0] + 0.5) * s0, lo1 + (c[1] + 0.5) * s1,
                         lo2 + (c[2] + 0.5) * s2};
  const int p0 = leaf_start[a], p1 = leaf_start[a + 1];
  const int per = D * M;
  for (long long t = threadIdx.x; t < (long long)(p1 - p0) * per; t += blockDim.x) {
    const long long i = p0 + t / per;
    const int k = static_cast<int>((t / M) % D), m = static_cast<int>(t % M);
    const double xk = k == 0 ? x0[i] : (k == 1 ? x1[i] : x2[i]);
    ph[i * per + k * M + m] = polar1(xi[m] * (xk - ctr[k]));
  }
}

// ---------------------------------------------------- FP64 DMMA helpers
// mma.sync.aligned.m8n8k4 f64 (sm_80+ DMMA, 8x8x4 per warp): lane holds
// A[m = lane/4][k = lane%4], B[k = lane%4][n = lane/4] and
// C[m = lane/4][n = 2*(lane%4) + v], v = 0, 1 (cute SM80_8x8x4_F64F64F64F64_TN).
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}
// complex C += A B with four real DMMAs (A_im passed negated for the real part)
struct CTile {
  double re[2], im[2];
};
__device__ __forceinline__ void cdmma(CTile& c, double are, double aim, double anim, double bre,
                                      double bim) {
  dmma(c.re[0], c.re[1], are, bre);
  dmma(c.re[0], c.re[1], anim, bim);
  dmma(c.im[0], c.im[1], are, bim);
  dmma(c.im[0], c.im[1], aim, bre);
}

// complex C += A B with three real DMMAs (3M: T1 = (Ar + Ai) Br,
// T2 = Ar (Bi - Br), T3 = Ai (Br + Bi); C = (T1 - T3, T1 + T2)); the operand
// sums are formed once per fragment by the caller.
struct CTile3 {
  double t1[2], t2[2], t3[2];
};
__device__ __forceinline__ void cdmma3(CTile3& c, double asum, double ar, double ai, double br,
                                       double bdiff, double bsum) {
  dmma(c.t1[0], c.t1[1], asum, br);
  dmma(c.t2[0], c.t2[1], ar, bdiff);
  dmma(c.t3[0], c.t3[1], ai, bsum);
}
__device__ __forceinline__ double2 ctile3_get(const CTile3& c, int v) {
  return make_double2(c.t1[v] - c.t3[v], c.t1[v] + c.t2[v]);
}
constexpr CTile3 kZeroTile3{{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};

// ---------------------------------------------------- P2M on FP64 DMMA
// V[row][c] = sum_j A[row][j] B[j][c] (complex), tiles 8 rows x 8 columns x 4
// points: A[row][j] = lambda_j conj(prod_{k<d-1} P_{k,j}[m_k]) is formed per
// fragment element from the plan-time phase table, B[j][c] =
// conj(P_{d-1,j}[c]). A warp owns WR x WC tiles; a CTA is 4 warps along rows.
template <int D, int WR, int WC>
__global__ void __launch_bounds__(128)
    k_p2m_mma(const int* __restrict__ leaf_list, const int* __restrict__ leaf_start,
              const double2* __restrict__ pht,
              const double* __restrict__ lam, int M, long long K, long long n, long long nleaf,
              int ncb, double2* __restrict__ mult) {
  const long long a = leaf_list ? leaf_list[blockIdx.x] : blockIdx.x;
  const int r = blockIdx.z;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, tq = lane & 3;
  const long long rows = K / M;
  const int rb = blockIdx.y / ncb, cb = blockIdx.y % ncb;
  const long long rt0 = ((long long)rb * 4 + warp) * WR;  // first row tile of this warp
  const int ct0 = cb * WC;
  const int per = D * M;
  int m1[WR], m2[WR];
  bool rv[WR];
#pragma unroll
  for (int q = 0; q < WR; ++q) {
    const long long row = (rt0 + q) * 8 + g;
    rv[q] = row < rows;
    const long long rc = rv[q] ? row : 0;
    m1[q] = D == 3 ? static_cast<int>(rc / M) : static_cast<int>(rc);
    m2[q] = D == 3 ? static_cast<int>(rc % M) : 0;
  }
  int cc[WC];
  bool cv[WC];
#pragma unroll
  for (int u = 0; u < WC; ++u) {
    const int col = (ct0 + u) * 8 + g;
    cv[u] = col < M;
    cc[u] = cv[u] ? col : 0;
  }
  CTile acc[WR][WC];
#pragma unroll
  for (int q = 0; q < WR; ++q)
#pragma unroll
    for (int u = 0; u < WC; ++u) acc[q][u] = CTile{{0.0, 0.0}, {0.0, 0.0}};
  const int p0 = leaf_start[a], p1 = leaf_start[a + 1];
  const double* lr = lam + (long long)r * n;
  for (int j0 = p0; j0 < p1; j0 += 4) {
    const int j = j0 + tq;
    const bool jv = j < p1;
    const double2* pj = pht + (long long)(jv ? j : p0) * per;
    const double w = jv ? __ldg(lr + j) : 0.0;
    double are[WR], aim[WR], anim[WR], bre[WC], bim[WC];
#pragma unroll
    for (int q = 0; q < WR; ++q) {
      double2 z = __ldg(pj + m1[q]);
      if (D == 3) z = cmul(z, __ldg(pj + M + m2[q]));
      const double ww = rv[q] ? w : 0.0;
      are[q] = ww * z.x;
      aim[q] = -ww * z.y;  // conj
      anim[q] = ww * z.y;
    }
#pragma unroll
    for (int u = 0; u < WC; ++u) {
      const double2 z = __ldg(pj + (D - 1) * M + cc[u]);
      bre[u] = cv[u] ? z.x : 0.0;
      bim[u] = cv[u] ? -z.y : 0.0;  // conj
    }
#pragma unroll
    for (int q = 0; q < WR; ++q)
#pragma unroll
      for (int u = 0; u < WC; ++u) cdmma(acc[q][u], are[q], aim[q], anim[q], bre[u], bim[u]);
  }
  double2* out = mult + ((long long)r * nleaf + a) * K;
#pragma unroll
  for (int q = 0; q < WR; ++q) {
    const long long row = (rt0 + q) * 8 + g;
    if (row >= rows) continue;
#pragma unroll
    for (int u = 0; u < WC; ++u) {
      const int col = (ct0 + u) * 8 + 2 * tq;
      if (col + 1 < M) {
        *reinterpret_cast<double4*>(out + row * M + col) =
            make_double4(acc[q][u].re[0], acc[q][u].im[0], acc[q][u].re[1], acc[q][u].im[1]);
      } else if (col < M) {
        out[row * M + col] = make_double2(acc[q][u].re[0], acc[q][u].im[0]);
      }
    }
  }
}

// ---------------------------------------------------- L2P on FP64 DMMA
// W[i][row] = sum_c P_{d-1,i}[c] L[row][c] as 8-point x 8-row x 4-column DMMA
// tiles (A = the points' phases, B = L^T), then
// u_i = w Re sum_row Prow_i[row] W[i][row] in the epilogue (vector FP64).
// CTA = 4 warps per (leaf, 8-point tile); warp w takes row tiles w, w+4, ...
// in groups of WN; the per-point sums finish with shuffles + shared memory.
template <int D, int WN>
__global__ void __launch_bounds__(128)
    k_l2p_mma(const int2* __restrict__ work, const int* __restrict__ leaf_start,
              const double2* __restrict__ pht,
              const double2* __restrict__ loc, int M, long long K, long long n,
              long long nleaf, double weight, double* __restrict__ far_,
              unsigned long long* __restrict__ imag_bits) {
  __shared__ double2 red[4][8];
  const int2 item = work[blockIdx.x];  // (leaf, first point of an 8-point tile)
  const long long a = item.x;
  const int r = blockIdx.z;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, tq = lane & 3;
  const long long rows = K / M;
  const long long rtiles = (rows + 7) / 8;
  const int p1 = leaf_start[a + 1];
  const int pb = item.y;
  const int per = D * M;
  const double2* la = loc + ((long long)r * nleaf + a) * K;
  // A fragment point (row of A): g; epilogue point (row of C): g as well
  const int ia = pb + g;
  const bool iv = ia < p1;
  const double2* pa = pht + (long long)(iv ? ia : pb) * per;
  double2 part = make_double2(0.0, 0.0);
  for (long long tb = (long long)warp * WN; tb < rtiles; tb += 4LL * WN) {
    CTile acc[WN];
#pragma unroll
    for (int u = 0; u < WN; ++u) acc[u] = CTile{{0.0, 0.0}, {0.0, 0.0}};
    const double2* lrow[WN];
    bool bv[WN];
#pragma unroll
    for (int u = 0; u < WN; ++u) {
      const long long row = (tb + u) * 8 + g;  // B column n = g
      bv[u] = (tb + u) < rtiles && row < rows;
      lrow[u] = la + (bv[u] ? row : 0) * M;
    }
    for (int k0 = 0; k0 < M; k0 += 4) {
      const int c = k0 + tq;
      const bool kv = c < M;
      double2 z = (iv && kv) ? __ldg(pa + (D - 1) * M + c) : make_double2(0.0, 0.0);
      const double are = z.x, aim = z.y, anim = -z.y;
#pragma unroll
      for (int u = 0; u < WN; ++u) {
        const double2 lv = (bv[u] && kv) ? __ldg(lrow[u] + c) : make_double2(0.0, 0.0);
        cdmma(acc[u], are, aim, anim, lv.x, lv.y);
      }
    }
    // epilogue: C[i = g][row = 8 (tb+u) + 2 tq + v]
#pragma unroll
    for (int u = 0; u < WN; ++u) {
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const long long row = (tb + u) * 8 + 2 * tq + v;
        if ((tb + u) >= rtiles || row >= rows || !iv) continue;
        const int mm1 = D == 3 ? static_cast<int>(row / M) : static_cast<int>(row);
        const int mm2 = D == 3 ? static_cast<int>(row % M) : 0;
        double2 pr = __ldg(pa + mm1);
        if (D == 3) pr = cmul(pr, __ldg(pa + M + mm2));
        cmac(part, pr, make_double2(acc[u].re[v], acc[u].im[v]));
      }
    }
  }
  // sum over the 4 lanes of a point (tq), then over warps
  for (int off = 1; off < 4; off <<= 1) {
    part.x += __shfl_xor_sync(0xffffffffu, part.x, off);
    part.y += __shfl_xor_sync(0xffffffffu, part.y, off);
  }
  if (tq == 0) red[warp][g] = part;
  __syncthreads();
  if (threadIdx.x < 8 && pb + threadIdx.x < p1) {
    double2 sum = red[0][threadIdx.x];
    for (int w = 1; w < 4; ++w) {
      sum.x += red[w][threadIdx.x].x;
      sum.y += red[w][threadIdx.x].y;
    }
    far_[(long long)r * n + pb + threadIdx.x] = weight * sum.x;
    const double im = fabs(weight * sum.y);
    if (im > 0.0)
      atomicMax(imag_bits, static_cast<unsigned long long>(__double_as_longlong(im)));
  }
}


// ------------------------- phases generated in registers (north star: the
// plane-wave factors e^{i xi_m t} of P2M / L2P are not read from a table)
// e^{ix} for the small arguments of leaf-relative phases (|x| <= 1/8: Taylor
// to x^13 / x^14, truncation < 1e-25 relative), the library sincos otherwise.
__device__ __forceinline__ double2 polar_small(double x) {
  if (fabs(x) > 0.125) return polar1(x);
  const double x2 = x * x;
  double sn = 1.0 / 6227020800.0;        // 1/13!
  sn = fma(sn, -x2, 1.0 / 39916800.0);   // 1/11!
  sn = fma(sn, -x2, 1.0 / 362880.0);     // 1/9!
  sn = fma(sn, -x2, 1.0 / 5040.0);       // 1/7!
  sn = fma(sn, -x2, 1.0 / 120.0);        // 1/5!
  sn = fma(sn, -x2, 1.0 / 6.0);          // 1/3!
  sn = fma(-sn * x2, x, x);
  double cs = 1.0 / 87178291200.0;       // 1/14!
  cs = fma(cs, -x2, 1.0 / 479001600.0);  // 1/12!
  cs = fma(cs, -x2, 1.0 / 3628800.0);    // 1/10!
  cs = fma(cs, -x2, 1.0 / 40320.0);      // 1/8!
  cs = fma(cs, -x2, 1.0 / 720.0);        // 1/6!
  cs = fma(cs, -x2, 1.0 / 24.0);         // 1/4!
  cs = fma(cs, -x2, 0.5);                // 1/2!
  cs = fma(-cs, x2, 1.0);
  return make_double2(cs, sn);
}
// The M = 16 phase row e^{i xi_m t}, m = 0..15: the grid -sigma + m dxi has
// xi_8 = 0 exactly and xi_{16-m} = -xi_m, so the row is the powers of
// s = e^{i dxi t}: s^{m-8} for m >= 8 and conj(s^{8-m}) below (one sincos,
// 7 products in a depth-3 tree).
__device__ __forceinline__ void gen_row16(double tv, double dxi, double2* __restrict__ row) {
  double2 pw[9];
  pw[0] = make_double2(1.0, 0.0);
  pw[1] = polar_small(dxi * tv);
  pw[2] = cmul(pw[1], pw[1]);
  pw[3] = cmul(pw[2], pw[1]);
  pw[4] = cmul(pw[2], pw[2]);
  pw[5] = cmul(pw[4], pw[1]);
  pw[6] = cmul(pw[4], pw[2]);
  pw[7] = cmul(pw[4], pw[3]);
  pw[8] = cmul(pw[4], pw[4]);
#pragma unroll
  for (int m = 0; m < 16; ++m) row[m] = m >= 8 ? pw[m - 8] : make_double2(pw[8 - m].x, -pw[8 - m].y);
}
// gen_row16 with a row stride (the 2-D kernels' [m][point] staging)
__device__ __forceinline__ void gen_row16s(double tv, double dxi, double2* __restrict__ out,
                                           int stride) {
  double2 pw[9];
  pw[0] = make_double2(1.0, 0.0);
  pw[1] = polar_small(dxi * tv);
  pw[2] = cmul(pw[1], pw[1]);
  pw[3] = cmul(pw[2], pw[1]);
  pw[4] = cmul(pw[2], pw[2]);
  pw[5] = cmul(pw[4], pw[1]);
  pw[6] = cmul(pw[4], pw[2]);
  pw[7] = cmul(pw[4], pw[3]);
  pw[8] = cmul(pw[4], pw[4]);
#pragma unroll
  for (int m = 0; m < 16; ++m)
    out[m * stride] = m >= 8 ? pw[m - 8] : make_double2(pw[8 - m].x, -pw[8 - m].y);
}

// ----------------------- 2-D, M = 16 (K = 256): P2M / L2P on FP64 DMMA
// One warp per leaf (P2M) or per 32-point chunk of a leaf (L2P); the point
// phases of a 16-point chunk are generated by the warp into shared memory
// (lanes 0-15: axis 0 of one point each, lanes 16-31: axis 1; gen_row16s: the
// M = 16 grid is symmetric about xi_8 = 0, so a row is the powers of
// e^{i dxi t} - one small-angle sincos and 7 products) and read back as DMMA
// fragments. Row strides are chosen so the fragment reads of a
// quarter warp hit distinct 16-byte bank groups.
constexpr int kP2D = 16;      // points per generated chunk
constexpr int kP2DSA = 20;    // P2M row stride (== 4 mod 8)
constexpr int kP2DS0 = 17;    // L2P P0 stride (odd)
constexpr int kP2DS1 = 18;    // L2P P1 stride (== 2 mod 8)

// V[m1][m2] = sum_j lambda_j conj(P0_j[m1]) conj(P1_j[m2]): A[m1][j] =
// lambda_j conj(P0_j[m1]), B[j][m2] = conj(P1_j[m2]); 2 x 2 tiles of 8 x 8
// per warp, k = 4 points per step (mlfmm.cpp:218-231).
__global__ void __launch_bounds__(128)
    k_p2m_2d16(const int* __restrict__ leaf_list, long long nitems,
               const uint32_t* __restrict__ leaf_key, const int* __restrict__ leaf_start,
               const double* __restrict__ x0, const double* __restrict__ x1,
               const double* __restrict__ lam, long long n, long long nleaf, int L, double lo0,
               double lo1, double s0, double s1, double sigma, double dxi,
               double2* __restrict__ mult) {
  __shared__ __align__(16) double2 sA[4][16][kP2DSA];
  __shared__ __align__(16) double2 sB[4][16][kP2DSA];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long item = (long long)blockIdx.x * 4 + warp;
  if (item >= nitems) return;
  const long long a = leaf_list ? leaf_list[item] : item;
  const int r = blockIdx.z;
  const int g = lane >> 2, tq = lane & 3;
  int c[2];
  morton_decode<2>(leaf_key[a], L, c);
  const int half = lane >> 4, pl = lane & 15;
  const double ctr = half ? lo1 + (c[1] + 0.5) * s1 : lo0 + (c[0] + 0.5) * s0;
  const double* __restrict__ xs = half ? x1 : x0;
  double2* gen = half ? &sB[warp][0][pl] : &sA[warp][0][pl];
  const double* lr = lam + (long long)r * n;
  CTile acc[2][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) acc[i][j] = CTile{{0.0, 0.0}, {0.0, 0.0}};
  const int p0 = leaf_start[a], p1 = leaf_start[a + 1];
  // the next chunk's coordinate and weight are loaded while this one is contracted
  double xn = p0 + pl < p1 ? __ldg(xs + p0 + pl) : ctr;
  double wn = (!half && p0 + pl < p1) ? __ldg(lr + p0 + pl) : 0.0;
  for (int j0 = p0; j0 < p1; j0 += kP2D) {
    {
      const double t = xn - ctr, w = wn;
      const int jn = j0 + kP2D + pl;
      xn = jn < p1 ? __ldg(xs + jn) : ctr;
      wn = (!half && jn < p1) ? __ldg(lr + jn) : 0.0;
      gen_row16s(-t, dxi, gen, kP2DSA);  // conj phases: e^{-i xi_m t}
      if (!half) {
#pragma unroll
        for (int m = 0; m < 16; ++m) {
          double2 z = sA[warp][m][pl];
          sA[warp][m][pl] = make_double2(w * z.x, w * z.y);
        }
      }
    }
    __syncwarp();
#pragma unroll
    for (int kk = 0; kk < kP2D / 4; ++kk) {
      const int pt = kk * 4 + tq;
      double2 av[2], bv[2];
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        av[i] = sA[warp][i * 8 + g][pt];
        bv[i] = sB[warp][i * 8 + g][pt];
      }
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) cdmma(acc[i][j], av[i].x, av[i].y, -av[i].y, bv[j].x, bv[j].y);
    }
    __syncwarp();
  }
  double2* out = mult + ((long long)r * nleaf + a) * 256;
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j)
      *reinterpret_cast<double4*>(out + (i * 8 + g) * 16 + j * 8 + 2 * tq) =
          make_double4(acc[i][j].re[0], acc[i][j].im[0], acc[i][j].re[1], acc[i][j].im[1]);
}

// u_i = w Re sum_{m1, m2} P0_i[m1] P1_i[m2] L[m1][m2] (mlfmm.cpp:342-357):
// W[i][m1] = sum_{m2} P1_i[m2] L[m1][m2] on DMMA (A = P1, 8 points x 4 nodes;
// B[m2][m1] = L[m1][m2], held in registers for the whole item), then
// u_i = w Re sum_{m1} P0_i[m1] W[i][m1] on the accumulator fragments.
// work[item] = (leaf, first point of a span of <= `span` points): a warp keeps
// the leaf's B fragments for the whole span (128: one load of the local
// expansion per 64-point leaf; the 32-point items left the kernel waiting on
// global loads, long-scoreboard 68 % of the stall samples).
__global__ void __launch_bounds__(128)
    k_l2p_2d16(const int2* __restrict__ work, long long nitems,
               const uint32_t* __restrict__ leaf_key, const int* __restrict__ leaf_start,
               const double* __restrict__ x0, const double* __restrict__ x1,
               const double2* __restrict__ loc, long long n, long long nleaf, int L, double lo0,
               double lo1, double s0, double s1, double sigma, double dxi, double weight,
               double* __restrict__ far_, unsigned long long* __restrict__ imag_bits, int span) {
  __shared__ __align__(16) double2 sP0[4][16][kP2DS0];
  __shared__ __align__(16) double2 sP1[4][16][kP2DS1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long item = (long long)blockIdx.x * 4 + warp;
  if (item >= nitems) return;
  const int2 it = work[item];
  const long long a = it.x;
  const int r = blockIdx.z;
  const int g = lane >> 2, tq = lane & 3;
  int c[2];
  morton_decode<2>(leaf_key[a], L, c);
  const int half = lane >> 4, pl = lane & 15;
  const double ctr = half ? lo1 + (c[1] + 0.5) * s1 : lo0 + (c[0] + 0.5) * s0;
  const double* __restrict__ xs = half ? x1 : x0;
  double2* gen = half ? &sP1[warp][0][pl] : &sP0[warp][0][pl];
  const int gstride = half ? kP2DS1 : kP2DS0;
  // B fragments: L[m1 = 8 nt + g][m2 = 4 ks + tq]
  const double2* la = loc + ((long long)r * nleaf + a) * 256;
  double2 bl[2][4];
#pragma unroll
  for (int nt = 0; nt < 2; ++nt)
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) bl[nt][ks] = __ldg(la + (nt * 8 + g) * 16 + ks * 4 + tq);
  const int p1 = leaf_start[a + 1];
  const int pend = min(p1, it.y + span);
  double* fr = far_ + (long long)r * n;
  double imax = 0.0;
  // the next chunk's coordinate is loaded while the current chunk is contracted
  double xn = it.y + pl < pend ? __ldg(xs + it.y + pl) : ctr;
  for (int j0 = it.y; j0 < pend; j0 += kP2D) {
    {
      const double t = xn - ctr;
      const int jn = j0 + kP2D + pl;
      xn = jn < pend ? __ldg(xs + jn) : ctr;
      gen_row16s(t, dxi, gen, gstride);
    }
    __syncwarp();
#pragma unroll
    for (int tile = 0; tile < kP2D / 8; ++tile) {
      CTile acc[2];
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) acc[nt] = CTile{{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        const double2 av = sP1[warp][ks * 4 + tq][tile * 8 + g];
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) cdmma(acc[nt], av.x, av.y, -av.y, bl[nt][ks].x, bl[nt][ks].y);
      }
      // C[i = g][m1 = 8 nt + 2 tq + v]
      double2 part = make_double2(0.0, 0.0);
#pragma unroll
      for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int v = 0; v < 2; ++v)
          cmac(part, sP0[warp][nt * 8 + 2 * tq + v][tile * 8 + g],
               make_double2(acc[nt].re[v], acc[nt].im[v]));
#pragma unroll
      for (int o = 1; o < 4; o <<= 1) {
        part.x += __shfl_xor_sync(0xffffffffu, part.x, o);
        part.y += __shfl_xor_sync(0xffffffffu, part.y, o);
      }
      const int i = j0 + tile * 8 + g;
      if (tq == 0 && i < pend) {
        fr[i] = weight * part.x;
        imax = fmax(imax, fabs(weight * part.y));
      }
    }
    __syncwarp();
  }
  if (imax > 0.0) atomicMax(imag_bits, static_cast<unsigned long long>(__double_as_longlong(imax)));
}

// ------------------------ 3-D full grid, large M (P2: M = 58, K = 195,112)
// The generic DMMA P2M above re-reads, per CTA, the leaf's point phases (one
// CTA per 128 x 16 output tile: ~80 GB of L2 traffic per P2 matvec). This one
// is a CTA per (leaf, 64-row block) with the leaf's P3 phases and weights
// staged in shared memory and all M3 column tiles per warp (P2 P2M 28.1 ->
// 24.6 ms). The same treatment of L2P (a CTA per 64-point span, every row
// tile of the local expansion read once, 8 or 4 point tiles per warp)
// measured slower than k_l2p_mma (33.8 / 26.3 vs 20.7 ms: 184 registers, and
// the epilogue's per-point P1 P2 loads), so L2P keeps the generic kernel.
constexpr int kBigPts = 64;  // points per CTA (P2M: leaf chunk; L2P: span)

// P2M: V[(m1, m2)][m3] = sum_j conj(P1_j[m1] P2_j[m2]) lambda_j conj(P3_j[m3]),
// warp w: row tile 8 blockIdx.y + w (8 warps), all ceil(M / 8) column tiles.
template <int MCT, int RPW = 1>
__global__ void __launch_bounds__(256, 1)
    k_p2m_big(const int* __restrict__ leaf_list, const int* __restrict__ leaf_start,
              const double2* __restrict__ pht, const double* __restrict__ lam, int M,
              long long K, long long n, long long nleaf, double2* __restrict__ mult,
              int coff, int ncol) {
  // columns m3 = coff .. coff + ncol - 1, stored at row * ncol + (m3 - coff):
  // the full grid (0, M), or block A of the half spectrum (M / 2, M / 2)
  extern __shared__ __align__(16) double2 big_dyn[];
  double2* s3 = big_dyn;                                   // [kBigPts][ncol]  lambda conj(P3)
  const long long a = leaf_list ? leaf_list[blockIdx.x] : blockIdx.x;
  const int r = blockIdx.z;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, tq = lane & 3;
  const long long rows = (long long)M * M;
  // RPW row tiles per warp: tiles (8 blockIdx.y + warp) RPW + q
  long long row[RPW];
  bool rv[RPW];
  int m1[RPW], m2[RPW];
#pragma unroll
  for (int q = 0; q < RPW; ++q) {
    row[q] = ((8LL * blockIdx.y + warp) * RPW + q) * 8 + g;  // this lane's A row
    rv[q] = row[q] < rows;
    m1[q] = rv[q] ? static_cast<int>(row[q] / M) : 0;
    m2[q] = rv[q] ? static_cast<int>(row[q] % M) : 0;
  }
  const int p0 = leaf_start[a], p1 = leaf_start[a + 1];
  const double* lr = lam + (long long)r * n;
  const int per = 3 * M;
  CTile acc[RPW][MCT];
#pragma unroll
  for (int q = 0; q < RPW; ++q)
#pragma unroll
    for (int u = 0; u < MCT; ++u) acc[q][u] = CTile{{0.0, 0.0}, {0.0, 0.0}};
  for (int c0 = p0; c0 < p1; c0 += kBigPts) {
    const int nb = min(kBigPts, p1 - c0);
    __syncthreads();
    for (int t = threadIdx.x; t < nb * ncol; t += blockDim.x) {
      const int j = t / ncol, c = t % ncol;
      const double2 z = __ldg(pht + (long long)(c0 + j) * per + 2 * M + coff + c);
      const double w = __ldg(lr + c0 + j);
      s3[j * ncol + c] = make_double2(w * z.x, -w * z.y);
    }
    __syncthreads();
    for (int j0 = 0; j0 < nb; j0 += 4) {
      const int j = j0 + tq;
      const bool jv = j < nb;
      double2 bv[MCT];
#pragma unroll
      for (int u = 0; u < MCT; ++u) {
        const int col = 8 * u + g;
        bv[u] = (jv && col < ncol) ? s3[j * ncol + col] : make_double2(0.0, 0.0);
      }
      const double2* pj = pht + (long long)(c0 + (jv ? j : 0)) * per;
#pragma unroll
      for (int q = 0; q < RPW; ++q) {
        double2 za = make_double2(0.0, 0.0);
        if (jv && rv[q]) za = cmul(__ldg(pj + m1[q]), __ldg(pj + M + m2[q]));
        const double are = za.x, aim = -za.y;  // conj(P1 P2)
#pragma unroll
        for (int u = 0; u < MCT; ++u) cdmma(acc[q][u], are, aim, -aim, bv[u].x, bv[u].y);
      }
    }
  }
  double2* out = mult + ((long long)r * nleaf + a) * K;
#pragma unroll
  for (int q = 0; q < RPW; ++q) {
    const long long orow = row[q];  // C row = g
    if (orow >= rows) continue;
#pragma unroll
    for (int u = 0; u < MCT; ++u) {
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const int col = 8 * u + 2 * tq + v;
        if (col < ncol) out[orow * ncol + col] = make_double2(acc[q][u].re[v], acc[q][u].im[v]);
      }
    }
  }
}

// Large-M P2M of a column window of at most 32 columns (block A of the half
// spectrum) in the 3-multiplication complex form: 3 real DMMAs per complex tile
// step instead of 4 (k_l2p_h16S's scheme). A CTA takes a leaf and a group of
// its row tiles: the B operand lambda conj(P3) of up to kBig3Pts points is
// staged ONCE as three real planes (b_r, b_i - b_r, b_r + b_i; row stride 36
// doubles = conflict-free quarter-warp LDS.64; zero filled beyond the leaf's
// points and the column window, so the contraction carries no predicates),
// then the warps loop over the group's row tiles (RPW per warp and pass); the
// A operand conj(P1 P2) of the next k step is loaded while the current one is
// contracted. k_p2m_big staged B once per 128 rows (27 times per P2 leaf) and
// waited on it: P2 P2M 11.9 -> see DESIGN.md §4. Leaves of more than kBig3Pts
// points take further chunks that add to the stored sums (same CTA, in order).
constexpr int kBig3CS = 36;   // plane row stride (doubles), = 4 mod 16
constexpr int kBig3Pts = 96;  // points per staged chunk
template <int RPW, int NW, int MINB>
__global__ void __launch_bounds__(32 * NW, MINB)
    k_p2m_big3(const int* __restrict__ leaf_list, const int* __restrict__ leaf_start,
               const double2* __restrict__ pht, const double* __restrict__ lam, int M,
               long long K, long long n, long long nleaf, double2* __restrict__ mult, int coff,
               int ncol, int ngroup) {
  constexpr int MCT = 4;
  extern __shared__ __align__(16) double big3_dyn[];  // [3][kBig3Pts][kBig3CS]
  double* const sr = big3_dyn;
  double* const sd = sr + kBig3Pts * kBig3CS;
  double* const ss = sd + kBig3Pts * kBig3CS;
  const long long li = blockIdx.x / ngroup;
  const int grp = static_cast<int>(blockIdx.x - li * ngroup);
  const long long a = leaf_list ? leaf_list[li] : li;
  const int r = blockIdx.z;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, tq = lane & 3;
  const int rows = M * M, rtiles = (rows + 7) / 8;
  // this group's row tiles [t_lo, t_hi), in passes of NW * RPW tiles
  const int per_grp = (rtiles + ngroup - 1) / ngroup;
  const int t_lo = grp * per_grp, t_hi = min(rtiles, t_lo + per_grp);
  const int p0 = leaf_start[a], p1 = leaf_start[a + 1];
  const double* lr = lam + (long long)r * n;
  const int per = 3 * M;
  double2* const out = mult + ((long long)r * nleaf + a) * K;
  for (int c0 = p0; c0 < p1; c0 += kBig3Pts) {
    const int nb = min(kBig3Pts, p1 - c0), nb4 = (nb + 3) & ~3;
    __syncthreads();
    for (int t = threadIdx.x; t < nb4 * 32; t += blockDim.x) {
      const int j = t >> 5, c = t & 31;
      double br = 0.0, bi = 0.0;
      if (j < nb && c < ncol) {
        const double2 z = __ldg(pht + (long long)(c0 + j) * per + 2 * M + coff + c);
        const double w = __ldg(lr + c0 + j);
        br = w * z.x;
        bi = -w * z.y;
      }
      sr[j * kBig3CS + c] = br;
      sd[j * kBig3CS + c] = bi - br;
      ss[j * kBig3CS + c] = br + bi;
    }
    __syncthreads();
    for (int tb = t_lo + warp * RPW; tb < t_hi; tb += NW * RPW) {
      int m1[RPW], m2[RPW], row[RPW];
#pragma unroll
      for (int q = 0; q < RPW; ++q) {
        row[q] = (tb + q) * 8 + g;  // this lane's A row
        // rows past the group / the grid: any finite A, never stored
        const int rc = (tb + q < t_hi && row[q] < rows) ? row[q] : 0;
        m1[q] = rc / M;
        m2[q] = rc - m1[q] * M;
      }
      CTile3 acc[RPW][MCT];
#pragma unroll
      for (int q = 0; q < RPW; ++q)
#pragma unroll
        for (int u = 0; u < MCT; ++u) acc[q][u] = kZeroTile3;
      double2 a1[RPW], a2[RPW];
      auto load_a = [&](int j0) {
        const double2* pj = pht + (long long)(c0 + min(j0 + tq, nb - 1)) * per;
#pragma unroll
        for (int q = 0; q < RPW; ++q) {
          a1[q] = __ldg(pj + m1[q]);
          a2[q] = __ldg(pj + M + m2[q]);
        }
      };
      load_a(0);
      for (int j0 = 0; j0 < nb; j0 += 4) {
        double are[RPW], aim[RPW];
#pragma unroll
        for (int q = 0; q < RPW; ++q) {
          const double2 za = cmul(a1[q], a2[q]);
          are[q] = za.x;
          aim[q] = -za.y;  // conj(P1 P2)
        }
        if (j0 + 4 < nb) load_a(j0 + 4);
        const int o = (j0 + tq) * kBig3CS + g;
#pragma unroll
        for (int u = 0; u < MCT; ++u) {
          const double br = sr[o + 8 * u], bd = sd[o + 8 * u], bs = ss[o + 8 * u];
#pragma unroll
          for (int q = 0; q < RPW; ++q)
            cdmma3(acc[q][u], are[q] + aim[q], are[q], aim[q], br, bd, bs);
        }
      }
#pragma unroll
      for (int q = 0; q < RPW; ++q) {
        if (tb + q >= t_hi || row[q] >= rows) continue;
        double2* orow = out + (long long)row[q] * ncol;  // C row = g
#pragma unroll
        for (int u = 0; u < MCT; ++u) {
#pragma unroll
          for (int v = 0; v < 2; ++v) {
            const int col = 8 * u + 2 * tq + v;
            if (col >= ncol) continue;
            double2 w = ctile3_get(acc[q][u], v);
            if (c0 > p0) {
              const double2 old = orow[col];
              w.x += old.x;
              w.y += old.y;
            }
            orow[col] = w;
          }
        }
      }
    }
  }
}
