// Tree build, scalar P2M and M2M kernels.
// Fragment of blfmm.cu (one translation unit): included inside
// namespace blfmm_gpu after the plan definition; not a standalone header.


// ================================================================ kernels
template <int D>
__global__ void k_bin(const double* __restrict__ xin, long long n, int L,
                      double lo0, double lo1, double lo2, double s0, double s1,
                      double s2, uint32_t* __restrict__ keys,
                      int* __restrict__ idx) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double lo[3] = {lo0, lo1, lo2}, side[3] = {s0, s1, s2};
  int c[3] = {0, 0, 0};
  const int nmax = (1 << L) - 1;
  for (int k = 0; k < D; ++k) {
    // leaf_of: static_cast<int>((x - lo) / side), clamped (geometry.cpp:254-262)
    int v = static_cast<int>((xin[i * D + k] - lo[k]) / side[k]);
    c[k] = min(max(v, 0), nmax);
  }
  keys[i] = morton_encode<D>(c, L);
  idx[i] = static_cast<int>(i);
}

template <int D>
__global__ void k_gather_coords(const double* __restrict__ xin,
                                const int* __restrict__ perm, long long n,
                                double* __restrict__ x0, double* __restrict__ x1,
                                double* __restrict__ x2) {
  long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (s >= n) return;
  long long i = perm[s];
  x0[s] = xin[i * D];
  if (D > 1) x1[s] = xin[i * D + 1];
  if (D > 2) x2[s] = xin[i * D + 2];
}

__global__ void k_shift_keys(const uint32_t* __restrict__ in, long long n,
                             int d, uint32_t* __restrict__ out) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) out[i] = in[i] >> d;
}

__global__ void k_fill_parent(const int* __restrict__ child_start,
                              long long nparent, int* __restrict__ parent) {
  long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (p >= nparent) return;
  for (int c = child_start[p]; c < child_start[p + 1]; ++c) parent[c] = static_cast<int>(p);
}

template <int D>
__global__ void k_slotmap(const uint32_t* __restrict__ key, long long nbox,
                          int level, int* __restrict__ slotmap) {
  long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (s >= nbox) return;
  int c[3];
  morton_decode<D>(key[s], level, c);
  slotmap[rowmajor_id<D>(c, level)] = static_cast<int>(s);
}

// near_pairs of every nonempty leaf (s_a * sum_{b in N(a)} s_b) and its
// count of nonempty neighbor leaves (for the single-level far_work count).
template <int D>
__global__ void k_pair_counts(const uint32_t* __restrict__ key,
                              const int* __restrict__ slotmap,
                              const int* __restrict__ leaf_start,
                              long long nleaf, int L,
                              unsigned long long* __restrict__ acc,
                              long long* __restrict__ leaf_src) {
  long long a = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (a >= nleaf) return;
  int c[3], b[3];
  morton_decode<D>(key[a], L, c);
  const int n = 1 << L;
  long long src = 0, nn = 0;
  int tot = D == 1 ? 3 : (D == 2 ? 9 : 27);
  for (int q = 0; q < tot; ++q) {
    int r = q;
    bool ok = true;
    for (int k = D - 1; k >= 0; --k) {
      b[k] = c[k] + (r % 3) - 1;
      r /= 3;
      ok = ok && b[k] >= 0 && b[k] < n;
    }
    if (!ok) continue;
    int s = slotmap[rowmajor_id<D>(b, L)];
    if (s < 0) continue;
    src += leaf_start[s + 1] - leaf_start[s];
    ++nn;
  }
  long long sa = leaf_start[a + 1] - leaf_start[a];
  leaf_src[a] = src;
  atomicAdd(&acc[0], static_cast<unsigned long long>(sa * src));
  atomicAdd(&acc[1], static_cast<unsigned long long>(nn));
}

// Number of nonempty (target, source) interaction-list pairs at one level.
template <int D>
__global__ void k_il_pairs(const uint32_t* __restrict__ key,
                           const int* __restrict__ slotmap, long long nbox,
                           int level, unsigned long long* __restrict__ acc) {
  long long a = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (a >= nbox) return;
  int c[3], b[3], base[3];
  morton_decode<D>(key[a], level, c);
  const int n = 1 << level;
  for (int k = 0; k < D; ++k) base[k] = (c[k] & 1) ? -3 : -2;
  long long cnt = 0;
  int tot = D == 1 ? 6 : (D == 2 ? 36 : 216);
  for (int q = 0; q < tot; ++q) {
    int r = q;
    bool ok = true, own = true;
    for (int k = D - 1; k >= 0; --k) {
      int o = base[k] + r % 6;
      r /= 6;
      b[k] = c[k] + o;
      ok = ok && b[k] >= 0 && b[k] < n;
      own = own && o >= -1 && o <= 1;
    }
    if (!ok || own) continue;
    if (slotmap[rowmajor_id<D>(b, level)] >= 0) ++cnt;
  }
  atomicAdd(acc, static_cast<unsigned long long>(cnt));
}

__global__ void k_gather_lambda(const double* __restrict__ lam_in,
                                const int* __restrict__ perm, long long n,
                                int R, double* __restrict__ lam, double* __restrict__ lamT) {
  long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (s >= n) return;
  long long i = perm[s];
  for (int r = 0; r < R; ++r) {
    const double v = lam_in[r * n + i];
    lam[r * n + s] = v;
    if (lamT) lamT[s * R + r] = v;  // point-major copy for the batched near field
  }
}

__global__ void k_combine(const double* __restrict__ far_,
                          const double* __restrict__ near_,
                          const int* __restrict__ perm, long long n, long long s0,
                          long long s1, int R, double* __restrict__ out,
                          const double* __restrict__ planes = nullptr,
                          const unsigned* __restrict__ pmask = nullptr) {
  long long s = s0 + blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (s >= s1) return;
  long long i = perm ? perm[s] : s;  // no perm: the sorted slice (gathered later)
  if (planes) {  // nrhs 1: symmetric-item planes summed in neighbour order (fixed)
    double v = near_[s];
    for (unsigned m = pmask[s]; m; m &= m - 1) v += planes[((long long)__ffs(m) - 1) * n + s];
    out[i] = far_[s] + v;
    return;
  }
  for (int r = 0; r < R; ++r) out[r * n + i] = far_[r * n + s] + near_[r * n + s];
}

// gathered sorted u -> caller order (distributed execute)
__global__ void k_scatter_sorted(const double* __restrict__ us, const int* __restrict__ perm,
                                 long long n, int R, double* __restrict__ out) {
  const long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (s >= n) return;
  const long long i = perm[s];
  for (int r = 0; r < R; ++r) out[r * n + i] = us[r * n + s];
}

// locals of the leaves whose interaction lists are empty at every level
// (plan_build: zero_far): the reference's exact zero
__global__ void k_zero_boxes(double2* __restrict__ loc, const int* __restrict__ slots, long long K,
                             long long nbox) {
  double2* o = loc + ((long long)blockIdx.y * nbox + slots[blockIdx.x]) * K;
  for (long long t = threadIdx.x; t < K; t += blockDim.x) o[t] = make_double2(0.0, 0.0);
}

// ---------------------------------------------------------------- P2M
// V_b[m] = sum_{j in b} lambda_j e^{i xi_m . (x_b - x_j)}  (mlfmm.cpp:218-231)
// One CTA per (leaf, node tile, rhs); per-axis phase tables of a batch of
// points in shared memory; the tensor-product phase is assembled per node.
constexpr int kP2MThreads = 256;
constexpr int kP2MNodesPerThread = 4;

template <int D>
__global__ void __launch_bounds__(kP2MThreads)
    k_p2m(const int* __restrict__ leaf_list, const uint32_t* __restrict__ leaf_key,
          const int* __restrict__ leaf_start,
          const double* __restrict__ x0, const double* __restrict__ x1,
          const double* __restrict__ x2, const double* __restrict__ lam,
          const double* __restrict__ xi, int M, long long K, int L, long long n,
          long long nleaf, double lo0, double lo1, double lo2, double s0,
          double s1, double s2, int batch, double2* __restrict__ mult) {
  extern __shared__ double2 smem[];
  const long long a = leaf_list ? leaf_list[blockIdx.x] : blockIdx.x;
  const int r = blockIdx.z;
  double2* ph = smem;                                     // [batch][D][M]
  double* lb = reinterpret_cast<double*>(ph + (size_t)batch * D * M);  // [batch]
  int c[3];
  morton_decode<D>(leaf_key[a], L, c);
  const double lo[3] = {lo0, lo1, lo2}, side[3] = {s0, s1, s2};
  double xb[3];
  for (int k = 0; k < D; ++k) xb[k] = lo[k] + (c[k] + 0.5) * side[k];
  const int p0 = leaf_start[a], p1 = leaf_start[a + 1];
  const double* xs[3] = {x0, x1, x2};

  long long e0 = (long long)blockIdx.y * kP2MThreads * kP2MNodesPerThread + threadIdx.x;
  double2 acc[kP2MNodesPerThread];
  int mk[kP2MNodesPerThread][3];
#pragma unroll
  for (int q = 0; q < kP2MNodesPerThread; ++q) {
    acc[q] = make_double2(0.0, 0.0);
    long long e = e0 + q * kP2MThreads;
    long long t = e < K ? e : 0;
    for (int k = D - 1; k >= 0; --k) {
      mk[q][k] = static_cast<int>(t % M);
      t /= M;
    }
  }
  if (D == 1) {
    // d = 1: node = m, every point-node phase is used by exactly one thread, so
    // it is formed in registers (no staged rows: any M fits, e.g. the 16,384
    // nodes of test_solver.cpp:244-285); same operations as the staged form
    double xq[kP2MNodesPerThread];
#pragma unroll
    for (int q = 0; q < kP2MNodesPerThread; ++q) xq[q] = xi[mk[q][0]];
    for (int j = p0; j < p1; ++j) {
      const double rk = xb[0] - x0[j];
      const double w = lam[(long long)r * n + j];
#pragma unroll
      for (int q = 0; q < kP2MNodesPerThread; ++q) {
        const double2 p = polar1(xq[q] * rk);
        acc[q].x = fma(w, p.x, acc[q].x);
        acc[q].y = fma(w, p.y, acc[q].y);
      }
    }
  } else
  for (int pb = p0; pb < p1; pb += batch) {
    int nb = min(batch, p1 - pb);
    __syncthreads();
    for (int t = threadIdx.x; t < nb * D * M; t += blockDim.x) {
      int j = t / (D * M), k = (t / M) % D, m = t % M;
      double rk = xb[k] - xs[k][pb + j];
      ph[t] = polar1(xi[m] * rk);
    }
    for (int t = threadIdx.x; t < nb; t += blockDim.x) lb[t] = lam[(long long)r * n + pb + t];
    __syncthreads();
    for (int j = 0; j < nb; ++j) {
      const double2* pj = ph + (size_t)j * D * M;
      const double w = lb[j];
#pragma unroll
      for (int q = 0; q < kP2MNodesPerThread; ++q) {
        double2 p = pj[mk[q][0]];
        if (D > 1) p = cmul(p, pj[M + mk[q][1]]);
        if (D > 2) p = cmul(p, pj[2 * M + mk[q][2]]);
        acc[q].x = fma(w, p.x, acc[q].x);
        acc[q].y = fma(w, p.y, acc[q].y);
      }
    }
  }
  double2* out = mult + ((long long)r * nleaf + a) * K;
#pragma unroll
  for (int q = 0; q < kP2MNodesPerThread; ++q) {
    long long e = e0 + q * kP2MThreads;
    if (e < K) out[e] = acc[q];
  }
}

// cp.async (LDGSTS) 16-byte copies global -> shared
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait_group() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::);
}

// Per-axis grid indices of stored node e: row-major decode of the full grid,
// or the plan's node table (packed m0 | m1 << 8 | m2 << 16) when the plan
// stores the Hermitian half spectrum.
template <int D>
__device__ __forceinline__ void node_axes(long long e, int M, const int* __restrict__ node_m,
                                          int mk[3]) {
  if (node_m) {
    const int v = __ldg(node_m + e);
    mk[0] = v & 255;
    mk[1] = (v >> 8) & 255;
    mk[2] = (v >> 16) & 255;
    return;
  }
  long long t = e;
  for (int k = D - 1; k >= 0; --k) {
    mk[k] = static_cast<int>(t % M);
    t /= M;
  }
}

// ---------------------------------------------------------------- M2M
// V_p[m] = sum_c e^{i xi_m . (x_p - x_c)} V_c[m]  (mlfmm.cpp:233-264, shared)
// tab[k][delta][m] = e^{i xi_m (1/2 - delta) h_{l,k}} for the child level l.
template <int D>
__global__ void k_m2m(const uint32_t* __restrict__ child_key,
                      const int* __restrict__ child_start,
                      const double2* __restrict__ child_mult,
                      long long nchild, long long nparent,
                      const double2* __restrict__ tab, int M, long long K,
                      const int* __restrict__ node_m, double2* __restrict__ parent_mult) {
  const long long p = blockIdx.x;
  const int r = blockIdx.z;
  long long e = (long long)blockIdx.y * blockDim.x + threadIdx.x;
  if (e >= K) return;
  int mk[3];
  node_axes<D>(e, M, node_m, mk);
  double2 acc = make_double2(0.0, 0.0);
  const double2* vc = child_mult + (long long)r * nchild * K;
  for (int c = child_start[p]; c < child_start[p + 1]; ++c) {
    uint32_t oct = child_key[c];
    double2 ph = make_double2(1.0, 0.0);
#pragma unroll
    for (int k = 0; k < D; ++k) {
      int delta = (oct >> (D - 1 - k)) & 1;
      double2 q = __ldg(&tab[(k * 2 + delta) * M + mk[k]]);
      ph = k == 0 ? q : cmul(ph, q);
    }
    cmac(acc, ph, vc[(long long)c * K + e]);
  }
  parent_mult[((long long)r * nparent + p) * K + e] = acc;
}

// Telescoped far field (shared grids): G_1 = C NS_1 and NS_1 covers every
// level-1 box, so G_L(a) = e^{i xi (x_a - x_0)} C V_0 with V_0 the root
// multipole. root[r][e] = C_e sum_{b at level 1} e^{i xi (x_0 - x_b)} V_1(b)
// (children in slot order, k_m2m's phase product), one thread per node.
template <int D>
__global__ void k_root(const uint32_t* __restrict__ key1, long long nbox1,
                       const double2* __restrict__ mult1, const double2* __restrict__ tab,
                       const double* __restrict__ ctab, int M, long long K,
                       const int* __restrict__ node_m, double2* __restrict__ root) {
  const int r = blockIdx.z;
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= K) return;
  int mk[3];
  node_axes<D>(e, M, node_m, mk);
  double2 acc = make_double2(0.0, 0.0);
  const double2* vc = mult1 + (long long)r * nbox1 * K;
  for (long long c = 0; c < nbox1; ++c) {
    const uint32_t oct = key1[c];
    double2 ph = make_double2(1.0, 0.0);
#pragma unroll
    for (int k = 0; k < D; ++k) {
      const int delta = (oct >> (D - 1 - k)) & 1;
      const double2 q = __ldg(&tab[(k * 2 + delta) * M + mk[k]]);
      ph = k == 0 ? q : cmul(ph, q);
    }
    cmac(acc, ph, vc[c * K + e]);
  }
  const double cm = ctab[e];
  root[(long long)r * K + e] = make_double2(cm * acc.x, cm * acc.y);
}

// M2M for the multi-GPU exchange mode: parents from a slot list (or a
// contiguous range), children restricted to slots [cmin, cmax), child and
// parent arrays possibly stored with an offset (partial "own" buffers):
// child c lives at (r*nchild_store + c - child_off)*K, parent p at
// (r*nparent_store + p - parent_off)*K.
template <int D>
__global__ void k_m2m_x(const uint32_t* __restrict__ child_key,
                        const int* __restrict__ child_start,
                        const double2* __restrict__ child_mult, long long child_off,
                        long long nchild_store, const int* __restrict__ plist,
                        long long pfirst, long long parent_off, long long nparent_store,
                        int cmin, int cmax, const double2* __restrict__ tab, int M, long long K,
                        const int* __restrict__ node_m, double2* __restrict__ parent_mult) {
  const long long p = plist ? plist[blockIdx.x] : pfirst + blockIdx.x;
  const int r = blockIdx.z;
  const long long e = (long long)blockIdx.y * blockDim.x + threadIdx.x;
  if (e >= K) return;
  int mk[3];
  node_axes<D>(e, M, node_m, mk);
  double2 acc = make_double2(0.0, 0.0);
  const double2* vc = child_mult + (long long)r * nchild_store * K;
  for (int c = max(child_start[p], cmin); c < min(child_start[p + 1], cmax); ++c) {
    const uint32_t oct = child_key[c];
    double2 ph = make_double2(1.0, 0.0);
#pragma unroll
    for (int k = 0; k < D; ++k) {
      const int delta = (oct >> (D - 1 - k)) & 1;
      const double2 q = __ldg(&tab[(k * 2 + delta) * M + mk[k]]);
      ph = k == 0 ? q : cmul(ph, q);
    }
    cmac(acc, ph, vc[(long long)(c - child_off) * K + e]);
  }
  parent_mult[((long long)r * nparent_store + (p - parent_off)) * K + e] = acc;
}
