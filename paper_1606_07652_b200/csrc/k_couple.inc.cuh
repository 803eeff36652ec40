// M2L (+ L2L) kernels: level sweep, per-parent and z-streamed column couple.
// Fragment of blfmm.cu (one translation unit): included inside
// namespace blfmm_gpu after the plan definition; not a standalone header.

// ---------------------------------------------------------- M2L (+ L2L)
// couple (mlfmm.cpp:268-299) and the L2L half of downsweep (307-340) for the
// 2^d children of one parent p at level l-1, all in shared grids.
//
// IL_l(a) = children(N_{l-1}(p)) \ N_l(a) (geometry.cpp:294-313), and with a
// shared grid the M2M is an exact phase shift (mlfmm.cpp:253-255), so
//   sum_{b in IL(a)} e^{i xi (x_a - x_b)} V_b
//     = e^{i xi (x_a - x_p)} NS_{l-1}(p) - NS_l(a),
//   NS_l(a) = sum_{b in N_l(a)} e^{i xi (x_a - x_b)} V_b   (3^d neighborhood)
// and the accumulated local of the downsweep obeys
//   L_l(a) = G_l(a) - C NS_l(a),  G_l(a) = e^{i xi (x_a - x_p)} G_{l-1}(p),
//   G_1 = C NS_1 (no locals exist at level 1; IL lists start at level 2).
// couple()'s own output is C (e^{i xi (x_a - x_p)} NS_{l-1}(p) - NS_l(a)).
// NS is evaluated separably on the 4^d block of level-l boxes around p's
// children (3 taps per axis), so a sibling group costs ~21 complex MACs per
// child and node instead of |IL| = 189.
//
// One CTA per (parent, node chunk, rhs); one thread per node.
// ns_tab[k*7 + o+1][m] = e^{-i xi_m o h_{l,k}}  (o = -1, 0, 1; a view into m2l_tab)
// sh_tab[k][delta][m] = e^{i xi_m (1/2 - delta) h_{l,k}} (conj = child shift)
constexpr int kCoupleThreads = 128;

template <int D>
__global__ void __launch_bounds__(kCoupleThreads, 4)
    k_couple(const int* __restrict__ region, long long pfirst, long long nparent,
             long long nb_all, int level,
             const int* __restrict__ slotmap, const double2* __restrict__ mult,
             long long nbox, const double2* __restrict__ ns_tab,
             const double2* __restrict__ sh_tab, const double* __restrict__ ctab, int M,
             long long K, const double2* __restrict__ g_parent,
             double2* __restrict__ g_out, double2* __restrict__ loc_out,
             const double2* __restrict__ ns_parent, double2* __restrict__ ns_out,
             double2* __restrict__ couple_out, int skip_empty, const int* __restrict__ node_m) {
  constexpr int E0 = 4, E1 = D >= 2 ? 4 : 1, E2 = D == 3 ? 4 : 1;
  constexpr int C0 = 2, C1 = D >= 2 ? 2 : 1, C2 = D == 3 ? 2 : 1;
  constexpr int O0 = 1, O1 = D >= 2 ? 1 : 0, O2 = D == 3 ? 1 : 0;
  constexpr int REG = E0 * E1 * E2;
  static_assert(REG <= 64 && kCoupleThreads >= 64, "region mask layout");
  __shared__ int slot[REG];
  __shared__ int voff[REG];
  __shared__ unsigned occw[2];
  __shared__ double2 phs[2][3][kCoupleThreads];  // x / y axis phases of each thread's node
  const long long p = pfirst + blockIdx.x;
  const int r = blockIdx.z;
  // plan-time region table of this parent (k_region_slots): one load per entry
  if (threadIdx.x < 64) {
    const int t = threadIdx.x;
    const int sl = t < REG ? region[p * REG + t] : -1;
    if (t < REG) {
      slot[t] = sl;
      // element offset of the box's expansion (R*nbox*K + K < 2^31 is checked
      // at plan time); empty / out-of-domain boxes read the zero expansion
      // stored after the last box unless they are skipped
      voff[t] = sl >= 0 ? static_cast<int>((long long)r * nbox * K + (long long)sl * K)
                        : static_cast<int>(nb_all * K);
    }
    // occupancy mask of the region: empty boxes issue no loads (36 % of the
    // 4^3 region of a P3 leaf parent is empty)
    const unsigned b = __ballot_sync(0xffffffffu, sl >= 0 || !skip_empty);
    if ((t & 31) == 0) occw[t >> 5] = b;
  }
  const long long e = (long long)blockIdx.y * blockDim.x + threadIdx.x;
  const long long ec = e < K ? e : K - 1;
  int mk[3] = {0, 0, 0};
  node_axes<D>(ec, M, node_m, mk);
  // phases: the last axis (innermost pass, most uses) in registers, the
  // others in shared memory (per thread) to keep register pressure down
  double2 ph[3][3];
  for (int k = 0; k < 3; ++k)
    for (int o = 0; o < 3; ++o) {
      double2 z = k < D ? __ldg(&ns_tab[(k * 7 + o) * M + mk[k]]) : make_double2(1.0, 0.0);
      if (k == 2) ph[2][o] = z;
      else phs[k][o][threadIdx.x] = z;
    }
  __syncthreads();
  if (e >= K) return;
#define PHX(o) phs[0][(o)][threadIdx.x]
#define PHY(o) phs[1][(o)][threadIdx.x]
  const double2* v = mult + e;
  const unsigned long long occ = ((unsigned long long)occw[1] << 32) | occw[0];
  auto ldv = [&](int t) {
    return (occ >> t) & 1ull ? __ldg(v + voff[t]) : make_double2(0.0, 0.0);
  };

  double2 ns[C0][C1][C2];
#pragma unroll
  for (int a = 0; a < C0; ++a)
#pragma unroll
    for (int b = 0; b < C1; ++b)
#pragma unroll
      for (int c = 0; c < C2; ++c) ns[a][b][c] = make_double2(0.0, 0.0);
  // The o = 0 tap of every axis is e^0 = 1 exactly: an add, not a MAC.
  auto tap = [](double2& acc, const double2& ph, const double2& v, int o) {
    if (o == 0) {
      acc.x += v.x;
      acc.y += v.y;
    } else {
      cmac(acc, ph, v);
    }
  };
  // region rows (x, y) stream in z-columns of E2 values, the next column's
  // loads issued before the current one is consumed (low register pressure)
  auto col = [&](int x, int y, int z) { return (x * E1 + y) * E2 + z; };
  double2 cur[E2];
#pragma unroll
  for (int z = 0; z < E2; ++z) cur[z] = ldv(col(0, 0, z));
#pragma unroll
  for (int x = 0; x < E0; ++x) {
    double2 y_acc[C1][C2];
#pragma unroll
    for (int b = 0; b < C1; ++b)
#pragma unroll
      for (int c = 0; c < C2; ++c) y_acc[b][c] = make_double2(0.0, 0.0);
#pragma unroll
    for (int y = 0; y < E1; ++y) {
      double2 vrow[E2];
#pragma unroll
      for (int z = 0; z < E2; ++z) vrow[z] = cur[z];
      {
        const int ny = (y + 1 < E1) ? y + 1 : 0, nx = (y + 1 < E1) ? x : x + 1;
        if (nx < E0) {
#pragma unroll
          for (int z = 0; z < E2; ++z) cur[z] = ldv(col(nx, ny, z));
        }
      }
      double2 zr[C2];
      if (D == 3) {
        // 3-tap filter v0 + q v(+1) + conj(q) v(-1), q = ph[2][2] (o = +1),
        // as v0 + q.x (a + b) + i q.y (a - b) with a = v(+1), b = v(-1)
        const double qx = ph[2][2].x, qy = ph[2][2].y;
#pragma unroll
        for (int c = 0; c < C2; ++c) {
          const double2 vm = vrow[c], v0 = vrow[c + 1], vp = vrow[c + 2];
          const double sx = vp.x + vm.x, sy = vp.y + vm.y;
          const double dx = vp.x - vm.x, dy = vp.y - vm.y;
          zr[c].x = fma(-qy, dy, fma(qx, sx, v0.x));
          zr[c].y = fma(qy, dx, fma(qx, sy, v0.y));
        }
      } else {
#pragma unroll
        for (int c = 0; c < C2; ++c) zr[c] = vrow[c];
      }
#pragma unroll
      for (int b = 0; b < C1; ++b) {
        const int o = y - (b + O1);
        if (o >= -1 && o <= 1) {
#pragma unroll
          for (int c = 0; c < C2; ++c) {
            if (D >= 2) tap(y_acc[b][c], o == 0 ? zr[c] : PHY(o + 1), zr[c], o);
            else y_acc[b][c] = zr[c];
          }
        }
      }
    }
#pragma unroll
    for (int a = 0; a < C0; ++a) {
      const int o = x - (a + O0);
      if (o >= -1 && o <= 1) {
#pragma unroll
        for (int b = 0; b < C1; ++b)
#pragma unroll
          for (int c = 0; c < C2; ++c) tap(ns[a][b][c], o == 0 ? y_acc[b][c] : PHX(o + 1), y_acc[b][c], o);
      }
    }
  }
  const double cm = ctab[e];
  double2 gp = make_double2(0.0, 0.0), nsp = make_double2(0.0, 0.0);
  if (g_parent) gp = g_parent[((long long)r * nparent + p) * K + e];
  if (ns_parent) nsp = ns_parent[((long long)r * nparent + p) * K + e];
#pragma unroll
  for (int a = 0; a < C0; ++a)
#pragma unroll
    for (int b = 0; b < C1; ++b)
#pragma unroll
      for (int c = 0; c < C2; ++c) {
        int s = slot[((a + O0) * E1 + (b + O1)) * E2 + (c + O2)];
        if (s < 0) continue;
        const int dl[3] = {a, b, c};
        double2 sh = make_double2(1.0, 0.0);
#pragma unroll
        for (int k = 0; k < D; ++k) {
          double2 q = __ldg(&sh_tab[(k * 2 + dl[k]) * M + mk[k]]);
          q.y = -q.y;  // e^{i xi (x_a - x_p)}
          sh = k == 0 ? q : cmul(sh, q);
        }
        const double2 cn = make_double2(cm * ns[a][b][c].x, cm * ns[a][b][c].y);
        double2 g;
        if (g_parent) {
          g = cmul(sh, gp);
        } else {
          g = cn;  // level 1: G_1 = C NS_1
        }
        const int idx = static_cast<int>((long long)r * nbox * K) + s * static_cast<int>(K) +
                        static_cast<int>(e);
        if (g_out) g_out[idx] = g;
        if (loc_out) loc_out[idx] = make_double2(g.x - cn.x, g.y - cn.y);
        if (ns_out) ns_out[idx] = ns[a][b][c];
        if (couple_out) {
          double2 t = cmul(sh, nsp);
          couple_out[idx] = make_double2(cm * (t.x - ns[a][b][c].x), cm * (t.y - ns[a][b][c].y));
        }
      }
#undef PHX
#undef PHY
}

// 3-D couple + L2L with NPT nodes per thread (nodes e, e + 128, ...): the
// region offsets, occupancy tests and address arithmetic of every load are
// shared by the thread's nodes and their FP64 chains interleave. Same math as
// k_couple<3>; the per-axis tap phase q_k = e^{-i xi h_k} (o = +1) stays in
// registers and the o = -1 tap uses conj(q_k).
template <int NPT, bool SKIP, int PF = 1, bool ROOT = false>
__device__ __forceinline__ void couple3_body(long long p, long long e0, int estride, const int* __restrict__ voff,
                                             const int* __restrict__ slot, unsigned long long occ,
                                             int r, long long nparent,
                                             const double2* __restrict__ mult, long long nbox,
                                             const double2* __restrict__ ns_tab,
                                             const double2* __restrict__ sh_tab,
                                             const double* __restrict__ ctab, int M, long long K,
                                             const double2* __restrict__ g_parent,
                                             double2* __restrict__ g_out,
                                             double2* __restrict__ loc_out,
                                             const double2* __restrict__ ns_parent,
                                             double2* __restrict__ ns_out,
                                             double2* __restrict__ couple_out,
                                             const int* __restrict__ node_m,
                                             const double2* __restrict__ root = nullptr,
                                             const double2* __restrict__ root_tab = nullptr,
                                             const int* __restrict__ pc = nullptr) {
  int mk[NPT][3];
  bool nv[NPT];
  double2 qx[NPT], qy[NPT], qz[NPT];
#pragma unroll
  for (int j = 0; j < NPT; ++j) {
    const long long e = e0 + (long long)j * estride;
    nv[j] = e < K;
    node_axes<3>(nv[j] ? e : K - 1, M, node_m, mk[j]);
    qx[j] = __ldg(&ns_tab[(0 * 7 + 2) * M + mk[j][0]]);
    qy[j] = __ldg(&ns_tab[(1 * 7 + 2) * M + mk[j][1]]);
    qz[j] = __ldg(&ns_tab[(2 * 7 + 2) * M + mk[j][2]]);
  }
  // thread's nodes past K read node e0 (valid) and are not stored
  const double2* v = mult + e0;
  auto ldcol = [&](int x, int y, double2 (&c)[NPT][4]) {
    const int4 o4 = *reinterpret_cast<const int4*>(&voff[(x * 4 + y) * 4]);
    const int oo[4] = {o4.x, o4.y, o4.z, o4.w};
#pragma unroll
    for (int z = 0; z < 4; ++z) {
      const bool on = !SKIP || ((occ >> ((x * 4 + y) * 4 + z)) & 1ull);
#pragma unroll
      for (int j = 0; j < NPT; ++j) {
        const long long dj = nv[j] ? (long long)j * estride : 0;
        c[j][z] = on ? __ldg(v + oo[z] + dj) : make_double2(0.0, 0.0);
      }
    }
  };
  double2 ns[NPT][2][2][2];
#pragma unroll
  for (int j = 0; j < NPT; ++j)
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b)
#pragma unroll
        for (int c = 0; c < 2; ++c) ns[j][a][b][c] = make_double2(0.0, 0.0);
  // tap helpers: o = 0 add; o = +1: acc += q v; o = -1: acc += conj(q) v
  auto tap = [](double2& acc, const double2& q, const double2& w, int o) {
    if (o == 0) {
      acc.x += w.x;
      acc.y += w.y;
    } else if (o > 0) {
      acc.x = fma(q.x, w.x, fma(-q.y, w.y, acc.x));
      acc.y = fma(q.x, w.y, fma(q.y, w.x, acc.y));
    } else {
      acc.x = fma(q.x, w.x, fma(q.y, w.y, acc.x));
      acc.y = fma(q.x, w.y, fma(-q.y, w.x, acc.y));
    }
  };
  // PF columns of loads in flight (register ring, column index x*4+y)
  double2 cur[PF][NPT][4];
#pragma unroll
  for (int f = 0; f < PF; ++f) ldcol(f / 4, f % 4, cur[f]);
#pragma unroll
  for (int x = 0; x < 4; ++x) {
    double2 yacc[NPT][2][2];
#pragma unroll
    for (int j = 0; j < NPT; ++j)
#pragma unroll
      for (int b = 0; b < 2; ++b)
#pragma unroll
        for (int c = 0; c < 2; ++c) yacc[j][b][c] = make_double2(0.0, 0.0);
#pragma unroll
    for (int y = 0; y < 4; ++y) {
      const int cidx = x * 4 + y;
      double2 col[NPT][4];
#pragma unroll
      for (int j = 0; j < NPT; ++j)
#pragma unroll
        for (int z = 0; z < 4; ++z) col[j][z] = cur[cidx % PF][j][z];
      {
        const int nxt = cidx + PF;
        if (nxt < 16) ldcol(nxt / 4, nxt % 4, cur[cidx % PF]);
      }
#pragma unroll
      for (int j = 0; j < NPT; ++j) {
        // z filter, conjugate-pair form: v0 + q.x (vp + vm) + i q.y (vp - vm)
        double2 zr[2];
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const double2 vm = col[j][c], v0 = col[j][c + 1], vp = col[j][c + 2];
          const double sx = vp.x + vm.x, sy = vp.y + vm.y;
          const double dx = vp.x - vm.x, dy = vp.y - vm.y;
          zr[c].x = fma(-qz[j].y, dy, fma(qz[j].x, sx, v0.x));
          zr[c].y = fma(qz[j].y, dx, fma(qz[j].x, sy, v0.y));
        }
#pragma unroll
        for (int b = 0; b < 2; ++b) {
          const int o = y - (b + 1);
          if (o >= -1 && o <= 1) {
#pragma unroll
            for (int c = 0; c < 2; ++c) tap(yacc[j][b][c], qy[j], zr[c], o);
          }
        }
      }
    }
#pragma unroll
    for (int j = 0; j < NPT; ++j)
#pragma unroll
      for (int a = 0; a < 2; ++a) {
        const int o = x - (a + 1);
        if (o >= -1 && o <= 1) {
#pragma unroll
          for (int b = 0; b < 2; ++b)
#pragma unroll
            for (int c = 0; c < 2; ++c) tap(ns[j][a][b][c], qx[j], yacc[j][b][c], o);
        }
      }
  }
#pragma unroll
  for (int j = 0; j < NPT; ++j) {
    if (!nv[j]) continue;
    const long long e = e0 + (long long)j * estride;
    const double cm = ctab[e];
    double2 gp = make_double2(0.0, 0.0), nsp = make_double2(0.0, 0.0);
    double2 sx[2], sy[2], sz[2];
    if (ROOT) {
      // telescoped: G_L(a) = e^{i xi (x_a - x_0)} Ct V_0, root[e] = Ct V_0,
      // root_tab[k][i][m] = e^{i xi_m (x_{a,k} - x_{0,k})} for leaf index i
      gp = root[(long long)r * K + e];
      const int nper = 2 * pc[3];
#pragma unroll
      for (int dl = 0; dl < 2; ++dl) {
        sx[dl] = __ldg(&root_tab[(0 * nper + 2 * pc[0] + dl) * M + mk[j][0]]);
        sy[dl] = __ldg(&root_tab[(1 * nper + 2 * pc[1] + dl) * M + mk[j][1]]);
        sz[dl] = __ldg(&root_tab[(2 * nper + 2 * pc[2] + dl) * M + mk[j][2]]);
      }
    } else {
      if (g_parent) gp = g_parent[((long long)r * nparent + p) * K + e];
      if (ns_parent) nsp = ns_parent[((long long)r * nparent + p) * K + e];
      // child shifts e^{i xi (x_a - x_p)} = prod_k conj(sh_tab[k][delta_k])
#pragma unroll
      for (int dl = 0; dl < 2; ++dl) {
        sx[dl] = __ldg(&sh_tab[(0 * 2 + dl) * M + mk[j][0]]);
        sy[dl] = __ldg(&sh_tab[(1 * 2 + dl) * M + mk[j][1]]);
        sz[dl] = __ldg(&sh_tab[(2 * 2 + dl) * M + mk[j][2]]);
        sx[dl].y = -sx[dl].y;
        sy[dl].y = -sy[dl].y;
        sz[dl].y = -sz[dl].y;
      }
    }
    double2 gz[2];
#pragma unroll
    for (int c = 0; c < 2; ++c) gz[c] = cmul(sz[c], gp);
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        const double2 sxy = cmul(sx[a], sy[b]);
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const int s = slot[((a + 1) * 4 + (b + 1)) * 4 + (c + 1)];
          if (s < 0) continue;
          const double2 nsv = ns[j][a][b][c];
          const double2 cn = make_double2(cm * nsv.x, cm * nsv.y);
          const double2 g = (ROOT || g_parent) ? cmul(sxy, gz[c]) : cn;  // level 1: G_1 = C NS_1
          const int idx = static_cast<int>((long long)r * nbox * K) + s * static_cast<int>(K) +
                          static_cast<int>(e);
          if (g_out) g_out[idx] = g;
          if (loc_out) loc_out[idx] = make_double2(g.x - cn.x, g.y - cn.y);
          if (ns_out) ns_out[idx] = nsv;
          if (couple_out) {
            const double2 t = cmul(cmul(sxy, sz[c]), nsp);
            couple_out[idx] = make_double2(cm * (t.x - nsv.x), cm * (t.y - nsv.y));
          }
        }
      }
  }
}


constexpr int kCouple3Threads = 128;
template <int NPT, bool SKIP, int MINB = 3, int PF = 1, bool ROOT = false>
__global__ void __launch_bounds__(kCouple3Threads, MINB)
    k_couple3(const int* __restrict__ region, long long pfirst, long long nparent,
              long long nb_all, const double2* __restrict__ mult, long long nbox,
              const double2* __restrict__ ns_tab, const double2* __restrict__ sh_tab,
              const double* __restrict__ ctab, int M, long long K,
              const double2* __restrict__ g_parent, double2* __restrict__ g_out,
              double2* __restrict__ loc_out, const double2* __restrict__ ns_parent,
              double2* __restrict__ ns_out, double2* __restrict__ couple_out,
              const int* __restrict__ node_m, const double2* __restrict__ root = nullptr,
              const double2* __restrict__ root_tab = nullptr,
              const uint32_t* __restrict__ pkey = nullptr, int plevel = 0) {
  __shared__ __align__(16) int voff[64];
  __shared__ int slot[64];
  __shared__ unsigned occw[2];
  __shared__ int pc[4];  // ROOT: the parent's box coordinates and 2^plevel
  const long long p = pfirst + blockIdx.x;
  const int r = blockIdx.z;
  if (ROOT && threadIdx.x == 64) {
    int c[3];
    morton_decode<3>(pkey[p], plevel, c);
    pc[0] = c[0];
    pc[1] = c[1];
    pc[2] = c[2];
    pc[3] = 1 << plevel;
  }
  if (threadIdx.x < 64) {
    const int t = threadIdx.x;
    const int sl = region[p * 64 + t];
    slot[t] = sl;
    voff[t] = sl >= 0 ? static_cast<int>((long long)r * nbox * K + (long long)sl * K)
                      : static_cast<int>(nb_all * K);
    const unsigned b = __ballot_sync(0xffffffffu, sl >= 0 || !SKIP);
    if ((t & 31) == 0) occw[t >> 5] = b;
  }
  __syncthreads();
  const unsigned long long occ = ((unsigned long long)occw[1] << 32) | occw[0];
  const long long e0 = (long long)blockIdx.y * kCouple3Threads * NPT + threadIdx.x;
  if (e0 >= K) return;
  couple3_body<NPT, SKIP, PF, ROOT>(p, e0, kCouple3Threads, voff, slot, occ, r, nparent, mult, nbox,
                                    ns_tab, sh_tab, ctab, M, K, g_parent, g_out, loc_out,
                                    ns_parent, ns_out, couple_out, node_m, root, root_tab, pc);
}

// Telescoped leaf couple, z-streamed column tiles (3-D shared grids).
// L_L(a) = e^{i xi (x_a - x_0)} C V_0 - C NS_L(a), NS_L(a) = sum over the 3^3
// leaf neighbourhood of a of e^{i xi (x_a - x_b)} V_b. NS is
// separable: per axis a 3-tap filter v0 + q v(+1) + conj(q) v(-1) with
// q = e^{-i xi h}. One CTA takes one segment = a 2 x TY block of leaf columns
// (x, y) and up to ZS consecutive output slabs z, for 128 stored nodes of one
// right-hand side (thread = node). The thread streams the 4 x (TY+2) input
// boxes of slabs z0-1 .. z0+nz through registers once: y filter, x filter
// (the slab's 2 x TY partial sums P(z)), then the z filter over the ring
// P(z-1), P(z), P(z+1) gives NS of output slab z. Each leaf multipole is read
// by ~4 (TY = 2) threads of its node instead of the 8 parent regions of
// k_couple3 (that kernel re-read every multipole 8 times through L2). At CTA
// start the segment's slots become element offsets in shared memory (empty /
// outside boxes -> the zero expansion after the level's last box; outputs ->
// -1 unless the leaf is owned), so the slab loop is one LDS.128 per window
// row and unpredicated loads; the ring is unrolled by 3 (register renaming).
// GO: grid order, 0 = segments along x (all segments of a node chunk, then
// the next chunk), 1 = node chunks along x (the chunks of one segment run
// together).
// seg_hdr[s] = {x0, y0, z0, nz}; seg_slot[s][ZS+2][4][TY+2] = input slot of
// box (x0-1+i, y0-1+j, z0-1+slab), -1 empty / outside.
template <int TY, int ZS, int MINB, int GO>
__global__ void __launch_bounds__(128, MINB)
    k_couple_col(const int4* __restrict__ seg_hdr, const int* __restrict__ seg_slot,
                 const double2* __restrict__ mult, long long nbox, int R,
                 const double2* __restrict__ ns_tab, const double* __restrict__ ctab, int M,
                 long long K, const int* __restrict__ node_m, const double2* __restrict__ root,
                 const double2* __restrict__ root_tab, int nper, int own_lo, int own_hi,
                 double2* __restrict__ loc_out) {
  constexpr int WY = TY + 2, NI = 4 * WY;
  __shared__ __align__(16) int off[ZS + 2][4][4];  // input element offsets, row i, col j < WY
  __shared__ __align__(16) int oof[ZS + 2][4];     // output offsets (-1: skip)
  const long long sg = GO ? blockIdx.y : blockIdx.x;
  const long long chunk = GO ? blockIdx.x : blockIdx.y;
  const int r = blockIdx.z;
  const int4 h = __ldg(&seg_hdr[sg]);
  const int nsl = h.w + 2;
  {
    const int zoff = static_cast<int>((long long)(R - r) * nbox * K);  // zero expansion
    const int ki = static_cast<int>(K);
    for (int t = threadIdx.x; t < nsl * NI; t += 128) {
      const int sl = t / NI, i = (t % NI) / WY, j = t % WY;
      const int bx = __ldg(&seg_slot[(sg * (ZS + 2) + sl) * NI + i * WY + j]);
      off[sl][i][j] = bx >= 0 ? bx * ki : zoff;
      if (i >= 1 && i <= 2 && j >= 1 && j <= TY)
        oof[sl][(i - 1) * TY + j - 1] = (bx >= own_lo && bx < own_hi) ? bx * ki : -1;
    }
  }
  __syncthreads();
  const long long e0 = chunk * 128 + threadIdx.x;
  const bool valid = e0 < K;
  const long long e = valid ? e0 : K - 1;
  int mk[3];
  node_axes<3>(e, M, node_m, mk);
  const double2 qx = __ldg(&ns_tab[(0 * 7 + 2) * M + mk[0]]);
  const double2 qy = __ldg(&ns_tab[(1 * 7 + 2) * M + mk[1]]);
  const double2 qz = __ldg(&ns_tab[(2 * 7 + 2) * M + mk[2]]);
  const double cm = __ldg(&ctab[e]);
  const double2* __restrict__ v = mult + (long long)r * nbox * K + e;
  double2* __restrict__ lo = loc_out + (long long)r * nbox * K + e;
  // opaque bases: every load / store address is then one IMAD.WIDE.U32 of
  // the 32-bit offset instead of a re-derived 64-bit index
  asm("" : "+l"(v));
  asm("" : "+l"(lo));
  const double2* __restrict__ rtz = root_tab + (long long)2 * nper * M + mk[2];
  // filt(q, vm, v0, vp) = v0 + q vp + conj(q) vm = v0 + q.x (vp + vm) + i q.y (vp - vm)
  auto filt = [](double2 q, double2 vm, double2 v0, double2 vp) {
    const double px = vp.x + vm.x, py = vp.y + vm.y;
    const double dx = vp.x - vm.x, dy = vp.y - vm.y;
    return make_double2(fma(-q.y, dy, fma(q.x, px, v0.x)), fma(q.y, dx, fma(q.x, py, v0.y)));
  };
  typedef double2 PT[2][TY];
  PT ra, rb, rc;
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < TY; ++j) ra[i][j] = rb[i][j] = rc[i][j] = make_double2(0.0, 0.0);
  // one slab: P(z) -> pn; for s >= 2 the outputs of slab z-1 from pm, p0, pn
  auto step = [&](int s, const PT& pm, const PT& p0, PT& pn) {
    double2 in[4][WY];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int4 o = *reinterpret_cast<const int4*>(&off[s][i][0]);
      const int oa[4] = {o.x, o.y, o.z, o.w};
#pragma unroll
      for (int j = 0; j < WY; ++j) in[i][j] = __ldg(v + static_cast<unsigned>(oa[j]));
    }
    double2 yv[4][TY];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < TY; ++j) yv[i][j] = filt(qy, in[i][j], in[i][j + 1], in[i][j + 2]);
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < TY; ++j) pn[i][j] = filt(qx, yv[i][j], yv[i + 1][j], yv[i + 2][j]);
    if (s >= 2) {
      // output slab z = z0 + s - 2 (the centre of input slab s - 1):
      // g = e^{i xi (x_a - x_0)} C V_0 as (sx sy)(sz CV_0), L = g - C NS
      const int4 oo = *reinterpret_cast<const int4*>(&oof[s - 1][0]);
      const int oa[4] = {oo.x, oo.y, oo.z, oo.w};
      const bool any = TY == 2 ? (oo.x & oo.y & oo.z & oo.w) != -1 : (oo.x & oo.y) != -1;
      if (valid && any) {
        const int zo = h.z + s - 2;
        const double2 gz = cmul(__ldg(rtz + (long long)zo * M), __ldg(&root[(long long)r * K + e]));
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int j = 0; j < TY; ++j) {
            const int o = oa[i * TY + j];
            if (o < 0) continue;
            const double2 sx = __ldg(&root_tab[((long long)h.x + i) * M + mk[0]]);
            const double2 sy = __ldg(&root_tab[((long long)nper + h.y + j) * M + mk[1]]);
            const double2 ns = filt(qz, pm[i][j], p0[i][j], pn[i][j]);
            const double2 g = cmul(cmul(sx, sy), gz);
            lo[static_cast<unsigned>(o)] = make_double2(g.x - cm * ns.x, g.y - cm * ns.y);
          }
      }
    }
  };
  for (int s = 0; s < nsl; s += 3) {
    step(s, rb, rc, ra);
    if (s + 1 < nsl) step(s + 1, rc, ra, rb);
    if (s + 2 < nsl) step(s + 2, ra, rb, rc);
  }
}
