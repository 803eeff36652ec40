// Batched right-hand sides: real-weight DMMA GEMM P2M / L2P.
// Fragment of blfmm.cu (one translation unit): included inside
// namespace blfmm_gpu after the plan definition; not a standalone header.

// -------------------- batched right-hand sides: real weights, DMMA GEMMs
// With R weight vectors the expansions are linear in real lambda, so P2M and
// L2P become dense real x complex contractions over the stored nodes of the
// half spectrum (3-D, M = 16), two real DMMA GEMMs instead of the four of a
// complex product, and each point-node phase is formed once for 32
// right-hand sides:
//   P2M  V_r[e] = sum_j lambda_rj conj(P_j[e])                (mlfmm.cpp:218-231)
//   L2P  u_r,i  = w Re sum_e P_i[e] L_r[e]                    (mlfmm.cpp:342-357)
// P_j[e] = P1_j[m1] P2_j[m2] P3_j[m3] (node table), the per-axis phases of the
// CTA's points generated in shared memory (gen_row16). Tiles: m = 8 right-hand
// sides, n = 8 nodes (P2M) or 8 points (L2P), k = 4 points (P2M) or 4 nodes (L2P).
constexpr int kMRSpan = 64;                 // points per CTA pass
constexpr int kMRRow = 52;                  // L2P phase row stride (48 used; == 4 mod 8:
                                            // points along g, nodes along tq)
constexpr int kMRRowP = 50;                 // P2M phase row stride (== 2 mod 8: points along
                                            // tq, nodes along g; 52 gave 2-way conflicts on
                                            // every row read)
constexpr int kMRNC = 32, kMRLS = 36;       // L2P node chunk, staged row stride (== 4 mod 8)
constexpr int kMRLam = 36;                  // P2M staged weight row stride (== 4 mod 16: the
                                            // half-warp LDS.64 of (point tq, rhs g) is conflict-free)

template <int RS>
__device__ __forceinline__ void mr_gen_rows(double2 (*rows)[RS], int t0, int np,
                                            const double* __restrict__ x0,
                                            const double* __restrict__ x1,
                                            const double* __restrict__ x2, const double c[3],
                                            double dxi) {
  for (int t = threadIdx.x; t < 3 * np; t += blockDim.x) {
    const int j = t / 3, k = t % 3;
    const double xv = __ldg((k == 0 ? x0 : (k == 1 ? x1 : x2)) + t0 + j);
    gen_row16(xv - (k == 0 ? c[0] : (k == 1 ? c[1] : c[2])), dxi, &rows[j][16 * k]);
  }
}

// P2M: CTA = (leaf, 32 right-hand sides); the leaf's points in spans of 64
// (phase rows + staged weights), then node chunks of 64 (4 warps x 2 node
// tiles, 4 right-hand-side tiles each, real and imaginary part). Spans after
// the first add to the stored partial sums (same CTA, fixed order).
template <int SPAN, int NW>
__global__ void __launch_bounds__(32 * NW, 384 / (32 * NW))
    k_p2m_mr(const int* __restrict__ leaf_list, const uint32_t* __restrict__ leaf_key,
             const int* __restrict__ leaf_start, const double* __restrict__ x0,
             const double* __restrict__ x1, const double* __restrict__ x2, LeafGeom geo,
             double dxi, const int* __restrict__ node_m, const double* __restrict__ lam, int R,
             long long n, long long nleaf, double2* __restrict__ mult) {
  extern __shared__ __align__(16) double2 mr_dyn[];
  double2 (*rows)[kMRRowP] = reinterpret_cast<double2 (*)[kMRRowP]>(mr_dyn);
  double (*slam)[kMRLam] = reinterpret_cast<double (*)[kMRLam]>(mr_dyn + SPAN * kMRRowP);
  const long long a = leaf_list ? leaf_list[blockIdx.x] : blockIdx.x;
  const int r0 = blockIdx.y * 32, rc = min(32, R - r0);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, tq = lane & 3;
  double c[3];
  geo.centre(leaf_key[a], c);
  const int p0 = leaf_start[a], p1 = leaf_start[a + 1];
  double2* vout = mult + ((long long)r0 * nleaf + a) * kH16Ks;
  const long long rstride = nleaf * kH16Ks;  // next right-hand side
  for (int t0 = p0; t0 < p1 || (t0 == p0 && p0 == p1); t0 += SPAN) {
    const int np = min(SPAN, p1 - t0);
    __syncthreads();  // the previous span's rows / weights are no longer read
    mr_gen_rows(rows, t0, np, x0, x1, x2, c, dxi);
    for (int t = threadIdx.x; t < SPAN * 32; t += 32 * NW) {
      const int r = t / SPAN, j = t % SPAN;  // coalesced along points
      slam[j][r] = (j < np && r < rc) ? __ldg(lam + (long long)(r0 + r) * n + t0 + j) : 0.0;
    }
    __syncthreads();
    for (int nc = 0; nc < kH16Ks; nc += 16 * NW) {
      double vr[4][2][2], vi[4][2][2];  // [rhs tile][node tile][element]
#pragma unroll
      for (int rt = 0; rt < 4; ++rt)
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
          for (int v = 0; v < 2; ++v) vr[rt][nt][v] = vi[rt][nt][v] = 0.0;
      int mk[2][3];
      bool tl[2];  // node tile inside the stored nodes (the last chunk is half full)
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {  // B column of this lane: node e = nc + 16 w + 8 nt + g
        tl[nt] = nc + 16 * warp + 8 * nt < kH16Ks;
        const int e = tl[nt] ? nc + 16 * warp + 8 * nt + g : 0;
        const int v = __ldg(node_m + e);
        mk[nt][0] = v & 255;
        mk[nt][1] = (v >> 8) & 255;
        mk[nt][2] = (v >> 16) & 255;
      }
      // the operands of k step k0 + 4 (weights, the two node phases: a chain
      // of two complex products) are formed while the DMMAs of k step k0
      // issue; formed inside the step they left the warp waiting on the DMUL /
      // DFMA chain in front of every DMMA group (44 % of the stall samples)
      double al[4], bq[2][2];
      auto operands = [&](int k0) {
        const int j = k0 + tq;  // this lane's point (A column, B row)
#pragma unroll
        for (int rt = 0; rt < 4; ++rt) al[rt] = slam[j][8 * rt + g];  // 0 past np
        const double2* rw = rows[j < np ? j : 0];
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
          const double2 q = cmul(cmul(rw[mk[nt][0]], rw[16 + mk[nt][1]]), rw[32 + mk[nt][2]]);
          bq[nt][0] = q.x;
          bq[nt][1] = -q.y;  // conj
        }
      };
      operands(0);
      for (int k0 = 0; k0 < np; k0 += 4) {
        double ac[4], bc[2][2];
#pragma unroll
        for (int rt = 0; rt < 4; ++rt) ac[rt] = al[rt];
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
          bc[nt][0] = bq[nt][0];
          bc[nt][1] = bq[nt][1];
        }
        if (k0 + 4 < np) operands(k0 + 4);
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
          if (!tl[nt]) continue;
#pragma unroll
          for (int rt = 0; rt < 4; ++rt) {
            dmma(vr[rt][nt][0], vr[rt][nt][1], ac[rt], bc[nt][0]);
            dmma(vi[rt][nt][0], vi[rt][nt][1], ac[rt], bc[nt][1]);
          }
        }
      }
      // C[rhs 8 rt + g][node 8 nt + 2 tq + v]
#pragma unroll
      for (int rt = 0; rt < 4; ++rt) {
        const int r = 8 * rt + g;
        if (r >= rc) continue;
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
          if (!tl[nt]) continue;
          const int e = nc + 16 * warp + 8 * nt + 2 * tq;
          double2* o = vout + r * rstride + e;
          double4 val = make_double4(vr[rt][nt][0], vi[rt][nt][0], vr[rt][nt][1], vi[rt][nt][1]);
          if (e >= kH16K) val = make_double4(0.0, 0.0, 0.0, 0.0);  // padding nodes stay 0
          if (t0 != p0) {
            const double4 prev = *reinterpret_cast<const double4*>(o);
            val.x += prev.x;
            val.y += prev.y;
            val.z += prev.z;
            val.w += prev.w;
          }
          *reinterpret_cast<double4*>(o) = val;
        }
      }
    }
    if (p0 == p1) break;
  }
}

// L2P: CTA = (leaf, span of <= 64 points, 32 right-hand sides); the span's
// phase rows generated once; the locals of the 32 right-hand sides stream
// through shared memory in node chunks of 32 (cp.async, double-buffered).
// Warp w owns point tiles 2w, 2w + 1; C = [8 right-hand sides][8 points].
// IM: the imaginary residual GEMM with the locals scaled by D (block A).
template <bool IM>
__global__ void __launch_bounds__(128, 2)
    k_l2p_mr(const int2* __restrict__ work, const uint32_t* __restrict__ leaf_key,
             const int* __restrict__ leaf_start, const double* __restrict__ x0,
             const double* __restrict__ x1, const double* __restrict__ x2, LeafGeom geo,
             double dxi, const int* __restrict__ node_m, const double* __restrict__ dtab,
             const double2* __restrict__ loc, int R, long long n, long long nleaf, double weight,
             double* __restrict__ far_, unsigned long long* __restrict__ imag_bits) {
  extern __shared__ __align__(16) double2 mr_dyn[];
  double2 (*rows)[kMRRow] = reinterpret_cast<double2 (*)[kMRRow]>(mr_dyn);
  double2 (*lch)[32][kMRLS] = reinterpret_cast<double2 (*)[32][kMRLS]>(mr_dyn + kMRSpan * kMRRow);
  const int2 item = work[blockIdx.x];
  const long long a = item.x;
  const int t0 = item.y;
  const int r0 = blockIdx.y * 32, rc = min(32, R - r0);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, tq = lane & 3;
  const int pend = min(leaf_start[a + 1], t0 + kMRSpan), np = pend - t0;
  double c[3];
  geo.centre(leaf_key[a], c);
  const double2* lsrc = loc + ((long long)r0 * nleaf + a) * kH16Ks;
  const long long rstride = nleaf * kH16Ks;
  auto stage = [&](int buf, int c0) {
    for (int t = threadIdx.x; t < rc * kMRNC; t += 128) {
      const int r = t / kMRNC, e = t % kMRNC;
      cp_async16(&lch[buf][r][e], lsrc + r * rstride + c0 + e);
    }
    cp_async_commit();
  };
  stage(0, 0);
  mr_gen_rows(rows, t0, np, x0, x1, x2, c, dxi);
  double ur[4][2][2], ui[4][2][2];  // [rhs tile][point tile][element]
#pragma unroll
  for (int rt = 0; rt < 4; ++rt)
#pragma unroll
    for (int pt = 0; pt < 2; ++pt)
#pragma unroll
      for (int v = 0; v < 2; ++v) ur[rt][pt][v] = ui[rt][pt][v] = 0.0;
  int pl[2];  // this lane's B column (point) per point tile
#pragma unroll
  for (int pt = 0; pt < 2; ++pt) pl[pt] = min(16 * warp + 8 * pt + g, max(np - 1, 0));
  int buf = 0;
  for (int c0 = 0; c0 < kH16Ks; c0 += kMRNC, buf ^= 1) {
    if (c0 + kMRNC < kH16Ks) {
      stage(buf ^ 1, c0 + kMRNC);
      cp_async_wait_group<1>();
    } else {
      cp_async_wait_group<0>();
    }
    __syncthreads();
#pragma unroll 2
    for (int ks = 0; ks < kMRNC; ks += 4) {
      const int e = c0 + ks + tq;  // this lane's node (A column, B row)
      const int v = __ldg(node_m + e);
      const int m1 = v & 255, m2 = (v >> 8) & 255, m3 = (v >> 16) & 255;
      double2 la[4];
#pragma unroll
      for (int rt = 0; rt < 4; ++rt) {
        const int r = 8 * rt + g;
        la[rt] = r < rc ? lch[buf][r][ks + tq] : make_double2(0.0, 0.0);
      }
      const double dv = IM ? __ldg(dtab + e) : 0.0;
#pragma unroll
      for (int pt = 0; pt < 2; ++pt) {
        const double2* rw = rows[pl[pt]];
        const double2 q = cmul(cmul(rw[m1], rw[16 + m2]), rw[32 + m3]);
#pragma unroll
        for (int rt = 0; rt < 4; ++rt) {
          dmma(ur[rt][pt][0], ur[rt][pt][1], la[rt].x, q.x);
          dmma(ur[rt][pt][0], ur[rt][pt][1], -la[rt].y, q.y);
          if (IM) {
            dmma(ui[rt][pt][0], ui[rt][pt][1], dv * la[rt].x, q.y);
            dmma(ui[rt][pt][0], ui[rt][pt][1], dv * la[rt].y, q.x);
          }
        }
      }
    }
    __syncthreads();  // buffer `buf` is refilled by the next iteration's stage
  }
  // C[rhs 8 rt + g][point 8 pt + 2 tq + v] of warp w's 16 points
  double imax = 0.0;
#pragma unroll
  for (int rt = 0; rt < 4; ++rt) {
    const int r = 8 * rt + g;
    if (r >= rc) continue;
#pragma unroll
    for (int pt = 0; pt < 2; ++pt)
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const int i = 16 * warp + 8 * pt + 2 * tq + v;
        if (i >= np) continue;
        far_[(long long)(r0 + r) * n + t0 + i] = weight * ur[rt][pt][v];
        if (IM) imax = fmax(imax, fabs(weight * ui[rt][pt][v]));
      }
  }
  if (IM && imax > 0.0)
    atomicMax(imag_bits, static_cast<unsigned long long>(__double_as_longlong(imax)));
}
