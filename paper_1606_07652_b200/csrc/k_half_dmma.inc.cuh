// Half-spectrum DMMA P2M (fused leaf M2M) and L2P, one right-hand side per CTA.
// Fragment of blfmm.cu (one translation unit): included inside
// namespace blfmm_gpu after the plan definition; not a standalone header.

// P2M: one CTA (4 warps) per leaf. Warp w: A row tiles 8w..8w+7 (m1 in
// [4w, 4w+4)), the B row tile w (rb = 8w + g) and the C tile (m1 tile w/2,
// m2 tile w%2). A fragment rows are conj(P1 P2) (conj(P1 P3[0]) for C), the B
// fragment columns carry lambda (lambda conj P3 / lambda conj P2).
__global__ void __launch_bounds__(128)
    k_p2m_h16w4(const int* __restrict__ leaf_list, const int* __restrict__ leaf_start,
              const double2* __restrict__ pht, const double* __restrict__ lam, long long n,
              long long nleaf, double2* __restrict__ mult) {
  // point rows padded by 32 B: the 4 points of a k step (tq) then start 8
  // banks apart, so the quarter-warp LDS.128 operand loads are conflict-free
  constexpr int MM = 16, PER = 3 * MM, PERP = PER + 2, CHUNK = 32;
  __shared__ __align__(16) double2 sph[CHUNK][PERP];
  __shared__ double slam[CHUNK];
  const long long a = leaf_list ? leaf_list[blockIdx.x] : blockIdx.x;
  const int r = blockIdx.z;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, tq = lane & 3;
  const int rbg = 8 * warp + g;
  const bool bvalid = rbg < kH16BR;
  int bm1, bm2;
  h16_brow(bvalid ? rbg : 0, bm1, bm2);
  const int cm1 = 8 * (warp >> 1) + g, cm2 = 8 * (warp & 1) + g;
  CTile accA[8], accB, accC;
#pragma unroll
  for (int q = 0; q < 8; ++q) accA[q] = CTile{{0.0, 0.0}, {0.0, 0.0}};
  accB = CTile{{0.0, 0.0}, {0.0, 0.0}};
  accC = CTile{{0.0, 0.0}, {0.0, 0.0}};
  const int p0 = leaf_start[a], p1 = leaf_start[a + 1];
  const double* lr = lam + (long long)r * n;
  for (int c0 = p0; c0 < p1; c0 += CHUNK) {
    const int nb = min(CHUNK, p1 - c0);
    __syncthreads();
    const double2* src = pht + (long long)c0 * PER;
    for (int t = threadIdx.x; t < nb * PER; t += blockDim.x)
      cp_async16(&sph[t / PER][t % PER], src + t);
    for (int t = threadIdx.x; t < CHUNK; t += blockDim.x) slam[t] = t < nb ? lr[c0 + t] : 0.0;
    cp_async_wait_all();
    __syncthreads();
    for (int j0 = 0; j0 < nb; j0 += 4) {
      const int j = j0 + tq;
      const double2* pj = sph[j < nb ? j : 0];
      const double w = slam[j];  // 0 for padding
      // B fragments (k = point, n = g)
      const double2 zA = pj[2 * MM + 8 + g], zB = pj[2 * MM + g], zC = pj[MM + cm2];
      const double bAr = w * zA.x, bAi = -w * zA.y;
      const double bBr = w * zB.x, bBi = -w * zB.y;
      const double bCr = w * zC.x, bCi = -w * zC.y;
      const double2 p2lo = pj[MM + g], p2hi = pj[MM + 8 + g];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const double2 z = cmul(pj[4 * warp + (q >> 1)], (q & 1) ? p2hi : p2lo);
        cdmma(accA[q], z.x, -z.y, z.y, bAr, bAi);
      }
      {
        double2 z = cmul(pj[bm1], pj[MM + bm2]);
        if (!bvalid) z = make_double2(0.0, 0.0);
        cdmma(accB, z.x, -z.y, z.y, bBr, bBi);
      }
      {
        const double2 z = cmul(pj[cm1], pj[2 * MM]);
        cdmma(accC, z.x, -z.y, z.y, bCr, bCi);
      }
    }
  }
  double2* out = mult + ((long long)r * nleaf + a) * kH16Ks;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int row = 8 * (8 * warp + q) + g;
    *reinterpret_cast<double4*>(out + row * 8 + 2 * tq) =
        make_double4(accA[q].re[0], accA[q].im[0], accA[q].re[1], accA[q].im[1]);
  }
  if (bvalid) {
#pragma unroll
    for (int v = 0; v < 2; ++v) {
      const int m3 = 2 * tq + v;
      if (m3 >= 1) out[kH16A + kH16C + rbg * 7 + m3 - 1] = make_double2(accB.re[v], accB.im[v]);
    }
  }
  *reinterpret_cast<double4*>(out + kH16A + cm1 * MM + 8 * (warp & 1) + 2 * tq) =
      make_double4(accC.re[0], accC.im[0], accC.re[1], accC.im[1]);
  if (threadIdx.x < kH16Ks - kH16K) out[kH16K + threadIdx.x] = make_double2(0.0, 0.0);
}

// P2M fused with the leaf-level M2M (half spectrum): one CTA per parent at
// level L-1 computes every child leaf's multipoles exactly as k_p2m_h16w4
// (16-point staging chunks), writes them, and adds each child's fragments,
// shifted by e^{i xi (x_p - x_c)}, into the parent's expansion held in shared
// memory (each fragment element is owned by one lane, children in slot order:
// the same operations and order as k_m2m). The leaf-level M2M's re-read of
// V_L from HBM disappears.
// Points are staged in chunks of 16 (cp.async); double-buffering the chunks
// measured slower.
__global__ void __launch_bounds__(128, 4)
    k_p2m_m2m_h16(const int* __restrict__ plist, const int* __restrict__ child_start,
                  const uint32_t* __restrict__ leaf_key, const int* __restrict__ leaf_start,
                  const double2* __restrict__ pht, const double* __restrict__ lam, long long n,
                  long long nleaf, long long nparent, const double2* __restrict__ tab,
                  double2* __restrict__ mult, double2* __restrict__ pmult) {
  constexpr int MM = 16, PER = 3 * MM, PERP = PER + 2;  // padded rows (k_p2m_h16w4)
  constexpr int CHUNK = 16;
  __shared__ __align__(16) double2 sph[CHUNK][PERP];
  __shared__ double slam[CHUNK];
  extern __shared__ __align__(16) double2 pacc[];  // [kH16Ks]
  const long long p = plist[blockIdx.x];
  const int r = blockIdx.z;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, tq = lane & 3;
  const int rbg = 8 * warp + g;
  const bool bvalid = rbg < kH16BR;
  int bm1, bm2;
  h16_brow(bvalid ? rbg : 0, bm1, bm2);
  const int cm1 = 8 * (warp >> 1) + g, cm2 = 8 * (warp & 1) + g;
  for (int t = threadIdx.x; t < kH16Ks; t += blockDim.x) pacc[t] = make_double2(0.0, 0.0);
  const double* lr = lam + (long long)r * n;
  // phase of stored node (m1, m2, m3) for child octant bits (d0, d1, d2)
  auto shift = [&](int m1, int m2, int m3, int d0, int d1, int d2) {
    double2 ph = __ldg(&tab[(0 * 2 + d0) * MM + m1]);
    ph = cmul(ph, __ldg(&tab[(1 * 2 + d1) * MM + m2]));
    return cmul(ph, __ldg(&tab[(2 * 2 + d2) * MM + m3]));
  };
  const int cfirst = child_start[p], clast = child_start[p + 1];
  // stage chunk [s0, s0 + CHUNK) of child cc
  auto stage = [&](int cc, int s0) {
    const int nb = min(CHUNK, leaf_start[cc + 1] - s0);
    const double2* src = pht + (long long)s0 * PER;
    for (int t = threadIdx.x; t < nb * PER; t += blockDim.x)
      cp_async16(&sph[t / PER][t % PER], src + t);
    for (int t = threadIdx.x; t < CHUNK; t += blockDim.x) slam[t] = t < nb ? lr[s0 + t] : 0.0;
  };
  for (int c = cfirst; c < clast; ++c) {
    CTile accA[8], accB, accC;
#pragma unroll
    for (int q = 0; q < 8; ++q) accA[q] = CTile{{0.0, 0.0}, {0.0, 0.0}};
    accB = CTile{{0.0, 0.0}, {0.0, 0.0}};
    accC = CTile{{0.0, 0.0}, {0.0, 0.0}};
    const int p0 = leaf_start[c], p1 = leaf_start[c + 1];
    for (int c0 = p0; c0 < p1; c0 += CHUNK) {
      const int nb = min(CHUNK, p1 - c0);
      __syncthreads();  // every thread is done with the stage about to be refilled
      stage(c, c0);
      cp_async_wait_all();
      __syncthreads();
      for (int j0 = 0; j0 < nb; j0 += 4) {
        const int j = j0 + tq;
        const double2* pj = sph[j < nb ? j : 0];
        const double w = slam[j];  // 0 for padding
        const double2 zA = pj[2 * MM + 8 + g], zB = pj[2 * MM + g], zC = pj[MM + cm2];
        const double bAr = w * zA.x, bAi = -w * zA.y;
        const double bBr = w * zB.x, bBi = -w * zB.y;
        const double bCr = w * zC.x, bCi = -w * zC.y;
        const double2 p2lo = pj[MM + g], p2hi = pj[MM + 8 + g];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const double2 z = cmul(pj[4 * warp + (q >> 1)], (q & 1) ? p2hi : p2lo);
          cdmma(accA[q], z.x, -z.y, z.y, bAr, bAi);
        }
        {
          double2 z = cmul(pj[bm1], pj[MM + bm2]);
          if (!bvalid) z = make_double2(0.0, 0.0);
          cdmma(accB, z.x, -z.y, z.y, bBr, bBi);
        }
        {
          const double2 z = cmul(pj[cm1], pj[2 * MM]);
          cdmma(accC, z.x, -z.y, z.y, bCr, bCi);
        }
      }
    }
    // child multipoles out; shifted fragments into the parent
    const uint32_t oct = leaf_key[c];
    const int d0 = (oct >> 2) & 1, d1 = (oct >> 1) & 1, d2 = oct & 1;
    double2* out = mult + ((long long)r * nleaf + c) * kH16Ks;
    // this lane's A elements span m1 = 4w + k (k < 4), m2 = 8h + g (h < 2),
    // m3 = 8 + 2tq + v (v < 2): 8 axis phases instead of 3 per element
    double2 px[4], py[2], pz[2];
#pragma unroll
    for (int k = 0; k < 4; ++k) px[k] = __ldg(&tab[(0 * 2 + d0) * MM + 4 * warp + k]);
#pragma unroll
    for (int h = 0; h < 2; ++h) py[h] = __ldg(&tab[(1 * 2 + d1) * MM + 8 * h + g]);
#pragma unroll
    for (int v = 0; v < 2; ++v) pz[v] = __ldg(&tab[(2 * 2 + d2) * MM + 8 + 2 * tq + v]);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int row = 8 * (8 * warp + q) + g;
      *reinterpret_cast<double4*>(out + row * 8 + 2 * tq) =
          make_double4(accA[q].re[0], accA[q].im[0], accA[q].re[1], accA[q].im[1]);
      const double2 pxy = cmul(px[q >> 1], py[q & 1]);  // (x y) z: k_m2m's order
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const int e = row * 8 + 2 * tq + v;
        double2 acc = pacc[e];
        cmac(acc, cmul(pxy, pz[v]), make_double2(accA[q].re[v], accA[q].im[v]));
        pacc[e] = acc;
      }
    }
    if (bvalid) {
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const int m3 = 2 * tq + v;
        if (m3 < 1) continue;
        const int e = kH16A + kH16C + rbg * 7 + m3 - 1;
        out[e] = make_double2(accB.re[v], accB.im[v]);
        double2 acc = pacc[e];
        cmac(acc, shift(bm1, bm2, m3, d0, d1, d2), make_double2(accB.re[v], accB.im[v]));
        pacc[e] = acc;
      }
    }
    {
      const int m2b = 8 * (warp & 1) + 2 * tq;
      *reinterpret_cast<double4*>(out + kH16A + cm1 * MM + m2b) =
          make_double4(accC.re[0], accC.im[0], accC.re[1], accC.im[1]);
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const int e = kH16A + cm1 * MM + m2b + v;
        double2 acc = pacc[e];
        cmac(acc, shift(cm1, m2b + v, 0, d0, d1, d2), make_double2(accC.re[v], accC.im[v]));
        pacc[e] = acc;
      }
    }
    if (threadIdx.x < kH16Ks - kH16K) out[kH16K + threadIdx.x] = make_double2(0.0, 0.0);
  }
  __syncthreads();
  double2* po = pmult + ((long long)r * nparent + p) * kH16Ks;
  for (int t = threadIdx.x; t < kH16Ks; t += blockDim.x) po[t] = pacc[t];
}

constexpr int kL2PSpan = 128;
// L2P, half spectrum, per (leaf, span of up to 128 points), with the leaf's
// local expansion staged once per span in shared memory (40 KB, cp.async)
// and read with conflict-free LDS for every 8-point tile. Warp w: A row
// tiles 8w..8w+7 (2 k steps over m3 in [8, 16)), the B row tile w (2 k steps
// over m3 in [0, 8), m3 = 0 reads zero), and half of the k steps (m2) of the
// C tile with m1 tile w/2; W on DMMA in the 3-multiplication complex form; the
// per-point sums finish with shuffles and shared memory.
template <int MINB, bool IM = true>
__global__ void __launch_bounds__(128, MINB)
    k_l2p_h16S(const int2* __restrict__ work, const int* __restrict__ leaf_start,
               const double2* __restrict__ pht, const double2* __restrict__ loc,
               const double* __restrict__ dtab, long long n, long long nleaf, double weight,
               double* __restrict__ far_, unsigned long long* __restrict__ imag_bits) {
  constexpr int MM = 16, PER = 3 * MM, AW = 2;
  __shared__ double2 red[4][8];
  __shared__ double redi[4][8];
  const int2 item = work[blockIdx.x];
  const long long a = item.x;
  const int r = blockIdx.z;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, tq = lane & 3;
  const int pend = min(leaf_start[a + 1], item.y + kL2PSpan);
  const double2 zero = make_double2(0.0, 0.0);
  // the 8-point tiles' phase rows (48 complex per point), double-buffered in
  // shared memory by cp.async one tile ahead; rows padded to 52 (64 B bank
  // shift) so the fragment loads of points g, g+1 do not collide
  constexpr int PERP = PER + 4;
  extern __shared__ __align__(16) double2 l2p_dyn[];  // [kH16Ks] expansion + [2][8][PERP] phases
  double2 (*sph)[8][PERP] = reinterpret_cast<double2 (*)[8][PERP]>(l2p_dyn + kH16Ks);
  auto stage = [&](int buf, int pb) {
    const int cnt = min(8, pend - pb);
    const double2* src = pht + (long long)pb * PER;
    for (int t = threadIdx.x; t < cnt * PER; t += blockDim.x)
      cp_async16(&sph[buf][t / PER][t % PER], src + t);
  };
  stage(0, item.y);
  // the span's leaf expansion, staged once in shared memory (cp.async); block
  // A rows (8 nodes, 128 B) are XOR-swizzled (column ^ 4 on odd rows) so the
  // quarter-warp fragment loads (rows g, g+1 x columns tq) hit 32 distinct banks
  double2* const sl = l2p_dyn;
  {
    const double2* src = loc + ((long long)r * nleaf + a) * kH16Ks;
    for (int t = threadIdx.x; t < kH16Ks; t += blockDim.x)
      cp_async16(&sl[t < kH16A ? (t ^ (((t >> 3) & 1) << 2)) : t], src + t);
    cp_async_wait_all();
    __syncthreads();
  }
  const double2* la = sl;
  const double* dw = dtab + 8 * (8 * (8 * warp) + g) + tq;  // D (L1-resident table)
  const double2* laA = la + 8 * (8 * (8 * warp) + g) + tq;   // swizzled block-A rows
  const int ksw = (g & 1) << 2;                                 // column ^ 4 on odd rows
  double2 lB[2], lC[2];
  {
    const int rbn = 8 * warp + g, m1n = 8 * (warp >> 1) + g;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int m3 = 4 * k + tq;
      lB[k] = (m3 >= 1 && rbn < kH16BR) ? la[kH16A + kH16C + rbn * 7 + m3 - 1] : zero;
      lC[k] = la[kH16A + m1n * MM + 4 * (2 * (warp & 1) + k) + tq];
    }
  }
  int buf = 0;
  for (int pb = item.y; pb < pend; pb += 8, buf ^= 1) {
    if (pb + 8 < pend) {
      stage(buf ^ 1, pb + 8);  // buffer buf^1 was released by the previous tile's last barrier
      cp_async_commit();
      cp_async_wait_group<1>();
    } else {
      cp_async_wait_group<0>();
    }
    __syncthreads();
    const int ia = pb + g;
    const bool iv = ia < pend;
    const double2* pa = sph[buf][iv ? g : 0];
    double2 zA[2], zB[2], zC[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      zA[k] = iv ? pa[2 * MM + 8 + 4 * k + tq] : zero;
      zB[k] = iv ? pa[2 * MM + 4 * k + tq] : zero;
      zC[k] = iv ? pa[MM + 4 * (2 * (warp & 1) + k) + tq] : zero;
    }
    double2 p2[2][2];
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int v = 0; v < 2; ++v) p2[h][v] = iv ? pa[MM + h * 8 + 2 * tq + v] : zero;
    double2 part = zero;
    double pim = 0.0;
#pragma unroll
    for (int q0 = 0; q0 < 8; q0 += AW) {
      CTile3 acc[AW], acd[AW];
#pragma unroll
      for (int u = 0; u < AW; ++u) {
        acc[u] = kZeroTile3;
        acd[u] = kZeroTile3;
      }
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const double as = zA[k].x + zA[k].y;
#pragma unroll
        for (int u = 0; u < AW; ++u) {
          const double2 lv = laA[64 * (q0 + u) + (k == 0 ? ksw : 4 - ksw)];
          cdmma3(acc[u], as, zA[k].x, zA[k].y, lv.x, lv.y - lv.x, lv.x + lv.y);
          if (IM) {  // imaginary residual (stats requested): the D-weighted GEMM
            const double dv = __ldg(dw + 64 * (q0 + u) + 4 * k);
            const double dx = dv * lv.x, dy = dv * lv.y;
            cdmma3(acd[u], as, zA[k].x, zA[k].y, dx, dy - dx, dx + dy);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < AW; ++u) {
        const int t = 8 * warp + q0 + u;
        const int m1 = t >> 1, h = t & 1;
        double2 t2 = cmul(p2[h][0], ctile3_get(acc[u], 0));
        cmac(t2, p2[h][1], ctile3_get(acc[u], 1));
        const double2 p1v = iv ? pa[m1] : zero;
        const double2 z = cmul(p1v, t2);
        part.x += z.x;
        part.y += z.y;
        if (IM) {
          double2 d2 = cmul(p2[h][0], ctile3_get(acd[u], 0));
          cmac(d2, p2[h][1], ctile3_get(acd[u], 1));
          pim += p1v.x * d2.y + p1v.y * d2.x;
        }
      }
    }
    {
      CTile3 acc = kZeroTile3;
#pragma unroll
      for (int k = 0; k < 2; ++k)
        cdmma3(acc, zB[k].x + zB[k].y, zB[k].x, zB[k].y, lB[k].x, lB[k].y - lB[k].x,
               lB[k].x + lB[k].y);
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const int rb = 8 * warp + 2 * tq + v;
        if (rb >= kH16BR || !iv) continue;
        int m1, m2;
        h16_brow(rb, m1, m2);
        const double2 z = cmul(cmul(pa[m1], pa[MM + m2]), ctile3_get(acc, v));
        part.x += z.x;
        part.y += z.y;
        pim += z.y;
      }
    }
    {
      CTile3 acc = kZeroTile3;
#pragma unroll
      for (int k = 0; k < 2; ++k)
        cdmma3(acc, zC[k].x + zC[k].y, zC[k].x, zC[k].y, lC[k].x, lC[k].y - lC[k].x,
               lC[k].x + lC[k].y);
      if (iv) {
        const int m1a = 8 * (warp >> 1) + 2 * tq;
        double2 zc = cmul(pa[m1a], ctile3_get(acc, 0));
        cmac(zc, pa[m1a + 1], ctile3_get(acc, 1));
        const double2 z = cmul(pa[2 * MM], zc);
        part.x += z.x;
        part.y += z.y;
        pim += z.y;
      }
    }
    for (int off = 1; off < 4; off <<= 1) {
      part.x += __shfl_xor_sync(0xffffffffu, part.x, off);
      part.y += __shfl_xor_sync(0xffffffffu, part.y, off);
      pim += __shfl_xor_sync(0xffffffffu, pim, off);
    }
    if (tq == 0) {
      red[warp][g] = part;
      redi[warp][g] = pim;
    }
    __syncthreads();
    if (threadIdx.x < 8 && pb + threadIdx.x < pend) {
      double sum = red[0][threadIdx.x].x, si = redi[0][threadIdx.x];
      for (int w = 1; w < 4; ++w) {
        sum += red[w][threadIdx.x].x;
        si += redi[w][threadIdx.x];
      }
      far_[(long long)r * n + pb + threadIdx.x] = weight * sum;
      const double im = fabs(weight * si);
      if (IM && im > 0.0)
        atomicMax(imag_bits, static_cast<unsigned long long>(__double_as_longlong(im)));
    }
    __syncthreads();
  }
}
