// Hermitian half spectrum for any even M (3-D, shared grids; M = 16 has its
// own fused kernels in k_half_dmma.inc.cuh). Stored nodes per box, H = M / 2:
//   A   rows (m1, m2) x m3 in [H, M)             e = (m1 M + m2) H + m3 - H
//   C   the m3 = 0 plane                          e = oC + m1 M + m2
//   B1  m1 = 0, m2 in [0, M), m3 in [1, H)       e = oB + m2 (H - 1) + m3 - 1
//   B2  m2 = 0, m1 in [1, M), m3 in [1, H)       e = oB + (M - 1 + m1)(H - 1) + m3 - 1
// (oC = M^2 H, oB = oC + M^2; the M = 16 layout of build_h16 is this one).
// The missing nodes are the mirrors (M - m1, M - m2, M - m3) of the block-A
// nodes with m1, m2 >= 1, m3 >= H + 1, whose C weights fold into Ct (see
// build_half). P2M / L2P of block A are the large-M DMMA GEMMs restricted to
// the upper m3 half (k_p2m_big with a column window, k_l2p_half_a); blocks C,
// B1, B2 are three small two-axis GEMMs per leaf / point tile (k_p2m_axes,
// k_l2p_axes) with the third axis folded into the per-point weight.
// Fragment of blfmm.cu (one translation unit): included inside namespace
// blfmm_gpu; not a standalone header.

struct HalfAxes {  // one of the blocks C / B1 / B2
  int ax, a0, na;  // row axis, first index, count
  int bx, b0, nb;  // column axis
  int fx, f0;      // fixed axis folded into the point weight
  long long off;   // element offset of the block inside the box
  int stride;      // row stride of the block
};
__device__ __forceinline__ HalfAxes half_block(int blk, int M) {
  const int H = M / 2;
  const long long oC = (long long)M * M * H, oB = oC + (long long)M * M;
  if (blk == 0) return HalfAxes{0, 0, M, 1, 0, M, 2, 0, oC, M};
  if (blk == 1) return HalfAxes{1, 0, M, 2, 1, H - 1, 0, 0, oB, H - 1};
  return HalfAxes{0, 1, M - 1, 2, 1, H - 1, 1, 0, oB + (long long)M * (H - 1), H - 1};
}

// P2M of blocks C / B1 / B2 (blockIdx.y): V[a][b] = sum_j conj(Pa_j[a])
// (lambda_j conj(Pf_j[f0]) conj(Pb_j[b])); 8 warps = 8 row tiles, all column
// tiles per warp, the B operand of a 64-point chunk staged in shared memory.
// NCT column tiles per warp: 8 for block C (M columns), 4 for the B blocks
// (H - 1 <= 31 columns: the 8-tile loop contracted four all-zero tiles);
// blk0 + blockIdx.y selects the block.
template <int NCT>
__global__ void __launch_bounds__(256, 1)
    k_p2m_axes(const int* __restrict__ leaf_list, const int* __restrict__ leaf_start,
               const double2* __restrict__ pht, const double* __restrict__ lam, int M,
               long long K, long long n, long long nleaf, double2* __restrict__ mult, int blk0) {
  extern __shared__ __align__(16) double2 ax_dyn[];  // [kBigPts][64]
  const HalfAxes hb = half_block(blk0 + blockIdx.y, M);
  const long long lf = leaf_list ? leaf_list[blockIdx.x] : blockIdx.x;
  const int r = blockIdx.z;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, tq = lane & 3;
  const int ra = 8 * warp + g;  // this lane's A row (block row a0 + ra)
  const bool rv = ra < hb.na;
  const int p0 = leaf_start[lf], p1 = leaf_start[lf + 1];
  const double* lr = lam + (long long)r * n;
  const int per = 3 * M;
  CTile acc[NCT];
#pragma unroll
  for (int u = 0; u < NCT; ++u) acc[u] = CTile{{0.0, 0.0}, {0.0, 0.0}};
  for (int c0 = p0; c0 < p1; c0 += kBigPts) {
    const int np = min(kBigPts, p1 - c0);
    __syncthreads();
    for (int t = threadIdx.x; t < np * hb.nb; t += blockDim.x) {
      const int j = t / hb.nb, c = t % hb.nb;
      const double2* pj = pht + (long long)(c0 + j) * per;
      const double w = __ldg(lr + c0 + j);
      const double2 z = cmul(__ldg(pj + hb.fx * M + hb.f0), __ldg(pj + hb.bx * M + hb.b0 + c));
      ax_dyn[j * 64 + c] = make_double2(w * z.x, -w * z.y);  // lambda conj(Pf Pb)
    }
    __syncthreads();
    for (int j0 = 0; j0 < np; j0 += 4) {
      const int j = j0 + tq;
      const bool jv = j < np;
      double2 za = make_double2(0.0, 0.0);
      if (jv && rv) za = __ldg(pht + (long long)(c0 + j) * per + hb.ax * M + hb.a0 + ra);
      const double are = za.x, aim = -za.y;  // conj(Pa)
#pragma unroll
      for (int u = 0; u < NCT; ++u) {
        const int col = 8 * u + g;
        const double2 b = (jv && col < hb.nb) ? ax_dyn[j * 64 + col] : make_double2(0.0, 0.0);
        cdmma(acc[u], are, aim, -aim, b.x, b.y);
      }
    }
  }
  if (!rv) return;
  double2* out = mult + ((long long)r * nleaf + lf) * K + hb.off + (long long)ra * hb.stride;
#pragma unroll
  for (int u = 0; u < NCT; ++u)
#pragma unroll
    for (int v = 0; v < 2; ++v) {
      const int col = 8 * u + 2 * tq + v;
      if (col < hb.nb) out[col] = make_double2(acc[u].re[v], acc[u].im[v]);
    }
}

// L2P of blocks C / B1 / B2 for PT 8-point tiles of one leaf (work8: PT = 1):
// for each block W_i[a] = sum_b Pb_i[b] L[a][b] on DMMA (A = the points' Pb,
// B = L^T, each B fragment loaded one k step ahead of its use; warp w takes row
// tiles w and w + 4), then part_i += Pf_i[f0] sum_a Pa_i[a] W_i[a]. Writes
// far_[i] = w Re part_i and imag_acc[i] = w Im part_i (block A adds to both
// afterwards). (PT = 4 on 32-point items measured the same as PT = 1: 10.04 vs
// 10.02 ms of P2 L2P; the same prefetch of k_p2m_axes' A fragment was slower,
// 7.75 -> 8.35 ms.)
template <int PT>
__global__ void __launch_bounds__(128)
    k_l2p_axes(const int2* __restrict__ work, const int* __restrict__ leaf_start,
               const double2* __restrict__ pht, const double2* __restrict__ loc, int M,
               long long K, long long n, long long nleaf, double weight,
               double* __restrict__ far_, double* __restrict__ imag_acc) {
  __shared__ double2 red[4][8 * PT];
  const int2 item = work[blockIdx.x];
  const long long lf = item.x;
  const int r = blockIdx.z;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, tq = lane & 3;
  const int pb = item.y, p1 = min(leaf_start[lf + 1], pb + 8 * PT);
  const int per = 3 * M;
  const double2 zero = make_double2(0.0, 0.0);
  const double2* pi[PT];  // A row / C row: point 8 pt + g
  bool iv[PT];
#pragma unroll
  for (int pt = 0; pt < PT; ++pt) {
    const int ia = pb + 8 * pt + g;
    iv[pt] = ia < p1;
    pi[pt] = pht + (long long)(iv[pt] ? ia : pb) * per;
  }
  const double2* la = loc + ((long long)r * nleaf + lf) * K;
  double2 part[PT];
#pragma unroll
  for (int pt = 0; pt < PT; ++pt) part[pt] = zero;
  for (int blk = 0; blk < 3; ++blk) {
    const HalfAxes hb = half_block(blk, M);
    double2 bpart[PT];
#pragma unroll
    for (int pt = 0; pt < PT; ++pt) bpart[pt] = zero;
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int rt = warp + 4 * q;  // row tile of a
      if (8 * rt >= hb.na) continue;
      const int arow = 8 * rt + g;  // B column n = g: row a of L
      const bool av = arow < hb.na;
      const double2* lrow = la + hb.off + (long long)(av ? arow : 0) * hb.stride;
      CTile acc[PT];
#pragma unroll
      for (int pt = 0; pt < PT; ++pt) acc[pt] = CTile{{0.0, 0.0}, {0.0, 0.0}};
      double2 lv = (av && tq < hb.nb) ? __ldg(lrow + tq) : zero;
      for (int k0 = 0; k0 < hb.nb; k0 += 4) {
        const int c = k0 + tq;
        const bool cv = c < hb.nb;
        const double2 lc = lv;
        lv = (av && c + 4 < hb.nb) ? __ldg(lrow + c + 4) : zero;
#pragma unroll
        for (int pt = 0; pt < PT; ++pt) {
          const double2 z = (iv[pt] && cv) ? __ldg(pi[pt] + hb.bx * M + hb.b0 + c) : zero;
          cdmma(acc[pt], z.x, z.y, -z.y, lc.x, lc.y);
        }
      }
      // C[point g][a = 8 rt + 2 tq + v]
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const int aa = 8 * rt + 2 * tq + v;
        if (aa >= hb.na) continue;
#pragma unroll
        for (int pt = 0; pt < PT; ++pt)
          if (iv[pt])
            cmac(bpart[pt], __ldg(pi[pt] + hb.ax * M + hb.a0 + aa),
                 make_double2(acc[pt].re[v], acc[pt].im[v]));
      }
    }
#pragma unroll
    for (int pt = 0; pt < PT; ++pt) cmac(part[pt], __ldg(pi[pt] + hb.fx * M + hb.f0), bpart[pt]);
  }
#pragma unroll
  for (int pt = 0; pt < PT; ++pt) {
    for (int off = 1; off < 4; off <<= 1) {
      part[pt].x += __shfl_xor_sync(0xffffffffu, part[pt].x, off);
      part[pt].y += __shfl_xor_sync(0xffffffffu, part[pt].y, off);
    }
    if (tq == 0) red[warp][8 * pt + g] = part[pt];
  }
  __syncthreads();
  if (threadIdx.x < 8 * PT && pb + threadIdx.x < p1) {
    double2 sum = red[0][threadIdx.x];
    for (int w = 1; w < 4; ++w) {
      sum.x += red[w][threadIdx.x].x;
      sum.y += red[w][threadIdx.x].y;
    }
    far_[(long long)r * n + pb + threadIdx.x] = weight * sum.x;
    imag_acc[(long long)r * n + pb + threadIdx.x] = weight * sum.y;
  }
}

// L2P of block A for an 8-point tile: W_i[row] = sum_{m3 >= H} P3_i[m3]
// L[row][m3 - H] on DMMA (k_l2p_mma's tiling, K = H), then u_i += w Re sum_row
// P1_i[m1] P2_i[m2] W_i[row]; IM: the imaginary residual of a mirrored pair is
// (C_m - C_m') Im T, so the imaginary part uses the locals scaled by D
// (dtab), added to the blocks' imag_acc and max-reduced.
template <int WN, int PT, bool IM>
__global__ void __launch_bounds__(128)
    k_l2p_half_a(const int2* __restrict__ work, const int* __restrict__ leaf_start,
                 const double2* __restrict__ pht, const double2* __restrict__ loc,
                 const double* __restrict__ dtab, int M, long long K, long long n,
                 long long nleaf, double weight, double* __restrict__ far_,
                 const double* __restrict__ imag_acc, unsigned long long* __restrict__ imag_bits) {
  // PT point tiles (8 PT points of one leaf) per CTA: every block-A local is
  // read once per 8 PT points instead of once per 8
  __shared__ double2 red[4][8 * PT];
  const int2 item = work[blockIdx.x];
  const long long lf = item.x;
  const int r = blockIdx.z;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, tq = lane & 3;
  const int H = M / 2;
  const long long rows = (long long)M * M, rtiles = (rows + 7) / 8;
  const int p1 = min(leaf_start[lf + 1], item.y + 8 * PT), pb = item.y;
  const int per = 3 * M;
  const double2* pa[PT];
  bool iv[PT];
#pragma unroll
  for (int pt = 0; pt < PT; ++pt) {
    const int ia = pb + 8 * pt + g;
    iv[pt] = ia < p1;
    pa[pt] = pht + (long long)(iv[pt] ? ia : pb) * per;
  }
  const double2* la = loc + ((long long)r * nleaf + lf) * K;
  double part[PT], pim[PT];
#pragma unroll
  for (int pt = 0; pt < PT; ++pt) part[pt] = pim[pt] = 0.0;
  for (long long tb = (long long)warp * WN; tb < rtiles; tb += 4LL * WN) {
    CTile acc[WN][PT], acd[WN][PT];
#pragma unroll
    for (int u = 0; u < WN; ++u)
#pragma unroll
      for (int pt = 0; pt < PT; ++pt) acc[u][pt] = acd[u][pt] = CTile{{0.0, 0.0}, {0.0, 0.0}};
    const double2* lrow[WN];
    bool bv[WN];
#pragma unroll
    for (int u = 0; u < WN; ++u) {
      const long long row = (tb + u) * 8 + g;
      bv[u] = (tb + u) < rtiles && row < rows;
      lrow[u] = la + (bv[u] ? row : 0) * H;
    }
    for (int k0 = 0; k0 < H; k0 += 4) {
      const int c = k0 + tq;
      const bool kv = c < H;
      double2 z[PT];
#pragma unroll
      for (int pt = 0; pt < PT; ++pt)
        z[pt] = (iv[pt] && kv) ? __ldg(pa[pt] + 2 * M + H + c) : make_double2(0.0, 0.0);
#pragma unroll
      for (int u = 0; u < WN; ++u) {
        const double2 lv = (bv[u] && kv) ? __ldg(lrow[u] + c) : make_double2(0.0, 0.0);
        double dv = 0.0;
        if (IM) {
          const long long row = (tb + u) * 8 + g;
          dv = (bv[u] && kv) ? __ldg(dtab + row * H + c) : 0.0;
        }
#pragma unroll
        for (int pt = 0; pt < PT; ++pt) {
          cdmma(acc[u][pt], z[pt].x, z[pt].y, -z[pt].y, lv.x, lv.y);
          if (IM) cdmma(acd[u][pt], z[pt].x, z[pt].y, -z[pt].y, dv * lv.x, dv * lv.y);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < WN; ++u)
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const long long row = (tb + u) * 8 + 2 * tq + v;
        if ((tb + u) >= rtiles || row >= rows) continue;
        const int m1 = static_cast<int>(row / M), m2 = static_cast<int>(row % M);
#pragma unroll
        for (int pt = 0; pt < PT; ++pt) {
          if (!iv[pt]) continue;
          const double2 p12 = cmul(__ldg(pa[pt] + m1), __ldg(pa[pt] + M + m2));
          part[pt] += p12.x * acc[u][pt].re[v] - p12.y * acc[u][pt].im[v];
          if (IM) pim[pt] += p12.x * acd[u][pt].im[v] + p12.y * acd[u][pt].re[v];
        }
      }
  }
#pragma unroll
  for (int pt = 0; pt < PT; ++pt) {
    for (int off = 1; off < 4; off <<= 1) {
      part[pt] += __shfl_xor_sync(0xffffffffu, part[pt], off);
      if (IM) pim[pt] += __shfl_xor_sync(0xffffffffu, pim[pt], off);
    }
    if (tq == 0) red[warp][8 * pt + g] = make_double2(part[pt], pim[pt]);
  }
  __syncthreads();
  if (threadIdx.x < 8 * PT && pb + threadIdx.x < p1) {
    double2 sum = red[0][threadIdx.x];
    for (int w = 1; w < 4; ++w) {
      sum.x += red[w][threadIdx.x].x;
      sum.y += red[w][threadIdx.x].y;
    }
    const long long i = (long long)r * n + pb + threadIdx.x;
    far_[i] += weight * sum.x;
    if (IM) {
      const double im = fabs(imag_acc[i] + weight * sum.y);
      if (im > 0.0)
        atomicMax(imag_bits, static_cast<unsigned long long>(__double_as_longlong(im)));
    }
  }
}

// Block-A L2P (no imaginary residual) for a span of up to 8 NPT points of one
// leaf per CTA (8 warps; the plan cuts a leaf into equal spans of <= 64 points
// and sorts them into classes NPT = 2, 4, 6, 8 by their tile count: one launch
// per class, no predicates in the contraction loop), in the 3-multiplication complex form (3 real DMMAs
// per complex tile step; k_l2p_h16S's scheme). The span's P3 phases (upper m3
// half) are staged once in shared memory (rows padded to 36 complex: the
// quarter-warp LDS.128 fragment loads are conflict-free, zeros beyond H; plus
// a plane of the 3M operand sums P3_r + P3_i), and
// every warp streams its row tiles of the leaf's local expansion (8 rows x H
// complex, contiguous) through a private double buffer with cp.async, one
// tile ahead: each local is read once per span, and no fragment load waits on
// global memory. W_i[row] = sum_{m3 >= H} P3_i[m3] L[row][m3 - H], then
// u_i += w Re sum_row P1_i[m1] P2_i[m2] W_i[row] (added to k_l2p_axes' far_).
constexpr int kHA3CS = 36;  // row stride (complex) of the staged phases / local tiles
template <int NPT, int NG>
__global__ void __launch_bounds__(256 * NG, (NG == 1 && NPT <= 4) ? 2 : 1)
    k_l2p_half_a3(const int4* __restrict__ work, const int* __restrict__ leaf_start,
                  const double2* __restrict__ pht, const double2* __restrict__ loc, int M,
                  long long K, long long n, long long nleaf, double weight,
                  double* __restrict__ far_) {
  extern __shared__ __align__(16) double2 ha3_dyn[];
  double2* const zsm = ha3_dyn;                          // [8 NPT][kHA3CS]
  double2* const lsm = zsm + 8 * NPT * kHA3CS;           // [8 NG warps][2][8][kHA3CS]
  double* const red = reinterpret_cast<double*>(lsm + 8 * NG * 2 * 8 * kHA3CS);  // [8][8 NPT]
  double* const zss = red + 8 * 8 * NPT;  // [8 NPT][kHA3CS] P3_r + P3_i (the 3M operand sum)
  const int4 item = work[blockIdx.x];  // (leaf, first point, end point, -)
  const long long lf = item.x;
  const int r = blockIdx.z;
  // warp = (point-tile group, row-tile lane): NG groups of NPW point tiles, 8
  // warps per group striding the row tiles. NG = 1 is what runs; two groups
  // (16 warps, 48 accumulator registers each) measured slower, P2 L2P 10.2 ->
  // 11.1 ms: every warp streams its own copy of the local tiles
  constexpr int NPW = NPT / NG;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int warp = wid & 7, grp = wid >> 3;
  const int g = lane >> 2, tq = lane & 3;
  const int H = M / 2;
  const int rows = M * M, rtiles = (rows + 7) / 8;
  const int pb = item.y, p1 = item.z;
  const int np = p1 - pb;  // <= 8 NPT (the item's class); padded point rows are zero
  const int per = 3 * M;
  const double2 zero = make_double2(0.0, 0.0);
  for (int t = threadIdx.x; t < 8 * NPT * kHA3CS; t += blockDim.x) {
    const int j = t / kHA3CS, c = t - j * kHA3CS;
    const double2 z =
        (j < np && c < H) ? __ldg(pht + (long long)(pb + j) * per + 2 * M + H + c) : zero;
    zsm[t] = z;
    zss[t] = z.x + z.y;
  }
  double2* const lbuf = lsm + wid * (2 * 8 * kHA3CS);
  for (int t = lane; t < 2 * 8 * kHA3CS; t += 32) lbuf[t] = zero;  // pad columns stay zero
  __syncthreads();
  const double2* la = loc + ((long long)r * nleaf + lf) * K;
  // stage row tile tb of the local expansion into buffer b (rows past the
  // grid re-read row 0: finite, never used)
  auto stage = [&](int b, int tb) {
    double2* dst = lbuf + b * (8 * kHA3CS);
    for (int t = lane; t < 8 * H; t += 32) {
      const int rr = t / H, c = t - rr * H;
      const int row = tb * 8 + rr;
      cp_async16(dst + rr * kHA3CS + c, la + (long long)(row < rows ? row : 0) * H + c);
    }
    cp_async_commit();
  };
  const double2* pa[NPW];
#pragma unroll
  for (int pt = 0; pt < NPW; ++pt)
    pa[pt] = pht + (long long)min(pb + 8 * (grp * NPW + pt) + g, p1 - 1) * per;
  double part[NPW];
#pragma unroll
  for (int pt = 0; pt < NPW; ++pt) part[pt] = 0.0;
  int buf = 0;
  if (warp < rtiles) stage(0, warp);
  for (int tb = warp; tb < rtiles; tb += 8, buf ^= 1) {
    if (tb + 8 < rtiles) {
      stage(buf ^ 1, tb + 8);
      cp_async_wait_group<1>();
    } else {
      cp_async_wait_group<0>();
    }
    __syncwarp();
    CTile3 acc[NPW];
#pragma unroll
    for (int pt = 0; pt < NPW; ++pt) acc[pt] = kZeroTile3;
    const double2* lt = lbuf + buf * (8 * kHA3CS) + g * kHA3CS + tq;
    const double2* zt = zsm + (grp * NPW * 8 + g) * kHA3CS + tq;
    const double* zst = zss + (grp * NPW * 8 + g) * kHA3CS + tq;
    for (int k0 = 0; k0 < H; k0 += 4) {
      const double2 lv = lt[k0];
      const double bd = lv.y - lv.x, bs = lv.x + lv.y;
#pragma unroll
      for (int pt = 0; pt < NPW; ++pt) {
        const double2 z = zt[pt * 8 * kHA3CS + k0];
        cdmma3(acc[pt], zst[pt * 8 * kHA3CS + k0], z.x, z.y, lv.x, bd, bs);
      }
    }
#pragma unroll
    for (int v = 0; v < 2; ++v) {
      const int row = tb * 8 + 2 * tq + v;
      if (row >= rows) continue;
      const int m1 = row / M, m2 = row - m1 * M;
#pragma unroll
      for (int pt = 0; pt < NPW; ++pt) {
        const double2 p12 = cmul(__ldg(pa[pt] + m1), __ldg(pa[pt] + M + m2));
        const double2 w = ctile3_get(acc[pt], v);
        part[pt] += p12.x * w.x - p12.y * w.y;
      }
    }
    __syncwarp();  // every lane is done with buffer `buf` before it is refilled
  }
#pragma unroll
  for (int pt = 0; pt < NPW; ++pt) {
    for (int off = 1; off < 4; off <<= 1) part[pt] += __shfl_xor_sync(0xffffffffu, part[pt], off);
    if (tq == 0) red[warp * (8 * NPT) + 8 * (grp * NPW + pt) + g] = part[pt];
  }
  __syncthreads();
  if (threadIdx.x < np) {
    double sum = red[threadIdx.x];
    for (int w = 1; w < 8; ++w) sum += red[w * (8 * NPT) + threadIdx.x];
    far_[(long long)r * n + pb + threadIdx.x] += weight * sum;
  }
}
