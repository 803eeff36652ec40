// Host: the launch sequence of a matvec, graphs, stats.
// Fragment of blfmm.cu (one translation unit): included inside
// namespace blfmm_gpu after the plan definition; not a standalone header.

// ------------------------------------------------------------- execute
inline double2* mult_ptr(blfmm_plan* p, int l) {
  if (p->xmode && p->xbuf && l >= 1 && l <= (p->xtele ? 1 : p->L - 2)) return p->xbuf + p->xoff[l];
  return p->lev[l].mult.as<double2>();
}

// phase 0: whole matvec; 1: exchange-mode upsweep (gather, halo P2M, own
// partial M2M into the exchange buffer); 2: exchange-mode downsweep (after the
// caller's all-reduce of the exchange buffer).
template <int D>
void launch_all(blfmm_plan* p, const double* d_lam_in, double* d_out, int phase = 0) {
  cudaStream_t st = p->stream;
  const long long n = p->n, K = p->Ks;  // stored nodes per expansion
  const int R = p->R, M = p->M, L = p->L;
  const LevelDev& leaf = p->lev[L];
  double side[3];
  for (int k = 0; k < 3; ++k) side[k] = (p->hi[k] - p->lo[k]) / static_cast<double>(1LL << L);
  LeafGeom geo;
  for (int k = 0; k < 3; ++k) {
    geo.lo[k] = p->lo[k];
    geo.side[k] = side[k];
  }
  geo.L = L;
  const bool profiling = p->profiling && phase == 0;
  // development builds: xp[3] = 1 records the stage events of the OVERLAPPED
  // schedule (near field on its own stream, times.ms[5] = its fork-to-end time)
  const bool serial_near = profiling && p->xp[3] != 1;
  // NVTX ranges name the stages' launch issue on the host timeline (nsys / ncu)
  static const char* const kStage[BLFMM_NSTAGES + 1] = {
      "blfmm gather", "blfmm p2m", "blfmm m2m", "blfmm m2l+l2l", "blfmm l2p", "blfmm near",
      "blfmm combine", "blfmm end"};
  auto mark = [&](int i) {
    if (profiling) CK(cudaEventRecord(p->ev[i], st));
    if (i > 0) nvtxRangePop();
    if (i < BLFMM_NSTAGES) nvtxRangePushA(kStage[i]);
  };
  const bool up = phase != 2, down = phase != 1;
  if (up) for (int i = 0; i < BLFMM_NSTAGES; ++i) p->times.launches[i] = 0;
  mark(0);
  if (up) CK(cudaMemsetAsync(p->imag_bits.p, 0, sizeof(unsigned long long), st));
  if (n && up) {
    k_gather_lambda<<<blocks_for(n, 256), 256, 0, st>>>(
        d_lam_in, p->perm.as<int>(), n, R, p->lam.as<double>(),
        R > 1 ? p->lamT.as<double>() : nullptr);
    p->times.launches[0]++;
  }
  mark(1);
  const double* x0 = p->xs[0].as<double>();
  const double* x1 = D > 1 ? p->xs[1].as<double>() : nullptr;
  const double* x2 = D > 2 ? p->xs[2].as<double>() : nullptr;
  // Near field (depends on the sorted lambda only): its own stream, so its
  // FP64 work can overlap the memory-bound far-field sweep.
  auto launch_near = [&](cudaStream_t sn) {
  if (leaf.nbox) {
    if (R == 1) {
      k_pack_src<<<blocks_for(n, 256), 256, 0, sn>>>(x0, x1, x2, p->lam.as<double>(), n, D,
                                                     p->src4.as<double4>());
      CK(cudaGetLastError());
      CK(cudaMemsetAsync(p->near_ctr.p, 0, sizeof(unsigned long long), sn));
      const long long ns = p->near_sym_min > 0 ? p->nsym : 0;
      // the serialised stage profile runs the near field alone at full occupancy
      const unsigned gp = (unsigned)(p->num_sms * (serial_near ? 5 : p->near_persist));
      auto launchp = [&](auto kern) {
        kern<<<gp, 32 * kNearWarps, 0, sn>>>(
            p->near_ctr.as<unsigned long long>(), p->sym_work.as<int4>(),
            p->sym_q.as<unsigned char>(), ns,
            p->sym_planes.as<double>(), p->near_work2.as<int2>(), p->nwork2,
            leaf.key.as<uint32_t>(), p->leaf_start.as<int>(), leaf.slotmap.as<int>(),
            p->src4.as<double4>(), L, p->kern.shape, n, p->near_.as<double>(),
            p->near_sym_min);
      };
      auto launchk = [&](auto kt) {
        constexpr int KT = decltype(kt)::value;
        if (p->near_minb == 6) launchp(k_near_all<D, KT, 3, 6>);
        else launchp(k_near_all<D, KT, 3, 1>);
      };
      if (p->kern.type == BLFMM_KERNEL_IMQ)
        launchk(std::integral_constant<int, BLFMM_KERNEL_IMQ>{});
      else if (p->kern.type == BLFMM_KERNEL_MQ)
        launchk(std::integral_constant<int, BLFMM_KERNEL_MQ>{});
      else
        launchk(std::integral_constant<int, BLFMM_KERNEL_GAUSSIAN>{});
      CK(cudaGetLastError());
      p->times.launches[5] += 2;
    } else if (R % 2 == 0 && R >= 8) {
      // batched right-hand sides on DMMA: one phi per pair for 32 of them
      k_pack_src<<<blocks_for(n, 256), 256, 0, sn>>>(x0, x1, x2, p->lam.as<double>(), n, D,
                                                     p->src4.as<double4>());
      CK(cudaGetLastError());
      auto launchd = [&](auto kern) {
        dim3 grid((unsigned)p->nwork128, (unsigned)((R + 31) / 32));
        kern<<<grid, 128, 0, sn>>>(p->work128.as<int2>(), leaf.key.as<uint32_t>(),
                                   p->leaf_start.as<int>(), leaf.slotmap.as<int>(),
                                   p->src4.as<double4>(), p->lamT.as<double>(), R, n, L,
                                   p->kern.shape, p->near_.as<double>());
      };
      const int kt = p->kern.type;
      if (kt == BLFMM_KERNEL_IMQ) launchd(k_near_dmma<D, BLFMM_KERNEL_IMQ>);
      else if (kt == BLFMM_KERNEL_MQ) launchd(k_near_dmma<D, BLFMM_KERNEL_MQ>);
      else launchd(k_near_dmma<D, BLFMM_KERNEL_GAUSSIAN>);
      p->times.launches[5] += 2;
    } else if (R % 16 == 0) {
      // batched right-hand sides (point-major weights, one phi per pair for
      // 16 right-hand sides)
      k_pack_src<<<blocks_for(n, 256), 256, 0, sn>>>(x0, x1, x2, p->lam.as<double>(), n, D,
                                                     p->src4.as<double4>());
      CK(cudaGetLastError());
      auto launch = [&](auto kern, int rt) {
        dim3 grid(blocks_for(p->nwork, kNearWarps), R / rt);
        kern<<<grid, 32 * kNearWarps, 0, sn>>>(
            p->near_work.as<int2>(), p->nwork, leaf.key.as<uint32_t>(), p->leaf_start.as<int>(),
            leaf.slotmap.as<int>(), p->src4.as<double4>(), p->lamT.as<double>(), R, n, L,
            p->kern.shape, p->near_.as<double>());
      };
      // (16 per chunk measured faster than 32: occupancy vs phi reuse)
      const int kt = p->kern.type;
      if (kt == BLFMM_KERNEL_IMQ) launch(k_near_warp_mr<D, BLFMM_KERNEL_IMQ, 16>, 16);
      else if (kt == BLFMM_KERNEL_MQ) launch(k_near_warp_mr<D, BLFMM_KERNEL_MQ, 16>, 16);
      else launch(k_near_warp_mr<D, BLFMM_KERNEL_GAUSSIAN, 16>, 16);
      p->times.launches[5] += 2;
    } else {
      dim3 grid((unsigned)leaf.nbox, blocks_for(R, 8));
      k_near<D, 8><<<grid, kNearThreads, 0, sn>>>(
          leaf.key.as<uint32_t>(), p->leaf_start.as<int>(), leaf.slotmap.as<int>(), x0, x1, x2,
          p->lam.as<double>(), n, R, L, p->kern.type, p->kern.shape, p->near_.as<double>());
      p->times.launches[5]++;
    }
    CK(cudaGetLastError());
  }
  };
  auto fork_near = [&]() {
    if (!serial_near) {
      CK(cudaEventRecord(p->fork, st));
      CK(cudaStreamWaitEvent(p->stream_near, p->fork, 0));
      if (profiling) CK(cudaEventRecord(p->ev_near[0], p->stream_near));
      launch_near(p->stream_near);
      if (profiling) CK(cudaEventRecord(p->ev_near[1], p->stream_near));
      CK(cudaEventRecord(p->join, p->stream_near));
    }
  };
  // P2M (exchange mode: the owned leaves and their halo only)
  // P2M fused with the leaf-level M2M (whole-matvec phase, half spectrum)
  const bool fuse_up =
      phase == 0 && p->h16 && !p->mr && p->n_p2m_plist > 0 && !p->scaled && !p->xbuf;
  const int* leaf_list = phase == 1 ? p->eleaf.as<int>() : nullptr;
  const long long np2m = phase == 1 ? p->n_eleaf : leaf.nbox;
  if (up && np2m) {
    if (D == 1) {
      // (d = 1 forms the phases in registers: no staged rows, any M)
      const int batch = 1;
      const size_t smem = 0;
      dim3 grid((unsigned)np2m, blocks_for(K, kP2MThreads * kP2MNodesPerThread), R);
      k_p2m<D><<<grid, kP2MThreads, smem, st>>>(
          leaf_list, leaf.key.as<uint32_t>(), p->leaf_start.as<int>(), x0, x1, x2, p->lam.as<double>(),
          p->xi.as<double>(), M, K, L, n, leaf.nbox, p->lo[0], p->lo[1], p->lo[2], side[0],
          side[1], side[2], batch, leaf.mult.as<double2>());
    } else if (D == 3 && fuse_up) {
      const size_t smem = sizeof(double2) * kH16Ks;
      CK(cudaFuncSetAttribute(k_p2m_m2m_h16, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)smem));
      const LevelDev& pl = p->lev[L - 1];
      dim3 grid((unsigned)p->n_p2m_plist, 1, R);
      k_p2m_m2m_h16<<<grid, 128, smem, st>>>(
          p->p2m_plist.as<int>(), pl.child_start.as<int>(), leaf.key.as<uint32_t>(),
          p->leaf_start.as<int>(), p->pht.as<double2>(), p->lam.as<double>(), n, leaf.nbox,
          pl.nbox, p->m2m_tab.as<double2>() + (size_t)L * 3 * 2 * M, leaf.mult.as<double2>(),
          mult_ptr(p, L - 1));
    } else if (D == 2 && p->g2d16) {
      dim3 grid((unsigned)((np2m + 3) / 4), 1, R);
      k_p2m_2d16<<<grid, 128, 0, st>>>(leaf_list, np2m, leaf.key.as<uint32_t>(),
                                       p->leaf_start.as<int>(), x0, x1, p->lam.as<double>(), n,
                                       leaf.nbox, L, p->lo[0], p->lo[1], side[0], side[1],
                                       p->sigma, 2.0 * p->sigma / M, leaf.mult.as<double2>());
    } else if (D == 3 && p->mr) {
      auto launch_mr = [&](auto kern, int span, int nw) {
        const int smem = (int)(sizeof(double2) * span * kMRRowP + sizeof(double) * span * kMRLam);
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        dim3 grid((unsigned)np2m, (unsigned)((R + 31) / 32));
        kern<<<grid, 32 * nw, smem, st>>>(leaf_list, leaf.key.as<uint32_t>(),
                                          p->leaf_start.as<int>(), x0, x1, x2, geo,
                                          2.0 * p->sigma / M, p->node_m.as<int>(),
                                          p->lam.as<double>(), R, n, leaf.nbox,
                                          leaf.mult.as<double2>());
      };
      // leaves of more than 64 points: one 128-point span (no partial-sum
      // read-back; 8 warps, 1 CTA per SM), else 64-point spans (3 CTAs / SM)
      if (p->max_leaf_pts > 64 && p->p2m_span != 64) launch_mr(k_p2m_mr<128, 8>, 128, 8);
      else launch_mr(k_p2m_mr<64, 4>, 64, 4);
    } else if (D == 3 && p->herm && !p->h16) {
      // half spectrum, even M != 16: block A on the large-M kernel (upper m3
      // half), blocks C / B1 / B2 as three small GEMMs
      const int H = M / 2;
      const long long rtiles = ((long long)M * M + 7) / 8;
      // block A: 3M DMMA, B staged once per (leaf, row-tile group); H <= 32
      // always holds here (even M <= 64)
      {
        constexpr int kGroups = 2;
        const int sm3 = (int)(sizeof(double) * 3 * kBig3Pts * kBig3CS);
        auto kern = k_p2m_big3<1, 8, 2>;
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, sm3));
        kern<<<dim3((unsigned)(np2m * kGroups), 1, R), 256, sm3, st>>>(
            leaf_list, p->leaf_start.as<int>(), p->pht.as<double2>(), p->lam.as<double>(), M, K, n,
            leaf.nbox, leaf.mult.as<double2>(), H, H, kGroups);
      }
      const int smx = (int)(sizeof(double2) * kBigPts * 64);
      // block C: M <= 64 columns (8 tiles); blocks B1 / B2: H - 1 <= 31 columns (4 tiles)
      CK(cudaFuncSetAttribute(k_p2m_axes<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smx));
      CK(cudaFuncSetAttribute(k_p2m_axes<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smx));
      k_p2m_axes<8><<<dim3((unsigned)np2m, 1, R), 256, smx, st>>>(
          leaf_list, p->leaf_start.as<int>(), p->pht.as<double2>(), p->lam.as<double>(), M, K, n,
          leaf.nbox, leaf.mult.as<double2>(), 0);
      k_p2m_axes<4><<<dim3((unsigned)np2m, 2, R), 256, smx, st>>>(
          leaf_list, p->leaf_start.as<int>(), p->pht.as<double2>(), p->lam.as<double>(), M, K, n,
          leaf.nbox, leaf.mult.as<double2>(), 1);
      if (p->hK < K)  // padding nodes stay zero
        CK(cudaMemset2DAsync(leaf.mult.as<double2>() + p->hK, sizeof(double2) * K, 0,
                             sizeof(double2) * (K - p->hK), (size_t)R * leaf.nbox, st));
    } else if (D == 3 && p->h16) {
      dim3 grid((unsigned)np2m, 1, R);
      k_p2m_h16w4<<<grid, 128, 0, st>>>(leaf_list, p->leaf_start.as<int>(), p->pht.as<double2>(),
                                        p->lam.as<double>(), n, leaf.nbox, leaf.mult.as<double2>());
    } else if (D == 3 && M >= 24 && M <= 64) {
      const long long rtiles = ((long long)M * M + 7) / 8;
      const int smem = (int)(sizeof(double2) * kBigPts * M);
      dim3 grid((unsigned)np2m, (unsigned)((rtiles + 7) / 8), R);
      auto lb = [&](auto kern) {
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        kern<<<grid, 256, smem, st>>>(leaf_list, p->leaf_start.as<int>(), p->pht.as<double2>(),
                                      p->lam.as<double>(), M, K, n, leaf.nbox,
                                      leaf.mult.as<double2>(), 0, M);
      };
      if (M <= 32) lb(k_p2m_big<4>);
      else lb(k_p2m_big<8>);
    } else {
      constexpr int WR = 4, WC = 2;
      const long long rtiles = (K / M + 7) / 8;
      const int ctiles = (M + 7) / 8;
      const int ncb = (ctiles + WC - 1) / WC;
      const long long nrb = (rtiles + 4 * WR - 1) / (4 * WR);
      dim3 grid((unsigned)np2m, (unsigned)(nrb * ncb), R);
      k_p2m_mma<D, WR, WC><<<grid, 128, 0, st>>>(leaf_list, p->leaf_start.as<int>(),
                                                 p->pht.as<double2>(),
                                                 p->lam.as<double>(), M, K, n, leaf.nbox, ncb,
                                                 leaf.mult.as<double2>());
    }
    CK(cudaGetLastError());
    p->times.launches[1]++;
  }
  mark(2);
  // the near field (FP64-bound) forked here co-runs with the HBM-bound M2M
  // (and, in exchange mode, with the caller's all-reduce)
  if (up) fork_near();
  if (phase == 0 && p->scaled) {
    // M2M with Lagrange interpolation onto each parent grid, leaf -> level 2
    const size_t smem = sizeof(double2) * 2 * K;
    CK(cudaFuncSetAttribute(k_m2m_scaled<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)smem));
    for (int l = L; l >= 3; --l) {
      const LevelDev& ch = p->lev[l];
      LevelDev& pa = p->lev[l - 1];
      if (!pa.nbox) continue;
      dim3 grid((unsigned)pa.nbox, R);
      if (D == 3 && K <= 8 * 512) {
        auto launchm = [&](auto kern) {
          CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)(sizeof(double2) * K)));
          kern<<<grid, 512, sizeof(double2) * K, st>>>(
              ch.key.as<uint32_t>(), pa.child_start.as<int>(), ch.mult.as<double2>(), ch.nbox,
              pa.nbox, p->plo_tab.as<int>() + (size_t)l * M,
              p->pw_tab.as<double>() + (size_t)l * M * p->stencil, p->stencil,
              p->m2m_tab.as<double2>() + (size_t)l * 3 * 2 * M, M, (int)K,
              pa.mult.as<double2>());
        };
        const long long kpt = (K + 511) / 512;
        if (kpt <= 2) launchm(k_m2m_scaled3<2, 512>);
        else if (kpt <= 4) launchm(k_m2m_scaled3<4, 512>);
        else launchm(k_m2m_scaled3<8, 512>);
        CK(cudaGetLastError());
        p->times.launches[2]++;
        continue;
      }
      k_m2m_scaled<D><<<grid, 256, smem, st>>>(
          ch.key.as<uint32_t>(), pa.child_start.as<int>(), ch.mult.as<double2>(), ch.nbox,
          pa.nbox, p->ptab.as<double>() + (size_t)l * M * M,
          p->m2m_tab.as<double2>() + (size_t)l * 3 * 2 * M, M, (int)K, pa.mult.as<double2>());
      CK(cudaGetLastError());
      p->times.launches[2]++;
    }
  } else if (phase == 0) {
    // M2M, leaf -> level 1 (level 1 feeds the parent-neighborhood sums of level 2)
    for (int l = fuse_up ? L - 1 : L; l >= 2; --l) {
      const LevelDev& ch = p->lev[l];
      LevelDev& pa = p->lev[l - 1];
      if (!pa.nbox) continue;
      dim3 grid((unsigned)pa.nbox, blocks_for(K, 256), R);
      k_m2m<D><<<grid, 256, 0, st>>>(ch.key.as<uint32_t>(), pa.child_start.as<int>(),
                                     mult_ptr(p, l), ch.nbox, pa.nbox,
                                     p->m2m_tab.as<double2>() + (size_t)l * 3 * 2 * M, M, K,
                                     p->node_m.as<int>(), mult_ptr(p, l - 1));
      CK(cudaGetLastError());
      p->times.launches[2]++;
    }
  } else if (phase == 1) {
    // exchange mode: complete V_{L-1} on the halo set E_{L-1}; partial "own"
    // multipoles (owned leaves only, disjoint across ranks) for levels <= L-2
    // in the exchange buffer, which the caller all-reduces
    CK(cudaMemsetAsync(p->xbuf, 0, sizeof(double2) * p->xcount, st));
    const LevelDev& lvL = p->lev[L];
    const LevelDev& lv1 = p->lev[L - 1];
    const double2* tabL = p->m2m_tab.as<double2>() + (size_t)L * 3 * 2 * M;
    const double2* tabL1 = p->m2m_tab.as<double2>() + (size_t)(L - 1) * 3 * 2 * M;
    const int la = static_cast<int>(p->own_lo[L]), lb = static_cast<int>(p->own_hi[L]);
    if (p->n_epar) {
      dim3 grid((unsigned)p->n_epar, blocks_for(K, 256), R);
      k_m2m_x<D><<<grid, 256, 0, st>>>(lvL.key.as<uint32_t>(), lv1.child_start.as<int>(),
                                       lvL.mult.as<double2>(), 0, lvL.nbox, p->epar.as<int>(), 0, 0,
                                       lv1.nbox, 0, (int)lvL.nbox, tabL, M, K,
                                       p->node_m.as<int>(), lv1.mult.as<double2>());
    }
    const long long c1 = p->own_hi[L - 1] - p->own_lo[L - 1];
    if (c1 > 0) {
      dim3 grid((unsigned)c1, blocks_for(K, 256), R);
      k_m2m_x<D><<<grid, 256, 0, st>>>(lvL.key.as<uint32_t>(), lv1.child_start.as<int>(),
                                       lvL.mult.as<double2>(), 0, lvL.nbox, nullptr,
                                       p->own_lo[L - 1], p->own_lo[L - 1], c1, la, lb, tabL, M, K,
                                       p->node_m.as<int>(), p->own_l1.as<double2>());
      const long long c2 = p->own_hi[L - 2] - p->own_lo[L - 2];
      if (c2 > 0) {
        dim3 grid2((unsigned)c2, blocks_for(K, 256), R);
        k_m2m_x<D><<<grid2, 256, 0, st>>>(
            lv1.key.as<uint32_t>(), p->lev[L - 2].child_start.as<int>(), p->own_l1.as<double2>(),
            p->own_lo[L - 1], c1, nullptr, p->own_lo[L - 2], 0, p->lev[L - 2].nbox,
            (int)p->own_lo[L - 1], (int)p->own_hi[L - 1], tabL1, M, K, p->node_m.as<int>(),
            mult_ptr(p, L - 2));
      }
    }
    for (int l = L - 2; l >= 2; --l) {
      const long long cp = p->own_hi[l - 1] - p->own_lo[l - 1];
      if (cp <= 0) continue;
      dim3 grid((unsigned)cp, blocks_for(K, 256), R);
      k_m2m_x<D><<<grid, 256, 0, st>>>(
          p->lev[l].key.as<uint32_t>(), p->lev[l - 1].child_start.as<int>(), mult_ptr(p, l), 0,
          p->lev[l].nbox, nullptr, p->own_lo[l - 1], 0, p->lev[l - 1].nbox, (int)p->own_lo[l],
          (int)p->own_hi[l], p->m2m_tab.as<double2>() + (size_t)l * 3 * 2 * M, M, K,
          p->node_m.as<int>(), mult_ptr(p, l - 1));
    }
    CK(cudaGetLastError());
    nvtxRangePop();  // the upsweep half ends here (exchange mode)
    return;
  }
  mark(3);
  if (p->scaled) {
    // couple at every level 2..L (direct interaction lists, per-level grid
    // and C), then L2L top-down with anterpolation
    for (int l = 2; l <= L; ++l) {
      LevelDev& lv = p->lev[l];
      if (!lv.nbox) continue;
      if (D == 3) {  // separable 6^3-block form
        const LevelDev& pa = p->lev[l - 1];
        dim3 g3((unsigned)pa.nbox, blocks_for(K, kCoupleS3Threads), R);
        k_couple_scaled3<4><<<g3, kCoupleS3Threads, 0, st>>>(
            pa.key.as<uint32_t>(), pa.nbox, l, lv.slotmap.as<int>(), lv.mult.as<double2>(),
            lv.nbox, p->m2l_tab.as<double2>() + (size_t)l * 3 * 7 * M,
            p->ctab.as<double>() + (size_t)l * K, M, (int)K, lv.loc.as<double2>());
        CK(cudaGetLastError());
        p->times.launches[3]++;
        if (p->keep_couple) {
          if (lv.couple.bytes != lv.loc.bytes) lv.couple.alloc(lv.loc.bytes);
          CK(cudaMemcpyAsync(lv.couple.p, lv.loc.p, lv.loc.bytes, cudaMemcpyDeviceToDevice, st));
        }
        continue;
      }
      dim3 grid((unsigned)lv.nbox, blocks_for(K, kCoupleSThreads), R);
      k_couple_scaled<D><<<grid, kCoupleSThreads, 0, st>>>(
          lv.key.as<uint32_t>(), lv.nbox, l, lv.slotmap.as<int>(), lv.mult.as<double2>(),
          p->m2l_tab.as<double2>() + (size_t)l * 3 * 7 * M, p->ctab.as<double>() + (size_t)l * K,
          M, (int)K, lv.loc.as<double2>());
      CK(cudaGetLastError());
      p->times.launches[3]++;
      if (p->keep_couple) {
        if (lv.couple.bytes != lv.loc.bytes) lv.couple.alloc(lv.loc.bytes);
        CK(cudaMemcpyAsync(lv.couple.p, lv.loc.p, lv.loc.bytes, cudaMemcpyDeviceToDevice, st));
      }
    }
    const size_t smem = sizeof(double2) * 2 * K;
    CK(cudaFuncSetAttribute(k_l2l_scaled<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)smem));
    const double wratio = 1.0 / static_cast<double>(1 << D);  // w_l / w_{l+1}
    for (int l = 2; l < L; ++l) {
      LevelDev& lv = p->lev[l];
      LevelDev& ch = p->lev[l + 1];
      if (!lv.nbox || !ch.nbox) continue;
      dim3 grid((unsigned)lv.nbox, R);
      if (D == 3 && K <= 8 * 512) {
        auto launchl = [&](auto kern) {
          CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)(sizeof(double2) * K)));
          kern<<<grid, 512, sizeof(double2) * K, st>>>(
              lv.child_start.as<int>(), ch.key.as<uint32_t>(), lv.loc.as<double2>(), lv.nbox,
              ch.loc.as<double2>(), ch.nbox, p->ptr_tab.as<int>() + (size_t)(l + 1) * M * p->kt,
              p->ptw_tab.as<double>() + (size_t)(l + 1) * M * p->kt, p->kt,
              p->l2l_tab.as<double2>() + (size_t)(l + 1) * 3 * 2 * M, wratio, M, (int)K);
        };
        const long long kpt = (K + 511) / 512;
        if (kpt <= 2) launchl(k_l2l_scaled3<2, 512>);
        else if (kpt <= 4) launchl(k_l2l_scaled3<4, 512>);
        else launchl(k_l2l_scaled3<8, 512>);
        CK(cudaGetLastError());
        p->times.launches[3]++;
        continue;
      }
      k_l2l_scaled<D><<<grid, 256, smem, st>>>(
          lv.child_start.as<int>(), ch.key.as<uint32_t>(), lv.loc.as<double2>(), lv.nbox,
          ch.loc.as<double2>(), ch.nbox, p->ptab.as<double>() + (size_t)(l + 1) * M * M,
          p->l2l_tab.as<double2>() + (size_t)(l + 1) * 3 * 2 * M, wratio, M, (int)K);
      CK(cudaGetLastError());
      p->times.launches[3]++;
    }
  }
  // telescoped (whole matvec, shared grids, 3-D): G_L(a) = e^{i xi (x_a - x_0)}
  // C V_0, so only the leaf-level couple runs (NS_L and the root phase in its
  // epilogue); levels 1..L-1 (NS, G) are skipped. Stage dumps keep the
  // level-by-level sweep.
  const bool tele = D == 3 && p->telescope && !p->keep_couple && !p->scaled && L >= 2 && p->lev[1].nbox > 0 && p->root.p && p->root_tab.p;
  if (tele) {
    LevelDev& lv = p->lev[L];
    const LevelDev& pa = p->lev[L - 1];
    const LevelDev& l1 = p->lev[1];
    dim3 gr(blocks_for(K, 128), 1, R);
    k_root<D><<<gr, 128, 0, st>>>(l1.key.as<uint32_t>(), l1.nbox, mult_ptr(p, 1),
                                   p->m2m_tab.as<double2>() + (size_t)1 * 3 * 2 * M,
                                   p->ctab.as<double>(), M, K, p->node_m.as<int>(),
                                   p->root.as<double2>());
    CK(cudaGetLastError());
    p->times.launches[3]++;
    const long long plo = p->own_lo[L - 1], pcnt = p->own_hi[L - 1] - p->own_lo[L - 1];
    if (pcnt > 0 && lv.nbox) {
      auto launch_t = [&](auto kern, int npt) {
        dim3 grid3((unsigned)pcnt, blocks_for(K, kCouple3Threads * npt), R);
        kern<<<grid3, kCouple3Threads, 0, st>>>(
            lv.region.as<int>(), plo, pa.nbox, R * lv.nbox, mult_ptr(p, L), lv.nbox,
            p->m2l_tab.as<double2>() + ((size_t)L * 3 * 7 + 2) * M,
            p->m2m_tab.as<double2>() + (size_t)L * 3 * 2 * M, p->ctab.as<double>(), M, K,
            nullptr, nullptr, lv.loc.as<double2>(), nullptr, nullptr, nullptr,
            p->node_m.as<int>(), p->root.as<double2>(), p->root_tab.as<double2>(),
            pa.key.as<uint32_t>(), L - 1);
      };
      if (p->couple_var == 0) {
        launch_t(k_couple3<1, false, 4, 1, true>, 1);
      } else if (p->nseg > 0) {
        auto launch_c = [&](auto kern, int go) {
          const unsigned nch = blocks_for(K, 128);
          dim3 gc(go ? nch : (unsigned)p->nseg, go ? (unsigned)p->nseg : nch, R);
          kern<<<gc, 128, 0, st>>>(
              p->seg_hdr.as<int4>(), p->seg_slot.as<int>(), mult_ptr(p, L), lv.nbox, (int)R,
              p->m2l_tab.as<double2>() + ((size_t)L * 3 * 7 + 2) * M, p->ctab.as<double>(), M, K,
              p->node_m.as<int>(), p->root.as<double2>(), p->root_tab.as<double2>(), 1 << L,
              (int)p->own_lo[L], (int)p->own_hi[L], lv.loc.as<double2>());
        };
        // 2 x 2 columns, runs of <= 32 slabs, 128 registers (4 CTAs/SM). Measured
        // on P3 (couple ms): z16 1.375, z32 1.324, node chunks along x 1.487,
        // 2 x 1 columns at 5 / 6 CTAs/SM 1.519 / 1.573, 2 x 2 at 5 CTAs/SM
        // (spills) 1.542, 4 x 2 / 4 x 4 sub-tiled CTAs 1.74 / 2.14, the window
        // staged by TMA bulk copies into a 2 / 3 / 4-stage ring 2.05 / 2.86 /
        // 5.04
        launch_c(k_couple_col<2, kColZS, 4, 0>, 0);
      }
      CK(cudaGetLastError());
      p->times.launches[3]++;
    }
  }
  // couple (M2L) + L2L, level 1 (G_1 only) -> leaf
  for (int l = 1; l <= L && !p->scaled && !tele; ++l) {
    LevelDev& lv = p->lev[l];
    const LevelDev& pa = p->lev[l - 1];
    if (!lv.nbox) continue;
    const bool keep = p->keep_couple;
    if (keep) {
      if (lv.ns.bytes != lv.mult.bytes) lv.ns.alloc(lv.mult.bytes);
      if (l >= 2 && lv.couple.bytes != lv.mult.bytes) lv.couple.alloc(lv.mult.bytes);
      if (l >= 2 && lv.loc.bytes != lv.mult.bytes) lv.loc.alloc(lv.mult.bytes);
    }
    const long long plo = p->own_lo[l - 1], pcnt = p->own_hi[l - 1] - p->own_lo[l - 1];
    if (pcnt <= 0) continue;
    if (D == 3) {
      // one node per thread, 128 registers, 4 CTAs/SM (measured best of the
      // variants in DESIGN.md §5.4)
      dim3 grid3((unsigned)pcnt, blocks_for(K, kCouple3Threads), R);
      k_couple3<1, false, 4><<<grid3, kCouple3Threads, 0, st>>>(
          lv.region.as<int>(), plo, pa.nbox, R * lv.nbox, mult_ptr(p, l), lv.nbox,
          p->m2l_tab.as<double2>() + ((size_t)l * 3 * 7 + 2) * M,
          p->m2m_tab.as<double2>() + (size_t)l * 3 * 2 * M, p->ctab.as<double>(), M, K,
          l >= 2 ? pa.glob.as<double2>() : nullptr, l < L ? lv.glob.as<double2>() : nullptr,
          (l == L || (keep && l >= 2)) ? lv.loc.as<double2>() : nullptr,
          (keep && l >= 2) ? pa.ns.as<double2>() : nullptr, keep ? lv.ns.as<double2>() : nullptr,
          (keep && l >= 2) ? lv.couple.as<double2>() : nullptr, p->node_m.as<int>());
      CK(cudaGetLastError());
      p->times.launches[3]++;
      continue;
    }
    dim3 grid((unsigned)pcnt, blocks_for(K, kCoupleThreads), R);
    k_couple<D><<<grid, kCoupleThreads, 0, st>>>(
        lv.region.as<int>(), plo, pa.nbox, R * lv.nbox, l, lv.slotmap.as<int>(),
        mult_ptr(p, l),
        lv.nbox,
        p->m2l_tab.as<double2>() + ((size_t)l * 3 * 7 + 2) * M,  // o = -1..1 of each axis block
        p->m2m_tab.as<double2>() + (size_t)l * 3 * 2 * M, p->ctab.as<double>(), M, K,
        l >= 2 ? pa.glob.as<double2>() : nullptr, l < L ? lv.glob.as<double2>() : nullptr,
        (l == L || (keep && l >= 2)) ? lv.loc.as<double2>() : nullptr,
        (keep && l >= 2) ? pa.ns.as<double2>() : nullptr, keep ? lv.ns.as<double2>() : nullptr,
        (keep && l >= 2) ? lv.couple.as<double2>() : nullptr, 0, p->node_m.as<int>());
    CK(cudaGetLastError());
    p->times.launches[3]++;
  }
  if (down && p->n_zero_far) {
    k_zero_boxes<<<dim3((unsigned)p->n_zero_far, R), 256, 0, st>>>(
        leaf.loc.as<double2>(), p->zero_far.as<int>(), K, leaf.nbox);
    CK(cudaGetLastError());
  }
  mark(4);
  // L2P
  if (leaf.nbox) {
    if (D == 1) {
      // 8 points per batch
      auto launch1 = [&](auto kern, int) {
        const size_t smem = 0;  // d = 1: phases in registers
        dim3 grid((unsigned)leaf.nbox, R);
        kern<<<grid, kL2PThreads, smem, st>>>(
            leaf.key.as<uint32_t>(), p->leaf_start.as<int>(), x0, x1, x2, leaf.loc.as<double2>(),
            p->xi.as<double>(), M, K, L, n, leaf.nbox, p->lo[0], p->lo[1], p->lo[2], side[0],
            side[1], side[2], p->weight, p->far_.as<double>(),
            p->imag_bits.as<unsigned long long>());
      };
      launch1(k_l2p<D, 8>, 8);
    } else if (D == 3 && p->mr) {
      auto l2pm = p->want_imag ? k_l2p_mr<true> : k_l2p_mr<false>;
      const int smem = (int)(sizeof(double2) * (kMRSpan * kMRRow + 2 * 32 * kMRLS));
      CK(cudaFuncSetAttribute(l2pm, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      dim3 grid((unsigned)p->nwork64, (unsigned)((R + 31) / 32));
      l2pm<<<grid, 128, smem, st>>>(p->work64.as<int2>(), leaf.key.as<uint32_t>(),
                                    p->leaf_start.as<int>(), x0, x1, x2, geo, 2.0 * p->sigma / M,
                                    p->node_m.as<int>(), p->dtab.as<double>(),
                                    leaf.loc.as<double2>(), R, n, leaf.nbox, p->weight,
                                    p->far_.as<double>(), p->imag_bits.as<unsigned long long>());
    } else if (D == 3 && p->herm && !p->h16) {
      k_l2p_axes<1><<<dim3((unsigned)p->nwork8, 1, R), 128, 0, st>>>(
          p->work8.as<int2>(), p->leaf_start.as<int>(), p->pht.as<double2>(),
          leaf.loc.as<double2>(), M, K, n, leaf.nbox, p->weight, p->far_.as<double>(),
          p->himag.as<double>());
      // block A: 8-point tiles with the imaginary-residual GEMM (stats requested), else the
      // 3-multiplication kernel on class-sorted spans
      auto la = [&](auto kern, const DevBuf& wk, long long nw) {
        kern<<<dim3((unsigned)nw, 1, R), 128, 0, st>>>(
            wk.as<int2>(), p->leaf_start.as<int>(), p->pht.as<double2>(), leaf.loc.as<double2>(),
            p->dtab.as<double>(), M, K, n, leaf.nbox, p->weight, p->far_.as<double>(),
            p->himag.as<double>(), p->imag_bits.as<unsigned long long>());
      };
      if (p->want_imag) la(k_l2p_half_a<2, 1, true>, p->work8, p->nwork8);
      else {
        // stats-free block A: 3M DMMA on class-sorted spans (<= 64 points)
        auto la3 = [&](auto kern, int c, int ng, long long off) {
          if (!p->nwork_ha[c]) return;
          const int npt = 2 * (c + 1);
          const int smem = (int)(sizeof(double2) * (8 * npt * kHA3CS + 8 * ng * 2 * 8 * kHA3CS) +
                                 sizeof(double) * (8 * 8 * npt + 8 * npt * kHA3CS));
          CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
          kern<<<dim3((unsigned)p->nwork_ha[c], 1, R), 256 * ng, smem, st>>>(
              p->work_ha.as<int4>() + off, p->leaf_start.as<int>(), p->pht.as<double2>(),
              leaf.loc.as<double2>(), M, K, n, leaf.nbox, p->weight, p->far_.as<double>());
        };
        long long off = 0;
        la3(k_l2p_half_a3<2, 1>, 0, 1, off);
        off += p->nwork_ha[0];
        la3(k_l2p_half_a3<4, 1>, 1, 1, off);
        off += p->nwork_ha[1];
        la3(k_l2p_half_a3<6, 1>, 2, 1, off);
        off += p->nwork_ha[2];
        // (16 warps as two point-tile groups, k_l2p_half_a3<8, 2>, measured
        // slower: P2 L2P 10.2 -> 11.1 ms)
        la3(k_l2p_half_a3<8, 1>, 3, 1, off);
      }
    } else if (D == 3 && p->h16) {
      dim3 grid((unsigned)p->nwork128, 1, R);
      // the D-weighted GEMM of max|Im| only when the caller asked for stats
      auto l2pS = p->want_imag ? k_l2p_h16S<4, true> : k_l2p_h16S<4, false>;
      const int l2p_smem = (int)(sizeof(double2) * (kH16Ks + 2 * 8 * 52));
      CK(cudaFuncSetAttribute(l2pS, cudaFuncAttributeMaxDynamicSharedMemorySize, l2p_smem));
      l2pS<<<grid, 128, l2p_smem, st>>>(p->work128.as<int2>(), p->leaf_start.as<int>(),
                                        p->pht.as<double2>(), leaf.loc.as<double2>(),
                                        p->dtab.as<double>(), n, leaf.nbox, p->weight,
                                        p->far_.as<double>(), p->imag_bits.as<unsigned long long>());
    } else if (D == 2 && p->g2d16) {
      // warp items of 128-point spans (k_l2p_2d16's header)
      dim3 grid((unsigned)((p->nwork128 + 3) / 4), 1, R);
      k_l2p_2d16<<<grid, 128, 0, st>>>(p->work128.as<int2>(), p->nwork128,
                                       leaf.key.as<uint32_t>(), p->leaf_start.as<int>(), x0, x1,
                                       leaf.loc.as<double2>(), n, leaf.nbox, L, p->lo[0], p->lo[1],
                                       side[0], side[1], p->sigma, 2.0 * p->sigma / M, p->weight,
                                       p->far_.as<double>(),
                                       p->imag_bits.as<unsigned long long>(), kL2PSpan);
    } else {
      constexpr int WN = 4;
      dim3 grid((unsigned)p->nwork8, 1, R);
      k_l2p_mma<D, WN><<<grid, 128, 0, st>>>(p->work8.as<int2>(), p->leaf_start.as<int>(),
                                             p->pht.as<double2>(),
                                             leaf.loc.as<double2>(), M, K, n, leaf.nbox,
                                             p->weight, p->far_.as<double>(),
                                             p->imag_bits.as<unsigned long long>());
    }
    CK(cudaGetLastError());
    p->times.launches[4]++;
  }
  mark(5);
  if (serial_near) launch_near(st);  // serialised for per-stage timing
  mark(6);
  if (!serial_near) CK(cudaStreamWaitEvent(st, p->join, 0));
  if (n) {
    if (p->world > 1 && !p->gather_sorted)  // non-owned entries are 0: a sum over ranks is u
      CK(cudaMemsetAsync(d_out, 0, sizeof(double) * R * n, st));
    const long long s0 = p->own_pt_lo, s1 = p->own_pt_hi;
    if (s1 > s0)
      k_combine<<<blocks_for(s1 - s0, 256), 256, 0, st>>>(
          p->far_.as<double>(), p->near_.as<double>(),
          p->gather_sorted ? nullptr : p->perm.as<int>(), n, s0, s1, R,
          p->gather_sorted ? p->usorted.as<double>() : d_out,
          (R == 1 && p->near_sym_min > 0) ? p->sym_planes.as<double>() : nullptr,
          p->sym_pmask.as<unsigned>());
    CK(cudaGetLastError());
    p->times.launches[6]++;
  }
  mark(7);
}

void run(blfmm_plan* p, const double* d_lam_in, double* d_out, cudaStream_t user,
         bool fence_default = false, int phase = 0) {
  // Work is issued on the plan stream; a caller stream is ordered before and
  // after it with events so either stream can be used for timing. With
  // fence_default a NULL caller stream means the legacy default stream (the
  // device-pointer API: data produced / consumed there must be ordered too).
  const bool fence = (user && user != p->stream) || (!user && fence_default);
  if (fence) {
    CK(cudaEventRecord(p->fence_in, user));
    CK(cudaStreamWaitEvent(p->stream, p->fence_in, 0));
  }
  auto issue = [&] {
    if (p->d == 1) launch_all<1>(p, d_lam_in, d_out, phase);
    if (p->d == 2) launch_all<2>(p, d_lam_in, d_out, phase);
    if (p->d == 3) launch_all<3>(p, d_lam_in, d_out, phase);
  };
  // (exchange-mode phases 1/2 are not captured: the near-field fork of the
  // upsweep joins in the downsweep, across the caller's all-reduce)
  if (p->use_graphs && !p->profiling && !p->keep_couple && phase == 0) {
    cudaGraphExec_t exec = nullptr;
    for (const auto& g : p->graphs)
      if (g.lam == d_lam_in && g.out == d_out && g.phase == phase && g.imag == p->want_imag)
        exec = g.exec;
    bool again = false;  // capture on the second use of a pointer pair only
    for (const auto& q : p->seen) again = again || (q.first == d_lam_in && q.second == d_out);
    if (!exec && !again) {
      if (p->seen.size() >= 16) p->seen.erase(p->seen.begin());
      p->seen.push_back({d_lam_in, d_out});
      issue();
      goto fenced;
    }
    if (!exec) {
      if (p->graphs.size() >= 8) {
        CK(cudaStreamSynchronize(p->stream));
        cudaGraphExecDestroy(p->graphs.front().exec);
        p->graphs.erase(p->graphs.begin());
      }
      cudaGraph_t graph = nullptr;
      CK(cudaStreamBeginCapture(p->stream, cudaStreamCaptureModeThreadLocal));
      try {
        issue();
      } catch (...) {
        cudaStreamEndCapture(p->stream, &graph);
        if (graph) cudaGraphDestroy(graph);
        cudaGetLastError();
        p->use_graphs = false;  // this plan launches directly from now on
        issue();
        goto fenced;
      }
      CK(cudaStreamEndCapture(p->stream, &graph));
      CK(cudaGraphInstantiate(&exec, graph, 0));
      CK(cudaGraphDestroy(graph));
      p->graphs.push_back({d_lam_in, d_out, phase, p->want_imag, exec});
    }
    CK(cudaGraphLaunch(exec, p->stream));
  } else {
    issue();
  }
fenced:
  if (fence) {
    CK(cudaEventRecord(p->fence_out, p->stream));
    CK(cudaStreamWaitEvent(user, p->fence_out, 0));
  }
}

void collect_times(blfmm_plan* p) {
  if (!p->profiling) return;
  CK(cudaEventSynchronize(p->ev[BLFMM_NSTAGES]));
  for (int i = 0; i < BLFMM_NSTAGES; ++i) {
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, p->ev[i], p->ev[i + 1]));
    p->times.ms[i] = ms;
  }
  if (p->xp[3] == 1) {
    float ms = 0.f;
    CK(cudaEventSynchronize(p->ev_near[1]));
    CK(cudaEventElapsedTime(&ms, p->ev_near[0], p->ev_near[1]));
    p->times.ms[5] = ms;
  }
}

void fill_stats(blfmm_plan* p, blfmm_stats* s, bool single) {
  if (!s) return;
  unsigned long long bits = 0;
  CK(cudaMemcpyAsync(&bits, p->imag_bits.p, sizeof(bits), cudaMemcpyDeviceToHost, p->stream));
  CK(cudaStreamSynchronize(p->stream));
  double v;
  std::memcpy(&v, &bits, sizeof(v));
  s->max_imag_residual = v;
  s->near_pairs = p->info.near_pairs;
  s->far_work = single ? p->info.far_work_single : p->info.far_work;
}
