// Host: plan creation (tree, tables, work lists, segment tables).
// Fragment of blfmm.cu (one translation unit): included inside
// namespace blfmm_gpu after the plan definition; not a standalone header.

// ============================================================ host helpers
void partition_ranges(const double* cost, long long n, int world, long long* bounds);
inline unsigned blocks_for(long long n, int t) {
  return static_cast<unsigned>((n + t - 1) / t);
}

void set_error(const Error& e) {
  g_last_error = e.what();
  g_last_value = e.achieved;
}
void set_error_message(const char* msg) { g_last_error = msg; }

template <class F>
int guarded(F&& f) {
  try {
    f();
    return BLFMM_OK;
  } catch (const Error& e) {
    set_error(e);
    return e.code;
  } catch (const std::bad_alloc&) {
    g_last_error = "host allocation failed";
    return BLFMM_ENOMEM;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return BLFMM_EINVAL;
  }
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    int cnt = 0;
    cudaError_t e = cudaGetDeviceCount(&cnt);
    if (e != cudaSuccess || cnt == 0)
      throw Error(BLFMM_ECUDA, std::string("no CUDA device available: ") +
                                   (e != cudaSuccess ? cudaGetErrorString(e) : "0 devices"));
    CK(cudaGetDevice(&prev));
    if (dev >= 0 && dev != prev) CK(cudaSetDevice(dev));
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

template <class T>
void upload(DevBuf& buf, const std::vector<T>& v) {
  buf.alloc(v.size() * sizeof(T));
  if (!v.empty()) CK(cudaMemcpy(buf.p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
}

template <class F>
void cub_call(DevBuf& scratch, cudaStream_t st, F&& f) {
  size_t bytes = 0;
  CK(f(nullptr, bytes));
  if (bytes > scratch.bytes) scratch.alloc(bytes);
  CK(f(scratch.p, bytes));
  (void)st;
}

// Per-level phase tables (host, double): m2m[l][k][delta][m] =
// e^{i xi_m (1/2 - delta) h_{l,k}}, m2l[l][k][o+3][m] = e^{-i xi_m o h_{l,k}}.
// Hermitian half-spectrum node table, Ct and D for an even M (layout in
// k_halfm.inc.cuh; M = 16 is the layout the k_*_h16* kernels tile): node[e] =
// m1 | m2 << 8 | m3 << 16; Ct = C_m + C_m' and D = (C_m - C_m') / Ct for the
// block-A nodes whose mirror m' = (M - m1, M - m2, M - m3) is not stored
// (m1, m2 >= 1, m3 >= M/2 + 1), Ct = C_m and D = 1 otherwise. Returns the
// stored count; the vectors are padded to a multiple of 32 nodes.
long long build_half(const std::vector<double>& c, int M, std::vector<int>& node,
                     std::vector<double>& ct, std::vector<double>& dt) {
  const int H = M / 2;
  const long long nA = (long long)M * M * H, nC = (long long)M * M,
                  nB = (long long)(2 * M - 1) * (H - 1);
  const long long K = nA + nC + nB, Ks = (K + 31) / 32 * 32;
  node.assign(Ks, 0);
  ct.assign(Ks, 0.0);
  dt.assign(Ks, 0.0);
  auto full = [M](int m1, int m2, int m3) { return ((long long)m1 * M + m2) * M + m3; };
  auto put = [&](long long e, int m1, int m2, int m3) {
    node[e] = m1 | (m2 << 8) | (m3 << 16);
    const double v = c[full(m1, m2, m3)];
    ct[e] = v;
    dt[e] = 1.0;
    if (m1 >= 1 && m2 >= 1 && m3 >= H + 1) {
      const double vm = c[full(M - m1, M - m2, M - m3)];
      ct[e] = v + vm;
      dt[e] = ct[e] != 0.0 ? (v - vm) / ct[e] : 0.0;
    }
  };
  for (int m1 = 0; m1 < M; ++m1)
    for (int m2 = 0; m2 < M; ++m2)
      for (int m3 = H; m3 < M; ++m3) put(((long long)m1 * M + m2) * H + m3 - H, m1, m2, m3);
  for (int m1 = 0; m1 < M; ++m1)
    for (int m2 = 0; m2 < M; ++m2) put(nA + (long long)m1 * M + m2, m1, m2, 0);
  for (int rb = 0; rb < 2 * M - 1; ++rb) {
    const int m1 = rb < M ? 0 : rb - M + 1, m2 = rb < M ? rb : 0;
    for (int m3 = 1; m3 < H; ++m3) put(nA + nC + (long long)rb * (H - 1) + m3 - 1, m1, m2, m3);
  }
  return K;
}

// Segment tables of the z-streamed leaf couple (k_couple_col): the leaf
// columns are cut into 2 x TY tiles; along z each tile is cut into runs of
// <= kColZS output slabs that hold at least one owned nonempty leaf.
// Per segment the 4 x (TY+2) input slots of its kColZS + 2 slabs
// (-1: empty or outside the domain).
constexpr int kColZS = 32;
void build_col_segments(blfmm_plan* p) {
  const int L = p->L;
  const LevelDev& leaf = p->lev[L];
  p->nseg = 0;
  if (!leaf.nbox) return;
  const int TX = 2, TY = 2, WX = TX + 2, WY = TY + 2, NI = WX * WY;
  const long long n = 1LL << L;
  std::vector<uint32_t> lk(leaf.nbox);
  CK(cudaMemcpy(lk.data(), leaf.key.p, sizeof(uint32_t) * leaf.nbox, cudaMemcpyDeviceToHost));
  std::vector<int> slot3((size_t)n * n * n, -1);
  auto at = [&](long long x, long long y, long long z) -> int {
    if (x < 0 || y < 0 || z < 0 || x >= n || y >= n || z >= n) return -1;
    return slot3[((size_t)x * n + y) * n + z];
  };
  for (long long a = 0; a < leaf.nbox; ++a) {
    int c[3];
    morton_decode<3>(lk[a], L, c);
    slot3[((size_t)c[0] * n + c[1]) * n + c[2]] = static_cast<int>(a);
  }
  const long long olo = p->own_lo[L], ohi = p->own_hi[L];
  struct Seg {
    int x0, y0, z0, nz, key;
  };
  std::vector<Seg> segs;
  for (long long x0 = 0; x0 < n; x0 += TX)
    for (long long y0 = 0; y0 < n; y0 += TY) {
      std::vector<char> out(n, 0);
      for (long long z = 0; z < n; ++z)
        for (int i = 0; i < TX; ++i)
          for (int j = 0; j < TY; ++j) {
            const int b = at(x0 + i, y0 + j, z);
            if (b >= olo && b < ohi) out[z] = 1;
          }
      for (long long z0 = 0; z0 < n;) {
        if (!out[z0]) {
          ++z0;
          continue;
        }
        // a run of kColZS slabs starting at the first slab with an output,
        // trimmed to its last output slab
        long long z1 = std::min(n, z0 + kColZS), last = z0;
        for (long long z = z0; z < z1; ++z)
          if (out[z]) last = z;
        int first = -1;
        for (int i = 0; i < TX && first < 0; ++i)
          for (int j = 0; j < TY && first < 0; ++j)
            for (long long z = z0; z <= last; ++z) {
              const int b = at(x0 + i, y0 + j, z);
              if (b >= 0) {
                first = first < 0 ? b : std::min(first, b);
              }
            }
        segs.push_back({(int)x0, (int)y0, (int)z0, (int)(last - z0 + 1), first});
        z0 = last + 1;
      }
    }
  // spatial (Morton) order of the segments' first leaf: neighbouring segments,
  // which re-read each other's halo boxes, run close in time (L2 reuse)
  std::stable_sort(segs.begin(), segs.end(),
                   [](const Seg& a, const Seg& b) { return a.key < b.key; });
  p->nseg = static_cast<long long>(segs.size());
  std::vector<int4> hdr(std::max<size_t>(segs.size(), 1));
  std::vector<int> tab(std::max<size_t>(segs.size(), 1) * (kColZS + 2) * NI, -1);
  for (size_t q = 0; q < segs.size(); ++q) {
    const Seg& g = segs[q];
    hdr[q] = make_int4(g.x0, g.y0, g.z0, g.nz);
    for (int sl = 0; sl < g.nz + 2; ++sl)
      for (int i = 0; i < WX; ++i)
        for (int j = 0; j < WY; ++j)
          tab[(q * (kColZS + 2) + sl) * NI + i * WY + j] =
              at(g.x0 - 1 + i, g.y0 - 1 + j, g.z0 - 1 + sl);
  }
  upload(p->seg_hdr, hdr);
  upload(p->seg_slot, tab);
}

// Per-level phase tables. Shared grids: every level uses the leaf nodes xi.
// Scaled grids: level l uses xi^l = -sigma_l + m dxi_l; m2m_tab[l] (child
// level l -> parent) is built on the PARENT grid (mlfmm.cpp:262), l2l_tab[l]
// (parent -> child level l) and m2l_tab[l] on grid l (mlfmm.cpp:293, 336).
void build_tables(blfmm_plan* p, const std::vector<double>& xi) {
  const int M = p->M, L = p->L;
  std::vector<double2> m2m((size_t)(L + 1) * 3 * 2 * M), m2l((size_t)(L + 1) * 3 * 7 * M),
      l2l((size_t)(L + 1) * 3 * 2 * M);
  auto level_xi = [&](int l, int m) {
    if (!p->scaled) return xi[m];
    const int ll = std::max(l, 2);
    const double sg = p->sig[ll];
    return -sg + m * (2.0 * sg / M);
  };
  for (int l = 0; l <= L; ++l)
    for (int k = 0; k < 3; ++k) {
      double h = (p->hi[k] - p->lo[k]) / static_cast<double>(1LL << l);
      for (int m = 0; m < M; ++m) {
        const double xl = level_xi(l, m), xp = level_xi(l - 1, m);
        for (int delta = 0; delta < 2; ++delta) {
          std::complex<double> z = std::polar(1.0, xp * ((0.5 - delta) * h));
          m2m[(((size_t)l * 3 + k) * 2 + delta) * M + m] = make_double2(z.real(), z.imag());
          std::complex<double> y = std::polar(1.0, xl * ((0.5 - delta) * h));
          l2l[(((size_t)l * 3 + k) * 2 + delta) * M + m] = make_double2(y.real(), y.imag());
        }
        for (int o = -3; o <= 3; ++o) {
          std::complex<double> z = std::polar(1.0, xl * (-o * h));
          m2l[(((size_t)l * 3 + k) * 7 + o + 3) * M + m] = make_double2(z.real(), z.imag());
        }
      }
    }
  upload(p->m2m_tab, m2m);
  upload(p->m2l_tab, m2l);
  upload(p->l2l_tab, l2l);
  if (!p->scaled && p->d == 3) {
    // root_tab[k][i][m] = e^{i xi_m (x_{a,k} - x_{0,k})}, leaf index i
    // (x_a = lo + (i + 1/2) h_L, x_0 = the root centre)
    const long long nper = 1LL << L;
    std::vector<double2> rt((size_t)3 * nper * M);
    for (int k = 0; k < 3; ++k) {
      const double h = (p->hi[k] - p->lo[k]) / static_cast<double>(nper);
      const double half = 0.5 * (p->hi[k] - p->lo[k]);
      for (long long i = 0; i < nper; ++i)
        for (int m = 0; m < M; ++m) {
          std::complex<double> z = std::polar(1.0, xi[m] * ((i + 0.5) * h - half));
          rt[((size_t)k * nper + i) * M + m] = make_double2(z.real(), z.imag());
        }
    }
    upload(p->root_tab, rt);
  }
}

// Dense per-axis k-point Lagrange transfer from grid `src` to grid `tgt`
// nodes (lagrange_matrix, mlfmm.cpp:42-80: window of the k nodes nearest the
// target, then the classical product formula), row-major [tgt][src].
std::vector<double> lagrange_dense(const std::vector<double>& src, const std::vector<double>& tgt,
                                   int k) {
  const int n = static_cast<int>(src.size()), rows = static_cast<int>(tgt.size());
  if (k < 1 || k > n) throw Error(BLFMM_EINVAL, "stencil size out of range");
  std::vector<double> P((size_t)rows * n, 0.0);
  for (int r = 0; r < rows; ++r) {
    const double t = tgt[r];
    int lo = static_cast<int>(std::lower_bound(src.begin(), src.end(), t) - src.begin()) - k / 2;
    lo = std::min(std::max(lo, 0), n - k);
    while (lo > 0 && t - src[lo - 1] < src[lo + k - 1] - t) --lo;
    while (lo + k < n && src[lo + k] - t < t - src[lo]) ++lo;
    for (int j = 0; j < k; ++j) {
      double w = 1.0;
      for (int q = 0; q < k; ++q) {
        if (q == j) continue;
        w *= (t - src[lo + q]) / (src[lo + j] - src[lo + q]);
      }
      P[(size_t)r * n + lo + j] = w;
    }
  }
  return P;
}

template <int D>
void plan_build_tree(blfmm_plan* p, const double* coords_host) {
  const long long n = p->n;
  const int L = p->L;
  cudaStream_t st = p->stream;
  DevBuf xin, keys, idx, skeys;
  xin.alloc(sizeof(double) * n * D);
  if (n) CK(cudaMemcpyAsync(xin.p, coords_host, sizeof(double) * n * D, cudaMemcpyHostToDevice, st));
  keys.alloc(sizeof(uint32_t) * std::max<long long>(n, 1));
  idx.alloc(sizeof(int) * std::max<long long>(n, 1));
  skeys.alloc(sizeof(uint32_t) * std::max<long long>(n, 1));
  p->perm.alloc(sizeof(int) * std::max<long long>(n, 1));
  double side[3];
  for (int k = 0; k < 3; ++k) side[k] = (p->hi[k] - p->lo[k]) / static_cast<double>(1LL << L);
  if (n) {
    k_bin<D><<<blocks_for(n, 256), 256, 0, st>>>(xin.as<double>(), n, L, p->lo[0], p->lo[1],
                                                 p->lo[2], side[0], side[1], side[2],
                                                 keys.as<uint32_t>(), idx.as<int>());
    CK(cudaGetLastError());
    cub_call(p->scratch, st, [&](void* tmp, size_t& bytes) {
      return cub::DeviceRadixSort::SortPairs(tmp, bytes, keys.as<uint32_t>(), skeys.as<uint32_t>(),
                                             idx.as<int>(), p->perm.as<int>(), (int)n, 0,
                                             std::max(1, D * L), st);
    });
  }
  for (int k = 0; k < 3; ++k) p->xs[k].alloc(k < D ? sizeof(double) * std::max<long long>(n, 1) : 0);
  if (n) {
    k_gather_coords<D><<<blocks_for(n, 256), 256, 0, st>>>(
        xin.as<double>(), p->perm.as<int>(), n, p->xs[0].as<double>(),
        D > 1 ? p->xs[1].as<double>() : nullptr, D > 2 ? p->xs[2].as<double>() : nullptr);
    CK(cudaGetLastError());
  }
  // Leaf level: run-length encode the sorted keys.
  DevBuf nruns, counts;
  nruns.alloc(sizeof(int));
  counts.alloc(sizeof(int) * (std::max<long long>(n, 1) + 1));
  LevelDev& leaf = p->lev[L];
  leaf.key.alloc(sizeof(uint32_t) * std::max<long long>(n, 1));
  int hruns = 0;
  if (n) {
    cub_call(p->scratch, st, [&](void* tmp, size_t& bytes) {
      return cub::DeviceRunLengthEncode::Encode(tmp, bytes, skeys.as<uint32_t>(),
                                                leaf.key.as<uint32_t>(), counts.as<int>(),
                                                nruns.as<int>(), (int)n, st);
    });
    CK(cudaMemcpyAsync(&hruns, nruns.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  }
  leaf.nbox = hruns;
  p->leaf_start.alloc(sizeof(int) * (hruns + 1));
  if (hruns) {
    CK(cudaMemsetAsync(counts.as<int>() + hruns, 0, sizeof(int), st));
    cub_call(p->scratch, st, [&](void* tmp, size_t& bytes) {
      return cub::DeviceScan::ExclusiveSum(tmp, bytes, counts.as<int>(), p->leaf_start.as<int>(),
                                           hruns + 1, st);
    });
  } else {
    CK(cudaMemsetAsync(p->leaf_start.p, 0, sizeof(int), st));
  }
  // Coarser levels: parent key = child key >> d.
  DevBuf shifted;
  shifted.alloc(sizeof(uint32_t) * std::max<long long>(hruns, 1));
  for (int l = L - 1; l >= 0; --l) {
    LevelDev& ch = p->lev[l + 1];
    LevelDev& pa = p->lev[l];
    long long nc = ch.nbox;
    pa.key.alloc(sizeof(uint32_t) * std::max<long long>(nc, 1));
    int np = 0;
    if (nc) {
      k_shift_keys<<<blocks_for(nc, 256), 256, 0, st>>>(ch.key.as<uint32_t>(), nc, D,
                                                         shifted.as<uint32_t>());
      cub_call(p->scratch, st, [&](void* tmp, size_t& bytes) {
        return cub::DeviceRunLengthEncode::Encode(tmp, bytes, shifted.as<uint32_t>(),
                                                  pa.key.as<uint32_t>(), counts.as<int>(),
                                                  nruns.as<int>(), (int)nc, st);
      });
      CK(cudaMemcpyAsync(&np, nruns.p, sizeof(int), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
    }
    pa.nbox = np;
    pa.child_start.alloc(sizeof(int) * (np + 1));
    ch.parent.alloc(sizeof(int) * std::max<long long>(nc, 1));
    if (np) {
      CK(cudaMemsetAsync(counts.as<int>() + np, 0, sizeof(int), st));
      cub_call(p->scratch, st, [&](void* tmp, size_t& bytes) {
        return cub::DeviceScan::ExclusiveSum(tmp, bytes, counts.as<int>(),
                                             pa.child_start.as<int>(), np + 1, st);
      });
      k_fill_parent<<<blocks_for(np, 256), 256, 0, st>>>(pa.child_start.as<int>(), np,
                                                          ch.parent.as<int>());
      CK(cudaGetLastError());
    }
  }
  // Dense slot maps (levels 1..L; level 0 is the root).
  for (int l = 1; l <= L; ++l) {
    LevelDev& lv = p->lev[l];
    long long cnt = 1LL << (D * l);
    lv.slotmap.alloc(sizeof(int) * cnt);
    CK(cudaMemsetAsync(lv.slotmap.p, 0xFF, sizeof(int) * cnt, st));
    if (lv.nbox)
      k_slotmap<D><<<blocks_for(lv.nbox, 256), 256, 0, st>>>(lv.key.as<uint32_t>(), lv.nbox, l,
                                                             lv.slotmap.as<int>());
    CK(cudaGetLastError());
  }
  // couple region tables (level l, grouped by parent at level l-1)
  for (int l = 1; l <= L; ++l) {
    LevelDev& lv = p->lev[l];
    const LevelDev& pa = p->lev[l - 1];
    constexpr int REG = D == 3 ? 64 : (D == 2 ? 16 : 4);
    lv.region.alloc(sizeof(int) * std::max<long long>(pa.nbox * REG, 1));
    if (pa.nbox)
      k_region_slots<D><<<blocks_for(pa.nbox * REG, 256), 256, 0, st>>>(
          pa.key.as<uint32_t>(), pa.nbox, l, lv.slotmap.as<int>(), lv.region.as<int>());
    CK(cudaGetLastError());
  }
  // Pair statistics.
  DevBuf acc, leaf_src;
  acc.alloc(sizeof(unsigned long long) * 2);
  leaf_src.alloc(sizeof(long long) * std::max<long long>(leaf.nbox, 1));
  CK(cudaMemsetAsync(acc.p, 0, acc.bytes, st));
  if (leaf.nbox)
    k_pair_counts<D><<<blocks_for(leaf.nbox, 128), 128, 0, st>>>(
        leaf.key.as<uint32_t>(), leaf.slotmap.as<int>(), p->leaf_start.as<int>(), leaf.nbox, L,
        acc.as<unsigned long long>(), leaf_src.as<long long>());
  // Near-field work list: (leaf, first target) per chunk of 32 targets,
  // heaviest (most sources) first.
  {
    std::vector<long long> hsrc(leaf.nbox);
    std::vector<int> hstart(leaf.nbox + 1);
    if (leaf.nbox) {
      CK(cudaMemcpyAsync(hsrc.data(), leaf_src.p, sizeof(long long) * leaf.nbox,
                         cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(hstart.data(), p->leaf_start.p, sizeof(int) * (leaf.nbox + 1),
                         cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
    }
    // Morton-range sharding (multi-GPU): leaves split into `world`
    // contiguous ranges of equal estimated cost (near pairs + per-point
    // expansion work + per-box translation work); this plan owns one range.
    long long la = 0, lb = leaf.nbox;
    if (p->world > 1 && leaf.nbox) {
      std::vector<double> cost(leaf.nbox);
      for (long long a = 0; a < leaf.nbox; ++a) {
        const double s_a = hstart[a + 1] - hstart[a];
        // calibrated on the P3 kernels (units of one near-field pair): near
        // pairs + P2M/L2P per point (1.1 K_s) + the leaf's share of the
        // translations (19 K_s), K_s = stored nodes per expansion
        const double ks = static_cast<double>(p->Ks);
        cost[a] = s_a * hsrc[a] + 1.1 * s_a * ks + 19.0 * ks;
      }
      std::vector<long long> bounds(p->world + 1);
      partition_ranges(cost.data(), leaf.nbox, p->world, bounds.data());
      la = bounds[p->rank];
      lb = bounds[p->rank + 1];
      p->pt_bounds.resize(p->world + 1);
      for (int q = 0; q <= p->world; ++q) p->pt_bounds[q] = hstart[bounds[q]];
    }
    p->own_lo[L] = la;
    p->own_hi[L] = lb;
    p->own_pt_lo = leaf.nbox ? hstart[la] : 0;
    p->own_pt_hi = leaf.nbox ? hstart[lb] : 0;
    long long own_pairs = 0;
    for (long long a = la; a < lb; ++a) own_pairs += (long long)(hstart[a + 1] - hstart[a]) * hsrc[a];
    p->own_near_pairs = own_pairs;
    // owned box range of every coarser level: the ancestors of leaves la..lb-1
    // (contiguous in Morton order)
    {
      std::vector<uint32_t> lk(leaf.nbox);
      if (leaf.nbox)
        CK(cudaMemcpy(lk.data(), leaf.key.p, sizeof(uint32_t) * leaf.nbox, cudaMemcpyDeviceToHost));
      for (int l = L - 1; l >= 0; --l) {
        const LevelDev& lv = p->lev[l];
        std::vector<uint32_t> kk(lv.nbox);
        if (lv.nbox)
          CK(cudaMemcpy(kk.data(), lv.key.p, sizeof(uint32_t) * lv.nbox, cudaMemcpyDeviceToHost));
        if (la >= lb) {
          p->own_lo[l] = p->own_hi[l] = 0;
          continue;
        }
        const int sh = D * (L - l);
        const uint32_t k0 = lk[la] >> sh, k1 = lk[lb - 1] >> sh;
        p->own_lo[l] = std::lower_bound(kk.begin(), kk.end(), k0) - kk.begin();
        p->own_hi[l] = (std::lower_bound(kk.begin(), kk.end(), k1) - kk.begin()) + 1;
      }
    }
    for (long long a = 0; a < leaf.nbox; ++a)
      p->max_leaf_pts = std::max(p->max_leaf_pts, hstart[a + 1] - hstart[a]);
    // Leaves whose 3^d neighbourhood holds EVERY point: their interaction lists
    // are empty at every level and the reference's far field there is an exact
    // zero. The neighbourhood-difference sweep would leave
    // eps |C| |NS| instead, which the pole cell of a singular spectrum (MQ:
    // |C| ~ 1e8 / dxi, the 1e-8 pole ball) lifts above the parity bar when
    // nothing else contributes; their locals are zeroed before L2P.
    {
      std::vector<int> zf;
      if (leaf.nbox <= (D == 1 ? 3 : (D == 2 ? 9 : 27)))
        for (long long a = 0; a < leaf.nbox; ++a)
          if (hsrc[a] == n) zf.push_back(static_cast<int>(a));
      p->n_zero_far = static_cast<long long>(zf.size());
      if (!zf.empty()) upload(p->zero_far, zf);
    }
    // batched right-hand sides: (leaf, first target) per chunk of 32 targets,
    // heaviest (most sources) first
    if (p->R > 1) {
      std::vector<std::pair<long long, int2>> items;
      for (long long a = la; a < lb; ++a)
        for (int t = hstart[a]; t < hstart[a + 1]; t += 32)
          items.push_back({-hsrc[a] * std::min(32, hstart[a + 1] - t), make_int2((int)a, t)});
      std::stable_sort(items.begin(), items.end(),
                       [](const auto& u, const auto& v) { return u.first < v.first; });
      std::vector<int2> w(items.size());
      for (size_t q = 0; q < items.size(); ++q) w[q] = items[q].second;
      upload(p->near_work, w);
      p->nwork = static_cast<long long>(w.size());
    }
    // one right-hand side: symmetric items for neighbouring leaves that both
    // hold >= near_sym_min points (per-leaf neighbour masks, the pair list,
    // and the sources each leaf's one-sided items still see), then one-sided
    // items of up to 96 targets; one queue, heaviest first within each kind
    std::vector<long long> hsrc1(hsrc);
    constexpr int TOT = D == 1 ? 3 : (D == 2 ? 9 : 27);
    if (p->R == 1 && p->near_sym_min > 0 && leaf.nbox) {
      const int T = p->near_sym_min;
      std::vector<uint32_t> lkey(leaf.nbox);
      CK(cudaMemcpy(lkey.data(), leaf.key.p, sizeof(uint32_t) * leaf.nbox, cudaMemcpyDeviceToHost));
      const int nper = 1 << L;
      auto npts = [&](long long a) { return hstart[a + 1] - hstart[a]; };
      std::vector<uint32_t> lmask(leaf.nbox, 0u);
      std::vector<std::pair<long long, int4>> sitems;
      for (long long a = 0; a < leaf.nbox; ++a) {
        if (npts(a) < T) continue;
        int c[3], b[3];
        morton_decode<D>(lkey[a], L, c);
        for (int q = 0; q < TOT; ++q) {
          if (q == TOT / 2) continue;  // the leaf itself
          bool ok = true;
          int rr = q;
          for (int k = D - 1; k >= 0; --k) {
            b[k] = c[k] + rr % 3 - 1;
            rr /= 3;
            ok = ok && b[k] >= 0 && b[k] < nper;
          }
          if (!ok) continue;
          const uint32_t kb = morton_encode<D>(b, L);
          const auto itb = std::lower_bound(lkey.begin(), lkey.end(), kb);
          if (itb == lkey.end() || *itb != kb) continue;
          const long long bs = itb - lkey.begin();
          if (npts(bs) < T) continue;
          lmask[a] |= 1u << q;
          hsrc1[a] -= npts(bs);
          if (q < TOT / 2) continue;  // each unordered pair once (forward half)
          // target side = the leaf whose lane rows (32 NT targets per warp
          // pass, NT <= 3) waste fewer slots; ties: the larger, then the lower slot
          auto slots = [&](long long nt, long long ns) {
            const long long per = nt > 64 ? 96 : (nt > 32 ? 64 : 32);
            return ((nt + per - 1) / per) * per * ns;
          };
          const long long sa = slots(npts(a), npts(bs)), sb = slots(npts(bs), npts(a));
          const bool ta = sa < sb || (sa == sb && (npts(a) > npts(bs) ||
                                                   (npts(a) == npts(bs) && a < bs)));
          const long long tl = ta ? a : bs, sl = ta ? bs : a;
          const bool mine = p->world == 1 || (tl >= la && tl < lb) || (sl >= la && sl < lb);
          if (mine)
            sitems.push_back({-(long long)npts(a) * npts(bs),
                              make_int4((int)tl, (int)sl, ta ? q : TOT - 1 - q, 0)});
        }
      }
      std::stable_sort(sitems.begin(), sitems.end(),
                       [&](const auto& u, const auto& v) { return u.first < v.first; });
      // device items carry the point ranges (targets [x, y), sources [z, w))
      // and the target-side neighbour index separately
      std::vector<int4> sw(sitems.size());
      std::vector<unsigned char> sqv(sitems.size());
      for (size_t q = 0; q < sitems.size(); ++q) {
        const int4 s = sitems[q].second;
        sw[q] = make_int4(hstart[s.x], hstart[s.x + 1], hstart[s.y], hstart[s.y + 1]);
        sqv[q] = static_cast<unsigned char>(s.z);
      }
      p->nsym = static_cast<long long>(sw.size());
      bool any = false;
      for (long long a = 0; a < leaf.nbox && !any; ++a) any = lmask[a] != 0;
      if (any) {
        upload(p->sym_work, sw);
        upload(p->sym_q, sqv);
        std::vector<unsigned> pm(n);
        for (long long a = 0; a < leaf.nbox; ++a)
          for (int i = hstart[a]; i < hstart[a + 1]; ++i) pm[i] = lmask[a];
        upload(p->sym_pmask, pm);
        p->sym_planes.alloc(sizeof(double) * TOT * std::max<long long>(n, 1));
      } else {
        p->near_sym_min = 0;
        p->nsym = 0;
      }
    } else {
      p->near_sym_min = 0;
    }
    if (p->R == 1) {
      std::vector<std::pair<long long, int2>> items2;
      for (long long a = la; a < lb; ++a)
        for (int t = hstart[a]; t < hstart[a + 1];) {
          const int cnt = std::min(kNearItemMax, hstart[a + 1] - t);
          items2.push_back({-hsrc1[a] * cnt, make_int2((int)a, t)});
          t += cnt;
        }
      std::stable_sort(items2.begin(), items2.end(),
                       [](const auto& u, const auto& v) { return u.first < v.first; });
      std::vector<int2> w(items2.size());
      for (size_t q = 0; q < items2.size(); ++q) w[q] = items2[q].second;
      upload(p->near_work2, w);
      p->nwork2 = static_cast<long long>(w.size());
      p->near_ctr.alloc(sizeof(unsigned long long));
    }
    // (leaf, 8-point tile) items for the DMMA L2P, heaviest leaves first
    std::vector<int2> w8;
    std::vector<long long> order;
    for (long long a = la; a < lb; ++a) order.push_back(a);
    std::stable_sort(order.begin(), order.end(), [&](long long u, long long v) {
      return hstart[u + 1] - hstart[u] > hstart[v + 1] - hstart[v];
    });
    for (long long a : order)
      for (int t = hstart[a]; t < hstart[a + 1]; t += 8) w8.push_back(make_int2((int)a, t));
    upload(p->work8, w8);
    p->nwork8 = static_cast<long long>(w8.size());
    std::vector<int2> w128;
    for (long long a : order)
      for (int t = hstart[a]; t < hstart[a + 1]; t += kL2PSpan) w128.push_back(make_int2((int)a, t));
    upload(p->work128, w128);
    p->nwork128 = static_cast<long long>(w128.size());
    std::vector<int2> w64;
    for (long long a : order)
      for (int t = hstart[a]; t < hstart[a + 1]; t += kMRSpan) w64.push_back(make_int2((int)a, t));
    upload(p->work64, w64);
    p->nwork64 = static_cast<long long>(w64.size());
    // block-A L2P of the general half spectrum (k_l2p_half_a3): spans of up to
    // 64 points in classes of 2, 4, 6, 8 point tiles (heaviest leaves first
    // inside a class)
    {
      std::vector<int4> wc[4];  // (leaf, first point, end point, -)
      const int cap = 64;
      for (long long a : order) {
        // a leaf's points in equal spans of whole tiles (70 points, cap 64: 40 + 30)
        const int cnt = hstart[a + 1] - hstart[a];
        const int nsp = (cnt + cap - 1) / cap;
        const int len = nsp ? ((cnt + nsp - 1) / nsp + 7) / 8 * 8 : 0;
        for (int t = hstart[a]; t < hstart[a + 1]; t += len) {
          const int end = std::min(t + len, hstart[a + 1]);
          wc[((end - t + 7) / 8 - 1) / 2].push_back(make_int4((int)a, t, end, 0));
        }
      }
      std::vector<int4> all;
      for (int c = 0; c < 4; ++c) {
        p->nwork_ha[c] = static_cast<long long>(wc[c].size());
        all.insert(all.end(), wc[c].begin(), wc[c].end());
      }
      upload(p->work_ha, all);
    }
    // parents of the leaves (level L-1) by decreasing point count: the fused
    // P2M + leaf-M2M kernel's work list
    if (L >= 2 && p->lev[L - 1].nbox) {
      const LevelDev& pl = p->lev[L - 1];
      std::vector<int> cs(pl.nbox + 1);
      CK(cudaMemcpy(cs.data(), pl.child_start.p, sizeof(int) * cs.size(), cudaMemcpyDeviceToHost));
      std::vector<long long> pts(pl.nbox);
      std::vector<int> plist(pl.nbox);
      for (long long q = 0; q < pl.nbox; ++q) {
        pts[q] = hstart[cs[q + 1]] - hstart[cs[q]];
        plist[q] = static_cast<int>(q);
      }
      std::stable_sort(plist.begin(), plist.end(), [&](int u, int v) { return pts[u] > pts[v]; });
      upload(p->p2m_plist, plist);
      p->n_p2m_plist = pl.nbox;
    }
  }
  unsigned long long hacc[2] = {0, 0};
  CK(cudaMemcpyAsync(hacc, acc.p, sizeof(hacc), cudaMemcpyDeviceToHost, st));
  DevBuf il;
  il.alloc(sizeof(unsigned long long));
  CK(cudaMemsetAsync(il.p, 0, il.bytes, st));
  for (int l = 2; l <= L; ++l)
    if (p->lev[l].nbox)
      k_il_pairs<D><<<blocks_for(p->lev[l].nbox, 128), 128, 0, st>>>(
          p->lev[l].key.as<uint32_t>(), p->lev[l].slotmap.as<int>(), p->lev[l].nbox, l,
          il.as<unsigned long long>());
  unsigned long long hil = 0;
  CK(cudaMemcpyAsync(&hil, il.p, sizeof(hil), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  CK(cudaGetLastError());
  p->info.near_pairs = static_cast<long long>(hacc[0]);
  long long nleaf = leaf.nbox;
  // fmm.cpp:152,179,209: 2 N K + (sum over nonempty a of nonempty non-neighbors) K
  p->info.far_work_single =
      2LL * n * p->K + (nleaf * nleaf - static_cast<long long>(hacc[1])) * p->K;
  p->info.il_pairs = static_cast<long long>(hil);
}

// Contiguous ranges of (approximately) equal total cost: bounds[0..world],
// bounds[r] = first index whose cost prefix reaches r/world of the total.
void partition_ranges(const double* cost, long long n, int world, long long* bounds) {
  double total = 0.0;
  for (long long i = 0; i < n; ++i) total += cost[i];
  bounds[0] = 0;
  long long i = 0;
  double pre = 0.0;
  for (int r = 1; r < world; ++r) {
    const double target = total * r / world;
    while (i < n && pre + 0.5 * cost[i] < target) pre += cost[i++];
    bounds[r] = i;
  }
  bounds[world] = n;
}

// sum_a |IL_l(a)| over the dense box set (factorises over the axes).
long long dense_il_sum(int d, int l) {
  long long n = 1LL << l, np = n / 2, s6 = 1, s3 = 1;
  for (int k = 0; k < d; ++k) {
    long long a6 = 0, a3 = 0;
    for (long long i = 0; i < n; ++i) {
      long long pi = i / 2;
      a6 += 2 * (std::min(np - 1, pi + 1) - std::max(0LL, pi - 1) + 1);
      a3 += std::min(n - 1, i + 1) - std::max(0LL, i - 1) + 1;
    }
    s6 *= a6;
    s3 *= a3;
  }
  return s6 - s3;
}

void create_plan(const blfmm_plan_desc* desc, const blfmm_tuning* tune, blfmm_plan** out) {
  if (!desc || !out) throw Error(BLFMM_EINVAL, "null descriptor or output");
  *out = nullptr;
  const int d = desc->d;
  if (d < 1 || d > 3) throw Error(BLFMM_EINVAL, "d must be 1, 2 or 3");
  if (desc->n < 0) throw Error(BLFMM_EINVAL, "n must be >= 0");
  if (desc->n > 0 && !desc->coords) throw Error(BLFMM_EINVAL, "request has no point set");
  if (desc->n > 2000000000LL) throw Error(BLFMM_EINVAL, "n exceeds 2^31 points");
  if (!(desc->sigma > 0.0)) throw Error(BLFMM_EINVAL, "sigma must be > 0");
  if (desc->m_per_dim < 2) throw Error(BLFMM_EINVAL, "m_per_dim must be >= 2");
  if (desc->leaf_level < 2) throw Error(BLFMM_EINVAL, "leaf_level must be >= 2");
  if (d * desc->leaf_level > 24) throw Error(BLFMM_EINVAL, "box count cap exceeded");
  if (desc->nrhs < 1) throw Error(BLFMM_EINVAL, "nrhs must be >= 1");
  if (desc->grid_mode != BLFMM_GRID_SHARED && desc->grid_mode != BLFMM_GRID_SCALED)
    throw Error(BLFMM_EINVAL, "unknown grid mode");
  if (desc->grid_mode == BLFMM_GRID_SCALED) {
    if (desc->world > 1)
      throw Error(BLFMM_EDOMAIN, "scaled grids are single-GPU on this path");
    long long kk = 1;
    for (int q = 0; q < d; ++q) kk *= desc->m_per_dim;
    if (kk > kScaledMaxK)
      throw Error(BLFMM_EDOMAIN, "scaled grids need M^d <= 6400 (shared-memory transfers)");
    if (desc->stencil_k < 1) throw Error(BLFMM_EINVAL, "stencil size out of range");
  }
  const int world = desc->world < 1 ? 1 : desc->world;
  if (desc->rank < 0 || desc->rank >= world) throw Error(BLFMM_EINVAL, "rank out of range");
  KernelSpec k{desc->kernel_type, desc->kernel_shape};
  if (!(k.shape > 0.0) || !std::isfinite(k.shape))
    throw Error(BLFMM_EINVAL, "kernel parameter must be positive");
  require_fmm_kernel(k);
  for (int q = 0; q < d; ++q)
    if (!(desc->domain_hi[q] > desc->domain_lo[q]))
      throw Error(BLFMM_EINVAL, "domain must have hi > lo on every axis");
  long long K = 1;
  for (int q = 0; q < d; ++q) K *= desc->m_per_dim;

  auto t0 = std::chrono::steady_clock::now();
  DeviceGuard guard(desc->device);
  std::unique_ptr<blfmm_plan> p(new blfmm_plan());
#ifdef BLFMM_DEV_KNOBS
  for (int i = 0; i < 4; ++i) {
    const std::string nm = "BLFMM_XP" + std::to_string(i);
    if (const char* e = std::getenv(nm.c_str())) p->xp[i] = std::atoi(e);
  }
#endif
  CK(cudaGetDevice(&p->device));
  CK(cudaDeviceGetAttribute(&p->num_sms, cudaDevAttrMultiProcessorCount, p->device));
  // Deep 3-D trees (leaf level >= 6, one right-hand side): the register-bound
  // leaf couple dominates the step, so the co-running near field is capped at 2
  // CTAs of 80 registers per SM (P3: 5.576 vs 5.707 ms). Shallower trees keep 3
  // CTAs of up to 128 registers (P2p 1.11 vs 1.63 ms, P4 11.07 vs 12.21 ms).
  if (!(d == 3 && desc->leaf_level >= 6 && desc->nrhs <= 1)) {
    p->near_minb = 1;
    p->near_persist = 3;
  }
  if (tune) {
    if (tune->telescope >= 0) p->telescope = tune->telescope != 0;
    if (tune->graphs >= 0) p->use_graphs = tune->graphs != 0;
    if (tune->near_sym_min >= 0) p->near_sym_min = tune->near_sym_min;
    if (tune->near_ctas_per_sm > 0) p->near_persist = std::min(tune->near_ctas_per_sm, 8);
    if (tune->near_reg_cap == 80) p->near_minb = 6;
    else if (tune->near_reg_cap > 0) p->near_minb = 1;
  }
  p->d = d;
  p->rank = desc->world > 1 ? desc->rank : 0;
  p->world = desc->world > 1 ? desc->world : 1;
  p->n = desc->n;
  p->M = desc->m_per_dim;
  p->L = desc->leaf_level;
  p->R = desc->nrhs;
  p->K = K;
  p->kern = k;
  p->sigma = desc->sigma;
  for (int q = 0; q < 3; ++q) {
    p->lo[q] = q < d ? desc->domain_lo[q] : 0.0;
    p->hi[q] = q < d ? desc->domain_hi[q] : 1.0;
  }
  const double dxi = 2.0 * p->sigma / p->M;
  p->weight = d == 1 ? dxi : (d == 2 ? dxi * dxi : dxi * dxi * dxi);
  CK(cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking));
  for (auto& e : p->ev) CK(cudaEventCreate(&e));
  for (auto& e : p->ev_near) CK(cudaEventCreate(&e));
  CK(cudaEventCreateWithFlags(&p->fence_in, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&p->fence_out, cudaEventDisableTiming));
  {
    int lo_prio = 0, hi_prio = 0;
    CK(cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio));
    // higher priority: its CTAs interleave with the far-field grids
    CK(cudaStreamCreateWithPriority(&p->stream_near, cudaStreamNonBlocking, hi_prio));
  }
  CK(cudaEventCreateWithFlags(&p->fork, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&p->join, cudaEventDisableTiming));
  if (tune && tune->couple_tile >= 0 && tune->couple_tile <= 1) p->couple_var = tune->couple_tile;

  std::vector<double> xi(p->M);
  for (int m = 0; m < p->M; ++m) xi[m] = -p->sigma + m * dxi;
  upload(p->xi, xi);
  p->scaled = desc->grid_mode == BLFMM_GRID_SCALED;
  p->stencil = std::min(desc->stencil_k, p->M);
  p->sig.assign(p->L + 1, p->sigma);
  if (p->scaled)
    for (int l = p->L - 1; l >= 0; --l) p->sig[l] = p->sig[l + 1] / 2.0;
  std::vector<double> c;
  if (p->scaled) {
    // one C table per level 2..L (desc->c_table, if given, holds them in order)
    c.assign((size_t)(p->L + 1) * K, 0.0);
    for (int l = 2; l <= p->L; ++l) {
      std::vector<double> cl =
          desc->c_table ? std::vector<double>(desc->c_table + (size_t)(l - 2) * K,
                                              desc->c_table + (size_t)(l - 1) * K)
                        : translation_spectrum(k, p->sig[l], p->M, d);
      std::copy(cl.begin(), cl.end(), c.begin() + (size_t)l * K);
    }
    std::vector<double> P((size_t)(p->L + 1) * p->M * p->M, 0.0);
    auto nodes = [&](int l) {
      std::vector<double> v(p->M);
      for (int m = 0; m < p->M; ++m) v[m] = -p->sig[l] + m * (2.0 * p->sig[l] / p->M);
      return v;
    };
    // CSR form: row r of P[l] holds the k consecutive sources lo .. lo+k-1
    std::vector<int> plo((size_t)(p->L + 1) * p->M, 0);
    std::vector<double> pw((size_t)(p->L + 1) * p->M * p->stencil, 0.0);
    for (int l = 3; l <= p->L; ++l) {
      std::vector<double> Pl = lagrange_dense(nodes(l), nodes(l - 1), p->stencil);
      std::copy(Pl.begin(), Pl.end(), P.begin() + (size_t)l * p->M * p->M);
      for (int r = 0; r < p->M; ++r) {
        int lo = 0;
        while (lo < p->M && Pl[(size_t)r * p->M + lo] == 0.0) ++lo;
        lo = std::min(lo, p->M - p->stencil);
        plo[(size_t)l * p->M + r] = lo;
        for (int j = 0; j < p->stencil; ++j)
          pw[((size_t)l * p->M + r) * p->stencil + j] = Pl[(size_t)r * p->M + lo + j];
      }
    }
    // transpose CSR: column c of P[l] -> rows r with P[r][c] != 0 (padded)
    int kt = 1;
    for (int l = 3; l <= p->L; ++l)
      for (int c = 0; c < p->M; ++c) {
        int cnt = 0;
        for (int r = 0; r < p->M; ++r) cnt += P[((size_t)l * p->M + r) * p->M + c] != 0.0;
        kt = std::max(kt, cnt);
      }
    std::vector<int> ptr((size_t)(p->L + 1) * p->M * kt, 0);
    std::vector<double> ptw((size_t)(p->L + 1) * p->M * kt, 0.0);
    for (int l = 3; l <= p->L; ++l)
      for (int c = 0; c < p->M; ++c) {
        int j = 0;
        for (int r = 0; r < p->M; ++r) {
          const double w = P[((size_t)l * p->M + r) * p->M + c];
          if (w == 0.0) continue;
          ptr[((size_t)l * p->M + c) * kt + j] = r;
          ptw[((size_t)l * p->M + c) * kt + j] = w;
          ++j;
        }
      }
    p->kt = kt;
    upload(p->ptab, P);
    upload(p->plo_tab, plo);
    upload(p->pw_tab, pw);
    upload(p->ptr_tab, ptr);
    upload(p->ptw_tab, ptw);
  } else {
    c = desc->c_table ? std::vector<double>(desc->c_table, desc->c_table + K)
                      : translation_spectrum(k, p->sigma, p->M, d);
  }
  p->Ks = K;
  // half spectrum: 3-D shared grids, even M in [16, 64] (M = 16: the tiled
  // k_*_h16* kernels; otherwise block GEMMs, k_halfm.inc.cuh)
  p->herm = d == 3 && !p->scaled && p->M % 2 == 0 && p->M >= 16 && p->M <= 64 &&
            !(tune && tune->half_spectrum == 0);
  p->h16 = p->herm && p->M == 16;
  p->mr = p->h16 && p->R >= 8 && !(tune && tune->rhs_gemm == 0);
  if (p->herm) {
    std::vector<double> dt;
    p->hK = build_half(c, p->M, p->node_host, p->c_st, dt);
    p->Ks = static_cast<long long>(p->node_host.size());
    upload(p->node_m, p->node_host);
    upload(p->dtab, dt);
    upload(p->ctab, p->c_st);
  } else {
    upload(p->ctab, c);
  }
  p->c_full = c;
  const long long Ks = p->Ks;
  build_tables(p.get(), xi);

  if (d == 1) plan_build_tree<1>(p.get(), desc->coords);
  if (d == 2) plan_build_tree<2>(p.get(), desc->coords);
  if (d == 3) plan_build_tree<3>(p.get(), desc->coords);
  if (d == 3 && !p->scaled && p->couple_var > 0) build_col_segments(p.get());

  const long long n = p->n, R = p->R;
  for (int l = 1; l <= p->L; ++l)
    if (R * p->lev[l].nbox * Ks + Ks >= (1LL << 31))
      throw Error(BLFMM_EDOMAIN, "expansion set exceeds 2^31 coefficients per level "
                                 "(reduce nrhs, M or leaf level)");
  for (int l = 1; l <= p->L; ++l) {
    LevelDev& lv = p->lev[l];
    size_t bytes = sizeof(double2) * R * lv.nbox * Ks;
    // + one zero expansion after the last box: the couple kernel reads it for
    // empty / out-of-domain region boxes (unconditional loads)
    lv.mult.alloc(bytes + sizeof(double2) * Ks);
    CK(cudaMemset(static_cast<char*>(lv.mult.p) + bytes, 0, sizeof(double2) * Ks));
    if (l == p->L || (p->scaled && l >= 2)) lv.loc.alloc(bytes);
    else if (!p->scaled) lv.glob.alloc(bytes);
  }
  p->lam_in.alloc(sizeof(double) * R * std::max<long long>(n, 1));
  p->lam.alloc(sizeof(double) * R * std::max<long long>(n, 1));
  p->far_.alloc(sizeof(double) * R * std::max<long long>(n, 1));
  p->near_.alloc(sizeof(double) * R * std::max<long long>(n, 1));
  p->out.alloc(sizeof(double) * R * std::max<long long>(n, 1));
  p->src4.alloc(sizeof(double4) * std::max<long long>(n, 1));
  if (R > 1) p->lamT.alloc(sizeof(double) * R * std::max<long long>(n, 1));
  // plan-time per-point phase tables (P2M / L2P operands) for the kernels
  // that read them; 2-D M = 16 generates the phases in registers
  p->g2d16 = d == 2 && p->M == 16 && !p->scaled;
  if (d >= 2 && p->lev[p->L].nbox && !p->g2d16 && !p->mr) {
    p->pht.alloc(sizeof(double2) * n * d * p->M);
    double side[3];
    for (int q = 0; q < 3; ++q) side[q] = (p->hi[q] - p->lo[q]) / static_cast<double>(1LL << p->L);
    const LevelDev& leaf = p->lev[p->L];
    if (d == 2)
      k_point_phases<2><<<(unsigned)leaf.nbox, 256, 0, p->stream>>>(
          leaf.key.as<uint32_t>(), p->leaf_start.as<int>(), leaf.nbox, p->xs[0].as<double>(),
          p->xs[1].as<double>(), nullptr, p->xi.as<double>(), p->M, p->L, p->lo[0], p->lo[1],
          p->lo[2], side[0], side[1], side[2], p->pht.as<double2>());
    else
      k_point_phases<3><<<(unsigned)leaf.nbox, 256, 0, p->stream>>>(
          leaf.key.as<uint32_t>(), p->leaf_start.as<int>(), leaf.nbox, p->xs[0].as<double>(),
          p->xs[1].as<double>(), p->xs[2].as<double>(), p->xi.as<double>(), p->M, p->L,
          p->lo[0], p->lo[1], p->lo[2], side[0], side[1], side[2], p->pht.as<double2>());
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(p->stream));
  }
  p->imag_bits.alloc(sizeof(unsigned long long));
  if (p->herm && !p->h16) p->himag.alloc(sizeof(double) * R * std::max<long long>(n, 1));
  if (d == 3 && !p->scaled) p->root.alloc(sizeof(double2) * R * Ks);

  // multi-GPU exchange mode: halo sets and exchange-buffer layout
  if (p->world > 1 && p->L >= 3 && p->lev[p->L].nbox) {
    const int L = p->L;
    constexpr int REG3 = 64;
    const int REG = d == 3 ? REG3 : (d == 2 ? 16 : 4);
    const LevelDev& l2 = p->lev[L - 2];
    const LevelDev& l1 = p->lev[L - 1];
    std::vector<int> region((size_t)l2.nbox * REG), cs(l1.nbox + 1);
    CK(cudaMemcpy(region.data(), l1.region.p, sizeof(int) * region.size(), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(cs.data(), l1.child_start.p, sizeof(int) * cs.size(), cudaMemcpyDeviceToHost));
    // E_{L-1}: region boxes (level L-1) of the owned parents at level L-2
    std::vector<int> epar;
    for (long long q = p->own_lo[L - 2]; q < p->own_hi[L - 2]; ++q)
      for (int t = 0; t < REG; ++t)
        if (region[q * REG + t] >= 0) epar.push_back(region[q * REG + t]);
    std::sort(epar.begin(), epar.end());
    epar.erase(std::unique(epar.begin(), epar.end()), epar.end());
    // E_L: their children (covers every leaf-level region of owned parents)
    std::vector<int> eleaf;
    for (int c : epar)
      for (int a = cs[c]; a < cs[c + 1]; ++a) eleaf.push_back(a);
    upload(p->epar, epar);
    upload(p->eleaf, eleaf);
    p->n_epar = static_cast<long long>(epar.size());
    p->n_eleaf = static_cast<long long>(eleaf.size());
    const long long c1 = p->own_hi[L - 1] - p->own_lo[L - 1];
    p->own_l1.alloc(sizeof(double2) * R * std::max<long long>(c1, 1) * Ks);
    // telescoped downsweep: only V_1 (-> the root multipole)
    // is read above the leaf level, so only level 1 is exchanged (8 boxes);
    // levels 2..L-2 stay rank-local partials in the plan's own buffers
    p->xtele = d == 3 && p->telescope && !p->scaled && p->lev[1].nbox > 0;
    long long off = 0;
    for (int l = 1; l <= (p->xtele ? 1 : L - 2); ++l) {
      p->xoff[l] = off;
      off += (R * p->lev[l].nbox + 1) * Ks;  // + the zero expansion
    }
    p->xcount = off;
    p->xmode = true;
  }
  blfmm_plan_info& in = p->info;
  in.d = d;
  in.m_per_dim = p->M;
  in.leaf_level = p->L;
  in.nrhs = p->R;
  in.n = n;
  in.K = K;
  in.stored_nodes = p->Ks;
  in.telescoped = (d == 3 && p->telescope && !p->scaled && p->L >= 2 &&
                   p->lev[1].nbox > 0)
                      ? 1
                      : 0;
  for (int l = 0; l <= p->L; ++l) in.boxes[l] = p->lev[l].nbox;
  long long far = 2LL * n * K;
  for (int l = 2; l <= p->L; ++l) far += dense_il_sum(d, l) * K;
  in.far_work = far;
  in.owned_begin = p->own_pt_lo;
  in.owned_end = p->own_pt_hi;
  if (p->world > 1) in.near_pairs = p->own_near_pairs;
  size_t free_b = 0, total_b = 0;
  CK(cudaMemGetInfo(&free_b, &total_b));
  long long dev = 0;
  for (int l = 1; l <= p->L; ++l)
    dev += 2LL * p->lev[l].mult.bytes + p->lev[l].slotmap.bytes;
  in.device_bytes = dev + 5LL * sizeof(double) * R * n;
  in.near_sym_items = p->nsym;
  in.near_items = p->R == 1 ? p->nwork2 : p->nwork;
  {
    const bool tele = in.telescoped != 0;
    std::string k = "p2m=";
    if (d == 1) k += "k_p2m";
    else if (p->mr) k += "k_p2m_mr";
    else if (p->h16 && p->n_p2m_plist > 0) k += "k_p2m_m2m_h16";
    else if (p->h16) k += "k_p2m_h16w4";
    else if (p->herm) k += "k_p2m_big3+k_p2m_axes";
    else if (p->g2d16) k += "k_p2m_2d16";
    else if (d == 3 && p->M >= 24 && p->M <= 64 && !p->scaled) k += "k_p2m_big";
    else k += "k_p2m_mma";
    k += p->scaled ? (d == 3 ? " m2m=k_m2m_scaled3" : " m2m=k_m2m_scaled") : " m2m=k_m2m";
    if (p->scaled) k += d == 3 ? " couple=k_couple_scaled3+k_l2l_scaled3" : " couple=k_couple_scaled+k_l2l_scaled";
    else if (tele && p->couple_var == 0) k += " couple=k_root+k_couple3<ROOT>";
    else if (tele) {
      k += " couple=k_root+k_couple_col<2x2,z32>";
    }
    else k += d == 3 ? " couple=k_couple3" : " couple=k_couple";
    k += d == 1 ? " l2p=k_l2p"
                : (p->mr ? " l2p=k_l2p_mr"
                         : (p->h16 ? " l2p=k_l2p_h16S"
                                   : p->herm ? " l2p=k_l2p_axes+k_l2p_half_a3"
                                    : (p->g2d16 ? " l2p=k_l2p_2d16" : " l2p=k_l2p_mma")));
    if (p->R == 1)
      k += " near=k_near_all(ctas_per_sm=" + std::to_string(p->near_persist) +
           ",regcap=" + (p->near_minb == 6 ? std::string("80") : std::string("none")) +
           ",sym_min=" + std::to_string(p->near_sym_min) + ")";
    else
      k += (p->R % 2 == 0 && p->R >= 8) ? " near=k_near_dmma"
                                         : (p->R % 16 == 0 ? " near=k_near_warp_mr" : " near=k_near");
    p->kernels = k;
    std::snprintf(in.kernels, sizeof(in.kernels), "%s", k.c_str());
  }
  in.plan_seconds =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  *out = p.release();
}
