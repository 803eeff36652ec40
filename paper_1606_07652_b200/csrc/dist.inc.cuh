// Host: NCCL / caller collectives and the distributed matvec.
// Fragment of blfmm.cu (one translation unit): included inside
// namespace blfmm_gpu after the plan definition; not a standalone header.

// ------------------------------------------------ NCCL (loaded on first use)
struct NcclApi {
  bool tried = false, ok = false;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
  const char* (*errorString)(ncclResult_t) = nullptr;
};
NcclApi& nccl_api() {
  static NcclApi api;
  if (api.tried) return api;
  api.tried = true;
  // the process's libnccl.so.2 (torch's, if loaded) or the system one
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return api;
  auto sym = [&](auto& f, const char* name) {
    f = reinterpret_cast<std::remove_reference_t<decltype(f)>>(dlsym(h, name));
    return f != nullptr;
  };
  api.ok = sym(api.getUniqueId, "ncclGetUniqueId") && sym(api.commInitRank, "ncclCommInitRank") &&
           sym(api.commDestroy, "ncclCommDestroy") && sym(api.allReduce, "ncclAllReduce") &&
           sym(api.broadcast, "ncclBroadcast") && sym(api.groupStart, "ncclGroupStart") &&
           sym(api.groupEnd, "ncclGroupEnd") && sym(api.errorString, "ncclGetErrorString");
  return api;
}
NcclApi& nccl_required() {
  NcclApi& a = nccl_api();
  if (!a.ok) throw Error(BLFMM_ENCCL, "libnccl.so.2 not found or incomplete");
  return a;
}
void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw Error(BLFMM_ENCCL, std::string(what) + ": " + nccl_api().errorString(r));
}

void comm_sum(blfmm_plan* p, double* d, long long cnt) {
  if (cnt <= 0) return;
  if (p->comm_kind == 1) {
    nccl_check(nccl_api().allReduce(d, d, (size_t)cnt, ncclDouble, ncclSum,
                                    static_cast<ncclComm_t>(p->nccl), p->stream),
               "ncclAllReduce");
  } else if (p->ops.all_reduce_sum(p->ops.ctx, d, cnt, p->stream) != 0) {
    throw Error(BLFMM_ENCCL, "all_reduce_sum callback failed");
  }
}
void comm_max(blfmm_plan* p, double* d, long long cnt) {
  if (p->comm_kind == 1) {
    nccl_check(nccl_api().allReduce(d, d, (size_t)cnt, ncclDouble, ncclMax,
                                    static_cast<ncclComm_t>(p->nccl), p->stream),
               "ncclAllReduce(max)");
  } else if (p->ops.all_reduce_max(p->ops.ctx, d, cnt, p->stream) != 0) {
    throw Error(BLFMM_ENCCL, "all_reduce_max callback failed");
  }
}
// every rank's owned sorted slice of u (per right-hand side) to every rank
void comm_gather(blfmm_plan* p) {
  const long long n = p->n;
  double* us = p->usorted.as<double>();
  if (p->comm_kind == 1) {
    NcclApi& a = nccl_api();
    nccl_check(a.groupStart(), "ncclGroupStart");
    for (int q = 0; q < p->world; ++q) {
      const long long lo = p->pt_bounds[q], cnt = p->pt_bounds[q + 1] - lo;
      if (cnt <= 0) continue;
      for (int r = 0; r < p->R; ++r) {
        double* d = us + (long long)r * n + lo;
        nccl_check(a.broadcast(d, d, (size_t)cnt, ncclDouble, q, static_cast<ncclComm_t>(p->nccl),
                               p->stream),
                   "ncclBroadcast");
      }
    }
    nccl_check(a.groupEnd(), "ncclGroupEnd");
    return;
  }
  for (int q = 0; q < p->world; ++q) {
    const long long lo = p->pt_bounds[q], cnt = p->pt_bounds[q + 1] - lo;
    if (cnt <= 0) continue;
    for (int r = 0; r < p->R; ++r)
      if (p->ops.broadcast(p->ops.ctx, us + (long long)r * n + lo, cnt, q, p->stream) != 0)
        throw Error(BLFMM_ENCCL, "broadcast callback failed");
  }
}

void attach_common(blfmm_plan* p) {
  // world 1: a one-rank group (the same gather / scatter / max path, trivial
  // collectives) - lets the NCCL build be exercised on a single GPU
  if (p->world == 1) p->pt_bounds = {0, p->n};
  if ((long long)p->pt_bounds.size() != p->world + 1) {
    p->pt_bounds.assign(p->world + 1, 0);  // empty tree: nothing owned
  }
  if (p->xmode && !p->xbuf) {
    p->xown.alloc(sizeof(double2) * std::max<long long>(p->xcount, 1));
    p->xbuf = p->xown.as<double2>();
  }
  p->usorted.alloc(sizeof(double) * p->R * std::max<long long>(p->n, 1));
  p->gather_sorted = true;
  p->use_graphs = false;
}

// The whole sharded matvec on a plan with a communicator: lambda (full, on
// the device) -> u (full, caller order) on every rank.
void run_dist(blfmm_plan* p, const double* d_lam, double* d_out, cudaStream_t user) {
  const bool fence = user && user != p->stream;
  if (fence) {
    CK(cudaEventRecord(p->fence_in, user));
    CK(cudaStreamWaitEvent(p->stream, p->fence_in, 0));
  }
  auto phase = [&](int ph) {
    if (p->d == 1) launch_all<1>(p, d_lam, d_out, ph);
    if (p->d == 2) launch_all<2>(p, d_lam, d_out, ph);
    if (p->d == 3) launch_all<3>(p, d_lam, d_out, ph);
  };
  if (p->xmode) {
    phase(1);                                            // partitioned upsweep
    comm_sum(p, reinterpret_cast<double*>(p->xbuf), 2 * p->xcount);  // expansion exchange
    phase(2);                                            // owned downsweep + near field
  } else {
    phase(0);  // replicated upsweep, owned downsweep
  }
  comm_gather(p);
  if (p->n)
    k_scatter_sorted<<<blocks_for(p->n, 256), 256, 0, p->stream>>>(
        p->usorted.as<double>(), p->perm.as<int>(), p->n, p->R, d_out);
  CK(cudaGetLastError());
  if (p->want_imag) comm_max(p, reinterpret_cast<double*>(p->imag_bits.p), 1);
  if (fence) {
    CK(cudaEventRecord(p->fence_out, p->stream));
    CK(cudaStreamWaitEvent(user, p->fence_out, 0));
  }
}

void execute_host(blfmm_plan* p, const double* lambda, double* out, blfmm_stats* s,
                  void* stream, bool single) {
  if (!p) throw Error(BLFMM_EINVAL, "null plan");
  if (p->n && (!lambda || !out)) throw Error(BLFMM_EINVAL, "null lambda/out");
  DeviceGuard g(p->device);
  cudaStream_t user = static_cast<cudaStream_t>(stream);
  cudaStream_t cs = user ? user : p->stream;
  size_t bytes = sizeof(double) * p->R * p->n;
  if (bytes) CK(cudaMemcpyAsync(p->lam_in.p, lambda, bytes, cudaMemcpyHostToDevice, cs));
  p->want_imag = s != nullptr;
  if (p->comm_kind) run_dist(p, p->lam_in.as<double>(), p->out.as<double>(), cs);
  else run(p, p->lam_in.as<double>(), p->out.as<double>(), user);
  if (bytes) CK(cudaMemcpyAsync(out, p->out.p, bytes, cudaMemcpyDeviceToHost, cs));
  CK(cudaStreamSynchronize(cs));
  CK(cudaStreamSynchronize(p->stream));
  collect_times(p);
  fill_stats(p, s, single);
}
