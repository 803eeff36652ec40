// C++ caller of the library's distributed matvec (blfmm_plan_attach_comm +
// blfmm_execute): `world` ranks as threads of one process, each with its own
// plan (rank / world) on one device, and host collectives supplied through
// blfmm_comm_ops (a shared slot table and a barrier: the ranks' kernels never
// wait on each other). Every rank's u must equal the one-rank matvec.
//   dist_threads <d> <n> <leaf> <world> <kernel spec> <sigma> <m> <nrhs>
// Exit code 0 and "OK" on success.
#include <cuda_runtime.h>

#include <barrier>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

#include "blfmm_gpu.h"

namespace {

struct Shared {
  int world;
  std::barrier<> bar;
  std::vector<std::vector<double>> slot;
  explicit Shared(int w) : world(w), bar(w), slot(w) {}
};
struct RankCtx {
  Shared* sh;
  int rank;
};

int dev_to_host(std::vector<double>& h, const double* d, long long cnt, void* stream) {
  h.resize(cnt);
  if (cudaStreamSynchronize(static_cast<cudaStream_t>(stream)) != cudaSuccess) return 1;
  return cudaMemcpy(h.data(), d, sizeof(double) * cnt, cudaMemcpyDeviceToHost) != cudaSuccess;
}
int host_to_dev(double* d, const std::vector<double>& h) {
  return cudaMemcpy(d, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice) !=
         cudaSuccess;
}

template <bool MAX>
int all_reduce(void* ctx, double* d, long long cnt, void* stream) {
  auto* c = static_cast<RankCtx*>(ctx);
  Shared& s = *c->sh;
  if (dev_to_host(s.slot[c->rank], d, cnt, stream)) return 1;
  s.bar.arrive_and_wait();
  std::vector<double> acc(s.slot[0]);
  for (int q = 1; q < s.world; ++q)  // rank order on every rank: identical sums
    for (long long i = 0; i < cnt; ++i)
      acc[i] = MAX ? std::fmax(acc[i], s.slot[q][i]) : acc[i] + s.slot[q][i];
  s.bar.arrive_and_wait();
  return host_to_dev(d, acc);
}
int broadcast(void* ctx, double* d, long long cnt, int root, void* stream) {
  auto* c = static_cast<RankCtx*>(ctx);
  Shared& s = *c->sh;
  if (c->rank == root && dev_to_host(s.slot[root], d, cnt, stream)) return 1;
  s.bar.arrive_and_wait();
  int rc = c->rank == root ? 0 : host_to_dev(d, s.slot[root]);
  s.bar.arrive_and_wait();
  return rc;
}

double u01(uint64_t seed, uint64_t i) {  // splitmix64
  uint64_t z = seed * 0x9E3779B97F4A7C15ull + i + 1;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z ^= z >> 31;
  return (z >> 11) * (1.0 / 9007199254740992.0);
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 9) {
    std::fprintf(stderr, "usage: %s d n leaf world spec sigma m nrhs\n", argv[0]);
    return 2;
  }
  const int d = std::atoi(argv[1]), leaf = std::atoi(argv[3]), world = std::atoi(argv[4]);
  const long long n = std::atoll(argv[2]);
  const double sigma = std::atof(argv[6]);
  const int m = std::atoi(argv[7]), nrhs = std::atoi(argv[8]);
  int kt;
  double shape;
  if (blfmm_parse_kernel_spec(argv[5], &kt, &shape)) return 3;
  // clustered points (4 blobs, clipped to the unit cube) and weights
  std::vector<double> x(n * d), lam(nrhs * n);
  for (long long i = 0; i < n; ++i) {
    const int b = static_cast<int>(i % 4);
    for (int k = 0; k < d; ++k) {
      double v = 0.2 + 0.2 * b + 0.15 * (u01(7, i * d + k) - 0.5) + 0.1 * u01(11, b * 3 + k);
      x[i * d + k] = std::fmin(1.0, std::fmax(0.0, v));
    }
  }
  for (long long i = 0; i < nrhs * n; ++i) lam[i] = 2.0 * u01(13, i) - 1.0;
  auto make = [&](int rank, int w, blfmm_plan** p) {
    blfmm_plan_desc desc;
    std::memset(&desc, 0, sizeof desc);
    desc.d = d;
    desc.n = n;
    desc.coords = x.data();
    for (int k = 0; k < d; ++k) desc.domain_hi[k] = 1.0;
    desc.kernel_type = kt;
    desc.kernel_shape = shape;
    desc.sigma = sigma;
    desc.m_per_dim = m;
    desc.leaf_level = leaf;
    desc.grid_mode = BLFMM_GRID_SHARED;
    desc.stencil_k = 10;
    desc.nrhs = nrhs;
    desc.device = 0;
    desc.rank = rank;
    desc.world = w;
    return blfmm_plan_create(&desc, p);
  };
  blfmm_plan* one = nullptr;
  if (make(0, 1, &one)) {
    std::fprintf(stderr, "plan: %s\n", blfmm_last_error());
    return 4;
  }
  std::vector<double> ref(nrhs * n);
  blfmm_stats rs;
  if (blfmm_execute(one, lam.data(), ref.data(), &rs, nullptr)) return 5;
  blfmm_plan_destroy(one);

  Shared sh(world);
  std::vector<std::vector<double>> got(world, std::vector<double>(nrhs * n));
  std::vector<double> imag(world);
  std::vector<int> rc(world, 0);
  std::vector<std::thread> th;
  std::vector<RankCtx> ctx(world);
  for (int r = 0; r < world; ++r) {
    ctx[r] = {&sh, r};
    th.emplace_back([&, r] {
      blfmm_plan* p = nullptr;
      if (make(r, world, &p)) {
        std::fprintf(stderr, "rank %d plan: %s\n", r, blfmm_last_error());
        rc[r] = 1;
        return;
      }
      blfmm_comm_ops ops{&ctx[r], all_reduce<false>, all_reduce<true>, broadcast};
      blfmm_stats st;
      if (blfmm_plan_attach_comm(p, &ops) ||
          blfmm_execute(p, lam.data(), got[r].data(), &st, nullptr) ||
          blfmm_execute(p, lam.data(), got[r].data(), &st, nullptr)) {
        std::fprintf(stderr, "rank %d: %s\n", r, blfmm_last_error());
        rc[r] = 1;
      }
      imag[r] = st.max_imag_residual;
      blfmm_plan_destroy(p);
    });
  }
  for (auto& t : th) t.join();
  double worst = 0.0, nrm = 0.0;
  for (long long i = 0; i < nrhs * n; ++i) nrm += ref[i] * ref[i];
  for (int r = 0; r < world; ++r) {
    if (rc[r]) return 6;
    double e = 0.0;
    for (long long i = 0; i < nrhs * n; ++i) e += (got[r][i] - ref[i]) * (got[r][i] - ref[i]);
    worst = std::fmax(worst, std::sqrt(e / nrm));
    if (std::fabs(imag[r] - rs.max_imag_residual) > 1e-8 * std::fmax(1.0, rs.max_imag_residual))
      return 7;
  }
  std::printf("world %d rel-l2 vs one rank %.3e\n", world, worst);
  if (!(worst <= 1e-13)) return 8;
  std::printf("OK\n");
  return 0;
}
