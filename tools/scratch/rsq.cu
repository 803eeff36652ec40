#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>
__global__ void k(const double* x, double* y0, double* y1, double* y2, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double v = x[i], y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(v));
  y0[i] = y;
  // quadratic Newton with the half taken on the exponent (integer op)
  double t = y * y;
  double e = fma(-v, t, 1.0);
  int hi = __double2hiint(y), lo = __double2loint(y);
  double h = __hiloint2double(hi - 0x00100000, lo);
  y1[i] = fma(h, e, y);
  y2[i] = fma(fma(0.375, e, 0.5) * e, y, y);
}
int main() {
  const int n = 1 << 24;
  double *x, *a, *b, *c;
  cudaMallocManaged(&x, n * 8); cudaMallocManaged(&a, n * 8); cudaMallocManaged(&b, n * 8); cudaMallocManaged(&c, n * 8);
  unsigned long long s = 12345;
  for (int i = 0; i < n; ++i) { s = s * 6364136223846793005ULL + 1442695040888963407ULL; double u = (s >> 11) * (1.0 / 9007199254740992.0); x[i] = 0.0025 + 3.0 * u * u; }
  k<<<(n + 255) / 256, 256>>>(x, a, b, c, n);
  cudaDeviceSynchronize();
  double m0 = 0, m1 = 0, m2 = 0, s1 = 0, s2 = 0;
  for (int i = 0; i < n; ++i) {
    long double ref = 1.0L / sqrtl((long double)x[i]);
    double e0 = fabs((double)((a[i] - ref) / ref)), e1 = fabs((double)((b[i] - ref) / ref)), e2 = fabs((double)((c[i] - ref) / ref));
    m0 = fmax(m0, e0); m1 = fmax(m1, e1); m2 = fmax(m2, e2); s1 += (double)((b[i]-ref)/ref); s2 += (double)((c[i]-ref)/ref);
  }
  printf("seed max rel %.3e (2^%.1f)\nquadratic max rel %.3e mean %.3e\ncubic max rel %.3e mean %.3e\n", m0, log2(m0), m1, s1 / n, m2, s2 / n);
}
