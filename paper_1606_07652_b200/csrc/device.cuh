// Device helpers shared by the CUDA translation units.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/blfmm_gpu.h"

namespace blfmm_gpu {

// complex double as (re, im)
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ void cmac(double2& acc, double2 a, double2 b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
}
__device__ __forceinline__ double2 polar1(double t) {
  double s, c;
  sincos(t, &s, &c);
  return make_double2(c, s);
}

// phi(r) from the squared distance (kernels.cpp:131-161 evaluates phi at
// r = sqrt(s); phi depends on r only through r^2 for these three kernels).
__device__ __forceinline__ double phi_of_r2(int type, double c, double s) {
  if (type == BLFMM_KERNEL_GAUSSIAN) return exp(-c * s);
  if (type == BLFMM_KERNEL_IMQ) return rsqrt(s + c * c);
  return sqrt(s + c * c);  // MQ
}

// Morton keys interleave the leaf-level integer coordinates with axis 0 as the
// most significant bit of each group, so key >> d is the parent's key.
template <int D>
__host__ __device__ __forceinline__ uint32_t morton_encode(const int* c, int bits) {
  uint32_t key = 0;
  for (int b = bits - 1; b >= 0; --b)
    for (int k = 0; k < D; ++k) key = (key << 1) | ((c[k] >> b) & 1u);
  return key;
}
template <int D>
__host__ __device__ __forceinline__ void morton_decode(uint32_t key, int bits, int* c) {
  for (int k = 0; k < D; ++k) c[k] = 0;
  for (int b = 0; b < bits; ++b)
    for (int k = D - 1; k >= 0; --k) {
      c[k] |= (key & 1u) << b;
      key >>= 1;
    }
}
// Row-major reference box id ((i*n)+j)*n+k (geometry.cpp:216-229).
template <int D>
__host__ __device__ __forceinline__ long long rowmajor_id(const int* c, int level) {
  long long id = 0;
  for (int k = 0; k < D; ++k) id = (id << level) | c[k];
  return id;
}

}  // namespace blfmm_gpu
