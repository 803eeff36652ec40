// Internal declarations shared by the host plan code and the CUDA sources.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/blfmm_gpu.h"

namespace blfmm_gpu {

struct Error : std::runtime_error {
  int code;
  double achieved = 0.0;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

struct KernelSpec {
  int type = BLFMM_KERNEL_GAUSSIAN;
  double shape = 1.0;
};

KernelSpec parse_spec(const std::string& spec);
// thread-local error state behind blfmm_last_error / blfmm_last_error_value
void set_error(const Error& e);
void set_error_message(const char* msg);
void require_fmm_kernel(const KernelSpec& k);
void require_radial_kernel(const KernelSpec& k);  // any RadialKernel::type with a valid shape
// dense kernel matvec on device vectors (blfmm.cu), the operator of blfmm_solve_dense
void direct_device(int d, long long n, const double* d_x, int type, double shape,
                   const double* d_in, double* d_out, void* stream);
double fourier_value(const KernelSpec& k, double xi, int d);
std::vector<double> translation_spectrum(const KernelSpec& k, double sigma,
                                         int m, int d);
// Phi_sigma in d = 1 (bandlimit.cpp:307-334) and its cubic-interpolation
// table of kRadialIntervals + 3 samples at step rmax / kRadialIntervals
// (bandlimit.cpp:229-262).
constexpr int kRadialIntervals = 1024;
double eval_bandlimited_1d(const KernelSpec& k, double sigma, double x, int refinement);
std::vector<double> bandlimited_radial_table(const KernelSpec& k, double sigma, double rmax,
                                             int refinement, double* step);

}  // namespace blfmm_gpu
