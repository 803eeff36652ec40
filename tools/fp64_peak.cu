// FP64 peak microbenchmark for the roofline denominators (profiles/fp64_peak.json):
// (1) DFMA: independent FMA chains per thread, all SMs;
// (2) DMMA: mma.sync.aligned.m8n8k4.row.col.f64 back to back (8 accumulators/warp).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
}

__global__ void dmma_kernel(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-6, b = 0.5;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  double* out;
  cudaMalloc(&out, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  // DFMA
  int blocks = sms * 8, threads = 256, iters = 20000;
  dfma_kernel<<<blocks, threads>>>(out, 100, 1.0000001, 1e-9);
  cudaEventRecord(e0);
  dfma_kernel<<<blocks, threads>>>(out, iters, 1.0000001, 1e-9);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  double dfma_tf = 2.0 * 16 * (double)iters * blocks * threads / (ms * 1e-3) / 1e12;
  // DMMA
  int wblocks = sms * 8, wthreads = 128, witers = 20000;
  dmma_kernel<<<wblocks, wthreads>>>(out, 100);
  cudaEventRecord(e0);
  dmma_kernel<<<wblocks, wthreads>>>(out, witers);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  double warps = (double)wblocks * wthreads / 32;
  double dmma_tf = 2.0 * 256 * 8 * (double)witers * warps / (ms * 1e-3) / 1e12;
  printf("{\"sms\": %d, \"clock_khz_attr\": %d, \"dfma_tflops\": %.3f, \"dmma_tflops\": %.3f, "
         "\"how\": \"tools/fp64_peak.cu: %d blocks x %d threads x %d iters x 16 independent DFMA chains; "
         "DMMA m8n8k4 f64, 8 independent accumulators per warp, %d blocks x %d threads x %d iters\"}\n",
         sms, clk, dfma_tf, dmma_tf, blocks, threads, iters, wblocks, wthreads, witers);
  return 0;
}
