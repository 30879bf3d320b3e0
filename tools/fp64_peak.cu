// fp64_peak.cu — measured FP64 roofline denominators on this GPU:
// DFMA throughput (vector FP64 pipe) and DMMA m8n8k4 (FP64 tensor path), plus
// the SM clock seen.  Prints one JSON line.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) x[k] = threadIdx.x * 1e-3 + k;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 16; ++k) x[k] = fma(x[k], a, b);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 16; ++k) s += x[k];
  if (s == 12345.678) out[0] = s;
}

__global__ void dmma_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[4][2] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 4; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int k = 0; k < 4; ++k) s += c[k][0] + c[k][1];
  if (s == 12345.678) out[0] = s;
}

__global__ void mixed_kernel(double* out, int iters, double a, double b) {
  // DFMA chains and DMMA issued from the same warps: does the tensor path add throughput?
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3 + k;
  double ma = threadIdx.x * 1e-3, mb = 1.0 - threadIdx.x * 1e-4;
  double c[2][2] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
#pragma unroll
    for (int k = 0; k < 2; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(ma), "d"(mb));
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  s += c[0][0] + c[1][1];
  if (s == 12345.678) out[0] = s;
}

int main() {
  int dev = 0, nsm, clk;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  double* out;
  cudaMalloc(&out, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = nsm * 8, threads = 256, iters = 4096;
  float ms;
  dfma_kernel<<<blocks, threads>>>(out, 64, 0.999999, 1e-7);
  cudaEventRecord(e0);
  dfma_kernel<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  const double dfma_tflops = 2.0 * blocks * threads * (double)iters * 16 / (ms * 1e-3) / 1e12;
  dmma_kernel<<<blocks, threads>>>(out, 64);
  cudaEventRecord(e0);
  dmma_kernel<<<blocks, threads>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  const double warps = blocks * threads / 32.0;
  const double dmma_tflops = 2.0 * 8 * 8 * 4 * warps * (double)iters * 4 / (ms * 1e-3) / 1e12;
  mixed_kernel<<<blocks, threads>>>(out, 64, 0.999999, 1e-7);
  cudaEventRecord(e0);
  mixed_kernel<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  // 8 DFMA per thread + 2 DMMA (256 FMA each) per warp per iteration
  const double mixed_tflops = (2.0 * blocks * threads * (double)iters * 8 + 2.0 * 256 * 2 * warps * iters) / (ms * 1e-3) / 1e12;
  printf("{\"mixed_dfma_dmma_tflops\": %.3f}\n", mixed_tflops);
  printf("{\"sm_count\": %d, \"clock_rate_mhz\": %.0f, \"dfma_tflops\": %.3f, \"dmma_tflops\": %.3f, "
         "\"nominal_fp64_tflops_at_max_clock\": %.3f}\n",
         nsm, clk / 1000.0, dfma_tflops, dmma_tflops, nsm * 64 * 2 * (clk / 1e6) / 1e3);
  return 0;
}
