// lat.cu — dependent-chain latencies on this GPU (cycles): DFMA, DADD, fp64 sqrt,
// fp64 div, fp64 rsqrt, SHFL (double), FFMA.  Development aid for the solver warp.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, double x0, int it) {
  double x = x0 + threadIdx.x * 1e-9;
  long long t0, t1;
  float f = (float)x;
#define BENCH(name, expr) \
  t0 = clock64(); for (int i = 0; i < it; ++i) { expr; } t1 = clock64(); \
  if (threadIdx.x == 0) printf("%-8s %.1f cycles\n", name, (double)(t1 - t0) / it);
  BENCH("dfma", x = fma(x, 1.0000001, 1e-9));
  BENCH("dadd", x = x + 1e-9);
  BENCH("dsqrt", x = sqrt(x) + 1.0);
  BENCH("ddiv", x = 1.0 / x + 1.0);
  BENCH("drsqrt", x = rsqrt(x) + 1.0);
  BENCH("shfl64", x = __shfl_sync(0xffffffff, x, (threadIdx.x + 1) & 31) + 1e-9);
  BENCH("ffma", f = fmaf(f, 1.0000001f, 1e-9f));
  BENCH("fsqrt", f = __fsqrt_rn(f) + 1.0f);
  BENCH("frsqrt", f = rsqrtf(f) + 1.0f);
  BENCH("fdiv", f = __fdividef(1.0f, f) + 1.0f);
  out[threadIdx.x] = x + f;
}
int main() {
  double* o; cudaMalloc(&o, 1024);
  k<<<1, 32>>>(o, 1.5, 1000);
  cudaDeviceSynchronize();
  return 0;
}
