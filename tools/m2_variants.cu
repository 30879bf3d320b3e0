// m2_variants.cu — development aid (not part of libjfb200.so): launch shapes
// of the n = 13 moment J-pass (jf_moment2.cuh) on one rank's C5 band
// (8192 x H rows), 20 launches in a CUDA graph.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//        -I include -I paper_2208_12187_b200/csrc -o tools/m2_variants tools/m2_variants.cu
#include <cmath>
#include <cstdio>
#include <vector>

#ifndef JF_DEV
#define JF_DEV 1
#endif
#include <algorithm>

#include "jf_moment2.cuh"

using namespace jf;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

static double ref[128];
static bool have_ref = false;

template <int L, int TC, int NW>
void run(const char* name, const double* dz, const double* dx, const double* pre, int W, int H, double* dpart,
         unsigned* dtick, double* dout, int* derr, int grid) {
  auto k = moment2_task_kernel<L, TC, NW, true>;
  const int smem = moment2_task_smem_bytes(NW);
  CK(cudaFuncSetAttribute((const void*)k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  PassArgs a;
  memset(&a, 0, sizeof(a));
  a.z = dz;
  a.m = (int64_t)W * H;
  a.W = W;
  a.coord = COORD_GRID;
  a.epilogue = EPI_NONE;
  a.x = dx;
  a.partials = dpart;
  a.ticket = dtick;
  a.out = dout;
  a.err = derr;
  memcpy(a.pre, pre, sizeof(double) * 15);
  a.has_pre = 1;
  cudaStream_t s;
  CK(cudaStreamCreate(&s));
  for (int i = 0; i < 3; ++i) k<<<grid, NW * 32, smem, s>>>(nullptr, nullptr, 0, 0, a);
  CK(cudaStreamSynchronize(s));
  CK(cudaGetLastError());
  if (!have_ref) {  // per-warp timeline of one launch
    const int NWT = grid * NW;
    unsigned long long* dd;
    CK(cudaMalloc(&dd, sizeof(unsigned long long) * 4 * 16384));
    CK(cudaMemset(dd, 0, sizeof(unsigned long long) * 4 * 16384));
    a.dbg = dd;
    k<<<grid, NW * 32, smem, s>>>(nullptr, nullptr, 0, 0, a);
    CK(cudaStreamSynchronize(s));
    a.dbg = nullptr;
    std::vector<unsigned long long> hd(4 * 16384);
    CK(cudaMemcpy(hd.data(), dd, sizeof(unsigned long long) * hd.size(), cudaMemcpyDeviceToHost));
    cudaFree(dd);
    unsigned long long t0 = ~0ull;
    for (int w = 0; w < NWT; ++w) t0 = std::min(t0, hd[w * 8 + 1]);
    auto q = [&](int c0, int c1, const char* nm) {
      std::vector<double> v;
      for (int w = 0; w < NWT; ++w) v.push_back(((double)hd[w * 8 + c1] - (double)(c0 < 0 ? t0 : hd[w * 8 + c0])) / 1e3);
      std::sort(v.begin(), v.end());
      printf("  %-18s min %6.2f med %6.2f max %6.2f us\n", nm, v[0], v[v.size() / 2], v.back());
    };
    q(-1, 1, "entry");
    q(1, 2, "setup");
    q(2, 3, "tasks");
    q(-1, 3, "tasks end");
    const unsigned long long* tl = hd.data() + 4 * 16384 - 16;
    printf("  tail from ticket: reduced %.2f, prologue %.2f, kalt2 %.2f, chain %.2f us\n", (double)(tl[2] - tl[1]) / 1965.0,
           (double)(tl[5] - tl[1]) / 1965.0, (double)(tl[6] - tl[1]) / 1965.0, (double)(tl[7] - tl[1]) / 1965.0);
  }
  cudaGraph_t g;
  cudaGraphExec_t ge;
  CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal));
  for (int i = 0; i < 20; ++i) k<<<grid, NW * 32, smem, s>>>(nullptr, nullptr, 0, 0, a);
  CK(cudaStreamEndCapture(s, &g));
  CK(cudaGraphInstantiate(&ge, g, 0));
  CK(cudaGraphLaunch(ge, s));
  CK(cudaStreamSynchronize(s));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0, s);
    CK(cudaGraphLaunch(ge, s));
    cudaEventRecord(e1, s);
    CK(cudaStreamSynchronize(s));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = fminf(best, ms);
  }
  double out[128];
  CK(cudaMemcpy(out, dout, sizeof(double) * 106, cudaMemcpyDeviceToHost));
  double maxd = 0.0;
  if (!have_ref) {
    memcpy(ref, out, sizeof(out));
    have_ref = true;
  } else {
    for (int i = 0; i < 105; ++i) maxd = fmax(maxd, fabs(out[i] - ref[i]) / (fabs(ref[i]) + 1e-300));
  }
  printf("{\"variant\": \"%s\", \"H\": %d, \"us\": %.2f, \"maxrel_vs_first\": %.2e}\n", name, H, best * 1e3 / 20, maxd);
  cudaGraphExecDestroy(ge);
  cudaGraphDestroy(g);
  cudaStreamDestroy(s);
}

int main(int argc, char** argv) {
  const int W = 8192, H = argc > 1 ? atoi(argv[1]) : 1024;
  const double p[13] = {1.0, 3000.0, 500.0, 900.0, 600.0, 0.5, 0.8, 5000.0, 700.0, 700.0, 1100.0, 1.2, 0.3};
  std::vector<double> h((size_t)W * H);
  for (int r = 0; r < H; ++r)
    for (int c = 0; c < W; ++c) {
      double v = 0.3 + 0.05 * sin(0.37 * c + 1.3 * r);
      for (int q = 0; q < 2; ++q) {
        const double* g = p + 6 * q;
        const double C = cos(g[5]), S = sin(g[5]);
        const double dx = c - g[1] * 1.02, dy = r - g[2] * 0.99;
        const double u = (C * dx - S * dy) / g[3], w = (S * dx + C * dy) / g[4];
        v += 1.05 * g[0] * exp(-0.5 * (u * u + w * w));
      }
      h[(size_t)r * W + c] = v;
    }
  double *dz, *dx, *dpart, *dout;
  unsigned* dtick;
  int* derr;
  CK(cudaMalloc(&dz, sizeof(double) * h.size()));
  CK(cudaMemcpy(dz, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice));
  CK(cudaMalloc(&dx, sizeof(double) * 16));
  CK(cudaMemcpy(dx, p, sizeof(p), cudaMemcpyHostToDevice));
  CK(cudaMalloc(&dpart, sizeof(double) * 4096 * 128));
  CK(cudaMalloc(&dtick, sizeof(unsigned) * 1024));
  CK(cudaMemset(dtick, 0, sizeof(unsigned) * 1024));
  CK(cudaMalloc(&dout, sizeof(double) * 128));
  CK(cudaMalloc(&derr, sizeof(int) * 4));
  double pre[16];
  gauss2d_x2_prologue(p, pre);
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
#define RUN(L, TC, NW) run<L, TC, NW>(#L " " #TC " " #NW, dz, dx, pre, W, H, dpart, dtick, dout, derr, nsm)
  RUN(8, 8, 12);
  RUN(8, 4, 12);
  RUN(8, 2, 12);
  RUN(16, 4, 12);
  RUN(16, 2, 12);
  RUN(8, 8, 12);
  return 0;
}
