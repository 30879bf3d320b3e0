// jpass_variants.cu — development aid (not part of libjfb200.so): times launch
// shapes of the production n = 7 moment J-pass (jf_moment_stream.cuh) on a
// synthetic 4096 x 4096 image (the T parameters), 20 launches in a CUDA graph,
// and checks each variant's K-vector against the first one.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//        -I include -I paper_2208_12187_b200/csrc -o tools/jpass_variants tools/jpass_variants.cu
#include <cmath>
#include <cstdio>
#include <vector>

#ifndef JF_DEV
#define JF_DEV 1  // per-warp globaltimer stamps (timeline of the first variant)
#endif
#include <algorithm>

#include "jf_moment_stream.cuh"

using namespace jf;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

static double ref[64];
static bool have_ref = false;

static const double* g_pre = nullptr;  // host-precomputed prologue (PassArgs::pre) or nullptr

template <int L, int NW, int SEEDN, int STG>
void run(const char* name, const double* dz, const double* dx, int W, int H, double* dpart, unsigned* dtick,
         double* dout, int* derr, int grid) {
  auto k = moment_stream_kernel<L, NW, SEEDN, STG>;
  const int smem = moment_stream_smem_bytes(NW, L, STG);
  CK(cudaFuncSetAttribute((const void*)k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  cudaFuncAttributes fa;
  CK(cudaFuncGetAttributes(&fa, (const void*)k));
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
  if (g_pre) {
    memcpy(a.pre, g_pre, sizeof(a.pre));
    a.has_pre = 1;
  }
  cudaStream_t s;
  CK(cudaStreamCreate(&s));
  for (int i = 0; i < 3; ++i) k<<<grid, NW * 32, smem, s>>>(nullptr, nullptr, 0, 0, a);
  CK(cudaStreamSynchronize(s));
  CK(cudaGetLastError());
  if (JF_DEV && !have_ref) {  // per-warp timeline of one launch (stamps: [smid, entry, prologue, loop end])
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
      printf("  %-22s min %6.2f med %6.2f p90 %6.2f max %6.2f us\n", nm, v[0], v[v.size() / 2], v[v.size() * 9 / 10], v.back());
    };
    q(-1, 1, "entry (from first)");
    q(1, 4, "args+issue");
    q(4, 5, "pass_begin");
    q(5, 6, "prologue compute");
    q(6, 2, "accuracy check");
    q(1, 2, "prologue dur");
    q(-1, 2, "prologue end");
    q(2, 3, "loop dur");
    q(-1, 3, "loop end");
    // per SM: last - first loop end
    std::vector<double> spread, last;
    for (int b = 0; b < grid; ++b) {
      double lo = 1e30, hi = 0;
      for (int w = 0; w < NW; ++w) {
        const double t = ((double)hd[(b * NW + w) * 8 + 3] - (double)t0) / 1e3;
        lo = std::min(lo, t);
        hi = std::max(hi, t);
      }
      spread.push_back(hi - lo);
      last.push_back(hi);
    }
    std::sort(spread.begin(), spread.end());
    std::sort(last.begin(), last.end());
    printf("  per-block loop-end spread med %.2f max %.2f us; block last loop end min %.2f med %.2f max %.2f us\n",
           spread[grid / 2], spread.back(), last[0], last[grid / 2], last.back());
    printf("  mean loop end by warp id:");
    for (int w = 0; w < NW; ++w) {
      double m = 0.0;
      for (int b = 0; b < grid; ++b) m += ((double)hd[(b * NW + w) * 8 + 3] - (double)t0) / 1e3;
      printf(" %.2f", m / grid);
    }
    printf("\n  mean loop dur by warp id:");
    for (int w = 0; w < NW; ++w) {
      double m = 0.0;
      for (int b = 0; b < grid; ++b) m += ((double)hd[(b * NW + w) * 8 + 3] - (double)hd[(b * NW + w) * 8 + 2]) / 1e3;
      printf(" %.2f", m / grid);
    }
    printf("\n");
    const unsigned long long* tl = hd.data() + 4 * 16384 - 16;  // last block's tail (clock64)
    printf("  tail from ticket (us at 1.965 GHz): loads+map %.2f, kvec %.2f, chain %.2f, hand-off %.2f\n",
           (double)(tl[2] - tl[1]) / 1965.0, (double)(tl[5] - tl[1]) / 1965.0, (double)(tl[6] - tl[1]) / 1965.0,
           (double)(tl[7] - tl[1]) / 1965.0);
  }
  const int NJ = 20;
  cudaGraph_t g;
  cudaGraphExec_t ge;
  CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal));
  for (int i = 0; i < NJ; ++i) k<<<grid, NW * 32, smem, s>>>(nullptr, nullptr, 0, 0, a);
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
  const double us = best * 1e3 / NJ;
  double out[64];
  CK(cudaMemcpy(out, dout, sizeof(double) * 37, cudaMemcpyDeviceToHost));
  double maxd = 0.0;
  if (!have_ref) {
    memcpy(ref, out, sizeof(out));
    have_ref = true;
  } else {
    for (int i = 0; i < 36; ++i) maxd = fmax(maxd, fabs(out[i] - ref[i]) / (fabs(ref[i]) + 1e-300));
  }
  const double m = (double)W * H;
  printf("{\"variant\": \"%s\", \"regs\": %d, \"smem\": %d, \"local\": %zu, \"us\": %.2f, \"hbm_frac\": %.3f, \"maxrel_vs_first\": %.2e, \"cost\": %.10e}\n",
         name, fa.numRegs, smem, fa.localSizeBytes, us, 8 * m / (us * 1e-6) / 6553.6e9, maxd, 0.5 * out[35]);
  cudaGraphExecDestroy(ge);
  cudaGraphDestroy(g);
  cudaStreamDestroy(s);
}

int main(int argc, char** argv) {
  const int W = argc > 1 ? atoi(argv[1]) : 4096, H = W;
  const double p[7] = {1.2183346542295974, 1851.3072104717621 * W / 4096, 1511.4287038505363 * W / 4096,
                       524.9889360025724 * W / 4096, 1158.6440554950686 * W / 4096, 1.7914207797496442,
                       0.40173085011841553};
  std::vector<double> h((size_t)W * H);
  const double C = cos(p[5]), S = sin(p[5]);
  for (int r = 0; r < H; ++r)
    for (int c = 0; c < W; ++c) {  // a rotated Gaussian near p (truth 5% off) plus a deterministic ripple
      const double dx = c - p[1] * 1.03, dy = r - p[2] * 0.98;
      const double u = (C * dx - S * dy) / (p[3] * 1.05), v = (S * dx + C * dy) / (p[4] * 0.97);
      h[(size_t)r * W + c] = 1.1 * p[0] * exp(-0.5 * (u * u + v * v)) + 0.38 + 0.1 * sin(0.37 * c + 1.3 * r);
    }
  double *dz, *dx, *dpart, *dout;
  unsigned* dtick;
  int* derr;
  CK(cudaMalloc(&dz, sizeof(double) * h.size()));
  CK(cudaMemcpy(dz, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice));
  CK(cudaMalloc(&dx, sizeof(double) * 16));
  CK(cudaMemcpy(dx, p, sizeof(p), cudaMemcpyHostToDevice));
  CK(cudaMalloc(&dpart, sizeof(double) * 4096 * 64));
  CK(cudaMalloc(&dtick, sizeof(unsigned) * 1024));
  CK(cudaMemset(dtick, 0, sizeof(unsigned) * 1024));
  CK(cudaMalloc(&dout, sizeof(double) * 64));
  CK(cudaMalloc(&derr, sizeof(int) * 4));
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
#define RUN(L, NW, S, STG) run<L, NW, S, STG>(#L " " #NW " " #S " " #STG, dz, dx, W, H, dpart, dtick, dout, derr, nsm)
  double pre[8];
  gauss2d_prologue(p, pre);
  g_pre = pre;
  RUN(16, 12, 8, 3);
  return 0;
}
