// jpass_probe.cu — design probe for the n = 7 moment-form J-pass hot loop
// (development aid, not part of libjfb200.so).  Streams a W x H fp64 image and
// runs the 19-FP64-op per-point moment update of jf_moment.cuh with several
// launch shapes / z-staging schemes, static contiguous split of warp-chunks
// per warp (no tasks, no epilogue), to measure what the hot loop alone can
// reach against the HBM (8 B/pt) and FP64 (19 op/pt) floors.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/jpass_probe tools/jpass_probe.cu
//   tools/jpass_probe [W]
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

struct Par { double A, off, ga, gb2, gc, x0, y0; };

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

template <int L>
struct Mom {
  double P[5], Q[3], R[3], sr, srr;
  __device__ void zero() {
#pragma unroll
    for (int i = 0; i < 5; ++i) P[i] = 0.0;
#pragma unroll
    for (int i = 0; i < 3; ++i) Q[i] = R[i] = 0.0;
    sr = srr = 0.0;
  }
  __device__ __forceinline__ void shift(double d) {
#pragma unroll
    for (int j = 1; j <= 4; ++j)
#pragma unroll
      for (int p = 4; p >= j; --p) P[p] = fma(d, P[p - 1], P[p]);
#pragma unroll
    for (int j = 1; j <= 2; ++j)
#pragma unroll
      for (int p = 2; p >= j; --p) {
        Q[p] = fma(d, Q[p - 1], Q[p]);
        R[p] = fma(d, R[p - 1], R[p]);
      }
  }
  template <class ZF>
  __device__ __forceinline__ void chunk(const Par& q, double& E, double& Rr, double rho, ZF zat) {
    constexpr double D = 32.0;
    double cs = 0.0;
#pragma unroll
    for (int k = 0; k < L; ++k) {
      const double u = E;
      const double r = fma(q.A, u, q.off) - zat(k);
      const double u2 = u * u;
      const double k1 = D * k, k2 = k1 * k1, k3 = k2 * k1, k4 = k2 * k2;
      const double ur = u * r;
      P[0] += u2;
      Q[0] += u;
      R[0] += ur;
      if (k > 0) {
        P[1] = fma(u2, k1, P[1]);
        P[2] = fma(u2, k2, P[2]);
        P[3] = fma(u2, k3, P[3]);
        P[4] = fma(u2, k4, P[4]);
        Q[1] = fma(u, k1, Q[1]);
        Q[2] = fma(u, k2, Q[2]);
        R[1] = fma(ur, k1, R[1]);
        R[2] = fma(ur, k2, R[2]);
      }
      sr += r;
      cs = fma(r, r, cs);
      E *= Rr;
      Rr *= rho;
    }
    srr += cs;
  }
  __device__ double sum() const {
    double s = sr + srr;
#pragma unroll
    for (int i = 0; i < 5; ++i) s += P[i];
#pragma unroll
    for (int i = 0; i < 3; ++i) s += Q[i] + R[i];
    return s;
  }
};

// MODE 0: register prefetch, copy zn -> zc per chunk
// MODE 1: register prefetch, two buffers, loop unrolled by 2 chunks (no copies)
// MODE 2: per-warp smem ring of STG chunk slots filled by cp.async.bulk (TMA), LDS reads
template <int L, int NW, int MODE, int STG, int MINB>
__global__ void __launch_bounds__(NW * 32, MINB) probe(const double* __restrict__ z, int W, int H, Par q, double* out) {
  constexpr int CW = 32 * L;
  constexpr double D = 32.0;
  extern __shared__ __align__(128) double ring_all[];
  __shared__ __align__(8) unsigned long long bars[MODE == 2 ? NW * STG : 1];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int cpr = W / CW;
  const int64_t nch = (int64_t)H * cpr;
  const int64_t nwt = (int64_t)gridDim.x * NW;
  const int64_t gw = (int64_t)blockIdx.x * NW + wid;
  const int64_t c0 = gw * nch / nwt, c1 = (gw + 1) * nch / nwt;
  const double rho = exp(-2.0 * q.ga * D * D);
  Mom<L> M;
  M.zero();
  double E = 0.0, Rr = 0.0;
  auto seed = [&](int64_t ch) {
    const int64_t row = ch / cpr;
    const int cc = (int)(ch - row * cpr);
    const double dy = (double)row - q.y0;
    const double dx0 = (double)(cc * CW + lane) - q.x0;
    const double q0 = dx0 * (q.ga * dx0 + q.gb2 * dy) + q.gc * (dy * dy);
    const double argR = D * (2.0 * q.ga * dx0 + q.gb2 * dy) + q.ga * D * D;
    E = exp(-q0);
    Rr = exp(-argR);
  };
  if constexpr (MODE == 0) {
    double zn[L];
    auto load = [&](int64_t ch) {
      const double* zp = z + ch * CW + lane;
#pragma unroll
      for (int k = 0; k < L; ++k) zn[k] = __ldcs(zp + 32 * k);
    };
    if (c0 < c1) load(c0);
    for (int64_t ch = c0; ch < c1; ++ch) {
      double zc[L];
#pragma unroll
      for (int k = 0; k < L; ++k) zc[k] = zn[k];
      if (ch + 1 < c1) load(ch + 1);
      if (((ch - c0) & 3) == 0) seed(ch);
      M.shift(-(double)CW);
      M.chunk(q, E, Rr, rho, [&](int k) { return zc[k]; });
    }
  } else if constexpr (MODE == 1) {
    double za[L], zb[L];
    auto load = [&](double (&zz)[L], int64_t ch) {
      const double* zp = z + ch * CW + lane;
#pragma unroll
      for (int k = 0; k < L; ++k) zz[k] = __ldcs(zp + 32 * k);
    };
    if (c0 < c1) load(za, c0);
    int64_t ch = c0;
    for (; ch + 1 < c1; ch += 2) {
      load(zb, ch + 1);
      if (((ch - c0) & 3) == 0) seed(ch);
      M.shift(-(double)CW);
      M.chunk(q, E, Rr, rho, [&](int k) { return za[k]; });
      if (ch + 2 < c1) load(za, ch + 2);
      M.shift(-(double)CW);
      M.chunk(q, E, Rr, rho, [&](int k) { return zb[k]; });
    }
    if (ch < c1) {
      M.shift(-(double)CW);
      M.chunk(q, E, Rr, rho, [&](int k) { return za[k]; });
    }
  } else {
    double* ring = ring_all + wid * STG * CW;
    unsigned long long* bar = bars + wid * STG;
    unsigned long long pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    if (lane == 0) {
#pragma unroll
      for (int s = 0; s < STG; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar + s)));
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    auto issue = [&](int s, int64_t ch) {
      if (lane == 0) {
        const unsigned b = su32(bar + s);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(CW * 8) : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
            ::"r"(su32(ring + s * CW)), "l"(z + ch * CW), "r"(CW * 8), "r"(b), "l"(pol) : "memory");
      }
    };
#pragma unroll
    for (int s = 0; s < STG; ++s)
      if (c0 + s < c1) issue(s, c0 + s);
    unsigned par = 0;
    int s = 0;
    for (int64_t ch = c0; ch < c1; ++ch) {
      const unsigned b = su32(bar + s);
      unsigned done = 0;
      do {
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                     : "=r"(done) : "r"(b), "r"((par >> s) & 1u) : "memory");
      } while (!done);
      par ^= 1u << s;
      if (((ch - c0) & 3) == 0) seed(ch);
      M.shift(-(double)CW);
      const double* zs = ring + s * CW + lane;
      M.chunk(q, E, Rr, rho, [&](int k) { return zs[32 * k]; });
      __syncwarp();
      if (ch + STG < c1) issue(s, ch + STG);
      s = (s + 1 == STG) ? 0 : s + 1;
    }
  }
  const double v = M.sum();
  if (v == 1.2345) out[gw] = v;
}

template <int L, int NW, int MODE, int STG, int MINB>
int run(const char* name, const double* z, int W, int H, int nsm, double* out, int blocks_per_sm = 1) {
  const Par q{1.3, 0.33, 1.0 / (2 * 640.0 * 640.0), 1e-7, 1.0 / (2 * 1016.0 * 1016.0), 1727.0, 1779.0};
  auto k = probe<L, NW, MODE, STG, MINB>;
  const int smem = MODE == 2 ? NW * STG * 32 * L * 8 : 0;
  if (smem > 48 * 1024) CK(cudaFuncSetAttribute((const void*)k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  cudaFuncAttributes fa;
  CK(cudaFuncGetAttributes(&fa, (const void*)k));
  int occ = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, NW * 32, smem));
  const int grid = nsm * blocks_per_sm;
  for (int i = 0; i < 3; ++i) k<<<grid, NW * 32, smem>>>(z, W, H, q, out);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int reps = 20;
  cudaEventRecord(e0);
  for (int i = 0; i < reps; ++i) k<<<grid, NW * 32, smem>>>(z, W, H, q, out);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double us = ms * 1e3 / reps;
  const double m = (double)W * H;
  printf("{\"variant\": \"%s\", \"regs\": %d, \"occ_blocks\": %d, \"grid\": %d, \"us\": %.2f, \"hbm_frac\": %.3f, \"fp64_frac\": %.3f}\n",
         name, fa.numRegs, occ, grid, us, 8 * m / (us * 1e-6) / 6539.5e9, 19 * m / (us * 1e-6) / (nsm * 64 * 1.965e9));
  return 0;
}

int main(int argc, char** argv) {
  const int W = argc > 1 ? atoi(argv[1]) : 4096, H = W;
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  double *z, *out;
  CK(cudaMalloc(&z, sizeof(double) * W * H));
  CK(cudaMalloc(&out, sizeof(double) * 65536));
  std::vector<double> h((size_t)W * H);
  for (size_t i = 0; i < h.size(); ++i) h[i] = 0.3 + 1e-3 * (double)(i % 977);
  CK(cudaMemcpy(z, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice));
  run<16, 12, 0, 1, 1>("L16 NW12 regcopy", z, W, H, nsm, out);
  run<16, 16, 0, 1, 1>("L16 NW16 regcopy", z, W, H, nsm, out);
  run<8, 12, 0, 1, 1>("L8 NW12 regcopy", z, W, H, nsm, out);
  run<8, 16, 0, 1, 1>("L8 NW16 regcopy", z, W, H, nsm, out);
  run<8, 16, 1, 1, 1>("L8 NW16 dbuf", z, W, H, nsm, out);
  run<8, 20, 1, 1, 1>("L8 NW20 dbuf", z, W, H, nsm, out);
  run<16, 12, 1, 1, 1>("L16 NW12 dbuf", z, W, H, nsm, out);
  run<8, 16, 2, 3, 1>("L8 NW16 tma3", z, W, H, nsm, out);
  run<8, 20, 2, 3, 1>("L8 NW20 tma3", z, W, H, nsm, out);
  run<8, 24, 2, 3, 1>("L8 NW24 tma3", z, W, H, nsm, out);
  run<8, 32, 2, 2, 1>("L8 NW32 tma2", z, W, H, nsm, out);
  run<16, 16, 2, 3, 1>("L16 NW16 tma3", z, W, H, nsm, out);
  run<16, 12, 2, 4, 1>("L16 NW12 tma4", z, W, H, nsm, out);
  run<8, 8, 2, 3, 2>("L8 NW8x2 tma3", z, W, H, nsm, out, 2);
  run<8, 8, 2, 3, 3>("L8 NW8x3 tma3", z, W, H, nsm, out, 3);
  run<16, 8, 2, 3, 2>("L16 NW8x2 tma3", z, W, H, nsm, out, 2);
  return 0;
}
