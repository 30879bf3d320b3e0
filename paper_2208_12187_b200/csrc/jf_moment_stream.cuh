// jf_moment_stream.cuh — the production J-pass for the rotated 2D Gaussian
// (n = 7) on an implicit pixel grid, unweighted: the moment form of R34
// (jf_moment.cuh) with a static, contiguous split of the image over warps.
//
// Same output as every other J-pass — the upper triangle of [J | r]^T [J | r]
// (Eq. 2, Eq. 4, Eq. 5) plus the non-finite count —
// from the 29 moments of jf_moment.cuh's MomLayout, mapped once per pass.
//
// Work split.  The image is a sequence of warp-chunks (32 L consecutive
// pixels of one row; a row's last chunk may be partial).  Warp w of the grid
// owns the contiguous chunk range [w nch / nw, (w+1) nch / nw): every warp
// streams the same number of pixels (to one chunk) with no scheduling work,
// so the warps of an SM finish together (measured: tools/jpass_probe.cu,
// profiles/r2_jpass_probe.txt).  Lane l owns pixels l + 32 k of a chunk, so
// every load of the warp reads 256 contiguous bytes; the next chunk is
// prefetched into registers (two buffers, the loop unrolled by two chunks:
// no register copies).
//
// Per point (the whole hot loop): u = E from the row recurrence
// E_{k+1} = E_k R_k, R_{k+1} = R_k rho (2 DMUL), r = A u + off - z (2),
// u^2, u r (2), the eleven step-index moments (11), sum r, sum r^2 (2):
// 19 FP64 operations.  A chunk's moments are taken about the lane's pixel
// k = (L-1)/2 of the chunk (compile-time powers of the step index), moved to
// dx = 0 by a Taylor shift when the chunk ends and added to the row's; the
// row's are folded with dy^q into the thread's column of a shared-memory
// table at each row change (reading R34).  A row segment whose exponent range
// is unsafe for the recurrence (q >= 600 or a step factor beyond e^300
// anywhere on it) is evaluated with exp per point instead, and a pass whose
// peak is narrower than MOMENT_MIN_WIDTH runs the dual-number body.
//
// Determinism: the chunk -> (warp, lane) map is a function of (m, W, grid),
// every per-thread sum runs in chunk order, the block partial sums the
// thread columns in thread order and the grid combine sums the block
// partials in block order — a pass is bitwise reproducible.
#pragma once

#include "jf_moment.cuh"

namespace jf {

// Row t of the finish map (R33 + R34 composed): K-vector slot t = (j, k) of
// [J | r]^T [J | r] in the paper's parameters as a linear combination of the
// 29 moments (C[t][i], i < NV) and the point count (C[t][NV]).  Column j < 6
// of J is f_j u psi_j(dx, dy) with psi_j a polynomial of degree <= 2 (6
// coefficients over the monomials mono(2, p, q)):
//   j = 0 (A):  f = 1,  psi = 1
//   j = 1 (x0): f = A,  psi = 2a dx + 2b dy
//   j = 2 (y0): f = A,  psi = 2b dx + 2 c2 dy
//   j = 3..5 (sx, sy, th; s = j - 3): f = -A,
//         psi = T[0][s] dx^2 + T[1][s] dx dy + T[2][s] dy^2   (T = d(a, 2b, c2)/d(sx, sy, th))
// column 6 (offset) is 1, column 7 is r.  So G_jk = f_j f_k sum u^2 psi_j psi_k
// (a product of two polynomials: the degree-4 family M2), G_j6 = f_j sum u psi_j
// (M1), G_j7 = f_j sum u r psi_j (MR), G_66 = m, G_67 = sum r, G_77 = sum r^2.
// Straight-line code per slot (one thread per slot).
__device__ __forceinline__ void psi_poly(const PreGauss2D& g, int j, double (&c)[6], double& f) {
  // monomial order mono(2, p, q): 1, dx, dx^2, dy, dx dy, dy^2
#pragma unroll
  for (int i = 0; i < 6; ++i) c[i] = 0.0;
  if (j == 0) {
    f = 1.0;
    c[0] = 1.0;
  } else if (j == 1) {
    f = g.A;
    c[1] = 2.0 * g.a;
    c[3] = g.b2;
  } else if (j == 2) {
    f = g.A;
    c[1] = g.b2;
    c[3] = 2.0 * g.c;
  } else {
    const int sidx = j - 3;
    f = -g.A;
    c[2] = g.T[0 + sidx];
    c[4] = g.T[3 + sidx];
    c[5] = g.T[6 + sidx];
  }
}
__device__ __forceinline__ void finish_map_row(const PreGauss2D& g, int t, double* row /* FMAP_COLS */) {
  constexpr int N = 7;
  int j = 0, rem = t;
  while (rem >= N + 1 - j) {
    rem -= N + 1 - j;
    ++j;
  }
  const int k = j + rem;
  double out[FMAP_COLS];
#pragma unroll
  for (int i = 0; i < FMAP_COLS; ++i) out[i] = 0.0;
  constexpr int MP[6] = {0, 1, 2, 0, 1, 0}, MQ[6] = {0, 0, 0, 1, 1, 2};  // (p, q) of mono(2, ., .)
  if (k < 6) {
    double cj[6], ck[6], fj, fk;
    psi_poly(g, j, cj, fj);
    psi_poly(g, k, ck, fk);
    const double f = fj * fk;
#pragma unroll
    for (int x = 0; x < 6; ++x)
#pragma unroll
      for (int y = 0; y < 6; ++y) {
        const int idx = MomLayout::O2 + mono(4, MP[x] + MP[y], MQ[x] + MQ[y]);
        out[idx] = fma(cj[x], ck[y], out[idx]);
      }
#pragma unroll
    for (int i = 0; i < MomLayout::N2; ++i) out[MomLayout::O2 + i] *= f;
  } else if (j < 6) {
    double cj[6], fj;
    psi_poly(g, j, cj, fj);
    const int base = (k == 6) ? MomLayout::O1 : MomLayout::OR;
#pragma unroll
    for (int x = 0; x < 6; ++x) out[base + x] = fj * cj[x];
  } else if (j == 6) {
    out[k == 6 ? MomLayout::NV : MomLayout::OSR] = 1.0;
  } else {
    out[MomLayout::OSRR] = 1.0;
  }
#pragma unroll
  for (int i = 0; i < FMAP_COLS; ++i) row[i] = out[i];
}

// Where the moment form keeps the pass's accuracy.  Its two regroupings
// cancel for some peak shapes: the chunk-to-row Taylor shift when the peak is
// narrow (amplification ~ (256 px / w)^4, w the smallest principal width
// sqrt(1 / (2 lambda_max)) of the quadratic form [[a, b], [b, c2]]), and the
// chain-rule map T^T (moment Gram) T when it is elongated (the columns
// -A u (dx^2, dx dy, dy^2) become nearly dependent; ~ aspect^4).  Outside
// (w < 48 px or aspect > 12) the pass runs the dual-number body, whose
// per-point rank-1 update does not cancel.
constexpr double MOMENT_MIN_WIDTH = 48.0, MOMENT_MAX_ASPECT = 12.0;
__device__ __forceinline__ bool moment_form_accurate(double a, double b2, double c) {
  const double hb = 0.5 * b2, hd = 0.5 * (a - c);
  const double rt = sqrt(fma(hd, hd, hb * hb));
  const double lmax = 0.5 * (a + c) + rt, lmin = 0.5 * (a + c) - rt;
  return 2.0 * lmax * MOMENT_MIN_WIDTH * MOMENT_MIN_WIDTH <= 1.0 &&
         lmax <= MOMENT_MAX_ASPECT * MOMENT_MAX_ASPECT * lmin;
}

// Out-of-line pieces of the moment kernel's rare paths (row changes, unsafe
// or partial chunks): kept out of the hot loop's register allocation.
struct StreamAcc {
  double P[5], Q[3], R[3], sr, srr;
  int bad;
};
// The thread's row moments (about dx = 0; shared-memory rows NR0.. of its
// column) times dy^q into its moment column (rows 0..26), row moments cleared.
static __device__ __noinline__ void stream_row_fold(double* __restrict__ colbase, int stride, double dy) {
  constexpr int NR0 = MomLayout::KS;
  auto c = [&](int i) -> double& { return colbase[i * stride]; };
  double dq[5];
  dq[0] = 1.0;
  dq[1] = dy;
  dq[2] = dy * dy;
  dq[3] = dq[2] * dy;
  dq[4] = dq[2] * dq[2];
  double rp[11];
#pragma unroll
  for (int i = 0; i < 11; ++i) {
    rp[i] = c(NR0 + i);
    c(NR0 + i) = 0.0;
  }
#pragma unroll
  for (int q = 0; q <= 4; ++q)
#pragma unroll
    for (int p = 0; p + q <= 4; ++p) {
      double& m2 = c(MomLayout::O2 + mono(4, p, q));
      m2 = fma(rp[p], dq[q], m2);
    }
#pragma unroll
  for (int q = 0; q <= 2; ++q)
#pragma unroll
    for (int p = 0; p + q <= 2; ++p) {
      double& m1 = c(MomLayout::O1 + mono(2, p, q));
      m1 = fma(rp[5 + p], dq[q], m1);
      double& mr = c(MomLayout::OR + mono(2, p, q));
      mr = fma(rp[8 + p], dq[q], mr);
    }
}
// A chunk by exp per point (row end, or an exponent range unsafe for the
// recurrence): points c0 + lane + 32 k < W, z read from global memory,
// moments about the chunk origin t = D (k - KC).
template <int L>
__device__ __noinline__ void stream_direct_chunk(StreamAcc& acc, const double* __restrict__ zp, int c0, int lane,
                                                 int W, double dx0, double dy, double ga, double gb2, double gc,
                                                 double A, double off) {
  constexpr int KC = (L - 1) / 2;
  constexpr double D = 32.0;
  for (int k = 0; k < L; ++k) {
    if (c0 + lane + 32 * k < W) {
      const double dx = dx0 + D * k;
      const double u = exp(-(dx * (ga * dx + gb2 * dy) + gc * (dy * dy)));
      const double r = fma(A, u, off) - zp[32 * k];
      acc.bad += isfinite(r) ? 0 : 1;
      const double u2 = u * u, t = D * (k - KC), t2 = t * t, ur = u * r;
      acc.P[0] += u2;
      acc.P[1] = fma(u2, t, acc.P[1]);
      acc.P[2] = fma(u2, t2, acc.P[2]);
      acc.P[3] = fma(u2, t2 * t, acc.P[3]);
      acc.P[4] = fma(u2, t2 * t2, acc.P[4]);
      acc.Q[0] += u;
      acc.Q[1] = fma(u, t, acc.Q[1]);
      acc.Q[2] = fma(u, t2, acc.Q[2]);
      acc.R[0] += ur;
      acc.R[1] = fma(ur, t, acc.R[1]);
      acc.R[2] = fma(ur, t2, acc.R[2]);
      acc.sr += r;
      acc.srr = fma(r, r, acc.srr);
    }
  }
}

// dynamic shared memory: the per-thread folded-moment table [KS][TPB + 1]
// followed by the per-thread row moments [11][TPB + 1]
__host__ __device__ constexpr int moment_stream_smem_bytes(int NW) {
  return (MomLayout::KS + 11) * (NW * 32 + 1) * 8;  // + the row moments (11 per thread)
}

// The end of a moment-form pass (both kernels): the block partial (the thread
// columns of the moment table col[KS][TPB + 1] summed in thread order), the
// grid combine (the last block sums the block partials in block order while
// it builds the finish map), the map, the hand-off.
template <int NW>
__device__ __forceinline__ void moment_stream_tail(const PassArgs& a, FitState* __restrict__ st,
                                                   cudaGraphConditionalHandle cond, int use_cond,
                                                   double* dyn_stream, const PreGauss2D& spre, double off) {
  constexpr int N = 7, KT = tri_count(N), KS2 = KT + 1;
  constexpr int TPB = NW * 32;
  constexpr int KS = MomLayout::KS, NV = MomLayout::NV;
  const int tid = threadIdx.x;
  __shared__ double red[NW][KS];
  __shared__ double vec[KMAX];
  __shared__ double scratch[combine_scratch(TPB)];
  __shared__ double mom[KS];
  // ---- block partial: the thread columns summed in thread order (NW segments of 32)
  static_assert(NW * KS <= TPB, "one (entry, segment) per thread");
  if (tid < NW * KS) {
    const int i = tid % KS, seg = tid / KS;
    const double* c = dyn_stream + i * (TPB + 1) + seg * 32;
    double s4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int j = 0; j < 32; ++j) s4[j & 3] += c[j];
    red[seg][i] = (s4[0] + s4[1]) + (s4[2] + s4[3]);
  }
  __syncthreads();
  if (tid < KS) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < NW; ++w) s += red[w][tid];
    // keep the partial in L2 for the last block (the image streams through evict-first)
    unsigned long long pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(a.partials + (size_t)blockIdx.x * KS + tid),
                 "d"(s), "l"(pol)
                 : "memory");
  }
  // ---- grid combine: the last block sums the block partials in block order
  // (one L2 batch) while it builds the finish map, then maps once
  __shared__ unsigned int tflag;
  const int nblk = gridDim.x;
  __syncthreads();
  if (tid == 0) {
    unsigned prev;
    asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(prev) : "l"(a.ticket) : "memory");
    tflag = (prev == (unsigned)(nblk - 1)) ? 1u : 0u;
  }
  __syncthreads();
  if (!tflag) return;
  dbg_tail(a, 1);
  constexpr int NSEG = TPB / KS;
  double v[16];
  const int rk = tid % KS, rseg = tid / KS;
  double s = 0.0;
  if (tid < NSEG * KS) {  // first batch of loads in flight while the map is built
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int r = rseg + i * NSEG;
      v[i] = (r < nblk) ? __ldcg(a.partials + (size_t)r * KS + rk) : 0.0;
    }
  }
  double (*fmap)[FMAP_COLS] = reinterpret_cast<double (*)[FMAP_COLS]>(dyn_stream);  // the column table is free now
  if (tid < KT) finish_map_row(spre, tid, fmap[tid]);
  if (tid < NSEG * KS) {
#pragma unroll
    for (int i = 0; i < 16; ++i) s += v[i];
    for (int r0 = rseg + 16 * NSEG; r0 < nblk; r0 += 16 * NSEG) {  // grids beyond 16 NSEG blocks
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int r = r0 + i * NSEG;
        v[i] = (r < nblk) ? __ldcg(a.partials + (size_t)r * KS + rk) : 0.0;
      }
#pragma unroll
      for (int i = 0; i < 16; ++i) s += v[i];
    }
    scratch[rseg * KS + rk] = s;
  }
  if (tid == 0) a.ticket[0] = 0u;
  __syncthreads();
  dbg_tail(a, 2);
  if (tid < KS) {
    double t = 0.0;
#pragma unroll
    for (int seg = 0; seg < NSEG; ++seg) t += scratch[seg * KS + tid];
    mom[tid] = t;
  }
  __syncthreads();
  if (tid < KT) {
    double w = fmap[tid][NV] * (double)a.m;
#pragma unroll
    for (int i = 0; i < NV; ++i) w = fma(fmap[tid][i], mom[i], w);
    vec[tid] = w;
  } else if (tid == KT) {
    vec[KT] = mom[NV];  // non-finite count
  }
  __syncthreads();
  dbg_tail(a, 5);
  if (a.no_chain) {  // debug: the K-vector in the alt coordinates (first stage of R33 only)
    moments_to_kvec(spre, (double)a.m, mom, vec);
    __syncthreads();
  }
  dbg_tail(a, 6);
  pass_tail<KS2, TPB, true>(a, st, vec, cond, use_cond);
  dbg_tail(a, 7);
}

template <int L, int NW, int SEEDN>
__global__ void __launch_bounds__(NW * 32, 1)
    moment_stream_kernel(const PassArgs* __restrict__ pa, FitState* __restrict__ st, cudaGraphConditionalHandle cond,
                         int use_cond, const PassArgs av) {
  using Model = ModelGauss2DRot;
  constexpr int N = Model::N, KT = tri_count(N), KS2 = KT + 1;
  constexpr int TPB = NW * 32;
  constexpr int KS = MomLayout::KS, NV = MomLayout::NV, NF = MomLayout::OSR;
  constexpr int CW = 32 * L;
  constexpr double D = 32.0;
  const PassArgs& a = pa ? *pa : av;  // fits: device-resident args (graph replay); else by value
  if (!pass_begin<true, false>(a, st)) {
    qr2_dispatch<Model, COORD_GRID, false, NW * 32>(a, st, cond, use_cond);  // TSQR second pass
    return;
  }
  const double* xs = (a.epilogue == EPI_FIT) ? st->x_eval : a.x;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  // development builds only (JF_DEV): per-warp globaltimer stamps (tools/stamps2.py)
  auto stamp = [&](int slot) {
    if (JF_DEV && a.dbg && lane == 0 && blockIdx.x * NW + wid < 8000) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      a.dbg[(blockIdx.x * NW + wid) * 8 + slot] = t;
      if (slot == 1) {
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        a.dbg[(blockIdx.x * NW + wid) * 8] = smid;
      }
    }
  };
  stamp(1);

  extern __shared__ __align__(16) double dyn_stream[];  // [KS][TPB + 1]
  auto col = [&](int i) -> double& { return dyn_stream[i * (TPB + 1) + tid]; };
  __shared__ PreGauss2D spre;  // the pass's parameters incl. the chain-rule block

  double A, off, ga, gb2, gc, x0, y0;
  {
    double xv[N];
#pragma unroll
    for (int j = 0; j < N; ++j) xv[j] = xs[j];
    const auto pre = Model::template prologue<true>(xv);
    A = pre.g.A, off = pre.off, ga = pre.g.a, gb2 = pre.g.b2, gc = pre.g.c, x0 = pre.g.x0, y0 = pre.g.y0;
    if (tid == 0) spre = pre.g;
  }
  if (!moment_form_accurate(ga, gb2, gc)) {
    pass_body_ool<Model, true, COORD_GRID, false, PassCfg<Model, true>::P, TPB, false>(a, st, cond, use_cond);
    return;
  }
#pragma unroll
  for (int i = 0; i < NF; ++i) col(i) = 0.0;
  stamp(2);

  // every thread reads the pass's parameters from spre below (row set-up,
  // exp seeds): the hot loop keeps only A, off, rho and lane - x0 in registers
  __syncthreads();
  const int W = (int)a.W;
  const int H = (int)(a.m / a.W);
  const int cpr = (W + CW - 1) / CW;
  const int64_t nch = (int64_t)H * cpr;
  const int64_t nw = (int64_t)gridDim.x * NW;
  const int64_t gw = (int64_t)blockIdx.x * NW + wid;
  const int64_t c_begin = gw * nch / nw, c_end = (gw + 1) * nch / nw;
  const int nmy = (int)(c_end - c_begin);  // this warp's chunks
  const double rho = exp(-2.0 * ga * D * D);
  const double xl = (double)lane - x0;     // dx of the lane's pixel in column 0
  const double dyb = (double)a.row0 - y0;  // dy of the shard's row 0

  // Moments of the current chunk about the lane's chunk origin o_c (its
  // pixel k = KC: t = D (k - KC), compile-time), and of the current row about
  // dx = 0 (each chunk folded in by a Taylor shift when it ends).  Keeping the
  // chunk moments local bounds the shift's cancellation by (|t| + |o_c|) / w
  // over the chunk that holds the mass (w: the peak's width along the row):
  // the origin never travels along the row with accumulated mass.
  constexpr int KC = (L - 1) / 2;
  constexpr int NR = 11;  // row moments: RP[0..4], RQ[0..2], RR[0..2] (shared-memory column, per thread)
  double P[5], Q[3], R[3];  // chunk, about o_c
#pragma unroll
  for (int i = 0; i < 5; ++i) P[i] = 0.0;
#pragma unroll
  for (int i = 0; i < 3; ++i) Q[i] = R[i] = 0.0;
  auto rowm = [&](int i) -> double& { return dyn_stream[(KS + i) * (TPB + 1) + tid]; };
#pragma unroll
  for (int i = 0; i < NR; ++i) rowm(i) = 0.0;
  double sr = 0.0, srr = 0.0;
  int bad = 0;

  // the chunk's moments about o_c -> about dx = 0 (Pascal scheme: t -> t + o_c),
  // added to the row's; the chunk's moments restart from zero
  auto chunk_fold = [&](double oc) {
#pragma unroll
    for (int j = 1; j <= 4; ++j)
#pragma unroll
      for (int p = 4; p >= j; --p) P[p] = fma(oc, P[p - 1], P[p]);
#pragma unroll
    for (int j = 1; j <= 2; ++j)
#pragma unroll
      for (int p = 2; p >= j; --p) {
        Q[p] = fma(oc, Q[p - 1], Q[p]);
        R[p] = fma(oc, R[p - 1], R[p]);
      }
#pragma unroll
    for (int i = 0; i < 5; ++i) {
      rowm(i) += P[i];
      P[i] = 0.0;
    }
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      rowm(5 + i) += Q[i];
      rowm(8 + i) += R[i];
      Q[i] = R[i] = 0.0;
    }
  };
  auto fold = [&](double dyv) { stream_row_fold(dyn_stream + tid, TPB + 1, dyv); };

  // position of the chunk being processed (advanced incrementally, 32-bit)
  int row = (int)(c_begin / cpr);
  int cc = (int)(c_begin - (int64_t)row * cpr) - 1;
  int cur_row = -1, jc = 0;
  double dy = 0.0;
  bool row_fast = false;   // the warp's chunks of this row are safe for the recurrence
  bool carried = false;    // E, Rr continue from the previous chunk
  int since_seed = 0;
  double E = 0.0, Rr = 0.0;

  // Load the next chunk in order (lane's points) into zz; a partial (row-end)
  // chunk is predicated.  (lp, lcc): the lane's first point and the column of
  // the next chunk to load.
  int lcc = cc + 1;
  const double* lp = a.z + (int64_t)row * W + lcc * CW + lane;
  const int row_step = W - (cpr - 1) * CW;  // last chunk of a row -> first chunk of the next
  // L2 prefetch PF chunks beyond the one loaded into registers (one bulk
  // prefetch per chunk by lane 0; the register loads then hit L2): rows must
  // start 16-byte aligned for the bulk copy engine, else no prefetch
  constexpr int PF = 2;
  const bool pf_ok = ((reinterpret_cast<uintptr_t>(a.z) & 15) == 0) && ((W & 1) == 0);
  int pcc = lcc, pleft = nmy;
  const double* pp = a.z + (int64_t)row * W + pcc * CW;
  auto prefetch_next = [&]() {  // the next chunk in the prefetch stream
    if (pleft > 0) {
      if (pf_ok && lane == 0) {
        const int c0p = pcc * CW;
        const unsigned bytes = (unsigned)(min(CW, W - c0p) * 8);
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(pp), "r"(bytes) : "memory");
      }
      --pleft;
      if (++pcc == cpr) {
        pcc = 0;
        pp += W - (cpr - 1) * CW;
      } else {
        pp += CW;
      }
    }
  };
#pragma unroll
  for (int q = 0; q < PF; ++q) prefetch_next();
  auto load = [&](double (&zz)[L]) {
    prefetch_next();
    const int c0l = lcc * CW;
    if (c0l + CW <= W) {  // warp-uniform
#pragma unroll
      for (int k = 0; k < L; ++k) zz[k] = __ldcs(lp + 32 * k);
    } else {
#pragma unroll
      for (int k = 0; k < L; ++k) zz[k] = (c0l + lane + 32 * k < W) ? __ldcs(lp + 32 * k) : 0.0;
    }
    if (++lcc == cpr) {
      lcc = 0;
      lp += row_step;
    } else {
      lp += CW;
    }
  };

  // One chunk: zc holds its points.
  auto process = [&](const double (&zc)[L]) {
    if (++cc == cpr) {
      cc = 0;
      ++row;
    }
    if (row != cur_row) {  // warp-uniform: fold the previous row, set up this one
      if (cur_row >= 0) fold(dy);
      cur_row = row;
      dy = (double)row + dyb;
      // the warp's chunks of this row: [cc, cl]; q is convex and argR linear
      // along the row, so the range ends bound them
      const int cl = min(cpr - 1, cc + (nmy - jc) - 1);
      const double sa = spre.a, sb2 = spre.b2, sc = spre.c;
      const double dxa = (double)(cc * CW) + xl;
      const double dxb = (double)(cl * CW + 32 * (L - 1)) + xl;
      const double qa = dxa * (sa * dxa + sb2 * dy) + sc * (dy * dy);
      const double qb = dxb * (sa * dxb + sb2 * dy) + sc * (dy * dy);
      const double ra = D * (2.0 * sa * dxa + sb2 * dy) + sa * D * D;
      const double rb = D * (2.0 * sa * dxb + sb2 * dy) + sa * D * D;
      const bool ok = qa < 600.0 && qb < 600.0 && fabs(ra) < 300.0 && fabs(rb) < 300.0 &&
                      2.0 * sa * D * D * L * SEEDN < 300.0;
      row_fast = __all_sync(FULL, ok);
      carried = false;
    }
    ++jc;
    const int c0 = cc * CW;
    const double dx0 = (double)c0 + xl;
    if (row_fast && c0 + CW <= W) {  // warp-uniform
      if (!carried || ++since_seed >= SEEDN) {
        const double sa = spre.a, sb2 = spre.b2, sc = spre.c;
        const double q0 = dx0 * (sa * dx0 + sb2 * dy) + sc * (dy * dy);
        const double argR = D * (2.0 * sa * dx0 + sb2 * dy) + sa * D * D;
        E = exp(-q0);
        Rr = exp(-argR);
        since_seed = 0;
        carried = true;
      }
      double cs = 0.0;
      const double E_in = E, R_in = Rr;
#pragma unroll
      for (int k = 0; k < L; ++k) {
        const double u = E;
        const double r = fma(A, u, off) - zc[k];  // Eq. 1: r = h - z
        const double u2 = u * u;
        const double k1 = D * (k - KC), k2 = k1 * k1, k3 = k2 * k1, k4 = k2 * k2;
        const double ur = u * r;
        P[0] += u2;
        Q[0] += u;
        R[0] += ur;
        if (k != KC) {
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
      if (!isfinite(cs)) {  // rare: replay the chunk's residuals and count the non-finite ones
        double e = E_in, rr = R_in;
#pragma unroll
        for (int k = 0; k < L; ++k) {
          bad += isfinite(fma(A, e, off) - zc[k]) ? 0 : 1;
          e *= rr;
          rr *= rho;
        }
      }
    } else {
      // row end or an unsafe exponent range: exp per point (out of line)
      carried = false;
      StreamAcc acc;
#pragma unroll
      for (int q = 0; q < 5; ++q) acc.P[q] = P[q];
#pragma unroll
      for (int q = 0; q < 3; ++q) acc.Q[q] = Q[q], acc.R[q] = R[q];
      acc.sr = sr;
      acc.srr = srr;
      acc.bad = bad;
      stream_direct_chunk<L>(acc, a.z + (int64_t)row * W + c0 + lane, c0, lane, W, dx0, dy, spre.a, spre.b2,
                             spre.c, A, off);
#pragma unroll
      for (int q = 0; q < 5; ++q) P[q] = acc.P[q];
#pragma unroll
      for (int q = 0; q < 3; ++q) Q[q] = acc.Q[q], R[q] = acc.R[q];
      sr = acc.sr;
      srr = acc.srr;
      bad = acc.bad;
    }
    chunk_fold(dx0 + D * KC);
  };

  {
    double za[L], zb[L];
    if (nmy > 0) load(za);
    for (int j = 0; j < nmy; j += 2) {
      if (j + 1 < nmy) load(zb);
      process(za);
      if (j + 1 < nmy) {
        if (j + 2 < nmy) load(za);
        process(zb);
      }
    }
  }
  if (cur_row >= 0) fold(dy);
  stamp(3);
  col(MomLayout::OSR) = sr;
  col(MomLayout::OSRR) = srr;
  col(NV) = (double)bad;
  __syncthreads();

  moment_stream_tail<NW>(a, st, cond, use_cond, dyn_stream, spre, off);
}

}  // namespace jf
