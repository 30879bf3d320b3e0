// jf_moment_stream.cuh — the production J-pass for the rotated 2D Gaussian
// (n = 7) on an implicit pixel grid, unweighted: the moment form of R34
// (jf_moment.cuh) with a static, contiguous split of the image over warps and
// the image staged into shared memory by TMA bulk copies.
//
// Same output as every other J-pass — the upper triangle of [J | r]^T [J | r]
// (Eq. 2, Eq. 4, Eq. 5) plus the non-finite count —
// from the 29 moments of jf_moment.cuh's MomLayout, mapped once per pass.
//
// Work split.  The image is a sequence of warp-chunks (32 L consecutive
// pixels of one row; a row's last chunk may be partial).  Warp g of the grid
// owns the contiguous chunk range [f(g), f(g + 1)), f(g) = floor(g nch / nw)
// in fp64 (a monotone partition, no 64-bit division at start-up): every warp
// streams the same number of pixels to one chunk with no scheduling work.
// Lane 0 of each warp streams its chunks into a STG-slot shared-memory ring
// with 1D bulk copies (cp.async.bulk, mbarrier completion, L2 evict-first):
// the first STG copies are issued at kernel entry, before the PDL wait on the
// preceding kernel of a fit and before the prologue; a slot is refilled as
// soon as the warp has consumed it.  Lane l reads pixels l + 32 k of a chunk
// from shared memory.  (Inputs that are not 16-byte aligned or have odd W are
// staged by the lanes.)
//
// Per point (the whole hot loop): u = E from the row recurrence
// E_{k+1} = E_k R_k, R_{k+1} = R_k rho (2 DMUL), r = A u + off - z (2),
// u^2, u r (2), the eleven step-index moments (11), sum r, sum r^2 (2):
// 19 FP64 operations.  A chunk's moments are taken about the lane's pixel
// k = (L-1)/2 of the chunk (compile-time powers of the step index), moved to
// dx = 0 by a Taylor shift when the chunk ends and added to the row's (all
// in registers); at a row change the row's moments are summed over the warp
// and lane i adds entry i of the folded moment vector (x dy^q).  A row
// segment whose exponent range is unsafe for the recurrence (q >= 600 or a
// step factor beyond e^300 anywhere on it) is evaluated with exp per point,
// and a pass whose peak is narrower than MOMENT_MIN_WIDTH or too elongated
// runs the dual-number body.  The parameter-only prologue comes precomputed
// (reading R36) or is computed here.
//
// Determinism: the chunk -> (warp, lane) map is a function of (m, W, grid),
// every per-lane sum runs in chunk order, the warp sums use a fixed xor
// butterfly, the block partial sums the warps in warp order and the grid
// combine sums the block partials in block order — a pass is bitwise
// reproducible.
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

// Out-of-line pieces of the moment kernel's rare paths (unsafe or partial
// chunks): kept out of the hot loop's register allocation.
struct StreamAcc {
  double P[5], Q[3], R[3], sr, srr;
  int bad;
};
// A chunk by exp per point (row end, or an exponent range unsafe for the
// recurrence): points c0 + lane + 32 k < W, z from zp[32 k], moments about
// dx = 0 directly (t = dx: no Taylor shift, so a chunk that holds only a few
// pixels — a row narrower than the chunk — keeps full accuracy).
template <int L>
__device__ __noinline__ void stream_direct_chunk(StreamAcc& acc, const double* __restrict__ zp, int c0, int lane,
                                                 int W, double dx0, double dy, double ga, double gb2, double gc,
                                                 double A, double off) {
  constexpr double D = 32.0;
  for (int k = 0; k < L; ++k) {
    if (c0 + lane + 32 * k < W) {
      const double dx = dx0 + D * k;
      const double u = exp(-(dx * (ga * dx + gb2 * dy) + gc * (dy * dy)));
      const double r = fma(A, u, off) - zp[32 * k];
      acc.bad += isfinite(r) ? 0 : 1;
      const double u2 = u * u, t = dx, t2 = t * t, ur = u * r;
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

// ---- TMA staging of z (1D bulk copies into a per-warp shared-memory ring)
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  unsigned done;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!done);
}
// One elected lane: bytes from global src into shared dst, completing on bar
// (L2 evict-first: the image is read once per pass).
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, unsigned bytes, unsigned long long* bar,
                                           unsigned long long pol) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

// dynamic shared memory of the n = 7 moment J-pass: the z ring [NW][STG][32 L]
__host__ __device__ constexpr int moment_stream_smem_bytes(int NW, int L, int STG) { return NW * STG * 32 * L * 8; }

// The end of a moment-form pass: the block partial (the warps' moment vectors
// wpart[NW][KS] summed in warp order), the grid combine (the last block sums
// the block partials in block order), the finish map (fmap_mem: KT rows of
// FMAP_COLS, built by the block's first idle warp), the hand-off.
template <int NW>
__device__ __forceinline__ void moment_stream_tail(const PassArgs& a, FitState* __restrict__ st,
                                                   cudaGraphConditionalHandle cond, int use_cond,
                                                   const double (*wpart)[MomLayout::KS], const double* fmap_mem,
                                                   const PreGauss2D& spre) {
  constexpr int N = 7, KT = tri_count(N), KS2 = KT + 1;
  constexpr int TPB = NW * 32;
  constexpr int KS = MomLayout::KS, NV = MomLayout::NV;
  const int tid = threadIdx.x;
  __shared__ double vec[KMAX];
  __shared__ double scratch[combine_scratch(TPB)];
  __shared__ double mom[KS];
  if (tid < KS) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < NW; ++w) s += wpart[w][tid];
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
  const double (*fmap)[FMAP_COLS] = reinterpret_cast<const double (*)[FMAP_COLS]>(fmap_mem);
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

// Moment entry i (< OSR) of the layout as (row-moment index v, dy power q):
// M2[mono(4, p, q)] <- RP[p] dy^q, M1 / MR[mono(2, p, q)] <- RQ[p] / RR[p] dy^q.
__device__ __forceinline__ void fold_index(int i, int& v, int& q) {
  q = 0;
  if (i < MomLayout::O1) {
    int r = i;
    while (r >= 5 - q) r -= 5 - q++;
    v = r;
  } else {
    const bool mr = i >= MomLayout::OR;
    int r = i - (mr ? MomLayout::OR : MomLayout::O1);
    while (r >= 3 - q) r -= 3 - q++;
    v = (mr ? 8 : 5) + r;
  }
}

template <int L, int NW, int SEEDN, int STG>
__global__ void __launch_bounds__(NW * 32, 1)
    moment_stream_kernel(const PassArgs* __restrict__ pa, FitState* __restrict__ st, cudaGraphConditionalHandle cond,
                         int use_cond, const PassArgs av) {
  using Model = ModelGauss2DRot;
  constexpr int KS = MomLayout::KS, NF = MomLayout::OSR;
  constexpr int CW = 32 * L;
  constexpr double D = 32.0;
  constexpr int KC = (L - 1) / 2;
  constexpr int NR = 11;  // row moments RP[0..4], RQ[0..2], RR[0..2]
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  // the arguments (fits: device-resident, graph replay; else by value) into
  // shared memory once: every later field access is a shared-memory load
  __shared__ __align__(16) PassArgs sargs;
  __shared__ int fmap_claim;
  {
    constexpr int NA = sizeof(PassArgs) / 8;
    static_assert(sizeof(PassArgs) % 8 == 0 && NA <= NW * 32, "PassArgs copy");
    if (tid < NA)
      reinterpret_cast<unsigned long long*>(&sargs)[tid] =
          pa ? __ldg(reinterpret_cast<const unsigned long long*>(pa) + tid)
             : reinterpret_cast<const unsigned long long*>(&av)[tid];
    if (tid == 0) fmap_claim = 0;
    __syncthreads();
  }
  const PassArgs& a = sargs;
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
  extern __shared__ __align__(128) double zring_all[];  // [NW][STG][CW]
  __shared__ __align__(8) unsigned long long zbar_all[NW * STG];
  __shared__ double wpart[NW][KS];
  __shared__ PreGauss2D spre;
  __shared__ double fmap_s[tri_count(7)][FMAP_COLS];  // finish map (built by the block's first idle warp)
  double* zring = zring_all + wid * STG * CW;
  unsigned long long* zbar = zbar_all + wid * STG;

  // ---- the warp's chunks: a function of (m, W, grid) only, so the first STG
  // copies are issued before this kernel waits for the solver kernel that
  // precedes it in a fit (PDL) and before the prologue
  const int W = (int)a.W;
  const int H = (int)((double)a.m / (double)W);  // (m = H W exactly)
  const int cpr = (W + CW - 1) / CW;
  const int64_t nch = (int64_t)H * cpr;
  // warp g owns chunks [f(g), f(g + 1)), f(g) = floor(g nch / nw) evaluated in
  // double (exact for nch nw < 2^53; any monotone f with f(0) = 0, f(nw) = nch
  // is a partition) — no 64-bit integer division on the start-up path
  const double fnw = (double)nch / (double)(gridDim.x * NW);
  const int gw = blockIdx.x * NW + wid;
  const int64_t c_begin = (int64_t)((double)gw * fnw);
  const int64_t c_end = (gw + 1 == (int)(gridDim.x * NW)) ? nch : (int64_t)((double)(gw + 1) * fnw);
  const int nmy = (int)(c_end - c_begin);
  int row_begin = (int)((double)c_begin / (double)cpr);  // exact quotient after the correction
  if ((int64_t)row_begin * cpr > c_begin) --row_begin;
  if ((int64_t)(row_begin + 1) * cpr <= c_begin) ++row_begin;
  const int cc_begin = (int)(c_begin - (int64_t)row_begin * cpr);
  const bool tma_ok = ((reinterpret_cast<uintptr_t>(a.z) & 15) == 0) && ((W & 1) == 0);
  unsigned long long pol = 0;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  int irow = row_begin, icc = cc_begin;  // the next chunk to copy
  auto issue = [&](int slot) {
    if (lane == 0) {
      const int c0 = icc * CW;
      JF_DCHECK(irow >= 0 && c0 < W && (int64_t)irow * W + min(CW, W - c0) + c0 <= a.m && slot < STG);
      tma_load_1d(zring + slot * CW, a.z + (int64_t)irow * W + c0, (unsigned)(min(CW, W - c0) * 8), zbar + slot, pol);
    }
    if (++icc == cpr) {
      icc = 0;
      ++irow;
    }
  };
  if (lane == 0) {
#pragma unroll
    for (int q = 0; q < STG; ++q) mbar_init(zbar + q);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  if (tma_ok) {
#pragma unroll
    for (int q = 0; q < STG; ++q)
      if (q < nmy) issue(q);
  }
  stamp(4);
  // the copies issued so far complete before the block leaves this kernel
  auto drain = [&]() {
    if (tma_ok)
      for (int q = 0; q < STG && q < nmy; ++q) mbar_wait(zbar + q, 0u);
  };

  // In a fit: the preceding kernel's state (phase, the precomputed prologue)
  // read in one batch of loads after the PDL wait, not one round trip each
  double pf[8];
  int pf_has = 0;
  if (a.epilogue == EPI_FIT) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int ph = __ldcg(&st->phase);
    pf_has = __ldcg(&st->has_pre);
#pragma unroll
    for (int i = 0; i < 8; ++i) pf[i] = __ldcg(&st->pre[i]);
    if (!(ph == PH_INIT_J || ph == PH_TRIAL_J || ph == PH_ACCEPT_J)) {
      pass_begin<true, false>(a, st);  // (the launch count and timeline; returns false)
      drain();
      qr2_dispatch<Model, COORD_GRID, false, NW * 32>(a, st, cond, use_cond);  // TSQR second pass
      return;
    }
  }
  pass_begin<true, false>(a, st);  // (fits: PDL trigger, launch count, timeline)
  const double* xs = (a.epilogue == EPI_FIT) ? st->x_eval : a.x;
  stamp(5);

  // ---- prologue: precomputed by the caller (a.has_pre, fits: by the solver
  // kernel, st->pre) or here (plain doubles; the expressions of
  // Gauss2DComponent::prologue)
  double A, off, ga, gb2, gc, x0, y0, rho;
  if (a.epilogue == EPI_FIT ? pf_has : a.has_pre) {
    const double* pr = (a.epilogue == EPI_FIT) ? pf : a.pre;
    A = pr[0], x0 = pr[1], y0 = pr[2], ga = pr[3], gb2 = pr[4], gc = pr[5], off = pr[6], rho = pr[7];
  } else {
    double pr[8];
    gauss2d_prologue(xs, pr);
    A = pr[0], x0 = pr[1], y0 = pr[2], ga = pr[3], gb2 = pr[4], gc = pr[5], off = pr[6], rho = pr[7];
  }
  stamp(6);
  if (!moment_form_accurate(ga, gb2, gc)) {
    drain();
    pass_body_ool<Model, true, COORD_GRID, false, PassCfg<Model, true>::P, NW * 32, false>(a, st, cond, use_cond);
    return;
  }
  stamp(2);
  const double xl = (double)lane - x0;     // dx of the lane's pixel in column 0
  const double dyb = (double)a.row0 - y0;  // dy of the shard's row 0

  // Moments of the current chunk about the lane's chunk origin o_c (its
  // pixel k = KC: t = D (k - KC), compile-time), of the current row about
  // dx = 0 (each chunk added by a Taylor shift when it ends), and of the
  // warp's rows so far (lane i < NF holds entry i of the moment layout: the
  // row totals over the warp times dy^q, added at each row change).  Keeping
  // the chunk moments local bounds the shift's cancellation by
  // (|t| + |o_c|) / w over the chunk that holds the mass (w: the peak's width
  // along the row): the origin never travels along the row with accumulated mass.
  double P[5], Q[3], R[3];  // chunk, about o_c
  double RM[NR];            // row, about dx = 0
#pragma unroll
  for (int i = 0; i < 5; ++i) P[i] = 0.0;
#pragma unroll
  for (int i = 0; i < 3; ++i) Q[i] = R[i] = 0.0;
#pragma unroll
  for (int i = 0; i < NR; ++i) RM[i] = 0.0;
  double sr = 0.0, srr = 0.0, wacc = 0.0;
  int bad = 0;
  int fv = 0, fq = 0;
  if (lane < NF) fold_index(lane, fv, fq);

  // the row's moments summed over the warp (xor butterfly: every lane gets the
  // same bits), times dy^q into the lane's entry; the row's restart from zero
  auto fold = [&](double dyv) {
#pragma unroll
    for (int v = 0; v < NR; ++v)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) RM[v] += __shfl_xor_sync(FULL, RM[v], o);
    double t = RM[0];
#pragma unroll
    for (int v = 1; v < NR; ++v) t = (fv == v) ? RM[v] : t;
    const double d2 = dyv * dyv;
    const double dq = (fq == 0) ? 1.0 : (fq == 1) ? dyv : (fq == 2) ? d2 : (fq == 3) ? d2 * dyv : d2 * d2;
    if (lane < NF) wacc = fma(t, dq, wacc);
#pragma unroll
    for (int v = 0; v < NR; ++v) RM[v] = 0.0;
  };
  auto chunk_fold = [&](double oc) {  // chunk moments about o_c -> about dx = 0 (Pascal scheme), into the row's
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
      RM[i] += P[i];
      P[i] = 0.0;
    }
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      RM[5 + i] += Q[i];
      RM[8 + i] += R[i];
      Q[i] = R[i] = 0.0;
    }
  };

  int row = row_begin, cc = cc_begin;
  int cur_row = -1;
  double dy = 0.0;
  bool row_fast = false;  // the warp's chunks of this row are safe for the recurrence
  bool carried = false;   // E, Rr continue from the previous chunk
  int since_seed = 0;
  double E = 0.0, Rr = 0.0;
  for (int j = 0; j < nmy; ++j) {
    const int slot = j % STG;
    double* zs = zring + slot * CW;
    const int c0 = cc * CW;
    if (tma_ok) {
      mbar_wait(zbar + slot, (unsigned)(j / STG) & 1u);
    } else {  // (odd W or unaligned z: no bulk copies) the lanes stage the chunk themselves
      const double* zg = a.z + (int64_t)row * W + c0;
      JF_DCHECK(row >= 0 && (int64_t)row * W + min(c0 + CW, W) <= a.m);
#pragma unroll
      for (int k = 0; k < L; ++k) zs[lane + 32 * k] = (c0 + lane + 32 * k < W) ? zg[lane + 32 * k] : 0.0;
      __syncwarp();
    }
    if (row != cur_row) {  // warp-uniform: fold the previous row, set up this one
      if (cur_row >= 0) fold(dy);
      cur_row = row;
      dy = (double)row + dyb;
      // the warp's chunks of this row: [cc, cl]; q is convex and argR linear
      // along the row, so the range ends bound them
      const int cl = min(cpr - 1, cc + (nmy - j) - 1);
      const double dxa = (double)(cc * CW) + xl;
      const double dxb = (double)(cl * CW + 32 * (L - 1)) + xl;
      const double qa = dxa * (ga * dxa + gb2 * dy) + gc * (dy * dy);
      const double qb = dxb * (ga * dxb + gb2 * dy) + gc * (dy * dy);
      const double ra = D * (2.0 * ga * dxa + gb2 * dy) + ga * D * D;
      const double rb = D * (2.0 * ga * dxb + gb2 * dy) + ga * D * D;
      const bool ok = qa < 600.0 && qb < 600.0 && fabs(ra) < 300.0 && fabs(rb) < 300.0 &&
                      2.0 * ga * D * D * L * SEEDN < 300.0;
      row_fast = __all_sync(FULL, ok);
      carried = false;
    }
    const double dx0 = (double)c0 + xl;
    const bool fast = row_fast && c0 + CW <= W;  // warp-uniform
    if (fast) {
      if (!carried || ++since_seed >= SEEDN) {
        const double q0 = dx0 * (ga * dx0 + gb2 * dy) + gc * (dy * dy);
        const double argR = D * (2.0 * ga * dx0 + gb2 * dy) + ga * D * D;
        E = exp(-q0);
        Rr = exp(-argR);
        since_seed = 0;
        carried = true;
      }
      double cs = 0.0;
      const double E_in = E, R_in = Rr;
      const double* zl = zs + lane;
#pragma unroll
      for (int k = 0; k < L; ++k) {
        const double u = E;
        const double r = fma(A, u, off) - zl[32 * k];  // Eq. 1: r = h - z
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
          bad += isfinite(fma(A, e, off) - zl[32 * k]) ? 0 : 1;
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
      stream_direct_chunk<L>(acc, zs + lane, c0, lane, W, dx0, dy, ga, gb2, gc, A, off);
#pragma unroll
      for (int q = 0; q < 5; ++q) P[q] = acc.P[q];
#pragma unroll
      for (int q = 0; q < 3; ++q) Q[q] = acc.Q[q], R[q] = acc.R[q];
      sr = acc.sr;
      srr = acc.srr;
      bad = acc.bad;
    }
    chunk_fold(fast ? dx0 + D * KC : 0.0);  // (direct chunks are already about dx = 0)
    // the slot is free again: refill it with the chunk STG ahead
    __syncwarp();
    if (tma_ok && j + STG < nmy) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(slot);
    }
    if (++cc == cpr) {
      cc = 0;
      ++row;
    }
  }
  if (cur_row >= 0) fold(dy);
  stamp(3);
  // the warp's moment vector: the folded entries (lanes < NF) and the lane sums
  // of sum r, sum r^2 and the non-finite count (xor butterfly)
  double bd = (double)bad;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    sr += __shfl_xor_sync(FULL, sr, o);
    srr += __shfl_xor_sync(FULL, srr, o);
    bd += __shfl_xor_sync(FULL, bd, o);
  }
  if (lane < NF) wpart[wid][lane] = wacc;
  if (lane == 0) {
    wpart[wid][MomLayout::OSR] = sr;
    wpart[wid][MomLayout::OSRR] = srr;
    wpart[wid][MomLayout::NV] = bd;
  }
  // the first warp of the block to get here builds the finish map (the chain
  // rule's T from the dual-number prologue) while the others still stream
  int first = 0;
  if (lane == 0) first = atomicAdd(&fmap_claim, 1);
  if (__shfl_sync(FULL, first, 0) == 0) {
    const PreGauss2D g = Model::template prologue<true>(xs).g;
    if (lane == 0) spre = g;
    for (int t = lane; t < tri_count(7); t += 32) finish_map_row(g, t, fmap_s[t]);
  }
  __syncthreads();
  moment_stream_tail<NW>(a, st, cond, use_cond, wpart, &fmap_s[0][0], spre);
}

}  // namespace jf
