// jf_moment.cuh — moment-form J-pass for the rotated 2D Gaussian (n = 7) on
// an implicit pixel grid, unweighted.
//
// Same output as pass_kernel<ModelGauss2DRot, JAC=true, COORD_GRID> — the
// upper triangle of [J | r]^T [J | r] (Eqs. 2, 4, 5: cost, J^T r, J^T J) —
// computed with fewer fp64 operations per point by using the model's
// structure.  In the alt coordinates (a, 2b, c2) of jf_models.cuh PreGauss2D
// every Jacobian column of the Gaussian is u = exp(-q) times a polynomial of
// degree <= 2 in (dx, dy):
//   J_A = u,  J_x0 = A u (2a dx + 2b dy),  J_y0 = A u (2b dx + 2 c2 dy),
//   J_a = -A u dx^2,  J_2b = -A u dx dy,  J_c2 = -A u dy^2,  J_off = 1,
// so every entry of the triangle is a fixed linear combination of the moments
//   M2[p][q] = sum u^2 dx^p dy^q  (p + q <= 4),   M1[p][q] = sum u dx^p dy^q,
//   MR[p][q] = sum u r dx^p dy^q  (p + q <= 2),   sum r,  sum r^2,  m.
// Exact algebra (the same sums, regrouped); the map moments -> triangle runs
// once per pass in the last block, then the chain-rule blocks T map the alt
// columns to (sx, sy, th) as for the dual-number kernel.
//
// Per point: u from the row recurrence (2 DMUL), r = A u + off - z (2), the
// moment updates along the row (dx powers; 8 + 4 + 5), sum r and sum r^2 (2),
// dx (1): 25 fp64 operations against ~60 for the rank-1 update of the
// 36-slot triangle.  The dy powers are folded in once per image row a lane
// visits: each warp walks a contiguous range of warp-chunks (32 L pixels of
// one row), so a row's chunks are consecutive.
#pragma once

#include "jf_pass.cuh"

#ifndef JF_TAIL_STAMPS
#define JF_TAIL_STAMPS 0
#endif

namespace jf {

// dynamic shared memory of moment_pass_kernel (the cp.async z ring)
__host__ __device__ constexpr int moment_zbuf_bytes(int L, int TPB, int STAGES) {
  return STAGES >= 2 ? (TPB / 32) * STAGES * L * 32 * 8 : 0;
}

// Moment vector layout: M2 (15) | M1 (6) | MR (6) | sum r | sum r^2 | bad
struct MomLayout {
  static constexpr int N2 = 15, N1 = 6;
  static constexpr int O2 = 0, O1 = 15, OR = 21, OSR = 27, OSRR = 28, NV = 29, KS = 30;
};
// index of dx^p dy^q among the monomials of degree <= D (q-major)
__host__ __device__ constexpr int mono(int D, int p, int q) { return (D + 1) * q - q * (q - 1) / 2 + p; }

// The moment vector -> the K-vector of [J_alt | r] (slot (j, k), j <= k <= 7).
// Thread t < KT computes slot t.  Column j of the Gaussian block is
// J_j = f_j u psi_j (f_0 = 1, f_j = A else) with psi_j = sum of at most two
// monomials c dx^p dy^q, from the formulas above.
struct Poly2 {
  double c[2];
  int p[2], q[2];
};
__device__ __forceinline__ Poly2 psi(const PreGauss2D& g, int j) {
  switch (j) {
    case 0: return {{1.0, 0.0}, {0, 0}, {0, 0}};
    case 1: return {{2.0 * g.a, g.b2}, {1, 0}, {0, 1}};
    case 2: return {{g.b2, 2.0 * g.c}, {1, 0}, {0, 1}};
    case 3: return {{-1.0, 0.0}, {2, 0}, {0, 0}};
    case 4: return {{-1.0, 0.0}, {1, 0}, {1, 0}};
    default: return {{-1.0, 0.0}, {0, 0}, {2, 0}};
  }
}
__device__ __forceinline__ void moments_to_kvec(const PreGauss2D& g, double m_pts, const double* mom, double* vec) {
  constexpr int N = 7, KT = tri_count(N);
  for (int t = threadIdx.x; t < KT; t += blockDim.x) {
    int j = 0, rem = t;
    while (rem >= N + 1 - j) {
      rem -= N + 1 - j;
      ++j;
    }
    const int k = j + rem;
    double v;
    if (k <= 5) {
      const Poly2 a = psi(g, j), b = psi(g, k);
      v = 0.0;
#pragma unroll
      for (int s = 0; s < 2; ++s)
#pragma unroll
        for (int u = 0; u < 2; ++u)
          v = fma(a.c[s] * b.c[u], mom[MomLayout::O2 + mono(4, a.p[s] + b.p[u], a.q[s] + b.q[u])], v);
      v *= (j == 0 ? 1.0 : g.A) * g.A;  // k >= 1 here unless j = k = 0
      if (k == 0) v = mom[MomLayout::O2 + mono(4, 0, 0)];
    } else if (j <= 5) {  // k = 6 (offset column) or k = 7 (residual)
      const int base = (k == 6) ? MomLayout::O1 : MomLayout::OR;
      const Poly2 a = psi(g, j);
      v = 0.0;
#pragma unroll
      for (int s = 0; s < 2; ++s) v = fma(a.c[s], mom[base + mono(2, a.p[s], a.q[s])], v);
      v *= (j == 0 ? 1.0 : g.A);
    } else if (j == 6) {
      v = (k == 6) ? m_pts : mom[MomLayout::OSR];
    } else {
      v = mom[MomLayout::OSRR];
    }
    vec[t] = v;
  }
}

// Last block: combine the grid's moment vectors, map them to the K-vector
// (alt coordinates), apply the chain rule, hand over (pass_tail).  Out of
// line so the prologue's 3x3 blocks never occupy the main loop's registers.
template <int TPB>
__device__ __noinline__ void moment_finish(const PassArgs& a, FitState* __restrict__ st, const double* xs,
                                           double* mom, double* vec, double* scratch,
                                           cudaGraphConditionalHandle cond, int use_cond) {
  using Model = ModelGauss2DRot;
  constexpr int N = Model::N, KT = tri_count(N), KS = KT + 1;
  auto stamp = [&]() {
    if (JF_TAIL_STAMPS && threadIdx.x == 0 && a.epilogue == EPI_FIT) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      const int k = atomicAdd(&st->tl_n, 1);
      if (k < 64) st->tl[k] = t;
    }
  };
  stamp();
  double xv[N];
#pragma unroll
  for (int j = 0; j < N; ++j) xv[j] = xs[j];
  const auto pre = Model::template prologue<true>(xv);
  stamp();
  moments_to_kvec(pre.g, (double)a.m, mom, vec);
  if (threadIdx.x == 0) vec[KT] = mom[MomLayout::NV];  // non-finite count
  __syncthreads();
  stamp();
  if (!a.no_chain) apply_chain_kvec<Model, TPB>(pre, vec, scratch);
  stamp();
  pass_tail<KS, TPB, true>(a, st, vec, cond, use_cond);
}

template <int L, int TPB, int MINB, int SEEDN = 4, int STAGES = 0>
__global__ void __launch_bounds__(TPB, MINB)
    moment_pass_kernel(const PassArgs* __restrict__ pa, FitState* __restrict__ st, cudaGraphConditionalHandle cond,
                       int use_cond) {
  using Model = ModelGauss2DRot;
  constexpr int N = Model::N, KT = tri_count(N), KS = KT + 1;
  constexpr int NV = MomLayout::NV;
  constexpr int CW = 32 * L;
  constexpr double D = 32.0;
  const PassArgs& a = *pa;
  if (!pass_begin<true, false>(a, st)) return;
  const double* xs = (a.epilogue == EPI_FIT) ? st->x_eval : a.x;
  double A, off, ga, gb2, gc, x0, y0;
  {
    double xv[N];
#pragma unroll
    for (int j = 0; j < N; ++j) xv[j] = xs[j];
    const auto pre = Model::template prologue<false>(xv);
    A = pre.g.A, off = pre.off, ga = pre.g.a, gb2 = pre.g.b2, gc = pre.g.c, x0 = pre.g.x0, y0 = pre.g.y0;
  }

  // per-thread moments with dy folded in: shared memory, one column per
  // thread (updated once per image row a lane visits; keeps the registers for
  // the per-point work and more resident warps)
  __shared__ double smom[MomLayout::KS][TPB + 1];  // + sum r, sum r^2, bad at the end; padded rows
  const int tid = threadIdx.x;
#pragma unroll
  for (int i = 0; i < MomLayout::OSR; ++i) smom[i][tid] = 0.0;
  double sr = 0.0, srr = 0.0;
  double P[5], Q[3], R[3];
#pragma unroll
  for (int i = 0; i < 5; ++i) P[i] = 0.0;
#pragma unroll
  for (int i = 0; i < 3; ++i) Q[i] = R[i] = 0.0;
  int bad = 0;

  auto fold = [&](double dy) {  // row moments x dy^q into the thread's moments
    double dq[5];
    dq[0] = 1.0;
    dq[1] = dy;
    dq[2] = dy * dy;
    dq[3] = dq[2] * dy;
    dq[4] = dq[2] * dq[2];
#pragma unroll
    for (int q = 0; q <= 4; ++q)
#pragma unroll
      for (int p = 0; p + q <= 4; ++p) {
        double& m2 = smom[MomLayout::O2 + mono(4, p, q)][tid];
        m2 = fma(P[p], dq[q], m2);
      }
#pragma unroll
    for (int q = 0; q <= 2; ++q)
#pragma unroll
      for (int p = 0; p + q <= 2; ++p) {
        double& m1 = smom[MomLayout::O1 + mono(2, p, q)][tid];
        m1 = fma(Q[p], dq[q], m1);
        double& mr = smom[MomLayout::OR + mono(2, p, q)][tid];
        mr = fma(R[p], dq[q], mr);
      }
#pragma unroll
    for (int i = 0; i < 5; ++i) P[i] = 0.0;
#pragma unroll
    for (int i = 0; i < 3; ++i) Q[i] = R[i] = 0.0;
  };
  // one point: u = exp(-q), dx, data z
  auto point = [&](double u, double dx, double z) {
    const double r = fma(A, u, off) - z;  // Eq. 1: r = h - z
    bad += isfinite(r) ? 0 : 1;
    const double u2 = u * u;
    P[0] += u2;
    P[1] = fma(u2, dx, P[1]);
    const double t1 = u2 * dx;
    P[2] = fma(t1, dx, P[2]);
    const double t2 = t1 * dx;
    P[3] = fma(t2, dx, P[3]);
    const double t3 = t2 * dx;
    P[4] = fma(t3, dx, P[4]);
    Q[0] += u;
    Q[1] = fma(u, dx, Q[1]);
    const double v1 = u * dx;
    Q[2] = fma(v1, dx, Q[2]);
    const double ur = u * r;
    R[0] += ur;
    R[1] = fma(ur, dx, R[1]);
    const double w1 = ur * dx;
    R[2] = fma(w1, dx, R[2]);
    sr += r;
    srr = fma(r, r, srr);
  };

  const int lane = threadIdx.x & 31;
  const int W = (int)a.W;
  const int64_t H = a.m / a.W;
  const int64_t row0 = a.row0;  // PassArgs fields read once (the loop must not reload them)
  const int cpr = (W + CW - 1) / CW;
  const int64_t nch = H * (int64_t)cpr;
  const int64_t nwt = (int64_t)gridDim.x * (TPB / 32);
  const int64_t gw = (int64_t)blockIdx.x * (TPB / 32) + (threadIdx.x >> 5);
  const int64_t c_begin = gw * nch / nwt, c_end = (gw + 1) * nch / nwt;
  const double rho = exp(-2.0 * ga * D * D);
  const double* __restrict__ z = a.z;
  // z staging.  STAGES == 0: the next chunk is prefetched into registers.
  // STAGES >= 2: each lane streams its own points of the next STAGES - 1
  // chunks into a per-warp shared-memory ring with cp.async (LDGSTS,
  // evict-first in L2), freeing the registers for the arithmetic.
  constexpr bool ASYNC = STAGES >= 2;
  extern __shared__ __align__(16) double zbuf[];  // dynamic: moment_zbuf_bytes(L, TPB, STAGES)
  double* wz = zbuf + (ASYNC ? (threadIdx.x >> 5) * STAGES * L * 32 : 0);
  unsigned long long pol = 0;
  if constexpr (ASYNC) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  double zn[ASYNC ? 1 : L];
  // chunk ch = row * cpr + cc; row and cc are advanced incrementally (no
  // 64-bit division in the loop)
  int64_t lrow = c_begin / cpr;  // position of the next chunk to load
  int lcc = (int)(c_begin - lrow * cpr);
  auto load = [&](int stage) {
    const int col = lcc * CW + lane;
    const double* zp = z + lrow * (int64_t)W + col;
    if constexpr (ASYNC) {
#pragma unroll
      for (int k = 0; k < L; ++k) {
        const bool v = col + 32 * k < W;
        const unsigned dst = (unsigned)__cvta_generic_to_shared(wz + (stage * L + k) * 32 + lane);
        asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 8, %2, %3;" ::"r"(dst),
                     "l"(v ? zp + 32 * k : z), "r"(v ? 8 : 0), "l"(pol)
                     : "memory");
      }
    } else {
#pragma unroll
      for (int k = 0; k < L; ++k) zn[k] = (col + 32 * k < W) ? __ldcs(zp + 32 * k) : 0.0;
    }
    if (++lcc == cpr) {
      lcc = 0;
      ++lrow;
    }
  };
  if constexpr (ASYNC) {
#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
      if (c_begin + s < c_end) load(s);
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
  } else {
    if (c_begin < c_end) load(0);
  }
  int64_t cur_row = c_begin / cpr;
  int cc = (int)(c_begin - cur_row * cpr) - 1;  // chunk column of the current chunk (advanced below)
  int64_t row = cur_row;
  double E = 0.0, Rr = 0.0;
  bool carried = false;
  int since_seed = 0;
  int stage = 0;
  for (int64_t ch = c_begin; ch < c_end; ++ch) {
    double zc[ASYNC ? 1 : L];
    const double* zs = wz + stage * L * 32 + lane;  // ASYNC: this chunk's points, stride 32
    if constexpr (ASYNC) {
      const int nxt = stage == 0 ? STAGES - 1 : stage - 1;  // the slot consumed last iteration
      if (ch + STAGES - 1 < c_end) load(nxt);
      asm volatile("cp.async.commit_group;" ::: "memory");
      asm volatile("cp.async.wait_group %0;" ::"n"(STAGES - 1) : "memory");
    } else {
#pragma unroll
      for (int k = 0; k < L; ++k) zc[k] = zn[k];
      if (ch + 1 < c_end) load(0);  // prefetch the next chunk
    }
    auto zat = [&](int k) -> double {
      if constexpr (ASYNC) return zs[32 * k];
      else return zc[k];
    };
    if (++cc == cpr) {
      cc = 0;
      ++row;
    }
    if (row != cur_row) {  // warp-uniform
      fold((double)(cur_row + row0) - y0);
      cur_row = row;
      carried = false;
    }
    const int c0 = cc * CW;
    const double dy = (double)(row + row0) - y0;
    const double dx0 = (double)(c0 + lane) - x0;
    const double q0 = dx0 * (ga * dx0 + gb2 * dy) + gc * (dy * dy);
    const double argR = D * (2.0 * ga * dx0 + gb2 * dy) + ga * D * D;
    const bool ok = fabs(q0) < 600.0 && fabs(argR) < 300.0 && 2.0 * ga * D * D * L < 300.0;
    const bool full = c0 + CW <= W;  // warp-uniform
    if (full && __all_sync(FULL, ok)) {
      // E, Rr continue from the previous chunk of the same row (its last
      // step lands on this chunk's first pixel); re-seeded by exp at a row
      // start, after a direct-evaluation chunk, and every SEEDN chunks so the
      // recurrence's rounding stays below ~(16 SEEDN)^2 / 2 ulp
      if (!carried || ++since_seed >= SEEDN) {  // warp-uniform
        E = exp(-q0);
        Rr = exp(-argR);
        since_seed = 0;
      }
      // moments in the local step index k (dx = dx0 + D k): the k^p are
      // compile-time constants, so each update is one FMA
      double a2[5] = {0.0, 0.0, 0.0, 0.0, 0.0}, a1[3] = {0.0, 0.0, 0.0}, ar[3] = {0.0, 0.0, 0.0};
#pragma unroll
      for (int k = 0; k < L; ++k) {
        const double u = E;
        const double r = fma(A, u, off) - zat(k);  // Eq. 1: r = h - z
        bad += isfinite(r) ? 0 : 1;
        const double u2 = u * u;
        const double k1 = (double)k, k2 = k1 * k1, k3 = k2 * k1, k4 = k2 * k2;
        a2[0] += u2;
        a2[1] = fma(u2, k1, a2[1]);
        a2[2] = fma(u2, k2, a2[2]);
        a2[3] = fma(u2, k3, a2[3]);
        a2[4] = fma(u2, k4, a2[4]);
        a1[0] += u;
        a1[1] = fma(u, k1, a1[1]);
        a1[2] = fma(u, k2, a1[2]);
        const double ur = u * r;
        ar[0] += ur;
        ar[1] = fma(ur, k1, ar[1]);
        ar[2] = fma(ur, k2, ar[2]);
        sr += r;
        srr = fma(r, r, srr);
        E *= Rr;
        Rr *= rho;
      }
      carried = true;
      // shift to dx: sum w (dx0 + D k)^p = sum_i C(p, i) dx0^(p-i) D^i sum w k^i
      const double d1 = dx0, d2 = d1 * d1, d3 = d2 * d1, d4 = d2 * d2;
      const double s1 = D * a2[1], s2 = (D * D) * a2[2], s3 = (D * D * D) * a2[3], s4 = (D * D * D * D) * a2[4];
      P[0] += a2[0];
      P[1] += fma(d1, a2[0], s1);
      P[2] += fma(d2, a2[0], fma(2.0 * d1, s1, s2));
      P[3] += fma(d3, a2[0], fma(3.0 * d2, s1, fma(3.0 * d1, s2, s3)));
      P[4] += fma(d4, a2[0], fma(4.0 * d3, s1, fma(6.0 * d2, s2, fma(4.0 * d1, s3, s4))));
      const double t1 = D * a1[1], t2 = (D * D) * a1[2];
      Q[0] += a1[0];
      Q[1] += fma(d1, a1[0], t1);
      Q[2] += fma(d2, a1[0], fma(2.0 * d1, t1, t2));
      const double v1 = D * ar[1], v2 = (D * D) * ar[2];
      R[0] += ar[0];
      R[1] += fma(d1, ar[0], v1);
      R[2] += fma(d2, ar[0], fma(2.0 * d1, v1, v2));
    } else {
      // ragged row end or unsafe exponent range: direct evaluation
      carried = false;
#pragma unroll
      for (int k = 0; k < L; ++k) {
        if (c0 + lane + 32 * k < W) {
          const double dx = dx0 + 32.0 * k;
          point(exp(-(dx * (ga * dx + gb2 * dy) + gc * (dy * dy))), dx, zat(k));
        }
      }
    }
    stage = (stage + 1 == (ASYNC ? STAGES : 1)) ? 0 : stage + 1;
  }
  if (c_begin < c_end) fold((double)(cur_row + row0) - y0);

  // block partial of the moment vector
  __shared__ double red[TPB / 32][MomLayout::KS];
  __shared__ double vec[KMAX];
  __shared__ double scratch[combine_scratch(TPB)];
  __shared__ double mom[MomLayout::KS];
  {
    // block partial: the threads' columns of smom summed by rows, NSEG
    // segments of 32 threads each, then the segments in order
    smom[MomLayout::OSR][tid] = sr;
    smom[MomLayout::OSRR][tid] = srr;
    smom[NV][tid] = (double)bad;
    __syncthreads();
    constexpr int NSEG = TPB / 32;
    static_assert(NSEG * MomLayout::KS <= TPB, "one (row, segment) per thread");
    if (tid < NSEG * MomLayout::KS) {
      const int i = tid % MomLayout::KS, seg = tid / MomLayout::KS;
      double s = 0.0;
#pragma unroll 8
      for (int j = 0; j < 32; ++j) s += smom[i][seg * 32 + j];
      red[seg][i] = s;
    }
    __syncthreads();
    for (int k = tid; k < MomLayout::KS; k += TPB) {
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < NSEG; ++w) s += red[w][k];
      a.partials[(size_t)blockIdx.x * MomLayout::KS + k] = s;
    }
  }
  if (!grid_reduce<MomLayout::KS, TPB>(a, mom, scratch)) return;
  moment_finish<TPB>(a, st, xs, mom, vec, scratch, cond, use_cond);
}

}  // namespace jf
