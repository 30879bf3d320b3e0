// jf_moment2.cuh — moment-form J-pass for the sum of two rotated 2D
// Gaussians (GAUSS2D_ROT_X2, n = 13) on an implicit pixel grid, unweighted.
//
// The same reading as jf_moment.cuh (R34) for the two-component model: in
// the alt coordinates every Jacobian column of component c is
// u_c = exp(-q_c) times a polynomial of degree <= 2 in (dX_c, dY_c) =
// (X - x0_c, Y - y0_c), the offset column is 1 and the last column of W is r.
// So every entry of [J|r]^T [J|r] is a fixed linear combination of
//   F11 = sum u1^2 dX1^p dY1^q, F22 = sum u2^2 dX2^p dY2^q,
//   F12 = sum u1 u2 dX1^p dY1^q (p + q <= 4),
//   G_c = sum u_c dX_c^p dY_c^q, H_c = sum u_c r dX_c^p dY_c^q (p + q <= 2),
//   sum r, sum r^2 and m
// (72 moments; component c's families in its own frame, the cross family in
// component 1's).  Per point: two row recurrences (4 DMUL), r (3), u1^2,
// u2^2, u1 u2 (3), fifteen step-index moments of the three products (15),
// six of u_c (6), u_c r (2) and six of them (6), sum r and sum r^2 (2):
// 41 fp64 operations against ~300 for the dual-number rank-1 form of the
// n = 13 triangle (computed twice over, once per grid half).
//
// Scheduling: tasks of TC chunks of one row, taken by the block's warps from
// a shared-memory counter; every task's lane sums land in the task's own slot
// and the block partial adds the slots in task order (bitwise reproducible
// whichever warp ran which task).  The last block maps the summed moment
// vector to the alt-coordinate K-vector (kalt2_slot), applies the two
// chain-rule blocks (apply_chain_kvec) and hands off.
#pragma once

#include "jf_moment_stream.cuh"

namespace jf {

// Moment vector layout of the two-component pass
struct Mom2 {
  static constexpr int F11 = 0, F22 = 15, F12 = 30, G1 = 45, G2 = 51, H1 = 57, H2 = 63;
  static constexpr int OSR = 69, OSRR = 70, NV = 71, KS = 72;
  // running per-lane families (step index t): P11 P22 P12 (5 each), Q1 Q2, R1 R2 (3 each), sr, srr
  static constexpr int NRUN = 29;
};

// (family base in the 72-vector) for the lane-sum rows of the running
// families: rows 0-4 P11, 5-9 P22, 10-14 P12, 15-17 Q1, 18-20 Q2, 21-23 R1,
// 24-26 R2, 27 sr, 28 srr.
__host__ __device__ constexpr int run_row(int fam) {  // fam: 0 P11 1 P22 2 P12 3 Q1 4 Q2 5 R1 6 R2
  return fam < 3 ? 5 * fam : 15 + 3 * (fam - 3);
}

// monomial (p, q) of (dX, dY) relative to the other component's frame:
// (dX1 + dx) for frame shifts — coefficient list of dX1^a dY1^b in
// (dX1 + sx)^p (dY1 + sy)^q, p + q <= 2.
struct ShiftTerms {
  double c[4];
  int p[4], q[4];
  int n;
};
__device__ __forceinline__ ShiftTerms shift_mono(int p, int q, double sx, double sy) {
  ShiftTerms t{};
  t.n = 0;
  // binomial expansion: sum_i sum_k C(p,i) C(q,k) sx^(p-i) sy^(q-k) dX^i dY^k
  for (int i = 0; i <= p; ++i) {
    const double ci = (p == 2 && i == 1) ? 2.0 : 1.0;
    double sxp = 1.0;
    for (int e = 0; e < p - i; ++e) sxp *= sx;
    for (int k = 0; k <= q; ++k) {
      const double ck = (q == 2 && k == 1) ? 2.0 : 1.0;
      double syp = 1.0;
      for (int e = 0; e < q - k; ++e) syp *= sy;
      t.c[t.n] = ci * ck * sxp * syp;
      t.p[t.n] = i;
      t.q[t.n] = k;
      ++t.n;
    }
  }
  return t;
}

// Alt-coordinate K-vector slot (j, k), j <= k <= 13, of the two-component
// model from the moment vector (parameters: the components' PreGauss2D).
__device__ __forceinline__ double kalt2_slot(const PreGauss2D& g1, const PreGauss2D& g2, double m_pts,
                                             const double* mom, int j, int k) {
  constexpr int OFF = 12, RES = 13;
  if (j == OFF) return (k == OFF) ? m_pts : mom[Mom2::OSR];
  if (j == RES) return mom[Mom2::OSRR];
  const int cj = j / 6, jj = j % 6;
  const PreGauss2D& gj = cj == 0 ? g1 : g2;
  const Poly2 a = psi(gj, jj);
  const double fa = (jj == 0 ? 1.0 : gj.A);
  if (k == OFF || k == RES) {
    const int base = (k == OFF) ? (cj == 0 ? Mom2::G1 : Mom2::G2) : (cj == 0 ? Mom2::H1 : Mom2::H2);
    double v = 0.0;
    for (int s = 0; s < 2; ++s) v = fma(a.c[s], mom[base + mono(2, a.p[s], a.q[s])], v);
    return v * fa;
  }
  const int ck = k / 6, kk = k % 6;
  const PreGauss2D& gk = ck == 0 ? g1 : g2;
  const Poly2 b = psi(gk, kk);
  const double f = fa * (kk == 0 ? 1.0 : gk.A);
  double v = 0.0;
  if (cj == ck) {  // F11 / F22 in the component's own frame
    const int base = cj == 0 ? Mom2::F11 : Mom2::F22;
    for (int s = 0; s < 2; ++s)
      for (int u = 0; u < 2; ++u) v = fma(a.c[s] * b.c[u], mom[base + mono(4, a.p[s] + b.p[u], a.q[s] + b.q[u])], v);
  } else {  // F12 in component 1's frame: component 2's monomials shifted (dX2 = dX1 + x0_1 - x0_2)
    const double sx = g1.x0 - g2.x0, sy = g1.y0 - g2.y0;
    for (int s = 0; s < 2; ++s) {
      if (a.c[s] == 0.0) continue;
      for (int u = 0; u < 2; ++u) {
        if (b.c[u] == 0.0) continue;
        const ShiftTerms t = shift_mono(b.p[u], b.q[u], sx, sy);
        double w = 0.0;
        for (int e = 0; e < t.n; ++e) w = fma(t.c[e], mom[Mom2::F12 + mono(4, a.p[s] + t.p[e], a.q[s] + t.q[e])], w);
        v = fma(a.c[s] * b.c[u], w, v);
      }
    }
  }
  return v * f;
}

// The same slot as a short list of (coefficient, moment index) terms —
// kalt2_slot's products expanded (the map is linear in the moments; the
// point count is index M2_COUNT) — so the last block applies a precomputed
// map instead of evaluating kalt2_slot.  At most M2_TERMS terms per slot:
// psi has <= 2 monomials, a shifted monomial of degree <= 2 <= 4 terms, and a
// column's monomials shift to <= 4 terms in all.
constexpr int M2_TERMS = 8, M2_COUNT = 255;
__device__ __forceinline__ int kalt2_terms(const PreGauss2D& g1, const PreGauss2D& g2, int j, int k, double* coef,
                                           unsigned char* idx) {
  constexpr int OFF = 12, RES = 13;
  int n = 0;
  auto add = [&](double c, int i) {
    coef[n] = c;
    idx[n] = (unsigned char)i;
    ++n;
  };
  if (j == OFF) {
    add(1.0, k == OFF ? M2_COUNT : Mom2::OSR);
    return n;
  }
  if (j == RES) {
    add(1.0, Mom2::OSRR);
    return n;
  }
  const int cj = j / 6, jj = j % 6;
  const PreGauss2D& gj = cj == 0 ? g1 : g2;
  const Poly2 a = psi(gj, jj);
  const double fa = (jj == 0 ? 1.0 : gj.A);
  if (k == OFF || k == RES) {
    const int base = (k == OFF) ? (cj == 0 ? Mom2::G1 : Mom2::G2) : (cj == 0 ? Mom2::H1 : Mom2::H2);
    for (int s = 0; s < 2; ++s)
      if (a.c[s] != 0.0) add(fa * a.c[s], base + mono(2, a.p[s], a.q[s]));
    return n;
  }
  const int ck = k / 6, kk = k % 6;
  const PreGauss2D& gk = ck == 0 ? g1 : g2;
  const Poly2 b = psi(gk, kk);
  const double f = fa * (kk == 0 ? 1.0 : gk.A);
  if (cj == ck) {  // F11 / F22 in the component's own frame
    const int base = cj == 0 ? Mom2::F11 : Mom2::F22;
    for (int s = 0; s < 2; ++s)
      for (int u = 0; u < 2; ++u)
        if (a.c[s] != 0.0 && b.c[u] != 0.0)
          add(f * (a.c[s] * b.c[u]), base + mono(4, a.p[s] + b.p[u], a.q[s] + b.q[u]));
  } else {  // F12 in component 1's frame: component 2's monomials shifted
    const double sx = g1.x0 - g2.x0, sy = g1.y0 - g2.y0;
    for (int s = 0; s < 2; ++s) {
      if (a.c[s] == 0.0) continue;
      for (int u = 0; u < 2; ++u) {
        if (b.c[u] == 0.0) continue;
        const ShiftTerms t = shift_mono(b.p[u], b.q[u], sx, sy);
        for (int e = 0; e < t.n; ++e)
          add(f * (a.c[s] * b.c[u]) * t.c[e], Mom2::F12 + mono(4, a.p[s] + t.p[e], a.q[s] + t.q[e]));
      }
    }
  }
  return n;
}

constexpr int MOMENT2_MAXT = 96;  // task slots per block
__host__ __device__ constexpr int moment2_task_smem_bytes(int NW) {
  // task slots, per-warp lane-sum rows, the moments -> K-vector term lists
  return (MOMENT2_MAXT * Mom2::KS + NW * Mom2::NRUN * 33) * 8 + 105 * M2_TERMS * 8 + 105 * M2_TERMS + 105 * 4 + 16;
}

template <int L, int TC, int NW, bool ROLLED = false>
__global__ void __launch_bounds__(NW * 32, 1)
    moment2_task_kernel(const PassArgs* __restrict__ pa, FitState* __restrict__ st, cudaGraphConditionalHandle cond,
                        int use_cond, const PassArgs av) {
  using Model = ModelGauss2DRotX2;
  using Pre = typename Model::Pre;
  constexpr int N = Model::N, KT = tri_count(N), KS2 = KT + 1;
  constexpr int TPB = NW * 32;
  constexpr int KS = Mom2::KS, NR = Mom2::NRUN;
  constexpr int CW = 32 * L;
  constexpr int MAXT = MOMENT2_MAXT;
  constexpr double D = 32.0;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  // the arguments (fits: device-resident, graph replay; else by value) into
  // shared memory once: every later field access is a shared-memory load
  __shared__ __align__(16) PassArgs sargs;
  {
    constexpr int NA = sizeof(PassArgs) / 8;
    static_assert(sizeof(PassArgs) % 8 == 0 && NA <= NW * 32, "PassArgs copy");
    if (tid < NA)
      reinterpret_cast<unsigned long long*>(&sargs)[tid] =
          pa ? __ldg(reinterpret_cast<const unsigned long long*>(pa) + tid)
             : reinterpret_cast<const unsigned long long*>(&av)[tid];
    __syncthreads();
  }
  const PassArgs& a = sargs;
  // in a fit: the state's phase and the precomputed prologue (reading R36)
  // in one batch of loads after the PDL wait
  double pf[15];
  int pf_has = 0;
  if (a.epilogue == EPI_FIT) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int ph = __ldcg(&st->phase);
    pf_has = __ldcg(&st->has_pre);
#pragma unroll
    for (int i = 0; i < 15; ++i) pf[i] = __ldcg(&st->pre[i]);
    if (!(ph == PH_INIT_J || ph == PH_TRIAL_J || ph == PH_ACCEPT_J)) {
      pass_begin<true, false>(a, st);  // (the launch count and timeline; returns false)
      qr2_dispatch<ModelGauss2DRotX2, COORD_GRID, false, NW * 32>(a, st, cond, use_cond);  // TSQR second pass
      return;
    }
  }
  pass_begin<true, false>(a, st);
  const double* xs = (a.epilogue == EPI_FIT) ? st->x_eval : a.x;
  // development builds only (JF_DEV): per-warp globaltimer stamps
  auto stamp = [&](int slot) {
    if (JF_DEV && a.dbg && lane == 0 && blockIdx.x * NW + wid < 8000) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      a.dbg[(blockIdx.x * NW + wid) * 8 + slot] = t;
    }
  };
  stamp(1);

  extern __shared__ __align__(16) double dyn_task2[];
  double (*tslot)[KS] = reinterpret_cast<double (*)[KS]>(dyn_task2);                 // [MAXT][KS]
  double (*wred)[NR][33] = reinterpret_cast<double (*)[NR][33]>(dyn_task2 + MAXT * KS);  // [NW]
  __shared__ double red[NW][KS];
  __shared__ double vec[KMAX];
  __shared__ double scratch[combine_scratch(TPB)];
  __shared__ double mom[KS];
  __shared__ int next_task;
  __shared__ double binom[5][5];

  double A1, A2, off, a1, b1, c1, a2, b2, c2, x01, y01, x02, y02, rho1, rho2;
  {
    double pr[15];
    const double* p = pr;
    if (a.epilogue == EPI_FIT ? pf_has : a.has_pre) {  // precomputed once per pass (R36)
      p = (a.epilogue == EPI_FIT) ? pf : a.pre;
    } else {
      double xv[N];
#pragma unroll
      for (int j = 0; j < N; ++j) xv[j] = xs[j];
      gauss2d_x2_prologue(xv, pr);
    }
    A1 = p[0], x01 = p[1], y01 = p[2], a1 = p[3], b1 = p[4], c1 = p[5];
    A2 = p[6], x02 = p[7], y02 = p[8], a2 = p[9], b2 = p[10], c2 = p[11];
    off = p[12], rho1 = p[13], rho2 = p[14];
  }
  if (!moment_form_accurate(a1, b1, c1) || !moment_form_accurate(a2, b2, c2)) {  // (jf_moment_stream.cuh)
    pass_body_ool<Model, true, COORD_GRID, false, PassCfg<Model, true>::P, TPB, false>(a, st, cond, use_cond);
    return;
  }

  if (tid == 0) next_task = 0;
  if (tid < 25) {
    const int p = tid / 5, i = tid % 5;
    double c = 0.0;
    if (i <= p) {
      c = 1.0;
      for (int j = 0; j < i; ++j) c = c * (p - j) / (j + 1);
    }
    binom[p][i] = c;
  }
  __syncthreads();

  const int W = (int)a.W;
  const int64_t H = a.m / a.W;
  const int64_t row0 = a.row0;
  const int cpr = (W + CW - 1) / CW;
  const int nblk = gridDim.x;
  int tcr = TC < cpr ? TC : cpr;
  // longer tasks (whole sub-runs of TC chunks, at most a row) while the block
  // would have more than MAXT; beyond that the block runs rounds of MAXT tasks
  while (((H * (int64_t)((cpr + tcr - 1) / tcr)) + nblk - 1) / nblk > MAXT && tcr < cpr)
    tcr += (tcr < TC) ? 1 : TC;
  const int tpr = (cpr + tcr - 1) / tcr;
  const int64_t ntask = H * (int64_t)tpr;
  const int64_t t_begin = (int64_t)blockIdx.x * ntask / nblk, t_end = (int64_t)(blockIdx.x + 1) * ntask / nblk;
  const int nt_all = (int)(t_end - t_begin);
  const int nround = nt_all > MAXT ? (nt_all + MAXT - 1) / MAXT : 1;
  int rbase = 0;                             // first task of the current round
  int nt = nt_all < MAXT ? nt_all : MAXT;    // tasks of the current round
  const int64_t row_b = t_begin / tpr;
  const int k_b = (int)(t_begin - row_b * tpr);
  auto task_pos = [&](int t, int64_t& row, int& cc0, int& ncc) {
    const int g = k_b + rbase + t;
    const int dr = g / tpr;
    row = row_b + dr;
    cc0 = (g - dr * tpr) * tcr;
    ncc = min(tcr, cpr - cc0);
  };
  auto grab = [&]() {
    int t = 0;
    if (lane == 0) t = atomicAdd(&next_task, 1);
    return __shfl_sync(FULL, t, 0);
  };
  const double* __restrict__ z = a.z;

  double P11[5], P22[5], P12[5], Q1[3], Q2[3], R1[3], R2[3], sr, srr;
  int bad;
  auto shift = [&](double d) {  // running moments about o -> about o - d (Pascal scheme)
#pragma unroll
    for (int j = 1; j <= 4; ++j)
#pragma unroll
      for (int p = 4; p >= j; --p) {
        P11[p] = fma(d, P11[p - 1], P11[p]);
        P22[p] = fma(d, P22[p - 1], P22[p]);
        P12[p] = fma(d, P12[p - 1], P12[p]);
      }
#pragma unroll
    for (int j = 1; j <= 2; ++j)
#pragma unroll
      for (int p = 2; p >= j; --p) {
        Q1[p] = fma(d, Q1[p - 1], Q1[p]);
        Q2[p] = fma(d, Q2[p - 1], Q2[p]);
        R1[p] = fma(d, R1[p - 1], R1[p]);
        R2[p] = fma(d, R2[p - 1], R2[p]);
      }
  };
  // one point at step t from the origin (any path): u1, u2, z
  auto point = [&](double u1, double u2, double t, double zv, bool count) {
    const double r = fma(A1, u1, fma(A2, u2, off)) - zv;  // Eq. 1
    if (count) bad += isfinite(r) ? 0 : 1;
    const double w11 = u1 * u1, w22 = u2 * u2, w12 = u1 * u2, ur1 = u1 * r, ur2 = u2 * r;
    const double t2 = t * t, t3 = t2 * t, t4 = t2 * t2;
    P11[0] += w11; P11[1] = fma(w11, t, P11[1]); P11[2] = fma(w11, t2, P11[2]); P11[3] = fma(w11, t3, P11[3]); P11[4] = fma(w11, t4, P11[4]);
    P22[0] += w22; P22[1] = fma(w22, t, P22[1]); P22[2] = fma(w22, t2, P22[2]); P22[3] = fma(w22, t3, P22[3]); P22[4] = fma(w22, t4, P22[4]);
    P12[0] += w12; P12[1] = fma(w12, t, P12[1]); P12[2] = fma(w12, t2, P12[2]); P12[3] = fma(w12, t3, P12[3]); P12[4] = fma(w12, t4, P12[4]);
    Q1[0] += u1; Q1[1] = fma(u1, t, Q1[1]); Q1[2] = fma(u1, t2, Q1[2]);
    Q2[0] += u2; Q2[1] = fma(u2, t, Q2[1]); Q2[2] = fma(u2, t2, Q2[2]);
    R1[0] += ur1; R1[1] = fma(ur1, t, R1[1]); R1[2] = fma(ur1, t2, R1[2]);
    R2[0] += ur2; R2[1] = fma(ur2, t, R2[1]); R2[2] = fma(ur2, t2, R2[2]);
    sr += r;
    srr = fma(r, r, srr);
  };

  double zn[L];
  auto load = [&](int64_t row, int cc) {
    const int c0l = cc * CW;
    const double* zp = z + row * (int64_t)W + c0l + lane;
    JF_DCHECK(row >= 0 && row * (int64_t)W + min(c0l + CW, W) <= a.m);
    if (c0l + CW <= W) {  // warp-uniform
#pragma unroll
      for (int k = 0; k < L; ++k) zn[k] = __ldcs(zp + 32 * k);
    } else {
#pragma unroll
      for (int k = 0; k < L; ++k) zn[k] = (c0l + lane + 32 * k < W) ? __ldcs(zp + 32 * k) : 0.0;
    }
  };

  // the components' chain-rule blocks for the last block's tail (dual-number
  // prologue), by one thread of every block at its start: its warp takes
  // fewer tasks (the block's warps grab tasks dynamically)
  __shared__ Pre spre2;
  if (tid == 4 * 32) {
    double xv[N];
#pragma unroll
    for (int j = 0; j < N; ++j) xv[j] = xs[j];
    spre2 = Model::template prologue<true>(xv);
  }
  // ... and the moments -> alt-coordinate K-vector map as term lists, by
  // the block's last four warps (likewise absorbed by the dynamic task grab)
  static_assert(KT == 105, "term-list layout");
  double (*m2coef)[M2_TERMS] = reinterpret_cast<double (*)[M2_TERMS]>(dyn_task2 + MAXT * KS + NW * NR * 33);
  unsigned char (*m2idx)[M2_TERMS] = reinterpret_cast<unsigned char (*)[M2_TERMS]>(m2coef + KT);
  int* m2n = reinterpret_cast<int*>(reinterpret_cast<unsigned char*>(m2idx + KT) + 8 - (KT * M2_TERMS) % 8);
  static_assert(NW >= 4, "four builder warps");
  if (wid >= NW - 4) {
    PreGauss2D g1, g2;
    g1.A = A1, g1.x0 = x01, g1.y0 = y01, g1.a = a1, g1.b2 = b1, g1.c = c1;
    g2.A = A2, g2.x0 = x02, g2.y0 = y02, g2.a = a2, g2.b2 = b2, g2.c = c2;
    for (int t = lane + 32 * (wid - (NW - 4)); t < KT; t += 128) {
      int j = 0, rem = t;
      while (rem >= N + 1 - j) {
        rem -= N + 1 - j;
        ++j;
      }
      m2n[t] = kalt2_terms(g1, g2, j, j + rem, m2coef[t], m2idx[t]);
    }
  }
  constexpr int NSEG = TPB / KS > 0 ? (TPB / KS < NW ? TPB / KS : NW) : 1;
  double bsum = 0.0;  // this thread's (entry, segment) share of the block partial, over the rounds
  for (int rd = 0; rd < nround; ++rd) {
  if (rd > 0) {
    rbase = rd * MAXT;
    nt = min(MAXT, nt_all - rbase);
    if (tid == 0) next_task = 0;
    __syncthreads();
  }
  stamp(2);
  int task = grab();
  int64_t trow = 0;
  int tcc0 = 0, tncc = 0;
  if (task < nt) {
    task_pos(task, trow, tcc0, tncc);
    load(trow, tcc0);
  }
  while (task < nt) {
    const int64_t row = trow;
    const int cc0 = tcc0, ncc = tncc;
    const int my = task;
    const double Y = (double)(row + row0);
    const double dy1 = Y - y01, dy2 = Y - y02;
    int next = nt;
#pragma unroll
    for (int i = 0; i < 5; ++i) P11[i] = P22[i] = P12[i] = 0.0;
#pragma unroll
    for (int i = 0; i < 3; ++i) Q1[i] = Q2[i] = R1[i] = R2[i] = 0.0;
    sr = srr = 0.0;
    bad = 0;
    // origin of the running moments: X of the lane's first pixel of the
    // current sub-run (runs of TC chunks; a task longer than TC chunks —
    // large images, MAXT — is several sub-runs, the origin advanced between
    // them by a Taylor shift)
    double Xo = (double)(cc0 * CW + lane);
    const int nsub = (ncc + TC - 1) / TC;
    for (int sub = 0; sub < nsub; ++sub) {
      if (sub > 0) {  // origin -> the sub-run's first pixel
        const double Xn = (double)((cc0 + sub * TC) * CW + lane);
        shift(Xo - Xn);
        Xo = Xn;
      }
      const int ncs = min(TC, ncc - sub * TC);
      const int ccs = cc0 + sub * TC;
      const bool last_sub = (sub + 1 == nsub);
      const int c0 = ccs * CW;
      const double da1 = Xo - x01, db1 = da1 + D * (TC * L - 1);
      const double da2 = Xo - x02, db2 = da2 + D * (TC * L - 1);
      const double qa1 = da1 * (a1 * da1 + b1 * dy1) + c1 * (dy1 * dy1);
      const double qb1 = db1 * (a1 * db1 + b1 * dy1) + c1 * (dy1 * dy1);
      const double qa2 = da2 * (a2 * da2 + b2 * dy2) + c2 * (dy2 * dy2);
      const double qb2 = db2 * (a2 * db2 + b2 * dy2) + c2 * (dy2 * dy2);
      const double ra1 = D * (2.0 * a1 * da1 + b1 * dy1) + a1 * D * D;
      const double rb1 = D * (2.0 * a1 * db1 + b1 * dy1) + a1 * D * D;
      const double ra2 = D * (2.0 * a2 * da2 + b2 * dy2) + a2 * D * D;
      const double rb2 = D * (2.0 * a2 * db2 + b2 * dy2) + a2 * D * D;
      const bool ok = qa1 < 600.0 && qb1 < 600.0 && qa2 < 600.0 && qb2 < 600.0 && fabs(ra1) < 300.0 &&
                      fabs(rb1) < 300.0 && fabs(ra2) < 300.0 && fabs(rb2) < 300.0 &&
                      2.0 * a1 * D * D * (TC * L) < 300.0 && 2.0 * a2 * D * D * (TC * L) < 300.0;
      const bool fast = (ncs == TC) && (c0 + TC * CW <= W) && __all_sync(FULL, ok);  // warp-uniform
      if (fast) {
        // TC chunks: two row recurrences, t = D (L j + k) from the sub-run's first pixel
        double E1 = exp(-qa1), S1 = exp(-ra1), E2 = exp(-qa2), S2 = exp(-ra2);
#pragma unroll(ROLLED ? 1 : TC)
        for (int j = 0; j < TC; ++j) {
          if (ROLLED && j > 0) {  // rolled: t = D k within the chunk, origin moved per chunk
            shift(-(double)CW);
            Xo += (double)CW;
          }
          double zc[L];
#pragma unroll
          for (int k = 0; k < L; ++k) zc[k] = zn[k];
          if (j + 1 < TC || !last_sub) {
            load(row, ccs + j + 1);
          } else {
            next = grab();
            if (next < nt) {
              task_pos(next, trow, tcc0, tncc);
              load(trow, tcc0);
            }
          }
          const double srr_in = srr;
          const double E1i = E1, S1i = S1, E2i = E2, S2i = S2;
#pragma unroll
          for (int k = 0; k < L; ++k) {
            point(E1, E2, ROLLED ? D * k : D * (L * j + k), zc[k], false);
            E1 *= S1;
            S1 *= rho1;
            E2 *= S2;
            S2 *= rho2;
          }
          if (!isfinite(srr - srr_in)) {  // rare: replay the chunk's residuals, count non-finite ones
            double e1 = E1i, s1 = S1i, e2 = E2i, s2 = S2i;
#pragma unroll
            for (int k = 0; k < L; ++k) {
              bad += isfinite(fma(A1, e1, fma(A2, e2, off)) - zc[k]) ? 0 : 1;
              e1 *= s1;
              s1 *= rho1;
              e2 *= s2;
              s2 *= rho2;
            }
          }
        }
      } else {
        for (int j = 0; j < ncs; ++j) {
          // ragged row end or unsafe exponent range: direct evaluation, t from the sub-run's first pixel
          double zc[L];
#pragma unroll
          for (int k = 0; k < L; ++k) zc[k] = zn[k];
          if (j + 1 < ncs || !last_sub) {
            load(row, ccs + j + 1);
          } else {
            next = grab();
            if (next < nt) {
              task_pos(next, trow, tcc0, tncc);
              load(trow, tcc0);
            }
          }
          const int cj0 = (ccs + j) * CW;
#pragma unroll
          for (int k = 0; k < L; ++k) {
            if (cj0 + lane + 32 * k < W) {
              const double X = (double)(cj0 + lane + 32 * k);
              const double d1 = X - x01, d2 = X - x02;
              const double u1 = exp(-(d1 * (a1 * d1 + b1 * dy1) + c1 * (dy1 * dy1)));
              const double u2 = exp(-(d2 * (a2 * d2 + b2 * dy2) + c2 * (dy2 * dy2)));
              point(u1, u2, X - Xo, zc[k], true);
            }
          }
        }
      }
    }
    // ---- the task's moment vector: lane moments to the common origin
    // (lane 0's first pixel), summed across the warp in lane order, moved to
    // each family's frame and folded with its dY^q
    shift((double)lane);
    {
      double (*wr)[33] = wred[wid];
#pragma unroll
      for (int i = 0; i < 5; ++i) {
        wr[i][lane] = P11[i];
        wr[5 + i][lane] = P22[i];
        wr[10 + i][lane] = P12[i];
      }
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        wr[15 + i][lane] = Q1[i];
        wr[18 + i][lane] = Q2[i];
        wr[21 + i][lane] = R1[i];
        wr[24 + i][lane] = R2[i];
      }
      wr[27][lane] = sr;
      wr[28][lane] = srr;
      const int nbad = __reduce_add_sync(FULL, bad);
      __syncwarp();
      if (lane < NR) {
        double s4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int l = 0; l < 32; ++l) s4[l & 3] += wr[lane][l];
        wr[lane][32] = (s4[0] + s4[1]) + (s4[2] + s4[3]);
      }
      __syncwarp();
      const double X0 = __shfl_sync(FULL, Xo, 0);  // the common origin (absolute X)
      for (int e = lane; e < KS; e += 32) {
        double v;
        if (e < Mom2::OSR) {
          // entry e: family, (p, q), frame
          int fam, base, deg;
          if (e < Mom2::F22) fam = 0, base = Mom2::F11, deg = 4;
          else if (e < Mom2::F12) fam = 1, base = Mom2::F22, deg = 4;
          else if (e < Mom2::G1) fam = 2, base = Mom2::F12, deg = 4;
          else if (e < Mom2::G2) fam = 3, base = Mom2::G1, deg = 2;
          else if (e < Mom2::H1) fam = 4, base = Mom2::G2, deg = 2;
          else if (e < Mom2::H2) fam = 5, base = Mom2::H1, deg = 2;
          else fam = 6, base = Mom2::H2, deg = 2;
          int p = e - base, q = 0;
          while (p > deg - q) {
            p -= deg - q + 1;
            ++q;
          }
          const bool f2 = (fam == 1 || fam == 4 || fam == 6);  // component 2's frame
          const double o = X0 - (f2 ? x02 : x01);              // X0 in the family's frame
          const double dyf = f2 ? dy2 : dy1;
          const int rb = run_row(fam);
          double mv = 0.0;
          for (int i = 0; i <= p; ++i) {  // sum_i C(p, i) o^(p-i) M_i  (Horner in o)
            mv = fma(mv, o, binom[p][i] * wr[rb + i][32]);
          }
          double dq = 1.0;
          for (int t = 0; t < q; ++t) dq *= dyf;
          v = mv * dq;
        } else if (e == Mom2::OSR) {
          v = wr[27][32];
        } else if (e == Mom2::OSRR) {
          v = wr[28][32];
        } else {
          v = (double)nbad;
        }
        tslot[my][e] = v;
      }
      __syncwarp();
    }
    task = next;
  }
  __syncthreads();
  if (tid < NSEG * KS) {  // the round's slots, in slot order, into this thread's share
    const int i = tid % KS, seg = tid / KS;
    for (int t = seg; t < nt; t += NSEG) bsum += tslot[t][i];
  }
  __syncthreads();  // the slots are reused by the next round
  }  // rounds
  stamp(3);

  // ---- block partial: the task slots summed in task order (round by round)
  {
    if (tid < NSEG * KS) red[tid / KS][tid % KS] = bsum;
    __syncthreads();
    unsigned long long pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    for (int k = tid; k < KS; k += TPB) {
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < NSEG; ++w) s += red[w][k];
      asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(a.partials + (size_t)blockIdx.x * KS + k), "d"(s),
                   "l"(pol)
                   : "memory");
    }
  }
  if (!grid_reduce1<KS, TPB>(a, mom, scratch)) return;
  // ---- last block: moments -> alt-coordinate K-vector (the term lists built
  // at the block's start) -> chain rule (the blocks of spre2) -> hand-off
  dbg_tail(a, 5);
  if (tid < KT) {
    const double m_pts = (double)a.m;
    double v = 0.0;
    for (int e = 0; e < m2n[tid]; ++e) {
      const int i = m2idx[tid][e];
      v = fma(m2coef[tid][e], i == M2_COUNT ? m_pts : mom[i], v);
    }
    vec[tid] = v;
  }
  if (tid == 0) vec[KT] = mom[Mom2::NV];
  __syncthreads();
  dbg_tail(a, 6);
  if (!a.no_chain) apply_chain_kvec<Model, TPB>(spre2, vec, scratch);
  dbg_tail(a, 7);
  pass_tail<KS2, TPB, true>(a, st, vec, cond, use_cond);
}

}  // namespace jf
