// jf_solver.cuh — the n x n trust-region subproblem and the iteration control
// of a fit, run on the device between passes.
//
// Everything the paper runs "in NumPy on the CPU" between passes (P:226, P:343:
// the alpha sub-problem and the radius logic) runs here, in the solver kernel
// that follows every pass kernel, so a fit never returns to the host.
//
//   Alg. 1  outer loop; Gauss-Newton trial p_t = -B^-1 g (l.141)
//   Alg. 2  LM parameter alpha: Eq. 13 phi, Eq. 14 Newton update,
//                       safeguard max{0.001 u, sqrt(l u)}
//   Alg. 3  accept / reject and radius update, Eq. 15 gain ratio
//   App. B  SVD basis: here the eigendecomposition of the scaled
//                       Gram  B_hat = D^-1 J^T J D^-1 = V diag(s^2) V^T, so
//                       S^T U^T r = V^T g_hat ("suf") — identical in exact
//                       arithmetic.
// Readings R3-R27 of DESIGN.md §3 fix what the paper leaves open (SciPy TRF
// semantics, P:42 / P:246), including the Coleman-Li bounded path (R19, R20).
//
// Execution model: the work between passes is a few hundred flops on n <= 16
// vectors, a chain of dependent steps.  It runs as plain scalar code on lane 0
// over shared memory (no shuffle or barrier latency per step); the one
// parallel kernel, the Jacobi eigensolver, uses the whole warp and is only
// entered when a trial needs alpha > 0 or the rank test cannot be certified
// from the Cholesky factor (gn_fastpath below).
#pragma once

#include <cfloat>
#include <cmath>

#include "jf_common.cuh"
#include "jf_state.cuh"

namespace jf {

constexpr int MS = NMAX + 1;  // shared-memory matrix row stride

struct SolverSmem {
  double A[NMAX][MS];   // eigensolver input / output (diagonal)
  double V[NMAX][MS];   // eigenvectors (columns)
  double M[NMAX][MS];   // B_hat (incl. diag_h): quadratic forms
  double T[NMAX][MS];   // scratch (Cholesky factor, warm-start product)
  double M2[NMAX][MS];  // scratch
  double lam[NMAX];     // eigenvalues, descending
  double w1[NMAX], w2[NMAX], w3[NMAX], w4[NMAX], w5[NMAX];
  double cinv[NMAX];
  double kvs[KMAX];  // the pass's K-vector (shared-memory copy)
  double Q[2 * NMAX][MS];  // TSQR: [R_hat; diag(sqrt(diag_h))] (rows x n), SVD input
  double caug[2 * NMAX];   // TSQR: [c; 0]
  double sufq[NMAX];       // TSQR: suf = a_k . [c; 0] from the one-sided Jacobi
  int need_eig, need_trial, fast;
};

// ------------------------------------------------------ scalar vector helpers
template <int n>
__device__ __forceinline__ double vdot(const double* a, const double* b) {
  double s = 0.0;
#pragma unroll
  for (int j = 0; j < n; ++j) s = fma(a[j], b[j], s);
  return s;
}
template <int n>
__device__ __forceinline__ double vnorm(const double* a) { return sqrt(vdot<n>(a, a)); }
// y = M x (row-major, stride MS)
template <int n>
__device__ __forceinline__ void vmatvec(const double (*M)[MS], const double* x, double* y) {
  for (int i = 0; i < n; ++i) {
    double s = 0.0;
    for (int k = 0; k < n; ++k) s = fma(M[i][k], x[k], s);
    y[i] = s;
  }
}
// x^T M x
template <int n>
__device__ __forceinline__ double vquad(const double (*M)[MS], const double* x) {
  double s = 0.0;
  for (int i = 0; i < n; ++i) {
    double r = 0.0;
    for (int k = 0; k < n; ++k) r = fma(M[i][k], x[k], r);
    s = fma(x[i], r, s);
  }
  return s;
}

// ---------------------------------------------------- symmetric eigensolver
// Parallel (round-robin) cyclic Jacobi on the n x n symmetric matrix in S.A,
// the whole warp cooperating: on return S.lam holds the eigenvalues sorted
// descending and the columns of S.V the matching orthonormal eigenvectors —
// App. B's SVD of the scaled Jacobian computed through its Gram (c.1b).
//
// Register-resident: lane j owns column j of A and of V (n padded to an even
// N2 with a zero row/column).  Round r of a sweep rotates the N2/2 disjoint
// pairs of the circle schedule (partner of i: 2r - i mod N2-1, N2-1 <-> r)
// at once: both lanes of a pair compute the same rotation, the column update
// takes the partner's column by shuffle, the row update every pair's (c, s);
// the round loop is unrolled so every row index is static.
//
// warm != 0: S.V holds an orthogonal V0 on entry (an earlier iterate's
// eigenvectors); the sweeps run on V0^T A V0 and accumulate onto V0.  A
// rotation is skipped when |a_pq| <= eps sqrt(|a_pp a_qq|) or |a_pq| <=
// 2^-60 max_i |a_ii|; the sweeps stop when one applies none.
template <int N2>
__device__ __forceinline__ int jacobi_regs(double (&a)[N2], double (&v)[N2], int lane, double abs_tol) {
  int sweeps = 0;
  for (int sweep = 0; sweep < 40; ++sweep) {
    ++sweeps;
    bool any = false;
#pragma unroll
    for (int r = 0; r < N2 - 1; ++r) {
      int pj;
      if (lane == N2 - 1) pj = r;
      else if (lane == r) pj = N2 - 1;
      else pj = ((2 * r - lane) % (N2 - 1) + (N2 - 1)) % (N2 - 1);
      const bool act = lane < N2;
      if (!act) pj = lane;
      double dj = 0.0, apq = 0.0;
#pragma unroll
      for (int i = 0; i < N2; ++i) {
        if (i == lane) dj = a[i];
        if (i == pj) apq = a[i];
      }
      const double dq = __shfl_sync(FULL, dj, pj);
      const bool lo = lane < pj;
      const double app = lo ? dj : dq, aqq = lo ? dq : dj;
      double c = 1.0, s = 0.0;
      const double aa = fabs(apq);
      bool rot = false;
      if (act && !(aa <= abs_tol || aa <= 1.1102230246251565e-16 * sqrt(fabs(app) * fabs(aqq)))) {
        // t = tan(phi), the smaller root: 2 apq sgn(d) / (|d| + sqrt(d^2 + 4 apq^2)), d = aqq - app
        const double d = aqq - app;
        const double t = (2.0 * apq) * (d >= 0.0 ? 1.0 : -1.0) / (fabs(d) + sqrt(fma(d, d, 4.0 * apq * apq)));
        c = rsqrt(fma(t, t, 1.0));
        s = t * c;
        rot = true;
      }
      // P[p][p] = P[q][q] = c, P[p][q] = s, P[q][p] = -s;  e_j = P[partner j][j]
      const double e = lo ? -s : s;
      if (!__any_sync(FULL, rot)) continue;
      any = true;
#pragma unroll
      for (int i = 0; i < N2; ++i) {  // B = A P
        const double pc = __shfl_sync(FULL, a[i], pj);
        a[i] = fma(c, a[i], e * pc);
      }
      double na[N2];
#pragma unroll
      for (int i = 0; i < N2; ++i) {  // A' = P^T B
        const int pi = (i == N2 - 1) ? r : (i == r ? N2 - 1 : ((2 * r - i) % (N2 - 1) + (N2 - 1)) % (N2 - 1));
        const double ci = __shfl_sync(FULL, c, i), ei = __shfl_sync(FULL, e, i);
        na[i] = fma(ci, a[i], ei * a[pi]);
      }
#pragma unroll
      for (int i = 0; i < N2; ++i) a[i] = (rot && i == pj) ? 0.0 : na[i];
#pragma unroll
      for (int i = 0; i < N2; ++i) {  // V' = V P
        const double pv = __shfl_sync(FULL, v[i], pj);
        v[i] = fma(c, v[i], e * pv);
      }
    }
    if (!any) break;
  }
  return sweeps;
}

template <int N2>
__device__ __forceinline__ int eig_regs(SolverSmem& S, int n, int lane, double abs_tol) {
  double a[N2], v[N2];
#pragma unroll
  for (int i = 0; i < N2; ++i) {
    a[i] = (lane < n && i < n) ? S.A[i][lane] : 0.0;
    v[i] = (lane < n && i < n) ? S.V[i][lane] : ((i == lane) ? 1.0 : 0.0);
  }
  const int sw = jacobi_regs<N2>(a, v, lane, abs_tol);
  __syncwarp();
#pragma unroll
  for (int i = 0; i < N2; ++i) {
    if (lane < n && i < n) {
      S.V[i][lane] = v[i];
      if (i == lane) S.A[i][i] = a[i];
    }
  }
  __syncwarp();
  return sw;
}

// All 32 lanes.  In: S.A (n x n symmetric), S.V = V0 if warm.  Out: S.lam, S.V.
static __device__ __noinline__ int warp_eig(SolverSmem& S, int n, int warm) {
  const int lane = threadIdx.x & 31;
  if (!warm) {
    for (int e = lane; e < NMAX * NMAX; e += 32) {
      const int i = e / NMAX, j = e % NMAX;
      S.V[i][j] = (i == j) ? 1.0 : 0.0;
    }
    __syncwarp();
  } else {
    for (int e = lane; e < n * n; e += 32) {  // T = A V0
      const int i = e / n, j = e % n;
      double t = 0.0;
      for (int k = 0; k < n; ++k) t = fma(S.A[i][k], S.V[k][j], t);
      S.T[i][j] = t;
    }
    __syncwarp();
    for (int e = lane; e < n * n; e += 32) {  // V0^T T (upper half)
      const int i = e / n, j = e % n;
      if (i <= j) {
        double t = 0.0;
        for (int k = 0; k < n; ++k) t = fma(S.V[k][i], S.T[k][j], t);
        S.M2[i][j] = t;
      }
    }
    __syncwarp();
    for (int e = lane; e < n * n; e += 32) {
      const int i = e / n, j = e % n;
      S.A[i][j] = (i <= j) ? S.M2[i][j] : S.M2[j][i];  // exactly symmetric
    }
    __syncwarp();
  }
  double amax = 0.0;
  for (int i = 0; i < n; ++i) amax = fmax(amax, fabs(S.A[i][i]));
  const double abs_tol = amax * 8.673617379884035e-19;  // 2^-60
  const int N2 = (n + 1) & ~1;
  int sweeps;
  switch (N2) {
    case 2: sweeps = eig_regs<2>(S, n, lane, abs_tol); break;
    case 4: sweeps = eig_regs<4>(S, n, lane, abs_tol); break;
    case 6: sweeps = eig_regs<6>(S, n, lane, abs_tol); break;
    case 8: sweeps = eig_regs<8>(S, n, lane, abs_tol); break;
    case 10: sweeps = eig_regs<10>(S, n, lane, abs_tol); break;
    case 12: sweeps = eig_regs<12>(S, n, lane, abs_tol); break;
    case 14: sweeps = eig_regs<14>(S, n, lane, abs_tol); break;
    default: sweeps = eig_regs<16>(S, n, lane, abs_tol); break;
  }
  // sort descending (ties by index); permute the columns of V accordingly
  int rank = 0;
  const double lj = (lane < n) ? S.A[lane][lane] : 0.0;
  for (int k = 0; k < n; ++k) {
    const double lk = S.A[k][k];
    if (lane < n && (lk > lj || (lk == lj && k < lane))) ++rank;
  }
  for (int e = lane; e < n * n; e += 32) {
    const int i = e / n, j = e % n;
    S.T[i][j] = S.V[i][j];
  }
  __syncwarp();
  if (lane < n) {
    S.lam[rank] = lj;
    for (int i = 0; i < n; ++i) S.V[i][rank] = S.T[i][lane];
  }
  __syncwarp();
  return sweeps;
}

// One-sided (Hestenes) Jacobi SVD of the rows x n matrix in S.Q (rows <= 32),
// the whole warp: lane j owns column j (padded to an even N2 with zero
// columns); a round of the circle schedule orthogonalises N2/2 disjoint column
// pairs (p, q) at once by the rotation that zeroes a_p . a_q (both lanes
// compute it from alpha = |a_p|^2, beta = |a_q|^2, gamma = a_p . a_q after
// exchanging columns by shuffle).  At convergence the columns are
// a_j = s_j u_j: S.lam = s^2 (descending), S.V, S.sufq = a_j . [c; 0]
// (= s_j u_j^T [c; 0] = suf, App. B's S^T U^T r for the TSQR mode).
template <int N2>
__device__ __forceinline__ int svd_regs(SolverSmem& S, int n, int rows, int lane) {
  constexpr int R = 2 * NMAX;
  double a[R], v[N2];
#pragma unroll
  for (int i = 0; i < R; ++i) a[i] = (lane < n && i < rows) ? S.Q[i][lane] : 0.0;
#pragma unroll
  for (int i = 0; i < N2; ++i) v[i] = (i == lane) ? 1.0 : 0.0;
  int sweeps = 0;
  for (int sweep = 0; sweep < 40; ++sweep) {
    ++sweeps;
    bool any = false;
#pragma unroll
    for (int r = 0; r < N2 - 1; ++r) {
      int pj;
      if (lane == N2 - 1) pj = r;
      else if (lane == r) pj = N2 - 1;
      else pj = ((2 * r - lane) % (N2 - 1) + (N2 - 1)) % (N2 - 1);
      const bool act = lane < N2;
      if (!act) pj = lane;
      double pc[R];
      double al = 0.0, be = 0.0, ga = 0.0;
#pragma unroll
      for (int i = 0; i < R; ++i) {
        pc[i] = __shfl_sync(FULL, a[i], pj);
        al = fma(a[i], a[i], al);
        be = fma(pc[i], pc[i], be);
        ga = fma(a[i], pc[i], ga);
      }
      const bool lo = lane < pj;
      const double app = lo ? al : be, aqq = lo ? be : al;
      double c = 1.0, sn = 0.0;
      bool rot = false;
      if (act && fabs(ga) > 2.220446049250313e-16 * sqrt(app * aqq) && ga != 0.0) {
        // zeta = (aqq - app) / (2 gamma); t = sgn(zeta) / (|zeta| + sqrt(1 + zeta^2))
        const double zeta = (aqq - app) / (2.0 * ga);
        const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(fma(zeta, zeta, 1.0)));
        c = rsqrt(fma(t, t, 1.0));
        sn = c * t;
        rot = true;
      }
      // a_p' = c a_p - s a_q, a_q' = s a_p + c a_q  ->  own' = c own + e partner
      const double e = lo ? -sn : sn;
      if (!__any_sync(FULL, rot)) continue;
      any = true;
#pragma unroll
      for (int i = 0; i < R; ++i) a[i] = fma(c, a[i], e * pc[i]);
#pragma unroll
      for (int i = 0; i < N2; ++i) {
        const double pv = __shfl_sync(FULL, v[i], pj);
        v[i] = fma(c, v[i], e * pv);
      }
    }
    if (!any) break;
  }
  // singular values, suf = a_j . c_aug, sort descending
  double s2 = 0.0, sf = 0.0;
#pragma unroll
  for (int i = 0; i < R; ++i) {
    s2 = fma(a[i], a[i], s2);
    sf = fma(a[i], S.caug[i], sf);
  }
  if (lane >= n) {
    s2 = 0.0;
    sf = 0.0;
  }
  int rank = 0;
  for (int k = 0; k < n; ++k) {
    const double sk = __shfl_sync(FULL, s2, k);
    if (lane < n && (sk > s2 || (sk == s2 && k < lane))) ++rank;
  }
  __syncwarp();
  if (lane < n) {
    S.lam[rank] = s2;
    S.sufq[rank] = sf;
#pragma unroll
    for (int i = 0; i < N2; ++i)
      if (i < n) S.V[i][rank] = v[i];
  }
  __syncwarp();
  return sweeps;
}

static __device__ __noinline__ int warp_svd(SolverSmem& S, int n, int rows) {
  const int lane = threadIdx.x & 31;
  const int N2 = (n + 1) & ~1;
  switch (N2) {
    case 2: return svd_regs<2>(S, n, rows, lane);
    case 4: return svd_regs<4>(S, n, rows, lane);
    case 6: return svd_regs<6>(S, n, rows, lane);
    case 8: return svd_regs<8>(S, n, rows, lane);
    case 10: return svd_regs<10>(S, n, rows, lane);
    case 12: return svd_regs<12>(S, n, rows, lane);
    case 14: return svd_regs<14>(S, n, rows, lane);
    default: return svd_regs<16>(S, n, rows, lane);
  }
}

// ---------------------------------------------- TSQR: CholeskyQR2 factors
// W = [J | r] (m x (n+1)).  Pass 1 gives G1 = W^T W; R1 = chol(G1) (upper),
// P = R1^-1 is applied to every row in pass 2, whose Gram G2 = P^T G1 P ~ I
// gives R2 = chol(G2) and R = R2 R1 with the accuracy of a Householder TSQR
// for cond(W) < ~1e8 (one Gram pass alone loses cond(W)^2).  R = [[R_J, c],
// [0, rho]]: g = R_J^T c, J^T J = R_J^T R_J, 2 cost = |c|^2 + rho^2.
// Lane 0; matrices row-major with stride n+1.

// upper Cholesky of the Gram packed in a K-vector; false if not SPD
template <int n>
__device__ __forceinline__ bool chol_kv(const double* kv, double* R, double shift = 0.0) {
  constexpr int N1 = n + 1;
  for (int i = 0; i < N1; ++i)
    for (int j = 0; j < N1; ++j) R[i * N1 + j] = (j >= i) ? kv[tri_slot(n, i, j)] + (i == j ? shift : 0.0) : 0.0;
  for (int k = 0; k < N1; ++k) {
    double d = R[k * N1 + k];
    for (int j = 0; j < k; ++j) d = fma(-R[j * N1 + k], R[j * N1 + k], d);
    if (!(d > 0.0)) return false;
    const double rk = sqrt(d);
    const double inv = 1.0 / rk;
    R[k * N1 + k] = rk;
    for (int i = k + 1; i < N1; ++i) {
      double t = R[k * N1 + i];
      for (int j = 0; j < k; ++j) t = fma(-R[j * N1 + k], R[j * N1 + i], t);
      R[k * N1 + i] = t * inv;
    }
  }
  return true;
}

// P = R^-1 for upper-triangular R
template <int n>
__device__ __forceinline__ void tri_inv(const double* R, double* P) {
  constexpr int N1 = n + 1;
  for (int i = 0; i < N1 * N1; ++i) P[i] = 0.0;
  for (int j = 0; j < N1; ++j) {
    P[j * N1 + j] = 1.0 / R[j * N1 + j];
    for (int i = j - 1; i >= 0; --i) {
      double t = 0.0;
      for (int k = i + 1; k <= j; ++k) t = fma(R[i * N1 + k], P[k * N1 + j], t);
      P[i * N1 + j] = -t / R[i * N1 + i];
    }
  }
}

// --------------------------------------------------- Alg. 2 + App. B (scalar)
// In: S.lam (descending eigenvalues of B_hat), S.V, suf = V^T g_hat, radius
// Delta, warm-start alpha, m (number of residuals, R6).  Out: p, alpha;
// returns the number of Moré iterations (0 = Gauss-Newton step).
template <int n>
__device__ __noinline__ int solve_tr(SolverSmem& S, int64_t m, const double* suf, double Delta, double& alpha, double* p) {
  double* s = S.w4;  // singular values s = sqrt(max(lam, 0))
  double* coef = S.w5;
  for (int j = 0; j < n; ++j) s[j] = sqrt(fmax(S.lam[j], 0.0));
  const bool full_rank = (m >= n) && (s[n - 1] > DBL_EPSILON * (double)m * s[0]);  // R6
  if (full_rank) {  // Alg. 1 l.141: p_t = -V (uf / s), uf = suf / s
    for (int j = 0; j < n; ++j) coef[j] = -((suf[j] / s[j]) / s[j]);
    vmatvec<n>(S.V, coef, p);
    if (vnorm<n>(p) <= Delta) {  // Alg. 1 l.142
      alpha = 0.0;
      return 0;
    }
  }
  double u = vnorm<n>(suf) / Delta;  // Alg. 2 l.160
  double l = 0.0;
  // phi(alpha) = ||suf / (s^2 + alpha)|| - Delta  (Eq. 13);  phi' per R11
  auto phi_d = [&](double a, double& phi, double& dphi) {
    double pn2 = 0.0, t = 0.0;
    for (int j = 0; j < n; ++j) {
      const double den = s[j] * s[j] + a;
      const double q = suf[j] / den;
      pn2 = fma(q, q, pn2);
      t += suf[j] * suf[j] / (den * den * den);
    }
    const double pn = sqrt(pn2);
    phi = pn - Delta;
    dphi = -t / pn;
  };
  if (full_rank) {
    double phi, dphi;
    phi_d(0.0, phi, dphi);
    l = -phi / dphi;  // Alg. 2 l.161
  }
  if (!full_rank && alpha == 0.0) alpha = fmax(0.001 * u, sqrt(l * u));
  int it = 0;
  for (it = 0; it < 10; ++it) {  // R9
    if (alpha < l || alpha > u) alpha = fmax(0.001 * u, sqrt(l * u));
    double phi, dphi;
    phi_d(alpha, phi, dphi);
    if (phi < 0.0) u = alpha;  // Alg. 2 l.173
    const double ratio = phi / dphi;
    l = fmax(l, alpha - ratio);                       // Alg. 2 l.172
    alpha = alpha - ((phi + Delta) / Delta) * ratio;  // Eq. 14
    if (fabs(phi) < 0.01 * Delta) break;              // R9
  }
  for (int j = 0; j < n; ++j) coef[j] = -(suf[j] / (s[j] * s[j] + alpha));  // Eq. B4 (sign R8)
  vmatvec<n>(S.V, coef, p);
  const double sc = Delta / vnorm<n>(p);  // R12
  for (int j = 0; j < n; ++j) p[j] *= sc;
  return it + 1;
}

// ------------------------------------------- Alg. 1 l.141: p_t = -B^-1 g
// The Gauss-Newton trial of Alg. 1 by a Cholesky solve of the
// scaled Gram, B_hat p = -g_hat.  App. B obtains the same p from the SVD; the
// SVD (here: the eigendecomposition) is only needed when the trial is
// rejected (||p|| > Delta) and Alg. 2 searches for alpha > 0, or when the rank
// test R6 (s_min > EPS m s_max) cannot be certified.  The certificate is
// conservative: s_max^2 <= trace(B_hat) and s_min^2 >= 1 / ||L^-1||_F^2
// (B_hat = L L^T), so 1/||L^-1||_F > 2 EPS m sqrt(trace) implies R6.
// Returns 1 with p when the certified trial lies inside the trust region.
// Register-resident Cholesky (lane 0, n compile-time so every loop unrolls
// and every index is static): lower L of the SPD matrix in L (in place),
// cinv = 1 / diag(L); false if a pivot is not positive.
template <int n>
__device__ __forceinline__ bool chol_reg(double (&L)[n][n], double (&cinv)[n]) {
#pragma unroll
  for (int k = 0; k < n; ++k) {
    double d = L[k][k];
#pragma unroll
    for (int j = 0; j < k; ++j) d = fma(-L[k][j], L[k][j], d);
    if (!(d > 0.0)) return false;
    const double r = rsqrt(d);
    L[k][k] = d * r;
    cinv[k] = r;
#pragma unroll
    for (int i = k + 1; i < n; ++i) {
      double t = L[i][k];
#pragma unroll
      for (int j = 0; j < k; ++j) t = fma(-L[i][j], L[k][j], t);
      L[i][k] = t * r;
    }
  }
  return true;
}
// ||L^-1||_F^2 with Y = L^-1 (lower) returned
template <int n>
__device__ __forceinline__ double inv_fro2(const double (&L)[n][n], const double (&cinv)[n], double (&Y)[n][n]) {
  double fro = 0.0;
#pragma unroll
  for (int c = 0; c < n; ++c) {
#pragma unroll
    for (int i = c; i < n; ++i) {
      double t = (i == c) ? 1.0 : 0.0;
#pragma unroll
      for (int k = c; k < i; ++k) t = fma(-L[i][k], Y[k][c], t);
      Y[i][c] = t * cinv[i];
      fro = fma(Y[i][c], Y[i][c], fro);
    }
  }
  return fro;
}

template <int n>
__device__ __noinline__ int gn_fastpath(SolverSmem& S, int64_t m, const double* gh, double Delta, double* p,
                                        double& kappa2) {
  double L[n][n], Y[n][n], cinv[n];
  double tr = 0.0;
  kappa2 = INFINITY;
#pragma unroll
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int j = 0; j <= i; ++j) L[i][j] = S.M[i][j];
    tr += L[i][i];
  }
  if (!chol_reg<n>(L, cinv)) return 0;
  const double fro = inv_fro2<n>(L, cinv, Y);
  kappa2 = tr * fro;  // >= cond(B_hat) (lambda_max <= tr, lambda_min >= 1 / ||L^-1||_F^2)
  if (!(m >= n && rsqrt(fro) > 2.0 * DBL_EPSILON * (double)m * sqrt(tr))) return 0;
  double w[n], pr[n];
#pragma unroll
  for (int i = 0; i < n; ++i) {  // L w = -g_hat
    double t = -gh[i];
#pragma unroll
    for (int k = 0; k < i; ++k) t = fma(-L[i][k], w[k], t);
    w[i] = t * cinv[i];
  }
#pragma unroll
  for (int i = n - 1; i >= 0; --i) {  // L^T p = w
    double t = w[i];
#pragma unroll
    for (int k = i + 1; k < n; ++k) t = fma(-L[k][i], pr[k], t);
    pr[i] = t * cinv[i];
  }
  double pn = 0.0;
#pragma unroll
  for (int i = 0; i < n; ++i) {
    p[i] = pr[i];
    pn = fma(pr[i], pr[i], pn);
  }
  return sqrt(pn) <= Delta ? 1 : 0;
}

// --------------------------------------------------- Coleman-Li helpers (R19)
// Smallest t >= 0 with x + t s on a bound; hits[j] = sign(s_j) where attained.
__device__ __forceinline__ double step_to_bound(const double* x, const double* s, const double* lb, const double* ub,
                                                int n, int* hits) {
  double tmin = INFINITY;
  double st[NMAX];
  for (int j = 0; j < n; ++j) {
    st[j] = INFINITY;
    if (s[j] != 0.0) st[j] = fmax((lb[j] - x[j]) / s[j], (ub[j] - x[j]) / s[j]);
    tmin = fmin(tmin, st[j]);
  }
  if (hits) {
    for (int j = 0; j < n; ++j) hits[j] = (st[j] == tmin) ? (s[j] > 0.0 ? 1 : (s[j] < 0.0 ? -1 : 0)) : 0;
  }
  return tmin;
}

// 1-D quadratic minimiser on [lo, hi]: candidates lo, hi, vertex (R20)
__device__ __forceinline__ void min_quad_1d(double a, double b, double lo, double hi, double c, double& t_out,
                                            double& y_out) {
  double ts[3] = {lo, hi, 0.0};
  int nt = 2;
  if (a != 0.0) {
    const double ext = -0.5 * b / a;
    if (lo < ext && ext < hi) ts[nt++] = ext;
  }
  double best = ts[0] * (a * ts[0] + b) + c;
  double bt = ts[0];
  for (int k = 1; k < nt; ++k) {
    const double y = ts[k] * (a * ts[k] + b) + c;
    if (y < best) {
      best = y;
      bt = ts[k];
    }
  }
  t_out = bt;
  y_out = best;
}

// Q(s) = 1/2 s^T B s + g^T s  (B = B_hat incl. diag_h; R13)
template <int n>
__device__ __forceinline__ double eval_quad(const SolverSmem& S, const double* gh, const double* s) {
  return 0.5 * vquad<n>(S.M, s) + vdot<n>(s, gh);
}

// Coleman-Li step selection (R19, R20).  In: p_h, d, x, lb, ub, g_hat.
// Out: step (original space), step_h (hat space), predicted reduction, branch
// (0 interior, 1 reflected, 2 truncated, 3 scaled gradient).
template <int n>
__device__ __noinline__ void select_step(SolverSmem& S, const double* x, const double* lb, const double* ub, const double* gh, const double* d, const double* p_h, double Delta, double theta, double* step, double* step_h, double& pred, int& branch) {
  double p[NMAX], ph[NMAX], r_h[NMAX], r[NMAX], xb[NMAX], ag_h[NMAX], ag[NMAX], tmp[NMAX];
  bool inb = true;
  for (int j = 0; j < n; ++j) {
    p[j] = d[j] * p_h[j];
    const double xn = x[j] + p[j];
    inb = inb && xn >= lb[j] && xn <= ub[j];
  }
  if (inb) {
    for (int j = 0; j < n; ++j) {
      step[j] = p[j];
      step_h[j] = p_h[j];
    }
    pred = -eval_quad<n>(S, gh, p_h);
    branch = 0;
    return;
  }
  int hits[NMAX];
  const double t_b = step_to_bound(x, p, lb, ub, n, hits);
  for (int j = 0; j < n; ++j) {
    r_h[j] = hits[j] ? -p_h[j] : p_h[j];
    r[j] = d[j] * r_h[j];
    p[j] *= t_b;
    ph[j] = p_h[j] * t_b;
    xb[j] = x[j] + p[j];
  }
  double to_tr;  // positive root of ||ph + t r_h|| = Delta (stable form)
  {
    const double a = vdot<n>(r_h, r_h), b = vdot<n>(ph, r_h), c = vdot<n>(ph, ph) - Delta * Delta;
    const double dd = sqrt(b * b - a * c);
    const double q = -(b + copysign(dd, b));
    to_tr = fmax(q / a, c / q);
  }
  const double to_bd = step_to_bound(xb, r, lb, ub, n, nullptr);
  const double rs = fmin(to_bd, to_tr);
  double lo, hi;
  if (rs > 0.0) {
    lo = (1.0 - theta) * t_b / rs;
    hi = (rs == to_bd) ? theta * to_bd : to_tr;
  } else {
    lo = 0.0;
    hi = -1.0;
  }
  double r_val;
  if (lo <= hi) {  // Q(ph + t r_h) = a t^2 + b t + c
    vmatvec<n>(S.M, r_h, tmp);
    const double a = 0.5 * vdot<n>(r_h, tmp);
    const double b = vdot<n>(gh, r_h) + vdot<n>(ph, tmp);
    const double c = 0.5 * vquad<n>(S.M, ph) + vdot<n>(gh, ph);
    double rt;
    min_quad_1d(a, b, lo, hi, c, rt, r_val);
    for (int j = 0; j < n; ++j) {
      r_h[j] = ph[j] + rt * r_h[j];
      r[j] = r_h[j] * d[j];
    }
  } else {
    r_val = INFINITY;
  }
  for (int j = 0; j < n; ++j) {
    p[j] *= theta;
    ph[j] *= theta;
  }
  const double p_val = eval_quad<n>(S, gh, ph);
  for (int j = 0; j < n; ++j) {
    ag_h[j] = -gh[j];
    ag[j] = d[j] * ag_h[j];
  }
  const double t_tr = Delta / vnorm<n>(ag_h);
  const double t_bd = step_to_bound(x, ag, lb, ub, n, nullptr);
  const double stride = (t_bd < t_tr) ? theta * t_bd : t_tr;
  double at, ag_val;
  {
    const double a = 0.5 * vquad<n>(S.M, ag_h);
    const double b = vdot<n>(gh, ag_h);
    min_quad_1d(a, b, 0.0, stride, 0.0, at, ag_val);
  }
  for (int j = 0; j < n; ++j) {
    ag_h[j] *= at;
    ag[j] *= at;
  }
  const double* ss;
  const double* sh;
  if (p_val < r_val && p_val < ag_val) {
    ss = p;
    sh = ph;
    pred = -p_val;
    branch = 2;
  } else if (r_val < p_val && r_val < ag_val) {
    ss = r;
    sh = r_h;
    pred = -r_val;
    branch = 1;
  } else {
    ss = ag;
    sh = ag_h;
    pred = -ag_val;
    branch = 3;
  }
  for (int j = 0; j < n; ++j) {
    step[j] = ss[j];
    step_h[j] = sh[j];
  }
}

// rstep = 0 strict feasibility (R19): x <= lb -> nextafter(lb, ub), x >= ub ->
// nextafter(ub, lb); still outside -> midpoint.
__device__ __forceinline__ double strict_feasible0(double x, double lb, double ub) {
  double xn = x;
  if (x <= lb) xn = nextafter(lb, ub);
  else if (x >= ub) xn = nextafter(ub, lb);
  if (xn < lb || xn > ub) xn = 0.5 * (lb + ub);
  return xn;
}

// strict feasibility with rstep > 0 (R18/R19: the bounded start): an active
// bound (within rstep max(1, |bound|)) moves to bound +- that; still outside
// -> midpoint.
__device__ __forceinline__ double strict_feasible_r(double x, double lb, double ub, double rstep) {
  double xn = x;
  const double ld = x - lb, ud = ub - x;
  const double lt = rstep * fmax(1.0, fabs(lb)), ut = rstep * fmax(1.0, fabs(ub));
  if (isfinite(lb) && ld <= fmin(ud, lt)) xn = lb + lt;
  else if (isfinite(ub) && ud <= fmin(ld, ut)) xn = ub - ut;
  if (xn < lb || xn > ub) xn = 0.5 * (lb + ub);
  return xn;
}

// Coleman-Li vector v, dv (R19)
__device__ __forceinline__ void cl_vector(double x, double g, double lb, double ub, double& v, double& dv) {
  v = 1.0;
  dv = 0.0;
  if (g < 0.0 && isfinite(ub)) {
    v = ub - x;
    dv = -1.0;
  }
  if (g > 0.0 && isfinite(lb)) {
    v = x - lb;
    dv = 1.0;
  }
}

// ======================================================= the state machine
// Everything below runs on lane 0 only (st and S are in shared memory).

__device__ __forceinline__ void st_trace(FitState* st, double cost_new, double ratio) {
  if (st->trace_cap > 0 && st->trace_len < st->trace_cap) {
    double* rec = st->trace + (int64_t)st->trace_len * TRACE_FIELDS;
    rec[0] = st->nit;
    rec[1] = st->nfev;
    rec[2] = st->njev;
    rec[3] = st->cost;
    rec[4] = cost_new;
    rec[5] = st->Delta_used;
    rec[6] = st->alpha;
    rec[7] = ratio;
    rec[8] = st->hn;
    rec[9] = st->step_norm;
    rec[10] = st->pred;
    rec[11] = st->bounded ? st->branch : -1;
    st->trace_len = st->trace_len + 1;
  }
}

// (cost, g, G) at the current iterate from a J-pass K-vector.
template <int n>
__device__ __forceinline__ void st_take_pass(FitState* st, const double* kv) {
  for (int j = 0; j < n; ++j) {
    st->g[j] = kv[tri_slot(n, j, n)];
    for (int k = j; k < n; ++k) {
      const double v = kv[tri_slot(n, j, k)];
      st->G[j * NMAX + k] = v;
      st->G[k * NMAX + j] = v;
    }
  }
  st->cost = 0.5 * kv[tri_slot(n, n, n)];
}

// scale_inv from the Gram diagonal (reading R3: column norms of J = sqrt(G_jj))
template <int n>
__device__ __forceinline__ void st_update_scale(FitState* st, bool first) {
  for (int j = 0; j < n; ++j) {
    double si = sqrt(st->G[j * NMAX + j]);
    if (first) {
      if (si == 0.0) si = 1.0;
    } else {
      si = fmax(si, st->scale_inv[j]);
    }
    st->scale_inv[j] = si;
  }
}

// Trial, part 1: the Gauss-Newton fast path; sets S.need_eig when Alg. 2 or
// the exact rank test needs the eigendecomposition (computed by the warp).
template <int n>
__device__ __noinline__ void st_trial_begin(FitState* st, SolverSmem& S, bool have_M = false) {
  if (!have_M) {
    double M[n][n];
#pragma unroll
    for (int i = 0; i < n; ++i)
#pragma unroll
      for (int j = 0; j < n; ++j) M[i][j] = st->Gh[i * NMAX + j];
#pragma unroll
    for (int i = 0; i < n; ++i)
#pragma unroll
      for (int j = 0; j < n; ++j) S.M[i][j] = M[i][j];
  }
  S.need_trial = 1;
  S.fast = 0;
  S.need_eig = 0;
  if (!st->have_eig && st->qr_mode) {
    S.need_eig = 1;  // TSQR: the SVD of R_hat, no Cholesky shortcut
  } else if (!st->have_eig) {
    const long long c0 = clock64();
    double k2;
    S.fast = gn_fastpath<n>(S, st->m_global, st->gh, st->Delta, S.w3, k2);
    st->kappa2_gn = k2;
    st->prof[1] += clock64() - c0;
    if (!S.fast) S.need_eig = 1;
  }
}

// Trial, part 2: Alg. 2 (if not fast), the Coleman-Li selection, the trial
// point x_new staged in x_eval, and the phase of the next pass.
template <int n>
__device__ __noinline__ void st_trial_finish(FitState* st, SolverSmem& S) {
  const double Delta = st->Delta;
  double alpha = st->alpha;
  double* p_h = S.w3;
  if (S.fast) {
    alpha = 0.0;  // Alg. 1 l.142-144: p_k = p_t (SciPy returns alpha = 0)
  } else {
    if (S.need_eig) {  // the warp just computed it: keep it for retried trials
      for (int j = 0; j < n; ++j) {
        st->lam[j] = S.lam[j];
        for (int i = 0; i < n; ++i) st->V[i * NMAX + j] = S.V[i][j];
      }
      for (int j = 0; j < n; ++j) {  // S^T U^T r = V^T g_hat (c.1b); TSQR: a_j . [c; 0]
        double t = 0.0;
        for (int i = 0; i < n; ++i) t = fma(S.V[i][j], st->gh[i], t);
        st->suf[j] = st->qr_mode ? S.sufq[j] : t;
      }
      st->have_eig = 1;
      st->have_V = 1;
    } else {
      for (int j = 0; j < n; ++j) {
        S.lam[j] = st->lam[j];
        for (int i = 0; i < n; ++i) S.V[i][j] = st->V[i * NMAX + j];
      }
    }
    const long long c0 = clock64();
    solve_tr<n>(S, st->m_global, st->suf, Delta, alpha, p_h);
    st->prof[2] += clock64() - c0;
  }
  double pred;
  int branch = -1;
  if (st->bounded) {
    select_step<n>(S, st->x, st->lb, st->ub, st->gh, st->d, p_h, Delta, st->theta, st->step, st->step_h, pred, branch);
    for (int j = 0; j < n; ++j) st->x_eval[j] = strict_feasible0(st->x[j] + st->step[j], st->lb[j], st->ub[j]);
  } else {
    for (int j = 0; j < n; ++j) st->step_h[j] = p_h[j];
    pred = -eval_quad<n>(S, st->gh, p_h);  // Eq. 15 denominator (R13)
    for (int j = 0; j < n; ++j) {
      st->step[j] = st->d[j] * p_h[j];  // Alg. 3 l.185: w = D^-1 p
      st->x_eval[j] = st->x[j] + st->step[j];
    }
  }
  st->alpha = alpha;
  st->pred = pred;
  st->hn = vnorm<n>(st->step_h);
  st->step_norm = vnorm<n>(st->step);
  st->Delta_used = Delta;
  st->branch = branch;
  st->phase = (st->policy == 1) ? PH_TRIAL_R : PH_TRIAL_J;
  S.need_trial = 0;
}

// Alg. 1 loop top: termination by gtol / max_nfev, then the hat space of the
// new iterate (Eq. 7-8).  Requests a trial unless the fit is over.
template <int n>
__device__ __noinline__ void st_outer_top(FitState* st, SolverSmem& S) {
  double gnorm = 0.0;
  double v[NMAX], dv[NMAX];
  for (int j = 0; j < n; ++j) {
    v[j] = 1.0;
    dv[j] = 0.0;
    if (st->bounded) cl_vector(st->x[j], st->g[j], st->lb[j], st->ub[j], v[j], dv[j]);
    gnorm = fmax(gnorm, fabs(st->g[j] * v[j]));
  }
  if (gnorm < st->gtol) st->status = 1;  // R16
  st->gnorm = gnorm;
  if (st->status != STATUS_NONE || st->nfev == st->max_nfev) {
    if (st->status == STATUS_NONE) st->status = 0;
    st->phase = PH_DONE;
    st->cont = 0;
    return;
  }
  // register copies first: every load is issued before any store (the
  // state lives in shared memory; interleaved stores would serialise them).
  // n > 8: G read in place (a register copy would spill)
  constexpr int NG = n <= 8 ? n : 1;
  double dd[n], dh[n], gj[n], G[NG][NG];
  const bool bounded = st->bounded;
#pragma unroll
  for (int j = 0; j < n; ++j) {
    gj[j] = st->g[j];
    if constexpr (n <= 8) {
#pragma unroll
      for (int k = 0; k < n; ++k) G[j][k] = st->G[j * NMAX + k];
    }
  }
#pragma unroll
  for (int j = 0; j < n; ++j) {
    const double si = st->scale_inv[j];
    if (bounded) {
      double vj = v[j];
      if (dv[j] != 0.0) vj *= si;
      dd[j] = sqrt(vj) / si;          // R19: d = v^0.5 * scale
      dh[j] = gj[j] * dv[j] / si;      // C = diag(g * scale) Jv
    } else {
      dd[j] = 1.0 / si;  // Eq. 8: J_hat = J D^-1
      dh[j] = 0.0;
    }
  }
#pragma unroll
  for (int j = 0; j < n; ++j) {
    st->d[j] = dd[j];
    st->diag_h[j] = dh[j];
    st->gh[j] = dd[j] * gj[j];
  }
#pragma unroll
  for (int i = 0; i < n; ++i) {  // B_hat = d G d (+ diag_h)
#pragma unroll
    for (int j = 0; j < n; ++j) {
      double b;
      if constexpr (n <= 8) b = dd[i] * G[i][j] * dd[j];
      else b = dd[i] * st->G[i * NMAX + j] * dd[j];
      if (i == j) b += dh[i];
      st->Gh[i * NMAX + j] = b;
      S.M[i][j] = b;  // the trial's copy (st_trial_begin)
    }
  }
  st->theta = fmax(0.995, 1.0 - gnorm);
  st->actual = -1.0;
  st->have_eig = 0;
  st_trial_begin<n>(st, S, true);
}

// TSQR (reading R31): the R factor of W = [J | r] from passes that reduce
// (W P)^T (W P) for preconditioners P built from the earlier passes.
//  - CholeskyQR2: R1 = chol(W^T W), R = chol((W R1^-1)^T (W R1^-1)) R1 — one
//    preconditioned pass; accurate while cond(W) stays below ~u^-1/2, here
//    while the certificate trace(G1) ||R1^-1||_F^2 >= cond(W)^2 is <= 1e14.
//  - beyond that (or when chol(G1) fails): shifted CholeskyQR3 (Fukaya,
//    Kannan, Nakatsukasa, Yamamoto, Yanagisawa 2020): R1 = chol(G1 + s I)
//    with s = 11 (m (n+1) + (n+1)(n+2)) u ||W||_2^2 (||W||_2^2 <= trace G1),
//    which exists for any cond(W); then CholeskyQR2 on W R1^-1 — two
//    preconditioned passes, R accurate for cond(W) up to ~u^-1.
constexpr double QR2_KAPPA2_MAX = 1.0e14;

// Start TSQR at the current x from the first pass's Gram (kv): the first
// preconditioner into the QR working set, phase PH_QR2.  Returns false only if
// G1 is not finite or not even the shifted Gram factors (the fit then
// continues in Gram mode).
template <int n>
__device__ __forceinline__ bool st_qr_begin(FitState* st, SolverSmem& S, const double* kv, int after) {
  constexpr int N1 = n + 1;
  double* R1 = &S.T[0][0];
  double* P = &S.M2[0][0];
  double tr = 0.0;
  for (int i = 0; i < N1; ++i) tr += kv[tri_slot(n, i, i)];
  bool ok = chol_kv<n>(kv, R1);
  if (ok) {
    tri_inv<n>(R1, P);
    double fro = 0.0;
    for (int i = 0; i < N1 * N1; ++i) fro = fma(P[i], P[i], fro);
    ok = tr * fro <= QR2_KAPPA2_MAX;
  }
  int stage = 0;
  if (!ok) {  // shifted CholeskyQR3
    const double u = 0.5 * DBL_EPSILON;
    const double shift = 11.0 * ((double)st->m_global * N1 + (double)(N1 * (N1 + 1))) * u * tr;
    if (!(tr > 0.0 && tr < INFINITY) || !chol_kv<n>(kv, R1, shift)) {
      st->qr_mode = 0;
      return false;
    }
    tri_inv<n>(R1, P);
    stage = 1;
  }
  for (int i = 0; i < N1 * N1; ++i) {
    st->qr->R1[i] = R1[i];
    st->qr->prec[i] = P[i];
  }
  st->qr_stage = stage;
  st->qr_after = after;
  st->phase = PH_QR2;
  return true;
}

// TSQR: after a preconditioned pass (Gram G2 of W P, P = R1^-1), R = chol(G2)
// R1.  Shifted CholeskyQR3's first preconditioned pass: R becomes the next
// R1 (another PH_QR2 pass follows; returns false).  Otherwise (g, G) from R
// (g = R_J^T c, G = R_J^T R_J); returns true.
template <int n>
__device__ __forceinline__ bool st_qr_finish(FitState* st, SolverSmem& S, const double* kv) {
  constexpr int N1 = n + 1;
  double* R2 = &S.T[0][0];
  double* R = &S.M2[0][0];
  const double* R1 = st->qr->R1;
  if (!chol_kv<n>(kv, R2)) {  // G2 ~ I in exact arithmetic; keep R1 if rounding broke it
    for (int i = 0; i < N1 * N1; ++i) R2[i] = (i % (N1 + 1) == 0) ? 1.0 : 0.0;
  }
  for (int i = 0; i < N1; ++i)
    for (int j = 0; j < N1; ++j) {
      double t = 0.0;
      for (int k = i; k <= j; ++k) t = fma(R2[i * N1 + k], R1[k * N1 + j], t);
      R[i * N1 + j] = (j >= i) ? t : 0.0;
    }
  if (st->qr_stage == 1) {  // shifted CholeskyQR3: CholeskyQR2 on W R^-1 next
    double* P = &S.T[0][0];
    tri_inv<n>(R, P);
    for (int i = 0; i < N1 * N1; ++i) {
      st->qr->R1[i] = R[i];
      st->qr->prec[i] = P[i];
    }
    st->qr_stage = 2;
    return false;
  }
  for (int i = 0; i < N1 * N1; ++i) st->qr->R[i] = R[i];
  for (int j = 0; j < n; ++j) {  // g = R_J^T c, G = R_J^T R_J
    double t = 0.0;
    for (int k = 0; k <= j; ++k) t = fma(R[k * N1 + j], R[k * N1 + n], t);
    st->g[j] = t;
    for (int l = j; l < n; ++l) {
      double u = 0.0;
      for (int k = 0; k <= j; ++k) u = fma(R[k * N1 + j], R[k * N1 + l], u);
      st->G[j * NMAX + l] = u;
      st->G[l * NMAX + j] = u;
    }
  }
  return true;
}

// AUTO solver choice (jf.h jf_solver): an upper bound on cond(J D^-1)^2 for
// the column-scaled Gram B = D^-1 G D^-1 (D = column norms): lambda_max <=
// trace(B) = n and lambda_min >= 1/||L^-1||_F^2 (B = L L^T); +inf if B is not
// numerically SPD.
template <int n>
__device__ __forceinline__ double kappa2_estimate(FitState* st, SolverSmem& S) {
  double dinv[n], L[n][n], Y[n][n], cinv[n];
#pragma unroll
  for (int j = 0; j < n; ++j) {
    const double gjj = st->G[j * NMAX + j];
    dinv[j] = gjj > 0.0 ? rsqrt(gjj) : 1.0;
  }
  double tr = 0.0;
#pragma unroll
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int j = 0; j <= i; ++j) L[i][j] = dinv[i] * st->G[i * NMAX + j] * dinv[j];
    tr += L[i][i];
  }
  if (!chol_reg<n>(L, cinv)) return INFINITY;
  return tr * inv_fro2<n>(L, cinv, Y);
}

// AUTO along the trajectory: at an accepted step of a Gram-mode fit whose last
// Gauss-Newton Cholesky bounded cond(B_hat)^2 above 1e6 (or failed), the
// column-scaled Gram at the new x decides whether the fit continues in TSQR
// mode (the same test as at x0; a cheap trigger keeps it off the common path).
template <int n>
__device__ __forceinline__ void st_auto_recheck(FitState* st, SolverSmem& S) {
  if (st->auto_mode && !st->qr_mode && !(st->kappa2_gn <= 1.0e6) && kappa2_estimate<n>(st, S) > 1.0e6)
    st->qr_mode = 1;
}

// Initialisation after the J-pass at x0 (Alg. 1 l.137-138; R3, R4, R18).
template <int n>
__device__ __noinline__ void st_init_finish(FitState* st, SolverSmem& S) {
  if (st->jacmode) {
    st_update_scale<n>(st, true);
  } else {
    for (int j = 0; j < n; ++j) st->scale_inv[j] = st->xs_inv[j];
  }
  double s2 = 0.0;  // R4: Delta0 = ||x0 * scale_inv (/ sqrt(v))||
  for (int j = 0; j < n; ++j) {
    double t = st->x[j] * st->scale_inv[j];
    if (st->bounded) {
      double v, dv;
      cl_vector(st->x[j], st->g[j], st->lb[j], st->ub[j], v, dv);
      if (dv != 0.0) v *= st->scale_inv[j];
      t /= sqrt(v);
    }
    s2 = fma(t, t, s2);
  }
  double Delta = sqrt(s2);
  if (Delta == 0.0) Delta = 1.0;
  st->Delta = Delta;
  st_outer_top<n>(st, S);
}

template <int n>
__device__ __noinline__ void st_init(FitState* st, SolverSmem& S, const double* kv) {
  if (kv[tri_count(n)] != 0.0) {  // R18: residuals at x0 must be finite
    st->error = -3;
    st->status = -3;
    st->phase = PH_DONE;
    st->cont = 0;
    return;
  }
  st_take_pass<n>(st, kv);
  st->nfev = 1;
  st->njev = 1;
  st->nit = 0;
  st->alpha = 0.0;
  st->status = STATUS_NONE;
  if (st->qr_mode == 2) {  // AUTO: TSQR iff the column-scaled Gram at x0 is ill-conditioned
    st->qr_mode = (kappa2_estimate<n>(st, S) > 1.0e6) ? 1 : 0;
  }
  if (st->qr_mode && st_qr_begin<n>(st, S, kv, 0)) return;  // R from the second pass first
  st_init_finish<n>(st, S);
}

// End of the inner (retry) loop: accept or keep x, count the iteration.  For
// the conservative policy an accepted step first needs the J-pass at x_new.
template <int n>
__device__ __noinline__ void st_end_inner(FitState* st, SolverSmem& S, bool have_jac) {
  if (st->actual > 0.0) {
    for (int j = 0; j < n; ++j) st->x[j] = st->x_eval[j];
    if (!have_jac) {  // conservative: J at the new x (counts as njev there)
      st->cost = st->cost_new;
      st->phase = PH_ACCEPT_J;
      return;
    }
    const long long c0 = clock64();
    st_take_pass<n>(st, st->kv);
    st->cost = st->cost_new;  // SciPy keeps the trial's cost
    st->njev = st->njev + 1;
    st_auto_recheck<n>(st, S);
    if (st->qr_mode && st_qr_begin<n>(st, S, st->kv, 1)) return;  // nit counts after the QR pass
    if (st->jacmode) st_update_scale<n>(st, false);
    st->prof[5] += clock64() - c0;
  }
  st->nit = st->nit + 1;  // R27
  const long long c1 = clock64();
  st_outer_top<n>(st, S);
  st->prof[6] += clock64() - c1;
}

// After a trial pass at x_eval (speculative J-pass or conservative r-pass).
template <int n>
__device__ __noinline__ void st_after_trial(FitState* st, SolverSmem& S, const double* kv, bool jac) {
  const double rr = jac ? kv[tri_slot(n, n, n)] : kv[0];
  const double bad = jac ? kv[tri_count(n)] : kv[1];
  st->nfev = st->nfev + 1;
  if (bad != 0.0) {  // R17: shrink and retry, no termination test
    st->Delta = 0.25 * st->hn;
    st_trace(st, NAN, NAN);
    if (st->nfev < st->max_nfev) {
      st_trial_begin<n>(st, S);
      return;
    }
    st->actual = -1.0;
    st_end_inner<n>(st, S, jac);
    return;
  }
  const double cost_new = 0.5 * rr;
  const double actual = st->cost - cost_new;
  const double pred = st->pred;
  double ratio;  // Eq. 15 (R14)
  if (pred > 0.0) ratio = actual / pred;
  else if (pred == 0.0 && actual == 0.0) ratio = 1.0;
  else ratio = 0.0;
  double Delta_new = st->Delta;  // Alg. 3 with SciPy's rules (R15)
  if (ratio < 0.25) Delta_new = 0.25 * st->hn;
  else if (ratio > 0.75 && st->hn > 0.95 * st->Delta) Delta_new = 2.0 * st->Delta;
  const double xnorm = vnorm<n>(st->x);  // termination (R16), pre-step x
  const bool ft = actual < st->ftol * st->cost && ratio > 0.25;
  const bool xt = st->step_norm < st->xtol * (st->xtol + xnorm);
  const int status = (ft && xt) ? 4 : (ft ? 2 : (xt ? 3 : STATUS_NONE));
  st->cost_new = cost_new;
  st->actual = actual;
  st->ratio = ratio;
  st_trace(st, cost_new, ratio);
  if (status != STATUS_NONE) {
    st->status = status;
    st_end_inner<n>(st, S, jac);
    return;
  }
  st->alpha = st->alpha * (st->Delta / Delta_new);  // R5
  st->Delta = Delta_new;
  if (actual <= 0.0 && st->nfev < st->max_nfev) {
    st_trial_begin<n>(st, S);  // R15: same hat space, new radius
    return;
  }
  st_end_inner<n>(st, S, jac);
}

// Lane 0: advance the state machine with the K-vector of the pass that just
// finished.  A requested trial is left half done (S.need_trial) for
// solver_step: warp eigensolver if S.need_eig, then st_trial_finish.
template <int n>
__device__ __noinline__ void fit_after_pass(FitState* st, SolverSmem& S, const double* kv, bool jac) {
  const int KS = jac ? tri_count(n) + 1 : 2;
  for (int k = 0; k < KS; ++k) st->kv[k] = kv[k];
  st->launches = st->launches + 1;
  S.need_trial = 0;
  S.need_eig = 0;
  const int phase = st->phase;
  if (phase == PH_INIT_J) {
    st_init<n>(st, S, st->kv);
  } else if (phase == PH_TRIAL_J && jac) {
    const long long c0 = clock64();
    st_after_trial<n>(st, S, st->kv, true);
    st->prof[4] += clock64() - c0;
  } else if (phase == PH_TRIAL_R && !jac) {
    st_after_trial<n>(st, S, st->kv, false);
  } else if (phase == PH_ACCEPT_J && jac) {
    const long long c0 = clock64();
    st_take_pass<n>(st, st->kv);  // g, G at the accepted x (cost kept: SciPy)
    st->cost = st->cost_new;
    st->njev = st->njev + 1;
    st_auto_recheck<n>(st, S);
    if (st->qr_mode && st_qr_begin<n>(st, S, st->kv, 1)) return;
    if (st->jacmode) st_update_scale<n>(st, false);
    st->nit = st->nit + 1;
    const long long c1 = clock64();
    st->prof[5] += c1 - c0;
    st_outer_top<n>(st, S);
    st->prof[6] += clock64() - c1;
  } else if (phase == PH_QR2 && jac) {
    if (!st_qr_finish<n>(st, S, st->kv)) return;  // (shifted CholeskyQR3: one more preconditioned pass)
    if (st->qr_after == 0) {
      st_init_finish<n>(st, S);
    } else {
      if (st->jacmode) st_update_scale<n>(st, false);
      st->nit = st->nit + 1;
      st_outer_top<n>(st, S);
    }
  }
}

// Warp Cholesky of the SPD matrix A (shared memory, rows padded to MS) with
// the rank certificate: L (lower) in Lm, cinv = 1 / diag(L), Y = L^-1 in Ym,
// fro = ||L^-1||_F^2, tr = trace(A) — the same arithmetic in the same order
// as chol_reg + inv_fro2 (lane i forms row i's entries of column k; lane c
// column c of L^-1; the sums in their serial order).  false: not SPD.
template <int n>
__device__ __forceinline__ bool warp_chol_cert(const double (*A)[MS], double (*Lm)[MS], double* cinv,
                                               double (*Ym)[MS], double& tr, double& fro) {
  const int lane = threadIdx.x & 31;
  tr = 0.0;
#pragma unroll
  for (int i = 0; i < n; ++i) tr += A[i][i];
  // (loops fully unrolled, the lane's own row of L in registers: the loads
  // are issued together instead of one shared-memory round trip per fma)
  double lrow[n];
#pragma unroll
  for (int k = 0; k < n; ++k) {
    double t = 0.0;
    if (lane >= k && lane < n) {
      t = A[lane][k];
#pragma unroll
      for (int j = 0; j < k; ++j) t = fma(-lrow[j], Lm[k][j], t);
    }
    const double d = __shfl_sync(FULL, t, k);
    if (!(d > 0.0)) return false;
    const double r = rsqrt(d);
    lrow[k] = (lane == k) ? d * r : t * r;
    if (lane == k) {
      Lm[k][k] = d * r;
      cinv[k] = r;
    } else if (lane > k && lane < n) {
      Lm[lane][k] = t * r;
    }
    __syncwarp();
  }
  if (lane < n) {  // lane c: column c of L^-1, rows i >= c (k increasing from c, as before)
    const int c = lane;
    double y[n];
#pragma unroll
    for (int i = 0; i < n; ++i) {
      double t = (i == c) ? 1.0 : 0.0;
#pragma unroll
      for (int k = 0; k < i; ++k)
        if (k >= c) t = fma(-Lm[i][k], y[k], t);
      y[i] = t * cinv[i];
      if (i >= c) Ym[i][c] = y[i];
    }
  }
  __syncwarp();
  fro = 0.0;
#pragma unroll
  for (int c = 0; c < n; ++c)
#pragma unroll
    for (int i = c; i < n; ++i) fro = fma(Ym[i][c], Ym[i][c], fro);
  return true;
}

// Fast path of the covariance: when the Cholesky certificate (warp_chol_cert)
// shows no singular value of J falls below the cut-off
// (1/||L^-1||_F > 2 EPS max(m, n) sqrt(trace G) => s_min > EPS max(m, n) s_max),
// the pseudo-inverse is the inverse, (L L^T)^-1 = L^-T L^-1: n^3/2 fmas in
// place of an eigendecomposition (st_pcov below).
// Whole warp, once at the end of a fit: the parameter covariance curve_fit
// returns with the parameters: the Moore-Penrose
// inverse of J^T J at the final x, discarding singular values of J below
// EPS * max(m, n) * s_max, scaled by 2 cost / (m - n) (m > n; else +inf).
// J^T J = V diag(s^2) V^T is the final pass's Gram (the same eigensolver as
// the trust-region subproblem) unless pcov_chol certifies full rank.
template <int n>
__device__ __noinline__ void st_pcov(FitState* st, SolverSmem& S) {
  const int lane = threadIdx.x & 31;
  const int64_t m = st->m_global;
  const double s_sq = (m > n) ? 2.0 * st->cost / (double)(m - n) : INFINITY;
  if (!st->qr_mode) {  // pcov_chol on the warp: the same arithmetic (warp_chol_cert), entries on the lanes
    if (lane < n)
      for (int j = 0; j <= lane; ++j) S.A[lane][j] = st->G[lane * NMAX + j];
    __syncwarp();
    double tr, fro;
    const bool spd = warp_chol_cert<n>(S.A, S.T, S.w4, S.M2, tr, fro);
    if (spd && m >= n && rsqrt(fro) > 2.0 * DBL_EPSILON * (double)(m > n ? m : n) * sqrt(tr)) {
      for (int e = lane; e < n * n; e += 32) {
        const int i = e / n, j = e % n;
        if (j < i) continue;
        double t = 0.0;
        for (int k = j; k < n; ++k) t = fma(S.M2[k][i], S.M2[k][j], t);
        st->pcov[i * NMAX + j] = st->pcov[j * NMAX + i] = t * s_sq;
      }
      __syncwarp();
      if (lane == 0) st->pcov_done = 1;
      __syncwarp();
      return;
    }
  }
  if (st->qr_mode) {  // TSQR: singular values of J from R_J (one-sided Jacobi), not squared
    constexpr int N1 = n + 1;
    for (int e = lane; e < 2 * NMAX * n; e += 32) {
      const int i = e / n, j = e % n;
      S.Q[i][j] = (i < n) ? st->qr->R[i * N1 + j] : 0.0;
    }
    for (int i = lane; i < 2 * NMAX; i += 32) S.caug[i] = 0.0;
    __syncwarp();
    warp_svd(S, n, n);
  } else {
    for (int e = lane; e < n * n; e += 32) {
      const int i = e / n, j = e % n;
      S.A[i][j] = st->G[i * NMAX + j];
    }
    __syncwarp();
    warp_eig(S, n, 0);
  }
  if (lane == 0) {
    const double smax = sqrt(fmax(S.lam[0], 0.0));
    const double thr = DBL_EPSILON * (double)(m > n ? m : n) * smax;
    double* is2 = S.w1;  // 1 / s_k^2 of the kept singular values, else 0
    for (int k = 0; k < n; ++k) {
      const double sk = sqrt(fmax(S.lam[k], 0.0));
      is2[k] = (sk > thr) ? 1.0 / (sk * sk) : 0.0;
    }
    for (int i = 0; i < n; ++i) {
      for (int j = 0; j < n; ++j) {
        double t = 0.0;
        for (int k = 0; k < n; ++k) t += S.V[i][k] * S.V[j][k] * is2[k];
        st->pcov[i * NMAX + j] = t * s_sq;
      }
    }
    st->pcov_done = 1;
  }
  __syncwarp();
}

// Warp fast path of the common solver steps of a speculative, unbounded,
// Gram-mode fit (every step of every BASELINE fit but the last):
//  - PH_INIT_J: the J-pass at x0 (st_init: AUTO keeps the Gram path, scale,
//    Delta0), then Alg. 1's loop top and a certified Gauss-Newton trial;
//  - PH_TRIAL_J: the J-pass at the trial point is accepted with no
//    termination test firing, then the loop top and the next certified
//    Gauss-Newton trial inside the new radius.
// Bitwise the same arithmetic, in the same order, as the general path
// (fit_after_pass -> st_init / st_after_trial -> st_end_inner ->
// st_outer_top -> gn_fastpath -> st_trial_finish), with the independent parts
// on the warp's lanes and over shared memory rather than lane 0's long serial
// chain.  Everything is decided before the state is written: any other case
// returns false and the general path runs from the untouched state.  All
// lanes call it.
template <int n>
__device__ __noinline__ bool warp_gn_step(FitState* st, SolverSmem& S, const double* kv) {
  const int lane = threadIdx.x & 31;
#if JF_DEV  // development: cycles of the phases (prof[1] decide + g/G, [4] B_hat + Cholesky, [6] solves, [7] pred + commit)
  long long dq0 = clock64(), dq1 = 0, dq2 = 0, dq3 = 0;
#endif
  // (the gating fields read together, ahead of the first branch)
  const int phase = st->phase, bounded = st->bounded, policy = st->policy, trace_cap = st->trace_cap;
  const int qr_mode = st->qr_mode, status0 = st->status, nfev0 = st->nfev, max_nfev = st->max_nfev;
  const int auto_mode = st->auto_mode;
  const double cost = st->cost, pred_old = st->pred, Delta = st->Delta, hn_old = st->hn, ftol = st->ftol,
               xtol = st->xtol, step_norm = st->step_norm, kappa2_gn = st->kappa2_gn, alpha0 = st->alpha;
  const double kv_flag = kv[tri_count(n)], kv_rr = kv[tri_slot(n, n, n)];
  const bool init = (phase == PH_INIT_J);
  if ((phase != PH_TRIAL_J && !init) || bounded || policy != 0 || trace_cap > 0 ||
      (init ? qr_mode == 1 : (qr_mode != 0 || status0 != STATUS_NONE)))
    return false;
  if (kv_flag != 0.0) return false;  // R17 / R18 paths
  const double cost_new = 0.5 * kv_rr;
  double ratio = 0.0, Delta_new = 0.0, alpha_new = 0.0;
  int nfev = 1;
  if (!init) {  // ---- st_after_trial (read-only)
    const double actual = cost - cost_new;
    if (pred_old > 0.0) ratio = actual / pred_old;
    else if (pred_old == 0.0 && actual == 0.0) ratio = 1.0;
    else ratio = 0.0;
    Delta_new = Delta;
    if (ratio < 0.25) Delta_new = 0.25 * hn_old;
    else if (ratio > 0.75 && hn_old > 0.95 * Delta) Delta_new = 2.0 * Delta;
    const double xnorm = vnorm<n>(st->x);
    const bool ft = actual < ftol * cost && ratio > 0.25;
    const bool xt = step_norm < xtol * (xtol + xnorm);
    if (ft || xt || !(actual > 0.0)) return false;
    nfev = nfev0 + 1;
    if (auto_mode && !(kappa2_gn <= 1.0e6)) return false;  // AUTO re-check: general path
    alpha_new = alpha0 * (Delta / Delta_new);
  }
  if (nfev == max_nfev) return false;
  // ---- the new iterate's g, G (from the K-vector) and scale (lane j: entry j)
  double gj = 0.0, gjj = 0.0, si = 1.0;
  if (lane < n) {
    gj = kv[tri_slot(n, lane, n)];
    gjj = kv[tri_slot(n, lane, lane)];
    const double sq = sqrt(gjj);
    if (init) {
      si = st->jacmode ? (sq == 0.0 ? 1.0 : sq) : st->xs_inv[lane];
    } else {
      si = st->jacmode ? fmax(sq, st->scale_inv[lane]) : st->scale_inv[lane];
    }
    S.w1[lane] = gj;
  }
  __syncwarp();
  if (init && st->qr_mode == 2) {  // AUTO at x0: kappa2_estimate of the column-scaled Gram
    if (lane < n) S.w2[lane] = gjj > 0.0 ? rsqrt(gjj) : 1.0;
    __syncwarp();
    if (lane < n) {
      for (int j = 0; j <= lane; ++j) S.A[lane][j] = S.w2[lane] * kv[tri_slot(n, j, lane)] * S.w2[j];
    }
    __syncwarp();
    double tr0, fro0;
    if (!warp_chol_cert<n>(S.A, S.T, S.w4, S.M2, tr0, fro0)) return false;  // (kappa2 = inf: TSQR)
    if (tr0 * fro0 > 1.0e6) return false;                                    // TSQR: general path
  }
  double gnorm = 0.0;
#pragma unroll
  for (int j = 0; j < n; ++j) gnorm = fmax(gnorm, fabs(S.w1[j] * 1.0));
  if (gnorm < st->gtol) return false;  // gtol termination: general path
  if (init) {  // R4: Delta0 = ||x0 scale_inv||, 0 -> 1
    if (lane < n) S.w5[lane] = si;
    __syncwarp();
    double s2 = 0.0;
#pragma unroll
    for (int j = 0; j < n; ++j) {
      const double t = st->x[j] * S.w5[j];
      s2 = fma(t, t, s2);
    }
    Delta_new = sqrt(s2);
    if (Delta_new == 0.0) Delta_new = 1.0;
    __syncwarp();
  }
#if JF_DEV
  dq1 = clock64();
#endif
  // B_hat = d G d (+ diag_h = 0 on the diagonal; row i on lane i), g_hat
  const double dd = (lane < n) ? 1.0 / si : 0.0;
  if (lane < n) S.w2[lane] = dd;
  __syncwarp();
  if (lane < n) {
#pragma unroll
    for (int j = 0; j < n; ++j) {
      const int a = lane < j ? lane : j, b = lane < j ? j : lane;
      double bij = dd * kv[tri_slot(n, a, b)] * S.w2[j];
      if (lane == j) bij += 0.0;
      S.M[lane][j] = bij;
    }
    S.w3[lane] = dd * gj;  // g_hat
  }
  __syncwarp();
  // ---- gn_fastpath: Cholesky + certificate, L w = -g_hat, L^T p = w
  double tr, fro;
  double* cinv = S.w4;
  if (!warp_chol_cert<n>(S.M, S.T, cinv, S.M2, tr, fro)) return false;
  const int64_t m = st->m_global;
  if (!(m >= n && rsqrt(fro) > 2.0 * DBL_EPSILON * (double)m * sqrt(tr))) return false;
#if JF_DEV
  dq2 = clock64();
#endif
  double t = (lane < n) ? -S.w3[lane] : 0.0;
#pragma unroll
  for (int k = 0; k < n; ++k) {  // lane i accumulates row i as w_k become known (k increasing)
    const double wk = __shfl_sync(FULL, t * cinv[k], k);
    if (lane > k && lane < n) t = fma(-S.T[lane][k], wk, t);
    if (lane == k) S.w5[k] = wk;
  }
  __syncwarp();
  double pr[n];  // L^T p = w in gn_fastpath's order (k increasing from i + 1), every lane
#pragma unroll
  for (int i = n - 1; i >= 0; --i) {
    double u = S.w5[i];
#pragma unroll
    for (int k = i + 1; k < n; ++k) u = fma(-S.T[k][i], pr[k], u);
    pr[i] = u * cinv[i];
  }
  double pn = 0.0;
#pragma unroll
  for (int i = 0; i < n; ++i) pn = fma(pr[i], pr[i], pn);
  if (!(sqrt(pn) <= Delta_new)) return false;
#if JF_DEV
  dq3 = clock64();
#endif
  // pred = -(0.5 p^T B p + p^T g_hat): rows of B p on the lanes, sums in vquad's order
  if (lane < n) {
    double r = 0.0;
#pragma unroll
    for (int k = 0; k < n; ++k) r = fma(S.M[lane][k], pr[k], r);
    S.V[0][lane] = r;
  }
  __syncwarp();
  // ---- commit (the general path's state, field by field)
  if (lane == 0) {
    double q = 0.0;
#pragma unroll
    for (int i = 0; i < n; ++i) q = fma(pr[i], S.V[0][i], q);
    double gp = 0.0;
#pragma unroll
    for (int j = 0; j < n; ++j) gp = fma(pr[j], S.w3[j], gp);
    st->launches = st->launches + 1;
    st->nfev = nfev;
    if (init) {
      st->njev = 1;
      st->nit = 0;
      st->status = STATUS_NONE;
      if (st->qr_mode == 2) st->qr_mode = 0;
    } else {
      st->cost_new = cost_new;
      st->ratio = ratio;
      st->njev = st->njev + 1;
      st->nit = st->nit + 1;
#pragma unroll
      for (int j = 0; j < n; ++j) st->x[j] = st->x_eval[j];
    }
    st->cost = cost_new;
    st->Delta = Delta_new;
    st->gnorm = gnorm;
    st->theta = fmax(0.995, 1.0 - gnorm);
    st->actual = -1.0;
    st->have_eig = 0;
    st->kappa2_gn = tr * fro;
    (void)alpha_new;  // (the trial's alpha: 0, a Gauss-Newton step)
    st->alpha = 0.0;
    st->pred = -(0.5 * q + gp);
    double h2 = 0.0, s2 = 0.0;
#pragma unroll
    for (int j = 0; j < n; ++j) {
      const double stp = S.w2[j] * pr[j];
      st->step_h[j] = pr[j];
      st->step[j] = stp;
      st->x_eval[j] = st->x[j] + stp;
      h2 = fma(pr[j], pr[j], h2);
      s2 = fma(stp, stp, s2);
    }
    st->hn = sqrt(h2);
    st->step_norm = sqrt(s2);
    st->Delta_used = Delta_new;
    st->branch = -1;
    st->phase = PH_TRIAL_J;
  }
  for (int k = lane; k < tri_count(n) + 1; k += 32) st->kv[k] = kv[k];  // (the K-vector, lane-parallel)
  if (lane < n) {
    st->g[lane] = gj;
    st->scale_inv[lane] = si;
    st->d[lane] = dd;
    st->diag_h[lane] = 0.0;
    st->gh[lane] = S.w3[lane];
#pragma unroll
    for (int j = 0; j < n; ++j) {
      const int a = lane < j ? lane : j, b = lane < j ? j : lane;
      st->G[lane * NMAX + j] = kv[tri_slot(n, a, b)];
      st->Gh[lane * NMAX + j] = S.M[lane][j];
    }
  }
  __syncwarp();
#if JF_DEV
  if (lane == 0) {
    st->prof[1] += dq1 - dq0;
    st->prof[4] += dq2 - dq1;
    st->prof[6] += dq3 - dq2;
    st->prof[7] += clock64() - dq3;
  }
#endif
  return true;
}

template <int n>
__device__ __forceinline__ void solver_step_n(FitState* st, SolverSmem& S, const double* kv, bool jac) {
  const int lane = threadIdx.x & 31;
  const long long c0 = clock64();
  if (jac && warp_gn_step<n>(st, S, kv)) {  // (the common step, on the whole warp)
    if (lane == 0) st->prof[3] += clock64() - c0;
    __syncwarp();
    return;
  }
  if (lane == 0) fit_after_pass<n>(st, S, kv, jac);
  __syncwarp();
  if (S.need_trial && S.need_eig && st->qr_mode) {
    // TSQR: SVD of [R_J diag(d); diag(sqrt(diag_h))] and [c; 0] (App. B on R)
    constexpr int N1 = n + 1;
    const double* R = st->qr->R;
    const int rows = st->bounded ? 2 * n : n;
    for (int e = lane; e < 2 * NMAX * n; e += 32) {
      const int i = e / n, j = e % n;
      double q = 0.0;
      if (i < n) q = R[i * N1 + j] * st->d[j];
      else if (i < rows) q = (i - n == j) ? sqrt(st->diag_h[j]) : 0.0;
      S.Q[i][j] = q;
    }
    for (int i = lane; i < 2 * NMAX; i += 32) S.caug[i] = (i < n) ? R[i * N1 + n] : 0.0;
    __syncwarp();
    const long long c1 = clock64();
    warp_svd(S, n, rows);
    if (lane == 0) st->prof[0] += clock64() - c1;
  } else if (S.need_trial && S.need_eig) {
    const int warm = st->have_V;
    for (int e = lane; e < n * n; e += 32) {
      const int i = e / n, j = e % n;
      S.A[i][j] = S.M[i][j];
      if (warm) S.V[i][j] = st->V[i * NMAX + j];
    }
    __syncwarp();
    const long long c1 = clock64();
    warp_eig(S, n, warm);
    if (lane == 0) st->prof[0] += clock64() - c1;
  }
  __syncwarp();
  if (lane == 0 && S.need_trial) {
    const long long c2 = clock64();
    st_trial_finish<n>(st, S);
    st->prof[7] += clock64() - c2;
  }
  __syncwarp();
  if (!st->cont && st->error == 0 && !st->pcov_done) st_pcov<n>(st, S);
  if (lane == 0) st->prof[3] += clock64() - c0;
  __syncwarp();
}

// Whole warp: one solver step after a pass (state machine on lane 0, the
// eigensolver on all lanes when a trial needs it).  NC = 0: dispatch on st->n.
template <int NC>
__device__ __forceinline__ void solver_step(FitState* st, SolverSmem& S, const double* kv, bool jac) {
  if constexpr (NC > 0) {
    solver_step_n<NC>(st, S, kv, jac);
  } else {
    switch (st->n) {
      case 2: solver_step_n<2>(st, S, kv, jac); break;
      case 3: solver_step_n<3>(st, S, kv, jac); break;
      case 4: solver_step_n<4>(st, S, kv, jac); break;
      case 7: solver_step_n<7>(st, S, kv, jac); break;
      case 13: solver_step_n<13>(st, S, kv, jac); break;
      default: break;
    }
  }
}

// Whole warp: load the fit state and the pass's K-vector (global, just
// written by the pass) into shared memory — every load issued before any is
// consumed — run one solver step, write the state back, set the CUDA-graph
// WHILE condition.  Used by the solver kernel and by the fused J-pass.
template <int NC>
__device__ __forceinline__ void solver_run(FitState* __restrict__ st, SolverSmem& S, FitState& sst, const double* kv,
                                           bool jac, cudaGraphConditionalHandle cond, int use_cond) {
  const int lane = threadIdx.x & 31;
  unsigned long long t0, t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  if (lane == 0) {
    const int k = atomicAdd(&st->tl_n, 1);
    if (k < 64) st->tl[k] = t0;
  }
  __syncwarp();
  constexpr int NW = sizeof(FitState) / 8;
  constexpr int PER = (NW + 31) / 32;
  constexpr int KPER = (KMAX + 31) / 32;
  const unsigned long long* src = reinterpret_cast<const unsigned long long*>(st);
  unsigned long long* dst = reinterpret_cast<unsigned long long*>(&sst);
  unsigned long long buf[PER];
  double kvb[KPER];
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int k = lane + 32 * q;
    buf[q] = (k < NW) ? __ldcg(src + k) : 0ull;
  }
#pragma unroll
  for (int q = 0; q < KPER; ++q) {
    const int k = lane + 32 * q;
    kvb[q] = (k < KMAX) ? __ldcg(kv + k) : 0.0;
  }
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int k = lane + 32 * q;
    if (k < NW) dst[k] = buf[q];
  }
#pragma unroll
  for (int q = 0; q < KPER; ++q) {
    const int k = lane + 32 * q;
    if (k < KMAX) S.kvs[k] = kvb[q];
  }
  __syncwarp();
  solver_step<NC>(&sst, S, S.kvs, jac);
  __syncwarp();
  if (sst.n == 7) {  // the next n = 7 moment J-pass's prologue at x_eval
    gauss2d_prologue_warp(sst.x_eval, sst.pre);
    if (lane == 0) sst.has_pre = 1;
  } else if (sst.n == 13) {  // (the two-Gaussian moment J-pass's)
    gauss2d_x2_prologue_warp(sst.x_eval, sst.pre);
    if (lane == 0) sst.has_pre = 1;
  }
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  if (lane == 0) {
    sst.pass_ready = 0;
    sst.epi_ns += (t1 - t0);
    const int k = sst.tl_n;
    if (k < 64) sst.tl[k] = t1;
    sst.tl_n = k + 1;
  }
  __syncwarp();
  unsigned long long* back = reinterpret_cast<unsigned long long*>(st);
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int k = lane + 32 * q;
    if (k < NW) back[k] = dst[k];
  }
  if (lane == 0 && use_cond) cudaGraphSetConditional(cond, sst.cont ? 1u : 0u);
}

// Scratch of the fused solver step (SolverSmem, then a FitState copy).
__host__ __device__ constexpr size_t fused_solver_smem_bytes() {
  return ((sizeof(SolverSmem) + 15) & ~(size_t)15) + sizeof(FitState);
}

// The solver step run by warp 0 of the last block of a fused J-pass (reading
// PassArgs::fused): the same as the solver kernel's solver_run with the
// pass's combined K-vector read from shared memory (vec) and the kernel's
// dynamic shared memory (>= fused_solver_smem_bytes()) as scratch.  The next
// pass kernel waits for this grid (PDL griddepcontrol.wait) and reads the
// state it leaves.
template <int NC>
__device__ __noinline__ void fused_solver_step(FitState* __restrict__ st, const double* vec,
                                               cudaGraphConditionalHandle cond, int use_cond) {
  extern __shared__ __align__(16) unsigned char fused_dyn[];
  SolverSmem& S = *reinterpret_cast<SolverSmem*>(fused_dyn);
  FitState& sst = *reinterpret_cast<FitState*>(fused_dyn + ((sizeof(SolverSmem) + 15) & ~(size_t)15));
  const int lane = threadIdx.x & 31;
#if JF_DEV
  const long long dvs = clock64();
#endif
  unsigned long long t0, t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  constexpr int NW = sizeof(FitState) / 8;
  constexpr int PER = (NW + 31) / 32;
  const unsigned long long* src = reinterpret_cast<const unsigned long long*>(st);
  unsigned long long* dst = reinterpret_cast<unsigned long long*>(&sst);
  unsigned long long buf[PER];
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int k = lane + 32 * q;
    buf[q] = (k < NW) ? __ldcg(src + k) : 0ull;
  }
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int k = lane + 32 * q;
    if (k < NW) dst[k] = buf[q];
  }
  for (int k = lane; k < KMAX; k += 32) S.kvs[k] = vec[k];
  __syncwarp();
#if JF_DEV
  const long long dv0 = clock64();
#endif
  if (lane == 0) {
    const int k = sst.tl_n;
    if (k < 64) sst.tl[k] = t0;
    sst.tl_n = k + 1;
  }
  __syncwarp();
  solver_step<NC>(&sst, S, S.kvs, true);
  __syncwarp();
#if JF_DEV
  const long long dv1 = clock64();
#endif
  if (sst.n == 7) {  // the next pass's prologue at x_eval
    gauss2d_prologue_warp(sst.x_eval, sst.pre);
    if (lane == 0) sst.has_pre = 1;
  } else if (sst.n == 13) {  // (the two-Gaussian moment J-pass's)
    gauss2d_x2_prologue_warp(sst.x_eval, sst.pre);
    if (lane == 0) sst.has_pre = 1;
  }
#if JF_DEV  // development: cycles of the state load (prof[0]) and of the prologue (prof[2])
  if (lane == 0) {
    sst.prof[0] += dv0 - dvs;
    sst.prof[2] += clock64() - dv1;
  }
#endif
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  if (lane == 0) {
    sst.pass_ready = 0;
    sst.epi_ns += (t1 - t0);
    const int k = sst.tl_n;
    if (k < 64) sst.tl[k] = t1;
    sst.tl_n = k + 1;
  }
  __syncwarp();
  unsigned long long* back = reinterpret_cast<unsigned long long*>(st);
#if JF_DEV  // development: cycles of the state write-back (prof[5], accumulated in the global state)
  const long long dvw = clock64();
#endif
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int k = lane + 32 * q;
    if (k < NW) back[k] = dst[k];
  }
#if JF_DEV
  __syncwarp();
  __threadfence();
  if (lane == 0) atomicAdd(reinterpret_cast<unsigned long long*>(&st->prof[5]), (unsigned long long)(clock64() - dvw));
#endif
  if (lane == 0 && use_cond) cudaGraphSetConditional(cond, sst.cont ? 1u : 0u);
}

}  // namespace jf
