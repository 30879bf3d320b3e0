// jf_solver.cuh — the n x n trust-region subproblem and the iteration control,
// executed by ONE warp on the device.
//
// Everything the paper runs "in NumPy on the CPU" between passes (P:226, P:343:
// the alpha sub-problem and the radius logic) runs here, in the last block of
// each pass kernel, so a fit never returns to the host between iterations.
//
//   Alg. 1  outer loop, Gauss-Newton trial p_t = -B^-1 g
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
// Warp conventions: vector element j lives in lane j (j < n; other lanes hold
// 0); scalars are computed redundantly and identically by all 32 lanes (every
// reduction is a commutative xor-butterfly, so all lanes see bit-identical
// values); matrices live in shared memory.
#pragma once

#include <cfloat>
#include <cmath>

#include "jf_common.cuh"

namespace jf {

enum Phase : int32_t {
  PH_INIT_J = 0,    // J-pass at x0
  PH_TRIAL_J = 1,   // speculative policy: J-pass at a trial point
  PH_TRIAL_R = 2,   // conservative policy: residual pass at a trial point
  PH_ACCEPT_J = 3,  // conservative policy: J-pass at the accepted point
  PH_DONE = 4
};

constexpr int TRACE_FIELDS = 12;
constexpr int STATUS_NONE = -100;

struct FitState {
  // ---- configuration (written by the host before the first launch)
  int32_t n, bounded, jacmode, max_nfev;
  int32_t policy, trace_cap, pad0, pad1;
  int64_t m_global;
  double ftol, xtol, gtol;
  double lb[NMAX], ub[NMAX], xs_inv[NMAX];
  double* trace;
  // ---- iteration state
  int32_t phase, status, nfev, njev, nit, cont, error, trace_len;
  int32_t full_rank, branch, launches, have_V;
  unsigned long long comm_epoch;
  unsigned long long epi_ns;  // device time spent in the solver epilogue (globaltimer)
  long long prof[4];          // SM cycles: eig, solve_tr, select_step, fit_after_pass
  double cost, cost_new, Delta, alpha, gnorm, theta, actual;
  double pred, hn, step_norm, Delta_used, ratio, pad4;
  double x[NMAX], x_eval[NMAX];
  double g[NMAX], G[NMAX * NMAX], scale_inv[NMAX];
  // hat space of the current iterate (reused by rejected trials, R15)
  double d[NMAX], diag_h[NMAX], gh[NMAX], Gh[NMAX * NMAX], lam[NMAX], V[NMAX * NMAX], suf[NMAX];
  double step[NMAX], step_h[NMAX];
  double kv[KMAX];  // K-vector of the last pass
};

struct SolverSmem {
  double A[NMAX][NMAX + 1];
  double V[NMAX][NMAX + 1];
  double M[NMAX][NMAX + 1];  // scaled Gram (incl. diag_h) for quadratic forms
  double T[NMAX][NMAX + 1];  // scratch
  double c[NMAX], e[NMAX];
  int partner[NMAX];
};

// ------------------------------------------------------------ warp helpers
static __device__ __forceinline__ double wsum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}
static __device__ __forceinline__ double wmin(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(FULL, v, o));
  return v;
}
static __device__ __forceinline__ double wmax(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(FULL, v, o));
  return v;
}
static __device__ __forceinline__ bool wall(bool b) { return __all_sync(FULL, b); }
static __device__ __forceinline__ bool wany(bool b) { return __any_sync(FULL, b); }
static __device__ __forceinline__ double lanev(double v, int src) { return __shfl_sync(FULL, v, src); }
static __device__ __forceinline__ double wdot(double a, double b) { return wsum(a * b); }
static __device__ __forceinline__ double wnorm(double a) { return sqrt(wsum(a * a)); }

// y = M x for an n x n matrix in shared memory (row-major, stride NMAX+1).
static __device__ __forceinline__ double wmatvec(const double (*M)[NMAX + 1], double x, int n, int lane) {
  double y = 0.0;
  for (int k = 0; k < n; ++k) {
    const double xk = lanev(x, k);
    if (lane < n) y = fma(M[lane][k], xk, y);
  }
  return lane < n ? y : 0.0;
}
// y = V x (V columns are eigenvectors)
static __device__ __forceinline__ double wVx(const double (*V)[NMAX + 1], double x, int n, int lane) {
  return wmatvec(V, x, n, lane);
}
// y = V^T x
static __device__ __forceinline__ double wVtx(const double (*V)[NMAX + 1], double x, int n, int lane) {
  double y = 0.0;
  for (int k = 0; k < n; ++k) {
    const double xk = lanev(x, k);
    if (lane < n) y = fma(V[k][lane], xk, y);
  }
  return lane < n ? y : 0.0;
}
// s^T M s
static __device__ __forceinline__ double wquad(const double (*M)[NMAX + 1], double s, int n, int lane) {
  return wdot(s, wmatvec(M, s, n, lane));
}
// u^T M v
static __device__ __forceinline__ double wbilin(const double (*M)[NMAX + 1], double u, double v, int n, int lane) {
  return wdot(u, wmatvec(M, v, n, lane));
}

// ---------------------------------------------------- symmetric eigensolver
// Parallel (round-robin) cyclic Jacobi on the n x n symmetric matrix in S.A:
// on return lam (lane j, j < n) holds the eigenvalues sorted descending and
// the columns of S.V the matching orthonormal eigenvectors.  This is App. B's
// SVD of the scaled Jacobian computed through its Gram matrix (c.1b).
//
// warm != 0: S.V holds an orthogonal matrix V0 on entry (the previous
// iterate's eigenvectors); the sweeps run on V0^T A V0, which is nearly
// diagonal between consecutive iterations, and accumulate onto V0 — one or
// two sweeps instead of six.  Rotations are skipped when
// |a_pq| <= eps sqrt(|a_pp a_qq|) or |a_pq| <= 2^-60 max_i |a_ii|; the
// sweep loop ends when a sweep applies none.
static __device__ __noinline__ int warp_eig(SolverSmem& S, int n, int lane, double& lam_out, int warm) {
  const int N2 = (n + 1) & ~1;  // pad to even with a zero row / column
  if (!warm) {
    for (int e = lane; e < NMAX * NMAX; e += 32) {
      const int i = e / NMAX, j = e % NMAX;
      if (i >= n || j >= n) S.A[i][j] = 0.0;
      S.V[i][j] = (i == j) ? 1.0 : 0.0;
    }
    __syncwarp();
  } else {
    // T = A V0, then A = V0^T T (lane-parallel over elements)
    for (int e = lane; e < n * n; e += 32) {
      const int i = e / n, j = e % n;
      double t = 0.0;
      for (int k = 0; k < n; ++k) t = fma(S.A[i][k], S.V[k][j], t);
      S.T[i][j] = t;
    }
    __syncwarp();
    for (int e = lane; e < NMAX * NMAX; e += 32) {
      const int i = e / NMAX, j = e % NMAX;
      double t = 0.0;
      if (i < n && j < n) {
        for (int k = 0; k < n; ++k) t = fma(S.V[k][i], S.T[k][j], t);
      }
      S.A[i][j] = t;
      if (i >= n || j >= n) S.V[i][j] = (i == j) ? 1.0 : 0.0;
    }
    __syncwarp();
    // exact symmetry
    for (int e = lane; e < n * n; e += 32) {
      const int i = e / n, j = e % n;
      if (i < j) S.A[j][i] = S.A[i][j];
    }
    __syncwarp();
  }
  double amax = (lane < n) ? fabs(S.A[lane][lane]) : 0.0;
  amax = wmax(amax);
  const double abs_tol = amax * 8.673617379884035e-19;  // 2^-60
  int sweeps = 0;
  for (int sweep = 0; sweep < 40; ++sweep) {
    bool rotated = false;
    ++sweeps;
    for (int r = 0; r < N2 - 1; ++r) {
      // pair k: (p, q) from the circle method
      if (lane < N2 / 2) {
        int p, q;
        if (lane == 0) {
          p = r;
          q = N2 - 1;
        } else {
          p = (r + lane) % (N2 - 1);
          q = (r - lane + (N2 - 1)) % (N2 - 1);
        }
        if (p > q) {
          const int t = p;
          p = q;
          q = t;
        }
        const double apq = S.A[p][q], app = S.A[p][p], aqq = S.A[q][q];
        double c = 1.0, s = 0.0;
        const double aa = fabs(apq);
        const bool tiny = aa <= abs_tol || aa <= 1.1102230246251565e-16 * sqrt(fabs(app) * fabs(aqq));
        if (!tiny) {
          // t = tan(phi), the smaller root: t = 2 apq sgn(d) / (|d| + sqrt(d^2 + 4 apq^2)), d = aqq - app
          const double d = aqq - app;
          const double t = (2.0 * apq) * (d >= 0.0 ? 1.0 : -1.0) / (fabs(d) + sqrt(fma(d, d, 4.0 * apq * apq)));
          c = rsqrt(fma(t, t, 1.0));
          s = t * c;
          rotated = true;
        }
        // P[p][p] = c, P[p][q] = s, P[q][p] = -s, P[q][q] = c; A' = P^T A P
        S.c[p] = c;
        S.c[q] = c;
        S.e[p] = -s;  // P[q][p]
        S.e[q] = s;   // P[p][q]
        S.partner[p] = q;
        S.partner[q] = p;
      }
      __syncwarp();
      rotated = wany(rotated);
      if (!rotated) continue;
      // write phase: A' = P^T A P, V' = V P (each lane owns up to 8 elements)
      double newA[8], newV[8];
      int cnt = 0;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int e = lane + 32 * k;
        if (e < N2 * N2) {
          const int i = e / N2, j = e % N2;
          const int ib = S.partner[i], jb = S.partner[j];
          const double ci = S.c[i], ei = S.e[i], cj = S.c[j], ej = S.e[j];
          newA[k] = ci * (cj * S.A[i][j] + ej * S.A[i][jb]) + ei * (cj * S.A[ib][j] + ej * S.A[ib][jb]);
          newV[k] = cj * S.V[i][j] + ej * S.V[i][jb];
        }
      }
      (void)cnt;
      __syncwarp();
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int e = lane + 32 * k;
        if (e < N2 * N2) {
          const int i = e / N2, j = e % N2;
          S.A[i][j] = (S.partner[i] == j && i != j) ? 0.0 : newA[k];
          S.V[i][j] = newV[k];
        }
      }
      __syncwarp();
    }
    if (!__any_sync(FULL, rotated)) break;
  }
  // sort descending (ties by index); permute V columns accordingly
  double lam = (lane < n) ? S.A[lane][lane] : 0.0;
  int rank = 0;
  for (int k = 0; k < n; ++k) {
    const double lk = lanev(lam, k);
    if (lane < n && (lk > lam || (lk == lam && k < lane))) ++rank;
  }
  for (int e = lane; e < n * n; e += 32) {
    const int i = e / n, j = e % n;
    S.T[i][j] = S.V[i][j];
  }
  __syncwarp();
  for (int j = 0; j < n; ++j) {
    const int rj = __shfl_sync(FULL, rank, j);
    if (lane < n) S.V[lane][rj] = S.T[lane][j];
  }
  __syncwarp();
  double sorted = 0.0;
  for (int j = 0; j < n; ++j) {
    const int rj = __shfl_sync(FULL, rank, j);
    const double lj = lanev(lam, j);
    if (lane == rj) sorted = lj;
  }
  lam_out = (lane < n) ? sorted : 0.0;
  return sweeps;
}

// --------------------------------------------------- Alg. 2 + App. B on device
// Inputs: lam (descending eigenvalues of B_hat, lane j), V (S.V), suf = V^T g_hat
// (lane j), radius Delta, warm-start alpha, m (number of residuals, R6).
// Output: p (lane j), alpha, number of Moré iterations (0 = Gauss-Newton).
static __device__ __noinline__ int warp_solve_tr(const SolverSmem& S, int n, int64_t m, double lam, double suf, double Delta,
                             double& alpha, double& p_out, int lane, int* full_rank_out) {
  const bool act = lane < n;
  const double s = act ? sqrt(fmax(lam, 0.0)) : 0.0;
  const double s2 = s * s;
  const double s_max = lanev(s, 0), s_min = lanev(s, n - 1);
  const bool full_rank = (m >= n) && (s_min > DBL_EPSILON * (double)m * s_max);  // R6
  if (full_rank_out) *full_rank_out = full_rank ? 1 : 0;
  if (full_rank) {
    // Alg. 1 l.141: p_t = -V (uf / s), uf = suf / s
    const double coef = act ? (suf / s) / s : 0.0;
    const double p = -wVx(S.V, coef, n, lane);
    if (wnorm(p) <= Delta) {  // Alg. 1 l.142
      p_out = p;
      alpha = 0.0;
      return 0;
    }
  }
  // phi(alpha) = ||suf / (s^2 + alpha)|| - Delta;  phi' per R11
  auto phi_d = [&](double a, double& phi, double& dphi) {
    const double den = s2 + a;
    const double q = act ? suf / den : 0.0;
    const double pn = sqrt(wsum(q * q));
    phi = pn - Delta;
    const double t = act ? suf * suf / (den * den * den) : 0.0;
    dphi = -wsum(t) / pn;
  };
  double u = sqrt(wsum(act ? suf * suf : 0.0)) / Delta;  // Alg. 2 l.160
  double l = 0.0;
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
    l = fmax(l, alpha - ratio);                          // Alg. 2 l.172
    alpha = alpha - ((phi + Delta) / Delta) * ratio;     // Eq. 14
    if (fabs(phi) < 0.01 * Delta) break;                 // R9
  }
  const double coef = act ? suf / (s2 + alpha) : 0.0;
  double p = -wVx(S.V, coef, n, lane);  // Eq. B4 (sign R8)
  p = p * (Delta / wnorm(p));           // R12
  p_out = act ? p : 0.0;
  return it + 1;
}

// --------------------------------------------------- Coleman-Li helpers (R19)
// Smallest t >= 0 with x + t s on a bound; hit pattern sign(s_j) where attained.
static __device__ __forceinline__ double w_step_to_bound(double x, double s, double lb, double ub, bool act, int& hit) {
  double st = INFINITY;
  if (act && s != 0.0) st = fmax((lb - x) / s, (ub - x) / s);
  const double t = wmin(st);
  hit = (act && st == t) ? (s > 0.0 ? 1 : (s < 0.0 ? -1 : 0)) : 0;
  return t;
}

// 1-D quadratic minimiser on [lo, hi]: candidates lo, hi, vertex (R20)
static __device__ __forceinline__ void min_quad_1d(double a, double b, double lo, double hi, double c, double& t_out,
                                            double& y_out) {
  double ts[3] = {lo, hi, 0.0};
  int nt = 2;
  if (a != 0.0) {
    const double ext = -0.5 * b / a;
    if (lo < ext && ext < hi) ts[nt++] = ext;
  }
  double best = INFINITY;
  double bt = lo;
  bool first = true;
  for (int k = 0; k < nt; ++k) {
    const double y = ts[k] * (a * ts[k] + b) + c;
    if (first || y < best) {
      best = y;
      bt = ts[k];
      first = false;
    }
  }
  t_out = bt;
  y_out = best;
}

// Q(s) = 1/2 s^T B s + g^T s  (B = B_hat incl. diag_h; R13)
static __device__ __forceinline__ double w_eval_quad(const SolverSmem& S, double gh, double s, int n, int lane) {
  return 0.5 * wquad(S.M, s, n, lane) + wdot(s, gh);
}

// Coleman-Li step selection (R19, R20).  In: p_h (lane), d, x, lb, ub, g_hat.
// Out: step (original space), step_h (hat space), predicted reduction, branch.
static __device__ __noinline__ void w_select_step(const SolverSmem& S, int n, int lane, double x, double lb, double ub, double gh,
                              double d, double p_h, double Delta, double theta, double& step, double& step_h,
                              double& pred, int& branch) {
  const bool act = lane < n;
  double p = d * p_h;
  const bool inb = wall(!act || ((x + p) >= lb && (x + p) <= ub));
  if (inb) {
    step = p;
    step_h = p_h;
    pred = -w_eval_quad(S, gh, p_h, n, lane);
    branch = 0;
    return;
  }
  int hit;
  const double t_b = w_step_to_bound(x, p, lb, ub, act, hit);
  double r_h = (hit != 0) ? -p_h : p_h;
  double r = d * r_h;
  p = p * t_b;
  double ph = p_h * t_b;
  const double x_b = x + p;
  // to_tr: the positive root of ||ph + t r_h|| = Delta (stable form)
  double to_tr;
  {
    const double a = wdot(r_h, r_h), b = wdot(ph, r_h), c = wdot(ph, ph) - Delta * Delta;
    const double dd = sqrt(b * b - a * c);
    const double q = -(b + copysign(dd, b));
    const double t1 = q / a, t2 = c / q;
    to_tr = fmax(t1, t2);
  }
  int hit2;
  const double to_bd = w_step_to_bound(x_b, r, lb, ub, act, hit2);
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
  if (lo <= hi) {
    // Q(ph + t r_h) = a t^2 + b t + c
    const double Mr = wmatvec(S.M, r_h, n, lane);
    const double a = 0.5 * wdot(r_h, Mr);
    const double b = wdot(gh, r_h) + wdot(ph, Mr);
    const double c = 0.5 * wquad(S.M, ph, n, lane) + wdot(gh, ph);
    double rt;
    min_quad_1d(a, b, lo, hi, c, rt, r_val);
    r_h = ph + rt * r_h;
    r = r_h * d;
  } else {
    r_val = INFINITY;
  }
  p = p * theta;
  ph = ph * theta;
  const double p_val = w_eval_quad(S, gh, ph, n, lane);
  double ag_h = -gh;
  double ag = d * ag_h;
  const double t_tr = Delta / wnorm(ag_h);
  int hit3;
  const double t_bd = w_step_to_bound(x, ag, lb, ub, act, hit3);
  const double stride = (t_bd < t_tr) ? theta * t_bd : t_tr;
  double at, ag_val;
  {
    const double a = 0.5 * wquad(S.M, ag_h, n, lane);
    const double b = wdot(gh, ag_h);
    min_quad_1d(a, b, 0.0, stride, 0.0, at, ag_val);
  }
  ag_h = ag_h * at;
  ag = ag * at;
  if (p_val < r_val && p_val < ag_val) {
    step = p;
    step_h = ph;
    pred = -p_val;
    branch = 2;
  } else if (r_val < p_val && r_val < ag_val) {
    step = r;
    step_h = r_h;
    pred = -r_val;
    branch = 1;
  } else {
    step = ag;
    step_h = ag_h;
    pred = -ag_val;
    branch = 3;
  }
  if (!act) {
    step = 0.0;
    step_h = 0.0;
  }
}

// rstep = 0 strict feasibility (R19): x <= lb -> nextafter(lb, ub), x >= ub ->
// nextafter(ub, lb); still outside -> midpoint.
static __device__ __forceinline__ double strict_feasible0(double x, double lb, double ub) {
  double xn = x;
  if (x <= lb) xn = nextafter(lb, ub);
  else if (x >= ub) xn = nextafter(ub, lb);
  if (xn < lb || xn > ub) xn = 0.5 * (lb + ub);
  return xn;
}

// ----------------------------------------------------------- control logic
static __device__ __forceinline__ void st_trace(FitState* st, int lane, double cost_new, double ratio) {
  if (st->trace_cap > 0 && st->trace_len < st->trace_cap) {
    if (lane == 0) {
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
    }
    __syncwarp();
    if (lane == 0) st->trace_len = st->trace_len + 1;
    __syncwarp();
  }
}

// Unpack the K-vector into (cost, g, G) at the current iterate.
static __device__ __forceinline__ void st_take_pass(FitState* st, const double* kv, int n, int lane) {
  if (lane < n) {
    st->g[lane] = kv[tri_slot(n, lane, n)];
    for (int k = 0; k < n; ++k) {
      const int a = lane < k ? lane : k, b = lane < k ? k : lane;
      st->G[lane * NMAX + k] = kv[tri_slot(n, a, b)];
    }
  }
  if (lane == 0) st->cost = 0.5 * kv[tri_slot(n, n, n)];
  __syncwarp();
}

// scale_inv from the Gram diagonal (reading R3: column norms of J = sqrt(G_jj))
static __device__ __forceinline__ void st_update_scale(FitState* st, int n, int lane, bool first) {
  if (lane < n) {
    double si = sqrt(st->G[lane * NMAX + lane]);
    if (first) {
      if (si == 0.0) si = 1.0;
    } else {
      si = fmax(si, st->scale_inv[lane]);
    }
    st->scale_inv[lane] = si;
  }
  __syncwarp();
}

// Coleman-Li vector v, dv (R19)
static __device__ __forceinline__ void cl_vector(double x, double g, double lb, double ub, double& v, double& dv) {
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

// Solve the subproblem for the current hat space and stage the trial point
// in st->x_eval (Alg. 1 l.141-148 / Alg. 2 / select_step).  Then set the phase
// of the next pass.
static __device__ void st_make_trial(FitState* st, SolverSmem& S, int n, int lane) {
  const bool act = lane < n;
  // restore the hat space (S.V, S.M) from global state
  for (int e = lane; e < n * n; e += 32) {
    const int i = e / n, j = e % n;
    S.V[i][j] = st->V[i * NMAX + j];
    S.M[i][j] = st->Gh[i * NMAX + j];
  }
  __syncwarp();
  const double lam = act ? st->lam[lane] : 0.0;
  const double suf = act ? st->suf[lane] : 0.0;
  const double Delta = st->Delta;
  double alpha = st->alpha;
  double p_h;
  const long long c0 = clock64();
  warp_solve_tr(S, n, st->m_global, lam, suf, Delta, alpha, p_h, lane, nullptr);
  if (lane == 0) st->prof[1] += clock64() - c0;
  const double x = act ? st->x[lane] : 0.0;
  const double d = act ? st->d[lane] : 0.0;
  const double gh = act ? st->gh[lane] : 0.0;
  double step, step_h, pred, x_new;
  int branch = -1;
  if (st->bounded) {
    const double lb = act ? st->lb[lane] : 0.0, ub = act ? st->ub[lane] : 0.0;
    const long long c1 = clock64();
    w_select_step(S, n, lane, x, lb, ub, gh, d, p_h, Delta, st->theta, step, step_h, pred, branch);
    if (lane == 0) st->prof[2] += clock64() - c1;
    x_new = act ? strict_feasible0(x + step, lb, ub) : 0.0;
  } else {
    step_h = p_h;
    pred = -w_eval_quad(S, gh, step_h, n, lane);  // Eq. 15 denominator (R13)
    step = d * step_h;                            // Alg. 3 l.185: w = D^-1 p
    x_new = x + step;
  }
  const double hn = wnorm(act ? step_h : 0.0);
  const double sn = wnorm(act ? step : 0.0);
  if (act) {
    st->x_eval[lane] = x_new;
    st->step[lane] = step;
    st->step_h[lane] = step_h;
  }
  if (lane == 0) {
    st->alpha = alpha;
    st->pred = pred;
    st->hn = hn;
    st->step_norm = sn;
    st->Delta_used = Delta;
    st->branch = branch;
    st->phase = (st->policy == 1) ? PH_TRIAL_R : PH_TRIAL_J;
  }
  __syncwarp();
}

// Alg. 1 loop top: termination by gtol / max_nfev, then the hat space of the
// new iterate (Eq. 7-8, App. B) and the first trial.
static __device__ void st_outer_top(FitState* st, SolverSmem& S, int n, int lane) {
  const bool act = lane < n;
  const double x = act ? st->x[lane] : 0.0;
  const double g = act ? st->g[lane] : 0.0;
  const double lb = act ? st->lb[lane] : 0.0, ub = act ? st->ub[lane] : 0.0;
  double v = 1.0, dv = 0.0;
  double gnorm;
  if (st->bounded) {
    if (act) cl_vector(x, g, lb, ub, v, dv);
    gnorm = wmax(act ? fabs(g * v) : 0.0);
  } else {
    gnorm = wmax(act ? fabs(g) : 0.0);
  }
  int status = st->status;
  if (gnorm < st->gtol) status = 1;  // R16
  if (lane == 0) {
    st->gnorm = gnorm;
    st->status = status;
  }
  __syncwarp();
  if (status != STATUS_NONE || st->nfev == st->max_nfev) {
    if (lane == 0) {
      if (status == STATUS_NONE) st->status = 0;
      st->phase = PH_DONE;
      st->cont = 0;
    }
    __syncwarp();
    return;
  }
  const double si = act ? st->scale_inv[lane] : 1.0;
  double d, diag_h = 0.0;
  if (st->bounded) {
    if (dv != 0.0) v *= si;
    d = sqrt(v) / si;          // R19: d = v^0.5 * scale
    diag_h = g * dv / si;      // C = diag(g * scale) Jv
  } else {
    d = 1.0 / si;              // Eq. 8: J_hat = J D^-1
  }
  if (!act) {
    d = 0.0;
    diag_h = 0.0;
  }
  const double gh = d * g;
  if (act) {
    st->d[lane] = d;
    st->diag_h[lane] = diag_h;
    st->gh[lane] = gh;
  }
  __syncwarp();
  // B_hat = d G d (+ diag_h): the scaled Gram (Eq. 8), eigensolver input S.A
  // and quadratic-form matrix S.M
  for (int e = lane; e < n * n; e += 32) {
    const int i = e / n, j = e % n;
    double b = st->d[i] * st->G[i * NMAX + j] * st->d[j];
    if (i == j) b += st->diag_h[i];
    S.A[i][j] = b;
    S.M[i][j] = b;
    st->Gh[i * NMAX + j] = b;
  }
  const int warm = st->have_V;
  if (warm) {
    for (int e = lane; e < NMAX * NMAX; e += 32) {
      const int i = e / NMAX, j = e % NMAX;
      S.V[i][j] = (i < n && j < n) ? st->V[i * NMAX + j] : 0.0;
    }
  }
  __syncwarp();
  double lam;
  const long long c0 = clock64();
  warp_eig(S, n, lane, lam, warm);
  if (lane == 0) st->prof[0] += clock64() - c0;
  const double suf = wVtx(S.V, gh, n, lane);  // S^T U^T r = V^T g_hat (c.1b)
  if (act) {
    st->lam[lane] = lam;
    st->suf[lane] = suf;
  }
  for (int e = lane; e < n * n; e += 32) {
    const int i = e / n, j = e % n;
    st->V[i * NMAX + j] = S.V[i][j];
  }
  if (lane == 0) {
    st->theta = fmax(0.995, 1.0 - gnorm);
    st->actual = -1.0;
    st->have_V = 1;
  }
  __syncwarp();
  st_make_trial(st, S, n, lane);
}

// Initialisation after the J-pass at x0 (Alg. 1 l.137-138; R3, R4, R18).
static __device__ void st_init(FitState* st, SolverSmem& S, const double* kv, int n, int lane) {
  const bool act = lane < n;
  if (kv[tri_count(n)] != 0.0) {  // R18: residuals at x0 must be finite
    if (lane == 0) {
      st->error = -3;
      st->status = -3;
      st->phase = PH_DONE;
      st->cont = 0;
    }
    __syncwarp();
    return;
  }
  st_take_pass(st, kv, n, lane);
  if (lane == 0) {
    st->nfev = 1;
    st->njev = 1;
    st->nit = 0;
    st->alpha = 0.0;
    st->status = STATUS_NONE;
  }
  if (st->jacmode) {
    st_update_scale(st, n, lane, true);
  } else if (act) {
    st->scale_inv[lane] = st->xs_inv[lane];
  }
  __syncwarp();
  const double x = act ? st->x[lane] : 0.0;
  const double si = act ? st->scale_inv[lane] : 0.0;
  double Delta;
  if (st->bounded) {  // R4
    double v = 1.0, dv = 0.0;
    if (act) cl_vector(x, st->g[lane], st->lb[lane], st->ub[lane], v, dv);
    if (dv != 0.0) v *= si;
    Delta = wnorm(act ? x * si / sqrt(v) : 0.0);
  } else {
    Delta = wnorm(act ? x * si : 0.0);
  }
  if (Delta == 0.0) Delta = 1.0;
  if (lane == 0) st->Delta = Delta;
  __syncwarp();
  st_outer_top(st, S, n, lane);
}

// End of the inner (retry) loop: accept or keep x, count the iteration.
// For the conservative policy an accepted step first needs the J-pass at x_new.
static __device__ void st_end_inner(FitState* st, SolverSmem& S, int n, int lane, bool have_jac) {
  const bool act = lane < n;
  if (st->actual > 0.0) {
    if (!have_jac) {  // conservative: J at the new x (counts as njev there)
      if (act) st->x[lane] = st->x_eval[lane];
      if (lane == 0) {
        st->cost = st->cost_new;
        st->phase = PH_ACCEPT_J;
      }
      __syncwarp();
      return;
    }
    if (act) st->x[lane] = st->x_eval[lane];
    __syncwarp();
    st_take_pass(st, st->kv, n, lane);
    if (lane == 0) {
      st->cost = st->cost_new;  // SciPy keeps the trial's cost
      st->njev = st->njev + 1;
    }
    __syncwarp();
    if (st->jacmode) st_update_scale(st, n, lane, false);
  }
  if (lane == 0) st->nit = st->nit + 1;  // R27
  __syncwarp();
  st_outer_top(st, S, n, lane);
}

// After a trial pass at x_eval (speculative J-pass or conservative r-pass).
static __device__ void st_after_trial(FitState* st, SolverSmem& S, const double* kv, int n, int lane, bool jac) {
  const double rr = jac ? kv[tri_slot(n, n, n)] : kv[0];
  const double bad = jac ? kv[tri_count(n)] : kv[1];
  if (lane == 0) st->nfev = st->nfev + 1;
  __syncwarp();
  if (bad != 0.0) {  // R17: shrink and retry, no termination test
    if (lane == 0) st->Delta = 0.25 * st->hn;
    __syncwarp();
    st_trace(st, lane, NAN, NAN);
    if (st->nfev < st->max_nfev) {
      st_make_trial(st, S, n, lane);
      return;
    }
    if (lane == 0) st->actual = -1.0;
    __syncwarp();
    st_end_inner(st, S, n, lane, jac);
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
  // termination (R16), x_norm of the pre-step x
  const bool act = lane < n;
  const double xnorm = wnorm(act ? st->x[lane] : 0.0);
  const bool ft = actual < st->ftol * st->cost && ratio > 0.25;
  const bool xt = st->step_norm < st->xtol * (st->xtol + xnorm);
  const int status = (ft && xt) ? 4 : (ft ? 2 : (xt ? 3 : STATUS_NONE));
  if (lane == 0) {
    st->cost_new = cost_new;
    st->actual = actual;
    st->ratio = ratio;
  }
  __syncwarp();
  st_trace(st, lane, cost_new, ratio);
  if (status != STATUS_NONE) {
    if (lane == 0) st->status = status;
    __syncwarp();
    st_end_inner(st, S, n, lane, jac);
    return;
  }
  if (lane == 0) {
    st->alpha = st->alpha * (st->Delta / Delta_new);  // R5
    st->Delta = Delta_new;
  }
  __syncwarp();
  if (actual <= 0.0 && st->nfev < st->max_nfev) {
    st_make_trial(st, S, n, lane);  // R15: same hat space, new radius
    return;
  }
  st_end_inner(st, S, n, lane, jac);
}

// Entry point: called by warp 0 of the last block of every pass kernel in a
// fit, with the combined K-vector of the pass that just finished.
static __device__ __noinline__ void fit_after_pass(FitState* st, SolverSmem& S, const double* kv, bool jac) {
  const int lane = threadIdx.x & 31;
  const long long cstart = clock64();
  const int n = st->n;
  const int KS = jac ? tri_count(n) + 1 : 2;
  for (int k = lane; k < KS; k += 32) st->kv[k] = kv[k];
  if (lane == 0) st->launches = st->launches + 1;
  __syncwarp();
  const int phase = st->phase;
  if (phase == PH_INIT_J) {
    st_init(st, S, kv, n, lane);
  } else if (phase == PH_TRIAL_J && jac) {
    st_after_trial(st, S, kv, n, lane, true);
  } else if (phase == PH_TRIAL_R && !jac) {
    st_after_trial(st, S, kv, n, lane, false);
  } else if (phase == PH_ACCEPT_J && jac) {
    st_take_pass(st, kv, n, lane);  // g, G at the accepted x (cost kept: SciPy)
    if (lane == 0) {
      st->cost = st->cost_new;
      st->njev = st->njev + 1;
    }
    __syncwarp();
    if (st->jacmode) st_update_scale(st, n, lane, false);
    if (lane == 0) st->nit = st->nit + 1;
    __syncwarp();
    st_outer_top(st, S, n, lane);
  }
  __syncwarp();
  if (lane == 0) st->prof[3] += clock64() - cstart;
  __syncwarp();
}

}  // namespace jf
