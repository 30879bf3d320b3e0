// jf_state.cuh — the device-resident state of one fit and
// the phases of the pass / solver alternation.  Shared by the pass kernels
// (which read the phase and the point to evaluate) and the solver kernel.
#pragma once

#include <cstddef>

#include "jf_common.cuh"

namespace jf {

enum Phase : int32_t {
  PH_INIT_J = 0,    // J-pass at x0
  PH_TRIAL_J = 1,   // speculative policy: J-pass at a trial point
  PH_TRIAL_R = 2,   // conservative policy: residual pass at a trial point
  PH_ACCEPT_J = 3,  // conservative policy: J-pass at the accepted point
  PH_DONE = 4,
  PH_QR2 = 5        // TSQR (CholeskyQR2): preconditioned J-pass at the current x
};

// TSQR working set (device, one per fit context): CholeskyQR2 factors of
// W = [J | r], (n+1) x (n+1) row-major upper triangular.
struct QRState {
  double prec[(NMAX + 1) * (NMAX + 1)];  // P = R1^-1 (read by the preconditioned pass)
  double R1[(NMAX + 1) * (NMAX + 1)];    // chol(W^T W)
  double R[(NMAX + 1) * (NMAX + 1)];     // R = R2 R1
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
  int32_t kernels;     // kernel launches of this fit (pass kernels incl. predicated-out ones + solver kernels)
  int32_t tl_n;        // timeline entries written
  int32_t pass_ready;  // set by a pass kernel's last block: 1 J-pass, 2 r-pass result in kv_in
  int32_t have_eig;    // eigendecomposition of the current B_hat computed (lazy, per iteration)
  unsigned long long comm_epoch;
  unsigned long long epi_ns;  // device time spent in the solver epilogue (globaltimer)
  long long prof[8];          // SM cycles: eig, trial solve, select_step, fit_after_pass, after_trial,
                              // accept (take_pass + scale), outer_top (pre-trial), trial finish
  double cost, cost_new, Delta, alpha, gnorm, theta, actual;
  double pred, hn, step_norm, Delta_used, ratio;
  double kappa2_gn;  // cond(B_hat)^2 bound from the last Gauss-Newton Cholesky (tr B_hat ||L^-1||_F^2; +inf if none)
  double x[NMAX], x_eval[NMAX];
  double g[NMAX], scale_inv[NMAX];
  // hat space of the current iterate (reused by rejected trials, R15)
  double d[NMAX], diag_h[NMAX], gh[NMAX], suf[NMAX];
  double step[NMAX], step_h[NMAX];
  int32_t pcov_done, qr_mode;  // qr_mode: TSQR (CholeskyQR2 + SVD of R) instead of the Gram eigensolver
  int32_t qr_after;            // what follows the PH_QR2 pass: 0 initialisation, 1 an accepted step
  int32_t qr_stage;            // 0: CholeskyQR2's second pass pending; 1, 2: shifted CholeskyQR3's
                               // first / second preconditioned pass pending (reading R31)
  int32_t pad_qr;
  int32_t auto_mode;           // solver AUTO: Gram until the conditioning calls for TSQR (checked at x0 and at accepted steps)
  QRState* qr;                 // device TSQR working set
  double* prec;                // = qr->prec (read by the preconditioned pass kernel)
  int32_t has_pre, pad_pre;    // pre: the moment J-pass prologue at x_eval (gauss2d_prologue, _x2)
  double pre[16];
  // ---- bulk: every entry is written on the device before it is read (the
  // host uploads only the fields above, FITSTATE_UPLOAD bytes, per fit)
  unsigned long long tl[64];  // device timeline (globaltimer ns): pass start/end, solver start/end
  double G[NMAX * NMAX];      // J^T J at the current iterate
  double Gh[NMAX * NMAX];     // B_hat of the current iterate
  double lam[NMAX], V[NMAX * NMAX];  // its eigendecomposition (valid while have_eig / have_V)
  double kv[KMAX];            // K-vector of the last pass
  double pcov[NMAX * NMAX];   // parameter covariance at the final x (curve_fit's pcov)
};
constexpr size_t FITSTATE_UPLOAD = offsetof(FitState, tl);

// The parameter-only prologue of the n = 7 moment J-pass (the rotated 2D
// Gaussian, SPEC S:463 form; the expressions of Gauss2DComponent::prologue):
// pre = {A, x0, y0, a, 2b, c2, off, rho}, rho = exp(-2 a 32^2) the row
// recurrence's step factor (lane stride 32).  Computed once per pass by the
// caller — the host for a host x, the solver kernel for the next pass of a
// fit — instead of by every thread of the pass.
__host__ __device__ inline void gauss2d_prologue(const double* x, double* pre) {
  const double sx = x[3], sy = x[4], th = x[5];
  const double C = cos(th), S = sin(th);
  const double ix = 0.5 / (sx * sx), iy = 0.5 / (sy * sy);
  const double CC = C * C, SS = S * S;
  const double a = CC * ix + SS * iy;
  pre[0] = x[0];
  pre[1] = x[1];
  pre[2] = x[2];
  pre[3] = a;
  pre[4] = 2.0 * ((S * C) * (iy - ix));
  pre[5] = SS * ix + CC * iy;
  pre[6] = x[6];
  pre[7] = exp(-2.0 * a * 32.0 * 32.0);
}
// The two-Gaussian model (n = 13): pre = {A1, x01, y01, a1, 2b1, c21, A2,
// x02, y02, a2, 2b2, c22, off, rho1, rho2} (the expressions of
// ModelGauss2DRotX2::prologue, rho_c = exp(-2 a_c 32^2)).
__host__ __device__ inline void gauss2d_x2_prologue(const double* x, double* pre) {
  for (int c = 0; c < 2; ++c) {
    const double* xc = x + 6 * c;
    const double sx = xc[3], sy = xc[4], th = xc[5];
    const double C = cos(th), S = sin(th);
    const double ix = 0.5 / (sx * sx), iy = 0.5 / (sy * sy);
    const double CC = C * C, SS = S * S;
    const double a = CC * ix + SS * iy;
    double* pc = pre + 6 * c;
    pc[0] = xc[0];
    pc[1] = xc[1];
    pc[2] = xc[2];
    pc[3] = a;
    pc[4] = 2.0 * ((S * C) * (iy - ix));
    pc[5] = SS * ix + CC * iy;
    pre[13 + c] = exp(-2.0 * a * 32.0 * 32.0);
  }
  pre[12] = x[12];
}
#ifdef __CUDACC__
// The same on a whole warp (lane values equal on entry), without divergent
// lanes: sin and cos from one sincos, the two reciprocals on two lanes of the
// same instruction stream; lane 0 writes pre.  (sincos may differ from the
// separate cos / sin in the last bit: a fit's passes agree with a plain pass
// at the same x to ~1e-15, like host- and device-computed prologues, R36.)
__device__ __forceinline__ void gauss2d_prologue_warp(const double* x, double* pre) {
  const int lane = threadIdx.x & 31;
  double S, C;
  sincos(x[5], &S, &C);
  const double sg = (lane & 1) ? x[4] : x[3];
  const double rinv = 0.5 / (sg * sg);
  const double ix = __shfl_sync(0xffffffffu, rinv, 0), iy = __shfl_sync(0xffffffffu, rinv, 1);
  const double CC = C * C, SS = S * S;
  const double a = CC * ix + SS * iy;
  const double rho = exp(-2.0 * a * 32.0 * 32.0);
  if (lane == 0) {
    pre[0] = x[0];
    pre[1] = x[1];
    pre[2] = x[2];
    pre[3] = a;
    pre[4] = 2.0 * ((S * C) * (iy - ix));
    pre[5] = SS * ix + CC * iy;
    pre[6] = x[6];
    pre[7] = rho;
  }
}
// n = 13 on a whole warp: lanes 0-1 the two components' sincos... each lane
// of a pair (lane & 1) one component, the rest on every lane; lane 0 writes.
__device__ __forceinline__ void gauss2d_x2_prologue_warp(const double* x, double* pre) {
  const int lane = threadIdx.x & 31;
  const double* xc = x + 6 * (lane & 1);
  double S, C;
  sincos(xc[5], &S, &C);
  const double ix = 0.5 / (xc[3] * xc[3]), iy = 0.5 / (xc[4] * xc[4]);
  const double CC = C * C, SS = S * S;
  const double a = CC * ix + SS * iy;
  const double b2 = 2.0 * ((S * C) * (iy - ix));
  const double c2 = SS * ix + CC * iy;
  const double rho = exp(-2.0 * a * 32.0 * 32.0);
  const double a_1 = __shfl_sync(0xffffffffu, a, 1), b_1 = __shfl_sync(0xffffffffu, b2, 1);
  const double c_1 = __shfl_sync(0xffffffffu, c2, 1), r_1 = __shfl_sync(0xffffffffu, rho, 1);
  if (lane == 0) {
    for (int c = 0; c < 2; ++c) {
      pre[6 * c + 0] = x[6 * c + 0];
      pre[6 * c + 1] = x[6 * c + 1];
      pre[6 * c + 2] = x[6 * c + 2];
    }
    pre[3] = a;
    pre[4] = b2;
    pre[5] = c2;
    pre[9] = a_1;
    pre[10] = b_1;
    pre[11] = c_1;
    pre[12] = x[12];
    pre[13] = rho;
    pre[14] = r_1;
  }
}
#endif

}  // namespace jf
