// jf_solver.cu — the single-warp solver kernel and the
// stand-alone subproblem hook (jf_trust_region_step).
//
// One launch of solver_kernel follows every pass kernel of a fit: it takes
// the pass's combined K-vector, advances the device state machine of
// jf_solver.cuh (accept/reject, radius, termination, the next trust-region
// step) and sets the CUDA-graph WHILE condition.  Keeping it out of the pass
// kernels leaves their register allocation to the data-parallel loop.
#include <cstdio>

#include "jf_solver.cuh"

namespace jf {

__global__ void __launch_bounds__(32, 1)
    solver_kernel(FitState* __restrict__ st, const double* __restrict__ kv, cudaGraphConditionalHandle cond,
                  int use_cond) {
  __shared__ SolverSmem S;
  __shared__ FitState sst;
  const int lane = threadIdx.x;
  (void)lane;
  // PDL: wait for the pass kernel before us (a no-op for a plain launch)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  // the next pass kernel may be scheduled now; it waits for this grid
  asm volatile("griddepcontrol.launch_dependents;");
  if (lane == 0) atomicAdd(&st->kernels, 1);
  __syncwarp();
  if (st->pass_ready != 0) {
    solver_run<0>(st, S, sst, kv, st->pass_ready == 1, cond, use_cond);
  } else if (lane == 0 && use_cond) {
    cudaGraphSetConditional(cond, st->cont ? 1u : 0u);
  }
}

const void* solver_kernel_ptr() { return (const void*)solver_kernel; }

int launch_solver(FitState* st, const double* kv, cudaStream_t s) {
  solver_kernel<<<1, 32, 0, s>>>(st, kv, (cudaGraphConditionalHandle)0, 0);
  return cudaGetLastError() == cudaSuccess ? 0 : -4;
}

__global__ void tr_step_kernel(const double* hatG, const double* hatg, int n, int64_t m, double Delta,
                               double alpha_in, double* out, int dbg) {
  __shared__ SolverSmem S;
  const int lane = threadIdx.x;
  for (int e = lane; e < n * n; e += 32) {
    const int i = e / n, j = e % n;
    S.A[i][j] = hatG[e];
    S.M[i][j] = hatG[e];
  }
  __syncwarp();
  const long long c0 = clock64();
  const int sw = warp_eig(S, n, 0);
  const long long c1 = clock64();
  if (lane == 0) {
    double suf[NMAX], p[NMAX];
    for (int j = 0; j < n; ++j) {  // suf = V^T g_hat
      double t = 0.0;
      for (int i = 0; i < n; ++i) t = fma(S.V[i][j], hatg[i], t);
      suf[j] = t;
    }
    double alpha = alpha_in;
    int it = -1;
    switch (n) {
#define JF_TR_CASE(N) \
  case N: it = solve_tr<N>(S, m, suf, Delta, alpha, p); break;
      JF_TR_CASE(1) JF_TR_CASE(2) JF_TR_CASE(3) JF_TR_CASE(4) JF_TR_CASE(5) JF_TR_CASE(6) JF_TR_CASE(7)
      JF_TR_CASE(8) JF_TR_CASE(9) JF_TR_CASE(10) JF_TR_CASE(11) JF_TR_CASE(12) JF_TR_CASE(13)
      JF_TR_CASE(14) JF_TR_CASE(15) JF_TR_CASE(16)
#undef JF_TR_CASE
      default: break;
    }
    const long long c2 = clock64();
    if (dbg) printf("tr_step n=%d sweeps=%d eig_cycles=%lld solve_cycles=%lld iters=%d\n", n, sw, c1 - c0, c2 - c1, it);
    for (int j = 0; j < n; ++j) {
      out[j] = p[j];
      out[NMAX + j] = S.lam[j];
    }
    out[2 * NMAX] = alpha;
    out[2 * NMAX + 1] = it;
  }
}

int launch_tr_step(const double* hatG, const double* hatg, int n, int64_t m, double Delta, double alpha_in,
                   double* out, int dbg, cudaStream_t s) {
  tr_step_kernel<<<1, 32, 0, s>>>(hatG, hatg, n, m, Delta, alpha_in, out, dbg);
  return cudaGetLastError() == cudaSuccess ? 0 : -4;
}

// The Coleman-Li step selection alone (jf_select_step, parity hook): lane 0
// runs select_step<n> on the scaled quadratic model B_hat (incl. diag_h).
__global__ void select_step_kernel(const double* in, int n, double Delta, double theta, double* out) {
  __shared__ SolverSmem S;
  // in: B_hat (n*n) | g_hat | x | lb | ub | d | p_h   (n each)
  const int lane = threadIdx.x;
  for (int e = lane; e < n * n; e += 32) S.M[e / n][e % n] = in[e];
  __syncwarp();
  if (lane == 0) {
    const double* gh = in + n * n;
    const double* x = gh + n;
    const double* lb = x + n;
    const double* ub = lb + n;
    const double* d = ub + n;
    const double* ph = d + n;
    double step[NMAX], step_h[NMAX], pred = 0.0;
    int branch = -1;
    switch (n) {
#define JF_SEL_CASE(N) \
  case N: select_step<N>(S, x, lb, ub, gh, d, ph, Delta, theta, step, step_h, pred, branch); break;
      JF_SEL_CASE(1) JF_SEL_CASE(2) JF_SEL_CASE(3) JF_SEL_CASE(4) JF_SEL_CASE(5) JF_SEL_CASE(6) JF_SEL_CASE(7)
      JF_SEL_CASE(8) JF_SEL_CASE(9) JF_SEL_CASE(10) JF_SEL_CASE(11) JF_SEL_CASE(12) JF_SEL_CASE(13)
      JF_SEL_CASE(14) JF_SEL_CASE(15) JF_SEL_CASE(16)
#undef JF_SEL_CASE
      default: break;
    }
    for (int j = 0; j < n; ++j) {
      out[j] = step[j];
      out[NMAX + j] = step_h[j];
    }
    out[2 * NMAX] = pred;
    out[2 * NMAX + 1] = branch;
  }
}

int launch_select_step(const double* in, int n, double Delta, double theta, double* out, cudaStream_t s) {
  select_step_kernel<<<1, 32, 0, s>>>(in, n, Delta, theta, out);
  return cudaGetLastError() == cudaSuccess ? 0 : -4;
}

}  // namespace jf
