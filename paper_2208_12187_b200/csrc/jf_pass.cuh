// jf_pass.cuh — the data-parallel pass over the m points.
//
// One kernel template serves both passes of the method:
//   J-pass (JAC = true):  per point i, the model value and Jacobian row through
//       dual numbers, r_i = h - z_i (Eq. 1), and the fp64 upper
//       triangle of [J_i | r_i]^T [J_i | r_i] accumulated in registers: that
//       is the Gram B = J^T J (Eq. 5), the gradient g = J^T r (Eq. 4) and
//       r^T r = 2 f (Eq. 2) at once, without ever storing J.
//   r-pass (JAC = false): r^T r only, at a trial point (Eq. 15 numerator).
// Both also count non-finite residuals (reading R17).
//
// Reduction: per-thread registers -> warp xor-butterfly -> shared memory in
// warp order -> one partial K-vector per block in HBM -> the LAST block to
// finish (atomic ticket) sums the partials in block order.  The grid size is
// a pure function of m, each thread visits a fixed index sequence and every
// sum has a fixed order, so a pass is bitwise reproducible (H4).  No floating
// point atomics.
//
// Multi-GPU (use_comm): the last block pushes its K-vector into every peer's
// mailbox over NVLink (P2P stores), raises its epoch flag there, waits for all
// peers' flags in its own mailbox and sums the R vectors in rank order — an
// all-reduce fused into the pass kernel, identical on every rank.
//
// Epilogue EPI_FIT: warp 0 of the last block then runs the solver state
// machine (jf_solver.cuh) and, inside a CUDA graph, sets the WHILE node's
// condition — so a whole fit is one graph launch.
#pragma once

#include "jf_common.cuh"
#include "jf_dual.cuh"
#include "jf_models.cuh"
#include "jf_solver.cuh"

namespace jf {

template <class Model, bool JAC>
struct PassShape {
  static constexpr int N = Model::N;
  static constexpr int KT = JAC ? tri_count(N) : 1;  // accumulated slots
  static constexpr int KS = KT + 1;                   // + non-finite count
};

template <class Model>
struct MinBlocks {
  static constexpr int value = Model::N <= 7 ? 2 : 1;
};

// Accumulate one point's contribution.
template <class Model, bool JAC, class H>
__device__ __forceinline__ void accumulate(double (&acc)[PassShape<Model, JAC>::KT], int& bad, const H& h, double z,
                                           double wsig, bool weighted) {
  constexpr int N = Model::N;
  if constexpr (JAC) {
    double w[N + 1];
    static_for<N>([&](auto J) {
      constexpr int j = decltype(J)::value;
      w[j] = h.template partial<j>();
    });
    w[N] = h.v - z;  // Eq. 1
    if (weighted) {
#pragma unroll
      for (int j = 0; j <= N; ++j) w[j] *= wsig;  // App. C Eq. C13-C16
    }
    bad += isfinite(w[N]) ? 0 : 1;
    int s = 0;
#pragma unroll
    for (int j = 0; j <= N; ++j) {
#pragma unroll
      for (int k = j; k <= N; ++k) {
        acc[s] = fma(w[j], w[k], acc[s]);
        ++s;
      }
    }
  } else {
    double r = h - z;
    if (weighted) r *= wsig;
    bad += isfinite(r) ? 0 : 1;
    acc[0] = fma(r, r, acc[0]);
  }
}

// Block-level combine of per-thread accumulators into partials[blockIdx.x].
template <int KT>
__device__ __forceinline__ void block_partial(double (&acc)[KT], int bad, double* __restrict__ part,
                                              double (*red)[KT + 1]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < KT; ++k) {
    double v = acc[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    if (lane == 0) red[warp][k] = v;
  }
  const int b = __reduce_add_sync(FULL, bad);
  if (lane == 0) red[warp][KT] = (double)b;
  __syncthreads();
  for (int k = threadIdx.x; k < KT + 1; k += BLOCK) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < NWARP; ++w) s += red[w][k];
    part[(size_t)blockIdx.x * (KT + 1) + k] = s;
  }
}

// Last-block deterministic sum over the grid's partials; result in out[0..KS).
template <int KS>
__device__ __forceinline__ void grid_combine(const double* __restrict__ part, int nblk, double* out,
                                             double* scratch /* BLOCK doubles */) {
  constexpr int NSEG = (BLOCK / KS) > 0 ? (BLOCK / KS) : 1;
  const int t = threadIdx.x;
  if (t < NSEG * KS) {
    const int k = t % KS, seg = t / KS;
    double s = 0.0;
    for (int b = seg; b < nblk; b += NSEG) s += __ldcg(part + (size_t)b * KS + k);
    scratch[seg * KS + k] = s;
  }
  __syncthreads();
  for (int k = t; k < KS; k += BLOCK) {
    double s = 0.0;
#pragma unroll
    for (int seg = 0; seg < NSEG; ++seg) s += scratch[seg * KS + k];
    out[k] = s;
  }
  __syncthreads();
}

// Cross-rank combine through the NVLink mailboxes (see jf_comm.cu).
template <int KS>
__device__ __forceinline__ bool comm_combine(const CommDev& cm, unsigned long long epoch, double* vec /* smem */) {
  const int R = cm.nranks, me = cm.rank;
  const int par = (int)(epoch & 1ull);
  // 1. push my vector into slot [par][me] of every mailbox (peer stores over NVLink)
  for (int p = 0; p < R; ++p) {
    double* dst = cm.mbox_data[p] + ((size_t)par * R + me) * KMAX;
    for (int k = threadIdx.x; k < KS; k += BLOCK) dst[k] = vec[k];
  }
  __threadfence_system();
  __syncthreads();
  // 2. raise my flag in every mailbox
  if (threadIdx.x < R) {
    volatile unsigned long long* f = cm.mbox_flag[threadIdx.x] + me;
    *f = epoch;
  }
  __threadfence_system();
  // 3. wait for every rank's flag in my mailbox
  __shared__ int timed_out;
  if (threadIdx.x == 0) timed_out = 0;
  __syncthreads();
  if (threadIdx.x < R) {
    volatile unsigned long long* f = cm.mbox_flag[me] + threadIdx.x;
    long long spins = 0;
    while (*f < epoch) {
      if (++spins > (1ll << 31)) {
        timed_out = 1;
        break;
      }
    }
  }
  __threadfence_system();
  __syncthreads();
  if (timed_out) return false;
  // 4. sum in rank order (identical on every rank)
  const double* box = cm.mbox_data[me] + (size_t)par * R * KMAX;
  for (int k = threadIdx.x; k < KS; k += BLOCK) {
    double s = 0.0;
    for (int p = 0; p < R; ++p) s += __ldcv(box + (size_t)p * KMAX + k);
    vec[k] = s;
  }
  __syncthreads();
  return true;
}

// Per-thread point iterator over the shard: index i and its coordinates.
template <int D, int COORD>
struct PointIter {
  int64_t i, S;
  // grid state
  int64_t row, col, dr, dc, W;
  double row0d;
  __device__ __forceinline__ void init(const PassArgs& a, int64_t i0, int64_t stride) {
    i = i0;
    S = stride;
    if constexpr (COORD == COORD_GRID) {
      W = a.W;
      row = i0 / W;
      col = i0 - row * W;
      dr = stride / W;
      dc = stride - dr * W;
      row0d = (double)a.row0;
    }
  }
  __device__ __forceinline__ void advance() {
    i += S;
    if constexpr (COORD == COORD_GRID) {
      col += dc;
      row += dr;
      if (col >= W) {
        col -= W;
        ++row;
      }
    }
  }
};

// The pass kernel.  st != nullptr and epilogue == EPI_FIT: part of a fit.
template <class Model, bool JAC, int COORD>
__global__ void __launch_bounds__(BLOCK, MinBlocks<Model>::value)
    pass_kernel(const PassArgs* __restrict__ pa, FitState* __restrict__ st, cudaGraphConditionalHandle cond,
                int use_cond) {
  using Sh = PassShape<Model, JAC>;
  constexpr int KT = Sh::KT, KS = Sh::KS;
  const PassArgs& a = *pa;

  // Phase predication inside a fit: run only when this pass type is wanted.
  if (a.epilogue == EPI_FIT) {
    const int ph = st->phase;
    const bool want = JAC ? (ph == PH_INIT_J || ph == PH_TRIAL_J || ph == PH_ACCEPT_J) : (ph == PH_TRIAL_R);
    if (!want) return;
  }
  const double* xs = (a.epilogue == EPI_FIT) ? st->x_eval : a.x;
  double xv[Model::N];
#pragma unroll
  for (int j = 0; j < Model::N; ++j) xv[j] = xs[j];
  const auto pre = Model::template prologue<JAC>(xv);

  double acc[KT];
#pragma unroll
  for (int k = 0; k < KT; ++k) acc[k] = 0.0;
  int bad = 0;

  const int64_t m = a.m;
  const int64_t stride = (int64_t)gridDim.x * BLOCK;
  PointIter<Model::D, COORD> it;
  it.init(a, (int64_t)blockIdx.x * BLOCK + threadIdx.x, stride);
  const double* __restrict__ z = a.z;
  const double* __restrict__ y0 = a.y0;
  const double* __restrict__ y1 = a.y1;
  const double* __restrict__ ws = a.wsig;
  const bool weighted = ws != nullptr;
  for (; it.i < m; it.advance()) {
    const int64_t i = it.i;
    const double zi = __ldg(z + i);
    const double wi = weighted ? __ldg(ws + i) : 1.0;
    if constexpr (Model::D == 1) {
      double t;
      if constexpr (COORD == COORD_IMPLICIT_T) t = fma((double)(a.index0 + i), a.dt, a.t0);
      else t = __ldg(y0 + i);
      const auto h = Model::template point<JAC>(pre, t);
      accumulate<Model, JAC>(acc, bad, h, zi, wi, weighted);
    } else {
      double X, Y;
      if constexpr (COORD == COORD_GRID) {
        X = (double)it.col;
        Y = (double)it.row + it.row0d;
      } else {
        X = __ldg(y0 + i);
        Y = __ldg(y1 + i);
      }
      const auto h = Model::template point<JAC>(pre, X, Y);
      accumulate<Model, JAC>(acc, bad, h, zi, wi, weighted);
    }
  }

  __shared__ double red[NWARP][KT + 1];
  __shared__ double vec[KMAX];
  __shared__ double scratch[BLOCK];
  __shared__ unsigned int is_last;
  block_partial<KT>(acc, bad, a.partials, red);
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) is_last = (atomicAdd(a.ticket, 1u) == gridDim.x - 1) ? 1u : 0u;
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  grid_combine<KS>(a.partials, gridDim.x, vec, scratch);
  if (threadIdx.x == 0) *a.ticket = 0u;  // ready for the next launch

  if (a.use_comm) {
    const unsigned long long epoch = (a.epilogue == EPI_FIT) ? (st->comm_epoch + 1) : (a.comm.epoch + 1);
    const bool ok = comm_combine<KS>(a.comm, epoch, vec);
    if (threadIdx.x == 0 && a.epilogue == EPI_FIT) st->comm_epoch = epoch;
    if (!ok) {
      if (threadIdx.x == 0 && a.epilogue == EPI_FIT) {
        st->error = -5;
        st->status = -5;
        st->cont = 0;
        st->phase = PH_DONE;
      }
      if (threadIdx.x == 0 && use_cond) cudaGraphSetConditional(cond, 0u);
      return;
    }
  }

  if (a.epilogue != EPI_FIT) {
    for (int k = threadIdx.x; k < KS; k += BLOCK) a.out[k] = vec[k];
    return;
  }
  // ---- fit epilogue: one warp runs the solver state machine
  if (threadIdx.x < 32) {
    __shared__ SolverSmem S;
    fit_after_pass(st, S, vec, JAC);
    if (threadIdx.x == 0 && use_cond) cudaGraphSetConditional(cond, st->cont ? 1u : 0u);
  }
}

}  // namespace jf
