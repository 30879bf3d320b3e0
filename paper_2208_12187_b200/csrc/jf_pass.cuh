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

// Accumulate one point's contribution.  CONST_COL: a parameter whose partial
// is identically 1 (the offset); unweighted, its diagonal slot is the point
// count, kept as an integer instead of an fp64 add per point.
template <class Model, bool JAC, class H>
__device__ __forceinline__ void accumulate(double (&acc)[PassShape<Model, JAC>::KT], int& bad, int& cnt,
                                           const H& h, double z, double wsig, bool weighted) {
  constexpr int N = Model::N;
  if constexpr (JAC) {
    constexpr int CC = Model::CONST_COL;
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
    ++cnt;
    int s = 0;
#pragma unroll
    for (int j = 0; j <= N; ++j) {
#pragma unroll
      for (int k = j; k <= N; ++k) {
        if (j == CC && k == CC) {
          if (weighted) acc[s] = fma(w[j], w[k], acc[s]);
        } else {
          acc[s] = fma(w[j], w[k], acc[s]);
        }
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
template <int KT, int TPB>
__device__ __forceinline__ void block_partial(double (&acc)[KT], int bad, double* __restrict__ part,
                                              double (*red)[KT + 1]) {
  constexpr int NW = TPB / 32;
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
  for (int k = threadIdx.x; k < KT + 1; k += TPB) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < NW; ++w) s += red[w][k];
    part[(size_t)blockIdx.x * (KT + 1) + k] = s;
  }
}

// Last-block deterministic sum over the grid's partials; result in out[0..KS).
template <int KS, int TPB>
__device__ __forceinline__ void grid_combine(const double* __restrict__ part, int nblk, double* out,
                                             double* scratch /* TPB doubles */) {
  constexpr int NSEG = (TPB / KS) > 0 ? (TPB / KS) : 1;
  const int t = threadIdx.x;
  if (t < NSEG * KS) {
    const int k = t % KS, seg = t / KS;
    double s = 0.0;
    for (int b = seg; b < nblk; b += NSEG) s += __ldcg(part + (size_t)b * KS + k);
    scratch[seg * KS + k] = s;
  }
  __syncthreads();
  for (int k = t; k < KS; k += TPB) {
    double s = 0.0;
#pragma unroll
    for (int seg = 0; seg < NSEG; ++seg) s += scratch[seg * KS + k];
    out[k] = s;
  }
  __syncthreads();
}

// Cross-rank combine through the NVLink mailboxes (see jf_comm.cu).
template <int KS, int TPB>
__device__ __forceinline__ bool comm_combine(const CommDev& cm, unsigned long long epoch, double* vec /* smem */) {
  const int R = cm.nranks, me = cm.rank;
  const int par = (int)(epoch & 1ull);
  // 1. push my vector into slot [par][me] of every mailbox (peer stores over NVLink)
  for (int p = 0; p < R; ++p) {
    double* dst = cm.mbox_data[p] + ((size_t)par * R + me) * KMAX;
    for (int k = threadIdx.x; k < KS; k += TPB) dst[k] = vec[k];
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
    unsigned long long t0, t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    while (*f < epoch) {
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
      if (t1 - t0 > 20000000000ull) {  // 20 s: a peer is gone
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
  for (int k = threadIdx.x; k < KS; k += TPB) {
    double s = 0.0;
    for (int p = 0; p < R; ++p) s += __ldcv(box + (size_t)p * KMAX + k);
    vec[k] = s;
  }
  __syncthreads();
  return true;
}

// Per-thread point iterator over the shard: index i and, for the implicit
// pixel grid, (row, col) maintained incrementally (no division per point).
template <int COORD>
struct PointIter {
  int64_t i, S;
  int32_t row, col, dr, dc, W;
  __device__ __forceinline__ void init(const PassArgs& a, int64_t i0, int64_t stride) {
    i = i0;
    S = stride;
    if constexpr (COORD == COORD_GRID) {
      W = (int32_t)a.W;
      row = (int32_t)(i0 / a.W);
      col = (int32_t)(i0 - (int64_t)row * a.W);
      dr = (int32_t)(stride / a.W);
      dc = (int32_t)(stride - (int64_t)dr * a.W);
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

// Launch shape per (model, pass): points per thread per iteration (ILP) and
// minimum resident blocks per SM (register budget).
template <class Model, bool JAC>
struct PassCfg {
  static constexpr bool BIG = JAC && Model::N >= 7;
  static constexpr int P = JAC ? (Model::N == 7 ? 2 : 1) : 4;
  static constexpr int TPB = (JAC && Model::N == 7) ? 384 : 256;
  static constexpr int MINB = BIG ? 1 : 2;
};

// The pass kernel.  epilogue == EPI_FIT: one pass of a fit (st is the state).
template <class Model, bool JAC, int COORD, bool WGT>
__global__ void __launch_bounds__((PassCfg<Model, JAC>::TPB), (PassCfg<Model, JAC>::MINB))
    pass_kernel(const PassArgs* __restrict__ pa, FitState* __restrict__ st, cudaGraphConditionalHandle cond,
                int use_cond) {
  using Sh = PassShape<Model, JAC>;
  constexpr int KT = Sh::KT, KS = Sh::KS;
  constexpr int P = PassCfg<Model, JAC>::P;
  constexpr int TPB = PassCfg<Model, JAC>::TPB;
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
  int bad = 0, cnt = 0;

  const int64_t m = a.m;
  const int64_t S = (int64_t)gridDim.x * TPB;
  PointIter<COORD> it;
  it.init(a, (int64_t)blockIdx.x * TPB + threadIdx.x, S);
  const double* __restrict__ z = a.z;
  const double* __restrict__ y0 = a.y0;
  const double* __restrict__ y1 = a.y1;
  const double* __restrict__ ws = a.wsig;
  constexpr bool weighted = WGT;
  constexpr bool EXPL = (COORD == COORD_EXPLICIT);
  constexpr bool TWO = (Model::D == 2);

  // Software pipeline: the loads of the next group of P points are issued
  // before the current group is computed, so HBM latency hides behind the
  // fp64 work of the current points.
  double qz[P], qw[P], qa[P], qb[P];
  auto issue = [&](int64_t base) {
#pragma unroll
    for (int p = 0; p < P; ++p) {
      const int64_t idx = base + p * S;
      const bool v = idx < m;
      qz[p] = v ? __ldg(z + idx) : 0.0;
      qw[p] = (v && weighted) ? __ldg(ws + idx) : 1.0;
      if constexpr (EXPL) {
        qa[p] = v ? __ldg(y0 + idx) : 0.0;
        if constexpr (TWO) qb[p] = v ? __ldg(y1 + idx) : 0.0;
      }
    }
  };
  issue(it.i);
  while (it.i < m) {
    double cz[P], cw[P], cx[P], cy[P];
    bool cv[P];
#pragma unroll
    for (int p = 0; p < P; ++p) {
      cv[p] = it.i < m;
      cz[p] = qz[p];
      cw[p] = qw[p];
      if constexpr (EXPL) {
        cx[p] = qa[p];
        if constexpr (TWO) cy[p] = qb[p];
      } else if constexpr (COORD == COORD_GRID) {
        cx[p] = (double)it.col;
        cy[p] = (double)(it.row + (int32_t)a.row0);
      } else {
        cx[p] = fma((double)(a.index0 + it.i), a.dt, a.t0);
      }
      it.advance();
    }
    issue(it.i);
#pragma unroll
    for (int p = 0; p < P; ++p) {
      if (P == 1 || cv[p]) {
        if constexpr (TWO) {
          const auto h = Model::template point<JAC>(pre, cx[p], cy[p]);
          accumulate<Model, JAC>(acc, bad, cnt, h, cz[p], cw[p], weighted);
        } else {
          const auto h = Model::template point<JAC>(pre, cx[p]);
          accumulate<Model, JAC>(acc, bad, cnt, h, cz[p], cw[p], weighted);
        }
      }
    }
  }
  if constexpr (JAC) {
    constexpr int CC = Model::CONST_COL;
    if (!weighted) acc[tri_slot(Model::N, CC, CC)] = (double)cnt;
  }

  __shared__ double red[TPB / 32][KT + 1];
  __shared__ double vec[KMAX];
  __shared__ double scratch[TPB];
  __shared__ unsigned int is_last;
  block_partial<KT, TPB>(acc, bad, a.partials, red);
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) is_last = (atomicAdd(a.ticket, 1u) == gridDim.x - 1) ? 1u : 0u;
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  grid_combine<KS, TPB>(a.partials, gridDim.x, vec, scratch);
  if (threadIdx.x == 0) *a.ticket = 0u;  // ready for the next launch

  if (a.use_comm) {
    const unsigned long long epoch = (a.epilogue == EPI_FIT) ? (st->comm_epoch + 1) : (a.comm.epoch + 1);
    const bool ok = comm_combine<KS, TPB>(a.comm, epoch, vec);
    if (threadIdx.x == 0 && a.epilogue == EPI_FIT) st->comm_epoch = epoch;
    if (!ok) {
      if (threadIdx.x == 0 && a.epilogue != EPI_FIT && a.err) *a.err = -5;
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
    for (int k = threadIdx.x; k < KS; k += TPB) a.out[k] = vec[k];
    return;
  }
  // ---- fit epilogue: one warp runs the solver state machine on a shared-
  // memory copy of the state (no global-latency chains), then writes it back.
  if (threadIdx.x < 32) {
    __shared__ SolverSmem S;
    __shared__ FitState sst;
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    constexpr int NW = sizeof(FitState) / 8;
    const unsigned long long* src = reinterpret_cast<const unsigned long long*>(st);
    unsigned long long* dst = reinterpret_cast<unsigned long long*>(&sst);
    for (int k = threadIdx.x; k < NW; k += 32) dst[k] = src[k];
    __syncwarp();
    fit_after_pass(&sst, S, vec, JAC);
    __syncwarp();
    unsigned long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    if (threadIdx.x == 0) sst.epi_ns += (t1 - t0);
    __syncwarp();
    unsigned long long* back = reinterpret_cast<unsigned long long*>(st);
    for (int k = threadIdx.x; k < NW; k += 32) back[k] = dst[k];
    __syncwarp();
    if (threadIdx.x == 0 && use_cond) cudaGraphSetConditional(cond, sst.cont ? 1u : 0u);
  }
}

}  // namespace jf
