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

#include <cstdio>

#include "jf_common.cuh"
#include "jf_dual.cuh"
#include "jf_models.cuh"
#include "jf_solver.cuh"
#include "jf_state.cuh"

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

// A contiguous range [RL, RH) of rows j of the W^T W upper triangle (slots
// (j, k), j <= k <= n).  The n = 13 J-pass splits the triangle in two parts
// computed by the two halves of the grid, so each thread holds ~half the
// 105 accumulators (the model is evaluated by both halves).
__host__ __device__ constexpr int part_count(int n, int rl, int rh) {
  return rl >= rh ? 0 : (n + 1 - rl) + part_count(n, rl + 1, rh);
}
template <class Model, bool JAC, int RL, int RH>
struct Part {
  static constexpr int K = JAC ? part_count(Model::N, RL, RH) : 1;
};

// Accumulate one point's contribution to the part's slots.  CONST_COL: a
// parameter whose partial is identically 1 (the offset); unweighted, its
// diagonal slot is the point count, kept as an integer (cnt).  The non-finite
// count is kept by the part that starts at row 0.
//
// Rotated Gaussians (Model::NT > 0): the dual numbers give the row in the
// alternative coordinates (a, 2b, c2) of each quadratic form; the chain-rule
// block T (R33) maps it to (sx, sy, th) here, per point, before the rank-1
// update (chain = true; false: the alt-coordinate Gram, JF_FLAG_ALT_COORDS).
// Per point, not on the reduced Gram: for an elongated peak the alt columns
// -A u (dx^2, dx dy, dy^2) are nearly dependent and T^T (W_alt^T W_alt) T
// would cancel catastrophically.
template <class Model, bool JAC, int RL, int RH, bool PREC = false, class H, class Pre>
__device__ __forceinline__ void accumulate(double (&acc)[Part<Model, JAC, RL, RH>::K], int& bad, int& cnt,
                                           const H& h, double z, double wsig, bool weighted,
                                           const double* __restrict__ prec, const Pre& pre, bool chain) {
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
    if constexpr (RL == 0) bad += isfinite(w[N]) ? 0 : 1;
    ++cnt;
    if constexpr (!PREC && Model::NT > 0) {
      if (chain) {
#pragma unroll
        for (int g = 0; g < Model::NT; ++g) {
          const int b = Model::tbase(g);
          const double* T = Model::tblock(pre, g);
          const double u0 = w[b], u1 = w[b + 1], u2 = w[b + 2];
#pragma unroll
          for (int q = 0; q < 3; ++q) w[b + q] = fma(u0, T[q], fma(u1, T[3 + q], u2 * T[6 + q]));
        }
      }
    }
    if constexpr (PREC) {
      // TSQR (CholeskyQR2) second pass: the row of W P, P = R1^-1 upper
      // triangular ((n+1) x (n+1), shared memory), so the accumulated Gram is
      // P^T (W^T W) P and its Cholesky factor R2 gives R = R2 R1.  The row is
      // first mapped to the paper's parameters by the chain-rule blocks T
      // (jf_models.cuh PreGauss2D), stored after P.
#pragma unroll
      for (int g = 0; g < Model::NT; ++g) {
        constexpr int N1 = N + 1;
        const int b = Model::tbase(g);
        const double* T = prec + N1 * N1 + 9 * g;
        const double u0 = w[b], u1 = w[b + 1], u2 = w[b + 2];
#pragma unroll
        for (int q = 0; q < 3; ++q) w[b + q] = fma(u0, T[q], fma(u1, T[3 + q], u2 * T[6 + q]));
      }
      double u[N + 1];
#pragma unroll
      for (int k = 0; k <= N; ++k) {
        double t = 0.0;
#pragma unroll
        for (int j = 0; j <= k; ++j) t = fma(w[j], prec[j * (N + 1) + k], t);
        u[k] = t;
      }
#pragma unroll
      for (int k = 0; k <= N; ++k) w[k] = u[k];
    }
    int s = 0;
#pragma unroll
    for (int j = RL; j < RH; ++j) {
#pragma unroll
      for (int k = j; k <= N; ++k) {
        if (j == CC && k == CC && !PREC) {
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

// Block-level combine of one part's per-thread accumulators into the block's
// full partial K-vector (slots outside the part are zero).
template <class Model, bool JAC, int RL, int RH, int TPB>
__device__ __forceinline__ void block_partial_part(double (&acc)[Part<Model, JAC, RL, RH>::K], int bad,
                                                   double* __restrict__ part,
                                                   double (*red)[PassShape<Model, JAC>::KT + 1]) {
  constexpr int N = Model::N;
  constexpr int KT = PassShape<Model, JAC>::KT;
  constexpr int NW = TPB / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int k = lane; k < KT + 1; k += 32) red[warp][k] = 0.0;
  __syncwarp();
  if constexpr (JAC) {
    int s = 0;
#pragma unroll
    for (int j = RL; j < RH; ++j) {
#pragma unroll
      for (int k = j; k <= N; ++k) {
        double v = acc[s];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
        if (lane == 0) red[warp][tri_slot(N, j, k)] = v;
        ++s;
      }
    }
  } else {
    double v = acc[0];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    if (lane == 0) red[warp][0] = v;
  }
  const int b = __reduce_add_sync(FULL, bad);
  if (lane == 0) red[warp][KT] = (double)b;
  __syncthreads();
  for (int k = threadIdx.x; k < KT + 1; k += TPB) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < NW; ++w) s += red[w][k];
    part[k] = s;  // the caller passes this block's row
  }
}

// Map the reduced W_alt^T W_alt (columns (a, 2b, c2) of each Gaussian) to the
// paper's parameters: T^T M T with the 3x3 chain-rule blocks of the model
// (jf_models.cuh PreGauss2D).  Once per pass on the K-vector, one slot per
// thread:  M'[j][k] = sum_{r in S(j), r' in S(k)} T(r, j) T(r', k) M[r][r'],
// S(j) = {j} for a column outside every block, else the block's 3 columns.
template <class Model>
__device__ __forceinline__ int chain_block(int j) {
#pragma unroll
  for (int g = 0; g < Model::NT; ++g)
    if (j >= Model::tbase(g) && j < Model::tbase(g) + 3) return g;
  return -1;
}
template <class Model, int TPB, class Pre>
__device__ __forceinline__ void apply_chain_kvec(const Pre& pre, double* vec, double* tmp /* KT doubles */) {
  constexpr int N = Model::N, N1 = N + 1, KT = tri_count(N);
  for (int t = threadIdx.x; t < KT; t += TPB) {
    int j = 0, rem = t;
    while (rem >= N1 - j) {
      rem -= N1 - j;
      ++j;
    }
    const int k = j + rem;
    const int gj = chain_block<Model>(j), gk = chain_block<Model>(k);
    const int nj = gj < 0 ? 1 : 3, nk = gk < 0 ? 1 : 3;
    const int bj = gj < 0 ? j : Model::tbase(gj), bk = gk < 0 ? k : Model::tbase(gk);
    const double* Tj = gj < 0 ? nullptr : Model::tblock(pre, gj);
    const double* Tk = gk < 0 ? nullptr : Model::tblock(pre, gk);
    double s = 0.0;
    for (int r = 0; r < nj; ++r) {
      const double cj = gj < 0 ? 1.0 : Tj[3 * r + (j - bj)];
      double u = 0.0;
      for (int q = 0; q < nk; ++q) {
        const double ck = gk < 0 ? 1.0 : Tk[3 * q + (k - bk)];
        const int x = bj + r, y = bk + q;
        u = fma(ck, vec[x <= y ? tri_slot(N, x, y) : tri_slot(N, y, x)], u);
      }
      s = fma(cj, u, s);
    }
    tmp[t] = s;
  }
  __syncthreads();
  for (int t = threadIdx.x; t < KT; t += TPB) vec[t] = tmp[t];
  __syncthreads();
}

__host__ __device__ constexpr int combine_scratch(int tpb) { return tpb; }

// Two-level deterministic grid reduction of the per-block partials
// (partials[b][0..KS), written by every block before calling).  Blocks form
// groups of GROUP consecutive indices; the last block of a group to finish
// (atomic ticket) sums the group's rows in block order into a group row
// (stored after the nblk block rows); the last group to finish sums the group
// rows in group order into out[0..KS) and returns true — exactly one block of
// the grid gets true.  Every sum has a fixed order (bitwise reproducible) and
// at most two L2 round trips sit on the critical path after the last block
// arrives (one for its group, one for the group rows).
// Tickets: a.ticket[0] (groups), a.ticket[1 + g] (blocks of group g); each
// is reset by its last user, ready for the next launch.
constexpr int GROUP = 16;
// Development builds only (JF_DEV=1 python -m paper_2208_12187_b200.build):
// timestamps of the last block's tail phases for tools/stamps2.py.
#ifndef JF_DEV
#define JF_DEV 0
#endif
__device__ __forceinline__ void dbg_tail(const PassArgs& a, int i) {
#if JF_DEV
  if (a.dbg && threadIdx.x == 0) {
    a.dbg[4 * 16384 - 16 + i] = clock64();  // SM cycles (all tail stamps are on the last block's SM)
  }
#else
  (void)a;
  (void)i;
#endif
}
template <int KS, int TPB>
__device__ __forceinline__ bool grid_reduce(const PassArgs& a, double* out, double* scratch /* TPB doubles */) {
  __shared__ unsigned int flag;
  const int t = threadIdx.x;
  const int nblk = gridDim.x;
  const int ngrp = (nblk + GROUP - 1) / GROUP;
  const int g = blockIdx.x / GROUP;
  const int b0 = g * GROUP, nb = min(GROUP, nblk - b0);
  const double* part = a.partials;
  double* grp = a.partials + (size_t)nblk * KS;
  __threadfence();
  __syncthreads();
  if (t == 0) flag = (atomicAdd(a.ticket + 1 + g, 1u) == (unsigned)(nb - 1)) ? 1u : 0u;
  __syncthreads();
  if (!flag) return false;
  dbg_tail(a, 1);
  __threadfence();
  for (int k = t; k < KS; k += TPB) {
    double v[GROUP];
#pragma unroll
    for (int i = 0; i < GROUP; ++i) v[i] = (i < nb) ? __ldcg(part + (size_t)(b0 + i) * KS + k) : 0.0;
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < GROUP; ++i) s += v[i];
    grp[(size_t)g * KS + k] = s;
  }
  if (t == 0) a.ticket[1 + g] = 0u;
  __threadfence();
  __syncthreads();
  if (t == 0) flag = (atomicAdd(a.ticket, 1u) == (unsigned)(ngrp - 1)) ? 1u : 0u;
  __syncthreads();
  if (!flag) return false;
  dbg_tail(a, 2);
  __threadfence();
  // group rows: NSEG segments per column, each up to 16 rows in one batch
  constexpr int NSEG = (TPB / KS) > 0 ? (TPB / KS) : 1;
  if (t < NSEG * KS) {
    const int k = t % KS, seg = t / KS;
    double s = 0.0;
    for (int r0 = seg; r0 < ngrp; r0 += 16 * NSEG) {
      double v[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int r = r0 + i * NSEG;
        v[i] = (r < ngrp) ? __ldcg(grp + (size_t)r * KS + k) : 0.0;
      }
#pragma unroll
      for (int i = 0; i < 16; ++i) s += v[i];
    }
    if (t == 0) dbg_tail(a, 10);
    scratch[seg * KS + k] = s;
  }
  if (t == 0) a.ticket[0] = 0u;
  __syncthreads();
  for (int k = t; k < KS; k += TPB) {
    double s = 0.0;
#pragma unroll
    for (int seg = 0; seg < NSEG; ++seg) s += scratch[seg * KS + k];
    out[k] = s;
  }
  __syncthreads();
  return true;
}

// Single-level variant for small grids (one block per SM): the last block
// sums all gridDim.x partials, NSEG interleaved segments per entry in
// parallel, then the segments in order (fixed order: bitwise reproducible).
template <int KS, int TPB>
__device__ __forceinline__ bool grid_reduce1(const PassArgs& a, double* out, double* scratch /* TPB doubles */) {
  __shared__ unsigned int flag;
  const int t = threadIdx.x;
  const int nblk = gridDim.x;
  // the block's partial (written by threads < KS) is released by thread 0
  // after the barrier (release is cumulative); the last block acquires
  __syncthreads();
  if (t == 0) {
    unsigned prev;
    asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(prev) : "l"(a.ticket) : "memory");
    flag = (prev == (unsigned)(nblk - 1)) ? 1u : 0u;
  }
  __syncthreads();
  if (!flag) return false;
  dbg_tail(a, 1);
  constexpr int NSEG = (TPB / KS) > 0 ? (TPB / KS) : 1;
  const double* part = a.partials;  // read once (each L2 load below would otherwise re-read the field)
  if (t < NSEG * KS) {
    const int k = t % KS, seg = t / KS;
    double s = 0.0;
    for (int r0 = seg; r0 < nblk; r0 += 16 * NSEG) {  // one batch of loads for nblk <= 16 NSEG
      double v[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int r = r0 + i * NSEG;
        v[i] = (r < nblk) ? __ldcg(part + (size_t)r * KS + k) : 0.0;
      }
#pragma unroll
      for (int i = 0; i < 16; ++i) s += v[i];
    }
    if (t == 0) dbg_tail(a, 10);
    scratch[seg * KS + k] = s;
  }
  if (t == 0) a.ticket[0] = 0u;
  __syncthreads();
  for (int k = t; k < KS; k += TPB) {
    double s = 0.0;
#pragma unroll
    for (int seg = 0; seg < NSEG; ++seg) s += scratch[seg * KS + k];
    out[k] = s;
  }
  __syncthreads();
  dbg_tail(a, 2);
  return true;
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
      if (t1 - t0 > cm.timeout_ns) {  // a peer is gone (jf_comm_set_timeout)
        timed_out = 1;
        break;
      }
    }
  }
  __threadfence_system();
  __syncthreads();
#if JF_DEV
  if (timed_out && threadIdx.x == 0) {
    printf("comm timeout: rank %d epoch %llu flags:", me, epoch);
    for (int p = 0; p < R; ++p) printf(" %llu", *(volatile unsigned long long*)(cm.mbox_flag[me] + p));
    printf("\n");
  }
#endif
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

// Implicit-grid pass with the row recurrence for exp (models with NEXP > 0).
//
// Work unit: a warp-chunk of 32 L consecutive pixels of one image row; lane l
// owns pixels col0 + l + 32 k, k < L, so every load instruction of the warp
// reads 32 consecutive doubles.  Along such a run the exponent of each
// Gaussian factor is quadratic in k:  q(k+1) - q(k) = D (2a dx_k + 2b dy) + a D^2
// with D = 32, so  E_{k+1} = E_k R_k,  R_{k+1} = R_k rho,  rho = exp(-2 a D^2):
// two multiplications per point instead of an fp64 exp (two exps per chunk
// start).  Relative error grows by a few ulp per step (<= ~4e-15 at L = 8).
// A lane whose chunk start is outside a safe exponent range (|q| > 600 or a
// step factor beyond e^300) evaluates exp directly for that chunk.
template <class Model, bool JAC, bool WGT, int L, int TPB, int RL, int RH, bool PREC>
__device__ __forceinline__ void grid_recur_loop(const PassArgs& a, const auto& pre,
                                                double (&acc)[Part<Model, JAC, RL, RH>::K], int& bad, int& cnt,
                                                int blk, int nblk, const double* prec) {
  constexpr int NE = Model::NEXP;
  constexpr int CW = 32 * L;
  constexpr double D = 32.0;
  const int lane = threadIdx.x & 31;
  const int W = (int)a.W;
  const int64_t H = a.m / a.W;
  const int cpr = (W + CW - 1) / CW;
  const int64_t nch = H * (int64_t)cpr;
  const int64_t nw = (int64_t)nblk * (TPB / 32);
  int64_t ch = (int64_t)blk * (TPB / 32) + (threadIdx.x >> 5);
  const double* __restrict__ z = a.z;
  const double* __restrict__ ws = a.wsig;
  double ra[NE], rb2[NE], rx0[NE], ry0[NE], rho[NE];
#pragma unroll
  for (int g = 0; g < NE; ++g) {
    if (g == 0) Model::template rec_coeffs<0>(pre, ra[g], rb2[g], rx0[g], ry0[g]);
    if constexpr (NE > 1) {
      if (g == 1) Model::template rec_coeffs<1>(pre, ra[g], rb2[g], rx0[g], ry0[g]);
    }
    rho[g] = exp(-2.0 * ra[g] * D * D);
  }
  double zn[L], wn[L];
  auto load = [&](int64_t c) {
    if (c < nch) {
      const int64_t row = c / cpr;
      const int col = (int)(c - row * cpr) * CW + lane;
      const double* zp = z + row * a.W + col;
#pragma unroll
      for (int k = 0; k < L; ++k) {
        const bool v = col + 32 * k < W;
        JF_DCHECK(!v || row * a.W + col + 32 * k < a.m);
        zn[k] = v ? __ldcs(zp + 32 * k) : 0.0;
        if constexpr (WGT) wn[k] = v ? __ldcs(ws + row * a.W + col + 32 * k) : 0.0;
      }
    }
  };
  load(ch);
  for (; ch < nch; ch += nw) {
    double zc[L], wc[L];
#pragma unroll
    for (int k = 0; k < L; ++k) {
      zc[k] = zn[k];
      if constexpr (WGT) wc[k] = wn[k];
    }
    load(ch + nw);  // prefetch the next chunk
    const int64_t row = ch / cpr;
    const int col0 = (int)(ch - row * cpr) * CW + lane;
    const double Y = (double)(row + a.row0);
    const double X0 = (double)col0;
    double E[NE], R[NE];
    bool ok = true;
#pragma unroll
    for (int g = 0; g < NE; ++g) {
      double q0;
      if (g == 0) q0 = Model::template qval<0>(pre, X0, Y);
      if constexpr (NE > 1) {
        if (g == 1) q0 = Model::template qval<1>(pre, X0, Y);
      }
      const double argR = D * (2.0 * ra[g] * (X0 - rx0[g]) + rb2[g] * (Y - ry0[g])) + ra[g] * D * D;
      ok = ok && fabs(q0) < 600.0 && fabs(argR) < 300.0 && 2.0 * ra[g] * D * D * L < 300.0;
      E[g] = exp(-q0);
      R[g] = exp(-argR);
    }
    const bool full = (int)(ch - row * cpr) * CW + CW <= W;  // warp-uniform
    if (full && __all_sync(FULL, ok)) {
#pragma unroll
      for (int k = 0; k < L; ++k) {
        const double X = X0 + 32.0 * k;
        const auto h = Model::template point_e<JAC>(pre, X, Y, E);
        accumulate<Model, JAC, RL, RH, PREC>(acc, bad, cnt, h, zc[k], WGT ? wc[k] : 1.0, WGT, prec, pre, !a.no_chain);
#pragma unroll
        for (int g = 0; g < NE; ++g) {
          E[g] *= R[g];
          R[g] *= rho[g];
        }
      }
    } else {
      // ragged row end or unsafe exponent range: direct evaluation
#pragma unroll
      for (int k = 0; k < L; ++k) {
        if (col0 + 32 * k < W) {
          const double X = X0 + 32.0 * k;
          const auto h = Model::template point<JAC>(pre, X, Y);
          accumulate<Model, JAC, RL, RH, PREC>(acc, bad, cnt, h, zc[k], WGT ? wc[k] : 1.0, WGT, prec, pre, !a.no_chain);
        }
      }
    }
  }
}

// Launch shape per (model, pass): points per thread per iteration (ILP) and
// minimum resident blocks per SM (register budget).
template <class Model, bool JAC>
struct PassCfg {
  static constexpr bool BIG = JAC && Model::N >= 7;
  static constexpr int P = JAC ? (Model::N == 7 ? 4 : 1) : (Model::N > 7 ? 2 : 4);
  static constexpr int TPB = 256;
  static constexpr int MINB = BIG ? 1 : 2;
  static constexpr int L = JAC ? (Model::N > 7 ? 2 : 8) : (Model::N > 7 ? 8 : 16);  // points per lane per warp-chunk (grid recurrence)
  static constexpr bool SPLIT = JAC && Model::N > 7;  // two-part triangle (see run_part)
};

// One part [RL, RH) of the triangle over all points, by blocks [blk of nblk]:
// the per-thread loop (grid recurrence or generic prefetching loop) and the
// block partial into a.partials[blockIdx.x].
template <class Model, bool JAC, int COORD, bool WGT, int P, int TPB, int RL, int RH, bool PREC, class Pre>
__device__ __forceinline__ void run_part(const PassArgs& a, const Pre& pre, int blk, int nblk,
                                         double (*red)[PassShape<Model, JAC>::KT + 1], double* part_out,
                                         const double* prec) {
  constexpr int KP = Part<Model, JAC, RL, RH>::K;
  double acc[KP];
#pragma unroll
  for (int k = 0; k < KP; ++k) acc[k] = 0.0;
  int bad = 0, cnt = 0;

  const int64_t m = a.m;
  const int64_t S = (int64_t)nblk * TPB;
  PointIter<COORD> it;
  it.init(a, (int64_t)blk * TPB + threadIdx.x, S);
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
      JF_DCHECK(!v || idx >= 0);
      qz[p] = v ? __ldcs(z + idx) : 0.0;
      qw[p] = (v && weighted) ? __ldcs(ws + idx) : 1.0;
      if constexpr (EXPL) {
        qa[p] = v ? __ldcs(y0 + idx) : 0.0;
        if constexpr (TWO) qb[p] = v ? __ldcs(y1 + idx) : 0.0;
      }
    }
  };
  if constexpr (COORD == COORD_GRID && Model::NEXP > 0) {
    grid_recur_loop<Model, JAC, WGT, PassCfg<Model, JAC>::L, TPB, RL, RH, PREC>(a, pre, acc, bad, cnt, blk, nblk, prec);
  } else {
  auto coords = [&](double& X, double& Y) {
    if constexpr (COORD == COORD_GRID) {
      X = (double)it.col;
      Y = (double)(it.row + (int32_t)a.row0);
    } else if constexpr (COORD == COORD_IMPLICIT_T) {
      X = fma((double)(a.index0 + it.i), a.dt, a.t0);
    }
  };
  auto eval = [&](double X, double Y, double zz, double ww) {
    if constexpr (TWO) {
      const auto h = Model::template point<JAC>(pre, X, Y);
      accumulate<Model, JAC, RL, RH, PREC>(acc, bad, cnt, h, zz, ww, weighted, prec, pre, !a.no_chain);
    } else {
      const auto h = Model::template point<JAC>(pre, X);
      accumulate<Model, JAC, RL, RH, PREC>(acc, bad, cnt, h, zz, ww, weighted, prec, pre, !a.no_chain);
    }
  };
  // main loop: full groups of P points, straight-line (no per-point predicate)
  const int64_t full_end = m - (int64_t)(P - 1) * S;
  issue(it.i);
  while (it.i < full_end) {
    double cz[P], cw[P], cx[P], cy[P];
#pragma unroll
    for (int p = 0; p < P; ++p) {
      cz[p] = qz[p];
      cw[p] = qw[p];
      if constexpr (EXPL) {
        cx[p] = qa[p];
        if constexpr (TWO) cy[p] = qb[p];
      } else {
        coords(cx[p], cy[p]);
      }
      it.advance();
    }
    issue(it.i);
#pragma unroll
    for (int p = 0; p < P; ++p) eval(cx[p], cy[p], cz[p], cw[p]);
  }
  // tail: fewer than P points left for this thread
  if constexpr (P > 1) {
#pragma unroll 1
    for (int p = 0; p < P - 1 && it.i < m; ++p) {
      double X = 0.0, Y = 0.0;
      if constexpr (EXPL) {
        X = qa[p];
        if constexpr (TWO) Y = qb[p];
      } else {
        coords(X, Y);
      }
      eval(X, Y, qz[p], qw[p]);
      it.advance();
    }
  }
  }
  if constexpr (JAC) {
    constexpr int CC = Model::CONST_COL;
    if constexpr (CC >= RL && CC < RH && !PREC) {
      if (!weighted) acc[tri_slot(Model::N, CC, CC) - tri_slot(Model::N, RL, RL)] = (double)cnt;
    }
  }
  block_partial_part<Model, JAC, RL, RH, TPB>(acc, bad, part_out, red);

}

// Common start of every pass kernel: inside a fit, count the launch, stamp
// the timeline, let the dependent solver kernel launch early (PDL; it waits
// for this grid in griddepcontrol.wait) and run only when the fit's phase
// wants this pass type.
template <bool JAC, bool PREC>
__device__ __forceinline__ bool pass_begin(const PassArgs& a, FitState* __restrict__ st) {
  if (a.epilogue != EPI_FIT) return true;
  // PDL: the solver kernel before this pass in the graph has finished and its
  // state is visible (a no-op without a programmatic dependency)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    atomicAdd(&st->kernels, 1);
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    const int k = atomicAdd(&st->tl_n, 1);
    if (k < 64) st->tl[k] = t;
  }
  const int ph = st->phase;
  return JAC ? (PREC ? (ph == PH_QR2) : (ph == PH_INIT_J || ph == PH_TRIAL_J || ph == PH_ACCEPT_J))
             : (ph == PH_TRIAL_R);
}

// Common end of every pass kernel's last block: the cross-rank combine
// (multi-GPU), then either the K-vector to a.out (plain pass) or the hand-off
// to the solver kernel (fit).  vec: the block's combined K-vector (smem).
template <int KS, int TPB, bool JAC>
__device__ __forceinline__ void pass_tail(const PassArgs& a, FitState* __restrict__ st, double* vec,
                                          cudaGraphConditionalHandle cond, int use_cond) {
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

  // ---- fit: hand the combined K-vector to the solver kernel (jf_solver.cu)
  for (int k = threadIdx.x; k < KS; k += TPB) a.out[k] = vec[k];
  if constexpr (JAC && (KS == tri_count(7) + 1 || KS == tri_count(13) + 1)) {
    if (a.fused) {  // the solver step here, by warp 0 (the kernel's dynamic shared memory as scratch)
      __syncthreads();
      if (threadIdx.x < 32) fused_solver_step<(KS == tri_count(7) + 1) ? 7 : 13>(st, vec, cond, use_cond);
      return;
    }
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    st->pass_ready = JAC ? 1 : 2;
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    const int k = atomicAdd(&st->tl_n, 1);
    if (k < 64) st->tl[k] = t;
  }
}

// The body of a pass (everything after pass_begin).  PREC: the TSQR
// (CholeskyQR2) second pass, rows of W multiplied by P = R1^-1.
template <class Model, bool JAC, int COORD, bool WGT, int P, int TPB, bool PREC>
__device__ __forceinline__ void pass_body(const PassArgs& a, FitState* __restrict__ st,
                                          cudaGraphConditionalHandle cond, int use_cond) {
  using Sh = PassShape<Model, JAC>;
  constexpr int KT = Sh::KT, KS = Sh::KS;
  const double* xs = (a.epilogue == EPI_FIT) ? st->x_eval : a.x;
  double xv[Model::N];
#pragma unroll
  for (int j = 0; j < Model::N; ++j) xv[j] = xs[j];
  const auto pre = Model::template prologue<JAC>(xv);

  // TSQR second pass: the preconditioner P = R1^-1 into shared memory
  __shared__ double prec_s[PREC ? (Model::N + 1) * (Model::N + 1) + 9 * Model::NT + 1 : 1];
  const double* prec = nullptr;
  if constexpr (PREC) {
    constexpr int N1 = Model::N + 1;
    const double* src = (a.epilogue == EPI_FIT) ? st->prec : a.precond;
    for (int k = threadIdx.x; k < N1 * N1; k += TPB) prec_s[k] = __ldcg(src + k);
    if (threadIdx.x == 0) {
      for (int g = 0; g < Model::NT; ++g)
        for (int q = 0; q < 9; ++q) prec_s[N1 * N1 + 9 * g + q] = Model::tblock(pre, g)[q];
    }
    __syncthreads();
    prec = prec_s;
  }

  __shared__ double red[TPB / 32][KT + 1];
  __shared__ double vec[KMAX];
  __shared__ double scratch[combine_scratch(TPB)];
  constexpr int NP1 = Model::N + 1;
  if constexpr (JAC && Model::N > 7) {
    // split triangle: rows [0, 4) by the first half of the grid, [4, n+1) by the second
    const int half = gridDim.x / 2;
    if ((int)blockIdx.x < half) {
      run_part<Model, JAC, COORD, WGT, P, TPB, 0, 4, PREC>(a, pre, blockIdx.x, half, red, a.partials + (size_t)blockIdx.x * KS, prec);
    } else {
      run_part<Model, JAC, COORD, WGT, P, TPB, 4, NP1, PREC>(a, pre, blockIdx.x - half, gridDim.x - half, red,
                                                            a.partials + (size_t)blockIdx.x * KS, prec);
    }
  } else {
    run_part<Model, JAC, COORD, WGT, P, TPB, 0, (JAC ? NP1 : 1), PREC>(a, pre, blockIdx.x, gridDim.x, red,
                                                                       a.partials + (size_t)blockIdx.x * KS, prec);
  }
  if (!grid_reduce<KS, TPB>(a, vec, scratch)) return;

  pass_tail<KS, TPB, JAC>(a, st, vec, cond, use_cond);
}

// The same body out of line: a fallback inside another kernel (the moment
// kernels) keeps its registers out of the caller's hot loop.
template <class Model, bool JAC, int COORD, bool WGT, int P, int TPB, bool PREC>
__device__ __noinline__ void pass_body_ool(const PassArgs& a, FitState* __restrict__ st,
                                           cudaGraphConditionalHandle cond, int use_cond) {
  pass_body<Model, JAC, COORD, WGT, P, TPB, PREC>(a, st, cond, use_cond);
}

// In a fit, a J-pass kernel also serves the TSQR second pass (phase PH_QR2):
// the graph needs no separate node (and no empty launch per trial) for it.
template <class Model, int COORD, bool WGT, int TPB>
__device__ __forceinline__ bool qr2_dispatch(const PassArgs& a, FitState* __restrict__ st,
                                             cudaGraphConditionalHandle cond, int use_cond) {
  if (a.epilogue != EPI_FIT || st->phase != PH_QR2) return false;
  pass_body_ool<Model, true, COORD, WGT, PassCfg<Model, true>::P, TPB, true>(a, st, cond, use_cond);
  return true;
}

// The pass kernel.  epilogue == EPI_FIT: one pass of a fit (st is the state).
template <class Model, bool JAC, int COORD, bool WGT, int P = PassCfg<Model, JAC>::P,
          int TPB = PassCfg<Model, JAC>::TPB, int MINB = PassCfg<Model, JAC>::MINB, bool PREC = false>
__global__ void __launch_bounds__(TPB, MINB)
    pass_kernel(const PassArgs* __restrict__ pa, FitState* __restrict__ st, cudaGraphConditionalHandle cond,
                int use_cond, const PassArgs av) {
  // the arguments (fits: device-resident, graph replay; else by value) into
  // shared memory once: a reference that may name either the kernel's
  // parameters or global memory makes every field access a generic load
  __shared__ __align__(16) PassArgs sargs;
  {
    constexpr int NA = sizeof(PassArgs) / 8;
    static_assert(sizeof(PassArgs) % 8 == 0 && NA <= TPB, "PassArgs copy");
    if ((int)threadIdx.x < NA)
      reinterpret_cast<unsigned long long*>(&sargs)[threadIdx.x] =
          pa ? __ldg(reinterpret_cast<const unsigned long long*>(pa) + threadIdx.x)
             : reinterpret_cast<const unsigned long long*>(&av)[threadIdx.x];
    __syncthreads();
  }
  const PassArgs& a = sargs;
  if (!pass_begin<JAC, PREC>(a, st)) {
    if constexpr (JAC && !PREC) qr2_dispatch<Model, COORD, WGT, TPB>(a, st, cond, use_cond);
    return;
  }
  pass_body<Model, JAC, COORD, WGT, P, TPB, PREC>(a, st, cond, use_cond);
}

// ---------------------------------------------------------------- small m
// The whole fit in ONE single-block kernel, for small m (the regime where
// launch latency, not the data pass, dominates; Gpufit "runs
// entirely in CUDA" and wins below v = 3e4).  The state lives in shared
// memory for the whole fit; every iteration: the block's J-pass over all m
// points (the same run_part as the grid kernels, one block) -> warp 0 runs
// the solver step -> barrier.  Speculative policy (a J-pass per trial).
template <class Model, int COORD, bool WGT>
__global__ void __launch_bounds__(256, 1) fit_small_kernel(const PassArgs* __restrict__ pa, FitState* __restrict__ gst) {
  constexpr int TPB = 256;
  constexpr int KT = PassShape<Model, true>::KT;
  constexpr int NP1 = Model::N + 1;
  constexpr int P = (Model::N <= 4) ? 2 : 1;
  __shared__ FitState st;
  __shared__ SolverSmem S;
  __shared__ double red[TPB / 32][KT + 1];
  __shared__ double kvec[KT + 1];
  __shared__ double prec_s[NP1 * NP1 + 9 * Model::NT + 1];  // TSQR second pass: P = R1^-1 and the chain blocks
  const PassArgs& a = *pa;
  {
    constexpr int NW = sizeof(FitState) / 8;
    const unsigned long long* src = reinterpret_cast<const unsigned long long*>(gst);
    unsigned long long* dst = reinterpret_cast<unsigned long long*>(&st);
    for (int k = threadIdx.x; k < NW; k += TPB) dst[k] = src[k];
  }
  __syncthreads();
  if (threadIdx.x == 0) st.kernels = st.kernels + 1;
  for (int iter = 0; iter < 4 * st.max_nfev + 8; ++iter) {
    __syncthreads();
    if (!st.cont) break;
    double xv[Model::N];
#pragma unroll
    for (int j = 0; j < Model::N; ++j) xv[j] = st.x_eval[j];
    const auto pre = Model::template prologue<true>(xv);
    if (st.phase == PH_QR2) {  // TSQR (CholeskyQR2): the preconditioned pass at x (solver AUTO / TSQR)
      for (int k = threadIdx.x; k < NP1 * NP1; k += TPB) prec_s[k] = __ldcg(st.prec + k);  // written by lane 0 this launch
      if (threadIdx.x == 0) {
        for (int g = 0; g < Model::NT; ++g)
          for (int q = 0; q < 9; ++q) prec_s[NP1 * NP1 + 9 * g + q] = Model::tblock(pre, g)[q];
      }
      __syncthreads();
      run_part<Model, true, COORD, WGT, P, TPB, 0, NP1, true>(a, pre, 0, 1, red, kvec, prec_s);
      __syncthreads();
    } else {
      run_part<Model, true, COORD, WGT, P, TPB, 0, NP1, false>(a, pre, 0, 1, red, kvec, nullptr);
      __syncthreads();
    }
    if (threadIdx.x < 32) solver_step<Model::N>(&st, S, kvec, true);
  }
  __syncthreads();
  {
    constexpr int NW = sizeof(FitState) / 8;
    const unsigned long long* src = reinterpret_cast<const unsigned long long*>(&st);
    unsigned long long* dst = reinterpret_cast<unsigned long long*>(gst);
    for (int k = threadIdx.x; k < NW; k += TPB) dst[k] = src[k];
  }
}

// ------------------------------------------------------ batched small fits
// Many independent fits in ONE launch (Gpufit's regime, P:260/P:267 — "runs
// entirely in CUDA"): each block is one warp and runs whole fits, one after
// another (block b: fits b, b + grid, ...), with the fit state and the
// subproblem workspace in shared memory.  Per fit: the initial point
// (caller's p0 or curve_fit's default, strictly feasible when bounded), then
// [J-pass over the fit's m points by the warp -> solver step] until the state
// machine ends the fit; the result is written per fit.  The same pass body
// (run_part) and solver step (solver_step) as every other path.
template <class Model, int COORD, bool WGT>
__global__ void __launch_bounds__(32, 8) fit_batch_kernel(const BatchArgs ba) {
  constexpr int TPB = 32;
  constexpr int N = Model::N;
  constexpr int KT = PassShape<Model, true>::KT;
  constexpr int NP1 = N + 1;
  constexpr int P = (N <= 4) ? 2 : 1;
  __shared__ FitState st;
  __shared__ SolverSmem S;
  __shared__ PassArgs a;
  __shared__ double red[1][KT + 1];
  __shared__ double kvec[KT + 1];
  __shared__ double prec_s[NP1 * NP1 + 9 * Model::NT + 1];
  __shared__ int skip;
  const int lane = threadIdx.x;
  const int64_t nfits = ba.nfits;
  for (int64_t f = blockIdx.x; f < nfits; f += gridDim.x) {
    {  // the shared configuration, then this fit's initial point and data
      constexpr int NW = sizeof(FitState) / 8;
      const unsigned long long* src = reinterpret_cast<const unsigned long long*>(ba.tmpl);
      unsigned long long* dst = reinterpret_cast<unsigned long long*>(&st);
      for (int k = lane; k < NW; k += TPB) dst[k] = __ldg(src + k);
    }
    __syncwarp();
    if (lane == 0) {
      a = ba.base;
      a.z = ba.base.z + f * ba.z_stride;
      if (ba.base.wsig) a.wsig = ba.base.wsig + f * ba.z_stride;
      if (ba.base.y0) a.y0 = ba.base.y0 + f * ba.y_stride;
      if (ba.base.y1) a.y1 = ba.base.y1 + f * ba.y_stride;
      int bad = 0;
      for (int j = 0; j < N; ++j) {
        const double lo = st.lb[j], hi = st.ub[j];
        double x0;
        if (ba.p0) {
          x0 = ba.p0[f * N + j];
        } else {  // curve_fit's default initial guess
          const bool lf = isfinite(lo), uf = isfinite(hi);
          x0 = (lf && uf) ? 0.5 * (lo + hi) : (lf ? lo + 1.0 : (uf ? hi - 1.0 : 1.0));
        }
        if (!isfinite(x0)) bad = -1;
        else if (x0 < lo || x0 > hi) bad = bad ? bad : -2;  // R18: p0 outside the bounds
        if (st.bounded) x0 = strict_feasible_r(x0, lo, hi, 1e-10);
        st.x[j] = x0;
        st.x_eval[j] = x0;
      }
      st.qr = ba.qr + blockIdx.x;
      st.prec = st.qr->prec;
      skip = bad;
    }
    __syncwarp();
    if (skip) {
      if (lane == 0) {
        BatchResult& o = ba.out[f];
        for (int j = 0; j < NMAX; ++j) o.x[j] = j < N ? st.x[j] : 0.0;
        o.cost = o.optimality = 0.0;
        o.status = skip;
        o.nfev = o.njev = o.nit = 0;
      }
      __syncwarp();
      continue;
    }
    for (int iter = 0; iter < 4 * st.max_nfev + 8 && st.cont; ++iter) {
      double xv[N];
#pragma unroll
      for (int j = 0; j < N; ++j) xv[j] = st.x_eval[j];
      const auto pre = Model::template prologue<true>(xv);
      if (st.phase == PH_QR2) {  // TSQR (CholeskyQR2) second pass (solver AUTO / TSQR)
        for (int k = lane; k < NP1 * NP1; k += TPB) prec_s[k] = __ldcg(st.prec + k);
        if (lane == 0) {
          for (int g = 0; g < Model::NT; ++g)
            for (int q = 0; q < 9; ++q) prec_s[NP1 * NP1 + 9 * g + q] = Model::tblock(pre, g)[q];
        }
        __syncwarp();
        run_part<Model, true, COORD, WGT, P, TPB, 0, NP1, true>(a, pre, 0, 1, red, kvec, prec_s);
        __syncwarp();
      } else {
        run_part<Model, true, COORD, WGT, P, TPB, 0, NP1, false>(a, pre, 0, 1, red, kvec, nullptr);
        __syncwarp();
      }
      solver_step<N>(&st, S, kvec, true);
      __syncwarp();
    }
    if (lane == 0) {
      BatchResult& o = ba.out[f];
      for (int j = 0; j < NMAX; ++j) o.x[j] = j < N ? st.x[j] : 0.0;
      o.cost = st.cost;
      o.optimality = st.gnorm;
      o.status = st.error ? st.error : (st.cont ? -4 : st.status);
      o.nfev = st.nfev;
      o.njev = st.njev;
      o.nit = st.nit;
    }
    __syncwarp();
  }
}

}  // namespace jf
