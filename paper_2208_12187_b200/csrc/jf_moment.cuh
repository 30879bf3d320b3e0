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

// The alt-coordinate K-vector slot (x, y), x <= y <= 7, as <= 4 terms
// coef * mom[idx] (idx == NV stands for the point count m), the same
// formulas as moments_to_kvec.
__device__ __forceinline__ int kalt_terms(const PreGauss2D& g, int x, int y, int* idx, double* c) {
  if (y <= 5) {
    if (y == 0) {
      idx[0] = MomLayout::O2 + mono(4, 0, 0);
      c[0] = 1.0;
      return 1;
    }
    const Poly2 a = psi(g, x), b = psi(g, y);
    const double f = (x == 0 ? 1.0 : g.A) * g.A;
    int n = 0;
    for (int s = 0; s < 2; ++s)
      for (int u = 0; u < 2; ++u) {
        idx[n] = MomLayout::O2 + mono(4, a.p[s] + b.p[u], a.q[s] + b.q[u]);
        c[n++] = a.c[s] * b.c[u] * f;
      }
    return n;
  }
  if (x <= 5) {
    const int base = (y == 6) ? MomLayout::O1 : MomLayout::OR;
    const Poly2 a = psi(g, x);
    const double f = (x == 0 ? 1.0 : g.A);
    for (int s = 0; s < 2; ++s) {
      idx[s] = base + mono(2, a.p[s], a.q[s]);
      c[s] = a.c[s] * f;
    }
    return 2;
  }
  idx[0] = (x == 6) ? (y == 6 ? MomLayout::NV : MomLayout::OSR) : MomLayout::OSRR;
  c[0] = 1.0;
  return 1;
}

// The whole finish map as one matrix: K-vector slot t (paper coordinates,
// after the chain rule) = sum_i C[t][i] mom[i], i < NV, + C[t][NV] * m.
// Built by one warp from the pass's parameters (R33, R34): the same linear
// algebra as moments_to_kvec followed by apply_chain_kvec, composed once.
constexpr int FMAP_COLS = MomLayout::NV + 1;
template <class Pre>
__device__ __forceinline__ void build_finish_map(const Pre& pre, double (*C)[FMAP_COLS], int t0, int nthr) {
  using Model = ModelGauss2DRot;
  constexpr int N = Model::N, N1 = N + 1, KT = tri_count(N);
  for (int t = t0; t < KT; t += nthr) {
    for (int i = 0; i < FMAP_COLS; ++i) C[t][i] = 0.0;
    int j = 0, rem = t;
    while (rem >= N1 - j) {
      rem -= N1 - j;
      ++j;
    }
    const int k = j + rem;
    const int gj = chain_block<Model>(j), gk = chain_block<Model>(k);
    const int nj = gj < 0 ? 1 : 3, nk = gk < 0 ? 1 : 3;
    const int bj = gj < 0 ? j : Model::tbase(gj), bk = gk < 0 ? k : Model::tbase(gk);
    for (int r = 0; r < nj; ++r) {
      const double cj = gj < 0 ? 1.0 : pre.g.T[3 * r + (j - bj)];
      for (int q = 0; q < nk; ++q) {
        const double ck = gk < 0 ? 1.0 : pre.g.T[3 * q + (k - bk)];
        const int x = bj + r, y = bk + q;
        int idx[4];
        double c[4];
        const int n = kalt_terms(pre.g, x <= y ? x : y, x <= y ? y : x, idx, c);
        for (int u = 0; u < n; ++u) C[t][idx[u]] = fma(cj * ck, c[u], C[t][idx[u]]);
      }
    }
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
  dbg_tail(a, 3);
  double xv[N];
#pragma unroll
  for (int j = 0; j < N; ++j) xv[j] = xs[j];
  const auto pre = Model::template prologue<true>(xv);
  stamp();
  dbg_tail(a, 4);
  moments_to_kvec(pre.g, (double)a.m, mom, vec);
  if (threadIdx.x == 0) vec[KT] = mom[MomLayout::NV];  // non-finite count
  __syncthreads();
  stamp();
  dbg_tail(a, 5);
  if (!a.no_chain) apply_chain_kvec<Model, TPB>(pre, vec, scratch);
  stamp();
  dbg_tail(a, 6);
  pass_tail<KS, TPB, true>(a, st, vec, cond, use_cond);
  dbg_tail(a, 7);
}

// dynamic shared memory of moment_pass_kernel<.., STG> (the z ring; reused
// for the block-partial table after the main loop)
__host__ __device__ constexpr int moment_smem_bytes(int L, int TPB, int STG) {
  return STG > 0 ? ((TPB / 32) * STG * 32 * L * 8 > MomLayout::KS * (TPB + 1) * 8
                        ? (TPB / 32) * STG * 32 * L * 8
                        : MomLayout::KS * (TPB + 1) * 8)
                 : 0;
}

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  const unsigned a = smem_u32(bar);
  unsigned done = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
  } while (!done);
}

// STG == 0: each lane prefetches its points of the next chunk into registers.
// STG >= 2: z streams through a per-warp ring of STG chunk slots in shared
// memory, filled by TMA bulk copies (cp.async.bulk, one 32 L x 8 B copy per
// chunk, completion on an mbarrier per slot) issued STG - 1 chunks ahead by
// lane 0; the row moments then live in registers and the ring doubles as the
// block-partial table at the end.
template <int L, int TPB, int MINB, int SEEDN = 4, int STG = 0>
__global__ void __launch_bounds__(TPB, MINB)
    moment_pass_kernel(const PassArgs* __restrict__ pa, FitState* __restrict__ st, cudaGraphConditionalHandle cond,
                       int use_cond) {
  using Model = ModelGauss2DRot;
  constexpr int N = Model::N;
  constexpr int NV = MomLayout::NV;
  constexpr int CW = 32 * L;
  constexpr double D = 32.0;
  constexpr bool TMA = STG >= 2;
  constexpr int NF = MomLayout::OSR;  // folded moments per thread (27)
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

  // per-thread moments with dy folded in.  STG == 0: shared memory, one
  // column per thread (updated once per image row a lane visits; keeps the
  // registers for the z prefetch); STG >= 2: registers.
  extern __shared__ __align__(128) double dyn[];
  __shared__ double smom_s[TMA ? 1 : MomLayout::KS][TMA ? 1 : TPB + 1];  // + sum r, sum r^2, bad; padded rows
  auto smom = [&](int i, int t) -> double& {
    if constexpr (TMA) return dyn[i * (TPB + 1) + t];
    else return smom_s[i][t];
  };
  const int tid = threadIdx.x;
  double Mf[TMA ? NF : 1];
#pragma unroll
  for (int i = 0; i < NF; ++i) {
    if constexpr (TMA) Mf[i] = 0.0;
    else smom(i, tid) = 0.0;
  }
  auto macc = [&](int i) -> double& {
    if constexpr (TMA) return Mf[i];
    else return smom(i, tid);
  };
  double sr = 0.0, srr = 0.0;
  // The lane's running moments of the current image row, about a moving
  // origin o (the dx of the lane's first pixel of the current chunk):
  //   P[p] = sum u^2 t^p, Q[p] = sum u t^p, R[p] = sum u r t^p,  t = dx - o.
  // Within a chunk t = D k (k = step index), so every t^p is a compile-time
  // constant; moving the origin to the next chunk (o += CW) is a Taylor shift.
  double P[5], Q[3], R[3];
#pragma unroll
  for (int i = 0; i < 5; ++i) P[i] = 0.0;
#pragma unroll
  for (int i = 0; i < 3; ++i) Q[i] = R[i] = 0.0;
  int bad = 0;

  // moments about o -> about o - d:  M'_p = sum_i C(p, i) d^(p-i) M_i
  // (Pascal scheme: for j = 1..deg, for p = deg..j: M_p += d M_(p-1))
  auto shift = [&](double d) {
#pragma unroll
    for (int j = 1; j <= 4; ++j)
#pragma unroll
      for (int p = 4; p >= j; --p) P[p] = fma(d, P[p - 1], P[p]);
#pragma unroll
    for (int j = 1; j <= 2; ++j)
#pragma unroll
      for (int p = 2; p >= j; --p) {
        Q[p] = fma(d, Q[p - 1], Q[p]);
        R[p] = fma(d, R[p - 1], R[p]);
      }
  };
  double org = 0.0;  // o of the running row moments
  auto fold = [&](double dy) {  // row moments (about dx = 0) x dy^q into the thread's moments
    shift(org);
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
        double& m2 = macc(MomLayout::O2 + mono(4, p, q));
        m2 = fma(P[p], dq[q], m2);
      }
#pragma unroll
    for (int q = 0; q <= 2; ++q)
#pragma unroll
      for (int p = 0; p + q <= 2; ++p) {
        double& m1 = macc(MomLayout::O1 + mono(2, p, q));
        m1 = fma(Q[p], dq[q], m1);
        double& mr = macc(MomLayout::OR + mono(2, p, q));
        mr = fma(R[p], dq[q], mr);
      }
#pragma unroll
    for (int i = 0; i < 5; ++i) P[i] = 0.0;
#pragma unroll
    for (int i = 0; i < 3; ++i) Q[i] = R[i] = 0.0;
  };
  // one point at t = D k from the origin: u = exp(-q), data z
  auto point = [&](double u, double t, double z) {
    const double r = fma(A, u, off) - z;  // Eq. 1: r = h - z
    bad += isfinite(r) ? 0 : 1;
    const double u2 = u * u;
    const double t2 = t * t;
    P[0] += u2;
    P[1] = fma(u2, t, P[1]);
    P[2] = fma(u2, t2, P[2]);
    P[3] = fma(u2, t2 * t, P[3]);
    P[4] = fma(u2, t2 * t2, P[4]);
    Q[0] += u;
    Q[1] = fma(u, t, Q[1]);
    Q[2] = fma(u, t2, Q[2]);
    const double ur = u * r;
    R[0] += ur;
    R[1] = fma(ur, t, R[1]);
    R[2] = fma(ur, t2, R[2]);
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
  auto dbg_stamp = [&](int slot) {  // development aid (JF_DEBUG_STAMPS)
    if (a.dbg && lane == 0 && gw < 16384) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      unsigned smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      a.dbg[gw * 4 + 0] = smid;
      a.dbg[gw * 4 + slot] = t;
    }
  };
  dbg_stamp(1);

  // ---- z staging
  double zn[TMA ? 1 : L];  // STG == 0: the next chunk's points
  constexpr int NWB = TPB / 32;
  __shared__ __align__(8) unsigned long long mbar[TMA ? NWB * STG : 1];
  double* ring = dyn + (TMA ? (threadIdx.x >> 5) * STG * CW : 0);
  unsigned long long* wbar = mbar + (TMA ? (threadIdx.x >> 5) * STG : 0);
  unsigned direct = 0;  // TMA: slot s holds no copy (ragged or unaligned chunk: read from global)
  unsigned parity = 0;  // TMA: mbarrier phase parity per slot
  const bool z_al16 = (reinterpret_cast<uintptr_t>(z) & 15) == 0;
  unsigned long long pol = 0;
  if constexpr (TMA) {
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    if (lane == 0) {
#pragma unroll
      for (int s = 0; s < STG; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(wbar + s)));
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
  }
  // chunk ch = row * cpr + cc; row and cc are advanced incrementally (no
  // 64-bit division in the loop)
  int64_t lrow = c_begin / cpr;  // position of the next chunk to load
  int lcc = (int)(c_begin - lrow * cpr);
  auto load = [&](int slot) {
    const int c0l = lcc * CW;
    const int64_t g0 = lrow * (int64_t)W + c0l;
    if constexpr (TMA) {
      if (c0l + CW <= W && z_al16 && (g0 & 1) == 0) {  // warp-uniform
        direct &= ~(1u << slot);
        if (lane == 0) {
          const unsigned b = smem_u32(wbar + slot);
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(CW * 8) : "memory");
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], "
              "%4;" ::"r"(smem_u32(ring + slot * CW)),
              "l"(z + g0), "r"(CW * 8), "r"(b), "l"(pol)
              : "memory");
        }
      } else {
        direct |= 1u << slot;
      }
    } else {
      const double* zp = z + g0 + lane;
      if (c0l + CW <= W) {  // warp-uniform
#pragma unroll
        for (int k = 0; k < L; ++k) zn[k] = __ldcs(zp + 32 * k);
      } else {
#pragma unroll
        for (int k = 0; k < L; ++k) zn[k] = (c0l + lane + 32 * k < W) ? __ldcs(zp + 32 * k) : 0.0;
      }
    }
    if (++lcc == cpr) {
      lcc = 0;
      ++lrow;
    }
  };
  if constexpr (TMA) {
#pragma unroll
    for (int s = 0; s < STG; ++s)
      if (c_begin + s < c_end) load(s);
  } else {
    if (c_begin < c_end) load(0);
  }
  int64_t cur_row = c_begin / cpr;
  int cc = (int)(c_begin - cur_row * cpr) - 1;  // chunk column of the current chunk (advanced below)
  int64_t row = cur_row;
  double E = 0.0, Rr = 0.0;
  bool carried = false;
  int since_seed = 0;
  int slot = 0;
  for (int64_t ch = c_begin; ch < c_end; ++ch) {
    double zc[TMA ? 1 : L];
    if constexpr (!TMA) {
#pragma unroll
      for (int k = 0; k < L; ++k) zc[k] = zn[k];
      if (ch + 1 < c_end) load(0);  // prefetch the next chunk
    }
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
    const double* zrow = z + row * (int64_t)W + c0 + lane;  // this lane's first point of the chunk (global)
    const double* zsl = ring + slot * CW + lane;           // ... in the ring (TMA)
    bool from_ring = false;
    if constexpr (TMA) {
      if (!((direct >> slot) & 1u)) {
        mbar_wait(wbar + slot, (parity >> slot) & 1u);
        parity ^= 1u << slot;
        from_ring = true;
      }
    }
    // origin of the running moments -> this chunk's first pixel (zero
    // moments after a fold shift to zero)
    shift(-(double)CW);
    org = dx0;
    const double q0 = dx0 * (ga * dx0 + gb2 * dy) + gc * (dy * dy);
    const double argR = D * (2.0 * ga * dx0 + gb2 * dy) + ga * D * D;
    const bool ok = fabs(q0) < 600.0 && fabs(argR) < 300.0 && 2.0 * ga * D * D * L < 300.0;
    const bool full = c0 + CW <= W;  // warp-uniform
    // the chunk: recurrence for u, moments in t = D k (compile-time t^p)
    auto chunk = [&](auto zat) {
      // E, Rr continue from the previous chunk of the same row (its last
      // step lands on this chunk's first pixel); re-seeded by exp at a row
      // start, after a direct-evaluation chunk, and every SEEDN chunks so the
      // recurrence's rounding stays below ~(L SEEDN)^2 / 2 ulp
      if (!carried || ++since_seed >= SEEDN) {  // warp-uniform
        E = exp(-q0);
        Rr = exp(-argR);
        since_seed = 0;
      }
      // the chunk's sum r^2 doubles as its non-finite test (any non-finite
      // r makes it non-finite; the exact count is then taken below)
      double cs = 0.0;
      const double E_in = E, R_in = Rr;
#pragma unroll
      for (int k = 0; k < L; ++k) {
        const double u = E;
        const double r = fma(A, u, off) - zat(k);  // Eq. 1: r = h - z
        const double u2 = u * u;
        const double k1 = D * k, k2 = k1 * k1, k3 = k2 * k1, k4 = k2 * k2;
        const double ur = u * r;
        P[0] += u2;
        Q[0] += u;
        R[0] += ur;
        if (k > 0) {
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
      carried = true;
      srr += cs;
      if (!isfinite(cs)) {  // rare: replay the chunk's residuals and count the non-finite ones
        double e = E_in, rr = R_in;
#pragma unroll
        for (int k = 0; k < L; ++k) {
          bad += isfinite(fma(A, e, off) - zat(k)) ? 0 : 1;
          e *= rr;
          rr *= rho;
        }
      }
    };
    if (full && __all_sync(FULL, ok)) {
      if constexpr (TMA) {
        if (from_ring) chunk([&](int k) { return zsl[32 * k]; });
        else chunk([&](int k) { return __ldcs(zrow + 32 * k); });
      } else {
        chunk([&](int k) { return zc[k]; });
      }
    } else {
      // ragged row end or unsafe exponent range: direct evaluation
      carried = false;
#pragma unroll
      for (int k = 0; k < L; ++k) {
        if (c0 + lane + 32 * k < W) {
          const double dx = dx0 + D * k;
          double zk;
          if constexpr (TMA) zk = from_ring ? zsl[32 * k] : __ldcs(zrow + 32 * k);
          else zk = zc[k];
          point(exp(-(dx * (ga * dx + gb2 * dy) + gc * (dy * dy))), D * k, zk);
        }
      }
    }
    if constexpr (TMA) {
      __syncwarp();  // every lane has read the slot: refill it STG chunks ahead
      if (ch + STG < c_end) load(slot);
      slot = (slot + 1 == STG) ? 0 : slot + 1;
    }
  }
  if (c_begin < c_end) fold((double)(cur_row + row0) - y0);
  dbg_stamp(2);
  if constexpr (TMA) {
    __syncthreads();  // the ring becomes the block-partial table
#pragma unroll
    for (int i = 0; i < NF; ++i) smom(i, tid) = Mf[i];
  }

  // block partial of the moment vector
  __shared__ double red[TPB / 32][MomLayout::KS];
  __shared__ double vec[KMAX];
  __shared__ double scratch[combine_scratch(TPB)];
  __shared__ double mom[MomLayout::KS];
  {
    // block partial: the threads' columns of smom summed by rows, NSEG
    // segments of 32 threads each, then the segments in order
    smom(MomLayout::OSR, tid) = sr;
    smom(MomLayout::OSRR, tid) = srr;
    smom(NV, tid) = (double)bad;
    __syncthreads();
    constexpr int NSEG = TPB / 32;
    static_assert(NSEG * MomLayout::KS <= TPB, "one (row, segment) per thread");
    if (tid < NSEG * MomLayout::KS) {
      const int i = tid % MomLayout::KS, seg = tid / MomLayout::KS;
      double s = 0.0;
#pragma unroll 8
      for (int j = 0; j < 32; ++j) s += smom(i, seg * 32 + j);
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
  dbg_stamp(3);
  if (!grid_reduce<MomLayout::KS, TPB>(a, mom, scratch)) return;
  moment_finish<TPB>(a, st, xs, mom, vec, scratch, cond, use_cond);
  if (a.dbg && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.dbg[4 * 16384 - 1] = t;
  }
}

// ---------------------------------------------------------------------------
// Task-scheduled moment J-pass (the production kernel for the north-star
// configuration).  One block per SM (NW warps).  The block's share of the
// image is a fixed, contiguous range of TASKS — runs of up to TC chunks
// (32 L pixels each) of one image row — and the warps take tasks from a
// shared-memory counter as they become free, so the SM's warps finish
// together however the warp scheduler shares the FP64 pipe among them
// (with a static per-warp split, the fastest and slowest warps of an SM
// differed 2x).  The result does not depend on which warp ran a task: every
// task starts from zero moments and a fresh exp seed, its per-lane moments
// are summed across the warp in lane order and written, folded with dy, to
// the task's own slot; the block partial sums the slots in task order.
// Single-level grid combine (one partial per SM).
constexpr int MOMENT_MAXT = 112;  // task slots per block of moment_task_kernel
__host__ __device__ constexpr int moment_task_smem_bytes(int NW) {
  return (MOMENT_MAXT * MomLayout::KS + NW * 13 * 33) * 8;
}
template <int L, int TC, int NW, int SEEDN = 4, int DBGZ = 0, int FASTP = 1>
__global__ void __launch_bounds__(NW * 32, 1)
    moment_task_kernel(const PassArgs* __restrict__ pa, FitState* __restrict__ st, cudaGraphConditionalHandle cond,
                       int use_cond) {
  using Model = ModelGauss2DRot;
  using Pre = typename Model::Pre;
  constexpr int N = Model::N, KT = tri_count(N), KS2 = KT + 1;
  constexpr int TPB = NW * 32;
  constexpr int KS = MomLayout::KS, NV = MomLayout::NV;
  constexpr int CW = 32 * L;
  constexpr int MAXT = MOMENT_MAXT;
  constexpr double D = 32.0;
  const PassArgs& a = *pa;
  if (!pass_begin<true, false>(a, st)) return;
  const double* xs = (a.epilogue == EPI_FIT) ? st->x_eval : a.x;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;

  extern __shared__ __align__(16) double dyn_task[];  // moment_task_smem_bytes(NW)
  double (*tslot)[KS] = reinterpret_cast<double (*)[KS]>(dyn_task);                 // [MAXT][KS] per-task vectors
  double (*wred)[13][33] = reinterpret_cast<double (*)[13][33]>(dyn_task + MAXT * KS);  // [NW]: lane-sum transpose
  __shared__ double red[TPB / 32 > 0 ? NW : 1][KS];
  __shared__ double vec[KMAX];
  __shared__ double scratch[combine_scratch(TPB)];
  __shared__ double mom[KS];
  __shared__ double fmap[KT][FMAP_COLS];    // the finish map (warp 0, at the start)
  __shared__ int next_task;
  __shared__ double binom[5][5];            // C(p, i)

  double A, off, ga, gb2, gc, x0, y0;
  {
    double xv[N];
#pragma unroll
    for (int j = 0; j < N; ++j) xv[j] = xs[j];
    const auto pre = Model::template prologue<false>(xv);
    A = pre.g.A, off = pre.off, ga = pre.g.a, gb2 = pre.g.b2, gc = pre.g.c, x0 = pre.g.x0, y0 = pre.g.y0;
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
  // lane -> entry of the moment vector it folds at a task end: family row
  // base in the lane-sum table, dx power p, dy power q (MomLayout order)
  int f_base = 0, f_p = 0, f_q = 0;
  if (lane < MomLayout::OSR) {
    int deg, idx;
    if (lane < MomLayout::O1) f_base = 0, deg = 4, idx = lane;
    else if (lane < MomLayout::OR) f_base = 5, deg = 2, idx = lane - MomLayout::O1;
    else f_base = 8, deg = 2, idx = lane - MomLayout::OR;
    f_p = idx;
    while (f_p > deg - f_q) {
      f_p -= deg - f_q + 1;
      ++f_q;
    }
  }

  // ---- the block's tasks
  const int W = (int)a.W;
  const int64_t H = a.m / a.W;
  const int64_t row0 = a.row0;
  const int cpr = (W + CW - 1) / CW;
  const int nblk = gridDim.x;
  // task length: TC chunks, longer when the block would get more than MAXT tasks
  // (TSPLIT > 0: the block's last TSPLIT tasks are split into single-chunk
  // tasks so the warps run out of work within about one chunk of each other;
  // measured slower at 4096^2 — the per-task overhead outweighs the balance)
  constexpr int TSPLIT = 0;
  // More tasks than MAXT slots: the block runs them in rounds of MAXT (the
  // slot sums of each round are added in round order: still a fixed order).
  const int tcr = TC < cpr ? TC : cpr;
  const int tpr = (cpr + tcr - 1) / tcr;  // tasks per row
  const int64_t ntask = H * (int64_t)tpr;
  const int64_t t_begin = (int64_t)blockIdx.x * ntask / nblk, t_end = (int64_t)(blockIdx.x + 1) * ntask / nblk;
  const int nt_big = (int)(t_end - t_begin);
  const int nbig = nt_big > TSPLIT ? nt_big - TSPLIT : 0;  // tasks kept whole
  const int nt_all = nbig + (nt_big - nbig) * tcr;          // tasks (single-chunk tail tasks may be empty)
  const int nround = nt_all > MAXT ? (nt_all + MAXT - 1) / MAXT : 1;
  int rbase = 0;                                            // first task of the current round
  int nt = nt_all < MAXT ? nt_all : MAXT;                   // tasks of the current round

  const double rho = exp(-2.0 * ga * D * D);
  const double* __restrict__ z = a.z;
  if (a.dbg && lane == 0 && blockIdx.x * NW + wid < 16384) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    a.dbg[(blockIdx.x * NW + wid) * 4 + 0] = smid;
    a.dbg[(blockIdx.x * NW + wid) * 4 + 1] = t;
  }

  // one warp builds the finish map (any block may be the last one): warp 0
  // before its first task when the block has at least NW tasks (the task
  // counter balances its late start); otherwise the last warp, which then
  // takes no task, so the map is built while the other warps run the tasks
  // (with fewer tasks than warps, every warp beyond the task count builds a
  // share of the map's rows, one row per lane)
  const int map_warp = (nt_all < NW) ? NW - 1 : 0;
  const bool map_builder = (nt_all < NW) ? (wid >= nt_all) : (wid == 0);
  if (map_builder) {
    double xv[N];
#pragma unroll
    for (int j = 0; j < N; ++j) xv[j] = xs[j];
    const auto pre = Model::template prologue<true>(xv);
    if (nt_all < NW) build_finish_map(pre, fmap, (wid - nt_all) * 32 + lane, (NW - nt_all) * 32);
    else build_finish_map(pre, fmap, lane, 32);
  }

  double P[5], Q[3], R[3], sr, srr;
  int bad;
  auto shift = [&](double d) {  // moments about o -> about o - d (Pascal scheme)
#pragma unroll
    for (int j = 1; j <= 4; ++j)
#pragma unroll
      for (int p = 4; p >= j; --p) P[p] = fma(d, P[p - 1], P[p]);
#pragma unroll
    for (int j = 1; j <= 2; ++j)
#pragma unroll
      for (int p = 2; p >= j; --p) {
        Q[p] = fma(d, Q[p - 1], Q[p]);
        R[p] = fma(d, R[p - 1], R[p]);
      }
  };
  auto point = [&](double u, double t, double zv) {
    const double r = fma(A, u, off) - zv;  // Eq. 1: r = h - z
    bad += isfinite(r) ? 0 : 1;
    const double u2 = u * u;
    const double t2 = t * t;
    P[0] += u2;
    P[1] = fma(u2, t, P[1]);
    P[2] = fma(u2, t2, P[2]);
    P[3] = fma(u2, t2 * t, P[3]);
    P[4] = fma(u2, t2 * t2, P[4]);
    Q[0] += u;
    Q[1] = fma(u, t, Q[1]);
    Q[2] = fma(u, t2, Q[2]);
    const double ur = u * r;
    R[0] += ur;
    R[1] = fma(ur, t, R[1]);
    R[2] = fma(ur, t2, R[2]);
    sr += r;
    srr = fma(r, r, srr);
  };

  // task -> (row, first chunk column, chunks); 32-bit arithmetic relative to
  // the block's first task
  const int64_t row_b = t_begin / tpr;
  const int k_b = (int)(t_begin - row_b * tpr);
  auto task_pos = [&](int t, int64_t& row, int& cc0, int& ncc) {
    t += rbase;
    int sub = -1;
    if (t >= nbig) {  // single-chunk tail task: chunk sub of whole task bt
      sub = (t - nbig) % tcr;
      t = nbig + (t - nbig) / tcr;
    }
    const int g = k_b + t;
    const int dr = g / tpr;
    row = row_b + dr;
    cc0 = (g - dr * tpr) * tcr;
    ncc = min(tcr, cpr - cc0);
    if (sub >= 0) {
      cc0 += sub;
      ncc = sub < ncc ? 1 : 0;
    }
  };
  auto grab = [&]() {
    int t = 0;
    if (lane == 0) t = atomicAdd(&next_task, 1);
    return __shfl_sync(FULL, t, 0);
  };
  double zn[L];
  auto load = [&](int64_t row, int cc) {
    const int c0l = cc * CW;
    const double* zp = DBGZ ? z + lane : z + row * (int64_t)W + c0l + lane;  // DBGZ: compute-only probe (L1-resident z)
    if (c0l + CW <= W) {  // warp-uniform
#pragma unroll
      for (int k = 0; k < L; ++k) zn[k] = __ldcs(zp + 32 * k);
    } else {
#pragma unroll
      for (int k = 0; k < L; ++k) zn[k] = (c0l + lane + 32 * k < W) ? __ldcs(zp + 32 * k) : 0.0;
    }
  };

  (void)map_warp;
  // this thread's (entry, segment) share of the block partial, accumulated
  // over the rounds in shared memory (keeps it out of the hot loop's registers)
  if (tid < NW * KS) red[tid / KS][tid % KS] = 0.0;
  for (int rd = 0; rd < nround; ++rd) {
  if (rd > 0) {
    rbase = rd * MAXT;
    nt = min(MAXT, nt_all - rbase);
    if (tid == 0) next_task = 0;
    __syncthreads();
  }
  int task = (nt_all < NW && map_builder) ? nt : grab();
  int64_t trow = 0;
  int tcc0 = 0, tncc = 0;
  if (task < nt) {
    task_pos(task, trow, tcc0, tncc);
    load(trow, tcc0);
  }
  while (task < nt) {
    // ---- one task: chunks tcc0 .. tcc0 + tncc - 1 of row trow
    const int64_t row = trow;
    const int cc0 = tcc0, ncc = tncc;
    const int my = task;
    const double dy = (double)(row + row0) - y0;
    int next = nt;
#pragma unroll
    for (int i = 0; i < 5; ++i) P[i] = 0.0;
#pragma unroll
    for (int i = 0; i < 3; ++i) Q[i] = R[i] = 0.0;
    sr = srr = 0.0;
    bad = 0;
    double E = 0.0, Rr = 0.0, org = 0.0;
    bool carried = false;
    int since_seed = 0;
    // Fast path: a whole task of TC chunks inside the row whose exponents are
    // safe over its full pixel range (q is convex along the row and argR is
    // linear, so the range ends bound them): the TC chunks are one unrolled
    // run of TC L points per lane with t = D (L j + k) measured from the
    // task's first pixel — compile-time t^p, no per-chunk shift or set-up,
    // one exp seed per task.
    bool fast = false;
    {
      const int c0 = cc0 * CW;
      const double dxa = (double)(c0 + lane) - x0, dxb = dxa + D * (TC * L - 1);
      const double qa = dxa * (ga * dxa + gb2 * dy) + gc * (dy * dy);
      const double qb = dxb * (ga * dxb + gb2 * dy) + gc * (dy * dy);
      const double ra = D * (2.0 * ga * dxa + gb2 * dy) + ga * D * D;
      const double rb = D * (2.0 * ga * dxb + gb2 * dy) + ga * D * D;
      const bool ok = qa < 600.0 && qb < 600.0 && fabs(ra) < 300.0 && fabs(rb) < 300.0 &&
                      2.0 * ga * D * D * (TC * L) < 300.0;
      fast = (FASTP != 0) && (ncc == TC) && (c0 + TC * CW <= W) && __all_sync(FULL, ok);  // warp-uniform
      if (fast && FASTP == 2) {
        // rolled variant: the TC chunks as a loop (a quarter of the hot code),
        // t = D k within the chunk, the origin moved per chunk (Taylor shift)
        org = dxa;
        E = exp(-qa);
        Rr = exp(-ra);
#pragma unroll 1
        for (int j = 0; j < TC; ++j) {
          double zc[L];
#pragma unroll
          for (int k = 0; k < L; ++k) zc[k] = zn[k];
          if (j + 1 < TC) {
            load(row, cc0 + j + 1);
          } else {
            next = grab();
            if (next < nt) {
              task_pos(next, trow, tcc0, tncc);
              load(trow, tcc0);
            }
          }
          if (j > 0) {
            shift(-(double)CW);
            org += (double)CW;
          }
          double cs = 0.0;
          const double E_in = E, R_in = Rr;
#pragma unroll
          for (int k = 0; k < L; ++k) {
            const double u = E;
            const double r = fma(A, u, off) - zc[k];  // Eq. 1: r = h - z
            const double u2 = u * u;
            const double k1 = D * k, k2 = k1 * k1, k3 = k2 * k1, k4 = k2 * k2;
            const double ur = u * r;
            P[0] += u2;
            Q[0] += u;
            R[0] += ur;
            if (k > 0) {
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
              bad += isfinite(fma(A, e, off) - zc[k]) ? 0 : 1;
              e *= rr;
              rr *= rho;
            }
          }
        }
      } else if (fast) {
        org = dxa;
        E = exp(-qa);
        Rr = exp(-ra);
#pragma unroll
        for (int j = 0; j < TC; ++j) {
          double zc[L];
#pragma unroll
          for (int k = 0; k < L; ++k) zc[k] = zn[k];
          if (j + 1 < TC) {
            load(row, cc0 + j + 1);
          } else {
            next = grab();
            if (next < nt) {
              task_pos(next, trow, tcc0, tncc);
              load(trow, tcc0);
            }
          }
          double cs = 0.0;
          const double E_in = E, R_in = Rr;
#pragma unroll
          for (int k = 0; k < L; ++k) {
            const double u = E;
            const double r = fma(A, u, off) - zc[k];  // Eq. 1: r = h - z
            const double u2 = u * u;
            const double k1 = D * (L * j + k), k2 = k1 * k1, k3 = k2 * k1, k4 = k2 * k2;
            const double ur = u * r;
            P[0] += u2;
            Q[0] += u;
            R[0] += ur;
            if (L * j + k > 0) {
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
              bad += isfinite(fma(A, e, off) - zc[k]) ? 0 : 1;
              e *= rr;
              rr *= rho;
            }
          }
        }
      }
    }
    for (int j = 0; j < (fast ? 0 : ncc); ++j) {
      double zc[L];
#pragma unroll
      for (int k = 0; k < L; ++k) zc[k] = zn[k];
      if (j + 1 < ncc) {
        load(row, cc0 + j + 1);  // prefetch the next chunk of this task
      } else {
        next = grab();  // ... or the first chunk of the next task
        if (next < nt) {
          task_pos(next, trow, tcc0, tncc);
          load(trow, tcc0);
        }
      }
      const int c0 = (cc0 + j) * CW;
      const double dx0 = (double)(c0 + lane) - x0;
      shift(-(double)CW);  // origin -> this chunk's first pixel (zero moments at j = 0)
      org = dx0;
      const double q0 = dx0 * (ga * dx0 + gb2 * dy) + gc * (dy * dy);
      const double argR = D * (2.0 * ga * dx0 + gb2 * dy) + ga * D * D;
      const bool ok = fabs(q0) < 600.0 && fabs(argR) < 300.0 && 2.0 * ga * D * D * L < 300.0;
      const bool full = c0 + CW <= W;  // warp-uniform
      if (full && __all_sync(FULL, ok)) {
        if (!carried || ++since_seed >= SEEDN) {  // warp-uniform
          E = exp(-q0);
          Rr = exp(-argR);
          since_seed = 0;
        }
        double cs = 0.0;
        const double E_in = E, R_in = Rr;
#pragma unroll
        for (int k = 0; k < L; ++k) {
          const double u = E;
          const double r = fma(A, u, off) - zc[k];  // Eq. 1: r = h - z
          const double u2 = u * u;
          const double k1 = D * k, k2 = k1 * k1, k3 = k2 * k1, k4 = k2 * k2;
          const double ur = u * r;
          P[0] += u2;
          Q[0] += u;
          R[0] += ur;
          if (k > 0) {
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
        carried = true;
        srr += cs;
        if (!isfinite(cs)) {  // rare: replay the chunk's residuals and count the non-finite ones
          double e = E_in, rr = R_in;
#pragma unroll
          for (int k = 0; k < L; ++k) {
            bad += isfinite(fma(A, e, off) - zc[k]) ? 0 : 1;
            e *= rr;
            rr *= rho;
          }
        }
      } else {
        // ragged row end or unsafe exponent range: direct evaluation
        carried = false;
#pragma unroll
        for (int k = 0; k < L; ++k) {
          if (c0 + lane + 32 * k < W) {
            const double dx = dx0 + D * k;
            point(exp(-(dx * (ga * dx + gb2 * dy) + gc * (dy * dy))), D * k, zc[k]);
          }
        }
      }
    }
    if (ncc == 0) {  // empty tail task: zero slot, next task
      next = grab();
      if (next < nt) {
        task_pos(next, trow, tcc0, tncc);
        load(trow, tcc0);
      }
    }
    // ---- the task's moment vector: lane moments to the common origin
    // o* = org - lane (lane 0's), summed across the warp in lane order,
    // then moved to dx = 0 and folded with dy^q (lane i: vector entry i)
    shift((double)lane);
    {
      double (*wr)[33] = wred[wid];
#pragma unroll
      for (int i = 0; i < 5; ++i) wr[i][lane] = P[i];
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        wr[5 + i][lane] = Q[i];
        wr[8 + i][lane] = R[i];
      }
      wr[11][lane] = sr;
      wr[12][lane] = srr;
      const int nbad = __reduce_add_sync(FULL, bad);
      __syncwarp();
      if (lane < 13) {  // four interleaved chains, then combined (fixed order)
        double s4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int l = 0; l < 32; ++l) s4[l & 3] += wr[lane][l];
        wr[lane][32] = (s4[0] + s4[1]) + (s4[2] + s4[3]);
      }
      __syncwarp();
      const double os = org - (double)lane;  // o*: the common origin (dx of lane 0's first pixel of the last chunk)
      const double o = __shfl_sync(FULL, os, 0);
      if (lane < KS) {
        double v;
        if (lane < MomLayout::OSR) {
          // about dx = 0: sum_i C(p, i) o^(p-i) M_i, times dy^q (branch-free:
          // binom[p][i] = 0 for i > p)
          const double o2 = o * o, y2 = dy * dy;
          auto pw = [](int e, double x1, double x2) {  // x^e, e <= 4
            const double lo = (e & 1) ? x1 : 1.0;
            return (e >= 2) ? ((e >= 4) ? x2 * x2 : x2 * lo) : lo;
          };
          double mv = 0.0;
#pragma unroll
          for (int i = 0; i < 5; ++i) {
            const int e = f_p - i;
            const double c = binom[f_p][i] * pw(e < 0 ? 0 : e, o, o2);
            mv = fma(c, wr[min(f_base + i, 12)][32], mv);
          }
          v = mv * pw(f_q, dy, y2);
        } else if (lane == MomLayout::OSR) {
          v = wr[11][32];
        } else if (lane == MomLayout::OSRR) {
          v = wr[12][32];
        } else {
          v = (double)nbad;
        }
        tslot[my][lane] = v;
      }
      __syncwarp();
    }
    task = next;
  }
  __syncthreads();
  if (tid < NW * KS) {  // the round's slots, in slot order, into this thread's share
    const int i = tid % KS, seg = tid / KS;
    double bsum = red[seg][i];
    for (int t = seg; t < nt; t += NW) bsum += tslot[t][i];
    red[seg][i] = bsum;
  }
  __syncthreads();  // the slots are reused by the next round
  }  // rounds
  if (a.dbg && lane == 0 && blockIdx.x * NW + wid < 16384) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.dbg[(blockIdx.x * NW + wid) * 4 + 2] = t;
  }

  // ---- block partial: the task slots summed in task order, then (unless
  // debugging the alt coordinates) mapped through the finish map here, so
  // the last block only sums the blocks' K-vectors
  const bool mapped = !a.no_chain;
  {
    static_assert(NW * KS <= TPB, "one (entry, segment) per thread");
    for (int k = tid; k < KS; k += TPB) {
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < NW; ++w) s += red[w][k];
      mom[k] = s;
    }
    __syncthreads();
    // keep the partial in L2 for the last block (the image streams through evict-first)
    unsigned long long pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    const int np = mapped ? KS2 : KS;
    if (tid < np) {
      double v;
      if (!mapped) {
        v = mom[tid];
      } else if (tid < KT) {
        v = 0.0;
#pragma unroll
        for (int i = 0; i < NV; ++i) v = fma(fmap[tid][i], mom[i], v);
      } else {
        v = mom[NV];  // non-finite count
      }
      asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(a.partials + (size_t)blockIdx.x * np + tid), "d"(v),
                   "l"(pol)
                   : "memory");
    }
  }
  if (a.dbg && lane == 0 && blockIdx.x * NW + wid < 16384) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.dbg[(blockIdx.x * NW + wid) * 4 + 3] = t;
  }
  if (mapped) {
    if (!grid_reduce1<KS2, TPB>(a, vec, scratch)) return;
    // ---- last block: + the point-count term of the map, hand-off
    dbg_tail(a, 3);
    if (tid < KT) vec[tid] = fma(fmap[tid][NV], (double)a.m, vec[tid]);
    __syncthreads();
  } else {
    // debug: the K-vector in the alt coordinates (the two-stage map)
    if (!grid_reduce1<KS, TPB>(a, mom, scratch)) return;
    Pre pre;
    {
      double xv[N];
#pragma unroll
      for (int j = 0; j < N; ++j) xv[j] = xs[j];
      pre = Model::template prologue<true>(xv);
    }
    moments_to_kvec(pre.g, (double)a.m, mom, vec);
    if (tid == 0) vec[KT] = mom[NV];
    __syncthreads();
  }
  dbg_tail(a, 6);
  pass_tail<KS2, TPB, true>(a, st, vec, cond, use_cond);
  dbg_tail(a, 7);
}

}  // namespace jf
