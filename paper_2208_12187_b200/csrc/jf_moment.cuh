// jf_moment.cuh — the moment form of the n = 7 J-pass (reading R34): the
// moment-vector layout and the map moments -> alt-coordinate K-vector shared
// by the moment kernels (jf_moment_stream.cuh, jf_moment2.cuh).
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
#pragma once

#include "jf_pass.cuh"

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

// (the production kernel is moment_stream_kernel, jf_moment_stream.cuh)
constexpr int FMAP_COLS = MomLayout::NV + 1;  // finish-map row: 29 moments + the point count

}  // namespace jf
