// jf_models.cuh — the built-in models h(y; x) of the hot path.
//
// P:44-48 §II Eq. 1: r_i(x) = h(y_i, x) - z_i.  Each model is written ONCE
// over a generic scalar: instantiated with JAC = true every parameter is a
// seeded dual number (jf_dual.cuh) and point() returns h together with the
// whole Jacobian row dh/dx; with JAC = false the same body is the
// residual-only evaluation used at trial points (Eq. 15).
//
// Each model splits into prologue(x) — parameter-only sub-expressions, once
// per thread per pass ("hoisted to a per-pass prologue") —
// and point(pre, y) — the per-data-point work.
//
// Parameter orders are jf.h's (reading R21).
#pragma once

#include "jf_dual.cuh"

namespace jf {

// Parameter j as a dual seed (J-pass) or a plain double (residual pass).
template <bool JAC, int N, int j>
__device__ __forceinline__ auto param(double v) {
  if constexpr (JAC) {
    return seed<N, j>(v);
  } else {
    return v;
  }
}

// ---------------------------------------------------------------- LINEAR (n=2)
struct ModelLinear {
  static constexpr int N = 2, D = 1, CONST_COL = 1;
  static constexpr int NEXP = 0;
  static constexpr int NT = 0;
  template <class P>
  __device__ __forceinline__ static const double* tblock(const P&, int) { return nullptr; }
  __host__ __device__ static constexpr int tbase(int) { return 0; }
  struct Pre {
    double x0, x1;
  };
  template <bool JAC>
  __device__ __forceinline__ static Pre prologue(const double* x) { return {x[0], x[1]}; }
  template <bool JAC>
  __device__ __forceinline__ static auto point(const Pre& p, double t) {
    return param<JAC, N, 0>(p.x0) * t + param<JAC, N, 1>(p.x1);
  }
};

// ------------------------------------------------------------ EXP_DECAY (n=3)
struct ModelExpDecay {
  static constexpr int N = 3, D = 1, CONST_COL = 2;
  static constexpr int NEXP = 0;
  static constexpr int NT = 0;
  template <class P>
  __device__ __forceinline__ static const double* tblock(const P&, int) { return nullptr; }
  __host__ __device__ static constexpr int tbase(int) { return 0; }
  struct Pre {
    double a, b, c;
  };
  template <bool JAC>
  __device__ __forceinline__ static Pre prologue(const double* x) { return {x[0], x[1], x[2]}; }
  template <bool JAC>
  __device__ __forceinline__ static auto point(const Pre& p, double t) {
    // a * exp(-b t) + c
    const auto a = param<JAC, N, 0>(p.a);
    const auto b = param<JAC, N, 1>(p.b);
    const auto c = param<JAC, N, 2>(p.c);
    return a * dexp(-(b * t)) + c;
  }
};

// --------------------------------------------------------------- GAUSS1D (n=4)
template <class TI>
struct PreGauss1D {
  double A, mu, c;
  TI inv2s2;  // 1 / (2 s^2), a dual in s
};
struct ModelGauss1D {
  static constexpr int N = 4, D = 1, CONST_COL = 3;
  static constexpr int NEXP = 0;
  static constexpr int NT = 0;
  template <class P>
  __device__ __forceinline__ static const double* tblock(const P&, int) { return nullptr; }
  __host__ __device__ static constexpr int tbase(int) { return 0; }
  template <bool JAC>
  __device__ __forceinline__ static auto prologue(const double* x) {
    const auto s = param<JAC, N, 2>(x[2]);
    auto inv = 0.5 / (s * s);
    return PreGauss1D<decltype(inv)>{x[0], x[1], x[3], inv};
  }
  template <bool JAC, class P>
  __device__ __forceinline__ static auto point(const P& p, double t) {
    // A * exp(-(t - mu)^2 / (2 s^2)) + c
    const auto dt = t - param<JAC, N, 1>(p.mu);
    const auto E = dexp(-((dt * dt) * p.inv2s2));
    return param<JAC, N, 0>(p.A) * E + param<JAC, N, 3>(p.c);
  }
};

// ------------------------------------------------------- GAUSS2D_ROT (n=7)
// h = A exp(-(a dx^2 + 2 b dx dy + c2 dy^2)) + off
//   a  = cos^2/(2 sx^2) + sin^2/(2 sy^2)
//   b  = sin(2 th) (1/(4 sy^2) - 1/(4 sx^2)) = sin cos (1/(2 sy^2) - 1/(2 sx^2))
//   c2 = sin^2/(2 sx^2) + cos^2/(2 sy^2)
// Two-stage forward mode (chain rule): per point, the dual numbers carry
// the partials w.r.t. the quadratic-form coefficients (a, 2b, c2) in place of
// (sx, sy, th) — simple monomials -dx^2, -dx dy, -dy^2 times A E — and the
// 3x3 block T = d(a, 2b, c2)/d(sx, sy, th), computed once per pass by dual
// numbers in the prologue, maps the reduced W^T W back to the paper's
// parameters: W_x = W_alt T, so W_x^T W_x = T^T (W_alt^T W_alt) T
// (jf_pass.cuh apply_chain_kvec).  Exact chain rule; fewer fp64 operations
// and registers per point than carrying (sx, sy, th) through every point.
struct PreGauss2D {
  double A, x0, y0, a, b2, c;  // b2 = 2b
  double T[9];                 // T[3r + s] = d coef_r / d param_s
};

// One rotated Gaussian component whose parameters start at index B of x.
template <int N, int B>
struct Gauss2DComponent {
  static constexpr int TBASE = B + 3;  // columns (a, 2b, c2) <-> (sx, sy, th)
  template <bool JAC>
  __device__ __forceinline__ static PreGauss2D prologue(const double* x) {
    const auto sx = seed<3, 0>(x[B + 3]);
    const auto sy = seed<3, 1>(x[B + 4]);
    const auto th = seed<3, 2>(x[B + 5]);
    const auto C = dcos(th);
    const auto S = dsin(th);
    const auto ix = 0.5 / (sx * sx);  // 1/(2 sx^2)
    const auto iy = 0.5 / (sy * sy);  // 1/(2 sy^2)
    const auto CC = C * C;
    const auto SS = S * S;
    const auto a = CC * ix + SS * iy;
    const auto b2 = 2.0 * ((S * C) * (iy - ix));
    const auto c = SS * ix + CC * iy;
    PreGauss2D p;
    p.A = x[B + 0];
    p.x0 = x[B + 1];
    p.y0 = x[B + 2];
    p.a = a.v;
    p.b2 = b2.v;
    p.c = c.v;
    static_for<3>([&](auto J) {
      constexpr int s = decltype(J)::value;
      p.T[0 + s] = a.template partial<s>();
      p.T[3 + s] = b2.template partial<s>();
      p.T[6 + s] = c.template partial<s>();
    });
    return p;
  }
  // A * exp(-q), q = dx (a dx + 2b dy) + c2 dy^2; seeds B+3..B+5 = (a, 2b, c2)
  template <bool JAC>
  __device__ __forceinline__ static auto qform(const PreGauss2D& p, double X, double Y) {
    const auto dx = X - param<JAC, N, B + 1>(p.x0);
    const auto dy = Y - param<JAC, N, B + 2>(p.y0);
    const auto a = param<JAC, N, B + 3>(p.a);
    const auto b2 = param<JAC, N, B + 4>(p.b2);
    const auto c = param<JAC, N, B + 5>(p.c);
    return dx * (a * dx + b2 * dy) + c * (dy * dy);
  }
  template <bool JAC>
  __device__ __forceinline__ static auto point(const PreGauss2D& p, double X, double Y) {
    return param<JAC, N, B + 0>(p.A) * dexp(-qform<JAC>(p, X, Y));
  }
  // The same with E = exp(-q(X, Y)) supplied by the caller (row recurrence).
  template <bool JAC>
  __device__ __forceinline__ static auto point_e(const PreGauss2D& p, double X, double Y, double E) {
    return param<JAC, N, B + 0>(p.A) * dexp_given(-qform<JAC>(p, X, Y), E);
  }
  // Plain-double quantities of the row recurrence.
  __device__ __forceinline__ static double qval(const PreGauss2D& p, double X, double Y) {
    const double dx = X - p.x0, dy = Y - p.y0;
    return dx * (p.a * dx + p.b2 * dy) + p.c * (dy * dy);
  }
  __device__ __forceinline__ static void rec_coeffs(const PreGauss2D& p, double& a, double& b2, double& x0,
                                                    double& y0) {
    a = p.a;
    b2 = p.b2;
    x0 = p.x0;
    y0 = p.y0;
  }
};

struct ModelGauss2DRot {
  static constexpr int N = 7, D = 2, CONST_COL = 6;
  static constexpr int NEXP = 1;  // exp factors with a quadratic argument (row recurrence)
  static constexpr int NT = 1;    // chain-rule blocks (see PreGauss2D)
  using G = Gauss2DComponent<N, 0>;
  struct Pre {
    PreGauss2D g;
    double off;
  };
  template <bool JAC>
  __device__ __forceinline__ static Pre prologue(const double* x) {
    return Pre{G::template prologue<JAC>(x), x[6]};
  }
  template <bool JAC>
  __device__ __forceinline__ static auto point(const Pre& p, double X, double Y) {
    return G::template point<JAC>(p.g, X, Y) + param<JAC, N, 6>(p.off);
  }
  template <bool JAC>
  __device__ __forceinline__ static auto point_e(const Pre& p, double X, double Y, const double (&E)[NEXP]) {
    return G::template point_e<JAC>(p.g, X, Y, E[0]) + param<JAC, N, 6>(p.off);
  }
  template <int g>
  __device__ __forceinline__ static double qval(const Pre& p, double X, double Y) {
    return G::qval(p.g, X, Y);
  }
  template <int g>
  __device__ __forceinline__ static void rec_coeffs(const Pre& p, double& a, double& b2, double& x0, double& y0) {
    G::rec_coeffs(p.g, a, b2, x0, y0);
  }
  __device__ __forceinline__ static const double* tblock(const Pre& p, int) { return p.g.T; }
  __host__ __device__ static constexpr int tbase(int) { return G::TBASE; }
};

// ---------------------------------------------------- GAUSS2D_ROT_X2 (n=13)
struct ModelGauss2DRotX2 {
  static constexpr int N = 13, D = 2, CONST_COL = 12;
  static constexpr int NEXP = 2;
  static constexpr int NT = 2;
  using G1 = Gauss2DComponent<N, 0>;
  using G2 = Gauss2DComponent<N, 6>;
  struct Pre {
    PreGauss2D g1, g2;
    double off;
  };
  template <bool JAC>
  __device__ __forceinline__ static Pre prologue(const double* x) {
    return Pre{G1::template prologue<JAC>(x), G2::template prologue<JAC>(x), x[12]};
  }
  template <bool JAC>
  __device__ __forceinline__ static auto point(const Pre& p, double X, double Y) {
    return (G1::template point<JAC>(p.g1, X, Y) + G2::template point<JAC>(p.g2, X, Y)) +
           param<JAC, N, 12>(p.off);
  }
  template <bool JAC>
  __device__ __forceinline__ static auto point_e(const Pre& p, double X, double Y, const double (&E)[NEXP]) {
    return (G1::template point_e<JAC>(p.g1, X, Y, E[0]) + G2::template point_e<JAC>(p.g2, X, Y, E[1])) +
           param<JAC, N, 12>(p.off);
  }
  template <int g>
  __device__ __forceinline__ static double qval(const Pre& p, double X, double Y) {
    if constexpr (g == 0) return G1::qval(p.g1, X, Y);
    else return G2::qval(p.g2, X, Y);
  }
  template <int g>
  __device__ __forceinline__ static void rec_coeffs(const Pre& p, double& a, double& b2, double& x0, double& y0) {
    if constexpr (g == 0) G1::rec_coeffs(p.g1, a, b2, x0, y0);
    else G2::rec_coeffs(p.g2, a, b2, x0, y0);
  }
  __device__ __forceinline__ static const double* tblock(const Pre& p, int g) { return g == 0 ? p.g1.T : p.g2.T; }
  __host__ __device__ static constexpr int tbase(int g) { return g == 0 ? G1::TBASE : G2::TBASE; }
};

}  // namespace jf
