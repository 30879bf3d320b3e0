// jf_dual.cuh — forward-mode dual numbers with compile-time sparsity.
//
// The paper obtains the Jacobian J by JAX autodiff ("we use
// JAX's in-built automatic differentiation").  The hot path instead carries,
// per data point, a dual number  v + sum_j d_j eps_j  through the model
// h(y; x): seeding parameter j with d_j = 1 yields dh/dx_j in one forward
// sweep.
//
// Dual<N, M>: N parameters; M is a compile-time bitmask of the partials that
// can be non-zero.  Only those are stored, so operations between values that
// depend on different parameter subsets cost only the non-zero terms, and the
// compiler sees every partial of a seed as the literal +1 (or -1 after a
// subtraction) and folds the multiplications by it.  Nothing here allocates
// or branches at run time; after inlining a model's dual evaluation compiles
// to straight-line fp64 code.
#pragma once

#include <cstdint>
#include <utility>

namespace jf {

__host__ __device__ constexpr int popc_c(unsigned m) { return m ? int(m & 1u) + popc_c(m >> 1) : 0; }
// position of partial j inside the compact storage of mask M
__host__ __device__ constexpr int pos_c(unsigned M, int j) { return popc_c(M & ((1u << j) - 1u)); }

template <int I>
using ic = std::integral_constant<int, I>;

template <class F, int... Is>
__device__ __forceinline__ void static_for_impl(F&& f, std::integer_sequence<int, Is...>) {
  (f(ic<Is>{}), ...);
}
// f(ic<0>), f(ic<1>), ..., f(ic<N-1>) — fully unrolled at compile time.
template <int N, class F>
__device__ __forceinline__ void static_for(F&& f) {
  static_for_impl(f, std::make_integer_sequence<int, N>{});
}

template <int N, unsigned M>
struct Dual {
  static constexpr int n = N;
  static constexpr unsigned mask = M;
  static constexpr int nnz = popc_c(M);
  double v;
  double d[nnz > 0 ? nnz : 1];

  // partial w.r.t. parameter j (0.0 when j is not in the mask)
  template <int j>
  __device__ __forceinline__ double partial() const {
    if constexpr (((M >> j) & 1u) != 0) {
      return d[pos_c(M, j)];
    } else {
      return 0.0;
    }
  }
};

// A parameter seeded for differentiation: value v, dv/dx_j = 1.
template <int N, int j>
__device__ __forceinline__ Dual<N, (1u << j)> seed(double v) {
  Dual<N, (1u << j)> r;
  r.v = v;
  r.d[0] = 1.0;
  return r;
}

// ---------------------------------------------------------------- arithmetic
template <int N, unsigned A, unsigned B>
__device__ __forceinline__ Dual<N, (A | B)> operator+(const Dual<N, A>& a, const Dual<N, B>& b) {
  constexpr unsigned M = A | B;
  Dual<N, M> r;
  r.v = a.v + b.v;
  static_for<N>([&](auto J) {
    constexpr int j = decltype(J)::value;
    if constexpr (((M >> j) & 1u) != 0) {
      constexpr bool ia = ((A >> j) & 1u) != 0, ib = ((B >> j) & 1u) != 0;
      if constexpr (ia && ib) r.d[pos_c(M, j)] = a.d[pos_c(A, j)] + b.d[pos_c(B, j)];
      else if constexpr (ia) r.d[pos_c(M, j)] = a.d[pos_c(A, j)];
      else r.d[pos_c(M, j)] = b.d[pos_c(B, j)];
    }
  });
  return r;
}

template <int N, unsigned A, unsigned B>
__device__ __forceinline__ Dual<N, (A | B)> operator-(const Dual<N, A>& a, const Dual<N, B>& b) {
  constexpr unsigned M = A | B;
  Dual<N, M> r;
  r.v = a.v - b.v;
  static_for<N>([&](auto J) {
    constexpr int j = decltype(J)::value;
    if constexpr (((M >> j) & 1u) != 0) {
      constexpr bool ia = ((A >> j) & 1u) != 0, ib = ((B >> j) & 1u) != 0;
      if constexpr (ia && ib) r.d[pos_c(M, j)] = a.d[pos_c(A, j)] - b.d[pos_c(B, j)];
      else if constexpr (ia) r.d[pos_c(M, j)] = a.d[pos_c(A, j)];
      else r.d[pos_c(M, j)] = -b.d[pos_c(B, j)];
    }
  });
  return r;
}

template <int N, unsigned A, unsigned B>
__device__ __forceinline__ Dual<N, (A | B)> operator*(const Dual<N, A>& a, const Dual<N, B>& b) {
  constexpr unsigned M = A | B;
  Dual<N, M> r;
  r.v = a.v * b.v;
  static_for<N>([&](auto J) {
    constexpr int j = decltype(J)::value;
    if constexpr (((M >> j) & 1u) != 0) {
      constexpr bool ia = ((A >> j) & 1u) != 0, ib = ((B >> j) & 1u) != 0;
      if constexpr (ia && ib) r.d[pos_c(M, j)] = a.d[pos_c(A, j)] * b.v + a.v * b.d[pos_c(B, j)];
      else if constexpr (ia) r.d[pos_c(M, j)] = a.d[pos_c(A, j)] * b.v;
      else r.d[pos_c(M, j)] = a.v * b.d[pos_c(B, j)];
    }
  });
  return r;
}

template <int N, unsigned A, unsigned B>
__device__ __forceinline__ Dual<N, (A | B)> operator/(const Dual<N, A>& a, const Dual<N, B>& b) {
  constexpr unsigned M = A | B;
  Dual<N, M> r;
  const double inv = 1.0 / b.v;
  r.v = a.v * inv;
  static_for<N>([&](auto J) {
    constexpr int j = decltype(J)::value;
    if constexpr (((M >> j) & 1u) != 0) {
      constexpr bool ia = ((A >> j) & 1u) != 0, ib = ((B >> j) & 1u) != 0;
      if constexpr (ia && ib) r.d[pos_c(M, j)] = (a.d[pos_c(A, j)] - r.v * b.d[pos_c(B, j)]) * inv;
      else if constexpr (ia) r.d[pos_c(M, j)] = a.d[pos_c(A, j)] * inv;
      else r.d[pos_c(M, j)] = -r.v * b.d[pos_c(B, j)] * inv;
    }
  });
  return r;
}

// ------------------------------------------------------ scalar (double) mixes
template <int N, unsigned A>
__device__ __forceinline__ Dual<N, A> operator+(const Dual<N, A>& a, double b) {
  Dual<N, A> r = a;
  r.v = a.v + b;
  return r;
}
template <int N, unsigned A>
__device__ __forceinline__ Dual<N, A> operator+(double b, const Dual<N, A>& a) { return a + b; }
template <int N, unsigned A>
__device__ __forceinline__ Dual<N, A> operator-(const Dual<N, A>& a, double b) {
  Dual<N, A> r = a;
  r.v = a.v - b;
  return r;
}
template <int N, unsigned A>
__device__ __forceinline__ Dual<N, A> operator-(double b, const Dual<N, A>& a) {
  Dual<N, A> r;
  r.v = b - a.v;
#pragma unroll
  for (int k = 0; k < Dual<N, A>::nnz; ++k) r.d[k] = -a.d[k];
  return r;
}
template <int N, unsigned A>
__device__ __forceinline__ Dual<N, A> operator-(const Dual<N, A>& a) {
  Dual<N, A> r;
  r.v = -a.v;
#pragma unroll
  for (int k = 0; k < Dual<N, A>::nnz; ++k) r.d[k] = -a.d[k];
  return r;
}
template <int N, unsigned A>
__device__ __forceinline__ Dual<N, A> operator*(const Dual<N, A>& a, double b) {
  Dual<N, A> r;
  r.v = a.v * b;
#pragma unroll
  for (int k = 0; k < Dual<N, A>::nnz; ++k) r.d[k] = a.d[k] * b;
  return r;
}
template <int N, unsigned A>
__device__ __forceinline__ Dual<N, A> operator*(double b, const Dual<N, A>& a) { return a * b; }
template <int N, unsigned A>
__device__ __forceinline__ Dual<N, A> operator/(double b, const Dual<N, A>& a) {
  Dual<N, A> r;
  const double inv = 1.0 / a.v;
  r.v = b * inv;
  const double s = -r.v * inv;
#pragma unroll
  for (int k = 0; k < Dual<N, A>::nnz; ++k) r.d[k] = s * a.d[k];
  return r;
}

// ------------------------------------------------------ elementary functions
// Value functions are overloaded for double too, so a model body written once
// over a generic scalar S instantiates to both the J-pass (S = Dual) and the
// residual-only pass (S = double).
__device__ __forceinline__ double dexp(double a) { return ::exp(a); }
__device__ __forceinline__ double dsin(double a) { return ::sin(a); }
__device__ __forceinline__ double dcos(double a) { return ::cos(a); }

template <int N, unsigned A>
__device__ __forceinline__ Dual<N, A> dexp(const Dual<N, A>& a) {
  Dual<N, A> r;
  r.v = ::exp(a.v);
#pragma unroll
  for (int k = 0; k < Dual<N, A>::nnz; ++k) r.d[k] = r.v * a.d[k];
  return r;
}
template <int N, unsigned A>
__device__ __forceinline__ Dual<N, A> dsin(const Dual<N, A>& a) {
  double s, c;
  ::sincos(a.v, &s, &c);
  Dual<N, A> r;
  r.v = s;
#pragma unroll
  for (int k = 0; k < Dual<N, A>::nnz; ++k) r.d[k] = c * a.d[k];
  return r;
}
template <int N, unsigned A>
__device__ __forceinline__ Dual<N, A> dcos(const Dual<N, A>& a) {
  double s, c;
  ::sincos(a.v, &s, &c);
  Dual<N, A> r;
  r.v = c;
#pragma unroll
  for (int k = 0; k < Dual<N, A>::nnz; ++k) r.d[k] = -s * a.d[k];
  return r;
}

// exp(a) when the value e = exp(a.v) is already known (the grid-stride
// recurrence of jf_pass.cuh supplies it): only the chain-rule partials remain.
__device__ __forceinline__ double dexp_given(double /*a*/, double e) { return e; }
template <int N, unsigned A>
__device__ __forceinline__ Dual<N, A> dexp_given(const Dual<N, A>& a, double e) {
  Dual<N, A> r;
  r.v = e;
#pragma unroll
  for (int k = 0; k < Dual<N, A>::nnz; ++k) r.d[k] = e * a.d[k];
  return r;
}

// value / partial accessors that also work on plain doubles
__device__ __forceinline__ double value(double a) { return a; }
template <int N, unsigned A>
__device__ __forceinline__ double value(const Dual<N, A>& a) { return a.v; }

}  // namespace jf
