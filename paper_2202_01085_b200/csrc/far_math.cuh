// Device math shared by the far-field kernels (global-sorted and tile-local variants).
// Sec. 3 "Lagrange interpolation": 1-D Lagrange basis on the P
// Chebyshev nodes of the 2nd kind, tensor-product basis over D dimensions (dimension 0
// fastest in the node index k = sum_d k_d P^d).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "f3m_internal.h"

namespace f3m {

template <int P, int D>
struct IPow { static constexpr int value = P * IPow<P, D - 1>::value; };
template <int P>
struct IPow<P, 0> { static constexpr int value = 1; };

__host__ __device__ constexpr int ipow_c(int p, int d) { return d == 0 ? 1 : p * ipow_c(p, d - 1); }

// L_k(tau) = c_k prod_{j != k} (tau - s_j), product form (the barycentric form of App. C
// evaluates the same polynomial); prefix/suffix products, no division, no node-hit branch.
template <int P>
__device__ __forceinline__ void lagrange(float tau, const NodeConsts& nc, float (&L)[P]) {
  float dl[P];
#pragma unroll
  for (int k = 0; k < P; ++k) dl[k] = tau - nc.s[k];
  // prefix pre[k] = prod_{j<k} dl[j], suffix suf[k] = prod_{j>k} dl[j]  (4P - 6 multiplies in all)
  float pre[P], suf[P];
  pre[0] = 1.f;
  pre[1] = dl[0];
#pragma unroll
  for (int k = 2; k < P; ++k) pre[k] = pre[k - 1] * dl[k - 1];
  suf[P - 1] = 1.f;
  suf[P - 2] = dl[P - 1];
#pragma unroll
  for (int k = P - 3; k >= 0; --k) suf[k] = suf[k + 1] * dl[k + 1];
  L[0] = nc.c[0] * suf[0];
  L[P - 1] = nc.c[P - 1] * pre[P - 1];
#pragma unroll
  for (int k = 1; k < P - 1; ++k) L[k] = (nc.c[k] * pre[k]) * suf[k];
}

// Chebyshev polynomials T_0..T_{P-1} at tau (T_0 = 1 folds away): the tile-local kernels
// accumulate Chebyshev moments M_k = sum b prod_d T_{k_d}(tau_d) and evaluate sum_k T_k(x) U~_k.
// The Lagrange basis of the P Chebyshev nodes is L_j = sum_k c_jk T_k exactly (both span the
// polynomials of degree <= P-1), so W = (C x...x C) M and U~ = (C^T x...x C^T) U per box
// (k_cheb_transform): the same interpolant as Sec. 3 / App. C, fewer operations per point.
template <int P>
__device__ __forceinline__ void chebyshev(float tau, float (&T)[P]) {
  T[0] = 1.f;
  if constexpr (P > 1) T[1] = tau;
  const float t2 = tau + tau;
#pragma unroll
  for (int k = 2; k < P; ++k) T[k] = fmaf(t2, T[k - 1], -T[k - 2]);
}

// box-local coordinate tau = (x - lo) (2/l) - 1 with the lower corner lo = lo_hi + lo_lo
__device__ __forceinline__ float local_tau(float x, float lo_hi, float lo_lo, float scale) {
  return fmaf(__fsub_rn(__fsub_rn(x, lo_hi), lo_lo), scale, -1.f);
}

// Tensor-product helpers written as template recursion so that every array index is a
// compile-time constant (no local-memory arrays).
// expand: w[j + len*k] = w[j] * L[d][k] for k < P, j < len   (len = P^d)
template <int P, int LEN>
__device__ __forceinline__ void tp_expand(float* w, const float (&Ld)[P]) {
#pragma unroll
  for (int k = P - 1; k >= 1; --k)
#pragma unroll
    for (int j = 0; j < LEN; ++j) w[j + LEN * k] = w[j] * Ld[k];
#pragma unroll
  for (int j = 0; j < LEN; ++j) w[j] = w[j] * Ld[0];
}

template <int D, int P, int d>
struct TPBuild {  // w (length P^d on entry) expanded over dimensions d .. D-2
  __device__ __forceinline__ static void run(float* w, const float (&L)[D][P]) {
    tp_expand<P, IPow<P, d>::value>(w, L[d]);
    TPBuild<D, P, d + 1>::run(w, L);
  }
};
template <int D, int P>
struct TPBuild<D, P, D - 1> {
  __device__ __forceinline__ static void run(float*, const float (&)[D][P]) {}
};

// acc[k] += b prod_d L_{k_d}
template <int D, int P>
__device__ __forceinline__ void s2m_accumulate(float b, const float (&L)[D][P], float (&acc)[IPow<P, D>::value]) {
  constexpr int MP = IPow<P, D - 1>::value;
  float w[MP];
  w[0] = b;
  TPBuild<D, P, 0>::run(w, L);
#pragma unroll
  for (int k = 0; k < P; ++k)
#pragma unroll
    for (int j = 0; j < MP; ++j) acc[j + MP * k] = fmaf(w[j], L[D - 1][k], acc[j + MP * k]);
}

// contraction over dimension d: t[r] = sum_k L[d][k] t[k + P r], r < LEN  (in place)
// (Chebyshev basis: Ld[0] = T_0 = 1, so the k = 0 term starts the sum)
template <int P, int LEN>
__device__ __forceinline__ void tp_contract(float* t, const float (&Ld)[P]) {
#pragma unroll
  for (int r = 0; r < LEN; ++r) {
    float s = t[P * r];
#pragma unroll
    for (int k = 1; k < P; ++k) s = fmaf(Ld[k], t[k + P * r], s);
    t[r] = s;
  }
}

template <int D, int P, int d>
struct TPContract {  // contract dimensions d .. D-1 of t (length P^{D-d})
  __device__ __forceinline__ static void run(float* t, const float (&L)[D][P]) {
    tp_contract<P, IPow<P, D - d - 1>::value>(t, L[d]);
    TPContract<D, P, d + 1>::run(t, L);
  }
};
template <int D, int P>
struct TPContract<D, P, D> {
  __device__ __forceinline__ static void run(float*, const float (&)[D][P]) {}
};

// sum_k prod_d T_{k_d} u[k] in the Chebyshev basis (T_0 = 1; contract dimension 0 first)
template <int D, int P>
__device__ __forceinline__ float l2t_contract(const float (&L)[D][P], const float (&u)[IPow<P, D>::value]) {
  constexpr int MP = IPow<P, D - 1>::value;
  float t[MP];
#pragma unroll
  for (int r = 0; r < MP; ++r) {
    float s = u[P * r];
#pragma unroll
    for (int k = 1; k < P; ++k) s = fmaf(L[0][k], u[k + P * r], s);
    t[r] = s;
  }
  TPContract<D, P, 1>::run(t, L);
  return t[0];
}

// warp reduce-scatter of M (multiple of 32) per-lane values: afterwards lane l owns the
// warp sums of indices [l*M/32, (l+1)*M/32) in out[0..M/32).
template <int M>
__device__ __forceinline__ void warp_reduce_scatter(float (&v)[M], float (&out)[M / 32]) {
  static_assert(M % 32 == 0, "M must be a multiple of 32");
  const int lane = threadIdx.x & 31;
  float a[M];
#pragma unroll
  for (int i = 0; i < M; ++i) a[i] = v[i];
  int len = M;
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    const int half = len / 2;
    const bool up = (lane & o) != 0;
#pragma unroll
    for (int i = 0; i < M / 2; ++i) {
      if (i < half) {
        const float keep = up ? a[i + half] : a[i];
        const float send = up ? a[i] : a[i + half];
        a[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
      }
    }
    len = half;
  }
#pragma unroll
  for (int i = 0; i < M / 32; ++i) out[i] = a[i];
}

}  // namespace f3m
