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

// box-local coordinate from a two-float offset (kernels_tma.cu tm_box_geometry):
// tau = fma(x, s, off_hi) + off_lo = x s - (lo s + 1)
__device__ __forceinline__ float local_tau_off(float x, float scale, float off_hi, float off_lo) {
  return fmaf(x, scale, off_hi) + off_lo;
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

// ---- packed FP32x2 forms (sm_100a FFMA2 / FMUL2 / FADD2: two lanes of fp32 per instruction,
// the same IEEE single-precision roundings as the scalar forms) for the headline grid D = 3,
// P = 4 (m = 64).  They halve the issue slots of the tensor-product work, which is what bounds
// the tile-local S2M / L2T kernels (instruction issue, not the FMA pipe or HBM).
__device__ __forceinline__ float2 f2b(float v) { return make_float2(v, v); }

// Box-local coordinates and Chebyshev values of one point for D = 3, P = 4, dimensions 0 and
// 1 as one packed pair (FFMA2 / FADD2: each lane rounds exactly as the scalar local_tau_off and
// chebyshev<4>, so the values are bit-identical), dimension 2 scalar.
__device__ __forceinline__ void cheb_d3p4_x2(const float (&x)[3], float scale, const float (&lh)[3],
                                             const float (&ll)[3], float (&T)[3][4]) {
  const float2 tau01 = __fadd2_rn(__ffma2_rn(make_float2(x[0], x[1]), f2b(scale), make_float2(lh[0], lh[1])),
                                  make_float2(ll[0], ll[1]));
  const float2 t2 = __fadd2_rn(tau01, tau01);
  const float2 c2 = __ffma2_rn(t2, tau01, f2b(-1.f));
  const float2 c3 = __ffma2_rn(t2, c2, make_float2(-tau01.x, -tau01.y));
  T[0][0] = 1.f; T[0][1] = tau01.x; T[0][2] = c2.x; T[0][3] = c3.x;
  T[1][0] = 1.f; T[1][1] = tau01.y; T[1][2] = c2.y; T[1][3] = c3.y;
  chebyshev<4>(local_tau_off(x[2], scale, lh[2], ll[2]), T[2]);
}

// S2M: acc2 holds the 64 moments as 32 pairs, pair q = (moment 2q, 2q + 1) with moment index
// k1 + 4 k2 + 16 k3 (dimension 0 fastest).  acc[j + 16 k3] += b T1[k1] T2[k2] T3[k3], j = k1 + 4 k2.
__device__ __forceinline__ void s2m_accumulate_d3p4_x2(float b, const float (&L)[3][4], float2 (&acc2)[32]) {
  // w[j] = b T1[k1] T2[k2] as 8 pairs (j, j + 1): pair (k2, h) = (w[2h + 4 k2], w[2h + 1 + 4 k2])
  const float2 bt0 = make_float2(b, b * L[0][1]);
  const float2 bt1 = make_float2(b * L[0][2], b * L[0][3]);
  float2 w2[8];
  w2[0] = bt0;
  w2[1] = bt1;
#pragma unroll
  for (int k2 = 1; k2 < 4; ++k2) {
    const float2 t = f2b(L[1][k2]);
    w2[2 * k2] = __fmul2_rn(bt0, t);
    w2[2 * k2 + 1] = __fmul2_rn(bt1, t);
  }
#pragma unroll
  for (int q = 0; q < 8; ++q) acc2[q] = __fadd2_rn(acc2[q], w2[q]);  // k3 = 0: T0 = 1
#pragma unroll
  for (int k3 = 1; k3 < 4; ++k3) {
    const float2 t = f2b(L[2][k3]);
#pragma unroll
    for (int q = 0; q < 8; ++q) acc2[q + 8 * k3] = __ffma2_rn(w2[q], t, acc2[q + 8 * k3]);
  }
}

// L2T: u2 holds the 64 Chebyshev coefficients of the box as 32 pairs in the order
// u2[(k2 + 4 h) * 4 + k1] = (u[k1 + 4 k2 + 16 (2h)], u[k1 + 4 k2 + 16 (2h + 1)])  (h = 0, 1):
// rows k3 and k3 + 1 of the same (k1, k2) share a pair (l2t_pair_index below lays U out so).
__device__ __forceinline__ float l2t_contract_d3p4_x2(const float (&L)[3][4], const float2 (&u2)[32]) {
  float2 t2[8];  // t[k2 + 4 k3] = sum_k1 T1[k1] u[..], pairs (k3 = 2h, 2h + 1) at t2[k2 + 4h]
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    float2 a = u2[r * 4];
#pragma unroll
    for (int k1 = 1; k1 < 4; ++k1) a = __ffma2_rn(f2b(L[0][k1]), u2[r * 4 + k1], a);
    t2[r] = a;
  }
  float2 s2[2];  // s[k3] = sum_k2 T2[k2] t[k2 + 4 k3], pairs (2h, 2h + 1)
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    float2 a = t2[4 * h];
#pragma unroll
    for (int k2 = 1; k2 < 4; ++k2) a = __ffma2_rn(f2b(L[1][k2]), t2[k2 + 4 * h], a);
    s2[h] = a;
  }
  // v = T3[0] s0 + T3[1] s1 + T3[2] s2 + T3[3] s3  (T3[0] = 1)
  const float2 v2 = __ffma2_rn(make_float2(L[2][2], L[2][3]), s2[1], __fmul2_rn(make_float2(1.f, L[2][1]), s2[0]));
  return v2.x + v2.y;
}
// position of coefficient k (= k1 + 4 k2 + 16 k3) in the pair layout of l2t_contract_d3p4_x2,
// as a float index into the 64 floats of u2
__host__ __device__ __forceinline__ int l2t_pair_index(int k) {
  const int k1 = k & 3, k2 = (k >> 2) & 3, k3 = k >> 4;
  return (((k2 + 4 * (k3 >> 1)) * 4 + k1) << 1) | (k3 & 1);
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
