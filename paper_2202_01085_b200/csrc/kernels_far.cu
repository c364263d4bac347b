// Far-field kernels for sm_100a: S2M (v1 = L_Y b), M2L (v2 = K v1), L2T (v += L_X^T v2).
//
// Paper: Sec. 3 "Interpolating k(x,y)" and Fig. 4;
// Chebyshev nodes of the 2nd kind; App. E Prop. 2 costs.
// B200 design:
//  * S2M/L2T work on box-sorted SoA coordinates in chunks of <= FAR_CHUNK points of one
//    box; the 1-D Lagrange weights (product form of PAPER.md:139, the same polynomial as
//    the barycentric form of App. C) and the tensor products live in registers; the
//    m = P^D accumulators are registers, reduced across the CTA, then across chunks in
//    fp64 in a fixed order (deterministic).
//  * M2L uses the separability of the Gaussian: K(nodes_p, nodes_q) = (x)_d T_d, with
//    T_d[k][j] = exp(-(Delta_d + l/2 (s_k - s_j))^2 / (2 gamma^2)) tabulated per level and
//    per integer box offset (on the device), applied as D mode products (D P^{D+1} FMAs
//    per pair instead of P^{2D}); fp64 accumulation over the interaction list.
#include <cuda_runtime.h>
#include <stdint.h>
#include <cstdlib>

#include "f3m_internal.h"

namespace f3m {

template <int P, int D>
struct IPow { static constexpr int value = P * IPow<P, D - 1>::value; };
template <int P>
struct IPow<P, 0> { static constexpr int value = 1; };

// 1-D Lagrange weights at tau (product form with precomputed 1/prod(s_k - s_j))
template <int P>
__device__ __forceinline__ void lagrange(float tau, const NodeConsts& nc, float (&L)[P]) {
  float dl[P];
#pragma unroll
  for (int k = 0; k < P; ++k) dl[k] = tau - nc.s[k];
  float acc = 1.f;
#pragma unroll
  for (int k = 0; k < P; ++k) { L[k] = acc; acc *= dl[k]; }
  acc = 1.f;
#pragma unroll
  for (int k = P - 1; k >= 0; --k) { L[k] *= acc * nc.c[k]; acc *= dl[k]; }
}

// Chebyshev polynomials T_0..T_{P-1} (the sorted kernels accumulate Chebyshev moments and
// evaluate Chebyshev coefficients; launch_cheb_transform converts to / from the nodal
// Lagrange values of Sec. 3 exactly, as in the tile-local kernels)
template <int P>
__device__ __forceinline__ void cheb_t(float tau, float (&T)[P]) {
  T[0] = 1.f;
  if constexpr (P > 1) T[1] = tau;
  const float t2 = tau + tau;
#pragma unroll
  for (int k = 2; k < P; ++k) T[k] = fmaf(t2, T[k - 1], -T[k - 2]);
}

template <int D, int P, bool CHEB>
__device__ __forceinline__ void point_weights(const float* __restrict__ xs, int64_t n, int64_t i, const BoxGeom& g,
                                              const NodeConsts& nc, float (&L)[D][P]) {
#pragma unroll
  for (int d = 0; d < D; ++d) {
    const float x = __ldg(xs + (int64_t)d * n + i);
    const float tau = fmaf(__fsub_rn(__fsub_rn(x, g.lo_hi[d]), g.lo_lo[d]), g.scale, -1.f);
    if constexpr (CHEB) cheb_t<P>(tau, L[d]);
    else lagrange<P>(tau, nc, L[d]);
  }
}

// the same from coordinates already in registers (software-pipelined loops)
template <int D, int P, bool CHEB>
__device__ __forceinline__ void point_weights_x(const float (&x)[D], const BoxGeom& g, const NodeConsts& nc,
                                                float (&L)[D][P]) {
#pragma unroll
  for (int d = 0; d < D; ++d) {
    const float tau = fmaf(__fsub_rn(__fsub_rn(x[d], g.lo_hi[d]), g.lo_lo[d]), g.scale, -1.f);
    if constexpr (CHEB) cheb_t<P>(tau, L[d]);
    else lagrange<P>(tau, nc, L[d]);
  }
}

// ---------------------------------------------------------------------------------------
// S2M: partials[chunk][k] = sum_{y in chunk} b_y prod_d T_{k_d}(tau_{y,d})  (Chebyshev moments)
// ---------------------------------------------------------------------------------------
template <int D, int P>
__global__ void __launch_bounds__(FAR_THREADS) k_s2m(const float* __restrict__ xs, const float* __restrict__ bs,
                                                     int64_t n, const BoxGeom* __restrict__ boxes,
                                                     const Chunk* __restrict__ chunks, NodeConsts nc,
                                                     float* __restrict__ partials) {
  constexpr int M = IPow<P, D>::value;
  constexpr int MP = M / P;
  const Chunk ch = chunks[blockIdx.x];
  const BoxGeom g = boxes[ch.box];
  float acc[M];
#pragma unroll
  for (int k = 0; k < M; ++k) acc[k] = 0.f;
  const int64_t end = ch.start + ch.len;
  // software pipeline: the next point's coordinates and weight are loaded before the current
  // point's products (one CTA per SM at these register counts: the loads' latency was exposed)
  float xn[D], bn;
  auto ld = [&](int64_t ii) {
    const bool ok = ii < end;
    const int64_t jj = ok ? ii : ch.start;
#pragma unroll
    for (int d = 0; d < D; ++d) xn[d] = __ldg(xs + (int64_t)d * n + jj);
    bn = __ldg(bs + jj);
  };
  ld(ch.start + threadIdx.x);
  for (int64_t i = ch.start + threadIdx.x; i < end; i += FAR_THREADS) {
    float x[D];
#pragma unroll
    for (int d = 0; d < D; ++d) x[d] = xn[d];
    const float bw = bn;
    ld(i + FAR_THREADS);
    float L[D][P];
    point_weights_x<D, P, true>(x, g, nc, L);
    float w[MP];
    w[0] = bw;
    // tensor product over dimensions 0..D-2 (dimension 0 fastest)
#pragma unroll
    for (int d = 0; d < D - 1; ++d) {
      const int len = (d == 0) ? 1 : (d == 1 ? P : (d == 2 ? P * P : (d == 3 ? P * P * P : (d == 4 ? P * P * P * P : P * P * P * P * P))));
#pragma unroll
      for (int k = P - 1; k >= 0; --k)
#pragma unroll
        for (int j = 0; j < len; ++j) w[j + len * k] = w[j] * L[d][k];
    }
#pragma unroll
    for (int k = 0; k < P; ++k)
#pragma unroll
      for (int j = 0; j < MP; ++j) acc[j + MP * k] = fmaf(w[j], L[D - 1][k], acc[j + MP * k]);
  }
  // CTA reduction
  __shared__ float red[FAR_THREADS / 32][M];
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < M; ++k) {
    float v = acc[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[wp][k] = v;
  }
  __syncthreads();
  for (int k = threadIdx.x; k < M; k += FAR_THREADS) {
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < FAR_THREADS / 32; ++j) s += red[j][k];
    partials[(int64_t)blockIdx.x * M + k] = s;
  }
}

// W[box][k] = sum over the box's chunks (fixed order, fp64)
__global__ void k_chunk_reduce(const float* __restrict__ partials, const int32_t* __restrict__ chunk_ptr,
                               int32_t nboxes, int m, double* __restrict__ W) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)nboxes * m) return;
  const int32_t b = (int32_t)(e / m);
  const int k = (int)(e - (int64_t)b * m);
  double s = 0.0;
  for (int32_t c = chunk_ptr[b]; c < chunk_ptr[b + 1]; ++c) s += (double)partials[(int64_t)c * m + k];
  W[e] = s;
}

// ---------------------------------------------------------------------------------------
// L2T: vs[x] += sum_k prod_d L_{k_d}(tau_{x,d}) U[box][k]  (nodal locals, Lagrange basis)
// ---------------------------------------------------------------------------------------
template <int D, int P>
__global__ void __launch_bounds__(FAR_THREADS) k_l2t(const float* __restrict__ xs, int64_t n,
                                                     const BoxGeom* __restrict__ boxes,
                                                     const Chunk* __restrict__ chunks, NodeConsts nc,
                                                     const double* __restrict__ U, float* __restrict__ vs) {
  constexpr int M = IPow<P, D>::value;
  constexpr int MP = M / P;
  const Chunk ch = chunks[blockIdx.x];
  const BoxGeom g = boxes[ch.box];
  __shared__ float su[M];
  for (int k = threadIdx.x; k < M; k += FAR_THREADS) su[k] = (float)U[(int64_t)ch.box * M + k];
  __syncthreads();
  float u[M];
#pragma unroll
  for (int k = 0; k < M; ++k) u[k] = su[k];
  const int64_t end = ch.start + ch.len;
  float xn[D];  // software pipeline (as k_s2m)
  auto ld = [&](int64_t ii) {
    const int64_t jj = ii < end ? ii : ch.start;
#pragma unroll
    for (int d = 0; d < D; ++d) xn[d] = __ldg(xs + (int64_t)d * n + jj);
  };
  ld(ch.start + threadIdx.x);
  for (int64_t i = ch.start + threadIdx.x; i < end; i += FAR_THREADS) {
    float x[D];
#pragma unroll
    for (int d = 0; d < D; ++d) x[d] = xn[d];
    ld(i + FAR_THREADS);
    float L[D][P];
    point_weights_x<D, P, false>(x, g, nc, L);
    float t[MP];
#pragma unroll
    for (int r = 0; r < MP; ++r) {
      float s = 0.f;
#pragma unroll
      for (int k = 0; k < P; ++k) s = fmaf(L[0][k], u[k + P * r], s);
      t[r] = s;
    }
#pragma unroll
    for (int d = 1; d < D; ++d) {
      const int len = MP / ((d == 1) ? P : (d == 2 ? P * P : (d == 3 ? P * P * P : (d == 4 ? P * P * P * P : (d == 5 ? P * P * P * P * P : P * P * P * P * P * P)))));
#pragma unroll
      for (int r = 0; r < len; ++r) {
        float s = 0.f;
#pragma unroll
        for (int k = 0; k < P; ++k) s = fmaf(L[d][k], t[k + P * r], s);
        t[r] = s;
      }
    }
    vs[i] += t[0];
  }
}

// ---------------------------------------------------------------------------------------
// M2L tables: tables[d][idx][k][j] = exp(-(Delta_d(idx) + l/2 (s_k - s_j))^2 / (2 gamma^2)),
// Delta_d(idx) = delta0[d] + idx * l  (= c_p - c_q along d)
// ---------------------------------------------------------------------------------------
template <int P, int D>
struct IPowFar { static constexpr int value = P * IPowFar<P, D - 1>::value; };
template <int P>
struct IPowFar<P, 0> { static constexpr int value = 1; };
__host__ __device__ constexpr int ipow_far(int p, int d) { return d == 0 ? 1 : p * ipow_far(p, d - 1); }

struct Nodes64 { double s[16]; };
struct DimInfo { double delta0[F3M_MAXD]; int32_t range[F3M_MAXD]; };

__global__ void k_m2l_tables(int D, int P, DimInfo di, double l, double gamma, Nodes64 nd, float* __restrict__ tables,
                             int table_stride) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int per = table_stride;
  if (e >= (int64_t)D * per) return;
  const int d = (int)(e / per);
  const int r = (int)(e - (int64_t)d * per);
  const int idx = r / (P * P);
  const int kj = r - idx * P * P;
  const int k = kj / P, j = kj - k * P;
  if (idx >= di.range[d]) { tables[e] = 0.f; return; }
  const double diff = (di.delta0[d] + (double)idx * l) + (l / 2.0) * (nd.s[k] - nd.s[j]);
  tables[e] = (float)exp(-(diff * diff) / (2.0 * gamma * gamma));
}

// One warp per target box (deterministic: its pairs in list order), no block barriers: per
// pair the source charges go through the D separable factor contractions in two per-warp
// shared buffers (__syncwarp between dimensions), the result is added to the box's fp64
// locals in a per-warp shared accumulator (the potential at a node is a long sum with
// cancellation).  Work per pair: D m P FMAs (separable).
__global__ void k_m2l(int D, int P, int m, int ntgt, const int32_t* __restrict__ csr_ptr,
                      const int32_t* __restrict__ src, const uint64_t* __restrict__ offs,
                      const float* __restrict__ tables, int table_stride, const float* __restrict__ W32,
                      double* __restrict__ U, int warps) {
  extern __shared__ __align__(16) unsigned char m2l_sm[];
  float* tbl = reinterpret_cast<float*>(m2l_sm);                        // [D][table_stride]
  const size_t tbytes = ((size_t)D * table_stride * 4 + 15) / 16 * 16;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* wb = m2l_sm + tbytes + (size_t)w * (size_t)m * 16;
  double* acc = reinterpret_cast<double*>(wb);                          // [m]
  float* bufA = reinterpret_cast<float*>(wb + (size_t)m * 8);          // [m]
  float* bufB = bufA + m;                                               // [m]
  for (int e = threadIdx.x; e < D * table_stride; e += blockDim.x) tbl[e] = tables[e];
  __syncthreads();
  for (int tgt = blockIdx.x * warps + w; tgt < ntgt; tgt += gridDim.x * warps) {
    for (int k = lane; k < m; k += 32) acc[k] = 0.0;
    for (int32_t p = csr_ptr[tgt]; p < csr_ptr[tgt + 1]; ++p) {
      const int32_t s = src[p];
      const uint64_t o = offs[p];
      const float* Ws = W32 + (int64_t)s * m;
      for (int k = lane; k < m; k += 32) bufA[k] = __ldg(Ws + k);
      __syncwarp();
      float* cur = bufA;
      float* nxt = bufB;
      int stride = 1;
      for (int d = 0; d < D; ++d) {
        const int idx = (int)((o >> (8 * d)) & 0xffu);
        const float* T = tbl + d * table_stride + idx * P * P;
        for (int k = lane; k < m; k += 32) {
          const int kd = (k / stride) % P;
          const int base = k - kd * stride;
          float sacc = 0.f;
          for (int j = 0; j < P; ++j) sacc = fmaf(T[kd * P + j], cur[base + j * stride], sacc);
          nxt[k] = sacc;
        }
        __syncwarp();
        float* tmp = cur;
        cur = nxt;
        nxt = tmp;
        stride *= P;
      }
      for (int k = lane; k < m; k += 32) acc[k] += (double)cur[k];
      __syncwarp();
    }
    for (int k = lane; k < m; k += 32) U[(int64_t)tgt * m + k] = acc[k];
    __syncwarp();
  }
}

// Compile-time (D, P) variant of k_m2l for m = P^D <= 1024: locals accumulate in fp64
// registers (lane owns k = lane + 32 i), the per-dimension index arithmetic is constant-folded
// and the P-term contractions are unrolled.
template <int D, int P>
__global__ void __launch_bounds__(256) k_m2l_t(int ntgt, const int32_t* __restrict__ csr_ptr,
                                               const int32_t* __restrict__ src, const uint64_t* __restrict__ offs,
                                               const float* __restrict__ tables, int table_stride,
                                               const float* __restrict__ W32, double* __restrict__ U) {
  constexpr int M = IPowFar<P, D>::value;
  constexpr int V = (M + 31) / 32;
  constexpr int WARPS = 8;
  extern __shared__ __align__(16) unsigned char m2l_sm[];
  float* tbl = reinterpret_cast<float*>(m2l_sm);
  const size_t tbytes = ((size_t)D * table_stride * 4 + 15) / 16 * 16;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* bufA = reinterpret_cast<float*>(m2l_sm + tbytes) + (size_t)w * 2 * M;
  float* bufB = bufA + M;
  for (int e = threadIdx.x; e < D * table_stride; e += blockDim.x) tbl[e] = tables[e];
  __syncthreads();
  for (int tgt = blockIdx.x * WARPS + w; tgt < ntgt; tgt += gridDim.x * WARPS) {
    double acc[V];
#pragma unroll
    for (int i = 0; i < V; ++i) acc[i] = 0.0;
    const int32_t pend = csr_ptr[tgt + 1];
    for (int32_t p = csr_ptr[tgt]; p < pend; ++p) {
      const int32_t s = src[p];
      const uint64_t o = offs[p];
      const float* Ws = W32 + (int64_t)s * M;
#pragma unroll
      for (int i = 0; i < V; ++i)
        if (M % 32 == 0 || lane + 32 * i < M) bufA[lane + 32 * i] = __ldg(Ws + lane + 32 * i);
      __syncwarp();
      float* cur = bufA;
      float* nxt = bufB;
      float last[V];
      if constexpr (M / P >= 64 && (M / P) % 32 == 0) {
        // column form: a lane takes whole columns (the P values that differ only in digit d),
        // with the P x P factor in registers -- P loads and P^2 FMAs per column instead of
        // 2 P shared loads per output.  Same products and summation order as below.
        constexpr int C = M / P / 32;
#pragma unroll
        for (int d = 0; d < D; ++d) {
          const int stride = ipow_far(P, d);
          const float* Tg = tbl + d * table_stride + (int)((o >> (8 * d)) & 0xffu) * P * P;
          float Tr[P][P];
#pragma unroll
          for (int a2 = 0; a2 < P; ++a2)
#pragma unroll
            for (int j = 0; j < P; ++j) Tr[a2][j] = Tg[a2 * P + j];
#pragma unroll
          for (int cc = 0; cc < C; ++cc) {
            const int c = lane + 32 * cc;
            const int base = (c % stride) + (c / stride) * stride * P;
            float in[P];
            if (P == 4 && d == 0) {  // contiguous column: one 16-byte access (scalar: 4-way conflicts)
              const float4 q = *reinterpret_cast<const float4*>(cur + base);
              in[0] = q.x; in[1 % P] = q.y; in[2 % P] = q.z; in[3 % P] = q.w;
            } else {
#pragma unroll
              for (int j = 0; j < P; ++j) in[j] = cur[base + j * stride];
            }
            float o[P];
#pragma unroll
            for (int kd = 0; kd < P; ++kd) {
              float sacc = 0.f;
#pragma unroll
              for (int j = 0; j < P; ++j) sacc = fmaf(Tr[kd][j], in[j], sacc);
              o[kd] = sacc;
            }
            if (P == 4 && d == 0) {
              *reinterpret_cast<float4*>(nxt + base) = make_float4(o[0], o[1 % P], o[2 % P], o[3 % P]);
            } else {
#pragma unroll
              for (int kd = 0; kd < P; ++kd) nxt[base + kd * stride] = o[kd];
            }
          }
          __syncwarp();
          float* tmp = cur;
          cur = nxt;
          nxt = tmp;
        }
#pragma unroll
        for (int i = 0; i < V; ++i) last[i] = cur[lane + 32 * i];
      } else {
#pragma unroll
      for (int d = 0; d < D; ++d) {
        const int stride = IPowFar<P, 0>::value * ipow_far(P, d);
        const float* T = tbl + d * table_stride + (int)((o >> (8 * d)) & 0xffu) * P * P;
#pragma unroll
        for (int i = 0; i < V; ++i) {
          const int k = lane + 32 * i;
          if (M % 32 == 0 || k < M) {
            const int kd = (k / stride) % P;
            const int base = k - kd * stride;
            float sacc = 0.f;
#pragma unroll
            for (int j = 0; j < P; ++j) sacc = fmaf(T[kd * P + j], cur[base + j * stride], sacc);
            if (d + 1 < D) nxt[k] = sacc;
            else last[i] = sacc;
          }
        }
        if (d + 1 < D) {
          __syncwarp();
          float* tmp = cur;
          cur = nxt;
          nxt = tmp;
        }
      }
      }
#pragma unroll
      for (int i = 0; i < V; ++i)
        if (M % 32 == 0 || lane + 32 * i < M) acc[i] += (double)last[i];
      __syncwarp();
    }
#pragma unroll
    for (int i = 0; i < V; ++i)
      if (M % 32 == 0 || lane + 32 * i < M) U[(int64_t)tgt * M + lane + 32 * i] = acc[i];
  }
}

// P = 2, D >= 5 (m = 2^D >= 32): one warp per target box, the m values of a pair in
// registers (lane owns k = lane V + i, V = m / 32): dimensions below log2 V contract inside a
// lane, the others pair lanes through one __shfl_xor each -- no shared memory traffic per pair
// besides the 2 x 2 factor of each dimension.  fp32 partial sums over up to 16 pairs, folded into
// fp64 locals; pairs in list order (deterministic).
template <int D>
__global__ void __launch_bounds__(256) k_m2l_p2(int ntgt, const int32_t* __restrict__ csr_ptr,
                                                const int32_t* __restrict__ src, const uint64_t* __restrict__ offs,
                                                const float* __restrict__ tables, int table_stride,
                                                const float* __restrict__ W32, double* __restrict__ U) {
  constexpr int M = 1 << D;
  constexpr int V = M / 32;
  constexpr int LB = D - 5;  // dimensions inside a lane
  constexpr int WARPS = 8;
  extern __shared__ __align__(16) float tsm2[];
  for (int e = threadIdx.x; e < D * table_stride; e += blockDim.x) tsm2[e] = tables[e];
  __syncthreads();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int tgt = blockIdx.x * WARPS + w; tgt < ntgt; tgt += gridDim.x * WARPS) {
    double acc[V];
    float part[V];  // fp32 partial sums over up to 16 pairs, folded into the fp64 locals
#pragma unroll
    for (int i = 0; i < V; ++i) { acc[i] = 0.0; part[i] = 0.f; }
    int cnt = 0;
    const int32_t pbeg = csr_ptr[tgt], pend = csr_ptr[tgt + 1];
    // the next pair's charges are loaded while this pair is contracted
    float cn[V];
    if (pbeg < pend) {
      const float* Ws = W32 + (int64_t)src[pbeg] * M + lane * V;
#pragma unroll
      for (int i = 0; i < V; ++i) cn[i] = __ldg(Ws + i);
    }
    for (int32_t p = pbeg; p < pend; ++p) {
      const uint64_t o = offs[p];
      float c[V];
#pragma unroll
      for (int i = 0; i < V; ++i) c[i] = cn[i];
      if (p + 1 < pend) {
        const float* Ws = W32 + (int64_t)src[p + 1] * M + lane * V;
#pragma unroll
        for (int i = 0; i < V; ++i) cn[i] = __ldg(Ws + i);
      }
#pragma unroll
      for (int d = 0; d < D; ++d) {
        const float4 t = *reinterpret_cast<const float4*>(tsm2 + d * table_stride + (int)((o >> (8 * d)) & 0xffu) * 4);
        // t = (T[0][0], T[0][1], T[1][0], T[1][1])
        if (d < LB) {
#pragma unroll
          for (int i = 0; i < V; ++i)
            if (!((i >> d) & 1)) {
              const float c0 = c[i], c1 = c[i | (1 << d)];
              c[i] = fmaf(t.x, c0, t.y * c1);
              c[i | (1 << d)] = fmaf(t.z, c0, t.w * c1);
            }
        } else {
          // lane pair (lo, hi): lo keeps T[0][0] own + T[0][1] other, hi T[1][1] own + T[1][0]
          // other -- the row is chosen once per dimension, not per value
          const int sh = 1 << (d - LB);
          const bool hi = (lane & sh) != 0;
          const float a_own = hi ? t.w : t.x, a_oth = hi ? t.z : t.y;
#pragma unroll
          for (int i = 0; i < V; ++i) {
            const float q = __shfl_xor_sync(0xffffffffu, c[i], sh);
            c[i] = fmaf(a_own, c[i], a_oth * q);
          }
        }
      }
#pragma unroll
      for (int i = 0; i < V; ++i) part[i] += c[i];
      if (++cnt == 16) {
#pragma unroll
        for (int i = 0; i < V; ++i) { acc[i] += (double)part[i]; part[i] = 0.f; }
        cnt = 0;
      }
    }
#pragma unroll
    for (int i = 0; i < V; ++i) acc[i] += (double)part[i];
#pragma unroll
    for (int i = 0; i < V; ++i) U[(int64_t)tgt * M + lane * V + i] = acc[i];
  }
}

// P = 2, D >= 5, four pairs per warp step: lanes 8g .. 8g+7 take pair g of the step and own
// V = 2^D / 8 node values each (k = j V + i, j = lane % 8): dimensions 0 .. D-4 contract inside
// a lane with packed FP32x2 arithmetic (FMUL2 / FFMA2 on value pairs), the top three across
// the eight lanes of the group (one __shfl_xor per value).  Per pair this issues about half the
// instructions of k_m2l_p2 (which spends 5 shuffle levels on 4 values per lane).  fp32 partial
// sums per group over up to 16 steps, folded into fp64, the four groups summed at the end
// (fixed order: deterministic).
template <int D>
__global__ void __launch_bounds__(256) k_m2l_p2x(int ntgt, const int32_t* __restrict__ csr_ptr,
                                                 const int32_t* __restrict__ src, const uint64_t* __restrict__ offs,
                                                 const float* __restrict__ tables, int table_stride,
                                                 const float* __restrict__ W32, double* __restrict__ U) {
  constexpr int M = 1 << D;
  constexpr int V = M / 8;
  constexpr int LB = D - 3;  // dimensions inside a lane
  constexpr int WARPS = 8;
  static_assert(V % 4 == 0, "D >= 5");
  extern __shared__ __align__(16) float tsm3[];
  for (int e = threadIdx.x; e < D * table_stride; e += blockDim.x) tsm3[e] = tables[e];
  __syncthreads();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 3, j = lane & 7;
  for (int tgt = blockIdx.x * WARPS + w; tgt < ntgt; tgt += gridDim.x * WARPS) {
    double acc[V];
    float2 part[V / 2];
#pragma unroll
    for (int i = 0; i < V; ++i) acc[i] = 0.0;
#pragma unroll
    for (int i = 0; i < V / 2; ++i) part[i] = make_float2(0.f, 0.f);
    int cnt = 0;
    const int32_t pbeg = csr_ptr[tgt], pend = csr_ptr[tgt + 1];
    for (int32_t p0 = pbeg; p0 < pend; p0 += 4) {
      // a group without a pair this step recomputes the last pair and discards it: every lane
      // runs the same shuffles
      const int32_t p = min(p0 + g, pend - 1);
      const bool valid = p0 + g < pend;
      {
        const uint64_t o = offs[p];
        float2 c[V / 2];
        const float4* Ws = reinterpret_cast<const float4*>(W32 + (int64_t)src[p] * M + j * V);
#pragma unroll
        for (int q = 0; q < V / 4; ++q) {
          const float4 v4 = __ldg(Ws + q);
          c[2 * q] = make_float2(v4.x, v4.y);
          c[2 * q + 1] = make_float2(v4.z, v4.w);
        }
#pragma unroll
        for (int d = 0; d < D; ++d) {
          const float4 t = *reinterpret_cast<const float4*>(tsm3 + d * table_stride + (int)((o >> (8 * d)) & 0xffu) * 4);
          // t = (T[0][0], T[0][1], T[1][0], T[1][1])
          if (d == 0) {  // within each value pair: (c0, c1) -> (T00 c0 + T01 c1, T10 c0 + T11 c1)
#pragma unroll
            for (int q = 0; q < V / 2; ++q)
              c[q] = __ffma2_rn(make_float2(t.x, t.z), make_float2(c[q].x, c[q].x),
                                __fmul2_rn(make_float2(t.y, t.w), make_float2(c[q].y, c[q].y)));
          } else if (d < LB) {  // value pairs q and q + 2^{d-1}
            const int sq = 1 << (d - 1);
#pragma unroll
            for (int q = 0; q < V / 2; ++q)
              if (!((q / sq) & 1)) {
                const float2 c0 = c[q], c1 = c[q + sq];
                c[q] = __ffma2_rn(make_float2(t.x, t.x), c0, __fmul2_rn(make_float2(t.y, t.y), c1));
                c[q + sq] = __ffma2_rn(make_float2(t.z, t.z), c0, __fmul2_rn(make_float2(t.w, t.w), c1));
              }
          } else {  // across the group's lanes
            const int sh = 1 << (d - LB);
            const bool hi = (j & sh) != 0;
            const float a_own = hi ? t.w : t.x, a_oth = hi ? t.z : t.y;
#pragma unroll
            for (int q = 0; q < V / 2; ++q) {
              const float2 oth = make_float2(__shfl_xor_sync(0xffffffffu, c[q].x, sh), __shfl_xor_sync(0xffffffffu, c[q].y, sh));
              c[q] = __ffma2_rn(make_float2(a_own, a_own), c[q], __fmul2_rn(make_float2(a_oth, a_oth), oth));
            }
          }
        }
        if (valid)
#pragma unroll
          for (int q = 0; q < V / 2; ++q) part[q] = __fadd2_rn(part[q], c[q]);
      }
      if (++cnt == 16) {
#pragma unroll
        for (int q = 0; q < V / 2; ++q) {
          acc[2 * q] += (double)part[q].x;
          acc[2 * q + 1] += (double)part[q].y;
          part[q] = make_float2(0.f, 0.f);
        }
        cnt = 0;
      }
    }
#pragma unroll
    for (int q = 0; q < V / 2; ++q) {
      acc[2 * q] += (double)part[q].x;
      acc[2 * q + 1] += (double)part[q].y;
    }
    // the four groups hold partial sums of the same node values: g0 + g1, then + (g2 + g3)
#pragma unroll
    for (int i = 0; i < V; ++i) {
      acc[i] += __shfl_xor_sync(0xffffffffu, acc[i], 8);
      acc[i] += __shfl_xor_sync(0xffffffffu, acc[i], 16);
    }
    if (g == 0)
#pragma unroll
      for (int i = 0; i < V; ++i) U[(int64_t)tgt * M + j * V + i] = acc[i];
  }
}

// P = 3, D >= 5 (m = 3^D): one warp per target box, 27 active lanes; lane owns the V = 3^{D-3}
// node values k = lane V + i, i.e. dimensions 0 .. D-4 inside a lane (3 x 3 factors applied to
// register triplets) and the top three dimensions across lanes (lane digit a of dimension d
// takes the two other lanes' values with two shuffles and applies row a of the 3 x 3 factor).
// fp32 partial sums over up to 16 pairs, folded into fp64 locals in shared memory (fixed pair
// order: deterministic).  Work per pair: D 3^{D+1} FMAs (separable).
template <int D>
__global__ void __launch_bounds__(256, 1) k_m2l_p3(int ntgt, const int32_t* __restrict__ csr_ptr,
                                                   const int32_t* __restrict__ src, const uint64_t* __restrict__ offs,
                                                   const float* __restrict__ tables, int table_stride,
                                                   const float* __restrict__ W32, double* __restrict__ U) {
  constexpr int M = IPowFar<3, D>::value;
  constexpr int V = M / 27;
  constexpr int LB = D - 3;  // dimensions inside a lane
  constexpr int WARPS = 8;
  constexpr int FLUSH = 16;
  extern __shared__ __align__(16) unsigned char p3_sm[];
  float* tsm = reinterpret_cast<float*>(p3_sm);
  const size_t tbytes = ((size_t)D * table_stride * 4 + 15) / 16 * 16;
  for (int e = threadIdx.x; e < D * table_stride; e += blockDim.x) tsm[e] = tables[e];
  __syncthreads();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* accw = reinterpret_cast<double*>(p3_sm + tbytes) + (size_t)w * M;
  const bool act = lane < 27;
  // lane digits of the cross-lane dimensions and the partner lanes
  int dig[3], src1[3], src2[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const int s = c == 0 ? 1 : (c == 1 ? 3 : 9);
    const int a = act ? (lane / s) % 3 : 0;
    dig[c] = a;
    src1[c] = act ? lane + (((a + 1) % 3) - a) * s : lane;
    src2[c] = act ? lane + (((a + 2) % 3) - a) * s : lane;
  }
  for (int tgt = blockIdx.x * WARPS + w; tgt < ntgt; tgt += gridDim.x * WARPS) {
    for (int e = lane; e < M; e += 32) accw[e] = 0.0;
    float acc[V];
#pragma unroll
    for (int i = 0; i < V; ++i) acc[i] = 0.f;
    int cnt = 0;
    auto flush = [&]() {
      __syncwarp();
      if (act)
#pragma unroll
        for (int i = 0; i < V; ++i) { accw[lane * V + i] += (double)acc[i]; acc[i] = 0.f; }
      __syncwarp();
    };
    const int32_t pend = csr_ptr[tgt + 1];
    for (int32_t p = csr_ptr[tgt]; p < pend; ++p) {
      const uint64_t o = offs[p];
      const float* Ws = W32 + (int64_t)src[p] * M + (act ? lane * V : 0);
      float c[V];
#pragma unroll
      for (int i = 0; i < V; ++i) c[i] = __ldg(Ws + i);
#pragma unroll
      for (int d = 0; d < LB; ++d) {
        const float* T = tsm + d * table_stride + (int)((o >> (8 * d)) & 0xffu) * 9;  // T[k][j]
        float t[9];
#pragma unroll
        for (int e = 0; e < 9; ++e) t[e] = T[e];
        const int st = d == 0 ? 1 : (d == 1 ? 3 : (d == 2 ? 9 : (d == 3 ? 27 : 81)));
#pragma unroll
        for (int i = 0; i < V; ++i) {
          if ((i / st) % 3 != 0) continue;
          const float c0 = c[i], c1 = c[i + st], c2 = c[i + 2 * st];
          c[i] = fmaf(t[0], c0, fmaf(t[1], c1, t[2] * c2));
          c[i + st] = fmaf(t[3], c0, fmaf(t[4], c1, t[5] * c2));
          c[i + 2 * st] = fmaf(t[6], c0, fmaf(t[7], c1, t[8] * c2));
        }
      }
#pragma unroll
      for (int cd = 0; cd < 3; ++cd) {
        const int d = LB + cd;
        const float* T = tsm + d * table_stride + (int)((o >> (8 * d)) & 0xffu) * 9 + dig[cd] * 3;  // row a
        const int a = dig[cd];
        const float ta = T[a], t1 = T[(a + 1) % 3], t2 = T[(a + 2) % 3];
#pragma unroll
        for (int i = 0; i < V; ++i) {
          const float x1 = __shfl_sync(0xffffffffu, c[i], src1[cd]);
          const float x2 = __shfl_sync(0xffffffffu, c[i], src2[cd]);
          c[i] = fmaf(ta, c[i], fmaf(t1, x1, t2 * x2));
        }
      }
#pragma unroll
      for (int i = 0; i < V; ++i) acc[i] += c[i];
      if (++cnt == FLUSH) { flush(); cnt = 0; }
    }
    flush();
    if (act)
#pragma unroll
      for (int i = 0; i < V; ++i) U[(int64_t)tgt * M + lane * V + i] = accw[lane * V + i];
    __syncwarp();
  }
}

__global__ void k_to_f32(const double* __restrict__ a, int64_t n, float* __restrict__ b) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    b[i] = (float)a[i];
}

// ---------------------------------------------------------------------------------------
// Exact translations between levels (SURVEY 8(a) note 1; Sec. 3: Lagrange
// interpolation on P nodes reproduces polynomials of degree <= P-1, and a parent's basis
// function restricted to a child box is such a polynomial):
//   M2M  W_p[k] = sum_c sum_j prod_d T_{bit_d(c)}[k_d][j_d] W_c[j]
//   L2L  U_c[j] += sum_k prod_d T_{bit_d(c)}[k_d][j_d] U_p[k]
// with T_b[k][j] = L_k((s_j + 2b - 1) / 2) (child node j in the parent's local coordinate).
// fp64 throughout; one block per output box, separable contraction through shared memory.
// ---------------------------------------------------------------------------------------
struct TransMats { double T[2][16][16]; };

__device__ __forceinline__ void trans_apply(int D, int P, int m, const TransMats& tm, int child_bits, bool transpose,
                                            double* cur, double* nxt) {
  int stride = 1;
  for (int d = 0; d < D; ++d) {
    const int b = (child_bits >> d) & 1;
    for (int k = threadIdx.x; k < m; k += blockDim.x) {
      const int kd = (k / stride) % P;
      const int base = k - kd * stride;
      double acc = 0.0;
      for (int j = 0; j < P; ++j)
        acc += (transpose ? tm.T[b][j][kd] : tm.T[b][kd][j]) * cur[base + j * stride];
      nxt[k] = acc;
    }
    __syncthreads();
    double* t = cur; cur = nxt; nxt = t;
    stride *= P;
  }
  if (D & 1) {  // result must end in the first buffer
    for (int k = threadIdx.x; k < m; k += blockDim.x) nxt[k] = cur[k];
    __syncthreads();
  }
}

// W_parent (all parents of level t) from W_child (all boxes of level t + 1).  Block (p, g) of
// G blocks per parent sums the children g, g + G, ... of parent p into Wp[p G + g] (G = 1: the
// parent row itself; G > 1: partial rows summed by k_m2m_sum in a fixed order -- few parents
// with many children, e.g. D = 7: 128 parents of 128 children, would leave the GPU idle).
__global__ void k_m2m(int D, int P, int m, TransMats tm, const int32_t* __restrict__ child0,
                      const int32_t* __restrict__ nchild, const int32_t* __restrict__ child_bits,
                      const double* __restrict__ Wc, double* __restrict__ Wp, int G) {
  extern __shared__ double tsm[];
  double* a = tsm;
  double* b = tsm + m;
  const int p = blockIdx.x / G, g = blockIdx.x - p * G;
  double acc[8];
#pragma unroll
  for (int r = 0; r < 8; ++r) acc[r] = 0.0;
  for (int c = child0[p] + g; c < child0[p] + nchild[p]; c += G) {
    for (int k = threadIdx.x; k < m; k += blockDim.x) a[k] = Wc[(int64_t)c * m + k];
    __syncthreads();
    trans_apply(D, P, m, tm, child_bits[c], false, a, b);
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const int k = threadIdx.x + r * blockDim.x;
      if (k < m) acc[r] += a[k];
    }
    __syncthreads();
  }
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int k = threadIdx.x + r * blockDim.x;
    if (k < m) Wp[(int64_t)blockIdx.x * m + k] = acc[r];
  }
}

__global__ void k_m2m_sum(const double* __restrict__ part, int nparents, int G, int m, double* __restrict__ Wp) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)nparents * m) return;
  const int64_t p = e / m, k = e - p * m;
  double s = 0.0;
  for (int g = 0; g < G; ++g) s += part[(p * G + g) * m + k];
  Wp[e] = s;
}

// U_child (all boxes of level t + 1) += L2L(U_parent)
__global__ void k_l2l(int D, int P, int m, TransMats tm, const int32_t* __restrict__ parent,
                      const int32_t* __restrict__ child_bits, const double* __restrict__ Up, double* __restrict__ Uc) {
  extern __shared__ double tsm[];
  double* a = tsm;
  double* b = tsm + m;
  const int c = blockIdx.x;
  const int p = parent[c];
  for (int k = threadIdx.x; k < m; k += blockDim.x) a[k] = Up[(int64_t)p * m + k];
  __syncthreads();
  trans_apply(D, P, m, tm, child_bits[c], true, a, b);
  for (int k = threadIdx.x; k < m; k += blockDim.x) Uc[(int64_t)c * m + k] += a[k];
}

// rows: dst[r] = src[idx[r]] (gather) or dst[idx[r]] += src[r] (scatter-add; idx distinct)
__global__ void k_rows(const double* __restrict__ src, const int32_t* __restrict__ idx, int64_t rows, int m,
                       double* __restrict__ dst, int scatter_add) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < rows * m; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / m;
    const int k = (int)(e - r * m);
    if (scatter_add) dst[(int64_t)idx[r] * m + k] += src[e];
    else dst[e] = src[(int64_t)idx[r] * m + k];
  }
}

static TransMats trans_mats(int P) {
  TransMats tm{};
  const double pi = 3.14159265358979323846;
  double sn[16];
  for (int k = 0; k < P; ++k) sn[k] = cos((double)k * pi / (double)(P - 1));
  for (int b = 0; b < 2; ++b)
    for (int j = 0; j < P; ++j) {
      const double tau = (sn[j] + 2.0 * b - 1.0) / 2.0;
      for (int k = 0; k < P; ++k) {  // Lagrange basis L_k(tau), product form
        double v = 1.0;
        for (int q = 0; q < P; ++q)
          if (q != k) v *= (tau - sn[q]) / (sn[k] - sn[q]);
        tm.T[b][k][j] = v;
      }
    }
  return tm;
}

static int trans_threads(int m) {
  int bd = m < 32 ? 32 : (m > 256 ? 256 : m);
  if (bd < (m + 7) / 8) bd = (m + 7) / 8;  // k_m2m keeps <= 8 outputs per thread (m = 2187: 288 threads)
  return (bd + 31) / 32 * 32;
}

int m2m_split(int D, int nparents) {
  int G = 1;
  while (G < (1 << D) && (int64_t)nparents * G < 2 * 148) G *= 2;
  return G;
}

void launch_m2m(int D, int P, int m, int nparents, const int32_t* child0, const int32_t* nchild,
                const int32_t* child_bits, const double* Wc, double* Wp, double* scratch, cudaStream_t st) {
  if (nparents <= 0) return;
  const int G = scratch ? m2m_split(D, nparents) : 1;
  k_m2m<<<nparents * G, trans_threads(m), 2 * m * sizeof(double), st>>>(D, P, m, trans_mats(P), child0, nchild,
                                                                         child_bits, Wc, G > 1 ? scratch : Wp, G);
  if (G > 1) {
    const int64_t work = (int64_t)nparents * m;
    k_m2m_sum<<<(unsigned)((work + 255) / 256), 256, 0, st>>>(scratch, nparents, G, m, Wp);
  }
}

void launch_l2l(int D, int P, int m, int nchildren, const int32_t* parent, const int32_t* child_bits,
                const double* Up, double* Uc, cudaStream_t st) {
  if (nchildren <= 0) return;
  k_l2l<<<nchildren, trans_threads(m), 2 * m * sizeof(double), st>>>(D, P, m, trans_mats(P), parent, child_bits, Up, Uc);
}

void launch_rows(const double* src, const int32_t* idx, int64_t rows, int m, double* dst, bool scatter_add,
                 cudaStream_t st) {
  const int64_t work = rows * m;
  if (work <= 0) return;
  const int64_t want = (work + 255) / 256;
  k_rows<<<(unsigned)(want < 148 * 8 ? want : 148 * 8), 256, 0, st>>>(src, idx, rows, m, dst, scatter_add ? 1 : 0);
}

// ---------------------------------------------------------------------------------------
// dispatch over the register-tiled instantiations (m = P^D <= 128)
// ---------------------------------------------------------------------------------------
#define F3M_FAR_CASES(X) \
  X(1, 2) X(1, 3) X(1, 4) X(1, 5) X(1, 6) X(1, 7) X(1, 8) \
  X(2, 2) X(2, 3) X(2, 4) X(2, 5) X(2, 6) X(2, 7) X(2, 8) \
  X(3, 2) X(3, 3) X(3, 4) X(3, 5) \
  X(4, 2) X(4, 3) X(5, 2) X(6, 2) X(7, 2)

bool far_supported(int D, int P) {
#define X(d, p) if (D == d && P == p) return true;
  F3M_FAR_CASES(X)
#undef X
  return false;
}

void launch_s2m(int D, int P, const float* xs, const float* bs, int64_t n, const BoxGeom* boxes, const Chunk* chunks,
                int64_t nchunks, const NodeConsts& nc, float* partials, cudaStream_t st) {
  if (nchunks <= 0) return;
#define X(d, p) \
  if (D == d && P == p) { k_s2m<d, p><<<(unsigned)nchunks, FAR_THREADS, 0, st>>>(xs, bs, n, boxes, chunks, nc, partials); return; }
  F3M_FAR_CASES(X)
#undef X
}

void launch_l2t(int D, int P, const float* xs, int64_t n, const BoxGeom* boxes, const Chunk* chunks, int64_t nchunks,
                const NodeConsts& nc, const double* U, float* vs, cudaStream_t st) {
  if (nchunks <= 0) return;
#define X(d, p) \
  if (D == d && P == p) { k_l2t<d, p><<<(unsigned)nchunks, FAR_THREADS, 0, st>>>(xs, n, boxes, chunks, nc, U, vs); return; }
  F3M_FAR_CASES(X)
#undef X
}

void launch_chunk_reduce(const float* partials, const int32_t* chunk_ptr, int32_t nboxes, int m, double* W,
                         cudaStream_t st) {
  const int64_t work = (int64_t)nboxes * m;
  if (work <= 0) return;
  k_chunk_reduce<<<(unsigned)((work + 255) / 256), 256, 0, st>>>(partials, chunk_ptr, nboxes, m, W);
}

void launch_m2l_tables(int D, int P, const double* delta0, double l, const int32_t* range, double gamma,
                       const NodeConsts& nc, float* tables, int table_stride, cudaStream_t st) {
  (void)nc;
  DimInfo di{};
  for (int d = 0; d < D; ++d) { di.delta0[d] = delta0[d]; di.range[d] = range[d]; }
  Nodes64 nd{};
  const double pi = 3.14159265358979323846;
  for (int k = 0; k < P; ++k) nd.s[k] = cos((double)k * pi / (double)(P - 1));
  const int64_t work = (int64_t)D * table_stride;
  k_m2l_tables<<<(unsigned)((work + 255) / 256), 256, 0, st>>>(D, P, di, l, gamma, nd, tables, table_stride);
}

void launch_m2l(int D, int P, int32_t ntgt, const int32_t* csr_ptr, const int32_t* src, const uint64_t* offs,
                const float* tables, int table_stride, const float* W32, double* U, cudaStream_t st) {
  if (ntgt <= 0) return;
  int m = 1;
  for (int d = 0; d < D; ++d) m *= P;
  const size_t tbytes = ((size_t)D * table_stride * 4 + 15) / 16 * 16;
  if (P == 2 && D >= 5) {
#define P2_CASE(d)                                                                                        \
    if (D == d) {                                                                                         \
      if (tbytes > 48 * 1024) cudaFuncSetAttribute(k_m2l_p2x<d>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tbytes); \
      k_m2l_p2x<d><<<(ntgt + 7) / 8, 256, tbytes, st>>>(ntgt, csr_ptr, src, offs, tables, table_stride, W32, U); \
      return;                                                                                             \
    }
    P2_CASE(5) P2_CASE(6) P2_CASE(7)
#undef P2_CASE
  }
  if (P == 3 && D >= 5) {
#define P3_CASE(d)                                                                                          \
    if (D == d) {                                                                                           \
      const size_t smp3 = tbytes + (size_t)8 * m * 8;                                                       \
      cudaFuncSetAttribute(k_m2l_p3<d>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smp3);            \
      k_m2l_p3<d><<<(ntgt + 7) / 8, 256, smp3, st>>>(ntgt, csr_ptr, src, offs, tables, table_stride, W32, U); \
      return;                                                                                               \
    }
    P3_CASE(5) P3_CASE(6) P3_CASE(7)
#undef P3_CASE
  }
#define M2L_CASE(d, p)                                                                                        \
  if (D == d && P == p) {                                                                                     \
    const size_t smt = tbytes + (size_t)8 * 2 * m * 4;                                                        \
    if (smt > 48 * 1024) cudaFuncSetAttribute(k_m2l_t<d, p>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smt); \
    k_m2l_t<d, p><<<(ntgt + 7) / 8, 256, smt, st>>>(ntgt, csr_ptr, src, offs, tables, table_stride, W32, U);  \
    return;                                                                                                   \
  }
  M2L_CASE(1, 2) M2L_CASE(1, 3) M2L_CASE(1, 4) M2L_CASE(1, 5) M2L_CASE(1, 6) M2L_CASE(1, 7) M2L_CASE(1, 8)
  M2L_CASE(2, 2) M2L_CASE(2, 3) M2L_CASE(2, 4) M2L_CASE(2, 5) M2L_CASE(2, 6) M2L_CASE(2, 7) M2L_CASE(2, 8)
  M2L_CASE(3, 2) M2L_CASE(3, 3) M2L_CASE(3, 4) M2L_CASE(3, 5) M2L_CASE(3, 6)
  M2L_CASE(4, 2) M2L_CASE(4, 3) M2L_CASE(4, 4) M2L_CASE(5, 2) M2L_CASE(5, 4)
  M2L_CASE(6, 2) M2L_CASE(7, 2)
#undef M2L_CASE
  const size_t per_warp = (size_t)m * 16;
  int warps = 8;
  while (warps > 1 && tbytes + warps * per_warp > 200 * 1024) warps >>= 1;
  const size_t sm = tbytes + warps * per_warp;
  static size_t attr = 0;
  if (sm > 48 * 1024 && sm > attr) {
    cudaFuncSetAttribute(k_m2l, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    attr = sm;
  }
  int blocks = (ntgt + warps - 1) / warps;
  k_m2l<<<blocks, 32 * warps, sm, st>>>(D, P, m, ntgt, csr_ptr, src, offs, tables, table_stride, W32, U, warps);
}

void launch_to_f32(const double* a, int64_t n, float* b, cudaStream_t st) {
  if (n <= 0) return;
  const int64_t want = (n + 255) / 256;
  k_to_f32<<<(unsigned)(want < 148 * 8 ? want : 148 * 8), 256, 0, st>>>(a, n, b);
}

}  // namespace f3m
