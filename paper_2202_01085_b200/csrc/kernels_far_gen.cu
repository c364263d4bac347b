// Far-field S2M / L2T for large interpolation grids (128 < m = P^D <= 4096), sm_100a.
//
// Same operators as kernels_far.cu (Sec. 3: v1 = L_Y b per box, and
// v += L_X^T v2), on box-sorted SoA chunks of <= FAR_CHUNK points, in the Lagrange basis
// (product form of PAPER.md:139).  m accumulators per thread no longer fit in registers,
// so the work is split the other way round:
//  * k_s2m_gen is NODE-parallel: node k = k0 + P * line; thread t owns lines t, t + 256, ...
//    and accumulates its P * LPT nodes in registers over the chunk.  Per sub-batch of
//    GEN_SB points the 1-D weights L_d(tau_{p,d}) (dimension 0 scaled by b_p) are staged
//    in shared memory; a thread forms R = prod_{d>=1} L_d[k_d(line)] and adds
//    (b L_0[k0]) R for k0 < P.  Each node is written by exactly one thread: no reduction,
//    deterministic.
//  * k_l2t_gen is POINT-parallel (GEN_PPT points per thread): U of the chunk's box in
//    shared memory (rows of P read as float4 where P % 4 == 0, shared by the thread's
//    points), dimensions 0 and 1 contracted from registers, dimensions >= 2 weighted by
//    per-thread columns of shared memory (runtime digits index shared memory, never
//    registers).
#include <cuda_runtime.h>
#include <stdint.h>
#include <cstdlib>

#include "f3m_internal.h"
#include "far_math.cuh"

namespace f3m {

constexpr int GEN_THREADS = 256;
constexpr int GEN_SB = 32;   // points per staged sub-batch (S2M)
constexpr int GEN_PPT = 2;   // points per thread (L2T)

template <int D, int P>
__device__ __forceinline__ float gen_tau(const float* __restrict__ xs, int64_t n, int64_t i, int d, const BoxGeom& g) {
  const float x = __ldg(xs + (int64_t)d * n + i);
  return local_tau(x, g.lo_hi[d], g.lo_lo[d], g.scale);
}

// ---------------------------------------------------------------------------------------
// S2M: partials[chunk][k0 + P line] = sum_p b_p L_0[k0](p) prod_{d>=1} L_d[k_d(line)](p)
// ---------------------------------------------------------------------------------------
template <int D, int P>
__global__ void __launch_bounds__(GEN_THREADS) k_s2m_gen(const float* __restrict__ xs, const float* __restrict__ bs,
                                                         int64_t n, const BoxGeom* __restrict__ boxes,
                                                         const Chunk* __restrict__ chunks, NodeConsts nc,
                                                         float* __restrict__ partials) {
  constexpr int M = IPow<P, D>::value;
  constexpr int LINES = M / P;
  constexpr int LPT = (LINES + GEN_THREADS - 1) / GEN_THREADS;
  constexpr int NPH = LINES >= GEN_THREADS ? 1 : GEN_THREADS / LINES;  // point phases (few lines)
  constexpr int ROW = D * P;                 // staged weights of one point
  __shared__ __align__(16) float Ls[GEN_SB * ROW];
  __shared__ float red[NPH > 1 ? NPH * M : 1];
  const int ph = NPH > 1 ? threadIdx.x / LINES : 0;
  const int tl = NPH > 1 ? threadIdx.x % LINES : threadIdx.x;
  const Chunk ch = chunks[blockIdx.x];
  const BoxGeom g = boxes[ch.box];
  // shared-memory offsets of this thread's lines' digits (dimensions 1..D-1)
  int off[LPT][D > 1 ? D - 1 : 1];
  bool own[LPT];
#pragma unroll
  for (int r = 0; r < LPT; ++r) {
    const int line = tl + r * GEN_THREADS;
    own[r] = line < LINES && ph < NPH;
    int q = line;
#pragma unroll
    for (int d = 1; d < D; ++d) {
      off[r][d - 1] = d * P + q % P;
      q /= P;
    }
  }
  // fp32 sums over one sub-batch, folded into fp64 after each (a chunk is up to FAR_CHUNK
  // points summed by one thread: plain fp32 accumulation would lose ~sqrt(n) ulps)
  double acc[LPT][P];
#pragma unroll
  for (int r = 0; r < LPT; ++r)
#pragma unroll
    for (int k = 0; k < P; ++k) acc[r][k] = 0.0;

  for (int base = 0; base < ch.len; base += GEN_SB) {
    const int nb = min(GEN_SB, ch.len - base);
    __syncthreads();  // previous sub-batch consumed
    for (int e = threadIdx.x; e < nb * D; e += GEN_THREADS) {
      const int p = e / D, d = e - p * D;
      const int64_t i = ch.start + base + p;
      float L[P];
      lagrange<P>(gen_tau<D, P>(xs, n, i, d, g), nc, L);
      const float sc = d == 0 ? __ldg(bs + i) : 1.f;
#pragma unroll
      for (int k = 0; k < P; ++k) Ls[p * ROW + d * P + k] = L[k] * sc;
    }
    __syncthreads();
    float sb[LPT][P];
#pragma unroll
    for (int r = 0; r < LPT; ++r)
#pragma unroll
      for (int k = 0; k < P; ++k) sb[r][k] = 0.f;
    for (int p = ph; p < nb; p += NPH) {
      const float* row = Ls + p * ROW;
      float a0[P];
#pragma unroll
      for (int k = 0; k < P; ++k) a0[k] = row[k];
#pragma unroll
      for (int r = 0; r < LPT; ++r) {
        if (!own[r]) continue;
        float R = 1.f;
#pragma unroll
        for (int d = 1; d < D; ++d) R *= row[off[r][d - 1]];
#pragma unroll
        for (int k = 0; k < P; ++k) sb[r][k] = fmaf(a0[k], R, sb[r][k]);
      }
    }
#pragma unroll
    for (int r = 0; r < LPT; ++r)
#pragma unroll
      for (int k = 0; k < P; ++k) acc[r][k] += (double)sb[r][k];
  }
  float* out = partials + (int64_t)blockIdx.x * M;
  if constexpr (NPH == 1) {
#pragma unroll
    for (int r = 0; r < LPT; ++r) {
      if (!own[r]) continue;
      const int line = tl + r * GEN_THREADS;
#pragma unroll
      for (int k = 0; k < P; ++k) out[k + P * line] = (float)acc[r][k];
    }
  } else {  // sum the phases in a fixed order
    if (own[0])
#pragma unroll
      for (int k = 0; k < P; ++k) red[ph * M + k + P * tl] = (float)acc[0][k];
    __syncthreads();
    for (int e = threadIdx.x; e < M; e += GEN_THREADS) {
      float s = 0.f;
      for (int q = 0; q < NPH; ++q) s += red[q * M + e];
      out[e] = s;
    }
  }
}

// ---------------------------------------------------------------------------------------
// The same S2M with P lines per thread (the P values of digit k_1 share a0 and the dims >= 2
// digits): per point a thread loads the staged weights once for P lines, i.e. ~40 % fewer
// instructions than one line per thread.  Every node still accumulates its points in the
// same order with the same products (R = ((L_1 L_2) L_3) ..., fp32 per sub-batch, folded into
// fp64 per sub-batch), so the charges are bit-identical to k_s2m_gen.
// ---------------------------------------------------------------------------------------
template <int D, int P>
__global__ void __launch_bounds__(IPow<P, D - 2>::value) k_s2m_gen4(const float* __restrict__ xs,
                                                                   const float* __restrict__ bs, int64_t n,
                                                                   const BoxGeom* __restrict__ boxes,
                                                                   const Chunk* __restrict__ chunks, NodeConsts nc,
                                                                   float* __restrict__ partials) {
  constexpr int M = IPow<P, D>::value;
  constexpr int NT = IPow<P, D - 2>::value;  // threads: line groups (digits k_2 .. k_{D-1})
  constexpr int ROW = D * P;
  __shared__ __align__(16) float Ls[GEN_SB * ROW];
  const Chunk ch = chunks[blockIdx.x];
  const BoxGeom g = boxes[ch.box];
  const int gq = threadIdx.x;  // lines gq P + k1, k1 < P
  int off[D > 2 ? D - 2 : 1];  // shared-memory offsets of the digits k_2 .. k_{D-1}
  {
    int q = gq;
#pragma unroll
    for (int d = 2; d < D; ++d) {
      off[d - 2] = d * P + q % P;
      q /= P;
    }
  }
  double acc[P][P];
#pragma unroll
  for (int r = 0; r < P; ++r)
#pragma unroll
    for (int k = 0; k < P; ++k) acc[r][k] = 0.0;
  for (int base = 0; base < ch.len; base += GEN_SB) {
    const int nb = min(GEN_SB, ch.len - base);
    __syncthreads();
    for (int e = threadIdx.x; e < nb * D; e += NT) {
      const int p = e / D, d = e - p * D;
      const int64_t i = ch.start + base + p;
      float L[P];
      lagrange<P>(gen_tau<D, P>(xs, n, i, d, g), nc, L);
      const float sc = d == 0 ? __ldg(bs + i) : 1.f;
#pragma unroll
      for (int k = 0; k < P; ++k) Ls[p * ROW + d * P + k] = L[k] * sc;
    }
    __syncthreads();
    float sb[P][P];
#pragma unroll
    for (int r = 0; r < P; ++r)
#pragma unroll
      for (int k = 0; k < P; ++k) sb[r][k] = 0.f;
    for (int p = 0; p < nb; ++p) {
      const float* row = Ls + p * ROW;
      float a0[P], l1[P], rest[D > 2 ? D - 2 : 1];
#pragma unroll
      for (int k = 0; k < P; ++k) { a0[k] = row[k]; l1[k] = row[P + k]; }
#pragma unroll
      for (int d = 2; d < D; ++d) rest[d - 2] = row[off[d - 2]];
#pragma unroll
      for (int r = 0; r < P; ++r) {  // line gq P + r: k_1 = r
        float R = 1.f;
        R *= l1[r];
#pragma unroll
        for (int d = 2; d < D; ++d) R *= rest[d - 2];
#pragma unroll
        for (int k = 0; k < P; ++k) sb[r][k] = fmaf(a0[k], R, sb[r][k]);
      }
    }
#pragma unroll
    for (int r = 0; r < P; ++r)
#pragma unroll
      for (int k = 0; k < P; ++k) acc[r][k] += (double)sb[r][k];
  }
  float* out = partials + (int64_t)blockIdx.x * M;
#pragma unroll
  for (int r = 0; r < P; ++r)
#pragma unroll
    for (int k = 0; k < P; ++k) out[k + P * (gq * P + r)] = (float)acc[r][k];
}

// ---------------------------------------------------------------------------------------
// L2T: vs[x] += sum_k prod_d L_{k_d}(tau_{x,d}) U[box][k]
// ---------------------------------------------------------------------------------------
template <int P>
__device__ __forceinline__ void gen_row(const float* su, float (&u)[P]) {
  if constexpr (P % 4 == 0) {
#pragma unroll
    for (int k = 0; k < P; k += 4) {
      const float4 v = *reinterpret_cast<const float4*>(su + k);
      u[k] = v.x; u[k + 1] = v.y; u[k + 2] = v.z; u[k + 3] = v.w;
    }
  } else {
#pragma unroll
    for (int k = 0; k < P; ++k) u[k] = su[k];
  }
}

template <int D, int P>
__global__ void __launch_bounds__(GEN_THREADS) k_l2t_gen(const float* __restrict__ xs, int64_t n,
                                                         const BoxGeom* __restrict__ boxes,
                                                         const Chunk* __restrict__ chunks, NodeConsts nc,
                                                         const double* __restrict__ U, float* __restrict__ vs) {
  constexpr int M = IPow<P, D>::value;
  constexpr int NO = D > 2 ? D - 2 : 1;           // outer dimensions (>= 2)
  constexpr int OUTER = D > 2 ? M / (P * P) : 1;
  // small outer grids: the outer loop is unrolled, so the outer digits are compile-time and
  // their weights stay in registers (no per-term shared-memory loads)
  constexpr bool OUTER_REG = D > 2 && OUTER <= 64;
  extern __shared__ __align__(16) float gsm[];
  float* su = gsm;                                  // [M]
  float* Lo = gsm + ((M + 3) / 4) * 4;              // [GEN_PPT][NO * P][GEN_THREADS]
  const Chunk ch = chunks[blockIdx.x];
  const BoxGeom g = boxes[ch.box];
  for (int k = threadIdx.x; k < M; k += GEN_THREADS) su[k] = (float)U[(int64_t)ch.box * M + k];
  __syncthreads();
  const int64_t end = ch.start + ch.len;
  for (int64_t i0 = ch.start; i0 < end; i0 += (int64_t)GEN_THREADS * GEN_PPT) {
    float L0[GEN_PPT][P], L1[GEN_PPT][P];
    float Lr[OUTER_REG ? GEN_PPT : 1][OUTER_REG ? NO : 1][P];  // outer-dimension weights in registers
    bool valid[GEN_PPT];
#pragma unroll
    for (int q = 0; q < GEN_PPT; ++q) {
      const int64_t i = i0 + threadIdx.x + (int64_t)q * GEN_THREADS;
      valid[q] = i < end;
      const int64_t ii = valid[q] ? i : ch.start;
      lagrange<P>(gen_tau<D, P>(xs, n, ii, 0, g), nc, L0[q]);
      if constexpr (D > 1) lagrange<P>(gen_tau<D, P>(xs, n, ii, 1, g), nc, L1[q]);
      if constexpr (D > 2) {
#pragma unroll
        for (int d = 2; d < D; ++d) {
          float L[P];
          lagrange<P>(gen_tau<D, P>(xs, n, ii, d, g), nc, L);
#pragma unroll
          for (int k = 0; k < P; ++k) {
            if constexpr (OUTER_REG) Lr[q][d - 2][k] = L[k];
            else Lo[((q * NO + d - 2) * P + k) * GEN_THREADS + threadIdx.x] = L[k];
          }
        }
      }
    }
    float v[GEN_PPT];
#pragma unroll
    for (int q = 0; q < GEN_PPT; ++q) v[q] = 0.f;
    if constexpr (D == 1) {
      float u[P];
      gen_row<P>(su, u);
#pragma unroll
      for (int q = 0; q < GEN_PPT; ++q)
#pragma unroll
        for (int k = 0; k < P; ++k) v[q] = fmaf(L0[q][k], u[k], v[q]);
    } else {
      int kd[NO];
#pragma unroll
      for (int e = 0; e < NO; ++e) kd[e] = 0;
#pragma unroll (OUTER_REG ? OUTER : 1)
      for (int o = 0; o < OUTER; ++o) {
        float s[GEN_PPT];
#pragma unroll
        for (int q = 0; q < GEN_PPT; ++q) s[q] = 0.f;
#pragma unroll
        for (int k1 = 0; k1 < P; ++k1) {
          float u[P];
          gen_row<P>(su + (o * P + k1) * P, u);
#pragma unroll
          for (int q = 0; q < GEN_PPT; ++q) {
            float t = 0.f;
#pragma unroll
            for (int k0 = 0; k0 < P; ++k0) t = fmaf(L0[q][k0], u[k0], t);
            s[q] = fmaf(L1[q][k1], t, s[q]);
          }
        }
        if constexpr (D > 2) {
#pragma unroll
          for (int q = 0; q < GEN_PPT; ++q) {
            float wo = 1.f;
            if constexpr (OUTER_REG) {
              int rem = o;  // compile-time after unrolling: digit e of o (dimension 2 fastest)
#pragma unroll
              for (int e = 0; e < NO; ++e) {
                wo *= Lr[q][e][rem % P];
                rem /= P;
              }
            } else {
#pragma unroll
              for (int e = 0; e < NO; ++e) wo *= Lo[((q * NO + e) * P + kd[e]) * GEN_THREADS + threadIdx.x];
            }
            v[q] = fmaf(wo, s[q], v[q]);
          }
          // odometer over the outer digits (dimension 2 fastest)
#pragma unroll
          for (int e = 0; e < NO; ++e) {
            if (++kd[e] < P) break;
            kd[e] = 0;
          }
        } else {
#pragma unroll
          for (int q = 0; q < GEN_PPT; ++q) v[q] += s[q];
        }
      }
    }
#pragma unroll
    for (int q = 0; q < GEN_PPT; ++q) {
      const int64_t i = i0 + threadIdx.x + (int64_t)q * GEN_THREADS;
      if (valid[q]) vs[i] += v[q];
    }
  }
}

// ---------------------------------------------------------------------------------------
// instantiations: the (D, P) with 128 < P^D <= 4096 that kernels_far.cu does not cover
#define F3M_GEN_CASES(X)                                                                   \
  X(1, 9) X(1, 10) X(1, 11) X(1, 12) X(1, 13) X(1, 14) X(1, 15) X(1, 16)                  \
  X(2, 9) X(2, 10) X(2, 11) X(2, 12) X(2, 13) X(2, 14) X(2, 15) X(2, 16)                  \
  X(3, 6) X(3, 7) X(3, 8) X(3, 9) X(3, 10) X(3, 11) X(3, 12) X(3, 13) X(3, 14) X(3, 15) X(3, 16) \
  X(4, 4) X(4, 5) X(4, 6) X(4, 7) X(4, 8)                                                  \
  X(5, 3) X(5, 4) X(5, 5) X(6, 3) X(6, 4) X(7, 3)

bool gen_supported(int D, int P) {
#define X(d, p) if (D == d && P == p) return true;
  F3M_GEN_CASES(X)
#undef X
  return false;
}

static size_t l2t_gen_smem(int D, int P) {
  int m = 1;
  for (int d = 0; d < D; ++d) m *= P;
  const int no = D > 2 ? D - 2 : 1;
  return sizeof(float) * ((size_t)(m + 3) / 4 * 4 + (size_t)GEN_PPT * no * P * GEN_THREADS);
}

void launch_s2m_gen(int D, int P, const float* xs, const float* bs, int64_t n, const BoxGeom* boxes,
                    const Chunk* chunks, int64_t nchunks, const NodeConsts& nc, float* partials, cudaStream_t st) {
  if (nchunks <= 0) return;
  {  // P lines per thread where P^{D-2} makes a sensible block
    if (D == 5 && P == 4) { k_s2m_gen4<5, 4><<<(unsigned)nchunks, 64, 0, st>>>(xs, bs, n, boxes, chunks, nc, partials); return; }
    if (D == 4 && P == 8) { k_s2m_gen4<4, 8><<<(unsigned)nchunks, 64, 0, st>>>(xs, bs, n, boxes, chunks, nc, partials); return; }
    if (D == 5 && P == 5) { k_s2m_gen4<5, 5><<<(unsigned)nchunks, 125, 0, st>>>(xs, bs, n, boxes, chunks, nc, partials); return; }
    if (D == 6 && P == 4) { k_s2m_gen4<6, 4><<<(unsigned)nchunks, 256, 0, st>>>(xs, bs, n, boxes, chunks, nc, partials); return; }
  }
#define X(d, p)                                                                                       \
  if (D == d && P == p) {                                                                             \
    k_s2m_gen<d, p><<<(unsigned)nchunks, GEN_THREADS, 0, st>>>(xs, bs, n, boxes, chunks, nc, partials); \
    return;                                                                                           \
  }
  F3M_GEN_CASES(X)
#undef X
}

void launch_l2t_gen(int D, int P, const float* xs, int64_t n, const BoxGeom* boxes, const Chunk* chunks,
                    int64_t nchunks, const NodeConsts& nc, const double* U, float* vs, cudaStream_t st) {
  if (nchunks <= 0) return;
  const size_t sm = l2t_gen_smem(D, P);
#define X(d, p)                                                                                  \
  if (D == d && P == p) {                                                                        \
    if (sm > 48 * 1024) cudaFuncSetAttribute(k_l2t_gen<d, p>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm); \
    k_l2t_gen<d, p><<<(unsigned)nchunks, GEN_THREADS, sm, st>>>(xs, n, boxes, chunks, nc, U, vs); \
    return;                                                                                      \
  }
  F3M_GEN_CASES(X)
#undef X
}

}  // namespace f3m
