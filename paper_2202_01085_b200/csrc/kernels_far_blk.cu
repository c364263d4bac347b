// Far-field S2M / L2T for large grids (config C5: D = 5, P = 4, m = 1024; D = 7, P = 3,
// m = 2187) as register-blocked contractions over the points of one box chunk, sm_100a.
//
// Paper: Sec. 3: v1 = L_Y b per box (S2M) and v += L_X^T v2 (L2T), with
// the tensor-product basis over D dimensions.  Per box, both are dense
// contractions over the points:  W[a + MA c] = sum_p A_p[a] C_p[c]  and
// v_p = sum_{a,c} A'_p[a] U[a + MA c] C_p[c], where the node index k = a + MA c splits the
// dimensions into the first DA (a, MA = P^DA) and the rest (c, MC = P^{D-DA}):
//   A_p[a] = b_p prod_{d < DA} L_{k_d}(tau_d)   (A' without b),   C_p[c] = prod_{d >= DA} L_{k_d}(tau_d)
// with the 1-D Lagrange basis of the P Chebyshev nodes (product form): the nodal
// charges and locals of Sec. 3 directly.  [The Chebyshev-moment form of the m <= 128 kernels
// was measured here too: its fp64 change of basis cancels for boxes whose far field is a few
// nearby nodes (tiny gamma), and the locals missed the 1e-5 stage parity by 100x.]
//
// B200 design.  kernels_far_gen.cu (k_s2m_gen4 / k_l2t_gen) reloads the staged weights from
// shared memory for every 16 (S2M) or 4 (L2T) FMAs; here the contraction is register-
// blocked like a GEMM with K = points:
//  * one CTA (8 warps) per chunk of <= FAR_CHUNK points of one box; per batch of 256 points
//    every thread produces one point's A and C rows (zero-padded to 8 TA and 4 TC) into shared
//    memory, as float4 stores with a row stride of 4 (mod 8) floats (8 consecutive rows fall on
//    distinct banks); the products come from two half-tensor tables per side (one multiply per
//    entry);
//  * lane (ia = lane & 7, ic = lane >> 3) owns the TA x TC block a in {32 q + 4 ia + 0..3},
//    c in {16 q + 4 ic + 0..3}: per point TA / 4 + TC / 4 float4 loads (eight lanes read one
//    contiguous 128 B span, the other 24 are broadcasts) feed TA TC / 2 packed FFMA2
//    (D = 5, P = 4: 8 x 4, 3 loads, 16 FFMA2; D = 7, P = 3: 12 x 8 on the 96 x 32 padded grid);
//  * S2M: every warp accumulates all m node charges over its 32 points of each batch (fp32),
//    one fixed-order sum over the 8 warps at the end of the chunk (deterministic), chunk
//    partials reduced in fp64 by launch_chunk_reduce;
//  * L2T: the lane's 32 coefficients U~ live in registers for the whole chunk; per point the
//    lane forms its partial sum, and one warp reduce-scatter per 32 points leaves point
//    (warp, lane) in lane `lane`, written once (vs += v, sorted order, no atomics).
#include <cuda_runtime.h>
#include <stdint.h>

#include "f3m_internal.h"
#include "far_math.cuh"

namespace f3m {

constexpr int BLK_THREADS = 256;

template <int D, int P, int DA, int TA, int TC>
struct BlkShape {
  static constexpr int MA = IPow<P, DA>::value, MC = IPow<P, D - DA>::value, M = MA * MC;
  static constexpr int MAP = 8 * TA, MCP = 4 * TC;  // padded row parts
  // TC % 4 == 0: c slices as float4 (c = 16 q + 4 ic + e); otherwise scalar (c = TC ic + e)
  static_assert(TA % 4 == 0 && MAP >= MA && MCP >= MC, "tile shape");
  static_assert(MCP % 4 == 0, "C row part in float4 stores");
  static constexpr int ROW0 = MAP + MCP;
  static constexpr int ROW = ROW0 + ((4 - ROW0 % 8) + 8) % 8;  // == 4 (mod 8) floats
  static constexpr int HA = DA / 2, HC = (D - DA) / 2;        // half-tensor splits
  static constexpr int ALO = IPow<P, HA>::value, CLO = IPow<P, HC>::value;
  static constexpr int AHI = MA / ALO, CHI = MC / CLO;
};

// box-local 1-D Lagrange weights of one point (local_tau: the sorted kernels' coordinate map)
template <int D, int P>
__device__ __forceinline__ void blk_weights(const float (&x)[D], const BoxGeom& g, const NodeConsts& nc,
                                            float (&T)[D][P]) {
#pragma unroll
  for (int d = 0; d < D; ++d) lagrange<P>(local_tau(x[d], g.lo_hi[d], g.lo_lo[d], g.scale), nc, T[d]);
}

// tensor product over dimensions [d0, d0 + ND) (dimension d0 fastest), scaled by w
template <int D, int P, int D0, int ND>
__device__ __forceinline__ void blk_tensor(const float (&T)[D][P], float w, float* out) {
  out[0] = w;
  int len = 1;
#pragma unroll
  for (int d = 0; d < ND; ++d) {
#pragma unroll
    for (int k = P - 1; k >= 0; --k)
#pragma unroll
      for (int j = 0; j < IPow<P, ND>::value / P; ++j)
        if (j < len) out[j + len * k] = out[j] * T[D0 + d][k];
    len *= P;
  }
}

// row = [A (MA, zero-padded to MAP) | C (MC, padded to MCP)] of one point, A scaled by w
template <int D, int P, int DA, int TA, int TC>
__device__ __forceinline__ void blk_row(const float (&T)[D][P], float w, float* row) {
  using S = BlkShape<D, P, DA, TA, TC>;
  float4* r4 = reinterpret_cast<float4*>(row);
  {
    float lo[S::ALO], hi[S::AHI];
    blk_tensor<D, P, 0, S::HA>(T, w, lo);
    blk_tensor<D, P, S::HA, DA - S::HA>(T, 1.f, hi);
#pragma unroll
    for (int q = 0; q < S::MAP / 4; ++q) {
      float v[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int a = 4 * q + e;
        v[e] = a < S::MA ? lo[a % S::ALO] * hi[a / S::ALO] : 0.f;
      }
      r4[q] = make_float4(v[0], v[1], v[2], v[3]);
    }
  }
  {
    float lo[S::CLO], hi[S::CHI];
    blk_tensor<D, P, DA, S::HC>(T, 1.f, lo);
    blk_tensor<D, P, DA + S::HC, D - DA - S::HC>(T, 1.f, hi);
#pragma unroll
    for (int q = 0; q < S::MCP / 4; ++q) {
      float v[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int c = 4 * q + e;
        v[e] = c < S::MC ? lo[c % S::CLO] * hi[c / S::CLO] : 0.f;
      }
      r4[S::MAP / 4 + q] = make_float4(v[0], v[1], v[2], v[3]);
    }
  }
}

// the lane's A / C slices of one staged row: a = 32 q + 4 ia + e, c = 16 q + 4 ic + e
template <int TA, int TC, int MAP>
__device__ __forceinline__ void blk_load(const float* row, int ia, int ic, float2 (&av)[TA / 2], float (&cv)[TC]) {
#pragma unroll
  for (int q = 0; q < TA / 4; ++q) {
    const float4 x = *reinterpret_cast<const float4*>(row + 32 * q + 4 * ia);
    av[2 * q] = make_float2(x.x, x.y);
    av[2 * q + 1] = make_float2(x.z, x.w);
  }
  if constexpr (TC % 4 == 0) {
#pragma unroll
    for (int q = 0; q < TC / 4; ++q) {
      const float4 x = *reinterpret_cast<const float4*>(row + MAP + 16 * q + 4 * ic);
      cv[4 * q] = x.x; cv[4 * q + 1] = x.y; cv[4 * q + 2] = x.z; cv[4 * q + 3] = x.w;
    }
  } else {
#pragma unroll
    for (int e = 0; e < TC; ++e) cv[e] = row[MAP + TC * ic + e];
  }
}
__device__ __forceinline__ int blk_a(int q2, int ia) { return 32 * (q2 >> 1) + 4 * ia + 2 * (q2 & 1); }  // pair q2
template <int TC>
__device__ __forceinline__ int blk_c(int c, int ic) {
  if constexpr (TC % 4 == 0) return 16 * (c >> 2) + 4 * ic + (c & 3);
  else return TC * ic + c;
}

// ---------------------------------------------------------------------------------------
// S2M: partials[chunk][a + MA c] = sum_{p in chunk} A_p[a] C_p[c]   (nodal charges)
// ---------------------------------------------------------------------------------------
template <int D, int P, int DA, int TA, int TC, int MINB>
__global__ void __launch_bounds__(BLK_THREADS, MINB) k_s2m_blk(const float* __restrict__ xs,
                                                               const float* __restrict__ bs, int64_t n,
                                                               const BoxGeom* __restrict__ boxes,
                                                               const Chunk* __restrict__ chunks, NodeConsts nc,
                                                               float* __restrict__ partials) {
  using S = BlkShape<D, P, DA, TA, TC>;
  extern __shared__ __align__(16) float srow[];  // [256][ROW], then the warp sums [8][M]
  const Chunk ch = chunks[blockIdx.x];
  const BoxGeom g = boxes[ch.box];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int ia = lane & 7, ic = lane >> 3;
  float2 acc[TA / 2][TC];
#pragma unroll
  for (int q = 0; q < TA / 2; ++q)
#pragma unroll
    for (int c = 0; c < TC; ++c) acc[q][c] = make_float2(0.f, 0.f);
  // software pipeline: the next batch's coordinates and weight are loaded before the
  // current batch is consumed
  float xn[D], bn = 0.f;
  auto load = [&](int base) {
    const int p = base + tid;
    const bool ok = p < ch.len;
    const int64_t i = ch.start + (ok ? p : 0);
#pragma unroll
    for (int d = 0; d < D; ++d) xn[d] = __ldg(xs + (int64_t)d * n + i);
    bn = ok ? __ldg(bs + i) : 0.f;  // rows past the chunk contribute nothing
  };
  load(0);
  for (int base = 0; base < ch.len; base += BLK_THREADS) {
    {
      float T[D][P];
      blk_weights<D, P>(xn, g, nc, T);
      blk_row<D, P, DA, TA, TC>(T, bn, srow + tid * S::ROW);
    }
    __syncthreads();
    if (base + BLK_THREADS < ch.len) load(base + BLK_THREADS);
    const int np = min(32, ch.len - base - w * 32);  // this warp's valid rows of the batch
    const float* rw = srow + (w * 32) * S::ROW;
#pragma unroll 2
    for (int j = 0; j < np; ++j) {
      float2 av[TA / 2];
      float cv[TC];
      blk_load<TA, TC, S::MAP>(rw + j * S::ROW, ia, ic, av, cv);
#pragma unroll
      for (int c = 0; c < TC; ++c)
#pragma unroll
        for (int q = 0; q < TA / 2; ++q) acc[q][c] = __ffma2_rn(av[q], f2b(cv[c]), acc[q][c]);
    }
    __syncthreads();  // rows consumed
  }
  // fixed-order sum over the 8 warps (padded entries are never written out)
  float* ws = srow;  // [8][M]
#pragma unroll
  for (int q = 0; q < TA / 2; ++q)
#pragma unroll
    for (int c = 0; c < TC; ++c) {
      const int a = blk_a(q, ia), cc = blk_c<TC>(c, ic);
      if (cc < S::MC) {
        if (a < S::MA) ws[w * S::M + a + S::MA * cc] = acc[q][c].x;
        if (a + 1 < S::MA) ws[w * S::M + a + 1 + S::MA * cc] = acc[q][c].y;
      }
    }
  __syncthreads();
  float* out = partials + (int64_t)blockIdx.x * S::M;
  for (int k = tid; k < S::M; k += BLK_THREADS) {
    float s = ws[k];
#pragma unroll
    for (int w2 = 1; w2 < 8; ++w2) s += ws[w2 * S::M + k];
    out[k] = s;
  }
}

// ---------------------------------------------------------------------------------------
// L2T: vs[p] += sum_{a,c} A'_p[a] U[box][a + MA c] C_p[c]   (U: nodal locals)
// ---------------------------------------------------------------------------------------
template <int D, int P, int DA, int TA, int TC, int MINB>
__global__ void __launch_bounds__(BLK_THREADS, MINB) k_l2t_blk(const float* __restrict__ xs, int64_t n,
                                                               const BoxGeom* __restrict__ boxes,
                                                               const Chunk* __restrict__ chunks, NodeConsts nc,
                                                               const double* __restrict__ Ug,
                                                               float* __restrict__ vs) {
  using S = BlkShape<D, P, DA, TA, TC>;
  extern __shared__ __align__(16) float srow[];  // [256][ROW]
  const Chunk ch = chunks[blockIdx.x];
  const BoxGeom g = boxes[ch.box];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int ia = lane & 7, ic = lane >> 3;
  // the lane's TA x TC block of U, pairs of consecutive a for one c (zero on the padding)
  float2 u2[TA / 2][TC];
  {
    const double* U = Ug + (int64_t)ch.box * S::M;
#pragma unroll
    for (int q = 0; q < TA / 2; ++q)
#pragma unroll
      for (int c = 0; c < TC; ++c) {
        const int a = blk_a(q, ia), cc = blk_c<TC>(c, ic);
        const bool okc = cc < S::MC;
        u2[q][c] = make_float2(okc && a < S::MA ? (float)__ldg(U + a + S::MA * cc) : 0.f,
                               okc && a + 1 < S::MA ? (float)__ldg(U + a + 1 + S::MA * cc) : 0.f);
      }
  }
  float xn[D];
  auto load = [&](int base) {
    const int p = base + tid;
    const int64_t i = ch.start + (p < ch.len ? p : 0);
#pragma unroll
    for (int d = 0; d < D; ++d) xn[d] = __ldg(xs + (int64_t)d * n + i);
  };
  load(0);
  for (int base = 0; base < ch.len; base += BLK_THREADS) {
    {
      float T[D][P];
      blk_weights<D, P>(xn, g, nc, T);
      blk_row<D, P, DA, TA, TC>(T, 1.f, srow + tid * S::ROW);
    }
    __syncthreads();
    if (base + BLK_THREADS < ch.len) load(base + BLK_THREADS);
    const float* rw = srow + (w * 32) * S::ROW;
    auto partial = [&](int j) {  // the lane's share of point j of the warp's 32 rows
      float2 av[TA / 2];
      float cv[TC];
      blk_load<TA, TC, S::MAP>(rw + j * S::ROW, ia, ic, av, cv);
      float2 t = make_float2(0.f, 0.f);
#pragma unroll
      for (int q = 0; q < TA / 2; ++q) {
        float2 s = __fmul2_rn(u2[q][0], f2b(cv[0]));
#pragma unroll
        for (int c = 1; c < TC; ++c) s = __ffma2_rn(u2[q][c], f2b(cv[c]), s);
        t = __ffma2_rn(s, av[q], t);
      }
      return t.x + t.y;
    };
    // warp reduce-scatter of the 32 points' partials (rows past the chunk are finite and never
    // written back), its first level (xor 16) fused into the point loop so that 16 partials
    // are live: afterwards lane l holds the warp sum of point l
    const bool up16 = (lane & 16) != 0;
    float r[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const float pa = partial(j), pb = partial(j + 16);
      r[j] = (up16 ? pb : pa) + __shfl_xor_sync(0xffffffffu, up16 ? pa : pb, 16);
    }
#pragma unroll
    for (int o = 8, len = 16; o >= 1; o >>= 1, len >>= 1) {
      const bool up = (lane & o) != 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (i < len / 2) {
          const float keep = up ? r[i + len / 2] : r[i];
          const float send = up ? r[i] : r[i + len / 2];
          r[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
      }
    }
    const int p = base + w * 32 + lane;
    if (p < ch.len) vs[ch.start + p] += r[0];
    __syncthreads();  // rows consumed
  }
}

// instantiations: (D, P, DA, TA, TC, min CTAs per SM); the other (D, P) keep k_s2m / k_s2m_gen.
// [D = 7, P = 2 as (5, 4, 1): S2M 3.49 -> 3.27 ms but L2T 2.2 -> 3.0 ms at 1e8 (the 32-lane
// reduce-scatter per 32 points dominates at m = 128), so the register-tiled k_s2m / k_l2t stay.]
#define F3M_BLK_CASES(X) \
  X(5, 4, 3, 8, 4, 2)    \
  X(7, 3, 4, 12, 7, 1)   \
  X(4, 4, 3, 8, 1, 4)    \
  X(5, 3, 3, 4, 3, 4)    \
  X(6, 3, 3, 4, 8, 2)

bool blk_supported(int D, int P) {
#define X(d, p, da, ta, tc, mb) if (D == d && P == p) return true;
  F3M_BLK_CASES(X)
#undef X
  return false;
}

template <int D, int P, int DA, int TA, int TC>
static size_t blk_smem() {
  using S = BlkShape<D, P, DA, TA, TC>;
  const size_t rows = sizeof(float) * BLK_THREADS * S::ROW, sums = sizeof(float) * 8 * S::M;
  return rows > sums ? rows : sums;
}

void launch_s2m_blk(int D, int P, const float* xs, const float* bs, int64_t n, const BoxGeom* boxes,
                    const Chunk* chunks, int64_t nchunks, const NodeConsts& nc, float* partials, cudaStream_t st) {
  if (nchunks <= 0) return;
#define X(d, p, da, ta, tc, mb)                                                                               \
  if (D == d && P == p) {                                                                                     \
    const size_t sm = blk_smem<d, p, da, ta, tc>();                                                           \
    cudaFuncSetAttribute(k_s2m_blk<d, p, da, ta, tc, mb>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm); \
    k_s2m_blk<d, p, da, ta, tc, mb><<<(unsigned)nchunks, BLK_THREADS, sm, st>>>(xs, bs, n, boxes, chunks, nc, partials); \
    return;                                                                                                   \
  }
  F3M_BLK_CASES(X)
#undef X
}

void launch_l2t_blk(int D, int P, const float* xs, int64_t n, const BoxGeom* boxes, const Chunk* chunks,
                    int64_t nchunks, const NodeConsts& nc, const double* U, float* vs, cudaStream_t st) {
  if (nchunks <= 0) return;
#define X(d, p, da, ta, tc, mb)                                                                               \
  if (D == d && P == p) {                                                                                     \
    const size_t sm = sizeof(float) * BLK_THREADS * BlkShape<d, p, da, ta, tc>::ROW;                          \
    cudaFuncSetAttribute(k_l2t_blk<d, p, da, ta, tc, mb>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm); \
    k_l2t_blk<d, p, da, ta, tc, mb><<<(unsigned)nchunks, BLK_THREADS, sm, st>>>(xs, n, boxes, chunks, nc, U, vs); \
    return;                                                                                                   \
  }
  F3M_BLK_CASES(X)
#undef X
}

}  // namespace f3m
