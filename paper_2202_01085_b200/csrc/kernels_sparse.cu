// Far field on Smolyak sparse grids (Sec. 4.2 "Sparse grids": "we implement sparse
// grids [Smolyak] to allow for a finer selection of interpolation nodes"; reading R27 of
// combination technique over nested Chebyshev / Clenshaw-Curtis levels).
//
// The level-q interpolant spans the polynomials prod_d T_{k_d}(tau_d) for k in the downward-
// closed index set K_q = { k : k_d <= deg(j_d) for some |j| = q }, deg(0) = 0, deg(j) = 2^j, and
// |K_q| = |H| (nested nodes).  Its cardinal functions are Phi_h = sum_k A[h][k] T_k with
// A = (V^T)^-1, V[h][k] = T_k(node_h) (host, fp64, sparse_grid.cu).  So the three stages of
// Sec. 3 become
//   S2M  M_k = sum_y b_y T_k(tau_y) per box (k_s2m_sparse), W = A M       (k_dense_rows)
//   M2L  U_p[h] += sum_{q, h'} K(n_p^h, n_q^h') W_q[h'], the node-pair kernel evaluated on the
//        fly from per-dimension factor tables (the Gaussian factorises)
//   L2T  Ut = A^T U (k_dense_rows), v_x += sum_k Ut_k T_k(tau_x)       (k_l2t_sparse)
// Every k has at most q dimensions with k_d > 0: its basis function is a product of <= 3 (q <= 3)
// one-dimensional factors, addressed through a per-k table of row offsets (unused factors point
// at T_0 = 1).
#include <cuda_runtime.h>
#include <stdint.h>

#include "f3m_internal.h"
#include "far_math.cuh"

namespace f3m {

constexpr int SP_THREADS = 256;
constexpr int SP_SB = 32;      // staged points per sub-batch (S2M)
constexpr int SP_NMAX = 9;     // finest 1-D grid of level q <= 3
constexpr int SP_KPT = 8;      // index-set entries per thread (m <= 2048)

// T_0..T_{n1-1}(tau) by the three-term recurrence
__device__ __forceinline__ void sp_cheb(float tau, int n1, float* T) {
  T[0] = 1.f;
  T[1] = tau;
  const float t2 = tau + tau;
  for (int j = 2; j < n1; ++j) T[j] = fmaf(t2, T[j - 1], -T[j - 2]);
}

// ---------------------------------------------------------------------------------------
// S2M: partials[chunk][k] = sum_{p in chunk} b_p prod_{factors f of k} T[f](p)
// ---------------------------------------------------------------------------------------
template <int D>
__global__ void __launch_bounds__(SP_THREADS) k_s2m_sparse(const float* __restrict__ xs, const float* __restrict__ bs,
                                                           int64_t n, const BoxGeom* __restrict__ boxes,
                                                           const Chunk* __restrict__ chunks, int n1, int m,
                                                           const uint2* __restrict__ fac, float* __restrict__ partials) {
  constexpr int ROW = D * SP_NMAX;
  __shared__ float Ts[SP_SB][ROW];
  __shared__ float bsh[SP_SB];
  const Chunk ch = chunks[blockIdx.x];
  const BoxGeom g = boxes[ch.box];
  uint32_t f[SP_KPT][4];
  bool own[SP_KPT];
#pragma unroll
  for (int r = 0; r < SP_KPT; ++r) {
    const int e = threadIdx.x + r * SP_THREADS;
    own[r] = e < m;
    const uint2 fe = own[r] ? fac[e] : make_uint2(0u, 0u);
    f[r][0] = fe.x & 0xffffu; f[r][1] = fe.x >> 16; f[r][2] = fe.y & 0xffffu; f[r][3] = fe.y >> 16;
  }
  double acc[SP_KPT];
#pragma unroll
  for (int r = 0; r < SP_KPT; ++r) acc[r] = 0.0;
  for (int base = 0; base < ch.len; base += SP_SB) {
    const int nb = min(SP_SB, ch.len - base);
    __syncthreads();  // previous sub-batch consumed
    for (int e = threadIdx.x; e < nb * D; e += SP_THREADS) {
      const int p = e / D, d = e - p * D;
      const int64_t i = ch.start + base + p;
      const float tau = local_tau(__ldg(xs + (int64_t)d * n + i), g.lo_hi[d], g.lo_lo[d], g.scale);
      sp_cheb(tau, n1, &Ts[p][d * n1]);
      if (d == 0) bsh[p] = __ldg(bs + i);
    }
    __syncthreads();
    float sb[SP_KPT];
#pragma unroll
    for (int r = 0; r < SP_KPT; ++r) sb[r] = 0.f;
    for (int p = 0; p < nb; ++p) {
      const float* row = Ts[p];
      const float bp = bsh[p];
#pragma unroll
      for (int r = 0; r < SP_KPT; ++r)
        if (own[r]) sb[r] = fmaf(bp * row[f[r][0]] * row[f[r][1]] * row[f[r][2]], row[f[r][3]], sb[r]);
    }
#pragma unroll
    for (int r = 0; r < SP_KPT; ++r) acc[r] += (double)sb[r];  // fp64 across sub-batches
  }
  float* out = partials + (int64_t)blockIdx.x * m;
#pragma unroll
  for (int r = 0; r < SP_KPT; ++r)
    if (own[r]) out[threadIdx.x + r * SP_THREADS] = (float)acc[r];
}

// ---------------------------------------------------------------------------------------
// out[r][i] = sum_j mat[i][j] in[r][j] for R rows of length m (fp64), given matT = mat^T:
// 64 x 64 output tiles, 256 threads with 4 x 4 outputs each, 16-wide k panels in shared memory
// ---------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_dense_rows(const double* __restrict__ in, int64_t R, int m,
                                                    const double* __restrict__ matT, double* __restrict__ out) {
  __shared__ double As[16][64 + 1];  // in  [row][k] panel, transposed: As[k][row]
  __shared__ double Bs[16][64 + 1];  // matT[k][col]
  const int tr = threadIdx.x / 16, tc = threadIdx.x % 16;
  const int64_t r0 = (int64_t)blockIdx.y * 64;
  const int c0 = blockIdx.x * 64;
  double c[4][4] = {};
  for (int k0 = 0; k0 < m; k0 += 16) {
    for (int e = threadIdx.x; e < 16 * 64; e += 256) {
      const int kk = e % 16, rr = e / 16;
      const int64_t row = r0 + rr;
      As[kk][rr] = (row < R && k0 + kk < m) ? in[row * m + k0 + kk] : 0.0;
      const int kb = e / 64, cc = e % 64;
      Bs[kb][cc] = (k0 + kb < m && c0 + cc < m) ? matT[(int64_t)(k0 + kb) * m + c0 + cc] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) { a[i] = As[kk][tr + 16 * i]; b[i] = Bs[kk][tc + 16 * i]; }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) c[i][j] = fma(a[i], b[j], c[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t row = r0 + tr + 16 * i;
    if (row >= R) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int col = c0 + tc + 16 * j;
      if (col < m) out[row * m + col] = c[i][j];
    }
  }
}

// ---------------------------------------------------------------------------------------
// M2L on the sparse nodes: one block per target box, threads own target nodes; per pair the
// source charges and the pair's D factor tables are staged in shared memory, and
// K(n_p^h, n_q^h') = prod_d G_d[h_d][h'_d] is evaluated on the fly (fp32 per pair, fp64 over
// the interaction list).
// ---------------------------------------------------------------------------------------
template <int D>
__global__ void __launch_bounds__(SP_THREADS) k_m2l_sparse(int m, int n1, const int32_t* __restrict__ csr_ptr,
                                                           const int32_t* __restrict__ src, const uint64_t* __restrict__ offs,
                                                           const float* __restrict__ tables, int table_stride,
                                                           const float* __restrict__ W32, const uint8_t* __restrict__ nodes,
                                                           double* __restrict__ U) {
  extern __shared__ __align__(16) unsigned char sp_sm[];
  float* Ws = reinterpret_cast<float*>(sp_sm);                        // [m]
  float* Gs = Ws + ((m + 3) / 4) * 4;                                 // [D][n1 * n1]
  uint8_t* nd = reinterpret_cast<uint8_t*>(Gs + D * n1 * n1);         // [m][D]
  const int p = blockIdx.x;
  for (int e = threadIdx.x; e < m * D; e += SP_THREADS) nd[e] = nodes[e];
  int hb[SP_KPT][D];
  bool own[SP_KPT];
#pragma unroll
  for (int r = 0; r < SP_KPT; ++r) {
    const int h = threadIdx.x + r * SP_THREADS;
    own[r] = h < m;
#pragma unroll
    for (int d = 0; d < D; ++d) hb[r][d] = d * n1 * n1 + (own[r] ? nodes[h * D + d] : 0) * n1;
  }
  double acc[SP_KPT];
#pragma unroll
  for (int r = 0; r < SP_KPT; ++r) acc[r] = 0.0;
  for (int e = csr_ptr[p]; e < csr_ptr[p + 1]; ++e) {
    const int q = src[e];
    const uint64_t pk = offs[e];
    __syncthreads();  // previous pair consumed
    for (int i = threadIdx.x; i < m; i += SP_THREADS) Ws[i] = W32[(int64_t)q * m + i];
    for (int i = threadIdx.x; i < D * n1 * n1; i += SP_THREADS) {
      const int d = i / (n1 * n1), kj = i - d * n1 * n1;
      const int idx = (int)((pk >> (8 * d)) & 0xffu);
      Gs[i] = tables[(int64_t)d * table_stride + (int64_t)idx * n1 * n1 + kj];
    }
    __syncthreads();
    float s[SP_KPT];
#pragma unroll
    for (int r = 0; r < SP_KPT; ++r) s[r] = 0.f;
    for (int j = 0; j < m; ++j) {
      int sj[D];
#pragma unroll
      for (int d = 0; d < D; ++d) sj[d] = nd[j * D + d];
      const float wj = Ws[j];
#pragma unroll
      for (int r = 0; r < SP_KPT; ++r) {
        if (!own[r]) continue;
        float kv = Gs[hb[r][0] + sj[0]];
#pragma unroll
        for (int d = 1; d < D; ++d) kv *= Gs[hb[r][d] + sj[d]];
        s[r] = fmaf(kv, wj, s[r]);
      }
    }
#pragma unroll
    for (int r = 0; r < SP_KPT; ++r) acc[r] += (double)s[r];
  }
#pragma unroll
  for (int r = 0; r < SP_KPT; ++r)
    if (own[r]) U[(int64_t)p * m + threadIdx.x + r * SP_THREADS] = acc[r];
}

// ---------------------------------------------------------------------------------------
// L2T: vs[i] += sum_k Ut[box][k] prod_{factors f of k} T[f](x_i), one thread per point, the
// box's coefficients and the factor table in shared memory, each thread's Chebyshev row in
// its own shared-memory column (runtime factor offsets index shared memory, never registers)
// ---------------------------------------------------------------------------------------
template <int D>
__global__ void __launch_bounds__(SP_THREADS) k_l2t_sparse(const float* __restrict__ xs, int64_t n,
                                                           const BoxGeom* __restrict__ boxes,
                                                           const Chunk* __restrict__ chunks, int n1, int m,
                                                           const uint2* __restrict__ fac, const double* __restrict__ Ut,
                                                           float* __restrict__ vs) {
  constexpr int ROW = D * SP_NMAX + 1;  // odd stride: conflict-free per-thread rows
  extern __shared__ __align__(16) unsigned char sp_sm[];
  float* Us = reinterpret_cast<float*>(sp_sm);                         // [m]
  uint2* fs = reinterpret_cast<uint2*>(Us + ((m + 1) / 2) * 2);        // [m]
  float* Tr = reinterpret_cast<float*>(fs + m);                        // [THREADS][ROW]
  const Chunk ch = chunks[blockIdx.x];
  const BoxGeom g = boxes[ch.box];
  for (int e = threadIdx.x; e < m; e += SP_THREADS) {
    Us[e] = (float)Ut[(int64_t)ch.box * m + e];
    fs[e] = fac[e];
  }
  __syncthreads();
  float* T = Tr + threadIdx.x * ROW;
  for (int p = threadIdx.x; p < ch.len; p += SP_THREADS) {
    const int64_t i = ch.start + p;
#pragma unroll
    for (int d = 0; d < D; ++d)
      sp_cheb(local_tau(__ldg(xs + (int64_t)d * n + i), g.lo_hi[d], g.lo_lo[d], g.scale), n1, T + d * n1);
    float v = 0.f;
    for (int k = 0; k < m; ++k) {
      const uint2 fe = fs[k];
      const float t = T[fe.x & 0xffffu] * T[fe.x >> 16] * T[fe.y & 0xffffu] * T[fe.y >> 16];
      v = fmaf(Us[k], t, v);
    }
    vs[i] += v;
  }
}

// ---------------------------------------------------------------------------------------
bool sparse_supported(int D, int q, int64_t m) { return D >= 1 && D <= 7 && q >= 1 && q <= 3 && m <= SP_KPT * SP_THREADS; }

void launch_s2m_sparse(int D, int n1, int m, const float* xs, const float* bs, int64_t n, const BoxGeom* boxes,
                       const Chunk* chunks, int64_t nchunks, const uint2* fac, float* partials, cudaStream_t st) {
  if (nchunks <= 0) return;
#define X(d) \
  if (D == d) { k_s2m_sparse<d><<<(unsigned)nchunks, SP_THREADS, 0, st>>>(xs, bs, n, boxes, chunks, n1, m, fac, partials); return; }
  X(1) X(2) X(3) X(4) X(5) X(6) X(7)
#undef X
}

void launch_dense_rows(const double* in, int64_t R, int m, const double* matT, double* out, cudaStream_t st) {
  if (R <= 0) return;
  dim3 grid((unsigned)((m + 63) / 64), (unsigned)((R + 63) / 64));
  k_dense_rows<<<grid, 256, 0, st>>>(in, R, m, matT, out);
}

static size_t m2l_sparse_smem(int D, int m, int n1) {
  return (size_t)((m + 3) / 4) * 16 + (size_t)D * n1 * n1 * 4 + (size_t)m * D + 16;
}

void launch_m2l_sparse(int D, int n1, int m, int32_t ntgt, const int32_t* csr_ptr, const int32_t* src,
                       const uint64_t* offs, const float* tables, int table_stride, const float* W32,
                       const uint8_t* nodes, double* U, cudaStream_t st) {
  if (ntgt <= 0) return;
  const size_t sm = m2l_sparse_smem(D, m, n1);
#define X(d)                                                                                           \
  if (D == d) {                                                                                        \
    cudaFuncSetAttribute(k_m2l_sparse<d>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);       \
    k_m2l_sparse<d><<<(unsigned)ntgt, SP_THREADS, sm, st>>>(m, n1, csr_ptr, src, offs, tables, table_stride, W32, \
                                                            nodes, U);                                 \
    return;                                                                                            \
  }
  X(1) X(2) X(3) X(4) X(5) X(6) X(7)
#undef X
}

void launch_l2t_sparse(int D, int n1, int m, const float* xs, int64_t n, const BoxGeom* boxes, const Chunk* chunks,
                       int64_t nchunks, const uint2* fac, const double* Ut, float* vs, cudaStream_t st) {
  if (nchunks <= 0) return;
  const size_t sm = (size_t)((m + 1) / 2) * 8 + (size_t)m * 8 + (size_t)SP_THREADS * (D * SP_NMAX + 1) * 4;
#define X(d)                                                                                      \
  if (D == d) {                                                                                   \
    cudaFuncSetAttribute(k_l2t_sparse<d>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);  \
    k_l2t_sparse<d><<<(unsigned)nchunks, SP_THREADS, sm, st>>>(xs, n, boxes, chunks, n1, m, fac, Ut, vs); \
    return;                                                                                       \
  }
  X(1) X(2) X(3) X(4) X(5) X(6) X(7)
#undef X
}

}  // namespace f3m
