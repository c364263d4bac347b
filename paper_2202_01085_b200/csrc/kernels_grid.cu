// M2L over a complete level as Kronecker mode products (sm_100a).
//
// Paper: Sec. 3, stage 2 "v2 = K v1": for every far / smooth pair of boxes
// (p, q) at depth t, U_p += K(nodes_p, nodes_q) W_q, with the Gaussian kernel separable over the
// dimensions: K = (x)_d K_d.  kernels_far.cu applies that per pair (D mode
// products of P x P factors, D P^{D+1} FMAs per pair); for D = 5 / 7 the interaction lists of
// the uniform configurations hold 1e6 - 1e8 pairs and that loop is the step's largest phase.
//
// When level t is a complete grid (every one of the 2^{Dt} boxes present on both sides, X = Y)
// and the group's pairs are exactly the children of the near pairs of depth t - 1, the pair set
// has a product structure: with o = cell(parent p) - cell(parent q), the near rule of Alg. 1
// (dist^2 = sum_d o_d^2 < 4, integer offsets) admits precisely the o in {-1, 0, 1}^D with at most
// three non-zero entries (max-norm rule, F3M_ADMISSIBLE_MAXNORM: every o in {-1, 0, 1}^D).  So
//   U = sum_{o admitted} (x)_d B_d^{(o_d)} W,
// where W, U are tensors over the combined per-dimension index i_d = cell_d P + k_d (N = 2^t P
// values per dimension) and B_d^{(o)}[i][j] = K_d(x_i, y_j) if parent(cell_i) - parent(cell_j) = o,
// else 0.  The sum over the admitted patterns is carried by a "degree" index (the number of
// non-zero o_d so far): each mode product maps degree g to g through B^{(0)} and to g + 1 through
// B^{(+1)} + B^{(-1)}, degrees above 3 are dropped, and U is the sum over the degrees.  Every
// (node pair, box pair) product of the list is formed exactly once: the same sum as the
// pairwise M2L, in another order, accumulated in fp64 (reading R29).
//
// Cost: D mode products over ndeg N^D values, 2N FMAs each (D = 7, P = 3, t = 2: 1.5e9 fp64
// FMAs in place of 1.2e16 flop of pairwise separable products).
#include <cuda_runtime.h>
#include <stdint.h>

#include "f3m_internal.h"

namespace f3m {

// Z[g][I] = 0 (every degree), then Z[0][base(slot) + off(k)] = W[slot][k]
__global__ void k_grid_scatter(const double* __restrict__ W, int nslots, int m, int P, int D, int64_t N,
                               const int64_t* __restrict__ base, double* __restrict__ Z) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)nslots * m) return;
  const int s = (int)(e / m), k = (int)(e - (int64_t)s * m);
  int64_t off = 0, stride = 1;
  int r = k;
  for (int d = 0; d < D; ++d) {
    off += (int64_t)(r % P) * stride;
    r /= P;
    stride *= N;
  }
  Z[base[s] + off] = W[e];
}

// one mode product along dimension d: for every degree g < ndeg and index I,
//   Zo[g][I] = sum_j B0[i][j] Zi[g][I_j] + (g > 0 ? sum_j B1[i][j] Zi[g - 1][I_j] : 0)
// with i = digit d of I and I_j = I with digit d replaced by j (B1 = B^{(+1)} + B^{(-1)};
// ndeg = 1: B1 == 0 and B0 carries every admitted offset)
__global__ void k_grid_mode(const double* __restrict__ Zi, double* __restrict__ Zo, int ndeg, int64_t total,
                            int N, int64_t stride, const double* __restrict__ B0, const double* __restrict__ B1) {
  extern __shared__ double bsm[];  // B0 | B1, N x N each
  for (int e = threadIdx.x; e < 2 * N * N; e += blockDim.x) bsm[e] = e < N * N ? B0[e] : B1[e - N * N];
  __syncthreads();
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)ndeg * total) return;
  const int g = (int)(e / total);
  const int64_t I = e - (int64_t)g * total;
  const int i = (int)((I / stride) % N);
  const int64_t b = I - (int64_t)i * stride;
  const double* r0 = bsm + i * N;
  const double* z0 = Zi + (int64_t)g * total + b;
  double s = 0.0;
  for (int j = 0; j < N; ++j) s = fma(r0[j], z0[(int64_t)j * stride], s);
  if (g > 0) {
    const double* r1 = bsm + N * N + i * N;
    const double* z1 = z0 - total;
    for (int j = 0; j < N; ++j) s = fma(r1[j], z1[(int64_t)j * stride], s);
  }
  Zo[e] = s;
}

// The same mode product, one thread per (column, degree): the column (the N values of one line
// along dimension d) at degrees g and g - 1 is read into registers and the N outputs of degree g
// written once; the block structure of B is compile-time (combined index i = cell P + k, parent
// = i / BS, BS = 2P: B0 is block-diagonal, B1 couples adjacent blocks; MAXN (max-norm rule,
// one degree): B0 spans the diagonal and both adjacent blocks).
template <int N, int BS, bool MAXN>
__global__ void __launch_bounds__(128) k_grid_col(const double* __restrict__ Zi, double* __restrict__ Zo, int64_t total,
                                                  int64_t stride, const double* __restrict__ B0,
                                                  const double* __restrict__ B1) {
  __shared__ double b0[N * N], b1[N * N];
  for (int e = threadIdx.x; e < N * N; e += blockDim.x) { b0[e] = B0[e]; b1[e] = B1[e]; }
  __syncthreads();
  const int64_t col = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int g = blockIdx.y;
  if (col >= total / N) return;
  const int64_t o = col / stride, r = col - o * stride;
  const int64_t base = (int64_t)g * total + o * (int64_t)N * stride + r;
  double zc[N], zl[N];
#pragma unroll
  for (int j = 0; j < N; ++j) zc[j] = Zi[base + (int64_t)j * stride];
  if (g > 0) {
#pragma unroll
    for (int j = 0; j < N; ++j) zl[j] = Zi[base - total + (int64_t)j * stride];
  }
#pragma unroll
  for (int i = 0; i < N; ++i) {
    const int blk = i / BS;
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < N; ++j)
      if (j / BS == blk || (MAXN && (j / BS == blk - 1 || j / BS == blk + 1))) s = fma(b0[i * N + j], zc[j], s);
    if (!MAXN && g > 0) {
#pragma unroll
      for (int j = 0; j < N; ++j)
        if (j / BS == blk - 1 || j / BS == blk + 1) s = fma(b1[i * N + j], zl[j], s);
    }
    Zo[base + (int64_t)i * stride] = s;
  }
}

#define F3M_GRID_COL_CASES(X) X(4, 4) X(8, 4) X(16, 4) X(6, 6) X(12, 6) X(8, 8) X(16, 8) X(10, 10)

static bool grid_col(int N, int P, int ndeg, const double* zi, double* zo, int64_t total, int64_t stride,
                     const double* B0, const double* B1, cudaStream_t st) {
  const int64_t ncol = total / N;
  const dim3 grid((unsigned)((ncol + 127) / 128), (unsigned)ndeg);
#define X(n, bs)                                                              \
  if (N == n && 2 * P == bs) {                                               \
    if (ndeg == 1) k_grid_col<n, bs, true><<<grid, 128, 0, st>>>(zi, zo, total, stride, B0, B1); \
    else k_grid_col<n, bs, false><<<grid, 128, 0, st>>>(zi, zo, total, stride, B0, B1); \
    return true;                                                             \
  }
  F3M_GRID_COL_CASES(X)
#undef X
  return false;
}

// U[slot][k] = sum_g Z[g][base(slot) + off(k)]
__global__ void k_grid_gather(const double* __restrict__ Z, int ndeg, int64_t total, int nslots, int m, int P, int D,
                              int64_t N, const int64_t* __restrict__ base, double* __restrict__ U) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)nslots * m) return;
  const int s = (int)(e / m), k = (int)(e - (int64_t)s * m);
  int64_t off = 0, stride = 1;
  int r = k;
  for (int d = 0; d < D; ++d) {
    off += (int64_t)(r % P) * stride;
    r /= P;
    stride *= N;
  }
  double u = 0.0;
  for (int g = 0; g < ndeg; ++g) u += Z[(int64_t)g * total + base[s] + off];
  U[e] = u;
}

void launch_grid_m2l(int D, int P, int N, int ndeg, const double* B0, const double* B1, const double* W,
                     const int64_t* src_base, int nsrc, const int64_t* tgt_base, int ntgt, double* Za, double* Zb,
                     double* U, cudaStream_t st) {
  int m = 1;
  int64_t total = 1;
  for (int d = 0; d < D; ++d) { m *= P; total *= N; }
  cudaMemsetAsync(Za, 0, sizeof(double) * (size_t)ndeg * total, st);
  const int64_t ws = (int64_t)nsrc * m;
  k_grid_scatter<<<(unsigned)((ws + 255) / 256), 256, 0, st>>>(W, nsrc, m, P, D, N, src_base, Za);
  double* zi = Za;
  double* zo = Zb;
  int64_t stride = 1;
  const size_t sm = sizeof(double) * 2 * N * N;
  if (sm > 48 * 1024) cudaFuncSetAttribute(k_grid_mode, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  for (int d = 0; d < D; ++d) {
    const int64_t work = (int64_t)ndeg * total;
    const double* b0 = B0 + (size_t)d * N * N;
    const double* b1 = B1 + (size_t)d * N * N;
    if (!grid_col(N, P, ndeg, zi, zo, total, stride, b0, b1, st))
      k_grid_mode<<<(unsigned)((work + 255) / 256), 256, sm, st>>>(zi, zo, ndeg, total, N, stride, b0, b1);
    double* t = zi; zi = zo; zo = t;
    stride *= N;
  }
  const int64_t wt = (int64_t)ntgt * m;
  k_grid_gather<<<(unsigned)((wt + 255) / 256), 256, 0, st>>>(zi, ndeg, total, ntgt, m, P, D, N, tgt_base, U);
}

}  // namespace f3m
