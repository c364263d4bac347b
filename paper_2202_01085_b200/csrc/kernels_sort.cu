// Binning kernels for sm_100a: enclosing cube, bit-exact box keys, warp-aggregated tile
// histograms, exclusive scan, deterministic stable counting-sort scatter, run-length box
// tables and the output permutation.
//
// Paper: Sec. 3 "Enclosing"; Sec. 4.1 count-and-increment grouping
// (made deterministic and stable: reading R13); Sec. 4.2 box index
// (reading R12); sigma.
#include <cuda_runtime.h>
#include <stdint.h>

#include "f3m_internal.h"
#include "keys.cuh"

namespace f3m {

// ======================================================================================
// enclosing cube: per-dimension min / max and a non-finite flag
// ======================================================================================
constexpr int BBOX_THREADS = 256;

int bbox_blocks(int64_t n) {
  int64_t b = (n + BBOX_THREADS - 1) / BBOX_THREADS;
  if (b > 148 * 8) b = 148 * 8;
  if (b < 1) b = 1;
  return (int)b;
}

__global__ void __launch_bounds__(BBOX_THREADS) k_bbox(const float* __restrict__ X, int64_t n, int D,
                                                       float* __restrict__ partials) {
  float mn[F3M_MAXD], mx[F3M_MAXD];
  float bad = 0.f;
#pragma unroll
  for (int d = 0; d < F3M_MAXD; ++d) { mn[d] = __int_as_float(0x7f800000); mx[d] = -mn[d]; }
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
    for (int d = 0; d < F3M_MAXD; ++d) {
      if (d < D) {
        float v = __ldg(X + r * D + d);
        if (!isfinite(v)) bad = 1.f;
        mn[d] = fminf(mn[d], v);
        mx[d] = fmaxf(mx[d], v);
      }
    }
  }
  __shared__ float s[BBOX_THREADS / 32][2 * F3M_MAXD + 1];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int d = 0; d < F3M_MAXD; ++d) {
    for (int o = 16; o > 0; o >>= 1) {
      mn[d] = fminf(mn[d], __shfl_xor_sync(0xffffffffu, mn[d], o));
      mx[d] = fmaxf(mx[d], __shfl_xor_sync(0xffffffffu, mx[d], o));
    }
  }
  for (int o = 16; o > 0; o >>= 1) bad = fmaxf(bad, __shfl_xor_sync(0xffffffffu, bad, o));
  if (lane == 0) {
    for (int d = 0; d < F3M_MAXD; ++d) { s[w][d] = mn[d]; s[w][F3M_MAXD + d] = mx[d]; }
    s[w][2 * F3M_MAXD] = bad;
  }
  __syncthreads();
  if (threadIdx.x < 2 * F3M_MAXD + 1) {
    const int k = threadIdx.x;
    float a = s[0][k];
    for (int j = 1; j < BBOX_THREADS / 32; ++j)
      a = (k < F3M_MAXD) ? fminf(a, s[j][k]) : fmaxf(a, s[j][k]);
    partials[(int64_t)blockIdx.x * (2 * F3M_MAXD + 1) + k] = a;
  }
}

// vectorised variant: a unit of D float4 = 4 rows, dims known at compile time (16-B aligned X)
template <int D>
__global__ void __launch_bounds__(BBOX_THREADS) k_bbox_vec(const float* __restrict__ X, int64_t n,
                                                           float* __restrict__ partials) {
  float mn[D], mx[D];
  float bad = 0.f;
#pragma unroll
  for (int d = 0; d < D; ++d) { mn[d] = __int_as_float(0x7f800000); mx[d] = -mn[d]; }
  const int64_t units = n / 4;
  const float4* X4 = reinterpret_cast<const float4*>(X);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < units; u += 2 * stride) {
    float4 v[2][D];
    const bool second = u + stride < units;
#pragma unroll
    for (int k = 0; k < D; ++k) v[0][k] = __ldg(X4 + u * D + k);
#pragma unroll
    for (int k = 0; k < D; ++k) v[1][k] = second ? __ldg(X4 + (u + stride) * D + k) : v[0][k];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
#pragma unroll
      for (int k = 0; k < D; ++k) {
        const float e[4] = {v[h][k].x, v[h][k].y, v[h][k].z, v[h][k].w};
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int d = (4 * k + c) % D;
          if (!isfinite(e[c])) bad = 1.f;
          mn[d] = fminf(mn[d], e[c]);
          mx[d] = fmaxf(mx[d], e[c]);
        }
      }
    }
  }
  // tail rows (n % 4)
  if (blockIdx.x == 0 && threadIdx.x < (int)(n - units * 4)) {
    const int64_t r = units * 4 + threadIdx.x;
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const float e = X[r * D + d];
      if (!isfinite(e)) bad = 1.f;
      mn[d] = fminf(mn[d], e);
      mx[d] = fmaxf(mx[d], e);
    }
  }
  __shared__ float s[BBOX_THREADS / 32][2 * F3M_MAXD + 1];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int d = 0; d < D; ++d) {
    for (int o = 16; o > 0; o >>= 1) {
      mn[d] = fminf(mn[d], __shfl_xor_sync(0xffffffffu, mn[d], o));
      mx[d] = fmaxf(mx[d], __shfl_xor_sync(0xffffffffu, mx[d], o));
    }
  }
  for (int o = 16; o > 0; o >>= 1) bad = fmaxf(bad, __shfl_xor_sync(0xffffffffu, bad, o));
  if (lane == 0) {
    for (int d = 0; d < F3M_MAXD; ++d) {
      s[w][d] = d < D ? mn[d] : 0.f;
      s[w][F3M_MAXD + d] = d < D ? mx[d] : 0.f;
    }
    s[w][2 * F3M_MAXD] = bad;
  }
  __syncthreads();
  if (threadIdx.x < 2 * F3M_MAXD + 1) {
    const int k = threadIdx.x;
    float a = s[0][k];
    for (int j = 1; j < BBOX_THREADS / 32; ++j)
      a = (k < F3M_MAXD) ? fminf(a, s[j][k]) : fmaxf(a, s[j][k]);
    partials[(int64_t)blockIdx.x * (2 * F3M_MAXD + 1) + k] = a;
  }
}

__global__ void k_bbox_final(const float* __restrict__ partials, int nblocks, int D, float* __restrict__ out) {
  const int k = threadIdx.x;
  if (k >= 2 * F3M_MAXD + 1) return;
  float a = partials[k];
  for (int j = 1; j < nblocks; ++j) {
    float v = partials[(int64_t)j * (2 * F3M_MAXD + 1) + k];
    a = (k < F3M_MAXD) ? fminf(a, v) : fmaxf(a, v);
  }
  // compact layout [min_0..min_{D-1}, max_0..max_{D-1}, bad]
  if (k < D) out[k] = a;
  else if (k >= F3M_MAXD && k < F3M_MAXD + D) out[D + (k - F3M_MAXD)] = a;
  else if (k == 2 * F3M_MAXD) out[2 * D] = a;
}

void launch_bbox(const float* X, int64_t n, int D, float* partials, int nblocks, cudaStream_t st) {
  if ((reinterpret_cast<uintptr_t>(X) & 15) == 0) {
    switch (D) {
#define CASE(d) case d: k_bbox_vec<d><<<nblocks, BBOX_THREADS, 0, st>>>(X, n, partials); return;
      CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7)
#undef CASE
      default: break;
    }
  }
  k_bbox<<<nblocks, BBOX_THREADS, 0, st>>>(X, n, D, partials);
}
void launch_bbox_final(const float* partials, int nblocks, int D, float* out, cudaStream_t st) {
  k_bbox_final<<<1, 32, 0, st>>>(partials, nblocks, D, out);
}

// ======================================================================================
// bit-exact keys
// ======================================================================================
// Integer cell at depth T of one coordinate (reading R12).  Fast path: q = RN32(RN32(x-a) s)
// differs from the exact fp64 value RN64(RN64(x-a)/E) 2^T by < 2^(T-22) (three fp32
// roundings on |q| <= 2^T plus two fp64 ones); when frac(q) keeps that margin from both
// integers the floor is the same, otherwise the exact fp64 path (the oracle's arithmetic)
// decides.  T >= 22 always takes the exact path.

// (cell_of in keys.cuh; the nested Morton order key of reading R13 -- level groups of D bits,
// most significant level first, dimension d at bit d of its group -- is built by key_from_x.)

// lanes of the warp holding the same digit (<= 8 bits) among `valid` lanes (ballot multisplit)
__device__ __forceinline__ unsigned peers_ballot(uint32_t dig, int bits, unsigned valid) {
  unsigned peers = valid;
#pragma unroll
  for (int b = 0; b < MAX_DIGIT_BITS; ++b) {
    if (b < bits) {
      const unsigned bit = (dig >> b) & 1u;
      const unsigned bal = __ballot_sync(0xffffffffu, bit);
      peers &= bit ? bal : ~bal;
    }
  }
  return peers;
}


// ======================================================================================
// tile histograms (warp-aggregated with __match_any_sync into warp-private SMEM bins)
// counts layout: [bin][tile] so one exclusive scan yields every (bin, tile) destination
// ======================================================================================


// ======================================================================================
// exclusive scan (uint32), reduce-then-scan in three launches
// ======================================================================================
constexpr int SCAN_THREADS = 1024;
constexpr int SCAN_ITEMS = 4;
constexpr int SCAN_BLOCK = SCAN_THREADS * SCAN_ITEMS;

int64_t scan_tmp_words(int64_t len) { return (len + SCAN_BLOCK - 1) / SCAN_BLOCK + 1; }

__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t* warp_tot, uint32_t& total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  uint32_t inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) warp_tot[w] = inc;
  __syncthreads();
  if (w == 0) {
    uint32_t t = lane < nw ? warp_tot[lane] : 0u;
    uint32_t ti = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, ti, o);
      if (lane >= o) ti += y;
    }
    if (lane < nw) warp_tot[lane] = ti - t;
    if (lane == 31) warp_tot[32] = ti;
  }
  __syncthreads();
  const uint32_t r = warp_tot[w] + inc - v;
  total = warp_tot[32];
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(SCAN_THREADS) k_scan_reduce(const uint32_t* __restrict__ a, int64_t len,
                                                              uint32_t* __restrict__ sums) {
  const int64_t base = (int64_t)blockIdx.x * SCAN_BLOCK + threadIdx.x * SCAN_ITEMS;
  uint32_t s = 0;
#pragma unroll
  for (int k = 0; k < SCAN_ITEMS; ++k)
    if (base + k < len) s += a[base + k];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  __shared__ uint32_t ws[32];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    uint32_t t = ws[threadIdx.x];
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (threadIdx.x == 0) sums[blockIdx.x] = t;
  }
}

__global__ void __launch_bounds__(SCAN_THREADS) k_scan_top(uint32_t* __restrict__ sums, int64_t nb) {
  __shared__ uint32_t wt[33];
  uint32_t carry = 0;
  for (int64_t base = 0; base < nb; base += SCAN_THREADS) {
    const int64_t i = base + threadIdx.x;
    uint32_t v = i < nb ? sums[i] : 0u;
    uint32_t tot;
    uint32_t e = block_exclusive_scan(v, wt, tot);
    if (i < nb) sums[i] = e + carry;
    carry += tot;
  }
}

__global__ void __launch_bounds__(SCAN_THREADS) k_scan_down(uint32_t* __restrict__ a, int64_t len,
                                                            const uint32_t* __restrict__ sums) {
  __shared__ uint32_t wt[33];
  const int64_t base = (int64_t)blockIdx.x * SCAN_BLOCK + threadIdx.x * SCAN_ITEMS;
  uint32_t v[SCAN_ITEMS];
  uint32_t s = 0;
#pragma unroll
  for (int k = 0; k < SCAN_ITEMS; ++k) {
    v[k] = (base + k < len) ? a[base + k] : 0u;
    s += v[k];
  }
  uint32_t tot;
  uint32_t e = block_exclusive_scan(s, wt, tot) + sums[blockIdx.x];
#pragma unroll
  for (int k = 0; k < SCAN_ITEMS; ++k) {
    if (base + k < len) a[base + k] = e;
    e += v[k];
  }
}

void launch_scan_u32(uint32_t* data, int64_t len, uint32_t* tmp, cudaStream_t st) {
  const int64_t nb = (len + SCAN_BLOCK - 1) / SCAN_BLOCK;
  if (nb <= 0) return;
  k_scan_reduce<<<(unsigned)nb, SCAN_THREADS, 0, st>>>(data, len, tmp);
  k_scan_top<<<1, SCAN_THREADS, 0, st>>>(tmp, nb);
  k_scan_down<<<(unsigned)nb, SCAN_THREADS, 0, st>>>(data, len, tmp);
}

constexpr int NB_MAX = 1 << MAX_DIGIT_BITS;

// ======================================================================================
// LSD counting-sort pass with stored tile orders (multi-pass sorts, D T_sort > 8 bits).
//   k_lsd_rank:    per 4096-point tile, the digit of every point, its stable rank (ballot
//                  multisplit, warp-private histograms, bin-major scan), the tile's bin counts
//                  [bin][tile] and its order (sorted position -> original local index).
//   k_lsd_scatter: per tile, each payload array is staged in shared memory once (coalesced
//                  loads) and written as contiguous per-bin runs (one warp per bin) at the
//                  scanned destinations: every global access is coalesced.
// ======================================================================================
constexpr int LSD_THREADS = 512;
constexpr int LSD_WARPS = LSD_THREADS / 32;
constexpr int LSD_ITEMS = 8;
constexpr int LSD_TILE = LSD_THREADS * LSD_ITEMS;  // 4096
constexpr int LSD_WP = LSD_WARPS + 1;

template <int D>
__device__ __forceinline__ uint64_t key_from_x(const float* x, const KeyParams& kp) {
  uint64_t c[D];
#pragma unroll
  for (int d = 0; d < D; ++d) c[d] = cell_of(x[d], d, kp);
  uint64_t K = 0;
  for (int sl = kp.T - 1; sl >= 0; --sl)
#pragma unroll
    for (int d = D - 1; d >= 0; --d) K = (K << 1) | ((c[d] >> sl) & 1ull);
  return K;
}

template <bool FIRST, int D>
__global__ void __launch_bounds__(LSD_THREADS) k_lsd_rank(const float* __restrict__ X, const uint64_t* __restrict__ keys,
                                                          int64_t n, KeyParams kp, int shift, int bits, int num_tiles,
                                                          uint32_t* __restrict__ counts, uint16_t* __restrict__ order) {
  __shared__ uint32_t whist[NB_MAX * LSD_WP];
  __shared__ uint32_t wt[33];
  __shared__ __align__(16) uint16_t sorig[LSD_TILE];
  const int nb = 1 << bits;
  const uint32_t mask = (uint32_t)nb - 1u;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  const int tile = blockIdx.x;
  const int64_t tile0 = (int64_t)tile * LSD_TILE;
  const int tvalid = (int)min((int64_t)LSD_TILE, n - tile0);
  const int segl = w * (LSD_TILE / LSD_WARPS);
  for (int b = lane; b < nb; b += 32) whist[b * LSD_WP + w] = 0;
  __syncwarp();
  uint32_t dig[LSD_ITEMS];
  int wrank[LSD_ITEMS];
#pragma unroll
  for (int j = 0; j < LSD_ITEMS; ++j) {
    const int o = segl + j * 32 + lane;
    const bool valid = o < tvalid;
    uint64_t K = 0;
    if (valid) {
      if (FIRST) {
        float x[D];
#pragma unroll
        for (int d = 0; d < D; ++d) x[d] = __ldg(X + (tile0 + o) * D + d);
        K = key_from_x<D>(x, kp);
      } else {
        K = keys[tile0 + o];
      }
    }
    dig[j] = (uint32_t)(K >> shift) & mask;
  }
#pragma unroll
  for (int j = 0; j < LSD_ITEMS; ++j) {
    const bool valid = segl + j * 32 + lane < tvalid;
    const unsigned vm = __ballot_sync(0xffffffffu, valid);
    const unsigned peers = peers_ballot(dig[j], bits, vm);
    wrank[j] = valid ? (int)(whist[dig[j] * LSD_WP + w] + __popc(peers & lt)) : -1;
    __syncwarp();
    if (valid && (peers & lt) == 0) whist[dig[j] * LSD_WP + w] += __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  // exclusive scan of whist in bin-major order (bin, warp): nb * 16 <= 4096 entries
  {
    const int E = nb * LSD_WARPS;
    const int K = (E + LSD_THREADS - 1) / LSD_THREADS;  // <= 8
    const int e0 = threadIdx.x * K;
    uint32_t loc[8];
    uint32_t sum = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int e = e0 + q;
      loc[q] = (q < K && e < E) ? whist[(e / LSD_WARPS) * LSD_WP + (e % LSD_WARPS)] : 0u;
      sum += loc[q];
    }
    uint32_t tot;
    uint32_t run = block_exclusive_scan(sum, wt, tot);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int e = e0 + q;
      if (q < K && e < E) {
        whist[(e / LSD_WARPS) * LSD_WP + (e % LSD_WARPS)] = run;
        run += loc[q];
      }
    }
  }
  __syncthreads();
  for (int b = threadIdx.x; b < nb; b += LSD_THREADS) {
    const uint32_t st0 = whist[b * LSD_WP];
    const uint32_t nx = b + 1 < nb ? whist[(b + 1) * LSD_WP] : (uint32_t)tvalid;
    counts[(int64_t)b * num_tiles + tile] = nx - st0;
  }
#pragma unroll
  for (int j = 0; j < LSD_ITEMS; ++j)
    if (wrank[j] >= 0) sorig[whist[dig[j] * LSD_WP + w] + wrank[j]] = (uint16_t)(segl + j * 32 + lane);
  __syncthreads();
  if (tvalid == LSD_TILE) {
    reinterpret_cast<uint4*>(order + tile0)[threadIdx.x] = reinterpret_cast<const uint4*>(sorig)[threadIdx.x];
  } else {
    for (int e = threadIdx.x; e < tvalid; e += LSD_THREADS) order[tile0 + e] = sorig[e];
  }
}

template <bool FIRST, int D>
__global__ void __launch_bounds__(LSD_THREADS) k_lsd_scatter(ScatterIO io, int64_t n, KeyParams kp, int bits,
                                                             int num_tiles, const uint32_t* __restrict__ offsets,
                                                             const uint16_t* __restrict__ order) {
  extern __shared__ __align__(16) unsigned char lsm[];
  const int nb = 1 << bits;
  uint16_t* so = reinterpret_cast<uint16_t*>(lsm);                  // [TILE]
  uint32_t* lstart = reinterpret_cast<uint32_t*>(so + LSD_TILE);    // [nb]
  uint32_t* ltot = lstart + NB_MAX;
  uint32_t* goff = ltot + NB_MAX;
  uint32_t* wt = goff + NB_MAX;                                      // [33]
  float* xb = reinterpret_cast<float*>(wt + 36);                     // FIRST: [TILE * D] row-major x; else [TILE * 2]
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int tile = blockIdx.x;
  const int64_t tile0 = (int64_t)tile * LSD_TILE;
  const int tvalid = (int)min((int64_t)LSD_TILE, n - tile0);
  const int64_t scan_len = (int64_t)nb * num_tiles;
  for (int e = threadIdx.x; e < tvalid; e += LSD_THREADS) so[e] = order[tile0 + e];
  for (int b = threadIdx.x; b < nb; b += LSD_THREADS) {
    const int64_t idx = (int64_t)b * num_tiles + tile;
    const uint32_t cur = offsets[idx];
    const uint32_t nxt = (idx + 1 < scan_len) ? offsets[idx + 1] : (uint32_t)n;
    ltot[b] = nxt - cur;
    goff[b] = cur;
  }
  __syncthreads();
  {
    const uint32_t v = threadIdx.x < nb ? ltot[threadIdx.x] : 0u;
    uint32_t tot;
    const uint32_t e = block_exclusive_scan(v, wt, tot);
    if (threadIdx.x < nb) lstart[threadIdx.x] = e;
  }
  __syncthreads();
  // one warp per bin: sorted position q = lstart + e -> source local index so[q]; a skewed tile
  // (one bin > 1/8 of it) goes position-parallel with a binary search for the bin instead
  const bool skew = __syncthreads_or(threadIdx.x < nb && ltot[threadIdx.x] > LSD_TILE / 8);
  auto bin_of = [&](int q) {  // the largest b with lstart[b] <= q (a non-empty bin)
    int lo = 0, hi = nb;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if ((int)lstart[mid] <= q) lo = mid;
      else hi = mid;
    }
    return lo;
  };
  auto emit32 = [&](const uint32_t* src, uint32_t* dst) {  // src: the tile's values in smem
    if (skew) {
      for (int q = threadIdx.x; q < tvalid; q += LSD_THREADS) {
        const int b = bin_of(q);
        dst[goff[b] + (uint32_t)(q - (int)lstart[b])] = src[so[q]];
      }
      return;
    }
    for (int b = w; b < nb; b += LSD_WARPS) {
      const int ls = (int)lstart[b], ln = (int)ltot[b];
      uint32_t* out = dst + goff[b];
      for (int e = lane; e < ln; e += 32) out[e] = src[so[ls + e]];
    }
  };
  uint32_t* buf = reinterpret_cast<uint32_t*>(xb);
  if (FIRST) {
    for (int e = threadIdx.x; e < tvalid * D; e += LSD_THREADS) xb[e] = __ldg(io.X + tile0 * D + e);
    // a tile whose points crowd into a few bins (clustered, BM, fBm data) would leave one warp
    // per crowded bin doing most of the tile: there every thread takes sorted positions
    // q = tid + k THREADS and finds its bin by a binary search over the bin starts
    __syncthreads();
    auto emit_one = [&](int b, int e) {
      const int o = so[(int)lstart[b] + e];
      const uint32_t dst = goff[b] + (uint32_t)e;
      io.perm_out[dst] = (int32_t)(tile0 + o);
      float x[D];
#pragma unroll
      for (int d = 0; d < D; ++d) {
        x[d] = xb[o * D + d];
        io.xs_out[(int64_t)d * n + dst] = x[d];
      }
      if (io.keys_out) io.keys_out[dst] = key_from_x<D>(x, kp);
      if (io.bs_out) io.bs_out[dst] = __ldg(io.b + tile0 + o);
    };
    if (skew) {
      for (int q = threadIdx.x; q < tvalid; q += LSD_THREADS) {
        const int b = bin_of(q);
        emit_one(b, q - (int)lstart[b]);
      }
    } else {
      for (int b = w; b < nb; b += LSD_WARPS) {
        const int ln = (int)ltot[b];
        for (int e = lane; e < ln; e += 32) emit_one(b, e);
      }
    }
  } else {
    // perm, the D coordinate arrays, b: one shared staging buffer per payload.  [Double buffering
    // (payload j + 1 loaded into registers while j is emitted) measured no change: 3.73 ms for the
    // second pass at D = 7, n = 1e8 -- the scattered 128-byte bin runs of the writes bound it.]
    for (int e = threadIdx.x; e < tvalid; e += LSD_THREADS) buf[e] = (uint32_t)io.perm_in[tile0 + e];
    __syncthreads();
    emit32(buf, reinterpret_cast<uint32_t*>(io.perm_out));
    __syncthreads();
    for (int d = 0; d < D; ++d) {
      for (int e = threadIdx.x; e < tvalid; e += LSD_THREADS) buf[e] = __float_as_uint(io.xs_in[(int64_t)d * n + tile0 + e]);
      __syncthreads();
      emit32(buf, reinterpret_cast<uint32_t*>(io.xs_out + (int64_t)d * n));
      __syncthreads();
    }
    if (io.bs_out) {
      for (int e = threadIdx.x; e < tvalid; e += LSD_THREADS) buf[e] = __float_as_uint(io.bs_in[tile0 + e]);
      __syncthreads();
      emit32(buf, reinterpret_cast<uint32_t*>(io.bs_out));
      __syncthreads();
    }
    if (io.keys_out) {
      uint2* kb = reinterpret_cast<uint2*>(buf);
      for (int e = threadIdx.x; e < tvalid; e += LSD_THREADS) {
        const uint64_t k = io.keys_in[tile0 + e];
        kb[e] = make_uint2((uint32_t)k, (uint32_t)(k >> 32));
      }
      __syncthreads();
      uint2* ko = reinterpret_cast<uint2*>(io.keys_out);
      if (skew) {
        for (int q = threadIdx.x; q < tvalid; q += LSD_THREADS) {
          const int b = bin_of(q);
          ko[goff[b] + (uint32_t)(q - (int)lstart[b])] = kb[so[q]];
        }
      } else {
        for (int b = w; b < nb; b += LSD_WARPS) {
          const int ls = (int)lstart[b], ln = (int)ltot[b];
          uint2* out = ko + goff[b];
          for (int e = lane; e < ln; e += 32) out[e] = kb[so[ls + e]];
        }
      }
    }
  }
}

// Two-digit (MSD) path, first digit: the stable counting-sort scatter of one 4096-point tile into
// top-digit buckets laid out on whole tiles (bucket b starts pad[b] past its packed offset, so every
// bucket begins on a tile boundary and is TMA-aligned): row-major coordinates and the weights,
// staged in shared memory and written as per-bin coalesced runs (one warp per bin).
template <int D>
__global__ void __launch_bounds__(LSD_THREADS) k_scatter_msd(const float* __restrict__ X, const float* __restrict__ b,
                                                             int64_t n, int bits, int num_tiles,
                                                             const uint32_t* __restrict__ offsets,
                                                             const uint32_t* __restrict__ pad,
                                                             const uint16_t* __restrict__ order, float* __restrict__ xp,
                                                             float* __restrict__ bp) {
  extern __shared__ __align__(16) unsigned char msm[];
  const int nb = 1 << bits;
  uint16_t* so = reinterpret_cast<uint16_t*>(msm);                  // [TILE]
  uint32_t* lstart = reinterpret_cast<uint32_t*>(so + LSD_TILE);    // [NB_MAX]
  uint32_t* ltot = lstart + NB_MAX;
  uint32_t* goff = ltot + NB_MAX;
  uint32_t* wt = goff + NB_MAX;                                      // [36]
  float* xb = reinterpret_cast<float*>(wt + 36);                     // [TILE * D]
  float* bb = xb + LSD_TILE * D;                                     // [TILE]
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int tile = blockIdx.x;
  const int64_t tile0 = (int64_t)tile * LSD_TILE;
  const int tvalid = (int)min((int64_t)LSD_TILE, n - tile0);
  const int64_t scan_len = (int64_t)nb * num_tiles;
  for (int e = threadIdx.x; e < tvalid; e += LSD_THREADS) so[e] = order[tile0 + e];
  for (int e = threadIdx.x; e < tvalid * D; e += LSD_THREADS) xb[e] = __ldg(X + tile0 * D + e);
  for (int e = threadIdx.x; e < tvalid; e += LSD_THREADS) bb[e] = __ldg(b + tile0 + e);
  for (int q = threadIdx.x; q < nb; q += LSD_THREADS) {
    const int64_t idx = (int64_t)q * num_tiles + tile;
    const uint32_t cur = offsets[idx];
    const uint32_t nxt = (idx + 1 < scan_len) ? offsets[idx + 1] : (uint32_t)n;
    ltot[q] = nxt - cur;
    goff[q] = cur + pad[q];
  }
  __syncthreads();
  {
    const uint32_t v = threadIdx.x < nb ? ltot[threadIdx.x] : 0u;
    uint32_t tot;
    const uint32_t e = block_exclusive_scan(v, wt, tot);
    if (threadIdx.x < nb) lstart[threadIdx.x] = e;
  }
  __syncthreads();
  for (int q = w; q < nb; q += LSD_WARPS) {
    const int ls = (int)lstart[q], ln = (int)ltot[q];
    const int64_t g0 = goff[q];
    for (int e = lane; e < ln; e += 32) {
      const int o = so[ls + e];
      const int64_t dst = g0 + e;
#pragma unroll
      for (int d = 0; d < D; ++d) xp[dst * D + d] = xb[o * D + d];
      bp[dst] = bb[o];
    }
  }
}

void launch_scatter_msd(int D, const float* X, const float* b, int64_t n, int bits, int num_tiles,
                        const uint32_t* offsets, const uint32_t* pad, const uint16_t* order, float* xp, float* bp,
                        cudaStream_t st) {
  if (num_tiles <= 0) return;
  const size_t sm = (size_t)LSD_TILE * 2 + 4 * (3 * NB_MAX + 36) + (size_t)LSD_TILE * (D + 1) * 4;
#define X_(d)                                                                                        \
  if (D == d) {                                                                                      \
    cudaFuncSetAttribute(k_scatter_msd<d>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);    \
    k_scatter_msd<d><<<num_tiles, LSD_THREADS, sm, st>>>(X, b, n, bits, num_tiles, offsets, pad, order, xp, bp); \
    return;                                                                                          \
  }
  X_(1) X_(2) X_(3)
#undef X_
}

// Inverse of one LSD pass for a per-point result: out[i] (pass input order) = in[dst(i)]
// (pass output order).  Per tile, one warp per bin reads the bin's contiguous run of `in`
// (coalesced) and stages it in shared memory by original local index; the tile then leaves
// coalesced.  Undoing the passes in reverse replaces a random-scatter un-permutation.
// FWD: the pass itself on a float payload (out = the pass's output order of `in`): the tile is
// read coalesced into shared memory and every bin's run leaves as one contiguous store run.
template <bool FWD>
__global__ void __launch_bounds__(LSD_THREADS) k_lsd_unscatter(const float* __restrict__ in, float* __restrict__ out,
                                                               int64_t n, int bits, int num_tiles,
                                                               const uint32_t* __restrict__ offsets,
                                                               const uint16_t* __restrict__ order,
                                                               const uint32_t* __restrict__ pad) {
  __shared__ __align__(16) uint16_t so[LSD_TILE];
  __shared__ __align__(16) float buf[LSD_TILE];
  __shared__ uint32_t lstart[NB_MAX], ltot[NB_MAX], goff[NB_MAX], wt[36];
  const int nb = 1 << bits;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int tile = blockIdx.x;
  const int64_t tile0 = (int64_t)tile * LSD_TILE;
  const int tvalid = (int)min((int64_t)LSD_TILE, n - tile0);
  const int64_t scan_len = (int64_t)nb * num_tiles;
  for (int e = threadIdx.x; e < tvalid; e += LSD_THREADS) so[e] = order[tile0 + e];
  for (int b = threadIdx.x; b < nb; b += LSD_THREADS) {
    const int64_t idx = (int64_t)b * num_tiles + tile;
    const uint32_t cur = offsets[idx];
    const uint32_t nxt = (idx + 1 < scan_len) ? offsets[idx + 1] : (uint32_t)n;
    ltot[b] = nxt - cur;
    goff[b] = cur + (pad ? pad[b] : 0u);  // padded layout: runs of bin b start pad[b] later
  }
  __syncthreads();
  {
    const uint32_t v = threadIdx.x < nb ? ltot[threadIdx.x] : 0u;
    uint32_t tot;
    const uint32_t e = block_exclusive_scan(v, wt, tot);
    if (threadIdx.x < nb) lstart[threadIdx.x] = e;
  }
  __syncthreads();
  // skewed tile (one bin > 1/8 of it): position-parallel with a binary search for the bin
  const bool skew = __syncthreads_or(threadIdx.x < nb && ltot[threadIdx.x] > LSD_TILE / 8);
  auto bin_of = [&](int q) {
    int lo = 0, hi = nb;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if ((int)lstart[mid] <= q) lo = mid;
      else hi = mid;
    }
    return lo;
  };
  if constexpr (FWD) {
    for (int e = threadIdx.x; e < tvalid; e += LSD_THREADS) buf[e] = in[tile0 + e];
    __syncthreads();
    if (skew) {
      for (int q = threadIdx.x; q < tvalid; q += LSD_THREADS) {
        const int b = bin_of(q);
        out[goff[b] + (uint32_t)(q - (int)lstart[b])] = buf[so[q]];
      }
    } else {
      for (int b = w; b < nb; b += LSD_WARPS) {
        const int ls = (int)lstart[b], ln = (int)ltot[b];
        float* dst = out + goff[b];
        for (int e = lane; e < ln; e += 32) dst[e] = buf[so[ls + e]];
      }
    }
  } else {
    if (skew) {
      for (int q = threadIdx.x; q < tvalid; q += LSD_THREADS) {
        const int b = bin_of(q);
        buf[so[q]] = in[goff[b] + (uint32_t)(q - (int)lstart[b])];
      }
    } else {
      for (int b = w; b < nb; b += LSD_WARPS) {
        const int ls = (int)lstart[b], ln = (int)ltot[b];
        const float* src = in + goff[b];
        for (int e = lane; e < ln; e += 32) buf[so[ls + e]] = src[e];
      }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < tvalid; e += LSD_THREADS) out[tile0 + e] = buf[e];
  }
}

void launch_lsd_unscatter(const float* in, float* out, int64_t n, int bits, int num_tiles, const uint32_t* offsets,
                          const uint16_t* order, cudaStream_t st, const uint32_t* pad) {
  if (num_tiles <= 0) return;
  k_lsd_unscatter<false><<<num_tiles, LSD_THREADS, 0, st>>>(in, out, n, bits, num_tiles, offsets, order, pad);
}

void launch_lsd_rescatter(const float* in, float* out, int64_t n, int bits, int num_tiles, const uint32_t* offsets,
                          const uint16_t* order, cudaStream_t st) {
  if (num_tiles <= 0) return;
  k_lsd_unscatter<true><<<num_tiles, LSD_THREADS, 0, st>>>(in, out, n, bits, num_tiles, offsets, order, nullptr);
}

// out[i] = in[idx[i]]
__global__ void k_gather_u32(const uint32_t* __restrict__ in, const int64_t* __restrict__ idx, int64_t n,
                             uint32_t* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = in[idx[i]];
}

// two-digit path: per tile of the padded bucket layout, {bucket | valid points << 8, tile of
// the bucket} (bucket = the largest k with tile0[k] <= g, a non-empty bucket)
__global__ void k_bucket_tiles(const int32_t* __restrict__ tile0, const int64_t* __restrict__ nb_pts, int nbuckets,
                               int ntiles, int2* __restrict__ out) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= ntiles) return;
  int lo = 0, hi = nbuckets;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (tile0[mid] <= g) lo = mid;
    else hi = mid;
  }
  const int lt = g - tile0[lo];
  const int64_t rem = nb_pts[lo] - (int64_t)lt * 4096;
  const int tv = (int)(rem < 4096 ? rem : 4096);
  out[g] = make_int2(lo | (tv << 8), lt);
}

void launch_bucket_tiles(const int32_t* tile0, const int64_t* nb_pts, int nbuckets, int ntiles, int2* out,
                         cudaStream_t st) {
  if (ntiles <= 0) return;
  k_bucket_tiles<<<(ntiles + 255) / 256, 256, 0, st>>>(tile0, nb_pts, nbuckets, ntiles, out);
}

void launch_gather_u32(const uint32_t* in, const int64_t* idx, int64_t n, uint32_t* out, cudaStream_t st) {
  if (n <= 0) return;
  k_gather_u32<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(in, idx, n, out);
}

int lsd_tile() { return LSD_TILE; }

void launch_lsd_rank(bool first, const float* X, const uint64_t* keys, int64_t n, int D, const KeyParams& kp, int shift,
                     int bits, int num_tiles, uint32_t* counts, uint16_t* order, cudaStream_t st) {
#define X_(d)                                                                                                   \
  if (D == d) {                                                                                                 \
    if (first) k_lsd_rank<true, d><<<num_tiles, LSD_THREADS, 0, st>>>(X, keys, n, kp, shift, bits, num_tiles, counts, order); \
    else k_lsd_rank<false, d><<<num_tiles, LSD_THREADS, 0, st>>>(X, keys, n, kp, shift, bits, num_tiles, counts, order);     \
    return;                                                                                                     \
  }
  X_(1) X_(2) X_(3) X_(4) X_(5) X_(6) X_(7)
#undef X_
}

void launch_lsd_scatter(bool first, const ScatterIO& io, int64_t n, int D, const KeyParams& kp, int bits, int num_tiles,
                        const uint32_t* offsets, const uint16_t* order, cudaStream_t st) {
  const size_t base = (size_t)LSD_TILE * 2 + 4 * (3 * NB_MAX + 36);
  const size_t sm = base + (first ? (size_t)LSD_TILE * D * 4 : (size_t)LSD_TILE * 8);
#define X_(d)                                                                                                    \
  if (D == d) {                                                                                                  \
    if (first) {                                                                                                 \
      cudaFuncSetAttribute(k_lsd_scatter<true, d>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);        \
      k_lsd_scatter<true, d><<<num_tiles, LSD_THREADS, sm, st>>>(io, n, kp, bits, num_tiles, offsets, order);     \
    } else {                                                                                                     \
      cudaFuncSetAttribute(k_lsd_scatter<false, d>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);       \
      k_lsd_scatter<false, d><<<num_tiles, LSD_THREADS, sm, st>>>(io, n, kp, bits, num_tiles, offsets, order);    \
    }                                                                                                            \
    return;                                                                                                      \
  }
  X_(1) X_(2) X_(3) X_(4) X_(5) X_(6) X_(7)
#undef X_
}


// ======================================================================================
// small elementwise kernels
// ======================================================================================
__global__ void k_key_heads(const uint64_t* __restrict__ keys, int64_t n, uint32_t* __restrict__ flags) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j <= n; j += (int64_t)gridDim.x * blockDim.x)
    flags[j] = (j < n && (j == 0 || keys[j] != keys[j - 1])) ? 1u : 0u;
}
__global__ void k_compact_heads(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ fs, int64_t n,
                                uint64_t* __restrict__ box_key, int64_t* __restrict__ box_start) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    if (fs[j + 1] != fs[j]) {
      box_key[fs[j]] = keys[j];
      box_start[fs[j]] = j;
    }
  }
}
// 8 independent gathers in flight per thread (the gather is latency-bound)
__global__ void k_unpermute(const float* __restrict__ vs, const int32_t* __restrict__ sigma, int64_t n,
                            float* __restrict__ v) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < n; i0 += 8 * stride) {
    int32_t s[8];
    float r[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) s[k] = (i0 + k * stride < n) ? __ldg(sigma + i0 + k * stride) : 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) r[k] = (i0 + k * stride < n) ? __ldg(vs + s[k]) : 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (i0 + k * stride < n) v[i0 + k * stride] = r[k];
  }
}
// sigma-free un-permutation: v[pi[j]] = vs[j] (coalesced reads, one random 4-byte write each)
__global__ void k_unpermute_perm(const float* __restrict__ vs, const int32_t* __restrict__ perm, int64_t n,
                                 float* __restrict__ v) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
    v[perm[j]] = vs[j];
}
__global__ void k_to_soa(const float* __restrict__ X, int64_t n, int D, float* __restrict__ xs) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n * D; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / D;
    const int d = (int)(e - i * D);
    xs[(int64_t)d * n + i] = X[e];
  }
}

static inline unsigned grid_for(int64_t work, int threads) {
  int64_t g = (work + threads - 1) / threads;
  if (g > 148 * 16) g = 148 * 16;
  if (g < 1) g = 1;
  return (unsigned)g;
}

void launch_key_heads(const uint64_t* keys, int64_t n, uint32_t* flags, cudaStream_t st) {
  k_key_heads<<<grid_for(n + 1, 256), 256, 0, st>>>(keys, n, flags);
}
void launch_compact_heads(const uint64_t* keys, const uint32_t* fs, int64_t n, uint64_t* box_key,
                          int64_t* box_start, cudaStream_t st) {
  k_compact_heads<<<grid_for(n, 256), 256, 0, st>>>(keys, fs, n, box_key, box_start);
}
void launch_unpermute(const float* vs, const int32_t* sigma, int64_t n, float* v, cudaStream_t st) {
  k_unpermute<<<grid_for(n, 256), 256, 0, st>>>(vs, sigma, n, v);
}
void launch_unpermute_perm(const float* vs, const int32_t* perm, int64_t n, float* v, cudaStream_t st) {
  k_unpermute_perm<<<grid_for(n, 256), 256, 0, st>>>(vs, perm, n, v);
}
void launch_to_soa(const float* X, int64_t n, int D, float* xs, cudaStream_t st) {
  k_to_soa<<<grid_for(n * D, 256), 256, 0, st>>>(X, n, D, xs);
}

}  // namespace f3m
