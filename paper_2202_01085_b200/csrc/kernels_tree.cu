// Interaction division + classification on the device (App. F Algorithm 1, PAPER.md:724-733;
// Sec. 4.1 Fig. 6 "dividing the interaction"; far criterion Sec. 3
// PAPER.md:135; smoothness Sec. 4.3; adaptive far field PAPER.md:240-250;
// small field Sec. 4.2).
//
// One depth t.  The near list of depth t-1 is a set of runs (one run per parent target box p,
// partners q_r ascending).  Candidate c of a run enumerates, in the canonical order of the
// oracle (R9):
//     for pc in children(p):  for r in run:  for qc in children(q_r)
// so c = base_run + i * Q_run + S_r + j with Q_run = sum_r nchild(q_r), S_r its exclusive
// prefix inside the run.  Every candidate is classified with the precedence far > smooth >
// small > near (reading R11) using the same fp64 operations as the host / oracle (dist2 is
// summed left to right with explicitly rounded multiplies and adds: no FMA contraction).
//
// Stable 5-way partition: a counting pass writes per-block class counts (blocks of
// DIV_BLOCK candidates), the host scans them, and a scatter pass recomputes each candidate and
// writes it into its list at (block offset + rank inside the block).  Ranks come from one
// block-wide exclusive scan of five 12-bit counters packed in a uint64.
#include <cuda_runtime.h>
#include <stdint.h>

#include "f3m_internal.h"

namespace f3m {

constexpr int DIV_THREADS = 512;
constexpr int DIV_ITEMS = 4;
constexpr int DIV_BLOCK = DIV_THREADS * DIV_ITEMS;  // 2048 < 2^12: five 12-bit counters fit a u64
static_assert(DIV_BLOCK < 4096, "packed 12-bit class counters");

__device__ __forceinline__ int div_class(const DivArgs& a, int32_t pc, int32_t qc) {
  double dist2 = 0.0, distmax = 0.0;
#pragma unroll
  for (int d = 0; d < F3M_MAXD; ++d) {
    if (d < a.D) {
      const double o = __dadd_rn((double)(a.cellX[(int64_t)pc * F3M_MAXD + d] - a.cellY[(int64_t)qc * F3M_MAXD + d]),
                                 a.delta[d]);
      dist2 = __dadd_rn(dist2, __dmul_rn(o, o));
      distmax = fmax(distmax, fabs(o));
    }
  }
  const bool far = a.maxnorm ? distmax >= 2.0 : dist2 >= 4.0;         // ||c_p - c_q|| >= 2l
  if (far) return a.pfar > 0 ? DIV_FAR : DIV_DROP;
  if (a.smooth_level) return DIV_SMOOTH;                               // level-wide O(1) bound
  if (!a.no_small && a.gX[pc] + a.gY[qc] <= a.rho) return DIV_SMALL;  // #B_p + #B_q <= rho
  return DIV_NEAR;
}

// candidate index -> (pc, qc)
__device__ __forceinline__ void div_decode(const DivArgs& a, uint64_t c, int32_t& pc, int32_t& qc) {
  int lo = 0, hi = a.nruns - 1;  // last run with base <= c
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (a.run_base[mid] <= c) lo = mid;
    else hi = mid - 1;
  }
  const int run = lo;
  const uint64_t local = c - a.run_base[run];
  const uint32_t Q = a.run_Q[run];
  const uint32_t i = (uint32_t)(local / Q);
  const uint32_t rem = (uint32_t)(local - (uint64_t)i * Q);
  int r0 = a.run_r0[run], r1 = a.run_r0[run + 1] - 1;  // last pair r with S_r <= rem
  while (r0 < r1) {
    const int mid = (r0 + r1 + 1) >> 1;
    if (a.pair_S[mid] <= rem) r0 = mid;
    else r1 = mid - 1;
  }
  pc = a.childX0[a.run_p[run]] + (int32_t)i;
  qc = a.childY0[a.pair_q[r0]] + (int32_t)(rem - a.pair_S[r0]);
}

__device__ __forceinline__ uint64_t cls_unit(int cls) { return 1ull << (12 * cls); }

template <bool SCATTER>
__global__ void __launch_bounds__(DIV_THREADS) k_divide(DivArgs a) {
  const uint64_t base = (uint64_t)blockIdx.x * DIV_BLOCK + (uint64_t)threadIdx.x * DIV_ITEMS;
  int32_t pc[DIV_ITEMS], qc[DIV_ITEMS];
  int cls[DIV_ITEMS];
  uint64_t mine = 0;
#pragma unroll
  for (int k = 0; k < DIV_ITEMS; ++k) {
    cls[k] = -1;
    if (base + k < a.M) {
      div_decode(a, base + k, pc[k], qc[k]);
      cls[k] = div_class(a, pc[k], qc[k]);
      mine += cls_unit(cls[k]);
      if (!SCATTER && a.dbg_tag) {
        a.dbg_pc[base + k] = pc[k];
        a.dbg_qc[base + k] = qc[k];
        a.dbg_tag[base + k] = (int8_t)cls[k];
      }
    }
  }
  // block exclusive scan of the packed counters
  __shared__ uint64_t wsum[DIV_THREADS / 32 + 1];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint64_t inc = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) wsum[w] = inc;
  __syncthreads();
  if (w == 0) {
    const uint64_t v = lane < DIV_THREADS / 32 ? wsum[lane] : 0ull;
    uint64_t vi = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t y = __shfl_up_sync(0xffffffffu, vi, o);
      if (lane >= o) vi += y;
    }
    if (lane < DIV_THREADS / 32) wsum[lane] = vi - v;
    if (lane == 31) wsum[DIV_THREADS / 32] = vi;
  }
  __syncthreads();
  if (!SCATTER) {
    if (threadIdx.x < DIV_NCLS) {
      const uint64_t tot = wsum[DIV_THREADS / 32];
      a.blockcnt[(uint64_t)blockIdx.x * DIV_NCLS + threadIdx.x] = (uint32_t)((tot >> (12 * threadIdx.x)) & 0xfffu);
    }
    return;
  }
  uint64_t run = wsum[w] + inc - mine;  // exclusive prefix of this thread's first item
#pragma unroll
  for (int k = 0; k < DIV_ITEMS; ++k) {
    if (cls[k] < 0) continue;
    const uint32_t rank = (uint32_t)((run >> (12 * cls[k])) & 0xfffu);
    run += cls_unit(cls[k]);
    const int list = a.cls_list[cls[k]];
    if (list < 0) continue;
    // merged lists (far + smooth at the same node count) rank by both classes
    uint32_t pos = a.blockoff[(uint64_t)blockIdx.x * DIV_NCLS + cls[k]] + rank;
    const int other = a.cls_merge[cls[k]];
    if (other >= 0) pos += (uint32_t)((run - cls_unit(cls[k])) >> (12 * other) & 0xfffu);
    a.outP[list][pos] = pc[k];
    a.outQ[list][pos] = qc[k];
  }
}

// ---- far-group CSR on the device (consumers: M2L) ---------------------------------------
// mark used target / source boxes, count pairs per target, offset ranges per dimension
__global__ void k_far_marks(const int32_t* __restrict__ P, const int32_t* __restrict__ Q, int64_t n,
                            const int32_t* __restrict__ cellX, const int32_t* __restrict__ cellY, int D,
                            uint32_t* __restrict__ tcount, uint32_t* __restrict__ smark, int* __restrict__ omin,
                            int* __restrict__ omax) {
  int lmin[F3M_MAXD], lmax[F3M_MAXD];
#pragma unroll
  for (int d = 0; d < F3M_MAXD; ++d) { lmin[d] = INT32_MAX; lmax[d] = INT32_MIN; }
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int32_t p = P[e], q = Q[e];
    // the list is sorted by target: each target's run head records the run start (no atomics;
    // the host turns the starts into the CSR pointer)
    if (e == 0 || P[e - 1] != p) tcount[p] = (uint32_t)e;
    smark[q] = 1u;
#pragma unroll
    for (int d = 0; d < F3M_MAXD; ++d)
      if (d < D) {
        const int o = cellX[(int64_t)p * F3M_MAXD + d] - cellY[(int64_t)q * F3M_MAXD + d];
        lmin[d] = min(lmin[d], o);
        lmax[d] = max(lmax[d], o);
      }
  }
#pragma unroll
  for (int d = 0; d < F3M_MAXD; ++d)
    if (d < D) {
      int a = lmin[d], b = lmax[d];
      for (int o = 16; o > 0; o >>= 1) {
        a = min(a, __shfl_xor_sync(0xffffffffu, a, o));
        b = max(b, __shfl_xor_sync(0xffffffffu, b, o));
      }
      if ((threadIdx.x & 31) == 0) {
        atomicMin(&omin[d], a);
        atomicMax(&omax[d], b);
      }
    }
}

// col = source slot (exclusive scan of the source marks), packed per-dimension offset index
__global__ void k_far_cols(const int32_t* __restrict__ P, const int32_t* __restrict__ Q, int64_t n,
                           const int32_t* __restrict__ cellX, const int32_t* __restrict__ cellY, int D,
                           const uint32_t* __restrict__ sslot, const int* __restrict__ omin, int32_t* __restrict__ col,
                           uint64_t* __restrict__ off) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int32_t p = P[e], q = Q[e];
    col[e] = (int32_t)sslot[q];
    uint64_t pk = 0;
    for (int d = 0; d < D; ++d)
      pk |= (uint64_t)(cellX[(int64_t)p * F3M_MAXD + d] - cellY[(int64_t)q * F3M_MAXD + d] - omin[d]) << (8 * d);
    off[e] = pk;
  }
}

void launch_divide(const DivArgs& a, bool scatter, cudaStream_t st) {
  const uint64_t blocks = (a.M + DIV_BLOCK - 1) / DIV_BLOCK;
  if (blocks == 0) return;
  if (scatter) k_divide<true><<<(unsigned)blocks, DIV_THREADS, 0, st>>>(a);
  else k_divide<false><<<(unsigned)blocks, DIV_THREADS, 0, st>>>(a);
}
int64_t divide_blocks(uint64_t M) { return (int64_t)((M + DIV_BLOCK - 1) / DIV_BLOCK); }

void launch_far_marks(const int32_t* P, const int32_t* Q, int64_t n, const int32_t* cellX, const int32_t* cellY, int D,
                      uint32_t* tcount, uint32_t* smark, int* omin, int* omax, cudaStream_t st) {
  if (n <= 0) return;
  const int64_t want = (n + 255) / 256;
  k_far_marks<<<(unsigned)(want < 148 * 16 ? want : 148 * 16), 256, 0, st>>>(P, Q, n, cellX, cellY, D, tcount, smark,
                                                                           omin, omax);
}

void launch_far_cols(const int32_t* P, const int32_t* Q, int64_t n, const int32_t* cellX, const int32_t* cellY, int D,
                     const uint32_t* sslot, const int* omin, int32_t* col, uint64_t* off, cudaStream_t st) {
  if (n <= 0) return;
  const int64_t want = (n + 255) / 256;
  k_far_cols<<<(unsigned)(want < 148 * 16 ? want : 148 * 16), 256, 0, st>>>(P, Q, n, cellX, cellY, D, sslot, omin,
                                                                          col, off);
}

}  // namespace f3m
