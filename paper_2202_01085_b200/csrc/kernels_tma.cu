// TMA-pipelined tile-local far field for sm_100a (one persistent 512-thread CTA per SM).
//
// Same method as kernels_local.cu (Sec. 4.1 grouping by box; Sec. 3 far
// field; Chebyshev-moment form of the Lagrange interpolant, far_math.cuh), with
// the B200 memory pipeline: the raw 4096-point tile of the ORIGINAL order (row-major
// coordinates, weights / ranks) is brought into shared memory by one elected thread with
// cp.async.bulk (TMA, UBLKCP) completing on an mbarrier, double-buffered so that tile k+1
// streams in while tile k is ranked and evaluated.  Points are never copied into key order:
// the ranking produces sorig (sorted position -> original local index) and the 4-lane groups
// read coordinates through it.
//   * k_s2m_tma: rank (match_any multisplit, warp histograms, per-bin prefix), per-tile key
//     histogram + tile-local ranks to global (the counting sort's first half), owned-group
//     Chebyshev moments accumulated in shared memory slices (deterministic).
//   * k_l2t_tma: ranks come from the S2M pass; L2T per sorted position, result by original
//     index, pi scattered at the counting-sort destination, v written coalesced.
#include <cuda_runtime.h>
#include <stdint.h>
#include <cstdlib>
#include <type_traits>

#include "f3m_internal.h"
#include "far_math.cuh"

namespace f3m {

constexpr int TM_THREADS = 512;
constexpr int TM_WARPS = TM_THREADS / 32;
constexpr int TM_ITEMS = 8;
constexpr int TM_TILE = TM_THREADS * TM_ITEMS;  // 4096
static_assert(TM_TILE == LT_TILE_PTS, "tile size must match the count/scan tiles");
constexpr int TM_G = 4;
constexpr int TM_GROUPS = TM_THREADS / TM_G;    // 128
constexpr int TM_WP = TM_WARPS + 1;             // per-bin row of the warp histogram (padded)

// ---- PTX helpers: mbarrier + bulk async copy (TMA) ------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "TM_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra TM_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// the same wait with a suspend-time hint: a waiting warp sleeps in the barrier unit instead of
// re-issuing try_wait (warp-specialised kernels: the other group keeps the issue slots)
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "TM_WAITS_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra TM_WAITS_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(0x100000u)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void fence_barrier_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// ---- bit-exact keys (reading R12/R13), same arithmetic as kernels_sort.cu ----------------
__device__ __forceinline__ uint32_t tm_cell(float x, float alpha_f, double alpha, const KeyParams& kp) {
  const float dd = __fsub_rn(x, alpha_f);
  const float q = __fmul_rn(dd, kp.scale_f);
  const float fl = floorf(q);
  const float fr = __fsub_rn(q, fl);
  if (fr > kp.margin && fr < 1.0f - kp.margin) return (uint32_t)fl;
  const double u = __ddiv_rn(__dsub_rn((double)x, alpha), kp.E);
  const double f = floor(__dmul_rn(u, kp.twoT));
  const uint32_t cmax = (uint32_t)kp.twoT - 1u;
  const uint32_t c = (uint32_t)f;
  return c > cmax ? cmax : c;
}
template <int D, int T>
__device__ __forceinline__ uint32_t tm_digit_t(const float* x, const float* af, const double* ad, const KeyParams& kp) {
  uint32_t c[D];
#pragma unroll
  for (int d = 0; d < D; ++d) c[d] = tm_cell(x[d], af[d], ad[d], kp);
  uint32_t K = 0;
#pragma unroll
  for (int s = T - 1; s >= 0; --s)
#pragma unroll
    for (int d = D - 1; d >= 0; --d) K = (K << 1) | ((c[d] >> s) & 1u);
  return K;
}
template <int D>
__device__ __forceinline__ uint32_t tm_digit(const float* x, const float* af, const double* ad, const KeyParams& kp) {
  switch (kp.T) {
    case 1: return tm_digit_t<D, 1>(x, af, ad, kp);
    case 2: if constexpr (D * 2 <= 8) return tm_digit_t<D, 2>(x, af, ad, kp); break;
    case 3: if constexpr (D * 3 <= 8) return tm_digit_t<D, 3>(x, af, ad, kp); break;
    case 4: if constexpr (D * 4 <= 8) return tm_digit_t<D, 4>(x, af, ad, kp); break;
    case 5: if constexpr (D * 5 <= 8) return tm_digit_t<D, 5>(x, af, ad, kp); break;
    case 6: if constexpr (D * 6 <= 8) return tm_digit_t<D, 6>(x, af, ad, kp); break;
    case 7: if constexpr (D * 7 <= 8) return tm_digit_t<D, 7>(x, af, ad, kp); break;
    default: if constexpr (D * 8 <= 8) return tm_digit_t<D, 8>(x, af, ad, kp); break;
  }
  return 0;
}

// digits from exact per-dimension thresholds (thr: [D][2^T - 1] ascending; thr[d][j] is the
// smallest float whose cell is >= j + 1, so cell = #{j : x >= thr[d][j]}).
template <int D, int T>
__host__ __device__ constexpr uint32_t tm_spread(uint32_t c) {  // cell bits -> nested Morton positions
  uint32_t K = 0;
  for (int s = 0; s < T; ++s) K |= ((c >> s) & 1u) << (D * s);
  return K;
}
template <int D, int T>
__device__ __forceinline__ uint32_t tm_digit_thr(const float* x, const float* th) {
  constexpr int NT = (1 << T) - 1;
  uint32_t K = 0;
  if constexpr (NT <= 7) {
    // Morton-weighted threshold count: passing thr[d][j] adds spread(j+1) - spread(j) at dim d
#pragma unroll
    for (int d = 0; d < D; ++d)
#pragma unroll
      for (int j = 0; j < NT; ++j)
        K += (x[d] >= th[d * NT + j]) ? ((tm_spread<D, T>(j + 1) - tm_spread<D, T>(j)) << d) : 0u;
  } else {
#pragma unroll
    for (int d = 0; d < D; ++d) {
      int lo = 0;
#pragma unroll
      for (int step = 1 << (T - 1); step > 0; step >>= 1)
        if (lo + step <= NT && x[d] >= th[d * NT + lo + step - 1]) lo += step;
      K |= tm_spread<D, T>((uint32_t)lo) << d;
    }
  }
  return K;
}

// The D*T bits of the digit as predicates (bit D s + d = bit s of dimension d's cell): with
// the exact thresholds the cell is c = #{j : x >= thr[j]} and the predicates are monotone in j,
// so bit s of c is the XOR of the predicates of the multiples of 2^s.  The ranking ballots on
// these predicates directly (no bit extraction).
template <int D, int T>
__device__ __forceinline__ void tm_bits_thr(const float* x, const float* th, bool (&bits)[D * T]) {
  constexpr int NT = (1 << T) - 1;
#pragma unroll
  for (int d = 0; d < D; ++d) {
    bool p[NT + 1];
#pragma unroll
    for (int j = 1; j <= NT; ++j) p[j] = x[d] >= th[d * NT + j - 1];
#pragma unroll
    for (int sb = 0; sb < T; ++sb) {
      bool v = false;
#pragma unroll
      for (int j = 1 << sb; j <= NT; j += 1 << sb) v ^= p[j];
      bits[D * sb + d] = v;
    }
  }
}

// Digits of this thread's items from the raw tile (thresholds in registers for 2^T - 1 <= 7)
// and their stable ranks among the warp's items of equal digit: peers from D*T ballots,
// running per-warp counts in whist[digit * TM_WP + w].
template <int D, int T>
__device__ __forceinline__ void tm_rank_thr(const float* rx, int segl, int lane, int tvalid, const float* sthr,
                                            uint32_t* whist, int w, uint32_t (&dig)[TM_ITEMS],
                                            int (&wrank)[TM_ITEMS]) {
  constexpr int NT = (1 << T) - 1;
  constexpr int BITS = D * T;
  constexpr int NTR = NT <= 7 ? D * NT : 1;
  float th[NTR];
  if constexpr (NT <= 7) {
#pragma unroll
    for (int e = 0; e < NTR; ++e) th[e] = sthr[e];
  }
#pragma unroll
  for (int j = 0; j < TM_ITEMS; ++j) {
    const int o = segl + j * 32 + lane;
    float x[D];
#pragma unroll
    for (int d = 0; d < D; ++d) x[d] = rx[o * D + d];
    if constexpr (NT <= 7) dig[j] = tm_digit_thr<D, T>(x, th);
    else dig[j] = tm_digit_thr<D, T>(x, sthr);
  }
  const unsigned lt = (1u << lane) - 1u;
#pragma unroll
  for (int j = 0; j < TM_ITEMS; ++j) {
    const uint32_t d = dig[j];
    const bool valid = segl + j * 32 + lane < tvalid;
    unsigned peers = __ballot_sync(0xffffffffu, valid);
#pragma unroll
    for (int i = 0; i < BITS; ++i) {
      const bool bit = (d >> i) & 1u;
      const unsigned bb = __ballot_sync(0xffffffffu, bit);
      peers &= bit ? bb : ~bb;
    }
    wrank[j] = valid ? (int)(whist[d * TM_WP + w] + __popc(peers & lt)) : -1;
    __syncwarp();
    if (valid && (peers & lt) == 0) whist[d * TM_WP + w] += __popc(peers);
    __syncwarp();
  }
}

// ---- shared-memory layout --------------------------------------------------------------
struct TmTables {
  uint32_t* whist;   // [nb][TM_WP]: per-warp counts of each bin, then their bin-major exclusive scan
  uint32_t* wsum;    // [32] block-scan scratch
  uint32_t* ltot;    // [nb]
  uint32_t* lstart;  // [nb]
  uint32_t* goff;    // [nb]
  int nb;
};
__host__ __device__ inline size_t tm_tables_bytes(int nb) {
  return ((size_t)4 * (TM_WP * nb + 32 + 3 * nb) + 15) / 16 * 16;
}
__device__ __forceinline__ TmTables tm_tables(unsigned char* base, int nb) {
  TmTables t;
  uint32_t* u = reinterpret_cast<uint32_t*>(base);
  t.whist = u; u += TM_WP * nb;
  t.wsum = u; u += 32;
  t.ltot = u; u += nb;
  t.lstart = u; u += nb;
  t.goff = u;
  t.nb = nb;
  return t;
}

// one warp: exclusive scan of ltot -> lstart (nb <= 256 bins, 8 per lane)
__device__ __forceinline__ void tm_scan_bins(const TmTables& S) {
  const int lane = threadIdx.x & 31;
  constexpr int BPL = 8;
  uint32_t loc = 0;
#pragma unroll
  for (int r = 0; r < BPL; ++r) {
    const int b = lane * BPL + r;
    if (b < S.nb) loc += S.ltot[b];
  }
  uint32_t inc = loc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  uint32_t run = inc - loc;
#pragma unroll
  for (int r = 0; r < BPL; ++r) {
    const int b = lane * BPL + r;
    if (b < S.nb) {
      S.lstart[b] = run;
      run += S.ltot[b];
    }
  }
}

// Exclusive scan of the warp histogram in bin-major order (bin b, warp w): afterwards
// whist[b][w] = first tile-local sorted position of warp w's items of bin b; then
// lstart/ltot per bin (tvalid = number of ranked items).  Contains __syncthreads.
__device__ __forceinline__ void tm_scan_whist(const TmTables& S, int tvalid) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int E = S.nb * TM_WARPS;
  const int K = (E + TM_THREADS - 1) / TM_THREADS;  // <= 8 (nb <= 256)
  const int e0 = threadIdx.x * K;
  uint32_t loc[8];
  uint32_t sum = 0;
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int e = e0 + r;
    loc[r] = (r < K && e < E) ? S.whist[(e / TM_WARPS) * TM_WP + (e % TM_WARPS)] : 0u;
    sum += loc[r];
  }
  uint32_t inc = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) S.wsum[w] = inc;
  __syncthreads();
  if (w == 0) {
    const uint32_t v = lane < TM_WARPS ? S.wsum[lane] : 0u;
    uint32_t vi = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, vi, o);
      if (lane >= o) vi += y;
    }
    if (lane < TM_WARPS) S.wsum[lane] = vi - v;
  }
  __syncthreads();
  uint32_t run = S.wsum[w] + inc - sum;
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int e = e0 + r;
    if (r < K && e < E) {
      S.whist[(e / TM_WARPS) * TM_WP + (e % TM_WARPS)] = run;
      run += loc[r];
    }
  }
  __syncthreads();
  for (int b = threadIdx.x; b < S.nb; b += TM_THREADS) {
    const uint32_t st = S.whist[b * TM_WP];
    const uint32_t nx = b + 1 < S.nb ? S.whist[(b + 1) * TM_WP] : (uint32_t)tvalid;
    S.lstart[b] = st;
    S.ltot[b] = nx - st;
  }
}

// 4-lane group reduce-scatter (see kernels_local.cu)
template <int M>
__device__ __forceinline__ void tm_group4_reduce_scatter(float (&a)[M]) {
  const int lane = threadIdx.x & 31;
  const bool up2 = (lane & 2) != 0, up1 = (lane & 1) != 0;
#pragma unroll
  for (int i = 0; i < M / 2; ++i) {
    const float keep = up2 ? a[i + M / 2] : a[i];
    const float send = up2 ? a[i] : a[i + M / 2];
    a[i] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
  }
#pragma unroll
  for (int i = 0; i < M / 4; ++i) {
    const float keep = up1 ? a[i + M / 4] : a[i];
    const float send = up1 ? a[i] : a[i + M / 4];
    a[i] = keep + __shfl_xor_sync(0xffffffffu, send, 1);
  }
}

// group sums of acc into the group's slice (ADD: accumulate into it, else overwrite)
template <int M, bool ADD>
__device__ __forceinline__ void tm_owned_flush(float (&acc)[M], float* slice, int gl) {
  if constexpr (M % 4 == 0) {
    tm_group4_reduce_scatter<M>(acc);
#pragma unroll
    for (int r = 0; r < M / 4; ++r) {
      float* q = slice + gl * (M / 4) + r;
      *q = ADD ? *q + acc[r] : acc[r];
    }
  } else {
#pragma unroll
    for (int k2 = 0; k2 < M; ++k2) {
      float v = acc[k2];
      v += __shfl_xor_sync(0xffffffffu, v, 2);
      v += __shfl_xor_sync(0xffffffffu, v, 1);
      if (gl == 0) slice[k2] = ADD ? slice[k2] + v : v;
    }
  }
}

// Per box and dimension the two-float offset of tau = x s - (lo s + 1), s = fp32(2 / l), lo =
// alpha + cell l (fp64): tau = fma(x, s, off_hi) + off_lo (local_tau_off) -- the product x s is
// exact inside the FMA, so this is (x - lo) s - 1 with two roundings, two instructions per
// dimension instead of three for (x - lo_hi - lo_lo) s - 1.
template <int D>
__device__ __forceinline__ void tm_box_geometry(int nbox, int t, const double* alpha, double l, float* geo) {
  const double s = (double)(float)(2.0 / l);
  for (int B = threadIdx.x; B < nbox; B += TM_THREADS) {
    int cell[D];
#pragma unroll
    for (int d = 0; d < D; ++d) cell[d] = 0;
    for (int q = 0; q < t; ++q)
#pragma unroll
      for (int d = 0; d < D; ++d) cell[d] |= ((B >> (D * q + d)) & 1) << q;
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const double lo = alpha[d] + (double)cell[d] * l;
      const double off = -fma(lo, s, 1.0);
      const float hi = (float)off;
      geo[(B * D + d) * 2] = hi;
      geo[(B * D + d) * 2 + 1] = (float)(off - (double)hi);
    }
  }
}

// ---------------------------------------------------------------------------------------
// S2M: ranks + key histogram of every tile, Chebyshev moments of its boxes
// ---------------------------------------------------------------------------------------
template <int D, int P>
__global__ void __launch_bounds__(TM_THREADS, 1) k_s2m_tma(LocalS2MArgs a) {
  constexpr int M = IPow<P, D>::value;
  constexpr bool PERSIST = M <= 64;  // moments live in registers across tiles
  extern __shared__ __align__(128) unsigned char smraw[];
  const int nb = 1 << a.bits;
  // layout: rawx[2][TILE*D] | rawb[2][TILE] | sorig[TILE] u16 | tables | wsl[GROUPS][M] | geo | bars
  float* rawx = reinterpret_cast<float*>(smraw);
  float* rawb = rawx + 2 * TM_TILE * D;
  uint16_t* sorig = reinterpret_cast<uint16_t*>(rawb + 2 * TM_TILE);
  unsigned char* tb = reinterpret_cast<unsigned char*>(sorig + TM_TILE);
  const TmTables S = tm_tables(tb, nb);
  float* wsl = reinterpret_cast<float*>(tb + tm_tables_bytes(nb));
  float* geo = wsl + TM_GROUPS * M;
  float* sthr = geo + ((2 * D * a.nbox + 3) / 4) * 4;                // [D][2^T - 1]
  const int nthr = a.kp.thr ? D * ((1 << a.kp.T) - 1) : 0;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sthr + ((nthr + 3) / 4) * 4);
  for (int e = threadIdx.x; e < nthr; e += TM_THREADS) sthr[e] = a.kp.thr[e];

  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int grp = threadIdx.x / TM_G, gl = threadIdx.x % TM_G;
  const int t = (a.bits - a.shift) / D;
  const bool owned = a.do_s2m && a.nbox <= TM_GROUPS;
  float af[D];
  double ad[D];
#pragma unroll
  for (int d = 0; d < D; ++d) { af[d] = a.kp.alpha_f[d]; ad[d] = a.kp.alpha[d]; }
  if (a.do_s2m) tm_box_geometry<D>(a.nbox, t, a.alpha, a.l, geo);
  for (int e = threadIdx.x; e < TM_GROUPS * M; e += TM_THREADS) wsl[e] = 0.f;
  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_barrier_init();
  }
  __syncthreads();

  const int tpb = (a.num_tiles + gridDim.x - 1) / gridDim.x;
  const int t_begin = blockIdx.x * tpb, t_end = min(a.num_tiles, t_begin + tpb);
  const float scale = (float)(2.0 / a.l);
  const bool aligned = ((reinterpret_cast<uintptr_t>(a.X) | reinterpret_cast<uintptr_t>(a.b)) & 15) == 0;
  auto full_tile = [&](int tile) { return aligned && (int64_t)(tile + 1) * TM_TILE <= a.n; };
  auto issue = [&](int tile, int buf) {
    if (tile < t_end && full_tile(tile) && threadIdx.x == 0) {
      fence_proxy_async();
      const int64_t r0 = (int64_t)tile * TM_TILE;
      mbar_expect_tx(&bars[buf], (uint32_t)(TM_TILE * (D + 1) * 4));
      tma_g2s(rawx + buf * TM_TILE * D, a.X + r0 * D, (uint32_t)(TM_TILE * D * 4), &bars[buf]);
      tma_g2s(rawb + buf * TM_TILE, a.b + r0, (uint32_t)(TM_TILE * 4), &bars[buf]);
    }
  };
  float acc[PERSIST ? M : 1];
#pragma unroll
  for (int k2 = 0; k2 < (PERSIST ? M : 1); ++k2) acc[k2] = 0.f;
  issue(t_begin, 0);
  uint32_t phase = 0;  // bit b: mbarrier parity of buffer b
  for (int tile = t_begin, k = 0; tile < t_end; ++tile, ++k) {
    const int buf = k & 1;
    issue(tile + 1, buf ^ 1);  // buffer buf^1 was released by the previous tile's final barrier
    const int64_t tile0 = (int64_t)tile * TM_TILE;
    const int tvalid = (int)min((int64_t)TM_TILE, a.n - tile0);
    float* rx = rawx + buf * TM_TILE * D;
    float* rb = rawb + buf * TM_TILE;
    if (full_tile(tile)) {
      mbar_wait(&bars[buf], (phase >> buf) & 1u);
      phase ^= 1u << buf;
    } else {  // partial / unaligned tile: plain loads
      for (int e = threadIdx.x; e < tvalid * D; e += TM_THREADS) rx[e] = __ldg(a.X + tile0 * D + e);
      for (int e = threadIdx.x; e < tvalid; e += TM_THREADS) rb[e] = __ldg(a.b + tile0 + e);
      __syncthreads();
    }
    // ---- rank: warp w owns local items [w*256, (w+1)*256), lane l items 32j + l
    for (int b = lane; b < nb; b += 32) S.whist[b * TM_WP + w] = 0;
    __syncwarp();
    uint32_t dig[TM_ITEMS];
    int wrank[TM_ITEMS];
    const int segl = w * (TM_TILE / TM_WARPS);
    if (nthr) {
      switch (a.kp.T) {
        case 1: tm_rank_thr<D, 1>(rx, segl, lane, tvalid, sthr, S.whist, w, dig, wrank); break;
        case 2: if constexpr (D * 2 <= 8) tm_rank_thr<D, 2>(rx, segl, lane, tvalid, sthr, S.whist, w, dig, wrank); break;
        case 3: if constexpr (D * 3 <= 8) tm_rank_thr<D, 3>(rx, segl, lane, tvalid, sthr, S.whist, w, dig, wrank); break;
        case 4: if constexpr (D * 4 <= 8) tm_rank_thr<D, 4>(rx, segl, lane, tvalid, sthr, S.whist, w, dig, wrank); break;
        case 5: if constexpr (D * 5 <= 8) tm_rank_thr<D, 5>(rx, segl, lane, tvalid, sthr, S.whist, w, dig, wrank); break;
        case 6: if constexpr (D * 6 <= 8) tm_rank_thr<D, 6>(rx, segl, lane, tvalid, sthr, S.whist, w, dig, wrank); break;
        case 7: if constexpr (D * 7 <= 8) tm_rank_thr<D, 7>(rx, segl, lane, tvalid, sthr, S.whist, w, dig, wrank); break;
        default: if constexpr (D * 8 <= 8) tm_rank_thr<D, 8>(rx, segl, lane, tvalid, sthr, S.whist, w, dig, wrank); break;
      }
    } else {
#pragma unroll
      for (int j = 0; j < TM_ITEMS; ++j) {
        const int o = segl + j * 32 + lane;
        float x[D];
#pragma unroll
        for (int d = 0; d < D; ++d) x[d] = rx[o * D + d];
        dig[j] = (o < tvalid) ? tm_digit<D>(x, af, ad, a.kp) : 0xffffffffu;
      }
      const unsigned lt = (1u << lane) - 1u;
#pragma unroll
      for (int j = 0; j < TM_ITEMS; ++j) {
        const uint32_t d = dig[j];
        const bool valid = d != 0xffffffffu;
        const unsigned peers = __match_any_sync(0xffffffffu, d);
        wrank[j] = valid ? (int)(S.whist[d * TM_WP + w] + __popc(peers & lt)) : -1;
        __syncwarp();
        if (valid && (peers & lt) == 0) S.whist[d * TM_WP + w] += __popc(peers);
        __syncwarp();
      }
    }
    __syncthreads();
    tm_scan_whist(S, tvalid);
    if (a.counts)
      for (int b = threadIdx.x; b < nb; b += TM_THREADS) a.counts[(int64_t)b * a.num_tiles + tile] = S.ltot[b];
    __syncthreads();
#pragma unroll
    for (int j = 0; j < TM_ITEMS; ++j) {
      if (wrank[j] >= 0) {
        const int o = segl + j * 32 + lane;
        const int lp = (int)S.whist[dig[j] * TM_WP + w] + wrank[j];
        sorig[lp] = (uint16_t)o;
      }
    }
    __syncthreads();
    // the tile's stable order for the L2T pass: sorted position -> original local index
    if (a.lrank) {
      if (tvalid == TM_TILE && aligned) {  // 8 entries (16 B) per thread
        const uint4 q = reinterpret_cast<const uint4*>(sorig)[threadIdx.x];
        reinterpret_cast<uint4*>(a.lrank + tile0)[threadIdx.x] = q;
      } else {
        for (int e = threadIdx.x; e < tvalid; e += TM_THREADS) a.lrank[tile0 + e] = sorig[e];
      }
    }
    // ---- owned-group Chebyshev moments: group g takes box g % nbox (sub-slot g / nbox).
    // The assignment is the same in every tile, so the moments stay in registers across the
    // CTA's whole tile range and are reduced once at the end (fixed order: deterministic).
    if (owned) {
      const int G = TM_GROUPS / a.nbox;
      const int B = grp % a.nbox, sub = grp / a.nbox;
      const int per = 1 << a.shift;
      uint32_t beg = S.lstart[B * per], cnt = 0;
      for (int q = 0; q < per; ++q) cnt += S.ltot[B * per + q];
      const int end = (int)(beg + cnt);
      auto own_box = [&](float (&ac)[M]) {
        if ((int)beg < end) {
          float lh[D], ll[D];
#pragma unroll
          for (int d = 0; d < D; ++d) { lh[d] = geo[(B * D + d) * 2]; ll[d] = geo[(B * D + d) * 2 + 1]; }
          for (int p = (int)beg + sub * TM_G + gl; p < end; p += TM_G * G) {
            const int o = sorig[p];
            float T[D][P];
#pragma unroll
            for (int d = 0; d < D; ++d) chebyshev<P>(local_tau_off(rx[o * D + d], scale, lh[d], ll[d]), T[d]);
            s2m_accumulate<D, P>(rb[o], T, ac);
          }
        }
      };
      if constexpr (PERSIST) {
        own_box(acc);
      } else {  // M > 64: per-tile accumulators flushed into the slice (register budget)
        float ac[M];
#pragma unroll
        for (int k2 = 0; k2 < M; ++k2) ac[k2] = 0.f;
        own_box(ac);
        __syncwarp();
        tm_owned_flush<M, true>(ac, wsl + grp * M, gl);
      }
    }
    __syncthreads();  // releases rx/rb/sorig of this tile
  }
  if (owned) {
    if constexpr (PERSIST) tm_owned_flush<M, false>(acc, wsl + grp * M, gl);
    __syncthreads();
    const int G = TM_GROUPS / a.nbox;
    float* out = a.Wpart + (int64_t)blockIdx.x * a.nbox * M;
    for (int e = threadIdx.x; e < a.nbox * M; e += TM_THREADS) {
      const int B = e / M, k2 = e - B * M;
      float sum = 0.f;
      for (int sub = 0; sub < G; ++sub) sum += wsl[(sub * a.nbox + B) * M + k2];
      out[e] = sum;
    }
  }
}

// ---------------------------------------------------------------------------------------
// L2T with the first pass's tile order; pi at the counting-sort destinations
// ---------------------------------------------------------------------------------------
// cp.async (LDGSTS) of one 4-byte word: the bin offsets of the next tile stream into shared
// memory without holding registers across the compute phase
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
// explicit shared-state-space accesses through 32-bit addresses (the generic-pointer form made
// the compiler re-derive the shared window base inside the inner loops)
__device__ __forceinline__ float lds_f32(uint32_t addr) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ uint32_t lds_u16(uint32_t addr) {
  unsigned short v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ void sts_f32(uint32_t addr, float v) {
  asm volatile("st.shared.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}

// One barrier per tile.  Iteration k: wait for tile k (TMA: coordinates + the first pass's
// sorted-order local indices, so no re-ranking and no scatter), warp 0 turns the prefetched
// bin offsets into the tile's bin table; __syncthreads; thread 0 issues the TMA of tile k+1;
// every thread writes v of tile k-1 (coalesced, from the other sv buffer) and then evaluates
// tile k: 4-lane group g owns box g % nbox with its coefficients in registers, result into
// sv[k & 1] by original index, pi straight to its counting-sort destination.
template <int D, int P, bool PER1>  // PER1: one leaf bin per box (shift = 0, the C4 case)
__global__ void __launch_bounds__(TM_THREADS, 1) k_l2t_tma(LocalL2TArgs a) {
  constexpr int M = IPow<P, D>::value;
  constexpr int MROW = (M % 4 == 0) ? M + 4 : M;
  extern __shared__ __align__(128) unsigned char smraw[];
  const int nb = 1 << a.bits;
  // rawx[2][TILE*D] | rawo[2][TILE] u16 | sv[2][TILE] | Us | geo | tab[2][3 nb] | off[2][2 nb] | bars
  float* rawx = reinterpret_cast<float*>(smraw);
  uint16_t* rawo = reinterpret_cast<uint16_t*>(rawx + 2 * TM_TILE * D);
  float* sv = reinterpret_cast<float*>(rawo + 2 * TM_TILE);
  float* Us = sv + 2 * TM_TILE;
  float* geo = Us + a.nbox * MROW;
  uint32_t* tab = reinterpret_cast<uint32_t*>(geo + ((2 * D * a.nbox + 3) / 4) * 4);  // lstart | cnt | goff
  uint32_t* off = tab + 2 * 3 * nb;
  uint64_t* bars = reinterpret_cast<uint64_t*>(off + ((2 * 2 * nb + 3) / 4) * 4);

  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int grp = threadIdx.x / TM_G, gl = threadIdx.x % TM_G;
  const int t = (a.bits - a.shift) / D;
  const int per = PER1 ? 1 : 1 << a.shift;  // leaf bins per box
  tm_box_geometry<D>(a.nbox, t, a.alpha, a.l, geo);
  for (int e = threadIdx.x; e < a.nbox * M; e += TM_THREADS) {
    const int B = e / M, k2 = e - B * M;
    const int sl = a.box_slot[B];
    const int at = (D == 3 && P == 4) ? l2t_pair_index(k2) : k2;  // FFMA2 pair layout (far_math.cuh)
    Us[B * MROW + at] = sl >= 0 ? (float)a.U[(int64_t)sl * M + k2] : 0.f;
  }
  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_barrier_init();
  }
  const int tpb = (a.num_tiles + gridDim.x - 1) / gridDim.x;
  const int t_begin = blockIdx.x * tpb, t_end = min(a.num_tiles, t_begin + tpb);
  const float scale = (float)(2.0 / a.l);
  const bool aligned = (reinterpret_cast<uintptr_t>(a.X) & 15) == 0;
  const int64_t scan_len = (int64_t)nb * a.sort_tiles;
  auto full_tile = [&](int tile) { return aligned && (int64_t)(tile + 1) * TM_TILE <= a.n; };
  auto issue = [&](int tile, int buf) {
    if (tile < t_end && full_tile(tile) && threadIdx.x == 0) {
      fence_proxy_async();
      const int64_t r0 = (int64_t)tile * TM_TILE;
      mbar_expect_tx(&bars[buf], (uint32_t)(TM_TILE * (D * 4 + 2)));
      tma_g2s(rawx + buf * TM_TILE * D, a.X + r0 * D, (uint32_t)(TM_TILE * D * 4), &bars[buf]);
      tma_g2s(rawo + buf * TM_TILE, a.lrank + r0, (uint32_t)(TM_TILE * 2), &bars[buf]);
    }
  };
  // warp 0: cp.async of tile `tile`'s scanned offsets (bin b: [b][tile] and the next entry)
  auto prefetch_offsets = [&](int tile, int buf) {
    if (w == 0 && tile < t_end) {
      uint32_t* o = off + buf * 2 * nb;
      for (int b = lane; b < nb; b += 32) {
        const int64_t idx = (int64_t)b * a.sort_tiles + tile;
        cp_async4(o + b, a.offsets + idx);
        if (idx + 1 < scan_len) cp_async4(o + nb + b, a.offsets + idx + 1);
        else o[nb + b] = (uint32_t)a.n;
      }
    }
  };
  const bool v_vec = !a.vs && !a.accumulate && (reinterpret_cast<uintptr_t>(a.v) & 15) == 0;
  auto write_v = [&](int tile, int buf) {
    const int64_t tile0 = (int64_t)tile * TM_TILE;
    const int tvalid = (int)min((int64_t)TM_TILE, a.n - tile0);
    const float* s = sv + buf * TM_TILE;
    if (v_vec && tvalid == TM_TILE) {  // 8 consecutive results (two 16-byte stores) per thread
      const float4* s4 = reinterpret_cast<const float4*>(s) + 2 * threadIdx.x;
      float4* d4 = reinterpret_cast<float4*>(a.v + tile0) + 2 * threadIdx.x;
      d4[0] = s4[0];
      d4[1] = s4[1];
      return;
    }
    for (int o = threadIdx.x; o < tvalid; o += TM_THREADS) {
      const int64_t i = tile0 + o;
      float r = s[o];
      if (a.vs) r += a.vs[a.sigma[i]];
      if (a.accumulate) r += a.v[i];
      a.v[i] = r;
    }
  };
  __syncthreads();
  issue(t_begin, 0);
  prefetch_offsets(t_begin, 0);
  uint32_t phase = 0;  // bit b: mbarrier parity of buffer b
  for (int tile = t_begin, k = 0; tile < t_end; ++tile, ++k) {
    const int buf = k & 1;
    const int64_t tile0 = (int64_t)tile * TM_TILE;
    const int tvalid = (int)min((int64_t)TM_TILE, a.n - tile0);
    float* rx = rawx + buf * TM_TILE * D;
    uint16_t* ro = rawo + buf * TM_TILE;
    uint32_t* lstart = tab + buf * 3 * nb;
    uint32_t* lcnt = lstart + nb;
    uint32_t* goff = lcnt + nb;
    if (w == 0) {  // bin table of this tile: counts, destinations, exclusive scan -> lstart
      cp_async_wait_all();
      __syncwarp();
      const uint32_t* o = off + buf * 2 * nb;
      constexpr int BPL = 8;  // nb <= 256
      uint32_t c[BPL];
      uint32_t loc = 0;
#pragma unroll
      for (int r = 0; r < BPL; ++r) {
        const int b = lane * BPL + r;
        c[r] = b < nb ? o[nb + b] - o[b] : 0u;
        loc += c[r];
      }
      uint32_t inc = loc;
#pragma unroll
      for (int sh = 1; sh < 32; sh <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, sh);
        if (lane >= sh) inc += y;
      }
      uint32_t run = inc - loc;
#pragma unroll
      for (int r = 0; r < BPL; ++r) {
        const int b = lane * BPL + r;
        if (b < nb) {
          lstart[b] = run;
          lcnt[b] = c[r];
          goff[b] = o[b];
          run += c[r];
        }
      }
    }
    if (full_tile(tile)) {
      mbar_wait(&bars[buf], (phase >> buf) & 1u);
      phase ^= 1u << buf;
    } else {  // partial / unaligned tile: plain loads
      for (int e = threadIdx.x; e < tvalid * D; e += TM_THREADS) rx[e] = __ldg(a.X + tile0 * D + e);
      for (int e = threadIdx.x; e < tvalid; e += TM_THREADS) ro[e] = __ldg(a.lrank + tile0 + e);
    }
    __syncthreads();  // the only barrier of the iteration
    issue(tile + 1, buf ^ 1);
    prefetch_offsets(tile + 1, buf ^ 1);
    if (k > 0) write_v(tile - 1, buf ^ 1);
    float* svb = sv + buf * TM_TILE;
    // evaluate the points of box B at sorted positions first, first + step, ...
    auto eval_box = [&](int B, int first, int step) {
      const int beg = (int)lstart[B * per];
      const int end = (B + 1) * per < nb ? (int)lstart[(B + 1) * per] : tvalid;
      if (beg + first >= end) return;
      float lh[D], ll[D];
#pragma unroll
      for (int d = 0; d < D; ++d) { lh[d] = geo[(B * D + d) * 2]; ll[d] = geo[(B * D + d) * 2 + 1]; }
      constexpr bool X2 = (D == 3 && P == 4);  // packed FFMA2 contraction (far_math.cuh)
      float u[X2 ? 1 : M];
      float2 u2[X2 ? M / 2 : 1];
      if constexpr (X2) {
#pragma unroll
        for (int k2 = 0; k2 < M; k2 += 4) {
          const float4 v4 = *reinterpret_cast<const float4*>(Us + B * MROW + k2);
          u2[k2 / 2] = make_float2(v4.x, v4.y);
          u2[k2 / 2 + 1] = make_float2(v4.z, v4.w);
        }
      } else if constexpr (M % 4 == 0) {
#pragma unroll
        for (int k2 = 0; k2 < M; k2 += 4) {
          const float4 v4 = *reinterpret_cast<const float4*>(Us + B * MROW + k2);
          u[k2] = v4.x; u[k2 + 1] = v4.y; u[k2 + 2] = v4.z; u[k2 + 3] = v4.w;
        }
      } else {
#pragma unroll
        for (int k2 = 0; k2 < M; ++k2) u[k2] = Us[B * MROW + k2];
      }
      // pi destination of sorted position p inside bin b: goff[b] + p - lstart[b]
      int bin = B * per;
      int32_t* pdst = a.perm ? a.perm + (int64_t)goff[bin] - (int64_t)lstart[bin] : nullptr;
      // software pipeline: the next point's order entry and coordinates load while this one is
      // evaluated (hides the dependent shared-memory latencies)
      int on = ro[beg + first];
      float xn[D];
#pragma unroll
      for (int d = 0; d < D; ++d) xn[d] = rx[on * D + d];
      for (int p = beg + first; p < end; p += step) {
        const int o = on;
        float xo[D];
#pragma unroll
        for (int d = 0; d < D; ++d) xo[d] = xn[d];
        if (p + step < end) {
          on = ro[p + step];
#pragma unroll
          for (int d = 0; d < D; ++d) xn[d] = rx[on * D + d];
        }
        float T[D][P];
#pragma unroll
        for (int d = 0; d < D; ++d) chebyshev<P>(local_tau_off(xo[d], scale, lh[d], ll[d]), T[d]);
        if constexpr (X2) svb[o] = l2t_contract_d3p4_x2(T, u2);
        else svb[o] = l2t_contract<D, P>(T, u);
        if (a.perm) {
          if (!PER1 && per > 1) {  // bins finer than boxes: last bin of the box with lstart <= p
            int bb = B * per;
            for (int q = 1; q < per; ++q)
              if ((int)lstart[B * per + q] <= p) bb = B * per + q;
            if (bb != bin) {
              bin = bb;
              pdst = a.perm + (int64_t)goff[bin] - (int64_t)lstart[bin];
            }
          }
          pdst[p] = (int32_t)(tile0 + o);
          if (a.keys) a.keys[(int64_t)goff[bin] + p - lstart[bin]] = (uint64_t)bin;
        }
      }
    };
    {
      // 4-lane group g owns box g % nbox (boxes <= 128); larger trees stride over boxes
      const int G = a.nbox <= TM_GROUPS ? TM_GROUPS / a.nbox : 1;
      for (int B = grp % a.nbox; B < a.nbox; B += (a.nbox <= TM_GROUPS ? a.nbox : TM_GROUPS)) {
        const int sub = a.nbox <= TM_GROUPS ? grp / a.nbox : 0;
        eval_box(B, sub * TM_G + gl, TM_G * G);
      }
    }
  }
  __syncthreads();
  if (t_end > t_begin) write_v(t_end - 1, (t_end - 1 - t_begin) & 1);
}

// ---------------------------------------------------------------------------------------
// L2T with register-resident coefficients (the headline configuration: one leaf bin per box and
// at most 128 boxes, so 4-lane group g owns box g % nbox in every tile).  Same pipeline as
// k_l2t_tma (TMA double buffer, one barrier per tile, coalesced v write-out), but a group's 64
// Chebyshev coefficients and box geometry are loaded into registers once per kernel instead of
// once per tile and box (ncu on k_l2t_tma: that per-tile prologue was ~24 % of the warp-stall
// samples, waiting on its shared-memory loads).  Arithmetic per point is that of k_l2t_tma
// (bit-identical v).
// ---------------------------------------------------------------------------------------
template <int D, int P>
__global__ void __launch_bounds__(TM_THREADS, 1) k_l2t_fix(LocalL2TArgs a) {
  constexpr int M = IPow<P, D>::value;
  static_assert(M <= 64, "register-resident coefficients");
  extern __shared__ __align__(128) unsigned char smraw[];
  const int nb = 1 << a.bits;  // == nbox
  // rawx[2][TILE*D] | rawo[2][TILE] u16 | sv[2][TILE] | tab[2][2 nb] | off[2][2 nb] | bars
  float* rawx = reinterpret_cast<float*>(smraw);
  uint16_t* rawo = reinterpret_cast<uint16_t*>(rawx + 2 * TM_TILE * D);
  float* sv = reinterpret_cast<float*>(rawo + 2 * TM_TILE);
  uint32_t* tab = reinterpret_cast<uint32_t*>(sv + 2 * TM_TILE);  // lstart | goff
  uint32_t* off = tab + 2 * 2 * nb;
  uint64_t* bars = reinterpret_cast<uint64_t*>(off + ((2 * 2 * nb + 3) / 4) * 4);

  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int grp = threadIdx.x / TM_G, gl = threadIdx.x % TM_G;
  const int B = grp % a.nbox, sub = grp / a.nbox;
  const int step = TM_G * (TM_GROUPS / a.nbox);
  const int t = a.bits / D;
  const float scale = (float)(2.0 / a.l);
  // box geometry (the arithmetic of tm_box_geometry) and coefficients, once
  float lh[D], ll[D];
  {
    const double sc = (double)(float)(2.0 / a.l);
#pragma unroll
    for (int d = 0; d < D; ++d) {
      int cell = 0;
      for (int q = 0; q < t; ++q) cell |= ((B >> (D * q + d)) & 1) << q;
      cell += a.cell_base[d];
      const double lo = a.alpha[d] + (double)cell * a.l;
      const double of = -fma(lo, sc, 1.0);
      lh[d] = (float)of;
      ll[d] = (float)(of - (double)lh[d]);
    }
  }
  constexpr bool X2 = (D == 3 && P == 4);  // packed FFMA2 contraction (far_math.cuh)
  float u[X2 ? 1 : M];
  float2 u2[X2 ? M / 2 : 1];
  {
    const int sl = a.box_slot[B];
    float uf[M];
#pragma unroll
    for (int k2 = 0; k2 < M; ++k2) uf[k2] = sl >= 0 ? (float)a.U[(int64_t)sl * M + k2] : 0.f;
    if constexpr (X2) {
      float pf[M];
#pragma unroll
      for (int k2 = 0; k2 < M; ++k2) pf[l2t_pair_index(k2)] = uf[k2];
#pragma unroll
      for (int q = 0; q < M / 2; ++q) u2[q] = make_float2(pf[2 * q], pf[2 * q + 1]);
    } else {
#pragma unroll
      for (int k2 = 0; k2 < M; ++k2) u[k2] = uf[k2];
    }
  }
  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_barrier_init();
  }
  const int tpb = (a.num_tiles + gridDim.x - 1) / gridDim.x;
  const int t_begin = blockIdx.x * tpb, t_end = min(a.num_tiles, t_begin + tpb);
  const bool aligned = (reinterpret_cast<uintptr_t>(a.X) & 15) == 0;
  const int64_t scan_len = (int64_t)nb * a.sort_tiles;
  auto full_tile = [&](int tile) { return aligned && (int64_t)(tile + 1) * TM_TILE <= a.n; };
  auto issue = [&](int tile, int buf) {
    if (tile < t_end && full_tile(tile) && threadIdx.x == 0) {
      fence_proxy_async();
      const int64_t r0 = (int64_t)tile * TM_TILE;
      mbar_expect_tx(&bars[buf], (uint32_t)(TM_TILE * (D * 4 + 2)));
      tma_g2s(rawx + buf * TM_TILE * D, a.X + r0 * D, (uint32_t)(TM_TILE * D * 4), &bars[buf]);
      tma_g2s(rawo + buf * TM_TILE, a.lrank + r0, (uint32_t)(TM_TILE * 2), &bars[buf]);
    }
  };
  auto prefetch_offsets = [&](int tile, int buf) {
    if (w == 0 && tile < t_end) {
      uint32_t* o = off + buf * 2 * nb;
      for (int b = lane; b < nb; b += 32) {
        const int64_t idx = (int64_t)b * a.sort_tiles + tile;
        cp_async4(o + b, a.offsets + idx);
        if (a.offsets_tail || idx + 1 < scan_len) cp_async4(o + nb + b, a.offsets + idx + 1);
        else o[nb + b] = (uint32_t)a.n;
      }
    }
  };
  const bool v_vec = !a.vs && !a.accumulate && (reinterpret_cast<uintptr_t>(a.v) & 15) == 0;
  auto write_v = [&](int tile, int buf) {
    const int64_t tile0 = (int64_t)tile * TM_TILE;
    const int tvalid = (int)min((int64_t)TM_TILE, a.n - tile0);
    const float* s = sv + buf * TM_TILE;
    if (v_vec && tvalid == TM_TILE) {  // 8 consecutive results (two 16-byte stores) per thread
      const float4* s4 = reinterpret_cast<const float4*>(s) + 2 * threadIdx.x;
      float4* d4 = reinterpret_cast<float4*>(a.v + tile0) + 2 * threadIdx.x;
      d4[0] = s4[0];
      d4[1] = s4[1];
      return;
    }
    for (int o = threadIdx.x; o < tvalid; o += TM_THREADS) {
      const int64_t i = tile0 + o;
      float r = s[o];
      if (a.vs) r += a.vs[a.sigma[i]];
      if (a.accumulate) r += a.v[i];
      a.v[i] = r;
    }
  };
  __syncthreads();
  issue(t_begin, 0);
  prefetch_offsets(t_begin, 0);
  uint32_t phase = 0;  // bit b: mbarrier parity of buffer b
  for (int tile = t_begin, k = 0; tile < t_end; ++tile, ++k) {
    const int buf = k & 1;
    const int64_t tile0 = (int64_t)tile * TM_TILE;
    const int tvalid = (int)min((int64_t)TM_TILE, a.n - tile0);
    float* rx = rawx + buf * TM_TILE * D;
    uint16_t* ro = rawo + buf * TM_TILE;
    uint32_t* lstart = tab + buf * 2 * nb;
    uint32_t* goff = lstart + nb;
    if (w == 0) {  // bin table of this tile: destinations, exclusive scan of the counts -> lstart
      cp_async_wait_all();
      __syncwarp();
      const uint32_t* o = off + buf * 2 * nb;
      constexpr int BPL = 4;  // nb <= 128
      uint32_t c[BPL];
      uint32_t loc = 0;
#pragma unroll
      for (int r = 0; r < BPL; ++r) {
        const int b = lane * BPL + r;
        c[r] = b < nb ? o[nb + b] - o[b] : 0u;
        loc += c[r];
      }
      uint32_t inc = loc;
#pragma unroll
      for (int sh = 1; sh < 32; sh <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, sh);
        if (lane >= sh) inc += y;
      }
      uint32_t run = inc - loc;
#pragma unroll
      for (int r = 0; r < BPL; ++r) {
        const int b = lane * BPL + r;
        if (b < nb) {
          lstart[b] = run;
          goff[b] = o[b];
          run += c[r];
        }
      }
    }
    if (full_tile(tile)) {
      mbar_wait(&bars[buf], (phase >> buf) & 1u);
      phase ^= 1u << buf;
    } else {  // partial / unaligned tile: plain loads
      for (int e = threadIdx.x; e < tvalid * D; e += TM_THREADS) rx[e] = __ldg(a.X + tile0 * D + e);
      for (int e = threadIdx.x; e < tvalid; e += TM_THREADS) ro[e] = __ldg(a.lrank + tile0 + e);
    }
    __syncthreads();  // the only barrier of the iteration
    issue(tile + 1, buf ^ 1);
    prefetch_offsets(tile + 1, buf ^ 1);
    if (k > 0) write_v(tile - 1, buf ^ 1);
    const uint32_t rx_s = smem_u32(rx), ro_s = smem_u32(ro), sv_s = smem_u32(sv + buf * TM_TILE);
    const int beg = (int)lstart[B];
    const int end = B + 1 < nb ? (int)lstart[B + 1] : tvalid;
    // evaluate the group's points (sorted positions beg + sub*4 + gl, + step, ...): result into sv
    // by original index; MODE 1: pi at its counting-sort destination, 2: also the sorted keys
    auto run = [&](auto mode_c) {
      constexpr int MODE = decltype(mode_c)::value;
      int32_t* pdst = MODE ? a.perm + (int64_t)goff[B] - (int64_t)beg : nullptr;
      int p = beg + sub * TM_G + gl;
      if (p >= end) return;
      const int last = end - 1;
      // two points per iteration with two register sets: set 1 is reloaded (next pair) only after
      // its point is evaluated, so the loads overlap the other point's arithmetic and no
      // loop-carried copies are needed; indices are clamped to the box (no branches on loads)
      auto load = [&](int q, uint32_t& o4, float (&x)[D]) {
        o4 = lds_u16(ro_s + 2u * q) << 2;                 // 4 o: sv byte offset
        const uint32_t ob = rx_s + o4 * D;                // coordinate row
#pragma unroll
        for (int d = 0; d < D; ++d) x[d] = lds_f32(ob + 4u * d);
      };
      auto eval = [&](int q, uint32_t o4, const float (&x)[D]) {
        float Tc[D][P];
        float r;
        if constexpr (X2) {
          cheb_d3p4_x2(x, scale, lh, ll, Tc);
          r = l2t_contract_d3p4_x2(Tc, u2);
        } else {
#pragma unroll
          for (int d = 0; d < D; ++d) chebyshev<P>(local_tau_off(x[d], scale, lh[d], ll[d]), Tc[d]);
          r = l2t_contract<D, P>(Tc, u);
        }
        sts_f32(sv_s + o4, r);
        if constexpr (MODE >= 1) pdst[q] = (int32_t)(tile0 + (o4 >> 2));
        if constexpr (MODE == 2) a.keys[(int64_t)goff[B] + q - beg] = (uint64_t)B;
      };
      uint32_t o1, o2;
      float x1[D], x2[D];
      load(p, o1, x1);
      for (; p < end; p += 2 * step) {
        const int q2 = p + step;
        load(min(q2, last), o2, x2);
        eval(p, o1, x1);
        load(min(q2 + step, last), o1, x1);
        if (q2 < end) eval(q2, o2, x2);
      }
    };
    if (!a.perm) run(std::integral_constant<int, 0>{});
    else if (!a.keys) run(std::integral_constant<int, 1>{});
    else run(std::integral_constant<int, 2>{});
  }
  __syncthreads();
  if (t_end > t_begin) write_v(t_end - 1, (t_end - 1 - t_begin) & 1);
}

static size_t l2t_fix_smem(int D, int nb) {
  return (size_t)2 * TM_TILE * D * 4 + (size_t)2 * TM_TILE * 2 + (size_t)2 * TM_TILE * 4 + (size_t)4 * 2 * 2 * nb +
         (size_t)((2 * 2 * nb + 3) / 4) * 16 + 64;
}

bool l2t_fix_supported(int D, int P, int nb, int nbox, int shift) {
  if (shift != 0 || nb != nbox || nbox > TM_GROUPS) return false;
  int m = 1;
  for (int d = 0; d < D; ++d) m *= P;
  if (m > 64 || l2t_fix_smem(D, nb) > 227 * 1024) return false;
  return (D == 3 && P >= 2 && P <= 4) || (D == 2 && P >= 2 && P <= 8) || (D == 1 && P >= 2 && P <= 8);
}

void launch_l2t_fix(int D, int P, const LocalL2TArgs& a, int grid, cudaStream_t st) {
  const size_t sm = l2t_fix_smem(D, 1 << a.bits);
#define X(d, p)                                                                                  \
  if (D == d && P == p) {                                                                        \
    cudaFuncSetAttribute(k_l2t_fix<d, p>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm); \
    k_l2t_fix<d, p><<<grid, TM_THREADS, sm, st>>>(a);                                            \
    return;                                                                                      \
  }
  X(3, 4) X(3, 3) X(3, 2) X(2, 2) X(2, 3) X(2, 4) X(2, 5) X(2, 6) X(2, 7) X(2, 8)
  X(1, 2) X(1, 3) X(1, 4) X(1, 5) X(1, 6) X(1, 7) X(1, 8)
#undef X
}

// ---------------------------------------------------------------------------------------
// S2M with a stored tile order (operator reuse): the tree, the counting-sort
// histogram and each tile's stable order do not depend on b, so a new right-hand side needs
// only the moments.  TMA brings coordinates, weights and the tile order; one barrier per tile
// (inputs and bin tables double-buffered); 4-lane group g owns box g % nbox with its moments
// in registers across the CTA's tiles, reduced once at the end (fixed order: deterministic).
// ---------------------------------------------------------------------------------------
template <int D, int P>
__global__ void __launch_bounds__(TM_THREADS, 1) k_s2m_ord(LocalS2MArgs a) {
  constexpr int M = IPow<P, D>::value;
  static_assert(M <= 64, "register-resident moments");
  extern __shared__ __align__(128) unsigned char smraw[];
  const int nb = 1 << a.bits;
  // rawx[2][TILE*D] | rawb[2][TILE] | rawo[2][TILE] u16 | wsl[GROUPS][M] | geo | tab[2][2 nb] | off[2][2 nb] | bars
  float* rawx = reinterpret_cast<float*>(smraw);
  float* rawb = rawx + 2 * TM_TILE * D;
  uint16_t* rawo = reinterpret_cast<uint16_t*>(rawb + 2 * TM_TILE);
  float* wsl = reinterpret_cast<float*>(rawo + 2 * TM_TILE);
  float* geo = wsl + TM_GROUPS * M;
  uint32_t* tab = reinterpret_cast<uint32_t*>(geo + ((2 * D * a.nbox + 3) / 4) * 4);  // lstart | cnt
  uint32_t* off = tab + 2 * 2 * nb;
  uint64_t* bars = reinterpret_cast<uint64_t*>(off + ((2 * 2 * nb + 3) / 4) * 4);

  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int grp = threadIdx.x / TM_G, gl = threadIdx.x % TM_G;
  const int t = (a.bits - a.shift) / D;
  const int per = 1 << a.shift;
  tm_box_geometry<D>(a.nbox, t, a.alpha, a.l, geo);
  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_barrier_init();
  }
  const int tpb = (a.num_tiles + gridDim.x - 1) / gridDim.x;
  const int t_begin = blockIdx.x * tpb, t_end = min(a.num_tiles, t_begin + tpb);
  const float scale = (float)(2.0 / a.l);
  const bool aligned = ((reinterpret_cast<uintptr_t>(a.X) | reinterpret_cast<uintptr_t>(a.b)) & 15) == 0;
  const int64_t scan_len = (int64_t)nb * a.sort_tiles;
  auto full_tile = [&](int tile) { return aligned && (int64_t)(tile + 1) * TM_TILE <= a.n; };
  auto issue = [&](int tile, int buf) {
    if (tile < t_end && full_tile(tile) && threadIdx.x == 0) {
      fence_proxy_async();
      const int64_t r0 = (int64_t)tile * TM_TILE;
      mbar_expect_tx(&bars[buf], (uint32_t)(TM_TILE * (D * 4 + 4 + 2)));
      tma_g2s(rawx + buf * TM_TILE * D, a.X + r0 * D, (uint32_t)(TM_TILE * D * 4), &bars[buf]);
      tma_g2s(rawb + buf * TM_TILE, a.b + r0, (uint32_t)(TM_TILE * 4), &bars[buf]);
      tma_g2s(rawo + buf * TM_TILE, a.lrank + r0, (uint32_t)(TM_TILE * 2), &bars[buf]);
    }
  };
  auto prefetch_offsets = [&](int tile, int buf) {
    if (w == 0 && tile < t_end) {
      uint32_t* o = off + buf * 2 * nb;
      for (int b = lane; b < nb; b += 32) {
        const int64_t idx = (int64_t)b * a.sort_tiles + tile;
        cp_async4(o + b, a.offsets + idx);
        if (idx + 1 < scan_len) cp_async4(o + nb + b, a.offsets + idx + 1);
        else o[nb + b] = (uint32_t)a.n;
      }
    }
  };
  constexpr bool X2 = (D == 3 && P == 4);  // packed FFMA2 accumulation (far_math.cuh)
  float acc[X2 ? 1 : M];
  float2 acc2[X2 ? M / 2 : 1];
#pragma unroll
  for (int k2 = 0; k2 < (X2 ? 1 : M); ++k2) acc[k2] = 0.f;
#pragma unroll
  for (int k2 = 0; k2 < (X2 ? M / 2 : 1); ++k2) acc2[k2] = make_float2(0.f, 0.f);
  const int G = TM_GROUPS / a.nbox;
  const int B = grp % a.nbox, sub = grp / a.nbox;
  float lh[D], ll[D];
  __syncthreads();
#pragma unroll
  for (int d = 0; d < D; ++d) { lh[d] = geo[(B * D + d) * 2]; ll[d] = geo[(B * D + d) * 2 + 1]; }
  issue(t_begin, 0);
  prefetch_offsets(t_begin, 0);
  uint32_t phase = 0;
  for (int tile = t_begin, k = 0; tile < t_end; ++tile, ++k) {
    const int buf = k & 1;
    const int64_t tile0 = (int64_t)tile * TM_TILE;
    const int tvalid = (int)min((int64_t)TM_TILE, a.n - tile0);
    float* rx = rawx + buf * TM_TILE * D;
    float* rb = rawb + buf * TM_TILE;
    uint16_t* ro = rawo + buf * TM_TILE;
    uint32_t* lstart = tab + buf * 2 * nb;
    if (w == 0) {  // exclusive scan of the tile's bin counts -> lstart
      cp_async_wait_all();
      __syncwarp();
      const uint32_t* o = off + buf * 2 * nb;
      constexpr int BPL = 8;
      uint32_t c[BPL];
      uint32_t loc = 0;
#pragma unroll
      for (int r = 0; r < BPL; ++r) {
        const int b = lane * BPL + r;
        c[r] = b < nb ? o[nb + b] - o[b] : 0u;
        loc += c[r];
      }
      uint32_t inc = loc;
#pragma unroll
      for (int sh = 1; sh < 32; sh <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, sh);
        if (lane >= sh) inc += y;
      }
      uint32_t run = inc - loc;
#pragma unroll
      for (int r = 0; r < BPL; ++r) {
        const int b = lane * BPL + r;
        if (b < nb) {
          lstart[b] = run;
          run += c[r];
        }
      }
    }
    if (full_tile(tile)) {
      mbar_wait(&bars[buf], (phase >> buf) & 1u);
      phase ^= 1u << buf;
    } else {
      for (int e = threadIdx.x; e < tvalid * D; e += TM_THREADS) rx[e] = __ldg(a.X + tile0 * D + e);
      for (int e = threadIdx.x; e < tvalid; e += TM_THREADS) {
        rb[e] = __ldg(a.b + tile0 + e);
        ro[e] = __ldg(a.lrank + tile0 + e);
      }
    }
    __syncthreads();  // the only barrier of the iteration
    issue(tile + 1, buf ^ 1);
    prefetch_offsets(tile + 1, buf ^ 1);
    const int beg = (int)lstart[B * per];
    const int end = (B + 1) * per < nb ? (int)lstart[(B + 1) * per] : tvalid;
    int p = beg + sub * TM_G + gl;
    if (p < end) {
      // software pipeline: the next point's order entry, coordinates and weight load while this
      // one is accumulated
      int on = ro[p];
      float xn[D], bn = rb[on];
#pragma unroll
      for (int d = 0; d < D; ++d) xn[d] = rx[on * D + d];
      for (; p < end; p += TM_G * G) {
        float xo[D];
#pragma unroll
        for (int d = 0; d < D; ++d) xo[d] = xn[d];
        const float bo = bn;
        if (p + TM_G * G < end) {
          on = ro[p + TM_G * G];
          bn = rb[on];
#pragma unroll
          for (int d = 0; d < D; ++d) xn[d] = rx[on * D + d];
        }
        float T[D][P];
#pragma unroll
        for (int d = 0; d < D; ++d) chebyshev<P>(local_tau_off(xo[d], scale, lh[d], ll[d]), T[d]);
        if constexpr (X2) s2m_accumulate_d3p4_x2(bo, T, acc2);
        else s2m_accumulate<D, P>(bo, T, acc);
      }
    }
  }
  __syncthreads();
  if constexpr (X2) {
    float accs[M];
#pragma unroll
    for (int q = 0; q < M / 2; ++q) { accs[2 * q] = acc2[q].x; accs[2 * q + 1] = acc2[q].y; }
    tm_owned_flush<M, false>(accs, wsl + grp * M, gl);
  } else {
    tm_owned_flush<M, false>(acc, wsl + grp * M, gl);
  }
  __syncthreads();
  float* out = a.Wpart + (int64_t)blockIdx.x * a.nbox * M;
  for (int e = threadIdx.x; e < a.nbox * M; e += TM_THREADS) {
    const int Bx = e / M, k2 = e - Bx * M;
    float sum = 0.f;
    for (int s2 = 0; s2 < G; ++s2) sum += wsl[(s2 * a.nbox + Bx) * M + k2];
    out[e] = sum;
  }
}

// ---------------------------------------------------------------------------------------
// Deferred counting-sort scatter from the stored tile orders (the global-sorted far field and
// the near field need the points in box order, Sec. 4.1): one CTA per tile
// stages the tile's coordinates, weights and sorted order in shared memory, then one warp per
// bin writes that bin's run (pi, sorted SoA coordinates, sorted weights, keys) contiguously
// at its scanned destination, and sigma (original -> sorted) for the tile's points.
// ---------------------------------------------------------------------------------------
template <int D>
__global__ void __launch_bounds__(TM_THREADS) k_scatter_ord(LocalS2MArgs a) {
  extern __shared__ __align__(16) unsigned char smraw[];
  const int nb = 1 << a.bits;
  float* rx = reinterpret_cast<float*>(smraw);               // [TILE * D]
  float* rb = rx + TM_TILE * D;                              // [TILE]
  uint16_t* ro = reinterpret_cast<uint16_t*>(rb + TM_TILE);  // [TILE]
  uint32_t* lstart = reinterpret_cast<uint32_t*>(ro + TM_TILE);
  uint32_t* ltot = lstart + nb;
  uint32_t* goff = ltot + nb;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int tile = blockIdx.x;
  const int64_t tile0 = (int64_t)tile * TM_TILE;
  const int tvalid = (int)min((int64_t)TM_TILE, a.n - tile0);
  const int64_t scan_len = (int64_t)nb * a.sort_tiles;
  for (int e = threadIdx.x; e < tvalid * D; e += TM_THREADS) rx[e] = __ldg(a.X + tile0 * D + e);
  for (int e = threadIdx.x; e < tvalid; e += TM_THREADS) {
    if (a.xs) rb[e] = __ldg(a.b + tile0 + e);
    ro[e] = __ldg(a.lrank + tile0 + e);
  }
  for (int b = threadIdx.x; b < nb; b += TM_THREADS) {
    const int64_t idx = (int64_t)b * a.sort_tiles + tile;
    const uint32_t cur = a.offsets[idx];
    const uint32_t nxt = (idx + 1 < scan_len) ? a.offsets[idx + 1] : (uint32_t)a.n;
    ltot[b] = nxt - cur;
    goff[b] = cur;
  }
  __syncthreads();
  if (w == 0) {
    constexpr int BPL = 8;
    uint32_t loc = 0;
#pragma unroll
    for (int r = 0; r < BPL; ++r) {
      const int b = lane * BPL + r;
      if (b < nb) loc += ltot[b];
    }
    uint32_t inc = loc;
#pragma unroll
    for (int sh = 1; sh < 32; sh <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, inc, sh);
      if (lane >= sh) inc += y;
    }
    uint32_t run = inc - loc;
#pragma unroll
    for (int r = 0; r < BPL; ++r) {
      const int b = lane * BPL + r;
      if (b < nb) {
        lstart[b] = run;
        run += ltot[b];
      }
    }
  }
  __syncthreads();
  for (int bin = w; bin < nb; bin += TM_WARPS) {
    const int ls = (int)lstart[bin], lt = (int)ltot[bin];
    const uint32_t g0 = goff[bin];
    for (int e = lane; e < lt; e += 32) {
      const int o = ro[ls + e];
      const uint32_t dst = g0 + (uint32_t)e;
      a.perm[dst] = (int32_t)(tile0 + o);
      if (a.xs) {
#pragma unroll
        for (int d = 0; d < D; ++d) a.xs[(int64_t)d * a.n + dst] = rx[o * D + d];
        a.bs[dst] = rb[o];
      }
      if (a.sigma) a.sigma[tile0 + o] = (int32_t)dst;
      if (a.keys) a.keys[dst] = (uint64_t)bin;
    }
  }
}

static size_t scatter_ord_smem(int D, int nb) {
  return (size_t)TM_TILE * (D * 4 + 4 + 2) + (size_t)3 * 4 * nb;
}

void launch_scatter_ord(int D, const LocalS2MArgs& a, cudaStream_t st) {
  const size_t sm = scatter_ord_smem(D, 1 << a.bits);
#define X(d)                                                                                      \
  if (D == d) {                                                                                   \
    cudaFuncSetAttribute(k_scatter_ord<d>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm); \
    k_scatter_ord<d><<<a.num_tiles, TM_THREADS, sm, st>>>(a);                                     \
    return;                                                                                       \
  }
  X(1) X(2) X(3) X(4) X(5) X(6) X(7)
#undef X
}

// ---------------------------------------------------------------------------------------
// Warp-specialised S2M (the headline configuration's dominant kernel).  The fused kernel
// above runs ranking and moments back to back in every tile, separated by CTA barriers, so
// the FP32 pipe idles while the tile is ranked and the integer/ballot work idles while the
// moments accumulate.  Here warps 0-7 (the rank group) rank tile k+1 while warps 8-15 (the
// moment group) accumulate the moments of tile k, with a three-stage shared-memory ring
// (coordinates, weights, tile order, bin table) and mbarrier hand-offs instead of
// __syncthreads:
//   full[s]     TMA bytes of the stage landed (or the rank group's plain loads, partial tile)
//   ranked[s]   the rank group published the tile order and bin table of the stage (256 arrivals)
//   consumed[s] the moment group is done with the stage (256 arrivals) -> TMA may refill it
// Outputs are those of k_s2m_tma: per-tile bin counts, the tile orders (sorted form), and
// per-CTA moments of every box (owned groups, fixed order: deterministic).
// Requirements: exact-threshold digits with 2^T - 1 <= 7, nb = 2^{D T} <= 64, nbox <= 64,
// m <= 64 (launch_s2m_ws_supported).
// ---------------------------------------------------------------------------------------
constexpr int WS_RW = 8;                  // rank warps
constexpr int WS_MW = 8;                  // moment warps
constexpr int WS_ITEMS = TM_TILE / (WS_RW * 32);  // 16 items per rank lane
constexpr int WS_WP = WS_RW + 1;
constexpr int WS_STAGES = 3;
constexpr int WS_NBMAX = 64;
constexpr int WS_GROUPS = WS_MW * 32 / TM_G;     // 64 moment groups

// Named barriers of the two groups.  barrier.sync (not the .aligned bar.sync) because a warp
// may arrive with diverged lanes after its data-dependent loops (compute-sanitizer synccheck).
__device__ __forceinline__ void ws_bar_rank() { asm volatile("barrier.sync 1, %0;" ::"n"(WS_RW * 32) : "memory"); }
__device__ __forceinline__ void ws_bar_all() { asm volatile("barrier.sync 2, %0;" ::"n"(TM_THREADS) : "memory"); }

// Stable warp-local ranks of the rank lane's WS_ITEMS items (items j*32 + lane of the warp's
// segment), in two phases so that the per-item histogram read-modify-write is the only serial
// chain: (1) for every item, digits from the exact thresholds as D*T predicates and the peers
// (same-digit lanes) from one ballot per predicate -- independent across items, so the loads,
// compares and ballots of all items overlap; (2) the running per-warp counts whist[digit][rw]
// item by item (one shared load, one leader store each).  FULL: every item is valid (no
// validity ballot, the common case); otherwise items at or beyond tvalid get rank -1.
template <int D, int T, bool FULL>
__device__ __forceinline__ void ws_rank_items(const float* rx, int segl, int lane, int tvalid, const float (&th)[D * ((1 << T) - 1)],
                                              uint32_t* whist, int rw, uint32_t (&dig)[WS_ITEMS], int (&wrank)[WS_ITEMS]) {
  constexpr int BITS = D * T;
  const unsigned lt = (1u << lane) - 1u;
  unsigned peers[WS_ITEMS];
#pragma unroll
  for (int j = 0; j < WS_ITEMS; ++j) {
    const int o = segl + j * 32 + lane;
    float x[D];
#pragma unroll
    for (int d = 0; d < D; ++d) x[d] = rx[o * D + d];
    const bool valid = FULL || o < tvalid;
    bool bits[BITS];
    tm_bits_thr<D, T>(x, th, bits);
    unsigned pj = FULL ? 0xffffffffu : __ballot_sync(0xffffffffu, valid);
    uint32_t dj = 0;
#pragma unroll
    for (int i = 0; i < BITS; ++i) {
      const unsigned bb = __ballot_sync(0xffffffffu, bits[i]);
      pj &= bits[i] ? bb : ~bb;
      dj |= bits[i] ? (1u << i) : 0u;
    }
    dig[j] = dj;
    peers[j] = valid ? pj : 0u;
  }
#pragma unroll
  for (int j = 0; j < WS_ITEMS; ++j) {
    const uint32_t base = whist[dig[j] * WS_WP + rw];
    const unsigned pj = peers[j];
    wrank[j] = pj ? (int)(base + __popc(pj & lt)) : -1;
    __syncwarp();
    if (pj && (pj & lt) == 0) whist[dig[j] * WS_WP + rw] = base + __popc(pj);
    __syncwarp();
  }
}

// MODE 0: the single-pass headline kernel; 1: one launch over the two-digit path's buckets;
// 2: ranking only (tile orders and counts, no moments: the two-digit path's top digit)
template <int D, int P, int T, int MODE>
__global__ void __launch_bounds__(TM_THREADS, 1) k_s2m_ws(LocalS2MArgs a) {
  constexpr bool BK = MODE == 1, MOM = MODE != 2;
  constexpr int M = IPow<P, D>::value;
  static_assert(M <= 64, "register-resident moments");
  constexpr int NT = (1 << T) - 1;
  constexpr int BITS = D * T;
  static_assert(BITS <= 6, "nb <= 64");
  constexpr int NB = 1 << BITS;
  constexpr int BPL = NB > 32 ? 2 : 1;  // bins per lane in the offset computation
  constexpr int STAGE_BYTES = TM_TILE * (D * 4 + 4 + 2);
  extern __shared__ __align__(128) unsigned char smraw[];
  // [stage]{ rx[TILE*D] f32 | rb[TILE] f32 | so[TILE] u16 } | tab[stage][2 NB] | whist[2][NB][WS_WP] |
  // offw[WS_RW][NB] | bars[3 * STAGES]
  uint32_t* tab = reinterpret_cast<uint32_t*>(smraw + WS_STAGES * STAGE_BYTES);
  uint32_t* whist2 = tab + WS_STAGES * 2 * NB;
  uint32_t* offw = whist2 + 2 * NB * WS_WP;
  uint64_t* bars = reinterpret_cast<uint64_t*>(offw + WS_RW * NB);
  uint64_t* full = bars;
  uint64_t* ranked = bars + WS_STAGES;
  uint64_t* consumed = bars + 2 * WS_STAGES;
  auto stage_rx = [&](int s) { return reinterpret_cast<float*>(smraw + s * STAGE_BYTES); };
  auto stage_rb = [&](int s) { return stage_rx(s) + TM_TILE * D; };
  auto stage_so = [&](int s) { return reinterpret_cast<uint16_t*>(stage_rb(s) + TM_TILE); };

  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int t = (a.bits - a.shift) / D;
  if (threadIdx.x == 0) {
    for (int s = 0; s < WS_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&ranked[s], WS_RW * 32);    // every rank thread arrives after its own writes
      mbar_init(&consumed[s], WS_MW * 32);  // every moment thread arrives after its last read
    }
    fence_barrier_init();
  }
  const int tpb = (a.num_tiles + gridDim.x - 1) / gridDim.x;
  const int t_begin = blockIdx.x * tpb, t_end = min(a.num_tiles, t_begin + tpb);
  const int ntile = max(0, t_end - t_begin);
  const bool aligned = ((reinterpret_cast<uintptr_t>(a.X) | reinterpret_cast<uintptr_t>(a.b)) & 15) == 0;
  // tile g -> (bucket, tile of the bucket, valid points); one bucket outside MODE 1
  struct TileInfo { int bk, lt, tvalid; };
  auto tinfo = [&](int g) -> TileInfo {
    if (!BK) return {0, g, (int)min((int64_t)TM_TILE, a.n - (int64_t)g * TM_TILE)};
    const int2 e = __ldg(a.bk_tile + g);
    return {e.x & 0xff, e.y, e.x >> 8};
  };
  auto full_tile = [&](int r) { return aligned && tinfo(t_begin + r).tvalid == TM_TILE; };
  auto issue = [&](int r) {  // one thread: TMA of relative tile r into stage r % 3
    if (r < ntile && full_tile(r)) {
      const int s = r % WS_STAGES;
      fence_proxy_async();
      const int64_t r0 = (int64_t)(t_begin + r) * TM_TILE;
      mbar_expect_tx(&full[s], (uint32_t)(TM_TILE * (D + 1) * 4));
      tma_g2s(stage_rx(s), a.X + r0 * D, (uint32_t)(TM_TILE * D * 4), &full[s]);
      tma_g2s(stage_rb(s), a.b + r0, (uint32_t)(TM_TILE * 4), &full[s]);
    }
  };
  __syncthreads();
  if (threadIdx.x == 0) { issue(0); issue(1); issue(2); }
  const float scale = (float)(2.0 / a.l);
  const int G = WS_GROUPS / a.nbox;
  // rank group = warps 8-15, moment group = warps 0-7 (each SM sub-partition runs two of each;
  // placing the groups on separate sub-partitions halves the FMA pipes the moment group can use
  // and was measured 2x slower)
  const bool is_rank = w >= WS_MW;
  const int gw = w & 7;  // warp index inside its group
  const int grp = (gw * 32 + lane) / TM_G, gl = lane % TM_G;

  if (is_rank) {
    // ================= rank group =================
    // One named barrier per tile: the warp histograms are double-buffered by tile parity, and
    // every warp derives its own scatter offsets from all of them (no block-wide scan).
    const int rw = gw, rt = gw * 32 + lane;
    float th[D * NT];
    int cur_bk = -1;
    const int segl = rw * (TM_TILE / WS_RW);
    uint32_t* myoff = offw + rw * NB;
    for (int r = 0; r < ntile; ++r) {
      const int s = r % WS_STAGES, u = r / WS_STAGES;
      const int64_t tile0 = (int64_t)(t_begin + r) * TM_TILE;
      const TileInfo ti = tinfo(t_begin + r);
      const int tvalid = ti.tvalid;
      if (ti.bk != cur_bk) {  // exact thresholds of the tile's bucket
        const float* src = BK ? a.bk_thr + (size_t)ti.bk * D * NT : a.kp.thr;
#pragma unroll
        for (int e = 0; e < D * NT; ++e) th[e] = src[e];
        cur_bk = ti.bk;
      }
      float* rx = stage_rx(s);
      float* rb = stage_rb(s);
      uint16_t* so = stage_so(s);
      uint32_t* whist = whist2 + (r & 1) * NB * WS_WP;
      if (full_tile(r)) {
        mbar_wait_sleep(&full[s], u & 1);
        __syncwarp();
      } else {  // partial / unaligned tile: the rank group loads it (published via ranked[s])
        if (r >= WS_STAGES) mbar_wait(&consumed[s], ((r - WS_STAGES) / WS_STAGES) & 1);  // stage free
        for (int e = rt; e < tvalid * D; e += WS_RW * 32) rx[e] = __ldg(a.X + tile0 * D + e);
        for (int e = rt; e < tvalid; e += WS_RW * 32) rb[e] = __ldg(a.b + tile0 + e);
        ws_bar_rank();
        // complete the stage's `full` phase without bytes, so that its parity stays in step
        // with the stage's uses (bucket mode has partial tiles inside the CTA's range)
        if (rt == 0) mbar_arrive(&full[s]);
      }
      for (int b = lane; b < NB; b += 32) whist[b * WS_WP + rw] = 0;
      __syncwarp();
      uint32_t dig[WS_ITEMS];
      int wrank[WS_ITEMS];
      const bool fullt = tvalid == TM_TILE;
      if (fullt) ws_rank_items<D, T, true>(rx, segl, lane, tvalid, th, whist, rw, dig, wrank);
      else ws_rank_items<D, T, false>(rx, segl, lane, tvalid, th, whist, rw, dig, wrank);
      ws_bar_rank();  // every warp's histogram of this tile is complete
      // offsets: bin b of warp rw starts at sum_{b' < b} tot[b'] + sum_{w' < rw} whist[b][w']
      uint32_t tot[BPL], pre[BPL];
      uint32_t loc = 0;
#pragma unroll
      for (int q = 0; q < BPL; ++q) {
        const int b = lane * BPL + q;
        tot[q] = 0u;
        pre[q] = 0u;
        if (b < NB) {
#pragma unroll
          for (int w2 = 0; w2 < WS_RW; ++w2) {
            const uint32_t c = whist[b * WS_WP + w2];
            tot[q] += c;
            pre[q] += w2 < rw ? c : 0u;
          }
        }
        loc += tot[q];
      }
      uint32_t inc = loc;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
      }
      uint32_t run = inc - loc;
      uint32_t* lstart = tab + s * 2 * NB;
      uint32_t* ltot = lstart + NB;
#pragma unroll
      for (int q = 0; q < BPL; ++q) {
        const int b = lane * BPL + q;
        if (b < NB) {
          myoff[b] = run + pre[q];
          if (rw == 0) {
            lstart[b] = run;
            ltot[b] = tot[q];
            if (a.counts) {
              if (BK)
                a.counts[a.bk_coff[ti.bk] + (int64_t)b * (a.bk_tile0[ti.bk + 1] - a.bk_tile0[ti.bk]) + ti.lt] = tot[q];
              else
                a.counts[(int64_t)b * a.num_tiles + t_begin + r] = tot[q];
            }
          }
        }
        run += tot[q];
      }
      __syncwarp();
#pragma unroll
      for (int j = 0; j < WS_ITEMS; ++j)
        if (wrank[j] >= 0) so[(int)myoff[dig[j]] + wrank[j]] = (uint16_t)(segl + j * 32 + lane);
      mbar_arrive(&ranked[s]);
    }
    __syncwarp();
    ws_bar_all();
  } else {
    // ================= moment group =================
    const int B = grp % a.nbox, sub = grp / a.nbox;
    const int per = 1 << a.shift;
    const int mt = gw * 32 + lane;
    float lh[D], ll[D];  // box geometry (the arithmetic of tm_box_geometry)
    auto geometry = [&](int bk) {
      const double sc = (double)(float)(2.0 / a.l);
#pragma unroll
      for (int d = 0; d < D; ++d) {
        int cell = 0;
        for (int q = 0; q < t; ++q) cell |= ((B >> (D * q + d)) & 1) << q;
        cell += BK ? a.bk_cell[bk * D + d] : a.cell_base[d];
        const double lo = a.alpha[d] + (double)cell * a.l;
        const double of = -fma(lo, sc, 1.0);
        lh[d] = (float)of;
        ll[d] = (float)(of - (double)lh[d]);
      }
    };
    int cur_bk = (BK && ntile > 0) ? tinfo(t_begin).bk : 0;
    geometry(cur_bk);
    constexpr bool X2 = (D == 3 && P == 4);  // packed FFMA2 accumulation (far_math.cuh)
    float acc[X2 ? 1 : M];
    float2 acc2[X2 ? M / 2 : 1];
#pragma unroll
    for (int k2 = 0; k2 < (X2 ? 1 : M); ++k2) acc[k2] = 0.f;
#pragma unroll
    for (int k2 = 0; k2 < (X2 ? M / 2 : 1); ++k2) acc2[k2] = make_float2(0.f, 0.f);
    // bucket mode: the group's moments of one bucket go straight to Wpart[bucket][CTA][box]
    // (one group per box) when the CTA's tile range leaves the bucket, and at the end
    auto flush_bucket = [&](int bk) {
      float accs[M];
      if constexpr (X2) {
#pragma unroll
        for (int q = 0; q < M / 2; ++q) {
          accs[2 * q] = acc2[q].x;
          accs[2 * q + 1] = acc2[q].y;
          acc2[q] = make_float2(0.f, 0.f);
        }
      } else {
#pragma unroll
        for (int q = 0; q < M; ++q) { accs[q] = acc[q]; acc[q] = 0.f; }
      }
      tm_group4_reduce_scatter<M>(accs);
      float* out = a.Wpart + (((int64_t)bk * gridDim.x + blockIdx.x) * a.nbox + B) * M + gl * (M / 4);
#pragma unroll
      for (int q = 0; q < M / 4; ++q) out[q] = accs[q];
    };
    for (int r = 0; r < ntile; ++r) {
      const int s = r % WS_STAGES, u = r / WS_STAGES;
      const int64_t tile0 = (int64_t)(t_begin + r) * TM_TILE;
      const TileInfo ti = tinfo(t_begin + r);
      const int tvalid = ti.tvalid;
      if (BK && ti.bk != cur_bk) {
        flush_bucket(cur_bk);
        cur_bk = ti.bk;
        geometry(cur_bk);
      }
      mbar_wait_sleep(&ranked[s], u & 1);
      __syncwarp();
      const float* rx = stage_rx(s);
      const float* rb = stage_rb(s);
      const uint16_t* so = stage_so(s);
      const uint32_t* lstart = tab + s * 2 * NB;
      const int beg = (int)lstart[B * per];
      const int end = (B + 1) * per < NB ? (int)lstart[(B + 1) * per] : tvalid;
      int p = beg + sub * TM_G + gl;
      if (MOM && p < end) {
        // software pipeline: the next point's order entry, coordinates and weight are loaded
        // while the current one is accumulated (prefetch index clamped to the box: no branch)
        // [a two-register-set unroll like k_l2t_fix's measured slower here: 6.6 -> 7.0 ms]
        const uint32_t rx_s = smem_u32(rx), rb_s = smem_u32(rb), so_s = smem_u32(so);
        const int stp = TM_G * G;
        int on = (int)lds_u16(so_s + 2u * p);
        float xn[D], bn = lds_f32(rb_s + 4u * on);
#pragma unroll
        for (int d = 0; d < D; ++d) xn[d] = lds_f32(rx_s + 4u * (on * D + d));
        for (; p < end; p += stp) {
          float xo[D];
#pragma unroll
          for (int d = 0; d < D; ++d) xo[d] = xn[d];
          const float bo = bn;
          on = (int)lds_u16(so_s + 2u * min(p + stp, end - 1));
          bn = lds_f32(rb_s + 4u * on);
#pragma unroll
          for (int d = 0; d < D; ++d) xn[d] = lds_f32(rx_s + 4u * (on * D + d));
          float Tc[D][P];
          if constexpr (X2) {
            cheb_d3p4_x2(xo, scale, lh, ll, Tc);
            s2m_accumulate_d3p4_x2(bo, Tc, acc2);
          } else {
#pragma unroll
            for (int d = 0; d < D; ++d) chebyshev<P>(local_tau_off(xo[d], scale, lh[d], ll[d]), Tc[d]);
            s2m_accumulate<D, P>(bo, Tc, acc);
          }
        }
      }
      // the tile's stable order for the L2T pass (sorted position -> original local index)
      if (a.lrank) {
        if (tvalid == TM_TILE && aligned) {  // 16 entries (32 B) per thread
          const uint4* src = reinterpret_cast<const uint4*>(so) + mt * 2;
          uint4* dst = reinterpret_cast<uint4*>(a.lrank + tile0) + mt * 2;
          dst[0] = src[0];
          dst[1] = src[1];
        } else {
          for (int e = mt; e < tvalid; e += WS_MW * 32) a.lrank[tile0 + e] = so[e];
        }
      }
      mbar_arrive(&consumed[s]);
      // refill: once all moment warps released the stage (tile order copied out too), moment
      // warp 0 brings relative tile r + 3 into it (the rank group never waits on the moment group)
      if (gw == 0 && r + WS_STAGES < ntile) {
        if (lane == 0) {
          mbar_wait(&consumed[s], u & 1);
          issue(r + WS_STAGES);
        }
        __syncwarp();
      }
    }
    __syncwarp();
    if (BK && ntile > 0) flush_bucket(cur_bk);
    ws_bar_all();  // both groups are done with the ring: flush into the stage-0 coordinates
    if (BK || !MOM) {
      // moments already written per bucket, or a ranking-only pass
    } else if constexpr (X2) {
      float accs[M];
#pragma unroll
      for (int q = 0; q < M / 2; ++q) { accs[2 * q] = acc2[q].x; accs[2 * q + 1] = acc2[q].y; }
      tm_owned_flush<M, false>(accs, stage_rx(0) + grp * M, gl);
    } else {
      tm_owned_flush<M, false>(acc, stage_rx(0) + grp * M, gl);
    }
  }
  __syncthreads();
  if (BK || !MOM) return;
  const float* wsl = stage_rx(0);
  float* out = a.Wpart + (int64_t)blockIdx.x * a.nbox * M;
  for (int e = threadIdx.x; e < a.nbox * M; e += TM_THREADS) {
    const int Bx = e / M, k2 = e - Bx * M;
    float sum = 0.f;
    for (int s2 = 0; s2 < G; ++s2) sum += wsl[(s2 * a.nbox + Bx) * M + k2];
    out[e] = sum;
  }
}

static size_t s2m_ws_smem(int D, int nbox) {
  return (size_t)WS_STAGES * TM_TILE * (D * 4 + 4 + 2) +
         (size_t)4 * (WS_STAGES * 2 * WS_NBMAX + 2 * WS_NBMAX * WS_WP + WS_RW * WS_NBMAX) + 8 * 3 * WS_STAGES + 16;
}

bool s2m_ws_supported(int D, int P, int T, int nbox) {
  if (!((D == 3 && P == 4 && T == 2) || (D == 3 && P == 3 && T == 2) || (D == 2 && P == 4 && T == 3) ||
        (D == 2 && P == 6 && T == 3) || (D == 3 && P == 4 && T == 1) || (D == 2 && P == 8 && T == 3)))
    return false;
  if (nbox > WS_GROUPS) return false;
  return s2m_ws_smem(D, nbox) <= 227 * 1024;
}

void launch_s2m_ws(int D, int P, int T, const LocalS2MArgs& a, int grid, cudaStream_t st) {
  const size_t sm = s2m_ws_smem(D, a.nbox);
#define X(d, p, tt, mode)                                                                                 \
  if (D == d && P == p && T == tt) {                                                                      \
    cudaFuncSetAttribute(k_s2m_ws<d, p, tt, mode>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm); \
    k_s2m_ws<d, p, tt, mode><<<grid, TM_THREADS, sm, st>>>(a);                                            \
    return;                                                                                               \
  }
  if (!a.do_s2m) {  // ranking only (two-digit path, top digit)
    X(3, 4, 2, 2)
  } else if (a.nbuckets) {  // one launch over the two-digit path's buckets
    X(3, 4, 2, 1) X(3, 3, 2, 1)
  } else {
    X(3, 4, 2, 0) X(3, 3, 2, 0) X(2, 4, 3, 0) X(2, 6, 3, 0) X(3, 4, 1, 0) X(2, 8, 3, 0)
  }
#undef X
}

#define F3M_ORD_CASES(X) \
  X(1, 2) X(1, 3) X(1, 4) X(1, 5) X(1, 6) X(1, 7) X(1, 8) \
  X(2, 2) X(2, 3) X(2, 4) X(2, 5) X(2, 6) X(2, 7) X(2, 8) \
  X(3, 2) X(3, 3) X(3, 4) X(4, 2) X(5, 2) X(6, 2)

static size_t s2m_ord_smem(int D, int nb, int nbox, int m) {
  return (size_t)2 * TM_TILE * (D * 4 + 4 + 2) + (size_t)TM_GROUPS * m * 4 + (size_t)((2 * D * nbox + 3) / 4) * 16 +
         (size_t)4 * 2 * 2 * nb + (size_t)((2 * 2 * nb + 3) / 4) * 16 + 64;
}

bool s2m_ord_supported(int D, int P, int nb, int nbox) {
  int m = 1;
  for (int d = 0; d < D; ++d) m *= P;
  if (m > 64 || nbox > TM_GROUPS || nb > 256 || s2m_ord_smem(D, nb, nbox, m) > 227 * 1024) return false;
#define X(d, p) if (D == d && P == p) return true;
  F3M_ORD_CASES(X)
#undef X
  return false;
}

void launch_s2m_ord(int D, int P, const LocalS2MArgs& a, int grid, cudaStream_t st) {
  int m = 1;
  for (int d = 0; d < D; ++d) m *= P;
  const size_t sm = s2m_ord_smem(D, 1 << a.bits, a.nbox, m);
#define X(d, p)                                                                                \
  if (D == d && P == p) {                                                                      \
    cudaFuncSetAttribute(k_s2m_ord<d, p>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm); \
    k_s2m_ord<d, p><<<grid, TM_THREADS, sm, st>>>(a);                                          \
    return;                                                                                    \
  }
  F3M_ORD_CASES(X)
#undef X
}

// ---------------------------------------------------------------------------------------
#define F3M_TMA_CASES(X) \
  X(1, 2) X(1, 3) X(1, 4) X(1, 5) X(1, 6) X(1, 7) X(1, 8) \
  X(2, 2) X(2, 3) X(2, 4) X(2, 5) X(2, 6) X(2, 7) X(2, 8) \
  X(3, 2) X(3, 3) X(3, 4) \
  X(4, 2) X(5, 2) X(6, 2) X(7, 2)

static size_t s2m_tma_smem(int D, int nb, int nbox, int m) {
  return (size_t)2 * TM_TILE * D * 4 + (size_t)2 * TM_TILE * 4 + (size_t)TM_TILE * 2 + tm_tables_bytes(nb) +
         (size_t)TM_GROUPS * m * 4 + (size_t)((2 * D * nbox + 3) / 4) * 16 + (size_t)((D * 255 + 3) / 4) * 16 + 64;
}
static size_t l2t_tma_smem(int D, int nb, int nbox, int m) {
  const int mrow = (m % 4 == 0) ? m + 4 : m;
  return (size_t)2 * TM_TILE * D * 4 + (size_t)2 * TM_TILE * 2 + (size_t)2 * TM_TILE * 4 + (size_t)nbox * mrow * 4 +
         (size_t)((2 * D * nbox + 3) / 4) * 16 + (size_t)4 * 2 * 3 * nb + (size_t)((2 * 2 * nb + 3) / 4) * 16 + 64;
}

// inverse of the per-tile permutation: out[tile0 + in[i]] = i - tile0 (tile-local ranks <->
// sorted-order local indices; only when the two tile-local passes use different kernels)
__global__ void k_tile_invert(const uint16_t* __restrict__ in, int64_t n, uint16_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t tile0 = i / TM_TILE * TM_TILE;
    out[tile0 + in[i]] = (uint16_t)(i - tile0);
  }
}

void launch_tile_invert(const uint16_t* in, int64_t n, uint16_t* out, cudaStream_t st) {
  if (n <= 0) return;
  k_tile_invert<<<148 * 8, 256, 0, st>>>(in, n, out);
}

bool tma_supported(int D, int P, int nb, int nbox, bool s2m_owned) {
  int m = 1;
  for (int d = 0; d < D; ++d) m *= P;
  if (s2m_owned && nbox > TM_GROUPS) return false;
  if (s2m_tma_smem(D, nb, nbox, m) > 227 * 1024 || l2t_tma_smem(D, nb, nbox, m) > 227 * 1024) return false;
#define X(d, p) if (D == d && P == p) return true;
  F3M_TMA_CASES(X)
#undef X
  return false;
}

int tma_grid(int num_tiles) {
  int g = 148;
  if (g > num_tiles) g = num_tiles;
  return g < 1 ? 1 : g;
}

void launch_s2m_tma(int D, int P, const LocalS2MArgs& a, int grid, cudaStream_t st) {
  int m = 1;
  for (int d = 0; d < D; ++d) m *= P;
  const size_t sm = s2m_tma_smem(D, 1 << a.bits, a.nbox, m);
#define X(d, p)                                                                                \
  if (D == d && P == p) {                                                                      \
    cudaFuncSetAttribute(k_s2m_tma<d, p>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm); \
    k_s2m_tma<d, p><<<grid, TM_THREADS, sm, st>>>(a);                                          \
    return;                                                                                    \
  }
  F3M_TMA_CASES(X)
#undef X
}

void launch_l2t_tma(int D, int P, const LocalL2TArgs& a, int grid, cudaStream_t st) {
  int m = 1;
  for (int d = 0; d < D; ++d) m *= P;
  const size_t sm = l2t_tma_smem(D, 1 << a.bits, a.nbox, m);
#define X(d, p)                                                                                       \
  if (D == d && P == p) {                                                                             \
    if (a.shift == 0) {                                                                               \
      cudaFuncSetAttribute(k_l2t_tma<d, p, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);  \
      k_l2t_tma<d, p, true><<<grid, TM_THREADS, sm, st>>>(a);                                         \
    } else {                                                                                          \
      cudaFuncSetAttribute(k_l2t_tma<d, p, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm); \
      k_l2t_tma<d, p, false><<<grid, TM_THREADS, sm, st>>>(a);                                        \
    }                                                                                                 \
    return;                                                                                           \
  }
  F3M_TMA_CASES(X)
#undef X
}

}  // namespace f3m
