// Tile-local far field for sm_100a: S2M fused with the stable counting-sort scatter, and
// L2T fused with the output permutation.  Used for far levels whose boxes fit one <= 8-bit
// digit of the key (D*t <= 8: every far level of config C4, EV = 1).
//
// Paper: Sec. 4.1 grouping by box and "box-to-threadblock alignment"
// (PAPER.md:165); Sec. 3 three-stage far field.  B200 design (DESIGN.md
// sec. 6): a persistent CTA owns a contiguous range of 4096-point tiles of the ORIGINAL
// order.  Per tile it
//   1. ranks the points by key in registers + shared memory (one ballot-multisplit pass,
//      warp-private histograms: the same stable order as the global counting sort) and
//      stages the coordinates (and weights) in key order in SMEM;
//   2. splits every box's run into pieces of <= 64 points; 4-lane groups (64 per CTA)
//      process one piece each:
//      * k_local_s2m: register accumulators for the P^D charges, 4-lane reduce-scatter,
//        piece partials to SMEM, then fixed-order per-(box, node) sums in fp64 registers
//        (deterministic); the permutation pi is written at the scanned counting-sort
//        destinations (and sigma / sorted copies when the global-sorted path needs them);
//      * k_local_l2t: the box's locals in registers, L2T sum per point, then v is written
//        back in the original order (coalesced) -- no global un-permutation pass.
// HBM: S2M reads X, b (4D+4 B/pt) and writes pi (4 B/pt); L2T reads X (4D B/pt), writes v.
#include <cuda_runtime.h>
#include <stdint.h>

#include "f3m_internal.h"
#include "far_math.cuh"

namespace f3m {

constexpr int LT_THREADS = 256;
constexpr int LT_WARPS = LT_THREADS / 32;
constexpr int LT_ITEMS = 16;
constexpr int LT_TILE = LT_THREADS * LT_ITEMS;  // 4096
static_assert(LT_TILE == LT_TILE_PTS, "tile size");
constexpr int LT_G = 4;                          // lanes per group
constexpr int LT_GROUPS = LT_THREADS / LT_G;     // 64 groups per CTA
constexpr int LT_PIECE = 128;                    // points per piece (32 per lane)
constexpr int LT_MAXPIECES = LT_TILE / LT_PIECE + 256;

// bit-exact cell (same arithmetic as kernels_sort.cu; reading R12)
__device__ __forceinline__ uint32_t lt_cell(float x, float alpha_f, double alpha, const KeyParams& kp) {
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

// nested Morton digit of T levels, D*T <= 8 (reading R13)
template <int D, int T>
__device__ __forceinline__ uint32_t lt_digit(const float (&x)[D], const float (&af)[D], const double (&ad)[D],
                                             const KeyParams& kp) {
  uint32_t c[D];
#pragma unroll
  for (int d = 0; d < D; ++d) c[d] = lt_cell(x[d], af[d], ad[d], kp);
  uint32_t K = 0;
#pragma unroll
  for (int s = T - 1; s >= 0; --s) {
#pragma unroll
    for (int d = D - 1; d >= 0; --d) K = (K << 1) | ((c[d] >> s) & 1u);
  }
  return K;
}

template <int BITS>
__device__ __forceinline__ unsigned lt_peers_t(uint32_t dig, unsigned valid) {
  unsigned peers = valid;
#pragma unroll
  for (int b = 0; b < BITS; ++b) {
    const unsigned bit = (dig >> b) & 1u;
    const unsigned bal = __ballot_sync(0xffffffffu, bit);
    peers &= bit ? bal : ~bal;
  }
  return peers;
}


// the ranking part of the shared memory, sized for nb digit bins and nbox boxes
struct LtShared {
  uint32_t* whist;    // [LT_WARPS][nb] warp histograms, then per-warp exclusive prefixes
  uint32_t* ltot;     // [nb] tile counts
  uint32_t* lstart;   // [nb] tile-local bin starts
  uint32_t* goff;     // [nb] global counting-sort destinations of the tile's bins
  uint32_t* bcnt;     // [nbox]
  uint32_t* pstart;   // [nbox + 1] first piece of each box
  int32_t* piece_box;
  int32_t* piece_beg;
  int32_t* piece_len;
  int32_t* npieces;
  int nb;
};

__host__ __device__ inline size_t lt_shared_bytes(int nb, int nbox) {
  const size_t maxp = LT_TILE / LT_PIECE + nbox;
  size_t b = 4 * ((size_t)LT_WARPS * nb + 3 * nb + nbox + nbox + 1) + 12 * maxp + 4;
  return (b + 15) / 16 * 16;
}

__device__ __forceinline__ LtShared lt_layout(unsigned char* base, int nb, int nbox) {
  LtShared S;
  uint32_t* u = reinterpret_cast<uint32_t*>(base);
  S.whist = u; u += LT_WARPS * nb;
  S.ltot = u; u += nb;
  S.lstart = u; u += nb;
  S.goff = u; u += nb;
  S.bcnt = u; u += nbox;
  S.pstart = u; u += nbox + 1;
  const int maxp = LT_TILE / LT_PIECE + nbox;
  int32_t* q = reinterpret_cast<int32_t*>(u);
  S.piece_box = q; q += maxp;
  S.piece_beg = q; q += maxp;
  S.piece_len = q; q += maxp;
  S.npieces = q;
  S.nb = nb;
  return S;
}

__device__ __forceinline__ uint32_t lt_block_scan(uint32_t v, uint32_t* wt, uint32_t& total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) wt[w] = inc;
  __syncthreads();
  if (w == 0) {
    const uint32_t t = lane < LT_WARPS ? wt[lane] : 0u;
    uint32_t ti = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, ti, o);
      if (lane >= o) ti += y;
    }
    if (lane < LT_WARPS) wt[lane] = ti - t;
    if (lane == 31) wt[32] = ti;
  }
  __syncthreads();
  const uint32_t r = wt[w] + inc - v;
  total = wt[32];
  __syncthreads();
  return r;
}

// Rank one tile.  Items: warp w owns the contiguous segment [w*512, (w+1)*512) of the tile,
// lane l its rows 32j + l (coalesced loads).  On return: x[j][d] (coordinates), dig[j],
// lpos[j] (local sorted position, -1 for padding), S.lstart/S.ltot per digit, and the
// piece list for boxes = digit >> shift.
// histogram pass for compile-time T (D*T <= 8): digits, warp ranks, warp histograms
template <int D, int T>
__device__ __forceinline__ void lt_hist(int64_t n, int64_t seg, const KeyParams& kp, const float (&af)[D],
                                        const double (&ad)[D], const LtShared& S, const float (&x)[LT_ITEMS][D],
                                        uint32_t (&dig)[LT_ITEMS], int (&wrank)[LT_ITEMS]) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  const int lim = (int)min((int64_t)(LT_TILE / LT_WARPS), max((int64_t)0, n - seg));
  uint32_t* wh = S.whist + w * S.nb;
#pragma unroll
  for (int j = 0; j < LT_ITEMS; ++j) {   // digits first (independent, full ILP)
    const bool valid = j * 32 + lane < lim;
    dig[j] = valid ? lt_digit<D, T>(x[j], af, ad, kp) : 0xffffffffu;
  }
#pragma unroll
  for (int j = 0; j < LT_ITEMS; ++j) {
    const uint32_t d = dig[j];
    const bool valid = d != 0xffffffffu;
    const unsigned peers = __match_any_sync(0xffffffffu, d);   // lanes with the same digit
    wrank[j] = valid ? (int)(wh[d] + __popc(peers & lt)) : -1;
    __syncwarp();
    if (valid && (peers & lt) == 0) wh[d] += __popc(peers);
    __syncwarp();
    if (!valid) dig[j] = 0;
  }
}

// One warp: (from_whist) per-bin prefix over the warps and tile bin counts ltot, then the
// tile bin starts lstart, box counts and the piece list of boxes = bin >> shift.
__device__ __forceinline__ void lt_tables(const LtShared& S, int nb, int shift, int nbox, bool from_whist,
                                          bool pieces) {
  const int lane = threadIdx.x & 31;
    constexpr int BPL = 256 / 32;  // bins per lane (nb <= 256)
    uint32_t loc = 0;
#pragma unroll
    for (int r = 0; r < BPL; ++r) {
      const int bin = lane * BPL + r;
      if (bin < nb) {
        if (from_whist) {
          uint32_t run = 0;
#pragma unroll
          for (int k = 0; k < LT_WARPS; ++k) {
            const uint32_t c = S.whist[(k) * S.nb + (bin)];
            S.whist[(k) * S.nb + (bin)] = run;
            run += c;
          }
          S.ltot[bin] = run;
        }
        loc += S.ltot[bin];
      }
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
      const int bin = lane * BPL + r;
      if (bin < nb) {
        S.lstart[bin] = run;
        run += S.ltot[bin];
      }
    }
    __syncwarp();
    // boxes B = bin >> shift (lane handles boxes lane*BPL .. +BPL)
    const int per = 1 << shift;
    uint32_t bcl[BPL], npl = 0;
#pragma unroll
    for (int r = 0; r < BPL; ++r) {
      const int B = lane * BPL + r;
      uint32_t c = 0;
      if (B < nbox)
        for (int k = 0; k < per; ++k) c += S.ltot[B * per + k];
      bcl[r] = c;
      npl += (c + LT_PIECE - 1) / LT_PIECE;
    }
    uint32_t pinc = npl;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, pinc, o);
      if (lane >= o) pinc += y;
    }
    uint32_t q = pinc - npl;
#pragma unroll
    for (int r = 0; r < BPL; ++r) {
      const int B = lane * BPL + r;
      if (B < nbox) {
        S.pstart[B] = q;
        S.bcnt[B] = bcl[r];
        const uint32_t b0 = S.lstart[B * per];
        for (uint32_t s0 = 0; pieces && s0 < bcl[r]; s0 += LT_PIECE, ++q) {
          S.piece_box[q] = B;
          S.piece_beg[q] = (int32_t)(b0 + s0);
          S.piece_len[q] = (int32_t)min((uint32_t)LT_PIECE, bcl[r] - s0);
        }
      }
    }
    if (lane == 31) {
      *S.npieces = (int)pinc;
      S.pstart[nbox] = pinc;
    }
  }

template <int D>
__device__ __forceinline__ void lt_rank(const float* __restrict__ X, int64_t n, int64_t tile0, const KeyParams& kp,
                                        const float (&af)[D], const double (&ad)[D], int bits, int shift, int nbox,
                                        const LtShared& S, float (&x)[LT_ITEMS][D], uint32_t (&dig)[LT_ITEMS],
                                        int (&lpos)[LT_ITEMS]) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  const int nb = 1 << bits;
  const int64_t seg = tile0 + (int64_t)w * (LT_TILE / LT_WARPS);
  for (int b = lane; b < nb; b += 32) S.whist[(w) * S.nb + (b)] = 0;
  const int lim = (int)min((int64_t)(LT_TILE / LT_WARPS), max((int64_t)0, n - seg));  // valid items of this warp
  const float* Xs = X + seg * D;
#pragma unroll
  for (int j = 0; j < LT_ITEMS; ++j) {
    const int o = j * 32 + lane;
#pragma unroll
    for (int d = 0; d < D; ++d) x[j][d] = (o < lim) ? __ldg(Xs + o * D + d) : 0.f;
  }
  __syncwarp();
  int wrank[LT_ITEMS];
  switch (kp.T) {  // warp-uniform: the digit and its ballots unrolled for the exact depth
    case 1: lt_hist<D, 1>(n, seg, kp, af, ad, S, x, dig, wrank); break;
    case 2: if constexpr (D * 2 <= 8) { lt_hist<D, 2>(n, seg, kp, af, ad, S, x, dig, wrank); } break;
    case 3: if constexpr (D * 3 <= 8) { lt_hist<D, 3>(n, seg, kp, af, ad, S, x, dig, wrank); } break;
    case 4: if constexpr (D * 4 <= 8) { lt_hist<D, 4>(n, seg, kp, af, ad, S, x, dig, wrank); } break;
    case 5: if constexpr (D * 5 <= 8) { lt_hist<D, 5>(n, seg, kp, af, ad, S, x, dig, wrank); } break;
    case 6: if constexpr (D * 6 <= 8) { lt_hist<D, 6>(n, seg, kp, af, ad, S, x, dig, wrank); } break;
    case 7: if constexpr (D * 7 <= 8) { lt_hist<D, 7>(n, seg, kp, af, ad, S, x, dig, wrank); } break;
    default: if constexpr (D * 8 <= 8) { lt_hist<D, 8>(n, seg, kp, af, ad, S, x, dig, wrank); } break;
  }
  __syncthreads();
  // per-bin prefix over the warps (all threads, one bin each), then the tables (warp 0)
  for (int b = threadIdx.x; b < nb; b += LT_THREADS) {
    uint32_t run = 0;
#pragma unroll
    for (int k = 0; k < LT_WARPS; ++k) {
      const uint32_t c = S.whist[k * S.nb + b];
      S.whist[k * S.nb + b] = run;
      run += c;
    }
    S.ltot[b] = run;
  }
  __syncthreads();
  if (w == 0) lt_tables(S, nb, shift, nbox, false, nbox > LT_GROUPS);
  __syncthreads();
#pragma unroll
  for (int j = 0; j < LT_ITEMS; ++j)
    lpos[j] = (wrank[j] >= 0) ? (int)(S.lstart[dig[j]] + S.whist[w * S.nb + dig[j]]) + wrank[j] : -1;
}

// box lower corners (two-float) for the boxes of level t, staged once per CTA
template <int D>
__device__ __forceinline__ void lt_box_geometry_t(int nbox, int t, const double* alpha, double l, float* geo,
                                                  int nthreads) {
  for (int B = threadIdx.x; B < nbox; B += nthreads) {
    int cell[D];
#pragma unroll
    for (int d = 0; d < D; ++d) cell[d] = 0;
    for (int s = 0; s < t; ++s) {
#pragma unroll
      for (int d = 0; d < D; ++d) cell[d] |= ((B >> (D * s + d)) & 1) << s;
    }
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const double lo = alpha[d] + (double)cell[d] * l;
      const float hi = (float)lo;
      geo[(B * D + d) * 2] = hi;
      geo[(B * D + d) * 2 + 1] = (float)(lo - (double)hi);
    }
  }
}
template <int D>
__device__ __forceinline__ void lt_box_geometry(int nbox, int t, const double* alpha, double l, float* geo) {
  lt_box_geometry_t<D>(nbox, t, alpha, l, geo, LT_THREADS);
}

// 4-lane group reduce-scatter of M (multiple of 4) values: lane g of the group ends with
// the group sums of indices [g*M/4, (g+1)*M/4) in a[0 .. M/4)
template <int M>
__device__ __forceinline__ void group4_reduce_scatter(float (&a)[M]) {
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

// ---------------------------------------------------------------------------------------
// S2M (+ scatter)
// ---------------------------------------------------------------------------------------
template <int D, int P>
__global__ void __launch_bounds__(LT_THREADS, 2) k_local_s2m(LocalS2MArgs a) {
  constexpr int M = IPow<P, D>::value;
  constexpr int MPAD = (M % 4 == 0) ? M : (M + 3) / 4 * 4;
  extern __shared__ __align__(16) unsigned char smraw[];
  const LtShared S = lt_layout(smraw, 1 << a.bits, a.nbox);
  float* sx = reinterpret_cast<float*>(smraw + lt_shared_bytes(1 << a.bits, a.nbox));   // [D][LT_TILE]
  float* sb = sx + D * LT_TILE;                                      // [LT_TILE]
  float* pbuf = sb + LT_TILE;                                        // [LT_GROUPS][MPAD]: one batch of pieces
  float* wacc = pbuf + LT_GROUPS * MPAD;                             // [nbox][M] per-CTA charges
  float* geo = wacc + a.nbox * M;                                    // [nbox][D][2]
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int grp = threadIdx.x / LT_G, gl = threadIdx.x % LT_G;
  const int t = (a.bits - a.shift) / D;
  float af[D];
  double ad[D];
#pragma unroll
  for (int d = 0; d < D; ++d) { af[d] = a.kp.alpha_f[d]; ad[d] = a.kp.alpha[d]; }
  // owned mode (nbox <= 64 groups): group g always takes box g % nbox (sub-slot g / nbox) and
  // adds its per-tile partial to its own slice of pbuf -- no batches, no cross-group sums
  const bool owned = a.nbox <= LT_GROUPS;
  if (a.do_s2m) {
    lt_box_geometry<D>(a.nbox, t, a.alpha, a.l, geo);
    for (int e = threadIdx.x; e < a.nbox * M; e += LT_THREADS) wacc[e] = 0.f;
    if (owned)
      for (int e = threadIdx.x; e < LT_GROUPS * MPAD; e += LT_THREADS) pbuf[e] = 0.f;
  }
  const int tpb = (a.num_tiles + gridDim.x - 1) / gridDim.x;
  const int t_begin = blockIdx.x * tpb, t_end = min(a.num_tiles, t_begin + tpb);
  const float scale = (float)(2.0 / a.l);
  for (int tile = t_begin; tile < t_end; ++tile) {
    const int64_t tile0 = (int64_t)tile * LT_TILE;
    {
      float x[LT_ITEMS][D];
      uint32_t dig[LT_ITEMS];
      int lpos[LT_ITEMS];
      lt_rank<D>(a.X, a.n, tile0, a.kp, af, ad, a.bits, a.shift, a.nbox, S, x, dig, lpos);
      if (a.counts)
        for (int b = threadIdx.x; b < (1 << a.bits); b += LT_THREADS)
          a.counts[(int64_t)b * a.num_tiles + tile] = S.ltot[b];
      if (a.offsets)
        for (int b = threadIdx.x; b < (1 << a.bits); b += LT_THREADS)
          S.goff[b] = a.offsets[(int64_t)b * a.sort_tiles + tile];
      __syncthreads();
      const int64_t seg = tile0 + (int64_t)w * (LT_TILE / LT_WARPS);
#pragma unroll
      for (int j = 0; j < LT_ITEMS; ++j) {
        if (lpos[j] >= 0) {
          const int64_t i = seg + j * 32 + lane;
          const float bv = __ldg(a.b + i);
#pragma unroll
          for (int d = 0; d < D; ++d) sx[d * LT_TILE + lpos[j]] = x[j][d];
          sb[lpos[j]] = bv;
          if (a.lrank) a.lrank[i] = (uint16_t)lpos[j];
          if (a.perm) {
            const uint32_t dst = S.goff[dig[j]] + (uint32_t)lpos[j] - S.lstart[dig[j]];
            a.perm[dst] = (int32_t)i;
            if (a.sigma) a.sigma[i] = (int32_t)dst;
            if (a.keys) a.keys[dst] = (uint64_t)dig[j];
            if (a.xs) {
#pragma unroll
              for (int d = 0; d < D; ++d) a.xs[(int64_t)d * a.n + dst] = x[j][d];
              a.bs[dst] = bv;
            }
          }
        }
      }
    }
    __syncthreads();
    if (a.do_s2m && owned) {
      const int G = LT_GROUPS / a.nbox;
      const int B = grp % a.nbox, sub = grp / a.nbox;
      const int per = 1 << a.shift;
      const int beg = (int)S.lstart[B * per], end = beg + (int)S.bcnt[B];
      float acc[M];
#pragma unroll
      for (int k = 0; k < M; ++k) acc[k] = 0.f;
      if (beg < end) {
        float lh[D], ll[D];
#pragma unroll
        for (int d = 0; d < D; ++d) { lh[d] = geo[(B * D + d) * 2]; ll[d] = geo[(B * D + d) * 2 + 1]; }
        for (int p = beg + sub * LT_G + gl; p < end; p += LT_G * G) {
          float L[D][P];
#pragma unroll
          for (int d = 0; d < D; ++d) chebyshev<P>(local_tau(sx[d * LT_TILE + p], lh[d], ll[d], scale), L[d]);
          s2m_accumulate<D, P>(sb[p], L, acc);
        }
      }
      __syncwarp();
      if constexpr (M % 4 == 0) {
        group4_reduce_scatter<M>(acc);
#pragma unroll
        for (int r = 0; r < M / 4; ++r) pbuf[grp * MPAD + gl * (M / 4) + r] += acc[r];
      } else {
#pragma unroll
        for (int k = 0; k < M; ++k) {
          float v = acc[k];
          v += __shfl_xor_sync(0xffffffffu, v, 2);
          v += __shfl_xor_sync(0xffffffffu, v, 1);
          if (gl == 0) pbuf[grp * MPAD + k] += v;
        }
      }
      __syncthreads();
    } else
if (a.do_s2m) {
      const int np = *S.npieces;
      for (int q0 = 0; q0 < np; q0 += LT_GROUPS) {   // one piece per 4-lane group per batch
        const int q = q0 + grp;
        float acc[M];
#pragma unroll
        for (int k = 0; k < M; ++k) acc[k] = 0.f;
        if (q < np) {
          const int B = S.piece_box[q];
          const int beg = S.piece_beg[q], end = beg + S.piece_len[q];
          float lh[D], ll[D];
#pragma unroll
          for (int d = 0; d < D; ++d) { lh[d] = geo[(B * D + d) * 2]; ll[d] = geo[(B * D + d) * 2 + 1]; }
          for (int p = beg + gl; p < end; p += LT_G) {
            float L[D][P];
#pragma unroll
            for (int d = 0; d < D; ++d) chebyshev<P>(local_tau(sx[d * LT_TILE + p], lh[d], ll[d], scale), L[d]);
            s2m_accumulate<D, P>(sb[p], L, acc);
          }
        }
        __syncwarp();
        if constexpr (M % 4 == 0) {
          group4_reduce_scatter<M>(acc);
          if constexpr ((M / 4) % 4 == 0) {
#pragma unroll
            for (int r = 0; r < M / 4; r += 4)
              *reinterpret_cast<float4*>(pbuf + grp * MPAD + gl * (M / 4) + r) =
                  make_float4(acc[r], acc[r + 1], acc[r + 2], acc[r + 3]);
          } else {
#pragma unroll
            for (int r = 0; r < M / 4; ++r) pbuf[grp * MPAD + gl * (M / 4) + r] = acc[r];
          }
        } else {
#pragma unroll
          for (int k = 0; k < M; ++k) {
            float v = acc[k];
            v += __shfl_xor_sync(0xffffffffu, v, 2);
            v += __shfl_xor_sync(0xffffffffu, v, 1);
            if (gl == 0) pbuf[grp * MPAD + k] = v;
          }
        }
        __syncthreads();
        // fixed-order accumulation of the batch's piece partials into the CTA charges
        const int q1 = min(np, q0 + LT_GROUPS);
        for (int e = threadIdx.x; e < a.nbox * M; e += LT_THREADS) {
          const int B = e / M, k = e - B * M;
          const int lo = max((int)S.pstart[B], q0), hi = min((int)S.pstart[B + 1], q1);
          if (lo < hi) {
            float s = 0.f;
            for (int pq = lo; pq < hi; ++pq) s += pbuf[(pq - q0) * MPAD + k];
            wacc[e] += s;
          }
        }
        __syncthreads();
      }
    }
  }
  if (a.do_s2m) {
    float* out = a.Wpart + (int64_t)blockIdx.x * a.nbox * M;
    if (owned) {  // fixed-order sum of the sub-slots of each box
      __syncthreads();
      const int G = LT_GROUPS / a.nbox;
      for (int e = threadIdx.x; e < a.nbox * M; e += LT_THREADS) {
        const int B = e / M, k = e - B * M;
        float sum = 0.f;
        for (int sub = 0; sub < G; ++sub) sum += pbuf[(sub * a.nbox + B) * MPAD + k];
        out[e] = sum;
      }
    } else {
      for (int e = threadIdx.x; e < a.nbox * M; e += LT_THREADS) out[e] = wacc[e];
    }
  }
}

// Per-box change of basis between Chebyshev moments and nodal values (D mode products):
//   forward (transpose = 0): W_j = sum_k prod_d C[j_d][k_d] M_k     (moments -> nodal charges)
//   adjoint (transpose = 1): U~_k = sum_j prod_d C[j_d][k_d] U_j     (nodal locals -> Chebyshev)
struct ChebMat { double c[16 * 16]; };
__global__ void k_cheb_transform(double* __restrict__ V, int nslots, int D, int P, int m, ChebMat cm, int transpose) {
  extern __shared__ double tb[];
  double* cur = tb;
  double* nxt = tb + m;
  const int slot = blockIdx.x;
  for (int k = threadIdx.x; k < m; k += blockDim.x) cur[k] = V[(int64_t)slot * m + k];
  __syncthreads();
  int stride = 1;
  for (int d = 0; d < D; ++d) {
    for (int k = threadIdx.x; k < m; k += blockDim.x) {
      const int kd = (k / stride) % P;
      const int base = k - kd * stride;
      double s = 0.0;
      for (int j = 0; j < P; ++j) {
        const double c = transpose ? cm.c[j * P + kd] : cm.c[kd * P + j];
        s += c * cur[base + j * stride];
      }
      nxt[k] = s;
    }
    __syncthreads();
    double* t = cur; cur = nxt; nxt = t;
    stride *= P;
  }
  for (int k = threadIdx.x; k < m; k += blockDim.x) V[(int64_t)slot * m + k] = cur[k];
}

void launch_cheb_transform(double* V, int nslots, int D, int P, int transpose, cudaStream_t st) {
  if (nslots <= 0) return;
  // C[j][k]: Lagrange basis of the P Chebyshev points in the Chebyshev basis, C = (Vm^{-1})^T,
  // Vm[i][k] = T_k(s_i); solved once on the host in fp64 (Gauss-Jordan, P <= 16)
  static thread_local int cachedP = -1;
  static thread_local ChebMat cm;
  if (cachedP != P) {
    const double pi = 3.14159265358979323846;
    double A[16][32];
    for (int i = 0; i < P; ++i) {
      const double si = cos((double)i * pi / (double)(P - 1));
      double t0 = 1.0, t1 = si;
      for (int k = 0; k < P; ++k) {
        double tk = (k == 0) ? 1.0 : (k == 1 ? si : 0.0);
        if (k >= 2) { tk = 2.0 * si * t1 - t0; t0 = t1; t1 = tk; }
        A[i][k] = tk;
        A[i][P + k] = (i == k) ? 1.0 : 0.0;
      }
    }
    for (int c = 0; c < P; ++c) {  // Gauss-Jordan with partial pivoting
      int piv = c;
      for (int r = c + 1; r < P; ++r) if (fabs(A[r][c]) > fabs(A[piv][c])) piv = r;
      for (int k = 0; k < 2 * P; ++k) { double t = A[c][k]; A[c][k] = A[piv][k]; A[piv][k] = t; }
      const double inv = 1.0 / A[c][c];
      for (int k = 0; k < 2 * P; ++k) A[c][k] *= inv;
      for (int r = 0; r < P; ++r)
        if (r != c) {
          const double f = A[r][c];
          for (int k = 0; k < 2 * P; ++k) A[r][k] -= f * A[c][k];
        }
    }
    // Vm^{-1} = A[:, P:]; C[j][k] = Vm^{-1}[k][j]
    for (int j = 0; j < P; ++j)
      for (int k = 0; k < P; ++k) cm.c[j * P + k] = A[k][P + j];
    cachedP = P;
  }
  int m = 1;
  for (int d = 0; d < D; ++d) m *= P;
  const int bd = m < 32 ? 32 : (m > 256 ? 256 : (m + 31) / 32 * 32);
  const size_t sm = sizeof(double) * 2 * m;
  if (sm > 48 * 1024) cudaFuncSetAttribute(k_cheb_transform, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  k_cheb_transform<<<nslots, bd, sm, st>>>(V, nslots, D, P, m, cm, transpose);
}

// W[slot][k] = sum_cta Wpart[cta][box(slot)][k] (fixed order, fp64)
__global__ void k_local_reduce(const float* __restrict__ Wpart, int nctas, int nbox, int m,
                               const int32_t* __restrict__ slot_box, int nslots, double* __restrict__ W) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)nslots * m) return;
  const int s = (int)(e / m), k = (int)(e - (int64_t)s * m);
  const int B = slot_box[s];
  double acc = 0.0;
  for (int c = 0; c < nctas; ++c) acc += (double)Wpart[((int64_t)c * nbox + B) * m + k];
  W[e] = acc;
}

// ---------------------------------------------------------------------------------------
// L2T in the original order
// ---------------------------------------------------------------------------------------
template <int D, int P>
__global__ void __launch_bounds__(LT_THREADS, 2) k_local_l2t(LocalL2TArgs a) {
  constexpr int M = IPow<P, D>::value;
  constexpr int MROW = (M % 4 == 0) ? M + 4 : M;  // padded rows: the 8 groups of a warp hit distinct banks
  extern __shared__ __align__(16) unsigned char smraw[];
  const LtShared S = lt_layout(smraw, 1 << a.bits, a.nbox);
  float* sx = reinterpret_cast<float*>(smraw + lt_shared_bytes(1 << a.bits, a.nbox));  // [D][LT_TILE]
  float* sv = sx + D * LT_TILE;                                     // [LT_TILE] by ORIGINAL local index
  float* Us = sv + LT_TILE;                                         // [nbox][MROW]
  float* geo = Us + a.nbox * MROW;                                  // [nbox][D][2]
  uint16_t* sorig = reinterpret_cast<uint16_t*>(geo + 2 * D * a.nbox);  // [LT_TILE] sorted -> original local
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int grp = threadIdx.x / LT_G, gl = threadIdx.x % LT_G;
  const int t = (a.bits - a.shift) / D;
  float af[D];
  double ad[D];
#pragma unroll
  for (int d = 0; d < D; ++d) { af[d] = a.kp.alpha_f[d]; ad[d] = a.kp.alpha[d]; }
  lt_box_geometry<D>(a.nbox, t, a.alpha, a.l, geo);
  for (int e = threadIdx.x; e < a.nbox * M; e += LT_THREADS) {
    const int B = e / M, k = e - B * M;
    const int s = a.box_slot[B];
    Us[B * MROW + k] = s >= 0 ? (float)a.U[(int64_t)s * M + k] : 0.f;
  }
  const int tpb = (a.num_tiles + gridDim.x - 1) / gridDim.x;
  const int t_begin = blockIdx.x * tpb, t_end = min(a.num_tiles, t_begin + tpb);
  const float scale = (float)(2.0 / a.l);
  __syncthreads();
  for (int tile = t_begin; tile < t_end; ++tile) {
    const int64_t tile0 = (int64_t)tile * LT_TILE;
    {
      float x[LT_ITEMS][D];
      uint32_t dig[LT_ITEMS];
      int lpos[LT_ITEMS];
      const int nb = 1 << a.bits;
      if (a.lrank) {  // reuse the first pass's ranks: no digits, no ballots
        const int64_t seg = tile0 + (int64_t)w * (LT_TILE / LT_WARPS);
#pragma unroll
        for (int j = 0; j < LT_ITEMS; ++j) {
          const int64_t i = seg + j * 32 + lane;
#pragma unroll
          for (int d = 0; d < D; ++d) x[j][d] = (i < a.n) ? __ldg(a.X + i * D + d) : 0.f;
          lpos[j] = (i < a.n) ? (int)__ldg(a.lrank + i) : -1;
        }
        if (w == 0) {
          const int64_t len = (int64_t)nb * a.sort_tiles;
          for (int b = lane; b < nb; b += 32) {
            const int64_t idx = (int64_t)b * a.sort_tiles + tile;
            const uint32_t cur = a.offsets[idx];
            const uint32_t nxt = (idx + 1 < len) ? a.offsets[idx + 1] : (uint32_t)a.n;
            S.ltot[b] = nxt - cur;
            S.goff[b] = cur;
          }
          __syncwarp();
          lt_tables(S, nb, a.shift, a.nbox, false, a.nbox > LT_GROUPS);
        }
        __syncthreads();
      } else {
        lt_rank<D>(a.X, a.n, tile0, a.kp, af, ad, a.bits, a.shift, a.nbox, S, x, dig, lpos);
        if (a.perm) {
          for (int b = threadIdx.x; b < nb; b += LT_THREADS)
            S.goff[b] = a.offsets[(int64_t)b * a.sort_tiles + tile];
          __syncthreads();
        }
      }
#pragma unroll
      for (int j = 0; j < LT_ITEMS; ++j)
        if (lpos[j] >= 0) {
#pragma unroll
          for (int d = 0; d < D; ++d) sx[d * LT_TILE + lpos[j]] = x[j][d];
          sorig[lpos[j]] = (uint16_t)(w * (LT_TILE / LT_WARPS) + j * 32 + lane);
        }
    }
    __syncthreads();
    const bool owned = a.nbox <= LT_GROUPS;  // group g takes box g % nbox every tile
    const int np = owned ? (grp < LT_GROUPS ? 1 : 0) : *S.npieces;
    for (int q = grp; q < (owned ? LT_GROUPS : np); q += LT_GROUPS) {
      int B, beg, end, step = LT_G, first;
      if (owned) {
        const int G = LT_GROUPS / a.nbox, sub = grp / a.nbox;
        B = grp % a.nbox;
        beg = (int)S.lstart[B * (1 << a.shift)];
        end = beg + (int)S.bcnt[B];
        step = LT_G * G;
        first = beg + sub * LT_G + gl;
      } else {
        B = S.piece_box[q];
        beg = S.piece_beg[q];
        end = beg + S.piece_len[q];
        first = beg + gl;
      }
      float lh[D], ll[D];
#pragma unroll
      for (int d = 0; d < D; ++d) { lh[d] = geo[(B * D + d) * 2]; ll[d] = geo[(B * D + d) * 2 + 1]; }
      float u[M];
      if constexpr (M % 4 == 0) {
#pragma unroll
        for (int k = 0; k < M; k += 4) {
          const float4 v4 = *reinterpret_cast<const float4*>(Us + B * MROW + k);
          u[k] = v4.x; u[k + 1] = v4.y; u[k + 2] = v4.z; u[k + 3] = v4.w;
        }
      } else {
#pragma unroll
        for (int k = 0; k < M; ++k) u[k] = Us[B * MROW + k];
      }
      for (int p = first; p < end; p += step) {
        float L[D][P];
#pragma unroll
        for (int d = 0; d < D; ++d) chebyshev<P>(local_tau(sx[d * LT_TILE + p], lh[d], ll[d], scale), L[d]);
        const int o = sorig[p];
        sv[o] = l2t_contract<D, P>(L, u);
        if (a.perm) {  // the counting-sort permutation (Sec. 4.1): stable destination of p
          int bin = B;
          if (a.shift) {  // last bin with lstart <= p
            int lo = 0, hi = (1 << a.bits) - 1;
            while (lo < hi) {
              const int mid = (lo + hi + 1) >> 1;
              if ((int)S.lstart[mid] <= p) lo = mid; else hi = mid - 1;
            }
            bin = lo;
          }
          const uint32_t dst = S.goff[bin] + (uint32_t)p - S.lstart[bin];
          a.perm[dst] = (int32_t)(tile0 + o);
          if (a.keys) a.keys[dst] = (uint64_t)bin;
        }
      }
    }
    __syncthreads();
    const int tvalid = (int)min((int64_t)LT_TILE, a.n - tile0);
    for (int o = threadIdx.x; o < tvalid; o += LT_THREADS) {   // coalesced, original order
      const int64_t i = tile0 + o;
      float r = sv[o];
      if (a.vs) r += a.vs[a.sigma[i]];
      if (a.accumulate) r += a.v[i];
      a.v[i] = r;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------------------
#define F3M_LOCAL_CASES(X) \
  X(1, 2) X(1, 3) X(1, 4) X(1, 5) X(1, 6) X(1, 7) X(1, 8) \
  X(2, 2) X(2, 3) X(2, 4) X(2, 5) X(2, 6) X(2, 7) X(2, 8) \
  X(3, 2) X(3, 3) X(3, 4) \
  X(4, 2) X(5, 2) X(6, 2) X(7, 2)

static int mpad_of(int m) { return (m % 4 == 0) ? m : (m + 3) / 4 * 4; }
static size_t s2m_smem(int D, int nb, int nbox, int m) {
  return lt_shared_bytes(nb, nbox) + (size_t)(D + 1) * LT_TILE * 4 + (size_t)LT_GROUPS * mpad_of(m) * 4 +
         (size_t)nbox * m * 4 + (size_t)2 * D * nbox * 4 + 16;
}
static size_t l2t_smem(int D, int nb, int nbox, int m) {
  const int mrow = (m % 4 == 0) ? m + 4 : m;
  return lt_shared_bytes(nb, nbox) + (size_t)(D + 1) * LT_TILE * 4 + (size_t)nbox * mrow * 4 + (size_t)2 * D * nbox * 4 +
         (size_t)LT_TILE * 2 + 16;
}

int local_grid(int num_tiles) {
  int g = 148 * 2;
  if (g > num_tiles) g = num_tiles;
  return g < 1 ? 1 : g;
}

bool local_supported(int D, int P, int nbox) {
  int m = 1;
  for (int d = 0; d < D; ++d) m *= P;
  if (s2m_smem(D, 256, nbox, m) > 227 * 1024 || l2t_smem(D, 256, nbox, m) > 227 * 1024) return false;
#define X(d, p) if (D == d && P == p) return true;
  F3M_LOCAL_CASES(X)
#undef X
  return false;
}

void launch_local_s2m(int D, int P, const LocalS2MArgs& a, int grid, cudaStream_t st) {
  int m = 1;
  for (int d = 0; d < D; ++d) m *= P;
  const size_t sm = s2m_smem(D, 1 << a.bits, a.nbox, m);
#define X(d, p)                                                                                  \
  if (D == d && P == p) {                                                                        \
    cudaFuncSetAttribute(k_local_s2m<d, p>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm); \
    k_local_s2m<d, p><<<grid, LT_THREADS, sm, st>>>(a);                                          \
    return;                                                                                      \
  }
  F3M_LOCAL_CASES(X)
#undef X
}

void launch_local_reduce(const float* Wpart, int nctas, int nbox, int m, const int32_t* slot_box, int nslots,
                         double* W, cudaStream_t st) {
  const int64_t work = (int64_t)nslots * m;
  if (work <= 0) return;
  k_local_reduce<<<(unsigned)((work + 255) / 256), 256, 0, st>>>(Wpart, nctas, nbox, m, slot_box, nslots, W);
}



void launch_local_l2t(int D, int P, const LocalL2TArgs& a, int grid, cudaStream_t st) {
  int m = 1;
  for (int d = 0; d < D; ++d) m *= P;
  const size_t sm = l2t_smem(D, 1 << a.bits, a.nbox, m);
#define X(d, p)                                                                                  \
  if (D == d && P == p) {                                                                        \
    cudaFuncSetAttribute(k_local_l2t<d, p>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm); \
    k_local_l2t<d, p><<<grid, LT_THREADS, sm, st>>>(a);                                          \
    return;                                                                                      \
  }
  F3M_LOCAL_CASES(X)
#undef X
}

}  // namespace f3m
