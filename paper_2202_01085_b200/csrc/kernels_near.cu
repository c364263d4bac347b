// Near / small field and exact direct KMVM for sm_100a: KeOps-style tiled map-reduce
// over box-pair lists (Sec. 3 Eq. (1); small field
// Sec. 4.2; final near flush, Alg. 1).
//
// One CTA = up to NEAR_TILE targets of one target box (one per thread, coordinates in
// registers).  Source boxes of its CSR list stream through shared memory as float4
// records (x, y, z, b) -- one broadcast LDS.128 per source per warp -- and each thread
// sums exp2(-d2 * log2(e)/(2 gamma^2)) b on MUFU.EX2.  Tile partial sums are fp32 and are
// accumulated across tiles in fp64 (bounded rounding).
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "f3m_internal.h"

namespace f3m {

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// records per source: RW = 4 floats (D <= 3) or 8 floats (D <= 7); last slot = b
template <int D>
struct Rec { static constexpr int W = (D + 1 <= 4) ? 4 : 8; };

template <int D>
__global__ void __launch_bounds__(NEAR_TILE) k_near(const float* __restrict__ xs_t, int64_t nt,
                                                    const float* __restrict__ xs_s, const float* __restrict__ bs,
                                                    int64_t ns, const NearJob* __restrict__ jobs,
                                                    const int32_t* __restrict__ list_ptr,
                                                    const int64_t* __restrict__ src_start,
                                                    const int64_t* __restrict__ src_count, float c,
                                                    float* __restrict__ vs) {
  constexpr int RW = Rec<D>::W;
  __shared__ __align__(16) float sy[NEAR_TILE * RW];
  const NearJob job = jobs[blockIdx.x];
  const int tid = threadIdx.x;
  const bool active = tid < job.tlen;
  const int64_t i = job.tstart + tid;
  float x[D];
#pragma unroll
  for (int d = 0; d < D; ++d) x[d] = active ? __ldg(xs_t + (int64_t)d * nt + i) : 0.f;
  double acc = 0.0;
  for (int32_t L = list_ptr[job.list]; L < list_ptr[job.list + 1]; ++L) {
    const int64_t s0 = src_start[L];
    const int64_t sc = src_count[L];
    for (int64_t base = 0; base < sc; base += NEAR_TILE) {
      const int cnt = (int)min((int64_t)NEAR_TILE, sc - base);
      if (tid < cnt) {
        const int64_t j = s0 + base + tid;
        float r[RW];
#pragma unroll
        for (int d = 0; d < RW; ++d) r[d] = 0.f;
#pragma unroll
        for (int d = 0; d < D; ++d) r[d] = __ldg(xs_s + (int64_t)d * ns + j);
        r[RW - 1] = __ldg(bs + j);
#pragma unroll
        for (int q = 0; q < RW; q += 4)
          *reinterpret_cast<float4*>(sy + tid * RW + q) = make_float4(r[q], r[q + 1], r[q + 2], r[q + 3]);
      }
      __syncthreads();
      float part = 0.f;
#pragma unroll 4
      for (int j = 0; j < cnt; ++j) {
        float r[RW];
#pragma unroll
        for (int q = 0; q < RW; q += 4) {
          const float4 v = *reinterpret_cast<const float4*>(sy + j * RW + q);
          r[q] = v.x; r[q + 1] = v.y; r[q + 2] = v.z; r[q + 3] = v.w;
        }
        float d2 = 0.f;
#pragma unroll
        for (int d = 0; d < D; ++d) {
          const float df = x[d] - r[d];
          d2 = fmaf(df, df, d2);
        }
        part = fmaf(ex2_approx(-d2 * c), r[RW - 1], part);
      }
      acc += (double)part;
      __syncthreads();
    }
  }
  if (active) vs[i + job.out_off] += (float)acc;
}

// exact reference: fp64 evaluation (exp in double) and fp64 accumulation
template <int D>
__global__ void __launch_bounds__(NEAR_TILE) k_direct_f64(const float* __restrict__ xs_t, int64_t nt,
                                                          const float* __restrict__ xs_s,
                                                          const float* __restrict__ bs, int64_t ns,
                                                          double inv2g2, double* __restrict__ partial) {
  __shared__ double sy[NEAR_TILE][D + 1];
  const int tid = threadIdx.x;
  const int64_t i = (int64_t)blockIdx.x * NEAR_TILE + tid;
  const bool active = i < nt;
  double x[D];
#pragma unroll
  for (int d = 0; d < D; ++d) x[d] = active ? (double)xs_t[(int64_t)d * nt + i] : 0.0;
  double acc = 0.0;
  const int64_t per = (ns + gridDim.y - 1) / gridDim.y;
  const int64_t s0 = (int64_t)blockIdx.y * per;
  const int64_t s1 = min(ns, s0 + per);
  for (int64_t base = s0; base < s1; base += NEAR_TILE) {
    const int cnt = (int)min((int64_t)NEAR_TILE, s1 - base);
    if (tid < cnt) {
#pragma unroll
      for (int d = 0; d < D; ++d) sy[tid][d] = (double)xs_s[(int64_t)d * ns + base + tid];
      sy[tid][D] = (double)bs[base + tid];
    }
    __syncthreads();
    for (int j = 0; j < cnt; ++j) {
      double d2 = 0.0;
#pragma unroll
      for (int d = 0; d < D; ++d) {
        const double df = x[d] - sy[j][d];
        d2 += df * df;
      }
      acc += exp(-d2 * inv2g2) * sy[j][D];
    }
    __syncthreads();
  }
  if (active) partial[(int64_t)blockIdx.y * nt + i] = acc;
}

template <typename T>
__global__ void k_reduce_splits(const T* __restrict__ partial, int splits, int64_t nt, T* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nt; i += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int k = 0; k < splits; ++k) s += (double)partial[(int64_t)k * nt + i];
    out[i] = (T)s;
  }
}

void launch_near(int D, const float* xs_t, int64_t nt, const float* xs_s, const float* bs, int64_t ns,
                 const NearJob* jobs, int64_t njobs, const int32_t* list_ptr, const int64_t* src_start,
                 const int64_t* src_count, double gamma, float* vs, cudaStream_t st) {
  if (njobs <= 0) return;
  const float c = (float)(1.4426950408889634 / (2.0 * gamma * gamma));
  switch (D) {
#define CASE(d) case d: k_near<d><<<(unsigned)njobs, NEAR_TILE, 0, st>>>(xs_t, nt, xs_s, bs, ns, jobs, list_ptr, src_start, src_count, c, vs); break;
    CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7)
#undef CASE
    default: break;
  }
}

void launch_direct_f64(int D, const float* xs_t, int64_t nt, const float* xs_s, const float* bs, int64_t ns,
                       double gamma, int splits, double* partial, cudaStream_t st) {
  if (nt <= 0) return;
  const dim3 g((unsigned)((nt + NEAR_TILE - 1) / NEAR_TILE), (unsigned)splits);
  const double inv2g2 = 1.0 / (2.0 * gamma * gamma);
  switch (D) {
#define CASE(d) case d: k_direct_f64<d><<<g, NEAR_TILE, 0, st>>>(xs_t, nt, xs_s, bs, ns, inv2g2, partial); break;
    CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7)
#undef CASE
    default: break;
  }
}

void launch_reduce_splits_f64(const double* partial, int splits, int64_t nt, double* out, cudaStream_t st) {
  const unsigned g = (unsigned)std::min<int64_t>((nt + 255) / 256, 148 * 8);
  k_reduce_splits<double><<<g > 0 ? g : 1, 256, 0, st>>>(partial, splits, nt, out);
}
void launch_reduce_splits_f32(const float* partial, int splits, int64_t nt, float* out, cudaStream_t st) {
  const unsigned g = (unsigned)std::min<int64_t>((nt + 255) / 256, 148 * 8);
  k_reduce_splits<float><<<g > 0 ? g : 1, 256, 0, st>>>(partial, splits, nt, out);
}

}  // namespace f3m
