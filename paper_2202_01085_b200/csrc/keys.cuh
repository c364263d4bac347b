// Bit-exact integer cell of one coordinate (Sec. 4.2 box index; reading R12):
//   c = min(floor(RN64(RN64(x - alpha) / E) * 2^T), 2^T - 1)
// fp32 fast path with an error margin, exact fp64 division when the fast path is ambiguous
// (DESIGN.md "Bit-exact binning").  Shared by the sort kernels and the original-order L2T.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "f3m_internal.h"

namespace f3m {

__device__ __forceinline__ uint64_t cell_of(float x, int d, const KeyParams& kp) {
  const float dd = __fsub_rn(x, kp.alpha_f[d]);
  const float q = __fmul_rn(dd, kp.scale_f);
  const float fl = floorf(q);
  const float fr = __fsub_rn(q, fl);
  if (fr > kp.margin && fr < 1.0f - kp.margin) return (uint64_t)fl;
  const double u = __ddiv_rn(__dsub_rn((double)x, kp.alpha[d]), kp.E);
  const double f = floor(__dmul_rn(u, kp.twoT));
  uint64_t c = (uint64_t)f;
  const uint64_t cmax = (uint64_t)kp.twoT - 1ull;
  return c > cmax ? cmax : c;
}

}  // namespace f3m
