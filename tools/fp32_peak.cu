// FP32 FFMA throughput microbenchmark (the denominator of the "alu" roofline in bench.py).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp32_peak tools/fp32_peak.cu
//   tools/fp32_peak            -> one JSON line per variant
//
// Each thread runs NCH independent FFMA chains (enough ILP to cover the 4-cycle latency)
// for ITERS iterations; the grid is 148 x BLOCKS_PER_SM persistent blocks.  Two variants:
//   reg3: a = fma(a, b, c) with b, c in registers (three register operands, as in the S2M /
//         L2T inner loops), and
//   mix:  half the chains use a register multiplier, half an immediate one.
// flops = 2 x threads x ITERS x NCH; time = CUDA events around the launch (best of 5).
#include <cuda_runtime.h>
#include <stdio.h>

constexpr int NCH = 16;
constexpr int ITERS = 1 << 14;

template <int MODE>
__global__ void __launch_bounds__(512) k_ffma(float* out, float b, float c) {
  float a[NCH];
#pragma unroll
  for (int i = 0; i < NCH; ++i) a[i] = threadIdx.x * 1e-3f + i;
  float bb[NCH], cc[NCH];
#pragma unroll
  for (int i = 0; i < NCH; ++i) { bb[i] = b + i * 1e-7f; cc[i] = c - i * 1e-7f; }
#pragma unroll 4
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < NCH; ++i) {
      if (MODE == 0) a[i] = fmaf(a[i], bb[i], cc[i]);
      else if (MODE == 3) a[i] = fmaf(a[i], 0.999f, cc[i]);  // immediate multiplier (FFMA imm form)
      else a[i] = (i & 1) ? fmaf(a[i], 0.999f, cc[i]) : fmaf(a[i], bb[i], cc[i]);
    }
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < NCH; ++i) s += a[i];
  if (s == 12345.678f) out[threadIdx.x] = s;  // keep the chains live
}

// packed FFMA2 (sm_100a fma.rn.f32x2): NCH/2 float2 chains, two FMAs per instruction
__global__ void __launch_bounds__(512) k_ffma2(float* out, float b, float c) {
  float2 a[NCH / 2], bb[NCH / 2], cc[NCH / 2];
#pragma unroll
  for (int i = 0; i < NCH / 2; ++i) {
    a[i] = make_float2(threadIdx.x * 1e-3f + i, threadIdx.x * 1e-3f - i);
    bb[i] = make_float2(b + i * 1e-7f, b - i * 1e-7f);
    cc[i] = make_float2(c - i * 1e-7f, c + i * 1e-7f);
  }
#pragma unroll 4
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < NCH / 2; ++i) a[i] = __ffma2_rn(a[i], bb[i], cc[i]);
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < NCH / 2; ++i) s += a[i].x + a[i].y;
  if (s == 12345.678f) out[threadIdx.x] = s;
}

// outer-product form of the S2M inner loop: acc[i][j] += a[i] * c[j] (4 x 16 accumulators; each
// multiplier is reused by 16 consecutive FFMAs, so operands come from the reuse cache)
__global__ void __launch_bounds__(512) k_outer(float* out, float b, float c) {
  float acc[4][16], x[4], y[16];
#pragma unroll
  for (int i = 0; i < 4; ++i) x[i] = b + i * 1e-7f;
#pragma unroll
  for (int j = 0; j < 16; ++j) y[j] = c + j * 1e-7f;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 16; ++j) acc[i][j] = threadIdx.x * 1e-6f;
#pragma unroll 2
  for (int it = 0; it < ITERS / 4; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 16; ++j) acc[i][j] = fmaf(x[i], y[j], acc[i][j]);
    x[it & 3] += 1e-9f;  // keep the multipliers loop-variant (one FADD per 64 FFMA)
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 16; ++j) s += acc[i][j];
  if (s == 12345.678f) out[threadIdx.x] = s;
}

template <int MODE>
static void run(const char* name, int threads, int bps) {
  float* out;
  cudaMalloc(&out, 4096);
  int dev = 0, sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = sms * bps;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  if (MODE == 2) k_outer<<<grid, threads>>>(out, 0.9999f, 1e-4f);  // warm-up
  else if (MODE == 4) k_ffma2<<<grid, threads>>>(out, 0.9999f, 1e-4f);
  else k_ffma<MODE><<<grid, threads>>>(out, 0.9999f, 1e-4f);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    if (MODE == 2) k_outer<<<grid, threads>>>(out, 0.9999f, 1e-4f);
    else if (MODE == 4) k_ffma2<<<grid, threads>>>(out, 0.9999f, 1e-4f);
    else k_ffma<MODE><<<grid, threads>>>(out, 0.9999f, 1e-4f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double flops = MODE == 2 ? 2.0 * grid * threads * (double)(ITERS / 4) * 64
                                 : 2.0 * grid * threads * (double)ITERS * NCH;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("{\"variant\": \"%s\", \"threads\": %d, \"blocks_per_sm\": %d, \"sms\": %d, \"ms\": %.4f, "
         "\"tflops\": %.3f, \"per_sm_per_clk_at_max\": %.2f, \"clock_rate_khz\": %d, \"err\": \"%s\"}\n",
         name, threads, bps, sms, best, flops / best * 1e-9, flops / (best * 1e-3) / sms / (clk * 1e3), clk,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(out);
}

int main() {
  run<0>("reg3", 512, 2);
  run<0>("reg3", 256, 4);
  run<2>("outer4x16", 512, 1);
  run<2>("outer4x16", 256, 2);
  run<1>("mix", 512, 2);
  run<3>("imm", 512, 2);
  run<4>("ffma2", 512, 2);
  run<4>("ffma2", 256, 4);
  return 0;
}
