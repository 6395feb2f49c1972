// ffma_peak.cu — FP32 FMA-pipe throughput on this GPU (the roofline denominator of the
// ALU-bound kernels).  8 independent register-operand FFMA chains per thread,
// grid = SMs x 8 CTAs of 256 threads.  Prints lane-FFMA/s and the implied FLOP/s.
#include <cstdio>
#include <cuda_runtime.h>

template <int CH>
__global__ void ffma_loop(float *out, int iters, float a, float b) {
  float x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = threadIdx.x * 1e-3f + c;
  float y = a, z = b;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = fmaf(x[c], y, z);      // 3-register FFMA
    y = __int_as_float(__float_as_int(y) ^ (i & 1));           // keep y/z live registers
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c];
  if (s == 1234.5f) out[threadIdx.x] = s;
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  float *out;
  cudaMalloc(&out, 4096);
  const int blocks = p.multiProcessorCount * 8, threads = 256, iters = 1 << 16;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  ffma_loop<8><<<blocks, threads>>>(out, 1024, 0.999f, 1e-4f);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    ffma_loop<8><<<blocks, threads>>>(out, iters, 0.999f, 1e-4f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double ffma = (double)blocks * threads * iters * 8;
  const double rate = ffma / (best * 1e-3);
  printf("{\"sms\": %d, \"ffma_lane_per_s\": %.4e, \"tflops\": %.2f, \"ms\": %.3f, "
         "\"lanes_per_clk_per_sm_at_max_clock\": %.1f, \"max_clock_mhz\": %.0f}\n",
         p.multiProcessorCount, rate, 2 * rate / 1e12, best,
         rate / (p.multiProcessorCount * clk * 1e3), clk / 1e3);
  return 0;
}
