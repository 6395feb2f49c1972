// ffma2_peak.cu — packed fp32x2 FMA (FFMA2, sm_100a) vs scalar FFMA throughput, and a mixed
// stream (FFMA2 interleaved with integer ALU work) to see whether FFMA2 frees issue slots.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long f2(unsigned long long a, unsigned long long b, unsigned long long c) {
  unsigned long long d;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

template <int CH, bool ALU>
__global__ void ffma2_loop(float *out, int iters, float a, float b) {
  unsigned long long x[CH];
  unsigned cnt[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    float2 v = make_float2(threadIdx.x * 1e-3f + c, c * 0.5f);
    x[c] = *reinterpret_cast<unsigned long long *>(&v);
    cnt[c] = 0;
  }
  float2 yv = make_float2(a, a), zv = make_float2(b, b);
  unsigned long long y = *reinterpret_cast<unsigned long long *>(&yv), z = *reinterpret_cast<unsigned long long *>(&zv);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      x[c] = f2(x[c], y, z);
      if (ALU) cnt[c] += ((unsigned)x[c] & ~(unsigned)(x[c] >> 32)) >> 31;
    }
    y ^= (unsigned long long)(i & 1);
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += __int_as_float((int)x[c]) + cnt[c];
  if (s == 1234.5f) out[threadIdx.x] = s;
}

template <int CH, bool ALU>
__global__ void ffma_loop(float *out, int iters, float a, float b) {
  float x[CH];
  unsigned cnt[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) { x[c] = threadIdx.x * 1e-3f + c; cnt[c] = 0; }
  float y = a, z = b;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      x[c] = fmaf(x[c], y, z);
      if (ALU) cnt[c] += (__float_as_uint(x[c]) & ~__float_as_uint(x[c ^ 1])) >> 31;
    }
    y = __int_as_float(__float_as_int(y) ^ (i & 1));
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c] + cnt[c];
  if (s == 1234.5f) out[threadIdx.x] = s;
}

template <typename K>
float run(K kern, int blocks, int threads, float *out, int iters) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  kern<<<blocks, threads>>>(out, 1024, 0.999f, 1e-4f);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    kern<<<blocks, threads>>>(out, iters, 0.999f, 1e-4f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  float *out;
  cudaMalloc(&out, 4096);
  const int blocks = p.multiProcessorCount * 8, threads = 256, iters = 1 << 15;
  const double lanes = (double)blocks * threads * iters * 8;
  const float t1 = run(ffma_loop<8, false>, blocks, threads, out, iters);
  const float t2 = run(ffma2_loop<8, false>, blocks, threads, out, iters);
  const float t3 = run(ffma_loop<8, true>, blocks, threads, out, iters);
  const float t4 = run(ffma2_loop<8, true>, blocks, threads, out, iters);
  printf("{\"ffma_tflops\": %.2f, \"ffma2_tflops\": %.2f, \"ffma+alu_tflops\": %.2f, \"ffma2+alu_tflops\": %.2f}\n",
         2 * lanes / (t1 * 1e9), 4 * lanes / (t2 * 1e9), 2 * lanes / (t3 * 1e9), 4 * lanes / (t4 * 1e9));
  return 0;
}
