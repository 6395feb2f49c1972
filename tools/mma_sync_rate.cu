// mma_sync_rate.cu — throughput of the warp-level mma.sync.m16n8k16 (f16 x f16 -> f32) on this
// GPU (the legacy tensor-core path, for small gathered GEMMs where tcgen05's tiles do not fit).
// 8 independent accumulators per warp, grid = SMs x 4 CTAs of 256 threads.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mma_sync_rate tools/mma_sync_rate.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void mma_loop(float *out, int iters, uint32_t seed) {
  uint32_t a[4], b[2];
#pragma unroll
  for (int k = 0; k < 4; ++k) a[k] = seed * (k + 1) + threadIdx.x;
  b[0] = seed ^ threadIdx.x; b[1] = seed + 7 * threadIdx.x;
  float c[8][4];
#pragma unroll
  for (int t = 0; t < 8; ++t)
#pragma unroll
    for (int k = 0; k < 4; ++k) c[t][k] = 0.f;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < 8; ++t)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+f"(c[t][0]), "+f"(c[t][1]), "+f"(c[t][2]), "+f"(c[t][3])
                   : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
  }
  float s = 0.f;
#pragma unroll
  for (int t = 0; t < 8; ++t)
#pragma unroll
    for (int k = 0; k < 4; ++k) s += c[t][k];
  if (s == 1234.5f) out[threadIdx.x] = s;
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  float *out;
  cudaMalloc(&out, 4096);
  const int blocks = p.multiProcessorCount * 4, threads = 256, iters = 4096;
  mma_loop<<<blocks, threads>>>(out, 16, 3u);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(e0);
    mma_loop<<<blocks, threads>>>(out, iters, 3u);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  const double flop = 2.0 * 16 * 8 * 16 * 8.0 * iters * (blocks * threads / 32);
  printf("{\"mma_sync_m16n8k16_f16_f32_tflops\": %.1f, \"err\": \"%s\"}\n", flop / (best * 1e-3) / 1e12,
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
