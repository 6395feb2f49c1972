// minmax_pipes.cu — which pipe runs FMNMX (float min/max) vs VIMNMX (integer) on sm_100a:
// throughput of each alone and of an interleaved mix (if they are on different pipes the
// mix runs ~2x the single-pipe rate).
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void mm_loop(unsigned *out, int iters, unsigned seed) {
  unsigned a[8], b = seed ^ threadIdx.x;
  float fa[8], fb = __uint_as_float((seed >> 9) | 0x3f800000u);
#pragma unroll
  for (int k = 0; k < 8; ++k) { a[k] = seed * (k + 1) + threadIdx.x; fa[k] = __uint_as_float(a[k] >> 9 | 0x3f800000u); }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (MODE == 0 || MODE == 2) { a[k] = min(a[k], b); b = max(b, a[(k + 1) & 7]); }
      if (MODE == 1 || MODE == 2) { fa[k] = fminf(fa[k], fb); fb = fmaxf(fb, fa[(k + 1) & 7]); }
    }
    b ^= i;
    fb = __uint_as_float(__float_as_uint(fb) ^ (i & 1));
  }
  unsigned s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += a[k] + __float_as_uint(fa[k]);
  if (s == 12345u) out[threadIdx.x] = s;
}

template <typename K>
float run(K kern, int blocks, unsigned *out, int iters) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  kern<<<blocks, 256>>>(out, 256, 7u);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    kern<<<blocks, 256>>>(out, iters, 7u);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  return best;
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  unsigned *out;
  cudaMalloc(&out, 4096);
  const int blocks = p.multiProcessorCount * 8, iters = 1 << 14;
  const double ops = (double)blocks * 256 * iters * 16;                   // min/max ops per mode-0/1 run
  const float ti = run(mm_loop<0>, blocks, out, iters), tf = run(mm_loop<1>, blocks, out, iters),
              tm = run(mm_loop<2>, blocks, out, iters);
  printf("{\"vimnmx_per_clk_per_sm\": %.1f, \"fmnmx_per_clk_per_sm\": %.1f, \"mix_ops_per_clk_per_sm\": %.1f}\n",
         ops / (ti * 1e-3) / (p.multiProcessorCount * 1.965e9), ops / (tf * 1e-3) / (p.multiProcessorCount * 1.965e9),
         2 * ops / (tm * 1e-3) / (p.multiProcessorCount * 1.965e9));
  return 0;
}
