// umma_rate.cu — tcgen05.mma kind::f16 throughput on this GPU for the matching kernel's shapes:
// M = 128, K = 16 per instruction, N in {64, 128, 256}, A from shared memory (SS) or from TMEM
// (TS), 1 or 2 CTAs per SM.  One thread per CTA issues `iters` x 8 MMAs (K = 128) into one
// accumulator, commits, waits; cycles per MMA per SM = elapsed SM cycles / (MMAs per SM).
// Operand values are zero (only the rate is measured).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/umma_rate tools/umma_rate.cu -lcuda
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_sw128(uint32_t addr) {
  return ((uint64_t)(addr & 0x3FFFF) >> 4) | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
}

template <int N, bool TS>
__global__ void __launch_bounds__(128, 1) umma_loop(long long *out, int iters) {
  extern __shared__ uint8_t raw[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  uint8_t *base = raw + ((1024u - (su32(raw) & 1023u)) & 1023u);
  uint8_t *sA = base, *sB = base + 32768;
  for (int i = threadIdx.x; i < (32768 + N * 256) / 16; i += blockDim.x)
    reinterpret_cast<uint4 *>(base)[i] = make_uint4(0, 0, 0, 0);
  constexpr int cols = N + (TS ? 64 : 0) <= 128 ? 128 : (N + (TS ? 64 : 0) <= 256 ? 256 : 512);
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tbase)), "r"(cols) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tbase;
  const uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  long long t0 = 0, t1 = 0;
  if (threadIdx.x == 0) {
    t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int kb = k >> 2, ks = k & 3;
        const uint64_t bd = desc_sw128(su32(sB + kb * (N * 128) + ks * 32));
        const uint32_t acc = (it | k) ? 1u : 0u;
        if (TS) {
          // A operand in TMEM columns N .. N + 63 (128 lanes x 128 fp16 = 64 columns)
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem),
                       "r"(tmem + N + k * 8), "l"(bd), "r"(idesc), "r"(acc)
                       : "memory");
        } else {
          const uint64_t ad = desc_sw128(su32(sA + kb * 16384 + ks * 32));
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem), "l"(ad),
                       "l"(bd), "r"(idesc), "r"(acc)
                       : "memory");
        }
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(ok) : "r"(su32(&bar)) : "memory");
    t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(cols) : "memory");
  }
}

template <int N, bool TS>
void run(int sms, int per_sm) {
  const size_t smem = 1024 + 32768 + N * 256;
  auto k = umma_loop<N, TS>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  long long *d;
  cudaMalloc(&d, sizeof(long long) * sms * per_sm);
  const int iters = 2000;
  k<<<sms * per_sm, 128, smem>>>(d, 10);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<<<sms * per_sm, 128, smem>>>(d, iters);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  long long h[1024];
  cudaMemcpy(h, d, sizeof(long long) * sms * per_sm, cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int i = 0; i < sms * per_sm; ++i) mx = h[i] > mx ? h[i] : mx;
  const double mmas_per_sm = (double)iters * 8 * per_sm;
  const double flop = 2.0 * 128 * N * 16 * iters * 8 * sms * per_sm;
  printf("{\"N\": %d, \"A\": \"%s\", \"ctas_per_sm\": %d, \"smem_kb\": %zu, \"cycles_per_mma_per_sm\": %.1f, "
         "\"floor\": %.1f, \"tflops\": %.1f, \"err\": \"%s\"}\n",
         N, TS ? "tmem" : "smem", per_sm, smem / 1024, mx / mmas_per_sm, 128.0 * N / 256, flop / (ms * 1e-3) / 1e12,
         cudaGetErrorString(err));
  cudaFree(d);
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  const int sms = p.multiProcessorCount;
  run<64, false>(sms, 1);
  run<64, false>(sms, 2);
  run<128, false>(sms, 1);
  run<128, false>(sms, 2);
  run<256, false>(sms, 1);
  run<64, true>(sms, 1);
  run<64, true>(sms, 2);
  run<128, true>(sms, 1);
  run<128, true>(sms, 2);
  run<256, true>(sms, 1);
  return 0;
}
