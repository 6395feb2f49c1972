// bt_match.cu — mutual nearest-neighbour descriptor matching (P:4 "feature matching",
// P:25 "n keypoints ... feature descriptor D_i in R^128"), readings R1-R4 of DESIGN.md:
// squared Euclidean distance, ties -> lowest index, mutual NN, optional Lowe ratio,
// output ascending in i.  The result is the EXACT brute-force one; the tensor cores only
// prune candidates under a proven error bound.
//
//  k_desc_prep   per frame and keypoint: |a| (fp32) and the frame's max |a| = M_f.
//  k_desc_half   a / M_f in fp16 ([F][n_pad][128], zero padded; |a / M_f| <= 1).
//  k_match_ws    persistent, warp-specialized (2 CTAs per SM) over the items (128-row tile,
//                pair, direction a->b / b->a): a producer warp issues the TMA (128B-swizzled
//                boxes of 64 x 128 fp16) of the A tile once per item and of B in 128-column
//                chunks (double buffered), stages each chunk's column constants and issues
//                tcgen05.mma.cta_group::1.kind::f16 (M = 128, N = 128, K = 8 x 16) into one of two
//                128-column fp32 TMEM accumulators, S'' = (A / M_a) . (B / M_b)^T; 8 epilogue
//                warps (two warpgroups, half the columns each) read TMEM with tcgen05.ld, rank
//                d' = |b|^2 - 2 M_a M_b S'' (= d_hat - |a|^2; one FFMA with the per-column
//                |b|^2 + 2.01 M_a M_b) and keep the three smallest as packed (order-preserving
//                value | index) keys, merging two keys per step with 3-input mins (columns past
//                n_b rank at +inf: no per-element bound check).  Both directions recompute the
//                tile on the tensor cores rather than reducing columns across lanes.  The
//                epilogue certifies each row (below) and decides it, queues it for top-2
//                rescoring, or lists it in the item's full-scan list.
//  certificate   With the bound
//                eps = 2.2e-3 |a| M_b + 1e-6 (|a|^2 + M_b^2) + 3e-6 M_a M_b (+ key truncation) —
//                fp16 elements of a / M_a have relative error 2^-11, so |S_hat - S''| <= (2^-10 +
//                128 * 2^-23) |a||b| / (M_a M_b) (fp32 accumulation, any rounding mode) and
//                |d_hat - d| <= 2.0e-3 |a||b| + subnormal and fp32 evaluation terms — a reference
//                ranked at position >= L cannot be the nearest neighbour when d'_(L) - d'_(1) >
//                2 eps: L = 2 certifies the best candidate; L = 3 leaves the top two, rescored
//                exactly in fp32; otherwise (ties, ratio test, BT_FORCE_FALLBACK) the row is
//                rescanned exactly over all references, batched per row tile by k_fullscan (the
//                same summation tree as the top-2 rescoring, bit for bit).
//  k_rescore     blockIdx.y 0: warps over the top-2 queue (two exact distances per row);
//                1: CTAs over the full-scan queue (one row per CTA, references split over 8
//                warps) — used when n_max < 1024.
//  k_fullscan    n_max >= 1024: per (pair, direction) its undecided rows, compacted per row
//                tile by k_match_ws, in groups of 32 against all references (chunks of 64)
//                staged in shared memory, 8 exact distances per thread (a reference is read
//                once per 32 rows instead of once per row); few rows: one row per CTA.
//  k_mutual      keep (i, NN_ab(i)) iff NN_ba(NN_ab(i)) == i (+ ratio flag), compact ascending.
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <math_constants.h>

#include "bt_internal.cuh"
#include "bt_tc.cuh"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>


namespace bt {
namespace {

constexpr int kWarpsPerBlock = 8;
constexpr unsigned kNone = 0xFFFFFFFFu;

// small PTX wrappers (mbarrier, TMA, UMMA descriptors, tcgen05): bt_tc.cuh

__device__ __forceinline__ float key_value(unsigned k) { return __uint_as_float(k); }

// ---------------------------------------------------------------- descriptor prep
constexpr int kPrepPerWarp = 4;                // keypoints per warp (loads issued together)

__global__ void __launch_bounds__(kWarpsPerBlock * 32)
k_desc_prep(KpView kp, MatchScratch S, int n_pad) {
  pdl_wait();
  __shared__ unsigned wmax[kWarpsPerBlock];
  const int f = blockIdx.y;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int i0 = (blockIdx.x * kWarpsPerBlock + warp) * kPrepPerWarp;
  const int n = min(kp.n_kp[f], kp.n_max);
  float4 a[kPrepPerWarp];
#pragma unroll
  for (int q = 0; q < kPrepPerWarp; ++q) {
    const int i = i0 + q;
    a[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (i < n) a[q] = __ldg(reinterpret_cast<const float4 *>(kp.desc + ((size_t)f * kp.n_max + i) * kDim) + lane);
  }
  unsigned mx = 0u;
#pragma unroll
  for (int q = 0; q < kPrepPerWarp; ++q) {
    const int i = i0 + q;
    float s = __fmul_rn(a[q].x, a[q].x);
    s = __fmaf_rn(a[q].y, a[q].y, s);
    s = __fmaf_rn(a[q].z, a[q].z, s);
    s = __fmaf_rn(a[q].w, a[q].w, s);
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    const float nrm = sqrtf(s);
    const float inv = nrm > 0.f ? 1.0f / nrm : 0.f;
    (void)inv;
    if (i < n_pad && lane == 0) S.norm[(size_t)f * n_pad + i] = nrm;
    if (i < n) mx = max(mx, __float_as_uint(nrm));                 // nrm >= 0: bits are monotone
  }
  if (lane == 0) wmax[warp] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned m = 0u;
#pragma unroll
    for (int w = 0; w < kWarpsPerBlock; ++w) m = max(m, wmax[w]);
    if (m) atomicMax(S.maxnorm + f, m);
  }
}

// the frame's scale P_f = max_i |a_i| (1 for an empty / all-zero frame)
__device__ __forceinline__ float frame_scale(unsigned maxbits) {
  const float m = __uint_as_float(maxbits);
  return m > 0.f ? m : 1.f;
}

// fp16 descriptors scaled by the frame's max norm: a / P_f (|a / P_f| <= 1; the fp32 scaling
// adds 2^-24 to fp16's 2^-11), zero rows past n (the TMA source of k_match_ws)
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
k_desc_half(KpView kp, MatchScratch S, int n_pad) {
  pdl_wait();
  // the matching kernel may launch now: it allocates TMEM and sets up its barriers before its
  // own griddepcontrol.wait (which still waits for this grid to complete)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int f = blockIdx.y;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int i0 = (blockIdx.x * kWarpsPerBlock + warp) * kPrepPerWarp;
  const int n = min(kp.n_kp[f], kp.n_max);
  const float inv = 1.f / frame_scale(S.maxnorm[f]);
  float4 a[kPrepPerWarp];
#pragma unroll
  for (int q = 0; q < kPrepPerWarp; ++q) {
    const int i = i0 + q;
    a[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (i < n) a[q] = __ldg(reinterpret_cast<const float4 *>(kp.desc + ((size_t)f * kp.n_max + i) * kDim) + lane);
  }
#pragma unroll
  for (int q = 0; q < kPrepPerWarp; ++q) {
    const int i = i0 + q;
    if (i < n_pad) {
      const float x0 = a[q].x * inv, x1 = a[q].y * inv, x2 = a[q].z * inv, x3 = a[q].w * inv;
      __half2 h01 = __floats2half2_rn(x0, x1), h23 = __floats2half2_rn(x2, x3);
      uint2 packed;
      packed.x = *reinterpret_cast<uint32_t *>(&h01);
      packed.y = *reinterpret_cast<uint32_t *>(&h23);
      reinterpret_cast<uint2 *>(S.desc16 + ((size_t)f * n_pad + i) * kDim)[lane] = packed;
      if (S.desc16lo) {                                            // the remainders (exact in fp32)
        const float2 f01 = __half22float2(h01), f23 = __half22float2(h23);
        __half2 l01 = __floats2half2_rn(x0 - f01.x, x1 - f01.y), l23 = __floats2half2_rn(x2 - f23.x, x3 - f23.y);
        packed.x = *reinterpret_cast<uint32_t *>(&l01);
        packed.y = *reinterpret_cast<uint32_t *>(&l23);
        reinterpret_cast<uint2 *>(S.desc16lo + ((size_t)f * n_pad + i) * kDim)[lane] = packed;
      }
    }
  }
}

// ---------------------------------------------------------------- tcgen05 candidate search
struct TcArgs {
  KpView kp;
  const int32_t *pairs;
  MatchScratch S;
  int n_pad, ibits, P, force_fallback;
  float ratio2;
  int fs_batched;                              // undecided rows -> per-tile lists (k_fullscan), else queue 1
  unsigned kmul;                               // 2^kshift (IMAD keys): a runtime operand keeps it an IMAD
  int kshift;                                  // IMAD keys: index bits, max(ibits, 9)
  float kwin;                                  // IMAD keys: value window width 2^-(kshift - 9)
  unsigned kpad;                               // IMAD keys: largest float below 1 + kwin (padded columns)
};

constexpr int kN = 128;                       // B columns per MMA chunk (N); B and TMEM double-buffered

// certificate of a row's packed top-3 keys: 1 = the best is the nearest neighbour, 2 = it is
// one of the top two, 0 = undecided.  A reference ranked >= L cannot be the nearest
// neighbour when d'_(L) - d'_(1) > 2 eps + (truncated key bits).
__device__ __forceinline__ int certify(unsigned k1, unsigned k2, unsigned k3, float qn, float mr, float pp, int ibits) {
  const unsigned imask = (1u << ibits) - 1u;
  if (k1 == kNone) return 0;
  if (k2 == kNone) return 1;
  // |d_hat - d| <= 2.2e-3 |a||b| (fp16 rounding of a / P_a and b / P_b, fp32 accumulation)
  //   + 1e-6 (|a|^2 + |b|^2) + 3e-6 P_a P_b (fp16 subnormals, the fp32 key evaluation around the
  //   offset 2.01 P_a P_b)
  const float eps2 = 2.f * (2.2e-3f * qn * mr + 1e-6f * (qn * qn + mr * mr) + 3e-6f * pp);
  const float v1 = key_value(k1 & ~imask);
  const float v2 = key_value(k2 & ~imask);
  // truncated key bits + the rounding of the offset sum: a few ulps of the values compared
  if ((v2 - v1) > eps2 + ldexpf(fabsf(v1) + fabsf(v2), ibits - 21) + 1e-30f) return 1;
  if (k3 == kNone) return 2;
  const float v3 = key_value(k3 & ~imask);
  if ((v3 - v1) > eps2 + ldexpf(fabsf(v1) + fabsf(v3), ibits - 21) + 1e-30f) return 2;
  return 0;
}

// IMAD keys (s = max(index bits, 9) <= 16): the ranked value is mapped into the window
// [1, 1 + w), w = 2^-(s - 9) — v = 1 + c d'' with c = w / (M_b^2 + 4.02 M_a M_b), still ONE FFMA
// per element (column constant 1 + c(|b|^2 + 2.01 M_a M_b), scale -2 M_a M_b c) — so its float
// bits are 0x3F8xxxxx with a fixed exponent and the top s - 9 mantissa bits zero, and
// bits * 2^s + j (mod 2^32; exponent and zero bits shift out) is the remaining 32 - s mantissa
// bits followed by the s-bit column index: the key is ONE IMAD on the FMA pipe instead of a
// LOP3 on the ALU pipe (the epilogue is ALU-bound: min / max of the top-3), and no value bit
// is truncated (the value's resolution is 2^-23 / c = (M_b^2 + 4.02 M_a M_b) 2^(s - 32)).
// d'' in [0.008 M_a M_b, M_b^2 + 4.012 M_a M_b] (S'' <= 1 + 1e-3) keeps v strictly inside
// [1, 1 + w (1 - 1.6e-3)); a padded column's constant is the largest float below 1 + w (key
// 0xFFFFFFFF << s | j).  Certificate in key units u = 2^-23 / c: each key's value is within
// 2.5 u of 1 + c d'' (the FFMA, the constant's and the scale's fp32 rounding; all values lie in
// [1, 2) where the ulp is 2^-23), so 8 u covers a difference of two.
__device__ __forceinline__ int certify_imad(unsigned k1, unsigned k2, unsigned k3, float qn, float mr, float pp,
                                            float ma, float mb, int s) {
  if (k1 == kNone) return 0;
  if (k2 == kNone) return 1;
  const float u = ldexpf(mb * mb + 4.02f * ma * mb, s - 32);
  const float eps2 = 2.f * (2.2e-3f * qn * mr + 1e-6f * (qn * qn + mr * mr) + 3e-6f * pp) + 8.f * u;
  const float d21 = (float)((k2 >> s) - (k1 >> s)) * u;
  if (d21 > eps2) return 1;
  if (k3 == kNone) return 2;
  const float d31 = (float)((k3 >> s) - (k1 >> s)) * u;
  if (d31 > eps2) return 2;
  return 0;
}

// ---------------------------------------------------------------- persistent, warp-specialized
// Same items, arithmetic and outputs as k_match_tc (bit for bit), restructured so no CTA barrier
// sits in the chunk loop.  Persistent CTAs (2 per SM) walk the items blockIdx.x, + gridDim.x, ...;
// the chunks of successive items form one stream g = 0, 1, 2, ... per CTA.
//   producer warp (warp 8): lane 0 issues the TMA of A (once per item, after the previous item's
//     last MMA has read the old one) and of B into buffer g & 1 (after MMA g - 2 consumed it), the
//     32 lanes stage chunk g's column constants once the epilogue released buffer g & 1, then
//     lane 0 issues the 8 tcgen05.mma of chunk g into TMEM buffer g & 1 and commits to mma[g & 1].
//   epilogue warps 0-7: wait mma[g & 1] and the constants, tcgen05.ld their TMEM lanes, rank,
//     release the buffer (one arrive per warp on free[g & 1]); at an item's end the two
//     warpgroups merge through shared memory (named barrier 1, epilogue warps only), certify
//     and decide or queue each row exactly as k_match_tc.
// mbarrier phases: buffer b's k-th use has parity k & 1 (k = g >> 1); no barrier can run two
// phases ahead of its waiter (each is gated by the other side), so parity waits are exact.
constexpr int kWsEpiWarps = 8;
constexpr int kWsThreads = (kWsEpiWarps + 1) * 32;
constexpr size_t kWsSmem = 1024 /*align*/ + 32768 /*A*/ + 2 * 32768 /*B x2*/ + 2 * kN * 8 /*consts x2*/;


struct TcItem {
  int fa, fb, na, nb, nchunks, rt, p, dir;
  bool skip;
};
// item it = (dir * P + p) * rtc + rt  (= the full-scan list index of k_match_tc)
__device__ __forceinline__ TcItem tc_item(const TcArgs &A, int it) {
  TcItem I;
  const int rtc = A.n_pad / 128;
  I.rt = it % rtc;
  const int q = it / rtc;
  I.p = q % A.P;
  I.dir = q / A.P;
  I.fa = A.pairs[2 * I.p + I.dir];
  I.fb = A.pairs[2 * I.p + 1 - I.dir];
  I.na = min(A.kp.n_kp[I.fa], A.kp.n_max);
  I.nb = min(A.kp.n_kp[I.fb], A.kp.n_max);
  I.nchunks = (I.nb + kN - 1) / kN;
  I.skip = I.rt * 128 >= I.na || I.nb == 0;
  return I;
}

// kTop2 (the batched path, n_max >= 1024, where undecided rows go to the level-2 pass): four
// interleaved top-2 sets per thread instead of two top-3 sets — 2.5 instead of 4 ALU min / max
// per element.  The global top-2 is exact (each of its keys is in its set's top-2); for the
// third-best value only a lower bound is known: LB = min(3rd of the union of the sets' top-2s,
// min over sets of their 2nd) — if all of the global top-3 are in the union, LB <= the union's
// 3rd = the true 3rd; else a global top-3 key lies beyond its set's 2nd, so the true 3rd >= that
// set's 2nd >= LB.  The certificate takes LB for the third-best value (level 2 only), so a row
// may be left undecided where the exact top-3 would have certified it, never the converse.
template <bool kImad, bool kTop2>
__global__ void __launch_bounds__(kWsThreads, 2) k_match_ws(const __grid_constant__ CUtensorMap tmap, TcArgs A) {
  extern __shared__ uint8_t tc_smem_raw[];
  __shared__ __align__(8) uint64_t bar_a, bar_b[2], bar_mma[2], bar_free[2], bar_c[2];
  __shared__ uint32_t tmem_base_sh;
  __shared__ __align__(16) uint4 rmerge[2][128];
  __shared__ int fs_warp[4];
  // 1024-B aligned by an offset from the shared array itself (not an integer round trip), so the
  // compiler keeps the shared address space: LDS for the column constants, not generic LD
  uint8_t *base = tc_smem_raw + ((1024u - (smem_u32(tc_smem_raw) & 1023u)) & 1023u);
  uint8_t *sA = base;                                           // [2 K-atoms][128 rows][128 B]
  uint8_t *sB = base + 32768;                                   // [2 buffers][2 K-atoms][128 rows][128 B]
  float2 *cconst = reinterpret_cast<float2 *>(base + 3 * 32768);  // [2][kN] (|b_j|^2 + 2.01 P_a P_b, j bits)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n_pad = A.n_pad;
  const int n_items = 2 * A.P * (n_pad / 128);
  const unsigned imask = (1u << A.ibits) - 1u;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_sh)),
                 "r"(2 * kN)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (tid == 0) {
    mbar_init(&bar_a, 1);
    for (int b = 0; b < 2; ++b) {
      mbar_init(&bar_b[b], 1); mbar_init(&bar_mma[b], 1); mbar_init(&bar_free[b], kWsEpiWarps); mbar_init(&bar_c[b], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_wait();                       // the setup above (no global memory) overlapped k_desc_half's end
  const uint32_t tmem = tmem_base_sh;
  // instruction descriptor: D f32, A/B f16, K-major both, N = 128, M = 128
  const uint32_t idesc = (1u << 4) | ((uint32_t)(kN >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);

  if (warp == kWsEpiWarps) {
    // ------------------------------------------------------------ producer
    // item descriptors and the column norms are prefetched one item / one chunk ahead, so no
    // dependent global load sits between the epilogue's release of a buffer and the next MMA
    uint32_t g = 0, nitem = 0;
    int it = blockIdx.x;
    TcItem I;
    if (it < n_items) I = tc_item(A, it);
    float nv[kN / 32];                                            // norms of the next chunk's columns
    bool nv_ok = false;
    while (it < n_items) {
      const int itn = it + gridDim.x;
      TcItem In;
      In.skip = true;
      if (itn < n_items) In = tc_item(A, itn);
      if (!I.skip) {
        const float ma_ = frame_scale(A.S.maxnorm[I.fa]), mb_ = frame_scale(A.S.maxnorm[I.fb]);
        const float coff = 2.01f * ma_ * mb_;
        const float cinv = kImad ? A.kwin / (mb_ * mb_ + 4.02f * ma_ * mb_) : 0.f;
        for (int c = 0; c < I.nchunks; ++c, ++g) {
          const int b = g & 1;
          if (!nv_ok) {
#pragma unroll
            for (int q = 0; q < kN / 32; ++q) {
              const int j = c * kN + q * 32 + lane;
              nv[q] = j < I.nb ? A.S.norm[(size_t)I.fb * n_pad + j] : 0.f;
            }
          }
          if (lane == 0) {
            if (c == 0) {                                         // A of this item, once the old one is read
              if (g > 0) mbar_wait(&bar_mma[(g - 1) & 1], ((g - 1) >> 1) & 1);
              mbar_expect_tx(&bar_a, 32768u);
              tma_load_2d(sA, &tmap, 0, I.fa * n_pad + I.rt * 128, &bar_a);
              tma_load_2d(sA + 16384, &tmap, 64, I.fa * n_pad + I.rt * 128, &bar_a);
            }
            if (g >= 2) mbar_wait(&bar_mma[b], ((g - 2) >> 1) & 1);   // B buffer b consumed by MMA g - 2
            mbar_expect_tx(&bar_b[b], 32768u);
            uint8_t *dst = sB + b * 32768;
            tma_load_2d(dst, &tmap, 0, I.fb * n_pad + c * kN, &bar_b[b]);
            tma_load_2d(dst + 16384, &tmap, 64, I.fb * n_pad + c * kN, &bar_b[b]);
          }
          if (g >= 2) mbar_wait(&bar_free[b], ((g - 2) >> 1) & 1);    // epilogue done with chunk g - 2
#pragma unroll
          for (int q = 0; q < kN / 32; ++q) {
            const int jj = q * 32 + lane, j = c * kN + jj;
            // |b_j|^2 + the offset that keeps every ranked value >= 0; a column past n_b ranks at
            // +inf (no per-element bound check in the epilogue)
            if (kImad)
              cconst[b * kN + jj] = make_float2(j < I.nb ? __fmaf_rn(cinv, __fmaf_rn(nv[q], nv[q], coff), 1.0f)
                                                         : __uint_as_float(A.kpad),
                                                __uint_as_float((unsigned)j));
            else
              cconst[b * kN + jj] = make_float2(j < I.nb ? __fmaf_rn(nv[q], nv[q], coff) : CUDART_INF_F,
                                                __uint_as_float((unsigned)j));
          }
          __syncwarp();
          if (lane == 0) {
            mbar_arrive(&bar_c[b]);                               // release: the constants are visible
            if (c == 0) mbar_wait(&bar_a, nitem & 1);
            mbar_wait(&bar_b[b], (g >> 1) & 1);
            tc_fence_after();
#pragma unroll
            for (int k = 0; k < 8; ++k) {                         // K = 128 = 8 x 16
              const int kb = k >> 2, ks = k & 3;
              umma_f16(tmem + b * kN, umma_desc_sw128(sA + kb * 16384 + ks * 32),
                       umma_desc_sw128(sB + b * 32768 + kb * 16384 + ks * 32), idesc, k > 0 ? 1u : 0u);
            }
            umma_commit(&bar_mma[b]);
          }
          __syncwarp();
          // prefetch the next chunk's column norms (this item's, else the next item's first)
          const bool same = c + 1 < I.nchunks;
          nv_ok = same || !In.skip;
          if (nv_ok) {
            const int fbn = same ? I.fb : In.fb, nbn = same ? I.nb : In.nb, cn = same ? c + 1 : 0;
#pragma unroll
            for (int q = 0; q < kN / 32; ++q) {
              const int j = cn * kN + q * 32 + lane;
              nv[q] = j < nbn ? A.S.norm[(size_t)fbn * n_pad + j] : 0.f;
            }
          }
        }
        ++nitem;
      }
      I = In;
      it = itn;
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const int wg = warp >> 2;
    const int lrow = (warp & 3) * 32 + lane;                      // TMEM lane = tile row
    uint32_t g = 0, nitem = 0;
    int it = blockIdx.x;
    TcItem In;
    float na_nx = 0.f, mr_nx = 0.f;                               // the next item's row norm / max |b|
    unsigned ma_nx = 0u, mb_nx = 0u;                              // max-norm bits of its frames
    if (it < n_items) {
      In = tc_item(A, it);
      na_nx = A.S.norm[(size_t)In.fa * n_pad + In.rt * 128 + lrow];
      ma_nx = A.S.maxnorm[In.fa]; mb_nx = A.S.maxnorm[In.fb];
      mr_nx = __uint_as_float(mb_nx);
    }
    for (; it < n_items; it += gridDim.x) {
      const TcItem I = In;
      const float na_n = na_nx, mr = mr_nx;
      // S'' = (a / P_a).(b / P_b): d' = |b|^2 - 2 P_a P_b S''
      const float fsa = frame_scale(ma_nx), fsb = frame_scale(mb_nx);
      const float pp = fsa * fsb;
      const float kscale = kImad ? -2.f * pp * (A.kwin / (fsb * fsb + 4.02f * pp)) : -2.f * pp;
      if (it + (int)gridDim.x < n_items) {                        // prefetch the next item
        In = tc_item(A, it + gridDim.x);
        na_nx = A.S.norm[(size_t)In.fa * n_pad + In.rt * 128 + lrow];
        ma_nx = A.S.maxnorm[In.fa]; mb_nx = A.S.maxnorm[In.fb];
        mr_nx = __uint_as_float(mb_nx);
      }
      if (I.skip) {
        if (A.fs_batched && tid == 0) A.S.fs_count[it] = 0;
        continue;
      }
      const int i = I.rt * 128 + lrow;
      unsigned r1 = kNone, r2 = kNone, r3 = kNone, s1 = kNone, s2 = kNone, s3 = kNone;
      unsigned x1[4] = {kNone, kNone, kNone, kNone}, x2[4] = {kNone, kNone, kNone, kNone};   // kTop2 sets
      for (int c = 0; c < I.nchunks; ++c, ++g) {
        const int b = g & 1;
        mbar_wait(&bar_mma[b], (g >> 1) & 1);
        mbar_wait(&bar_c[b], (g >> 1) & 1);
        tc_fence_after();
#pragma unroll 1
        for (int cc = wg * 2; cc < wg * 2 + 2; ++cc) {
          const int j0 = c * kN + cc * 32;
          if (j0 >= I.nb) break;                                  // warpgroup-uniform
          uint32_t v[32];
          BT_TMEM_LD32(tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)(b * kN + cc * 32), v);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          const float4 *cb = reinterpret_cast<const float4 *>(cconst + b * kN + cc * 32);   // 2 columns per load
#pragma unroll
          for (int col = 0; col < 32; col += 2) {
            const float4 cc2 = cb[col >> 1];
            // d'' = d' + 2.01 P_a P_b >= 0 (one FFMA), so the float bits order like the values
            const float d0 = __fmaf_rn(kscale, __uint_as_float(v[col]), cc2.x);
            const float d1 = __fmaf_rn(kscale, __uint_as_float(v[col + 1]), cc2.z);
            unsigned k0, k1;
            if (kImad) {                                          // one IMAD each (FMA pipe)
              asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(k0) : "r"(__float_as_uint(d0)), "r"(A.kmul), "r"(__float_as_uint(cc2.y)));
              asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(k1) : "r"(__float_as_uint(d1)), "r"(A.kmul), "r"(__float_as_uint(cc2.w)));
            } else {
              k0 = (__float_as_uint(d0) & ~imask) | __float_as_uint(cc2.y);
              k1 = (__float_as_uint(d1) & ~imask) | __float_as_uint(cc2.w);
            }
            const unsigned m = min(k0, k1), M = max(k0, k1);
            if (kTop2) {
              const int st = (col >> 1) & 3;
              x2[st] = min(min(x2[st], max(x1[st], m)), M);
              x1[st] = min(x1[st], m);
            } else if ((col & 2) == 0) {
              const unsigned n3 = min(min(r3, max(r2, m)), max(r1, M)), n2 = min(min(r2, max(r1, m)), M);
              r1 = min(r1, m); r2 = n2; r3 = n3;
            } else {
              const unsigned n3 = min(min(s3, max(s2, m)), max(s1, M)), n2 = min(min(s2, max(s1, m)), M);
              s1 = min(s1, m); s2 = n2; s3 = n3;
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bar_free[b]);                 // TMEM + constants of buffer b released
      }
      // merge the even/odd sets, then the two warpgroups' top-3; certify; decide the row or queue it
      unsigned mr2 = kNone;                                        // kTop2: min of the sets' 2nd
      if (kTop2) {
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          const unsigned k = t < 4 ? x1[t] : x2[t - 4];
          const unsigned n3 = min(r3, max(r2, k)), n2 = min(r2, max(r1, k));
          r1 = min(r1, k); r2 = n2; r3 = n3;
        }
        mr2 = min(min(x2[0], x2[1]), min(x2[2], x2[3]));
      } else {
        const unsigned ks[3] = {s1, s2, s3};
#pragma unroll
        for (int t = 0; t < 3; ++t) {
          const unsigned k = ks[t];
          const unsigned n3 = min(r3, max(r2, k)), n2 = min(r2, max(r1, k));
          r1 = min(r1, k); r2 = n2; r3 = n3;
        }
      }
      uint4 *rm = rmerge[nitem & 1];
      if (wg == 1) rm[lrow] = make_uint4(r1, r2, r3, mr2);
      named_bar(1, kWsEpiWarps * 32);
      int level = 1;
      if (wg == 0 && i < I.na) {
        const uint4 o = rm[lrow];
        const unsigned ks[3] = {o.x, o.y, o.z};
#pragma unroll
        for (int t = 0; t < 3; ++t) {
          const unsigned k = ks[t];
          const unsigned n3 = min(r3, max(r2, k)), n2 = min(r2, max(r1, k));
          r1 = min(r1, k); r2 = n2; r3 = n3;
        }
        if (kTop2) r3 = min(r3, min(mr2, o.w));                   // the third-best lower bound
        level = 0;
        if (!A.force_fallback && A.ratio2 >= 1.f)
          level = kImad ? certify_imad(r1, r2, r3, na_n, mr, pp, fsa, fsb, A.kshift) : certify(r1, r2, r3, na_n, mr, pp, A.ibits);
        const size_t o_nn = (size_t)I.p * A.kp.n_max + i;
        if (level == 1) {
          (I.dir == 0 ? A.S.nn_ab : A.S.nn_ba)[o_nn] = (int32_t)(r1 & imask);
          if (I.dir == 0) A.S.ratio_ok[o_nn] = 1;
        } else if (level == 2 || !A.fs_batched) {               // queue: [0] top-2 rescoring, [1] full scan
          const int qi = level == 2 ? 0 : 1;
          const unsigned slot = atomicAdd(A.S.work_count + qi, 1u);
          A.S.work[(size_t)qi * A.S.work_cap + slot] = make_uint4((unsigned)I.dir | ((unsigned)i << 1), (unsigned)I.p, r1, r2);
        }
      }
      if (A.fs_batched && wg == 0) {                              // undecided rows -> this item's list
        const bool fs = i < I.na && level == 0;
        const unsigned bal = __ballot_sync(0xffffffffu, fs);
        if (lane == 0) fs_warp[warp] = __popc(bal);
        named_bar(2, 128);                                        // warpgroup 0 only
        int off = 0;
        for (int w = 0; w < warp; ++w) off += fs_warp[w];
        if (fs) A.S.fs_rows[(size_t)it * 128 + off + __popc(bal & ((1u << lane) - 1u))] = i;
        if (tid == 0) A.S.fs_count[it] = fs_warp[0] + fs_warp[1] + fs_warp[2] + fs_warp[3];
      }
      ++nitem;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * kN) : "memory");
  }
}

// ---------------------------------------------------------------- exact fp32 rescoring
// warp-cooperative brute force over nr references (lane l owns words 4l..4l+3, 32 references
// per step, transpose reduction — the butterfly's tree): best, index (ties lowest), second
__device__ void exact_scan(const float4 a, const float4 *R, int nr, int lane, float &b1, int &j1, float &b2) {
  b1 = CUDART_INF_F; b2 = CUDART_INF_F; j1 = -1;
  for (int j0 = 0; j0 < nr; j0 += 32) {
    float v[32];
#pragma unroll
    for (int c = 0; c < 32; ++c) {
      const int j = j0 + c;
      float s = 0.f;
      if (j < nr) {
        const float4 b = __ldg(R + (size_t)j * 32 + lane);
        const float dx = __fsub_rn(a.x, b.x), dy = __fsub_rn(a.y, b.y);
        const float dz = __fsub_rn(a.z, b.z), dw = __fsub_rn(a.w, b.w);
        s = __fmul_rn(dx, dx);
        s = __fmaf_rn(dy, dy, s);
        s = __fmaf_rn(dz, dz, s);
        s = __fmaf_rn(dw, dw, s);
      }
      v[c] = s;
    }
    // transpose reduction: lane l ends with the distance to reference j0 + l
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
      const bool upper = (lane & o) != 0;
#pragma unroll
      for (int c = 0; c < o; ++c) {
        const float send = upper ? v[c] : v[c + o];
        const float keep = upper ? v[c + o] : v[c];
        v[c] = __fadd_rn(keep, __shfl_xor_sync(0xffffffffu, send, o));
      }
    }
    const int j = j0 + lane;
    if (j < nr) {
      if (v[0] < b1) { b2 = b1; b1 = v[0]; j1 = j; }
      else if (v[0] < b2) b2 = v[0];
    }
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    const float ob1 = __shfl_xor_sync(0xffffffffu, b1, o);
    const int oj1 = __shfl_xor_sync(0xffffffffu, j1, o);
    const float ob2 = __shfl_xor_sync(0xffffffffu, b2, o);
    const bool mine = (b1 < ob1) || (b1 == ob1 && (unsigned)j1 < (unsigned)oj1);
    if (mine) b2 = fminf(b2, ob1);
    else { b2 = fminf(ob2, b1); b1 = ob1; j1 = oj1; }
  }
}

// fp32 distance of one reference: 4 sequential terms per lane (words 4l..4l+3), then the lane
// tree bit 4, 3, 2, 1, 0 (a butterfly) — k_fullscan reproduces this tree bit for bit
__device__ __forceinline__ float exact_one(const float4 a, const float4 *R, int j, int lane) {
  const float4 b = __ldg(R + (size_t)j * 32 + lane);
  const float dx = __fsub_rn(a.x, b.x), dy = __fsub_rn(a.y, b.y);
  const float dz = __fsub_rn(a.z, b.z), dw = __fsub_rn(a.w, b.w);
  float s = __fmul_rn(dx, dx);
  s = __fmaf_rn(dy, dy, s);
  s = __fmaf_rn(dz, dz, s);
  s = __fmaf_rn(dw, dw, s);
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) s = __fadd_rn(s, __shfl_xor_sync(0xffffffffu, s, o));
  return s;
}


struct RescoreArgs {
  KpView kp;
  const int32_t *pairs;
  MatchScratch S;
  int ibits;
  float ratio2;
};

// blockIdx.y == 0: warps over the top-2 queue (two exact distances per row);
// blockIdx.y == 1: CTAs over the full-scan queue, the references split across the 8 warps
__global__ void __launch_bounds__(kWarpsPerBlock * 32) k_rescore(RescoreArgs A) {
  pdl_wait();
  __shared__ float sb1[kWarpsPerBlock], sb2[kWarpsPerBlock];
  __shared__ int sj1[kWarpsPerBlock];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned imask = (1u << A.ibits) - 1u;
  if (blockIdx.y == 0) {
    const unsigned n_work = A.S.work_count[0];
    const int gw = blockIdx.x * kWarpsPerBlock + warp, nw = gridDim.x * kWarpsPerBlock;
    for (unsigned w = gw; w < n_work; w += nw) {
      const uint4 it = A.S.work[w];
      const int dir = it.x & 1, q = (int)(it.x >> 1), p = (int)it.y;
      const int fq = A.pairs[2 * p + dir], fr = A.pairs[2 * p + 1 - dir];
      const float4 a = reinterpret_cast<const float4 *>(A.kp.desc + ((size_t)fq * A.kp.n_max + q) * kDim)[lane];
      const float4 *R = reinterpret_cast<const float4 *>(A.kp.desc + (size_t)fr * A.kp.n_max * kDim);
      const int ja = (int)(it.z & imask), jb = (int)(it.w & imask);
      const float da = exact_one(a, R, ja, lane), db = exact_one(a, R, jb, lane);
      if (lane == 0) {
        const size_t o = (size_t)p * A.kp.n_max + q;
        (dir == 0 ? A.S.nn_ab : A.S.nn_ba)[o] = (db < da || (db == da && jb < ja)) ? jb : ja;
        if (dir == 0) A.S.ratio_ok[o] = 1;
      }
    }
    return;
  }
  const unsigned n_work = A.S.work_count[1];
  for (unsigned w = blockIdx.x; w < n_work; w += gridDim.x) {
    const uint4 it = A.S.work[(size_t)A.S.work_cap + w];
    const int dir = it.x & 1, q = (int)(it.x >> 1), p = (int)it.y;
    const int fq = A.pairs[2 * p + dir], fr = A.pairs[2 * p + 1 - dir];
    const int nr = min(A.kp.n_kp[fr], A.kp.n_max);
    const float4 a = reinterpret_cast<const float4 *>(A.kp.desc + ((size_t)fq * A.kp.n_max + q) * kDim)[lane];
    const float4 *R = reinterpret_cast<const float4 *>(A.kp.desc + (size_t)fr * A.kp.n_max * kDim);
    // warp w scans references [w*span, (w+1)*span) (span a multiple of 32: same per-column tree)
    const int span = ((nr + kWarpsPerBlock * 32 - 1) / (kWarpsPerBlock * 32)) * 32;
    const int j0 = min(nr, warp * span), j1e = min(nr, j0 + span);
    float b1, b2;
    int jb;
    exact_scan(a, R + (size_t)j0 * 32, j1e - j0, lane, b1, jb, b2);
    if (lane == 0) { sb1[warp] = b1; sb2[warp] = b2; sj1[warp] = jb < 0 ? -1 : jb + j0; }
    __syncthreads();
    if (threadIdx.x == 0) {
      float B1 = CUDART_INF_F, B2 = CUDART_INF_F;
      int J1 = -1;
      for (int w2 = 0; w2 < kWarpsPerBlock; ++w2) {                // ascending index order: ties -> lowest
        if (sj1[w2] < 0) continue;
        if (sb1[w2] < B1) { B2 = fminf(B1, sb2[w2]); B1 = sb1[w2]; J1 = sj1[w2]; }
        else B2 = fminf(B2, sb1[w2]);
      }
      const size_t o = (size_t)p * A.kp.n_max + q;
      (dir == 0 ? A.S.nn_ab : A.S.nn_ba)[o] = J1;
      if (dir == 0) A.S.ratio_ok[o] = (A.ratio2 >= 1.f) || (nr < 2) || (B1 < A.ratio2 * B2);
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- level-2 certification
// The rows k_match_ws could not certify (fp16 operands: |d_hat - d| <= 2.2e-3 |a| M_b) are
// re-ranked by warp-level tensor-core MMAs (mma.sync m16n8k16, fp32 accumulation) on hi + lo
// fp16 operands — S'' = A_hi B_hi + A_hi B_lo + A_lo B_hi of the frame-max-scaled descriptors,
// which leaves out only A_lo B_lo (<= 2^-22 |a||b| / M_a M_b) — over ALL references, with a
// certificate 9x tighter: |S''_hat - S''| <= 2^-13 |a||b| / (M_a M_b) (the dropped term, the hi /
// lo representation, and the fp32 accumulation of 24 MMA steps, with margin), so
// |d_hat - d| <= 2.5e-4 |a| M_b + 1e-6 (|a|^2 + M_b^2) + 3e-6 M_a M_b.  A row is then decided (its
// best certified), queued for the exact top-2 rescoring (k_rescore), or left for the exact full
// scan (k_fullscan, the l3 list).  Keys: the ranked value mapped into [1, 2) (one FFMA with a
// per-column constant, as k_match_ws) and packed as its top 20 mantissa bits above the 12-bit
// column index (n_pad <= 4096): the 3 truncated bits are in the certificate.
// CTA = 4 warps x 16 rows of one (pair, direction); references in chunks of 128 (hi + lo staged
// with cp.async, rows padded to 136 halves: conflict-free ldmatrix).
constexpr int kL2Rows = 64, kL2Refs = 128, kL2Pitch = 136;      // halves per staged row
constexpr size_t kL2Smem = (size_t)(2 * kL2Rows + 2 * kL2Refs) * kL2Pitch * 2 + kL2Refs * 8;

struct L2Args {
  KpView kp;
  const int32_t *pairs;
  MatchScratch S;
  int P, n_pad;
  int certify;                                 // 0: ratio test / forced fallback — forward every row
};

__device__ __forceinline__ void cp_async16(void *dst, const void *src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], const void *p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(smem_u32(p)));
}
__device__ __forceinline__ void ldsm_x2(uint32_t (&r)[2], const void *p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0,%1}, [%2];" : "=r"(r[0]), "=r"(r[1]) : "r"(smem_u32(p)));
}
__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
               "{%0,%1,%2,%3};"
               : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
               : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

__global__ void __launch_bounds__(128) k_match_l2(L2Args A) {
  pdl_wait();
  extern __shared__ __align__(16) uint8_t l2sm[];
  __half *sAh = reinterpret_cast<__half *>(l2sm);                 // [64][136]
  __half *sAl = sAh + kL2Rows * kL2Pitch;
  __half *sBh = sAl + kL2Rows * kL2Pitch;                          // [128][136]
  __half *sBl = sBh + kL2Refs * kL2Pitch;
  float2 *sC = reinterpret_cast<float2 *>(sBl + kL2Refs * kL2Pitch);   // [128] (column constant, j)
  __shared__ int toff[65];
  __shared__ int grow[kL2Rows];
  const int g = blockIdx.x, p = blockIdx.y, dir = blockIdx.z;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n_tiles = A.n_pad / 128;
  const int tile0 = (dir * A.P + p) * n_tiles;
  if (tid == 0) {                                                  // the (pair, direction)'s rows, in tile order
    int acc = 0;
    for (int t = 0; t < n_tiles; ++t) { toff[t] = acc; acc += A.S.fs_count[tile0 + t]; }
    toff[n_tiles] = acc;
  }
  __syncthreads();
  const int u = toff[n_tiles];
  for (int gg = g; gg * kL2Rows < u; gg += gridDim.x) {             // groups of 64 rows, block-uniform
  const int g0 = gg * kL2Rows;
  const int gn = min(kL2Rows, u - g0);
  __syncthreads();                                                 // the previous group's smem reads done
  if (tid < kL2Rows) {
    int r = -1;
    if (tid < gn) {
      const int gi = g0 + tid;
      int t = 0;
      while (toff[t + 1] <= gi) ++t;
      r = A.S.fs_rows[(size_t)(tile0 + t) * 128 + (gi - toff[t])];
    }
    grow[tid] = r;
  }
  __syncthreads();
  const int lq = (dir * A.P + p);
  int32_t *l3 = A.S.l3_rows + (size_t)lq * A.n_pad;
  if (!A.certify) {                                                // forward the rows to the exact scan
    if (tid < gn) l3[atomicAdd(A.S.l3_count + lq, 1)] = grow[tid];
    continue;
  }
  const int fq = A.pairs[2 * p + dir], fr = A.pairs[2 * p + 1 - dir];
  const int nr = min(A.kp.n_kp[fr], A.kp.n_max);
  const int n_pad = A.n_pad;
  const __half *Qh = A.S.desc16 + (size_t)fq * n_pad * kDim, *Ql = A.S.desc16lo + (size_t)fq * n_pad * kDim;
  const __half *Rh = A.S.desc16 + (size_t)fr * n_pad * kDim, *Rl = A.S.desc16lo + (size_t)fr * n_pad * kDim;
  // A rows: 64 x (256 B hi + 256 B lo) in 16-B pieces
  for (int x = tid; x < kL2Rows * 16; x += 128) {
    const int r = x >> 4, c = x & 15;
    const int row = grow[r] < 0 ? 0 : grow[r];                    // padded rows: any row (ignored)
    cp_async16(sAh + r * kL2Pitch + c * 8, Qh + (size_t)row * kDim + c * 8);
    cp_async16(sAl + r * kL2Pitch + c * 8, Ql + (size_t)row * kDim + c * 8);
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
  const float ma = frame_scale(A.S.maxnorm[fq]), mb = frame_scale(A.S.maxnorm[fr]);
  const float pp = ma * mb;
  const float cinv = 1.0f / (mb * mb + 4.02f * pp);
  const float kscale = -2.f * pp * cinv;
  // per thread: rows r0 = 16 warp + lane / 4 and r0 + 8, columns 2 (lane % 4) + {0, 1} of each n-tile
  unsigned t0[3] = {kNone, kNone, kNone}, t1[3] = {kNone, kNone, kNone};
  auto ins = [](unsigned (&t)[3], unsigned k) {
    const unsigned n3 = min(t[2], max(t[1], k)), n2 = min(t[1], max(t[0], k));
    t[0] = min(t[0], k); t[1] = n2; t[2] = n3;
  };
  for (int jc = 0; jc < nr; jc += kL2Refs) {
    __syncthreads();                                               // the previous chunk consumed
    for (int x = tid; x < kL2Refs * 16; x += 128) {
      const int j = x >> 4, c = x & 15;
      const int jj = min(jc + j, n_pad - 1);                       // rows past n_r: zero-padded rows
      cp_async16(sBh + j * kL2Pitch + c * 8, Rh + (size_t)jj * kDim + c * 8);
      cp_async16(sBl + j * kL2Pitch + c * 8, Rl + (size_t)jj * kDim + c * 8);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    {                                                              // column constants (IMAD-free: value in [1, 2))
      const int j = jc + tid;
      const float nb = j < nr ? A.S.norm[(size_t)fr * n_pad + j] : 0.f;
      sC[tid] = make_float2(j < nr ? __fmaf_rn(cinv, __fmaf_rn(nb, nb, 2.01f * pp), 1.0f)
                                   : __uint_as_float(0x3FFFFFFFu), __uint_as_float((unsigned)j));
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    float acc[16][4];
#pragma unroll
    for (int nt = 0; nt < 16; ++nt)
#pragma unroll
      for (int k = 0; k < 4; ++k) acc[nt][k] = 0.f;
#pragma unroll 2
    for (int kk = 0; kk < 8; ++kk) {
      uint32_t ah[4], al[4];
      // A fragment (16 x 16 at rows 16 warp, k 16 kk): ldmatrix x4, lane -> row (lane & 15), k-half (lane >> 4)
      const int ar = 16 * warp + (lane & 15), ak = 16 * kk + 8 * (lane >> 4);
      ldsm_x4(ah, sAh + ar * kL2Pitch + ak);
      ldsm_x4(al, sAl + ar * kL2Pitch + ak);
#pragma unroll
      for (int nt = 0; nt < 16; ++nt) {
        uint32_t bh[2], bl[2];
        // B fragment (16 k x 8 n, "col"): the 8 reference rows 8 nt.., k halves by lanes 0-7 / 8-15
        const int br = 8 * nt + (lane & 7), bk = 16 * kk + 8 * ((lane >> 3) & 1);
        ldsm_x2(bh, sBh + br * kL2Pitch + bk);
        ldsm_x2(bl, sBl + br * kL2Pitch + bk);
        mma16816(acc[nt], ah, bh);
        mma16816(acc[nt], ah, bl);
        mma16816(acc[nt], al, bh);
      }
    }
    // ranking: d'' mapped into [1, 2), key = top 20 mantissa bits | 12-bit column
#pragma unroll
    for (int nt = 0; nt < 16; ++nt) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const float2 cc = sC[8 * nt + 2 * (lane & 3) + e];
        const float v0 = __fmaf_rn(kscale, acc[nt][e], cc.x), v1 = __fmaf_rn(kscale, acc[nt][2 + e], cc.x);
        const unsigned k0 = ((__float_as_uint(v0) << 9) & 0xFFFFF000u) | __float_as_uint(cc.y);
        const unsigned k1 = ((__float_as_uint(v1) << 9) & 0xFFFFF000u) | __float_as_uint(cc.y);
        ins(t0, k0);
        ins(t1, k1);
      }
    }
  }
  // merge the 4 lanes of each row (xor 1, 2), then certify
#pragma unroll
  for (int o = 1; o <= 2; o <<= 1) {
    unsigned x0[3], x1[3];                                         // the partner's lists, read first
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      x0[q] = __shfl_xor_sync(0xffffffffu, t0[q], o);
      x1[q] = __shfl_xor_sync(0xffffffffu, t1[q], o);
    }
#pragma unroll
    for (int q = 0; q < 3; ++q) {                                  // columns are disjoint across lanes
      ins(t0, x0[q]);
      ins(t1, x1[q]);
    }
  }
  if ((lane & 3) == 0) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int r = 16 * warp + (lane >> 2) + 8 * h;
      if (r >= gn) continue;                                       // (the row loop)
      const int i = grow[r];
      const unsigned *t = h ? t1 : t0;
      const float qn = A.S.norm[(size_t)fq * n_pad + i];
      // key units: 2^-20 of the [1, 2) value = 2^-20 / c in d; each key within 3 units of 1 + c d''
      const float uk = ldexpf(mb * mb + 4.02f * pp, -20);
      const float eps2 = 2.f * (2.5e-4f * qn * mb + 1e-6f * (qn * qn + mb * mb) + 3e-6f * pp) + 8.f * uk;
      int level = 0;
      if (t[0] != kNone) {
        if (t[1] == kNone) level = 1;
        else if ((float)((t[1] >> 12) - (t[0] >> 12)) * uk > eps2) level = 1;
        else if (t[2] == kNone || (float)((t[2] >> 12) - (t[0] >> 12)) * uk > eps2) level = 2;
      }
      const size_t o_nn = (size_t)p * A.kp.n_max + i;
      if (level == 1) {
        (dir == 0 ? A.S.nn_ab : A.S.nn_ba)[o_nn] = (int32_t)(t[0] & 0xFFFu);
        if (dir == 0) A.S.ratio_ok[o_nn] = 1;
      } else if (level == 2) {                                     // the exact top-2 (k_rescore, queue 0)
        const unsigned slot = atomicAdd(A.S.work_count, 1u);
        A.S.work[slot] = make_uint4((unsigned)dir | ((unsigned)i << 1), (unsigned)p, t[0] & 0xFFFu, t[1] & 0xFFFu);
      } else {
        l3[atomicAdd(A.S.l3_count + lq, 1)] = i;
      }
    }
  }
  }
}

// ---------------------------------------------------------------- exact full scans, batched
// One CTA per (group of 32, pair, direction): the undecided rows of a (pair, direction) — the
// row tiles' lists of k_match_tc concatenated in order — in groups of 32 against all
// references in chunks of 64, both staged in shared memory, so a reference is read once per 32
// rows instead of once per row; warps without rows skip the arithmetic.  With few rows or few
// references (C2: n ~ 500) one CTA takes one row and its 8 warps split the references instead.  Warp w owns rows 4w..4w+3 of the
// group, lane l references 2l, 2l+1 of the chunk: 8 exact fp32 distances per thread.  Each
// distance is bitwise the value exact_one computes: the 32 "lane" partials (4
// sequential terms over words 4l..4l+3) combined in the butterfly's tree — leaves visited in
// bit-reversed order and merged as a binary counter.  Best (ties: lowest index) and second
// best are combined across lanes order-independently.
constexpr int kFsRows = 32, kFsRefs = 64, kFsPitch = kFsRefs + 2;   // sB row pitch (8-B aligned pairs)
constexpr int kFsSmall = 4;                      // (pair, dir)s with at most this many rows: per-row path
constexpr int kFsBatchRefs = 1024;               // batch only when a row scan reads >= 512 KB
#ifndef BT_L2_MIN_NMAX
#define BT_L2_MIN_NMAX 1024
#endif
// n_max from which the rows the first level leaves undecided go to the level-2 pass (per-tile
// lists) instead of the per-row exact queue
constexpr int kL2MinNmax = BT_L2_MIN_NMAX;
constexpr size_t kFsSmem = (size_t)(kFsRows * kDim + kDim * kFsPitch) * sizeof(float);

struct FullScanArgs {
  KpView kp;
  const int32_t *pairs;
  MatchScratch S;
  int P, n_pad, ibits;
  float ratio2;
};

__host__ __device__ constexpr int bitrev5(int s) {
  return ((s & 1) << 4) | ((s & 2) << 2) | (s & 4) | ((s & 8) >> 2) | ((s & 16) >> 4);
}

__global__ void __launch_bounds__(256) k_fullscan(FullScanArgs A) {
  pdl_wait();
  extern __shared__ __align__(16) float fsm[];
  float *sA = fsm;                                   // [32][128] rows (broadcast reads)
  float *sB = fsm + kFsRows * kDim;                  // [128][kFsPitch] k-major reference chunk
  __shared__ int grow[kFsRows];                      // this group's rows
  const int g = blockIdx.x, p = blockIdx.y, dir = blockIdx.z;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // the (pair, direction)'s rows the level-2 pass left uncertified (k_match_l2)
  const int u = A.S.l3_count[dir * A.P + p];
  const int32_t *l3 = A.S.l3_rows + (size_t)(dir * A.P + p) * A.n_pad;
  const int fq = A.pairs[2 * p + dir], fr = A.pairs[2 * p + 1 - dir];
  const int nr = min(A.kp.n_kp[fr], A.kp.n_max);
  const float *Q = A.kp.desc + (size_t)fq * A.kp.n_max * kDim;
  const float *R = A.kp.desc + (size_t)fr * A.kp.n_max * kDim;
  auto row_of = [&](int gi) { return l3[gi]; };     // gi-th undecided row of (p, dir)
  if (u <= kFsSmall || nr < kFsBatchRefs) {
    // few rows (or few references in this pair): one row per CTA, the 8 warps split the
    // references and read them straight from L2 (exact_scan — the same distances, bit for bit)
    __shared__ float sb1[8], sb2[8];
    __shared__ int sj1[8];
    const int span = ((nr + 8 * 32 - 1) / (8 * 32)) * 32;
    const int j0 = min(nr, warp * span), j1e = min(nr, j0 + span);
    for (int gi = g; gi < u; gi += gridDim.x) {
      const int i = row_of(gi);
      const float4 a = __ldg(reinterpret_cast<const float4 *>(Q + (size_t)i * kDim) + lane);
      float b1, b2;
      int jb;
      exact_scan(a, reinterpret_cast<const float4 *>(R) + (size_t)j0 * 32, j1e - j0, lane, b1, jb, b2);
      if (lane == 0) { sb1[warp] = b1; sb2[warp] = b2; sj1[warp] = jb < 0 ? -1 : jb + j0; }
      __syncthreads();
      if (threadIdx.x == 0) {
        float B1 = CUDART_INF_F, B2 = CUDART_INF_F;
        int J1 = -1;
        for (int w2 = 0; w2 < 8; ++w2) {                            // ascending index order: ties -> lowest
          if (sj1[w2] < 0) continue;
          if (sb1[w2] < B1) { B2 = fminf(B1, sb2[w2]); B1 = sb1[w2]; J1 = sj1[w2]; }
          else B2 = fminf(B2, sb1[w2]);
        }
        const size_t o = (size_t)p * A.kp.n_max + i;
        (dir == 0 ? A.S.nn_ab : A.S.nn_ba)[o] = J1;
        if (dir == 0) A.S.ratio_ok[o] = (A.ratio2 >= 1.f) || (nr < 2) || (B1 < A.ratio2 * B2);
      }
      __syncthreads();
    }
    return;
  }
  for (int gg = g; gg * kFsRows < u; gg += gridDim.x) {             // groups of 32 rows, block-uniform
  const int g0 = gg * kFsRows;
  const int gn = min(kFsRows, u - g0);
  __syncthreads();                                   // the previous group's grow / sA reads done
  if (threadIdx.x < kFsRows) grow[threadIdx.x] = threadIdx.x < gn ? row_of(g0 + threadIdx.x) : -1;
  __syncthreads();                                   // grow visible to every thread
  const bool active = 4 * warp < gn;                 // warp-uniform: this warp has rows
  {
    __syncthreads();
    for (int x = threadIdx.x; x < kFsRows * (kDim / 4); x += blockDim.x) {
      const int r = x / (kDim / 4), c4 = x % (kDim / 4);
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (r < gn) v = __ldg(reinterpret_cast<const float4 *>(Q + (size_t)grow[r] * kDim) + c4);
      reinterpret_cast<float4 *>(sA)[x] = v;
    }
    float b1[4], b2[4];
    int j1[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) { b1[q] = CUDART_INF_F; b2[q] = CUDART_INF_F; j1[q] = -1; }
    for (int jc = 0; jc < nr; jc += kFsRefs) {
      __syncthreads();                               // previous chunk consumed
      for (int x = threadIdx.x; x < kFsRefs * (kDim / 4); x += blockDim.x) {
        const int j = x / (kDim / 4), c4 = x % (kDim / 4);
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (jc + j < nr) v = __ldg(reinterpret_cast<const float4 *>(R + (size_t)(jc + j) * kDim) + c4);
        float *col = sB + (4 * c4) * kFsPitch + j;
        col[0] = v.x; col[kFsPitch] = v.y; col[2 * kFsPitch] = v.z; col[3 * kFsPitch] = v.w;
      }
      __syncthreads();
      if (!active) continue;                         // still takes part in the staging barriers
      float lv[4][2][5];                             // binary-counter partial sums per distance
#pragma unroll
      for (int s = 0; s < 32; ++s) {
        const int l = bitrev5(s);
        float2 bw[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) bw[c] = *reinterpret_cast<const float2 *>(sB + (4 * l + c) * kFsPitch + 2 * lane);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float4 a = *reinterpret_cast<const float4 *>(sA + (4 * warp + q) * kDim + 4 * l);
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const float bx = e ? bw[0].y : bw[0].x, by = e ? bw[1].y : bw[1].x;
            const float bz = e ? bw[2].y : bw[2].x, bv = e ? bw[3].y : bw[3].x;
            const float dx = __fsub_rn(a.x, bx), dy = __fsub_rn(a.y, by);
            const float dz = __fsub_rn(a.z, bz), dw = __fsub_rn(a.w, bv);
            float x = __fmul_rn(dx, dx);
            x = __fmaf_rn(dy, dy, x);
            x = __fmaf_rn(dz, dz, x);
            x = __fmaf_rn(dw, dw, x);
            // merge leaf s into the pairwise tree (binary counter, resolved at compile time)
#pragma unroll
            for (int b = 0; b < 5; ++b) {
              if (s & (1 << b)) x = __fadd_rn(lv[q][e][b], x);
              else { lv[q][e][b] = x; break; }
            }
            if (s == 31) {                           // x is the full distance
              const int j = jc + 2 * lane + e;
              if (j < nr) {
                if (x < b1[q]) { b2[q] = b1[q]; b1[q] = x; j1[q] = j; }
                else if (x < b2[q]) b2[q] = x;
              }
            }
          }
        }
      }
    }
    // combine the lanes' (best, index, second) per row: lowest distance, ties -> lowest index
#pragma unroll
    for (int q = 0; q < 4; ++q) {
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) {
        const float ob1 = __shfl_xor_sync(0xffffffffu, b1[q], o);
        const int oj1 = __shfl_xor_sync(0xffffffffu, j1[q], o);
        const float ob2 = __shfl_xor_sync(0xffffffffu, b2[q], o);
        const bool mine = (b1[q] < ob1) || (b1[q] == ob1 && (unsigned)j1[q] < (unsigned)oj1);
        if (mine) b2[q] = fminf(b2[q], ob1);
        else { b2[q] = fminf(ob2, b1[q]); b1[q] = ob1; j1[q] = oj1; }
      }
      const int r = 4 * warp + q;
      if (lane == 0 && r < gn) {
        const int i = grow[r];
        const size_t o = (size_t)p * A.kp.n_max + i;
        (dir == 0 ? A.S.nn_ab : A.S.nn_ba)[o] = j1[q];
        if (dir == 0) A.S.ratio_ok[o] = (A.ratio2 >= 1.f) || (nr < 2) || (b1[q] < A.ratio2 * b2[q]);
      }
    }
  }
  }
}

// keep (i, nn_ab(i)) iff nn_ba(nn_ab(i)) == i (and the ratio flag); compact ascending in i
__global__ void __launch_bounds__(1024)
k_mutual(KpView kp, const int32_t *__restrict__ pairs, const int32_t *__restrict__ nn_ab,
         const int32_t *__restrict__ nn_ba, const uint8_t *__restrict__ ratio_ok,
         int32_t *__restrict__ matches, int32_t *__restrict__ n_matches, MatchScratch S) {
  pdl_wait();
  __shared__ int warp_tot[32];
  const int p = blockIdx.x;
  if (p == 0) {                            // last reader done: zero for the next call (no memsets)
    for (int f = threadIdx.x; f < kp.n_frames; f += blockDim.x) S.maxnorm[f] = 0u;
    if (threadIdx.x < 2) S.work_count[threadIdx.x] = 0u;
  }
  if (S.l3_count && threadIdx.x < 2) S.l3_count[threadIdx.x * gridDim.x + p] = 0;   // k_fullscan is done
  const int fa = pairs[2 * p], fb = pairs[2 * p + 1];
  const int na = min(kp.n_kp[fa], kp.n_max), nb = min(kp.n_kp[fb], kp.n_max);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const size_t row0 = (size_t)p * kp.n_max;
  int base = 0;
  for (int i0 = 0; i0 < na; i0 += blockDim.x) {
    const int i = i0 + threadIdx.x;
    int j = -1;
    bool keep = false;
    if (i < na && nb > 0) {
      j = nn_ab[row0 + i];
      keep = j >= 0 && nn_ba[row0 + j] == i && ratio_ok[row0 + i];
    }
    const unsigned bal = __ballot_sync(0xffffffffu, keep);
    if (lane == 0) warp_tot[warp] = __popc(bal);
    __syncthreads();
    int off = 0, tot = 0;
    for (int w = 0; w < nw; ++w) {
      const int c = warp_tot[w];
      off += (w < warp) ? c : 0;
      tot += c;
    }
    if (keep) {
      const int pos = base + off + __popc(bal & ((1u << lane) - 1u));
      matches[(row0 + pos) * 2] = i;
      matches[(row0 + pos) * 2 + 1] = j;
    }
    base += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) n_matches[p] = base;
}

int ceil_log2(int x) {
  int b = 0;
  while ((1 << b) < x) ++b;
  return b;
}

}  // namespace

int match_n_pad(int n_max) { return (n_max + 127) / 128 * 128; }

size_t match_scratch_bytes(int max_frames, int max_pairs, int n_max) {
  const size_t np = match_n_pad(n_max), F = max_frames, P = max_pairs, rt = np / 128;
  auto al = [](size_t b) { return (b + 255) / 256 * 256; };
  (void)rt;
  return al(F * np * kDim * 2) + al(F * np * 4) + al(F * 4) + al(2 * 2 * P * n_max * 16) + al(16) +
         al(P * n_max * 4) * 2 + al(P * n_max) + al(2 * P * np * 4) + al(2 * P * (np / 128) * 4) +
         (n_max >= kL2MinNmax ? al(F * np * kDim * 2) + al(2 * P * np * 4) + al(2 * P * 4) : 0);
}

MatchScratch carve_match_scratch(void *p, int max_frames, int max_pairs, int n_max) {
  const size_t np = match_n_pad(n_max), F = max_frames, P = max_pairs, rt = np / 128;
  auto al = [](size_t b) { return (b + 255) / 256 * 256; };
  char *c = (char *)p;
  MatchScratch S;
  S.desc16 = (__half *)c;        c += al(F * np * kDim * 2);
  S.norm = (float *)c;           c += al(F * np * 4);
  S.maxnorm = (unsigned *)c;     c += al(F * 4);
  S.work = (uint4 *)c;           c += al(2 * 2 * P * n_max * 16);
  S.work_cap = 2 * P * n_max;
  S.work_count = (unsigned *)c;  c += al(16);
  (void)rt;
  S.nn_ab = (int32_t *)c;        c += al(P * n_max * 4);
  S.nn_ba = (int32_t *)c;        c += al(P * n_max * 4);
  S.ratio_ok = (uint8_t *)c;     c += al(P * n_max);
  S.fs_rows = (int32_t *)c;      c += al(2 * P * np * 4);
  S.fs_count = (int32_t *)c;     c += al(2 * P * (np / 128) * 4);
  S.desc16lo = nullptr; S.l3_rows = nullptr; S.l3_count = nullptr;
  if (n_max >= kL2MinNmax) {                                     // the level-2 pass (batched full scans only)
    S.desc16lo = (__half *)c;    c += al(F * np * kDim * 2);
    S.l3_rows = (int32_t *)c;    c += al(2 * P * np * 4);
    S.l3_count = (int32_t *)c;
    cudaMemset(S.l3_count, 0, 2 * P * 4);
  }
  // maxnorm and the queue counters are zero between calls: zeroed here, re-zeroed by k_mutual
  cudaMemset(S.maxnorm, 0, F * 4);
  cudaMemset(S.work_count, 0, 16);
  return S;
}

void launch_match(const KpView &kp, const int32_t *pairs, int P, float ratio, const MatchScratch &S,
                  const CUtensorMap *tmap, int force_fallback, int32_t *matches, int32_t *n_matches,
                  cudaStream_t s, Launch &L) {
  if (P <= 0) return;
  const int n_pad = match_n_pad(kp.n_max);
  const int rt_count = n_pad / 128;
  const int ibits = ceil_log2(n_pad);
  L.begin(K_DESC_PREP, s);
  constexpr int per_cta = kWarpsPerBlock * kPrepPerWarp;
  launch_pdl(k_desc_prep, dim3((n_pad + per_cta - 1) / per_cta, kp.n_frames), kWarpsPerBlock * 32, 0, s, kp, S,
             n_pad);
  L.end(K_DESC_PREP, s);
  L.begin(K_DESC_PREP, s);
  launch_pdl(k_desc_half, dim3((n_pad + per_cta - 1) / per_cta, kp.n_frames), kWarpsPerBlock * 32, 0, s, kp, S,
             n_pad);
  L.end(K_DESC_PREP, s);
  const float ratio2 = ratio >= 1.f ? 1.f : ratio * ratio;
  // batched full scans pay off when a row's scan reads >= 512 KB of references (n >= 1024);
  // below that the per-row queue (one CTA per row, 8 warps split the references) is faster
  const int fs_batched = kp.n_max >= kL2MinNmax ? 1 : 0;
  const int kshift = std::max(ibits, 9);
  TcArgs ta{kp, pairs, S, n_pad, ibits, P, force_fallback, ratio2, fs_batched, 1u << kshift, kshift,
            ldexpf(1.f, 9 - kshift), 0x3F800000u + (1u << (32 - kshift)) - 1u};
  const bool imad_keys = kshift <= 16 && !getenv("BT_MATCH_LOP3");   // BT_MATCH_LOP3: dev A/B of the key packing
  // four top-2 sets where the level-2 pass takes the rows they leave undecided (BT_MATCH_TOP3:
  // dev A/B against the exact top-3)
  const bool top2 = fs_batched && !getenv("BT_MATCH_TOP3");
  auto kws = imad_keys ? (top2 ? k_match_ws<true, true> : k_match_ws<true, false>)
                       : (top2 ? k_match_ws<false, true> : k_match_ws<false, false>);
  L.begin(K_MATCH_TC, s);
  // two CTAs per SM by design (2 x 108 KB of shared memory, 2 x 256 TMEM columns, 96 registers;
  // ncu: block limits 2 / 2); the occupancy API reports 1 for this configuration, so the grid
  // is sized directly (a CTA that does not fit only waits: no CTA depends on another)
  smem_optin((const void *)kws, kWsSmem);
  cudaFuncSetAttribute(kws, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  const int ws_grid = sm_count() * 2;
  launch_pdl(kws, std::min(ws_grid, 2 * P * rt_count), kWsThreads, kWsSmem, s, *tmap, ta);
  L.end(K_MATCH_TC, s);
  if (getenv("BT_MATCH_STATS") && fs_batched) {                   // dev aid (synchronizes): first-level outcome
    unsigned c0 = 0;
    cudaStreamSynchronize(s);
    cudaMemcpy(&c0, S.work_count, 4, cudaMemcpyDeviceToHost);
    std::vector<int32_t> fc(2 * P * rt_count);
    cudaMemcpy(fc.data(), S.fs_count, fc.size() * 4, cudaMemcpyDeviceToHost);
    long long t = 0;
    for (int v : fc) t += v;
    fprintf(stderr, "bt matching: first level left %u rows top-2, %lld rows undecided\n", c0, t);
  }
  L.begin(K_RESOLVE, s);
  RescoreArgs ra{kp, pairs, S, ibits, ratio2};
  if (fs_batched) {
    // level 2: tensor-core hi + lo re-ranking of the rows k_match_ws left undecided; what it
    // cannot certify goes to the exact batched scan
    L2Args la{kp, pairs, S, P, n_pad, (!force_fallback && ratio2 >= 1.f && n_pad <= 4096) ? 1 : 0};
    smem_optin((const void *)k_match_l2, kL2Smem);
    launch_pdl(k_match_l2, dim3(std::min(n_pad / kL2Rows, 4), P, 2), 128, kL2Smem, s, la);
    L.end(K_RESOLVE, s);
    L.begin(K_RESOLVE, s);
    FullScanArgs fa{kp, pairs, S, P, n_pad, ibits, ratio2};
    smem_optin((const void *)k_fullscan, kFsSmem);
    launch_pdl(k_fullscan, dim3(std::min(n_pad / kFsRows, 4), P, 2), 256, kFsSmem, s, fa);
    L.end(K_RESOLVE, s);
    L.begin(K_RESOLVE, s);
  }
  launch_pdl(k_rescore, dim3(2 * 148, 2), kWarpsPerBlock * 32, 0, s, ra);
  L.end(K_RESOLVE, s);
  if (getenv("BT_MATCH_STATS")) {                                 // dev aid (synchronizes): queue sizes
    unsigned c[2] = {0, 0};
    cudaStreamSynchronize(s);
    cudaMemcpy(c, S.work_count, 8, cudaMemcpyDeviceToHost);
    fprintf(stderr, "bt matching: %u rows top-2 rescored, %u rows full-scanned\n", c[0], c[1]);
    if (fs_batched && S.l3_count) {
      std::vector<int32_t> l3(2 * P);
      cudaMemcpy(l3.data(), S.l3_count, 2 * P * 4, cudaMemcpyDeviceToHost);
      long long t = 0;
      for (int v : l3) t += v;
      fprintf(stderr, "bt matching: %lld rows left to the exact batched scan after the level-2 pass\n", t);
    }
  }
  L.begin(K_MUTUAL, s);
  launch_pdl(k_mutual, P, 512, 0, s, kp, pairs, (const int32_t *)S.nn_ab, (const int32_t *)S.nn_ba,
             (const uint8_t *)S.ratio_ok, matches, n_matches, S);
  L.end(K_MUTUAL, s);
}

}  // namespace bt
