// bt_ransac.cu — RANSAC over 3-pair samples, best-hypothesis refit and the Eq. (2)
// feature-edge blocks.
//
//  k_ransac_hyp     per hypothesis: Philox4x32-10 (counter (h, uid, 0, 0), key = seed) ->
//                   distinct triple (reading R6) -> closed-form 3-point Arun in fp64
//                   (triangle frames + 2x2 Procrustes, reading R7) -> R, t in fp32, written to
//                   an L2-resident buffer in the scoring kernel's f32x2 pair layout.
//  k_ransac_score   balanced: the flat (pair, 512-hypothesis block, correspondence) work range
//                   is cut into one equal slice per resident CTA slot (no partial last wave).
//                   Two hypotheses per lane packed in f32x2 registers: every FMA of the
//                   distance gate (15 FMA-pipe ops) and normal gate (9) is one FFMA2 for both
//                   (sm_100a), the correspondence (staged in shared memory, 64 B each: p_a,
//                   -p_b, O = n_b n_a^T) a broadcast operand; the normal gate is skipped by a
//                   warp vote when no lane's distance gate passes; counts are integer atomics.
//  k_ransac_finish  one CTA per pair: best key ((count+1) << 32 | ~h) over the counts — max
//                   count, ties -> lowest h (R11) — reads T of h* from the hypothesis buffer,
//                   inlier mask by ballot, refit by fp64 cross-covariance + Jacobi SVD with
//                   the det fix (north star, R12), status, and — when node poses are given —
//                   the Eq. (2) J^T W J blocks at those poses in fp64, reduced in a fixed order.
#include <cuda_runtime.h>
#include <math_constants.h>

#include <algorithm>
#include <climits>
#include <cstdio>
#include <cmath>
#include <cstdlib>

#include "bt_internal.cuh"
#include "bt_tc.cuh"

#ifndef BT_TC_EPI_WARPS
#define BT_TC_EPI_WARPS 8
#endif

namespace bt {
namespace {

constexpr int kScoreThreads = 256;
constexpr int kHypPerThread = 2;
constexpr int kHypPerBlock = kScoreThreads * kHypPerThread;
constexpr int kMaxChunk = 512;            // correspondences staged per smem pass (32 KB)

// ---------------------------------------------------------------- Philox4x32-10
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
    const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
    c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}

// distinct ordered triple in [0, M): floor(r * n / 2^32) with skips (R6)
__device__ __forceinline__ void sample_triple(uint4 r, int M, int &i0, int &i1, int &i2) {
  const uint32_t a = __umulhi(r.x, (uint32_t)M);
  uint32_t b = __umulhi(r.y, (uint32_t)(M - 1));
  if (b >= a) ++b;
  uint32_t c = __umulhi(r.z, (uint32_t)(M - 2));
  const uint32_t lo = min(a, b), hi = max(a, b);
  if (c >= lo) ++c;
  if (c >= hi) ++c;
  i0 = (int)a; i1 = (int)b; i2 = (int)c;
}

// ---------------------------------------------------------------- fp64 3-point Arun
// Every fp64 operation is an explicit _rn intrinsic, so the (inlined) solver yields the same
// bits in the scoring and the finish kernel whatever the compiler contracts around it.
struct d3 { double x, y, z; };
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dfma(double a, double b, double c) { return __fma_rn(a, b, c); }
__device__ __forceinline__ d3 vsub(d3 a, d3 b) { return {dsub(a.x, b.x), dsub(a.y, b.y), dsub(a.z, b.z)}; }
__device__ __forceinline__ d3 vscale(d3 a, double s) { return {dmul(a.x, s), dmul(a.y, s), dmul(a.z, s)}; }
__device__ __forceinline__ double vdot(d3 a, d3 b) { return dfma(a.x, b.x, dfma(a.y, b.y, dmul(a.z, b.z))); }
__device__ __forceinline__ d3 vcross(d3 a, d3 b) {
  return {dfma(a.y, b.z, -dmul(a.z, b.y)), dfma(a.z, b.x, -dmul(a.x, b.z)), dfma(a.x, b.y, -dmul(a.y, b.x))};
}

// R, t minimising sum_k |R a_k + t - b_k|^2 for three correspondences.  Centred points of a
// triangle lie in its plane: in orthonormal in-plane frames (e1, e2) / (f1, f2) the
// cross-covariance is E_a M E_b^T with the 2x2 M = sum alpha_k beta_k^T, so its singular
// values are those of M: s1,2 = (p +- q)/2 with p = |(m00+m11, m01-m10)|,
// q = |(m00-m11, m01+m10)|.  The optimal proper rotation maps n_a -> +n_b with an in-plane
// rotation (value p) or n_a -> -n_b with an in-plane reflection (value q); the larger wins.
// Degenerate (false) when s2/s1 < tau (R8) — tested as (p - q)^2 < tau^2 (p + q)^2 — or for a
// collinear / coincident triangle.
__device__ __forceinline__ bool solve3(const float *A, const float *B, double tau, float *out) {
  const d3 a0 = {A[0], A[1], A[2]}, a1 = {A[3], A[4], A[5]}, a2 = {A[6], A[7], A[8]};
  const d3 b0 = {B[0], B[1], B[2]}, b1 = {B[3], B[4], B[5]}, b2 = {B[6], B[7], B[8]};
  const double third = 1.0 / 3.0;
  const d3 ac = vscale({dadd(dadd(a0.x, a1.x), a2.x), dadd(dadd(a0.y, a1.y), a2.y), dadd(dadd(a0.z, a1.z), a2.z)}, third);
  const d3 bc = vscale({dadd(dadd(b0.x, b1.x), b2.x), dadd(dadd(b0.y, b1.y), b2.y), dadd(dadd(b0.z, b1.z), b2.z)}, third);
  const d3 ua = vsub(a1, a0), ub = vsub(b1, b0);
  const d3 na = vcross(ua, vsub(a2, a0)), nb = vcross(ub, vsub(b2, b0));
  const double lua = vdot(ua, ua), lub = vdot(ub, ub), lna = vdot(na, na), lnb = vdot(nb, nb);
  if (!(lua > 0.0) || !(lub > 0.0) || !(lna > 0.0) || !(lnb > 0.0)) return false;
  const d3 e1 = vscale(ua, rsqrt(lua)), n = vscale(na, rsqrt(lna)), e2 = vcross(n, e1);
  const d3 f1 = vscale(ub, rsqrt(lub)), m = vscale(nb, rsqrt(lnb)), f2 = vcross(m, f1);
  double m00 = 0, m01 = 0, m10 = 0, m11 = 0;
  const d3 as[3] = {vsub(a0, ac), vsub(a1, ac), vsub(a2, ac)};
  const d3 bs[3] = {vsub(b0, bc), vsub(b1, bc), vsub(b2, bc)};
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double x0 = vdot(e1, as[k]), x1 = vdot(e2, as[k]);
    const double y0 = vdot(f1, bs[k]), y1 = vdot(f2, bs[k]);
    m00 = dfma(x0, y0, m00); m01 = dfma(x0, y1, m01); m10 = dfma(x1, y0, m10); m11 = dfma(x1, y1, m11);
  }
  const double pr = dadd(m00, m11), pi = dsub(m01, m10), qr = dsub(m00, m11), qi = dadd(m01, m10);
  const double P2 = dfma(pr, pr, dmul(pi, pi)), Q2 = dfma(qr, qr, dmul(qi, qi));
  const double PQ = __dsqrt_rn(dmul(P2, Q2));
  const double sum2 = dadd(P2, Q2);                              // (p +- q)^2 = P2 + Q2 +- 2 PQ
  if (!(sum2 > 0.0) || dsub(sum2, dmul(2.0, PQ)) < dmul(dmul(tau, tau), dadd(sum2, dmul(2.0, PQ)))) return false;
  double q00, q01, q10, q11, sg;
  if (P2 >= Q2) {                                                // rotation branch, R n_a = n_b
    const double ip = rsqrt(P2), c = dmul(pr, ip), s = dmul(pi, ip);
    q00 = c; q01 = -s; q10 = s; q11 = c; sg = 1.0;
  } else {                                                       // reflection branch, R n_a = -n_b
    const double iq = rsqrt(Q2), c = dmul(qr, iq), s = dmul(qi, iq);
    q00 = c; q01 = s; q10 = s; q11 = -c; sg = -1.0;
  }
  // R = [f1 f2 m] diag(Q, sg) [e1 e2 n]^T
  const d3 c0 = {dfma(q00, f1.x, dmul(q10, f2.x)), dfma(q00, f1.y, dmul(q10, f2.y)), dfma(q00, f1.z, dmul(q10, f2.z))};
  const d3 c1 = {dfma(q01, f1.x, dmul(q11, f2.x)), dfma(q01, f1.y, dmul(q11, f2.y)), dfma(q01, f1.z, dmul(q11, f2.z))};
  const d3 c2 = vscale(m, sg);
  const double cx[3] = {c0.x, c0.y, c0.z}, cy[3] = {c1.x, c1.y, c1.z}, cz[3] = {c2.x, c2.y, c2.z};
  const double ex[3] = {e1.x, e1.y, e1.z}, ey[3] = {e2.x, e2.y, e2.z}, ez[3] = {n.x, n.y, n.z};
  double R[9];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) R[3 * r + c] = dfma(cx[r], ex[c], dfma(cy[r], ey[c], dmul(cz[r], ez[c])));
#pragma unroll
  for (int k = 0; k < 9; ++k) out[k] = __double2float_rn(R[k]);
  out[9] = __double2float_rn(dsub(bc.x, dfma(R[0], ac.x, dfma(R[1], ac.y, dmul(R[2], ac.z)))));
  out[10] = __double2float_rn(dsub(bc.y, dfma(R[3], ac.x, dfma(R[4], ac.y, dmul(R[5], ac.z)))));
  out[11] = __double2float_rn(dsub(bc.z, dfma(R[6], ac.x, dfma(R[7], ac.y, dmul(R[8], ac.z)))));
  return true;
}

// solve hypothesis h of a pair from its matched points staged as sab[m] = (a_m, b_m)
__device__ __forceinline__ bool make_hypothesis_staged(int h, uint32_t uid, uint32_t k0, uint32_t k1, int M,
                                                       const float *sab, double tau, float *out) {
  const uint4 r = philox4x32_10(make_uint4((uint32_t)h, uid, 0u, 0u), k0, k1);
  int s[3];
  sample_triple(r, M, s[0], s[1], s[2]);
  float A[9], B[9];
#pragma unroll
  for (int k = 0; k < 3; ++k)
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      A[3 * k + c] = sab[6 * s[k] + c];
      B[3 * k + c] = sab[6 * s[k] + 3 + c];
    }
  return solve3(A, B, tau, out);
}


// ---------------------------------------------------------------- the inlier test
// Correspondence m as four float4: q0 = (ax, ay, az, -bx), q1 = (-by, -bz, O00, O01),
// q2 = (O02, O10, O11, O12), q3 = (O20, O21, O22, 0) with O = n_b n_a^T, so that
// (R n_a) . n_b = <R, O>_F.  The gates are folded into the FMA chains:
//   d' = |R a + t - b|^2 - delta^2  (< 0: distance gate, 15 FMA-pipe ops),
//   c' = <R, O> - cos(alpha)        (> 0: normal gate, 9 FFMA).
// x + (-b) is x - b exactly.  Explicit _rn intrinsics: the scoring kernel (packed f32x2, one
// IEEE fma.rn per lane) and the finish kernel (scalar) compute identical bits.
__device__ __forceinline__ float dist_term(const float *T, const float4 q0, const float4 q1, float ndelta2) {
  const float ex = __fadd_rn(__fmaf_rn(T[0], q0.x, __fmaf_rn(T[1], q0.y, __fmaf_rn(T[2], q0.z, T[9]))), q0.w);
  const float ey = __fadd_rn(__fmaf_rn(T[3], q0.x, __fmaf_rn(T[4], q0.y, __fmaf_rn(T[5], q0.z, T[10]))), q1.x);
  const float ez = __fadd_rn(__fmaf_rn(T[6], q0.x, __fmaf_rn(T[7], q0.y, __fmaf_rn(T[8], q0.z, T[11]))), q1.y);
  return __fmaf_rn(ex, ex, __fmaf_rn(ey, ey, __fmaf_rn(ez, ez, ndelta2)));
}
__device__ __forceinline__ float normal_term(const float *T, const float4 q1, const float4 q2, const float4 q3,
                                             float ncosa) {
  float c = __fmaf_rn(T[0], q1.z, ncosa);
  c = __fmaf_rn(T[1], q1.w, c);
  c = __fmaf_rn(T[2], q2.x, c);
  c = __fmaf_rn(T[3], q2.y, c);
  c = __fmaf_rn(T[4], q2.z, c);
  c = __fmaf_rn(T[5], q2.w, c);
  c = __fmaf_rn(T[6], q3.x, c);
  c = __fmaf_rn(T[7], q3.y, c);
  c = __fmaf_rn(T[8], q3.z, c);
  return c;
}
// inlier <=> sign(d') = 1 and sign(c') = 0 (differs from d' < 0 && c' > 0 only at exact
// ties d' = -0 / c' = +0, which the band rule leaves undecided); both kernels use it
__device__ __forceinline__ unsigned pass_bit(float d, float c) {
  return (__float_as_uint(d) & ~__float_as_uint(c)) >> 31;
}
__device__ __forceinline__ bool inlier(const float *T, const float4 q0, const float4 q1, const float4 q2,
                                       const float4 q3, float ndelta2, float ncosa) {
  return pass_bit(dist_term(T, q0, q1, ndelta2), normal_term(T, q1, q2, q3, ncosa)) != 0u;
}

// ---- packed fp32x2 (sm_100a FFMA2 / FADD2): lane .x = hypothesis 0, .y = hypothesis 1 of a
// thread; a correspondence scalar is a broadcast operand (no extra instruction in SASS)
typedef unsigned long long f32x2;
__device__ __forceinline__ f32x2 pk(float lo, float hi) {
  f32x2 d;
  asm("mov.b64 %0, {%1, %2};" : "=l"(d) : "f"(lo), "f"(hi));
  return d;
}
__device__ __forceinline__ f32x2 fma2(f32x2 a, float b, f32x2 c) {      // a * {b, b} + c
  f32x2 d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(pk(b, b)), "l"(c));
  return d;
}
__device__ __forceinline__ f32x2 fma2v(f32x2 a, f32x2 b, f32x2 c) {
  f32x2 d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ f32x2 add2(f32x2 a, float b) {               // a + {b, b}
  f32x2 d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(pk(b, b)));
  return d;
}
__device__ __forceinline__ void split(f32x2 x, unsigned &lo, unsigned &hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=r"(lo), "=r"(hi) : "l"(x));
}
// the scalar dist_term / normal_term, op for op, on both hypotheses of a thread
__device__ __forceinline__ f32x2 dist_term2(const f32x2 *T, const float4 q0, const float4 q1, f32x2 nd2) {
  const f32x2 ex = add2(fma2(T[0], q0.x, fma2(T[1], q0.y, fma2(T[2], q0.z, T[9]))), q0.w);
  const f32x2 ey = add2(fma2(T[3], q0.x, fma2(T[4], q0.y, fma2(T[5], q0.z, T[10]))), q1.x);
  const f32x2 ez = add2(fma2(T[6], q0.x, fma2(T[7], q0.y, fma2(T[8], q0.z, T[11]))), q1.y);
  return fma2v(ex, ex, fma2v(ey, ey, fma2v(ez, ez, nd2)));
}
__device__ __forceinline__ f32x2 normal_term2(const f32x2 *T, const float4 q1, const float4 q2, const float4 q3,
                                              f32x2 nc2) {
  f32x2 c = fma2(T[0], q1.z, nc2);
  c = fma2(T[1], q1.w, c);
  c = fma2(T[2], q2.x, c);
  c = fma2(T[3], q2.y, c);
  c = fma2(T[4], q2.z, c);
  c = fma2(T[5], q2.w, c);
  c = fma2(T[6], q3.x, c);
  c = fma2(T[7], q3.y, c);
  c = fma2(T[8], q3.z, c);
  return c;
}

__device__ __forceinline__ void pack_corr(const float *pa, const float *na, const float *pb,
                                          const float *nb, float4 &q0, float4 &q1, float4 &q2,
                                          float4 &q3) {
  q0 = make_float4(pa[0], pa[1], pa[2], -pb[0]);
  q1 = make_float4(-pb[1], -pb[2], __fmul_rn(nb[0], na[0]), __fmul_rn(nb[0], na[1]));
  q2 = make_float4(__fmul_rn(nb[0], na[2]), __fmul_rn(nb[1], na[0]), __fmul_rn(nb[1], na[1]),
                   __fmul_rn(nb[1], na[2]));
  q3 = make_float4(__fmul_rn(nb[2], na[0]), __fmul_rn(nb[2], na[1]), __fmul_rn(nb[2], na[2]), 0.f);
}

struct ScoreArgs {
  KpView kp;
  const int32_t *pairs;
  const uint32_t *uid;
  const int32_t *matches;
  const int32_t *n_matches;
  int P, n_hyp, nb, chunk;
  uint32_t k0, k1;
  float ndelta2, ncosa;
  double tau;
  f32x2 *hyp;                  // [P][nb][12][kScoreThreads]: T (R row-major, t) of hypotheses
                               // (b*512 + t, b*512 + 256 + t) packed per thread; never-passing
                               // sentinel when degenerate or h >= n_hyp
  int32_t *counts;             // [P][n_hyp] inlier counts (accumulated); < 0 => degenerate
  int32_t *work;               // slice counter of the scoring kernel (zeroed by k_ransac_hyp)
  int slices;                  // slices the scoring work is cut into (grabbed dynamically)
};

// One thread per hypothesis: Philox4x32-10 (counter (h, uid, 0, 0), key = seed) -> distinct
// triple (R6) -> closed-form 3-point Arun in fp64 (R7) -> R, t rounded to fp32, written to the
// L2-resident hypothesis buffer in the scoring kernel's f32x2 pair layout; the count is
// initialised to 0, or to a very negative value when degenerate (it stays < 0 whatever the
// scoring adds — degenerate hypotheses never pass the distance gate anyway).
constexpr int kHypThreads = 256;
#ifndef BT_HYP_ITER
#define BT_HYP_ITER 8
#endif
constexpr int kHypIter = BT_HYP_ITER;                             // hypotheses per thread (loop)

// One CTA = kHypThreads x kHypIter hypotheses of one pair.  The pair's matched points are first
// staged in shared memory (match list, then a_m / b_m), then one thread per hypothesis per
// iteration: Philox4x32-10 (counter (h, uid, 0, 0), key = seed) -> distinct triple (R6) ->
// closed-form 3-point Arun in fp64 (R7) -> R, t rounded to fp32, written to the L2-resident
// hypothesis buffer in the scoring kernel's f32x2 pair layout.  The count is initialised to 0,
// or to a very negative value when degenerate (it stays < 0 whatever the scoring adds).
__global__ void __launch_bounds__(kHypThreads) k_ransac_hyp(ScoreArgs A) {
  pdl_wait();
  extern __shared__ float sab[];                                  // [M][6] = (a_m, b_m)
  const int p = blockIdx.y;
  if ((blockIdx.x | blockIdx.y | threadIdx.x) == 0) *A.work = 0;   // the previous score kernel is done
  const int M = A.n_matches[p];
  if (M < 3) return;
  const int fa = A.pairs[2 * p], fb = A.pairs[2 * p + 1];
  const int32_t *mt = A.matches + (size_t)p * A.kp.n_max * 2;
  const float *pa_f = A.kp.pts + (size_t)fa * A.kp.n_max * 3, *pb_f = A.kp.pts + (size_t)fb * A.kp.n_max * 3;
  const uint32_t uid = A.uid[p];
  for (int x = threadIdx.x; x < 2 * M; x += kHypThreads) {
    const int m = x >> 1, side = x & 1;
    const float *src = (side ? pb_f : pa_f) + 3 * mt[x];
    sab[6 * m + 3 * side] = src[0];
    sab[6 * m + 3 * side + 1] = src[1];
    sab[6 * m + 3 * side + 2] = src[2];
  }
  __syncthreads();
#pragma unroll 1
  for (int it = 0; it < kHypIter; ++it) {
    const int h = (blockIdx.x * kHypIter + it) * kHypThreads + threadIdx.x;
    if (h >= A.nb * kHypPerBlock) break;                           // past the pair's slots
    float T[12];
    bool v = false;
    if (h < A.n_hyp) {
      v = make_hypothesis_staged(h, uid, A.k0, A.k1, M, sab, A.tau, T);
      A.counts[(size_t)p * A.n_hyp + h] = v ? 0 : INT_MIN / 2;
    }
    if (!v) {                                                      // never passes the distance gate
#pragma unroll
      for (int q = 0; q < 12; ++q) T[q] = 0.f;
      T[11] = 3.0e38f;
    }
    const int b = h / kHypPerBlock, r = h - b * kHypPerBlock;
    const int t = r % kScoreThreads, k = r / kScoreThreads;
    float *dst = reinterpret_cast<float *>(A.hyp + ((size_t)p * A.nb + b) * 12 * kScoreThreads + t) + k;
#pragma unroll
    for (int q = 0; q < 12; ++q) dst[2 * q * kScoreThreads] = T[q];
  }
}

constexpr int kPlanChunk = kScoreThreads;
// slices of the scoring work per resident CTA slot (grabbed dynamically; 2 measured best of
// 1/2/3/4/8/16 on C2 — tools/sweep history in DESIGN.md)
constexpr int kScoreSlicesPerSlot = 2;                         // pairs per prefix chunk

// exclusive prefix of the scoring work W_q = nb * M_q (M_q >= 3) over pairs [c0, c0 + 256),
// offset by carry: cpre[k] for pair c0 + k, cpre[256] = end of the chunk (CTA-uniform call)
__device__ void plan_chunk(const ScoreArgs &A, int c0, long long carry, long long *cpre, long long *wsum) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int q = c0 + threadIdx.x;
  const int Mq = q < A.P ? A.n_matches[q] : 0;
  const long long w = Mq >= 3 ? (long long)A.nb * Mq : 0;
  long long incl = w;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long long y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  __syncthreads();                                                 // previous chunk fully read
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  long long woff = 0, tot = 0;
#pragma unroll
  for (int w2 = 0; w2 < kScoreThreads / 32; ++w2) { woff += w2 < warp ? wsum[w2] : 0; tot += wsum[w2]; }
  cpre[threadIdx.x] = carry + woff + incl - w;
  if (threadIdx.x == 0) cpre[kPlanChunk] = carry + tot;
  __syncthreads();
}

// Balanced scoring.  The work of all pairs — (pair p, block b of kHypPerBlock hypotheses,
// correspondence m) steps, W_p = nb * M_p — is one flat range cut into A.slices equal slices
// that the CTAs grab from a counter, so the tests spread evenly whatever the pairs' match
// counts and however many SMs the concurrent dense stream leaves free.  A slice crosses segment
// boundaries.  Per segment the CTA loads its 512 hypotheses (two per thread, coalesced 8-B f32x2
// loads), stages the segment's correspondences in shared memory (AoS, 64 B each, read as warp
// broadcasts) and scores with packed f32x2 FMAs (both hypotheses of a thread in one FFMA2; a
// correspondence scalar is a broadcast operand).  Per correspondence a warp vote skips the
// normal gate when no lane's distance gate passes.  Counts are added with integer atomics
// (exact, order-independent).
__global__ void __launch_bounds__(kScoreThreads, 3) k_ransac_score(ScoreArgs A) {
  pdl_wait();
  extern __shared__ float4 sq[];                                  // [chunk][4] correspondences
  __shared__ long long cpre[kPlanChunk + 1];
  __shared__ long long wsum[kScoreThreads / 32];
  __shared__ int s_slice;
  const int H = A.n_hyp;
  // total work: prefix over all pairs, chunk by chunk (one chunk for P <= 256)
  long long total = 0;
  int c0 = 0;
  for (int c = 0; c < A.P; c += kPlanChunk) {
    plan_chunk(A, c, total, cpre, wsum);
    total = cpre[kPlanChunk];
    c0 = c;
  }
  bool fresh = true;                                               // cpre holds the last chunk
  for (;;) {
    if (threadIdx.x == 0) s_slice = atomicAdd(A.work, 1);
    __syncthreads();
    const int sl = s_slice;
    __syncthreads();
    if (sl >= A.slices) break;                                       // CTA-uniform
    const long long lo0 = total * sl / A.slices, hi = total * (sl + 1) / A.slices;
    if (lo0 >= hi) continue;
    if (A.P > kPlanChunk && (fresh || cpre[0] > lo0)) {              // re-plan from the chunk holding lo0
      long long carry = 0;
      for (c0 = 0;; c0 += kPlanChunk) {
        plan_chunk(A, c0, carry, cpre, wsum);
        if (cpre[kPlanChunk] > lo0 || c0 + kPlanChunk >= A.P) break;
        carry = cpre[kPlanChunk];
      }
    } else if (A.P > kPlanChunk) {                                   // slices ascend: step forward
      while (cpre[kPlanChunk] <= lo0 && c0 + kPlanChunk < A.P) {
        const long long carry = cpre[kPlanChunk];
        c0 += kPlanChunk;
        plan_chunk(A, c0, carry, cpre, wsum);
      }
    }
    fresh = false;
    int p;
    {
      int a = 0, b = min(kPlanChunk, A.P - c0);                      // cpre[a] <= lo0 < cpre[b]
      while (b - a > 1) { const int mid = (a + b) >> 1; if (cpre[mid] <= lo0) a = mid; else b = mid; }
      p = c0 + a;
    }
    long long lo = lo0;
    while (lo < hi) {
      for (;;) {                                                     // skip pairs without work
        if (p - c0 >= kPlanChunk) {
          const long long carry = cpre[kPlanChunk];
          c0 += kPlanChunk;
          plan_chunk(A, c0, carry, cpre, wsum);
        }
        const long long end_p = p + 1 - c0 < kPlanChunk ? cpre[p + 1 - c0] : cpre[kPlanChunk];
        if (end_p > lo) break;
        ++p;
      }
      const int M = A.n_matches[p];
      const long long rel = lo - cpre[p - c0];
      const int b = (int)(rel / M), m0 = (int)(rel - (long long)b * M);
      const int m1 = (int)min((long long)M, m0 + (hi - lo));
      const int fa = A.pairs[2 * p], fb = A.pairs[2 * p + 1];
      const int32_t *mt = A.matches + (size_t)p * A.kp.n_max * 2;
      const float *pa_f = A.kp.pts + (size_t)fa * A.kp.n_max * 3, *pb_f = A.kp.pts + (size_t)fb * A.kp.n_max * 3;
      const float *na_f = A.kp.nrm + (size_t)fa * A.kp.n_max * 3, *nb_f = A.kp.nrm + (size_t)fb * A.kp.n_max * 3;
      static_assert(kHypPerThread == 2, "packed f32x2 scoring holds two hypotheses per thread");
      f32x2 T2[12];                                                  // coalesced 8-B loads, L2-resident
      {
        const f32x2 *src = A.hyp + ((size_t)p * A.nb + b) * 12 * kScoreThreads + threadIdx.x;
#pragma unroll
        for (int q = 0; q < 12; ++q) T2[q] = __ldcg(src + q * kScoreThreads);
      }
      const f32x2 nd2 = pk(A.ndelta2, A.ndelta2), nc2 = pk(A.ncosa, A.ncosa);
      unsigned cnt[kHypPerThread];
#pragma unroll
      for (int k = 0; k < kHypPerThread; ++k) cnt[k] = 0u;
      for (int cs = m0; cs < m1; cs += A.chunk) {
        const int len = min(A.chunk, m1 - cs);
        __syncthreads();
        for (int k = threadIdx.x; k < len; k += kScoreThreads) {
          const int i = mt[2 * (cs + k)], j = mt[2 * (cs + k) + 1];
          float4 q0, q1, q2, q3;
          pack_corr(pa_f + 3 * i, na_f + 3 * i, pb_f + 3 * j, nb_f + 3 * j, q0, q1, q2, q3);
          sq[4 * k] = q0; sq[4 * k + 1] = q1; sq[4 * k + 2] = q2; sq[4 * k + 3] = q3;
        }
        __syncthreads();
#pragma unroll 2
        for (int m = 0; m < len; ++m) {
          const float4 q0 = sq[4 * m], q1 = sq[4 * m + 1];
          const f32x2 d = dist_term2(T2, q0, q1, nd2);
          unsigned d0, d1;
          split(d, d0, d1);
          if (__any_sync(0xffffffffu, (int)(d0 | d1) < 0)) {
            const float4 q2 = sq[4 * m + 2], q3 = sq[4 * m + 3];
            unsigned c0_, c1_;
            split(normal_term2(T2, q1, q2, q3, nc2), c0_, c1_);
            cnt[0] += (d0 & ~c0_) >> 31;
            cnt[1] += (d1 & ~c1_) >> 31;
          }
        }
      }
#pragma unroll
      for (int k = 0; k < kHypPerThread; ++k) {
        const int h = b * kHypPerBlock + k * kScoreThreads + threadIdx.x;
        if (h < H && cnt[k]) atomicAdd(A.counts + (size_t)p * H + h, (int)cnt[k]);
      }
      lo += m1 - m0;
    }
  }
}

// ---------------------------------------------------------------- finish: refit + Eq. (2)
// one-sided Jacobi SVD of a 3x3 (fp64): A = U diag(s) V^T, s descending
__device__ void svd3_jacobi(const double *Ain, double *U, double *s, double *V) {
  double a[9], v[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
  for (int k = 0; k < 9; ++k) a[k] = Ain[k];
  for (int sweep = 0; sweep < 60; ++sweep) {
    bool rot = false;
    for (int pq = 0; pq < 3; ++pq) {
      const int p = pq == 2 ? 1 : 0, q = pq == 0 ? 1 : 2;
      double al = 0, be = 0, ga = 0;
      for (int r = 0; r < 3; ++r) {
        al += a[3 * r + p] * a[3 * r + p];
        be += a[3 * r + q] * a[3 * r + q];
        ga += a[3 * r + p] * a[3 * r + q];
      }
      // the off-diagonal test squared (no sqrt) and c by one rsqrt: a shorter fp64 latency chain
      // on the refit's single thread (k_ransac_finish 18.2 -> 16.9 us standalone at C2)
      if (ga == 0.0 || ga * ga <= 4.930380657631324e-32 * (al * be)) continue;
      rot = true;
      const double z = (be - al) / (2.0 * ga);
      const double t = (z >= 0 ? 1.0 : -1.0) / (fabs(z) + sqrt(fma(z, z, 1.0)));
      const double c = rsqrt(fma(t, t, 1.0)), sn = c * t;
      for (int r = 0; r < 3; ++r) {
        const double x = a[3 * r + p], y = a[3 * r + q];
        a[3 * r + p] = c * x - sn * y;
        a[3 * r + q] = sn * x + c * y;
        const double vx = v[3 * r + p], vy = v[3 * r + q];
        v[3 * r + p] = c * vx - sn * vy;
        v[3 * r + q] = sn * vx + c * vy;
      }
    }
    if (!rot) break;
  }
  double sv[3];
  int o[3] = {0, 1, 2};
  for (int k = 0; k < 3; ++k) sv[k] = sqrt(a[k] * a[k] + a[3 + k] * a[3 + k] + a[6 + k] * a[6 + k]);
  for (int i = 0; i < 3; ++i)
    for (int j = i + 1; j < 3; ++j)
      if (sv[o[j]] > sv[o[i]]) { const int t = o[i]; o[i] = o[j]; o[j] = t; }
  for (int k = 0; k < 3; ++k) {
    s[k] = sv[o[k]];
    for (int r = 0; r < 3; ++r) V[3 * r + k] = v[3 * r + o[k]];
  }
  const double tiny = 1e-300 + s[0] * 1e-15;
  for (int k = 0; k < 2; ++k) {
    if (s[k] > tiny) {
      for (int r = 0; r < 3; ++r) U[3 * r + k] = a[3 * r + o[k]] / s[k];
    } else {                                  // rank <= k: any orthonormal completion
      double e[3] = {0, 0, 0};
      int ax = 0;
      double best = 2.0;
      for (int r = 0; r < 3; ++r) {
        const double c = k > 0 ? fabs(U[3 * r]) : 0.0;
        if (c < best) { best = c; ax = r; }
      }
      e[ax] = 1.0;
      for (int j = 0; j < k; ++j) {
        const double d = e[0] * U[j] + e[1] * U[3 + j] + e[2] * U[6 + j];
        for (int r = 0; r < 3; ++r) e[r] -= d * U[3 * r + j];
      }
      const double nr = sqrt(e[0] * e[0] + e[1] * e[1] + e[2] * e[2]);
      for (int r = 0; r < 3; ++r) U[3 * r + k] = e[r] / nr;
    }
  }
  U[2] = U[3] * U[7] - U[6] * U[4];           // u3 = u1 x u2 (sign is fixed by the det fix)
  U[5] = U[6] * U[1] - U[0] * U[7];
  U[8] = U[0] * U[4] - U[3] * U[1];
}

__device__ __forceinline__ double det3(const double *M) {
  return M[0] * (M[4] * M[8] - M[5] * M[7]) - M[1] * (M[3] * M[8] - M[5] * M[6]) +
         M[2] * (M[3] * M[7] - M[4] * M[6]);
}

// fixed-order block sums of N doubles (256 threads; results valid in every thread)
template <int N>
__device__ void block_sum_n(double (&v)[N], double *red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < N; ++k)
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
  __syncthreads();
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < N; ++k) red[warp * N + k] = v[k];
  __syncthreads();
  // lane k of warp 0 sums value k over the warps (the same order as before: w = 0, 1, ...)
  // and every thread then reads the N totals — instead of every thread summing all of them
  const int nw = (int)(blockDim.x >> 5);
  if (warp == 0 && lane < N) {
    double t = 0.0;
    for (int w = 0; w < nw; ++w) t += red[w * N + lane];
    red[nw * N + lane] = t;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < N; ++k) v[k] = red[nw * N + k];
}

struct FinishArgs {
  KpView kp;
  const int32_t *pairs;
  const uint32_t *uid;
  const int32_t *matches;
  const int32_t *n_matches;
  int n_hyp, min_inliers;
  uint32_t k0, k1;
  float ndelta2, ncosa;
  double tau;
  const int32_t *counts;         // [P][n_hyp] from k_ransac_score (< 0: degenerate)
  const f32x2 *hyp;              // hypothesis buffer of k_ransac_hyp (same bits as a re-solve)
  int nb;
  int32_t *hyp_counts;           // optional [P][n_hyp] output (-1: degenerate / no samples)
  uint32_t *records;
  int rec_stride;
  const bt_pose *node_pose;      // null: no feature blocks
  double huber;
  PeerRec peers;                 // NEXT-3: the record words also go to the peers' gather buffers
};

constexpr int kFinThreads = 256;
constexpr int kFeatChunk = 512;                  // feature rows staged per pass (smem)
// per-inlier feature data staged in smem: e(3) J(3x12) w rho
constexpr int kFeatRow = 3 * 13 + 2;             // per residual component q: J_q (12), e_q; w; rho

// Eq. (2) feature-edge blocks of one pair at the node poses, all kFinThreads threads.
// inl[0 .. n_feat) = the inlier match indices in ascending order (C_ij), frow: smem rows.
__device__ void feature_blocks(const int *inl, int n_feat, const int32_t *mt, const float *pa_f, const float *pb_f,
                               const bt_pose &Pi, const bt_pose &Pj, double huber, float *frow,
                               float (*fpart)[96], uint32_t *feat_out, const PeerRec *pr = nullptr, int pp = 0,
                               int pw = 0) {
  // e = R_i^T (p_m - t_i) - R_j^T (p_n - t_j) (fp64: it cancels ~0.5 m coordinates);
  // J_i = -R_i^T [I | -[p_m]x], J_j = R_j^T [I | -[p_n]x];  H += w J^T J, g += w J^T e,
  // E += rho(|e|).  Every thread builds rows (fp32 after the fp64 residual) into smem; warp w
  // accumulates rows w, w + 8, ... for outputs lane, lane + 32, lane + 64; a fixed-order
  // combine over the 8 warps keeps the result bitwise deterministic.
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double Ri[9], ti[3], Rj[9], tj[3];
  for (int k = 0; k < 9; ++k) { Ri[k] = Pi.R[k]; Rj[k] = Pj.R[k]; }
  for (int k = 0; k < 3; ++k) { ti[k] = Pi.t[k]; tj[k] = Pj.t[k]; }
  // the three outputs of this lane: kind 0 H(a,b), 1 g(a), 2 E, 3 count, -1 none
  int okind[3], oa[3], ob[3];
#pragma unroll
  for (int s = 0; s < 3; ++s) {
    int k = lane + 32 * s;
    okind[s] = -1; oa[s] = ob[s] = 0;
    if (k < 21) {                      // H_ii upper
      int a = 0;
      while (k >= 6 - a) { k -= 6 - a; ++a; }
      oa[s] = a; ob[s] = a + k; okind[s] = 0;
    } else if (k < 57) {               // H_ij
      k -= 21; oa[s] = k / 6; ob[s] = 6 + k % 6; okind[s] = 0;
    } else if (k < 78) {               // H_jj upper
      k -= 57;
      int a = 0;
      while (k >= 6 - a) { k -= 6 - a; ++a; }
      oa[s] = 6 + a; ob[s] = 6 + a + k; okind[s] = 0;
    } else if (k < 90) { oa[s] = k - 78; ob[s] = 12; okind[s] = 1; }
    else if (k == 90) okind[s] = 2;
    else if (k == 91) okind[s] = 3;
  }
  float acc[3] = {0.f, 0.f, 0.f};
  for (int done = 0; done < n_feat; done += kFeatChunk) {
    const int nc = min(kFeatChunk, n_feat - done);
    __syncthreads();
    for (int r = tid; r < nc; r += kFinThreads) {
      const int m = inl[done + r];
      const int i = mt[2 * m], j = mt[2 * m + 1];
      const double pm[3] = {pa_f[3 * i], pa_f[3 * i + 1], pa_f[3 * i + 2]};
      const double pn[3] = {pb_f[3 * j], pb_f[3 * j + 1], pb_f[3 * j + 2]};
      float *row = frow + r * kFeatRow;
      double e[3];
#pragma unroll
      for (int q = 0; q < 3; ++q)
        e[q] = Ri[q] * (pm[0] - ti[0]) + Ri[3 + q] * (pm[1] - ti[1]) + Ri[6 + q] * (pm[2] - ti[2]) -
               (Rj[q] * (pn[0] - tj[0]) + Rj[3 + q] * (pn[1] - tj[1]) + Rj[6 + q] * (pn[2] - tj[2]));
      const double Sp[9] = {0, -pm[2], pm[1], pm[2], 0, -pm[0], -pm[1], pm[0], 0};
      const double Sq[9] = {0, -pn[2], pn[1], pn[2], 0, -pn[0], -pn[1], pn[0], 0};
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        row[13 * q + 12] = (float)e[q];
        // (R^T)[q][c] = R[c][q];  (R^T [p]x)[q][c] = sum_k R[k][q] S[k][c]
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          row[13 * q + c] = (float)-Ri[3 * c + q];
          row[13 * q + 6 + c] = (float)Rj[3 * c + q];
          double x = 0, y = 0;
#pragma unroll
          for (int k = 0; k < 3; ++k) { x += Ri[3 * k + q] * Sp[3 * k + c]; y += Rj[3 * k + q] * Sq[3 * k + c]; }
          row[13 * q + 3 + c] = (float)x;
          row[13 * q + 9 + c] = (float)-y;
        }
      }
      const double nrm = sqrt(e[0] * e[0] + e[1] * e[1] + e[2] * e[2]);
      double w, rho;
      if (nrm <= huber) { w = 1.0; rho = 0.5 * nrm * nrm; }
      else { w = huber / nrm; rho = huber * (nrm - 0.5 * huber); }
      row[39] = (float)w;
      row[40] = (float)rho;
    }
    __syncthreads();
    // branch-free: H(a, b) and g(a) = H(a, 12) are the same 3-term dot product of row columns
    // (g's column 12 is e); E and the count are selects.  Rows r and r + 8 per step (loads of
    // both in flight), accumulated in the same row order as a one-row loop.
    auto term = [&](const float *row, int s) {
      const int a = oa[s], b = ob[s];
      const float d = fmaf(row[a], row[b], fmaf(row[13 + a], row[13 + b], row[26 + a] * row[26 + b]));
      return okind[s] <= 1 ? row[39] * d : (okind[s] == 2 ? row[40] : 1.f);
    };
    for (int r = warp; r < nc; r += 2 * (kFinThreads / 32)) {
      const float *r0 = frow + r * kFeatRow;
      const int r1i = r + kFinThreads / 32;
      const float *r1 = frow + (r1i < nc ? r1i : r) * kFeatRow;
#pragma unroll
      for (int s = 0; s < 3; ++s) {
        if (okind[s] < 0) continue;
        const float t0 = term(r0, s), t1 = term(r1, s);
        acc[s] += t0;
        if (r1i < nc) acc[s] += t1;
      }
    }
  }
#pragma unroll
  for (int s = 0; s < 3; ++s) fpart[warp][lane + 32 * s] = acc[s];
  __syncthreads();
  if (tid < 96) {
    float t = 0.f;
    for (int w = 0; w < kFinThreads / 32; ++w) t += fpart[w][tid];
    feat_out[tid] = __float_as_uint(tid < 92 ? t : 0.f);
    if (pr) peer_put(*pr, pp, pw + tid, __float_as_uint(tid < 92 ? t : 0.f));
  }
}

__global__ void __launch_bounds__(kFinThreads) k_ransac_finish(FinishArgs A) {
  pdl_wait();
  extern __shared__ int inl[];                     // [n_max] inlier match indices, in order
  __shared__ float Tb[12];
  __shared__ double red[(kFinThreads / 32 + 1) * 9];
  __shared__ int wcnt[kFinThreads / 32];
  __shared__ double shT[12];
  __shared__ int sh_status;
  // blockIdx.y == 0: h*, C_ij mask, refit, record words; blockIdx.y == 1 (launched only with
  // node poses): the same h* and inlier list, then the Eq. (2) blocks — the two latency chains
  // of a pair run side by side
  const int p = blockIdx.x;
  const bool feat_cta = blockIdx.y == 1;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n_max = A.kp.n_max, W = mask_words(n_max);
  unsigned long long key_all;
  const int M = A.n_matches[p];
  uint32_t *rec = A.records + (size_t)p * A.rec_stride;
  const int fa = A.pairs[2 * p], fb = A.pairs[2 * p + 1];
  const int32_t *mt = A.matches + (size_t)p * n_max * 2;
  const float *pa_f = A.kp.pts + (size_t)fa * n_max * 3, *pb_f = A.kp.pts + (size_t)fb * n_max * 3;
  const float *na_f = A.kp.nrm + (size_t)fa * n_max * 3, *nb_f = A.kp.nrm + (size_t)fb * n_max * 3;

  // best hypothesis: key ((count + 1) << 32 | ~h) — max count, ties -> lowest h (R11)
  __shared__ unsigned long long wkey[kFinThreads / 32];
  {
    unsigned long long kk = 0ull;
    const int32_t *cp = A.counts + (size_t)p * A.n_hyp;
    if ((A.n_hyp & 3) == 0) {                                      // int4 loads, 4 hypotheses each
      for (int h4 = tid; h4 < (A.n_hyp >> 2); h4 += kFinThreads) {
        int4 c4 = make_int4(-1, -1, -1, -1);
        if (M >= 3) c4 = __ldcg(reinterpret_cast<const int4 *>(cp) + h4);
        const int cs[4] = {max(c4.x, -1), max(c4.y, -1), max(c4.z, -1), max(c4.w, -1)};
        if (A.hyp_counts && !feat_cta)
          reinterpret_cast<int4 *>(A.hyp_counts + (size_t)p * A.n_hyp)[h4] = make_int4(cs[0], cs[1], cs[2], cs[3]);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint32_t h = 4 * h4 + q;
          const unsigned long long x = ((unsigned long long)(uint32_t)(cs[q] + 1) << 32) | (0xFFFFFFFFu - h);
          kk = x > kk ? x : kk;
        }
      }
    } else {
      for (int h = tid; h < A.n_hyp; h += kFinThreads) {
        const int cnt = M >= 3 ? max(cp[h], -1) : -1;
        if (A.hyp_counts && !feat_cta) A.hyp_counts[(size_t)p * A.n_hyp + h] = cnt;
        const unsigned long long x = ((unsigned long long)(uint32_t)(cnt + 1) << 32) | (0xFFFFFFFFu - (uint32_t)h);
        kk = x > kk ? x : kk;
      }
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
      const unsigned long long other = __shfl_xor_sync(0xffffffffu, kk, o);
      kk = other > kk ? other : kk;
    }
    if (lane == 0) wkey[warp] = kk;
    __syncthreads();
    kk = 0ull;
#pragma unroll
    for (int w = 0; w < kFinThreads / 32; ++w) kk = wkey[w] > kk ? wkey[w] : kk;
    key_all = kk;
  }
  int status = BT_PAIR_OK, best_h = -1;
  const unsigned long long key = key_all;
  const uint32_t c1 = (uint32_t)(key >> 32);
  if (M < 3) status = BT_PAIR_FEW_MATCHES;
  else if (c1 == 0u) status = BT_PAIR_FEW_INLIERS;                 // every hypothesis degenerate
  else best_h = (int)(0xFFFFFFFFu - (uint32_t)key);

  if (tid < 12) {                                                  // T of h* from the hypothesis buffer
    if (best_h >= 0) {                                             // (count >= 0: non-degenerate)
      const int b = best_h / kHypPerBlock, r = best_h - b * kHypPerBlock;
      const float *src = reinterpret_cast<const float *>(A.hyp + ((size_t)p * A.nb + b) * 12 * kScoreThreads +
                                                         r % kScoreThreads) + r / kScoreThreads;
      Tb[tid] = __ldcg(src + 2 * tid * kScoreThreads);
    } else {
      Tb[tid] = (tid == 0 || tid == 4 || tid == 8) ? 1.f : 0.f;
    }
  }
  __syncthreads();
  // inlier mask C_ij of h* (all words up to n_max written; bit m = match m) and the
  // ordered inlier list, by ballots + a block prefix over warps
  float T[12];
#pragma unroll
  for (int k = 0; k < 12; ++k) T[k] = Tb[k];
  int n_in = 0;
  for (int m0 = 0; m0 < W * 32; m0 += kFinThreads) {
    const int m = m0 + tid;
    bool in = false;
    if (best_h >= 0 && m < M) {
      const int i = mt[2 * m], j = mt[2 * m + 1];
      float4 q0, q1, q2, q3;
      pack_corr(pa_f + 3 * i, na_f + 3 * i, pb_f + 3 * j, nb_f + 3 * j, q0, q1, q2, q3);
      in = inlier(T, q0, q1, q2, q3, A.ndelta2, A.ncosa);
    }
    const unsigned bal = __ballot_sync(0xffffffffu, in);
    if (lane == 0) {
      if (!feat_cta && (m0 >> 5) + warp < W) {
        rec[kRecMask + (m0 >> 5) + warp] = bal;
        peer_put(A.peers, p, kRecMask + (m0 >> 5) + warp, bal);
      }
      wcnt[warp] = __popc(bal);
    }
    __syncthreads();
    int off = 0, tot = 0;
    for (int w = 0; w < kFinThreads / 32; ++w) {
      off += w < warp ? wcnt[w] : 0;
      tot += wcnt[w];
    }
    if (in) inl[n_in + off + __popc(bal & ((1u << lane) - 1u))] = m;
    n_in += tot;
    __syncthreads();
  }
  const int best_count = n_in;
  __shared__ float fpart[kFinThreads / 32][96];
  if (feat_cta) {
    // ---- Eq. (2) feature edge at the node poses ----------------------------------
    feature_blocks(inl, best_h >= 0 ? best_count : 0, mt, pa_f, pb_f, A.node_pose[fa], A.node_pose[fb], A.huber,
                   reinterpret_cast<float *>(inl + ((n_max + 3) & ~3)), fpart, rec + rec_feat(n_max),
                   A.peers.n ? &A.peers : nullptr, p, rec_feat(n_max));
    return;
  }
  if (best_h >= 0 && best_count < A.min_inliers) status = BT_PAIR_FEW_INLIERS;

  // refit: Arun on all inliers (fp64), two-pass centroid / cross-covariance
  double Rr[9], tr[3];
  bool refit_ok = false;
  if (status == BT_PAIR_OK) {
    double s6[6] = {0, 0, 0, 0, 0, 0};
    for (int k = tid; k < best_count; k += kFinThreads) {
      const int m = inl[k];
      const int i = mt[2 * m], j = mt[2 * m + 1];
#pragma unroll
      for (int c = 0; c < 3; ++c) { s6[c] += pa_f[3 * i + c]; s6[3 + c] += pb_f[3 * j + c]; }
    }
    block_sum_n<6>(s6, red);
    double ca[3], cb[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) { ca[c] = s6[c] / best_count; cb[c] = s6[3 + c] / best_count; }
    double Hl[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    for (int k = tid; k < best_count; k += kFinThreads) {
      const int m = inl[k];
      const int i = mt[2 * m], j = mt[2 * m + 1];
      double da[3], db[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) { da[c] = pa_f[3 * i + c] - ca[c]; db[c] = pb_f[3 * j + c] - cb[c]; }
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) Hl[3 * r + c] += da[r] * db[c];
    }
    block_sum_n<9>(Hl, red);
    if (tid == 0) {
      double U[9], s[3], V[9];
      svd3_jacobi(Hl, U, s, V);
      const double ratio = s[0] > 0 ? s[1] / s[0] : 0.0;
      if (ratio < A.tau) {
        sh_status = BT_PAIR_REFIT_DEGENERATE;
      } else {
        sh_status = BT_PAIR_OK;
        const double d = det3(V) * det3(U) > 0 ? 1.0 : -1.0;
        for (int r = 0; r < 3; ++r)
          for (int c = 0; c < 3; ++c)
            shT[3 * r + c] = V[3 * r] * U[3 * c] + V[3 * r + 1] * U[3 * c + 1] + d * V[3 * r + 2] * U[3 * c + 2];
        for (int r = 0; r < 3; ++r)
          shT[9 + r] = cb[r] - (shT[3 * r] * ca[0] + shT[3 * r + 1] * ca[1] + shT[3 * r + 2] * ca[2]);
      }
    }
    __syncthreads();
    status = sh_status;
    refit_ok = status == BT_PAIR_OK;
#pragma unroll
    for (int k = 0; k < 9; ++k) Rr[k] = shT[k];
#pragma unroll
    for (int k = 0; k < 3; ++k) tr[k] = shT[9 + k];
  }
  if (tid == 0) {
    rec[kRecStatus] = (uint32_t)status;
    rec[kRecNMatch] = (uint32_t)M;
    rec[kRecBestHyp] = (uint32_t)best_h;
    rec[kRecBestCount] = (uint32_t)(best_h >= 0 ? best_count : 0);
    for (int k = 0; k < 12; ++k) rec[kRecTBest + k] = __float_as_uint(Tb[k]);
    for (int k = 0; k < 12; ++k)
      rec[kRecTRefit + k] = __float_as_uint(refit_ok ? (float)(k < 9 ? Rr[k] : tr[k - 9]) : Tb[k]);
    if (A.peers.n)
      for (int w = 0; w < kRecMask; ++w) peer_put(A.peers, p, w, rec[w]);
  }
}


// Re-linearization of the Eq. (2) blocks at new node poses with C_ij reused: the
// ascending inlier list is rebuilt from the record's mask, then the same accumulation as the
// finish kernel (bitwise identical to a registration at these poses).
struct FeatArgs {
  KpView kp;
  const int32_t *pairs;
  const int32_t *matches;
  const int32_t *n_matches;
  uint32_t *records;
  int rec_stride;
  const bt_pose *node_pose;
  double huber;
};

__global__ void __launch_bounds__(kFinThreads) k_feature_edges(FeatArgs A) {
  extern __shared__ int inl[];
  __shared__ int wcnt[kFinThreads / 32];
  __shared__ float fpart[kFinThreads / 32][96];
  const int p = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n_max = A.kp.n_max, W = mask_words(n_max);
  const int M = A.n_matches[p];
  uint32_t *rec = A.records + (size_t)p * A.rec_stride;
  const int fa = A.pairs[2 * p], fb = A.pairs[2 * p + 1];
  int n_in = 0;
  for (int m0 = 0; m0 < W * 32; m0 += kFinThreads) {
    const int m = m0 + tid;
    const bool in = m < M && ((rec[kRecMask + (m >> 5)] >> (m & 31)) & 1u);
    const unsigned bal = __ballot_sync(0xffffffffu, in);
    if (lane == 0) wcnt[warp] = __popc(bal);
    __syncthreads();
    int off = 0, tot = 0;
    for (int w = 0; w < kFinThreads / 32; ++w) { off += w < warp ? wcnt[w] : 0; tot += wcnt[w]; }
    if (in) inl[n_in + off + __popc(bal & ((1u << lane) - 1u))] = m;
    n_in += tot;
    __syncthreads();
  }
  const float *pa_f = A.kp.pts + (size_t)fa * n_max * 3, *pb_f = A.kp.pts + (size_t)fb * n_max * 3;
  feature_blocks(inl, n_in, A.matches + (size_t)p * n_max * 2, pa_f, pb_f, A.node_pose[fa], A.node_pose[fb],
                 A.huber, reinterpret_cast<float *>(inl + ((n_max + 3) & ~3)), fpart, rec + rec_feat(n_max));
}

__device__ __forceinline__ f32x2 add2v(f32x2 a, f32x2 b) {               // a + b
  f32x2 d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ f32x2 sub2s(float a, f32x2 b) {               // {a, a} - b
  f32x2 d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(pk(a, a)), "l"(b));
  return d;
}

// ---------------------------------------------------------------- scoring on the tensor cores
// The inlier test of every (hypothesis h, correspondence m) as two small contractions
// (reading R27 of DESIGN.md).  With the pair's centroids a_bar, b_bar (fp32), a' = a - a_bar,
// b' = b - b_bar and t' = t + R a_bar - b_bar:
//   |R a + t - b|^2 = |R a' + t' - b'|^2
//                   = |t'|^2 + [ 2 R^T t' | -2 vec R | -2 t' | 1 ] . [ a' | vec(b' a'^T) | b' | |a'|^2 + |b'|^2 ]
//                     (|R a'|^2 = |a'|^2 up to the fp32 rounding of R, bounded below)
//   (R n_a) . n_b   = vec R . vec(n_b n_a^T)
// i.e. D1 = X1(h) . Y1(m) (K = 16) and D2 = X2(h) . Y2(m) (K = 9, padded to 16).  Each fp32
// feature x (scaled by a power of two into fp16 range) is split x = hi + lo (fp16 each,
// |x - hi - lo| <= 2^-22 |x|) and the products run as kind::f16 tcgen05.mma with fp32
// accumulation: D = X_hi.Y_hi + X_hi.Y_lo + X_lo.Y_hi (K = 48 per test type).
// Exactness: per row h the kernel bounds |D - exact| (split + dropped lo.lo + accumulation,
// from sum_k |X_hk| max_m |Y_mk|) plus the error of the fp32 FMA formula the finish kernel
// uses (dist_term / normal_term), and counts twice: "certain" inliers (both gates pass with
// margin) and "possible" ones (neither gate fails with margin).  Equal counts are the count
// of the fp32 formula exactly; a row where they differ (a test within ~1e-6 of a gate, ~1e-4
// of the tests) is listed and recounted with the fp32 formula itself (k_score_fix).  So the
// counts are bit-identical to the FMA kernel's.
constexpr int kTcRows = 128;                 // hypotheses per item (UMMA M)
#ifndef BT_TC_COLS
#define BT_TC_COLS 64
#endif
constexpr int kTcCols = BT_TC_COLS;          // correspondences per chunk (UMMA N)
#ifndef BT_TC_CTAS
#define BT_TC_CTAS 2
#endif
constexpr int kTcCtas = BT_TC_CTAS;            // CTAs per SM (each owns 512 / kTcCtas TMEM columns)
constexpr int kTcTmem = 512 / kTcCtas;
constexpr int kTcTBuf = kTcTmem / (2 * kTcCols);  // TMEM buffers (D1 + D2 of a chunk each)
constexpr int kTcWc = kTcCols / (BT_TC_EPI_WARPS / 4);  // columns per warpgroup and chunk
constexpr int kTcPad = 128;                  // feature rows per pair: multiple of 128
constexpr int kTcFeat = 64;                  // fp16 per feature row: X1/Y1 hi, lo | X2/Y2 hi, lo
constexpr int kTcEpiWarps = BT_TC_EPI_WARPS;  // warpgroups x (columns of a chunk / warpgroups)
constexpr int kTcWgs = kTcEpiWarps / 4;
constexpr int kTcThreads = (kTcEpiWarps + 2) * 32;   // + MMA warp + TMA warp
#ifndef BT_TC_BBUF
#define BT_TC_BBUF 0
#endif
constexpr int kTcBBuf = BT_TC_BBUF ? BT_TC_BBUF : (kTcCtas == 1 ? 6 : 3);
constexpr size_t kTcSmem = 1024 + 2 * kTcRows * 128 + kTcBBuf * kTcCols * 128;
constexpr float kTcSentinel = 65504.f;       // padded correspondence: D1 = 65504 * s_x > any threshold

struct PairFeat {                            // per pair, written by k_corr_feat
  float abar[3], bbar[3];
  float sy1;                                 // power-of-two scale of Y1 (Y2: 2^14)
  float ab;                                  // 2 max |a| + max |b| (reference-formula error)
  float korth;                               // 2e-6 max |a'|^2 (|R a'|^2 vs |a'|^2, fp32 R)
  float apmax2;
  float ymax1[16], ymax2[16];                // max_m |Y_mk| (unscaled, rounded up)
  int M, pad[3];
};
struct ScoreConst {                          // per launch (host-computed)
  float delta2, cosa;                        // the fp32 gate values of dist_term / normal_term
  float c_rel;                               // |D - exact| <= c_rel * sum |X||Y|
  float e_a, e_b;                            // eref1 = E (e_a + 3 E) + e_b,  E = 2^-21 (ab + |t|_1)
  float k2;                                  // constant part of eps2
};

struct ScoreTcArgs {
  KpView kp;
  const int32_t *pairs;
  const int32_t *matches;
  const int32_t *n_matches;
  int P, n_hyp, nb, nht, m_pad;
  float ndelta2, ncosa;
  ScoreConst sc;
  const f32x2 *hyp;
  int32_t *counts;
  PairFeat *pf;
  __half *feat;                              // [P][m_pad][64]
  int4 *elist;                               // undecided tests (p, h, m): evaluated by k_score_fix
  int32_t *ecount;                           // [2]: undecided tests, overflowed rows
  int ecap;
  int2 *fix;                                 // rows whose tests overflowed elist: recounted whole
  uint32_t *ofl;                             // [P][ceil(H / 32)] bit = row in fix (cleared by k_corr_feat)
};


// One CTA per pair (512 threads, fp32): pass 1 gathers the pair's correspondences (kept in
// registers for the first 512) and reduces the centroids and max |a|, |b|; pass 2 forms the
// centred features, reduces their maxima (the error bound's max_m |Y_mk|, and the Y1 scale)
// and writes the fp16 hi/lo rows (padded rows: Y1 = (0, ..., 0, 65504) so that D1 exceeds every
// distance threshold, Y2 = 0).  The centroid need not be exact — any centring is algebraically
// exact; fp32 feature rounding (2^-24) is inside the certificate's 2^-22 feature term.
constexpr int kFeatThreads = 512;
// Y1 of a correspondence: [2 a', -2 vec(b' a'^T), -2 b', |a'|^2 + |b'|^2] (X1 = [R^T t', vec R, t', 1])
__device__ __forceinline__ void corr_y1f(const float *ap, const float *bp, float *y1) {
#pragma unroll
  for (int k = 0; k < 3; ++k) { y1[k] = 2.f * ap[k]; y1[12 + k] = -2.f * bp[k]; }
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) y1[3 + 3 * i + j] = -2.f * bp[i] * ap[j];
  y1[15] = fmaf(ap[0], ap[0], fmaf(ap[1], ap[1], fmaf(ap[2], ap[2], fmaf(bp[0], bp[0], fmaf(bp[1], bp[1], bp[2] * bp[2])))));
}
template <int N, bool SUM>
__device__ __forceinline__ void block_reduce_f(float (&v)[N], float (*red)[32]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < N; ++k)
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
      const float y = __shfl_xor_sync(0xffffffffu, v[k], o);
      v[k] = SUM ? v[k] + y : fmaxf(v[k], y);
    }
  __syncthreads();
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < N; ++k) red[k][warp] = v[k];
  __syncthreads();
#pragma unroll
  for (int k = 0; k < N; ++k) {
    float t = SUM ? 0.f : 0.f;
    for (int w = 0; w < kFeatThreads / 32; ++w) t = SUM ? t + red[k][w] : fmaxf(t, red[k][w]);
    v[k] = t;
  }
}
__global__ void __launch_bounds__(kFeatThreads) k_corr_feat(ScoreTcArgs A) {
  pdl_wait();
  __shared__ float red[26][32];
  const int p = blockIdx.x, tid = threadIdx.x;
  if (p == 0 && tid < 2) A.ecount[tid] = 0;
  for (int w = tid, nw = (A.n_hyp + 31) / 32; w < nw; w += kFeatThreads) A.ofl[(size_t)p * nw + w] = 0u;
  const int M = A.n_matches[p];
  PairFeat *pf = A.pf + p;
  if (tid == 0) pf->M = M;
  if (M < 3) return;
  const int fa = A.pairs[2 * p], fb = A.pairs[2 * p + 1];
  const int32_t *mt = A.matches + (size_t)p * A.kp.n_max * 2;
  const float *pa = A.kp.pts + (size_t)fa * A.kp.n_max * 3, *pb = A.kp.pts + (size_t)fb * A.kp.n_max * 3;
  const float *na = A.kp.nrm + (size_t)fa * A.kp.n_max * 3, *nb = A.kp.nrm + (size_t)fb * A.kp.n_max * 3;
  auto gather = [&](int m, float *x, float *y, float *u, float *w) {
    const int i = mt[2 * m], j = mt[2 * m + 1];
#pragma unroll
    for (int k = 0; k < 3; ++k) { x[k] = pa[3 * i + k]; y[k] = pb[3 * j + k]; u[k] = na[3 * i + k]; w[k] = nb[3 * j + k]; }
  };
  float x0[3] = {0, 0, 0}, y0[3] = {0, 0, 0}, u0[3] = {0, 0, 0}, w0[3] = {0, 0, 0};
  if (tid < M) gather(tid, x0, y0, u0, w0);
  float s[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int m = tid; m < M; m += kFeatThreads) {
    float x[3], y[3], u[3], w[3];
    if (m == tid) { for (int k = 0; k < 3; ++k) { x[k] = x0[k]; y[k] = y0[k]; } }
    else gather(m, x, y, u, w);
    s[0] += x[0]; s[1] += x[1]; s[2] += x[2]; s[3] += y[0]; s[4] += y[1]; s[5] += y[2];
    s[6] = fmaxf(s[6], sqrtf(fmaf(x[0], x[0], fmaf(x[1], x[1], x[2] * x[2]))));
    s[7] = fmaxf(s[7], sqrtf(fmaf(y[0], y[0], fmaf(y[1], y[1], y[2] * y[2]))));
  }
  {
    float sm[6] = {s[0], s[1], s[2], s[3], s[4], s[5]}, mx[2] = {s[6], s[7]};
    block_reduce_f<6, true>(sm, red);
    block_reduce_f<2, false>(mx, red + 8);
    for (int k = 0; k < 6; ++k) s[k] = sm[k] / (float)M;
    s[6] = mx[0]; s[7] = mx[1];
  }
  const float cen[6] = {s[0], s[1], s[2], s[3], s[4], s[5]};
  // pass 2: feature maxima
  float mxv[26];
#pragma unroll
  for (int k = 0; k < 26; ++k) mxv[k] = 0.f;
  for (int m = tid; m < M; m += kFeatThreads) {
    float x[3], y[3], u[3], w[3];
    if (m == tid) { for (int k = 0; k < 3; ++k) { x[k] = x0[k]; y[k] = y0[k]; u[k] = u0[k]; w[k] = w0[k]; } }
    else gather(m, x, y, u, w);
    float ap[3], bp[3], y1[16];
    for (int k = 0; k < 3; ++k) { ap[k] = x[k] - cen[k]; bp[k] = y[k] - cen[3 + k]; }
    corr_y1f(ap, bp, y1);
#pragma unroll
    for (int k = 0; k < 16; ++k) mxv[k] = fmaxf(mxv[k], fabsf(y1[k]));
#pragma unroll
    for (int k = 0; k < 9; ++k) mxv[16 + k] = fmaxf(mxv[16 + k], fabsf(w[k / 3] * u[k % 3]));
    mxv[25] = fmaxf(mxv[25], fmaf(ap[0], ap[0], fmaf(ap[1], ap[1], ap[2] * ap[2])));
  }
  block_reduce_f<26, false>(mxv, red);
  // Y1 scale: max |Y1| * sy1 < 2^14, and >= delta^2 so that the padded rows' 65504 * s_x
  // exceeds every distance threshold (65504 / sy1 > 4 max(|Y1|max, delta^2))
  float ymx = A.sc.delta2;
#pragma unroll
  for (int k = 0; k < 16; ++k) ymx = fmaxf(ymx, mxv[k]);
  const int e = ((__float_as_int(ymx) >> 23) & 255) - 126;   // ymx < 2^e
  const float sy1 = __int_as_float((127 + 14 - e) << 23), sy2 = 16384.f;
  if (tid < 16) pf->ymax1[tid] = mxv[tid] * 1.0000002f;
  else if (tid < 25) pf->ymax2[tid - 16] = mxv[tid] * 1.0000002f;
  else if (tid < 32) pf->ymax2[tid - 16] = 0.f;
  if (tid == 0) {
    for (int k = 0; k < 6; ++k) (k < 3 ? pf->abar[k] : pf->bbar[k - 3]) = cen[k];
    pf->sy1 = sy1;
    pf->ab = (2.f * s[6] + s[7]) * 1.00001f;
    pf->korth = 2e-6f * mxv[25] * 1.0001f;
    pf->apmax2 = mxv[25];
  }
  const int mp = (M + kTcCols - 1) / kTcCols * kTcCols;
  __half *F = A.feat + (size_t)p * A.m_pad * kTcFeat;
  for (int m = tid; m < mp; m += kFeatThreads) {
    __align__(16) __half h1[16], l1[16], h2[16], l2[16];
    if (m < M) {
      float x[3], y[3], u[3], w[3];
      if (m == tid) { for (int k = 0; k < 3; ++k) { x[k] = x0[k]; y[k] = y0[k]; u[k] = u0[k]; w[k] = w0[k]; } }
      else gather(m, x, y, u, w);
      float ap[3], bp[3], y1[16];
      for (int k = 0; k < 3; ++k) { ap[k] = x[k] - cen[k]; bp[k] = y[k] - cen[3 + k]; }
      corr_y1f(ap, bp, y1);
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const float v1 = y1[k] * sy1;
        h1[k] = __float2half_rn(v1);
        l1[k] = __float2half_rn(v1 - __half2float(h1[k]));
        const float v2 = k < 9 ? w[k / 3] * u[k % 3] * sy2 : 0.f;
        h2[k] = __float2half_rn(v2);
        l2[k] = __float2half_rn(v2 - __half2float(h2[k]));
      }
    } else {
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        h1[k] = __float2half_rn(k == 15 ? kTcSentinel : 0.f); l1[k] = h2[k] = l2[k] = __float2half_rn(0.f);
      }
    }
    uint4 *dst = reinterpret_cast<uint4 *>(F + (size_t)m * kTcFeat);
    const uint4 *s1 = reinterpret_cast<const uint4 *>(h1), *s2 = reinterpret_cast<const uint4 *>(l1);
    const uint4 *s3 = reinterpret_cast<const uint4 *>(h2), *s4 = reinterpret_cast<const uint4 *>(l2);
    dst[0] = s1[0]; dst[1] = s1[1]; dst[2] = s2[0]; dst[3] = s2[1];
    dst[4] = s3[0]; dst[5] = s3[1]; dst[6] = s4[0]; dst[7] = s4[1];
  }
}

// T of hypothesis h of pair p from the f32x2 hypothesis buffer (k_ransac_hyp's layout)
__device__ __forceinline__ void load_T(const ScoreTcArgs &A, int p, int h, float *T) {
  const int b = h / kHypPerBlock, r = h - b * kHypPerBlock;
  const int t = r % kScoreThreads, k = r / kScoreThreads;
  const float *src = reinterpret_cast<const float *>(A.hyp + ((size_t)p * A.nb + b) * 12 * kScoreThreads + t) + k;
#pragma unroll
  for (int q = 0; q < 12; ++q) T[q] = __ldcg(src + 2 * q * kScoreThreads);
}

struct RowConst {
  float lo1B, lo2, hi2;                      // lo1B = lo1 * kSatB (certain-count thresholds pre-scaled)
  float lo1, hi1, hi2B, lo2r;
  bool valid;
};
constexpr float kSatB = 18446744073709551616.f;   // 2^64: sat((lo - x) 2^64) is 1 iff x < lo (scaled units)
// Per-row thresholds (scaled units) and one quarter of the row's fp16 features, written into
// the 128B-swizzled A tile (16-B chunk c of row r lands at c ^ (r & 7)): part 0 X1 hi, 1 X1 lo,
// 2 X2 hi, 3 X2 lo.  fp32 throughout: the features' own rounding (2^-22 relative) is in c_rel,
// the thresholds carry a 2^-21 (delta^2 + |t'|^2) slack for their fp32 evaluation.
__device__ __forceinline__ RowConst row_setup(const ScoreTcArgs &A, const PairFeat *pf, const float *T, uint8_t *arow,
                                              int r, int part) {
  RowConst rc;
  rc.valid = T[11] < 1e30f;
  float R[9];
#pragma unroll
  for (int k = 0; k < 9; ++k) R[k] = rc.valid ? T[k] : 0.f;
  __align__(16) __half h[16];
  if (part >= 2) {                                         // X2 = vec R (scaled 2^14): hi or lo
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const float x = k < 9 ? R[k] * 16384.f : 0.f;
      const __half hi = __float2half_rn(x);
      h[k] = part == 3 ? __float2half_rn(x - __half2float(hi)) : hi;
    }
  } else {
    float t[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) t[k] = rc.valid ? T[9 + k] : 0.f;
    const float ab0 = pf->abar[0], ab1 = pf->abar[1], ab2 = pf->abar[2];
    float x1[16];                                          // [R^T t', vec R, t', 1]
#pragma unroll
    for (int i = 0; i < 3; ++i)
      x1[12 + i] = t[i] + fmaf(R[3 * i], ab0, fmaf(R[3 * i + 1], ab1, R[3 * i + 2] * ab2)) - pf->bbar[i];
#pragma unroll
    for (int j = 0; j < 3; ++j) x1[j] = fmaf(R[j], x1[12], fmaf(R[3 + j], x1[13], R[6 + j] * x1[14]));
#pragma unroll
    for (int k = 0; k < 9; ++k) x1[3 + k] = R[k];
    x1[15] = 1.f;
    const float tn2 = fmaf(x1[12], x1[12], fmaf(x1[13], x1[13], x1[14] * x1[14]));
    // max |X1| <= max(1.0001, 1.0001 |t'|) < 2^e  ->  sx = 2^(14 - e)
    const float xm = fmaxf(1.0001f, 1.0001f * sqrtf(tn2) + 1e-6f);
    const int e = ((__float_as_int(xm) >> 23) & 255) - 126;
    const float sx = __int_as_float((127 + 14 - e) << 23);
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const float x = x1[k] * sx;
      const __half hi = __float2half_rn(x);
      h[k] = part == 1 ? __float2half_rn(x - __half2float(hi)) : hi;
    }
    if (part == 0) {                                       // the row's thresholds
      float s1 = 0.f, s2 = 0.f;
#pragma unroll
      for (int k = 0; k < 16; ++k) s1 = fmaf(fabsf(x1[k]), pf->ymax1[k], s1);
#pragma unroll
      for (int k = 0; k < 9; ++k) s2 = fmaf(fabsf(R[k]), pf->ymax2[k], s2);
      const float E = 0x1p-21f * (pf->ab + fabsf(t[0]) + fabsf(t[1]) + fabsf(t[2]));
      const float eref1 = fmaf(E, fmaf(3.f, E, A.sc.e_a), A.sc.e_b);
      const float eps1 = fmaf(A.sc.c_rel, s1, pf->korth + eref1 + 0x1p-21f * (A.sc.delta2 + tn2)) * 1.0001f;
      const float eps2 = fmaf(A.sc.c_rel, s2, A.sc.k2) * 1.0001f;
      const float sc1 = sx * pf->sy1, sc2 = 268435456.f;     // D1, D2 scales (powers of two)
      const float thr = A.sc.delta2 - tn2;
      rc.lo1 = sc1 * (thr - eps1);
      rc.hi1 = sc1 * (thr + eps1);
      rc.lo2 = sc2 * (A.sc.cosa - eps2);
      rc.hi2 = sc2 * (A.sc.cosa + eps2);
      rc.lo1B = rc.lo1 * kSatB;
      rc.hi2B = rc.hi2 * kSatB;
      rc.lo2r = rc.lo2;
    }
  }
  const uint4 *src = reinterpret_cast<const uint4 *>(h);
  uint4 *dst = reinterpret_cast<uint4 *>(arow);
  dst[(2 * part) ^ (r & 7)] = src[0];
  dst[(2 * part + 1) ^ (r & 7)] = src[1];
  return rc;
}

// Persistent, warp-specialized: items (pair p, tile of 128 hypotheses) walk blockIdx.x,
// + gridDim.x, ...; chunks of 128 correspondences form one stream g per CTA.
//   producer warp 16: TMA of feature chunk g into B buffer g % 3 (after the MMAs of g - 3
//     released it), then 6 tcgen05.mma (D1: X1hi.Y1hi + X1hi.Y1lo + X1lo.Y1hi, D2 likewise)
//     into TMEM buffer g & 1 (D1 columns 0-127, D2 128-255) once the epilogue released it.
//   epilogue warps 0-15: warpgroup 0 builds the next item's A tile (features of its 128
//     hypotheses) at the start of each item; every warp reads 32 columns of D1 and D2 for its
//     32 TMEM lanes, releases the buffer, and counts certain / possible inliers per row.
__global__ void __launch_bounds__(kTcThreads, kTcCtas) k_score_tc(const __grid_constant__ CUtensorMap fmap, ScoreTcArgs A) {
  pdl_wait();
  extern __shared__ uint8_t tc_smem_raw[];
  __shared__ __align__(8) uint64_t bar_a[2], bar_bfull[kTcBBuf], bar_bfree[kTcBBuf], bar_mma[kTcTBuf], bar_tfree[kTcTBuf];
  __shared__ uint32_t tmem_base_sh;
  __shared__ float4 rowc[4][kTcRows];
  __shared__ bool rowv[4][kTcRows];
  uint8_t *base = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(tc_smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t *sA = base;                                       // [2][128 rows][128 B]
  uint8_t *sB = base + 2 * kTcRows * 128;                   // [3][128 rows][128 B]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n_items = A.P * A.nht;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_sh)),
                 "r"(kTcTmem)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (tid == 0) {
    for (int b = 0; b < 2; ++b) mbar_init(&bar_a[b], kTcEpiWarps);
    for (int b = 0; b < kTcTBuf; ++b) { mbar_init(&bar_mma[b], 1); mbar_init(&bar_tfree[b], kTcEpiWarps); }
    for (int b = 0; b < kTcBBuf; ++b) { mbar_init(&bar_bfull[b], 1); mbar_init(&bar_bfree[b], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_sh;
  const uint32_t idesc = (1u << 4) | ((uint32_t)(kTcCols >> 3) << 17) | ((uint32_t)(kTcRows >> 4) << 24);

  if (warp == kTcEpiWarps + 1) {
    // ------------------------------------------------------------ TMA warp: runs up to
    // kTcBBuf chunks ahead of the MMAs (a buffer is refilled once the MMAs of its last chunk ended)
    if (lane == 0) {
      uint32_t g = 0;
      for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
        const int p = it / A.nht;
        const int M = A.n_matches[p];
        if (M < 3) continue;
        const int nch = (M + kTcCols - 1) / kTcCols;
        for (int c = 0; c < nch; ++c, ++g) {
          const int bb = g % kTcBBuf;
          const uint32_t use = g / kTcBBuf;
          if (use > 0) mbar_wait_sleep(&bar_bfree[bb], (use - 1) & 1);
          mbar_expect_tx(&bar_bfull[bb], kTcCols * 128);
          tma_load_2d(sB + bb * kTcCols * 128, &fmap, 0, p * A.m_pad + c * kTcCols, &bar_bfull[bb]);
        }
      }
    }
  } else if (warp == kTcEpiWarps) {
    // ------------------------------------------------------------ MMA warp
    if (lane == 0) {
      uint32_t g = 0, k = 0;
      for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
        const int p = it / A.nht;
        const int M = A.n_matches[p];
        if (M < 3) continue;
        const int nch = (M + kTcCols - 1) / kTcCols;
        for (int c = 0; c < nch; ++c, ++g) {
          const int bb = g % kTcBBuf, tb = g % kTcTBuf;
          const uint32_t use = g / kTcBBuf;
          if (c == 0) mbar_wait_sleep(&bar_a[k & 1], (k >> 1) & 1);
          if (g >= kTcTBuf) mbar_wait_sleep(&bar_tfree[tb], ((g - kTcTBuf) / kTcTBuf) & 1);
          mbar_wait_sleep(&bar_bfull[bb], use & 1);
          tc_fence_after();
          const uint8_t *a = sA + (k & 1) * kTcRows * 128, *b = sB + bb * kTcCols * 128;
          const uint32_t d1 = tmem + tb * 2 * kTcCols, d2 = d1 + kTcCols;
          // the operands' 32-B K slices: the descriptors' start-address field (16-B units, 14 bits;
          // shared memory < 228 KB, so + 6 never carries) advanced by 2 per slice
          const uint64_t da = umma_desc_sw128(a), db = umma_desc_sw128(b);
          umma_f16(d1, da, db, idesc, 0u);                          // X1hi . Y1hi
          umma_f16(d1, da, db + 2, idesc, 1u);                      // X1hi . Y1lo
          umma_f16(d1, da + 2, db, idesc, 1u);                      // X1lo . Y1hi
          umma_f16(d2, da + 4, db + 4, idesc, 0u);                  // X2hi . Y2hi
          umma_f16(d2, da + 4, db + 6, idesc, 1u);                  // X2hi . Y2lo
          umma_f16(d2, da + 6, db + 4, idesc, 1u);                  // X2lo . Y2hi
          umma_commit(&bar_mma[tb]);
          umma_commit(&bar_bfree[bb]);
        }
        ++k;
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const int wg = warp >> 2, q = warp & 3;
    const int lrow = q * 32 + lane;                         // TMEM lane = hypothesis row
    uint32_t g = 0, k = 0;
    // Every warp builds its quarter of the A tile of the next item (warpgroup 0 also its row
    // thresholds, into rowc[k & 3]) and arrives on bar_a; at an item's start every warp waits on
    // bar_a and reads the thresholds (no warp can be a phase behind: all 16 arrive per item;
    // rowc is 4 deep because a warp may lag the builders by up to two items).
    int it = blockIdx.x;
    while (it < n_items && A.n_matches[it / A.nht] < 3) it += gridDim.x;
    float Tn[12];
    auto build = [&](int itb, uint32_t kb) {
      const int pb = itb / A.nht, hb = (itb - pb * A.nht) * kTcRows + lrow;
      load_T(A, pb, hb, Tn);
      RowConst r = row_setup(A, A.pf + pb, Tn, sA + (kb & 1) * kTcRows * 128 + lrow * 128, lrow, wg);
      for (int part = wg + kTcWgs; part < 4; part += kTcWgs)
        row_setup(A, A.pf + pb, Tn, sA + (kb & 1) * kTcRows * 128 + lrow * 128, lrow, part);
      if (wg == 0) {
        rowc[kb & 3][lrow] = make_float4(r.lo1B, r.hi1, r.lo2, r.hi2B);
        rowv[kb & 3][lrow] = r.valid;
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar_a[kb & 1]);
    };
    if (it < n_items) build(it, 0);
    while (it < n_items) {
      const int p = it / A.nht, ht = it - p * A.nht;
      const int M = A.n_matches[p];
      const int nch = (M + kTcCols - 1) / kTcCols;
      int itn = it + gridDim.x;
      while (itn < n_items && A.n_matches[itn / A.nht] < 3) itn += gridDim.x;
      if (itn < n_items) build(itn, k + 1);
      mbar_wait_sleep(&bar_a[k & 1], (k >> 1) & 1);               // this item's thresholds
      RowConst rc;
      {
        const float4 v = rowc[k & 3][lrow];
        rc.lo1B = v.x; rc.hi1 = v.y; rc.lo2 = v.z; rc.hi2B = v.w;
        rc.lo1 = rc.lo1B * (1.f / kSatB); rc.hi2 = rc.hi2B * (1.f / kSatB); rc.lo2r = rc.lo2;
        rc.valid = rowv[k & 3][lrow];
      }
      unsigned cert = 0;
      bool overflow = false;
      for (int c = 0; c < nch; ++c, ++g) {
        const int tb = g % kTcTBuf;
#ifndef BT_TC_SLEEP
#define BT_TC_SLEEP 200
#endif
        mbar_wait_sleep(&bar_mma[tb], (g / kTcTBuf) & 1, BT_TC_SLEEP);
        tc_fence_after();
        const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(tb * 2 * kTcCols + wg * kTcWc);
        if (c * kTcCols + wg * kTcWc >= M) {                        // all columns padding: release only
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&bar_tfree[tb]);
          continue;
        }
        const f32x2 hi1 = pk(-rc.hi1, -rc.hi1);
        // the warp's columns of D1 and D2 in 16-column loads, all issued before one wait; the
        // buffer is released as soon as they are in registers
        constexpr int kH = kTcWc / 16;
        uint32_t v1a[kH][16], v2a[kH][16];
#pragma unroll
        for (int hf = 0; hf < kH; ++hf) {
          BT_TMEM_LD16(ta + hf * 16, v1a[hf]);
          BT_TMEM_LD16(ta + kTcCols + hf * 16, v2a[hf]);
        }
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bar_tfree[tb]);
#pragma unroll
        for (int hf = 0; hf < kH; ++hf) {
          const uint32_t *v1 = v1a[hf], *v2 = v2a[hf];
          // certain (D1 < lo1 and D2 > hi2) on the FMA pipe: sat((lo1 - x) 2^64) * sat((y - hi2) 2^64);
          // possible (D1 < hi1 and D2 > lo2) from sign bits
          f32x2 cacc[4] = {pk(0.f, 0.f), pk(0.f, 0.f), pk(0.f, 0.f), pk(0.f, 0.f)};   // 4 short chains
          unsigned pcs[2] = {0u, 0u};
#pragma unroll
          for (int col = 0; col < 16; col += 2) {
            const float x0 = __uint_as_float(v1[col]), x1 = __uint_as_float(v1[col + 1]);
            const float y0 = __uint_as_float(v2[col]), y1 = __uint_as_float(v2[col + 1]);
            const f32x2 ia = pk(__saturatef(__fmaf_rn(x0, -kSatB, rc.lo1B)), __saturatef(__fmaf_rn(x1, -kSatB, rc.lo1B)));
            const f32x2 ib = pk(__saturatef(__fmaf_rn(y0, kSatB, -rc.hi2B)), __saturatef(__fmaf_rn(y1, kSatB, -rc.hi2B)));
            cacc[(col >> 1) & 3] = fma2v(ia, ib, cacc[(col >> 1) & 3]);
            unsigned c0_, c1_, e0, e1;
            split(add2v(pk(x0, x1), hi1), c0_, c1_);
            split(sub2s(rc.lo2r, pk(y0, y1)), e0, e1);
            pcs[(col >> 1) & 1] += ((c0_ & e0) >> 31) + ((c1_ & e1) >> 31);
          }
          const unsigned pc = pcs[0] + pcs[1];
          unsigned ca_, cb_;
          split(add2v(add2v(cacc[0], cacc[1]), add2v(cacc[2], cacc[3])), ca_, cb_);
          const unsigned cc = (unsigned)(__uint_as_float(ca_) + __uint_as_float(cb_));
          cert += cc;
          if (__any_sync(0xffffffffu, pc != cc)) {                // rare: list the undecided tests
            if (pc != cc) {
              const int h = ht * kTcRows + lrow;
              for (int col = 0; col < 16; ++col) {
                const float x = __uint_as_float(v1[col]), y = __uint_as_float(v2[col]);
                const bool sure = x < rc.lo1 && y > rc.hi2, maybe = x < rc.hi1 && y > rc.lo2;
                if (maybe && !sure && h < A.n_hyp && rc.valid) {
                  const int slot = atomicAdd(A.ecount, 1);
                  if (slot < A.ecap) A.elist[slot] = make_int4(p, h, c * kTcCols + wg * kTcWc + hf * 16 + col, 0);
                  else overflow = true;
                }
              }
            }
          }
        }
      }
      // this warpgroup's columns of the row (integer atomics: exact, order-free)
      const int h = ht * kTcRows + lrow;
      if (h < A.n_hyp && rc.valid) {
        if (cert) atomicAdd(A.counts + (size_t)p * A.n_hyp + h, (int)cert);
        if (overflow) {                                            // both warpgroups may overflow one row:
          const unsigned bit = 1u << (h & 31);                     // only the first to set its bit lists it,
          if (!(atomicOr(A.ofl + (size_t)p * ((A.n_hyp + 31) / 32) + (h >> 5), bit) & bit))   // so fix holds
            A.fix[atomicAdd(A.ecount + 1, 1)] = make_int2(p, h);   // <= P * H rows (its capacity)
        }
      }
      it = itn;
      ++k;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTcTmem) : "memory");
  }
}

// The undecided tests, one thread each, with the fp32 formula of the finish kernel (the
// tensor-core count holds the certain inliers; an undecided test that passes adds one) — and
// the safety net, never taken at the configured list capacity: rows whose undecided tests did
// not all fit the list are recounted whole (warp per row) and their listed tests skipped.
__global__ void __launch_bounds__(256) k_score_fix(ScoreTcArgs A) {
  pdl_wait();
  const int n = min(A.ecount[0], A.ecap), nrow = A.ecount[1];
  const int nw = (A.n_hyp + 31) / 32;
  for (int w = blockIdx.x * blockDim.x + threadIdx.x; w < n; w += gridDim.x * blockDim.x) {
    const int4 e = A.elist[w];
    const int p = e.x, h = e.y, m = e.z;
    if (nrow && (A.ofl[(size_t)p * nw + (h >> 5)] >> (h & 31)) & 1u) continue;   // recounted below
    float T[12];
    load_T(A, p, h, T);
    const int fa = A.pairs[2 * p], fb = A.pairs[2 * p + 1];
    const int32_t *mt = A.matches + (size_t)p * A.kp.n_max * 2;
    const int i = mt[2 * m], j = mt[2 * m + 1];
    float4 q0, q1, q2, q3;
    pack_corr(A.kp.pts + ((size_t)fa * A.kp.n_max + i) * 3, A.kp.nrm + ((size_t)fa * A.kp.n_max + i) * 3,
              A.kp.pts + ((size_t)fb * A.kp.n_max + j) * 3, A.kp.nrm + ((size_t)fb * A.kp.n_max + j) * 3, q0, q1, q2, q3);
    if (inlier(T, q0, q1, q2, q3, A.ndelta2, A.ncosa)) atomicAdd(A.counts + (size_t)p * A.n_hyp + h, 1);
  }
  const int lane = threadIdx.x & 31;
  for (int w = blockIdx.x * 8 + (threadIdx.x >> 5); w < nrow; w += gridDim.x * 8) {
    const int2 ph = A.fix[w];
    const int p = ph.x, h = ph.y;
    float T[12];
    load_T(A, p, h, T);
    const int M = A.n_matches[p];
    const int fa = A.pairs[2 * p], fb = A.pairs[2 * p + 1];
    const int32_t *mt = A.matches + (size_t)p * A.kp.n_max * 2;
    const float *pa = A.kp.pts + (size_t)fa * A.kp.n_max * 3, *pb = A.kp.pts + (size_t)fb * A.kp.n_max * 3;
    const float *na = A.kp.nrm + (size_t)fa * A.kp.n_max * 3, *nb = A.kp.nrm + (size_t)fb * A.kp.n_max * 3;
    int cnt = 0;
    for (int m0 = 0; m0 < M; m0 += 32) {
      const int m = m0 + lane;
      bool in = false;
      if (m < M) {
        const int i = mt[2 * m], j = mt[2 * m + 1];
        float4 q0, q1, q2, q3;
        pack_corr(pa + 3 * i, na + 3 * i, pb + 3 * j, nb + 3 * j, q0, q1, q2, q3);
        in = inlier(T, q0, q1, q2, q3, A.ndelta2, A.ncosa);
      }
      cnt += __popc(__ballot_sync(0xffffffffu, in));
    }
    if (lane == 0) A.counts[(size_t)p * A.n_hyp + h] = cnt;
  }
}

}  // namespace

static size_t hyp_slots(int max_pairs, int max_hyp) {
  return (size_t)max_pairs * ((max_hyp + kHypPerBlock - 1) / kHypPerBlock) * kHypPerBlock;
}

static size_t al256(size_t b) { return (b + 255) / 256 * 256; }
int score_m_pad(int n_max) { return (n_max + kTcPad - 1) / kTcPad * kTcPad; }
int score_chunk() { return kTcCols; }

size_t ransac_scratch_bytes(int max_pairs, int max_hyp, int n_max) {
  return al256(hyp_slots(max_pairs, max_hyp) * 48) + al256((size_t)max_pairs * max_hyp * 4) + 256 +
         al256((size_t)max_pairs * score_m_pad(n_max) * kTcFeat * 2) + al256((size_t)max_pairs * sizeof(PairFeat)) +
         al256((size_t)max_pairs * max_hyp * 8) + al256((size_t)max_pairs * max_hyp * 16) +
         al256((size_t)max_pairs * ((max_hyp + 31) / 32) * 4) + 256;
}

RansacScratch carve_ransac_scratch(void *scratch, int max_pairs, int max_hyp, int n_max) {
  RansacScratch r;
  char *c = (char *)scratch;
  r.hyp = c;                      c += al256(hyp_slots(max_pairs, max_hyp) * 48);
  r.counts = (int32_t *)c;        c += al256((size_t)max_pairs * max_hyp * 4);
  r.work = (int32_t *)c;          c += 256;
  r.feat = c;                     c += al256((size_t)max_pairs * score_m_pad(n_max) * kTcFeat * 2);
  r.pfeat = c;                    c += al256((size_t)max_pairs * sizeof(PairFeat));
  r.fix = c;                      c += al256((size_t)max_pairs * max_hyp * 8);
  r.elist = c;                    c += al256((size_t)max_pairs * max_hyp * 16);
  r.ecap = (int)std::min<size_t>((size_t)max_pairs * max_hyp, 0x7fffffff);
  r.ofl = (uint32_t *)c;          c += al256((size_t)max_pairs * ((max_hyp + 31) / 32) * 4);
  r.fix_count = (int32_t *)c;
  r.m_pad = score_m_pad(n_max);
  r.fmap = nullptr;
  return r;
}

void launch_ransac(const KpView &kp, const int32_t *pairs, const uint32_t *uid, int P,
                   const int32_t *matches, const int32_t *n_matches, const bt_ransac_params &prm,
                   const RansacScratch &rs, uint32_t *records, int rec_stride,
                   int32_t *hyp_counts, const bt_pose *node_pose, float huber, cudaStream_t s,
                   Launch &L, const PeerRec *peers) {
  if (P <= 0) return;
  const int chunk = kp.n_max < kMaxChunk ? ((kp.n_max + 31) / 32) * 32 : kMaxChunk;   // multiple of 32
  const size_t smem = (size_t)4 * chunk * sizeof(float4);
  const int score_slots = resident_grid((const void *)k_ransac_score, kScoreThreads, 4 * kMaxChunk * sizeof(float4));
  ScoreArgs a;
  a.hyp = (f32x2 *)rs.hyp;
  a.counts = rs.counts;
  a.work = rs.work;
  a.slices = score_slots * kScoreSlicesPerSlot;
  a.kp = kp; a.pairs = pairs; a.uid = uid; a.matches = matches; a.n_matches = n_matches;
  a.P = P; a.n_hyp = prm.n_hyp; a.nb = (prm.n_hyp + kHypPerBlock - 1) / kHypPerBlock; a.chunk = chunk;
  a.k0 = (uint32_t)(prm.seed & 0xffffffffull); a.k1 = (uint32_t)(prm.seed >> 32);
  a.ndelta2 = (float)(-(double)prm.delta_m * (double)prm.delta_m);
  a.ncosa = -prm.cos_alpha;
  a.tau = prm.min_sigma_ratio;
  const size_t hyp_smem = (size_t)kp.n_max * 6 * sizeof(float);
  smem_optin((const void *)k_ransac_hyp, hyp_smem);
  L.begin(K_RANSAC_HYP, s);
  launch_pdl(k_ransac_hyp, dim3((a.nb * kHypPerBlock / kHypThreads + kHypIter - 1) / kHypIter, P), kHypThreads,
             hyp_smem, s, a);
  L.end(K_RANSAC_HYP, s);
  const char *fma_env = getenv("BT_SCORE_FMA");                  // 1: the FFMA2 kernel (A/B, equality test)
  const bool use_fma = fma_env && fma_env[0] == '1';
  if (use_fma || !rs.fmap) {
    L.begin(K_RANSAC_SCORE, s);
    launch_pdl(k_ransac_score, score_slots, kScoreThreads, smem, s, a);
    L.end(K_RANSAC_SCORE, s);
  } else {
    ScoreTcArgs t;
    t.kp = kp; t.pairs = pairs; t.matches = matches; t.n_matches = n_matches;
    t.P = P; t.n_hyp = prm.n_hyp; t.nb = a.nb; t.nht = (prm.n_hyp + kTcRows - 1) / kTcRows; t.m_pad = rs.m_pad;
    t.ndelta2 = a.ndelta2; t.ncosa = a.ncosa; t.hyp = a.hyp; t.counts = a.counts;
    {
      const double d2 = -(double)a.ndelta2, d = std::sqrt(d2);
      t.sc.delta2 = -a.ndelta2;
      t.sc.cosa = -a.ncosa;
      t.sc.c_rel = (float)((4.0 * 0x1p-22 + 51.0 * 0x1p-23) * 1.01);
      t.sc.e_a = (float)(4.0 * std::sqrt(3.0) * d * 1.0001);
      t.sc.e_b = (float)(0x1p-21 * 5.0 * d2 * 1.0001);
      t.sc.k2 = (float)(40.0 * 0x1p-24 + 0x1p-22 * (1.0 + std::fabs((double)a.ncosa)));
    }
    t.pf = (PairFeat *)rs.pfeat; t.feat = (__half *)rs.feat; t.fix = (int2 *)rs.fix; t.ecount = rs.fix_count;
    t.elist = (int4 *)rs.elist; t.ecap = rs.ecap; t.ofl = rs.ofl;
    if (const char *ec = getenv("BT_SCORE_ECAP")) t.ecap = std::max(0, std::min(t.ecap, atoi(ec)));   // tests: overflow path
    smem_optin((const void *)k_score_tc, kTcSmem);
    const int tc_grid = sm_count() * kTcCtas;                      // kTcCtas CTAs per SM (TMEM split)
    L.begin(K_RANSAC_SCORE, s);
    launch_pdl(k_corr_feat, P, kFeatThreads, 0, s, t);
    L.end(K_RANSAC_SCORE, s);
    L.begin(K_RANSAC_SCORE, s);
    launch_pdl(k_score_tc, std::min(tc_grid, P * t.nht), kTcThreads, kTcSmem, s, *rs.fmap, t);
    L.end(K_RANSAC_SCORE, s);
    L.begin(K_RANSAC_SCORE, s);
    launch_pdl(k_score_fix, 148, 256, 0, s, t);
    L.end(K_RANSAC_SCORE, s);
    if (getenv("BT_SCORE_STATS")) {                                // dev aid (synchronizes): undecided tests
      int32_t c[2] = {0, 0};
      cudaStreamSynchronize(s);
      cudaMemcpy(c, rs.fix_count, 8, cudaMemcpyDeviceToHost);
      fprintf(stderr, "bt scoring: %d undecided tests, %d overflowed rows\n", c[0], c[1]);
    }
  }
  FinishArgs f;
  f.kp = kp; f.pairs = pairs; f.uid = uid; f.matches = matches; f.n_matches = n_matches;
  f.n_hyp = prm.n_hyp; f.min_inliers = prm.min_inliers;
  f.k0 = a.k0; f.k1 = a.k1; f.ndelta2 = a.ndelta2; f.ncosa = a.ncosa; f.tau = a.tau;
  f.counts = a.counts; f.hyp = a.hyp; f.nb = a.nb; f.hyp_counts = hyp_counts; f.records = records; f.rec_stride = rec_stride;
  f.node_pose = node_pose; f.huber = huber;
  if (peers) f.peers = *peers;
  L.begin(K_RANSAC_FINISH, s);
  const size_t fin_smem = (size_t)((mask_words(kp.n_max) * 32 + 3) & ~3) * sizeof(int) +
                          (node_pose ? (size_t)kFeatChunk * kFeatRow * sizeof(float) : 0);
  smem_optin((const void *)k_ransac_finish, fin_smem);
  launch_pdl(k_ransac_finish, dim3(P, node_pose ? 2 : 1), kFinThreads, fin_smem, s, f);
  L.end(K_RANSAC_FINISH, s);
}

}  // namespace bt

namespace bt {
void launch_feature_edges(const KpView &kp, const int32_t *pairs, int P, const int32_t *matches,
                          const int32_t *n_matches, uint32_t *records, int rec_stride, const bt_pose *node_pose,
                          float huber, cudaStream_t s, Launch &L) {
  if (P <= 0) return;
  FeatArgs f;
  f.kp = kp; f.pairs = pairs; f.matches = matches; f.n_matches = n_matches; f.records = records;
  f.rec_stride = rec_stride; f.node_pose = node_pose; f.huber = huber;
  const size_t smem = (size_t)((mask_words(kp.n_max) * 32 + 3) & ~3) * sizeof(int) +
                      (size_t)kFeatChunk * kFeatRow * sizeof(float);
  smem_optin((const void *)k_feature_edges, smem);
  L.begin(K_RANSAC_FINISH, s);
  k_feature_edges<<<P, kFinThreads, smem, s>>>(f);
  L.end(K_RANSAC_FINISH, s);
}
}  // namespace bt
