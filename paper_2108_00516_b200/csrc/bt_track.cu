// bt_track.cu — NEXT-2: the causal tracker's per-frame decisions on the device, so a frame step
// needs no host round trip for them (§IV-B, §IV-C, §IV-E):
//
//  k_coarse_pose  T~_t = T_rel . T_{t-1} (reading R13), T_rel = the consecutive pair's best
//                 sampled hypothesis (record words 4..15); T_{t-1} when the pair has none (status
//                 FEW_MATCHES / FEW_INLIERS).  fp64 products in the oracle's order, rounded.
//  k_select       greedy keyframe selection: one CTA; score_k = geo(k, I_t) + sum over the
//                 selected keyframes of geo(k, q), starting from {I_0}; each round a block argmin
//                 (ties -> lowest pool index) and one geodesic per candidate to the new keyframe.
//                 The pool size is read from device memory, so the call is graph-capturable while
//                 the pool grows.
//  k_admit        pool augmentation: the optimized T_t joins the pool iff its rotation
//                 geodesic to every pool keyframe exceeds the threshold (10 deg, reading R21).
// geo(a, b) = arccos((tr(R_a^T R_b) - 1) / 2) in fp64 with explicit _rn operations in the
// oracle's summation order (no FMA contraction), so the decisions match bto_* bit for bit up to
// acos' last ulp.
#include <cuda_runtime.h>
#include <math_constants.h>

#include "bt_internal.cuh"

namespace bt {
namespace {

constexpr int kSelThreads = 256;

__device__ __forceinline__ double geodesic(const bt_pose &a, const bt_pose &b) {
  double tr = 0.0;
#pragma unroll
  for (int k = 0; k < 9; ++k) tr = __dadd_rn(tr, __dmul_rn((double)a.R[k], (double)b.R[k]));
  double c = __dmul_rn(__dadd_rn(tr, -1.0), 0.5);
  c = c > 1.0 ? 1.0 : (c < -1.0 ? -1.0 : c);
  return acos(c);
}

__global__ void k_coarse_pose(const uint32_t *record, const bt_pose *prev, bt_pose *out) {
  if (threadIdx.x != 0) return;
  const int status = (int)record[kRecStatus];
  const bt_pose P = *prev;
  if (status != BT_PAIR_OK && status != BT_PAIR_REFIT_DEGENERATE) {
    *out = P;
    return;
  }
  float T[12];
#pragma unroll
  for (int k = 0; k < 12; ++k) T[k] = __uint_as_float(record[kRecTBest + k]);
  bt_pose O;
#pragma unroll
  for (int r = 0; r < 3; ++r) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      double x = 0.0;
#pragma unroll
      for (int k = 0; k < 3; ++k) x = __dadd_rn(x, __dmul_rn((double)T[3 * r + k], (double)P.R[3 * k + c]));
      O.R[3 * r + c] = (float)x;
    }
    double y = T[9 + r];
#pragma unroll
    for (int k = 0; k < 3; ++k) y = __dadd_rn(y, __dmul_rn((double)T[3 * r + k], (double)P.t[k]));
    O.t[r] = (float)y;
  }
  *out = O;
}

__global__ void __launch_bounds__(kSelThreads) k_select(const bt_pose *pool, const int32_t *n_pool_p, int cap,
                                                        const bt_pose *cur_p, int K, int32_t *sel, int32_t *n_sel) {
  extern __shared__ double score[];                                   // [cap]; taken: +inf
  __shared__ double red_v[kSelThreads / 32];
  __shared__ int red_i[kSelThreads / 32];
  __shared__ int pick;
  const int n = min(*n_pool_p, cap);
  const bt_pose cur = *cur_p;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int want = min(K, n);
  if (want <= 0) {
    if (threadIdx.x == 0) *n_sel = 0;
    return;
  }
  for (int k = threadIdx.x; k < n; k += kSelThreads) score[k] = geodesic(pool[k], cur);
  __syncthreads();
  int last = 0;                                                       // I_0 first
  if (threadIdx.x == 0) sel[0] = 0;
  for (int s = 1; s < want; ++s) {
    const bt_pose q = pool[last];
    double bv = CUDART_INF;
    int bi = 0x7fffffff;
    for (int k = threadIdx.x; k < n; k += kSelThreads) {
      double v = score[k];
      if (k == last) v = CUDART_INF;                                  // taken
      else if (v < CUDART_INF) v = __dadd_rn(v, geodesic(pool[k], q));
      score[k] = v;
      if (v < bv || (v == bv && k < bi)) { bv = v; bi = k; }
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov < bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
    }
    if (lane == 0) { red_v[warp] = bv; red_i[warp] = bi; }
    __syncthreads();
    if (threadIdx.x == 0) {
      double v = red_v[0];
      int i = red_i[0];
      for (int w = 1; w < kSelThreads / 32; ++w)
        if (red_v[w] < v || (red_v[w] == v && red_i[w] < i)) { v = red_v[w]; i = red_i[w]; }
      pick = i;
      sel[s] = i;
    }
    __syncthreads();
    last = pick;
  }
  if (threadIdx.x == 0) *n_sel = want;
}

__global__ void __launch_bounds__(kSelThreads) k_admit(bt_pose *pool, int32_t *n_pool_p, int cap, const bt_pose *cur_p,
                                                       double thresh, int32_t *admitted) {
  __shared__ int any_close;
  const int n = min(*n_pool_p, cap);
  const bt_pose cur = *cur_p;
  if (threadIdx.x == 0) any_close = 0;
  __syncthreads();
  int close = 0;
  for (int k = threadIdx.x; k < n; k += kSelThreads) close |= !(geodesic(pool[k], cur) > thresh);
  if (close) atomicOr(&any_close, 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    const bool novel = !any_close && n < cap;
    if (novel) {
      pool[n] = cur;
      *n_pool_p = n + 1;
    }
    if (admitted) *admitted = novel ? n : -1;
  }
}

}  // namespace

void launch_coarse_pose(const uint32_t *record, const bt_pose *prev, bt_pose *out, cudaStream_t s, Launch &L) {
  L.begin(K_TRACK, s);
  k_coarse_pose<<<1, 32, 0, s>>>(record, prev, out);
  L.end(K_TRACK, s);
}

void launch_select(const bt_pose *pool, const int32_t *n_pool, int cap, const bt_pose *cur, int K, int32_t *sel,
                   int32_t *n_sel, cudaStream_t s, Launch &L) {
  const size_t smem = (size_t)cap * sizeof(double);
  smem_optin((const void *)k_select, smem);
  L.begin(K_TRACK, s);
  k_select<<<1, kSelThreads, smem, s>>>(pool, n_pool, cap, cur, K, sel, n_sel);
  L.end(K_TRACK, s);
}

void launch_admit(bt_pose *pool, int32_t *n_pool, int cap, const bt_pose *cur, double thresh, int32_t *admitted,
                  cudaStream_t s, Launch &L) {
  L.begin(K_TRACK, s);
  k_admit<<<1, kSelThreads, 0, s>>>(pool, n_pool, cap, cur, thresh, admitted);
  L.end(K_TRACK, s);
}

}  // namespace bt
