// bt_match.cu — mutual nearest-neighbour descriptor matching (P:4 "feature matching",
// P:25 "n keypoints ... feature descriptor D_i in R^128"), readings R1-R4 of DESIGN.md:
// squared Euclidean distance, ties -> lowest index, mutual NN, optional Lowe ratio,
// output ascending in i.
//
// Exact fp32 distances on the FP32 pipe, one warp per query descriptor:
//   lane l owns descriptor words [4l, 4l+4) (one LDG.128 per reference descriptor, a warp
//   reads 512 contiguous bytes); 32 reference descriptors are processed per step and their
//   32 lane-partials are combined by a 5-level "transpose reduction" (31 shuffles for 32
//   sums) after which lane l holds the distance to reference j0 + l.  The summation order
//   (4 sequential terms per lane, then a fixed binary tree) is the same for every (i, j).
#include <cuda_runtime.h>
#include <math_constants.h>

#include "bt_internal.cuh"

namespace bt {
namespace {

constexpr int kWarpsPerBlock = 8;

__device__ __forceinline__ void top2_update(float d, int j, float &b1, int &j1, float &b2) {
  if (d < b1) { b2 = b1; b1 = d; j1 = j; }
  else if (d < b2) { b2 = d; }
}

// nn[p][q] = argmin_r d(query q, reference r) for queries of frame pairs[p][dir] against
// references of frame pairs[p][1-dir]; for dir == 0 also the ratio-test flag.
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
k_nearest(KpView kp, const int32_t *__restrict__ pairs, int dir, float ratio2,
          int32_t *__restrict__ nn, uint8_t *__restrict__ ratio_ok) {
  const int p = blockIdx.y;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int fq = pairs[2 * p + dir], fr = pairs[2 * p + 1 - dir];
  const int nq = min(kp.n_kp[fq], kp.n_max), nr = min(kp.n_kp[fr], kp.n_max);
  const int q = blockIdx.x * kWarpsPerBlock + warp;
  if (q >= nq) return;                                           // warp-uniform
  const float4 a = reinterpret_cast<const float4 *>(kp.desc + ((size_t)fq * kp.n_max + q) * kDim)[lane];
  const float4 *R = reinterpret_cast<const float4 *>(kp.desc + (size_t)fr * kp.n_max * kDim);
  float b1 = CUDART_INF_F, b2 = CUDART_INF_F;
  int j1 = -1;
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
    // transpose reduction: after the step with offset o, lane keeps the half of its
    // columns selected by (lane & o) and adds the partner's copy of that half.
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
      const bool upper = (lane & o) != 0;
#pragma unroll
      for (int c = 0; c < o; ++c) {
        const float send = upper ? v[c] : v[c + o];
        const float keep = upper ? v[c + o] : v[c];
        const float recv = __shfl_xor_sync(0xffffffffu, send, o);
        v[c] = __fadd_rn(keep, recv);
      }
    }
    const int j = j0 + lane;                                      // column owned by this lane
    if (j < nr) top2_update(v[0], j, b1, j1, b2);
  }
  // warp merge of (best, index, second) with ties -> lowest index
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    const float ob1 = __shfl_xor_sync(0xffffffffu, b1, o);
    const int oj1 = __shfl_xor_sync(0xffffffffu, j1, o);
    const float ob2 = __shfl_xor_sync(0xffffffffu, b2, o);
    const bool mine = (b1 < ob1) || (b1 == ob1 && (unsigned)j1 < (unsigned)oj1);
    if (mine) { b2 = fminf(b2, ob1); }
    else { b2 = fminf(ob2, b1); b1 = ob1; j1 = oj1; }
  }
  if (lane == 0) {
    nn[(size_t)p * kp.n_max + q] = j1;
    if (dir == 0) ratio_ok[(size_t)p * kp.n_max + q] = (ratio2 >= 1.f) || (nr < 2) || (b1 < ratio2 * b2);
  }
}

// keep (i, nn_ab(i)) iff nn_ba(nn_ab(i)) == i (and the ratio flag); compact ascending in i
__global__ void __launch_bounds__(1024)
k_mutual(KpView kp, const int32_t *__restrict__ pairs, const int32_t *__restrict__ nn_ab,
         const int32_t *__restrict__ nn_ba, const uint8_t *__restrict__ ratio_ok,
         int32_t *__restrict__ matches, int32_t *__restrict__ n_matches) {
  __shared__ int warp_tot[32];
  const int p = blockIdx.x;
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

}  // namespace

void launch_match(const KpView &kp, const int32_t *pairs, int P, float ratio, int32_t *nn_ab,
                  int32_t *nn_ba, uint8_t *ratio_ok, int32_t *matches, int32_t *n_matches,
                  cudaStream_t s, Launch &L) {
  if (P <= 0) return;
  const float ratio2 = ratio >= 1.f ? 1.f : ratio * ratio;
  dim3 grid((kp.n_max + kWarpsPerBlock - 1) / kWarpsPerBlock, P);
  L.begin(K_NEAREST, s);
  k_nearest<<<grid, kWarpsPerBlock * 32, 0, s>>>(kp, pairs, 0, ratio2, nn_ab, ratio_ok);
  L.end(K_NEAREST, s);
  L.begin(K_NEAREST, s);
  k_nearest<<<grid, kWarpsPerBlock * 32, 0, s>>>(kp, pairs, 1, ratio2, nn_ba, nullptr);
  L.end(K_NEAREST, s);
  L.begin(K_MUTUAL, s);
  k_mutual<<<P, 512, 0, s>>>(kp, pairs, nn_ab, nn_ba, ratio_ok, matches, n_matches);
  L.end(K_MUTUAL, s);
}

}  // namespace bt
