// bt_dense.cu — dense geometric edges of Eq. (3):
//   E_g(i,j) = sum_{p in I_i} rho( n_i(x) . (T_i T_j^-1 pi_D^-1(pi(T_j T_i^-1 p)) - p) ),
// "dense pixel-wise correspondences are associated by point re-projection, while outliers
// are filtered based on the distance between the point pair and the angle formed by their
// normals".  Readings: nearest pixel (R14), gates (R15), normals compared in camera i (R16),
// Huber (R17), J = [n_i^T, (q x n_i)^T] for the left perturbation of T_i (R18).
//
// k_dense: one CTA per (edge, span of 256 x kPix pixels): coalesced reads of the source
// mask / depth / normal rows, the gathered target pixel, and 29 running fp32 sums per
// thread (H 21, g 6, E, count) reduced by warp shuffles + shared memory into one partial
// per CTA.  k_dense_reduce: fixed-order fp64 sum of the partials of an edge (bitwise
// deterministic, no float atomics).
#include <cuda_runtime.h>

#include "bt_internal.cuh"

namespace bt {
namespace {

constexpr int kDenseThreads = 256;
constexpr int kPix = 8;                       // pixels per thread
constexpr int kAcc = 29;                      // H 21, g 6, E, count
constexpr int kPartStride = 32;

struct DenseArgs {
  MapView mp;
  float fx, fy, cx, cy, ifx, ify;
  double cxd, cyd, ifxd, ifyd;
  const bt_pose *node_pose;
  const int32_t *edges;       // [E][2] or null (then derived from pairs)
  const int32_t *pairs;
  int E, stride;
  float gate2, cos_gate, huber;
  float *partials;            // [E][nblk][32]
  int nblk;
};

__device__ __forceinline__ void edge_frames(const DenseArgs &A, int e, int &fi, int &fj) {
  if (A.edges) { fi = A.edges[2 * e]; fj = A.edges[2 * e + 1]; }
  else {
    const int p = e >> 1;
    fi = A.pairs[2 * p + (e & 1)];
    fj = A.pairs[2 * p + 1 - (e & 1)];
  }
}

__global__ void __launch_bounds__(kDenseThreads) k_dense(DenseArgs A) {
  __shared__ float C[24];                     // Rji(9) tji(3) Rij(9) tij(3)
  __shared__ double Cd[12];                   // Rij(9) tij(3) in fp64 for the residual
  __shared__ float red[kDenseThreads / 32][kAcc];
  const int e = blockIdx.y;
  int fi, fj;
  edge_frames(A, e, fi, fj);
  if (threadIdx.x == 0) {
    // T_j T_i^-1: R = R_j R_i^T, t = t_j - R t_i ;  T_i T_j^-1: R = R_i R_j^T, t = t_i - R t_j
    const bt_pose Pi = A.node_pose[fi], Pj = A.node_pose[fj];
    double Rji[9], Rij[9];
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) {
        double x = 0, y = 0;
        for (int k = 0; k < 3; ++k) {
          x += (double)Pj.R[3 * r + k] * Pi.R[3 * c + k];
          y += (double)Pi.R[3 * r + k] * Pj.R[3 * c + k];
        }
        Rji[3 * r + c] = x;
        Rij[3 * r + c] = y;
      }
    for (int k = 0; k < 9; ++k) { C[k] = (float)Rji[k]; C[12 + k] = (float)Rij[k]; Cd[k] = Rij[k]; }
    for (int r = 0; r < 3; ++r) {
      C[9 + r] = (float)(Pj.t[r] - (Rji[3 * r] * Pi.t[0] + Rji[3 * r + 1] * Pi.t[1] + Rji[3 * r + 2] * Pi.t[2]));
      Cd[9 + r] = Pi.t[r] - (Rij[3 * r] * Pj.t[0] + Rij[3 * r + 1] * Pj.t[1] + Rij[3 * r + 2] * Pj.t[2]);
      C[21 + r] = (float)Cd[9 + r];
    }
  }
  __syncthreads();
  float Rji[9], tji[3], Rij[9], tij[3];
#pragma unroll
  for (int k = 0; k < 9; ++k) { Rji[k] = C[k]; Rij[k] = C[12 + k]; }
#pragma unroll
  for (int k = 0; k < 3; ++k) { tji[k] = C[9 + k]; tij[k] = C[21 + k]; }

  const int W = A.mp.W, H = A.mp.H, npx = W * H;
  const size_t off_i = (size_t)fi * npx, off_j = (size_t)fj * npx;
  const float *dep_i = A.mp.depth + off_i, *dep_j = A.mp.depth + off_j;
  const float *nor_i = A.mp.normal + 3 * off_i, *nor_j = A.mp.normal + 3 * off_j;
  const uint8_t *msk_i = A.mp.mask + off_i, *msk_j = A.mp.mask + off_j;

  float acc[kAcc];
#pragma unroll
  for (int k = 0; k < kAcc; ++k) acc[k] = 0.f;
  const int base = blockIdx.x * kDenseThreads * kPix;
#pragma unroll 1
  for (int it = 0; it < kPix; ++it) {
    const int pix = base + it * kDenseThreads + threadIdx.x;
    if (pix >= npx) break;
    const int v = pix / W, u = pix - v * W;
    if (A.stride > 1 && (u % A.stride || v % A.stride)) continue;
    if (!msk_i[pix]) continue;
    const float d = dep_i[pix];
    const float n0 = nor_i[3 * pix], n1 = nor_i[3 * pix + 1], n2 = nor_i[3 * pix + 2];
    if (!(d > 0.f) || (n0 == 0.f && n1 == 0.f && n2 == 0.f)) continue;
    // p = pi^-1(x, d)
    const float px = ((float)u - A.cx) * d * A.ifx, py = ((float)v - A.cy) * d * A.ify, pz = d;
    // y = T_j T_i^-1 p
    const float yx = fmaf(Rji[0], px, fmaf(Rji[1], py, fmaf(Rji[2], pz, tji[0])));
    const float yy = fmaf(Rji[3], px, fmaf(Rji[4], py, fmaf(Rji[5], pz, tji[1])));
    const float yz = fmaf(Rji[6], px, fmaf(Rji[7], py, fmaf(Rji[8], pz, tji[2])));
    if (!(yz > 0.f)) continue;
    const float iz = 1.0f / yz;
    const float up = fmaf(A.fx * yx, iz, A.cx), vp = fmaf(A.fy * yy, iz, A.cy);
    const float xu = floorf(up + 0.5f), xv = floorf(vp + 0.5f);
    if (!(xu >= 0.f && xu < (float)W && xv >= 0.f && xv < (float)H)) continue;
    const int uj = (int)xu, vj = (int)xv, pj = vj * W + uj;
    if (!msk_j[pj]) continue;
    const float dj = dep_j[pj];
    const float m0 = nor_j[3 * pj], m1 = nor_j[3 * pj + 1], m2 = nor_j[3 * pj + 2];
    if (!(dj > 0.f) || (m0 == 0.f && m1 == 0.f && m2 == 0.f)) continue;
    // s = pi_D^-1(x'), q = T_i T_j^-1 s, n_j in camera i
    const float sx = ((float)uj - A.cx) * dj * A.ifx, sy = ((float)vj - A.cy) * dj * A.ify, sz = dj;
    const float qx = fmaf(Rij[0], sx, fmaf(Rij[1], sy, fmaf(Rij[2], sz, tij[0])));
    const float qy = fmaf(Rij[3], sx, fmaf(Rij[4], sy, fmaf(Rij[5], sz, tij[1])));
    const float qz = fmaf(Rij[6], sx, fmaf(Rij[7], sy, fmaf(Rij[8], sz, tij[2])));
    const float k0 = fmaf(Rij[0], m0, fmaf(Rij[1], m1, Rij[2] * m2));
    const float k1 = fmaf(Rij[3], m0, fmaf(Rij[4], m1, Rij[5] * m2));
    const float k2 = fmaf(Rij[6], m0, fmaf(Rij[7], m1, Rij[8] * m2));
    const float dx = qx - px, dy = qy - py, dz = qz - pz;
    const float dist2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
    const float c = fmaf(n0, k0, fmaf(n1, k1, n2 * k2));
    if (!(dist2 < A.gate2 && c > A.cos_gate)) continue;
    // the point-to-plane residual cancels two ~0.5 m positions down to ~1e-5 m near the
    // optimum: evaluate it in fp64 (B200 FP64 runs at half the FP32 rate)
    double r_d;
    {
      const double pxd = ((double)u - A.cxd) * (double)d * A.ifxd, pyd = ((double)v - A.cyd) * (double)d * A.ifyd;
      const double sxd = ((double)uj - A.cxd) * (double)dj * A.ifxd, syd = ((double)vj - A.cyd) * (double)dj * A.ifyd;
      const double szd = dj;
      const double qxd = fma(Cd[0], sxd, fma(Cd[1], syd, fma(Cd[2], szd, Cd[9])));
      const double qyd = fma(Cd[3], sxd, fma(Cd[4], syd, fma(Cd[5], szd, Cd[10])));
      const double qzd = fma(Cd[6], sxd, fma(Cd[7], syd, fma(Cd[8], szd, Cd[11])));
      r_d = fma((double)n0, qxd - pxd, fma((double)n1, qyd - pyd, (double)n2 * (qzd - (double)d)));
    }
    const float r = (float)r_d;
    const float ar = fabsf(r);
    const float w = ar <= A.huber ? 1.f : A.huber / ar;
    const float rho = ar <= A.huber ? 0.5f * r * r : A.huber * (ar - 0.5f * A.huber);
    const float J[6] = {n0, n1, n2, qy * n2 - qz * n1, qz * n0 - qx * n2, qx * n1 - qy * n0};
    int k = 0;
#pragma unroll
    for (int a = 0; a < 6; ++a) {
      const float wa = w * J[a];
#pragma unroll
      for (int b = a; b < 6; ++b) { acc[k] = fmaf(wa, J[b], acc[k]); ++k; }
    }
#pragma unroll
    for (int a = 0; a < 6; ++a) acc[21 + a] = fmaf(w * J[a], r, acc[21 + a]);
    acc[27] += rho;
    acc[28] += 1.f;
  }
  // block reduction (fixed order)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < kAcc; ++k) {
    float x = acc[k];
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if (lane == 0) red[warp][k] = x;
  }
  __syncthreads();
  if (threadIdx.x < kAcc) {
    float t = 0.f;
#pragma unroll
    for (int w = 0; w < kDenseThreads / 32; ++w) t += red[w][threadIdx.x];
    A.partials[((size_t)e * A.nblk + blockIdx.x) * kPartStride + threadIdx.x] = t;
  }
}

__global__ void k_dense_reduce(const float *__restrict__ partials, int nblk, int E, const int32_t *edges,
                               float *out, int out_stride, uint32_t *records, int rec_stride,
                               int off_ij, int off_ji) {
  const int e = blockIdx.x;
  const int k = threadIdx.x;                  // 32 threads
  double t = 0.0;
  if (k < kAcc)
    for (int b = 0; b < nblk; ++b) t += (double)partials[((size_t)e * nblk + b) * kPartStride + k];
  const float v = k < kAcc ? (float)t : 0.f;
  if (records) {
    const int p = e >> 1;
    records[(size_t)p * rec_stride + ((e & 1) ? off_ji : off_ij) + k] = __float_as_uint(v);
  } else {
    out[(size_t)e * out_stride + k] = v;
  }
  (void)E; (void)edges;
}

__global__ void k_compose(const bt_pose *a, const bt_pose *b, bt_pose *out, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const bt_pose A = a[i], B = b[i];
  bt_pose O;
  for (int r = 0; r < 3; ++r) {
    for (int c = 0; c < 3; ++c) {
      double x = 0;
      for (int k = 0; k < 3; ++k) x += (double)A.R[3 * r + k] * B.R[3 * k + c];
      O.R[3 * r + c] = (float)x;
    }
    O.t[r] = (float)((double)A.R[3 * r] * B.t[0] + (double)A.R[3 * r + 1] * B.t[1] +
                     (double)A.R[3 * r + 2] * B.t[2] + A.t[r]);
  }
  out[i] = O;
}

}  // namespace

int dense_partials_per_edge(int W, int H) {
  return (W * H + kDenseThreads * kPix - 1) / (kDenseThreads * kPix);
}

void launch_dense(const MapView &mp, const bt_intrinsics &K, const bt_pose *node_pose,
                  const int32_t *edges, const int32_t *pairs, int E, const bt_edge_params &prm,
                  float *partials, int max_partials_per_edge, float *out, int out_stride,
                  uint32_t *records, int rec_stride, int rec_off_ij, int rec_off_ji,
                  cudaStream_t s, Launch &L) {
  if (E <= 0) return;
  DenseArgs a;
  a.mp = mp;
  a.fx = K.fx; a.fy = K.fy; a.cx = K.cx; a.cy = K.cy;
  a.ifx = 1.0f / K.fx; a.ify = 1.0f / K.fy;
  a.cxd = K.cx; a.cyd = K.cy; a.ifxd = 1.0 / (double)K.fx; a.ifyd = 1.0 / (double)K.fy;
  a.node_pose = node_pose; a.edges = edges; a.pairs = pairs; a.E = E;
  a.stride = prm.stride < 1 ? 1 : prm.stride;
  a.gate2 = (float)((double)prm.dist_gate_m * (double)prm.dist_gate_m);
  a.cos_gate = prm.cos_gate;
  a.huber = prm.huber_m;
  a.partials = partials;
  a.nblk = dense_partials_per_edge(mp.W, mp.H);
  (void)max_partials_per_edge;
  dim3 grid(a.nblk, E);
  L.begin(K_DENSE, s);
  k_dense<<<grid, kDenseThreads, 0, s>>>(a);
  L.end(K_DENSE, s);
  L.begin(K_DENSE_REDUCE, s);
  k_dense_reduce<<<E, 32, 0, s>>>(partials, a.nblk, E, edges, out, out_stride, records, rec_stride,
                                  rec_off_ij, rec_off_ji);
  L.end(K_DENSE_REDUCE, s);
}

void launch_compose(const bt_pose *a, const bt_pose *b, bt_pose *out, int n, cudaStream_t s,
                    Launch &L) {
  if (n <= 0) return;
  L.begin(K_COMPOSE, s);
  k_compose<<<(n + 127) / 128, 128, 0, s>>>(a, b, out, n);
  L.end(K_COMPOSE, s);
}

}  // namespace bt
