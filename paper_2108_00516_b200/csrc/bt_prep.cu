// bt_prep.cu — NEXT-4 input prep: the normal map n_i(x) of Eq. (3) (method
// unspecified; SPEC estimate_normals S:157-165) from the depth map alone.
//
//  k_normals  one thread per 4 x 2 pixel block: float4 loads of rows v-1 .. v+2 (+ the side
//             neighbours), each depth read once from HBM and its re-reads served by L1 / L2 (a
//             shared-memory staged tile measured slower), each row's 12 output floats as three
//             aligned float4 stores.  Central differences of the unprojected cloud,
//               t_u = P(u+1, v) - P(u-1, v),  t_v = P(u, v+1) - P(u, v-1),  n = t_u x t_v,
//             in fp32 with the differences regrouped so the depth differences are exact
//             (Sterbenz): x(u+1) - x(u-1) = ((u - cx)(d_R - d_L) + d_R + d_L) / fx, ...;
//             normalized, flipped to face the camera (n . P < 0).  Invalid (0, 0, 0) at the
//             border, for depth <= 0 at the pixel or a 4-neighbour, and for a neighbour
//             farther than `jump` in depth.  HBM roofline: 4 B read + 12 B written per pixel.
#include <cuda_runtime.h>

#include "bt_internal.cuh"

namespace bt {
namespace {

constexpr int kNormThreads = 256;                 // one thread per 4 horizontally adjacent pixels

struct NormArgs {
  const float *depth;
  float *normal;
  int F, W, H;
  int vec;                                        // W % 4 == 0 and depth 16-B aligned: float4 rows
  float fx, fy, cx, cy, ifx, ify, jump;
};

__device__ __forceinline__ float4 ld4(const float *p) { return __ldg(reinterpret_cast<const float4 *>(p)); }

// normals of 4 horizontally adjacent pixels of row v from the row's depths c[0..5] (c[0], c[5]
// the side neighbours) and the rows above / below
__device__ __forceinline__ void normals4(const NormArgs &A, int v, int ub, const float *c, const float *up,
                                         const float *dn, float *out) {
  const int W = A.W, H = A.H;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int u = ub + k;
    float n0 = 0.f, n1 = 0.f, n2 = 0.f;
    const float d = c[k + 1], dl = c[k], dr = c[k + 2], du = up[k], dd = dn[k];
    const bool ok = u > 0 && u < W - 1 && v > 0 && v < H - 1 && d > 0.f && dl > 0.f && dr > 0.f && du > 0.f &&
                    dd > 0.f && !(fabsf(dl - d) > A.jump) && !(fabsf(dr - d) > A.jump) &&
                    !(fabsf(du - d) > A.jump) && !(fabsf(dd - d) > A.jump);
    if (ok) {
      const float xu = (float)u - A.cx, yv = (float)v - A.cy;
      const float dh = dr - dl, dvv = dd - du;                    // exact (Sterbenz)
      const float tu0 = fmaf(xu, dh, dr + dl) * A.ifx, tu1 = yv * dh * A.ify, tu2 = dh;
      const float tv0 = xu * dvv * A.ifx, tv1 = fmaf(yv, dvv, dd + du) * A.ify, tv2 = dvv;
      const float m0 = tu1 * tv2 - tu2 * tv1, m1 = tu2 * tv0 - tu0 * tv2, m2 = tu0 * tv1 - tu1 * tv0;
      const float nn = m0 * m0 + m1 * m1 + m2 * m2;
      if (nn > 0.f) {
        const float px = xu * d * A.ifx, py = yv * d * A.ify;
        float s = rsqrtf(nn);
        if (m0 * px + m1 * py + m2 * d > 0.f) s = -s;
        n0 = m0 * s; n1 = m1 * s; n2 = m2 * s;
      }
    }
    out[3 * k] = n0; out[3 * k + 1] = n1; out[3 * k + 2] = n2;
  }
}

// a warp's 32 x 12 output floats: when its 4-pixel groups are consecutive in memory, staged in
// shared memory and written as three fully contiguous 512-byte float4 stores (direct 48-byte
// strided stores would hit every 32-byte sector with partial writes)
__device__ __forceinline__ void store4(const NormArgs &A, int f, int v, int ub, const float *out, float4 *stg,
                                       bool active) {
  const int W = A.W, lane = threadIdx.x & 31;
  const size_t pix = (size_t)f * W * A.H + (size_t)v * W + ub;
  float *dst = A.normal + 3 * pix;
  const unsigned m = __activemask();
  const size_t pix0 = __shfl_sync(m, pix, 0);
  const bool contig = m == 0xffffffffu && (W & 3) == 0 &&
                      __all_sync(m, active && pix == pix0 + 4 * (size_t)lane);
  if (contig) {
    stg[3 * lane] = make_float4(out[0], out[1], out[2], out[3]);
    stg[3 * lane + 1] = make_float4(out[4], out[5], out[6], out[7]);
    stg[3 * lane + 2] = make_float4(out[8], out[9], out[10], out[11]);
    __syncwarp();
    float4 *base = reinterpret_cast<float4 *>(A.normal + 3 * pix0);
#pragma unroll
    for (int i = 0; i < 3; ++i) __stcs(base + 32 * i + lane, stg[32 * i + lane]);
    __syncwarp();
    return;
  }
  if (!active) return;
  if ((W & 3) == 0) {
    float4 *d4 = reinterpret_cast<float4 *>(dst);
    d4[0] = make_float4(out[0], out[1], out[2], out[3]);
    d4[1] = make_float4(out[4], out[5], out[6], out[7]);
    d4[2] = make_float4(out[8], out[9], out[10], out[11]);
  } else {
    for (int k = 0; k < 4 && ub + k < W; ++k)
      for (int q = 0; q < 3; ++q) dst[3 * k + q] = out[3 * k + q];
  }
}

// row r of frame D: 4 depths at ub.. (zero outside) + the 2 side neighbours in c[0], c[5]
__device__ __forceinline__ void load_row(const float *D, int W, int H, int r, int ub, bool vec, float *c) {
  if (r < 0 || r >= H) {
#pragma unroll
    for (int k = 0; k < 6; ++k) c[k] = 0.f;
    return;
  }
  const float *row = D + (size_t)r * W;
  if (vec) {
    const float4 x = ld4(row + ub);
    c[1] = x.x; c[2] = x.y; c[3] = x.z; c[4] = x.w;
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k) c[k + 1] = ub + k < W ? __ldg(row + ub + k) : 0.f;
  }
  c[0] = ub > 0 ? __ldg(row + ub - 1) : 0.f;
  c[5] = ub + 4 < W ? __ldg(row + ub + 4) : 0.f;
}

// one thread per 4 x 2 pixel block: rows v-1 .. v+2 loaded once, two rows of normals out
__global__ void __launch_bounds__(kNormThreads) k_normals(NormArgs A) {
  __shared__ float4 stage[kNormThreads / 32][96];
  const int W = A.W, H = A.H, W4 = (W + 3) >> 2, H2 = (H + 1) >> 1;
  const size_t g = (size_t)blockIdx.x * kNormThreads + threadIdx.x;
  const int f0 = (int)(g / ((size_t)W4 * H2));
  const bool live = f0 < A.F;                                      // warps stay converged for the stores
  const int f = live ? f0 : A.F - 1;
  const int rem = (int)(g - (size_t)f0 * W4 * H2);
  const int v = live ? (rem / W4) * 2 : 0, ub = live ? (rem - (rem / W4) * W4) * 4 : 0;
  const float *D = A.depth + (size_t)f * W * H;
  float r0[6], r1[6], r2[6], r3[6], out[12];
  load_row(D, W, H, v - 1, ub, A.vec, r0);
  load_row(D, W, H, v, ub, A.vec, r1);
  load_row(D, W, H, v + 1, ub, A.vec, r2);
  load_row(D, W, H, v + 2, ub, A.vec, r3);
  float4 *stg = stage[threadIdx.x >> 5];
  normals4(A, v, ub, r1, r0 + 1, r2 + 1, out);
  store4(A, f, v, ub, out, stg, live);
  normals4(A, v + 1, ub, r2, r1 + 1, r3 + 1, out);
  store4(A, f, v + 1, ub, out, stg, live && v + 1 < H);
}

}  // namespace

void launch_normals(const float *depth, int F, int W, int H, const bt_intrinsics &K, float jump, float *normal,
                    cudaStream_t s, Launch &L) {
  if (F <= 0 || W <= 0 || H <= 0) return;
  NormArgs a;
  a.depth = depth; a.normal = normal; a.F = F; a.W = W; a.H = H;
  a.vec = (W % 4 == 0) && ((uintptr_t)depth % 16 == 0);
  a.fx = K.fx; a.fy = K.fy; a.cx = K.cx; a.cy = K.cy;
  a.ifx = 1.0f / K.fx; a.ify = 1.0f / K.fy; a.jump = jump;
  L.begin(K_NORMALS, s);
  const size_t groups = (size_t)F * ((H + 1) / 2) * ((W + 3) / 4);
  k_normals<<<(unsigned)((groups + kNormThreads - 1) / kNormThreads), kNormThreads, 0, s>>>(a);
  L.end(K_NORMALS, s);
}

}  // namespace bt
