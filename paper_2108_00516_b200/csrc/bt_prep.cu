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
//
//  k_lift     NEXT-4 keypoint lifting (reading R29; P:25 keypoints x_i + D_i, P:72 pi_D^-1 "looking
//             up the depth value on the pixel location", SPEC S:247 / S:262): one CTA per frame,
//             a thread per keypoint in blocks of kLiftThreads: nearest pixel (floor(u + 0.5)),
//             validity (in frame, mask, depth > 0, normal != 0), block-scan compaction in input
//             order, the point in fp64 ((u - cx) d / fx, (v - cy) d / fy, d) rounded to fp32 and
//             the pixel's normal; then each warp copies its lanes' kept descriptors (128 floats
//             as one float4 per lane, coalesced).  HBM: 8 B (uv) + 512 B (desc) read and 512 +
//             24 B written per keypoint + 17 B of map lookups.
#include <cuda_runtime.h>

#include "bt_internal.cuh"

namespace bt {
namespace {

constexpr int kLiftThreads = 512;
constexpr int kLiftSplit = 8;                      // CTAs per frame, each writing 1/8 of the output slots

struct LiftArgs {
  int F, n_max, W, H, span;                        // span = output slots per CTA
  const float *uv, *desc_in;
  const int32_t *n_in;
  MapView mp;
  double fx, fy, cx, cy;
  int32_t *n_out;
  float *desc, *pts, *nrm;
};

// grid (F, kLiftSplit): every CTA of a frame evaluates all of the frame's keypoints (8 B of uv +
// 17 B of map lookups each: cheap) and their output slots (block scan in input order), but writes
// only the slots [lo, lo + span) — so the 512-B descriptor copies spread over F x 8 CTAs with
// several rows in flight per warp instead of one frame's rows serialised in one CTA
__global__ void __launch_bounds__(kLiftThreads) k_lift(LiftArgs A) {
  extern __shared__ int src_of[];                  // [span] input index of each of this CTA's slots
  __shared__ int wsum[kLiftThreads / 32];
  const int f = blockIdx.x, lo = blockIdx.y * A.span, hi = lo + A.span;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int n = min(A.n_in[f], A.n_max);
  const size_t fpx = (size_t)f * A.W * A.H;
  int base = 0;
  for (int k0 = 0; k0 < n; k0 += kLiftThreads) {
    const int k = k0 + threadIdx.x;
    bool keep = false;
    float p0 = 0.f, p1 = 0.f, p2 = 0.f, m0 = 0.f, m1 = 0.f, m2 = 0.f;
    if (k < n) {
      const float2 uv = __ldg(reinterpret_cast<const float2 *>(A.uv) + (size_t)f * A.n_max + k);
      const double u = uv.x, v = uv.y;
      const double xu = floor(u + 0.5), xv = floor(v + 0.5);      // nearest pixel (R14)
      if (xu >= 0.0 && xu < (double)A.W && xv >= 0.0 && xv < (double)A.H) {
        const size_t px = fpx + (size_t)xv * A.W + (size_t)xu;
        const float d = __ldg(A.mp.depth + px);
        m0 = __ldg(A.mp.normal + 3 * px); m1 = __ldg(A.mp.normal + 3 * px + 1); m2 = __ldg(A.mp.normal + 3 * px + 2);
        keep = A.mp.mask[px] != 0 && d > 0.f && !(m0 == 0.f && m1 == 0.f && m2 == 0.f);
        const double dd = d;
        p0 = (float)__ddiv_rn(__dmul_rn(__dsub_rn(u, A.cx), dd), A.fx);   // pi_D^-1 at the keypoint
        p1 = (float)__ddiv_rn(__dmul_rn(__dsub_rn(v, A.cy), dd), A.fy);
        p2 = d;
      }
    }
    const unsigned bal = __ballot_sync(0xffffffffu, keep);        // block scan in input order
    if (lane == 0) wsum[warp] = __popc(bal);
    __syncthreads();
    int off = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < kLiftThreads / 32; ++w) { off += w < warp ? wsum[w] : 0; tot += wsum[w]; }
    const int slot = base + off + __popc(bal & ((1u << lane) - 1u));
    if (keep && slot >= lo && slot < hi) {
      const size_t o = (size_t)f * A.n_max + slot;
      A.pts[3 * o] = p0; A.pts[3 * o + 1] = p1; A.pts[3 * o + 2] = p2;
      A.nrm[3 * o] = m0; A.nrm[3 * o + 1] = m1; A.nrm[3 * o + 2] = m2;
      src_of[slot - lo] = k;
    }
    base += tot;
    __syncthreads();                                               // wsum reused
  }
  if (blockIdx.y == 0 && threadIdx.x == 0) A.n_out[f] = base;
  // this CTA's descriptor rows: warp w copies rows w, w + 16, ... four at a time (loads in flight)
  const int rows = max(0, min(hi, base) - lo);
  constexpr int kW = kLiftThreads / 32;
  for (int r0 = warp; r0 < rows; r0 += 4 * kW) {
    float4 x[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int r = r0 + q * kW;
      if (r < rows)
        x[q] = __ldg(reinterpret_cast<const float4 *>(A.desc_in + ((size_t)f * A.n_max + src_of[r]) * kDim) + lane);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int r = r0 + q * kW;
      if (r < rows) reinterpret_cast<float4 *>(A.desc + ((size_t)f * A.n_max + lo + r) * kDim)[lane] = x[q];
    }
  }
}

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

void launch_lift(int F, int n_max, const float *uv, const float *desc_in, const int32_t *n_in, const MapView &mp,
                 const bt_intrinsics &K, int32_t *n_out, float *desc, float *pts, float *nrm, cudaStream_t s,
                 Launch &L) {
  if (F <= 0) return;
  LiftArgs a;
  a.F = F; a.n_max = n_max; a.W = mp.W; a.H = mp.H;
  a.uv = uv; a.desc_in = desc_in; a.n_in = n_in; a.mp = mp;
  a.fx = K.fx; a.fy = K.fy; a.cx = K.cx; a.cy = K.cy;
  a.n_out = n_out; a.desc = desc; a.pts = pts; a.nrm = nrm;
  a.span = (n_max + kLiftSplit - 1) / kLiftSplit;
  L.begin(K_NORMALS, s);
  k_lift<<<dim3(F, kLiftSplit), kLiftThreads, (size_t)a.span * sizeof(int), s>>>(a);
  L.end(K_NORMALS, s);
}

// uint16 depth (the sensor format) -> metres: (float)v * scale, one fp32 rounding; 8 pixels per
// thread (16-B load, two 16-B stores) where the buffers are 16-B aligned, else one.  HBM-bound
// (2 B read + 4 B written per pixel).
__global__ void __launch_bounds__(256) k_depth_u16(const uint16_t *__restrict__ in, float scale, size_t n,
                                                   float *__restrict__ out, int vec) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (vec) {
    for (; 8 * i + 7 < n; i += stride) {
      const uint4 w = __ldg(reinterpret_cast<const uint4 *>(in) + i);
      const unsigned u[4] = {w.x, w.y, w.z, w.w};
      float o[8];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        o[2 * k] = __fmul_rn((float)(u[k] & 0xffffu), scale);
        o[2 * k + 1] = __fmul_rn((float)(u[k] >> 16), scale);
      }
      reinterpret_cast<float4 *>(out)[2 * i] = make_float4(o[0], o[1], o[2], o[3]);
      reinterpret_cast<float4 *>(out)[2 * i + 1] = make_float4(o[4], o[5], o[6], o[7]);
    }
    for (size_t j = (n & ~(size_t)7) + (size_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += stride)
      out[j] = __fmul_rn((float)in[j], scale);
  } else {
    for (; i < n; i += stride) out[i] = __fmul_rn((float)in[i], scale);
  }
}

// packed-bit mask rows (ceil(W / 8) bytes, LSB first) -> one byte per pixel: a thread per
// output byte group of 8 pixels (one input byte), 8-B stores where the row allows
__global__ void __launch_bounds__(256) k_mask_bits(const uint8_t *__restrict__ bits, int W, size_t rows, int rb,
                                                   uint8_t *__restrict__ mask) {
  const size_t n = rows * (size_t)rb, st = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += st) {
    const size_t row = i / rb;
    const int u0 = (int)(i - row * rb) * 8;
    const unsigned b = bits[i];
    uint8_t *o = mask + row * (size_t)W + u0;
    if (u0 + 8 <= W && ((uintptr_t)o & 7) == 0) {
      unsigned lo = 0, hi = 0;
#pragma unroll
      for (int k = 0; k < 4; ++k) { lo |= ((b >> k) & 1u) << (8 * k); hi |= ((b >> (4 + k)) & 1u) << (8 * k); }
      *reinterpret_cast<uint2 *>(o) = make_uint2(lo, hi);
    } else {
      for (int k = 0; k < 8 && u0 + k < W; ++k) o[k] = (uint8_t)((b >> k) & 1u);
    }
  }
}

void launch_mask_bits(const uint8_t *bits, int F, int W, int H, uint8_t *mask, cudaStream_t s, Launch &L) {
  if (F <= 0 || W <= 0 || H <= 0) return;
  L.begin(K_NORMALS, s);
  k_mask_bits<<<sm_count() * 8, 256, 0, s>>>(bits, W, (size_t)F * H, (W + 7) / 8, mask);
  L.end(K_NORMALS, s);
}

void launch_depth_u16(const uint16_t *in, float scale, size_t n, float *out, cudaStream_t s, Launch &L) {
  if (n == 0) return;
  const int vec = ((uintptr_t)in % 16 == 0) && ((uintptr_t)out % 16 == 0);
  L.begin(K_NORMALS, s);
  k_depth_u16<<<sm_count() * 8, 256, 0, s>>>(in, scale, n, out, vec);
  L.end(K_NORMALS, s);
}

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
