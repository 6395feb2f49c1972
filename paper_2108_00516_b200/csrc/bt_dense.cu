// bt_dense.cu — dense geometric edges of Eq. (3):
//   E_g(i,j) = sum_{p in I_i} rho( n_i(x) . (T_i T_j^-1 pi_D^-1(pi(T_j T_i^-1 p)) - p) ),
// "dense pixel-wise correspondences are associated by point re-projection, while outliers
// are filtered based on the distance between the point pair and the angle formed by their
// normals".  Readings: nearest pixel (R14), gates (R15), normals compared in camera i (R16),
// Huber (R17), J = [n_i^T, (q x n_i)^T] for the left perturbation of T_i (R18).
//
// Factored formulation (the oracle's algebra, regrouped — no use of R^-1 = R^T, which does
// not hold exactly for float32-rounded rotations):
//   q - p = R_i R_j^T (s - t_j) + t_i - p = R_i x_s - (p - t_i),  x_s = R_j^T (s - t_j),
//   r = n_i . (q - p),  |q - p|,  n_i . (R_i R_j^T n_j) = (R_i^T n_i) . (R_j^T n_j).
// The residual cancels two ~0.5 m positions down to ~1e-5 m near the optimum, so x_s and
// p - t_i are fp64 and x_s is computed ONCE per target pixel per call (not per edge); R_i is
// a per-CTA constant.
//
//  k_edge_setup   one thread per edge: T_j T_i^-1 (fp32, for the projection); one CTA per
//                 source frame builds that frame's ordered list of outgoing edges.
//  k_dense_prep   one CTA per (frame, 32x32 tile): coalesced vector reads (uchar4 mask,
//                 float4 depth, 3 x float4 normals) of 4 pixels per thread; per valid pixel the
//                 fp64 object-frame point and fp32 object-frame normal go to a per-frame map
//                 (gathered as a TARGET) tagged with the call's epoch (the tag is the pixel's
//                 validity: no per-pixel validity map), and a block scan compacts the tile's valid source pixels (pixel order, stride
//                 applied) into 32-byte entries.
//  k_dense_scan   one CTA per frame: exclusive scan of the tile counts, so the frame's valid
//                 source pixels form one compacted sequence cut into chunks of kTile entries.
//  k_dense        one CTA per (frame, chunk) work item (grid-stride) — every chunk but a
//                 frame's last is full.  A chunk's entries (located by binary search in the tile
//                 offsets) + their fp64 points are staged in shared memory once and reused for
//                 every edge leaving the frame; each warp owns whole edges (gathers pipelined
//                 two entries ahead in three fixed slots, one transpose reduction per (warp,
//                 edge)).
//                 Per (entry, edge): fp32 projection, gather of the target's map entry (valid iff
//                 it carries this call's epoch),
//                 fp64 residual difference then fp32 gates / Huber, 29 running sums.
//  k_dense_reduce fixed-order fp64 sum of the per-tile partials of an edge (deterministic), then
//                 the object-frame blocks to camera i: H = M H_o M^T, g = M g_o (reading R32).
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <type_traits>

#include "bt_internal.cuh"
#include "bt_tc.cuh"


namespace bt {
namespace {

constexpr int kTS = 32;                       // tile side (pixels)
constexpr int kTile = kTS * kTS;
constexpr int kDenseThreads = 256;
constexpr int kPer = kTile / kDenseThreads;   // 4 pixels / entries per thread
constexpr int kAcc = 29;                      // H 21, g 6, E, count
constexpr int kPartStride = 32;

// x_s = R^T (p - t) is computed in fp64 and stored as fp32 hi + fp16 lo: lo = (x - hi) * 2^24
// in fp16 (|x - hi| <= ulp(hi) / 2, so |lo| <= 2^24 * 2^-24 * |x| / 2: in range up to |x| of
// 65 km; below fp16's normal range the subnormals still resolve 2^-48 m).  hi + lo * 2^-24
// reproduces x to ~1e-12 relative — the cancelling difference of Eq. (3) keeps its fp64-level
// accuracy (reading R26) from one 32-byte sector.
constexpr double kLoScale = 16777216.0;       // 2^24
constexpr float kLoInv = 5.9604644775390625e-08f;  // 2^-24
struct __align__(32) MapEntry {                // 32 bytes (one sector, one 256-bit load), per valid pixel
  float x, y, z;                              // hi parts of x_s (object frame)
  float nx, ny, nz;                           // object-frame normal
  __half lx, ly, lz;                          // lo parts * 2^24
  unsigned short epoch;                       // the call that wrote it (valid iff == this call's)
};

struct DenseArgs {
  MapView mp;
  float fx, fy, cx, cy, ifx, ify;
  double cxd, cyd, ifxd, ifyd;
  const bt_pose *node_pose;
  const int32_t *edges;       // [E][2] or null (then derived from pairs)
  const int32_t *pairs;
  int E, stride, tx, ty, tiles;
  double gate2;
  float gate2f, cos_gate, huber;
  float *tji;                 // [E][12] T_j T_i^-1
  int32_t *elist;             // [F][E] outgoing edges per source frame, ascending
  int32_t *ecount;            // [F]
  float4 *entries;            // [F][tiles][2][kTile]: per tile its points (p, u | v << 16), then its normals
  int32_t *counts;            // [F][tiles]
  int32_t *offs;              // [F][tiles + 1] exclusive scan of counts (entries of frame f before tile t)
  int32_t *nch;               // [F] chunks of kTile compacted entries (0 if the frame has no outgoing edge)
  MapEntry *pmap;             // [F][H*W]: valid pixels' entries, tagged with the call's epoch
  uint32_t *hdr;              // [0] call counter (epoch = low 16 bits, never 0), [1] wrap flag,
                              // [2] map entries reserved (bt_reserve); zeroed with the maps
  int32_t *tlist;             // [F * tiles] masked tiles (f * tiles + t), k_dense_mask -> k_dense_prep
  int32_t *tcount;            // [1] list length (zeroed by k_edge_setup)
  float *partials;            // [E][tiles][32] (per chunk of the edge's source frame; chunks <= tiles)
  int32_t *assoc;             // debug (bt_dense_assoc): [E][H][W] associated target pixel or -1
};

__device__ __forceinline__ void edge_frames(const int32_t *edges, const int32_t *pairs, int e, int &fi, int &fj) {
  if (edges) { fi = edges[2 * e]; fj = edges[2 * e + 1]; }
  else {
    const int p = e >> 1;
    fi = pairs[2 * p + (e & 1)];
    fj = pairs[2 * p + 1 - (e & 1)];
  }
}

// one launch for the per-edge / per-frame setup: blocks [0, F) build frame f's ascending list
// of outgoing edges (deterministic ballot compaction); blocks F.. compute T_j T_i^-1 per edge
__global__ void __launch_bounds__(256) k_edge_setup(DenseArgs A) {
  pdl_wait();
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *A.tcount = 0;                                                 // k_dense_mask's work list
    // this call's epoch: a map entry is a valid target iff it carries it, so no per-pixel
    // validity map is written or gathered; every 65535 calls the tags wrap and the maps are
    // cleared (k_dense_mask) before any entry is written
    uint32_t e = A.hdr[0] + 1;
    if ((e & 0xFFFFu) == 0u) ++e;
    A.hdr[0] = e;
    A.hdr[1] = (e & 0xFFFFu) == 1u && e > 1u;
  }
  if ((int)blockIdx.x >= A.mp.n_frames) {
    const int e = (blockIdx.x - A.mp.n_frames) * blockDim.x + threadIdx.x;
    if (e >= A.E) return;
    int fi, fj;
    edge_frames(A.edges, A.pairs, e, fi, fj);
    // T_j T_i^-1: R = R_j R_i^T, t = t_j - R t_i
    const bt_pose Pi = A.node_pose[fi], Pj = A.node_pose[fj];
    double R[9];
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) {
        double x = 0;
        for (int k = 0; k < 3; ++k) x += (double)Pj.R[3 * r + k] * Pi.R[3 * c + k];
        R[3 * r + c] = x;
      }
    float *o = A.tji + 12 * e;
    for (int k = 0; k < 9; ++k) o[k] = (float)R[k];
    for (int r = 0; r < 3; ++r)
      o[9 + r] = (float)(Pj.t[r] - (R[3 * r] * Pi.t[0] + R[3 * r + 1] * Pi.t[1] + R[3 * r + 2] * Pi.t[2]));
    return;
  }
  __shared__ int wsum[8];
  const int f = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int base = 0;
  for (int e0 = 0; e0 < A.E; e0 += 256) {
    const int e = e0 + threadIdx.x;
    bool mine = false;
    if (e < A.E) {
      int fi, fj;
      edge_frames(A.edges, A.pairs, e, fi, fj);
      mine = fi == f;
    }
    const unsigned bal = __ballot_sync(0xffffffffu, mine);
    if (lane == 0) wsum[warp] = __popc(bal);
    __syncthreads();
    int off = 0, tot = 0;
    for (int w = 0; w < 8; ++w) { off += w < warp ? wsum[w] : 0; tot += wsum[w]; }
    if (mine) A.elist[(size_t)f * A.E + base + off + __popc(bal & ((1u << lane) - 1u))] = e;
    base += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) A.ecount[f] = base;
}

// map entry of one valid pixel: x = R^T (p - t) in fp64 from the exact inputs (stored hi + lo,
// reading R26), n_o = R^T n
__device__ __forceinline__ void write_map_entry(const DenseArgs &A, const bt_pose &P, MapEntry *dst, int u, int v,
                                                float dep, float n0, float n1, float n2, unsigned epoch) {
  const double d = dep;
  const double p0 = ((double)u - A.cxd) * d * A.ifxd - P.t[0];
  const double p1 = ((double)v - A.cyd) * d * A.ifyd - P.t[1];
  const double p2 = d - P.t[2];
  MapEntry me;
  const double X0 = P.R[0] * p0 + P.R[3] * p1 + P.R[6] * p2;
  const double X1 = P.R[1] * p0 + P.R[4] * p1 + P.R[7] * p2;
  const double X2 = P.R[2] * p0 + P.R[5] * p1 + P.R[8] * p2;
  me.x = (float)X0; me.y = (float)X1; me.z = (float)X2;
  me.lx = __double2half((X0 - (double)me.x) * kLoScale);
  me.ly = __double2half((X1 - (double)me.y) * kLoScale);
  me.lz = __double2half((X2 - (double)me.z) * kLoScale);
  me.epoch = (unsigned short)epoch;
  const double m0 = n0, m1 = n1, m2 = n2;
  me.nx = (float)(P.R[0] * m0 + P.R[3] * m1 + P.R[6] * m2);
  me.ny = (float)(P.R[1] * m0 + P.R[4] * m1 + P.R[7] * m2);
  me.nz = (float)(P.R[2] * m0 + P.R[5] * m1 + P.R[8] * m2);
  *dst = me;
}

// one masked 32x32 tile, 4 pixels per thread (CTA-uniform call)
__device__ __forceinline__ void prep_tile(const DenseArgs &A, const int f, const int t, int *wsum, unsigned epoch) {
  const int W = A.mp.W, H = A.mp.H, npx = W * H;
  const int ty = t / A.tx, tx = t - ty * A.tx;
  const int row = threadIdx.x >> 3, col0 = (threadIdx.x & 7) * 4;
  const int v = ty * kTS + row, u0 = tx * kTS + col0;
  const size_t off = (size_t)f * npx;
  const int pix0 = v * W + u0;
  bool in[kPer];
  float dep[kPer], nr[kPer * 3];
#pragma unroll
  for (int k = 0; k < kPer; ++k) { in[k] = false; dep[k] = 0.f; nr[3 * k] = nr[3 * k + 1] = nr[3 * k + 2] = 0.f; }
  if (v < H) {
    if ((W & 3) == 0 && u0 + kPer <= W) {
      // the mask first; depth and normals only where one of the 4 pixels is in the mask
      // (~1/8 of the frame): one extra round trip, ~5x fewer bytes
      const uchar4 m4 = __ldg(reinterpret_cast<const uchar4 *>(A.mp.mask + off + pix0));
      in[0] = m4.x != 0; in[1] = m4.y != 0; in[2] = m4.z != 0; in[3] = m4.w != 0;
      if (in[0] | in[1] | in[2] | in[3]) {
        const float4 d4 = __ldg(reinterpret_cast<const float4 *>(A.mp.depth + off + pix0));
        const float4 *n4 = reinterpret_cast<const float4 *>(A.mp.normal + 3 * (off + pix0));
        const float4 a = __ldg(n4), b = __ldg(n4 + 1), c = __ldg(n4 + 2);
        dep[0] = d4.x; dep[1] = d4.y; dep[2] = d4.z; dep[3] = d4.w;
        nr[0] = a.x; nr[1] = a.y; nr[2] = a.z; nr[3] = a.w; nr[4] = b.x; nr[5] = b.y;
        nr[6] = b.z; nr[7] = b.w; nr[8] = c.x; nr[9] = c.y; nr[10] = c.z; nr[11] = c.w;
      }
    } else {
#pragma unroll
      for (int k = 0; k < kPer; ++k) {
        const int u = u0 + k;
        if (u < W && A.mp.mask[off + pix0 + k]) {
          in[k] = true;
          dep[k] = A.mp.depth[off + pix0 + k];
          for (int c = 0; c < 3; ++c) nr[3 * k + c] = A.mp.normal[3 * (off + pix0 + k) + c];
        }
      }
    }
  }
  const bt_pose P = A.node_pose[f];
  bool src[kPer];
  int n_mine = 0;
  bool vv[kPer];
#pragma unroll
  for (int k = 0; k < kPer; ++k)
    vv[k] = in[k] && dep[k] > 0.f && !(nr[3 * k] == 0.f && nr[3 * k + 1] == 0.f && nr[3 * k + 2] == 0.f);
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    const int u = u0 + k;
    const bool valid = vv[k];
    if (valid) write_map_entry(A, P, A.pmap + off + pix0 + k, u, v, dep[k], nr[3 * k], nr[3 * k + 1], nr[3 * k + 2], epoch);
    src[k] = valid && (A.stride <= 1 || (u % A.stride == 0 && v % A.stride == 0));
    n_mine += src[k];
  }
  // block exclusive scan of n_mine (thread order = row-major pixel order within the tile)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int incl = n_mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  int woff = 0, total = 0;
#pragma unroll
  for (int w = 0; w < kDenseThreads / 32; ++w) {
    woff += w < warp ? wsum[w] : 0;
    total += wsum[w];
  }
  int pos = woff + incl - n_mine;
  float4 *out = A.entries + ((size_t)f * A.tiles + t) * kTile * 2;
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    if (!src[k]) continue;
    const int u = u0 + k;
    const float d = dep[k];
    out[pos] = make_float4(((float)u - A.cx) * d * A.ifx, ((float)v - A.cy) * d * A.ify, d,
                           __int_as_float(u | (v << 16)));
    out[kTile + pos] = make_float4(nr[3 * k], nr[3 * k + 1], nr[3 * k + 2], 0.f);
    ++pos;
  }
  if (threadIdx.x == 0) A.counts[(size_t)f * A.tiles + t] = total;
}

// persistent: the CTAs drain the list of masked tiles written by k_dense_mask
// 4 CTAs per SM (64 registers, no spill): 592 resident CTAs for the ~800 masked tiles of C2
// (3 at 103 registers) — step 0.2826 -> 0.2806 ms (A/B, same box)
#ifndef BT_PREP_MINB
#define BT_PREP_MINB 4
#endif
__global__ void __launch_bounds__(kDenseThreads, BT_PREP_MINB) k_dense_prep(DenseArgs A) {
  pdl_wait();
  __shared__ int wsum[kDenseThreads / 32];
  const int n_work = *A.tcount;
  const unsigned epoch = A.hdr[0] & 0xFFFFu;
  for (int w = blockIdx.x; w < n_work; w += gridDim.x) {
    __syncthreads();                                                 // wsum of the previous tile read
    const int f = A.tlist[w] / A.tiles, t = A.tlist[w] - f * A.tiles;
    prep_tile(A, f, t, wsum, epoch);
  }
}


// Masked-tile classification, warp per 32x32 tile (8 tiles per CTA): lane r reads row r of the
// tile's mask as two 16-B vectors, so a whole tile is 2 loads per lane (the mask pass is ~85 %
// of the frame and was latency-bound at one 4-B load per thread).  A tile without a masked
// pixel is finished here (no source entries, no map entries); the others are appended to a
// work list (slot order is irrelevant: each tile writes only its own outputs) that the
// persistent k_dense_prep drains with 256 threads per tile.
__global__ void __launch_bounds__(kDenseThreads) k_dense_mask(DenseArgs A) {
  pdl_wait();
  if (A.hdr[1]) {                                                  // epoch wrap: clear every reserved entry
    const size_t n = (size_t)A.hdr[2] * 2, st = (size_t)gridDim.x * gridDim.y * blockDim.x;
    uint4 *m = reinterpret_cast<uint4 *>(A.pmap);
    for (size_t i = ((size_t)blockIdx.y * gridDim.x + blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += st)
      m[i] = make_uint4(0u, 0u, 0u, 0u);
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int f = blockIdx.y, t = blockIdx.x * (kDenseThreads / 32) + warp;
  if (t >= A.tiles) return;                                        // warp-uniform
  const int W = A.mp.W, H = A.mp.H;
  const int ty = t / A.tx, tx = t - ty * A.tx;
  const int v = ty * kTS + lane, u0 = tx * kTS;
  const size_t row = (size_t)f * W * H + (size_t)v * W + u0;
  const bool full = (W & 15) == 0 && u0 + kTS <= W;                // 16-B aligned full-width tile row
  bool any = false;
  if (v < H) {
    if (full) {
      const uint4 *m = reinterpret_cast<const uint4 *>(A.mp.mask + row);
      const uint4 a = __ldg(m), b = __ldg(m + 1);
      any = (a.x | a.y | a.z | a.w | b.x | b.y | b.z | b.w) != 0u;
    } else {
      for (int u = u0; u < min(W, u0 + kTS); ++u) any |= A.mp.mask[row + (u - u0)] != 0;
    }
  }
  if (__ballot_sync(0xffffffffu, any) == 0u) {
    if (lane == 0) A.counts[(size_t)f * A.tiles + t] = 0;
  } else if (lane == 0) {
    A.tlist[atomicAdd(A.tcount, 1)] = f * A.tiles + t;
  }
}

// per frame: exclusive scan of the tile counts -> offs, and the number of kTile-entry chunks
__global__ void __launch_bounds__(kDenseThreads) k_dense_scan(DenseArgs A) {
  pdl_wait();
  __shared__ int wsum[kDenseThreads / 32];
  const int f = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int32_t *cnt = A.counts + (size_t)f * A.tiles;
  int32_t *off = A.offs + (size_t)f * (A.tiles + 1);
  int carry = 0;
  for (int t0 = 0; t0 < A.tiles; t0 += kDenseThreads) {
    const int t = t0 + threadIdx.x;
    const int c = t < A.tiles ? cnt[t] : 0;
    int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    int woff = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < kDenseThreads / 32; ++w) { woff += w < warp ? wsum[w] : 0; tot += wsum[w]; }
    if (t < A.tiles) off[t] = carry + woff + incl - c;
    carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    off[A.tiles] = carry;
    A.nch[f] = A.ecount[f] > 0 ? (carry + kTile - 1) / kTile : 0;
  }
}

constexpr size_t kDenseSmem = kTile * (16 + 16 + 8 + 24);
constexpr int kEdgeThreads = 256;                // k_dense CTA (8 warps, each owning edges)

// target-pixel gather of one (entry, edge) item, issued ahead of its use
struct Gather {
  float g[8];                 // one 32-B map entry: x_s hi, n_o,j, x_s lo (fp16 x 3), epoch tag
  bool in;                    // projected into the frame
  int tj;                     // target pixel index (read only by the association output)
};

// project entry k of the staged chunk with T = T_j T_i^-1 and issue its target gathers
// (kCheck false: the caller guarantees k < n)
template <bool kCheck = true>
__device__ __forceinline__ void issue_gather(const float4 *sP, int k, int n, const float (&T)[12], float fx, float fy,
                                             float cx, float cy, int W, int H, const float *pm, Gather &G) {
  // straight-line (no branches between the gathers of consecutive entries): out-of-range
  // entries and failed projections are predicated off through tj = -1
  const float4 a = sP[!kCheck || k < n ? k : 0];
  const float yx = fmaf(T[0], a.x, fmaf(T[1], a.y, fmaf(T[2], a.z, T[9])));
  const float yy = fmaf(T[3], a.x, fmaf(T[4], a.y, fmaf(T[5], a.z, T[10])));
  const float yz = fmaf(T[6], a.x, fmaf(T[7], a.y, fmaf(T[8], a.z, T[11])));
  // 1 / z as one MUFU.RCP (what __fdividef(1, z) computes for a normal z, without its
  // denormal-range fix-up: a projection with z <= 0 or a far-off pixel fails the tests below)
  float iz;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(iz) : "f"(yz));
  const float up = fmaf(fx * yx, iz, cx), vp = fmaf(fy * yy, iz, cy);
  // nearest pixel (R14): floor(x + 0.5) as one F2I.FLOOR (saturating: far-off projections fail
  // the unsigned range test like the float one)
  const int xu = __float2int_rd(up + 0.5f), xv = __float2int_rd(vp + 0.5f);
  const bool ok = (!kCheck || k < n) && yz > 0.f && (unsigned)xu < (unsigned)W && (unsigned)xv < (unsigned)H;
  const int tj = ok ? xv * W + xu : -1;
  const int tt = tj < 0 ? 0 : tj;                                  // the map entry (its tag = validity)
  G.in = tj >= 0;
  G.tj = tj;
  asm("ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
      : "=f"(G.g[0]), "=f"(G.g[1]), "=f"(G.g[2]), "=f"(G.g[3]), "=f"(G.g[4]), "=f"(G.g[5]), "=f"(G.g[6]),
        "=f"(G.g[7])
      : "l"(pm + 8 * (size_t)tt));
}

// Each warp owns whole edges of the chunk: warp w walks edges w, w + 8, ... leaving the frame,
// and for each one all of the chunk's entries (lane l: entries l, l + 32, ...), with the target
// gathers software-pipelined two entries ahead so loads stay in flight.  One 31-shuffle
// transpose reduction per (warp, edge) puts the 29 sums straight into the edge's chunk partial:
// no shared reduction buffer, no barrier between edges.
// kAssoc (bt_dense_assoc, a debug entry): the same arithmetic, plus one store per (entry, edge)
// of the associated target pixel (-1 when rejected) — the per-pixel decision the parity tests
// compare with the oracle's; a separate instantiation, so the product kernel carries no trace
template <bool kAssoc>
__global__ void __launch_bounds__(kEdgeThreads, 2) k_dense(DenseArgs A) {
  pdl_wait();
  extern __shared__ __align__(16) unsigned char dsm[];
  // the chunk's entries as the prep stored them per tile (points, normals: two arrays), copied
  // in by the TMA engine; the normal's pad word is replaced by n_o,i.x once staged
  float4 *sP = reinterpret_cast<float4 *>(dsm);                    // p (camera, fp32), (u | v << 16)
  float4 *sN = sP + kTile;                                         // n_i (camera), n_o,i.x
  float4 *sYh = sN + kTile;                                        // y_p = R_i^-1 (p - t_i) hi, n_o,i.y
  float4 *sYl = sYh + kTile;                                       //   and lo (fp32 + fp32), n_o,i.z
  int *sCb = reinterpret_cast<int *>(sYl + kTile);             // [F + 1] chunk base per frame
  int *sOff = sCb + A.mp.n_frames + 1;                             // [tiles + 1] of the current frame
  const int F = A.mp.n_frames;
  const int W = A.mp.W, H = A.mp.H, npx = W * H;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned epoch = A.hdr[0] & 0xFFFFu;                      // this call's map-entry tag
  __shared__ __align__(8) uint64_t bar_e;                           // the chunk's bulk copies landed
  if (threadIdx.x == 0) {
    mbar_init(&bar_e, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  uint32_t e_phase = 0;
  if (warp == 0) {                                                 // chunk bases: prefix over frames
    int carry = 0;
    for (int f0 = 0; f0 < F; f0 += 32) {
      const int c = f0 + lane < F ? A.nch[f0 + lane] : 0;
      int incl = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      if (f0 + lane < F) sCb[f0 + lane] = carry + incl - c;
      carry += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) sCb[F] = carry;
  }
  __syncthreads();
  const int total = sCb[F];
  for (int ch = blockIdx.x; ch < total; ch += gridDim.x) {
    int f = 0;
    {
      int lo = 0, hi = F;                                          // sCb[lo] <= ch < sCb[hi]
      while (hi - lo > 1) { const int mid = (lo + hi) >> 1; if (sCb[mid] <= ch) lo = mid; else hi = mid; }
      f = lo;
    }
    const int cl = ch - sCb[f];                                    // chunk of frame f
    const int32_t *offg = A.offs + (size_t)f * (A.tiles + 1);
    __syncthreads();                                               // previous chunk done with smem
    for (int k = threadIdx.x; k <= A.tiles; k += kEdgeThreads) sOff[k] = offg[k];
    __syncthreads();
    const int n = min(kTile, sOff[A.tiles] - cl * kTile);
    const int ne = A.ecount[f];
    // the chunk's compacted entries [g0, g0 + n) are contiguous runs of 32-B entries, one per
    // tile they overlap: staged by the TMA engine (one bulk copy per run) while the pose's
    // inverse is computed
    const float4 *src = A.entries + (size_t)f * A.tiles * kTile * 2;
    if (threadIdx.x == 0 && n > 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // previous chunk's accesses of sP / sN
      mbar_expect_tx(&bar_e, (uint32_t)n * 32u);                 // two 16-B words per entry
      const int g0 = cl * kTile;
      int t = 0, hi = A.tiles;                                     // tile holding g0: sOff[t] <= g0 < sOff[t + 1]
      while (hi - t > 1) { const int mid = (t + hi) >> 1; if (sOff[mid] <= g0) t = mid; else hi = mid; }
      for (; t < A.tiles && sOff[t] < g0 + n; ++t) {
        const int lo_ = max(g0, sOff[t]), hi_ = min(g0 + n, sOff[t + 1]);
        if (hi_ > lo_) {
          const float4 *tp = src + (size_t)t * kTile * 2 + (lo_ - sOff[t]);
          bulk_load(sP + (lo_ - g0), tp, (uint32_t)(hi_ - lo_) * 16u, &bar_e);
          bulk_load(sN + (lo_ - g0), tp + kTile, (uint32_t)(hi_ - lo_) * 16u, &bar_e);
        }
      }
    }
    {
      const bt_pose P = A.node_pose[f];
      double Rd[9], Ri[9];                                         // R_i and its exact inverse (fp64)
#pragma unroll
      for (int k = 0; k < 9; ++k) Rd[k] = P.R[k];
      {
        const double c0 = Rd[4] * Rd[8] - Rd[5] * Rd[7], c1 = Rd[5] * Rd[6] - Rd[3] * Rd[8],
                     c2 = Rd[3] * Rd[7] - Rd[4] * Rd[6];
        const double idet = 1.0 / (Rd[0] * c0 + Rd[1] * c1 + Rd[2] * c2);
        Ri[0] = c0 * idet; Ri[1] = (Rd[2] * Rd[7] - Rd[1] * Rd[8]) * idet; Ri[2] = (Rd[1] * Rd[5] - Rd[2] * Rd[4]) * idet;
        Ri[3] = c1 * idet; Ri[4] = (Rd[0] * Rd[8] - Rd[2] * Rd[6]) * idet; Ri[5] = (Rd[2] * Rd[3] - Rd[0] * Rd[5]) * idet;
        Ri[6] = c2 * idet; Ri[7] = (Rd[1] * Rd[6] - Rd[0] * Rd[7]) * idet; Ri[8] = (Rd[0] * Rd[4] - Rd[1] * Rd[3]) * idet;
      }
      const double t0 = P.t[0], t1 = P.t[1], t2 = P.t[2];
      if (n > 0) {
        mbar_wait(&bar_e, e_phase);
        e_phase ^= 1u;
      }
      for (int k = threadIdx.x; k < n; k += kEdgeThreads) {
        const float4 a = sP[k], b = sN[k];
        const int uv = __float_as_int(a.w), u = uv & 0xffff, v = uv >> 16;
        const double d = a.z;                                      // p.z = depth exactly
        const double x0 = ((double)u - A.cxd) * d * A.ifxd - t0, x1 = ((double)v - A.cyd) * d * A.ifyd - t1,
                     x2 = d - t2;                                  // p - t_i
        const double y[3] = {Ri[0] * x0 + Ri[1] * x1 + Ri[2] * x2, Ri[3] * x0 + Ri[4] * x1 + Ri[5] * x2,
                             Ri[6] * x0 + Ri[7] * x1 + Ri[8] * x2};
        float yh[3], yl[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          yh[c] = (float)y[c];
          yl[c] = (float)(y[c] - (double)yh[c]);
        }
        const double m0 = b.x, m1 = b.y, m2 = b.z;                 // n_o,i = R_i^T n_i
        const float o0 = (float)(Rd[0] * m0 + Rd[3] * m1 + Rd[6] * m2);
        const float o1 = (float)(Rd[1] * m0 + Rd[4] * m1 + Rd[7] * m2);
        const float o2 = (float)(Rd[2] * m0 + Rd[5] * m1 + Rd[8] * m2);
        sN[k].w = o0;
        sYh[k] = make_float4(yh[0], yh[1], yh[2], o1);               // one 16-B entry each: two
        sYl[k] = make_float4(yl[0], yl[1], yl[2], o2);               // LDS.128 per (entry, edge)
      }
    }
    __syncthreads();

    for (int ie = warp; ie < ne; ie += kEdgeThreads / 32) {
      const int e = A.elist[(size_t)f * A.E + ie];
      int fi, fj;
      edge_frames(A.edges, A.pairs, e, fi, fj);
      float T[12];
#pragma unroll
      for (int q = 0; q < 12; ++q) T[q] = __ldg(A.tji + 12 * e + q);
      const size_t off_j = (size_t)fj * npx;
      const float *pm = reinterpret_cast<const float *>(A.pmap + off_j);
      float acc[32];
#pragma unroll
      for (int q = 0; q < 32; ++q) acc[q] = 0.f;
      // three prefetch slots in a fixed rotation (unrolled by 3, so no loaded register is moved
      // and every gather has two entries of work to hide behind)
      // branch-free: rejected items (not in the frame, invalid target, gates failed) run the
      // same straight-line code with w = rho = 0 and zeroed map values (stale map words of
      // invalid pixels never reach the arithmetic), so the scheduler keeps the gathers of the
      // next entries in flight across it; accepted items compute exactly as before
      auto consume = [&](const Gather &G, int k0, auto checked) {
        const bool hit = G.in && (__float_as_uint(G.g[7]) >> 16) == epoch;   // a valid target of this call
        const int k = !decltype(checked)::value || k0 < n ? k0 : 0;   // tail: any staged entry (masked)
        // no select on the gathered words: a rejected item reads either pixel 0's entry or an
        // invalid pixel's (a stale entry of an earlier call, or zeros) — the map region sits at a
        // fixed offset, zeroed by bt_reserve and only ever written with finite map entries, so
        // its words are finite and w = rho = 0 cancel them
        const float *g = G.g;
        // q - p = R_i x_s - (p - t_i) = R_i (x_s - y_p), y_p = R_i^-1 (p - t_i) (exact algebra
        // for the fp32 R_i as given, reading R26).  x_s - y_p cancels ~0.1 m coordinates: with
        // both as hi + lo pairs, hi_s - hi_y is exact (Sterbenz) when they are close and the lo
        // parts carry the rest, so the difference is fp64-accurate in fp32 arithmetic; the
        // rotation of the small difference is fp32 (~1e-7 relative: inside the band rule, R22)
        const unsigned w6 = __float_as_uint(g[6]), w7 = __float_as_uint(g[7]);
        const float ls0 = __half2float(__ushort_as_half((unsigned short)(w6 & 0xffffu)));
        const float ls1 = __half2float(__ushort_as_half((unsigned short)(w6 >> 16)));
        const float ls2 = __half2float(__ushort_as_half((unsigned short)(w7 & 0xffffu)));
        const float4 yh = sYh[k], yl = sYl[k];
        const float D0 = (g[0] - yh.x) + fmaf(ls0, kLoInv, -yl.x);
        const float D1 = (g[1] - yh.y) + fmaf(ls1, kLoInv, -yl.y);
        const float D2 = (g[2] - yh.z) + fmaf(ls2, kLoInv, -yl.z);
        const float mj0 = g[3], mj1 = g[4], mj2 = g[5];
        // everything in the object frame (reading R32): q - p = R_i D, so r = n_i . (R_i D) =
        // (R_i^T n_i) . D = n_o,i . D exactly, |q - p|^2 = |D|^2 for the (orthonormal to fp32
        // rounding) R_i — a ~1e-7 relative difference, far inside the gate's band (R22) — and
        // J = [n_i, q x n_i] = M_i [n_o,i, x_s x n_o,i] with the per-frame 6 x 6
        // M_i = [[R_i, 0], [[t_i]x R_i, R_i]]: the blocks are accumulated with J_o and rotated
        // once per edge, in fp64, by k_dense_reduce (no per-item rotation of D, no q)
        const float dist2 = fmaf(D0, D0, fmaf(D1, D1, D2 * D2));
        const float o0 = sN[k].w, o1 = yh.w, o2 = yl.w;            // n_o,i
        const float c = fmaf(o0, mj0, fmaf(o1, mj1, o2 * mj2));
        const bool acc_ok = hit && dist2 < A.gate2f && c > A.cos_gate;
        const float r = fmaf(o0, D0, fmaf(o1, D1, o2 * D2));
        const float xs0 = g[0], xs1 = g[1], xs2 = g[2];             // x_s (hi): the target point, object frame
        const float ar = fabsf(r);
        // Huber (R17) without branches: with m = min(|r|, h), rho = m (|r| - m / 2) is 0.5 r^2
        // inside and h (|r| - h / 2) beyond (the same roundings as the two formulas); the weight
        // h / |r| beyond is h * rcp(|r|) (|r| > h > 0: no range fix-up needed)
        const float m = fminf(ar, A.huber);
        float rcp;
        asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rcp) : "f"(ar));
        const float w = acc_ok ? (ar <= A.huber ? 1.f : A.huber * rcp) : 0.f;
        const float rho = acc_ok ? m * fmaf(-0.5f, m, ar) : 0.f;
        const float J[6] = {o0, o1, o2, xs1 * o2 - xs2 * o1, xs2 * o0 - xs0 * o2, xs0 * o1 - xs1 * o0};
        int q = 0;
#pragma unroll
        for (int aa = 0; aa < 6; ++aa) {
          const float wa = w * J[aa];
#pragma unroll
          for (int b = aa; b < 6; ++b) { acc[q] = fmaf(wa, J[b], acc[q]); ++q; }
        }
#pragma unroll
        for (int aa = 0; aa < 6; ++aa) acc[21 + aa] = fmaf(w * J[aa], r, acc[21 + aa]);
        acc[27] += rho;
        acc[28] += acc_ok ? 1.f : 0.f;
        if constexpr (kAssoc) {
          if (!decltype(checked)::value || k0 < n) {
            const int uv = __float_as_int(sP[k].w);
            A.assoc[(size_t)e * npx + (size_t)(uv >> 16) * W + (uv & 0xffff)] = acc_ok ? G.tj : -1;
          }
        }
      };
      Gather GA, GB, GC;
      issue_gather(sP, lane, n, T, A.fx, A.fy, A.cx, A.cy, W, H, pm, GA);
      issue_gather(sP, lane + 32, n, T, A.fx, A.fy, A.cx, A.cy, W, H, pm, GB);
      // while every lane's six items of an iteration are inside the chunk (warp-uniform bound),
      // the range checks are compiled out; the tail iterations keep them
      const std::true_type chk;
      const std::false_type nochk;
      int k = lane;
      for (; k - lane + 31 + 128 < n; k += 96) {
        issue_gather<false>(sP, k + 64, n, T, A.fx, A.fy, A.cx, A.cy, W, H, pm, GC);
        consume(GA, k, nochk);
        issue_gather<false>(sP, k + 96, n, T, A.fx, A.fy, A.cx, A.cy, W, H, pm, GA);
        consume(GB, k + 32, nochk);
        issue_gather<false>(sP, k + 128, n, T, A.fx, A.fy, A.cx, A.cy, W, H, pm, GB);
        consume(GC, k + 64, nochk);
      }
      for (; k < n; k += 96) {
        issue_gather(sP, k + 64, n, T, A.fx, A.fy, A.cx, A.cy, W, H, pm, GC);
        consume(GA, k, chk);
        issue_gather(sP, k + 96, n, T, A.fx, A.fy, A.cx, A.cy, W, H, pm, GA);
        consume(GB, k + 32, chk);
        issue_gather(sP, k + 128, n, T, A.fx, A.fy, A.cx, A.cy, W, H, pm, GB);
        consume(GC, k + 64, chk);
      }
      // warp transpose reduction: lane l ends with the warp total of acc[l]
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) {
        const bool upper = (lane & o) != 0;
#pragma unroll
        for (int c = 0; c < o; ++c) {
          const float send = upper ? acc[c] : acc[c + o];
          const float keep = upper ? acc[c + o] : acc[c];
          acc[c] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
      }
      A.partials[((size_t)e * A.tiles + cl) * kPartStride + lane] = acc[0];
    }
  }
}

__global__ void __launch_bounds__(256) k_dense_reduce(const float *__restrict__ partials, const int32_t *__restrict__ nch,
                                                       int tiles, const int32_t *edges, const int32_t *pairs,
                                                       const bt_pose *node_pose, float *out,
                                                       int out_stride, uint32_t *records, int rec_stride, int off_ij,
                                                       int off_ji, PeerRec peers) {
  pdl_wait();
  __shared__ double wsum[8][32];
  __shared__ double Ho[6][6], go[6], Mi[6][6];
  const int e = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int fi, fj;
  edge_frames(edges, pairs, e, fi, fj);
  double s = 0.0;                                 // warp w: chunks w, w + 8, ... in order; lane = value
  const int nc = nch[fi];
  for (int t = warp; t < nc; t += 8) s += (double)partials[((size_t)e * tiles + t) * kPartStride + lane];
  wsum[warp][lane] = s;
  __syncthreads();
  if (warp != 0) return;
  double tsum = 0.0;
#pragma unroll
  for (int w = 0; w < 8; ++w) tsum += wsum[w][lane];
  // the object-frame blocks (J_o = [n_o, x_s x n_o]) to the camera frame of frame i (reading
  // R32): H = M Ho M^T, g = M go, with M = [[R, 0], [[t]x R, R]] of T_i — fp64, once per edge
  {
    int a = 0, b = 0, q = lane;
    if (q < 21) { while (q >= 6 - a) { q -= 6 - a; ++a; } b = a + q; Ho[a][b] = tsum; Ho[b][a] = tsum; }
    else if (lane < 27) go[lane - 21] = tsum;
    if (lane < 9) {
      const bt_pose P = node_pose[fi];
      const int r = lane / 3, c = lane % 3;
      const double R_rc = P.R[3 * r + c];
      const double t0 = P.t[0], t1 = P.t[1], t2 = P.t[2];
      // ([t]x R)[r][c] = sum_k [t]x[r][k] R[k][c]
      const double tx[3][3] = {{0.0, -t2, t1}, {t2, 0.0, -t0}, {-t1, t0, 0.0}};
      double v = 0.0;
      for (int k = 0; k < 3; ++k) v += tx[r][k] * (double)P.R[3 * k + c];
      Mi[r][c] = R_rc; Mi[r][3 + c] = 0.0; Mi[3 + r][c] = v; Mi[3 + r][3 + c] = R_rc;
    }
  }
  __syncwarp();
  double outv = tsum;
  if (lane < 21) {
    int a = 0, q = lane;
    while (q >= 6 - a) { q -= 6 - a; ++a; }
    const int b = a + q;
    double h = 0.0;
    for (int c = 0; c < 6; ++c) {
      double mh = 0.0;
      for (int d = 0; d < 6; ++d) mh += Ho[c][d] * Mi[b][d];
      h += Mi[a][c] * mh;
    }
    outv = h;
  } else if (lane < 27) {
    double gg = 0.0;
    for (int c = 0; c < 6; ++c) gg += Mi[lane - 21][c] * go[c];
    outv = gg;
  }
  const float v = lane < kAcc ? (float)outv : 0.f;
  if (records) {
    const int p = e >> 1;
    records[(size_t)p * rec_stride + ((e & 1) ? off_ji : off_ij) + lane] = __float_as_uint(v);
    peer_put(peers, p, ((e & 1) ? off_ji : off_ij) + lane, __float_as_uint(v));
  } else {
    out[(size_t)e * out_stride + lane] = v;
  }
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

size_t align256(size_t b) { return (b + 255) / 256 * 256; }

}  // namespace

int dense_tiles(int W, int H) { return ((W + kTS - 1) / kTS) * ((H + kTS - 1) / kTS); }

size_t dense_scratch_bytes(int max_frames, int max_edges, int W, int H) {
  const size_t tiles = dense_tiles(W, H), F = max_frames, npx = (size_t)W * H;
  return align256(F * tiles * kTile * 32) + align256(F * tiles * 4) + align256(F * (tiles + 1) * 4) + align256(F * 4) + align256((size_t)max_edges * tiles * kPartStride * 4) +
         align256((size_t)max_edges * 48) + align256(F * max_edges * 4) + align256(F * 4) +
         256 + align256(F * npx * sizeof(MapEntry)) + align256(F * tiles * 4) + align256(4);
}

void launch_dense(const MapView &mp, const bt_intrinsics &K, const bt_pose *node_pose, const int32_t *edges,
                  const int32_t *pairs, int E, const bt_edge_params &prm, void *scratch, size_t map_cap,
                  float *out, int out_stride, uint32_t *records, int rec_stride, int rec_off_ij, int rec_off_ji,
                  cudaStream_t s, Launch &L, int32_t *assoc, const PeerRec *peers) {
  if (E <= 0) return;
  DenseArgs a;
  a.assoc = assoc;
  a.mp = mp;
  a.fx = K.fx; a.fy = K.fy; a.cx = K.cx; a.cy = K.cy;
  a.ifx = 1.0f / K.fx; a.ify = 1.0f / K.fy;
  a.cxd = K.cx; a.cyd = K.cy; a.ifxd = 1.0 / (double)K.fx; a.ifyd = 1.0 / (double)K.fy;
  a.node_pose = node_pose;
  a.edges = edges; a.pairs = pairs; a.E = E;
  a.stride = prm.stride < 1 ? 1 : prm.stride;
  a.tx = (mp.W + kTS - 1) / kTS;
  a.ty = (mp.H + kTS - 1) / kTS;
  a.tiles = a.tx * a.ty;
  a.gate2 = (double)prm.dist_gate_m * (double)prm.dist_gate_m;
  a.gate2f = (float)a.gate2;
  a.cos_gate = prm.cos_gate;
  a.huber = prm.huber_m;
  // carve the scratch
  char *p = (char *)scratch;
  const size_t tiles = a.tiles, F = mp.n_frames, npx = (size_t)mp.W * mp.H;
  a.hdr = (uint32_t *)p;     p += 256;                                     // header + maps: zeroed by bt_reserve
  // the maps at their reserved size (map_cap entries: what bt_reserve zeroed and the epoch wrap
  // clears), so no other region of a call with fewer frames / pixels ever overlaps them
  a.pmap = (MapEntry *)p;    p += align256(std::max(map_cap, F * npx) * sizeof(MapEntry));
  a.entries = (float4 *)p;   p += align256(F * tiles * kTile * 32);
  a.counts = (int32_t *)p;   p += align256(F * tiles * 4);
  a.offs = (int32_t *)p;     p += align256(F * (tiles + 1) * 4);
  a.nch = (int32_t *)p;      p += align256(F * 4);
  a.partials = (float *)p;   p += align256((size_t)E * tiles * kPartStride * 4);
  a.tji = (float *)p;        p += align256((size_t)E * 48);
  a.elist = (int32_t *)p;    p += align256(F * E * 4);
  a.ecount = (int32_t *)p;   p += align256(F * 4);
  a.tlist = (int32_t *)p;    p += align256(F * tiles * 4);
  a.tcount = (int32_t *)p;
  L.begin(K_DENSE_PREP, s);
  launch_pdl(k_edge_setup, mp.n_frames + (E + 255) / 256, 256, 0, s, a);
  L.end(K_DENSE_PREP, s);
  L.begin(K_DENSE_PREP, s);
  launch_pdl(k_dense_mask, dim3((a.tiles + kDenseThreads / 32 - 1) / (kDenseThreads / 32), mp.n_frames),
             kDenseThreads, 0, s, a);
  L.end(K_DENSE_PREP, s);
  L.begin(K_DENSE_PREP, s);
  const int prep_grid = resident_grid((const void *)k_dense_prep, kDenseThreads, 0);
  launch_pdl(k_dense_prep, std::min(prep_grid, a.tiles * mp.n_frames), kDenseThreads, 0, s, a);
  L.end(K_DENSE_PREP, s);
  L.begin(K_DENSE_PREP, s);
  launch_pdl(k_dense_scan, mp.n_frames, kDenseThreads, 0, s, a);
  L.end(K_DENSE_PREP, s);
  const size_t smem = kDenseSmem + (size_t)(mp.n_frames + 1 + a.tiles + 1) * 4;
  auto kd = assoc ? k_dense<true> : k_dense<false>;
  smem_optin((const void *)kd, smem);
  if (assoc) cudaMemsetAsync(assoc, 0xff, (size_t)E * mp.W * mp.H * sizeof(int32_t), s);   // -1: no source entry
  // CTAs walk the chunks ch = blockIdx.x, + gridDim.x, ...: at most 8 per SM (a C2 step has
  // ~600 chunks, so most CTAs take one and their boundaries still let the higher-priority match /
  // RANSAC kernels interleave, bt_api.cu register_pairs_dev) — one CTA per possible chunk (4800
  // at C2, most exiting at once) measured 1.5 us slower per step
  const int grid = std::min(a.tiles * mp.n_frames, 8 * sm_count());
  L.begin(K_DENSE, s);
  launch_pdl(kd, grid, kEdgeThreads, smem, s, a);
  L.end(K_DENSE, s);
  L.begin(K_DENSE_REDUCE, s);
  launch_pdl(k_dense_reduce, E, 256, 0, s, a.partials, a.nch, a.tiles, edges, pairs, a.node_pose, out, out_stride, records,
             rec_stride, rec_off_ij, rec_off_ji, peers ? *peers : PeerRec{});
  L.end(K_DENSE_REDUCE, s);
}

void launch_compose(const bt_pose *a, const bt_pose *b, bt_pose *out, int n, cudaStream_t s, Launch &L) {
  if (n <= 0) return;
  L.begin(K_COMPOSE, s);
  k_compose<<<(n + 127) / 128, 128, 0, s>>>(a, b, out, n);
  L.end(K_COMPOSE, s);
}

}  // namespace bt
