// bt_graph.cu — NEXT-1: one Gauss-Newton step of the pose graph (§IV-D).
//
// Eq. (1): E = sum_{i != j} lambda_1 E_f(i,j) + lambda_2 E_g(i,j).  The per-pair records of
// bt_register_pairs already hold the IRLS-weighted Gauss-Newton blocks at the node poses
// (Eq. (2): H_ii, H_ij, H_jj, g_i, g_j over (T_i, T_j); Eq. (3): H, g of each directed edge
// w.r.t. T_i).  A directed dense edge i -> j only sees T_i T_j^-1, so its Jacobian w.r.t. T_j
// is J_j = -J_i Adj(T_i T_j^-1) with Adj = [[R, [t]x R], [0, R]] on (v, w) twists (reading
// R18): A_ii += H, A_ij += -H Adj, A_jj += Adj^T H Adj, b_i += g, b_j += -Adj^T g.
//
//  k_graph_contrib   one CTA per pair: the pair's 12 x 12 fp64 contribution over (T_i, T_j)
//                    (lambda_1 Eq. (2) block + lambda_2 x both expanded Eq. (3) edges), its
//                    12-vector and energies.
//  k_graph_assemble  one CTA per 6 x 6 node block of A: fixed-order sum over the pairs (no
//                    atomics: bitwise reproducible), the diagonal blocks also sum b.
//  k_graph_pcg       one CTA: preconditioned conjugate gradients on A d = -b in fp64 — the
//                    preconditioner is the diagonal of J^T W J ("the diagonal matrix J^T W J is
//                    used as the preconditioner") or its 6 x 6 node blocks (reading R23:
//                    a node's rotation and translation DOFs are strongly coupled under left
//                    perturbations about the camera origin) — A staged in shared memory when it
//                    fits, warp-per-row mat-vec, fixed-order block reductions; the fixed node's
//                    and unconstrained DOFs held at 0; then T_i <- exp(d_i) T_i.
#include <cuda_runtime.h>

#include "bt_internal.cuh"

namespace bt {
namespace {

constexpr int kContrib = 144 + 12 + 2;          // 12 x 12 over (i, j) row-major, vector, (E_f, E_g)
constexpr int kPcgThreads = 256;

struct GraphArgs {
  int N, P, n_max, rec_stride, fixed, max_iter, precond, stage_a;
  double lf, lg, tol;
  const bt_pose *pose;
  const int32_t *pairs;
  const uint32_t *records;
  double *contrib;                              // [P][kContrib]
  double *A;                                    // [6N][6N]
  double *b;                                    // [6N]
  double *energy;                               // [2]
  bt_pose *new_pose;
  double *delta;
  float *stats;
};

__device__ __forceinline__ bool pair_ok(int i, int j, int N) { return i >= 0 && j >= 0 && i < N && j < N && i != j; }

// Adj(T_a T_b^-1) on (v, w) twists: T_a T_b^-1 = (R_a R_b^T, t_a - R_a R_b^T t_b)
__device__ void adjoint_rel(const bt_pose &Pa, const bt_pose &Pb, double *Adj) {
  double R[9], t[3];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) {
      double x = 0.0;
      for (int k = 0; k < 3; ++k) x += (double)Pa.R[3 * r + k] * (double)Pb.R[3 * c + k];
      R[3 * r + c] = x;
    }
  for (int r = 0; r < 3; ++r)
    t[r] = (double)Pa.t[r] - (R[3 * r] * Pb.t[0] + R[3 * r + 1] * Pb.t[1] + R[3 * r + 2] * Pb.t[2]);
  const double S[9] = {0.0, -t[2], t[1], t[2], 0.0, -t[0], -t[1], t[0], 0.0};
  for (int k = 0; k < 36; ++k) Adj[k] = 0.0;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) {
      double x = 0.0;
      for (int k = 0; k < 3; ++k) x += S[3 * r + k] * R[3 * k + c];
      Adj[6 * r + c] = R[3 * r + c];
      Adj[6 * r + 3 + c] = x;
      Adj[6 * (3 + r) + 3 + c] = R[3 * r + c];
    }
}

// entry (r, c) of a symmetric 6 x 6 stored as its 21-entry upper triangle, row-major
__device__ __forceinline__ int up21(int r, int c) {
  if (r > c) { const int x = r; r = c; c = x; }
  return r * 6 - r * (r - 1) / 2 + (c - r);
}

__global__ void __launch_bounds__(64) k_graph_contrib(GraphArgs A) {
  __shared__ double H1[36], H2[36], Adj1[36], Adj2[36], HA1[36], HA2[36], g1[6], g2[6];
  __shared__ float F[96];
  const int p = blockIdx.x, tid = threadIdx.x;
  const int i = A.pairs[2 * p], j = A.pairs[2 * p + 1];
  double *C = A.contrib + (size_t)p * kContrib;
  if (!pair_ok(i, j, A.N)) {                                       // skipped entry: zero contribution
    for (int k = tid; k < kContrib; k += blockDim.x) C[k] = 0.0;
    return;
  }
  const uint32_t *rec = A.records + (size_t)p * A.rec_stride;
  const float *dij = reinterpret_cast<const float *>(rec + rec_dense_ij(A.n_max));
  const float *dji = reinterpret_cast<const float *>(rec + rec_dense_ji(A.n_max));
  const float *feat = reinterpret_cast<const float *>(rec + rec_feat(A.n_max));
  // a failed registration (S:290's signal: FEW_MATCHES / FEW_INLIERS) contributes no Eq. (2)
  // term — its few "inliers" are not correspondences (reading R30); its dense edges stay
  const int st = (int)rec[kRecStatus];
  const double lf = (st == BT_PAIR_FEW_MATCHES || st == BT_PAIR_FEW_INLIERS) ? 0.0 : A.lf;
  if (tid < 36) {
    const int r = tid / 6, c = tid % 6;
    H1[tid] = dij[up21(r, c)];
    H2[tid] = dji[up21(r, c)];
  } else if (tid < 42) {
    g1[tid - 36] = dij[21 + tid - 36];
    g2[tid - 36] = dji[21 + tid - 36];
  } else if (tid == 42) {
    adjoint_rel(A.pose[i], A.pose[j], Adj1);                       // edge i -> j: Adj(T_i T_j^-1)
  } else if (tid == 43) {
    adjoint_rel(A.pose[j], A.pose[i], Adj2);                       // edge j -> i: Adj(T_j T_i^-1)
  }
  for (int k = tid; k < 96; k += blockDim.x) F[k] = feat[k];
  __syncthreads();
  if (tid < 36) {
    const int r = tid / 6, c = tid % 6;
    double x = 0.0, y = 0.0;
    for (int k = 0; k < 6; ++k) { x += H1[6 * r + k] * Adj1[6 * k + c]; y += H2[6 * r + k] * Adj2[6 * k + c]; }
    HA1[tid] = x;
    HA2[tid] = y;
  }
  __syncthreads();
  for (int e = tid; e < 144; e += blockDim.x) {
    const int R = e / 12, Cc = e % 12, bi = R / 6, bj = Cc / 6, r = R % 6, c = Cc % 6;
    double f, d1, d2;
    if (bi == 0 && bj == 0) {                                      // (i, i)
      f = F[up21(r, c)];
      d1 = H1[6 * r + c];
      d2 = 0.0;
      for (int k = 0; k < 6; ++k) d2 += Adj2[6 * k + r] * HA2[6 * k + c];
    } else if (bi == 1 && bj == 1) {                               // (j, j)
      f = F[57 + up21(r, c)];
      d1 = 0.0;
      for (int k = 0; k < 6; ++k) d1 += Adj1[6 * k + r] * HA1[6 * k + c];
      d2 = H2[6 * r + c];
    } else if (bi == 0) {                                          // (i, j)
      f = F[21 + 6 * r + c];
      d1 = -HA1[6 * r + c];
      d2 = -HA2[6 * c + r];
    } else {                                                       // (j, i)
      f = F[21 + 6 * c + r];
      d1 = -HA1[6 * c + r];
      d2 = -HA2[6 * r + c];
    }
    C[e] = lf * f + A.lg * d1 + A.lg * d2;
  }
  if (tid < 12) {
    const int bi = tid / 6, r = tid % 6;
    double d1, d2;
    if (bi == 0) {
      d1 = g1[r];
      d2 = 0.0;
      for (int k = 0; k < 6; ++k) d2 -= Adj2[6 * k + r] * g2[k];
    } else {
      d1 = 0.0;
      for (int k = 0; k < 6; ++k) d1 -= Adj1[6 * k + r] * g1[k];
      d2 = g2[r];
    }
    C[144 + tid] = lf * (double)F[78 + tid] + A.lg * d1 + A.lg * d2;
  } else if (tid == 12) {
    C[156] = lf * (double)F[90];
    C[157] = A.lg * ((double)dij[27] + (double)dji[27]);
  }
}

// one CTA per node block (a, bn): the pairs touching the block are listed in ascending p
// (ballot compaction over the pair table), then thread (r, c) sums their contributions in that
// order — the same fixed order as a sequential scan, without a serial walk over all P pairs
constexpr int kAsmThreads = 64;
constexpr int kAsmList = 1024;                                     // list capacity per pass

__global__ void __launch_bounds__(kAsmThreads) k_graph_assemble(GraphArgs A) {
  __shared__ int lst[kAsmList];                                    // p << 2 | role
  __shared__ int wcnt[kAsmThreads / 32];
  const int a = blockIdx.y, bn = blockIdx.x, t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int n = 6 * A.N;
  const bool diag = a == bn, energy = a == 0 && bn == 0;
  double s = 0.0;                                                  // t < 36: A block entry; 36..41: b
  for (int p0 = 0; p0 < A.P; p0 += kAsmList) {
    const int p1 = min(A.P, p0 + kAsmList);
    int cnt = 0;
    for (int q0 = p0; q0 < p1; q0 += kAsmThreads) {               // list the touching pairs in order
      const int p = q0 + t;
      int role = -1;
      if (p < p1) {
        const int i = A.pairs[2 * p], j = A.pairs[2 * p + 1];
        if (pair_ok(i, j, A.N)) {
          if (a == i && bn == i) role = 0;
          else if (a == j && bn == j) role = 1;
          else if (a == i && bn == j) role = 2;
          else if (a == j && bn == i) role = 3;
        }
      }
      const unsigned bal = __ballot_sync(0xffffffffu, role >= 0);
      if (lane == 0) wcnt[warp] = __popc(bal);
      __syncthreads();
      int off = cnt;
      for (int w = 0; w < warp; ++w) off += wcnt[w];
      int tot = 0;
      for (int w = 0; w < kAsmThreads / 32; ++w) tot += wcnt[w];
      if (role >= 0) lst[off + __popc(bal & ((1u << lane) - 1u))] = (p << 2) | role;
      cnt += tot;
      __syncthreads();
    }
    if (t < 36) {
      const int r = t / 6, c = t % 6;
      const int o[4] = {12 * r + c, 12 * (6 + r) + 6 + c, 12 * r + 6 + c, 12 * (6 + r) + c};
#pragma unroll 4
      for (int k = 0; k < cnt; ++k) {
        const int v = lst[k];
        s += A.contrib[(size_t)(v >> 2) * kContrib + o[v & 3]];
      }
    } else if (diag && t < 42) {
      const int r = t - 36;
#pragma unroll 4
      for (int k = 0; k < cnt; ++k) {
        const int v = lst[k];
        s += A.contrib[(size_t)(v >> 2) * kContrib + ((v & 3) == 0 ? 144 : 150) + r];
      }
    }
    __syncthreads();                                               // lst reused by the next pass
  }
  if (t < 36) A.A[(size_t)(6 * a + t / 6) * n + 6 * bn + t % 6] = s;
  else if (diag && t < 42) A.b[6 * a + t - 36] = s;
  if (energy && warp == 1) {                                       // energies: fixed-order warp sums
    for (int k = 0; k < 2; ++k) {
      double acc = 0.0;
      for (int p0 = 0; p0 < A.P; p0 += 32) {
        const int p = p0 + lane;
        double v = 0.0;
        if (p < A.P && pair_ok(A.pairs[2 * p], A.pairs[2 * p + 1], A.N)) v = A.contrib[(size_t)p * kContrib + 156 + k];
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        acc += v;
      }
      if (lane == 0) A.energy[k] = acc;
    }
  }
}

// fixed-order block sums of two doubles per thread (results in every thread)
__device__ void block_sum2(double &u, double &v, double *red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    u += __shfl_xor_sync(0xffffffffu, u, o);
    v += __shfl_xor_sync(0xffffffffu, v, o);
  }
  __syncthreads();
  if (lane == 0) { red[warp] = u; red[32 + warp] = v; }
  __syncthreads();
  double su = 0.0, sv = 0.0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) { su += red[w]; sv += red[32 + w]; }
  u = su;
  v = sv;
}

// SE(3) exponential of a (v, w) twist: Rodrigues + V (series below th = 1e-6)
__device__ void se3_exp(const double *xi, double *R, double *t) {
  const double w0 = xi[3], w1 = xi[4], w2 = xi[5];
  const double th2 = w0 * w0 + w1 * w1 + w2 * w2, th = sqrt(th2);
  double a, bb, cc;
  if (th < 1e-6) { a = 1.0 - th2 / 6.0; bb = 0.5 - th2 / 24.0; cc = 1.0 / 6.0 - th2 / 120.0; }
  else { a = sin(th) / th; bb = (1.0 - cos(th)) / th2; cc = (th - sin(th)) / (th2 * th); }
  const double W[9] = {0.0, -w2, w1, w2, 0.0, -w0, -w1, w0, 0.0};
  double W2[9];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) W2[3 * r + c] = W[3 * r] * W[c] + W[3 * r + 1] * W[3 + c] + W[3 * r + 2] * W[6 + c];
  for (int k = 0; k < 9; ++k) R[k] = (k % 4 == 0 ? 1.0 : 0.0) + a * W[k] + bb * W2[k];
  for (int r = 0; r < 3; ++r) {
    double x = 0.0;
    for (int c = 0; c < 3; ++c) x += ((r == c ? 1.0 : 0.0) + bb * W[3 * r + c] + cc * W2[3 * r + c]) * xi[c];
    t[r] = x;
  }
}

// inverse of node i's 6 x 6 diagonal block (pinned rows / columns excluded, 0 in the result)
// by Cholesky; false if the free block is not positive definite
__device__ bool block_inverse(const double *Am, int n, int i, const double *dinv, double *Mi) {
  double M[36], L[36], Li[36];
  for (int r = 0; r < 6; ++r)
    for (int c = 0; c < 6; ++c) {
      const bool fr = dinv[6 * i + r] != 0.0, fc = dinv[6 * i + c] != 0.0;
      M[6 * r + c] = (fr && fc) ? Am[(size_t)(6 * i + r) * n + 6 * i + c] : (r == c ? 1.0 : 0.0);
      L[6 * r + c] = 0.0;
      Li[6 * r + c] = 0.0;
    }
  for (int r = 0; r < 6; ++r)
    for (int c = 0; c <= r; ++c) {
      double s = M[6 * r + c];
      for (int k = 0; k < c; ++k) s -= L[6 * r + k] * L[6 * c + k];
      if (r == c) {
        if (!(s > 0.0)) return false;
        L[6 * r + r] = sqrt(s);
      } else {
        L[6 * r + c] = s / L[6 * c + c];
      }
    }
  for (int c = 0; c < 6; ++c) {                                    // Li = L^-1 (lower)
    Li[6 * c + c] = 1.0 / L[6 * c + c];
    for (int r = c + 1; r < 6; ++r) {
      double s = 0.0;
      for (int k = c; k < r; ++k) s -= L[6 * r + k] * Li[6 * k + c];
      Li[6 * r + c] = s / L[6 * r + r];
    }
  }
  for (int r = 0; r < 6; ++r)                                      // M^-1 = Li^T Li
    for (int c = 0; c < 6; ++c) {
      double s = 0.0;
      for (int k = (r > c ? r : c); k < 6; ++k) s += Li[6 * k + r] * Li[6 * k + c];
      const bool fr = dinv[6 * i + r] != 0.0, fc = dinv[6 * i + c] != 0.0;
      Mi[6 * r + c] = (fr && fc) ? s : 0.0;
    }
  return true;
}

// Graphs of up to 16 nodes (n <= 96 unknowns) keep A in registers: two threads per row, 48
// columns each (A is symmetric, so row `row` is read as column `row` once from global memory);
// the mat-vec then reads only p (broadcast).  Larger graphs read A from shared memory (staged,
// up to kStageLimit) or global memory.
constexpr int kRegN = 96, kRegHalf = kRegN / 2;

__global__ void __launch_bounds__(kPcgThreads, 1) k_graph_pcg(GraphArgs A) {
  extern __shared__ double gsm[];
  const int n = 6 * A.N;
  const bool reg = n <= kRegN;
  const int nv = reg ? kRegN : n;                                  // vector stride (p padded with 0)
  double *x = gsm, *r = x + nv, *z = r + nv, *p = z + nv, *q = p + nv, *dinv = q + nv, *r2 = dinv + nv;
  double *Minv = r2 + nv;                                          // [N][36] block-Jacobi
  double *As = Minv + 36 * A.N;                                    // [n][n] when staged
  const double *Am = A.stage_a ? As : A.A;
  __shared__ double red[64];
  __shared__ double wred[2][kPcgThreads / 32][2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  if (A.stage_a) {                                                 // n even: double2, 8 loads in flight
    const double2 *src = reinterpret_cast<const double2 *>(A.A);
    double2 *dst = reinterpret_cast<double2 *>(As);
    const int n2 = n * n / 2;
#pragma unroll 8
    for (int k = tid; k < n2; k += kPcgThreads) dst[k] = __ldcg(src + k);
  }
  for (int k = tid; k < n; k += blockDim.x) {
    const double dg = A.A[(size_t)k * n + k];
    const bool pin = (k / 6 == A.fixed) || dg == 0.0;
    dinv[k] = pin ? 0.0 : 1.0 / dg;
  }
  __syncthreads();
  if (A.precond == 1)
    for (int i = tid; i < A.N; i += blockDim.x)
      if (!block_inverse(Am, n, i, dinv, Minv + 36 * i))
        for (int k = 0; k < 36; ++k) Minv[36 * i + k] = (k % 7 == 0) ? dinv[6 * i + k / 7] : 0.0;
  for (int k = tid; k < n; k += blockDim.x) {
    x[k] = 0.0;
    r[k] = dinv[k] != 0.0 ? -A.b[k] : 0.0;
  }
  for (int k = n + tid; k < nv; k += blockDim.x) p[k] = 0.0;
  double areg[kRegHalf];
  const int rrow = tid >> 1, rh = tid & 1;
  if (reg) {
    const bool act = rrow < n && dinv[rrow] != 0.0;
#pragma unroll
    for (int j = 0; j < kRegHalf; ++j) {
      const int c = rh * kRegHalf + j;
      areg[j] = (act && c < n) ? __ldcg(A.A + (size_t)c * n + rrow) : 0.0;
    }
  }
  __syncthreads();
  auto apply_m = [&](int k) {                                      // z = M^-1 r
    if (A.precond == 1) {
      const int i = k / 6, rr0 = k % 6;
      double s = 0.0;
      for (int c = 0; c < 6; ++c) s += Minv[36 * i + 6 * rr0 + c] * r[6 * i + c];
      return s;
    }
    return dinv[k] * r[k];
  };
  double bb = 0.0, rz = 0.0;
  for (int k = tid; k < n; k += blockDim.x) {
    z[k] = apply_m(k);
    p[k] = z[k];
    bb += r[k] * r[k];
    rz += r[k] * z[k];
  }
  block_sum2(bb, rz, red);
  double rr = bb;
  const double stop = A.tol * A.tol * bb;
  // Three barriers per iteration: (1) q = A p with the p.q partials, (2) the residual update
  // (double-buffered r, so a node's z = M^-1 r_new is formed from r_old and q without waiting)
  // with the r.r / r.z partials, (3) p = z + beta p.  Warp partials go to alternating halves of
  // `wred`, so a reduction needs one barrier.  A is symmetric: row `row` is read as column
  // `row` (consecutive rows -> consecutive addresses); S threads share a row when 2n <= T.
  const int T = blockDim.x, S = 2 * n <= T ? 2 : 1, h = tid % S;
  double *rn = r2;
  int par = 0, it = 0;
  auto wsum = [&](double &u, double &v) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
      u += __shfl_xor_sync(0xffffffffu, u, o);
      v += __shfl_xor_sync(0xffffffffu, v, o);
    }
    if (lane == 0) { wred[par][warp][0] = u; wred[par][warp][1] = v; }
    __syncthreads();
    double su = 0.0, sv = 0.0;
    for (int w = 0; w < nw; ++w) { su += wred[par][w][0]; sv += wred[par][w][1]; }
    u = su;
    v = sv;
    par ^= 1;
  };
  for (; it < A.max_iter && rr > stop; ++it) {
    double pq = 0.0, dummy = 0.0;
    if (reg) {                                                     // (1) q = A p, A in registers
      double s0 = 0.0, s1 = 0.0;
      const double2 *p2 = reinterpret_cast<const double2 *>(p + rh * kRegHalf);
#pragma unroll
      for (int j = 0; j < kRegHalf / 2; ++j) {
        const double2 pv = p2[j];
        s0 = fma(areg[2 * j], pv.x, s0);
        s1 = fma(areg[2 * j + 1], pv.y, s1);
      }
      double sr = s0 + s1;
      sr += __shfl_xor_sync(0xffffffffu, sr, 1);
      if (rrow < n && rh == 0) {
        q[rrow] = sr;
        pq = p[rrow] * sr;
      }
    } else
    for (int base = 0; base < n; base += T / S) {                  // (1) q = A p
      const int row = base + tid / S;
      double s0 = 0.0, s1 = 0.0;
      if (row < n && dinv[row] != 0.0) {
        const int c0 = h * (n / S), c1 = c0 + n / S;
        int c = c0;
        for (; c + 1 < c1; c += 2) {
          s0 = fma(Am[(size_t)c * n + row], p[c], s0);
          s1 = fma(Am[(size_t)(c + 1) * n + row], p[c + 1], s1);
        }
        if (c < c1) s0 = fma(Am[(size_t)c * n + row], p[c], s0);
      }
      double sr = s0 + s1;
      if (S == 2) sr += __shfl_xor_sync(0xffffffffu, sr, 1);
      if (row < n && h == 0) {
        q[row] = sr;
        pq = fma(p[row], sr, pq);
      }
    }
    wsum(pq, dummy);
    if (!(pq > 0.0)) break;
    const double alpha = rz / pq;
    double rr_l = 0.0, rzn = 0.0;
    for (int k = tid; k < n; k += T) {                             // (2) x, r, z
      x[k] = fma(alpha, p[k], x[k]);
      const double rk = fma(-alpha, q[k], r[k]);
      double zk;
      if (A.precond == 1) {
        const int i = k / 6, a0 = k % 6;
        zk = 0.0;
        for (int c = 0; c < 6; ++c) zk = fma(Minv[36 * i + 6 * a0 + c], fma(-alpha, q[6 * i + c], r[6 * i + c]), zk);
      } else {
        zk = dinv[k] * rk;
      }
      rn[k] = rk;
      z[k] = zk;
      rr_l = fma(rk, rk, rr_l);
      rzn = fma(rk, zk, rzn);
    }
    wsum(rr_l, rzn);
    rr = rr_l;
    const double beta = rzn / rz;
    rz = rzn;
    for (int k = tid; k < n; k += T) p[k] = fma(beta, p[k], z[k]);  // (3)
    double *t_ = r; r = rn; rn = t_;
    __syncthreads();
  }
  __syncthreads();
  for (int i = tid; i < A.N; i += blockDim.x) {                   // T_i <- exp(d_i) T_i
    const bt_pose P0 = A.pose[i];
    double Rd[9], td[3];
    se3_exp(x + 6 * i, Rd, td);
    bt_pose O;
    for (int a = 0; a < 3; ++a) {
      for (int c = 0; c < 3; ++c)
        O.R[3 * a + c] = (float)(Rd[3 * a] * P0.R[c] + Rd[3 * a + 1] * P0.R[3 + c] + Rd[3 * a + 2] * P0.R[6 + c]);
      O.t[a] = (float)(Rd[3 * a] * P0.t[0] + Rd[3 * a + 1] * P0.t[1] + Rd[3 * a + 2] * P0.t[2] + td[a]);
    }
    A.new_pose[i] = O;
    if (A.delta)
      for (int k = 0; k < 6; ++k) A.delta[6 * i + k] = x[6 * i + k];
  }
  if (tid == 0 && A.stats) {
    A.stats[0] = (float)A.energy[0];
    A.stats[1] = (float)A.energy[1];
    A.stats[2] = (float)it;
    A.stats[3] = bb > 0.0 ? (float)sqrt(rr / bb) : 0.f;
  }
}

size_t al256(size_t b) { return (b + 255) / 256 * 256; }

}  // namespace

size_t graph_scratch_bytes(int max_nodes, int max_pairs) {
  const size_t n = 6 * (size_t)max_nodes;
  return al256((size_t)max_pairs * kContrib * 8) + al256(n * n * 8) + al256(n * 8) + al256(16);
}

constexpr size_t kStageLimit = 160 * 1024;     // A staged in shared memory up to this size

bool graph_stage_a(int n_nodes) {
  return 6 * n_nodes > kRegN && (size_t)36 * n_nodes * n_nodes * 8 <= kStageLimit;
}

size_t graph_pcg_smem(int n_nodes) {
  const size_t n = 6 * (size_t)n_nodes, nv = n < (size_t)kRegN ? (size_t)kRegN : n;
  return (7 * nv + 36 * (size_t)n_nodes + (graph_stage_a(n_nodes) ? n * n : 0)) * sizeof(double);
}

void launch_graph(int N, const bt_pose *pose, const int32_t *pairs, int P, const uint32_t *records, int n_max,
                  const bt_graph_params &prm, void *scratch, bt_pose *new_pose, double *delta, float *stats,
                  cudaStream_t s, Launch &L) {
  GraphArgs a;
  a.N = N; a.P = P; a.n_max = n_max; a.rec_stride = rec_words(n_max); a.fixed = prm.fixed_node;
  a.max_iter = prm.max_iter;
  a.precond = prm.precond;
  a.stage_a = graph_stage_a(N) ? 1 : 0;
  a.lf = prm.lambda_feat; a.lg = prm.lambda_dense; a.tol = prm.rel_tol;
  a.pose = pose; a.pairs = pairs; a.records = records;
  char *c = (char *)scratch;
  const size_t n = 6 * (size_t)N;
  a.contrib = (double *)c;  c += al256((size_t)(P > 0 ? P : 1) * kContrib * 8);
  a.A = (double *)c;        c += al256(n * n * 8);
  a.b = (double *)c;        c += al256(n * 8);
  a.energy = (double *)c;
  a.new_pose = new_pose; a.delta = delta; a.stats = stats;
  if (P > 0) {
    L.begin(K_GRAPH, s);
    k_graph_contrib<<<P, 64, 0, s>>>(a);
    L.end(K_GRAPH, s);
  }
  L.begin(K_GRAPH, s);
  k_graph_assemble<<<dim3(N, N), kAsmThreads, 0, s>>>(a);
  L.end(K_GRAPH, s);
  const size_t smem = graph_pcg_smem(N);
  smem_optin((const void *)k_graph_pcg, smem);
  L.begin(K_GRAPH, s);
  k_graph_pcg<<<1, kPcgThreads, smem, s>>>(a);
  L.end(K_GRAPH, s);
}

}  // namespace bt
