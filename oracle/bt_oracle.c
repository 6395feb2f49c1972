/* bt_oracle.c — TEST INFRASTRUCTURE ONLY (see bt_oracle.h).
 *
 * Plain, slow, double-precision CPU oracle of BundleTrack's pairwise registration hot
 * path, written from the paper (arXiv 2108.00516, /root/reference/PAPER.md, "P:n" = line n).
 * It follows the paper's steps in the paper's order; where the paper is silent the reading
 * adopted is the one listed in DESIGN.md §2 ("R1".."R22").  No blocking, fusion or
 * reordering: every loop is the definition written out.  Shares no code with the CUDA path.
 *
 * Parity pins (tests/test_oracle_*.py): Random123 KATs, triple-mapping enumeration,
 * exact SE(3) recovery, brute-force SO(3) search, exhaustive triple enumeration, finite
 * differences of the residuals, analytic plane / identity closed forms.
 */
#include "bt_oracle.h"

#include <float.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

static double band(double th) { return BTO_BAND_REL * (fabs(th) > 1.0 ? fabs(th) : 1.0); }

/* ---------------------------------------------------------------------------------------
 * Counter-based sampler.  P:25 only says "RANSAC"; the north star fixes a counter-based
 * Philox sampler shared by both sides (reading R6).  Philox4x32-10 as published by
 * Salmon et al. (SC'11): 10 rounds of
 *   (hi0,lo0) = M0 * c0, (hi1,lo1) = M1 * c2,  c = (hi1^c1^k0, lo1, hi0^c3^k1, lo0),
 * with the key bumped by the Weyl constants between rounds.
 * ------------------------------------------------------------------------------------- */
void bto_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
  uint32_t k0 = key[0], k1 = key[1];
  for (int round = 0; round < 10; ++round) {
    uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
    uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* "Each registration sample consists of 3 pairs of keypoints": a uniformly random
 * ordered triple of DISTINCT match indices in [0, M), reading R6:
 *   i0 = floor(r0*M / 2^32); i1 = floor(r1*(M-1)/2^32), skip i0; i2 = floor(r2*(M-2)/2^32),
 *   skip min(i0,i1) then max(i0,i1). */
void bto_triple(const uint32_t r[4], int32_t M, int32_t out[3]) {
  uint32_t i0 = (uint32_t)(((uint64_t)r[0] * (uint64_t)M) >> 32);
  uint32_t i1 = (uint32_t)(((uint64_t)r[1] * (uint64_t)(M - 1)) >> 32);
  if (i1 >= i0) i1 += 1;
  uint32_t i2 = (uint32_t)(((uint64_t)r[2] * (uint64_t)(M - 2)) >> 32);
  uint32_t lo = i0 < i1 ? i0 : i1, hi = i0 < i1 ? i1 : i0;
  if (i2 >= lo) i2 += 1;
  if (i2 >= hi) i2 += 1;
  out[0] = (int32_t)i0; out[1] = (int32_t)i1; out[2] = (int32_t)i2;
}

/* ---------------------------------------------------------------------------------------
 * Feature matching, "feature matching and outlier pruning" (P:4).  Readings R1-R4:
 * squared Euclidean distance d(i,j) = sum_k (a_ik - b_jk)^2 (k ascending, double);
 * NN ties -> lowest index; mutual NN; optional Lowe ratio on squared distances;
 * output ascending in i.
 * ------------------------------------------------------------------------------------- */
int32_t bto_match(const float *A, int32_t na, const float *B, int32_t nb, int32_t dim, double ratio,
                  int32_t *pairs, int32_t *nn_ab, int32_t *nn_ba, uint8_t *row_border,
                  uint8_t *col_border, double *d_ab_best) {
  double *D = (double *)malloc(sizeof(double) * (size_t)(na > 0 ? na : 1) * (size_t)(nb > 0 ? nb : 1));
  uint8_t *row_ratio_ok = (uint8_t *)malloc((size_t)(na > 0 ? na : 1));
  for (int32_t i = 0; i < na; ++i)
    for (int32_t j = 0; j < nb; ++j) {
      double s = 0.0;
      for (int32_t k = 0; k < dim; ++k) {
        double d = (double)A[(size_t)i * dim + k] - (double)B[(size_t)j * dim + k];
        s += d * d;
      }
      D[(size_t)i * nb + j] = s;
    }
  double r2 = ratio * ratio;
  for (int32_t i = 0; i < na; ++i) {
    double b1 = INFINITY, b2 = INFINITY;
    int32_t j1 = -1;
    for (int32_t j = 0; j < nb; ++j) {
      double d = D[(size_t)i * nb + j];
      if (d < b1) { b2 = b1; b1 = d; j1 = j; }
      else if (d < b2) { b2 = d; }
    }
    nn_ab[i] = j1;
    if (d_ab_best) d_ab_best[i] = b1;
    uint8_t bd = (nb >= 2) && (b2 - b1 <= band(b1));
    row_ratio_ok[i] = 1;
    if (ratio < 1.0 && nb >= 2) {
      row_ratio_ok[i] = b1 < r2 * b2;
      if (fabs(b1 - r2 * b2) <= band(r2 * b2)) bd = 1;
    }
    row_border[i] = bd;
  }
  for (int32_t j = 0; j < nb; ++j) {
    double b1 = INFINITY, b2 = INFINITY;
    int32_t i1 = -1;
    for (int32_t i = 0; i < na; ++i) {
      double d = D[(size_t)i * nb + j];
      if (d < b1) { b2 = b1; b1 = d; i1 = i; }
      else if (d < b2) { b2 = d; }
    }
    nn_ba[j] = i1;
    col_border[j] = (na >= 2) && (b2 - b1 <= band(b1));
  }
  int32_t M = 0;
  for (int32_t i = 0; i < na; ++i) {
    int32_t j = nn_ab[i];
    if (j >= 0 && nn_ba[j] == i && row_ratio_ok[i]) {
      pairs[2 * M] = i;
      pairs[2 * M + 1] = j;
      ++M;
    }
  }
  free(row_ratio_ok);
  free(D);
  return M;
}

/* ---------------------------------------------------------------------------------------
 * Least squares rigid pose, "generated from a sample via least squares \cite{arun1987least}"
 * (P:25).  Arun, Huang & Blostein 1987, with the det(VU^T) correction (reading R7).
 * ------------------------------------------------------------------------------------- */
void bto_svd3(const double A[9], double U[9], double s[3], double V[9]) {
  double a[9], v[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
  memcpy(a, A, sizeof a);
  /* one-sided (Hestenes) Jacobi: rotate column pairs of a (and v) until orthogonal */
  for (int sweep = 0; sweep < 100; ++sweep) {
    int rotated = 0;
    for (int p = 0; p < 2; ++p)
      for (int q = p + 1; q < 3; ++q) {
        double alpha = 0, beta = 0, gamma = 0;
        for (int r = 0; r < 3; ++r) {
          alpha += a[r * 3 + p] * a[r * 3 + p];
          beta += a[r * 3 + q] * a[r * 3 + q];
          gamma += a[r * 3 + p] * a[r * 3 + q];
        }
        if (gamma == 0.0 || fabs(gamma) <= DBL_EPSILON * sqrt(alpha * beta)) continue;
        rotated = 1;
        double zeta = (beta - alpha) / (2.0 * gamma);
        double t = (zeta >= 0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        double c = 1.0 / sqrt(1.0 + t * t), sn = c * t;
        for (int r = 0; r < 3; ++r) {
          double ap = a[r * 3 + p], aq = a[r * 3 + q];
          a[r * 3 + p] = c * ap - sn * aq;
          a[r * 3 + q] = sn * ap + c * aq;
          double vp = v[r * 3 + p], vq = v[r * 3 + q];
          v[r * 3 + p] = c * vp - sn * vq;
          v[r * 3 + q] = sn * vp + c * vq;
        }
      }
    if (!rotated) break;
  }
  double sv[3];
  for (int k = 0; k < 3; ++k)
    sv[k] = sqrt(a[0 * 3 + k] * a[0 * 3 + k] + a[1 * 3 + k] * a[1 * 3 + k] + a[2 * 3 + k] * a[2 * 3 + k]);
  int ord[3] = {0, 1, 2};
  for (int i = 0; i < 3; ++i)          /* sort descending by singular value */
    for (int j = i + 1; j < 3; ++j)
      if (sv[ord[j]] > sv[ord[i]]) { int tmp = ord[i]; ord[i] = ord[j]; ord[j] = tmp; }
  for (int k = 0; k < 3; ++k) {
    s[k] = sv[ord[k]];
    for (int r = 0; r < 3; ++r) V[r * 3 + k] = v[r * 3 + ord[k]];
  }
  /* U columns: a_k / s_k; completed by orthogonality where s_k vanishes */
  double tiny = 1e-300 + s[0] * 1e-15;
  for (int k = 0; k < 3; ++k) {
    if (s[k] > tiny) {
      for (int r = 0; r < 3; ++r) U[r * 3 + k] = a[r * 3 + ord[k]] / s[k];
    } else if (k == 2) {
      U[0 * 3 + 2] = U[1 * 3 + 0] * U[2 * 3 + 1] - U[2 * 3 + 0] * U[1 * 3 + 1];
      U[1 * 3 + 2] = U[2 * 3 + 0] * U[0 * 3 + 1] - U[0 * 3 + 0] * U[2 * 3 + 1];
      U[2 * 3 + 2] = U[0 * 3 + 0] * U[1 * 3 + 1] - U[1 * 3 + 0] * U[0 * 3 + 1];
    } else {
      /* s1 (and s2) vanish: any unit vector orthogonal to the earlier columns */
      double e[3] = {0, 0, 0};
      int axis = 0;
      double best = 2.0;
      for (int r = 0; r < 3; ++r) {
        double c = fabs(k > 0 ? U[r * 3 + 0] : 0.0);
        if (c < best) { best = c; axis = r; }
      }
      e[axis] = 1.0;
      for (int j = 0; j < k; ++j) {
        double d = e[0] * U[0 * 3 + j] + e[1] * U[1 * 3 + j] + e[2] * U[2 * 3 + j];
        for (int r = 0; r < 3; ++r) e[r] -= d * U[r * 3 + j];
      }
      double nrm = sqrt(e[0] * e[0] + e[1] * e[1] + e[2] * e[2]);
      for (int r = 0; r < 3; ++r) U[r * 3 + k] = e[r] / nrm;
    }
  }
}

static double det3(const double M[9]) {
  return M[0] * (M[4] * M[8] - M[5] * M[7]) - M[1] * (M[3] * M[8] - M[5] * M[6]) +
         M[2] * (M[3] * M[7] - M[4] * M[6]);
}

void bto_arun(const double *pa, const double *pb, int32_t n, double R[9], double t[3],
              double *sig_ratio) {
  double abar[3] = {0, 0, 0}, bbar[3] = {0, 0, 0};
  for (int32_t k = 0; k < n; ++k)
    for (int r = 0; r < 3; ++r) { abar[r] += pa[3 * k + r]; bbar[r] += pb[3 * k + r]; }
  for (int r = 0; r < 3; ++r) { abar[r] /= n; bbar[r] /= n; }
  double Hm[9] = {0};
  for (int32_t k = 0; k < n; ++k)
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c)
        Hm[r * 3 + c] += (pa[3 * k + r] - abar[r]) * (pb[3 * k + c] - bbar[c]);
  double U[9], s[3], V[9];
  bto_svd3(Hm, U, s, V);
  *sig_ratio = s[0] > 0 ? s[1] / s[0] : 0.0;
  double d = det3(V) * det3(U);          /* = det(V U^T) = +-1 */
  double D[3] = {1.0, 1.0, d > 0 ? 1.0 : -1.0};
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) {
      double acc = 0.0;
      for (int k = 0; k < 3; ++k) acc += V[r * 3 + k] * D[k] * U[c * 3 + k];
      R[r * 3 + c] = acc;
    }
  for (int r = 0; r < 3; ++r)
    t[r] = bbar[r] - (R[r * 3 + 0] * abar[0] + R[r * 3 + 1] * abar[1] + R[r * 3 + 2] * abar[2]);
}

/* ---------------------------------------------------------------------------------------
 * Hypothesis evaluation: "inlier correspondences have a distance between
 * transformed point pairs below a threshold delta and an angle formed by the normals
 * within a threshold alpha" — strict gates (R9), unsigned angle without abs (R10).
 * ------------------------------------------------------------------------------------- */
/* returns 1 inlier / 0 outlier; *border = 1 when the decision is within the band */
static int inlier_test(const double R[9], const double t[3], const float *pa, const float *na,
                       const float *pb, const float *nb, double delta, double cos_alpha,
                       int *border) {
  double e[3], rn[3];
  for (int r = 0; r < 3; ++r) {
    e[r] = R[r * 3 + 0] * (double)pa[0] + R[r * 3 + 1] * (double)pa[1] + R[r * 3 + 2] * (double)pa[2] +
           t[r] - (double)pb[r];
    rn[r] = R[r * 3 + 0] * (double)na[0] + R[r * 3 + 1] * (double)na[1] + R[r * 3 + 2] * (double)na[2];
  }
  double dist = sqrt(e[0] * e[0] + e[1] * e[1] + e[2] * e[2]);
  double c = rn[0] * (double)nb[0] + rn[1] * (double)nb[1] + rn[2] * (double)nb[2];
  double bd = band(delta), bc = band(cos_alpha);
  int certain_out = (dist > delta + bd) || (c < cos_alpha - bc);
  int certain_in = (dist < delta - bd) && (c > cos_alpha + bc);
  *border = !certain_out && !certain_in;
  return (dist < delta) && (c > cos_alpha);
}

int32_t bto_inliers(const double T[12], const float *pa, const float *na, const float *pb,
                    const float *nb, int32_t M, double delta, double cos_alpha, uint32_t *mask,
                    uint8_t *border) {
  int32_t cnt = 0;
  if (mask) memset(mask, 0, sizeof(uint32_t) * (size_t)((M + 31) / 32));
  for (int32_t m = 0; m < M; ++m) {
    int bd;
    int in = inlier_test(T, T + 9, pa + 3 * m, na + 3 * m, pb + 3 * m, nb + 3 * m, delta, cos_alpha, &bd);
    if (border) border[m] = (uint8_t)bd;
    if (in) {
      ++cnt;
      if (mask) mask[m / 32] |= 1u << (m % 32);
    }
  }
  return cnt;
}

void bto_ransac_counts(const float *pa, const float *na, const float *pb, const float *nb, int32_t M,
                       int32_t n_hyp, uint32_t pair_uid, uint64_t seed, double delta,
                       double cos_alpha, double tau_deg, int32_t *cnt, int32_t *lo, int32_t *hi,
                       double *hyp, int32_t *tri) {
  const uint32_t key[2] = {(uint32_t)(seed & 0xffffffffu), (uint32_t)(seed >> 32)};
  for (int32_t h = 0; h < n_hyp; ++h) {
    if (M < 3) {                     /* no sample can be drawn (status FEW_MATCHES) */
      cnt[h] = lo[h] = hi[h] = -1;
      if (tri) tri[3 * h] = tri[3 * h + 1] = tri[3 * h + 2] = -1;
      if (hyp) memset(hyp + 12 * h, 0, 12 * sizeof(double));
      continue;
    }
    const uint32_t ctr[4] = {(uint32_t)h, pair_uid, 0u, 0u};
    uint32_t r[4];
    int32_t s3[3];
    bto_philox4x32_10(ctr, key, r);
    bto_triple(r, M, s3);
    double A[9], B[9];
    for (int k = 0; k < 3; ++k)
      for (int c = 0; c < 3; ++c) {
        A[3 * k + c] = (double)pa[3 * s3[k] + c];
        B[3 * k + c] = (double)pb[3 * s3[k] + c];
      }
    double T[12], sig;
    bto_arun(A, B, 3, T, T + 9, &sig);
    if (tri) { tri[3 * h] = s3[0]; tri[3 * h + 1] = s3[1]; tri[3 * h + 2] = s3[2]; }
    if (hyp) memcpy(hyp + 12 * h, T, sizeof T);
    int deg = sig < tau_deg;                                /* reading R8 */
    int deg_border = fabs(sig - tau_deg) <= band(tau_deg);
    if (deg && !deg_border) { cnt[h] = lo[h] = hi[h] = -1; continue; }
    int32_t n_in = 0, n_cin = 0, n_bd = 0;
    for (int32_t m = 0; m < M; ++m) {
      int bd;
      int in = inlier_test(T, T + 9, pa + 3 * m, na + 3 * m, pb + 3 * m, nb + 3 * m, delta, cos_alpha, &bd);
      n_in += in;
      n_bd += bd;
      n_cin += in && !bd;
    }
    cnt[h] = deg ? -1 : n_in;
    lo[h] = deg_border ? -1 : n_cin;
    hi[h] = n_cin + n_bd;
  }
}

static void identity12(double T[12]) {
  memset(T, 0, 12 * sizeof(double));
  T[0] = T[4] = T[8] = 1.0;
}

void bto_ransac_finish(const float *pa, const float *na, const float *pb, const float *nb, int32_t M,
                       int32_t n_hyp, const int32_t *cnt, const double *hyp, double delta,
                       double cos_alpha, double tau_deg, int32_t min_inliers, bto_pair_result *res,
                       uint32_t *mask) {
  memset(res, 0, sizeof *res);
  res->n_matches = M;
  res->best_hyp = -1;
  identity12(res->T_best);
  identity12(res->T_refit);
  int32_t words = (M + 31) / 32;
  if (mask && words > 0) memset(mask, 0, sizeof(uint32_t) * (size_t)words);
  if (M < 3) { res->status = 1; return; }                /* FEW_MATCHES */
  /* "T_t^{t-1} is the best sampled correspondence hypothesis": max count, ties ->
     lowest h (reading R11) */
  int32_t best = 0;
  for (int32_t h = 1; h < n_hyp; ++h)
    if (cnt[h] > cnt[best]) best = h;
  if (n_hyp <= 0 || cnt[best] < 0) { res->status = 2; return; }   /* all degenerate */
  res->best_hyp = best;
  memcpy(res->T_best, hyp + 12 * best, 12 * sizeof(double));
  memcpy(res->T_refit, hyp + 12 * best, 12 * sizeof(double));
  uint32_t *mk = (uint32_t *)calloc((size_t)(words > 0 ? words : 1), sizeof(uint32_t));
  res->best_count = bto_inliers(res->T_best, pa, na, pb, nb, M, delta, cos_alpha, mk, NULL);
  if (mask) memcpy(mask, mk, sizeof(uint32_t) * (size_t)words);
  if (res->best_count < min_inliers) { res->status = 2; free(mk); return; }  /* FEW_INLIERS */
  /* refit on all inliers of h* (north star; reading R12) */
  double *A = (double *)malloc(sizeof(double) * 3 * (size_t)res->best_count);
  double *B = (double *)malloc(sizeof(double) * 3 * (size_t)res->best_count);
  int32_t k = 0;
  for (int32_t m = 0; m < M; ++m)
    if (mk[m / 32] >> (m % 32) & 1u) {
      for (int c = 0; c < 3; ++c) { A[3 * k + c] = pa[3 * m + c]; B[3 * k + c] = pb[3 * m + c]; }
      ++k;
    }
  double T[12], sig;
  bto_arun(A, B, k, T, T + 9, &sig);
  res->refit_sig_ratio = sig;
  if (sig < tau_deg) res->status = 3;                   /* REFIT_DEGENERATE: keep T_best */
  else memcpy(res->T_refit, T, sizeof T);
  free(A); free(B); free(mk);
}

/* ---------------------------------------------------------------------------------------
 * Huber M-estimator, "rho is the M-estimator, where Huber loss is used"; IRLS
 * weight "W ... computed by the M-estimator rho and residual".
 * ------------------------------------------------------------------------------------- */
void bto_huber(double r, double delta, double *rho, double *w) {
  double a = fabs(r);
  if (a <= delta) { *rho = 0.5 * a * a; *w = 1.0; }
  else { *rho = delta * (a - 0.5 * delta); *w = delta / a; }
}

/* pose helpers (double) */
static void pose_of(const float T[12], double R[9], double t[3]) {
  for (int k = 0; k < 9; ++k) R[k] = T[k];
  for (int k = 0; k < 3; ++k) t[k] = T[9 + k];
}
/* x_obj = R^T (x_cam - t) */
static void inv_apply(const double R[9], const double t[3], const double x[3], double y[3]) {
  for (int r = 0; r < 3; ++r)
    y[r] = R[0 * 3 + r] * (x[0] - t[0]) + R[1 * 3 + r] * (x[1] - t[1]) + R[2 * 3 + r] * (x[2] - t[2]);
}
static void skew(const double p[3], double S[9]) {
  S[0] = 0;     S[1] = -p[2]; S[2] = p[1];
  S[3] = p[2];  S[4] = 0;     S[5] = -p[0];
  S[6] = -p[1]; S[7] = p[0];  S[8] = 0;
}

/* ---------------------------------------------------------------------------------------
 * Eq. (2): E_f(i,j) = sum_{(m,n) in C_ij} rho(|| T_i^-1 p_m - T_j^-1 p_n ||).
 * Gauss-Newton blocks ((J^T W J) dxi = J^T W E): J = [J_i | J_j] (3 x 12) of the
 * residual e with respect to the left perturbations T <- exp(d) T, d = (v, w) (R18):
 *   J_i = -R_i^T [ I | -[p_m]x ],   J_j = R_j^T [ I | -[p_n]x ].
 * ------------------------------------------------------------------------------------- */
void bto_feature_edge(const float *pa, const float *pb, const uint32_t *mask, int32_t M,
                      const float Ti[12], const float Tj[12], double huber_delta, double out[186]) {
  double Ri[9], ti[3], Rj[9], tj[3];
  pose_of(Ti, Ri, ti);
  pose_of(Tj, Rj, tj);
  double Hf[12][12], Hs[12][12], g[12], gs[12], E = 0.0;
  memset(Hf, 0, sizeof Hf);
  memset(Hs, 0, sizeof Hs);
  memset(g, 0, sizeof g);
  memset(gs, 0, sizeof gs);
  int32_t count = 0;
  for (int32_t m = 0; m < M; ++m) {
    if (!(mask[m / 32] >> (m % 32) & 1u)) continue;
    double p[3] = {pa[3 * m], pa[3 * m + 1], pa[3 * m + 2]};
    double q[3] = {pb[3 * m], pb[3 * m + 1], pb[3 * m + 2]};
    double xi[3], xj[3], e[3];
    inv_apply(Ri, ti, p, xi);
    inv_apply(Rj, tj, q, xj);
    for (int r = 0; r < 3; ++r) e[r] = xi[r] - xj[r];
    double nrm = sqrt(e[0] * e[0] + e[1] * e[1] + e[2] * e[2]);
    double rho, w;
    bto_huber(nrm, huber_delta, &rho, &w);
    double J[3][12], Sp[9], Sq[9];
    skew(p, Sp);
    skew(q, Sq);
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) {
        double RiT = Ri[c * 3 + r], RjT = Rj[c * 3 + r];   /* (R^T)[r][c] */
        J[r][c] = -RiT;
        J[r][6 + c] = RjT;
        double a = 0.0, b = 0.0;                          /* (R^T [p]x)[r][c] */
        for (int k = 0; k < 3; ++k) { a += Ri[k * 3 + r] * Sp[k * 3 + c]; b += Rj[k * 3 + r] * Sq[k * 3 + c]; }
        J[r][3 + c] = a;
        J[r][9 + c] = -b;
      }
    for (int a = 0; a < 12; ++a) {
      for (int b = 0; b < 12; ++b) {
        double s = 0.0, sa = 0.0;
        for (int r = 0; r < 3; ++r) { s += J[r][a] * J[r][b]; sa += fabs(J[r][a] * J[r][b]); }
        Hf[a][b] += w * s;
        Hs[a][b] += w * sa;
      }
      double s = 0.0, sa = 0.0;
      for (int r = 0; r < 3; ++r) { s += J[r][a] * e[r]; sa += fabs(J[r][a] * e[r]); }
      g[a] += w * s;
      gs[a] += w * sa;
    }
    E += rho;
    ++count;
  }
  memset(out, 0, 186 * sizeof(double));
  int k = 0;
  for (int a = 0; a < 6; ++a)
    for (int b = a; b < 6; ++b) out[k++] = Hf[a][b];               /* H_ii upper */
  for (int a = 0; a < 6; ++a)
    for (int b = 0; b < 6; ++b) out[k++] = Hf[a][6 + b];           /* H_ij */
  for (int a = 0; a < 6; ++a)
    for (int b = a; b < 6; ++b) out[k++] = Hf[6 + a][6 + b];       /* H_jj upper */
  for (int a = 0; a < 12; ++a) out[k++] = g[a];                    /* g_i, g_j */
  out[k++] = E;
  out[k++] = count;
  for (int a = 0; a < 12; ++a) out[96 + a] = gs[a];             /* tolerance scale of g */
  k = 108;                                                       /* tolerance scale of H, same packing */
  for (int a = 0; a < 6; ++a)
    for (int b = a; b < 6; ++b) out[k++] = Hs[a][b];
  for (int a = 0; a < 6; ++a)
    for (int b = 0; b < 6; ++b) out[k++] = Hs[a][6 + b];
  for (int a = 0; a < 6; ++a)
    for (int b = a; b < 6; ++b) out[k++] = Hs[6 + a][6 + b];
}

/* ---------------------------------------------------------------------------------------
 * Eq. (3): E_g(i,j) = sum_{p in I_i} rho( n_i(x) . (T_i T_j^-1 pi_D^-1(pi(T_j T_i^-1 p)) - p) ).
 * "dense pixel-wise correspondences are associated by point re-projection, while outliers
 * are filtered based on the distance between the point pair and the angle formed by their
 * normals".  Readings: nearest-pixel rounding (R14), gates (R15), normals compared
 * in camera i (R16), Huber delta (R17), left-perturbation Jacobian of T_i with the
 * association held fixed, J = [n_i^T, (q x n_i)^T] (R18), all masked valid pixels (R20).
 * ------------------------------------------------------------------------------------- */
/* Contribution of source point p (normal ni) associated with target pixel (uj, vj) of frame j,
   ignoring the gates: J = [n_i, q x n_i], r = n_i . (q - p), Huber weight.  Returns 0 when the
   target pixel is out of bounds or invalid.  Used only for the borderline allowance. */
static int dense_contrib(const float *depth_j, const float *normal_j, const uint8_t *mask_j, int32_t W,
                         int32_t H, double fx, double fy, double cx, double cy, const double Rij[9],
                         const double tij[3], const double p[3], const double ni[3], double huber_delta,
                         int32_t uj, int32_t vj, double *Hfro, double gabs[6], double *rho_out) {
  if (uj < 0 || uj >= W || vj < 0 || vj >= H) return 0;
  size_t pj = (size_t)vj * W + uj;
  double dj = depth_j[pj];
  const float *nj_f = normal_j + 3 * pj;
  if (!mask_j[pj] || !(dj > 0.0) || (nj_f[0] == 0.f && nj_f[1] == 0.f && nj_f[2] == 0.f)) return 0;
  double s[3] = {((double)uj - cx) * dj / fx, ((double)vj - cy) * dj / fy, dj};
  double q[3];
  for (int r = 0; r < 3; ++r)
    q[r] = Rij[r * 3 + 0] * s[0] + Rij[r * 3 + 1] * s[1] + Rij[r * 3 + 2] * s[2] + tij[r];
  double r = ni[0] * (q[0] - p[0]) + ni[1] * (q[1] - p[1]) + ni[2] * (q[2] - p[2]);
  double rho, w;
  bto_huber(r, huber_delta, &rho, &w);
  double J[6] = {ni[0], ni[1], ni[2],
                 q[1] * ni[2] - q[2] * ni[1], q[2] * ni[0] - q[0] * ni[2], q[0] * ni[1] - q[1] * ni[0]};
  double jj = 0.0;
  for (int a = 0; a < 6; ++a) { jj += J[a] * J[a]; gabs[a] = w * fabs(J[a] * r); }
  *Hfro = w * jj;                         /* |w J^T J|_F = w |J|^2 */
  *rho_out = rho;
  return 1;
}

void bto_dense_edge(const float *depth_i, const float *normal_i, const uint8_t *mask_i,
                    const float *depth_j, const float *normal_j, const uint8_t *mask_j,
                    int32_t W, int32_t H, double fx, double fy, double cx, double cy,
                    const float Ti[12], const float Tj[12], double dist_gate, double cos_gate,
                    double huber_delta, int32_t stride, double out[72], int32_t *pix_out,
                    uint8_t *pix_border, double *pix_allow) {
  double Ri[9], ti[3], Rj[9], tj[3];
  pose_of(Ti, Ri, ti);
  pose_of(Tj, Rj, tj);
  /* T_j T_i^-1 : R = R_j R_i^T, t = t_j - R t_i;  T_i T_j^-1 : R = R_i R_j^T, t = t_i - R t_j */
  double Rji[9], tji[3], Rij[9], tij[3];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) {
      double a = 0.0, b = 0.0;
      for (int k = 0; k < 3; ++k) { a += Rj[r * 3 + k] * Ri[c * 3 + k]; b += Ri[r * 3 + k] * Rj[c * 3 + k]; }
      Rji[r * 3 + c] = a;
      Rij[r * 3 + c] = b;
    }
  for (int r = 0; r < 3; ++r) {
    tji[r] = tj[r] - (Rji[r * 3 + 0] * ti[0] + Rji[r * 3 + 1] * ti[1] + Rji[r * 3 + 2] * ti[2]);
    tij[r] = ti[r] - (Rij[r * 3 + 0] * tj[0] + Rij[r * 3 + 1] * tj[1] + Rij[r * 3 + 2] * tj[2]);
  }
  double Hs[6][6], Ha[6][6], g[6], gs[6], E = 0.0;
  double al_g[6] = {0, 0, 0, 0, 0, 0}, al_E = 0.0, al_H = 0.0;   /* borderline allowance */
  memset(Hs, 0, sizeof Hs);
  memset(Ha, 0, sizeof Ha);
  memset(g, 0, sizeof g);
  memset(gs, 0, sizeof gs);
  int32_t count = 0, count_border = 0;
  if (stride < 1) stride = 1;
  for (int32_t v = 0; v < H; ++v)
    for (int32_t u = 0; u < W; ++u) {
      size_t pix = (size_t)v * W + u;
      if (pix_out) pix_out[pix] = -1;
      if (pix_border) pix_border[pix] = 0;
      if (pix_allow) memset(pix_allow + 8 * pix, 0, 8 * sizeof(double));
      if (u % stride || v % stride) continue;
      double d = depth_i[pix];
      const float *ni_f = normal_i + 3 * pix;
      if (!mask_i[pix] || !(d > 0.0) || (ni_f[0] == 0.f && ni_f[1] == 0.f && ni_f[2] == 0.f)) continue;
      double ni[3] = {ni_f[0], ni_f[1], ni_f[2]};
      /* p = pi^-1(x, d): unprojection with pixel centres at integer coordinates */
      double p[3] = {((double)u - cx) * d / fx, ((double)v - cy) * d / fy, d};
      double y[3];
      for (int r = 0; r < 3; ++r)
        y[r] = Rji[r * 3 + 0] * p[0] + Rji[r * 3 + 1] * p[1] + Rji[r * 3 + 2] * p[2] + tji[r];
      if (fabs(y[2]) <= band(0.0)) {      /* never in practice: counted, no allowance bound */
        ++count_border;
        if (pix_border) pix_border[pix] = 1;
        continue;
      }
      if (!(y[2] > 0.0)) continue;
      /* pi(y) and nearest pixel: x' = floor(u' + 0.5) */
      double up = fx * y[0] / y[2] + cx, vp = fy * y[1] / y[2] + cy;
      double fu = up + 0.5 - floor(up + 0.5), fv = vp + 0.5 - floor(vp + 0.5);
      double xu = floor(up + 0.5), xv = floor(vp + 0.5);
      /* targets a correct fp implementation may round to (band rule on the pixel coordinate) */
      int32_t cu[2] = {(int32_t)xu, (int32_t)xu}, cv[2] = {(int32_t)xv, (int32_t)xv};
      int nu = 1, nv = 1;
      if (fu <= band(up)) cu[nu++] = (int32_t)xu - 1;
      else if (1.0 - fu <= band(up)) cu[nu++] = (int32_t)xu + 1;
      if (fv <= band(vp)) cv[nv++] = (int32_t)xv - 1;
      else if (1.0 - fv <= band(vp)) cv[nv++] = (int32_t)xv + 1;
      int border = nu > 1 || nv > 1;
      int pass = 0;
      int32_t uj = (int32_t)xu, vj = (int32_t)xv;
      size_t pj = (size_t)vj * W + uj;
      double q[3], dq[3];
      if (xu >= 0 && xu < W && xv >= 0 && xv < H) {
        double dj = depth_j[pj];
        const float *nj_f = normal_j + 3 * pj;
        if (mask_j[pj] && dj > 0.0 && !(nj_f[0] == 0.f && nj_f[1] == 0.f && nj_f[2] == 0.f)) {
          /* s = pi_D^-1(x'), q = T_i T_j^-1 s */
          double s[3] = {((double)uj - cx) * dj / fx, ((double)vj - cy) * dj / fy, dj};
          double nj[3];
          for (int r = 0; r < 3; ++r) {
            q[r] = Rij[r * 3 + 0] * s[0] + Rij[r * 3 + 1] * s[1] + Rij[r * 3 + 2] * s[2] + tij[r];
            nj[r] = Rij[r * 3 + 0] * nj_f[0] + Rij[r * 3 + 1] * nj_f[1] + Rij[r * 3 + 2] * nj_f[2];
            dq[r] = q[r] - p[r];
          }
          double dist = sqrt(dq[0] * dq[0] + dq[1] * dq[1] + dq[2] * dq[2]);
          double c = ni[0] * nj[0] + ni[1] * nj[1] + ni[2] * nj[2];
          pass = (dist < dist_gate) && (c > cos_gate);
          int certain_out = (dist > dist_gate + band(dist_gate)) || (c < cos_gate - band(cos_gate));
          int certain_in = (dist < dist_gate - band(dist_gate)) && (c > cos_gate + band(cos_gate));
          if (!certain_out && !certain_in) border = 1;
        }
      }
      if (border) {
        /* allowance: the largest contribution over every target this pixel may round to */
        ++count_border;
        if (pix_border) pix_border[pix] = 1;
        double mh = 0.0, me = 0.0, mg[6] = {0, 0, 0, 0, 0, 0};
        for (int a = 0; a < nu; ++a)
          for (int b = 0; b < nv; ++b) {
            double hf, ga[6], rh;
            if (!dense_contrib(depth_j, normal_j, mask_j, W, H, fx, fy, cx, cy, Rij, tij, p, ni, huber_delta,
                               cu[a], cv[b], &hf, ga, &rh))
              continue;
            if (hf > mh) mh = hf;
            if (rh > me) me = rh;
            for (int k = 0; k < 6; ++k) if (ga[k] > mg[k]) mg[k] = ga[k];
          }
        al_H += mh;
        al_E += me;
        for (int k = 0; k < 6; ++k) al_g[k] += mg[k];
        if (pix_allow) {
          double *pa_ = pix_allow + 8 * pix;
          pa_[0] = mh;
          pa_[1] = me;
          for (int k = 0; k < 6; ++k) pa_[2 + k] = mg[k];
        }
      }
      if (!pass) continue;
      double r = ni[0] * dq[0] + ni[1] * dq[1] + ni[2] * dq[2];
      double rho, w;
      bto_huber(r, huber_delta, &rho, &w);
      double J[6] = {ni[0], ni[1], ni[2],
                     q[1] * ni[2] - q[2] * ni[1], q[2] * ni[0] - q[0] * ni[2], q[0] * ni[1] - q[1] * ni[0]};
      for (int a = 0; a < 6; ++a) {
        for (int b = 0; b < 6; ++b) { Hs[a][b] += w * J[a] * J[b]; Ha[a][b] += w * fabs(J[a] * J[b]); }
        g[a] += w * J[a] * r;
        gs[a] += w * fabs(J[a] * r);
      }
      E += rho;
      ++count;
      if (pix_out) pix_out[pix] = (int32_t)pj;
    }
  memset(out, 0, 72 * sizeof(double));
  int k = 48;                                                    /* tolerance scale of H (upper) */
  for (int a = 0; a < 6; ++a)
    for (int b = a; b < 6; ++b) out[k++] = Ha[a][b];
  k = 0;
  for (int a = 0; a < 6; ++a)
    for (int b = a; b < 6; ++b) out[k++] = Hs[a][b];
  for (int a = 0; a < 6; ++a) out[k++] = g[a];
  out[k++] = E;
  out[k++] = count;
  out[k++] = count_border;
  for (int a = 0; a < 6; ++a) out[32 + a] = gs[a];              /* tolerance scale of g */
  for (int a = 0; a < 6; ++a) out[38 + a] = al_g[a];            /* borderline allowances */
  out[44] = al_E;
  out[45] = al_H;
}

/* ======================================================================= NEXT-1: pose graph
   PAPER.md §IV-D: Gauss-Newton on Eq. (1) with IRLS weights, the update
   xi <- xi [+] d accumulated on the left, T_i = exp(xi_i); the initial frame's node fixed. */

void bto_se3_exp(const double xi[6], double R[9], double t[3]) {
  const double v[3] = {xi[0], xi[1], xi[2]}, w[3] = {xi[3], xi[4], xi[5]};
  const double th2 = w[0] * w[0] + w[1] * w[1] + w[2] * w[2], th = sqrt(th2);
  double A, B, Cc;                                 /* sin th / th, (1 - cos th)/th^2, (th - sin th)/th^3 */
  if (th < 1e-6) {
    A = 1.0 - th2 / 6.0;
    B = 0.5 - th2 / 24.0;
    Cc = 1.0 / 6.0 - th2 / 120.0;
  } else {
    A = sin(th) / th;
    B = (1.0 - cos(th)) / th2;
    Cc = (th - sin(th)) / (th2 * th);
  }
  double W[9], W2[9];
  skew(w, W);
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) {
      double x = 0.0;
      for (int k = 0; k < 3; ++k) x += W[3 * r + k] * W[3 * k + c];
      W2[3 * r + c] = x;
    }
  for (int k = 0; k < 9; ++k) {
    const double I = (k % 4 == 0) ? 1.0 : 0.0;
    R[k] = I + A * W[k] + B * W2[k];
  }
  for (int r = 0; r < 3; ++r) {
    double x = 0.0;
    for (int c = 0; c < 3; ++c) {
      const double I = (r == c) ? 1.0 : 0.0;
      x += (I + B * W[3 * r + c] + Cc * W2[3 * r + c]) * v[c];
    }
    t[r] = x;
  }
}

void bto_se3_adjoint(const double R[9], const double t[3], double Adj[36]) {
  double S[9];
  skew(t, S);
  for (int k = 0; k < 36; ++k) Adj[k] = 0.0;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) {
      double tr = 0.0;
      for (int k = 0; k < 3; ++k) tr += S[3 * r + k] * R[3 * k + c];
      Adj[6 * r + c] = R[3 * r + c];
      Adj[6 * r + 3 + c] = tr;
      Adj[6 * (3 + r) + 3 + c] = R[3 * r + c];
    }
}

/* unpack a 21-entry upper-triangular row-major 6x6 block */
static void sym6(const double *u, double H[36]) {
  int k = 0;
  for (int a = 0; a < 6; ++a)
    for (int b = a; b < 6; ++b) { H[6 * a + b] = u[k]; H[6 * b + a] = u[k]; ++k; }
}

static void add_block(double *A, int n, int bi, int bj, const double *M, double s) {
  for (int r = 0; r < 6; ++r)
    for (int c = 0; c < 6; ++c) A[(size_t)(6 * bi + r) * n + 6 * bj + c] += s * M[6 * r + c];
}

/* A_ii += H, A_ij += -H Adj, A_ji += -(H Adj)^T, A_jj += Adj^T H Adj, b_i += g, b_j += -Adj^T g */
static void add_dense(double *A, double *b, int n, int i, int j, const double *blk, const double Ri[9],
                      const double ti[3], const double Rj[9], const double tj[3], double lam) {
  double H[36], Adj[36], HA[36], AHA[36], R[9], t[3];
  sym6(blk, H);
  /* T_i T_j^-1 = (R_i R_j^T, t_i - R_i R_j^T t_j) */
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) {
      double x = 0.0;
      for (int k = 0; k < 3; ++k) x += Ri[3 * r + k] * Rj[3 * c + k];
      R[3 * r + c] = x;
    }
  for (int r = 0; r < 3; ++r) t[r] = ti[r] - (R[3 * r] * tj[0] + R[3 * r + 1] * tj[1] + R[3 * r + 2] * tj[2]);
  bto_se3_adjoint(R, t, Adj);
  for (int r = 0; r < 6; ++r)
    for (int c = 0; c < 6; ++c) {
      double x = 0.0;
      for (int k = 0; k < 6; ++k) x += H[6 * r + k] * Adj[6 * k + c];
      HA[6 * r + c] = x;
    }
  for (int r = 0; r < 6; ++r)
    for (int c = 0; c < 6; ++c) {
      double x = 0.0;
      for (int k = 0; k < 6; ++k) x += Adj[6 * k + r] * HA[6 * k + c];
      AHA[6 * r + c] = x;
    }
  double HAt[36];
  for (int r = 0; r < 6; ++r)
    for (int c = 0; c < 6; ++c) HAt[6 * r + c] = HA[6 * c + r];
  add_block(A, n, i, i, H, lam);
  add_block(A, n, i, j, HA, -lam);
  add_block(A, n, j, i, HAt, -lam);
  add_block(A, n, j, j, AHA, lam);
  for (int r = 0; r < 6; ++r) {
    double x = 0.0;
    for (int k = 0; k < 6; ++k) x += Adj[6 * k + r] * blk[21 + k];
    b[6 * i + r] += lam * blk[21 + r];
    b[6 * j + r] -= lam * x;
  }
}

int32_t bto_graph_system(int32_t n_nodes, const float *poses, const int32_t *pairs, int32_t P,
                         const double *feat, const double *dense_ij, const double *dense_ji,
                         const int32_t *status, double lambda_f, double lambda_g, double *A, double *b,
                         double energy[2]) {
  const int n = 6 * n_nodes;
  memset(A, 0, sizeof(double) * (size_t)n * n);
  memset(b, 0, sizeof(double) * (size_t)n);
  energy[0] = energy[1] = 0.0;
  for (int p = 0; p < P; ++p) {
    const int i = pairs[2 * p], j = pairs[2 * p + 1];
    if (i < 0 || j < 0 || i >= n_nodes || j >= n_nodes || i == j) return -1;
    /* Eq. (2) blocks, as given (12 x 12 over [i, j]); none for a failed registration (R30) */
    const double *f = feat + (size_t)96 * p;
    const double lf = (status && (status[p] == 1 || status[p] == 2)) ? 0.0 : lambda_f;
    double Hii[36], Hjj[36], Hij[36], Hji[36];
    sym6(f, Hii);
    sym6(f + 57, Hjj);
    for (int r = 0; r < 6; ++r)
      for (int c = 0; c < 6; ++c) { Hij[6 * r + c] = f[21 + 6 * r + c]; Hji[6 * c + r] = f[21 + 6 * r + c]; }
    add_block(A, n, i, i, Hii, lf);
    add_block(A, n, i, j, Hij, lf);
    add_block(A, n, j, i, Hji, lf);
    add_block(A, n, j, j, Hjj, lf);
    for (int r = 0; r < 6; ++r) { b[6 * i + r] += lf * f[78 + r]; b[6 * j + r] += lf * f[84 + r]; }
    energy[0] += lf * f[90];
    /* Eq. (3) blocks of both directed edges */
    double Ri[9], ti[3], Rj[9], tj[3];
    pose_of(poses + 12 * i, Ri, ti);
    pose_of(poses + 12 * j, Rj, tj);
    if (dense_ij) {
      add_dense(A, b, n, i, j, dense_ij + (size_t)32 * p, Ri, ti, Rj, tj, lambda_g);
      energy[1] += lambda_g * dense_ij[(size_t)32 * p + 27];
    }
    if (dense_ji) {
      add_dense(A, b, n, j, i, dense_ji + (size_t)32 * p, Rj, tj, Ri, ti, lambda_g);
      energy[1] += lambda_g * dense_ji[(size_t)32 * p + 27];
    }
  }
  return 0;
}

int32_t bto_graph_step(int32_t n_nodes, const float *poses, const int32_t *pairs, int32_t P,
                       const double *feat, const double *dense_ij, const double *dense_ji,
                       const int32_t *status, double lambda_f, double lambda_g, int32_t fixed_node,
                       double *delta, float *new_poses, double energy[2]) {
  const int n = 6 * n_nodes;
  double *A = (double *)malloc(sizeof(double) * (size_t)n * n);
  double *b = (double *)malloc(sizeof(double) * (size_t)n);
  int *free_idx = (int *)malloc(sizeof(int) * (size_t)n);
  int32_t st = bto_graph_system(n_nodes, poses, pairs, P, feat, dense_ij, dense_ji, status, lambda_f, lambda_g, A, b,
                                energy);
  int m = 0;
  for (int k = 0; k < n; ++k) {
    delta[k] = 0.0;
    if (k / 6 != fixed_node && A[(size_t)k * n + k] != 0.0) free_idx[m++] = k;
  }
  /* Cholesky of the free block, L L^T = A_ff (lower triangle in place in L) */
  double *L = (double *)calloc((size_t)m * m + 1, sizeof(double));
  double *y = (double *)calloc((size_t)m + 1, sizeof(double));
  for (int r = 0; r < m && st == 0; ++r)
    for (int c = 0; c <= r; ++c) {
      double s = A[(size_t)free_idx[r] * n + free_idx[c]];
      for (int k = 0; k < c; ++k) s -= L[(size_t)r * m + k] * L[(size_t)c * m + k];
      if (r == c) {
        if (!(s > 0.0)) { st = -1; break; }
        L[(size_t)r * m + r] = sqrt(s);
      } else {
        L[(size_t)r * m + c] = s / L[(size_t)c * m + c];
      }
    }
  if (st == 0) {
    for (int r = 0; r < m; ++r) {                  /* L y = -b_f */
      double s = -b[free_idx[r]];
      for (int k = 0; k < r; ++k) s -= L[(size_t)r * m + k] * y[k];
      y[r] = s / L[(size_t)r * m + r];
    }
    for (int r = m - 1; r >= 0; --r) {             /* L^T d = y */
      double s = y[r];
      for (int k = r + 1; k < m; ++k) s -= L[(size_t)k * m + r] * delta[free_idx[k]];
      delta[free_idx[r]] = s / L[(size_t)r * m + r];
    }
  }
  for (int i = 0; i < n_nodes; ++i) {              /* T_i <- exp(d_i) T_i */
    double Rd[9], td[3], R[9], t[3];
    bto_se3_exp(delta + 6 * i, Rd, td);
    pose_of(poses + 12 * i, R, t);
    for (int r = 0; r < 3; ++r) {
      for (int c = 0; c < 3; ++c) {
        double x = 0.0;
        for (int k = 0; k < 3; ++k) x += Rd[3 * r + k] * R[3 * k + c];
        new_poses[12 * i + 3 * r + c] = (float)x;
      }
      new_poses[12 * i + 9 + r] = (float)(Rd[3 * r] * t[0] + Rd[3 * r + 1] * t[1] + Rd[3 * r + 2] * t[2] + td[r]);
    }
  }
  free(A); free(b); free(free_idx); free(L); free(y);
  return st;
}

/* ============================================================ NEXT-2: tracker decisions */
double bto_rot_geodesic(const float Ta[12], const float Tb[12]) {
  double tr = 0.0;                                        /* tr(Ra^T Rb) = sum_ij Ra_ij Rb_ij */
  for (int k = 0; k < 9; ++k) tr += (double)Ta[k] * (double)Tb[k];
  double c = (tr - 1.0) / 2.0;
  if (c > 1.0) c = 1.0;
  if (c < -1.0) c = -1.0;
  return acos(c);
}

void bto_coarse_pose(int32_t status, const float T_best[12], const float T_prev[12], float out[12]) {
  if (status != 0 && status != 3) {                       /* no sampled hypothesis */
    for (int k = 0; k < 12; ++k) out[k] = T_prev[k];
    return;
  }
  for (int r = 0; r < 3; ++r) {
    for (int c = 0; c < 3; ++c) {
      double x = 0.0;
      for (int k = 0; k < 3; ++k) x += (double)T_best[3 * r + k] * (double)T_prev[3 * k + c];
      out[3 * r + c] = (float)x;
    }
    double y = T_best[9 + r];
    for (int k = 0; k < 3; ++k) y += (double)T_best[3 * r + k] * (double)T_prev[9 + k];
    out[9 + r] = (float)y;
  }
}

int32_t bto_select_keyframes(const float *pool, int32_t n_pool, const float cur[12], int32_t K, int32_t *sel) {
  if (n_pool <= 0 || K <= 0) return 0;
  int32_t n_sel = 0;
  sel[n_sel++] = 0;                                       /* I_0 */
  while (n_sel < K && n_sel < n_pool) {
    int32_t best = -1;
    double best_s = 0.0;
    for (int32_t k = 0; k < n_pool; ++k) {
      int taken = 0;
      for (int32_t q = 0; q < n_sel; ++q) taken |= sel[q] == k;
      if (taken) continue;
      double s = bto_rot_geodesic(pool + 12 * k, cur);
      for (int32_t q = 0; q < n_sel; ++q) s += bto_rot_geodesic(pool + 12 * k, pool + 12 * sel[q]);
      if (best < 0 || s < best_s) { best = k; best_s = s; }
    }
    sel[n_sel++] = best;
  }
  return n_sel;
}

int32_t bto_is_novel(const float *pool, int32_t n_pool, const float cur[12], double thresh_rad) {
  for (int32_t k = 0; k < n_pool; ++k)
    if (!(bto_rot_geodesic(pool + 12 * k, cur) > thresh_rad)) return 0;
  return 1;
}

/* ============================================================ NEXT-4: keypoint lifting (R29) */
void bto_lift_keypoints(int32_t F, int32_t n_max, int32_t dim, const float *uv, const float *desc_in,
                        const int32_t *n_in, const float *depth, const float *normal, const uint8_t *mask,
                        int32_t W, int32_t H, double fx, double fy, double cx, double cy, int32_t *n_out,
                        float *desc, float *pts, float *nrm, uint8_t *border) {
  for (int32_t f = 0; f < F; ++f) {
    int32_t m = 0;
    const int32_t n = n_in[f] < n_max ? n_in[f] : n_max;
    for (int32_t k = 0; k < n; ++k) {
      const size_t in = (size_t)f * n_max + k;
      const double u = uv[2 * in], v = uv[2 * in + 1];
      const double xu = floor(u + 0.5), xv = floor(v + 0.5);   /* nearest pixel (R14) */
      if (border) {
        const double fu = u + 0.5 - xu, fv = v + 0.5 - xv;
        border[in] = fu <= band(u + 0.5) || 1.0 - fu <= band(u + 0.5) || fv <= band(v + 0.5) ||
                     1.0 - fv <= band(v + 0.5);
      }
      if (!(xu >= 0.0 && xu < W && xv >= 0.0 && xv < H)) continue;
      const size_t px = (size_t)f * W * H + (size_t)xv * W + (size_t)xu;
      const double d = depth[px];
      const float *nm = normal + 3 * px;
      if (!mask[px] || !(d > 0.0) || (nm[0] == 0.f && nm[1] == 0.f && nm[2] == 0.f)) continue;
      const size_t o = (size_t)f * n_max + m;
      pts[3 * o + 0] = (float)((u - cx) * d / fx);         /* pi_D^-1 at the keypoint */
      pts[3 * o + 1] = (float)((v - cy) * d / fy);
      pts[3 * o + 2] = (float)d;
      for (int c = 0; c < 3; ++c) nrm[3 * o + c] = nm[c];
      for (int32_t c = 0; c < dim; ++c) desc[o * dim + c] = desc_in[in * dim + c];
      ++m;
    }
    n_out[f] = m;
  }
}

/* ======================================================================= NEXT-4: normals */
void bto_estimate_normals(const float *depth, int32_t F, int32_t W, int32_t H, double fx, double fy,
                          double cx, double cy, float jump, float *normal) {
  for (int f = 0; f < F; ++f)
    for (int v = 0; v < H; ++v)
      for (int u = 0; u < W; ++u) {
        const float *D = depth + (size_t)f * W * H;
        float *out = normal + 3 * ((size_t)f * W * H + (size_t)v * W + u);
        out[0] = out[1] = out[2] = 0.0f;
        const double d = D[v * W + u];
        if (!(d > 0.0) || u == 0 || v == 0 || u == W - 1 || v == H - 1) continue;
        const int nu[4] = {u - 1, u + 1, u, u};
        const int nv[4] = {v, v, v - 1, v + 1};
        double P[4][3];
        int ok = 1;
        for (int k = 0; k < 4; ++k) {
          const double dk = D[nv[k] * W + nu[k]];
          if (!(dk > 0.0) || fabs(dk - d) > (double)jump) { ok = 0; break; }
          P[k][0] = (nu[k] - cx) * dk / fx;
          P[k][1] = (nv[k] - cy) * dk / fy;
          P[k][2] = dk;
        }
        if (!ok) continue;
        const double tu[3] = {P[1][0] - P[0][0], P[1][1] - P[0][1], P[1][2] - P[0][2]};
        const double tv[3] = {P[3][0] - P[2][0], P[3][1] - P[2][1], P[3][2] - P[2][2]};
        double n[3] = {tu[1] * tv[2] - tu[2] * tv[1], tu[2] * tv[0] - tu[0] * tv[2], tu[0] * tv[1] - tu[1] * tv[0]};
        const double nn = sqrt(n[0] * n[0] + n[1] * n[1] + n[2] * n[2]);
        if (!(nn > 0.0)) continue;
        const double pc[3] = {(u - cx) * d / fx, (v - cy) * d / fy, d};
        const double s = (n[0] * pc[0] + n[1] * pc[1] + n[2] * pc[2]) > 0.0 ? -1.0 / nn : 1.0 / nn;
        for (int k = 0; k < 3; ++k) out[k] = (float)(n[k] * s);
      }
}
