/* bt_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, double-precision CPU oracle of BundleTrack's pairwise registration hot
 * path (arXiv 2108.00516, §IV-B P:25 and §IV-D Eq. (2)/(3) P:54-72).  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it.  It shares
 * no code, header, table or constant generator with the CUDA library
 * (paper_2108_00516_b200/csrc, include/bt.h); neither side includes the other.
 *
 * Inputs are the same float32 arrays the CUDA path receives; every value is converted
 * exactly to double before any arithmetic.  Layout conventions (identical by contract,
 * not by shared code): poses are 12 floats, R row-major then t, object->camera
 * (x_cam = R x_obj + t); points / normals are [n][3]; descriptors [n][dim].
 */
#ifndef BT_ORACLE_H
#define BT_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

/* band rule (north star "excluding points within 1e-6 of a threshold"):
   a decision on the double value x against threshold th is borderline iff
   |x - th| <= 1e-6 * max(1, |th|). */
#define BTO_BAND_REL 1e-6

/* Philox4x32-10 (Salmon et al., SC'11 "Parallel random numbers: as easy as 1, 2, 3"). */
void bto_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);

/* Distinct ordered triple in [0, M) from three 32-bit words (reading R6). */
void bto_triple(const uint32_t r[4], int32_t M, int32_t out[3]);

/* Brute-force mutual nearest neighbours (readings R1-R4).
   Returns the number of matches M; pairs[M][2] = (i, j) ascending in i.
   nn_ab[na], nn_ba[nb]: nearest neighbour indices (-1 if the other set is empty).
   row_border[na] / col_border[nb]: 1 iff best and second-best squared distances are
   within the band (ambiguous nearest neighbour), or the ratio test is borderline.
   d_ab_best[na] (may be NULL): the best squared distance per row. */
int32_t bto_match(const float *A, int32_t na, const float *B, int32_t nb, int32_t dim, double ratio,
                  int32_t *pairs, int32_t *nn_ab, int32_t *nn_ba, uint8_t *row_border,
                  uint8_t *col_border, double *d_ab_best);

/* Arun et al. 1987 least squares: R, t minimising sum ||R a_k + t - b_k||^2 over SO(3)
   via the SVD of H = sum (a_k - abar)(b_k - bbar)^T = U S V^T, R = V diag(1,1,det(VU^T)) U^T,
   t = bbar - R abar.  sig_ratio = s2/s1 (0 when s1 = 0).  pa, pb: [n][3] double. */
void bto_arun(const double *pa, const double *pb, int32_t n, double R[9], double t[3],
              double *sig_ratio);

/* One-sided Jacobi SVD of a 3x3 matrix (exposed for tests): A = U diag(s) V^T, s descending. */
void bto_svd3(const double A[9], double U[9], double s[3], double V[9]);

/* RANSAC over 3-correspondence samples.  pa/na/pb/nb: [M][3] float (the matched
   keypoint points and normals of frames a and b, in match order).  For every hypothesis h:
     cnt[h]  = the oracle's own count (double decisions), -1 if degenerate;
     lo[h], hi[h] = the interval any correct fp implementation's count must lie in
                    (borderline tests / degeneracy excluded per the band rule);
     hyp[h][12] (may be NULL) = the hypothesis pose (R row-major, t);
     tri[h][3]  (may be NULL) = the sampled triple. */
void bto_ransac_counts(const float *pa, const float *na, const float *pb, const float *nb, int32_t M,
                       int32_t n_hyp, uint32_t pair_uid, uint64_t seed, double delta,
                       double cos_alpha, double tau_deg, int32_t *cnt, int32_t *lo, int32_t *hi,
                       double *hyp, int32_t *tri);

/* Inlier test of one pose on all M correspondences (P:25 gates), double decisions.
   mask: ceil(M/32) words, bit m of word m/32.  border (may be NULL): per-m 1 iff the
   decision is borderline.  Returns the count. */
int32_t bto_inliers(const double T[12], const float *pa, const float *na, const float *pb,
                    const float *nb, int32_t M, double delta, double cos_alpha, uint32_t *mask,
                    uint8_t *border);

/* Per-pair record, oracle side (double). */
typedef struct {
  int32_t status;      /* 0 OK, 1 FEW_MATCHES, 2 FEW_INLIERS, 3 REFIT_DEGENERATE */
  int32_t n_matches;
  int32_t best_hyp;    /* -1 if none */
  int32_t best_count;
  double T_best[12];
  double T_refit[12];
  double refit_sig_ratio;
} bto_pair_result;

/* Select h* (max count, ties -> lowest h), build C_ij = inliers(h*), refit (Arun on
   C_ij, north star), status.  cnt from bto_ransac_counts.  mask: ceil(M/32) words out. */
void bto_ransac_finish(const float *pa, const float *na, const float *pb, const float *nb, int32_t M,
                       int32_t n_hyp, const int32_t *cnt, const double *hyp, double delta,
                       double cos_alpha, double tau_deg, int32_t min_inliers, bto_pair_result *res,
                       uint32_t *mask);

/* Huber M-estimator: value and IRLS weight of a residual magnitude r >= 0. */
void bto_huber(double r, double delta, double *rho, double *w);

/* Eq. (2) feature-edge linearization at node poses Ti, Tj (12 floats each):
   e = Ti^-1 p_m - Tj^-1 p_n over the masked correspondences; left perturbation
   T <- exp(d) T, twist order (v, w).  out[186]: H_ii(21, upper row-major) H_ij(36 row-major)
   H_jj(21) g_i(6) g_j(6) E(1) count(1) pad(4), then (oracle only) [96..107] the tolerance
   scale of g, sum w |J_k| . |e|, and [108..185] the tolerance scale of H in the same 78-entry
   packing, sum w sum_r |J_ra J_rb| (the sum of absolute contributions: the magnitude that
   floating-point summation error is relative to).  H = sum w J^T J, g = sum w J^T e,
   E = sum rho(||e||). */
void bto_feature_edge(const float *pa, const float *pb, const uint32_t *mask, int32_t M,
                      const float Ti[12], const float Tj[12], double huber_delta, double out[186]);

/* Eq. (3) dense point-to-plane edge i -> j.  Maps: depth [H][W], normal [H][W][3],
   mask [H][W].  out[72]: H(21 upper) g(6) E count count_border pad(2), then (oracle only)
   [32..37] sum w |J_k r| (the scale the g tolerance is relative to), the borderline
   allowance — summed over borderline pixels, the largest contribution over every target
   pixel the pixel may round to: [38..43] w |J_k r|, [44] rho, [45] w |J|^2 (>= |w J^T J|_F),
   pad(2), and [48..68] sum w |J_a J_b| (upper, the scale of an element-wise H tolerance).
   pix_out (may be NULL): [H][W] int32 per source pixel: -1 skipped or rejected by a gate,
   else the associated target pixel index y'*W+x' (both gates passed).  pix_border (may be
   NULL): [H][W] u8, 1 iff borderline.  pix_allow (may be NULL): [H][W][8] the allowance of
   each borderline pixel (w |J|^2, rho, w |J_k r| x 6; zero elsewhere), so a comparison can
   charge only the pixels whose decision actually differs. */
void bto_dense_edge(const float *depth_i, const float *normal_i, const uint8_t *mask_i,
                    const float *depth_j, const float *normal_j, const uint8_t *mask_j,
                    int32_t W, int32_t H, double fx, double fy, double cx, double cy,
                    const float Ti[12], const float Tj[12], double dist_gate, double cos_gate,
                    double huber_delta, int32_t stride, double out[72], int32_t *pix_out,
                    uint8_t *pix_border, double *pix_allow);

/* ---- NEXT-1: pose-graph Gauss-Newton step (§IV-D) -------------------
   Twists are (v, w) (translation first), perturbations are on the left: T <- exp(d) T
   (reading R18). */

/* SE(3) exponential: R = exp([w]x) (Rodrigues), t = V v with
   V = I + (1 - cos th)/th^2 [w]x + (th - sin th)/th^3 [w]x^2 (series below th = 1e-6). */
void bto_se3_exp(const double xi[6], double R[9], double t[3]);

/* Adjoint of T = (R, t) on (v, w) twists, 6x6 row-major: [[R, [t]x R], [0, R]], so that
   exp(Adj_T d) T = T exp(d). */
void bto_se3_adjoint(const double R[9], const double t[3], double Adj[36]);

/* The Gauss-Newton system of Eq. (1) at the node poses: A = sum J^T W J,
   b = sum J^T W r over
     * lambda_f x the Eq. (2) block of every pair (feat[96] as in bto_feature_edge, nodes
       (pairs[2p], pairs[2p+1]) = (i, j)), placed as given;
     * lambda_g x the Eq. (3) block of both directed edges of every pair (dense[32] as in
       bto_dense_edge: H, g w.r.t. T_i of edge i -> j), expanded to both nodes with
       J_j = -J_i Adj(T_i T_j^-1):  A_ii += H, A_ij += -H Adj, A_jj += Adj^T H Adj,
       b_i += g, b_j += -Adj^T g.
   poses [N][12]; A [6N][6N] row-major (symmetric), b [6N]; energies out[2] = (sum lambda_f
   E_f, sum lambda_g E_g).  Nodes outside [0, N) are an error (returns -1). */
int32_t bto_graph_system(int32_t n_nodes, const float *poses, const int32_t *pairs, int32_t P,
                         const double *feat, const double *dense_ij, const double *dense_ji,
                         const int32_t *status, double lambda_f, double lambda_g, double *A, double *b,
                         double energy[2]);
/* status [P] (may be NULL = all registered): a pair whose registration failed (1 FEW_MATCHES,
   2 FEW_INLIERS — S:290's signal) contributes no Eq. (2) term (reading R30); its Eq. (3)
   edges are kept. */

/* One Gauss-Newton step: solve A d = -b exactly (dense Cholesky, fp64) with the DOFs of
   fixed_node (I_0, kept constant) and every DOF whose diagonal is 0 (unconstrained)
   pinned to d = 0, then T_i <- exp(d_i) T_i (rounded to float).  delta [6N], new_poses
   [N][12] (may alias nothing).  Returns 0, or -1 if the free system is not positive
   definite. */
int32_t bto_graph_step(int32_t n_nodes, const float *poses, const int32_t *pairs, int32_t P,
                       const double *feat, const double *dense_ij, const double *dense_ji,
                       const int32_t *status, double lambda_f, double lambda_g, int32_t fixed_node,
                       double *delta, float *new_poses, double energy[2]);

/* ---- NEXT-4: input prep — normal map from depth (SPEC estimate_normals; the
   paper's n_i(x), method unspecified) ------------------------------------------------
   P(u, v) = ((u - cx) d / fx, (v - cy) d / fy, d) in fp64; n = (P(u+1,v) - P(u-1,v)) x
   (P(u,v+1) - P(u,v-1)), normalized, flipped to face the camera (n . P(u,v) < 0).  Invalid
   (0, 0, 0) when d(u,v) <= 0, a 4-neighbour is outside the image or has depth <= 0, a
   neighbour's |d_n - d(u,v)| > jump (compared in double on the float values), or |n| = 0.
   depth [F][H][W], normal [F][H][W][3] (float). */
void bto_estimate_normals(const float *depth, int32_t F, int32_t W, int32_t H, double fx, double fy,
                          double cx, double cy, float jump, float *normal);

/* ---- NEXT-4: keypoint lifting — the keypoints' 3-D points and normals from their pixels
   ("n keypoints x_i ... along with the feature descriptor D_i"; "pi_D^-1 ... recovers
   a 3D point in the camera's frame by looking up the depth value on the pixel location";
   n_i(x) "returns the normal of the pixel"; SPEC Keypoint invariant S:247 point =
   unproject(pixel, depth), detect_keypoints S:262 "inside the mask with valid depth").
   Reading R29: keypoint k of frame f at (u, v) (float pixel coordinates, centres at integers)
   looks up the pixel x' = (floor(u + 0.5), floor(v + 0.5)) (R14's rounding); it is KEPT iff x'
   lies in the frame, mask(x') != 0, depth(x') = d > 0 and normal(x') != 0; then
   point = ((u - cx) d / fx, (v - cy) d / fy, d) (fp64, rounded to float) and normal =
   normal(x').  Kept keypoints are compacted in their input order with their descriptors.
   uv [F][n_max][2], desc_in [F][n_max][dim], n_in [F]; maps [F][H][W] (normal [..][3]).
   Out: n_out [F], desc [F][n_max][dim], pts / nrm [F][n_max][3] (rows >= n_out untouched),
   border [F][n_max] (may be NULL): 1 iff input keypoint k's rounding is borderline (band rule
   R22: u + 0.5 or v + 0.5 within 1e-6 max(1, |.|) of an integer). */
void bto_lift_keypoints(int32_t F, int32_t n_max, int32_t dim, const float *uv, const float *desc_in,
                        const int32_t *n_in, const float *depth, const float *normal, const uint8_t *mask,
                        int32_t W, int32_t H, double fx, double fy, double cx, double cy, int32_t *n_out,
                        float *desc, float *pts, float *nrm, uint8_t *border);

/* ---- NEXT-2: the causal tracker's per-frame decisions (§IV-B/C/E) -----------------
   Poses are the 12-float (R row-major, t) layout above. */
/* rotation geodesic arccos((tr(R_a^T R_b) - 1) / 2) in fp64, argument clamped to [-1, 1] */
double bto_rot_geodesic(const float Ta[12], const float Tb[12]);
/* coarse pose: T~_t = T_{t-1} T_t^{t-1} read as T_rel . T_prev (reading R13), T_rel = the
   record's best sampled hypothesis T_best (maps frame t-1 points to frame t points); a pair
   without one (status FEW_MATCHES / FEW_INLIERS) leaves T~_t = T_prev.  fp64, rounded. */
void bto_coarse_pose(int32_t status, const float T_best[12], const float T_prev[12], float out[12]);
/* keyframe selection: start from {I_0} (pool index 0), then repeatedly add the pool
   keyframe with the smallest sum of geodesic distances against I_t (cur) and every keyframe
   selected so far (ties -> lowest pool index), until min(K, n_pool) are selected.  sel[] in
   selection order; returns the count. */
int32_t bto_select_keyframes(const float *pool, int32_t n_pool, const float cur[12], int32_t K, int32_t *sel);
/* pool augmentation: 1 iff the geodesic from cur to EVERY pool keyframe is larger than
   thresh_rad (reading R21: 10 degrees); an empty pool admits. */
int32_t bto_is_novel(const float *pool, int32_t n_pool, const float cur[12], double thresh_rad);

#ifdef __cplusplus
}
#endif
#endif
