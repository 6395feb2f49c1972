/* bt.h — C ABI of the B200-native BundleTrack pairwise-registration hot path.
 *
 * BundleTrack (Wen & Bekris, arXiv 2108.00516; PAPER.md = /root/reference/PAPER.md, "P:n" =
 * line n).  For every frame pair of the pose graph the library computes, on one sm_100a GPU:
 *   bt_match       feature matching (P:4 "feature matching and outlier pruning"):
 *                  mutual nearest neighbours of 128-d descriptors (D_i in R^128);
 *   bt_ransac      RANSAC over 3-pair samples ("Each registration sample consists of 3
 *                  pairs of keypoints"), Arun least-squares hypotheses ("generated from a
 *                  sample via least squares"), inlier gates delta = 5 mm / alpha = 45 deg,
 *                  best sampled hypothesis (T_t^{t-1}), refit on its inliers, C_ij;
 *   bt_dense_corr  dense reprojection association + point-to-plane residuals of Eq. (3)
 *                  (P:64-72), reduced to one 6x6 J^T W J block per directed edge;
 *   bt_register_pairs  all of the above for P pairs (matching, RANSAC, refit, Eq. (2)
 *                  feature-edge blocks at the node poses, both directed dense edges).
 * Readings of what the paper leaves open are listed in DESIGN.md §2 (R1..R22).
 *
 * Conventions
 *  - Every buffer pointer is a CUDA DEVICE pointer owned by the caller (except in
 *    bt_register_pairs_host / bt_register_raw_host), 16-byte aligned.  Inputs are read-only.  The library owns only
 *    the scratch reserved by bt_reserve; calls never allocate, never synchronise the host and
 *    only enqueue work on `stream` (a cudaStream_t passed as void*, NULL = legacy default
 *    stream), so they can be captured in a CUDA graph.  Outputs are valid once the stream
 *    reaches them.
 *  - Poses are object->camera, x_cam = R x_obj + t ("object pose in the camera's
 *    frame"), R row-major.  Points / normals are camera-frame metres / unit vectors.
 *  - Pixel centres sit at integer (u, v); pi(x) = (fx x/z + cx, fy y/z + cy); depth 0 =
 *    invalid; normal (0,0,0) = invalid; mask nonzero = object.
 *  - Twists are (v, w): translation first; Jacobians are w.r.t. the LEFT
 *    perturbation T <- exp(d) T (reading R18).
 *  - Errors: a call returns a bt_status; on failure nothing is enqueued and
 *    bt_last_error(ctx) describes why.  A CUDA launch error makes the context sticky-failed
 *    (every later call returns BT_ECUDA).  Per-pair outcomes are NOT errors: they are the
 *    status word of each output record ("registration-failure signal").
 *  - One context per host thread; a context is bound to the device given to bt_create.
 */
#ifndef BT_H
#define BT_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct bt_ctx bt_ctx;

typedef enum {
  BT_OK = 0,
  BT_EINVAL = 1,        /* bad argument: NULL / misaligned pointer, n_kp > n_max, ...      */
  BT_ENOMEM = 2,        /* bt_reserve could not allocate its scratch                          */
  BT_ECUDA = 3,         /* a CUDA call failed (sticky)                                        */
  BT_EUNSUPPORTED = 4,  /* device is not sm_100 (CC 10.0) or dim != 128                        */
  BT_ECAPACITY = 5      /* P, E, n_max, n_hyp, frames or map size beyond what bt_reserve got   */
} bt_status;

typedef enum {
  BT_PAIR_OK = 0,
  BT_PAIR_FEW_MATCHES = 1,       /* M < 3: no sample can be drawn                              */
  BT_PAIR_FEW_INLIERS = 2,       /* best count < min_inliers, or every hypothesis degenerate   */
  BT_PAIR_REFIT_DEGENERATE = 3   /* inliers of h* are degenerate: T_refit = T_best              */
} bt_pair_status;

typedef struct { float fx, fy, cx, cy; int32_t width, height; } bt_intrinsics;
typedef struct { float R[9]; float t[3]; } bt_pose;

/* keypoints of F frames, each padded to n_max entries */
typedef struct {
  int32_t n_frames, n_max, dim;  /* dim must be 128                                    */
  const int32_t *n_kp;           /* [F]              valid keypoints per frame, <= n_max       */
  const float *desc;             /* [F][n_max][128]  descriptors                               */
  const float *pts;              /* [F][n_max][3]    camera-frame points (metres)              */
  const float *nrm;              /* [F][n_max][3]    unit camera-frame normals                 */
} bt_keypoints;

/* dense depth / normal / mask maps of F frames */
typedef struct {
  int32_t n_frames, width, height;
  const float *depth;            /* [F][H][W]     metres, 0 = invalid                           */
  const float *normal;           /* [F][H][W][3]  unit, camera frame, (0,0,0) = invalid         */
  const uint8_t *mask;           /* [F][H][W]     nonzero = object                              */
} bt_maps;

typedef struct {
  float ratio;                   /* Lowe ratio on distances; >= 1 disables it (default 1: R2)   */
} bt_match_params;

typedef struct {
  float delta_m;                 /* inlier distance gate, 0.005                          */
  float cos_alpha;               /* cos of the normal-angle gate, cos 45 deg             */
  int32_t n_hyp;                 /* hypotheses per pair (1024 / 4096 / 16384), <= reserved      */
  uint32_t pad_;
  uint64_t seed;                 /* Philox key (lo, hi words)                                   */
  float min_sigma_ratio;         /* degeneracy: sigma2/sigma1 of the cross-covariance, 1e-3 (R8) */
  int32_t min_inliers;           /* FEW_INLIERS below this count, 3                     */
} bt_ransac_params;

typedef struct {
  float dist_gate_m;             /* dense association distance gate, 0.02 (R15)                 */
  float cos_gate;                /* dense normal-angle gate (cos), cos 45 deg (R15)             */
  float huber_m;                 /* Huber delta for E_g and E_f, 0.005 (R17)                    */
  int32_t stride;                /* use pixels with u % stride == 0 && v % stride == 0 (R20)    */
} bt_edge_params;

/* Context.  bt_create fails with BT_EUNSUPPORTED unless the device is compute capability 10.0. */
bt_status bt_create(bt_ctx **ctx, int cuda_device);
void bt_destroy(bt_ctx *ctx);
const char *bt_last_error(const bt_ctx *ctx);
const char *bt_status_string(bt_status s);

/* Reserve device scratch for calls up to these sizes (may be called again to grow).
   max_frames / width / height size the dense scratch, the pose-graph system and the staging
   of bt_register_pairs_host.  n_max <= 8192 (BT_EUNSUPPORTED beyond: a pair's point set is
   staged in shared memory); BT_EINVAL on non-positive pair / keypoint / hypothesis counts. */
bt_status bt_reserve(bt_ctx *ctx, int32_t max_pairs, int32_t n_max, int32_t max_hyp,
                     int32_t max_frames, int32_t width, int32_t height);

/* Per-pair output record, a fixed stride of bt_record_words(n_max) 4-byte words:
     [0] status  [1] n_matches M  [2] best_hyp h* (-1 none)  [3] best_count
     [4..15]  T_best  (f32: R row-major, t)   — the best SAMPLED hypothesis, a -> b
     [16..27] T_refit (f32)                   — Arun on the inliers of h* (north star)
     [28 .. 28+W)  inlier mask C_ij, W = ceil(n_max/32); bit m of word m/32 = match m
     then (bt_register_pairs only):
     dense_ij[32], dense_ji[32]  (f32, layout of bt_dense_corr's out rows)
     feat[96] (f32): H_ii(21, upper row-major) H_ij(36 row-major) H_jj(21) g_i(6) g_j(6)
                     E(1) count(1) pad(4)  — Eq. (2) at the node poses, i = pair.a, j = pair.b
   T maps frame-a points to frame-b points: p_b ~ R p_a + t. */
size_t bt_record_words(int32_t n_max);

/* Mutual nearest-neighbour matching of P frame pairs.
   pairs [P][2] (a, b) frame ids.  Out: matches [P][n_max][2] (i in a, j in b) ascending in
   i, n_matches [P].  Squared Euclidean distance; ties -> lowest index (R1-R4). */
bt_status bt_match(bt_ctx *ctx, const bt_keypoints *kp, const int32_t *pairs, int32_t P,
                   const bt_match_params *prm, int32_t *matches, int32_t *n_matches, void *stream);

/* RANSAC + refit of P pairs given their matches (as produced by bt_match).
   pair_uid [P]: the Philox counter word of each pair (a GLOBAL id: results do not depend on
   how pairs are batched or sharded).  Hypothesis h of pair p draws Philox4x32-10 with
   counter (h, uid, 0, 0), key (seed lo, seed hi) -> distinct triple (R6).
   Out: records [P][bt_record_words] words 0 .. 28+W; hyp_counts [P][n_hyp] (may be NULL):
   inlier count of each hypothesis, -1 if degenerate. */
bt_status bt_ransac(bt_ctx *ctx, const bt_keypoints *kp, const int32_t *pairs,
                    const uint32_t *pair_uid, int32_t P, const int32_t *matches,
                    const int32_t *n_matches, const bt_ransac_params *prm, uint32_t *records,
                    int32_t *hyp_counts, void *stream);

/* Eq. (3) dense edges.  edges [E][2] directed (i -> j) frame ids; node_pose [F] (device).
   Out: out [E][32] f32: H (21, upper row-major of sum w J^T J) g (6, sum w J^T r)
   E (sum rho(r)) count (associated pixels) pad(3); J = [n_i^T, (q x n_i)^T] w.r.t. the
   left perturbation of T_i (the caller expands the T_j blocks with Adj(T_i T_j^-1)). */
bt_status bt_dense_corr(bt_ctx *ctx, const bt_maps *maps, const bt_intrinsics *K,
                        const bt_pose *node_pose, const int32_t *edges, int32_t E,
                        const bt_edge_params *prm, float *out, void *stream);

/* Debug / verification entry of Eq. (3) ("dense pixel-wise correspondences are
   associated by point re-projection, while outliers are filtered based on the distance ...
   and the angle"): bt_dense_corr plus the per-pixel DECISION it took.  Same arguments and the
   same `out` (bitwise equal to bt_dense_corr's); in addition assoc [E][H][W] int32 (device,
   caller-owned, written in full): for each source pixel x of I_i, the target pixel index
   y'*W + x' it was associated with (projection in the frame, valid target, both gates passed),
   else -1 (not a source pixel: outside the mask / invalid / off-stride; or rejected).  A
   separate kernel instantiation: bt_dense_corr and bt_register_pairs never write it.  Errors
   as bt_dense_corr; BT_EINVAL if assoc is NULL. */
bt_status bt_dense_assoc(bt_ctx *ctx, const bt_maps *maps, const bt_intrinsics *K,
                         const bt_pose *node_pose, const int32_t *edges, int32_t E,
                         const bt_edge_params *prm, float *out, int32_t *assoc, void *stream);

/* The whole per-pair hot path for P pairs: bt_match -> bt_ransac -> Eq. (2) blocks at the
   node poses -> both directed Eq. (3) edges.  eprm may be NULL: dense + feature words are
   then left untouched (the first stage of a frame step). */
bt_status bt_register_pairs(bt_ctx *ctx, const bt_keypoints *kp, const bt_maps *maps,
                            const bt_intrinsics *K, const bt_pose *node_pose, const int32_t *pairs,
                            const uint32_t *pair_uid, int32_t P, const bt_match_params *mprm,
                            const bt_ransac_params *rprm, const bt_edge_params *eprm,
                            uint32_t *records, void *stream);

/* Same as bt_register_pairs but every pointer (including those inside kp and maps) is a
   HOST pointer (pinned memory gives full PCIe/C2C speed).  Copies the inputs into the
   context's staging, runs the path, copies the records back and synchronises `stream`
   before returning.  Needs bt_reserve(max_frames, width, height). */
bt_status bt_register_pairs_host(bt_ctx *ctx, const bt_keypoints *kp, const bt_maps *maps,
                                 const bt_intrinsics *K, const bt_pose *node_pose,
                                 const int32_t *pairs, const uint32_t *pair_uid, int32_t P,
                                 const bt_match_params *mprm, const bt_ransac_params *rprm,
                                 const bt_edge_params *eprm, uint32_t *records, void *stream);

/* NEXT-4 end to end: the whole path from the RAW per-frame inputs in HOST memory
   — depth, mask and the keypoint detector's output (2-D pixels + descriptors) — "only the RGB-D
   frames and the segmentation masks" plus the keypoints of P:25; the normal map n_i(x) of Eq. (3)
    and the keypoints' 3-D points / normals (pi_D^-1) are derived on the device.
   Equivalent to: bt_estimate_normals(depth, jump_m) -> bt_lift_keypoints(uv, desc, n_in, maps)
   -> bt_register_pairs on those outputs (bitwise the same records), with the host -> device
   copies of the inputs, and the device -> host copy of the records, inside the call; it
   synchronises `stream` before returning.  Needs bt_reserve(max_frames, width, height); the
   first raw call allocates two staging slots at that capacity (the raw inputs of two calls),
   which consecutive calls use in turn.  The copies run on the context's copy stream once the
   call that used the slot before is done with it.
   Layouts: depth [F][H][W] f32, mask [F][H][W] u8, uv [F][n_max][2] f32, desc [F][n_max][dim]
   f32, n_in [F] (detector counts); node_pose [F], pairs [P][2], pair_uid [P], records
   [P][bt_record_words(n_max)].  eprm may be NULL (no dense edges).  Errors: as bt_register_pairs
   plus BT_EUNSUPPORTED (dim != 128), BT_ECAPACITY (beyond the reserved staging), BT_EINVAL
   (NULL buffers, jump_m < 0, non-positive sizes). */
typedef struct {
  int32_t n_frames, width, height;
  int32_t n_max, dim;            /* keypoint rows per frame; descriptor length (128)              */
  float jump_m;                  /* normal estimation: neighbour depth-jump limit (SPEC: 0.05)    */
  const float *depth;            /* [F][H][W]  metres, <= 0 invalid                               */
  const uint8_t *mask;           /* [F][H][W]  nonzero = object                                    */
  const float *uv;               /* [F][n_max][2] keypoint pixel coordinates                      */
  const float *desc;             /* [F][n_max][dim] descriptors                                    */
  const int32_t *n_in;           /* [F] detected keypoints per frame                               */
  /* optional: depth as the sensor / the paper's datasets store it, [F][H][W] uint16 (0 invalid),
     metres = (float)value * depth_scale rounded to fp32 on the device (e.g. 0.001 for mm) — half
     the bytes of `depth` over PCIe.  Exactly one of depth / depth_u16 is non-NULL; the records
     equal those of `depth` holding the same fp32 values.                                         */
  const uint16_t *depth_u16;
  float depth_scale;             /* > 0 with depth_u16                                             */
  /* optional: the mask as packed bits, [F][H][ceil(W / 8)] bytes, pixel (u, v) = bit (u & 7)
     (LSB first) of byte (u >> 3) of row v — an eighth of the bytes of `mask` over PCIe, unpacked
     on the device.  Exactly one of mask / mask_bits is non-NULL.                                 */
  const uint8_t *mask_bits;
} bt_raw_frames;
bt_status bt_register_raw_host(bt_ctx *ctx, const bt_raw_frames *raw, const bt_intrinsics *K,
                               const bt_pose *node_pose, const int32_t *pairs, const uint32_t *pair_uid,
                               int32_t P, const bt_match_params *mprm, const bt_ransac_params *rprm,
                               const bt_edge_params *eprm, uint32_t *records, void *stream);
/* The same call without the final synchronisation — the streaming form for consecutive frame
   batches: the host -> device copies of call t + 1 (other slot) overlap the kernels of call t.
   On return the work is enqueued; `records` (pinned host memory) holds the result once `stream`
   has reached the call's end (cudaStreamSynchronize / an event recorded after the call).  The
   host input buffers must stay unchanged until then, and two calls in flight must not share a
   `records` buffer the caller still reads.  Errors found at enqueue time as above; a failure
   inside the kernels surfaces as BT_ECUDA on a later call. */
bt_status bt_register_raw_host_async(bt_ctx *ctx, const bt_raw_frames *raw, const bt_intrinsics *K,
                                     const bt_pose *node_pose, const int32_t *pairs, const uint32_t *pair_uid,
                                     int32_t P, const bt_match_params *mprm, const bt_ransac_params *rprm,
                                     const bt_edge_params *eprm, uint32_t *records, void *stream);

/* NEXT-3: fused record exchange.  The per-pair records are what every rank's
   pose-graph solve needs (the pair correspondences built "in parallel on GPU", §IV-D);
   instead of a separate all-gather, after this call every bt_register_pairs (device entry) on
   this context ALSO stores each word of local pair p's record into row (row_offset + p) of
   every peer buffer peers[k], k < n_peers: device addresses valid in this process (another
   rank's gather buffer mapped through CUDA IPC / symmetric memory, or a local buffer), each
   holding `rows` records of bt_record_words(n_max) words (the call's n_max).  The stores are
   issued by the kernels that produce the words (RANSAC finish: header, mask, Eq. (2) blocks;
   dense reduce: Eq. (3) blocks), so the exchange rides on them; the caller orders them before
   any reader on another device with a barrier after the call (e.g. the symmetric-memory
   barrier).  The local `records` output is written as before.  n_peers = 0 turns it off.
   Ownership: the peer buffers stay the caller's; the context keeps the addresses only.
   Errors: BT_EINVAL (n_peers outside [0, 8], peers NULL or holding a 0 address, row_offset < 0,
   rows < 1); bt_register_pairs then fails with BT_ECAPACITY when row_offset + P > rows. */
bt_status bt_set_record_peers(bt_ctx *ctx, int32_t n_peers, const uint64_t *peers, int32_t row_offset,
                              int32_t rows);

/* out[n] = a[n] * b[n] (device bt_pose arrays): the coarse pose T~_t = T_rel T_{t-1} of
   P:25 under object->camera poses (reading R13), without a host round trip. */
bt_status bt_compose_poses(bt_ctx *ctx, const bt_pose *a, const bt_pose *b, bt_pose *out,
                           int32_t n, void *stream);

/* ---- NEXT-1: pose-graph Gauss-Newton step (§IV-D) ---------------------
   Eq. (1): E = sum_{i != j} lambda_1 E_f(i,j) + lambda_2 E_g(i,j).  One Gauss-Newton step
   (J^T W J) d = -J^T W r (the IRLS weights W already in the blocks), solved with
   Jacobi-preconditioned CG ("the diagonal matrix J^T W J is used as the preconditioner"),
   then xi <- xi [+] d as the left update T_i <- exp(d_i) T_i (twists (v, w), reading R18). */
typedef struct {
  float lambda_feat;     /* lambda_1 (1) */
  float lambda_dense;    /* lambda_2 (1) */
  int32_t fixed_node;    /* node kept constant as the reference (I_0) */
  int32_t max_iter;      /* PCG iteration cap (>= 1) */
  float rel_tol;         /* PCG stops when |r| <= rel_tol |b| (e.g. 1e-10) */
  int32_t precond;       /* 0: the diagonal of J^T W J (Jacobi, P:83 as written);
                            1: its 6 x 6 node blocks (block-Jacobi, reading R23) */
} bt_graph_params;

/* One Gauss-Newton step of the pose graph from the blocks bt_register_pairs wrote at the
   node poses `node_pose` (device [n_nodes]):
     records  device [P][bt_record_words(n_max)] — per pair (pairs[p] = (i, j)): the Eq. (2)
              block `feat` over (T_i, T_j) used as given, and the Eq. (3) blocks dense_ij
              (edge i -> j, w.r.t. T_i) / dense_ji, each expanded to both nodes with
              J_j = -J_i Adj(T_i T_j^-1) (Adj = [[R, [t]x R], [0, R]]).
   The system is assembled in fp64 in a fixed order (bitwise reproducible).  DOFs of
   fixed_node and DOFs whose diagonal is 0 (nodes without edges) are held at d = 0.
   Outputs (device): new_pose [n_nodes] (may alias node_pose), delta [n_nodes][6] fp64 or
   NULL, stats [4] f32 or NULL = (lambda_1 sum E_f, lambda_2 sum E_g at the input poses, PCG
   iterations, final |r| / |b|).  Pair entries with i == j or a node outside [0, n_nodes) are
   skipped.  Errors: BT_EINVAL (NULL buffers, n_nodes < 1, fixed_node out of range, bad
   params), BT_ECAPACITY (n_nodes > reserved max_frames, P > reserved max_pairs). */
bt_status bt_pose_graph_step(bt_ctx *ctx, int32_t n_nodes, const bt_pose *node_pose,
                             const int32_t *pairs, int32_t P, const uint32_t *records, int32_t n_max,
                             const bt_graph_params *prm, bt_pose *new_pose, double *delta,
                             float *stats, void *stream);

/* Re-linearize the records' Eq. (2) and Eq. (3) blocks at new node poses for the next
   Gauss-Newton iteration (NEXT-1), reusing each pair's C_ij: "If C_ij has been built during a
   previous pose graph optimization, it is reused".  Feature blocks are recomputed from
   the record's inlier mask over the match lists the context kept from the LAST
   bt_register_pairs (device entry) on this context — the same P pairs and keypoints must be
   passed; the dense edges are re-associated at the new poses.  Matching, RANSAC and
   the other record words are untouched; the updated words are bitwise equal to what
   bt_register_pairs would write at these poses.  Errors: BT_EINVAL (NULL buffers / params, P
   different from the last bt_register_pairs), else as bt_register_pairs. */
bt_status bt_relinearize(bt_ctx *ctx, const bt_keypoints *kp, const bt_maps *maps, const bt_intrinsics *K,
                         const bt_pose *node_pose, const int32_t *pairs, int32_t P, const bt_edge_params *eprm,
                         uint32_t *records, void *stream);

/* The C_ij cache across calls ("If C_ij has been built during a previous pose graph
   optimization, it is reused"): a tracker keeps every pair's match list next to its record so
   that pairs registered in DIFFERENT bt_register_pairs calls (e.g. each frame's new pairs
   against the keyframes) can be re-linearized together.
   bt_copy_matches copies the match lists of the LAST bt_register_pairs (device entry) on this
   context to caller-owned device buffers: matches [P][n_max][2] i32 (row m of pair p = the
   m-th mutual match (i, j), ascending i; the record's inlier mask bit m refers to it; rows past
   n_matches[p] undefined), n_matches [P] i32.  Errors: BT_EINVAL (NULL buffers, P or n_max
   different from that call's).
   bt_relinearize_matches is bt_relinearize with the match lists given explicitly (device,
   layout as above, P pairs, kp->n_max rows each) instead of the context's; the updated words
   are bitwise equal to what bt_register_pairs writes at these poses.  Errors: BT_EINVAL (NULL
   buffers / params), BT_ECAPACITY (P > reserved max_pairs), else as bt_register_pairs. */
bt_status bt_copy_matches(bt_ctx *ctx, int32_t P, int32_t n_max, int32_t *matches, int32_t *n_matches,
                          void *stream);
bt_status bt_relinearize_matches(bt_ctx *ctx, const bt_keypoints *kp, const bt_maps *maps,
                                 const bt_intrinsics *K, const bt_pose *node_pose, const int32_t *pairs,
                                 int32_t P, const int32_t *matches, const int32_t *n_matches,
                                 const bt_edge_params *eprm, uint32_t *records, void *stream);

/* ---- NEXT-4: input prep — the normal map n_i(x) of Eq. (3) from depth (SPEC
   estimate_normals S:157-165) -----------------------------------------------------------
   depth [F][H][W] f32 device (<= 0: invalid) -> normal [F][H][W][3] f32 device (16-B
   aligned): central differences of the unprojected cloud P = ((u-cx) d/fx, (v-cy) d/fy, d),
   n = (P(u+1,v) - P(u-1,v)) x (P(u,v+1) - P(u,v-1)) normalized and facing the camera
   (n . P < 0); (0, 0, 0) at the image border, where the pixel or a 4-neighbour has depth
   <= 0, or where a neighbour's depth differs by more than jump_m (SPEC: 0.05).  Only K's
   fx, fy, cx, cy are used.  Errors: BT_EINVAL (NULL / misaligned buffers, fx or fy <= 0,
   jump_m < 0, negative sizes). */
bt_status bt_estimate_normals(bt_ctx *ctx, const float *depth, int32_t n_frames, int32_t width, int32_t height,
                              const bt_intrinsics *K, float jump_m, float *normal, void *stream);

/* ---- NEXT-4: input prep — keypoint lifting ("n keypoints x_i ... along with the feature
   descriptor D_i"; "pi_D^-1 ... recovers a 3D point in the camera's frame by looking up
   the depth value on the pixel location", n_i(x) "returns the normal of the pixel"
   point = unproject(pixel, depth), S:262 keypoints "inside the mask with valid depth") --------
   uv [F][n_max][2] f32 (pixel coordinates, centres at integers), desc_in [F][n_max][dim] f32,
   n_in [F]: the detector's raw output; maps: depth / normal (e.g. bt_estimate_normals) / mask
   of the same frames.  Keypoint k of frame f looks up x' = (floor(u + 0.5), floor(v + 0.5))
   (reading R29); it is kept iff x' is in the frame, mask(x') != 0, depth(x') = d > 0 and
   normal(x') != 0, with point ((u - cx) d / fx, (v - cy) d / fy, d) (fp64, rounded) and
   normal(x').  Out (device, caller-owned, NOT aliasing the inputs): n_kp [F], desc
   [F][n_max][dim], pts / nrm [F][n_max][3] — the kept keypoints compacted in input order (rows
   >= n_kp[f] are not written): exactly the bt_keypoints of the registration calls.
   Errors: BT_EUNSUPPORTED if dim != 128; BT_EINVAL for NULL / misaligned (16 B: uv, desc)
   buffers, maps that do not cover n_frames or mismatch K, n_max < 1. */
bt_status bt_lift_keypoints(bt_ctx *ctx, int32_t n_frames, int32_t n_max, int32_t dim, const float *uv,
                            const float *desc_in, const int32_t *n_in, const bt_maps *maps,
                            const bt_intrinsics *K, int32_t *n_kp, float *desc, float *pts, float *nrm,
                            void *stream);

/* ---- NEXT-2: the causal tracker's per-frame decisions, on the device (§IV-B/C/E) -----
   geo(a, b) = arccos((tr(R_a^T R_b) - 1) / 2), the rotation geodesic of P:33, in fp64.
   Pose arrays are device bt_pose; every call only enqueues (graph-capturable). */
/* Coarse pose of the current frame ("T~_t = T_{t-1} T_t^{t-1} where T_t^{t-1} is the best
   sampled correspondence hypothesis"; reading R13: out = T_rel . prev with T_rel = record's
   T_best, the (t-1 -> t) pair's record from bt_ransac / bt_register_pairs).  A record whose
   status is FEW_MATCHES / FEW_INLIERS (no hypothesis) gives out = prev.  `record`: one record
   (words 0..15 read); out may alias prev. */
bt_status bt_coarse_pose(bt_ctx *ctx, const uint32_t *record, const bt_pose *prev, bt_pose *out, void *stream);
/* Keyframe selection: from the pool poses pool[0 .. *n_pool) (pool[0] = I_0), the
   greedy minimum-H-subgraph heuristic — start with {I_0}; each round add the keyframe with the
   smallest sum of geodesics to cur (I_t) and to every keyframe selected so far (ties -> lowest
   index) — until min(K, *n_pool) are selected.  Out: sel [K] pool indices in selection order,
   *n_sel.  n_pool is a DEVICE int (bt_pool_admit grows it).  BT_EINVAL: pool_cap outside
   [1, 4096], K < 1, NULL buffers. */
bt_status bt_select_keyframes(bt_ctx *ctx, const bt_pose *pool, const int32_t *n_pool, int32_t pool_cap,
                              const bt_pose *cur, int32_t K, int32_t *sel, int32_t *n_sel, void *stream);
/* Memory-pool augmentation: if geo(cur, pool[k]) > thresh_rad for every k < *n_pool
   (reading R21: 10 degrees) and *n_pool < pool_cap, pool[*n_pool] = cur and ++*n_pool.
   *admitted (may be NULL) = the new pool index, or -1.  Device n_pool / admitted. */
bt_status bt_pool_admit(bt_ctx *ctx, bt_pose *pool, int32_t *n_pool, int32_t pool_cap, const bt_pose *cur,
                        float thresh_rad, int32_t *admitted, void *stream);

/* number of kernels the last bt_* call enqueued (for the bench's gpu_launches claim) */
int32_t bt_last_launch_count(const bt_ctx *ctx);

/* Per-kernel timing for roofline accounting.  When enabled, every kernel launch is bracketed
   by a pair of CUDA events recorded on the launching stream.  bt_profile_read waits for the
   recorded events, and returns (and resets) the accumulated time in ms and the launch count
   of kernel `kernel_id` (0 .. bt_profile_kernels()-1) since the previous read.  on: 0 off,
   1 every kernel, 2 + kernel_id only that kernel's launches (the others run unbracketed, so the
   overlap of the streams is perturbed less); BT_EINVAL outside [0, 2 + bt_profile_kernels()). */
bt_status bt_profile_enable(bt_ctx *ctx, int32_t on);
int32_t bt_profile_kernels(void);
const char *bt_profile_name(int32_t kernel_id);
bt_status bt_profile_read(bt_ctx *ctx, int32_t kernel_id, double *total_ms, int64_t *launches);

#ifdef __cplusplus
}
#endif
#endif /* BT_H */
