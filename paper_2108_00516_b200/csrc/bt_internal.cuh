// bt_internal.cuh — internal launch interfaces and device helpers of libbt (sm_100a).
// Not part of the ABI (include/bt.h is).  Nothing here is shared with oracle/.
#pragma once
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <utility>
#include <stdint.h>

#include "bt.h"

namespace bt {

constexpr int kDim = 128;               // descriptor length, D_i in R^128

// ---- record layout (see bt.h) -------------------------------------------------------
constexpr int kRecStatus = 0, kRecNMatch = 1, kRecBestHyp = 2, kRecBestCount = 3;
constexpr int kRecTBest = 4, kRecTRefit = 16, kRecMask = 28;
__host__ __device__ inline int mask_words(int n_max) { return (n_max + 31) / 32; }
__host__ __device__ inline int rec_dense_ij(int n_max) { return kRecMask + mask_words(n_max); }
__host__ __device__ inline int rec_dense_ji(int n_max) { return rec_dense_ij(n_max) + 32; }
__host__ __device__ inline int rec_feat(int n_max) { return rec_dense_ij(n_max) + 64; }
__host__ __device__ inline int rec_words(int n_max) { return rec_dense_ij(n_max) + 64 + 96; }

// ---- NEXT-3: fused record exchange (bt_set_record_peers) ----------------------------------
// The kernels that produce a record's words also store each word into row (row_off + p) of
// every peer's gather buffer (another rank's buffer mapped into this process through CUDA IPC /
// symmetric memory, or a local one): the all-gather of the records rides on the producers'
// own stores, no separate collective kernel.
constexpr int kMaxPeers = 8;
struct PeerRec {
  uint32_t *ptr[kMaxPeers];
  int n = 0, row_off = 0, stride = 0;
};
__device__ __forceinline__ void peer_put(const PeerRec &pr, int p, int w, uint32_t v) {
  for (int k = 0; k < pr.n; ++k) pr.ptr[k][(size_t)(pr.row_off + p) * pr.stride + w] = v;
}

// ---- device views of the ABI structs ---------------------------------------------------
struct KpView {
  int n_frames, n_max;
  const int32_t *n_kp;
  const float *desc, *pts, *nrm;
};
struct MapView {
  int n_frames, W, H;
  const float *depth, *normal;
  const uint8_t *mask;
};

// ---- launch bookkeeping: counts kernels and (optionally) brackets each with events ----
enum KernelId {
  K_DESC_PREP = 0, K_MATCH_TC, K_RESOLVE, K_MUTUAL, K_RANSAC_HYP, K_RANSAC_SCORE, K_RANSAC_FINISH, K_DENSE_PREP,
  K_DENSE, K_DENSE_REDUCE, K_COMPOSE, K_GRAPH, K_NORMALS, K_TRACK,
  K_COUNT
};

// matching scratch (carved from one allocation; see match_scratch_bytes)
struct MatchScratch {
  __half *desc16;          // [F][n_pad][128] unit descriptors (TMA source)
  __half *desc16lo;        // [F][n_pad][128] their fp16 remainders (a / M_f - hi): level-2 certification
  float *norm;             // [F][n_pad]
  unsigned *maxnorm;       // [F] float bits of max |a|
  uint4 *work;             // [2 queues][work_cap] undecided rows: (dir | i << 1, p, k1, k2);
                           // queue 0: top-2 rescoring, queue 1: full exact scan
  size_t work_cap;
  unsigned *work_count;    // [2]
  int32_t *nn_ab, *nn_ba;  // [P][n_max]
  uint8_t *ratio_ok;       // [P][n_max]
  int32_t *fs_rows;        // [2 dirs][P][n_pad / 128 tiles][128] undecided rows for the batched full scan
  int32_t *fs_count;       // [2][P][tiles]
  int32_t *l3_rows;        // [2][P][n_pad] rows left uncertified by the level-2 pass (k_fullscan's input)
  int32_t *l3_count;       // [2][P] (0 between calls: k_mutual resets it)
};
struct Launch {
  int count = 0;
  void (*hook)(void *user, int kernel_id, int phase, cudaStream_t s) = nullptr;
  void *user = nullptr;
  void begin(int k, cudaStream_t s) { if (hook) hook(user, k, 0, s); }
  void end(int k, cudaStream_t s) { ++count; if (hook) hook(user, k, 1, s); }
};

// ---- programmatic dependent launch (PDL) -----------------------------------------------
// Chain kernels are launched with programmatic stream serialization and call pdl_wait() before
// any memory access (griddepcontrol.wait returns once the predecessor grid has completed and
// its memory is visible): the dependent's launch overlaps the predecessor's completion
// (measured 0.385 -> 0.381 ms per step).  No early griddepcontrol.launch_dependents in general:
// CTAs launched early park on SM resources the low-priority dense stream needs (measured 0.459 ms
// with every kernel triggering).  One exception: k_desc_half triggers k_match_ws, which sets up
// TMEM and its barriers before its own wait (0.2868 -> 0.2834 ms); the same for k_corr_feat ->
// k_score_tc measured slower (0.2834 -> 0.287 ms).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       Args &&...args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
  static const bool dbg = getenv("BT_LAUNCH_DEBUG") != nullptr;   // dev aid: report the failing launch
  if (dbg && e != cudaSuccess)
    fprintf(stderr, "bt launch failed: grid %u x %u, block %u, smem %zu: %s\n", grid.x, grid.y, block.x, smem,
            cudaGetErrorString(e));
}

// ---- per-device launch setup (thread-safe, bt_api.cu) ---------------------------------
// cudaFuncSetAttribute applies to the CURRENT device only, so the dynamic shared-memory opt-in
// and the occupancy-derived grid sizes are cached per (device, kernel) behind a mutex: a second
// context on another GPU of the same process (or another host thread) sets its own.
void smem_optin(const void *kernel, size_t bytes);               // raise the kernel's opt-in if needed
int sm_count();                                                  // SMs of the current device
int resident_grid(const void *kernel, int threads, size_t smem); // SMs x max resident CTAs per SM (>= 1 per SM)

// ---- launchers (stream-ordered, no sync) -------------------------------------------
// matching
int match_n_pad(int n_max);
size_t match_scratch_bytes(int max_frames, int max_pairs, int n_max);
MatchScratch carve_match_scratch(void *p, int max_frames, int max_pairs, int n_max);
void launch_match(const KpView &kp, const int32_t *pairs, int P, float ratio, const MatchScratch &S,
                  const CUtensorMap *tmap, int force_fallback, int32_t *matches, int32_t *n_matches,
                  cudaStream_t s, Launch &L);
// RANSAC hypotheses + balanced scoring + finish (+ optional Eq. (2) blocks at node poses).
// Carved at capacity offsets: hypothesis buffer then per-hypothesis counts.
struct RansacScratch {
  void *hyp;
  int32_t *counts;
  int32_t *work;               // the scoring kernel's slice counter
  void *feat;                  // [P][m_pad][64] fp16 correspondence features (tensor-core scoring)
  void *pfeat;                 // [P] per-pair centroids / scales / feature maxima
  void *fix;                   // [P * H] (p, h) rows recounted whole (undecided-list overflow)
  void *elist;                 // [P * H] (p, h, m) undecided tests, evaluated by k_score_fix
  int ecap;
  uint32_t *ofl;               // [P][ceil(H / 32)] rows recounted whole (bitmap)
  int32_t *fix_count;          // [2]: undecided tests, overflowed rows
  int m_pad;
  const CUtensorMap *fmap;     // TMA view of feat: [P * m_pad][64] fp16, 64 x 128 boxes, 128B swizzle
};
size_t ransac_scratch_bytes(int max_pairs, int max_hyp, int n_max);
RansacScratch carve_ransac_scratch(void *scratch, int max_pairs, int max_hyp, int n_max);
int score_m_pad(int n_max);
int score_chunk();                 // rows of a scoring feature chunk (TMA box)
void launch_ransac(const KpView &kp, const int32_t *pairs, const uint32_t *uid, int P,
                   const int32_t *matches, const int32_t *n_matches, const bt_ransac_params &prm,
                   const RansacScratch &rs, uint32_t *records, int rec_stride,
                   int32_t *hyp_counts, const bt_pose *node_pose, float huber, cudaStream_t s,
                   Launch &L, const PeerRec *peers = nullptr);
// dense Eq. (3): edges either explicit (edges != null) or derived from pairs (2 per pair)
void launch_dense(const MapView &mp, const bt_intrinsics &K, const bt_pose *node_pose, const int32_t *edges,
                  const int32_t *pairs, int E, const bt_edge_params &prm, void *scratch, size_t map_cap,
                  float *out, int out_stride, uint32_t *records, int rec_stride, int rec_off_ij, int rec_off_ji,
                  cudaStream_t s, Launch &L, int32_t *assoc = nullptr, const PeerRec *peers = nullptr);
int dense_tiles(int W, int H);
size_t dense_scratch_bytes(int max_frames, int max_edges, int W, int H);
// Eq. (2) blocks re-linearized at new node poses from the records' inlier masks (C_ij reuse)
void launch_feature_edges(const KpView &kp, const int32_t *pairs, int P, const int32_t *matches,
                          const int32_t *n_matches, uint32_t *records, int rec_stride, const bt_pose *node_pose,
                          float huber, cudaStream_t s, Launch &L);
// NEXT-4 input prep: normal map from depth (bt_prep.cu)
void launch_depth_u16(const uint16_t *in, float scale, size_t n, float *out, cudaStream_t s, Launch &L);
void launch_mask_bits(const uint8_t *bits, int F, int W, int H, uint8_t *mask, cudaStream_t s, Launch &L);
void launch_normals(const float *depth, int F, int W, int H, const bt_intrinsics &K, float jump, float *normal,
                    cudaStream_t s, Launch &L);
// NEXT-4 keypoint lifting (bt_prep.cu)
void launch_lift(int F, int n_max, const float *uv, const float *desc_in, const int32_t *n_in, const MapView &mp,
                 const bt_intrinsics &K, int32_t *n_out, float *desc, float *pts, float *nrm, cudaStream_t s,
                 Launch &L);
// NEXT-2 tracker decisions (bt_track.cu)
void launch_coarse_pose(const uint32_t *record, const bt_pose *prev, bt_pose *out, cudaStream_t s, Launch &L);
void launch_select(const bt_pose *pool, const int32_t *n_pool, int cap, const bt_pose *cur, int K, int32_t *sel,
                   int32_t *n_sel, cudaStream_t s, Launch &L);
void launch_admit(bt_pose *pool, int32_t *n_pool, int cap, const bt_pose *cur, double thresh, int32_t *admitted,
                  cudaStream_t s, Launch &L);
// NEXT-1 pose-graph Gauss-Newton step (bt_graph.cu)
size_t graph_scratch_bytes(int max_nodes, int max_pairs);
void launch_graph(int N, const bt_pose *pose, const int32_t *pairs, int P, const uint32_t *records, int n_max,
                  const bt_graph_params &prm, void *scratch, bt_pose *new_pose, double *delta, float *stats,
                  cudaStream_t s, Launch &L);
void launch_compose(const bt_pose *a, const bt_pose *b, bt_pose *out, int n, cudaStream_t s,
                    Launch &L);

}  // namespace bt
