// bt_api.cu — the C ABI of include/bt.h: context, scratch reservation, argument validation and
// stream-ordered orchestration of the kernels in bt_match.cu / bt_ransac.cu / bt_dense.cu.
#include <cuda_runtime.h>

#include <cudaTypedefs.h>

#include <cstdarg>
#include <cstdlib>
#include <utility>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <new>
#include <tuple>
#include <vector>

#include "bt_internal.cuh"

struct bt_ctx {
  int device = 0;
  bool sticky = false;
  char err[512] = {0};
  bt::Launch launch;                          // kernels enqueued by the current / last call
  cudaStream_t side = nullptr;                // dense Eq.(3) path runs here, overlapping match + RANSAC
  cudaStream_t hi = nullptr;                  // match -> RANSAC chain (the longer one), high priority
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_join_hi = nullptr;
  // per-kernel event timing (bt_profile_*)
  struct Pending { int kid; cudaEvent_t start, stop; };
  bool prof_on = false;
  int prof_only = -1;                         // >= 0: bracket only this kernel bucket's launches
  std::vector<cudaEvent_t> ev_pool;
  std::vector<Pending> pending;
  double prof_ms[bt::K_COUNT] = {0};
  int64_t prof_n[bt::K_COUNT] = {0};
  // capacity
  int cap_pairs = 0, cap_nmax = 0, cap_hyp = 0, cap_frames = 0, cap_w = 0, cap_h = 0, cap_stage = 0;
  size_t cap_dense = 0;                       // bytes of dense scratch
  size_t dense_map_cap = 0;                   // dense map entries reserved (frames x pixels)
  // scratch
  void *match = nullptr;                      // matching scratch (bt::MatchScratch)
  bt::MatchScratch ms{};
  CUtensorMap tmap_desc;                      // TMA view of ms.desc16: [frames * n_pad][128] fp16
  CUtensorMap tmap_feat;                      // TMA view of rs.feat: [pairs * m_pad][64] fp16
  int force_fallback = 0;                     // BT_FORCE_FALLBACK: exact rescoring of every row
  int32_t *matches = nullptr, *n_matches = nullptr;
  void *rscratch = nullptr;                   // RANSAC hypotheses / counts (bt::RansacScratch)
  bt::RansacScratch rs{};
  void *dense = nullptr;
  void *graph = nullptr;                      // pose-graph step scratch (bt_graph.cu)
  int cached_P = -1;                          // pairs whose match lists c->matches holds (C_ij cache)
  int cached_nmax = -1;                       // ... and their row stride
  bt::PeerRec peers;                          // NEXT-3: fused record exchange (bt_set_record_peers)
  int peer_rows = 0;                          // rows each peer buffer holds
  // staging for bt_register_pairs_host
  int32_t *st_nkp = nullptr, *st_pairs = nullptr;
  uint32_t *st_uid = nullptr, *st_records = nullptr;
  float *st_desc = nullptr, *st_pts = nullptr, *st_nrm = nullptr, *st_depth = nullptr, *st_normal = nullptr;
  uint8_t *st_mask = nullptr;
  bt_pose *st_pose = nullptr;
  cudaEvent_t ev_maps = nullptr;                              // raw entry: maps + normals staged
  // bt_register_raw_host(_async) staging: two slots (allocated on the first raw call), used in
  // turn, so the copies of call t + 1 (on the copy stream) overlap the kernels of call t; a
  // slot's copies wait for ev_free, recorded once the call that used it last is done with it
  struct RawSlot {
    float *depth = nullptr, *normal = nullptr, *uv = nullptr, *desc_in = nullptr;
    uint16_t *depth_u16 = nullptr;
    uint8_t *mask = nullptr, *mask_bits = nullptr;
    int32_t *nin = nullptr, *pairs = nullptr;
    uint32_t *uid = nullptr;
    bt_pose *pose = nullptr;
    cudaEvent_t ev_in = nullptr, ev_free = nullptr;
  };
  RawSlot raw[2];
  int raw_next = 0;
  cudaStream_t h2d = nullptr;                                 // host -> device copies of the raw entry
};

namespace bt {
namespace {
std::mutex g_setup_mu;
std::map<std::pair<int, const void *>, size_t> g_smem;           // (device, kernel) -> opted-in bytes
std::map<int, int> g_sms;                                        // device -> SM count
std::map<std::tuple<int, const void *, int, size_t>, int> g_grid;
int current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev;
}
}  // namespace

void smem_optin(const void *kernel, size_t bytes) {
  // opt in when static + dynamic shared memory exceed the 48 KB default (not only the dynamic
  // part); the kernel's static size is looked up once
  const int dev = current_device();
  std::lock_guard<std::mutex> g(g_setup_mu);
  static std::map<std::pair<int, const void *>, size_t> statics;
  auto st = statics.find({dev, kernel});
  if (st == statics.end()) {
    cudaFuncAttributes fa;
    size_t v = 0;
    if (cudaFuncGetAttributes(&fa, kernel) == cudaSuccess) v = fa.sharedSizeBytes;
    else cudaGetLastError();
    st = statics.emplace(std::make_pair(dev, kernel), v).first;
  }
  if (st->second + bytes <= 48 * 1024) return;
  size_t &have = g_smem[{dev, kernel}];
  if (bytes > have) {
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    have = bytes;
  }
}

int sm_count() {
  const int dev = current_device();
  std::lock_guard<std::mutex> g(g_setup_mu);
  auto it = g_sms.find(dev);
  if (it != g_sms.end()) return it->second;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return g_sms[dev] = sms > 0 ? sms : 1;
}

int resident_grid(const void *kernel, int threads, size_t smem) {
  smem_optin(kernel, smem);
  const int sms = sm_count();
  const int dev = current_device();
  std::lock_guard<std::mutex> g(g_setup_mu);
  const auto key = std::make_tuple(dev, kernel, threads, smem);
  auto it = g_grid.find(key);
  if (it != g_grid.end()) return it->second;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem);
  return g_grid[key] = sms * (per_sm > 0 ? per_sm : 1);
}
}  // namespace bt

namespace {

bt_status fail(bt_ctx *c, bt_status s, const char *fmt, ...) {
  if (c) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(c->err, sizeof c->err, fmt, ap);
    va_end(ap);
    if (s == BT_ECUDA) c->sticky = true;
  }
  return s;
}

bool aligned16(const void *p) { return ((uintptr_t)p & 15u) == 0; }

template <class T>
void free_dev(T *&p) {
  if (p) cudaFree(p);
  p = nullptr;
}

void free_scratch(bt_ctx *c) {
  free_dev(c->match); free_dev(c->matches); free_dev(c->n_matches);
  free_dev(c->rscratch); free_dev(c->dense); free_dev(c->graph);
  free_dev(c->st_nkp); free_dev(c->st_pairs); free_dev(c->st_uid); free_dev(c->st_records);
  free_dev(c->st_desc); free_dev(c->st_pts); free_dev(c->st_nrm); free_dev(c->st_depth);
  free_dev(c->st_normal); free_dev(c->st_mask); free_dev(c->st_pose);
  for (auto &r : c->raw) {
    free_dev(r.depth); free_dev(r.normal); free_dev(r.uv); free_dev(r.desc_in); free_dev(r.mask);
    free_dev(r.nin); free_dev(r.pairs); free_dev(r.uid); free_dev(r.pose); free_dev(r.depth_u16);
    free_dev(r.mask_bits);
  }
}

#define BT_CHECK_CTX(c)                                                                  \
  do {                                                                                   \
    if (!(c)) return BT_EINVAL;                                                          \
    if ((c)->sticky) return BT_ECUDA;                                                    \
    if (cudaSetDevice((c)->device) != cudaSuccess)                                       \
      return fail((c), BT_ECUDA, "cudaSetDevice(%d) failed", (c)->device);               \
    (c)->launch.count = 0;                                                               \
  } while (0)

bt_status after_launch(bt_ctx *c, const char *what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(c, BT_ECUDA, "%s: %s", what, cudaGetErrorString(e));
  return BT_OK;
}

bt_status check_kp(bt_ctx *c, const bt_keypoints *kp) {
  if (!kp) return fail(c, BT_EINVAL, "keypoints: NULL");
  if (kp->dim != bt::kDim) return fail(c, BT_EUNSUPPORTED, "descriptor dim %d != 128", kp->dim);
  if (kp->n_frames < 1 || kp->n_max < 1) return fail(c, BT_EINVAL, "keypoints: n_frames/n_max < 1");
  if (kp->n_max > c->cap_nmax)
    return fail(c, BT_ECAPACITY, "n_max %d > reserved %d", kp->n_max, c->cap_nmax);
  if (kp->n_frames > c->cap_frames)
    return fail(c, BT_ECAPACITY, "keypoint frames %d > reserved %d", kp->n_frames, c->cap_frames);
  if (!kp->n_kp || !kp->desc || !kp->pts || !kp->nrm) return fail(c, BT_EINVAL, "keypoints: NULL buffer");
  if (!aligned16(kp->desc) || !aligned16(kp->pts) || !aligned16(kp->nrm) || !aligned16(kp->n_kp))
    return fail(c, BT_EINVAL, "keypoints: buffers must be 16-byte aligned");
  return BT_OK;
}

bt_status check_maps(bt_ctx *c, const bt_maps *mp, const bt_intrinsics *K) {
  if (!mp || !K) return fail(c, BT_EINVAL, "maps / intrinsics: NULL");
  if (mp->width != K->width || mp->height != K->height)
    return fail(c, BT_EINVAL, "maps %dx%d != intrinsics %dx%d", mp->width, mp->height, K->width, K->height);
  if (mp->width < 1 || mp->height < 1 || mp->n_frames < 1) return fail(c, BT_EINVAL, "maps: empty");
  // the dense scratch is carved per call from the frame count, the pixel count AND the 32x32
  // tile count (a 600x512 map has fewer pixels than 640x480 but more tiles): all three bounded
  if (mp->n_frames > c->cap_frames || (size_t)mp->width * mp->height > (size_t)c->cap_w * c->cap_h ||
      bt::dense_tiles(mp->width, mp->height) > bt::dense_tiles(c->cap_w, c->cap_h) || !c->dense)
    return fail(c, BT_ECAPACITY, "maps %d x %dx%d beyond reserved %d x %dx%d", mp->n_frames, mp->width, mp->height,
                c->cap_frames, c->cap_w, c->cap_h);
  if (!mp->depth || !mp->normal || !mp->mask) return fail(c, BT_EINVAL, "maps: NULL buffer");
  if (!aligned16(mp->depth) || !aligned16(mp->normal) || !aligned16(mp->mask))
    return fail(c, BT_EINVAL, "maps: buffers must be 16-byte aligned");
  if (!(K->fx > 0.f) || !(K->fy > 0.f)) return fail(c, BT_EINVAL, "intrinsics: fx, fy must be > 0");
  return BT_OK;
}

// the scratch one launch_dense carves (frames, edges, pixels, tiles) against the reservation
bt_status check_dense_bytes(bt_ctx *c, const bt_maps *mp, int E) {
  const size_t need = bt::dense_scratch_bytes(mp->n_frames, E, mp->width, mp->height);
  if (need > c->cap_dense)
    return fail(c, BT_ECAPACITY, "dense scratch %zu B for %d frames x %d edges at %dx%d > reserved %zu B", need,
                mp->n_frames, E, mp->width, mp->height, c->cap_dense);
  return BT_OK;
}

bt_status check_ransac(bt_ctx *c, const bt_ransac_params *r) {
  if (!r) return fail(c, BT_EINVAL, "ransac params: NULL");
  if (r->n_hyp < 1) return fail(c, BT_EINVAL, "n_hyp < 1");
  if (r->n_hyp > c->cap_hyp) return fail(c, BT_ECAPACITY, "n_hyp %d > reserved %d", r->n_hyp, c->cap_hyp);
  if (!(r->delta_m > 0.f)) return fail(c, BT_EINVAL, "delta_m must be > 0");
  return BT_OK;
}

bt_status check_edge(bt_ctx *c, const bt_edge_params *e) {
  if (!e) return fail(c, BT_EINVAL, "edge params: NULL");
  if (!(e->dist_gate_m > 0.f) || !(e->huber_m > 0.f)) return fail(c, BT_EINVAL, "edge gates must be > 0");
  return BT_OK;
}

bt::KpView kview(const bt_keypoints *kp) {
  return bt::KpView{kp->n_frames, kp->n_max, kp->n_kp, kp->desc, kp->pts, kp->nrm};
}
bt::MapView mview(const bt_maps *m) {
  return bt::MapView{m->n_frames, m->width, m->height, m->depth, m->normal, m->mask};
}

}  // namespace

extern "C" {

const char *bt_status_string(bt_status s) {
  switch (s) {
    case BT_OK: return "BT_OK";
    case BT_EINVAL: return "BT_EINVAL";
    case BT_ENOMEM: return "BT_ENOMEM";
    case BT_ECUDA: return "BT_ECUDA";
    case BT_EUNSUPPORTED: return "BT_EUNSUPPORTED";
    case BT_ECAPACITY: return "BT_ECAPACITY";
  }
  return "BT_?";
}

bt_status bt_create(bt_ctx **out, int cuda_device) {
  if (!out) return BT_EINVAL;
  *out = nullptr;
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, cuda_device) != cudaSuccess) return BT_ECUDA;
  if (prop.major != 10 || prop.minor != 0) return BT_EUNSUPPORTED;   // built for sm_100a only
  if (cudaSetDevice(cuda_device) != cudaSuccess) return BT_ECUDA;
  bt_ctx *c = new (std::nothrow) bt_ctx;
  if (!c) return BT_ENOMEM;
  c->device = cuda_device;
  int prio_lo = 0, prio_hi = 0;
  cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
  if (const char *sp = getenv("BT_STREAM_PRIO")) {                 // dev A/B: 1 swapped, 2 equal
    if (sp[0] == '1') std::swap(prio_lo, prio_hi);
    else if (sp[0] == '2') prio_lo = prio_hi;
  }
  if (cudaStreamCreateWithPriority(&c->side, cudaStreamNonBlocking, prio_lo) != cudaSuccess ||
      cudaStreamCreateWithPriority(&c->hi, cudaStreamNonBlocking, prio_hi) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_join_hi, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_maps, cudaEventDisableTiming) != cudaSuccess ||
      cudaStreamCreateWithFlags(&c->h2d, cudaStreamNonBlocking) != cudaSuccess) {
    delete c;
    return BT_ECUDA;
  }
  for (auto &r : c->raw)
    if (cudaEventCreateWithFlags(&r.ev_in, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&r.ev_free, cudaEventDisableTiming) != cudaSuccess) {
      delete c;
      return BT_ECUDA;
    }
  const char *ff = getenv("BT_FORCE_FALLBACK");
  c->force_fallback = ff && ff[0] && ff[0] != '0';
  *out = c;
  return BT_OK;
}

void bt_destroy(bt_ctx *c) {
  if (!c) return;
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  for (auto &p : c->pending) { cudaEventDestroy(p.start); if (p.stop) cudaEventDestroy(p.stop); }
  for (auto e : c->ev_pool) cudaEventDestroy(e);
  if (c->side) cudaStreamDestroy(c->side);
  if (c->hi) cudaStreamDestroy(c->hi);
  if (c->ev_join_hi) cudaEventDestroy(c->ev_join_hi);
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ev_maps) cudaEventDestroy(c->ev_maps);
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  if (c->h2d) cudaStreamDestroy(c->h2d);
  for (auto &r : c->raw) {
    if (r.ev_in) cudaEventDestroy(r.ev_in);
    if (r.ev_free) cudaEventDestroy(r.ev_free);
  }
  free_scratch(c);
  delete c;
}

const char *bt_last_error(const bt_ctx *c) { return c ? c->err : "no context"; }

int32_t bt_last_launch_count(const bt_ctx *c) { return c ? c->launch.count : 0; }

size_t bt_record_words(int32_t n_max) { return n_max < 1 ? 0 : (size_t)bt::rec_words(n_max); }

bt_status bt_set_record_peers(bt_ctx *c, int32_t n_peers, const uint64_t *peers, int32_t row_offset, int32_t rows) {
  BT_CHECK_CTX(c);
  if (n_peers < 0 || n_peers > bt::kMaxPeers) return fail(c, BT_EINVAL, "bt_set_record_peers: n_peers %d", n_peers);
  if (n_peers > 0 && (!peers || row_offset < 0 || rows < 1))
    return fail(c, BT_EINVAL, "bt_set_record_peers: bad peers / row_offset / rows");
  for (int k = 0; k < n_peers; ++k)
    if (!peers[k]) return fail(c, BT_EINVAL, "bt_set_record_peers: peer %d NULL", k);
  bt::PeerRec pr;
  for (int k = 0; k < bt::kMaxPeers; ++k) pr.ptr[k] = k < n_peers ? (uint32_t *)(uintptr_t)peers[k] : nullptr;
  pr.n = n_peers;
  pr.row_off = n_peers ? row_offset : 0;
  c->peers = pr;
  c->peer_rows = n_peers ? rows : 0;
  return BT_OK;
}

bt_status bt_reserve(bt_ctx *c, int32_t max_pairs, int32_t n_max, int32_t max_hyp, int32_t max_frames,
                     int32_t width, int32_t height) {
  BT_CHECK_CTX(c);
  if (max_pairs < 1 || n_max < 1 || max_hyp < 1 || max_frames < 0 || width < 0 || height < 0)
    return fail(c, BT_EINVAL, "bt_reserve: bad sizes");
  if (n_max > 8192)                                              // smem-staged per-pair point sets
    return fail(c, BT_EUNSUPPORTED, "bt_reserve: n_max %d > 8192", n_max);
  cudaDeviceSynchronize();
  free_scratch(c);
  c->cap_pairs = c->cap_nmax = c->cap_hyp = c->cap_frames = c->cap_w = c->cap_h = 0;
  c->cap_dense = 0;
  c->cached_P = c->cached_nmax = -1;                             // the match lists are gone with the scratch
  const size_t PN = (size_t)max_pairs * n_max;
  const size_t dense_bytes = (width > 0 && height > 0 && max_frames > 0)
                                 ? bt::dense_scratch_bytes(max_frames, 2 * max_pairs, width, height) : 0;
  const int mframes = max_frames > 0 ? max_frames : 1;
  bool ok = cudaMalloc(&c->match, bt::match_scratch_bytes(mframes, max_pairs, n_max)) == cudaSuccess &&
            cudaMalloc(&c->matches, PN * 8) == cudaSuccess && cudaMalloc(&c->n_matches, (size_t)max_pairs * 4) == cudaSuccess &&
            cudaMalloc(&c->rscratch, bt::ransac_scratch_bytes(max_pairs, max_hyp, n_max)) == cudaSuccess;
  if (ok) {
    c->ms = bt::carve_match_scratch(c->match, mframes, max_pairs, n_max);
    c->rs = bt::carve_ransac_scratch(c->rscratch, max_pairs, max_hyp, n_max);
    // TMA tensor map over the fp16 unit descriptors: 2-D [rows][128], 64 x 128 boxes, 128B swizzle
    // process-wide driver entry point (not per device); a magic static is initialized once, thread-safely
    static const PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
      PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
      cudaDriverEntryPointQueryResult q;
      if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&fn, cudaEnableDefault, &q) != cudaSuccess ||
          q != cudaDriverEntryPointSuccess)
        fn = nullptr;
      return fn;
    }();
    const cuuint64_t rows = (cuuint64_t)mframes * bt::match_n_pad(n_max);
    cuuint64_t dims[2] = {(cuuint64_t)bt::kDim, rows};
    cuuint64_t strides[1] = {(cuuint64_t)bt::kDim * 2};
    cuuint32_t box[2] = {64, 128};
    cuuint32_t estr[2] = {1, 1};
    ok = encode && encode(&c->tmap_desc, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, c->ms.desc16, dims, strides, box, estr,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    // TMA view of the scoring features: 2-D [pairs * m_pad][64] fp16, 64 x 128 boxes, 128B swizzle
    if (ok) {
      cuuint64_t fd[2] = {64, (cuuint64_t)max_pairs * c->rs.m_pad};
      cuuint64_t fs[1] = {128};
      cuuint32_t fbox[2] = {64, (cuuint32_t)bt::score_chunk()};
      ok = encode(&c->tmap_feat, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, c->rs.feat, fd, fs, fbox, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
      c->rs.fmap = &c->tmap_feat;
    }
  }
  // the dense scratch's header (call counter / map-entry epoch, offset 0) and map region (offset
  // 256) start zeroed — epoch 0 is never a call's, so no entry is valid — and the maps are only
  // ever written with finite entries: k_dense reads stale words of rejected items without a
  // select.  Header word 2: the reserved map entries (cleared when the epochs wrap).
  if (ok && dense_bytes > 0) {
    const size_t map_entries = (size_t)mframes * width * height;
    c->dense_map_cap = map_entries;
    const uint32_t hdr2 = (uint32_t)map_entries;
    ok = map_entries < 0xFFFFFFFFull && cudaMalloc(&c->dense, dense_bytes) == cudaSuccess &&
         cudaMemset(c->dense, 0, 256 + map_entries * 32) == cudaSuccess &&
         cudaMemcpy((char *)c->dense + 8, &hdr2, 4, cudaMemcpyHostToDevice) == cudaSuccess;
    if (ok) {
      if (const char *e0 = getenv("BT_DENSE_EPOCH0")) {           // tests: start near the epoch wrap
        const uint32_t v = (uint32_t)strtoul(e0, nullptr, 10);
        ok = cudaMemcpy(c->dense, &v, 4, cudaMemcpyHostToDevice) == cudaSuccess;
      }
    }
  }
  if (ok) ok = cudaMalloc(&c->graph, bt::graph_scratch_bytes(mframes, max_pairs)) == cudaSuccess;
  if (ok && max_frames > 0) {
    const size_t FN = (size_t)max_frames * n_max, FP = (size_t)max_frames * width * height;
    ok = cudaMalloc(&c->st_nkp, (size_t)max_frames * 4) == cudaSuccess &&
         cudaMalloc(&c->st_desc, FN * 128 * 4) == cudaSuccess && cudaMalloc(&c->st_pts, FN * 12) == cudaSuccess &&
         cudaMalloc(&c->st_nrm, FN * 12) == cudaSuccess && cudaMalloc(&c->st_pose, (size_t)max_frames * sizeof(bt_pose)) == cudaSuccess &&
         cudaMalloc(&c->st_pairs, (size_t)max_pairs * 8) == cudaSuccess && cudaMalloc(&c->st_uid, (size_t)max_pairs * 4) == cudaSuccess &&
         cudaMalloc(&c->st_records, (size_t)max_pairs * bt::rec_words(n_max) * 4) == cudaSuccess;
    if (ok && FP > 0)
      ok = cudaMalloc(&c->st_depth, FP * 4) == cudaSuccess && cudaMalloc(&c->st_normal, FP * 12) == cudaSuccess &&
           cudaMalloc(&c->st_mask, FP) == cudaSuccess;
  }
  if (!ok) {
    cudaGetLastError();
    free_scratch(c);
    return fail(c, BT_ENOMEM, "bt_reserve: cudaMalloc failed");
  }
  c->cap_pairs = max_pairs; c->cap_nmax = n_max; c->cap_hyp = max_hyp; c->cap_frames = mframes;
  c->cap_w = width; c->cap_h = height; c->cap_dense = dense_bytes; c->cap_stage = max_frames;
  return BT_OK;
}

bt_status bt_match(bt_ctx *c, const bt_keypoints *kp, const int32_t *pairs, int32_t P,
                   const bt_match_params *prm, int32_t *matches, int32_t *n_matches, void *stream) {
  BT_CHECK_CTX(c);
  bt_status s;
  if ((s = check_kp(c, kp)) != BT_OK) return s;
  if (P < 0) return fail(c, BT_EINVAL, "P < 0");
  if (P > c->cap_pairs) return fail(c, BT_ECAPACITY, "P %d > reserved %d", P, c->cap_pairs);
  if (P == 0) return BT_OK;
  if (!pairs || !matches || !n_matches) return fail(c, BT_EINVAL, "bt_match: NULL buffer");
  const float ratio = prm ? prm->ratio : 1.f;
  bt::launch_match(kview(kp), pairs, P, ratio, c->ms, &c->tmap_desc, c->force_fallback, matches, n_matches,
                   (cudaStream_t)stream, c->launch);
  return after_launch(c, "bt_match");
}

bt_status bt_ransac(bt_ctx *c, const bt_keypoints *kp, const int32_t *pairs, const uint32_t *pair_uid,
                    int32_t P, const int32_t *matches, const int32_t *n_matches, const bt_ransac_params *prm,
                    uint32_t *records, int32_t *hyp_counts, void *stream) {
  BT_CHECK_CTX(c);
  bt_status s;
  if ((s = check_kp(c, kp)) != BT_OK) return s;
  if ((s = check_ransac(c, prm)) != BT_OK) return s;
  if (P < 0) return fail(c, BT_EINVAL, "P < 0");
  if (P > c->cap_pairs) return fail(c, BT_ECAPACITY, "P %d > reserved %d", P, c->cap_pairs);
  if (P == 0) return BT_OK;
  if (!pairs || !pair_uid || !matches || !n_matches || !records) return fail(c, BT_EINVAL, "bt_ransac: NULL buffer");
  bt::launch_ransac(kview(kp), pairs, pair_uid, P, matches, n_matches, *prm, c->rs, records,
                    bt::rec_words(kp->n_max), hyp_counts, nullptr, 0.f, (cudaStream_t)stream, c->launch);
  return after_launch(c, "bt_ransac");
}

bt_status bt_dense_corr(bt_ctx *c, const bt_maps *maps, const bt_intrinsics *K, const bt_pose *node_pose,
                        const int32_t *edges, int32_t E, const bt_edge_params *prm, float *out, void *stream) {
  BT_CHECK_CTX(c);
  bt_status s;
  if ((s = check_maps(c, maps, K)) != BT_OK) return s;
  if ((s = check_edge(c, prm)) != BT_OK) return s;
  if (E < 0) return fail(c, BT_EINVAL, "E < 0");
  if (E > 2 * c->cap_pairs) return fail(c, BT_ECAPACITY, "E %d > 2 * reserved pairs %d", E, c->cap_pairs);
  if (E == 0) return BT_OK;
  if ((s = check_dense_bytes(c, maps, E)) != BT_OK) return s;
  if (!node_pose || !edges || !out) return fail(c, BT_EINVAL, "bt_dense_corr: NULL buffer");
  bt::launch_dense(mview(maps), *K, node_pose, edges, nullptr, E, *prm, c->dense, c->dense_map_cap, out, 32, nullptr, 0, 0, 0,
                   (cudaStream_t)stream, c->launch);
  return after_launch(c, "bt_dense_corr");
}

bt_status bt_dense_assoc(bt_ctx *c, const bt_maps *maps, const bt_intrinsics *K, const bt_pose *node_pose,
                         const int32_t *edges, int32_t E, const bt_edge_params *prm, float *out, int32_t *assoc,
                         void *stream) {
  BT_CHECK_CTX(c);
  bt_status s;
  if ((s = check_maps(c, maps, K)) != BT_OK) return s;
  if ((s = check_edge(c, prm)) != BT_OK) return s;
  if (E < 0) return fail(c, BT_EINVAL, "E < 0");
  if (E > 2 * c->cap_pairs) return fail(c, BT_ECAPACITY, "E %d > 2 * reserved pairs %d", E, c->cap_pairs);
  if (E == 0) return BT_OK;
  if ((s = check_dense_bytes(c, maps, E)) != BT_OK) return s;
  if (!node_pose || !edges || !out || !assoc) return fail(c, BT_EINVAL, "bt_dense_assoc: NULL buffer");
  bt::launch_dense(mview(maps), *K, node_pose, edges, nullptr, E, *prm, c->dense, c->dense_map_cap, out, 32, nullptr, 0, 0, 0,
                   (cudaStream_t)stream, c->launch, assoc);
  return after_launch(c, "bt_dense_assoc");
}

static bt_status register_pairs_dev(bt_ctx *c, const bt_keypoints *kp, const bt_maps *maps,
                                    const bt_intrinsics *K, const bt_pose *node_pose, const int32_t *pairs,
                                    const uint32_t *uid, int32_t P, const bt_match_params *mprm,
                                    const bt_ransac_params *rprm, const bt_edge_params *eprm,
                                    uint32_t *records, cudaStream_t st) {
  const int rw = bt::rec_words(kp->n_max);
  const float ratio = mprm ? mprm->ratio : 1.f;
  bt::PeerRec pr = c->peers;                                    // NEXT-3: stores into the peers' rows too
  pr.stride = rw;
  const bt::PeerRec *peers = pr.n ? &pr : nullptr;
  // fork: the dense edges only need the maps and node poses, so they run on the side stream
  // while matching and RANSAC run on the caller's stream (event fork / join: capturable)
  // with the dense edges forked off, match -> RANSAC (the longer chain) runs on a high-priority
  // internal stream so the block scheduler dispatches its CTAs ahead of the dense edges'
  cudaStream_t ms = eprm ? c->hi : st;
  if (eprm) {
    cudaEventRecord(c->ev_fork, st);
    cudaStreamWaitEvent(c->side, c->ev_fork, 0);
    if (ms != st) cudaStreamWaitEvent(ms, c->ev_fork, 0);
    bt::launch_dense(mview(maps), *K, node_pose, nullptr, pairs, 2 * P, *eprm, c->dense, c->dense_map_cap, nullptr, 0, records, rw,
                     bt::rec_dense_ij(kp->n_max), bt::rec_dense_ji(kp->n_max), c->side, c->launch, nullptr, peers);
  }
  bt::launch_match(kview(kp), pairs, P, ratio, c->ms, &c->tmap_desc, c->force_fallback, c->matches, c->n_matches,
                   ms, c->launch);
  bt::launch_ransac(kview(kp), pairs, uid, P, c->matches, c->n_matches, *rprm, c->rs, records, rw, nullptr,
                    eprm ? node_pose : nullptr, eprm ? eprm->huber_m : 0.f, ms, c->launch, peers);
  if (eprm) {
    cudaEventRecord(c->ev_join, c->side);
    cudaStreamWaitEvent(st, c->ev_join, 0);
    if (ms != st) {
      cudaEventRecord(c->ev_join_hi, ms);
      cudaStreamWaitEvent(st, c->ev_join_hi, 0);
    }
  }
  c->cached_P = P;
  c->cached_nmax = kp->n_max;
  return after_launch(c, "bt_register_pairs");
}

bt_status bt_register_pairs(bt_ctx *c, const bt_keypoints *kp, const bt_maps *maps, const bt_intrinsics *K,
                            const bt_pose *node_pose, const int32_t *pairs, const uint32_t *pair_uid, int32_t P,
                            const bt_match_params *mprm, const bt_ransac_params *rprm, const bt_edge_params *eprm,
                            uint32_t *records, void *stream) {
  BT_CHECK_CTX(c);
  bt_status s;
  if ((s = check_kp(c, kp)) != BT_OK) return s;
  if ((s = check_ransac(c, rprm)) != BT_OK) return s;
  if (eprm) {
    if ((s = check_edge(c, eprm)) != BT_OK) return s;
    if ((s = check_maps(c, maps, K)) != BT_OK) return s;
    if (!node_pose) return fail(c, BT_EINVAL, "bt_register_pairs: node_pose NULL");
    if (maps->n_frames < kp->n_frames) return fail(c, BT_EINVAL, "maps cover fewer frames than keypoints");
  }
  if (P < 0) return fail(c, BT_EINVAL, "P < 0");
  if (P > c->cap_pairs) return fail(c, BT_ECAPACITY, "P %d > reserved %d", P, c->cap_pairs);
  if (P == 0) return BT_OK;
  if (eprm && (s = check_dense_bytes(c, maps, 2 * P)) != BT_OK) return s;
  if (!pairs || !pair_uid || !records) return fail(c, BT_EINVAL, "bt_register_pairs: NULL buffer");
  if (c->peers.n && c->peers.row_off + P > c->peer_rows)
    return fail(c, BT_ECAPACITY, "bt_register_pairs: peer rows %d + P %d > %d", c->peers.row_off, P, c->peer_rows);
  return register_pairs_dev(c, kp, maps, K, node_pose, pairs, pair_uid, P, mprm, rprm, eprm, records,
                            (cudaStream_t)stream);
}

bt_status bt_register_pairs_host(bt_ctx *c, const bt_keypoints *kp, const bt_maps *maps, const bt_intrinsics *K,
                                 const bt_pose *node_pose, const int32_t *pairs, const uint32_t *pair_uid,
                                 int32_t P, const bt_match_params *mprm, const bt_ransac_params *rprm,
                                 const bt_edge_params *eprm, uint32_t *records, void *stream) {
  BT_CHECK_CTX(c);
  bt_status s;
  if (!kp) return fail(c, BT_EINVAL, "keypoints: NULL");
  if (kp->n_frames > c->cap_stage) return fail(c, BT_ECAPACITY, "frames %d > reserved staging %d", kp->n_frames, c->cap_stage);
  if ((s = check_ransac(c, rprm)) != BT_OK) return s;
  if (P < 0) return fail(c, BT_EINVAL, "P < 0");
  if (P > c->cap_pairs) return fail(c, BT_ECAPACITY, "P %d > reserved %d", P, c->cap_pairs);
  if (kp->n_max > c->cap_nmax) return fail(c, BT_ECAPACITY, "n_max %d > reserved %d", kp->n_max, c->cap_nmax);
  if (P == 0) return BT_OK;
  if (!pairs || !pair_uid || !records || !kp->n_kp || !kp->desc || !kp->pts || !kp->nrm)
    return fail(c, BT_EINVAL, "bt_register_pairs_host: NULL buffer");
  // every check before the first copy is enqueued (on failure nothing is enqueued): the staged
  // views carry the staging pointers, so the device-path checks apply to them unchanged
  bt_keypoints dk = *kp;
  dk.n_kp = c->st_nkp; dk.desc = c->st_desc; dk.pts = c->st_pts; dk.nrm = c->st_nrm;
  if ((s = check_kp(c, &dk)) != BT_OK) return s;                // dim == 128, n_max in [1, reserved]
  bt_maps dm{};
  if (eprm) {
    if (!maps || !K || !node_pose) return fail(c, BT_EINVAL, "bt_register_pairs_host: NULL maps/K/poses");
    if (!maps->depth || !maps->normal || !maps->mask) return fail(c, BT_EINVAL, "bt_register_pairs_host: NULL map buffer");
    if (maps->n_frames > c->cap_stage || (size_t)maps->width * maps->height > (size_t)c->cap_w * c->cap_h)
      return fail(c, BT_ECAPACITY, "maps beyond reserved staging");
    dm = *maps;
    dm.depth = c->st_depth; dm.normal = c->st_normal; dm.mask = c->st_mask;
    if ((s = check_maps(c, &dm, K)) != BT_OK) return s;
    if ((s = check_edge(c, eprm)) != BT_OK) return s;
    if ((s = check_dense_bytes(c, &dm, 2 * P)) != BT_OK) return s;
    if (maps->n_frames < kp->n_frames) return fail(c, BT_EINVAL, "maps cover fewer frames than keypoints");
  }
  const cudaStream_t st = (cudaStream_t)stream;
  const int F = kp->n_frames;
  const size_t FN = (size_t)F * kp->n_max;
  c->cached_P = -1;                                              // match lists from staged keypoints
  const int rw = bt::rec_words(kp->n_max);
  c->launch.count = 0;
  // keypoints first on the caller's stream: matching + RANSAC start as soon as they land,
  // while the (much larger) maps stream in on the side stream and feed the dense edges there
  cudaEventRecord(c->ev_fork, st);                               // staging buffers free
  cudaStreamWaitEvent(c->side, c->ev_fork, 0);
  cudaMemcpyAsync(c->st_nkp, kp->n_kp, (size_t)F * 4, cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(c->st_desc, kp->desc, FN * 128 * 4, cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(c->st_pts, kp->pts, FN * 12, cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(c->st_nrm, kp->nrm, FN * 12, cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(c->st_pairs, pairs, (size_t)P * 8, cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(c->st_uid, pair_uid, (size_t)P * 4, cudaMemcpyHostToDevice, st);
  if (eprm) {
    const size_t FP = (size_t)maps->n_frames * maps->width * maps->height;
    // poses on the caller's stream: the finish kernel (Eq. (2) blocks) reads them there
    cudaMemcpyAsync(c->st_pose, node_pose, (size_t)maps->n_frames * sizeof(bt_pose), cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(c->st_mask, maps->mask, FP, cudaMemcpyHostToDevice, c->side);
    cudaMemcpyAsync(c->st_depth, maps->depth, FP * 4, cudaMemcpyHostToDevice, c->side);
    cudaMemcpyAsync(c->st_normal, maps->normal, FP * 12, cudaMemcpyHostToDevice, c->side);
    // the dense kernels need the pair list and poses too: wait for the caller-stream copies
    cudaEventRecord(c->ev_join, st);
    cudaStreamWaitEvent(c->side, c->ev_join, 0);
    bt::launch_dense(mview(&dm), *K, c->st_pose, nullptr, c->st_pairs, 2 * P, *eprm, c->dense, c->dense_map_cap, nullptr, 0,
                     c->st_records, rw, bt::rec_dense_ij(kp->n_max), bt::rec_dense_ji(kp->n_max), c->side, c->launch);
  }
  const float ratio = mprm ? mprm->ratio : 1.f;
  bt::launch_match(kview(&dk), c->st_pairs, P, ratio, c->ms, &c->tmap_desc, c->force_fallback, c->matches,
                   c->n_matches, st, c->launch);
  bt::launch_ransac(kview(&dk), c->st_pairs, c->st_uid, P, c->matches, c->n_matches, *rprm, c->rs,
                    c->st_records, rw, nullptr, eprm ? c->st_pose : nullptr, eprm ? eprm->huber_m : 0.f, st,
                    c->launch);
  if (eprm) {
    cudaEventRecord(c->ev_join, c->side);
    cudaStreamWaitEvent(st, c->ev_join, 0);
  }
  if ((s = after_launch(c, "bt_register_pairs_host")) != BT_OK) return s;
  const int launches = c->launch.count;
  cudaMemcpyAsync(records, c->st_records, (size_t)P * rw * 4, cudaMemcpyDeviceToHost, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) return fail(c, BT_ECUDA, "bt_register_pairs_host: sync failed");
  c->launch.count = launches;
  return after_launch(c, "bt_register_pairs_host");
}

// NEXT-4 end to end: the raw per-frame inputs (depth, mask, the detector's 2-D keypoints and
// descriptors) from host memory; normals (bt_estimate_normals) and the keypoints' 3-D points /
// normals (bt_lift_keypoints) are derived on the device, then the whole per-pair path.
namespace {
// the raw entry's two staging slots, at the reserved capacity (first raw call only)
bool ensure_raw_slots(bt_ctx *c) {
  if (c->raw[0].depth) return true;
  const size_t F = (size_t)c->cap_stage, FN = F * c->cap_nmax, FP = F * c->cap_w * c->cap_h;
  bool ok = F > 0 && FP > 0;
  for (auto &r : c->raw)
    ok = ok && cudaMalloc(&r.depth, FP * 4) == cudaSuccess && cudaMalloc(&r.normal, FP * 12) == cudaSuccess &&
         cudaMalloc(&r.mask, FP) == cudaSuccess && cudaMalloc(&r.uv, FN * 8) == cudaSuccess &&
         cudaMalloc(&r.desc_in, FN * bt::kDim * 4) == cudaSuccess && cudaMalloc(&r.nin, F * 4) == cudaSuccess &&
         cudaMalloc(&r.pairs, (size_t)c->cap_pairs * 8) == cudaSuccess &&
         cudaMalloc(&r.uid, (size_t)c->cap_pairs * 4) == cudaSuccess && cudaMalloc(&r.pose, F * sizeof(bt_pose)) == cudaSuccess &&
         cudaMalloc(&r.depth_u16, FP * 2) == cudaSuccess &&
         cudaMalloc(&r.mask_bits, F * (size_t)c->cap_h * ((c->cap_w + 7) / 8) + 16) == cudaSuccess;
  if (!ok) {
    cudaGetLastError();
    for (auto &r : c->raw) {
      free_dev(r.depth); free_dev(r.normal); free_dev(r.uv); free_dev(r.desc_in); free_dev(r.mask);
      free_dev(r.nin); free_dev(r.pairs); free_dev(r.uid); free_dev(r.pose); free_dev(r.depth_u16);
      free_dev(r.mask_bits);
    }
  }
  return ok;
}

// validate, then enqueue one raw call on staging slot c->raw_next (see include/bt.h)
bt_status raw_enqueue(bt_ctx *c, const bt_raw_frames *raw, const bt_intrinsics *K, const bt_pose *node_pose,
                      const int32_t *pairs, const uint32_t *pair_uid, int32_t P, const bt_match_params *mprm,
                      const bt_ransac_params *rprm, const bt_edge_params *eprm, uint32_t *records, cudaStream_t st,
                      const char *what) {
  bt_status s;
  if (!raw || !K || !node_pose) return fail(c, BT_EINVAL, "%s: NULL raw / K / poses", what);
  if (raw->dim != bt::kDim) return fail(c, BT_EUNSUPPORTED, "%s: descriptor dim %d != 128", what, raw->dim);
  const int F = raw->n_frames, W = raw->width, H = raw->height, n_max = raw->n_max;
  if (F < 1 || W < 1 || H < 1 || n_max < 1 || P < 0) return fail(c, BT_EINVAL, "%s: bad sizes", what);
  if (!(raw->jump_m >= 0.f)) return fail(c, BT_EINVAL, "%s: jump < 0", what);
  if (F > c->cap_stage) return fail(c, BT_ECAPACITY, "frames %d > reserved staging %d", F, c->cap_stage);
  if ((size_t)W * H > (size_t)c->cap_w * c->cap_h) return fail(c, BT_ECAPACITY, "maps beyond reserved staging");
  if (n_max > c->cap_nmax) return fail(c, BT_ECAPACITY, "n_max %d > reserved %d", n_max, c->cap_nmax);
  if (P > c->cap_pairs) return fail(c, BT_ECAPACITY, "P %d > reserved %d", P, c->cap_pairs);
  if ((s = check_ransac(c, rprm)) != BT_OK) return s;
  if (P == 0) return BT_OK;
  if (!raw->uv || !raw->desc || !raw->n_in || !pairs || !pair_uid || !records)
    return fail(c, BT_EINVAL, "%s: NULL buffer", what);
  if (!raw->mask == !raw->mask_bits)
    return fail(c, BT_EINVAL, "%s: exactly one of mask / mask_bits must be given", what);
  if (!raw->depth == !raw->depth_u16)
    return fail(c, BT_EINVAL, "%s: exactly one of depth / depth_u16 must be given", what);
  if (raw->depth_u16 && !(raw->depth_scale > 0.f))
    return fail(c, BT_EINVAL, "%s: depth_scale %g <= 0 with depth_u16", what, (double)raw->depth_scale);
  if (raw->mask_bits && (size_t)H * ((W + 7) / 8) > (size_t)c->cap_h * ((c->cap_w + 7) / 8))
    return fail(c, BT_ECAPACITY, "%s: packed mask rows beyond the reserved staging", what);
  if (!c->st_depth) return fail(c, BT_ECAPACITY, "%s: no staging reserved", what);
  if (!ensure_raw_slots(c)) return fail(c, BT_ENOMEM, "%s: staging allocation failed", what);
  const int slot = c->raw_next;
  bt_ctx::RawSlot &r = c->raw[slot];
  bt_maps dm{};
  dm.n_frames = F; dm.width = W; dm.height = H;
  dm.depth = r.depth; dm.normal = r.normal; dm.mask = r.mask;
  if ((s = check_maps(c, &dm, K)) != BT_OK) return s;
  if (eprm) {
    if ((s = check_edge(c, eprm)) != BT_OK) return s;
    if ((s = check_dense_bytes(c, &dm, 2 * P)) != BT_OK) return s;
  }
  bt_keypoints dk{};
  dk.n_frames = F; dk.n_max = n_max; dk.dim = bt::kDim;
  dk.n_kp = c->st_nkp; dk.desc = c->st_desc; dk.pts = c->st_pts; dk.nrm = c->st_nrm;
  if ((s = check_kp(c, &dk)) != BT_OK) return s;
  c->raw_next ^= 1;
  const size_t FN = (size_t)F * n_max, FP = (size_t)F * W * H;
  c->cached_P = -1;                                              // match lists from staged keypoints
  const int rw = bt::rec_words(n_max);
  c->launch.count = 0;
  // copy stream: every input into the slot, once the call that used the slot before is done
  // with it (so they overlap the kernels of the previous call)
  cudaStreamWaitEvent(c->h2d, r.ev_free, 0);
  const size_t FB = (size_t)F * H * ((W + 7) / 8);                // packed mask bytes
  if (raw->mask) cudaMemcpyAsync(r.mask, raw->mask, FP, cudaMemcpyHostToDevice, c->h2d);
  else cudaMemcpyAsync(r.mask_bits, raw->mask_bits, FB, cudaMemcpyHostToDevice, c->h2d);
  if (raw->depth) cudaMemcpyAsync(r.depth, raw->depth, FP * 4, cudaMemcpyHostToDevice, c->h2d);
  else cudaMemcpyAsync(r.depth_u16, raw->depth_u16, FP * 2, cudaMemcpyHostToDevice, c->h2d);
  cudaMemcpyAsync(r.pairs, pairs, (size_t)P * 8, cudaMemcpyHostToDevice, c->h2d);
  cudaMemcpyAsync(r.uid, pair_uid, (size_t)P * 4, cudaMemcpyHostToDevice, c->h2d);
  cudaMemcpyAsync(r.pose, node_pose, (size_t)F * sizeof(bt_pose), cudaMemcpyHostToDevice, c->h2d);
  cudaMemcpyAsync(r.nin, raw->n_in, (size_t)F * 4, cudaMemcpyHostToDevice, c->h2d);
  cudaMemcpyAsync(r.uv, raw->uv, FN * 8, cudaMemcpyHostToDevice, c->h2d);
  cudaMemcpyAsync(r.desc_in, raw->desc, FN * bt::kDim * 4, cudaMemcpyHostToDevice, c->h2d);
  cudaEventRecord(r.ev_in, c->h2d);
  // side stream: the normal map from depth, then (after the caller's stream reached this call:
  // the previous call's records are read) the dense edges
  cudaStreamWaitEvent(c->side, r.ev_in, 0);
  if (!raw->depth) bt::launch_depth_u16(r.depth_u16, raw->depth_scale, FP, r.depth, c->side, c->launch);
  if (!raw->mask) bt::launch_mask_bits(r.mask_bits, F, W, H, r.mask, c->side, c->launch);
  bt::launch_normals(r.depth, F, W, H, *K, raw->jump_m, r.normal, c->side, c->launch);
  cudaEventRecord(c->ev_maps, c->side);
  if (eprm) {
    cudaEventRecord(c->ev_fork, st);
    cudaStreamWaitEvent(c->side, c->ev_fork, 0);
    bt::launch_dense(mview(&dm), *K, r.pose, nullptr, r.pairs, 2 * P, *eprm, c->dense, c->dense_map_cap, nullptr, 0, c->st_records, rw,
                     bt::rec_dense_ij(n_max), bt::rec_dense_ji(n_max), c->side, c->launch);
  }
  // caller's stream: lifting (needs the normal map), matching, RANSAC
  cudaStreamWaitEvent(st, c->ev_maps, 0);
  bt::launch_lift(F, n_max, r.uv, r.desc_in, r.nin, mview(&dm), *K, c->st_nkp, c->st_desc, c->st_pts, c->st_nrm, st,
                  c->launch);
  const float ratio = mprm ? mprm->ratio : 1.f;
  bt::launch_match(kview(&dk), r.pairs, P, ratio, c->ms, &c->tmap_desc, c->force_fallback, c->matches, c->n_matches,
                   st, c->launch);
  bt::launch_ransac(kview(&dk), r.pairs, r.uid, P, c->matches, c->n_matches, *rprm, c->rs, c->st_records, rw, nullptr,
                    eprm ? r.pose : nullptr, eprm ? eprm->huber_m : 0.f, st, c->launch);
  if (eprm) {
    cudaEventRecord(c->ev_join, c->side);
    cudaStreamWaitEvent(st, c->ev_join, 0);
  }
  cudaMemcpyAsync(records, c->st_records, (size_t)P * rw * 4, cudaMemcpyDeviceToHost, st);
  cudaEventRecord(r.ev_free, st);
  return after_launch(c, what);
}
}  // namespace

bt_status bt_register_raw_host(bt_ctx *c, const bt_raw_frames *raw, const bt_intrinsics *K,
                               const bt_pose *node_pose, const int32_t *pairs, const uint32_t *pair_uid, int32_t P,
                               const bt_match_params *mprm, const bt_ransac_params *rprm,
                               const bt_edge_params *eprm, uint32_t *records, void *stream) {
  BT_CHECK_CTX(c);
  const cudaStream_t st = (cudaStream_t)stream;
  bt_status s = raw_enqueue(c, raw, K, node_pose, pairs, pair_uid, P, mprm, rprm, eprm, records, st,
                            "bt_register_raw_host");
  if (s != BT_OK || P == 0) return s;
  const int launches = c->launch.count;
  if (cudaStreamSynchronize(st) != cudaSuccess) return fail(c, BT_ECUDA, "bt_register_raw_host: sync failed");
  c->launch.count = launches;
  return after_launch(c, "bt_register_raw_host");
}

bt_status bt_register_raw_host_async(bt_ctx *c, const bt_raw_frames *raw, const bt_intrinsics *K,
                                     const bt_pose *node_pose, const int32_t *pairs, const uint32_t *pair_uid,
                                     int32_t P, const bt_match_params *mprm, const bt_ransac_params *rprm,
                                     const bt_edge_params *eprm, uint32_t *records, void *stream) {
  BT_CHECK_CTX(c);
  return raw_enqueue(c, raw, K, node_pose, pairs, pair_uid, P, mprm, rprm, eprm, records, (cudaStream_t)stream,
                     "bt_register_raw_host_async");
}

bt_status bt_compose_poses(bt_ctx *c, const bt_pose *a, const bt_pose *b, bt_pose *out, int32_t n, void *stream) {
  BT_CHECK_CTX(c);
  if (n < 0) return fail(c, BT_EINVAL, "n < 0");
  if (n == 0) return BT_OK;
  if (!a || !b || !out) return fail(c, BT_EINVAL, "bt_compose_poses: NULL buffer");
  bt::launch_compose(a, b, out, n, (cudaStream_t)stream, c->launch);
  return after_launch(c, "bt_compose_poses");
}

bt_status bt_pose_graph_step(bt_ctx *c, int32_t n_nodes, const bt_pose *node_pose, const int32_t *pairs,
                             int32_t P, const uint32_t *records, int32_t n_max, const bt_graph_params *prm,
                             bt_pose *new_pose, double *delta, float *stats, void *stream) {
  BT_CHECK_CTX(c);
  if (!prm) return fail(c, BT_EINVAL, "bt_pose_graph_step: NULL params");
  if (n_nodes < 1) return fail(c, BT_EINVAL, "n_nodes %d < 1", n_nodes);
  if (n_nodes > c->cap_frames) return fail(c, BT_ECAPACITY, "n_nodes %d > reserved max_frames %d", n_nodes, c->cap_frames);
  if (P < 0) return fail(c, BT_EINVAL, "P < 0");
  if (P > c->cap_pairs) return fail(c, BT_ECAPACITY, "P %d > reserved %d", P, c->cap_pairs);
  if (n_max < 1) return fail(c, BT_EINVAL, "n_max < 1");
  if (prm->fixed_node < 0 || prm->fixed_node >= n_nodes)
    return fail(c, BT_EINVAL, "fixed_node %d outside [0, %d)", prm->fixed_node, n_nodes);
  if (prm->max_iter < 1 || !(prm->rel_tol >= 0.f) || !(prm->lambda_feat >= 0.f) || !(prm->lambda_dense >= 0.f) ||
      (prm->precond != 0 && prm->precond != 1))
    return fail(c, BT_EINVAL, "bt_pose_graph_step: bad params");
  if (!node_pose || !new_pose || (P > 0 && (!pairs || !records)))
    return fail(c, BT_EINVAL, "bt_pose_graph_step: NULL buffer");
  c->launch.count = 0;
  bt::launch_graph(n_nodes, node_pose, pairs, P, records, n_max, *prm, c->graph, new_pose, delta, stats,
                   (cudaStream_t)stream, c->launch);
  return after_launch(c, "bt_pose_graph_step");
}

bt_status bt_estimate_normals(bt_ctx *c, const float *depth, int32_t n_frames, int32_t width, int32_t height,
                              const bt_intrinsics *K, float jump_m, float *normal, void *stream) {
  BT_CHECK_CTX(c);
  if (n_frames < 0 || width < 0 || height < 0) return fail(c, BT_EINVAL, "bt_estimate_normals: negative size");
  if (!K || !(K->fx > 0.f) || !(K->fy > 0.f)) return fail(c, BT_EINVAL, "bt_estimate_normals: bad intrinsics");
  if (!(jump_m >= 0.f)) return fail(c, BT_EINVAL, "bt_estimate_normals: jump < 0");
  if ((size_t)n_frames * width * height == 0) return BT_OK;
  if (!depth || !normal) return fail(c, BT_EINVAL, "bt_estimate_normals: NULL buffer");
  if (((uintptr_t)normal & 15) != 0) return fail(c, BT_EINVAL, "bt_estimate_normals: normal not 16-B aligned");
  c->launch.count = 0;
  bt::launch_normals(depth, n_frames, width, height, *K, jump_m, normal, (cudaStream_t)stream, c->launch);
  return after_launch(c, "bt_estimate_normals");
}

bt_status bt_lift_keypoints(bt_ctx *c, int32_t n_frames, int32_t n_max, int32_t dim, const float *uv,
                            const float *desc_in, const int32_t *n_in, const bt_maps *maps, const bt_intrinsics *K,
                            int32_t *n_kp, float *desc, float *pts, float *nrm, void *stream) {
  BT_CHECK_CTX(c);
  if (dim != bt::kDim) return fail(c, BT_EUNSUPPORTED, "bt_lift_keypoints: descriptor dim %d != 128", dim);
  if (n_frames < 0 || n_max < 1) return fail(c, BT_EINVAL, "bt_lift_keypoints: bad sizes");
  if (n_frames == 0) return BT_OK;
  if (!maps || !K) return fail(c, BT_EINVAL, "bt_lift_keypoints: NULL maps / intrinsics");
  if (maps->n_frames < n_frames) return fail(c, BT_EINVAL, "bt_lift_keypoints: maps cover %d < %d frames",
                                             maps->n_frames, n_frames);
  if (maps->width != K->width || maps->height != K->height || maps->width < 1 || maps->height < 1)
    return fail(c, BT_EINVAL, "bt_lift_keypoints: maps %dx%d vs intrinsics %dx%d", maps->width, maps->height,
                K->width, K->height);
  if (!(K->fx > 0.f) || !(K->fy > 0.f)) return fail(c, BT_EINVAL, "bt_lift_keypoints: fx, fy must be > 0");
  if (!uv || !desc_in || !n_in || !maps->depth || !maps->normal || !maps->mask || !n_kp || !desc || !pts || !nrm)
    return fail(c, BT_EINVAL, "bt_lift_keypoints: NULL buffer");
  if (!aligned16(uv) || !aligned16(desc_in) || !aligned16(desc))
    return fail(c, BT_EINVAL, "bt_lift_keypoints: uv / desc buffers must be 16-byte aligned");
  c->launch.count = 0;
  bt::launch_lift(n_frames, n_max, uv, desc_in, n_in, mview(maps), *K, n_kp, desc, pts, nrm, (cudaStream_t)stream,
                  c->launch);
  return after_launch(c, "bt_lift_keypoints");
}

bt_status bt_coarse_pose(bt_ctx *c, const uint32_t *record, const bt_pose *prev, bt_pose *out, void *stream) {
  BT_CHECK_CTX(c);
  if (!record || !prev || !out) return fail(c, BT_EINVAL, "bt_coarse_pose: NULL buffer");
  bt::launch_coarse_pose(record, prev, out, (cudaStream_t)stream, c->launch);
  return after_launch(c, "bt_coarse_pose");
}

bt_status bt_select_keyframes(bt_ctx *c, const bt_pose *pool, const int32_t *n_pool, int32_t pool_cap,
                              const bt_pose *cur, int32_t K, int32_t *sel, int32_t *n_sel, void *stream) {
  BT_CHECK_CTX(c);
  if (pool_cap < 1 || pool_cap > 4096 || K < 1) return fail(c, BT_EINVAL, "bt_select_keyframes: pool_cap %d / K %d",
                                                            pool_cap, K);
  if (!pool || !n_pool || !cur || !sel || !n_sel) return fail(c, BT_EINVAL, "bt_select_keyframes: NULL buffer");
  bt::launch_select(pool, n_pool, pool_cap, cur, K, sel, n_sel, (cudaStream_t)stream, c->launch);
  return after_launch(c, "bt_select_keyframes");
}

bt_status bt_pool_admit(bt_ctx *c, bt_pose *pool, int32_t *n_pool, int32_t pool_cap, const bt_pose *cur,
                        float thresh_rad, int32_t *admitted, void *stream) {
  BT_CHECK_CTX(c);
  if (pool_cap < 1 || !(thresh_rad >= 0.f)) return fail(c, BT_EINVAL, "bt_pool_admit: pool_cap %d / thresh", pool_cap);
  if (!pool || !n_pool || !cur) return fail(c, BT_EINVAL, "bt_pool_admit: NULL buffer");
  bt::launch_admit(pool, n_pool, pool_cap, cur, (double)thresh_rad, admitted, (cudaStream_t)stream, c->launch);
  return after_launch(c, "bt_pool_admit");
}

static bt_status relinearize(bt_ctx *c, const char *what, const bt_keypoints *kp, const bt_maps *maps,
                             const bt_intrinsics *K, const bt_pose *node_pose, const int32_t *pairs, int32_t P,
                             const int32_t *matches, const int32_t *n_matches, const bt_edge_params *eprm,
                             uint32_t *records, void *stream) {
  bt_status s;
  if ((s = check_kp(c, kp)) != BT_OK) return s;
  if ((s = check_maps(c, maps, K)) != BT_OK) return s;
  if (!eprm) return fail(c, BT_EINVAL, "%s: NULL edge params", what);
  if ((s = check_edge(c, eprm)) != BT_OK) return s;
  if (P < 0) return fail(c, BT_EINVAL, "P < 0");
  if (P == 0) return BT_OK;
  if (P > c->cap_pairs) return fail(c, BT_ECAPACITY, "%s: P %d > reserved %d", what, P, c->cap_pairs);
  if ((s = check_dense_bytes(c, maps, 2 * P)) != BT_OK) return s;
  if (!node_pose || !pairs || !records || !matches || !n_matches) return fail(c, BT_EINVAL, "%s: NULL buffer", what);
  const cudaStream_t st = (cudaStream_t)stream;
  const int rw = bt::rec_words(kp->n_max);
  c->launch.count = 0;
  cudaEventRecord(c->ev_fork, st);                                 // dense edges beside the feature blocks
  cudaStreamWaitEvent(c->side, c->ev_fork, 0);
  bt::launch_dense(mview(maps), *K, node_pose, nullptr, pairs, 2 * P, *eprm, c->dense, c->dense_map_cap, nullptr, 0, records, rw,
                   bt::rec_dense_ij(kp->n_max), bt::rec_dense_ji(kp->n_max), c->side, c->launch);
  bt::launch_feature_edges(kview(kp), pairs, P, matches, n_matches, records, rw, node_pose, eprm->huber_m, st,
                           c->launch);
  cudaEventRecord(c->ev_join, c->side);
  cudaStreamWaitEvent(st, c->ev_join, 0);
  return after_launch(c, what);
}

bt_status bt_relinearize(bt_ctx *c, const bt_keypoints *kp, const bt_maps *maps, const bt_intrinsics *K,
                         const bt_pose *node_pose, const int32_t *pairs, int32_t P, const bt_edge_params *eprm,
                         uint32_t *records, void *stream) {
  BT_CHECK_CTX(c);
  if (P > 0 && (P != c->cached_P || (kp && kp->n_max != c->cached_nmax)))
    return fail(c, BT_EINVAL, "bt_relinearize: P %d does not match the last bt_register_pairs (%d pairs)", P,
                c->cached_P);
  return relinearize(c, "bt_relinearize", kp, maps, K, node_pose, pairs, P, c->matches, c->n_matches, eprm, records,
                     stream);
}

bt_status bt_relinearize_matches(bt_ctx *c, const bt_keypoints *kp, const bt_maps *maps, const bt_intrinsics *K,
                                 const bt_pose *node_pose, const int32_t *pairs, int32_t P, const int32_t *matches,
                                 const int32_t *n_matches, const bt_edge_params *eprm, uint32_t *records,
                                 void *stream) {
  BT_CHECK_CTX(c);
  return relinearize(c, "bt_relinearize_matches", kp, maps, K, node_pose, pairs, P, matches, n_matches, eprm, records,
                     stream);
}

bt_status bt_copy_matches(bt_ctx *c, int32_t P, int32_t n_max, int32_t *matches, int32_t *n_matches, void *stream) {
  BT_CHECK_CTX(c);
  if (!matches || !n_matches) return fail(c, BT_EINVAL, "bt_copy_matches: NULL buffer");
  if (P != c->cached_P || n_max != c->cached_nmax)
    return fail(c, BT_EINVAL, "bt_copy_matches: P %d / n_max %d do not match the last bt_register_pairs (%d / %d)", P,
                n_max, c->cached_P, c->cached_nmax);
  const cudaStream_t st = (cudaStream_t)stream;
  if (cudaMemcpyAsync(matches, c->matches, (size_t)P * n_max * 2 * sizeof(int32_t), cudaMemcpyDeviceToDevice, st) !=
          cudaSuccess ||
      cudaMemcpyAsync(n_matches, c->n_matches, (size_t)P * sizeof(int32_t), cudaMemcpyDeviceToDevice, st) !=
          cudaSuccess)
    return fail(c, BT_ECUDA, "bt_copy_matches: %s", cudaGetErrorString(cudaGetLastError()));
  return BT_OK;
}

static const char *kKernelNames[bt::K_COUNT] = {"k_desc_prep", "k_match_tc", "k_rescore", "k_mutual",
                                                 "k_ransac_hyp", "k_ransac_score", "k_ransac_finish", "k_dense_prep",
                                                 "k_dense", "k_dense_reduce", "k_compose", "k_graph", "k_normals",
                                                 "k_track"};

static cudaEvent_t take_event(bt_ctx *c) {
  if (c->ev_pool.empty()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
  }
  cudaEvent_t e = c->ev_pool.back();
  c->ev_pool.pop_back();
  return e;
}

static void prof_hook(void *user, int kid, int phase, cudaStream_t s) {
  bt_ctx *c = (bt_ctx *)user;
  if (c->prof_only >= 0 && kid != c->prof_only) return;
  cudaEvent_t e = take_event(c);
  cudaEventRecord(e, s);
  if (phase == 0) c->pending.push_back({kid, e, nullptr});
  else c->pending.back().stop = e;
}

bt_status bt_profile_enable(bt_ctx *c, int32_t on) {
  BT_CHECK_CTX(c);
  if (on < 0 || on >= 2 + bt::K_COUNT) return fail(c, BT_EINVAL, "bt_profile_enable: on = %d", on);
  c->prof_on = on != 0;
  c->prof_only = on >= 2 ? on - 2 : -1;
  c->launch.hook = c->prof_on ? prof_hook : nullptr;
  c->launch.user = c;
  return BT_OK;
}

int32_t bt_profile_kernels(void) { return bt::K_COUNT; }

const char *bt_profile_name(int32_t k) { return (k >= 0 && k < bt::K_COUNT) ? kKernelNames[k] : "?"; }

bt_status bt_profile_read(bt_ctx *c, int32_t kid, double *total_ms, int64_t *launches) {
  if (!c) return BT_EINVAL;
  if (kid < 0 || kid >= bt::K_COUNT || !total_ms || !launches) return fail(c, BT_EINVAL, "bt_profile_read: bad args");
  if (cudaSetDevice(c->device) != cudaSuccess) return fail(c, BT_ECUDA, "cudaSetDevice failed");
  for (auto &p : c->pending) {                 // fold every completed bracket into the totals
    if (!p.stop) continue;
    if (cudaEventSynchronize(p.stop) != cudaSuccess) return fail(c, BT_ECUDA, "bt_profile_read: event sync");
    float ms = 0.f;
    cudaEventElapsedTime(&ms, p.start, p.stop);
    c->prof_ms[p.kid] += ms;
    c->prof_n[p.kid] += 1;
    c->ev_pool.push_back(p.start);
    c->ev_pool.push_back(p.stop);
  }
  c->pending.clear();
  *total_ms = c->prof_ms[kid];
  *launches = c->prof_n[kid];
  c->prof_ms[kid] = 0.0;
  c->prof_n[kid] = 0;
  return BT_OK;
}

}  // extern "C"
