"""paper_2108_00516_b200 — B200-native BundleTrack pairwise-registration hot path.

Thin Python binding (argument marshalling only) over the C-ABI library libbt.so
(include/bt.h).  Every step of the path — matching, RANSAC, refit, Eq. (2) / Eq. (3)
linearization — runs in the library's sm_100a kernels; PyTorch is used only for device
memory, streams and (in bench.py / parallel tests) process groups.  There is no CPU
fallback: importing works anywhere, but creating a Context fails loudly when libbt.so is
missing or no sm_100 device is present.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BT_LIB") or os.path.join(_PKG, "libbt.so")   # BT_LIB: A/B builds (dev tools)

BT_OK, BT_EINVAL, BT_ENOMEM, BT_ECUDA, BT_EUNSUPPORTED, BT_ECAPACITY = range(6)
PAIR_OK, PAIR_FEW_MATCHES, PAIR_FEW_INLIERS, PAIR_REFIT_DEGENERATE = range(4)

# exported symbols (kept in sync with include/bt.h; tests check both)
SYMBOLS = ("bt_create", "bt_destroy", "bt_last_error", "bt_status_string", "bt_reserve",
           "bt_record_words", "bt_match", "bt_ransac", "bt_dense_corr", "bt_register_pairs",
           "bt_register_pairs_host", "bt_compose_poses", "bt_last_launch_count", "bt_profile_enable",
           "bt_profile_kernels", "bt_profile_name", "bt_profile_read", "bt_pose_graph_step",
           "bt_estimate_normals", "bt_relinearize", "bt_relinearize_matches", "bt_copy_matches",
           "bt_dense_assoc", "bt_lift_keypoints", "bt_coarse_pose", "bt_select_keyframes", "bt_pool_admit",
           "bt_set_record_peers", "bt_register_raw_host", "bt_register_raw_host_async")


class BtError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_STATUS.get(status, status)}: {msg}")
        self.status = status


_STATUS = {0: "BT_OK", 1: "BT_EINVAL", 2: "BT_ENOMEM", 3: "BT_ECUDA", 4: "BT_EUNSUPPORTED", 5: "BT_ECAPACITY"}


class Intrinsics(C.Structure):
    _fields_ = [("fx", C.c_float), ("fy", C.c_float), ("cx", C.c_float), ("cy", C.c_float),
                ("width", C.c_int32), ("height", C.c_int32)]


class Keypoints(C.Structure):
    _fields_ = [("n_frames", C.c_int32), ("n_max", C.c_int32), ("dim", C.c_int32),
                ("n_kp", C.c_void_p), ("desc", C.c_void_p), ("pts", C.c_void_p), ("nrm", C.c_void_p)]


class Maps(C.Structure):
    _fields_ = [("n_frames", C.c_int32), ("width", C.c_int32), ("height", C.c_int32),
                ("depth", C.c_void_p), ("normal", C.c_void_p), ("mask", C.c_void_p)]


class RawFrames(C.Structure):
    """bt_raw_frames: the raw per-frame inputs of bt_register_raw_host (host pointers)."""
    _fields_ = [("n_frames", C.c_int32), ("width", C.c_int32), ("height", C.c_int32), ("n_max", C.c_int32),
                ("dim", C.c_int32), ("jump_m", C.c_float), ("depth", C.c_void_p), ("mask", C.c_void_p),
                ("uv", C.c_void_p), ("desc", C.c_void_p), ("n_in", C.c_void_p), ("depth_u16", C.c_void_p),
                ("depth_scale", C.c_float), ("mask_bits", C.c_void_p)]


class MatchParams(C.Structure):
    _fields_ = [("ratio", C.c_float)]


class RansacParams(C.Structure):
    _fields_ = [("delta_m", C.c_float), ("cos_alpha", C.c_float), ("n_hyp", C.c_int32),
                ("pad_", C.c_uint32), ("seed", C.c_uint64), ("min_sigma_ratio", C.c_float),
                ("min_inliers", C.c_int32)]


class EdgeParams(C.Structure):
    _fields_ = [("dist_gate_m", C.c_float), ("cos_gate", C.c_float), ("huber_m", C.c_float),
                ("stride", C.c_int32)]


class GraphParams(C.Structure):
    _fields_ = [("lambda_feat", C.c_float), ("lambda_dense", C.c_float), ("fixed_node", C.c_int32),
                ("max_iter", C.c_int32), ("rel_tol", C.c_float), ("precond", C.c_int32)]


_lib = None


def lib():
    """Load libbt.so (built by __graft_entry__.build() / paper_2108_00516_b200.build)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"libbt.so not built ({LIB_PATH}); run python -c 'import __graft_entry__ as g; g.build()'")
        L = C.CDLL(LIB_PATH)
        vp, i32 = C.c_void_p, C.c_int32
        L.bt_create.argtypes = [C.POINTER(vp), C.c_int]
        L.bt_destroy.argtypes = [vp]
        L.bt_destroy.restype = None
        L.bt_last_error.argtypes = [vp]
        L.bt_last_error.restype = C.c_char_p
        L.bt_status_string.argtypes = [C.c_int]
        L.bt_status_string.restype = C.c_char_p
        L.bt_reserve.argtypes = [vp, i32, i32, i32, i32, i32, i32]
        L.bt_record_words.argtypes = [i32]
        L.bt_record_words.restype = C.c_size_t
        L.bt_match.argtypes = [vp, C.POINTER(Keypoints), vp, i32, C.POINTER(MatchParams), vp, vp, vp]
        L.bt_ransac.argtypes = [vp, C.POINTER(Keypoints), vp, vp, i32, vp, vp, C.POINTER(RansacParams), vp, vp, vp]
        L.bt_dense_corr.argtypes = [vp, C.POINTER(Maps), C.POINTER(Intrinsics), vp, vp, i32, C.POINTER(EdgeParams),
                                    vp, vp]
        L.bt_dense_assoc.argtypes = [vp, C.POINTER(Maps), C.POINTER(Intrinsics), vp, vp, i32, C.POINTER(EdgeParams),
                                     vp, vp, vp]
        rp = [vp, C.POINTER(Keypoints), C.POINTER(Maps), C.POINTER(Intrinsics), vp, vp, vp, i32,
              C.POINTER(MatchParams), C.POINTER(RansacParams), C.POINTER(EdgeParams), vp, vp]
        L.bt_register_pairs.argtypes = rp
        L.bt_register_pairs_host.argtypes = rp
        L.bt_compose_poses.argtypes = [vp, vp, vp, vp, i32, vp]
        L.bt_pose_graph_step.argtypes = [vp, i32, vp, vp, i32, vp, i32, C.POINTER(GraphParams), vp, vp, vp, vp]
        L.bt_estimate_normals.argtypes = [vp, vp, i32, i32, i32, C.POINTER(Intrinsics), C.c_float, vp, vp]
        L.bt_relinearize.argtypes = [vp, C.POINTER(Keypoints), C.POINTER(Maps), C.POINTER(Intrinsics), vp, vp, i32,
                                     C.POINTER(EdgeParams), vp, vp]
        L.bt_relinearize_matches.argtypes = [vp, C.POINTER(Keypoints), C.POINTER(Maps), C.POINTER(Intrinsics), vp, vp,
                                             i32, vp, vp, C.POINTER(EdgeParams), vp, vp]
        L.bt_copy_matches.argtypes = [vp, i32, i32, vp, vp, vp]
        L.bt_lift_keypoints.argtypes = [vp, i32, i32, i32, vp, vp, vp, C.POINTER(Maps), C.POINTER(Intrinsics), vp, vp,
                                        vp, vp, vp]
        L.bt_coarse_pose.argtypes = [vp, vp, vp, vp, vp]
        L.bt_select_keyframes.argtypes = [vp, vp, vp, i32, vp, i32, vp, vp, vp]
        L.bt_pool_admit.argtypes = [vp, vp, vp, i32, vp, C.c_float, vp, vp]
        L.bt_set_record_peers.argtypes = [vp, i32, C.POINTER(C.c_uint64), i32, i32]
        for f in ("bt_register_raw_host", "bt_register_raw_host_async"):
            getattr(L, f).argtypes = [vp, C.POINTER(RawFrames), C.POINTER(Intrinsics), vp, vp, vp, i32,
                                      C.POINTER(MatchParams), C.POINTER(RansacParams), C.POINTER(EdgeParams), vp, vp]
        L.bt_last_launch_count.argtypes = [vp]
        L.bt_last_launch_count.restype = i32
        L.bt_profile_enable.argtypes = [vp, i32]
        L.bt_profile_enable.restype = C.c_int
        L.bt_profile_kernels.argtypes = []
        L.bt_profile_kernels.restype = i32
        L.bt_profile_name.argtypes = [i32]
        L.bt_profile_name.restype = C.c_char_p
        L.bt_profile_read.argtypes = [vp, i32, C.POINTER(C.c_double), C.POINTER(C.c_int64)]
        L.bt_profile_read.restype = C.c_int
        for f in ("bt_create", "bt_reserve", "bt_match", "bt_ransac", "bt_dense_corr", "bt_dense_assoc", "bt_register_pairs",
                  "bt_register_pairs_host", "bt_compose_poses", "bt_pose_graph_step", "bt_estimate_normals", "bt_relinearize",
                  "bt_relinearize_matches", "bt_copy_matches", "bt_lift_keypoints", "bt_coarse_pose",
                  "bt_select_keyframes", "bt_pool_admit", "bt_set_record_peers", "bt_register_raw_host",
                  "bt_register_raw_host_async"):
            getattr(L, f).restype = C.c_int
        _lib = L
    return _lib


def record_words(n_max: int) -> int:
    return int(lib().bt_record_words(int(n_max)))


def mask_words(n_max: int) -> int:
    return (n_max + 31) // 32


def _ptr(t) -> int | None:
    if t is None:
        return None
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    return t.data_ptr()


def ransac_params(n_hyp: int, seed: int, delta_m: float = 0.005, alpha_deg: float = 45.0,
                  min_sigma_ratio: float = 1e-3, min_inliers: int = 3) -> RansacParams:
    """Defaults: delta = 5 mm and alpha = 45 deg; degeneracy and min-inlier readings R8."""
    return RansacParams(delta_m, float(np.cos(np.deg2rad(alpha_deg))), int(n_hyp), 0,
                        int(seed) & 0xFFFFFFFFFFFFFFFF, min_sigma_ratio, int(min_inliers))


def edge_params(dist_gate_m: float = 0.02, angle_deg: float = 45.0, huber_m: float = 0.005,
                stride: int = 1) -> EdgeParams:
    """Dense gates 2 cm / 45 deg and Huber 5 mm (readings R15, R17)."""
    return EdgeParams(dist_gate_m, float(np.cos(np.deg2rad(angle_deg))), huber_m, int(stride))


@dataclass
class FrameBatch:
    """Device (or pinned host) tensors of F frames in the layout include/bt.h expects."""
    n_kp: object      # [F] int32
    desc: object      # [F][n_max][128] float32
    pts: object       # [F][n_max][3] float32
    nrm: object       # [F][n_max][3] float32
    depth: object = None    # [F][H][W] float32
    normal: object = None   # [F][H][W][3] float32
    mask: object = None     # [F][H][W] uint8

    @property
    def n_max(self) -> int:
        return int(self.desc.shape[1])

    def keypoints(self) -> Keypoints:
        return Keypoints(int(self.desc.shape[0]), int(self.desc.shape[1]), int(self.desc.shape[2]),
                         _ptr(self.n_kp), _ptr(self.desc), _ptr(self.pts), _ptr(self.nrm))

    def maps(self) -> Maps | None:
        if self.depth is None:
            return None
        F, H, W = self.depth.shape
        return Maps(int(F), int(W), int(H), _ptr(self.depth), _ptr(self.normal), _ptr(self.mask))

    @staticmethod
    def from_scene(scene, device="cuda", pin: bool = False) -> "FrameBatch":
        import torch

        def t(a):
            x = torch.from_numpy(np.ascontiguousarray(a))
            if device == "cpu":
                return x.pin_memory() if pin else x
            return x.to(device)
        return FrameBatch(t(scene.n_kp), t(scene.desc), t(scene.pts), t(scene.nrm),
                          None if scene.depth is None else t(scene.depth),
                          None if scene.normal is None else t(scene.normal),
                          None if scene.mask is None else t(scene.mask))


def intrinsics(K) -> Intrinsics:
    return Intrinsics(K.fx, K.fy, K.cx, K.cy, int(K.width), int(K.height))


class Context:
    """One bt_ctx (one device, one host thread)."""

    def __init__(self, device: int = 0):
        L = lib()
        h = C.c_void_p()
        st = L.bt_create(C.byref(h), int(device))
        if st != BT_OK:
            raise BtError(st, f"bt_create(device={device}) failed (needs an sm_100 B200)")
        self._h = h
        self.device = device

    def close(self):
        if getattr(self, "_h", None):
            lib().bt_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    def _check(self, st: int, what: str):
        if st != BT_OK:
            raise BtError(st, f"{what}: {lib().bt_last_error(self._h).decode()}")

    @property
    def last_launches(self) -> int:
        return int(lib().bt_last_launch_count(self._h))

    def reserve(self, max_pairs: int, n_max: int, max_hyp: int, max_frames: int = 0, width: int = 0,
                height: int = 0):
        self._check(lib().bt_reserve(self._h, max_pairs, n_max, max_hyp, max_frames, width, height), "bt_reserve")

    @staticmethod
    def _stream(stream):
        if stream is None:
            import torch
            return torch.cuda.current_stream().cuda_stream
        return stream if isinstance(stream, int) else stream.cuda_stream

    def match(self, fb: FrameBatch, pairs, matches, n_matches, ratio: float = 1.0, stream=None):
        kp = fb.keypoints()
        self._check(lib().bt_match(self._h, C.byref(kp), _ptr(pairs), int(pairs.shape[0]),
                                   C.byref(MatchParams(ratio)), _ptr(matches), _ptr(n_matches),
                                   self._stream(stream)), "bt_match")

    def ransac(self, fb: FrameBatch, pairs, uid, matches, n_matches, prm: RansacParams, records,
               hyp_counts=None, stream=None):
        kp = fb.keypoints()
        self._check(lib().bt_ransac(self._h, C.byref(kp), _ptr(pairs), _ptr(uid), int(pairs.shape[0]),
                                    _ptr(matches), _ptr(n_matches), C.byref(prm), _ptr(records),
                                    _ptr(hyp_counts), self._stream(stream)), "bt_ransac")

    def dense_corr(self, fb: FrameBatch, K, node_pose, edges, prm: EdgeParams, out, stream=None):
        mp = fb.maps()
        Ki = intrinsics(K) if not isinstance(K, Intrinsics) else K
        self._check(lib().bt_dense_corr(self._h, C.byref(mp), C.byref(Ki), _ptr(node_pose), _ptr(edges),
                                        int(edges.shape[0]), C.byref(prm), _ptr(out), self._stream(stream)),
                    "bt_dense_corr")

    def dense_assoc(self, fb: FrameBatch, K, node_pose, edges, prm: EdgeParams, out, assoc, stream=None):
        """bt_dense_corr plus the per-source-pixel association assoc [E][H][W] int32 (target
        pixel index or -1) — the verification entry bt_dense_assoc."""
        mp = fb.maps()
        Ki = intrinsics(K) if not isinstance(K, Intrinsics) else K
        self._check(lib().bt_dense_assoc(self._h, C.byref(mp), C.byref(Ki), _ptr(node_pose), _ptr(edges),
                                         int(edges.shape[0]), C.byref(prm), _ptr(out), _ptr(assoc),
                                         self._stream(stream)), "bt_dense_assoc")

    def register_pairs(self, fb: FrameBatch, K, node_pose, pairs, uid, rprm: RansacParams,
                       eprm: EdgeParams | None, records, ratio: float = 1.0, stream=None, host=False):
        kp = fb.keypoints()
        mp = fb.maps()
        Ki = intrinsics(K) if not isinstance(K, Intrinsics) else K
        fn = lib().bt_register_pairs_host if host else lib().bt_register_pairs
        st = fn(self._h, C.byref(kp), C.byref(mp) if mp is not None else None, C.byref(Ki),
                _ptr(node_pose), _ptr(pairs), _ptr(uid), int(pairs.shape[0]), C.byref(MatchParams(ratio)),
                C.byref(rprm), C.byref(eprm) if eprm is not None else None, _ptr(records),
                self._stream(stream))
        self._check(st, "bt_register_pairs_host" if host else "bt_register_pairs")

    def register_raw(self, depth, mask, uv, desc, n_in, K, node_pose, pairs, uid, rprm: RansacParams,
                     eprm: EdgeParams | None, records, jump_m: float = 0.05, ratio: float = 1.0, stream=None,
                     blocking: bool = True, depth_scale: float = 0.0, mask_bits: bool = False):
        """bt_register_raw_host: depth [F][H][W] f32, mask [F][H][W] u8, uv [F][n_max][2] f32, desc
        [F][n_max][128] f32, n_in [F] i32, node_pose [F] (12 f32), pairs [P][2], uid [P], records
        [P][record_words] — all HOST tensors / arrays (pinned for full speed); normals and the
        keypoints' points / normals are derived on the device.  Synchronises the stream; with
        blocking=False (bt_register_raw_host_async) only enqueues: the copies of the next call
        overlap this call's kernels, and `records` is valid once the stream has passed the call;
        the host tensors passed in must stay alive and unchanged until then (the copies read them
        asynchronously — a temporary such as `t.pin_memory()` in the argument list is not safe).
        A uint16 `depth` (the sensor format; 0 invalid) is sent as is and scaled on the device:
        metres = value * depth_scale (fp32).  mask_bits=True: `mask` is packed bits [F][H][ceil(W/8)]
        (LSB first), unpacked on the device."""
        F, H, W = (int(x) for x in depth.shape)
        u16 = str(depth.dtype) in ("torch.uint16", "uint16")
        raw = RawFrames(F, W, H, int(uv.shape[1]), int(desc.shape[2]), float(jump_m), None if u16 else _ptr(depth),
                        None if mask_bits else _ptr(mask), _ptr(uv), _ptr(desc), _ptr(n_in),
                        _ptr(depth) if u16 else None, float(depth_scale), _ptr(mask) if mask_bits else None)
        Ki = intrinsics(K) if not isinstance(K, Intrinsics) else K
        name = "bt_register_raw_host" if blocking else "bt_register_raw_host_async"
        self._check(getattr(lib(), name)(self._h, C.byref(raw), C.byref(Ki), _ptr(node_pose), _ptr(pairs),
                                         _ptr(uid), int(pairs.shape[0]), C.byref(MatchParams(ratio)),
                                         C.byref(rprm), C.byref(eprm) if eprm is not None else None,
                                         _ptr(records), self._stream(stream)), name)

    def set_record_peers(self, peer_ptrs, row_offset: int = 0, rows: int = 0):
        """NEXT-3 (bt_set_record_peers): register_pairs also stores local pair p's record into row
        row_offset + p of every peer buffer (device addresses, e.g. symmetric-memory buffer_ptrs
        of the other ranks' gather buffers); an empty list turns it off."""
        ptrs = [int(x) for x in peer_ptrs]
        arr = (C.c_uint64 * max(1, len(ptrs)))(*ptrs)
        self._check(lib().bt_set_record_peers(self._h, len(ptrs), arr, int(row_offset), int(rows)),
                    "bt_set_record_peers")

    def profile(self, on: bool = True, only: str | None = None):
        """Bracket every kernel launch with CUDA events on its stream (bt_profile_enable); with
        `only` (a kernel name of profile_read) just that kernel's launches."""
        code = 1 if on else 0
        if on and only is not None:
            L = lib()
            names = [L.bt_profile_name(k).decode() for k in range(L.bt_profile_kernels())]
            code = 2 + names.index(only)
        self._check(lib().bt_profile_enable(self._h, code), "bt_profile_enable")

    def profile_read(self) -> dict:
        """{kernel name: (total ms, launches)} since the previous read (waits for the events)."""
        L = lib()
        out = {}
        for k in range(L.bt_profile_kernels()):
            ms = C.c_double()
            n = C.c_int64()
            self._check(L.bt_profile_read(self._h, k, C.byref(ms), C.byref(n)), "bt_profile_read")
            out[L.bt_profile_name(k).decode()] = (ms.value, n.value)
        return out

    def pose_graph_step(self, node_pose, pairs, records, n_max: int, new_pose, lambda_feat: float = 1.0,
                        lambda_dense: float = 1.0, fixed_node: int = 0, max_iter: int = 200, rel_tol: float = 1e-10,
                        precond: int = 1, delta=None, stats=None, stream=None):
        """One Gauss-Newton step of the pose graph from bt_register_pairs records
        (bt_pose_graph_step).  precond 0 = Jacobi, 1 = block-Jacobi."""
        prm = GraphParams(float(lambda_feat), float(lambda_dense), int(fixed_node), int(max_iter), float(rel_tol),
                          int(precond))
        self._check(lib().bt_pose_graph_step(self._h, int(node_pose.shape[0]), _ptr(node_pose), _ptr(pairs),
                                             int(pairs.shape[0]), _ptr(records), int(n_max), C.byref(prm),
                                             _ptr(new_pose), _ptr(delta), _ptr(stats), self._stream(stream)),
                    "bt_pose_graph_step")

    def relinearize(self, fb: FrameBatch, K, node_pose, pairs, eprm: EdgeParams, records, matches=None,
                    n_matches=None, stream=None):
        """Eq. (2) / Eq. (3) blocks of `records` at new node poses, C_ij reused: with the match
        lists of the last register_pairs (bt_relinearize), or with caller-kept lists
        `matches` [P][n_max][2] / `n_matches` [P] (bt_relinearize_matches)."""
        kp, mp = fb.keypoints(), fb.maps()
        Ki = intrinsics(K) if not isinstance(K, Intrinsics) else K
        if matches is None:
            self._check(lib().bt_relinearize(self._h, C.byref(kp), C.byref(mp), C.byref(Ki), _ptr(node_pose),
                                             _ptr(pairs), int(pairs.shape[0]), C.byref(eprm), _ptr(records),
                                             self._stream(stream)), "bt_relinearize")
        else:
            self._check(lib().bt_relinearize_matches(self._h, C.byref(kp), C.byref(mp), C.byref(Ki), _ptr(node_pose),
                                                     _ptr(pairs), int(pairs.shape[0]), _ptr(matches), _ptr(n_matches),
                                                     C.byref(eprm), _ptr(records), self._stream(stream)),
                        "bt_relinearize_matches")

    def copy_matches(self, matches, n_matches, stream=None):
        """The last register_pairs' match lists into caller buffers [P][n_max][2] / [P]
        (bt_copy_matches) — the C_ij cache a tracker keeps across frames."""
        self._check(lib().bt_copy_matches(self._h, int(matches.shape[0]), int(matches.shape[1]), _ptr(matches),
                                          _ptr(n_matches), self._stream(stream)), "bt_copy_matches")

    def estimate_normals(self, depth, K, normal, jump: float = 0.05, stream=None):
        """Normal map [F][H][W][3] from depth [F][H][W] (bt_estimate_normals; NEXT-4)."""
        F, H, W = (1,) + tuple(depth.shape) if depth.dim() == 2 else tuple(depth.shape)
        Ki = intrinsics(K) if not isinstance(K, Intrinsics) else K
        self._check(lib().bt_estimate_normals(self._h, _ptr(depth), int(F), int(W), int(H), C.byref(Ki),
                                              float(jump), _ptr(normal), self._stream(stream)), "bt_estimate_normals")

    def lift_keypoints(self, uv, desc_in, n_in, maps_fb: FrameBatch, K, out: FrameBatch, stream=None):
        """Raw detector output (uv [F][n_max][2], desc_in [F][n_max][128], n_in [F]) + the frames'
        depth / normal / mask maps (maps_fb) -> the registration inputs out.n_kp / desc / pts /
        nrm (bt_lift_keypoints; NEXT-4, reading R29)."""
        F, n_max, dim = (int(x) for x in desc_in.shape)
        mp = maps_fb.maps()
        Ki = intrinsics(K) if not isinstance(K, Intrinsics) else K
        self._check(lib().bt_lift_keypoints(self._h, F, n_max, dim, _ptr(uv), _ptr(desc_in), _ptr(n_in), C.byref(mp),
                                            C.byref(Ki), _ptr(out.n_kp), _ptr(out.desc), _ptr(out.pts),
                                            _ptr(out.nrm), self._stream(stream)), "bt_lift_keypoints")

    # ---- NEXT-2: the tracker's per-frame decisions (device-resident pool, P:25 / P:39 / P:88)
    def coarse_pose(self, record, prev, out, stream=None):
        """out = T_best(record) . prev, or prev when the pair has no hypothesis (bt_coarse_pose)."""
        self._check(lib().bt_coarse_pose(self._h, _ptr(record), _ptr(prev), _ptr(out), self._stream(stream)),
                    "bt_coarse_pose")

    def select_keyframes(self, pool, n_pool, cur, K, sel, n_sel, stream=None):
        """Greedy selection of P:39 over pool[0 .. n_pool) (device int) -> sel [K], n_sel [1]."""
        self._check(lib().bt_select_keyframes(self._h, _ptr(pool), _ptr(n_pool), int(pool.shape[0]), _ptr(cur), int(K),
                                              _ptr(sel), _ptr(n_sel), self._stream(stream)), "bt_select_keyframes")

    def pool_admit(self, pool, n_pool, cur, thresh_rad, admitted=None, stream=None):
        """cur joins the pool iff its rotation is > thresh from every keyframe (bt_pool_admit)."""
        self._check(lib().bt_pool_admit(self._h, _ptr(pool), _ptr(n_pool), int(pool.shape[0]), _ptr(cur),
                                        float(thresh_rad), _ptr(admitted), self._stream(stream)), "bt_pool_admit")

    def compose_poses(self, a, b, out, stream=None):
        self._check(lib().bt_compose_poses(self._h, _ptr(a), _ptr(b), _ptr(out), int(a.shape[0]),
                                           self._stream(stream)), "bt_compose_poses")


def decode_records(records, n_max: int) -> dict:
    """Split a [P][record_words] uint32 array (numpy or tensor) into named fields."""
    r = records.cpu().numpy() if hasattr(records, "cpu") else np.asarray(records)
    r = r.view(np.uint32).reshape(r.shape[0], -1)
    W = mask_words(n_max)
    f = r.view(np.float32)
    i = r.view(np.int32)
    o = 28 + W
    return dict(status=i[:, 0].copy(), n_matches=i[:, 1].copy(), best_hyp=i[:, 2].copy(),
                best_count=i[:, 3].copy(), T_best=f[:, 4:16].copy(), T_refit=f[:, 16:28].copy(),
                mask=r[:, 28:28 + W].copy(), dense_ij=f[:, o:o + 32].copy(), dense_ji=f[:, o + 32:o + 64].copy(),
                feat=f[:, o + 64:o + 160].copy())
