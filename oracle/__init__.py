"""CPU oracle (TEST INFRASTRUCTURE ONLY) — ctypes wrapper around oracle/bt_oracle.c.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
may import this package.  The product path (paper_2108_00516_b200) never does; it fails
loudly when its CUDA library is missing.

Everything here is marshalling: the arithmetic lives in bt_oracle.c (plain C, double),
written from PAPER.md (arXiv 2108.00516) §IV-B and §IV-D Eq. (2)/(3).
Functions with no independent pin: none (see tests/test_oracle_*.py and DESIGN.md §4).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "bt_oracle.c")
_HDR = os.path.join(_HERE, "bt_oracle.h")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

STATUS_OK, STATUS_FEW_MATCHES, STATUS_FEW_INLIERS, STATUS_REFIT_DEGENERATE = 0, 1, 2, 3


def build(force: bool = False) -> str:
    """Compile the oracle (gcc, -O2, no fast-math)."""
    stale = not os.path.exists(_LIB) or any(
        os.path.getmtime(p) > os.path.getmtime(_LIB) for p in (_SRC, _HDR))
    if force or stale:
        subprocess.check_call(["gcc", "-std=c99", "-O2", "-fPIC", "-shared", "-o", _LIB, _SRC, "-lm"])
    return _LIB


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        _setup(_lib)
    return _lib


_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_vp = C.c_void_p


class PairResult(C.Structure):
    _fields_ = [("status", C.c_int32), ("n_matches", C.c_int32), ("best_hyp", C.c_int32),
                ("best_count", C.c_int32), ("T_best", C.c_double * 12),
                ("T_refit", C.c_double * 12), ("refit_sig_ratio", C.c_double)]


def _setup(L):
    L.bto_philox4x32_10.argtypes = [_u32p, _u32p, _u32p]
    L.bto_triple.argtypes = [_u32p, C.c_int32, _i32p]
    L.bto_match.restype = C.c_int32
    L.bto_match.argtypes = [_f32p, C.c_int32, _f32p, C.c_int32, C.c_int32, C.c_double,
                            _i32p, _i32p, _i32p, _u8p, _u8p, _vp]
    L.bto_arun.argtypes = [_f64p, _f64p, C.c_int32, _f64p, _f64p, C.POINTER(C.c_double)]
    L.bto_svd3.argtypes = [_f64p, _f64p, _f64p, _f64p]
    L.bto_ransac_counts.argtypes = [_f32p, _f32p, _f32p, _f32p, C.c_int32, C.c_int32, C.c_uint32,
                                    C.c_uint64, C.c_double, C.c_double, C.c_double,
                                    _i32p, _i32p, _i32p, _vp, _vp]
    L.bto_inliers.restype = C.c_int32
    L.bto_inliers.argtypes = [_f64p, _f32p, _f32p, _f32p, _f32p, C.c_int32, C.c_double, C.c_double,
                              _vp, _vp]
    L.bto_ransac_finish.argtypes = [_f32p, _f32p, _f32p, _f32p, C.c_int32, C.c_int32, _i32p, _f64p,
                                    C.c_double, C.c_double, C.c_double, C.c_int32,
                                    C.POINTER(PairResult), _vp]
    L.bto_huber.argtypes = [C.c_double, C.c_double, C.POINTER(C.c_double), C.POINTER(C.c_double)]
    L.bto_feature_edge.argtypes = [_f32p, _f32p, _u32p, C.c_int32, _f32p, _f32p, C.c_double, _f64p]
    L.bto_dense_edge.argtypes = [_f32p, _f32p, _u8p, _f32p, _f32p, _u8p, C.c_int32, C.c_int32,
                                 C.c_double, C.c_double, C.c_double, C.c_double, _f32p, _f32p,
                                 C.c_double, C.c_double, C.c_double, C.c_int32, _f64p, _vp, _vp, _vp]
    L.bto_estimate_normals.argtypes = [_f32p, C.c_int32, C.c_int32, C.c_int32, C.c_double, C.c_double, C.c_double,
                                       C.c_double, C.c_float, _f32p]
    L.bto_lift_keypoints.argtypes = [C.c_int32, C.c_int32, C.c_int32, _f32p, _f32p, _vp, _f32p, _f32p, _u8p,
                                     C.c_int32, C.c_int32, C.c_double, C.c_double, C.c_double, C.c_double, _vp,
                                     _f32p, _f32p, _f32p, _vp]
    L.bto_se3_exp.argtypes = [_f64p, _f64p, _f64p]
    L.bto_se3_adjoint.argtypes = [_f64p, _f64p, _f64p]
    L.bto_graph_system.restype = C.c_int32
    L.bto_graph_system.argtypes = [C.c_int32, _f32p, _i32p, C.c_int32, _f64p, _vp, _vp, _vp, C.c_double, C.c_double,
                                   _f64p, _f64p, _f64p]
    L.bto_graph_step.restype = C.c_int32
    L.bto_graph_step.argtypes = [C.c_int32, _f32p, _i32p, C.c_int32, _f64p, _vp, _vp, _vp, C.c_double, C.c_double,
                                 C.c_int32, _f64p, _f32p, _f64p]


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


# ------------------------------------------------------------------------------ sampler
def philox(ctr, key) -> np.ndarray:
    out = np.zeros(4, np.uint32)
    lib().bto_philox4x32_10(_c(ctr, np.uint32), _c(key, np.uint32), out)
    return out


def triple(r, M: int) -> np.ndarray:
    out = np.zeros(3, np.int32)
    lib().bto_triple(_c(r, np.uint32), int(M), out)
    return out


# ----------------------------------------------------------------------------- matching
def match(A, B, ratio: float = 1.0):
    """Mutual NN of descriptor sets A [na][dim], B [nb][dim] (float32)."""
    A = _c(A, np.float32)
    B = _c(B, np.float32)
    na, nb = len(A), len(B)
    dim = A.shape[1] if A.ndim == 2 and na else (B.shape[1] if B.ndim == 2 and nb else 128)
    pairs = np.zeros((max(min(na, nb), 1), 2), np.int32)
    nn_ab = np.zeros(max(na, 1), np.int32)
    nn_ba = np.zeros(max(nb, 1), np.int32)
    rb = np.zeros(max(na, 1), np.uint8)
    cb = np.zeros(max(nb, 1), np.uint8)
    dbest = np.zeros(max(na, 1), np.float64)
    M = lib().bto_match(A.reshape(-1) if na else np.zeros(1, np.float32), na,
                        B.reshape(-1) if nb else np.zeros(1, np.float32), nb, dim, float(ratio),
                        pairs, nn_ab, nn_ba, rb, cb, _ptr(dbest))
    return dict(pairs=pairs[:M].copy(), nn_ab=nn_ab[:na], nn_ba=nn_ba[:nb],
                row_border=rb[:na].astype(bool), col_border=cb[:nb].astype(bool), d_best=dbest[:na])


# ------------------------------------------------------------------------- least squares
def svd3(A):
    U = np.zeros(9)
    s = np.zeros(3)
    V = np.zeros(9)
    lib().bto_svd3(_c(np.asarray(A).reshape(9), np.float64), U, s, V)
    return U.reshape(3, 3), s, V.reshape(3, 3)


def arun(pa, pb):
    pa = _c(pa, np.float64).reshape(-1, 3)
    pb = _c(pb, np.float64).reshape(-1, 3)
    R = np.zeros(9)
    t = np.zeros(3)
    sig = C.c_double()
    lib().bto_arun(pa.reshape(-1), pb.reshape(-1), len(pa), R, t, C.byref(sig))
    return R.reshape(3, 3), t, sig.value


# ---------------------------------------------------------------------------------- RANSAC
def ransac_counts(pa, na, pb, nb, n_hyp: int, pair_uid: int, seed: int, delta=0.005,
                  cos_alpha=float(np.cos(np.deg2rad(45.0))), tau=1e-3):
    pa, na, pb, nb = (_c(x, np.float32).reshape(-1) for x in (pa, na, pb, nb))
    M = len(pa) // 3
    cnt = np.zeros(n_hyp, np.int32)
    lo = np.zeros(n_hyp, np.int32)
    hi = np.zeros(n_hyp, np.int32)
    hyp = np.zeros((n_hyp, 12), np.float64)
    tri = np.zeros((n_hyp, 3), np.int32)
    z = np.zeros(3, np.float32)
    lib().bto_ransac_counts(pa if M else z, na if M else z, pb if M else z, nb if M else z, M, n_hyp,
                            int(pair_uid) & 0xffffffff, int(seed) & 0xffffffffffffffff,
                            float(delta), float(cos_alpha), float(tau), cnt, lo, hi, _ptr(hyp), _ptr(tri))
    return dict(cnt=cnt, lo=lo, hi=hi, hyp=hyp, tri=tri)


def inliers(T12, pa, na, pb, nb, delta=0.005, cos_alpha=float(np.cos(np.deg2rad(45.0)))):
    pa, na, pb, nb = (_c(x, np.float32).reshape(-1) for x in (pa, na, pb, nb))
    M = len(pa) // 3
    mask = np.zeros(max((M + 31) // 32, 1), np.uint32)
    border = np.zeros(max(M, 1), np.uint8)
    z = np.zeros(3, np.float32)
    n = lib().bto_inliers(_c(T12, np.float64), pa if M else z, na if M else z, pb if M else z,
                          nb if M else z, M, float(delta), float(cos_alpha), _ptr(mask), _ptr(border))
    return n, mask, border[:M].astype(bool)


def ransac_finish(pa, na, pb, nb, counts, delta=0.005, cos_alpha=float(np.cos(np.deg2rad(45.0))),
                  tau=1e-3, min_inliers=3):
    pa, na, pb, nb = (_c(x, np.float32).reshape(-1) for x in (pa, na, pb, nb))
    M = len(pa) // 3
    res = PairResult()
    mask = np.zeros(max((M + 31) // 32, 1), np.uint32)
    z = np.zeros(3, np.float32)
    H = len(counts["cnt"])
    lib().bto_ransac_finish(pa if M else z, na if M else z, pb if M else z, nb if M else z, M, H,
                            _c(counts["cnt"], np.int32), _c(counts["hyp"], np.float64).reshape(-1),
                            float(delta), float(cos_alpha), float(tau), int(min_inliers),
                            C.byref(res), _ptr(mask))
    return dict(status=res.status, n_matches=res.n_matches, best_hyp=res.best_hyp,
                best_count=res.best_count, T_best=np.array(res.T_best[:]),
                T_refit=np.array(res.T_refit[:]), refit_sig_ratio=res.refit_sig_ratio, mask=mask)


def huber(r: float, delta: float):
    rho = C.c_double()
    w = C.c_double()
    lib().bto_huber(float(r), float(delta), C.byref(rho), C.byref(w))
    return rho.value, w.value


# ------------------------------------------------------------------------------- edges
def feature_edge(pa, pb, mask, Ti, Tj, huber_delta=0.005) -> np.ndarray:
    pa = _c(pa, np.float32).reshape(-1)
    pb = _c(pb, np.float32).reshape(-1)
    M = len(pa) // 3
    out = np.zeros(186)
    mk = _c(mask, np.uint32) if M else np.zeros(1, np.uint32)
    z = np.zeros(3, np.float32)
    lib().bto_feature_edge(pa if M else z, pb if M else z, mk, M, _c(Ti, np.float32),
                           _c(Tj, np.float32), float(huber_delta), out)
    return out


def dense_edge(depth_i, normal_i, mask_i, depth_j, normal_j, mask_j, K, Ti, Tj, dist_gate=0.02,
               cos_gate=float(np.cos(np.deg2rad(45.0))), huber_delta=0.005, stride=1,
               want_pixels=False, want_allow=False):
    """Eq. (3) edge i -> j (bto_dense_edge).  Returns out[72]; with want_pixels also the per-pixel
    association [H][W] (target index or -1) and borderline flags; with want_allow also the
    per-pixel allowance [H][W][8] of the borderline pixels."""
    H, W = np.asarray(depth_i).shape
    out = np.zeros(72)
    pix = np.zeros(H * W, np.int32) if want_pixels else None
    pbd = np.zeros(H * W, np.uint8) if want_pixels else None
    pal = np.zeros(H * W * 8) if want_allow else None
    lib().bto_dense_edge(_c(depth_i, np.float32).reshape(-1), _c(normal_i, np.float32).reshape(-1),
                         _c(mask_i, np.uint8).reshape(-1), _c(depth_j, np.float32).reshape(-1),
                         _c(normal_j, np.float32).reshape(-1), _c(mask_j, np.uint8).reshape(-1),
                         W, H, float(K.fx), float(K.fy), float(K.cx), float(K.cy),
                         _c(Ti, np.float32), _c(Tj, np.float32), float(dist_gate), float(cos_gate),
                         float(huber_delta), int(stride), out, _ptr(pix), _ptr(pbd), _ptr(pal))
    res = (out,)
    if want_pixels:
        res += (pix.reshape(H, W), pbd.reshape(H, W).astype(bool))
    if want_allow:
        res += (pal.reshape(H, W, 8),)
    return res if len(res) > 1 else out


# --------------------------------------------------------------- whole pair registration
def register_pair(scene, a: int, b: int, uid: int, n_hyp: int, seed: int, node_poses=None,
                  delta=0.005, cos_alpha=float(np.cos(np.deg2rad(45.0))), tau=1e-3, min_inliers=3,
                  ratio=1.0, huber_delta=0.005, dense=None, counts_out=False):
    """The whole hot path for one frame pair (a, b), step by step in the paper's order:
    match -> RANSAC counts -> best + refit -> Eq. (2) blocks -> Eq. (3)
    blocks of both directed edges.  `dense` = dict(dist_gate, cos_gate, huber_delta,
    stride) or None to skip the dense edges."""
    na_, nb_ = int(scene.n_kp[a]), int(scene.n_kp[b])
    mt = match(scene.desc[a, :na_], scene.desc[b, :nb_], ratio)
    P = mt["pairs"]
    ia, ib = P[:, 0], P[:, 1]
    pa, pb = scene.pts[a][ia], scene.pts[b][ib]
    nra, nrb = scene.nrm[a][ia], scene.nrm[b][ib]
    cnt = ransac_counts(pa, nra, pb, nrb, n_hyp, uid, seed, delta, cos_alpha, tau)
    fin = ransac_finish(pa, nra, pb, nrb, cnt, delta, cos_alpha, tau, min_inliers)
    rec = dict(match=mt, counts=cnt if counts_out else None, **fin)
    if node_poses is not None:
        rec["feat"] = feature_edge(pa, pb, fin["mask"], node_poses[a], node_poses[b], huber_delta)
        if dense is not None:
            rec["dense_ij"] = dense_edge(scene.depth[a], scene.normal[a], scene.mask[a], scene.depth[b],
                                         scene.normal[b], scene.mask[b], scene.K, node_poses[a],
                                         node_poses[b], **dense)
            rec["dense_ji"] = dense_edge(scene.depth[b], scene.normal[b], scene.mask[b], scene.depth[a],
                                         scene.normal[a], scene.mask[a], scene.K, node_poses[b],
                                         node_poses[a], **dense)
    return rec


# ------------------------------------------------------------ NEXT-1: pose-graph GN step
def se3_exp(xi):
    """SE(3) exponential of a (v, w) twist -> (R [3][3], t [3]) (PAPER.md P:83 T = exp(xi))."""
    R = np.zeros(9)
    t = np.zeros(3)
    lib().bto_se3_exp(_c(xi, np.float64), R, t)
    return R.reshape(3, 3), t


def se3_adjoint(R, t):
    """6x6 adjoint of T = (R, t) on (v, w) twists: exp(Adj d) T = T exp(d)."""
    A = np.zeros(36)
    lib().bto_se3_adjoint(_c(R, np.float64).reshape(-1), _c(t, np.float64), A)
    return A.reshape(6, 6)


def _graph_inputs(poses, pairs, feat, dense_ij, dense_ji):
    poses = _c(poses, np.float32).reshape(-1, 12)
    pairs = _c(pairs, np.int32).reshape(-1, 2)
    feat = _c(feat, np.float64).reshape(len(pairs), -1)[:, :96]
    feat = _c(feat, np.float64)
    dij = None if dense_ij is None else _c(_c(dense_ij, np.float64).reshape(len(pairs), -1)[:, :32], np.float64)
    dji = None if dense_ji is None else _c(_c(dense_ji, np.float64).reshape(len(pairs), -1)[:, :32], np.float64)
    return poses, pairs, feat, dij, dji


def graph_system(poses, pairs, feat, dense_ij=None, dense_ji=None, lambda_f=1.0, lambda_g=1.0, status=None):
    """Gauss-Newton system of Eq. (1) from per-pair Eq. (2) blocks feat[P][96] and
    the Eq. (3) blocks of both directed edges [P][32] at node poses [N][12]: (A, b, (E_f, E_g)).
    status [P] (optional): pairs with status 1 / 2 (failed registration) bring no Eq. (2) term."""
    st_ = None if status is None else _c(status, np.int32)
    poses, pairs, feat, dij, dji = _graph_inputs(poses, pairs, feat, dense_ij, dense_ji)
    n = 6 * len(poses)
    A = np.zeros(n * n)
    b = np.zeros(n)
    e = np.zeros(2)
    st = lib().bto_graph_system(len(poses), poses, pairs.reshape(-1), len(pairs), feat.reshape(-1), _ptr(dij),
                                _ptr(dji), _ptr(st_), float(lambda_f), float(lambda_g), A, b, e)
    if st != 0:
        raise ValueError("bad pair list")
    return A.reshape(n, n), b, tuple(e)


def graph_step(poses, pairs, feat, dense_ij=None, dense_ji=None, lambda_f=1.0, lambda_g=1.0, fixed_node=0,
               status=None):
    """One Gauss-Newton step: solve A d = -b (Cholesky; the fixed node's and
    unconstrained DOFs pinned), T_i <- exp(d_i) T_i.  Returns (delta [N][6], poses [N][12],
    (E_f, E_g) at the input poses).  status: as graph_system."""
    st_ = None if status is None else _c(status, np.int32)
    poses, pairs, feat, dij, dji = _graph_inputs(poses, pairs, feat, dense_ij, dense_ji)
    N = len(poses)
    d = np.zeros(6 * N)
    out = np.zeros(12 * N, np.float32)
    e = np.zeros(2)
    st = lib().bto_graph_step(N, poses, pairs.reshape(-1), len(pairs), feat.reshape(-1), _ptr(dij), _ptr(dji),
                              _ptr(st_), float(lambda_f), float(lambda_g), int(fixed_node), d, out, e)
    if st != 0:
        raise np.linalg.LinAlgError("pose-graph system not positive definite")
    return d.reshape(N, 6), out.reshape(N, 12), tuple(e)


# ------------------------------------------------------------ NEXT-4: normals from depth
def estimate_normals(depth, K, jump: float = 0.05) -> np.ndarray:
    """Normal map [F][H][W][3] from depth [F][H][W] (or [H][W]) by central differences of the
    unprojected cloud, camera-facing, 5 cm jump test (SPEC estimate_normals S:157-165)."""
    d = _c(depth, np.float32)
    squeeze = d.ndim == 2
    if squeeze:
        d = d[None]
    F, H, W = d.shape
    out = np.zeros((F, H, W, 3), np.float32)
    lib().bto_estimate_normals(d.reshape(-1), F, W, H, float(K.fx), float(K.fy), float(K.cx), float(K.cy),
                               float(jump), out.reshape(-1))
    return out[0] if squeeze else out


# ------------------------------------------------------------ NEXT-4: keypoint lifting
def lift_keypoints(uv, desc, n_in, depth, normal, mask, K):
    """The keypoints' 3-D points and normals from their pixels (bto_lift_keypoints, reading R29;
    P:25, P:72 pi_D^-1): uv [F][n_max][2], desc [F][n_max][dim], n_in [F]; maps
    [F][H][W](.., 3).  Returns dict(n [F], desc, pts, nrm [F][n_max][..] (rows >= n zero),
    border [F][n_max] bool)."""
    uv = _c(uv, np.float32)
    desc = _c(desc, np.float32)
    F, n_max, dim = desc.shape
    depth = _c(depth, np.float32)
    Fd, H, W = depth.shape
    n_out = np.zeros(F, np.int32)
    od = np.zeros_like(desc)
    pts = np.zeros((F, n_max, 3), np.float32)
    nrm = np.zeros((F, n_max, 3), np.float32)
    bd = np.zeros((F, n_max), np.uint8)
    lib().bto_lift_keypoints(F, n_max, dim, uv.reshape(-1), desc.reshape(-1), _ptr(_c(n_in, np.int32)),
                             depth.reshape(-1), _c(normal, np.float32).reshape(-1), _c(mask, np.uint8).reshape(-1),
                             W, H, float(K.fx), float(K.fy), float(K.cx), float(K.cy), _ptr(n_out), od.reshape(-1),
                             pts.reshape(-1), nrm.reshape(-1), _ptr(bd))
    return dict(n=n_out, desc=od, pts=pts, nrm=nrm, border=bd.astype(bool))


# ------------------------------------------------------------ NEXT-2: tracker decisions
def _setup_track(L):
    L.bto_rot_geodesic.argtypes = [_f32p, _f32p]
    L.bto_rot_geodesic.restype = C.c_double
    L.bto_coarse_pose.argtypes = [C.c_int32, _f32p, _f32p, _f32p]
    L.bto_select_keyframes.argtypes = [_f32p, C.c_int32, _f32p, C.c_int32, _vp]
    L.bto_select_keyframes.restype = C.c_int32
    L.bto_is_novel.argtypes = [_f32p, C.c_int32, _f32p, C.c_double]
    L.bto_is_novel.restype = C.c_int32
    return L


def rot_geodesic(Ta, Tb) -> float:
    """arccos((tr(R_a^T R_b) - 1) / 2)."""
    return float(_setup_track(lib()).bto_rot_geodesic(_c(Ta, np.float32).reshape(-1), _c(Tb, np.float32).reshape(-1)))


def coarse_pose(status: int, T_best, T_prev) -> np.ndarray:
    """T~_t = T_rel . T_prev with T_rel the best sampled hypothesis (reading R13); T_prev
    when the pair has none (status FEW_MATCHES / FEW_INLIERS)."""
    out = np.zeros(12, np.float32)
    _setup_track(lib()).bto_coarse_pose(int(status), _c(T_best, np.float32).reshape(-1),
                                        _c(T_prev, np.float32).reshape(-1), out)
    return out


def select_keyframes(pool, cur, K: int) -> np.ndarray:
    """Greedy keyframe selection of P:39 over pool poses [N][12] for the current pose: pool
    indices in selection order (I_0 first)."""
    pool = _c(pool, np.float32).reshape(-1, 12)
    sel = np.zeros(max(K, 1), np.int32)
    n = _setup_track(lib()).bto_select_keyframes(pool.reshape(-1) if len(pool) else np.zeros(12, np.float32),
                                                 len(pool), _c(cur, np.float32).reshape(-1), int(K), _ptr(sel))
    return sel[:n]


def is_novel(pool, cur, thresh_rad=float(np.deg2rad(10.0))) -> bool:
    """the current pose is farther than thresh from every pool keyframe (rotation geodesic)."""
    pool = _c(pool, np.float32).reshape(-1, 12)
    return bool(_setup_track(lib()).bto_is_novel(pool.reshape(-1) if len(pool) else np.zeros(12, np.float32),
                                                 len(pool), _c(cur, np.float32).reshape(-1), float(thresh_rad)))
