"""Seeded synthetic RGB-D / keypoint workloads shaped like BundleTrack's (arXiv 2108.00516).

This module is the ONE piece shared by the CUDA path's tests/bench and by the CPU
oracle: it produces inputs only and holds none of the method's arithmetic (no matching,
no RANSAC, no least squares, no point-to-plane residuals).  The recipe is stated in
DESIGN.md §3 ("input recipe"):

* object: an analytic ellipsoid (semi-axes 11 x 8 x 6 cm) in its own frame; depth,
  normal and mask maps are exact analytic ray casts (SPEC.md synth_oracle idea);
* poses: object->camera T = (R, t), x_cam = R x_obj + t ("object pose in
  the camera's frame");
* keypoints: a global pool of surface points with a fixed "detector score"; each frame
  keeps the n best-scored visible pool points (n = 500, "n is 500 in all
  experiments"), with 128-d unit descriptors ("D_i in R^128") = normalize(global
  descriptor + 0.03 N(0, I));
* outliers: a fraction of each frame's keypoints carries the descriptor of a different
  pool point at least 5 cm away (10 x delta, delta = 5 mm of P:25), so that matching them
  produces geometric outliers ("outlier keypoints can arise").

Everything is float32 at the boundary, the layout the C ABI (include/bt.h) takes.
"""
from __future__ import annotations

import dataclasses
import numpy as np

DATA_SEED = 210800516
PHILOX_SEED = 0x0123456789ABCDEF

AXES = (0.11, 0.08, 0.06)          # ellipsoid semi-axes, metres


# ----------------------------------------------------------------------------------------
# small rigid-body helpers used only to POSE the synthetic scene
# ----------------------------------------------------------------------------------------
def rotvec_to_R(w: np.ndarray) -> np.ndarray:
    w = np.asarray(w, dtype=np.float64)
    th = float(np.linalg.norm(w))
    if th < 1e-12:
        return np.eye(3)
    k = w / th
    K = np.array([[0, -k[2], k[1]], [k[2], 0, -k[0]], [-k[1], k[0], 0]])
    return np.eye(3) + np.sin(th) * K + (1 - np.cos(th)) * (K @ K)


def random_rotation(rng: np.random.Generator, max_angle: float) -> np.ndarray:
    axis = rng.normal(size=3)
    axis /= np.linalg.norm(axis)
    return rotvec_to_R(axis * rng.uniform(0, max_angle))


def geodesic(Ra: np.ndarray, Rb: np.ndarray) -> float:
    c = (np.trace(Ra.T @ Rb) - 1.0) / 2.0
    return float(np.arccos(np.clip(c, -1.0, 1.0)))


def pose12(R: np.ndarray, t: np.ndarray) -> np.ndarray:
    """bt_pose layout: R row-major (9) then t (3), float32."""
    return np.concatenate([np.asarray(R).reshape(9), np.asarray(t).reshape(3)]).astype(np.float32)


# ----------------------------------------------------------------------------------------
# the object: an ellipsoid
# ----------------------------------------------------------------------------------------
def ellipsoid_normal(x: np.ndarray, axes=AXES) -> np.ndarray:
    a = np.asarray(axes)
    g = x / (a * a)
    return g / np.linalg.norm(g, axis=-1, keepdims=True)


def sample_surface(rng: np.random.Generator, n: int, axes=AXES, min_spacing: float | None = None) -> np.ndarray:
    """n points on the ellipsoid, roughly area-uniform, pairwise >= min_spacing apart (dart
    throwing with a grid hash).  Default spacing: 0.6 * sqrt(area / n), always satisfiable."""
    a = np.asarray(axes)
    if min_spacing is None:
        p = 1.6075                                         # Knud Thomsen's surface-area formula
        area = 4 * np.pi * ((a[0] ** p * a[1] ** p + a[0] ** p * a[2] ** p + a[1] ** p * a[2] ** p) / 3) ** (1 / p)
        min_spacing = min(0.004, 0.6 * np.sqrt(area / n))
    cell = min_spacing
    grid: dict = {}
    pts = []
    s2 = min_spacing ** 2
    while len(pts) < n:
        u = rng.normal(size=(4 * n, 3))
        u /= np.linalg.norm(u, axis=1, keepdims=True)
        w = np.linalg.norm(u / a, axis=1)              # area element ~ abc * |u/a|
        keep = rng.uniform(0, w.max(), size=len(w)) < w
        for c in u[keep] * a:
            key = tuple(np.floor(c / cell).astype(int))
            ok = True
            for dx in (-1, 0, 1):
                for dy in (-1, 0, 1):
                    for dz in (-1, 0, 1):
                        for q in grid.get((key[0] + dx, key[1] + dy, key[2] + dz), ()):
                            if (q[0] - c[0]) ** 2 + (q[1] - c[1]) ** 2 + (q[2] - c[2]) ** 2 < s2:
                                ok = False
                                break
                        if not ok:
                            break
                    if not ok:
                        break
                if not ok:
                    break
            if ok:
                grid.setdefault(key, []).append(c)
                pts.append(c)
                if len(pts) == n:
                    break
    return np.array(pts)


@dataclasses.dataclass
class Intrinsics:
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int


def render(R: np.ndarray, t: np.ndarray, K: Intrinsics, axes=AXES):
    """Analytic ray cast of the posed ellipsoid.  Returns depth [H][W] f32 (z, metres,
    0 = no surface), normal [H][W][3] f32 (camera frame, unit, 0 = invalid), mask u8."""
    W, H = K.width, K.height
    u, v = np.meshgrid(np.arange(W, dtype=np.float64), np.arange(H, dtype=np.float64))
    d = np.stack([(u - K.cx) / K.fx, (v - K.cy) / K.fy, np.ones_like(u)], axis=-1)   # z = 1 rays
    a = np.asarray(axes)
    o = -(R.T @ t)                       # camera centre in the object frame
    dd = d @ R                           # R^T d per pixel
    A = np.sum((dd / a) ** 2, axis=-1)
    B = 2 * np.sum(dd * o / (a * a), axis=-1)
    C = np.sum((o / a) ** 2) - 1.0
    disc = B * B - 4 * A * C
    hit = disc > 0
    s = np.where(hit, (-B - np.sqrt(np.maximum(disc, 0))) / (2 * A), 0.0)
    hit &= s > 0
    depth = np.where(hit, s, 0.0)                      # ray has d_z = 1, so s = z
    xo = o + s[..., None] * dd                         # hit point, object frame
    n_obj = ellipsoid_normal(np.where(hit[..., None], xo, 1.0), axes)
    n_cam = n_obj @ R.T
    normal = np.where(hit[..., None], n_cam, 0.0)
    return depth.astype(np.float32), normal.astype(np.float32), hit.astype(np.uint8)


# ----------------------------------------------------------------------------------------
# a multi-frame scene
# ----------------------------------------------------------------------------------------
@dataclasses.dataclass
class Scene:
    K: Intrinsics
    poses_R: np.ndarray          # [F][3][3] float64 ground truth
    poses_t: np.ndarray          # [F][3]
    n_kp: np.ndarray             # [F] int32
    desc: np.ndarray             # [F][n_max][128] f32
    pts: np.ndarray              # [F][n_max][3] f32 camera frame
    nrm: np.ndarray              # [F][n_max][3] f32 camera frame
    kp_pool: np.ndarray          # [F][n_max] int32: pool id whose POSITION the keypoint has (-1 pad)
    kp_desc_src: np.ndarray      # [F][n_max] int32: pool id whose DESCRIPTOR it carries
    depth: np.ndarray | None     # [F][H][W] f32
    normal: np.ndarray | None    # [F][H][W][3] f32
    mask: np.ndarray | None      # [F][H][W] u8

    @property
    def n_frames(self) -> int:
        return len(self.n_kp)

    def node_poses(self) -> np.ndarray:
        return np.stack([pose12(R, t) for R, t in zip(self.poses_R, self.poses_t)])

    def perturbed_poses(self, seed: int, rot_deg: float = 5.0, trans_m: float = 0.02,
                        fixed: int = 0) -> np.ndarray:
        """Node poses perturbed by <= rot_deg / trans_m, node `fixed` left exact."""
        rng = np.random.default_rng(seed)
        out = []
        for f, (R, t) in enumerate(zip(self.poses_R, self.poses_t)):
            if f == fixed:
                out.append(pose12(R, t))
                continue
            dR = random_rotation(rng, np.deg2rad(rot_deg))
            dt = rng.normal(size=3)
            dt *= rng.uniform(0, trans_m) / np.linalg.norm(dt)
            out.append(pose12(dR @ R, t + dt))          # rotate about the object origin
        return np.stack(out)


def make_scene(n_frames: int, n: int = 500, n_max: int = 512, width: int = 640, height: int = 480,
               seed: int = DATA_SEED, outlier_frac: float = 0.16, pool_size: int = 2000,
               desc_noise: float = 0.03, point_noise: float = 0.0, distance: float = 0.5,
               cone_deg: float = 60.0, min_geodesic_deg: float = 10.0, render_maps: bool = True,
               focal: float = 600.0, poses=None) -> Scene:
    """BundleTrack-shaped multi-view scene: node poses of one object seen from n_frames
    views inside a +-cone_deg cone whose pairwise rotation geodesics are >= 10 deg (the
    memory-pool novelty rule)."""
    rng = np.random.default_rng(seed)
    K = Intrinsics(focal, focal, (width - 1) / 2.0, (height - 1) / 2.0, width, height)
    pool = sample_surface(rng, pool_size)
    pool_n = ellipsoid_normal(pool)
    gdesc = rng.normal(size=(pool_size, 128))
    gdesc /= np.linalg.norm(gdesc, axis=1, keepdims=True)
    score = rng.uniform(size=pool_size)                      # fixed "detector response"
    R0 = rotvec_to_R(np.array([0.3, -0.5, 0.2]))

    Rs, ts = [], []
    if poses is not None:                                    # given (R, t) per frame (trajectories)
        Rs = [np.asarray(R, np.float64) for R, _ in poses]
        ts = [np.asarray(t, np.float64) for _, t in poses]
    tries = 0
    while len(Rs) < n_frames:
        tries += 1
        R = random_rotation(rng, np.deg2rad(cone_deg)) @ R0 if Rs else R0
        if all(geodesic(R, Q) >= np.deg2rad(min_geodesic_deg) for Q in Rs) or tries > 20000:
            Rs.append(R)
            ts.append(np.array([rng.uniform(-0.02, 0.02), rng.uniform(-0.02, 0.02),
                                distance + rng.uniform(-0.03, 0.03)]))
    F = n_frames
    n_kp = np.zeros(F, np.int32)
    desc = np.zeros((F, n_max, 128), np.float32)
    pts = np.zeros((F, n_max, 3), np.float32)
    nrm = np.zeros((F, n_max, 3), np.float32)
    kp_pool = -np.ones((F, n_max), np.int32)
    kp_src = -np.ones((F, n_max), np.int32)
    for f in range(F):
        R, t = Rs[f], ts[f]
        pc = pool @ R.T + t
        nc = pool_n @ R.T
        uvz = pc[:, 2]
        u = K.fx * pc[:, 0] / uvz + K.cx
        v = K.fy * pc[:, 1] / uvz + K.cy
        vis = (np.sum(nc * pc, axis=1) < -0.2 * np.linalg.norm(pc, axis=1)) & \
              (u >= 0) & (u <= width - 1) & (v >= 0) & (v <= height - 1)
        ids = np.nonzero(vis)[0]
        jitter = score[ids] + 0.05 * rng.uniform(size=len(ids))
        ids = ids[np.argsort(-jitter, kind="stable")][:n]
        rng.shuffle(ids)
        m = len(ids)
        n_kp[f] = m
        src = ids.copy()
        n_out = int(round(outlier_frac * m))
        for k in rng.choice(m, size=n_out, replace=False):
            far = np.nonzero(np.linalg.norm(pool - pool[ids[k]], axis=1) >= 0.05)[0]
            src[k] = far[rng.integers(len(far))]
        obs = gdesc[src] + desc_noise * rng.normal(size=(m, 128))
        obs /= np.linalg.norm(obs, axis=1, keepdims=True)
        desc[f, :m] = obs
        p = pc[ids] + (point_noise * rng.normal(size=(m, 3)) if point_noise > 0 else 0.0)
        pts[f, :m] = p
        nrm[f, :m] = nc[ids]
        kp_pool[f, :m] = ids
        kp_src[f, :m] = src
    depth = normal = mask = None
    if render_maps:
        maps = [render(Rs[f], ts[f], K) for f in range(F)]
        depth = np.stack([m[0] for m in maps])
        normal = np.stack([m[1] for m in maps])
        mask = np.stack([m[2] for m in maps])
    return Scene(K, np.stack(Rs), np.stack(ts), n_kp, desc, pts, nrm, kp_pool, kp_src,
                 depth, normal, mask)


def all_pairs(n_frames: int) -> np.ndarray:
    """Every unordered node pair (a < b) of the pose graph (|V| = k+1 nodes)."""
    return np.array([(a, b) for a in range(n_frames) for b in range(a + 1, n_frames)], np.int32)


def directed_edges(pairs: np.ndarray) -> np.ndarray:
    """Both directions of every pair: Eq. (1) sums over ordered i != j."""
    return np.concatenate([pairs, pairs[:, ::-1]], axis=0).astype(np.int32).copy()


# ----------------------------------------------------------------------------------------
# C1: one frame pair with a known SE(3) and 30 % outliers
# ----------------------------------------------------------------------------------------
def make_pair_c1(seed: int = DATA_SEED, n: int = 500, n_max: int = 512, outlier_frac: float = 0.30,
                 point_noise: float = 0.0, desc_noise: float = 0.03, width: int = 160,
                 height: int = 120, distance: float = 1.0):
    """Frame b observes the SAME n pool points as frame a, moved by T_true (rotation
    <= 30 deg, translation <= 5 cm).  outlier_frac of b's keypoints carry the descriptor
    of another of the n points that is >= 5 cm away (a derangement inside the outlier
    set), so mutual-NN matching yields exactly n matches of which outlier_frac are
    geometric outliers.  b's keypoint order is a random permutation.
    Returns (scene, T_true_R, T_true_t, gt_inlier_b) where gt_inlier_b[k] tells whether
    b-keypoint k is a true (inlier) observation."""
    rng = np.random.default_rng(seed)
    K = Intrinsics(600.0, 600.0, (width - 1) / 2.0, (height - 1) / 2.0, width, height)
    pool = sample_surface(rng, 3 * n)
    pool_n = ellipsoid_normal(pool)
    Ra = rotvec_to_R(np.array([0.3, -0.5, 0.2]))
    ta = np.array([0.0, 0.0, distance])
    pc = pool @ Ra.T + ta
    nc = pool_n @ Ra.T
    vis = np.nonzero(np.sum(nc * pc, axis=1) < -0.2 * np.linalg.norm(pc, axis=1))[0]
    ids = rng.permutation(vis)[:n]
    m = len(ids)
    Rrel = random_rotation(rng, np.deg2rad(30.0))
    dc = rng.normal(size=3)
    dc *= rng.uniform(0.0, 0.05) / np.linalg.norm(dc)
    trel = ta - Rrel @ ta + dc                         # object centre moves by <= 5 cm
    Rb = Rrel @ Ra
    tb = Rrel @ ta + trel
    gdesc = rng.normal(size=(m, 128))
    gdesc /= np.linalg.norm(gdesc, axis=1, keepdims=True)

    # outliers: a derangement pi inside the outlier set with partners >= 5 cm apart
    n_out = int(round(outlier_frac * m))
    x = pool[ids]
    out = rng.choice(m, size=n_out, replace=False)
    src = out[rng.permutation(n_out)]

    def ok(i, s):
        return np.linalg.norm(x[out[i]] - x[s]) >= 0.05

    for _ in range(200):                               # repair by random swaps
        bad = [i for i in range(n_out) if not ok(i, src[i])]
        if not bad:
            break
        for i in bad:
            j = int(rng.integers(n_out))
            if ok(i, src[j]) and ok(j, src[i]):
                src[i], src[j] = src[j], src[i]
    else:  # pragma: no cover
        raise RuntimeError("could not draw far outlier partners")
    desc_src_b = np.arange(m)
    desc_src_b[out] = src
    da = gdesc + desc_noise * rng.normal(size=(m, 128))
    db = gdesc[desc_src_b] + desc_noise * rng.normal(size=(m, 128))
    da /= np.linalg.norm(da, axis=1, keepdims=True)
    db /= np.linalg.norm(db, axis=1, keepdims=True)
    pa = x @ Ra.T + ta
    pb = x @ Rb.T + tb
    na = pool_n[ids] @ Ra.T
    nb = pool_n[ids] @ Rb.T
    if point_noise > 0:
        pa = pa + point_noise * rng.normal(size=pa.shape)
        pb = pb + point_noise * rng.normal(size=pb.shape)
    order = rng.permutation(m)                         # b's keypoint order
    inl = np.ones(m, bool)
    inl[out] = False

    F = 2
    desc = np.zeros((F, n_max, 128), np.float32)
    pts = np.zeros((F, n_max, 3), np.float32)
    nrm = np.zeros((F, n_max, 3), np.float32)
    kp_pool = -np.ones((F, n_max), np.int32)
    kp_src = -np.ones((F, n_max), np.int32)
    desc[0, :m], pts[0, :m], nrm[0, :m] = da, pa, na
    kp_pool[0, :m] = np.arange(m)
    kp_src[0, :m] = np.arange(m)
    desc[1, :m], pts[1, :m], nrm[1, :m] = db[order], pb[order], nb[order]
    kp_pool[1, :m] = order
    kp_src[1, :m] = desc_src_b[order]
    maps = [render(Ra, ta, K), render(Rb, tb, K)]
    scene = Scene(K, np.stack([Ra, Rb]), np.stack([ta, tb]), np.array([m, m], np.int32),
                  desc, pts, nrm, kp_pool, kp_src,
                  np.stack([q[0] for q in maps]), np.stack([q[1] for q in maps]),
                  np.stack([q[2] for q in maps]))
    return scene, Rrel, trel, inl[order]


# ----------------------------------------------------------------------------------------
# gathered correspondence sets (for stage-isolated RANSAC tests)
# ----------------------------------------------------------------------------------------
def make_correspondences(rng_or_seed, M: int, inlier_frac: float, noise: float = 0.0,
                         max_angle_deg: float = 30.0, spread: float = 0.05, distance: float = 0.6):
    """M correspondences (p_a, n_a, p_b, n_b) float32, a fraction inlier_frac related by a
    random T_true (+ Gaussian noise), the rest with partners displaced >= 5 cm.  Returns
    (pa, na, pb, nb, R, t, is_inlier)."""
    rng = rng_or_seed if isinstance(rng_or_seed, np.random.Generator) else np.random.default_rng(rng_or_seed)
    R = random_rotation(rng, np.deg2rad(max_angle_deg))
    t = rng.normal(size=3)
    t *= rng.uniform(0, 0.05) / max(np.linalg.norm(t), 1e-12)
    pa = rng.normal(scale=spread, size=(M, 3)) + np.array([0, 0, distance])
    na = rng.normal(size=(M, 3))
    na /= np.linalg.norm(na, axis=1, keepdims=True)
    pb = pa @ R.T + t
    nb = na @ R.T
    n_in = int(round(inlier_frac * M))
    inl = np.zeros(M, bool)
    inl[rng.choice(M, size=n_in, replace=False)] = True
    for m in np.nonzero(~inl)[0]:
        while True:
            d = rng.normal(size=3)
            d *= rng.uniform(0.05, 0.15) / np.linalg.norm(d)
            q = pb[m] + d
            if q[2] > 0.1:
                pb[m] = q
                break
        nn = rng.normal(size=3)
        nb[m] = nn / np.linalg.norm(nn)
    if noise > 0:
        pb[inl] += noise * rng.normal(size=(int(inl.sum()), 3))
    f = np.float32
    return pa.astype(f), na.astype(f), pb.astype(f), nb.astype(f), R, t, inl


def make_nearly_collinear(n_line: int = 200, length: float = 0.2, offset: float = 0.01, seed: int = 0,
                          distance: float = 0.6):
    """A correspondence set whose refit is degenerate while its best sample is not: n_line
    points evenly spaced on a segment of `length` along x plus ONE point displaced by `offset`
    along y, at `distance` in front of the camera, observed identically in both frames (p_b =
    p_a, normals (0, 0, -1)), in a seeded random order.  Returns (pa, na, pb, nb, off_index).
    The spread of the whole set across the line is ~offset^2 against ~n_line length^2 / 12
    along it, while a sample holding the displaced point sees offset^2 against length^2."""
    rng = np.random.default_rng(seed)
    x = np.linspace(-length / 2, length / 2, n_line)
    pts = np.zeros((n_line + 1, 3))
    pts[:n_line, 0] = x
    pts[n_line] = (rng.uniform(-length / 4, length / 4), offset, 0.0)
    pts[:, 2] += distance
    order = rng.permutation(n_line + 1)
    pts = pts[order].astype(np.float32)
    nrm = np.zeros_like(pts)
    nrm[:, 2] = -1.0
    return pts, nrm, pts.copy(), nrm.copy(), int(np.nonzero(order == n_line)[0][0])
