"""Pins of the oracle's pose-graph Gauss-Newton step (NEXT-1, §IV-D) against
what the mathematics fixes: the SE(3) exponential against the matrix exponential, the adjoint
identity, the assembled gradient against finite differences of the summed Eq. (2) energy, the
gauge null space of the Eq. (3) expansion (a directed dense edge only sees T_i T_j^-1), the
exact solve, and descent / convergence of the iterated step."""
import numpy as np
import pytest
import scipy.linalg

import oracle
import synth

RNG = np.random.default_rng(7)


def hat(xi):
    v, w = xi[:3], xi[3:]
    M = np.zeros((4, 4))
    M[:3, :3] = [[0, -w[2], w[1]], [w[2], 0, -w[0]], [-w[1], w[0], 0]]
    M[:3, 3] = v
    return M


def T44(R, t):
    M = np.eye(4)
    M[:3, :3] = R
    M[:3, 3] = t
    return M


def pose44(p12):
    p = np.asarray(p12, np.float64)
    return T44(p[:9].reshape(3, 3), p[9:])


def pose12(M):
    return np.concatenate([M[:3, :3].reshape(-1), M[:3, 3]]).astype(np.float32)


def left(p12, xi):
    """exp(xi) T (the perturbation convention of reading R18)."""
    R, t = oracle.se3_exp(xi)
    return pose12(T44(R, t) @ pose44(p12))


@pytest.mark.parametrize("scale", [1.0, 1e-3, 1e-8, 0.0])
def test_se3_exp_is_the_matrix_exponential(scale):
    for _ in range(5):
        xi = RNG.normal(size=6) * scale
        R, t = oracle.se3_exp(xi)
        E = scipy.linalg.expm(hat(xi))
        assert np.allclose(R, E[:3, :3], atol=1e-13)
        assert np.allclose(t, E[:3, 3], atol=1e-13)


def test_se3_exp_rodrigues_about_z():
    th = 0.7
    R, t = oracle.se3_exp([0, 0, 0, 0, 0, th])
    assert np.allclose(R, [[np.cos(th), -np.sin(th), 0], [np.sin(th), np.cos(th), 0], [0, 0, 1]], atol=1e-15)
    assert np.allclose(t, 0)
    R, t = oracle.se3_exp([0.1, -0.2, 0.3, 0, 0, 0])                # pure translation
    assert np.allclose(R, np.eye(3)) and np.allclose(t, [0.1, -0.2, 0.3])


def test_se3_adjoint_identity():
    for _ in range(5):
        R = synth.random_rotation(RNG, np.pi)
        t = RNG.normal(size=3)
        d = RNG.normal(size=6) * 0.3
        Adj = oracle.se3_adjoint(R, t)
        lhs = scipy.linalg.expm(hat(Adj @ d)) @ T44(R, t)
        rhs = T44(R, t) @ scipy.linalg.expm(hat(d))
        assert np.allclose(lhs, rhs, atol=1e-12)


# ------------------------------------------------------------------ a feature-only graph
def feature_graph(n_nodes=4, n_pts=60, noise=0.0, seed=3):
    rng = np.random.default_rng(seed)
    X = rng.uniform(-0.08, 0.08, size=(n_pts, 3))
    gt = [pose12(T44(np.eye(3), np.array([0.0, 0.0, 0.5])))]
    for _ in range(1, n_nodes):
        R = synth.random_rotation(rng, np.deg2rad(40))
        gt.append(pose12(T44(R, np.array([0.0, 0.0, 0.5]) + rng.uniform(-0.03, 0.03, 3))))
    gt = np.stack(gt)
    cam = [(X @ pose44(p)[:3, :3].T + pose44(p)[:3, 3] + noise * rng.normal(size=X.shape)).astype(np.float32)
           for p in gt]
    pairs = np.array([(a, b) for a in range(n_nodes) for b in range(a + 1, n_nodes)], np.int32)
    mask = np.full((n_pts + 31) // 32, 0xFFFFFFFF, np.uint32)
    if n_pts % 32:
        mask[-1] = (1 << (n_pts % 32)) - 1
    return gt, cam, pairs, mask


def feat_blocks(poses, cam, pairs, mask, huber=0.005):
    return np.stack([oracle.feature_edge(cam[a], cam[b], mask, poses[a], poses[b], huber)[:96] for a, b in pairs])


def perturb(gt, seed, rot_deg=3.0, trans=0.01, fixed=0):
    rng = np.random.default_rng(seed)
    out = gt.copy()
    for k in range(len(gt)):
        if k == fixed:
            continue
        xi = np.concatenate([rng.normal(size=3) * trans / np.sqrt(3), rng.normal(size=3) * np.deg2rad(rot_deg) / np.sqrt(3)])
        out[k] = left(gt[k], xi)
    return out


def total_feature_energy(poses, cam, pairs, mask):
    return float(sum(oracle.feature_edge(cam[a], cam[b], mask, poses[a], poses[b])[90] for a, b in pairs))


def test_graph_gradient_matches_finite_differences_of_eq2():
    gt, cam, pairs, mask = feature_graph()
    poses = perturb(gt, 1)
    feat = feat_blocks(poses, cam, pairs, mask)
    A, b, (Ef, Eg) = oracle.graph_system(poses, pairs, feat, lambda_f=1.0)
    assert Eg == 0.0 and Ef == pytest.approx(total_feature_energy(poses, cam, pairs, mask))
    assert np.allclose(A, A.T, atol=1e-12 * np.abs(A).max())
    h = 1e-4
    for k in range(len(poses)):
        for d in range(6):
            e = np.zeros(6)
            e[d] = h
            Pp, Pm = poses.copy(), poses.copy()
            Pp[k] = left(poses[k], e)
            Pm[k] = left(poses[k], -e)
            fd = (total_feature_energy(Pp, cam, pairs, mask) - total_feature_energy(Pm, cam, pairs, mask)) / (2 * h)
            assert fd == pytest.approx(b[6 * k + d], rel=2e-3, abs=2e-3 * np.abs(b).max()), (k, d)
    # lambda scales the system linearly
    A2, b2, _ = oracle.graph_system(poses, pairs, feat, lambda_f=2.5)
    assert np.allclose(A2, 2.5 * A) and np.allclose(b2, 2.5 * b)


def test_graph_feature_energy_is_gauge_invariant():
    """E_f only sees T_i^-1 p - T_j^-1 p: a common right perturbation leaves it unchanged, so
    the gradient is orthogonal to (Adj_{T_i} d, Adj_{T_j} d, ...)."""
    gt, cam, pairs, mask = feature_graph()
    poses = perturb(gt, 2)
    A, b, _ = oracle.graph_system(poses, pairs, feat_blocks(poses, cam, pairs, mask))
    for _ in range(4):
        d = RNG.normal(size=6)
        v = np.concatenate([oracle.se3_adjoint(pose44(p)[:3, :3], pose44(p)[:3, 3]) @ d for p in poses])
        # exact up to the float32 poses' non-orthonormality (~1e-7; Eq. (2) uses R^T as T^-1);
        # a wrong sign or block placement is O(1)
        assert abs(b @ v) <= 1e-7 * np.linalg.norm(b) * np.linalg.norm(v)


@pytest.fixture(scope="module")
def scene3():
    return synth.make_scene(3, n=300, seed=11)


def dense_blocks(sc, poses, pairs, **kw):
    dij, dji = [], []
    for a, b in pairs:
        dij.append(oracle.dense_edge(sc.depth[a], sc.normal[a], sc.mask[a], sc.depth[b], sc.normal[b], sc.mask[b],
                                     sc.K, poses[a], poses[b], **kw)[:32])
        dji.append(oracle.dense_edge(sc.depth[b], sc.normal[b], sc.mask[b], sc.depth[a], sc.normal[a], sc.mask[a],
                                     sc.K, poses[b], poses[a], **kw)[:32])
    return np.stack(dij), np.stack(dji)


def test_graph_dense_expansion_has_the_gauge_null_space(scene3):
    """A directed dense edge only sees T_i T_j^-1 (Eq. (3)), so its expanded blocks satisfy
    J_i Adj_{T_i} + J_j Adj_{T_j} = 0: A v = 0 and b . v = 0 for v = (Adj_{T_k} d)_k.  This
    pins J_j = -J_i Adj(T_i T_j^-1), the adjoint and the block placement."""
    sc = scene3
    poses = sc.perturbed_poses(5, rot_deg=2.0, trans_m=0.01)
    pairs = synth.all_pairs(3)
    dij, dji = dense_blocks(sc, poses, pairs)
    assert (dij[:, 28] > 1000).all() and (dji[:, 28] > 1000).all()      # real edges
    feat = np.zeros((len(pairs), 96))
    A, b, (Ef, Eg) = oracle.graph_system(poses, pairs, feat, dij, dji, lambda_f=0.0, lambda_g=1.0)
    assert Ef == 0 and Eg == pytest.approx(dij[:, 27].sum() + dji[:, 27].sum())
    assert np.allclose(A, A.T, atol=1e-12 * np.abs(A).max())
    for _ in range(4):
        d = RNG.normal(size=6)
        v = np.concatenate([oracle.se3_adjoint(pose44(p)[:3, :3], pose44(p)[:3, 3]) @ d for p in poses])
        # exact up to the float32 poses' non-orthonormality (~1e-7 relative)
        assert np.linalg.norm(A @ v) <= 1e-7 * np.abs(A).max() * np.linalg.norm(v)
        assert abs(b @ v) <= 1e-7 * np.linalg.norm(b) * np.linalg.norm(v)
    # a wrong sign / missing adjoint breaks it: the per-edge block alone (no j part) does not
    Ai = np.zeros_like(A)
    Ai[:6, :6] = A[:6, :6]
    d = RNG.normal(size=6)
    v = np.concatenate([oracle.se3_adjoint(pose44(p)[:3, :3], pose44(p)[:3, 3]) @ d for p in poses])
    assert np.linalg.norm(Ai @ v) > 1e-3 * np.abs(A).max() * np.linalg.norm(v)


def test_graph_step_solves_the_pinned_system():
    gt, cam, pairs, mask = feature_graph(n_nodes=5)
    poses = perturb(gt, 4)
    feat = feat_blocks(poses, cam, pairs, mask)
    # node 4 without edges: unconstrained, pinned
    keep = np.array([(a != 4 and b != 4) for a, b in pairs])
    pairs, feat = pairs[keep], feat[keep]
    d, newp, _ = oracle.graph_step(poses, pairs, feat, fixed_node=1)
    A, b, _ = oracle.graph_system(poses, pairs, feat)
    assert np.all(d[1] == 0) and np.all(d[4] == 0)
    assert np.array_equal(newp[1], poses[1]) and np.array_equal(newp[4], poses[4])
    free = [k for k in range(6 * 5) if k // 6 not in (1, 4)]
    res = A[np.ix_(free, free)] @ d.reshape(-1)[free] + b[free]
    assert np.linalg.norm(res) <= 1e-9 * np.linalg.norm(b)
    for k in (0, 2, 3):                                         # T_k <- exp(d_k) T_k
        assert np.allclose(newp[k], left(poses[k], d[k]), atol=1e-7)


def test_graph_steps_converge_to_ground_truth():
    gt, cam, pairs, mask = feature_graph(n_nodes=4)
    poses = perturb(gt, 6, rot_deg=5.0, trans=0.02)
    E = [total_feature_energy(poses, cam, pairs, mask)]
    for _ in range(8):
        _, poses, _ = oracle.graph_step(poses, pairs, feat_blocks(poses, cam, pairs, mask), fixed_node=0)
        E.append(total_feature_energy(poses, cam, pairs, mask))
    assert E[1] < E[0] and E[-1] < 1e-9 * E[0] + 1e-12
    for k in range(4):                      # (|R - R_gt|: arccos of the trace is blind below ~2e-4)
        Tk, Gk = pose44(poses[k]), pose44(gt[k])
        assert np.linalg.norm(Tk[:3, :3] - Gk[:3, :3]) < 1e-6 and np.linalg.norm(Tk[:3, 3] - Gk[:3, 3]) < 1e-6


def test_graph_step_with_dense_edges_descends(scene3):
    """Eq. (1) with both energies (lambda = 1): Gauss-Newton steps from perturbed poses
    lower E_f + E_g re-evaluated at the new poses (re-association included).  (Not a per-node
    pose-error claim: at lambda = 1 the dense term dominates and point-to-plane on the smooth
    ellipsoid leaves shallow directions a single step may overshoot along.)"""
    sc = scene3
    pairs = synth.all_pairs(3)
    gtp = sc.node_poses()
    poses = sc.perturbed_poses(9, rot_deg=2.0, trans_m=0.01)
    mask_all = {}
    cams = {}
    feat = []
    for a, b in pairs:                          # ground-truth correspondences via the pool ids
        ids_a = {int(i): k for k, i in enumerate(sc.kp_pool[a][:sc.n_kp[a]])}
        pa, pb = [], []
        for k, i in enumerate(sc.kp_pool[b][:sc.n_kp[b]]):
            if int(i) in ids_a:
                pa.append(sc.pts[a][ids_a[int(i)]])
                pb.append(sc.pts[b][k])
        pa, pb = np.array(pa, np.float32), np.array(pb, np.float32)
        M = len(pa)
        mk = np.full((M + 31) // 32, 0xFFFFFFFF, np.uint32)
        if M % 32:
            mk[-1] = (1 << (M % 32)) - 1
        cams[(a, b)] = (pa, pb)
        mask_all[(a, b)] = mk

    def energies(P):
        f = np.stack([oracle.feature_edge(*cams[(a, b)], mask_all[(a, b)], P[a], P[b])[:96] for a, b in pairs])
        dij, dji = dense_blocks(sc, P, pairs)
        return f, dij, dji, f[:, 90].sum() + dij[:, 27].sum() + dji[:, 27].sum()

    f, dij, dji, E0 = energies(poses)
    _, new, (Ef, Eg) = oracle.graph_step(poses, pairs, f, dij, dji, fixed_node=0)
    assert Ef + Eg == pytest.approx(E0)
    f, dij, dji, E1 = energies(new)
    _, new2, _ = oracle.graph_step(new, pairs, f, dij, dji, fixed_node=0)
    *_, E2 = energies(new2)
    assert E1 < 0.5 * E0 and E2 < E1
    assert np.array_equal(new[0], poses[0]) and np.array_equal(new2[0], poses[0])    # I_0 fixed
    del gtp


def test_failed_registration_status_drops_only_the_feature_term():
    """Reading R30: status 1 / 2 (S:290's registration-failure signal) zeroes the pair's Eq. (2)
    contribution and keeps its Eq. (3) edges — the same system as zeroing those feat rows."""
    rng = np.random.default_rng(4)
    N, pairs = 4, np.array([(0, 1), (1, 2), (0, 3), (2, 3)], np.int32)
    poses = np.stack([synth.pose12(synth.random_rotation(rng, 0.5), rng.normal(size=3) * 0.1 + [0, 0, 0.5])
                      for _ in range(N)])
    feat = rng.normal(size=(4, 96))
    dij, dji = rng.normal(size=(4, 32)), rng.normal(size=(4, 32))
    status = np.array([0, 2, 3, 1], np.int32)
    A, b, e = oracle.graph_system(poses, pairs, feat, dij, dji, status=status)
    fz = feat.copy()
    fz[[1, 3]] = 0.0
    A0, b0, e0 = oracle.graph_system(poses, pairs, fz, dij, dji)
    assert np.array_equal(A, A0) and np.array_equal(b, b0) and e == e0
    A1, _, _ = oracle.graph_system(poses, pairs, feat, dij, dji)
    assert not np.array_equal(A, A1)
