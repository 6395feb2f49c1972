"""Pins of the oracle's pose-graph edge linearizations: Eq. (2) feature edge and
Eq. (3) dense point-to-plane edge, Huber, Jacobians (reading R18)."""
import numpy as np

import oracle
import synth

COS45 = float(np.cos(np.deg2rad(45.0)))


def _exp_se3(xi):
    """exp of a twist (v, w) — test-side helper, used only to PERTURB poses."""
    v, w = np.asarray(xi[:3], float), np.asarray(xi[3:], float)
    R = synth.rotvec_to_R(w)
    th = np.linalg.norm(w)
    K = np.array([[0, -w[2], w[1]], [w[2], 0, -w[0]], [-w[1], w[0], 0]])
    if th < 1e-12:
        V = np.eye(3) + 0.5 * K
    else:
        V = np.eye(3) + (1 - np.cos(th)) / th ** 2 * K + (th - np.sin(th)) / th ** 3 * (K @ K)
    return R, V @ v


def _left(T12, xi):
    R, t = np.asarray(T12[:9], float).reshape(3, 3), np.asarray(T12[9:], float)
    dR, dt = _exp_se3(xi)
    return np.concatenate([(dR @ R).reshape(9), dR @ t + dt])


def _unpack_sym(v21):
    H = np.zeros((6, 6))
    k = 0
    for a in range(6):
        for b in range(a, 6):
            H[a, b] = H[b, a] = v21[k]
            k += 1
    return H


def _feat_blocks(out):
    Hii = _unpack_sym(out[0:21])
    Hij = out[21:57].reshape(6, 6)
    Hjj = _unpack_sym(out[57:78])
    g = out[78:90]
    H = np.block([[Hii, Hij], [Hij.T, Hjj]])
    return H, g, out[90], out[91]


def test_huber_values():
    """(0) -> (0, 1); (delta) -> (delta^2/2, 1); (2 delta) -> (1.5 delta^2, 0.5)."""
    d = 0.005
    assert oracle.huber(0.0, d) == (0.0, 1.0)
    rho, w = oracle.huber(d, d)
    assert abs(rho - 0.5 * d * d) < 1e-18 and w == 1.0
    rho, w = oracle.huber(2 * d, d)
    assert abs(rho - 1.5 * d * d) < 1e-18 and abs(w - 0.5) < 1e-15
    rho, w = oracle.huber(-2 * d, d)
    assert abs(rho - 1.5 * d * d) < 1e-18


def _feature_setup(seed, noise=0.0, n=40):
    rng = np.random.default_rng(seed)
    X = rng.normal(scale=0.05, size=(n, 3))                     # object-frame points
    Ti = synth.pose12(synth.random_rotation(rng, 1.0), rng.normal(scale=0.05, size=3) + [0, 0, 0.6])
    Tj = synth.pose12(synth.random_rotation(rng, 1.0), rng.normal(scale=0.05, size=3) + [0, 0, 0.6])
    Ri, ti = Ti[:9].reshape(3, 3).astype(float), Ti[9:].astype(float)
    Rj, tj = Tj[:9].reshape(3, 3).astype(float), Tj[9:].astype(float)
    pa = (X @ Ri.T + ti).astype(np.float32)
    pb = (X @ Rj.T + tj + noise * rng.normal(size=(n, 3))).astype(np.float32)
    mask = np.array([0xffffffff, (1 << (n - 32)) - 1], np.uint32)
    return pa, pb, mask, Ti, Tj


def test_feature_edge_zero_at_ground_truth():
    pa, pb, mask, Ti, Tj = _feature_setup(0)
    out = oracle.feature_edge(pa, pb, mask, Ti, Tj)
    H, g, E, count = _feat_blocks(out)
    assert count == 40 and E < 1e-12 and np.abs(g).max() < 1e-7


def test_feature_edge_single_gap_energy():
    """One correspondence whose object-frame gap is g (below Huber delta): E = |g|^2 / 2."""
    pa, pb, mask, Ti, Tj = _feature_setup(1)
    Rj = Tj[:9].reshape(3, 3).astype(float)
    gap = np.array([0.001, -0.002, 0.0015])
    pb2 = pb.astype(float).copy()
    pb2[0] = pb2[0] - Rj @ gap                                  # T_j^-1 p_n moves by -gap
    out = oracle.feature_edge(pa, pb2.astype(np.float32), np.array([1, 0], np.uint32), Ti, Tj)
    _, _, E, count = _feat_blocks(out)
    assert count == 1 and abs(E - 0.5 * gap @ gap) < 1e-9


def test_feature_edge_gradient_and_hessian_by_finite_differences():
    """Quadratic Huber branch: E(xi) = 1/2 sum |e|^2, so dE/dxi = g exactly, and at the
    ground truth (e = 0) d2E/dxi2 = H (Gauss-Newton is exact there)."""
    pa, pb, mask, Ti, Tj = _feature_setup(2, noise=0.0005)
    out0 = oracle.feature_edge(pa, pb, mask, Ti, Tj, huber_delta=1.0)     # keep quadratic
    H, g, E0, _ = _feat_blocks(out0)
    eps = 1e-3

    def E_at(k, s):
        # E depends on the poses only through T^-1 p, and (exp(d) T)^-1 p = T^-1 (exp(-d) p):
        # perturb the measurements by exp(-d) (in double, then float32 for the oracle)
        xi = np.zeros(12)
        xi[k] = s
        Rdi, tdi = _exp_se3(-xi[:6])
        Rdj, tdj = _exp_se3(-xi[6:])
        return _energy_double(pa.astype(float) @ Rdi.T + tdi, pb.astype(float) @ Rdj.T + tdj, Ti, Tj)

    for k in range(12):
        fd = (E_at(k, eps) - E_at(k, -eps)) / (2 * eps)
        assert abs(fd - g[k]) <= 1e-4 * np.abs(g).max(), (k, fd, g[k])
    # Hessian at the exact ground truth
    pa, pb, mask, Ti, Tj = _feature_setup(3)
    H, g, _, _ = _feat_blocks(oracle.feature_edge(pa, pb, mask, Ti, Tj))
    rng = np.random.default_rng(9)
    for _ in range(6):
        d = rng.normal(size=12)
        s = 1e-3
        Es = []
        for sg in (1, -1):                          # symmetric: odd-order terms cancel
            Rdi, tdi = _exp_se3(-sg * s * d[:6])
            Rdj, tdj = _exp_se3(-sg * s * d[6:])
            Es.append(_energy_double(pa.astype(float) @ Rdi.T + tdi, pb.astype(float) @ Rdj.T + tdj, Ti, Tj))
        E = 0.5 * (Es[0] + Es[1])
        assert abs(E / s ** 2 - 0.5 * d @ H @ d) <= 2e-4 * abs(0.5 * d @ H @ d)


def _energy_double(pa, pb, Ti, Tj):
    """1/2 sum |T_i^-1 p - T_j^-1 q|^2 with the oracle's own feature_edge on points given in
    double: evaluated by feeding the oracle exact float32 points relative to a shifted
    origin is not possible, so sum the oracle's E over single correspondences whose
    float32 rounding error is below 1e-9 m (points are O(1 m))."""
    # Use the oracle directly: float32 rounding of the perturbed points is ~3e-8 m, far
    # below the eps * |J| ~ 1e-5 m signal; the O(3e-8) noise is absorbed by the tolerance.
    out = oracle.feature_edge(pa.astype(np.float32), pb.astype(np.float32),
                              np.array([0xffffffff, 0xff], np.uint32), Ti, Tj, huber_delta=1.0)
    return out[90]


def _plane_maps(W, H, z, K):
    depth = np.full((H, W), z, np.float32)
    normal = np.zeros((H, W, 3), np.float32)
    normal[..., 2] = -1.0
    mask = np.ones((H, W), np.uint8)
    return depth, normal, mask


def test_dense_identical_frames_self_associate():
    """Identical frames and poses: every valid pixel associates with itself, r = 0,
    H = sum J^T J with J = [n, p x n]."""
    sc, *_ = synth.make_pair_c1()
    T = sc.node_poses()[0]
    out, pix, bd = oracle.dense_edge(sc.depth[0], sc.normal[0], sc.mask[0], sc.depth[0], sc.normal[0],
                                     sc.mask[0], sc.K, T, T, want_pixels=True)
    valid = np.nonzero(sc.mask[0].reshape(-1))[0]
    assert out[28] == len(valid) and out[29] == 0
    assert np.array_equal(np.nonzero(pix.reshape(-1) >= 0)[0], valid)
    assert np.array_equal(pix.reshape(-1)[valid], valid)
    # T T^-1 of a float32 pose is identity only to ~1e-7 (R^T R of a rounded rotation)
    assert abs(out[27]) < 1e-12 and np.abs(out[21:27]).max() < 1e-5
    # closed form of H
    v, u = np.divmod(valid, sc.K.width)
    d = sc.depth[0].reshape(-1)[valid].astype(float)
    p = np.stack([(u - sc.K.cx) * d / sc.K.fx, (v - sc.K.cy) * d / sc.K.fy, d], 1)
    n = sc.normal[0].reshape(-1, 3)[valid].astype(float)
    J = np.concatenate([n, np.cross(p, n)], 1)
    Hc = J.T @ J
    assert np.abs(_unpack_sym(out[:21]) - Hc).max() <= 1e-7 * np.abs(Hc).max()


def test_dense_plane_offset_one_millimetre():
    """Plane seen by two frames whose depth differs by 1 mm along the normal: every pixel
    associates with its own pixel and r = -1 mm; E = count * (1e-3)^2 / 2."""
    K = synth.Intrinsics(500.0, 500.0, 63.5, 47.5, 128, 96)
    di, ni, mi = _plane_maps(128, 96, 0.5, K)
    dj, nj, mj = _plane_maps(128, 96, 0.501, K)
    I = synth.pose12(np.eye(3), np.zeros(3))
    out, pix, bd = oracle.dense_edge(di, ni, mi, dj, nj, mj, K, I, I, want_pixels=True)
    assert out[28] == 128 * 96
    assert np.array_equal(pix.reshape(-1), np.arange(128 * 96))
    dz = float(np.float32(0.501)) - float(np.float32(0.5))      # the 1 mm offset as stored
    assert abs(out[27] - 128 * 96 * 0.5 * dz * dz) < 1e-9 * out[27]
    # g = sum J r with J = [n, p x n], r = -1e-3 (up to float32 depth rounding)
    v, u = np.divmod(np.arange(128 * 96), 128)
    p = np.stack([(u - K.cx) * 0.5 / K.fx, (v - K.cy) * 0.5 / K.fy, np.full(u.shape, 0.5)], 1)
    r_vec = -dz * np.ones(len(p))                      # r = n . (q - p) = -1 mm
    q = p * (float(np.float32(0.501)) / 0.5)
    n = np.array([0, 0, -1.0])
    J = np.concatenate([np.tile(n, (len(p), 1)), np.cross(q, n)], 1)
    gc = J.T @ r_vec
    assert np.allclose(out[21:27], gc, rtol=1e-6, atol=1e-12)


def test_dense_in_plane_sliding_invariance_and_gates():
    """Residual of a plane is invariant to in-plane sliding: shifting frame j's
    pose parallel to the plane changes the association but not r; a shift beyond the
    distance gate empties the edge."""
    K = synth.Intrinsics(500.0, 500.0, 63.5, 47.5, 128, 96)
    di, ni, mi = _plane_maps(128, 96, 0.5, K)
    dj, nj, mj = _plane_maps(128, 96, 0.501, K)
    I = synth.pose12(np.eye(3), np.zeros(3))
    Tj = synth.pose12(np.eye(3), np.array([0.0037, -0.0021, 0.0]))
    out = oracle.dense_edge(di, ni, mi, dj, nj, mj, K, I, Tj)
    base = oracle.dense_edge(di, ni, mi, dj, nj, mj, K, I, I)
    # residual per pixel is still -1 mm: E / count identical
    assert abs(out[27] / out[28] - base[27] / base[28]) < 1e-12
    far = synth.pose12(np.eye(3), np.array([0.0, 0.0, 0.05]))           # 5 cm along the normal
    assert oracle.dense_edge(di, ni, mi, dj, nj, mj, K, I, far)[28] == 0


def test_dense_gradient_by_finite_differences_on_a_tilted_plane():
    """At an offset plane the association is stable under tiny pose changes, so
    dE/dxi_i = g (quadratic Huber branch)."""
    K = synth.Intrinsics(500.0, 500.0, 63.5, 47.5, 128, 96)
    R = synth.rotvec_to_R([0.2, -0.1, 0.0])
    Ti = synth.pose12(R, np.array([0.0, 0.0, 0.5]))
    # render the plane z_obj = 0 (normal +z_obj facing camera after rotation) analytically
    def render_plane(T, offset):
        Rm, t = T[:9].reshape(3, 3).astype(float), T[9:].astype(float)
        n_cam = Rm @ np.array([0, 0, -1.0])
        c = n_cam @ t + offset
        u, v = np.meshgrid(np.arange(128.0), np.arange(96.0))
        d = np.stack([(u - K.cx) / K.fx, (v - K.cy) / K.fy, np.ones_like(u)], -1)
        s = c / (d @ n_cam)
        depth = s.astype(np.float32)
        normal = np.broadcast_to(n_cam, (96, 128, 3)).astype(np.float32)
        return depth, normal.copy(), np.ones((96, 128), np.uint8)
    di, ni, mi = render_plane(Ti, 0.0)
    dj, nj, mj = render_plane(Ti, 0.002)
    out = oracle.dense_edge(di, ni, mi, dj, nj, mj, K, Ti, Ti, huber_delta=1.0)
    g = out[21:27]
    eps = 2e-6
    for k in range(6):
        xi = np.zeros(6)
        xi[k] = eps
        Ep = oracle.dense_edge(di, ni, mi, dj, nj, mj, K, _left(Ti, xi).astype(np.float32), Ti,
                               huber_delta=1.0)
        Em = oracle.dense_edge(di, ni, mi, dj, nj, mj, K, _left(Ti, -xi).astype(np.float32), Ti,
                               huber_delta=1.0)
        assert Ep[28] == Em[28] == out[28]
        fd = (Ep[27] - Em[27]) / (2 * eps)
        assert abs(fd - g[k]) <= 2e-2 * np.abs(g).max(), (k, fd, g[k])


def test_dense_tolerance_scales_and_per_pixel_allowance():
    """The oracle's comparison aids of Eq. (3): the element-wise H scale sum w |J_a J_b| has
    the diagonal of H itself (w J_a^2 >= 0) and bounds |H| element-wise; the per-pixel
    allowances are non-zero only on borderline pixels and sum to the edge's allowance totals;
    the association map holds exactly `count` accepted pixels (P:72 gates)."""
    sc = synth.make_scene(4, seed=5)
    poses = sc.perturbed_poses(3)
    for i, j in ((0, 1), (2, 3), (3, 0)):
        out, pix, bd, pal = oracle.dense_edge(sc.depth[i], sc.normal[i], sc.mask[i], sc.depth[j], sc.normal[j],
                                              sc.mask[j], sc.K, poses[i], poses[j], want_pixels=True,
                                              want_allow=True)
        H, S = _unpack_sym(out[:21]), _unpack_sym(out[48:69])
        assert np.allclose(np.diag(S), np.diag(H), rtol=1e-12, atol=0)
        assert (np.abs(H) <= S * (1 + 1e-12)).all()
        assert (pix >= 0).sum() == out[28] > 1000
        assert not pal[~bd].any()
        tot = pal.reshape(-1, 8).sum(0)
        assert np.isclose(tot[0], out[45], rtol=1e-12) and np.isclose(tot[1], out[44], rtol=1e-12)
        assert np.allclose(tot[2:], out[38:44], rtol=1e-12)
        assert bd.sum() == out[29]


def test_dense_identical_frames_h_scale_closed_form():
    """Identical frames (all weights 1): the H scale is |J|^T |J| in closed form."""
    sc, *_ = synth.make_pair_c1()
    T = sc.node_poses()[0]
    out = oracle.dense_edge(sc.depth[0], sc.normal[0], sc.mask[0], sc.depth[0], sc.normal[0], sc.mask[0], sc.K, T, T)
    valid = np.nonzero(sc.mask[0].reshape(-1))[0]
    v, u = np.divmod(valid, sc.K.width)
    d = sc.depth[0].reshape(-1)[valid].astype(float)
    p = np.stack([(u - sc.K.cx) * d / sc.K.fx, (v - sc.K.cy) * d / sc.K.fy, d], 1)
    n = sc.normal[0].reshape(-1, 3)[valid].astype(float)
    J = np.abs(np.concatenate([n, np.cross(p, n)], 1))
    Sc = J.T @ J
    assert np.abs(_unpack_sym(out[48:69]) - Sc).max() <= 1e-7 * Sc.max()


def test_feature_edge_h_scale_invariants():
    """Eq. (2): the H scale sum w sum_r |J_ra J_rb| (out[108:186], same packing as H) equals H
    on the diagonal, bounds |H| element-wise, and for one correspondence at identity poses with
    p = 0 (J_i = -[I | 0], J_j = [I | 0]) is the 0/1 pattern of |J|^T |J|."""
    rng = np.random.default_rng(3)
    pa = rng.normal(scale=0.05, size=(40, 3)).astype(np.float32) + np.float32([0, 0, 0.6])
    pb = pa + rng.normal(scale=0.003, size=pa.shape).astype(np.float32)
    Ti = synth.pose12(synth.random_rotation(rng, 0.2), rng.normal(scale=0.05, size=3))
    Tj = synth.pose12(synth.random_rotation(rng, 0.2), rng.normal(scale=0.05, size=3))
    mask = np.array([0xffffffff, 0xff], np.uint32)
    out = oracle.feature_edge(pa, pb, mask, Ti, Tj)
    H, _, _, _ = _feat_blocks(out)
    S, _, _, _ = _feat_blocks(np.concatenate([out[108:186], out[78:108]]))
    assert np.allclose(np.diag(S), np.diag(H), rtol=1e-12, atol=0)
    assert (np.abs(H) <= S * (1 + 1e-12)).all()
    I = synth.pose12(np.eye(3), np.zeros(3))
    z = np.zeros((1, 3), np.float32)
    one = oracle.feature_edge(z, z, np.array([1], np.uint32), I, I)
    S1, _, _, _ = _feat_blocks(np.concatenate([one[108:186], one[78:108]]))
    Jabs = np.zeros((3, 12))
    Jabs[:, 0:3] = np.eye(3)
    Jabs[:, 6:9] = np.eye(3)
    assert np.array_equal(S1, Jabs.T @ Jabs)
