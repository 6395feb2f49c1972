"""Pins of the oracle's Arun least squares ("least squares \\cite{arun1987least}";
DESIGN.md reading R7) and its 3x3 SVD."""
import numpy as np

import oracle
import synth


def _cost(R, t, A, B):
    return float(np.sum((A @ R.T + t - B) ** 2))


def test_svd3_against_library_and_reconstruction():
    rng = np.random.default_rng(0)
    mats = [rng.normal(size=(3, 3)) for _ in range(200)]
    mats += [np.outer(rng.normal(size=3), rng.normal(size=3)) for _ in range(20)]        # rank 1
    mats += [sum(np.outer(rng.normal(size=3), rng.normal(size=3)) for _ in range(2)) for _ in range(20)]
    mats += [np.diag([2.0, 2.0, 1.0]), np.zeros((3, 3)), np.eye(3)]
    for A in mats:
        U, s, V = oracle.svd3(A)
        assert np.allclose(U @ np.diag(s) @ V.T, A, atol=1e-12)
        assert np.allclose(V.T @ V, np.eye(3), atol=1e-12)
        assert np.allclose(np.sort(s)[::-1], np.linalg.svd(A, compute_uv=False), atol=1e-12)
        if s[1] > 1e-12 * max(s[0], 1):
            assert np.allclose(U.T @ U, np.eye(3), atol=1e-10)


def test_exact_recovery_three_points():
    rng = np.random.default_rng(1)
    for _ in range(200):
        R = synth.random_rotation(rng, np.pi)
        t = rng.normal(size=3)
        A = rng.normal(size=(3, 3))
        B = A @ R.T + t
        Rh, th, sig = oracle.arun(A, B)
        assert np.abs(Rh - R).max() < 1e-12 and np.abs(th - t).max() < 1e-12
        assert sig > 0


def test_exact_recovery_many_points_and_identity():
    rng = np.random.default_rng(2)
    R = synth.random_rotation(rng, 2.0)
    t = rng.normal(size=3)
    A = rng.normal(size=(400, 3))
    Rh, th, _ = oracle.arun(A, A @ R.T + t)
    assert np.abs(Rh - R).max() < 1e-12 and np.abs(th - t).max() < 1e-12
    Rh, th, _ = oracle.arun(A, A)
    assert np.abs(Rh - np.eye(3)).max() < 1e-13 and np.abs(th).max() < 1e-13


def test_equilateral_triangle_repeated_singular_values():
    # s1 = s2 for an equilateral triangle; the rotation must still be exact
    A = np.array([[1, 0, 0], [-0.5, np.sqrt(3) / 2, 0], [-0.5, -np.sqrt(3) / 2, 0]])
    rng = np.random.default_rng(3)
    for _ in range(50):
        R = synth.random_rotation(rng, np.pi)
        t = rng.normal(size=3)
        Rh, th, sig = oracle.arun(A, A @ R.T + t)
        assert abs(sig - 1.0) < 1e-12
        assert np.abs(Rh - R).max() < 1e-12 and np.abs(th - t).max() < 1e-12


def test_mirrored_triangle_gives_proper_rotation():
    # b = mirror image of a: the optimal PROPER rotation flips the triangle normal
    rng = np.random.default_rng(4)
    for _ in range(50):
        A = rng.normal(size=(3, 3))
        B = A * np.array([1.0, 1.0, -1.0])
        Rh, th, _ = oracle.arun(A, B)
        assert abs(np.linalg.det(Rh) - 1) < 1e-12
        assert np.allclose(Rh.T @ Rh, np.eye(3), atol=1e-12)


def test_collinear_is_degenerate():
    A = np.array([[0, 0, 0], [1, 1, 1], [2, 2, 2.0]])
    _, _, sig = oracle.arun(A, A + 0.3)
    assert sig < 1e-12


def _rotvec_grid(step):
    g = np.arange(-np.pi, np.pi + 1e-9, step)
    W = np.stack(np.meshgrid(g, g, g, indexing="ij"), -1).reshape(-1, 3)
    return W[np.linalg.norm(W, axis=1) <= np.pi]


def test_brute_force_rotation_search_reaches_arun_cost():
    """Brute-force SO(3) search (grid of pi/24 + 30 local halvings) on a noisy 4-point set
    never goes below Arun's cost and reaches it to ~12 digits (SURVEY R-7)."""
    rng = np.random.default_rng(5)
    for trial in range(3):
        A = rng.normal(size=(4, 3))
        R = synth.random_rotation(rng, np.pi)
        B = A @ R.T + rng.normal(size=3) + 0.05 * rng.normal(size=(4, 3))
        Rh, th, _ = oracle.arun(A, B)
        best_arun = _cost(Rh, th, A, B)

        def cost_rv(w):
            Q = synth.rotvec_to_R(w)
            tt = B.mean(0) - Q @ A.mean(0)            # optimal t for fixed rotation
            return _cost(Q, tt, A, B)

        W = _rotvec_grid(np.pi / 24)
        Ac, Bc = A - A.mean(0), B - B.mean(0)
        # vectorised coarse pass
        best, bw = np.inf, None
        for w in W:
            c = cost_rv(w)
            if c < best:
                best, bw = c, w
        h = np.pi / 24
        offs = np.stack(np.meshgrid([-1, 0, 1], [-1, 0, 1], [-1, 0, 1], indexing="ij"), -1).reshape(-1, 3)
        for _ in range(30):
            cands = [bw + h * o for o in offs]
            cs = [cost_rv(w) for w in cands]
            k = int(np.argmin(cs))
            best, bw = cs[k], cands[k]
            h /= 2
        assert best >= best_arun * (1 - 1e-12) - 1e-15
        assert abs(best - best_arun) <= 1e-10 * max(best_arun, 1e-12), (best, best_arun)
        del Ac, Bc


def test_conjugation_invariance():
    """Pre-transforming both clouds by G conjugates the result: T' = G T G^-1."""
    rng = np.random.default_rng(6)
    A = rng.normal(size=(20, 3))
    B = A @ synth.random_rotation(rng, 1.0).T + 0.3 + 0.01 * rng.normal(size=(20, 3))
    R, t, _ = oracle.arun(A, B)
    G = synth.random_rotation(rng, 2.0)
    g = rng.normal(size=3)
    R2, t2, _ = oracle.arun(A @ G.T + g, B @ G.T + g)
    assert np.allclose(R2, G @ R @ G.T, atol=1e-12)
    assert np.allclose(t2, G @ t + g - G @ R @ G.T @ g, atol=1e-12)
