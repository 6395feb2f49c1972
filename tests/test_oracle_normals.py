"""Pins of the oracle's normal-map estimation (NEXT-4, SPEC estimate_normals S:157-165; the
paper's n_i(x)): central differences of the unprojected cloud are EXACT on planes
(any plane: its normal up to the float32 depth quantization, ~f * 2^-24 ~ 4e-5 — a wrong
sign, cross-product order or intrinsic is O(1); SPEC's fronto-parallel and 45-degree
examples), second
order on curved surfaces (a sphere's radial normal), and the validity rules (border, holes,
isolated pixels, the 5 cm jump) are checked case by case."""
import numpy as np
import pytest

import oracle
import synth

K = synth.Intrinsics(600.0, 600.0, 79.5, 59.5, 160, 120)


def plane_depth(n, c, K=K):
    """Depth of the plane n . X = c (camera frame) along each pixel ray."""
    H, W = K.height, K.width
    u, v = np.meshgrid(np.arange(W), np.arange(H))
    r = np.stack([(u - K.cx) / K.fx, (v - K.cy) / K.fy, np.ones_like(u, dtype=np.float64)], -1)
    return (c / (r @ np.asarray(n, np.float64))).astype(np.float32)


def test_fronto_parallel_plane():
    d = np.full((K.height, K.width), 0.8, np.float32)
    n = oracle.estimate_normals(d, K)
    assert np.array_equal(n[1:-1, 1:-1], np.broadcast_to(np.float32([0, 0, -1]), n[1:-1, 1:-1].shape))
    assert not n[0].any() and not n[-1].any() and not n[:, 0].any() and not n[:, -1].any()


def test_slanted_plane_z_equals_1_plus_x():
    d = plane_depth([-1.0, 0.0, 1.0], 1.0)                         # z - x = 1
    n = oracle.estimate_normals(d, K)
    want = np.array([1.0, 0.0, -1.0]) / np.sqrt(2.0)               # camera-facing
    assert np.abs(n[1:-1, 1:-1] - want).max() < 1e-4


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_any_plane_is_exact(seed):
    rng = np.random.default_rng(seed)
    nrm = rng.normal(size=3)
    nrm[2] = abs(nrm[2]) + 1.0                                     # facing the camera side
    nrm /= np.linalg.norm(nrm)
    d = plane_depth(nrm, 0.6 * nrm[2])
    ok = (d > 0.1) & (d < 5)
    d = np.where(ok, d, 0).astype(np.float32)
    n = oracle.estimate_normals(d, K, jump=10.0)
    valid = np.linalg.norm(n, axis=-1) > 0
    assert valid[1:-1, 1:-1].mean() > 0.9
    facing = -nrm if nrm[2] > 0 else nrm                           # n . P < 0 for P on the plane
    assert np.abs(n[valid] - facing).max() < 1e-4


def test_sphere_normals_are_radial_to_second_order():
    H, W = K.height, K.width
    C, R = np.array([0.0, 0.0, 0.5]), 0.08
    u, v = np.meshgrid(np.arange(W), np.arange(H))
    r = np.stack([(u - K.cx) / K.fx, (v - K.cy) / K.fy, np.ones((H, W))], -1)
    a = np.sum(r * r, -1)
    b = -2 * r @ C
    cc = C @ C - R * R
    disc = b * b - 4 * a * cc
    t = np.where(disc > 0, (-b - np.sqrt(np.maximum(disc, 0))) / (2 * a), 0.0)
    d = t.astype(np.float32)                                       # depth = z = t (ray z-component 1)
    n = oracle.estimate_normals(d, K)
    P = r * t[..., None]
    radial = (P - C) / R
    valid = np.linalg.norm(n, axis=-1) > 0
    inner = valid & (np.linalg.norm(P[..., :2] - C[:2], axis=-1) < 0.6 * R)
    assert inner.sum() > 500
    ang = np.arccos(np.clip(np.sum(n[inner] * radial[inner], -1), -1, 1))
    assert ang.max() < 2e-3                                        # O(h^2) with h ~ 1 px ~ 0.8 mm


def test_validity_rules():
    d = np.zeros((K.height, K.width), np.float32)
    d[50, 50] = 1.0                                                # isolated pixel
    assert not oracle.estimate_normals(d, K).any()
    d = np.full((K.height, K.width), 1.0, np.float32)
    d[40, 40] = 0.0                                                # hole: its 4 neighbours are invalid
    n = oracle.estimate_normals(d, K)
    for (y, x) in [(40, 40), (39, 40), (41, 40), (40, 39), (40, 41)]:
        assert not n[y, x].any()
    assert n[39, 39].any() and n[42, 40].any()
    d = np.full((K.height, K.width), 1.0, np.float32)
    d[:, 80:] = 1.06                                               # 6 cm step: both columns at the edge invalid
    n = oracle.estimate_normals(d, K, jump=0.05)
    assert not n[60, 79].any() and not n[60, 80].any() and n[60, 78].any() and n[60, 81].any()
    d[:, 80:] = 1.04                                               # 4 cm step: kept
    n = oracle.estimate_normals(d, K, jump=0.05)
    assert n[60, 79].any() and n[60, 80].any()


def test_rendered_ellipsoid_normals_agree():
    sc = synth.make_scene(2, n=100, seed=5)
    est = oracle.estimate_normals(sc.depth, sc.K)
    both = (np.linalg.norm(est, axis=-1) > 0) & (np.linalg.norm(sc.normal, axis=-1) > 0)
    assert both.sum() > 20000
    cosang = np.sum(est[both] * sc.normal[both], -1)
    assert np.median(cosang) > np.cos(np.deg2rad(0.2)) and np.mean(cosang > np.cos(np.deg2rad(2.0))) > 0.98
    # frames are independent: one call over two frames == two calls
    assert np.array_equal(est[1], oracle.estimate_normals(sc.depth[1], sc.K))
