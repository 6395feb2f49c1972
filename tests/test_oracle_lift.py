"""Pins of the oracle's keypoint lifting (NEXT-4, reading R29): a keypoint's 3-D point is
pi_D^-1 at its pixel with the depth looked up at the nearest pixel ("point =
unproject(pixel, depth)"), its normal the normal map's there (n_i(x)), and keypoints
outside the mask / without valid depth or normal are dropped, order kept.
Pinned by properties that do not restate the formula: the projection round trip, the
analytic ellipsoid the maps were ray-cast from (the lifted point lies ON the surface, its normal
is the surface's), lookups equal to the map values, and the validity / order rules case by case."""
import numpy as np
import pytest

import oracle
import synth

K = synth.Intrinsics(600.0, 600.0, 79.5, 59.5, 160, 120)


def _frame():
    R = synth.rotvec_to_R(np.array([0.2, -0.3, 0.1]))
    t = np.array([0.01, -0.005, 1.2])                                # ~110 x 80 px: background around
    d, n, m = synth.render(R, t, K)
    return R, t, d[None], n[None], m[None]


def _lift(uv, depth, normal, mask, desc=None):
    uv = np.asarray(uv, np.float32).reshape(1, -1, 2)
    n = uv.shape[1]
    if desc is None:
        desc = np.arange(n * 128, dtype=np.float32).reshape(1, n, 128)
    return oracle.lift_keypoints(uv, desc, np.array([n], np.int32), depth, normal, mask, K), desc


def test_lifted_points_lie_on_the_rendered_surface_with_its_normal():
    R, t, d, n, m = _frame()
    vv, uu = np.nonzero(m[0])
    rng = np.random.default_rng(0)
    pick = rng.choice(len(uu), 200, replace=False)
    uv = np.stack([uu[pick], vv[pick]], 1).astype(np.float32)             # pixel centres
    res, _ = _lift(uv, d, n, m)
    assert res["n"][0] == 200
    p = res["pts"][0, :200].astype(np.float64)
    x = (p - t) @ R                                                       # object frame
    a = np.asarray(synth.AXES)
    assert np.abs(np.sum((x / a) ** 2, 1) - 1.0).max() < 1e-5             # on the ellipsoid
    want_n = synth.ellipsoid_normal(x) @ R.T
    assert np.abs(res["nrm"][0, :200] - want_n).max() < 1e-5              # the surface normal


def test_projection_round_trip_and_nearest_pixel_lookup():
    _, _, d, n, m = _frame()
    vv, uu = np.nonzero(m[0])
    rng = np.random.default_rng(1)
    k = rng.choice(len(uu), 300, replace=False)
    off = rng.uniform(-0.45, 0.45, size=(300, 2))                        # sub-pixel, same nearest pixel
    uv = (np.stack([uu[k], vv[k]], 1) + off).astype(np.float32)
    res, _ = _lift(uv, d, n, m)
    assert res["n"][0] == 300
    p = res["pts"][0, :300].astype(np.float64)
    # z is the depth of the nearest pixel, exactly (a lookup)
    assert np.array_equal(res["pts"][0, :300, 2], d[0][vv[k], uu[k]])
    assert np.array_equal(res["nrm"][0, :300], n[0][vv[k], uu[k]])
    # pi(point) = the keypoint's own (sub-pixel) coordinates (SPEC S:95 round trip)
    u_back = K.fx * p[:, 0] / p[:, 2] + K.cx
    v_back = K.fy * p[:, 1] / p[:, 2] + K.cy
    assert np.abs(u_back - uv[:, 0]).max() < 1e-4 and np.abs(v_back - uv[:, 1]).max() < 1e-4


def test_rounding_side_of_a_half_pixel():
    d = np.zeros((1, K.height, K.width), np.float32)
    d[0, 50, 10] = 0.5
    d[0, 50, 11] = 0.7
    nm = np.zeros((1, K.height, K.width, 3), np.float32)
    nm[..., 2] = -1.0
    mk = np.ones((1, K.height, K.width), np.uint8)
    res, _ = _lift([[10.49, 50.0], [10.51, 50.0], [10.5, 50.0], [9.6, 49.6]], d, nm, mk)
    z = res["pts"][0, :res["n"][0], 2]
    assert list(z) == [np.float32(0.5), np.float32(0.7), np.float32(0.7), np.float32(0.5)]
    assert list(res["border"][0, :4]) == [False, False, True, False]      # 10.5: a tie (band rule)


def test_validity_rules_and_order():
    _, _, d, n, m = _frame()
    vv, uu = np.nonzero(m[0])
    inside = [(float(uu[i]), float(vv[i])) for i in (0, 10, 20, 30, 40)]
    off_mask = (0.0, 0.0)                                                 # corner: background
    assert m[0, 0, 0] == 0
    mk2 = m.copy()
    d2 = d.copy()
    n2 = n.copy()
    d2[0, int(inside[1][1]), int(inside[1][0])] = 0.0                    # depth invalid
    n2[0, int(inside[3][1]), int(inside[3][0])] = 0.0                    # normal invalid
    uv = [inside[0], off_mask, inside[1], (-0.6, 5.0), inside[2], (K.width - 0.4, 5.0), inside[3], inside[4]]
    desc = np.random.default_rng(3).normal(size=(1, len(uv), 128)).astype(np.float32)
    res, _ = _lift(uv, d2, n2, mk2, desc)
    kept = [0, 4, 7]                                                     # in order; the rest dropped
    assert res["n"][0] == len(kept)
    assert np.array_equal(res["desc"][0, :3], desc[0, kept])
    assert np.array_equal(res["pts"][0, :3, 2], [d[0, int(uv[i][1]), int(uv[i][0])] for i in kept])
    assert not res["pts"][0, 3:].any()


def test_empty_and_n_in_bound():
    _, _, d, n, m = _frame()
    uv = np.zeros((1, 4, 2), np.float32)
    res = oracle.lift_keypoints(uv, np.zeros((1, 4, 128), np.float32), np.array([0], np.int32), d, n, m, K)
    assert res["n"][0] == 0 and not res["pts"].any()
