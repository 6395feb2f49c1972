"""Pins of the oracle's NEXT-2 tracker decisions (§IV-B, §IV-C, §IV-E): the rotation
geodesic of P:33 against scipy's rotation-vector magnitude, the greedy keyframe selection of P:39
and the novelty rule of P:88 against a hand-worked example (tests/golden/keyframe_selection.txt),
and the coarse pose T~_t = T_rel . T_{t-1} of P:25 against ground-truth object motion."""
import os

import numpy as np
import pytest
from scipy.spatial.transform import Rotation

import oracle
import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "keyframe_selection.txt")


def rz(deg, t=(0.0, 0.0, 0.5)):
    return synth.pose12(synth.rotvec_to_R(np.array([0.0, 0.0, np.deg2rad(deg)])), np.asarray(t))


def test_geodesic_is_the_relative_rotation_angle():
    rng = np.random.default_rng(0)
    for _ in range(200):
        Ra = Rotation.random(random_state=rng).as_matrix()
        Rb = Rotation.random(random_state=rng).as_matrix()
        Ta, Tb = synth.pose12(Ra, np.zeros(3)), synth.pose12(Rb, np.zeros(3))
        want = Rotation.from_matrix(Ta[:9].reshape(3, 3).astype(np.float64).T @ Tb[:9].reshape(3, 3)).magnitude()
        tol = 2e-3 if want > 3.1 else 1e-5                             # acos is ill-conditioned near pi
        assert abs(oracle.rot_geodesic(Ta, Tb) - want) < tol
    assert oracle.rot_geodesic(rz(10), rz(10)) < 1e-3                # float rounding near 0 (acos)
    assert abs(oracle.rot_geodesic(rz(-20), rz(70)) - np.deg2rad(90)) < 1e-6


def _golden():
    g = {"novel": []}
    for line in open(GOLDEN):
        line = line.split("#")[0].split()
        if not line:
            continue
        if line[0] == "novel":
            g["novel"].append((float(line[1]), int(line[2])))
        else:
            g[line[0]] = [float(x) for x in line[1:]]
    return g


def test_selection_and_novelty_hand_worked_example():
    g = _golden()
    pool = np.stack([rz(a) for a in g["pool"]])
    sel = oracle.select_keyframes(pool, rz(g["cur"][0]), int(g["K"][0]))
    assert sel.tolist() == [int(x) for x in g["select"]]
    for cur, want in g["novel"]:
        assert oracle.is_novel(pool, rz(cur)) == bool(want)


def test_selection_small_pool_and_invariants():
    rng = np.random.default_rng(3)
    pool = np.stack([synth.pose12(synth.random_rotation(rng, 1.0), rng.normal(size=3)) for _ in range(9)])
    cur = synth.pose12(synth.random_rotation(rng, 1.0), np.zeros(3))
    for K in (1, 4, 9, 15):
        sel = oracle.select_keyframes(pool, cur, K)
        assert len(sel) == min(K, 9) and sel[0] == 0 and len(set(sel.tolist())) == len(sel)
        assert sel.min() >= 0 and sel.max() < 9
        if K > 1:                                                      # the first greedy step, by hand
            s = [oracle.rot_geodesic(pool[k], cur) + oracle.rot_geodesic(pool[k], pool[0]) for k in range(1, 9)]
            assert sel[1] == 1 + int(np.argmin(s))
    # translations play no part (rotation geodesics only)
    moved = pool.copy()
    moved[:, 9:] += 5.0
    assert np.array_equal(oracle.select_keyframes(moved, cur, 6), oracle.select_keyframes(pool, cur, 6))
    assert oracle.select_keyframes(pool[:0], cur, 5).size == 0
    assert oracle.is_novel(pool[:0], cur)                              # empty pool: the first frame joins


@pytest.mark.parametrize("seed", [0, 1])
def test_coarse_pose_chains_ground_truth_motion(seed):
    """p_t = T_rel p_{t-1} for every object point, so T_rel . T_{t-1} = T_t (object -> camera,
    reading R13); a pair without a hypothesis keeps T_{t-1}."""
    rng = np.random.default_rng(seed)
    R0, R1 = synth.random_rotation(rng, 1.0), synth.random_rotation(rng, 1.0)
    t0, t1 = rng.normal(size=3) * 0.1 + [0, 0, 0.5], rng.normal(size=3) * 0.1 + [0, 0, 0.5]
    Rr = R1 @ R0.T
    T_rel = synth.pose12(Rr, t1 - Rr @ t0)
    x = rng.normal(size=(20, 3)) * 0.05
    p0, p1 = x @ R0.T + t0, x @ R1.T + t1
    assert np.abs(p0 @ Rr.T + (t1 - Rr @ t0) - p1).max() < 1e-12         # T_rel maps t-1 points to t points
    T_prev = synth.pose12(R0, t0)
    got = oracle.coarse_pose(0, T_rel, T_prev)
    assert np.abs(got - synth.pose12(R1, t1)).max() < 1e-6
    assert np.array_equal(oracle.coarse_pose(3, T_rel, T_prev), got)    # REFIT_DEGENERATE still has T_best
    for st in (1, 2):
        assert np.array_equal(oracle.coarse_pose(st, T_rel, T_prev), T_prev.astype(np.float32))
