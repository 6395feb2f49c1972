"""Pins of the oracle's mutual-NN matching (P:4; readings R1-R4).
SPEC examples S:274-276 (identity, empty, permutation + noise), S:252 (no duplicates)."""
import numpy as np

import oracle
import synth


def _unit(rng, n, d=128):
    x = rng.normal(size=(n, d))
    return (x / np.linalg.norm(x, axis=1, keepdims=True)).astype(np.float32)


def test_identical_sets_give_identity():
    A = _unit(np.random.default_rng(0), 200)
    r = oracle.match(A, A)
    assert r["pairs"].tolist() == [[i, i] for i in range(200)]


def test_empty_inputs():
    A = _unit(np.random.default_rng(1), 5)
    E = np.zeros((0, 128), np.float32)
    assert len(oracle.match(E, A)["pairs"]) == 0
    assert len(oracle.match(A, E)["pairs"]) == 0
    assert len(oracle.match(E, E)["pairs"]) == 0


def test_known_permutation_with_noise():
    rng = np.random.default_rng(2)
    A = _unit(rng, 500)
    perm = rng.permutation(500)
    B = A[perm] + 0.03 * rng.normal(size=(500, 128)).astype(np.float32)
    B /= np.linalg.norm(B, axis=1, keepdims=True)
    r = oracle.match(A, B.astype(np.float32))
    inv = np.argsort(perm)          # A[i] sits at B[inv[i]]
    assert r["pairs"].tolist() == [[i, int(inv[i])] for i in range(500)]
    assert not r["row_border"].any() and not r["col_border"].any()


def test_swap_symmetry_and_no_duplicates():
    sc = synth.make_scene(2, render_maps=False, seed=5)
    A, B = sc.desc[0, :sc.n_kp[0]], sc.desc[1, :sc.n_kp[1]]
    r1 = oracle.match(A, B)["pairs"]
    r2 = oracle.match(B, A)["pairs"]
    assert sorted(map(tuple, r1.tolist())) == sorted((j, i) for i, j in r2.tolist())
    assert len(set(r1[:, 0])) == len(r1) and len(set(r1[:, 1])) == len(r1)
    assert np.all(np.diff(r1[:, 0]) > 0)                  # ascending in i (R4)


def test_ties_go_to_lowest_index():
    rng = np.random.default_rng(3)
    A = _unit(rng, 4)
    B = np.stack([A[1], A[0], A[0], A[2]])               # B[1] == B[2]
    r = oracle.match(A, B)
    assert r["nn_ab"][0] == 1                             # lowest of the tied columns
    assert r["row_border"][0]                              # and flagged as ambiguous
    assert r["pairs"].tolist() == [[0, 1], [1, 0], [2, 3]]


def test_squared_distance_values():
    # one-hot descriptors: d(e_i, e_j) = 2 for i != j, 0 for i == j; scaled copies
    A = np.eye(3, 128, dtype=np.float32)
    B = np.stack([2 * A[0], 3 * A[1]])
    r = oracle.match(A, B)
    # row 0: d(A0,B0) = 1, d(A0,B1) = 1 + 9 = 10 -> NN 0 with best d = 1 exactly
    assert r["nn_ab"][0] == 0 and r["d_best"][0] == 1.0
    # row 2 (e_2): d = 1 + 4 = 5 to B0 and 1 + 9 = 10 to B1
    assert r["nn_ab"][2] == 0 and r["d_best"][2] == 5.0
    assert r["pairs"].tolist() == [[0, 0], [1, 1]]


def test_ratio_test():
    # row 0: d1 = 1, d2 = 1 + 0.25 = 1.25 -> d1 < 0.8^2 d2 = 0.8 fails; ratio 0.95 passes
    A = np.zeros((1, 128), np.float32)
    B = np.zeros((2, 128), np.float32)
    B[0, 0] = 1.0
    B[1, 0] = 1.0
    B[1, 1] = 0.5
    assert len(oracle.match(A, B, ratio=0.8)["pairs"]) == 0
    assert oracle.match(A, B, ratio=0.95)["pairs"].tolist() == [[0, 0]]
    assert oracle.match(A, B, ratio=1.0)["pairs"].tolist() == [[0, 0]]
