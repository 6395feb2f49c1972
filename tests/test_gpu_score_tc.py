"""Tensor-core scoring (k_corr_feat / k_score_tc / k_score_fix, reading R27) against
the FFMA2 scoring kernel (BT_SCORE_FMA=1): every per-hypothesis inlier count and every record
word must be bit-identical — the certificate either decides a test with margin or the row is
recounted with the fp32 formula itself.  Oracle parity of the default (tensor-core) path is in
test_gpu_parity.py."""
import os

import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu
SEED = synth.PHILOX_SEED


@pytest.fixture(scope="module")
def bt():
    import paper_2108_00516_b200 as m
    return m


@pytest.fixture(scope="module")
def torch():
    import torch as t
    return t


def _run_both(bt, torch, ctx, sc, pairs, n_hyp, uids=None, match_lists=None):
    fb = bt.FrameBatch.from_scene(sc)
    P = len(pairs)
    n_max = sc.desc.shape[1]
    pr = torch.from_numpy(np.asarray(pairs, np.int32)).cuda()
    uid = np.arange(P, dtype=np.uint32) if uids is None else np.asarray(uids, np.uint32)
    tu = torch.from_numpy(uid.view(np.int32)).cuda()
    if match_lists is None:
        mt = torch.zeros((P, n_max, 2), dtype=torch.int32, device="cuda")
        nm = torch.zeros(P, dtype=torch.int32, device="cuda")
        ctx.match(fb, pr, mt, nm)
    else:
        m = np.zeros((P, n_max, 2), np.int32)
        n = np.zeros(P, np.int32)
        for p, l in enumerate(match_lists):
            m[p, :len(l)] = l
            n[p] = len(l)
        mt, nm = torch.from_numpy(m).cuda(), torch.from_numpy(n).cuda()
    out = {}
    for mode in ("fma", "tc"):
        if mode == "fma":
            os.environ["BT_SCORE_FMA"] = "1"
        else:
            os.environ.pop("BT_SCORE_FMA", None)
        rec = torch.zeros((P, bt.record_words(n_max)), dtype=torch.int32, device="cuda")
        cnt = torch.full((P, n_hyp), -5, dtype=torch.int32, device="cuda")
        ctx.ransac(fb, pr, tu, mt, nm, bt.ransac_params(n_hyp, SEED), rec, cnt)
        torch.cuda.synchronize()
        out[mode] = (rec.cpu().numpy(), cnt.cpu().numpy())
    os.environ.pop("BT_SCORE_FMA", None)
    return out, nm.cpu().numpy()


def _assert_equal(out, what):
    (rf, cf), (rt, ct) = out["fma"], out["tc"]
    bad = np.argwhere(cf != ct)
    assert bad.size == 0, f"{what}: {len(bad)} counts differ, first {bad[:5].tolist()} fma {cf[tuple(bad[0])]} tc {ct[tuple(bad[0])]}"
    assert np.array_equal(rf, rt), f"{what}: records differ"


def test_score_tc_equals_fma_c2(bt, torch):
    """All 120 C2 pairs at 4096 hypotheses (the bench workload)."""
    sc = synth.make_scene(16)
    pairs = synth.all_pairs(16)
    ctx = bt.Context(0)
    ctx.reserve(len(pairs), sc.desc.shape[1], 4096, 16, 640, 480)
    out, nm = _run_both(bt, torch, ctx, sc, pairs, 4096)
    ctx.close()
    assert (nm >= 3).all()
    _assert_equal(out, "C2")
    assert (out["tc"][1] > 0).any()


def test_score_tc_equals_fma_c1_and_ragged(bt, torch):
    """C1 (1024 hypotheses), a hypothesis count that is not a multiple of 128, noisy points."""
    ctx = bt.Context(0)
    ctx.reserve(4, 512, 2048, 2, 160, 120)
    sc, *_ = synth.make_pair_c1()
    out, _ = _run_both(bt, torch, ctx, sc, [(0, 1)], 1024)
    _assert_equal(out, "C1")
    sc, *_ = synth.make_pair_c1(seed=7, point_noise=0.001)
    out, _ = _run_both(bt, torch, ctx, sc, [(0, 1)], 1000)
    _assert_equal(out, "C1 noisy, H = 1000")
    ctx.close()


@pytest.mark.parametrize("M", [0, 1, 2, 3, 4, 127, 128, 129, 3000])
def test_score_tc_equals_fma_match_counts(bt, torch, M):
    """Degenerate and chunk-boundary correspondence counts (M = 3000: 24 chunks of 128)."""
    rng = np.random.default_rng(100 + M)
    n_max = 4096 if M > 512 else 512
    sc = synth.make_scene(2, render_maps=False, seed=3)
    Mm = max(M, 3)
    pa, na, pb, nb, R, t, inl = synth.make_correspondences(rng, Mm, 0.45, noise=0.0005)
    pts = np.zeros((2, n_max, 3), np.float32)
    nrm = np.zeros((2, n_max, 3), np.float32)
    nrm[:, :, 2] = -1.0
    pts[:, :, 2] = 0.5
    pts[0, :Mm], nrm[0, :Mm], pts[1, :Mm], nrm[1, :Mm] = pa, na, pb, nb
    sc.pts, sc.nrm = pts, nrm
    sc.desc = np.zeros((2, n_max, 128), np.float32)
    sc.n_kp = np.array([Mm, Mm], np.int32)
    sc.depth = sc.normal = sc.mask = None
    m = np.stack([np.arange(M), np.arange(M)], 1).astype(np.int32)
    ctx = bt.Context(0)
    ctx.reserve(1, n_max, 2048, 2, 0, 0)
    out, _ = _run_both(bt, torch, ctx, sc, [(0, 1)], 2048, match_lists=[m])
    ctx.close()
    _assert_equal(out, f"M = {M}")


def test_score_tc_list_overflow_recounts_rows(bt, torch):
    """The safety net: with the undecided-test list capped at 50 entries (BT_SCORE_ECAP), rows
    whose tests do not fit are recounted whole by k_score_fix — counts still equal the
    FFMA2 kernel's (C2, 24 pairs)."""
    sc = synth.make_scene(16)
    pairs = synth.all_pairs(16)[:24]
    ctx = bt.Context(0)
    ctx.reserve(len(pairs), sc.desc.shape[1], 4096, 16, 640, 480)
    os.environ["BT_SCORE_ECAP"] = "50"
    try:
        out, _ = _run_both(bt, torch, ctx, sc, pairs, 4096)
    finally:
        os.environ.pop("BT_SCORE_ECAP", None)
    ctx.close()
    _assert_equal(out, "C2 subset, list capped at 50")


@pytest.mark.parametrize("scale,shift", [(10.0, 0.0), (0.05, 0.0), (1.0, 3.0)])
def test_score_tc_equals_fma_scaled_scenes(bt, torch, scale, shift):
    """Object size x10 (1.2 m) and x0.05 (6 mm, below the 5 mm gate's scale), and a scene 3 m
    away: the per-pair feature scales and the per-row certificate adapt; counts equal the
    FFMA2 kernel's."""
    rng = np.random.default_rng(int(scale * 100 + shift))
    M = 600
    pa, na, pb, nb, R, t, inl = synth.make_correspondences(rng, M, 0.4, noise=0.0005)
    ca = pa.mean(0)
    pa = ((pa - ca) * scale + ca + [0, 0, shift]).astype(np.float32)
    pb = ((pb - ca) * scale + ca + [0, 0, shift]).astype(np.float32)
    n_max = 1024
    sc = synth.make_scene(2, render_maps=False, seed=5)
    pts = np.zeros((2, n_max, 3), np.float32)
    nrm = np.zeros((2, n_max, 3), np.float32)
    nrm[:, :, 2] = -1.0
    pts[:, :, 2] = 0.5
    pts[0, :M], nrm[0, :M], pts[1, :M], nrm[1, :M] = pa, na, pb, nb
    sc.pts, sc.nrm = pts, nrm
    sc.desc = np.zeros((2, n_max, 128), np.float32)
    sc.n_kp = np.array([M, M], np.int32)
    sc.depth = sc.normal = sc.mask = None
    m = np.stack([np.arange(M), np.arange(M)], 1).astype(np.int32)
    ctx = bt.Context(0)
    ctx.reserve(1, n_max, 4096, 2, 0, 0)
    out, _ = _run_both(bt, torch, ctx, sc, [(0, 1)], 4096, match_lists=[m])
    ctx.close()
    _assert_equal(out, f"scale {scale}, shift {shift}")


def test_score_tc_equals_fma_c5_shape(bt, torch):
    """BASELINE configs[4] shape (n = 4096 keypoints, ~2600 matches per pair, 16384
    hypotheses): 15 pairs of a 6-frame scene, every count bitwise equal to the FFMA2 kernel."""
    sc = synth.make_scene(6, n=4096, n_max=4096, pool_size=12000, seed=4242, outlier_frac=0.16,
                          render_maps=False)
    pairs = synth.all_pairs(6)
    ctx = bt.Context(0)
    ctx.reserve(len(pairs), 4096, 16384, 6, 0, 0)
    out, nm = _run_both(bt, torch, ctx, sc, pairs, 16384)
    ctx.close()
    assert (nm > 1500).all()
    _assert_equal(out, "C5 shape")


def test_score_tc_equals_fma_adversarial_exponent_spread(bt, torch):
    """an adversarial check of R27's accumulator model.  Correspondence sets whose
    centred features span many binades in ONE pair (points from 0.1 mm to 5 m from the centroid,
    so Y1's k-columns mix magnitudes ~1e-8 .. 25 m^2), hypotheses from triples that mix the
    scales (huge |t'|, heavy cancellation in |R a' + t' - b'|^2 - |t'|^2), near-gate
    inliers at exactly delta +- 1e-3 delta, and flipped / grazing normals.  The tensor-core counts
    must still equal the FFMA2 kernel's bit for bit: every test the certificate cannot decide is
    recounted by the fp32 formula."""
    rng = np.random.default_rng(1234)
    n_max = 1024
    F = 6
    sc = synth.make_scene(2, render_maps=False, seed=3)
    sc.n_kp = np.zeros(F, np.int32)
    sc.desc = np.zeros((F, n_max, 128), np.float32)
    sc.pts = np.zeros((F, n_max, 3), np.float32)
    sc.nrm = np.zeros((F, n_max, 3), np.float32)
    mls, pairs = [], []
    for q in range(F // 2):
        M = 900
        scale = 10.0 ** rng.uniform(-4, np.log10(5.0), size=(M, 1))      # 0.1 mm .. 5 m
        d = rng.normal(size=(M, 3))
        pa = d / np.linalg.norm(d, axis=1, keepdims=True) * scale + [0, 0, 0.6]
        R = synth.random_rotation(rng, np.pi)
        t = rng.normal(size=3) * 10.0 ** rng.uniform(-3, 1)
        pb = pa @ R.T + t
        # a third of the partners sit on the distance gate (delta = 5 mm) +- 1e-3 delta
        k = rng.permutation(M)[:M // 3]
        u = rng.normal(size=(len(k), 3))
        u /= np.linalg.norm(u, axis=1, keepdims=True)
        pb[k] += u * 0.005 * (1.0 + rng.choice([-1e-3, 1e-3], size=(len(k), 1)))
        na = rng.normal(size=(M, 3))
        na /= np.linalg.norm(na, axis=1, keepdims=True)
        nb = na @ R.T
        flip = rng.random(M) < 0.2
        nb[flip] *= -1.0                                                 # flipped normals
        a, b = 2 * q, 2 * q + 1
        sc.n_kp[a] = sc.n_kp[b] = M
        sc.pts[a, :M], sc.pts[b, :M] = pa, pb
        sc.nrm[a, :M], sc.nrm[b, :M] = na, nb
        mls.append(np.stack([np.arange(M), rng.permutation(M)], 1).astype(np.int32) if q == 2 else
                   np.stack([np.arange(M), np.arange(M)], 1).astype(np.int32))
        pairs.append((a, b))
    ctx = bt.Context(0)
    ctx.reserve(len(pairs), n_max, 4096, F)
    out, nm = _run_both(bt, torch, ctx, sc, pairs, 4096, match_lists=mls)
    ctx.close()
    _assert_equal(out, "adversarial")
    assert (out["tc"][1][:2] > 100).any()                                # real inliers exist
