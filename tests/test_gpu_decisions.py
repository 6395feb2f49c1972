"""Decision-level GPU parity: the CUDA path's per-pixel Eq. (3)
associations, its C_ij match lists from bt_register_pairs, its Eq. (2) blocks on its own inlier
set, and the REFIT_DEGENERATE branch — each against the oracle, through the C ABI.

* Eq. (3): bt_dense_assoc exposes the target pixel each source pixel was associated
  with; on EVERY directed edge of the C2 graph (240 edges, 640x480) it must equal the oracle's
  (bto_dense_edge pix_out) at every pixel outside the band (reading R22), and H / g / E must
  agree element by element (parity.dense_decisions).
* Eq. (2): the oracle's bto_feature_edge evaluated on the GPU's own inlier mask, so the
  comparison is unconditional (no "only if the masks agree").
* Matching: bt_register_pairs' own match lists (bt_copy_matches) against brute force.
* REFIT_DEGENERATE (reading R8 applied to the refit, status 3)."""
import numpy as np
import pytest

import oracle
import parity
import synth

pytestmark = pytest.mark.gpu

SEED = synth.PHILOX_SEED
COS45 = float(np.cos(np.deg2rad(45.0)))


@pytest.fixture(scope="module")
def bt():
    import paper_2108_00516_b200 as m
    return m


@pytest.fixture(scope="module")
def torch():
    import torch as t
    return t


@pytest.fixture(scope="module")
def ctx(bt):
    c = bt.Context(0)
    c.reserve(120, 512, 4096, 16, 640, 480)
    yield c
    c.close()


@pytest.fixture(scope="module")
def c2():
    return synth.make_scene(16)


def _dev(torch, a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def gpu_assoc(bt, torch, ctx, scene, poses, edges, **eprm):
    fb = bt.FrameBatch.from_scene(scene)
    E = len(edges)
    H, W = scene.depth.shape[1:]
    out = torch.zeros((E, 32), dtype=torch.float32, device="cuda")
    assoc = torch.zeros((E, H, W), dtype=torch.int32, device="cuda")
    ed = _dev(torch, np.asarray(edges, np.int32))
    prm = bt.edge_params(**eprm)
    ps = _dev(torch, poses)
    ctx.dense_assoc(fb, scene.K, ps, ed, prm, out, assoc)
    ref = torch.zeros_like(out)
    ctx.dense_corr(fb, scene.K, ps, ed, prm, ref)
    torch.cuda.synchronize()
    out = out.cpu().numpy()
    # the verification entry computes exactly what the product entry does
    assert np.array_equal(out.view(np.uint32), ref.cpu().numpy().view(np.uint32))
    return out, assoc.cpu().numpy()


def _check_edges(scene, poses, edges, out, assoc, what, dist_gate=0.02, stride=1):
    n_diff, worst, n_assoc = 0, 0.0, 0           # worst: max element-wise H error of the edges
    for e, (i, j) in enumerate(edges):          # where every pixel took the oracle's decision
        o, pix, border, allow = oracle.dense_edge(
            scene.depth[i], scene.normal[i], scene.mask[i], scene.depth[j], scene.normal[j], scene.mask[j],
            scene.K, poses[i], poses[j], dist_gate=dist_gate, stride=stride, want_pixels=True, want_allow=True)
        d, rel = parity.dense_decisions(out[e], assoc[e], o, pix, border, allow, f"{what} edge {i}->{j}")
        n_diff += d
        worst = max(worst, rel) if d == 0 else worst
        n_assoc += int(o[28])
    return n_diff, worst, n_assoc


@pytest.mark.parametrize("variant", ["gt", "perturbed"])
def test_dense_decisions_all_c2_edges(bt, torch, ctx, c2, variant):
    """All 240 directed edges of the C2 graph (16 nodes, 640x480): every pixel decision outside
    the band equals the oracle's, H/g/E element-wise within 1e-4."""
    poses = c2.node_poses() if variant == "gt" else c2.perturbed_poses(3)
    pairs = synth.all_pairs(16)
    edges = [tuple(x) for p in pairs for x in ((p[0], p[1]), (p[1], p[0]))]
    assert len(edges) == 240
    out, assoc = gpu_assoc(bt, torch, ctx, c2, poses, edges)
    n_diff, worst, n_assoc = _check_edges(c2, poses, edges, out, assoc, variant)
    print(f"\n{variant}: {n_assoc} associated pixels over 240 edges, {n_diff} borderline pixels decided "
          f"differently (all inside the band), max element-wise H error {worst:.2e} of sum w|J_a J_b| on the "
          f"edges without a flipped pixel")
    assert worst < 1e-5
    assert n_assoc > 240 * 1000
    assert n_diff <= 1e-4 * n_assoc


@pytest.mark.parametrize("variant", ["stride2", "gate5mm"])
def test_dense_decisions_variants(bt, torch, ctx, c2, variant):
    poses = c2.perturbed_poses(3)
    stride = 2 if variant == "stride2" else 1
    gate = 0.005 if variant == "gate5mm" else 0.02
    edges = [(0, 1), (1, 0), (0, 7), (5, 2), (15, 3), (9, 9), (4, 12), (12, 4)]
    out, assoc = gpu_assoc(bt, torch, ctx, c2, poses, edges, dist_gate_m=gate, stride=stride)
    _check_edges(c2, poses, edges, out, assoc, variant, dist_gate=gate, stride=stride)
    if stride == 2:
        assert (assoc[:, 1::2, :] == -1).all() and (assoc[:, :, 1::2] == -1).all()


def test_dense_decisions_c1_crop_and_ragged(bt, torch):
    """160x120 crop (C1) and a ragged 157x119 map (partial 32x32 tiles, W not a multiple of 4)."""
    sc, *_ = synth.make_pair_c1()
    c = bt.Context(0)
    c.reserve(2, 512, 256, 2, 160, 120)
    poses = sc.node_poses()
    edges = [(0, 1), (1, 0), (0, 0)]
    out, assoc = gpu_assoc(bt, torch, c, sc, poses, edges)
    _check_edges(sc, poses, edges, out, assoc, "c1")
    rag = synth.make_pair_c1()[0]
    rag.depth = np.ascontiguousarray(rag.depth[:, :119, :157])
    rag.normal = np.ascontiguousarray(rag.normal[:, :119, :157])
    rag.mask = np.ascontiguousarray(rag.mask[:, :119, :157])
    rag.K = synth.Intrinsics(rag.K.fx, rag.K.fy, rag.K.cx, rag.K.cy, 157, 119)
    out, assoc = gpu_assoc(bt, torch, c, rag, poses, edges)
    _check_edges(rag, poses, edges, out, assoc, "ragged")
    c.close()


def test_register_pairs_dense_blocks_are_the_associated_ones(bt, torch, ctx, c2):
    """bt_register_pairs' dense words (edges derived from the pairs, on the side stream) equal
    bt_dense_assoc's rows for the same directed edges bit for bit — the decisions checked above
    are the ones the product path takes."""
    pairs = synth.all_pairs(16)
    poses = c2.perturbed_poses(11)
    fb = bt.FrameBatch.from_scene(c2)
    rw = bt.record_words(512)
    rec = torch.zeros((len(pairs), rw), dtype=torch.int32, device="cuda")
    ctx.register_pairs(fb, c2.K, _dev(torch, poses), _dev(torch, np.asarray(pairs, np.int32)),
                       _dev(torch, np.arange(len(pairs), dtype=np.int32)), bt.ransac_params(4096, SEED),
                       bt.edge_params(), rec)
    torch.cuda.synchronize()
    r = bt.decode_records(rec, 512)
    edges = [tuple(x) for p in pairs for x in ((p[0], p[1]), (p[1], p[0]))]
    out, _ = gpu_assoc(bt, torch, ctx, c2, poses, edges)
    assert np.array_equal(r["dense_ij"].view(np.uint32), out[0::2].view(np.uint32))
    assert np.array_equal(r["dense_ji"].view(np.uint32), out[1::2].view(np.uint32))


def test_register_pairs_match_lists_and_feature_blocks(bt, torch, ctx, c2):
    """bt_register_pairs at the C2 size: its OWN match lists (bt_copy_matches) equal brute force
    on all 120 pairs, and every pair's Eq. (2) blocks equal the oracle's bto_feature_edge
    evaluated on the GPU's inlier set, element by element (unconditional)."""
    pairs = synth.all_pairs(16)
    P = len(pairs)
    poses = c2.perturbed_poses(11)
    fb = bt.FrameBatch.from_scene(c2)
    rw = bt.record_words(512)
    rec = torch.zeros((P, rw), dtype=torch.int32, device="cuda")
    ctx.register_pairs(fb, c2.K, _dev(torch, poses), _dev(torch, np.asarray(pairs, np.int32)),
                       _dev(torch, np.arange(P, dtype=np.int32)), bt.ransac_params(4096, SEED),
                       bt.edge_params(), rec)
    mt = torch.full((P, 512, 2), -7, dtype=torch.int32, device="cuda")
    nm = torch.zeros(P, dtype=torch.int32, device="cuda")
    ctx.copy_matches(mt, nm)
    torch.cuda.synchronize()
    r = bt.decode_records(rec, 512)
    mt, nm = mt.cpu().numpy(), nm.cpu().numpy()
    excluded, worst = 0, 0.0
    for p, (a, b) in enumerate(pairs):
        ml = mt[p, :nm[p]]
        o = oracle.match(c2.desc[a, :c2.n_kp[a]], c2.desc[b, :c2.n_kp[b]])
        excluded += parity.compare_matches(ml, o)
        assert r["n_matches"][p] == nm[p]
        pa, pb = c2.pts[a][ml[:, 0]], c2.pts[b][ml[:, 1]]
        of = oracle.feature_edge(pa, pb, r["mask"][p], poses[a], poses[b])
        assert of[91] == r["best_count"][p] > 100
        worst = max(worst, parity.feat_elementwise(r["feat"][p], of, f"pair {p} ({a},{b})"))
    print(f"\nmatch entries excluded by the band: {excluded}; max element-wise Eq. (2) H error {worst:.2e}")
    assert excluded <= 2


def test_refit_degenerate_status(bt, torch, ctx):
    """Status 3 on the GPU: 200 collinear points + one 1 cm off the line, identical in both
    frames (synth.make_nearly_collinear; the oracle pin is tests/test_oracle_ransac.py).  Samples
    holding the off-line point fit exactly (count M); the whole inlier set is degenerate for the
    refit (sigma ratio ~1.5e-4 < 1e-3), so T_refit = T_best and status = REFIT_DEGENERATE."""
    n_max = 512
    recs = []
    for seed in (0, 1, 2):
        pa, na, pb, nb, off = synth.make_nearly_collinear(seed=seed)
        M = len(pa)
        sc = synth.make_scene(2, render_maps=False, seed=seed)
        sc.n_kp = np.array([M, M], np.int32)
        sc.desc = np.zeros((2, n_max, 128), np.float32)
        sc.pts = np.zeros((2, n_max, 3), np.float32)
        sc.nrm = np.zeros((2, n_max, 3), np.float32)
        sc.pts[0, :M], sc.nrm[0, :M], sc.pts[1, :M], sc.nrm[1, :M] = pa, na, pb, nb
        fb = bt.FrameBatch.from_scene(sc)
        m = np.zeros((1, n_max, 2), np.int32)
        m[0, :M] = np.stack([np.arange(M), np.arange(M)], 1)
        rec = torch.zeros((1, bt.record_words(n_max)), dtype=torch.int32, device="cuda")
        cnt = torch.zeros((1, 512), dtype=torch.int32, device="cuda")
        ctx.ransac(fb, _dev(torch, np.array([[0, 1]], np.int32)), _dev(torch, np.array([7], np.int32)),
                   _dev(torch, m), _dev(torch, np.array([M], np.int32)), bt.ransac_params(512, SEED), rec, cnt)
        torch.cuda.synchronize()
        r = {k: v[0] for k, v in bt.decode_records(rec, n_max).items()}
        oc = oracle.ransac_counts(pa, na, pb, nb, 512, 7, SEED)
        fin = parity.compare_ransac(cnt.cpu().numpy()[0], r, oc, pa, na, pb, nb, what=f"collinear {seed}")
        assert fin is not None and fin["status"] == oracle.STATUS_REFIT_DEGENERATE
        assert r["status"] == bt.PAIR_REFIT_DEGENERATE and r["best_count"] == M
        assert np.array_equal(r["T_refit"].view(np.uint32), r["T_best"].view(np.uint32))
        recs.append(r)
    assert len(recs) == 3


def test_dense_map_epochs_stale_entries_and_wrap(bt, torch):
    """k_dense decides a target pixel's validity by the epoch tag of its map entry (no validity
    map): entries left by earlier calls on other frames must never count.  Two different scenes
    alternate on one context, through the epoch wrap (BT_DENSE_EPOCH0 starts the call counter
    three calls before it; the wrapping call clears every reserved entry — the maps are carved at
    their reserved size, so with more frames reserved than used the clear touches no other
    scratch): every call's dense blocks equal those of a fresh context."""
    import os
    scenes = [synth.make_scene(4, seed=s) for s in (61, 62)]
    pairs = synth.all_pairs(4)
    eprm = bt.edge_params()

    def dense(ctx, sc):
        fb = bt.FrameBatch.from_scene(sc)
        out = torch.zeros((2 * len(pairs), 32), dtype=torch.float32, device="cuda")
        edges = np.concatenate([pairs, pairs[:, ::-1]], 0).astype(np.int32)
        ctx.dense_corr(fb, sc.K, torch.from_numpy(sc.perturbed_poses(3)).cuda(),
                       torch.from_numpy(np.ascontiguousarray(edges)).cuda(), eprm, out)
        torch.cuda.synchronize()
        return out.cpu().numpy()

    want = []
    for sc in scenes:
        c = bt.Context(0)
        c.reserve(len(pairs), 512, 256, 4, 640, 480)
        want.append(dense(c, sc))
        c.close()
    assert not np.array_equal(want[0], want[1])
    os.environ["BT_DENSE_EPOCH0"] = str(65536 - 3)
    try:
        c = bt.Context(0)
        c.reserve(len(pairs), 512, 256, 9, 640, 480)     # more frames reserved than used: the
                                                          # wrap's clear must stay in the maps
    finally:
        os.environ.pop("BT_DENSE_EPOCH0", None)
    for k in range(8):                                  # epochs 65534, 65535, 1 (wrap), 2, ...
        got = dense(c, scenes[k % 2])
        assert np.array_equal(got, want[k % 2]), f"call {k}"
    c.close()


def test_dense_graph_replay_with_new_frames(bt, torch):
    """A CUDA graph of bt_dense_corr captured once and replayed on new frame content (the same
    device buffers, refilled): the epoch comes from device memory, bumped by every execution, so
    map entries the previous replay wrote for pixels no longer valid are never targets — each
    replay equals a fresh context's result for its frames."""
    scenes = [synth.make_scene(4, seed=s) for s in (71, 72)]
    pairs = synth.all_pairs(4)
    edges = torch.from_numpy(np.ascontiguousarray(np.concatenate([pairs, pairs[:, ::-1]], 0).astype(np.int32))).cuda()
    poses = torch.from_numpy(scenes[0].perturbed_poses(3)).cuda()
    eprm = bt.edge_params()
    want = []
    for sc in scenes:
        c = bt.Context(0)
        c.reserve(len(pairs), 512, 256, 4, 640, 480)
        fb = bt.FrameBatch.from_scene(sc)
        o = torch.zeros((edges.shape[0], 32), dtype=torch.float32, device="cuda")
        c.dense_corr(fb, sc.K, poses, edges, eprm, o)
        torch.cuda.synchronize()
        want.append(o.cpu().numpy())
        c.close()
    assert not np.array_equal(want[0], want[1])
    c = bt.Context(0)
    c.reserve(len(pairs), 512, 256, 4, 640, 480)
    fb = bt.FrameBatch.from_scene(scenes[0])
    out = torch.zeros((edges.shape[0], 32), dtype=torch.float32, device="cuda")
    s = torch.cuda.Stream()
    c.dense_corr(fb, scenes[0].K, poses, edges, eprm, out, stream=s)       # warm-up (attributes)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        c.dense_corr(fb, scenes[0].K, poses, edges, eprm, out, stream=s)
    for k in range(4):
        src = bt.FrameBatch.from_scene(scenes[k % 2])
        for name in ("depth", "normal", "mask"):
            getattr(fb, name).copy_(getattr(src, name))
        g.replay()
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy(), want[k % 2]), f"replay {k}"
    c.close()
