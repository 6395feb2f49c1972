"""NEXT-2 decisions on the GPU against the oracle (§IV-B/C/E): bt_coarse_pose,
bt_select_keyframes (incl. the hand-worked golden example) and bt_pool_admit, and
the causal tracker built from them (paper_2108_00516_b200.tracker) on a short ORBIT replay:
every frame's keyframe selection equals the oracle's on the GPU's own pose estimates (stage
isolation), the pool grows by the oracle's novelty rule, and the tracked poses stay within a
drift bound of the synthetic ground truth."""
import os

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "keyframe_selection.txt")


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
    yield c
    c.close()


def _d(torch, a, dt=None):
    return torch.from_numpy(np.ascontiguousarray(a if dt is None else np.asarray(a, dt))).cuda()


def test_coarse_pose_bitwise(bt, torch, ctx):
    rng = np.random.default_rng(0)
    for status in (0, 1, 2, 3):
        rec = np.zeros(bt.record_words(512), np.uint32)
        rec[0] = status
        Tb = synth.pose12(synth.random_rotation(rng, 1.0), rng.normal(size=3) * 0.1)
        rec.view(np.float32)[4:16] = Tb
        prev = synth.pose12(synth.random_rotation(rng, 2.0), rng.normal(size=3) * 0.1 + [0, 0, 0.5])
        out = torch.zeros(12, dtype=torch.float32, device="cuda")
        ctx.coarse_pose(_d(torch, rec.view(np.int32)), _d(torch, prev), out)
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy(), oracle.coarse_pose(status, Tb, prev)), status


def _select(bt, torch, ctx, pool, n, cur, K, cap=None):
    cap = cap or max(len(pool), 1)
    pp = np.zeros((cap, 12), np.float32)
    pp[:len(pool)] = pool
    sel = torch.full((K,), -7, dtype=torch.int32, device="cuda")
    ns = torch.zeros(1, dtype=torch.int32, device="cuda")
    ctx.select_keyframes(_d(torch, pp), _d(torch, [n], np.int32), _d(torch, cur), K, sel, ns)
    torch.cuda.synchronize()
    return sel.cpu().numpy()[:int(ns.item())]


def test_select_golden_and_random_pools(bt, torch, ctx):
    g = {}
    for line in open(GOLDEN):
        w = line.split("#")[0].split()
        if w and w[0] != "novel":
            g[w[0]] = [float(x) for x in w[1:]]

    def rz(a):
        return synth.pose12(synth.rotvec_to_R(np.array([0, 0, np.deg2rad(a)])), np.array([0, 0, 0.5]))
    pool = np.stack([rz(a) for a in g["pool"]])
    assert _select(bt, torch, ctx, pool, len(pool), rz(g["cur"][0]), int(g["K"][0])).tolist() == \
        [int(x) for x in g["select"]]
    rng = np.random.default_rng(1)
    for N, K in ((1, 15), (7, 15), (15, 15), (40, 15), (300, 15), (1000, 30)):
        pool = np.stack([synth.pose12(synth.random_rotation(rng, 1.2), rng.normal(size=3)) for _ in range(N)])
        cur = synth.pose12(synth.random_rotation(rng, 1.2), np.zeros(3))
        got = _select(bt, torch, ctx, pool, N, cur, K, cap=N + 5)
        assert got.tolist() == oracle.select_keyframes(pool, cur, K).tolist(), (N, K)
    # the pool count is read from device memory: a smaller *n_pool ignores the tail
    assert _select(bt, torch, ctx, pool, 20, cur, K=15, cap=len(pool)).tolist() == \
        oracle.select_keyframes(pool[:20], cur, 15).tolist()


def test_pool_admit_sequence(bt, torch, ctx):
    """Frames along a 2 deg / frame orbit with jitter: the device pool grows exactly as the
    oracle's novelty rule says, frame by frame."""
    rng = np.random.default_rng(2)
    cap = 64
    pool = torch.zeros((cap, 12), dtype=torch.float32, device="cuda")
    n_pool = torch.zeros(1, dtype=torch.int32, device="cuda")
    adm = torch.zeros(1, dtype=torch.int32, device="cuda")
    ref = []
    for t in range(150):
        R = synth.rotvec_to_R(np.array([0.1 * np.sin(t / 9.0), np.deg2rad(2.0 * t), 0.0])) @ \
            synth.random_rotation(rng, np.deg2rad(0.5))
        cur = synth.pose12(R, np.array([0, 0, 0.5]))
        ctx.pool_admit(pool, n_pool, _d(torch, cur), np.deg2rad(10.0), adm)
        torch.cuda.synchronize()
        want = oracle.is_novel(np.array(ref).reshape(-1, 12), cur)
        assert int(adm.item()) == (len(ref) if want else -1), t
        if want:
            ref.append(cur)
    assert int(n_pool.item()) == len(ref) > 10
    assert np.array_equal(pool.cpu().numpy()[:len(ref)], np.array(ref, np.float32))


def test_causal_tracker_orbit(bt, torch):
    """The causal tracker (coarse pose from the consecutive pair -> keyframe selection -> current x
    keyframe registrations with the keyframe pairs' C_ij cached -> Gauss-Newton with I_0 fixed ->
    pool refresh / augmentation) on a 120-frame ORBIT replay: each frame's selection equals the
    oracle's on the tracker's own estimates, admissions follow the oracle's novelty rule, and the
    tracked poses stay within 1 deg / 5 mm of ground truth.  The replay sweeps 60 views (2 deg
    apart) forth and back, so the way back revisits pool keyframes."""
    from paper_2108_00516_b200 import tracker
    scene, gt = tracker.orbit_scene(views=60, point_noise=0.0005, seed=17)
    order = list(range(60)) + list(range(58, -1, -1))
    tr = tracker.Tracker(scene.K, n_max=512, n_hyp=1024, gn_iters=2, log=True)
    out = tr.run(scene, order, T0=gt[0])
    rot, trans = tracker.pose_errors(out["poses"], [gt[v] for v in order])
    assert rot.max() < 1.0 and trans.max() < 0.005, (rot.max(), trans.max())
    pool = []
    for t, fr in enumerate(out["log"]):
        if t > 0:
            sel = oracle.select_keyframes(np.array(fr["pool"]), fr["coarse"], 15)
            assert sel.tolist() == fr["sel"], t
        nov = oracle.is_novel(np.array(fr["pool_after_refresh"]).reshape(-1, 12), fr["pose"]) if t > 0 else True
        assert fr["admitted"] == nov, t
    assert out["pool_size"] >= 6
    tr.close()
