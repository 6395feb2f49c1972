"""BASELINE configs[3] (C4) and configs[4] (C5) at FULL size, each in ONE bt_register_pairs call
in the bench's launch configuration, with sampled pairs compared end to end with the oracle
(the full-size batches were only checked for batch invariance).
C4: 64 tracks x 120 pairs = 7680 pairs (1024 frames of 640x480 maps, 15360 dense edges, 4096
hypotheses), track-major global pair ids as parallel.track_plan gives them; C5: 64 frames,
n = 4096, 2016 pairs, 16384 hypotheses, 4032 dense edges."""
import numpy as np
import pytest

import oracle
import parity
import synth
from paper_2108_00516_b200 import parallel

pytestmark = pytest.mark.gpu

SEED = synth.PHILOX_SEED
DENSE = dict(dist_gate=0.02, cos_gate=float(np.cos(np.deg2rad(45.0))), huber_delta=0.005, stride=1)


@pytest.fixture(scope="module")
def bt():
    import paper_2108_00516_b200 as m
    return m


@pytest.fixture(scope="module")
def torch():
    import torch as t
    return t


def _register(bt, torch, ctx, fb, K, poses, pairs, uids, n_max, n_hyp):
    rec = torch.zeros((len(pairs), bt.record_words(n_max)), dtype=torch.int32, device="cuda")
    ctx.register_pairs(fb, K, torch.from_numpy(np.ascontiguousarray(poses)).cuda(),
                       torch.from_numpy(np.ascontiguousarray(pairs, np.int32)).cuda(),
                       torch.from_numpy(np.ascontiguousarray(uids, np.uint32).view(np.int32)).cuda(),
                       bt.ransac_params(n_hyp, SEED), bt.edge_params(), rec)
    torch.cuda.synchronize()
    return bt.decode_records(rec, n_max)


def _check_pair(sc, a, b, uid, n_hyp, poses, r, what):
    o = oracle.register_pair(sc, a, b, int(uid), n_hyp, SEED, node_poses=poses, dense=DENSE, counts_out=True)
    assert r["n_matches"] == o["n_matches"], what
    P_ = o["match"]["pairs"]
    ia, ib = P_[:, 0], P_[:, 1]
    parity.compare_ransac(None, r, o["counts"], sc.pts[a][ia], sc.nrm[a][ia], sc.pts[b][ib], sc.nrm[b][ib], what=what)
    parity.assert_dense_close(r["dense_ij"], o["dense_ij"], f"{what} ij")
    parity.assert_dense_close(r["dense_ji"], o["dense_ji"], f"{what} ji")


def test_c4_full_batch_sampled(bt, torch):
    T, NF, S = 64, 16, 8
    scenes = [synth.make_scene(NF, seed=synth.DATA_SEED + 100 + s) for s in range(S)]
    tsc = [scenes[t % S] for t in range(T)]
    tp = synth.all_pairs(NF)
    plan = parallel.track_plan(T, NF, tp, 1, 0)
    poses = np.concatenate([tsc[t].perturbed_poses(seed=2000 + t) for t in range(T)])

    def field(f):
        return torch.cat([torch.from_numpy(np.ascontiguousarray(getattr(x, f))).cuda() for x in tsc], 0)
    fb = bt.FrameBatch(*(field(f) for f in ("n_kp", "desc", "pts", "nrm", "depth", "normal", "mask")))
    P = len(plan.pairs)
    assert P == T * len(tp) == 7680
    ctx = bt.Context(0)
    ctx.reserve(P, 512, 4096, T * NF, 640, 480)
    rec = _register(bt, torch, ctx, fb, tsc[0].K, poses, plan.pairs, plan.uids, 512, 4096)
    ctx.close()
    del fb
    torch.cuda.empty_cache()
    assert (rec["status"] == 0).all()
    for p in (0, 1337, 2999, 5555, 7679):
        t, k = divmod(p, len(tp))
        a, b = tp[k]
        r = {kk: v[p] for kk, v in rec.items()}
        _check_pair(tsc[t], a, b, plan.uids[p], 4096, poses[t * NF:(t + 1) * NF], r, f"c4 pair {p} (track {t})")


def test_c5_full_batch_sampled(bt, torch):
    sc = synth.make_scene(64, n=4096, n_max=4096, pool_size=14000, seed=5005, outlier_frac=0.16)
    pairs = synth.all_pairs(64)
    assert len(pairs) == 2016
    uids = np.arange(len(pairs), dtype=np.uint32)
    poses = sc.perturbed_poses(7)
    fb = bt.FrameBatch.from_scene(sc)
    ctx = bt.Context(0)
    ctx.reserve(len(pairs), 4096, 16384, 64, 640, 480)
    rec = _register(bt, torch, ctx, fb, sc.K, poses, pairs, uids, 4096, 16384)
    ctx.close()
    del fb
    torch.cuda.empty_cache()
    assert (rec["status"] == 0).all()
    for p in (0, 1000, 2015):
        a, b = pairs[p]
        _check_pair(sc, a, b, uids[p], 16384, poses, {k: v[p] for k, v in rec.items()}, f"c5 pair {p}")
