"""Shard invariance on the GPU: the partitions bench.py uses
under torchrun, run as virtual ranks one after another on ONE GPU (each shard a separate
bt_register_pairs call over only the frames that rank holds), concatenated in rank order, equal
the unsharded batch bit for bit — Philox is keyed by the global pair uid and every reduction is
fixed-order, so a record does not depend on which rank computes it or what else is in its batch.
No kernel of one virtual rank waits on another (B200_PROFILING: ranks that wait on each other
must not share a GPU)."""
import numpy as np
import pytest

import synth
from paper_2108_00516_b200 import parallel

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


def _cat(torch, scenes, field, idx):
    return torch.cat([torch.from_numpy(np.ascontiguousarray(getattr(scenes[i], field))) for i in idx], 0).cuda()


def _batch(bt, torch, scenes, idx):
    return bt.FrameBatch(*(_cat(torch, scenes, f, idx) for f in ("n_kp", "desc", "pts", "nrm", "depth", "normal",
                                                                 "mask")))


def _register(bt, torch, ctx, fb, K, poses, pairs, uids, n_max, n_hyp):
    rec = torch.zeros((len(pairs), bt.record_words(n_max)), dtype=torch.int32, device="cuda")
    ctx.register_pairs(fb, K, torch.from_numpy(np.ascontiguousarray(poses)).cuda(),
                       torch.from_numpy(np.ascontiguousarray(pairs, np.int32)).cuda(),
                       torch.from_numpy(np.ascontiguousarray(uids, np.uint32).view(np.int32)).cuda(),
                       bt.ransac_params(n_hyp, SEED), bt.edge_params(), rec)
    torch.cuda.synchronize()
    return rec.cpu().numpy()


def test_track_major_shards_equal_unsharded(bt, torch):
    """C4's partition: 8 tracks x 6 frames (15 pairs each, 640x480, 4096 hypotheses) — virtual
    ranks G = 2, 4, 8 each register only their own tracks' frames."""
    T, NF, S = 8, 6, 4
    scenes = [synth.make_scene(NF, seed=synth.DATA_SEED + s) for s in range(S)]
    tscene = [scenes[t % S] for t in range(T)]
    tp = synth.all_pairs(NF)
    poses = np.concatenate([tscene[t].perturbed_poses(seed=1000 + t) for t in range(T)])
    ctx = bt.Context(0)
    ctx.reserve(T * len(tp), 512, 4096, T * NF, 640, 480)
    full_plan = parallel.track_plan(T, NF, tp, 1, 0)
    full = _register(bt, torch, ctx, _batch(bt, torch, tscene, range(T)), scenes[0].K, poses, full_plan.pairs,
                     full_plan.uids, 512, 4096)
    rec = bt.decode_records(full, 512)
    assert (rec["status"] == 0).all() and rec["dense_ij"][:, 28].mean() > 5000
    for G in (2, 4, 8):
        parts = []
        for r in range(G):
            p = parallel.track_plan(T, NF, tp, G, r)
            t_lo, t_hi = p.frame_lo // NF, p.frame_hi // NF
            fb = _batch(bt, torch, tscene, range(t_lo, t_hi))
            parts.append(_register(bt, torch, ctx, fb, scenes[0].K, poses[p.frame_lo:p.frame_hi], p.pairs, p.uids,
                                   512, 4096))
            assert parts[-1].shape[0] == p.rows[r]
        assert np.array_equal(np.concatenate(parts), full), f"G = {G}: sharded records differ"
    ctx.close()


def test_pair_block_shards_equal_unsharded(bt, torch):
    """C5's partition: frames replicated on every rank, contiguous global pair-id blocks (uneven:
    28 pairs over 3 ranks too), n = 1024 keypoints, 8192 hypotheses."""
    NF = 8
    sc = synth.make_scene(NF, n=1024, n_max=1024, pool_size=3500, seed=5005, outlier_frac=0.16)
    pairs = synth.all_pairs(NF)
    poses = sc.perturbed_poses(7)
    ctx = bt.Context(0)
    ctx.reserve(len(pairs), 1024, 8192, NF, 640, 480)
    fb = bt.FrameBatch.from_scene(sc)
    full = _register(bt, torch, ctx, fb, sc.K, poses, pairs, np.arange(len(pairs)), 1024, 8192)
    assert (bt.decode_records(full, 1024)["status"] == 0).all()
    for G in (2, 3, 8):
        parts = []
        for r in range(G):
            p = parallel.pair_block_plan(pairs, NF, G, r)
            parts.append(_register(bt, torch, ctx, fb, sc.K, poses, p.pairs, p.uids, 1024, 8192))
        assert np.array_equal(np.concatenate(parts), full), f"G = {G}: sharded records differ"
    ctx.close()
