"""Multi-process (gloo, world size 2, CPU) tests of the sharding / record all-gather plumbing
used under torchrun: the partitions of SURVEY §8(e) (track-major C4, pair-block
C5), and the exchange end to end on REAL records — each rank registers its shard of frame pairs
(the oracle stands in for the GPU on this CPU-only box; the records are packed in include/bt.h's
layout and decoded by the binding), all-gathers them, and assembles the pose-graph system of
Eq. (1) from the gathered blocks; every rank's records and system equal the
unsharded computation bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2108_00516_b200 import parallel


def test_shard_range_partition():
    for n in range(0, 40):
        for world in (1, 2, 3, 4, 8):
            blocks = [parallel.shard_range(n, world, r) for r in range(world)]
            assert blocks[0][0] == 0 and blocks[-1][1] == n
            for (a, b), (c, d) in zip(blocks, blocks[1:]):
                assert b == c
            sizes = [b - a for a, b in blocks]
            assert max(sizes) - min(sizes) <= 1
            assert max(sizes) == parallel.shard_capacity(n, world) or n == 0
    with pytest.raises(ValueError):
        parallel.shard_range(5, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n_total, words, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lo, hi = parallel.shard_range(n_total, world, rank)
        # a record's content depends only on its global pair id (as with Philox keyed by uid)
        ids = torch.arange(lo, hi, dtype=torch.int32)
        local = (ids[:, None] * 1000 + torch.arange(words, dtype=torch.int32)[None, :]).contiguous()
        full = parallel.all_gather_records(local, n_total)
        q.put((rank, full.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n_total", [8, 7, 1])
def test_all_gather_records_gloo_world2(n_total):
    world, words = 2, 5
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_total, words, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    expect = np.arange(n_total)[:, None] * 1000 + np.arange(words)[None, :]
    for r in range(world):
        assert np.array_equal(results[r], expect)


# ------------------------------------------------------- partitions (host logic, no processes)
def test_track_plan_partitions_the_batch():
    tp = np.array([(a, b) for a in range(4) for b in range(a + 1, 4)], np.int32)     # 6 pairs / track
    for world in (1, 2, 3, 4, 8):
        full = parallel.track_plan(8, 4, tp, 1, 0, uid_base=100)
        seen_pairs, seen_uids = [], []
        for r in range(world):
            p = parallel.track_plan(8, 4, tp, world, r, uid_base=100)
            assert p.rows == [len(tp) * (b - a) for a, b in (parallel.shard_range(8, world, q) for q in range(world))]
            assert p.row_lo == sum(p.rows[:r]) and len(p.pairs) == p.rows[r] == len(p.uids)
            assert p.pairs.min(initial=0) >= 0 and p.pairs.max(initial=-1) < p.frame_hi - p.frame_lo
            seen_pairs.append(p.pairs + p.frame_lo)
            seen_uids.append(p.uids)
        assert np.array_equal(np.concatenate(seen_pairs), full.pairs)
        assert np.array_equal(np.concatenate(seen_uids), full.uids)
        assert np.array_equal(full.uids, 100 + np.arange(48))


def test_pair_block_plan_partitions_the_batch():
    pairs = np.array([(a, b) for a in range(7) for b in range(a + 1, 7)], np.int32)   # 21 pairs
    for world in (1, 2, 4, 8):
        plans = [parallel.pair_block_plan(pairs, 7, world, r) for r in range(world)]
        assert np.array_equal(np.concatenate([p.pairs for p in plans]), pairs)
        assert np.array_equal(np.concatenate([p.uids for p in plans]), np.arange(21))
        assert all(p.frame_lo == 0 and p.frame_hi == 7 for p in plans)
        assert max(plans[0].rows) - min(plans[0].rows) <= 1


# ----------------------------------------- the exchange end to end on records in bt.h's layout
N_MAX, N_HYP, NF = 128, 256, 3
DENSE = dict(dist_gate=0.02, cos_gate=float(np.cos(np.deg2rad(45.0))), huber_delta=0.005, stride=1)


def _tracks(n_tracks):
    import synth
    return [synth.make_scene(NF, n=96, n_max=N_MAX, pool_size=400, width=160, height=120, distance=0.35,
                             seed=4000 + t) for t in range(n_tracks)]


def _words(n_max):
    return 28 + (n_max + 31) // 32 + 160          # bt_record_words (test_abi pins it on the library)


def _pack(o, n_max):
    """One oracle pair result in include/bt.h's record layout (status, M, h*, count*, T_best,
    T_refit, inlier mask, dense_ij[32], dense_ji[32], feat[96])."""
    w = np.zeros(_words(n_max), np.uint32)
    f = w.view(np.float32)
    w.view(np.int32)[:4] = [o["status"], o["n_matches"], o["best_hyp"], o["best_count"]]
    f[4:16] = o["T_best"]
    f[16:28] = o["T_refit"]
    mw = (n_max + 31) // 32
    w[28:28 + len(o["mask"])] = o["mask"][:mw]
    f[28 + mw:60 + mw] = o["dense_ij"][:32]
    f[60 + mw:92 + mw] = o["dense_ji"][:32]
    f[92 + mw:188 + mw] = o["feat"][:96]
    return w


def _register_shard(scenes, plan, node_poses):
    import oracle
    import synth
    out = []
    for (a, b), uid in zip(plan.pairs, plan.uids):
        ga, gb = plan.frame_lo + int(a), plan.frame_lo + int(b)
        t, la, lb = ga // NF, ga % NF, gb % NF
        assert gb // NF == t
        o = oracle.register_pair(scenes[t], la, lb, int(uid), N_HYP, synth.PHILOX_SEED,
                                 node_poses=node_poses[t], dense=DENSE)
        out.append(_pack(o, N_MAX))
    return np.stack(out) if out else np.zeros((0, _words(N_MAX)), np.uint32)


def _systems(records, n_tracks, track_pairs, node_poses):
    """Pose-graph system of each track from the gathered records (decoded by the binding)."""
    import oracle
    import paper_2108_00516_b200 as bt
    d = bt.decode_records(records, N_MAX)
    k = len(track_pairs)
    res = []
    for t in range(n_tracks):
        sl = slice(k * t, k * (t + 1))
        A, b, e = oracle.graph_system(node_poses[t], track_pairs, d["feat"][sl], d["dense_ij"][sl], d["dense_ji"][sl])
        res.append((A, b))
    return res


def _record_worker(rank, world, port, n_tracks, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import synth
        scenes = _tracks(n_tracks)
        tp = synth.all_pairs(NF)
        poses = [sc.perturbed_poses(seed=77 + t) for t, sc in enumerate(scenes)]
        plan = parallel.track_plan(n_tracks, NF, tp, world, rank)
        local = torch.from_numpy(_register_shard(scenes, plan, poses).view(np.int32))
        full = parallel.all_gather_rows(local, plan.rows)
        rec = full.numpy().view(np.uint32)
        q.put((rank, rec, _systems(rec, n_tracks, tp, poses)))
    finally:
        dist.destroy_process_group()


def test_records_exchange_end_to_end_gloo_world2():
    """Track-major (C4's partition) with an uneven split: 3 tracks over 2 ranks."""
    import synth
    world, n_tracks = 2, 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_record_worker, args=(r, world, port, n_tracks, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = {}
    for _ in range(world):
        r, rec, sy = q.get(timeout=300)
        results[r] = (rec, sy)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    scenes = _tracks(n_tracks)
    tp = synth.all_pairs(NF)
    poses = [sc.perturbed_poses(seed=77 + t) for t, sc in enumerate(scenes)]
    serial = _register_shard(scenes, parallel.track_plan(n_tracks, NF, tp, 1, 0), poses)
    ref_sys = _systems(serial, n_tracks, tp, poses)
    mw = (N_MAX + 31) // 32
    assert (serial.view(np.int32)[:, 0] == 0).sum() >= 1           # registered pairs ...
    assert serial.view(np.float32)[:, 28 + mw + 28].any()           # ... with associated dense pixels
    for r in range(world):
        rec, sy = results[r]
        assert np.array_equal(rec, serial), f"rank {r}: gathered records differ from the unsharded batch"
        for (A, b), (A0, b0) in zip(sy, ref_sys):
            assert np.array_equal(A, A0) and np.array_equal(b, b0)
