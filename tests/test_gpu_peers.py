"""NEXT-3: the fused record exchange — bt_register_pairs' producer kernels
(RANSAC finish, Eq. (2) blocks, dense reduce) store every record word into the peers' gather
buffers too (bt_set_record_peers), replacing the separate all-gather of the records (the pair
correspondences "built in parallel on GPU" that every rank's pose-graph solve needs, PAPER.md
P:62, §IV-D).  On one GPU the "peers" are local buffers standing in for the other ranks' mapped
gather buffers: nothing waits on anything (B200_PROFILING), and the stores are the same
generic stores a peer mapping receives."""
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


@pytest.fixture(scope="module")
def setup(bt, torch):
    NF = 6
    sc = synth.make_scene(NF, seed=synth.DATA_SEED + 7)
    pairs = synth.all_pairs(NF)                                   # 15 pairs
    fb = bt.FrameBatch.from_scene(sc, "cuda")
    ctx = bt.Context(0)
    ctx.reserve(len(pairs), sc.desc.shape[1], 1024, NF, sc.K.width, sc.K.height)
    poses = torch.from_numpy(np.ascontiguousarray(sc.perturbed_poses(seed=3))).cuda()
    tp = torch.from_numpy(np.ascontiguousarray(pairs, np.int32)).cuda()
    uid = torch.from_numpy((np.arange(len(pairs)) + 100).astype(np.uint32).view(np.int32)).cuda()
    return sc, fb, ctx, poses, tp, uid


def _run(bt, torch, setup, eprm=True):
    sc, fb, ctx, poses, tp, uid = setup
    rec = torch.full((tp.shape[0], bt.record_words(sc.desc.shape[1])), -7, dtype=torch.int32, device="cuda")
    ctx.register_pairs(fb, sc.K, poses, tp, uid, bt.ransac_params(1024, SEED), bt.edge_params() if eprm else None,
                       rec)
    torch.cuda.synchronize()
    return rec


@pytest.mark.parametrize("eprm", [True, False])
def test_records_reach_every_peer_row(bt, torch, setup, eprm):
    """3 peer buffers, local rows land at global rows [4, 4 + P): every peer row equals the local
    record bit for bit (header, mask, Eq. (2) and both Eq. (3) blocks), rows outside the block
    and words the call does not produce (eprm None: dense / feature words) stay untouched, and
    the local output is the same as without peers."""
    sc, fb, ctx, poses, tp, uid = setup
    P, rw = tp.shape[0], bt.record_words(sc.desc.shape[1])
    ref = _run(bt, torch, setup, eprm)
    rows, off = P + 9, 4
    peers = [torch.full((rows, rw), 1234567 + k, dtype=torch.int32, device="cuda") for k in range(3)]
    ctx.set_record_peers([t.data_ptr() for t in peers], off, rows)
    try:
        got = _run(bt, torch, setup, eprm)
    finally:
        ctx.set_record_peers([])
    assert torch.equal(got, ref)
    for k, t in enumerate(peers):
        blk = t[off:off + P]
        if eprm:
            assert torch.equal(blk, ref), k
        else:                                                     # RANSAC words only
            n_ransac = 28 + (sc.desc.shape[1] + 31) // 32
            assert torch.equal(blk[:, :n_ransac], ref[:, :n_ransac]), k
            assert bool((blk[:, n_ransac:] == 1234567 + k).all()), k
        assert bool((t[:off] == 1234567 + k).all()) and bool((t[off + P:] == 1234567 + k).all()), k
    # peers off again: no stores into the old buffers
    snap = peers[0].clone()
    _run(bt, torch, setup, eprm)
    assert torch.equal(peers[0], snap)


def test_peer_capacity_and_arguments(bt, torch, setup):
    sc, fb, ctx, poses, tp, uid = setup
    P, rw = tp.shape[0], bt.record_words(sc.desc.shape[1])
    buf = torch.zeros((P, rw), dtype=torch.int32, device="cuda")
    ctx.set_record_peers([buf.data_ptr()], 1, P)                  # row_offset + P > rows
    try:
        with pytest.raises(bt.BtError, match="ECAPACITY|capacity|peer rows"):
            _run(bt, torch, setup)
    finally:
        ctx.set_record_peers([])
    with pytest.raises(bt.BtError):
        ctx.set_record_peers([0], 0, P)                           # NULL peer
    with pytest.raises(bt.BtError):
        ctx.set_record_peers([buf.data_ptr()] * 9, 0, P)          # more than 8 peers
    with pytest.raises(bt.BtError):
        ctx.set_record_peers([buf.data_ptr()], -1, P)


def test_peers_in_a_captured_graph(bt, torch, setup):
    """The peer stores are kernel arguments: a CUDA graph captured with peers set replays them."""
    sc, fb, ctx, poses, tp, uid = setup
    P, rw = tp.shape[0], bt.record_words(sc.desc.shape[1])
    ref = _run(bt, torch, setup)
    peer = torch.zeros((P, rw), dtype=torch.int32, device="cuda")
    rec = torch.zeros((P, rw), dtype=torch.int32, device="cuda")
    ctx.set_record_peers([peer.data_ptr()], 0, P)
    try:
        s = torch.cuda.Stream()
        _ = _run(bt, torch, setup)                                # warm-up outside the capture
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            ctx.register_pairs(fb, sc.K, poses, tp, uid, bt.ransac_params(1024, SEED), bt.edge_params(), rec,
                               stream=s)
        peer.zero_()
        rec.zero_()
        g.replay()
        torch.cuda.synchronize()
    finally:
        ctx.set_record_peers([])
    assert torch.equal(rec, ref) and torch.equal(peer, ref)


_SYMM_SCRIPT = r"""
import os, sys, numpy as np, torch, torch.distributed as dist
sys.path.insert(0, os.environ["BT_ROOT"])
import synth, paper_2108_00516_b200 as bt
from paper_2108_00516_b200 import parallel
dist.init_process_group("nccl", rank=0, world_size=1)
torch.cuda.set_device(0)
NF = 6
sc = synth.make_scene(NF, seed=synth.DATA_SEED + 7)
pairs = synth.all_pairs(NF)
fb = bt.FrameBatch.from_scene(sc, "cuda")
ctx = bt.Context(0)
ctx.reserve(len(pairs), sc.desc.shape[1], 1024, NF, sc.K.width, sc.K.height)
poses = torch.from_numpy(np.ascontiguousarray(sc.perturbed_poses(seed=3))).cuda()
tp = torch.from_numpy(np.ascontiguousarray(pairs, np.int32)).cuda()
uid = torch.from_numpy((np.arange(len(pairs)) + 100).astype(np.uint32).view(np.int32)).cuda()
rw = bt.record_words(sc.desc.shape[1])
rec = torch.zeros((len(pairs), rw), dtype=torch.int32, device="cuda")
assert parallel.FusedRecordExchange.available()
ex = parallel.FusedRecordExchange(ctx, [len(pairs)], rw, device="cuda")
ctx.register_pairs(fb, sc.K, poses, tp, uid, bt.ransac_params(1024, synth.PHILOX_SEED), bt.edge_params(), rec)
out = ex.finish()
torch.cuda.synchronize()
assert torch.equal(out, rec), "gathered rows differ"
ex.close()
dist.destroy_process_group()
print("SYMM_OK")
"""


def test_fused_exchange_symmetric_memory_single_rank(tmp_path):
    """parallel.FusedRecordExchange end to end on a one-rank NCCL group: symmetric-memory
    allocation, rendezvous, the peer addresses handed to bt_set_record_peers, the barrier — the
    gathered table equals the records (world > 1 differs only in the number of peers)."""
    import os
    import socket
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        port = s_.getsockname()[1]
    env = dict(os.environ, BT_ROOT=root, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK="0", WORLD_SIZE="1")
    script = tmp_path / "symm.py"
    script.write_text(_SYMM_SCRIPT)
    r = subprocess.run([sys.executable, str(script)], env=env, capture_output=True, text=True, timeout=300)
    if "SYMM_OK" not in r.stdout and ("symmetric" in r.stderr.lower() or "not supported" in r.stderr.lower()):
        pytest.skip("symmetric memory unavailable on this box: " + r.stderr.strip().splitlines()[-1][:200])
    assert "SYMM_OK" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]
