"""Multi-process (gloo, world size 2, CPU) tests of the sharding / record all-gather plumbing
used under torchrun."""
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
