"""Data-parallel plumbing of the hot path (one process per GPU, torch.distributed).

Frame pairs (and object tracks) are independent given the node poses, so they shard with no
data-path collective: every rank registers its own block of pairs — Philox is keyed by the
GLOBAL pair uid, so each record is bitwise identical whichever rank computes it — and the
fixed-stride per-pair records are exchanged once with all_gather_into_tensor (NCCL over
NVLink / NVSwitch on B200; gloo in the CPU tests).  This is the exchange the pose-graph solve
 needs: every rank then holds every edge's blocks.  The paper builds the
pairs' correspondences "in parallel on GPU" on one GPU (§IV-D); the sharding
over GPUs is this build's.

Two partitions:
  * track-major (C4, `track_plan`): rank r owns whole tracks (their frames' maps and keypoints
    stay resident on that rank only; no input replication), 64 / G tracks each;
  * pair blocks (C5, `pair_block_plan`): the frames are replicated, rank r registers the
    contiguous global pair-id block shard_range(P, G, r).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def shard_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """Balanced contiguous block [lo, hi) of n items for `rank` of `world` (sizes differ by <= 1,
    lower ranks take the extra items)."""
    if world < 1 or not 0 <= rank < world or n < 0:
        raise ValueError("bad shard arguments")
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def shard_capacity(n: int, world: int) -> int:
    """Rows every rank contributes to the gather (the largest shard)."""
    return -(-n // world) if world > 0 else 0


@dataclass
class ShardPlan:
    """One rank's share of a multi-pair batch.

    frame_lo / frame_hi: the global frames this rank needs resident ([lo, hi));
    pairs: [P_r][2] int32 frame ids RELATIVE to frame_lo (what bt_register_pairs receives);
    uids: [P_r] uint32 global pair ids (the Philox counter word: shard-invariant records);
    rows: per-rank record counts (identical on every rank; the gather's layout);
    row_lo: this rank's first global record row."""
    frame_lo: int
    frame_hi: int
    pairs: np.ndarray
    uids: np.ndarray
    rows: list
    row_lo: int


def track_plan(n_tracks: int, frames_per_track: int, track_pairs: np.ndarray, world: int, rank: int,
               uid_base: int = 0) -> ShardPlan:
    """Track-major partition (C4): tracks shard_range(n_tracks, world, rank); track t's frames are
    [t F, (t + 1) F) globally, its pairs track_pairs + t F, its global pair uids
    uid_base + t |track_pairs| + k — so the rank's records are rows [t_lo |tp|, t_hi |tp|) of the
    unsharded batch, in order."""
    tp = np.asarray(track_pairs, np.int32).reshape(-1, 2)
    t_lo, t_hi = shard_range(n_tracks, world, rank)
    F, k = frames_per_track, len(tp)
    pairs = np.concatenate([tp + F * (t - t_lo) for t in range(t_lo, t_hi)]) if t_hi > t_lo else np.zeros((0, 2), np.int32)
    uids = (uid_base + k * t_lo + np.arange(k * (t_hi - t_lo))).astype(np.uint32)
    rows = [k * (b - a) for a, b in (shard_range(n_tracks, world, r) for r in range(world))]
    return ShardPlan(F * t_lo, F * t_hi, pairs.astype(np.int32), uids, rows, k * t_lo)


def pair_block_plan(pairs: np.ndarray, n_frames: int, world: int, rank: int, uid_base: int = 0) -> ShardPlan:
    """Pair-block partition (C5): the global pair list cut into contiguous blocks
    shard_range(P, world, rank); every rank holds all n_frames frames (replicated inputs)."""
    pr = np.asarray(pairs, np.int32).reshape(-1, 2)
    lo, hi = shard_range(len(pr), world, rank)
    rows = [b - a for a, b in (shard_range(len(pr), world, r) for r in range(world))]
    return ShardPlan(0, n_frames, pr[lo:hi].copy(), (uid_base + np.arange(lo, hi)).astype(np.uint32), rows, lo)


def all_gather_rows(local, rows, group=None):
    """All-gather a row-sharded tensor: rank r holds rows[r] rows (`rows` identical on every rank,
    in rank order).  One all_gather_into_tensor of shards padded to max(rows); returns the
    [sum(rows)][...] tensor in global row order on every rank."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if len(rows) != world:
        raise ValueError(f"{len(rows)} shard sizes for world size {world}")
    if local.shape[0] != rows[rank]:
        raise ValueError(f"rank {rank}: {local.shape[0]} local records, shard has {rows[rank]}")
    cap = max(rows) if rows else 0
    send = local
    if local.shape[0] != cap:
        send = torch.zeros((cap,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
        send[: local.shape[0]] = local
    out = torch.empty((world * cap,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(out, send.contiguous(), group=group)
    if all(r == cap for r in rows):
        return out
    return torch.cat([out[r * cap: r * cap + rows[r]] for r in range(world)], 0)


def all_gather_records(local, n_total: int, group=None):
    """All-gather per-pair records sharded by shard_range(n_total, world, rank)."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rows = [b - a for a, b in (shard_range(n_total, world, r) for r in range(world))]
    return all_gather_rows(local, rows, group)


class FusedRecordExchange:
    """NEXT-3: the record exchange fused into the producers.  Every rank allocates
    the full [sum(rows)][rw] gather buffer in symmetric memory (torch.distributed
    _symmetric_memory: each rank's buffer mapped into every other rank over NVLink / NVSwitch);
    the rank's context gets every rank's buffer address (bt_set_record_peers), so the kernels
    that produce a record word (RANSAC finish, Eq. (2) blocks, dense reduce) store it straight
    into row (row_lo + p) of all ranks' buffers — no all-gather kernel.  `finish()` is the one
    synchronisation: a symmetric-memory barrier on the stream, after which this rank's buffer
    holds every rank's records.  Needs the NCCL backend and peer access between the GPUs."""

    def __init__(self, ctx, rows, rw: int, group=None, device=None):
        import torch
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm

        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        if len(rows) != self.world:
            raise ValueError(f"{len(rows)} shard sizes for world size {self.world}")
        self.rows = list(rows)
        self.row_lo = int(sum(self.rows[: self.rank]))
        total = int(sum(self.rows))
        self.buf = symm.empty((max(total, 1), rw), dtype=torch.int32, device=device)
        pg = group if group is not None else dist.group.WORLD
        self.handle = symm.rendezvous(self.buf, pg.group_name)
        self.ptrs = [int(self.handle.buffer_ptrs[r]) for r in range(self.world)]
        self.ctx = ctx
        ctx.set_record_peers(self.ptrs, self.row_lo, max(total, 1))

    def finish(self):
        """Barrier over all ranks (stream-ordered after this rank's register_pairs): afterwards the
        local gather buffer holds every rank's records in global row order."""
        self.handle.barrier(channel=0)
        return self.buf[: sum(self.rows)]

    def close(self):
        self.ctx.set_record_peers([])

    @staticmethod
    def available(group=None) -> bool:
        try:
            import torch.distributed as dist
            import torch.distributed._symmetric_memory  # noqa: F401
            return dist.is_initialized() and dist.get_backend(group) == "nccl"
        except Exception:
            return False
