"""Data-parallel plumbing of the hot path (one process per GPU, torch.distributed).

Frame pairs (and object tracks) are independent given the node poses, so they shard with no
data-path collective: every rank registers its own block of pairs — Philox is keyed by the
GLOBAL pair uid, so each record is bitwise identical whichever rank computes it — and the
fixed-stride per-pair records are exchanged once with all_gather_into_tensor (NCCL over
NVLink / NVSwitch on B200; gloo in the CPU tests).  This is the exchange the pose-graph solve
 needs: every rank then holds every edge's blocks.
"""
from __future__ import annotations


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


def all_gather_records(local, n_total: int, group=None):
    """All-gather per-pair records sharded by shard_range.  `local` is this rank's
    [hi - lo][words] tensor; returns the [n_total][words] tensor in global pair order on every
    rank.  Shards are padded to a common size for the single all_gather_into_tensor call."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    cap = shard_capacity(n_total, world)
    lo, hi = shard_range(n_total, world, rank)
    if local.shape[0] != hi - lo:
        raise ValueError(f"rank {rank}: {local.shape[0]} local records, shard has {hi - lo}")
    send = local
    if local.shape[0] != cap:
        send = torch.zeros((cap,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
        send[: local.shape[0]] = local
    out = torch.empty((world * cap,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(out, send.contiguous(), group=group)
    if cap * world == n_total:
        return out
    parts = []
    for r in range(world):
        a, b = shard_range(n_total, world, r)
        parts.append(out[r * cap: r * cap + (b - a)])
    return torch.cat(parts, 0)
