"""Data-parallel sharding of the global mini-batch.

The reference has no data parallelism; these are the host-side rules of the B200
build: contiguous row ranges, the first (B mod N) shards one row larger, every replica holding the
full parameters, gradients scaled by the GLOBAL batch (dlogits = (p - y) / B_global instead of
network.hpp:430's local divisor; lr / B_global for the RBM, energy.hpp:150), one allreduce of the
packed gradient buffer per step, then an identical update on every replica.
"""
from __future__ import annotations


def shard_bounds(batch: int, world: int, rank: int) -> tuple[int, int]:
    """Rows [lo, hi) of the global batch owned by `rank` (100 over 8 -> 13,13,13,13,12,12,12,12)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(batch, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return lo, hi


def shard_sizes(batch: int, world: int) -> list[int]:
    return [shard_bounds(batch, world, r)[1] - shard_bounds(batch, world, r)[0] for r in range(world)]
