"""Sample sharding across workers / GPUs (driver.py:175-186).

Samples are independent units keyed on their *global* id, so any
contiguous partition of [0, N) reproduces the single-worker output
exactly (bench.py:123-153).  ``worker_ranges`` is the reference's split:
contiguous, sizes differing by at most one, larger ranges first.
"""

from __future__ import annotations


def worker_ranges(n: int, workers: int) -> list[tuple[int, int]]:
    workers = max(1, min(workers, n)) if n else 1
    base, extra = divmod(n, workers)
    ranges, start = [], 0
    for w in range(workers):
        size = base + (1 if w < extra else 0)
        ranges.append((start, start + size))
        start += size
    return ranges


def shard_for_rank(n: int, world_size: int, rank: int) -> tuple[int, int]:
    """This rank's sample-id range; ranks beyond n get an empty range."""
    ranges = worker_ranges(n, world_size)
    if rank < len(ranges):
        return ranges[rank]
    return (n, n)


def piece_ranges(n: int, world_size: int, rank: int, chunks: int) -> list[tuple[int, int]]:
    """This rank's shard cut into `chunks` contiguous pieces (worker_ranges of
    the shard); ranks with fewer samples than pieces get empty pieces at the
    end, so every rank has exactly `chunks` pieces (multigpu.ShardedJob
    gathers piece c of every rank together)."""
    lo, hi = shard_for_rank(n, world_size, rank)
    chunks = max(1, int(chunks))
    pieces = [(lo + a, lo + b) for a, b in worker_ranges(hi - lo, chunks)] if hi > lo else []
    return pieces + [(hi, hi)] * (chunks - len(pieces))
