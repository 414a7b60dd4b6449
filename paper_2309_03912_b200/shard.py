"""Multi-GPU file sharding.

Units never resolve symbols across files (sema.py:152-218 works on one unit),
so a corpus shards across ranks with no data-path collective: each rank takes
a contiguous, byte-balanced range of the path-sorted corpus, analyses it on
its own GPU, and the ordered per-file results are gathered to rank 0 in rank
order -- which is path order, the order ``Diagnostic.sort_key`` imposes
(diagnostics.py:73-74).  One process per GPU, ``torch.distributed`` for the
plumbing (NCCL on the GPU box, gloo in the CPU tests).
"""
from __future__ import annotations

import bisect
from typing import Callable, Optional, Sequence


def shard_ranges(sizes: Sequence[int], world: int) -> list:
    """Contiguous ranges [lo, hi) of ``sizes`` with near-equal byte totals.

    Rank r gets the files whose byte prefix midpoints fall in
    [r * total / world, (r + 1) * total / world); every file lands on exactly
    one rank and ranks stay in input order.
    """
    if world < 1:
        raise ValueError("world must be >= 1")
    n = len(sizes)
    prefix = [0]
    for s in sizes:
        prefix.append(prefix[-1] + int(s))
    total = prefix[-1]
    if total == 0:
        # equal counts when there is nothing to balance
        return [(n * r // world, n * (r + 1) // world) for r in range(world)]
    mids = [(prefix[i] + prefix[i + 1]) / 2.0 for i in range(n)]
    bounds = [bisect.bisect_left(mids, total * r / world) for r in range(world)] + [n]
    return [(bounds[r], bounds[r + 1]) for r in range(world)]


def my_shard(units: Sequence, rank: int, world: int, size_of: Callable = None) -> tuple:
    size_of = size_of or (lambda u: len(u[1].encode("utf-8", "surrogateescape")))
    lo, hi = shard_ranges([size_of(u) for u in units], world)[rank]
    return lo, hi


def gather_in_rank_order(local: list, rank: int, world: int, group=None) -> Optional[list]:
    """Concatenate every rank's list on rank 0 in rank order (None elsewhere)."""
    import torch.distributed as dist
    if world == 1:
        return list(local)
    bucket = [None] * world if rank == 0 else None
    dist.gather_object(local, bucket, dst=0, group=group)
    if rank != 0:
        return None
    out = []
    for part in bucket:
        out.extend(part)
    return out


def analyze_sharded(units: Sequence, rank: int, world: int,
                    analyze_batch: Optional[Callable] = None, device: Optional[int] = None):
    """Analyse this rank's shard and gather ordered results to rank 0.

    ``units`` are (path, text[, profile, mode, cfg]) sorted by path;
    ``analyze_batch(shard) -> list`` defaults to the GPU engine on ``device``.
    Returns the full ordered list on rank 0 and None on other ranks.
    """
    lo, hi = my_shard(units, rank, world)
    shard = list(units[lo:hi])
    if analyze_batch is None:
        from .exspace import analyze_corpus
        dev = rank if device is None else device
        res = analyze_corpus(shard, device=dev) if shard else []
        local = [[(d.code, d.loc.file, d.loc.line, d.loc.col, d.message) for d in a.diagnostics]
                 for a in res]
    else:
        local = analyze_batch(shard)
    return gather_in_rank_order(local, rank, world)
