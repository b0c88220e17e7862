"""Host-side sharding of the hot path over ranks (one process per GPU).

The reorder stream shards by global-batch range: global batches are
independent (src/reorder.cpp:319-396 reads one batch), so
rank r reorders its contiguous range with no data-path collective.  The
orchestration search shards tuples by sorted index modulo the rank count and
folds the per-rank winners with the BestTracker order
(src/orchestrator.cpp:211-233), which is a total order — the fold is
independent of the rank count.  The device fold of the same order is
dtb_best_reduce_dev; this module is its host restatement for the collective
layer (and the multi-rank CPU tests).
"""
from __future__ import annotations


def batch_range(n_batches: int, rank: int, world: int) -> tuple[int, int]:
    """(first batch, batch count) of `rank`: contiguous, sizes differ by <= 1."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"rank {rank} of {world}")
    base, extra = divmod(n_batches, world)
    first = rank * base + min(rank, extra)
    return first, base + (1 if rank < extra else 0)


def tuple_shard(n_tuples: int, rank: int, world: int) -> range:
    """Sorted tuple indices i with i % world == rank (strided: balances the
    early infeasible exits)."""
    return range(rank, n_tuples, world)


def best_key(c) -> tuple:
    """BestTracker::offer order (src/orchestrator.cpp:219-227): t_iter, total
    GPUs, the parallelism tuple, then the PP triple.  `c` is an
    api.Candidate."""
    p = c.plan
    return (c.times[2], p.total_gpus(), tuple(c.tuple),
            p.encoder.pp, p.backbone.pp, p.generator.pp)


def fold_winners(cands):
    """Winner over feasible candidates (None when none is feasible)."""
    best = None
    for c in cands:
        if c is None or not c.feasible:
            continue
        if best is None or best_key(c) < best_key(best):
            best = c
    return best
