"""Multi-GPU exact solve: DFS-phase partitioning, one process per GPU.

Every rank runs phase 1 (the list steps are deterministic, so all ranks hold
identical L_BFS / L_IBFS and write identical trace prefixes), then explores
only the DFS subtrees rooted in its contiguous share of L_IBFS
(`dfs_shard_index/dfs_shard_count`, engine.cpp DfsRunner::run).  The DFS
returns the minimum depth at which any subtree meets L_BFS, so the threshold
of the whole search is the MIN over ranks (one all-reduce); the word comes
from the lowest rank attaining it.  Every reduction inside a DFS slice keeps a
dominating set in the same slice, so the partition cannot lose the optimum
(DESIGN.md §6).

The collective layer is injected (torch.distributed by default; tests pass a
gloo process group on CPU with a stand-in solver).
"""
from __future__ import annotations

from typing import Callable, Optional


def combine(results):
    """(threshold, word, rank) of the best shard: minimal threshold, lowest rank."""
    best = min(results, key=lambda r: (r[0], r[2]))
    return best


def solve_exact_sharded(aut, rank: int, world: int, solve: Optional[Callable] = None,
                        group=None, **opts):
    """Run this rank's shard and combine over the process group.

    Returns (threshold, word, per-rank result).  `solve(aut, **opts)` defaults to
    native.solve_exact; it must return an object with .threshold and .word.
    """
    import torch.distributed as dist
    if solve is None:
        from . import native
        solve = native.solve_exact
    res = solve(aut, dfs_shard_index=rank, dfs_shard_count=world, **opts)
    gathered = [None] * world
    dist.all_gather_object(gathered, (int(res.threshold), res.word, rank), group=group)
    thr, word, _ = combine(gathered)
    return thr, word, res
