"""Multi-GPU exact solve: DFS-phase partitioning, one process per GPU.

Every rank runs phase 1 (the list steps are deterministic, so all ranks hold
identical L_BFS / L_IBFS and write identical trace prefixes), then explores
only the DFS subtrees rooted in its interleaved share of L_IBFS (rows
i ≡ shard_index mod shard_count; `dfs_shard_index/dfs_shard_count`,
engine.cpp DfsRunner::run).  The DFS
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


# ------------------------------------------------------------------ hash ownership
def owner_hash(words, W: int, nranks: int):
    """Owner rank of each row (numpy uint64 [N*W]) — the hash of exchange.cu,
    restated for the CPU tests: h = 0x9E3779B97F4A7C15; per word w:
    h = (h ^ w) * 0xff51afd7ed558ccd; h ^= h >> 32; owner = h mod nranks."""
    import numpy as np
    rows = np.asarray(words, np.uint64).reshape(-1, W)
    h = np.full(rows.shape[0], 0x9E3779B97F4A7C15, np.uint64)
    with np.errstate(over="ignore"):
        for w in range(W):
            h = (h ^ rows[:, w]) * np.uint64(0xFF51AFD7ED558CCD)
            h ^= h >> np.uint64(32)
    return (h % np.uint64(nranks)).astype(np.int64)


def owner_exchange_dedupe(n: int, words, cards, group=None, partition=None, dedupe=None):
    """Exact distributed dedupe of one generated level by hash ownership
    (SURVEY §8(e)): every rank regroups its rows owner-major (device kernel,
    sw_dev_owner_partition), ONE all-to-all (NCCL over NVLink on GPUs) carries
    each row to its owner, and the owner dedupes what it received
    (sw_dev_hash_dedupe).  Equal rows share an owner, so the union over ranks
    of the returned lists is the deduplicated level, each value on exactly one
    rank.  words: int64 view of the u64 rows [N*W], cards: int32 [N], on this
    rank's device.  Returns (words, cards, bytes_sent) — bytes_sent counts the
    rows this rank sent to other ranks (the NVLink payload).
    `partition`/`dedupe` are injectable for the CPU (gloo) tests."""
    import torch
    import torch.distributed as dist
    from . import native
    W = native.W(n)
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if partition is None:
        partition = lambda w, c, k: native.dev_owner_partition(n, w, c, k)  # noqa: E731
    if dedupe is None:
        dedupe = lambda w, c: native.dev_hash_dedupe(n, w, c)  # noqa: E731
    pw, pc, counts = partition(words, cards, world)
    send = torch.tensor(counts, dtype=torch.int64, device=cards.device)
    recv = torch.empty_like(send)
    dist.all_to_all_single(recv, send, group=group)
    rcounts = [int(x) for x in recv.tolist()]
    rw = torch.empty(sum(rcounts) * W, dtype=words.dtype, device=words.device)
    rc = torch.empty(sum(rcounts), dtype=cards.dtype, device=cards.device)
    dist.all_to_all_single(rw, pw, [c * W for c in rcounts], [c * W for c in counts], group=group)
    dist.all_to_all_single(rc, pc, rcounts, counts, group=group)
    bytes_sent = sum(c for r, c in enumerate(counts) if r != rank) * (8 * W + 4)
    ow, oc = dedupe(rw, rc)
    return ow, oc, bytes_sent
