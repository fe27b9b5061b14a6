"""Multi-GPU exact solve, one process per GPU.

Two modes:

* `solve_exact_partitioned` (the north_star path, `sw_solve_exact_dist`): ONE solve
  partitioned by hash ownership of each subset — per level an all-to-all carries new
  subsets to their owner rank, which deduplicates them; containment runs against
  all-gathered lists; list statistics are all-reduced; the DFS runs interleaved shares
  with a MIN all-reduce.  Transport: NCCL (`make_comm("nccl")`) or
  host callbacks over a torch.distributed group (`make_comm("callback", group)`).
* `solve_exact_sharded` (DFS-phase sharding only, below):

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


# ------------------------------------------------------- partitioned solve
class TorchCallbacks:
    """Host-buffer collectives for sw_comm (SW_COMM_CALLBACK) over an
    initialised torch.distributed process group on CPU tensors (gloo): the
    engine stages its device buffers through host memory and calls these.
    Pairwise send/recv for the variable-size exchanges (gloo has no
    variable-size all-to-all), all_reduce for the statistics."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    @staticmethod
    def _view(ptr, nbytes):
        import ctypes
        import numpy as np
        import torch
        if nbytes == 0:
            return torch.empty(0, dtype=torch.uint8)
        arr = np.ctypeslib.as_array(ctypes.cast(ptr, ctypes.POINTER(ctypes.c_uint8)), (nbytes,))
        return torch.from_numpy(arr)

    def _exchange(self, sends, recvs):
        import torch.distributed as dist
        ops = []
        for r in range(self.world):
            if r == self.rank:
                if recvs[r].numel():
                    recvs[r].copy_(sends[r])
                continue
            if sends[r].numel():
                ops.append(dist.P2POp(dist.isend, sends[r], r, self.group))
            if recvs[r].numel():
                ops.append(dist.P2POp(dist.irecv, recvs[r], r, self.group))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()

    def all_to_allv(self, user, send, send_bytes, recv, recv_bytes):
        try:
            sb = [int(send_bytes[r]) for r in range(self.world)]
            rb = [int(recv_bytes[r]) for r in range(self.world)]
            st, rt = self._view(send, sum(sb)), self._view(recv, sum(rb))
            sends = list(st.split(sb)) if sum(sb) else [st[:0]] * self.world
            recvs = list(rt.split(rb)) if sum(rb) else [rt[:0]] * self.world
            self._exchange(sends, recvs)
            return 0
        except Exception:
            return 1

    def all_gather_v(self, user, send, nbytes, recv, recv_bytes):
        try:
            rb = [int(recv_bytes[r]) for r in range(self.world)]
            st, rt = self._view(send, int(nbytes)), self._view(recv, sum(rb))
            recvs = list(rt.split(rb)) if sum(rb) else [rt[:0]] * self.world
            self._exchange([st] * self.world, recvs)
            return 0
        except Exception:
            return 1

    def all_reduce_u64(self, user, values, count, op):
        import numpy as np
        import torch
        import torch.distributed as dist
        try:
            arr = np.ctypeslib.as_array(values, (int(count),))
            t = torch.from_numpy(arr.astype(np.int64))
            dop = {0: dist.ReduceOp.SUM, 1: dist.ReduceOp.MIN, 2: dist.ReduceOp.MAX}[int(op)]
            dist.all_reduce(t, op=dop, group=self.group)
            arr[:] = t.numpy().astype(np.uint64)
            return 0
        except Exception:
            return 1

    def callbacks(self):
        return (self.all_to_allv, self.all_gather_v, self.all_reduce_u64)


def make_comm(kind: str = "callback", group=None):
    """A native.Comm for this rank: "nccl" (rank 0 draws the unique id, one
    all_gather_object shares it) or "callback" (TorchCallbacks over `group`)."""
    import torch.distributed as dist
    from . import native
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    if kind == "nccl":
        box = [native.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(box, src=0, group=group)
        return native.Comm(rank, world, nccl_id=box[0])
    cb = TorchCallbacks(group)
    comm = native.Comm(rank, world, callbacks=cb.callbacks())
    comm._torch_callbacks = cb  # keep the bound methods alive
    return comm


def solve_exact_partitioned(aut, comm, trace_path=None, **opts):
    """sw_solve_exact_dist on this rank (all ranks call it): the frontier lists
    are partitioned by hash ownership, the per-level exchange is one
    all-to-all, the trace and threshold are the single-GPU solve's."""
    from . import native
    return native.solve_exact_dist(aut, comm, trace_path=trace_path, **opts)
