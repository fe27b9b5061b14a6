"""The N>1 host paths on CPU with a world_size-2 gloo process group:
  * DFS-partitioned solve: shard bookkeeping + MIN combination
    (paper_2207_05495_b200/distributed.py) with a stand-in solver;
  * instance-sharded experiment runner (one process per GPU in production):
    the shards of the two ranks partition the rows of the single-process run
    (solver=oracle runs on the host)."""
import os
import subprocess
import sys
import tempfile

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

WORKER = r"""
import os, sys, json
sys.path.insert(0, {root!r})
import torch.distributed as dist
dist.init_process_group("gloo", init_method="tcp://127.0.0.1:{port}", rank=int(sys.argv[1]), world_size=2)
rank = dist.get_rank()
from paper_2207_05495_b200 import distributed, native

class Res:
    def __init__(self, t, w): self.threshold, self.word = t, w

def fake_solve(aut, dfs_shard_index, dfs_shard_count, **kw):
    assert dfs_shard_count == 2 and dfs_shard_index == rank
    # shard 1 finds a shorter word in its half of L_IBFS
    return Res(7 if dfs_shard_index == 1 else 9, [dfs_shard_index] * (7 if dfs_shard_index == 1 else 9))

thr, word, mine = distributed.solve_exact_sharded(None, rank, 2, solve=fake_solve)
out = {{"rank": rank, "thr": thr, "word": word, "mine": mine.threshold}}
# instance sharding of the experiment runner (host-side oracle solver)
csv = os.path.join({tmp!r}, "shard%d.csv" % rank)
native.run_experiment([9, 10], 2, 8, 3, csv, solver="oracle", deterministic=True,
                      shard_index=rank, shard_count=2)
dist.barrier()
print(json.dumps(out))
dist.destroy_process_group()
"""


def test_two_rank_gloo_paths():
    import json
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    with tempfile.TemporaryDirectory() as tmp:
        code = WORKER.format(root=ROOT, port=port, tmp=tmp)
        procs = [subprocess.Popen([sys.executable, "-c", code, str(r)], stdout=subprocess.PIPE,
                                  stderr=subprocess.PIPE, text=True) for r in range(2)]
        outs = [p.communicate(timeout=240) for p in procs]
        for p, (o, e) in zip(procs, outs):
            assert p.returncode == 0, e
        res = [json.loads(o.strip().splitlines()[-1]) for o, _ in outs]
        for r in res:
            assert r["thr"] == 7 and r["word"] == [1] * 7
        assert {r["mine"] for r in res} == {7, 9}
        # the two instance shards partition the single-process rows
        from paper_2207_05495_b200 import native
        full = os.path.join(tmp, "full.csv")
        native.run_experiment([9, 10], 2, 8, 3, full, solver="oracle", deterministic=True)
        rows = []
        for r in range(2):
            rows += open(os.path.join(tmp, f"shard{r}.csv")).read().splitlines()[1:]
        assert sorted(rows) == sorted(open(full).read().splitlines()[1:])
        assert len(rows) == 16


def test_combine_prefers_min_then_lowest_rank():
    from paper_2207_05495_b200.distributed import combine
    assert combine([(5, "a", 0), (4, "b", 1), (4, "c", 2)]) == (4, "b", 1)


EXCHANGE_WORKER = r"""
import os, sys, json
sys.path.insert(0, {root!r})
import numpy as np
import torch
import torch.distributed as dist
dist.init_process_group("gloo", init_method="tcp://127.0.0.1:{port}", rank=int(sys.argv[1]), world_size=2)
rank = dist.get_rank()
from paper_2207_05495_b200 import distributed
n, W = 130, 3
rng = np.random.default_rng(5)
base = rng.integers(0, 2**63, size=(400, W), dtype=np.int64)
base[:, -1] &= ~((1 << 62) - 1)  # tail bits beyond n stay zero
mine = base[rng.integers(0, 400, 700 + 50 * rank)]  # both ranks draw from one pool: duplicates across ranks

def partition(w, c, k):  # test stand-in for the device kernel: same owner hash, grouped owner-major
    rows = w.numpy().reshape(-1, W)
    own = distributed.owner_hash(rows.view(np.uint64).reshape(-1), W, k)
    order = np.argsort(own, kind="stable")
    counts = np.bincount(own, minlength=k).tolist()
    return (torch.from_numpy(rows[order].reshape(-1).copy()), torch.from_numpy(c.numpy()[order].copy()),
            counts)

def dedupe(w, c):
    rows = w.numpy().reshape(-1, W)
    _, first = np.unique(rows, axis=0, return_index=True)
    return torch.from_numpy(rows[np.sort(first)].reshape(-1).copy()), c[np.sort(first)]

w = torch.from_numpy(mine.reshape(-1).copy())
c = torch.from_numpy(np.array([bin(int(x) & (2**64 - 1)).count("1") for x in mine.sum(axis=1)], np.int32))
ow, oc, sent = distributed.owner_exchange_dedupe(n, w, c, partition=partition, dedupe=dedupe)
out = {{"rank": rank, "rows": [list(map(int, r)) for r in ow.numpy().reshape(-1, W)], "sent": sent,
       "mine": [list(map(int, r)) for r in mine]}}
print(json.dumps(out))
dist.destroy_process_group()
"""


def test_owner_exchange_dedupe_two_ranks():
    """Hash-ownership exchange over a world_size-2 gloo group: every distinct row
    ends on exactly one rank (its owner), duplicates across ranks collapse."""
    import json
    import socket

    import numpy as np

    from paper_2207_05495_b200.distributed import owner_hash
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    code = EXCHANGE_WORKER.format(root=ROOT, port=port)
    procs = [subprocess.Popen([sys.executable, "-c", code, str(r)], stdout=subprocess.PIPE,
                              stderr=subprocess.PIPE, text=True) for r in range(2)]
    outs = [p.communicate(timeout=240) for p in procs]
    for p, (o, e) in zip(procs, outs):
        assert p.returncode == 0, e
    res = sorted((json.loads(o.strip().splitlines()[-1]) for o, _ in outs), key=lambda r: r["rank"])
    every = {tuple(r) for x in res for r in x["mine"]}
    got = [tuple(r) for x in res for r in x["rows"]]
    assert len(got) == len(set(got)) and set(got) == every
    for x in res:
        rows = np.array(x["rows"], np.int64).view(np.uint64).reshape(-1)
        assert (owner_hash(rows, 3, 2) == x["rank"]).all()
        sent_rows = sum(1 for r in x["mine"]
                        if owner_hash(np.array(r, np.int64).view(np.uint64), 3, 2)[0] != x["rank"])
        assert x["sent"] == sent_rows * (8 * 3 + 4)


def test_owner_hash_is_a_function_of_the_row():
    import numpy as np

    from paper_2207_05495_b200.distributed import owner_hash
    rows = np.arange(40, dtype=np.uint64).reshape(20, 2)
    a = owner_hash(rows.reshape(-1), 2, 8)
    b = owner_hash(np.concatenate([rows, rows[::-1]]).reshape(-1), 2, 8)
    assert (a == b[:20]).all() and (a[::-1] == b[20:]).all() and set(a.tolist()) <= set(range(8))


CALLBACK_WORKER = r"""
import ctypes as C, json, sys
import numpy as np
sys.path.insert(0, {root!r})
import torch.distributed as dist
dist.init_process_group("gloo", init_method="tcp://127.0.0.1:{port}", rank=int(sys.argv[1]),
                        world_size={world})
rank, world = dist.get_rank(), dist.get_world_size()
from paper_2207_05495_b200 import distributed, native
cb = distributed.TorchCallbacks()
# exactly the C signatures of sw_comm (include/synchro_b200.h), through ctypes thunks
a2a = native.A2A_CB(cb.all_to_allv)
ag = native.AG_CB(cb.all_gather_v)
ar = native.AR_CB(cb.all_reduce_u64)
# all_to_allv: rank r sends (r*10 + d) repeated (d+1) times to rank d
send = np.concatenate([np.full(d + 1, rank * 10 + d, np.uint8) for d in range(world)])
sb = (C.c_uint64 * world)(*[d + 1 for d in range(world)])
rb = (C.c_uint64 * world)(*[rank + 1 for _ in range(world)])
recv = np.zeros(sum(rb), np.uint8)
assert a2a(None, send.ctypes.data, sb, recv.ctypes.data, rb) == 0
# all_gather_v: rank r contributes r+1 bytes of value 100+r
mine = np.full(rank + 1, 100 + rank, np.uint8)
gb = (C.c_uint64 * world)(*[r + 1 for r in range(world)])
gath = np.zeros(sum(gb), np.uint8)
assert ag(None, mine.ctypes.data, mine.size, gath.ctypes.data, gb) == 0
# all_reduce_u64 sum / min / max
out = {{}}
for op in (0, 1, 2):
    v = (C.c_uint64 * 2)(rank + 5, 1000 - rank)
    assert ar(None, v, 2, op) == 0
    out[op] = list(v)
print(json.dumps({{"recv": recv.tolist(), "gath": gath.tolist(), "red": out}}))
dist.destroy_process_group()
"""


@pytest.mark.parametrize("world", [2, 3])
def test_partitioned_solve_host_collectives_gloo(world):
    """The host-buffer collectives the partitioned solve calls through sw_comm
    (distributed.TorchCallbacks over gloo, invoked via the C function-pointer
    types): variable-size all-to-all, all-gather and u64 all-reduces."""
    import json
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    code = CALLBACK_WORKER.format(root=ROOT, port=port, world=world)
    procs = [subprocess.Popen([sys.executable, "-c", code, str(r)], stdout=subprocess.PIPE,
                              stderr=subprocess.PIPE, text=True) for r in range(world)]
    outs = [p.communicate(timeout=240) for p in procs]
    for p, (o, e) in zip(procs, outs):
        assert p.returncode == 0, e[-2000:]
    res = [json.loads(o.strip().splitlines()[-1]) for o, _ in outs]
    for r, x in enumerate(res):
        assert x["recv"] == [v for src in range(world) for v in [src * 10 + r] * (r + 1)]
        assert x["gath"] == [v for src in range(world) for v in [100 + src] * (src + 1)]
        assert x["red"]["0"] == [sum(q + 5 for q in range(world)), sum(1000 - q for q in range(world))]
        assert x["red"]["1"] == [5, 1000 - (world - 1)]
        assert x["red"]["2"] == [world + 4, 1000]
