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
