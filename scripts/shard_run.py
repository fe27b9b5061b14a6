"""Per-shard DFS runs of one instance on one GPU (SolveOptions::dfs_shard_index/count).

On N GPUs the shards run concurrently with no communication except the final
MIN of their thresholds (distributed.py); run back to back on one B200, each
shard's engine time is what its own GPU would spend.  Appends one JSON line per
shard to the output file as it finishes (partial results survive a timeout).

usage: shard_run.py SPEC UPPER_BOUND SHARDS OUT.jsonl [FIRST_SHARD [COUNT]]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_05495_b200 import native as sw  # noqa: E402

spec, ub, shards, out = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
first = int(sys.argv[5]) if len(sys.argv) > 5 else 0
count = int(sys.argv[6]) if len(sys.argv) > 6 else shards - first
aut = sw.from_spec(spec)
for s in range(first, min(shards, first + count)):
    t = time.perf_counter()
    r = sw.solve_exact(aut, upper_bound=ub, dfs_shard_index=s, dfs_shard_count=shards)
    row = {"spec": spec, "shard": s, "shards": shards, "threshold": r.threshold,
           "upper_bound": ub, "used_dfs": bool(r.used_dfs), "engine_seconds": r.engine_seconds,
           "engine_device_ms": r.engine_device_ms, "expansions_phase1": r.expansions_phase1,
           "expansions_dfs": r.expansions_dfs, "wall_s": time.perf_counter() - t}
    with open(out, "a") as f:
        f.write(json.dumps(row) + "\n")
    print(json.dumps(row), flush=True)
