"""One full exact solve (heuristic included) of a workload; writes a JSON summary."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_05495_b200 import native as sw  # noqa: E402

spec, out = sys.argv[1], sys.argv[2]
aut = sw.from_spec(spec)
t = time.perf_counter()
r = sw.solve_exact(aut, track_word=True, trace_path=out + ".trace")
wall = time.perf_counter() - t
ok = r.word is not None and len(r.word) == r.threshold and sw.is_reset_word(aut, r.word)
row = {"spec": spec, "threshold": r.threshold, "upper_bound": r.upper_bound,
       "iterations": r.iterations, "bfs_steps": r.bfs_steps, "ibfs_steps": r.ibfs_steps,
       "used_dfs": bool(r.used_dfs), "peak_memory": r.peak_memory,
       "expansions_phase1": r.expansions_phase1, "expansions_dfs": r.expansions_dfs,
       "heuristic_seconds": r.heuristic_seconds, "engine_seconds": r.engine_seconds,
       "wall_s": wall, "word_verified": bool(ok)}
json.dump(row, open(out, "w"))
print(json.dumps(row))
