"""Full random:570,2,0 solve (R = 62 supplied), exact vs relaxed DFS slice order:
python scripts/r570_ab.py OUT.json [0|1 reference order]"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_05495_b200 import native as sw
aut = sw.from_spec("random:570,2,0")
ro = int(sys.argv[2]) if len(sys.argv) > 2 else 1
t = time.perf_counter()
r = sw.solve_exact(aut, upper_bound=62, dfs_reference_order=ro, timing=True)
row = {"spec": "random:570,2,0", "dfs_reference_order": ro, "threshold": r.threshold,
       "engine_seconds": r.engine_seconds, "engine_device_ms": r.engine_device_ms,
       "wall_s": time.perf_counter() - t, "expansions_dfs": r.expansions_dfs,
       "expansions_phase1": r.expansions_phase1, "contain_kernel_ms": r.contain_kernel_ms,
       "peak_memory": r.peak_memory, "iterations": r.iterations}
json.dump(row, open(sys.argv[1], "w"))
print(json.dumps(row))
