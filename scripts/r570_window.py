"""A bounded window of the random:570,2,0 solve (R = 62, relaxed DFS order):
python scripts/r570_window.py TIME_LIMIT [reference_order 0|1]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_05495_b200 import native as sw
aut = sw.from_spec("random:570,2,0")
t = time.perf_counter()
try:
    sw.solve_exact(aut, upper_bound=62, time_limit=float(sys.argv[1]),
                   dfs_reference_order=int(sys.argv[2]) if len(sys.argv) > 2 else 0)
except Exception as e:
    print("stopped", e)
print("wall", time.perf_counter() - t)
