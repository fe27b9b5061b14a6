"""Bounded n=570 solve with the progress log (stderr -> gpurun_out/<name>.err):
python scripts/r570_progress.py NAME TIME_LIMIT [track_word]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_05495_b200 import native as sw
aut = sw.from_spec("random:570,2,0")
try:
    r = sw.solve_exact(aut, upper_bound=62, time_limit=float(sys.argv[2]), track_word=len(sys.argv) > 3)
    print(r.threshold, r.engine_seconds, r.expansions_dfs)
except Exception as e:
    print("stopped", e)
