"""Heuristic vs engine split of single solves (wall clock)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_05495_b200 import native as sw
for spec in sys.argv[1:]:
    aut = sw.from_spec(spec)
    sw.solve_exact(aut)
    t = time.perf_counter()
    for _ in range(5):
        r = sw.solve_exact(aut)
    dt = (time.perf_counter() - t) / 5
    print(f"{spec}: wall {dt*1e3:.2f} ms heuristic {r.heuristic_seconds*1e3:.2f} ms engine {r.engine_seconds*1e3:.2f} ms launches {r.kernel_launches}")
