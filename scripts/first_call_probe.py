"""Fresh-process cost of the two config-2 instances that are slow only on
first use (one-time driver work), with the progress log timestamps."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_05495_b200 import native as sw
warm = sw.random_automaton(100, 2, 1)
t = time.perf_counter(); sw.solve_exact(warm); print(f"warm-up solve {1e3 * (time.perf_counter() - t):.1f} ms")
for seed in (12342737865669978812, 9676338588998210404):
    aut = sw.random_automaton(100, 2, seed)
    for rep in range(2):
        t = time.perf_counter()
        r = sw.solve_exact(aut)
        print(seed, rep, r.threshold, f"{1e3 * (time.perf_counter() - t):.1f} ms",
              f"heur {1e3 * r.heuristic_seconds:.1f} eng {1e3 * r.engine_seconds:.1f}", flush=True)
