"""Config-2 batch rate on the GPU: 1000 random n=100 solves through
run_experiment (experiment.hpp:133-188) at several thread counts."""
import os, sys, tempfile, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_05495_b200 import native as sw
for threads in [int(x) for x in (sys.argv[1:] or ["1", "8", "16", "32"])]:
    p = tempfile.mktemp()
    t = time.perf_counter()
    sw.run_experiment([100], 2, 1000, 0, p, solver="exact", threads=threads, deterministic=True)
    dt = time.perf_counter() - t
    print(f"threads {threads}: {dt:.2f} s, {1000 / dt:.0f} instances/s", flush=True)
