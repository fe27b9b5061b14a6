"""Where a fresh process's first solve spends its time: CUDA init, first
context, first solves (lazy kernel loading)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_05495_b200 import native as sw
t = time.perf_counter(); sw.device_count(); t1 = time.perf_counter()
print(f"cuInit + device query {1e3 * (t1 - t):.0f} ms", flush=True)
for spec in ["cerny:4", "random:100,2,0", "random:100,2,1", "random:300,2,0", "random:300,2,0"]:
    t = time.perf_counter()
    sw.solve_exact(sw.from_spec(spec))
    print(f"{spec}: {1e3 * (time.perf_counter() - t):.0f} ms", flush=True)
