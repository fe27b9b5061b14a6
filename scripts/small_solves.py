"""Full solves (heuristic included) of a few config-2 instances, for launch
lists: random:100,2,seed for seed in argv (default 0..4)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_05495_b200 import native as sw
for seed in [int(x) for x in (sys.argv[1:] or range(5))]:
    r = sw.solve_exact(sw.from_spec(f"random:100,2,{seed}"))
    print(seed, r.threshold, r.kernel_launches, f"{r.engine_device_ms:.3f}")
