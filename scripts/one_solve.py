"""One engine solve of a workload (for ncu launch lists / full captures)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_05495_b200 import native as sw
spec = sys.argv[1] if len(sys.argv) > 1 else "random:300,2,0"
ub = int(sys.argv[2]) if len(sys.argv) > 2 else 44
aut = sw.from_spec(spec)
r = sw.solve_exact(aut, upper_bound=ub)
print(spec, "threshold", r.threshold, "engine_ms", r.engine_device_ms, "launches", r.kernel_launches)
