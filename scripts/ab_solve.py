"""A/B helper: median engine device time of repeated solves (R supplied).
Usage: SYNCHRO_B200_LIB=... python scripts/ab_solve.py [spec:R ...]"""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_05495_b200 import native as sw
for item in sys.argv[1:] or ["random:300,2,0:44", "random:300,2,1:39"]:
    spec, ub = item.rsplit(":", 1)
    aut = sw.from_spec(spec)
    ms = []
    for i in range(6):
        r = sw.solve_exact(aut, upper_bound=int(ub))
        if i:
            ms.append(r.engine_device_ms)
    print(f"{spec} threshold {r.threshold} engine_ms median {statistics.median(ms):.2f} "
          f"min {min(ms):.2f} launches {r.kernel_launches}", flush=True)
