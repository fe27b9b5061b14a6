import os, sys, time
sys.path.insert(0, os.getcwd())
from paper_2207_05495_b200 import native as sw
aut = sw.from_spec("random:300,2,0")
for i in range(4):
    t = time.perf_counter()
    r = sw.solve_exact(aut, track_word=True)
    wall = time.perf_counter() - t
    print(f"wall {wall*1e3:.1f} ms heuristic {r.heuristic_seconds*1e3:.1f} engine {r.engine_seconds*1e3:.1f} engine_dev {r.engine_device_ms:.1f} launches {r.kernel_launches}")
