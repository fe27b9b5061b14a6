import os, sys, time, statistics
sys.path.insert(0, os.getcwd())
from paper_2207_05495_b200 import native as sw
for spec in ["random:300,2,0", "random:300,2,1", "random:200,3,0"]:
    aut = sw.from_spec(spec)
    b0 = sw.heuristic(aut, "adaptive")[0]
    ts = []
    for _ in range(3):
        t = time.perf_counter(); b = sw.heuristic(aut, "adaptive")[0]; ts.append(time.perf_counter() - t)
    print(spec, "bound", b, "adaptive ms", round(statistics.median(ts) * 1e3, 1), flush=True)
