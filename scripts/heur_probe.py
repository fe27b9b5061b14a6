"""Time the parts of the adaptive upper bound (heuristics.hpp:155-184) at n=300."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_05495_b200 import native as sw  # noqa: E402

aut = sw.from_spec(sys.argv[1] if len(sys.argv) > 1 else "random:300,2,0")
for alg, beam in [("eppstein", 0), ("beam", max(64, aut.n)), ("adaptive", 0)]:
    sw.heuristic(aut, alg, beam_size=beam)
    t = time.perf_counter()
    for _ in range(3):
        b, _w = sw.heuristic(aut, alg, beam_size=beam)
    print(alg, beam, "bound", b, "ms", (time.perf_counter() - t) / 3 * 1e3)
