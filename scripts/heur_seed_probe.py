"""Heuristic parts for one config-2 instance: Eppstein, beam(max(64,n)), adaptive."""
import math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_05495_b200 import native as sw
seed = int(sys.argv[1]) if len(sys.argv) > 1 else 9676338588998210404
aut = sw.random_automaton(100, 2, seed)
sw.heuristic(aut, "eppstein")
for alg, beam in (("eppstein", 0), ("beam", 100), ("adaptive", 0)):
    t = time.perf_counter()
    b, _ = sw.heuristic(aut, alg, beam_size=beam)
    print(alg, b, f"{1e3 * (time.perf_counter() - t):.1f} ms", flush=True)
R = min(sw.heuristic(aut, "eppstein")[0], sw.heuristic(aut, "beam", beam_size=100)[0])
target = 0.05 * 100 * 2 ** math.ceil(R / 2) / (2 * R)
print("R", R, "grown beam target", target)
