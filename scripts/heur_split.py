"""Heuristic components of one instance: Eppstein, beam(max(64,n)), adaptive (ms)."""
import math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_05495_b200 import native as sw
aut = sw.from_spec(sys.argv[1] if len(sys.argv) > 1 else "random:300,2,0")
sw.heuristic(aut, "adaptive")
out = {}
for alg, beam in (("eppstein", 0), ("beam", max(64, aut.n)), ("adaptive", 0)):
    t = time.perf_counter()
    try:
        b, _ = sw.heuristic(aut, alg, beam_size=beam)
    except sw.SynchroError:
        b = None
    out[alg] = (b, round(1e3 * (time.perf_counter() - t), 2))
R = min(v[0] for v in out.values() if v[0])
e, bm = out["eppstein"][0], out["beam"][0]
r0 = min(x for x in (e, bm) if x)
target = 0.05 * 512 * aut.n * aut.k ** math.ceil(r0 / 2) / (512 * aut.k * r0)
print(out, "grown beam target", int(target))
