"""End-to-end solve with word tracking (the bench's e2e call shape): wall time."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_05495_b200 import native as sw
for spec in sys.argv[1:] or ["random:300,2,0"]:
    aut = sw.from_spec(spec)
    sw.solve_exact(aut, track_word=True)
    t = time.perf_counter()
    for _ in range(5):
        r = sw.solve_exact(aut, track_word=True)
    dt = (time.perf_counter() - t) / 5
    ok = r.word is not None and len(r.word) == r.threshold and sw.is_reset_word(aut, r.word)
    print(f"{spec}: wall {dt * 1e3:.1f} ms heuristic {r.heuristic_seconds * 1e3:.1f} "
          f"engine {r.engine_seconds * 1e3:.1f} d2h {r.d2h_bytes} word_ok {ok}")
