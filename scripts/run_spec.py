"""Solve one generator spec on the GPU with a time limit; print result + trace path."""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_05495_b200 import native as sw
p = argparse.ArgumentParser()
p.add_argument("spec"); p.add_argument("--ub", type=int, default=0); p.add_argument("--time-limit", type=float, default=0)
p.add_argument("--trace", default=None); p.add_argument("--memory", type=int, default=4 << 30)
p.add_argument("--track-word", action="store_true")
a = p.parse_args()
aut = sw.from_spec(a.spec)
t = time.time()
try:
    r = sw.solve_exact(aut, trace_path=a.trace, upper_bound=a.ub, time_limit=a.time_limit, memory=a.memory,
                       track_word=a.track_word)
    out = {k: getattr(r, k) for k in ("threshold", "upper_bound", "iterations", "bfs_steps", "ibfs_steps",
                                      "used_dfs", "peak_memory", "expansions_phase1", "expansions_dfs",
                                      "heuristic_seconds", "engine_seconds", "phase", "kernel_launches")}
    if r.word is not None:
        out["word_ok"] = len(r.word) == r.threshold and sw.is_reset_word(aut, r.word)
except sw.SynchroError as e:
    out = {"error": str(e)}
out["spec"] = a.spec; out["wall_s"] = round(time.time() - t, 3)
print(json.dumps(out), flush=True)
