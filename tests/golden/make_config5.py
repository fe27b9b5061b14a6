"""Config 5 widened: slowly synchronizing series and a genuinely ternary
extremal automaton, as text-format fixtures (automaton.hpp:178-219) whose
thresholds are pinned by the REFERENCE's power-set oracle (oracle.hpp:17-57,
n <= 20) and whose solves are recorded from the reference's own solve_exact
(trace, counters, peak, DFS level log; same record as make_golden.py).

Families (n <= 20 so the oracle pins every threshold):
  * cerny:n, n = 13..19 (automaton.hpp:168-176; C_20 is in solve_small.json);
  * wielandt:n, n = 3..20 — the coloring of Wielandt's primitive digraph
    (delta(i,a) = delta(i,b) = i+1 for i < n-1, delta(n-1,a) = 0,
    delta(n-1,b) = 1), a slowly synchronizing series next to Černý's;
  * cerny_id:n, n = 4..12 — C_n with a third, identity letter (ternary);
  * ternary5_*: the n = 5 ternary automata at the Černý bound 16 found by
    find_ternary.c (letter a ranges over one representative per cycle type,
    b and c over all maps); ternary5_roman is the class in which no two
    letters synchronize (the Roman-type extremal automaton);
  * climb:n, n = 7..10 — binary automata found by local search for a large
    threshold (climb_slow.c), far above the random-automaton range.

Usage: python tests/golden/make_config5.py
"""
from __future__ import annotations

import json
import os
import subprocess
import sys
import tempfile
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import ref as R  # noqa: E402

# canonical tables from find_ternary.c (delta row-major, delta[q*3+x]); the
# first is the class in which every two-letter sub-automaton is not synchronizing
TERNARY5 = {
    "ternary5_roman": [0, 0, 1, 1, 2, 0, 3, 1, 4, 2, 1, 3, 4, 4, 2],
    "ternary5_cerny_ab": [0, 0, 1, 1, 1, 2, 2, 2, 3, 3, 3, 4, 0, 0, 0],
    "ternary5_cerny_ac": [0, 1, 1, 1, 2, 2, 2, 3, 3, 3, 4, 4, 0, 0, 0],
    "ternary5_mixed": [0, 0, 1, 1, 1, 2, 2, 2, 3, 3, 3, 4, 0, 4, 0],
}
# best automata of `climb_slow N 20 20000 N` (threshold, n, delta)
CLIMB = {
    7: [4, 0, 0, 6, 2, 3, 2, 4, 6, 5, 6, 3, 1, 1],
    8: [5, 2, 1, 0, 7, 3, 7, 1, 6, 7, 5, 1, 4, 6, 2, 4],
    9: [7, 5, 4, 2, 3, 1, 2, 6, 8, 8, 1, 0, 6, 3, 0, 2, 5, 4],
    10: [9, 5, 1, 0, 3, 2, 8, 8, 7, 6, 6, 9, 2, 3, 6, 1, 4, 4, 9, 7],
}


def wielandt(n):
    d = []
    for i in range(n):
        d += [i + 1, i + 1] if i < n - 1 else [0, 1]
    return d


def cerny_id(n):
    c = R.cerny_automaton(n).tolist()
    d = []
    for q in range(n):
        d += [c[2 * q], c[2 * q + 1], q]
    return d


def text(n, k, d):
    rows = [" ".join(str(d[q * k + x]) for x in range(k)) for q in range(n)]
    return f"{n} {k}\n" + "\n".join(rows) + "\n"


def record(name, n, k, d):
    import numpy as np
    delta = np.asarray(d, np.uint32)
    oracle = R.power_set_oracle(n, k, delta)
    with tempfile.TemporaryDirectory() as td:
        t0 = time.time()
        s = R.solve_instrumented(n, k, delta, os.path.join(td, "t"), os.path.join(td, "l"))
        wall = time.time() - t0
        s2 = R.solve_exact(n, k, delta, os.path.join(td, "t2"))
    assert s.threshold == s2.threshold == oracle, (name, s.threshold, s2.threshold, oracle)
    assert s.trace == s2.trace and s.peak_memory == s2.peak_memory, name
    return {"name": name, "n": n, "k": k, "text": text(n, k, d), "threshold": s.threshold,
            "oracle": oracle, "upper_bound": s.upper_bound, "iterations": s.iterations,
            "bfs_steps": s.bfs_steps, "ibfs_steps": s.ibfs_steps, "used_dfs": s.used_dfs,
            "peak_memory": s.peak_memory, "expansions_phase1": s.expansions_phase1,
            "expansions_dfs": s.expansions_dfs, "trace": s.trace or [],
            "dfs_levels": s.dfs_levels or [], "ref_wall_seconds": round(wall, 3)}


def main():
    out = []
    for n in range(13, 20):
        out.append(record(f"cerny:{n}", n, 2, R.cerny_automaton(n).tolist()))
    for n in range(3, 21):
        out.append(record(f"wielandt:{n}", n, 2, wielandt(n)))
    for n in range(4, 13):
        out.append(record(f"cerny_id:{n}", n, 3, cerny_id(n)))
    for name, d in TERNARY5.items():
        out.append(record(name, 5, 3, d))
    for n, d in CLIMB.items():
        out.append(record(f"climb:{n}", n, 2, d))
    for c in out:
        print(c["name"], c["threshold"], c["iterations"], c["ref_wall_seconds"], flush=True)
    with open(os.path.join(HERE, "slow_sync_series.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
