"""Config 5's slowly synchronizing family as fixtures: every isomorphism class of
binary automata with n = 4, 5 (and n = 6 when --n6 is given) whose reset
threshold is within a few of the Černý bound (n-1)^2, found by exhaustive
search (find_slow.c), each threshold pinned by the REFERENCE's power-set
oracle (oracle.hpp:17) and each solve recorded from the reference's own
solve_exact (trace, counters, peak) like make_golden.py.

Found (this search): n = 4: two classes at r = 9 = (n-1)^2; n = 5: one class
at r = 16 (Černý's C_5); n = 6: two classes at r = 25 (Černý's C_6 and a
second one — Kari's automaton is the published n = 6 example reaching the
bound) and none at r = 24.  The reference itself cannot generate these (its
generators are cerny:N and random:N,K,S).

Usage:  python tests/golden/make_slow.py [--n6 FILES...]
        (FILES: outputs of `find_slow 6 23 PART PARTS`, e.g. run in parallel)
"""
from __future__ import annotations

import itertools
import json
import os
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import ref as R  # noqa: E402

MIN = {4: 7, 5: 13, 6: 23}


def canonical(n, delta):
    """Lexicographically least relabelling (state permutation, letter swap)."""
    best = None
    for perm in itertools.permutations(range(n)):
        inv = [0] * n
        for q, p in enumerate(perm):
            inv[p] = q
        for swap in (False, True):
            d = []
            for p in range(n):  # new state p = old state inv[p]
                q = inv[p]
                a, b = delta[2 * q], delta[2 * q + 1]
                if swap:
                    a, b = b, a
                d += [perm[a], perm[b]]
            t = tuple(d)
            if best is None or t < best:
                best = t
    return best


def classes(lines):
    out = {}
    for line in lines:
        f = [int(x) for x in line.split()]
        r, n, delta = f[0], f[1], f[2:]
        c = canonical(n, delta)
        out.setdefault(c, (r, n))
    return out


def solve(n, delta):
    d = R.np.asarray(delta, R.np.uint32) if hasattr(R, "np") else delta
    with tempfile.TemporaryDirectory() as td:
        tp, lp = os.path.join(td, "trace"), os.path.join(td, "levels")
        s = R.solve_instrumented(n, 2, d, tp, lp)
        s2 = R.solve_exact(n, 2, d, os.path.join(td, "trace2"))
    assert s.threshold == s2.threshold and s.trace == s2.trace
    return {
        "n": n, "k": 2, "delta": list(delta), "options": {},
        "status": s.status, "threshold": s.threshold, "upper_bound": s.upper_bound,
        "iterations": s.iterations, "bfs_steps": s.bfs_steps, "ibfs_steps": s.ibfs_steps,
        "used_dfs": s.used_dfs, "peak_memory": s.peak_memory,
        "expansions_phase1": s.expansions_phase1, "expansions_dfs": s.expansions_dfs,
        "trace": s.trace or [], "dfs_levels": s.dfs_levels or [],
    }


def main():
    import numpy as np
    R.np = np
    exe = os.path.join(tempfile.mkdtemp(), "find_slow")
    subprocess.run(["gcc", "-O2", "-o", exe, os.path.join(HERE, "find_slow.c")], check=True)
    lines = []
    for n in (4, 5):
        lines += subprocess.run([exe, str(n), str(MIN[n])], check=True, capture_output=True,
                                text=True).stdout.splitlines()
    if "--n6" in sys.argv:
        for path in sys.argv[sys.argv.index("--n6") + 1:]:
            lines += open(path).read().splitlines()
    cases = []
    for c, (r, n) in sorted(classes(lines).items(), key=lambda kv: (kv[1][1], -kv[1][0], kv[0])):
        delta = list(c)
        pinned = R.power_set_oracle(n, 2, np.asarray(delta, np.uint32))
        assert pinned == r, (n, delta, r, pinned)
        case = solve(n, delta)
        assert case["threshold"] == r
        case["name"] = f"slow{n}_r{r}_{len([x for x in cases if x['n'] == n])}"
        cases.append(case)
        print(case["name"], r, flush=True)
    with open(os.path.join(HERE, "slow_sync.json"), "w") as f:
        json.dump(cases, f, indent=1)
    print("wrote", len(cases), "cases")


if __name__ == "__main__":
    main()
