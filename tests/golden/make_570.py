"""Config-4 (n=570) pinning fixture from the REFERENCE itself (oracle/_ref).

A full reference solve of random:570,2,0 is out of reach (~1 day single-core,
SURVEY.md Appendix), so the fixture pins what the reference can compute in a
session:
  * R: the reference's own adaptive_upper_bound (heuristics.hpp:155-184) at the
    default 4 GiB budget;
  * the per-iteration trace prefix (bibfs_engine.hpp:442-460) of the
    instrumented replay with upper_bound = R, stopped between iterations after
    a wall-clock budget (ref_solve_instrumented max_seconds).
The GPU test replays the same prefix (stop_after_iterations) and compares the
lines byte for byte.

Usage: python tests/golden/make_570.py [adaptive|prefix|all] [max_seconds]
"""
from __future__ import annotations

import json
import os
import sys
import tempfile
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import ref as R  # noqa: E402

SPEC = (570, 2, 0)


def _update(path: str, fields: dict) -> None:
    # re-read before writing: the two halves may run as separate processes
    cur = json.load(open(path)) if os.path.exists(path) else {}
    cur.update(fields)
    json.dump(cur, open(path, "w"), indent=1)


def main(which: str, max_seconds: float) -> None:
    n, k, seed = SPEC
    d = R.random_automaton(n, k, seed)
    out_path = os.path.join(HERE, "solve_random_570_2_0_prefix.json")
    out = json.load(open(out_path)) if os.path.exists(out_path) else {
        "spec": "random:%d,%d,%d" % SPEC, "n": n, "k": k}
    if which in ("adaptive", "all"):
        t0 = time.time()
        L, word = R.adaptive(n, k, d)
        assert R.is_reset_word(n, k, d, word) and len(word) == L
        _update(out_path, {"spec": out["spec"], "n": n, "k": k, "ref_adaptive_upper_bound": L,
                           "ref_adaptive_seconds": round(time.time() - t0, 1)})
        print("adaptive R =", L, flush=True)
    if which in ("prefix", "all"):
        ub = int(os.environ.get("UB", out.get("ref_adaptive_upper_bound", 0)))
        with tempfile.TemporaryDirectory() as td:
            tp = os.path.join(td, "trace")
            t0 = time.time()
            s = R.solve_instrumented(n, k, d, tp, None, upper_bound=ub, max_seconds=max_seconds)
            fields = {"spec": out["spec"], "n": n, "k": k, "prefix_upper_bound": ub,
                      "prefix_status": s.status, "prefix_iterations": s.iterations,
                      "prefix_trace": s.trace or [], "prefix_ref_seconds": round(time.time() - t0, 1),
                      "prefix_expansions_phase1": s.expansions_phase1}
        _update(out_path, fields)
        print("prefix lines", len(fields["prefix_trace"]), flush=True)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "all",
         float(sys.argv[2]) if len(sys.argv) > 2 else 1800.0)
