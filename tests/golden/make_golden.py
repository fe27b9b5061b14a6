"""Regenerate the golden fixtures in tests/golden/ from the REFERENCE itself.

Runs the unmodified reference (oracle/_ref/libsynchro_ref.so, built from
/root/reference/proj/include by oracle/Makefile) and records, per instance:
the threshold, SolveResult counters, the ledger peak, the full per-iteration
trace (bibfs_engine.hpp:442-460 — the per-level frontier-size parity artifact),
the DFS per-recurse sizes (logged re-drive, oracle/ref_driver.cpp) and the
engine expansion count.

Usage:  python tests/golden/make_golden.py [small|medium|large|batch|all]
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


def gen(spec: str):
    kind, args = spec.split(":")
    if kind == "cerny":
        n = int(args)
        return n, 2, R.cerny_automaton(n)
    n, k, seed = (int(x) for x in args.split(","))
    return n, k, R.random_automaton(n, k, seed)


def solve_case(spec: str, **opts) -> dict:
    n, k, d = gen(spec)
    with tempfile.TemporaryDirectory() as td:
        tp, lp = os.path.join(td, "trace"), os.path.join(td, "levels")
        t0 = time.time()
        s = R.solve_instrumented(n, k, d, tp, lp, **opts)
        wall = time.time() - t0
        s2 = R.solve_exact(n, k, d, os.path.join(td, "trace2"), **opts)
    assert s.status == s2.status, (s.status, s2.status)
    assert s.threshold == s2.threshold and s.peak_memory == s2.peak_memory, spec
    assert s.trace == s2.trace, spec
    out = {
        "spec": spec, "n": n, "k": k, "options": opts,
        "status": s.status, "threshold": s.threshold, "upper_bound": s.upper_bound,
        "iterations": s.iterations, "bfs_steps": s.bfs_steps, "ibfs_steps": s.ibfs_steps,
        "used_dfs": s.used_dfs, "peak_memory": s.peak_memory,
        "expansions_phase1": s.expansions_phase1, "expansions_dfs": s.expansions_dfs,
        "ref_heuristic_seconds": round(s.heuristic_seconds, 3),
        "ref_engine_seconds": round(s.engine_seconds, 3), "ref_wall_seconds": round(wall, 3),
        "trace": s.trace or [], "dfs_levels": s.dfs_levels or [],
    }
    if k * n <= 4096 and s.status == 0:
        e, _ = R.eppstein(n, k, d)
        b = R.beam(n, k, d, max(64, n))
        out["eppstein"] = e
        out["beam_default"] = b[0] if b else 0
    return out


def write(name: str, obj) -> None:
    path = os.path.join(HERE, name)
    with open(path, "w") as f:
        json.dump(obj, f, indent=1)
    print("wrote", path, flush=True)


SMALL = ["cerny:%d" % n for n in range(2, 13)] + ["cerny:20"] + \
        ["random:%d,%d,%d" % (n, k, s) for n in (20, 50, 100) for k in (2, 3) for s in range(3)]
MEDIUM = ["random:200,2,1", "random:300,2,1", "random:100,3,0", "random:100,3,1"]
LARGE = ["random:300,2,0", "random:300,2,2", "random:200,3,0"]
# Budgets under which the DFS cuts its levels into slices (dfs_phase.hpp:52-56,
# :153-158), with and without word tracking (meet_find copies L_IBFS, meet_check
# permutes it: the top-level slices follow that order), plus non-default
# EngineTuning / TuningParams fields (bibfs_engine.hpp:27-37, cost_model.hpp:26-36).
SLICING = [("random:200,2,1", dict(upper_bound=37, memory=m, track_word=tw))
           for m in (4 << 20, 8 << 20, 16 << 20) for tw in (0, 1)] + \
          [("random:300,2,1", dict(upper_bound=39, memory=16 << 20, track_word=tw)) for tw in (0, 1)]
TUNING = [("cerny:16", dict(history_growth=1.5)),
          ("cerny:12", dict(history_growth=3.0)),
          ("random:200,2,1", dict(dfs_largest=500)),
          ("random:200,2,1", dict(dfs_largest=3000, memory=16 << 20)),
          ("random:100,2,5", dict(reduction_of_reduction=0.3)),
          ("random:150,2,4", dict(beam_initial=100, beam_cost_fraction=0.2)),
          ("random:100,3,2", dict(beam_initial=16, beam_cost_fraction=0.01))]


def main(which: str) -> None:
    if which in ("small", "all"):
        cases = [solve_case(s) for s in SMALL]
        # schedule independence + memory-budget sensitivity + word tracking
        for sched in ("bfs", "ibfs", "dfs"):
            cases.append(solve_case("random:50,2,0", schedule=sched))
            cases.append(solve_case("cerny:10", schedule=sched))
        for mem in (1 << 20, 4 << 20, 16 << 20):
            cases.append(solve_case("random:100,2,1", memory=mem))
        write("solve_small.json", cases)
        # power-set oracle KATs (oracle.hpp:17) on the SPEC acceptance grid
        kats = []
        for n in range(6, 13):
            for k in (2, 3):
                for i in range(40):
                    seed = R.instance_seed(12345, 10 * n + k, i)
                    d = R.random_automaton(n, k, seed)
                    kats.append({"n": n, "k": k, "seed": seed,
                                 "oracle": R.power_set_oracle(n, k, d)})
        write("powerset_kats.json", kats)
    if which in ("medium", "all"):
        write("solve_medium.json", [solve_case(s) for s in MEDIUM])
    if which in ("large", "all"):
        for s in LARGE:
            write("solve_" + s.replace(":", "_").replace(",", "_") + ".json", solve_case(s))
    if which in ("slicing", "all"):
        cases = []
        for spec, opts in SLICING:
            c = solve_case(spec, **opts)
            depths = {}
            for lv in c["dfs_levels"]:
                depths[lv["r"]] = depths.get(lv["r"], 0) + 1
            assert max(depths.values()) > 1, (spec, opts)  # the DFS really slices
            cases.append(c)
        cases += [solve_case(spec, **opts) for spec, opts in TUNING]
        write("solve_slicing.json", cases)
    if which in ("batch", "all"):
        # config 2: 1000 random binary automata n=100, instance_seed(0, 100, i)
        rows = []
        t0 = time.time()
        for i in range(1000):
            seed = R.instance_seed(0, 100, i)
            d = R.random_automaton(100, 2, seed)
            s = R.solve_exact(100, 2, d)
            rows.append([i, seed, s.threshold if s.status == 0 else -s.status])
        write("batch_n100_k2.json", {"seed_base": 0, "n": 100, "k": 2,
                                     "ref_seconds": round(time.time() - t0, 2), "rows": rows})


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "small")
