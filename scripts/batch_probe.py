import json, os, sys, tempfile
sys.path.insert(0, os.getcwd())
from paper_2207_05495_b200 import native as sw
golden = {row[1]: (row[0], row[2]) for row in json.load(open("tests/golden/batch_n100_k2.json"))["rows"]}
for threads in (4, 1):
    p = tempfile.mktemp()
    sw.run_experiment([100], 2, 1000, 0, p, solver="exact", threads=threads, deterministic=True)
    bad = []
    for line in open(p).read().splitlines()[1:]:
        f = line.split(",")
        i, thr = golden[int(f[2])]
        ok = (f[5] == "nonsync") if thr < 0 else (f[5] == "ok" and int(f[4]) == thr)
        if not ok: bad.append((i, int(f[2]), f[4], f[5], thr))
    print("threads", threads, "bad", len(bad), bad[:8], flush=True)
    for i, seed, got, st, thr in bad[:3]:
        aut = sw.random_automaton(100, 2, seed)
        try:
            r = sw.solve_exact(aut)
            print("  single solve", i, r.threshold, thr, r.phase, flush=True)
        except Exception as e:
            print("  single solve", i, "error", e, flush=True)
