import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_05495_b200 import native as sw
for cnt in (1 << 20, 1 << 22, 1 << 24):
    for rep in range(2):
        ms, u = sw.bench_dedupe(300, cnt, 0.077, seed=1, dup_fraction=0.1, iters=3)
        ls, _ = sw.bench_dedupe(300, cnt, 0.077, seed=1, dup_fraction=0.1, iters=2, lex_sort=True)
        print(cnt, rep, "hash ms", round(ms, 3), "lex ms", round(ls, 3), "unique", u, flush=True)
