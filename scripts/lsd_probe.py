import os, sys
sys.path.insert(0, "/root/repo")
from paper_2207_05495_b200 import native as sw
for lg in (20, 22, 24):
    ms, u = sw.bench_dedupe(300, 1 << lg, 0.077, seed=1, dup_fraction=0.1, iters=2, lex_sort=True)
    print(lg, f"{ms:.2f} ms")
