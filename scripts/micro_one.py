"""One microbenchmark call (for ncu captures): expand image/preimage or dedupe
at 2^24 random parents.  Usage: micro_one.py img|pre|dedupe [spec]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_05495_b200 import native as sw
what = sys.argv[1]
aut = sw.from_spec(sys.argv[2] if len(sys.argv) > 2 else "random:300,2,0")
if what in ("img", "pre"):
    print(sw.bench_expand(aut, 1 << 24, 0.077, seed=1, inverse=what == "pre", iters=1))
else:
    print(sw.bench_dedupe(aut.n, 1 << 24, 0.077, seed=1, dup_fraction=0.1, iters=1))
