"""Hash dedupe microbenchmark vs list size (table L2 residency)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_05495_b200 import native as sw
n = int(sys.argv[1]) if len(sys.argv) > 1 else 300
W = (n + 63) // 64
row = 8 * W + 4
for lg in (20, 21, 22, 23, 24, 25):
    cnt = 1 << lg
    ms, uniq = sw.bench_dedupe(n, cnt, 0.077, seed=1, dup_fraction=0.1, iters=5)
    print(f"n={n} 2^{lg}: {ms:.3f} ms  {(cnt + uniq) * row / ms / 1e6:.0f} GB/s  {ms / cnt * 1e9:.1f} ps/row", flush=True)
