"""Expansion / dedupe microbenchmarks: 2^24 random parents at
density 0.077, algorithmic GB/s against the measured HBM peak."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_05495_b200 import native as sw  # noqa: E402

peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json"))).get("hbm_gbs", 6554.6)
count = 1 << int(os.environ.get("MICRO_LOG2", "24"))
for spec in sys.argv[1:] or ["random:300,2,0"]:
    aut = sw.from_spec(spec)
    W = (aut.n + 63) // 64
    unit = 8 * W / aut.k + 8 * W + 4
    for inv in (False, True):
        ms = sw.bench_expand(aut, count, 0.077, seed=1, inverse=inv, iters=5)
        gbs = count * aut.k * unit / ms / 1e6
        print(f"{spec} {'preimage' if inv else 'image   '} {ms:7.3f} ms  {gbs:7.1f} GB/s  "
              f"frac {gbs / peak:.3f}")
    ms, u = sw.bench_dedupe(aut.n, count, 0.077, seed=1, dup_fraction=0.1, iters=3)
    row = 8 * W + 4
    gbs = (count * row + u * row) / ms / 1e6
    print(f"{spec} hash-dedupe {ms:7.3f} ms  {gbs:7.1f} GB/s  frac {gbs / peak:.3f}  unique {u}")
