"""North-star kernel microbenchmarks: 2^24 random parents at
density 0.077 under random:300,2,0 (and n=570), expansion image/preimage and
the hash dedupe; prints GB/s of algorithmic bytes.  SYNCHRO_B200_LIB selects
the library (A/B)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_05495_b200 import native as sw
for spec in sys.argv[1:] or ["random:300,2,0", "random:570,2,0", "random:100,2,0"]:
    aut = sw.from_spec(spec)
    W = (aut.n + 63) // 64
    per = 8 * W / aut.k + 8 * W + 4
    cnt = 1 << 24
    out = []
    for inv in (False, True):
        ms = sw.bench_expand(aut, cnt, 0.077, seed=1, inverse=inv, iters=5)
        out.append(f"{'pre' if inv else 'img'} {ms:.3f} ms {cnt * aut.k * per / ms / 1e6:.0f} GB/s")
    ms, uniq = sw.bench_dedupe(aut.n, cnt, 0.077, seed=1, dup_fraction=0.1, iters=3)
    row = 8 * W + 4
    out.append(f"dedupe {ms:.3f} ms {(cnt + uniq) * row / ms / 1e6:.0f} GB/s")
    print(spec, " | ".join(out), flush=True)
