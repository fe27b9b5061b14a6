"""Slowest config-2 instances (one thread): seed, threshold, solve ms."""
import csv, os, sys, tempfile
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_05495_b200 import native as sw
p = tempfile.mktemp()
sw.run_experiment([100], 2, 1000, 0, p, solver="exact", threads=1, deterministic=False)
rows = list(csv.DictReader(open(p)))
ts = sorted(rows, key=lambda r: -float(r["time_s"]))
tot = sum(float(r["time_s"]) for r in rows)
print(f"total {tot:.2f} s over {len(rows)}; top 20 take {sum(float(r['time_s']) for r in ts[:20]):.2f} s")
for r in ts[:20]:
    print(r["seed"], r["threshold"], f"{1e3 * float(r['time_s']):.1f} ms")
buckets = [0] * 8
for r in rows:
    t = float(r["time_s"]) * 1e3
    buckets[min(7, int(t // 5))] += t
print("ms spent by 5-ms bucket:", [round(b) for b in buckets])
