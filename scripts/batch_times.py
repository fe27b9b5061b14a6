"""Per-instance solve time inside the config-2 batch at several thread counts
(how much concurrency inflates one solve)."""
import csv, os, sys, tempfile, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_05495_b200 import native as sw
for threads in [int(x) for x in (sys.argv[1:] or ["1", "4", "16"])]:
    p = tempfile.mktemp()
    t = time.perf_counter()
    sw.run_experiment([100], 2, 400, 0, p, solver="exact", threads=threads, deterministic=False)
    dt = time.perf_counter() - t
    ts = sorted(float(r["time_s"]) for r in csv.DictReader(open(p)))
    print(f"threads {threads}: {400 / dt:.0f} inst/s, per-instance mean {1e3 * sum(ts) / len(ts):.2f} ms "
          f"median {1e3 * ts[len(ts) // 2]:.2f} ms p90 {1e3 * ts[int(len(ts) * 0.9)]:.2f} ms", flush=True)
