"""Config 2 with P processes x T threads (instance shards, `--shard-index/--shard-count`):
each process has its own CUDA context, so host-side driver locks are not shared.
Checks every threshold against tests/golden/batch_n100_k2.json."""
import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
p = argparse.ArgumentParser()
p.add_argument("--samples", type=int, default=1000)
p.add_argument("--procs", type=int, default=4)
p.add_argument("--threads", type=int, default=2)
a = p.parse_args()

gold = {r[0]: r[2] for r in json.load(open(os.path.join(ROOT, "tests", "golden", "batch_n100_k2.json")))["rows"]}
child = (
    "import sys; sys.path.insert(0, {root!r}); from paper_2207_05495_b200 import native as sw; "
    "sw.run_experiment([100], 2, {samples}, 0, {csv!r}, threads={threads}, deterministic=True, "
    "shard_index={i}, shard_count={procs})")
with tempfile.TemporaryDirectory() as td:
    # warm the page cache / module load once
    subprocess.run([sys.executable, "-c", child.format(root=ROOT, samples=4, csv=os.path.join(td, "w.csv"),
                                                        threads=1, i=0, procs=1)], check=True)
    csvs = [os.path.join(td, f"s{i}.csv") for i in range(a.procs)]
    t = time.perf_counter()
    ps = [subprocess.Popen([sys.executable, "-c", child.format(root=ROOT, samples=a.samples, csv=csvs[i],
                                                               threads=a.threads, i=i, procs=a.procs)])
          for i in range(a.procs)]
    for q in ps:
        q.wait()
    dt = time.perf_counter() - t
    rows, bad = 0, 0
    for i, path in enumerate(csvs):
        for j, row in enumerate(open(path).read().splitlines()[1:]):
            f = row.split(",")
            idx = i + j * a.procs  # shard i holds grid indices i, i+P, ...
            thr = int(f[4]) if f[5] == "ok" else -2
            rows += 1
            if gold.get(idx) is not None and thr != gold[idx]:
                bad += 1
print(json.dumps({"procs": a.procs, "threads": a.threads, "samples": rows, "seconds": dt,
                  "instances_per_s": rows / dt, "mismatches_vs_reference": bad}))
