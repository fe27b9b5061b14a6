"""Config 2 (BASELINE.json): 1000 random binary automata n=100, instance_seed(0,100,i).

Runs our experiment runner (exact solver, T host threads, each solve on its own
CUDA stream on the visible GPU(s)) and, optionally, the reference's own
run_experiment on all host cores (oracle/_ref); checks every threshold against
tests/golden/batch_n100_k2.json and prints one JSON line with instances/s.
"""
import argparse
import json
import os
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

p = argparse.ArgumentParser()
p.add_argument("--samples", type=int, default=1000)
p.add_argument("--threads", type=int, default=16)
p.add_argument("--reference", action="store_true", help="also time the reference on all cores")
a = p.parse_args()

from paper_2207_05495_b200 import native as sw  # noqa: E402

gold = {r[0]: r[2] for r in json.load(open(os.path.join(ROOT, "tests", "golden", "batch_n100_k2.json")))["rows"]}


def check(path):
    rows = open(path).read().splitlines()[1:]
    bad = 0
    for i, row in enumerate(rows):
        f = row.split(",")
        thr = int(f[4]) if f[5] == "ok" else -2
        if gold.get(i) is not None and thr != gold[i]:
            bad += 1
    return len(rows), bad


out = {"config": "1000 x random:100,2,instance_seed(0,100,i) exact", "samples": a.samples}
with tempfile.TemporaryDirectory() as td:
    sw.run_experiment([100], 2, 4, 0, os.path.join(td, "warm.csv"), threads=2, deterministic=True)
    t = time.perf_counter()
    sw.run_experiment([100], 2, a.samples, 0, os.path.join(td, "ours.csv"), threads=a.threads,
                      deterministic=True)
    dt = time.perf_counter() - t
    n, bad = check(os.path.join(td, "ours.csv"))
    out.update({"ours_seconds": dt, "ours_instances_per_s": n / dt, "ours_threads": a.threads,
                "mismatches_vs_reference": bad})
    if a.reference:
        from oracle import ref as R
        cores = os.cpu_count() or 1
        t = time.perf_counter()
        R.run_experiment([100], 2, a.samples, 0, os.path.join(td, "ref.csv"), threads=cores)
        rdt = time.perf_counter() - t
        out.update({"reference_seconds": rdt, "reference_instances_per_s": a.samples / rdt,
                    "reference_threads": cores})
print(json.dumps(out))
