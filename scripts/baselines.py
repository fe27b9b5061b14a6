"""GPU-vs-reference lines for the configs the bench line does not cover,
measured in ONE run on the GPU box (its own host cores for the reference):

  * config 1  cerny:20 — exact solve, engine (R supplied) and end to end;
  * config 3  random:300,2,0 — one FULL reference solve (time to threshold),
              next to the GPU end-to-end time;
  * config 2  1000 random binary n=100 (instance_seed(0,100,i)) — the batch
              runner (experiment.hpp:133-188): GPU run_experiment vs the
              reference's run_experiment on all host cores.

Writes one JSON object (stdout and the path given).  The reference is
oracle/_ref (the unmodified headers, -O3), test infrastructure only.
Usage: python scripts/baselines.py OUT.json [--skip-full]"""
import json
import subprocess, os, sys, tempfile, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2207_05495_b200 import native as sw  # noqa: E402
from oracle import ref as R  # noqa: E402


def cpu_model():
    for line in open("/proc/cpuinfo"):
        if line.startswith("model name"):
            return line.split(":", 1)[1].strip()
    return "unknown"


def gpu_solve(spec, reps=3, **kw):
    aut = sw.from_spec(spec)
    sw.solve_exact(aut, **kw)  # warm-up
    best = None
    for _ in range(reps):
        t = time.perf_counter()
        r = sw.solve_exact(aut, **kw)
        wall = time.perf_counter() - t
        if best is None or wall < best[0]:
            best = (wall, r)
    return best


out = {"host_cpu": cpu_model(), "host_cores": os.cpu_count()}
# ---- config 1: C_20
aut = sw.from_spec("cerny:20")
wall, r = gpu_solve("cerny:20", track_word=True)
wall_e, re_ = gpu_solve("cerny:20", upper_bound=r.upper_bound)
d = R.cerny_automaton(20)
t = time.perf_counter()
rs = R.solve_exact(20, 2, d, track_word=1)
ref_wall = time.perf_counter() - t
rs_e = R.solve_instrumented(20, 2, d, upper_bound=r.upper_bound)
out["cerny20"] = {"threshold": r.threshold, "ref_threshold": rs.threshold,
                  "gpu_e2e_s": wall, "gpu_engine_device_ms": re_.engine_device_ms,
                  "gpu_engine_wall_s": wall_e, "gpu_launches": re_.kernel_launches,
                  "ref_e2e_s": ref_wall, "ref_engine_s": rs_e.engine_seconds,
                  "iterations": r.iterations, "cores": 1}
print(json.dumps({"cerny20": out["cerny20"]}), flush=True)
# ---- config 3: one full reference solve of random:300,2,0
if "--skip-full" not in sys.argv:
    wall, r = gpu_solve("random:300,2,0", track_word=True)
    d = R.random_automaton(300, 2, 0)
    t = time.perf_counter()
    rs = R.solve_exact(300, 2, d, track_word=1)
    ref_wall = time.perf_counter() - t
    out["random300_s0"] = {"threshold": r.threshold, "ref_threshold": rs.threshold,
                           "gpu_time_to_threshold_s": wall, "ref_time_to_threshold_s": ref_wall,
                           "speedup": ref_wall / wall, "cores": 1,
                           "ref_word_ok": bool(rs.word) and R.is_reset_word(300, 2, d, rs.word)}
    print(json.dumps({"random300_s0": out["random300_s0"]}), flush=True)
# ---- config 2: 1000 random binary n=100 through the batch runners
golden = {row[1]: row[2] for row in json.load(open(os.path.join(ROOT, "tests", "golden",
                                                                 "batch_n100_k2.json")))["rows"]}
rows = {}
with tempfile.TemporaryDirectory() as td:
    for threads in (8, 16):
        p = os.path.join(td, f"gpu{threads}.csv")
        t = time.perf_counter()
        sw.run_experiment([100], 2, 1000, 0, p, solver="exact", threads=threads, deterministic=True)
        rows[f"gpu_threads{threads}_s"] = time.perf_counter() - t
    # the same batch in a FRESH process (CUDA context creation, module loading and
    # the interpreter start included) — what a one-off batch run costs
    child = ("import sys; sys.path.insert(0, {r!r}); from paper_2207_05495_b200 import native as sw; "
             "sw.run_experiment([100], 2, 1000, 0, {p!r}, solver='exact', threads=16, "
             "deterministic=True)").format(r=ROOT, p=os.path.join(td, "cold.csv"))
    t = time.perf_counter()
    subprocess.run([sys.executable, "-c", child], check=True)
    rows["gpu_cold_process_threads16_s"] = time.perf_counter() - t
    ok = 0
    for line in open(p).read().splitlines()[1:]:
        f = line.split(",")
        thr = golden[int(f[2])]
        ok += (f[5] == "nonsync") if thr < 0 else (f[5] == "ok" and int(f[4]) == thr)
    cores = os.cpu_count() or 1
    p = os.path.join(td, "ref.csv")
    t = time.perf_counter()
    R.run_experiment([100], 2, 1000, 0, p, threads=cores)
    rows["ref_all_cores_s"] = time.perf_counter() - t
    rows["ref_cores"] = cores
rows["gpu_matches_golden"] = ok
best = min(v for k, v in rows.items() if k.startswith("gpu_threads"))
rows["gpu_instances_per_s"] = 1000 / best
rows["ref_instances_per_s"] = 1000 / rows["ref_all_cores_s"]
rows["gpu_cold_process_instances_per_s"] = 1000 / rows["gpu_cold_process_threads16_s"]
rows["note"] = ("gpu_threads*: warm process (context and kernels loaded by the solves above); "
                "gpu_cold_process*: a fresh interpreter + CUDA context for the batch alone")
out["batch_n100"] = rows
print(json.dumps({"batch_n100": rows}), flush=True)
json.dump(out, open(sys.argv[1], "w"), indent=1)
