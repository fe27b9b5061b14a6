"""Quick GPU probe: solve golden cases, compare trace/threshold, print timings."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_05495_b200 import native as sw

G = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")
names = sys.argv[1:] or ["solve_random_300_2_0.json"]
for name in names:
    case = json.load(open(os.path.join(G, name)))
    aut = sw.from_spec(case["spec"])
    for ub in (case["upper_bound"], 0):
        t = time.time()
        res = sw.solve_exact(aut, trace_path="/tmp/probe_trace.txt", upper_bound=ub, timing=1)
        wall = time.time() - t
        same = res.trace == case["trace"]
        print(f"{case['spec']} ub={ub}: thr={res.threshold} (ref {case['threshold']}) trace_equal={same} "
              f"peak={res.peak_memory} (ref {case['peak_memory']}) exp={res.expansions_phase1}+{res.expansions_dfs} "
              f"(ref {case['expansions_phase1']}+{case['expansions_dfs']}) heur={res.heuristic_seconds:.3f}s "
              f"engine={res.engine_seconds:.3f}s wall={wall:.3f}s expand_ms={res.expand_kernel_ms:.2f} "
              f"launches={res.kernel_launches} ref_engine={case['ref_engine_seconds']}s ref_heur={case['ref_heuristic_seconds']}s", flush=True)
        if not same:
            for i, (a, b) in enumerate(zip(res.trace, case["trace"])):
                if a != b:
                    print("first diff at line", i, "\n gpu:", a, "\n ref:", b)
                    break
