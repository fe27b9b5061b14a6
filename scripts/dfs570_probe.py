"""n=570 DFS-query A/B probe: one bounded solve of random:570,2,0 (R=62) with the
progress log on; prints the summed CUDA-event time of the first K DFS-phase
containment launches (deterministic sequence) and their query count.
Usage: SYNCHRO_B200_LIB=... python scripts/dfs570_probe.py [time_limit_s] [K]"""
import os, re, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tl = float(sys.argv[1]) if len(sys.argv) > 1 else 90
K = int(sys.argv[2]) if len(sys.argv) > 2 else 60
code = f"""
import sys; sys.path.insert(0, {ROOT!r})
from paper_2207_05495_b200 import native as sw
aut = sw.from_spec('random:570,2,0')
try:
    sw.solve_exact(aut, upper_bound=62, time_limit={tl})
except Exception as e:
    print('stopped', e)
"""
env = dict(os.environ, SYNCHRO_PROGRESS="1")
p = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
dfs = False
ms, q, n = 0.0, 0, 0
phase1 = 0.0
for line in p.stderr.splitlines():
    if "dfs r=" in line:
        dfs = True
    m = re.search(r"contain (exist|mark-proper) \|A\|=(\d+) \|B\|=(\d+) ([\d.]+) ms", line)
    if not m:
        continue
    if not dfs:
        phase1 += float(m.group(4))
    elif m.group(1) == "exist" and n < K:
        ms += float(m.group(4))
        q += int(m.group(3))
        n += 1
print(f"phase1 contain ms {phase1:.1f}; first {n} DFS exist launches: {ms:.1f} ms, {q} queries, "
      f"{ms / max(q, 1) * 1e6:.1f} ms per M queries", flush=True)
