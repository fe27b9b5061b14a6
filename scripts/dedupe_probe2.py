import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_05495_b200 import native as sw
mode = sys.argv[1]
aut = sw.from_spec("random:300,2,0")
if "torch" in mode:
    import torch
    buf = torch.empty(512 << 20, dtype=torch.uint8, device="cuda:0"); buf.zero_(); torch.cuda.synchronize()
if "solve" in mode:
    for _ in range(3): sw.solve_exact(aut, upper_bound=44, timing=True)
if "expand" in mode:
    print("expand ms", sw.bench_expand(aut, 1 << 24, 0.077, iters=5), flush=True)
for rep in range(2):
    ms, u = sw.bench_dedupe(300, 1 << 24, 0.077, seed=1, dup_fraction=0.1, iters=3)
    print(mode, rep, "hash ms", round(ms, 3), flush=True)
