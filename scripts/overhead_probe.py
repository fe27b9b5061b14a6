"""Fixed per-solve cost on the GPU path: tiny automata (lists of a few sets) in a
loop, plus the n=100 heuristic alone — what bounds the config-2 batch."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_05495_b200 import native as sw  # noqa: E402


def per_call(fn, reps):
    fn()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    return (time.perf_counter() - t) / reps * 1e3


tiny = sw.cerny_automaton(4)
small = sw.random_automaton(10, 2, 3)
n100 = sw.random_automaton(100, 2, sw.instance_seed(0, 100, 7))
print("cerny:4 solve ms", per_call(lambda: sw.solve_exact(tiny), 50))
print("random:10 solve ms", per_call(lambda: sw.solve_exact(small), 50))
r = sw.solve_exact(n100)
print("n100 solve ms", per_call(lambda: sw.solve_exact(n100), 20), "R", r.upper_bound,
      "launches", r.kernel_launches)
print("n100 solve(ub given) ms", per_call(lambda: sw.solve_exact(n100, upper_bound=r.upper_bound), 20))
