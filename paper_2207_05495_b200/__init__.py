"""B200-native exact shortest-reset-word search (arXiv 2207.05495).

The product is the C++/CUDA library in csrc/ (built to lib/libsynchro_b200.so
and bin/synchro); this package only exposes it to Python through the C-ABI
(include/synchro_b200.h) — see native.py.
"""
from .native import (  # noqa: F401
    Automaton, Engine, SolveResult, SynchroError, NotSynchronizingError, OutOfMemoryError,
    DeviceError, cerny_automaton, random_automaton, parse_automaton, from_spec, instance_seed,
    is_synchronizing, is_reset_word, solve_exact, heuristic, power_set_oracle, run_experiment,
    load, version, device_count, LIB_PATH, CLI_PATH,
)
