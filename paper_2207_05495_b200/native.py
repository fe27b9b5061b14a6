"""ctypes binding of lib/libsynchro_b200.so (the C-ABI in include/synchro_b200.h).

This is the Python-side mirror of the reference's public API (solve_exact,
heuristics, power-set oracle, generators, text format) used by the tests and
bench.py.  It never falls back to CPU code: if the shared library is missing
or no CUDA device is present, the device-backed calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SYNCHRO_B200_LIB") or os.path.join(HERE, "lib", "libsynchro_b200.so")
CLI_PATH = os.path.join(HERE, "bin", "synchro")

SW_OK = 0
STATUS_NAMES = {0: "ok", 1: "error", 2: "nonsync", 3: "parse", 4: "oom", 5: "refused",
                6: "timeout", 10: "device"}
SCHEDULES = {"auto": 0, "bfs": 1, "ibfs": 2, "dfs": 3}
STEP_KINDS = ["BFS", "BFS_NH", "IBFS", "IBFS_NH", "DFS"]

EXPORTED_SYMBOLS = [
    "sw_version", "sw_last_error", "sw_device_count", "sw_default_options",
    "sw_random_automaton", "sw_cerny_automaton", "sw_instance_seed", "sw_parse_automaton",
    "sw_is_synchronizing", "sw_pair_distances", "sw_is_reset_word", "sw_solve_exact", "sw_heuristic",
    "sw_power_set_oracle", "sw_engine_create", "sw_engine_destroy", "sw_engine_choose",
    "sw_engine_step", "sw_engine_meet", "sw_engine_dfs", "sw_engine_stats_get",
    "sw_list_expand", "sw_list_lex_sort_dedupe", "sw_list_sort_card_desc_lex",
    "sw_list_dedupe_sorted", "sw_list_hash_dedupe", "sw_list_self_reduce_minimal", "sw_list_mark",
    "sw_list_meet_check", "sw_trie_node_count", "sw_run_experiment", "sw_exp_mark",
    "sw_step_costs", "sw_bench_expand", "sw_bench_dedupe", "sw_dev_owner_partition",
    "sw_dev_hash_dedupe", "sw_solve_exact_ex", "sw_meet_check_order", "sw_list_trie_exists",
    "sw_nccl_unique_id", "sw_comm_create", "sw_comm_destroy", "sw_solve_exact_dist",
]


class SynchroError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{STATUS_NAMES.get(code, code)}] {msg}")
        self.code = code


class NotSynchronizingError(SynchroError):
    pass


class OutOfMemoryError(SynchroError):
    pass


class TimeoutError_(SynchroError):
    pass


class DeviceError(SynchroError):
    pass


_ERRORS = {2: NotSynchronizingError, 4: OutOfMemoryError, 6: TimeoutError_, 10: DeviceError}


class SolveOptions(C.Structure):
    _fields_ = [
        ("memory", C.c_uint64), ("time_limit", C.c_double), ("track_word", C.c_int32),
        ("schedule", C.c_int32), ("upper_bound", C.c_uint64), ("set_cost", C.c_double),
        ("dfs_set_weight", C.c_double), ("dfs_check_weight", C.c_double),
        ("min_brute", C.c_uint32), ("min_leaf", C.c_uint32), ("dedupe_cadence", C.c_uint32),
        ("reduce_cadence", C.c_uint32), ("device", C.c_int32), ("timing", C.c_int32),
        ("dfs_shard_index", C.c_uint32), ("dfs_shard_count", C.c_uint32),
        ("contain_stats", C.c_int32), ("dfs_largest", C.c_uint64),
        ("history_growth", C.c_double), ("beam_initial", C.c_uint64),
        ("beam_cost_fraction", C.c_double), ("reduction_of_reduction", C.c_double),
        ("stop_after_iterations", C.c_uint64), ("dfs_reference_order", C.c_int32),
        ("pad_", C.c_int32),
    ]


class SolveResultC(C.Structure):
    _fields_ = [
        ("threshold", C.c_uint64), ("upper_bound", C.c_uint64), ("iterations", C.c_uint64),
        ("bfs_steps", C.c_uint64), ("ibfs_steps", C.c_uint64), ("peak_memory", C.c_uint64),
        ("used_dfs", C.c_int32), ("has_word", C.c_int32), ("word_len", C.c_uint64),
        ("expansions_phase1", C.c_uint64), ("expansions_dfs", C.c_uint64),
        ("heuristic_seconds", C.c_double), ("engine_seconds", C.c_double),
        ("expand_kernel_ms", C.c_double), ("kernel_launches", C.c_uint64),
        ("phase", C.c_char * 16), ("engine_device_ms", C.c_double), ("h2d_bytes", C.c_uint64),
        ("d2h_bytes", C.c_uint64), ("contain_kernel_ms", C.c_double), ("contain_bytes", C.c_uint64),
        ("contain_visits", C.c_uint64), ("contain_pairs", C.c_uint64),
    ]


A2A_CB = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.POINTER(C.c_uint64), C.c_void_p,
                     C.POINTER(C.c_uint64))
AG_CB = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.POINTER(C.c_uint64))
AR_CB = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_uint64), C.c_uint64, C.c_int32)
SW_COMM_NCCL, SW_COMM_CALLBACK = 1, 2


class CommDesc(C.Structure):
    _fields_ = [
        ("kind", C.c_int32), ("rank", C.c_int32), ("nranks", C.c_int32), ("pad", C.c_int32),
        ("nccl_id", C.c_uint8 * 128), ("user", C.c_void_p), ("all_to_allv", A2A_CB),
        ("all_gather_v", AG_CB), ("all_reduce_u64", AR_CB),
    ]


class EngineStats(C.Structure):
    _fields_ = [
        ("iteration", C.c_uint64), ("bound", C.c_uint64), ("lbfs", C.c_uint64),
        ("libfs", C.c_uint64), ("hbfs", C.c_uint64), ("hibfs", C.c_uint64),
        ("d_lbfs", C.c_double), ("d_libfs", C.c_double), ("ledger_used", C.c_uint64),
        ("ledger_peak", C.c_uint64),
    ]


_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_lib = None


def lib_path() -> str:
    return LIB_PATH


def load():
    """Load the native library (raises if it was not built — no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"native library missing: {LIB_PATH} — run __graft_entry__.build() "
                           "or make -C paper_2207_05495_b200")
    L = C.CDLL(LIB_PATH)
    L.sw_version.restype = C.c_char_p
    L.sw_last_error.restype = C.c_char_p
    L.sw_instance_seed.restype = C.c_uint64
    L.sw_instance_seed.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32]
    L.sw_default_options.argtypes = [C.POINTER(SolveOptions)]
    L.sw_random_automaton.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, _u32p]
    L.sw_cerny_automaton.argtypes = [C.c_uint32, _u32p]
    L.sw_parse_automaton.argtypes = [C.c_char_p, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32),
                                     C.c_void_p, C.c_size_t]
    L.sw_is_synchronizing.argtypes = [C.c_uint32, C.c_uint32, _u32p, C.POINTER(C.c_int32)]
    L.sw_pair_distances.argtypes = [C.c_uint32, C.c_uint32, _u32p, C.c_int32, C.c_void_p,
                                    C.c_size_t]
    L.sw_is_reset_word.argtypes = [C.c_uint32, C.c_uint32, _u32p, C.c_void_p, C.c_size_t,
                                   C.POINTER(C.c_int32)]
    L.sw_solve_exact.argtypes = [C.c_uint32, C.c_uint32, _u32p, C.POINTER(SolveOptions),
                                 C.POINTER(SolveResultC), C.c_void_p, C.c_size_t, C.c_char_p]
    L.sw_solve_exact_ex.argtypes = [C.c_uint32, C.c_uint32, _u32p, C.POINTER(SolveOptions),
                                    C.POINTER(SolveResultC), C.c_void_p, C.c_size_t, C.c_char_p,
                                    C.c_void_p, C.c_size_t, C.POINTER(C.c_size_t)]
    L.sw_list_trie_exists.argtypes = [C.c_uint32, _u64p, C.c_size_t, _u64p, C.c_size_t,
                                      C.POINTER(C.c_int32), C.POINTER(C.c_uint64),
                                      C.POINTER(C.c_uint64)]
    L.sw_nccl_unique_id.argtypes = [C.c_void_p]
    L.sw_comm_create.argtypes = [C.POINTER(CommDesc), C.POINTER(C.c_void_p)]
    L.sw_comm_destroy.argtypes = [C.c_void_p]
    L.sw_solve_exact_dist.argtypes = [C.c_uint32, C.c_uint32, _u32p, C.POINTER(SolveOptions),
                                      C.c_void_p, C.POINTER(SolveResultC), C.c_void_p, C.c_size_t,
                                      C.c_char_p, C.POINTER(C.c_uint64)]
    L.sw_meet_check_order.argtypes = [C.c_uint32, _u64p, C.c_size_t, _u64p, C.c_size_t,
                                      C.c_uint32, _u32p]
    L.sw_heuristic.argtypes = [C.c_uint32, C.c_uint32, _u32p, C.c_int32, C.c_uint64, C.c_uint64,
                               C.c_double, C.POINTER(C.c_uint64), C.c_void_p, C.c_size_t]
    L.sw_power_set_oracle.argtypes = [C.c_uint32, C.c_uint32, _u32p, C.c_double,
                                      C.POINTER(C.c_uint64)]
    L.sw_engine_create.argtypes = [C.c_uint32, C.c_uint32, _u32p, C.POINTER(SolveOptions),
                                   C.c_uint64, C.POINTER(C.c_void_p)]
    L.sw_engine_destroy.argtypes = [C.c_void_p]
    L.sw_engine_choose.argtypes = [C.c_void_p, C.c_uint64, C.POINTER(C.c_int32)]
    L.sw_engine_step.argtypes = [C.c_void_p, C.c_int32]
    L.sw_engine_meet.argtypes = [C.c_void_p, C.POINTER(C.c_int32)]
    L.sw_engine_dfs.argtypes = [C.c_void_p, C.c_uint64, C.POINTER(C.c_uint64)]
    L.sw_engine_stats_get.argtypes = [C.c_void_p, C.POINTER(EngineStats)]
    L.sw_list_expand.argtypes = [C.c_uint32, C.c_uint32, _u32p, _u64p, C.c_size_t, C.c_int32,
                                 _u64p, _u32p]
    L.sw_list_lex_sort_dedupe.argtypes = [C.c_uint32, _u64p, _u32p, C.c_void_p, C.c_size_t,
                                          C.POINTER(C.c_size_t)]
    L.sw_list_sort_card_desc_lex.argtypes = [C.c_uint32, _u64p, _u32p, C.c_void_p, C.c_size_t]
    L.sw_list_dedupe_sorted.argtypes = [C.c_uint32, _u64p, _u32p, C.c_void_p, C.c_size_t,
                                        C.POINTER(C.c_size_t)]
    L.sw_list_hash_dedupe.argtypes = [C.c_uint32, _u64p, _u32p, C.c_void_p, C.c_size_t,
                                      C.POINTER(C.c_size_t)]
    L.sw_list_self_reduce_minimal.argtypes = [C.c_uint32, _u64p, _u32p, C.c_size_t,
                                              C.POINTER(C.c_size_t)]
    L.sw_list_mark.argtypes = [C.c_uint32, _u64p, C.c_size_t, _u64p, C.c_size_t, C.c_int32, _u8p]
    L.sw_list_meet_check.argtypes = [C.c_uint32, _u64p, C.c_size_t, _u64p, C.c_size_t,
                                     C.POINTER(C.c_int32)]
    L.sw_trie_node_count.argtypes = [C.c_uint32, _u64p, C.c_size_t, C.c_uint32,
                                     C.POINTER(C.c_uint64)]
    L.sw_run_experiment.argtypes = [_u32p, C.c_size_t, C.c_uint32, C.c_uint32, C.c_uint64,
                                    C.c_char_p, C.c_double, C.c_uint64, C.c_uint32, C.c_int32,
                                    C.c_uint32, C.c_uint32, C.c_char_p]
    L.sw_exp_mark.argtypes = [C.c_double] * 4
    L.sw_exp_mark.restype = C.c_double
    _dp = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
    _ip = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
    L.sw_step_costs.argtypes = [_dp, _ip, _dp, _dp, _dp, _ip, C.POINTER(C.c_int32)]
    L.sw_bench_expand.argtypes = [C.c_uint32, C.c_uint32, _u32p, C.c_uint64, C.c_double, C.c_uint64,
                                  C.c_int32, C.c_int32, C.POINTER(C.c_double)]
    L.sw_bench_dedupe.argtypes = [C.c_uint32, C.c_uint64, C.c_double, C.c_uint64, C.c_double, C.c_int32,
                                  C.c_int32, C.POINTER(C.c_double), C.POINTER(C.c_uint64)]
    L.sw_dev_owner_partition.argtypes = [C.c_uint32, C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint32,
                                         C.c_void_p, C.c_void_p, C.POINTER(C.c_uint64)]
    L.sw_dev_hash_dedupe.argtypes = [C.c_uint32, C.c_void_p, C.c_void_p, C.c_uint64,
                                     C.POINTER(C.c_uint64)]
    _lib = L
    return L


def bench_expand(aut, count: int, density: float, seed: int = 1, inverse: bool = False,
                 iters: int = 5) -> float:
    """Average ms of one expansion launch over `count` random parents (k children each)."""
    ms = C.c_double()
    _check(load().sw_bench_expand(aut.n, aut.k, aut.delta, count, density, seed, int(inverse), iters,
                                  C.byref(ms)))
    return ms.value


def bench_dedupe(n: int, count: int, density: float, seed: int = 1, dup_fraction: float = 0.1,
                 iters: int = 3, lex_sort: bool = False):
    """(avg ms of the hash dedupe [or lex sort + dedupe] over `count` random sets, unique count)."""
    ms, u = C.c_double(), C.c_uint64()
    _check(load().sw_bench_dedupe(n, count, density, seed, dup_fraction, iters, int(lex_sort),
                                  C.byref(ms), C.byref(u)))
    return ms.value, u.value


def exp_mark(a_size: float, b_size: float, a_density: float, b_density: float) -> float:
    """ExpMark (cost_model.hpp:67-74)."""
    return float(load().sw_exp_mark(a_size, b_size, a_density, b_density))


def step_costs(stats, flags, tuning):
    """compute_step_costs + select_step (cost_model.hpp:187-250); see sw_step_costs."""
    st = np.ascontiguousarray(stats, np.float64)
    fl = np.ascontiguousarray(flags, np.int32)
    tu = np.ascontiguousarray(tuning, np.float64)
    step, pred = np.zeros(5), np.zeros(5)
    feas = np.zeros(5, np.int32)
    sel = C.c_int32()
    _check(load().sw_step_costs(st, fl, tu, step, pred, feas, C.byref(sel)))
    return step, pred, feas, sel.value


def _check(rc: int) -> None:
    if rc != SW_OK:
        msg = load().sw_last_error().decode(errors="replace")
        raise _ERRORS.get(rc, SynchroError)(rc, msg)


def version() -> str:
    return load().sw_version().decode()


def device_count() -> int:
    return int(load().sw_device_count())


def exported_symbols() -> List[str]:
    L = load()
    return [s for s in EXPORTED_SYMBOLS if hasattr(L, s)]


# ------------------------------------------------------------------ automata
@dataclass
class Automaton:
    n: int
    k: int
    delta: np.ndarray  # uint32[n*k], delta[q*k + a]

    def next(self, q: int, a: int) -> int:
        return int(self.delta[q * self.k + a])


def random_automaton(n: int, k: int, seed: int) -> Automaton:
    d = np.zeros(n * k, np.uint32)
    _check(load().sw_random_automaton(n, k, seed, d))
    return Automaton(n, k, d)


def cerny_automaton(n: int) -> Automaton:
    d = np.zeros(max(n, 1) * 2, np.uint32)
    _check(load().sw_cerny_automaton(n, d))
    return Automaton(n, 2, d)


def instance_seed(base: int, n: int, i: int) -> int:
    return int(load().sw_instance_seed(base, n, i))


def parse_automaton(text: str) -> Automaton:
    n, k = C.c_uint32(), C.c_uint32()
    _check(load().sw_parse_automaton(text.encode(), C.byref(n), C.byref(k), None, 0))
    d = np.zeros(n.value * k.value, np.uint32)
    _check(load().sw_parse_automaton(text.encode(), C.byref(n), C.byref(k),
                                     d.ctypes.data_as(C.c_void_p), d.size))
    return Automaton(n.value, k.value, d)


def from_spec(spec: str) -> Automaton:
    kind, _, args = spec.partition(":")
    if kind == "cerny":
        return cerny_automaton(int(args))
    if kind == "random":
        n, k, s = (int(x) for x in args.split(","))
        return random_automaton(n, k, s)
    raise ValueError(f"unknown generator: {kind}")


def is_synchronizing(aut: Automaton) -> bool:
    r = C.c_int32()
    _check(load().sw_is_synchronizing(aut.n, aut.k, aut.delta, C.byref(r)))
    return bool(r.value)


def pair_distances(aut: Automaton, on_device: bool = True) -> np.ndarray:
    """Shortest merging word length of every pair {p <= q} at q(q+1)/2 + p
    (UINT32_MAX: unmergeable) — automaton.hpp:119-157; on_device: device/pairs.cu."""
    out = np.zeros(aut.n * (aut.n + 1) // 2, np.uint32)
    _check(load().sw_pair_distances(aut.n, aut.k, aut.delta, int(on_device),
                                    out.ctypes.data_as(C.c_void_p), out.size))
    return out


def is_reset_word(aut: Automaton, word: Sequence[int]) -> bool:
    w = np.ascontiguousarray(np.asarray(list(word), np.uint32))
    r = C.c_int32()
    _check(load().sw_is_reset_word(aut.n, aut.k, aut.delta, w.ctypes.data_as(C.c_void_p),
                                   w.size, C.byref(r)))
    return bool(r.value)


# --------------------------------------------------------------------- solve
@dataclass
class SolveResult:
    threshold: int
    word: Optional[List[int]]
    upper_bound: int
    iterations: int
    bfs_steps: int
    ibfs_steps: int
    used_dfs: bool
    peak_memory: int
    expansions_phase1: int
    expansions_dfs: int
    heuristic_seconds: float
    engine_seconds: float
    expand_kernel_ms: float
    kernel_launches: int
    phase: str
    engine_device_ms: float = 0.0
    h2d_bytes: int = 0
    d2h_bytes: int = 0
    contain_kernel_ms: float = 0.0
    contain_bytes: int = 0
    trace: Optional[List[str]] = field(default=None)
    contain_visits: int = 0
    contain_pairs: int = 0
    dfs_levels: List[List[int]] = field(default_factory=list)  # [r, level, in, generated, kept]

    @property
    def expansions(self) -> int:
        return self.expansions_phase1 + self.expansions_dfs


def default_options(**kw) -> SolveOptions:
    o = SolveOptions()
    load().sw_default_options(C.byref(o))
    for key, v in kw.items():
        if key == "schedule" and isinstance(v, str):
            v = SCHEDULES[v]
        if key in ("track_word", "timing", "contain_stats", "dfs_reference_order"):
            v = int(bool(v))
        if v is None:
            continue
        setattr(o, key, v)
    return o


def solve_exact(aut: Automaton, trace_path: Optional[str] = None, **opts) -> SolveResult:
    """synchro::solve_exact on the B200 data plane (bibfs_engine.hpp:467)."""
    o = default_options(**opts)
    r = SolveResultC()
    cap = 1 << 20 if o.track_word else 0
    buf = np.zeros(max(cap, 1), np.uint32)
    lcap = 1 << 16
    levels = np.zeros(5 * lcap, np.uint64)
    nlev = C.c_size_t()
    _check(load().sw_solve_exact_ex(aut.n, aut.k, np.ascontiguousarray(aut.delta, np.uint32),
                                    C.byref(o), C.byref(r), buf.ctypes.data_as(C.c_void_p), cap,
                                    trace_path.encode() if trace_path else None,
                                    levels.ctypes.data_as(C.c_void_p), lcap, C.byref(nlev)))
    word = buf[: r.word_len].tolist() if r.has_word else None
    dfs_levels = levels[: 5 * min(nlev.value, lcap)].reshape(-1, 5).tolist()
    trace = None
    if trace_path and os.path.exists(trace_path):
        with open(trace_path) as f:
            trace = f.read().splitlines()
    return SolveResult(r.threshold, word, r.upper_bound, r.iterations, r.bfs_steps, r.ibfs_steps,
                       bool(r.used_dfs), r.peak_memory, r.expansions_phase1, r.expansions_dfs,
                       r.heuristic_seconds, r.engine_seconds, r.expand_kernel_ms,
                       r.kernel_launches, r.phase.decode(), r.engine_device_ms, r.h2d_bytes,
                       r.d2h_bytes, r.contain_kernel_ms, r.contain_bytes, trace,
                       r.contain_visits, r.contain_pairs, dfs_levels)


def list_trie_exists(n: int, a_words, b_words):
    """(met, a_index, b_index) through the trie index (a in any order)."""
    W = (n + 63) // 64
    a = np.ascontiguousarray(a_words, np.uint64)
    b = np.ascontiguousarray(b_words, np.uint64)
    m, ai, bi = C.c_int32(), C.c_uint64(), C.c_uint64()
    _check(load().sw_list_trie_exists(n, a, a.size // W, b, b.size // W, C.byref(m), C.byref(ai),
                                      C.byref(bi)))
    return bool(m.value), int(ai.value), int(bi.value)


# ------------------------------------------------------- partitioned solve
def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    _check(load().sw_nccl_unique_id(buf))
    return bytes(buf)


class Comm:
    """A communicator for sw_solve_exact_dist: NCCL on device buffers
    (nccl_id from nccl_unique_id() on one rank, shared by the caller) or host
    callbacks (callbacks=(all_to_allv, all_gather_v, all_reduce_u64) with the
    C signatures of include/synchro_b200.h)."""

    def __init__(self, rank: int, nranks: int, nccl_id: Optional[bytes] = None, callbacks=None):
        d = CommDesc()
        d.rank, d.nranks = rank, nranks
        if nccl_id is not None:
            d.kind = SW_COMM_NCCL
            C.memmove(d.nccl_id, nccl_id, min(128, len(nccl_id)))
        else:
            d.kind = SW_COMM_CALLBACK
            self._cbs = (A2A_CB(callbacks[0]), AG_CB(callbacks[1]), AR_CB(callbacks[2]))
            d.all_to_allv, d.all_gather_v, d.all_reduce_u64 = self._cbs
        self._h = C.c_void_p()
        _check(load().sw_comm_create(C.byref(d), C.byref(self._h)))
        self.rank, self.nranks = rank, nranks

    def close(self):
        if self._h:
            load().sw_comm_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def solve_exact_dist(aut: Automaton, comm: Comm, trace_path: Optional[str] = None, **opts):
    """Partitioned sw_solve_exact_dist: (SolveResult, NVLink/transport bytes sent by this rank)."""
    o = default_options(**opts)
    r = SolveResultC()
    cap = 1 << 20 if o.track_word else 0
    buf = np.zeros(max(cap, 1), np.uint32)
    nv = C.c_uint64()
    _check(load().sw_solve_exact_dist(aut.n, aut.k, np.ascontiguousarray(aut.delta, np.uint32),
                                      C.byref(o), comm._h, C.byref(r),
                                      buf.ctypes.data_as(C.c_void_p), cap,
                                      trace_path.encode() if trace_path else None, C.byref(nv)))
    word = buf[: r.word_len].tolist() if r.has_word else None
    trace = None
    if trace_path and os.path.exists(trace_path):
        with open(trace_path) as f:
            trace = f.read().splitlines()
    res = SolveResult(r.threshold, word, r.upper_bound, r.iterations, r.bfs_steps, r.ibfs_steps,
                      bool(r.used_dfs), r.peak_memory, r.expansions_phase1, r.expansions_dfs,
                      r.heuristic_seconds, r.engine_seconds, r.expand_kernel_ms,
                      r.kernel_launches, r.phase.decode(), r.engine_device_ms, r.h2d_bytes,
                      r.d2h_bytes, r.contain_kernel_ms, r.contain_bytes, trace,
                      r.contain_visits, r.contain_pairs)
    return res, int(nv.value)


def meet_check_order(n: int, a_words, b_words, min_brute: int = 64) -> np.ndarray:
    """Host-side replay of the order the reference's meet_check leaves b in
    (subset_algebra.hpp:201-210; no device).  order[p] = original index."""
    W = (n + 63) // 64
    a = np.ascontiguousarray(a_words, np.uint64)
    b = np.ascontiguousarray(b_words, np.uint64)
    out = np.zeros(b.size // W, np.uint32)
    _check(load().sw_meet_check_order(n, a, a.size // W, b, b.size // W, min_brute, out))
    return out


ALGORITHMS = {"eppstein": 0, "beam": 1, "adaptive": 2}


def heuristic(aut: Automaton, algorithm: str = "adaptive", beam_size: int = 0,
              memory: int = 4 << 30, time_limit: float = 0.0):
    """(bound, word) — heuristics.hpp:26-184."""
    b = C.c_uint64()
    buf = np.zeros(aut.n * aut.n * 4 + 64, np.uint32)
    _check(load().sw_heuristic(aut.n, aut.k, aut.delta, ALGORITHMS[algorithm], beam_size, memory,
                               time_limit, C.byref(b), buf.ctypes.data_as(C.c_void_p), buf.size))
    return int(b.value), buf[: b.value].tolist()


def power_set_oracle(aut: Automaton, time_limit: float = 0.0) -> int:
    t = C.c_uint64()
    _check(load().sw_power_set_oracle(aut.n, aut.k, aut.delta, time_limit, C.byref(t)))
    return int(t.value)


def run_experiment(ns: Sequence[int], k: int, samples: int, seed_base: int, csv_path: str,
                   solver: str = "exact", time_limit: float = 0.0, memory: int = 4 << 30,
                   threads: int = 1, deterministic: bool = False, shard_index: int = 0,
                   shard_count: int = 1) -> None:
    arr = np.ascontiguousarray(np.asarray(ns, np.uint32))
    _check(load().sw_run_experiment(arr, arr.size, k, samples, seed_base, solver.encode(),
                                    time_limit, memory, threads, int(deterministic), shard_index,
                                    shard_count, csv_path.encode()))


# -------------------------------------------------------------------- engine
class Engine:
    """Step-by-step handle on the GPU engine (sw_engine_*)."""

    def __init__(self, aut: Automaton, upper_bound: int, **opts):
        self._h = C.c_void_p()
        o = default_options(**opts)
        _check(load().sw_engine_create(aut.n, aut.k, aut.delta, C.byref(o), upper_bound,
                                       C.byref(self._h)))

    def choose(self, r: int) -> str:
        kd = C.c_int32()
        _check(load().sw_engine_choose(self._h, r, C.byref(kd)))
        return STEP_KINDS[kd.value]

    def step(self, kind: str) -> None:
        _check(load().sw_engine_step(self._h, STEP_KINDS.index(kind)))

    def meet(self) -> bool:
        m = C.c_int32()
        _check(load().sw_engine_meet(self._h, C.byref(m)))
        return bool(m.value)

    def dfs(self, r: int) -> int:
        t = C.c_uint64()
        _check(load().sw_engine_dfs(self._h, r, C.byref(t)))
        return int(t.value)

    def stats(self) -> EngineStats:
        s = EngineStats()
        _check(load().sw_engine_stats_get(self._h, C.byref(s)))
        return s

    def close(self) -> None:
        if self._h:
            load().sw_engine_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---------------------------------------------------------------- primitives
def W(n: int) -> int:
    return (n + 63) // 64


def cards_of(n: int, words: np.ndarray) -> np.ndarray:
    w = np.ascontiguousarray(words, np.uint64).reshape(-1, W(n))
    bits = np.unpackbits(w.view(np.uint8), axis=1)
    return bits.sum(axis=1).astype(np.uint32)


def list_expand(aut: Automaton, words: np.ndarray, inverse: bool):
    words = np.ascontiguousarray(words, np.uint64)
    cnt = words.size // W(aut.n)
    ow = np.zeros(max(cnt * aut.k * W(aut.n), 1), np.uint64)
    oc = np.zeros(max(cnt * aut.k, 1), np.uint32)
    _check(load().sw_list_expand(aut.n, aut.k, aut.delta, words, cnt, int(inverse), ow, oc))
    return ow[: cnt * aut.k * W(aut.n)], oc[: cnt * aut.k]


def _tags_ptr(t):
    return t.ctypes.data_as(C.c_void_p) if t is not None else None


def list_lex_sort_dedupe(n: int, words: np.ndarray, tags: Optional[np.ndarray] = None):
    w = np.array(words, np.uint64).copy()
    c = cards_of(n, w)
    t = None if tags is None else np.array(tags, np.uint64).copy()
    out = C.c_size_t()
    _check(load().sw_list_lex_sort_dedupe(n, w, c, _tags_ptr(t), c.size, C.byref(out)))
    m = out.value
    return w[: m * W(n)], c[:m], (t[:m] if t is not None else None)


def list_sort_card_desc_lex(n: int, words: np.ndarray, tags: Optional[np.ndarray] = None):
    w = np.array(words, np.uint64).copy()
    c = cards_of(n, w)
    t = None if tags is None else np.array(tags, np.uint64).copy()
    _check(load().sw_list_sort_card_desc_lex(n, w, c, _tags_ptr(t), c.size))
    return w, c, t


def list_dedupe_sorted(n: int, words: np.ndarray, tags: Optional[np.ndarray] = None):
    w = np.array(words, np.uint64).copy()
    c = cards_of(n, w)
    t = None if tags is None else np.array(tags, np.uint64).copy()
    out = C.c_size_t()
    _check(load().sw_list_dedupe_sorted(n, w, c, _tags_ptr(t), c.size, C.byref(out)))
    m = out.value
    return w[: m * W(n)], c[:m], (t[:m] if t is not None else None)


def list_hash_dedupe(n: int, words: np.ndarray, tags: Optional[np.ndarray] = None):
    """First occurrence of every distinct row, original order (GPU hash dedupe)."""
    w = np.array(words, np.uint64).copy()
    c = cards_of(n, w)
    t = None if tags is None else np.array(tags, np.uint64).copy()
    out = C.c_size_t()
    _check(load().sw_list_hash_dedupe(n, w, c, _tags_ptr(t), c.size, C.byref(out)))
    m = out.value
    return w[: m * W(n)], c[:m], (t[:m] if t is not None else None)


def dev_owner_partition(n: int, words, cards, nranks: int):
    """Device tensors (torch, current CUDA device): rows regrouped owner-major by
    owner = h(row) mod nranks -> (words, cards, counts per owner)."""
    import torch
    words, cards = words.contiguous(), cards.contiguous()
    count = cards.numel()
    ow, oc = torch.empty_like(words), torch.empty_like(cards)
    counts = (C.c_uint64 * nranks)()
    _check(load().sw_dev_owner_partition(n, words.data_ptr(), cards.data_ptr(), count, nranks,
                                         ow.data_ptr(), oc.data_ptr(), counts))
    return ow, oc, [int(x) for x in counts]


def dev_hash_dedupe(n: int, words, cards):
    """Set-semantics dedupe of device tensors -> (words, cards) of the survivors."""
    words, cards = words.contiguous().clone(), cards.contiguous().clone()
    kept = C.c_uint64()
    _check(load().sw_dev_hash_dedupe(n, words.data_ptr(), cards.data_ptr(), cards.numel(),
                                     C.byref(kept)))
    m = kept.value
    return words.view(-1, W(n))[:m].reshape(-1), cards[:m]


def list_self_reduce_minimal(n: int, words: np.ndarray) -> np.ndarray:
    w = np.array(words, np.uint64).copy()
    c = cards_of(n, w)
    out = C.c_size_t()
    _check(load().sw_list_self_reduce_minimal(n, w, c, c.size, C.byref(out)))
    return w[: out.value * W(n)]


def list_mark(n: int, a_words: np.ndarray, b_words: np.ndarray, mode: int) -> np.ndarray:
    a = np.ascontiguousarray(a_words, np.uint64)
    b = np.ascontiguousarray(b_words, np.uint64)
    keep = np.zeros(max(b.size // W(n), 1), np.uint8)
    _check(load().sw_list_mark(n, a, a.size // W(n), b, b.size // W(n), mode, keep))
    return keep[: b.size // W(n)]


def list_meet_check(n: int, a_words: np.ndarray, b_words: np.ndarray) -> bool:
    a = np.ascontiguousarray(a_words, np.uint64)
    b = np.ascontiguousarray(b_words, np.uint64)
    m = C.c_int32()
    _check(load().sw_list_meet_check(n, a, a.size // W(n), b, b.size // W(n), C.byref(m)))
    return bool(m.value)


def trie_node_count(n: int, words: np.ndarray, min_leaf: int = 10) -> int:
    w = np.ascontiguousarray(words, np.uint64)
    out = C.c_uint64()
    _check(load().sw_trie_node_count(n, w, w.size // W(n), min_leaf, C.byref(out)))
    return int(out.value)
