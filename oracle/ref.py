"""ctypes wrapper over oracle/_ref/libsynchro_ref.so — TEST INFRASTRUCTURE ONLY.

The library is the unmodified reference (/root/reference/proj/include, header-only
C++20) compiled behind oracle/ref_driver.cpp.  Only tests/, __graft_entry__.smoke()
and bench.py (cpu_baseline / --impl reference) may import this module, and only
as the checker / the CPU baseline — never as the thing measured for the product.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import List, Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libsynchro_ref.so")
C_SO = os.path.join(HERE, "lib", "liboracle.so")

_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")


class RefOptions(C.Structure):
    _fields_ = [
        ("memory", C.c_uint64),
        ("time_limit", C.c_double),
        ("track_word", C.c_int32),
        ("schedule", C.c_int32),
        ("upper_bound", C.c_uint64),
        ("set_cost", C.c_double),
        ("dfs_set_weight", C.c_double),
        ("dfs_check_weight", C.c_double),
        ("min_brute", C.c_uint32),
        ("min_leaf", C.c_uint32),
        ("dedupe_cadence", C.c_uint32),
        ("reduce_cadence", C.c_uint32),
        ("max_seconds", C.c_double),
        ("dfs_largest", C.c_uint64),
        ("history_growth", C.c_double),
        ("beam_initial", C.c_uint64),
        ("beam_cost_fraction", C.c_double),
        ("reduction_of_reduction", C.c_double),
        ("stop_after_iterations", C.c_uint64),
    ]


class RefResult(C.Structure):
    _fields_ = [
        ("status", C.c_int32),
        ("used_dfs", C.c_int32),
        ("threshold", C.c_uint64),
        ("upper_bound", C.c_uint64),
        ("iterations", C.c_uint64),
        ("bfs_steps", C.c_uint64),
        ("ibfs_steps", C.c_uint64),
        ("peak_memory", C.c_uint64),
        ("word_len", C.c_uint64),
        ("expansions_phase1", C.c_uint64),
        ("expansions_dfs", C.c_uint64),
        ("heuristic_seconds", C.c_double),
        ("engine_seconds", C.c_double),
    ]


SCHEDULES = {"auto": 0, "bfs": 1, "ibfs": 2, "dfs": 3}


def default_options(**kw) -> RefOptions:
    o = RefOptions(
        memory=4 << 30, time_limit=0.0, track_word=0, schedule=0, upper_bound=0,
        set_cost=512.0, dfs_set_weight=0.25, dfs_check_weight=0.25, min_brute=64,
        min_leaf=10, dedupe_cadence=2, reduce_cadence=3, max_seconds=0.0, dfs_largest=20000,
        history_growth=2.0, beam_initial=0, beam_cost_fraction=0.05, reduction_of_reduction=0.0,
        stop_after_iterations=0)
    for k, v in kw.items():
        if k == "schedule" and isinstance(v, str):
            v = SCHEDULES[v]
        setattr(o, k, v)
    return o


_lib = None


def available() -> bool:
    return os.path.exists(REF_SO)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(REF_SO):
            raise RuntimeError(f"reference oracle not built: {REF_SO} (run make -C oracle ref)")
        L = C.CDLL(REF_SO)
        L.ref_random_automaton.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, _u32p]
        L.ref_cerny_automaton.argtypes = [C.c_uint32, _u32p]
        L.ref_instance_seed.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32]
        L.ref_instance_seed.restype = C.c_uint64
        L.ref_is_synchronizing.argtypes = [C.c_uint32, C.c_uint32, _u32p]
        L.ref_power_set_oracle.argtypes = [C.c_uint32, C.c_uint32, _u32p]
        L.ref_power_set_oracle.restype = C.c_int64
        L.ref_exp_mark.argtypes = [C.c_double] * 4
        L.ref_exp_mark.restype = C.c_double
        L.ref_is_reset_word.argtypes = [C.c_uint32, C.c_uint32, _u32p, _u32p, C.c_size_t]
        L.ref_expand.argtypes = [C.c_uint32, C.c_uint32, _u32p, _u64p, C.c_size_t, C.c_int,
                                 _u64p, _u32p]
        L.ref_lex_sort_dedupe.argtypes = [C.c_uint32, _u64p, _u32p, _u64p, C.c_size_t,
                                          C.POINTER(C.c_double)]
        L.ref_lex_sort_dedupe.restype = C.c_size_t
        L.ref_sort_lex.argtypes = [C.c_uint32, _u64p, _u32p, _u64p, C.c_size_t]
        L.ref_sort_card_desc_lex.argtypes = [C.c_uint32, _u64p, _u32p, _u64p, C.c_size_t]
        L.ref_dedupe_sorted.argtypes = [C.c_uint32, _u64p, _u32p, _u64p, C.c_size_t]
        L.ref_dedupe_sorted.restype = C.c_size_t
        L.ref_self_reduce_minimal.argtypes = [C.c_uint32, _u64p, _u32p, C.c_size_t]
        L.ref_self_reduce_minimal.restype = C.c_size_t
        L.ref_mark.argtypes = [C.c_uint32, _u64p, C.c_size_t, _u64p, C.c_size_t, C.c_int, _u8p]
        L.ref_mark.restype = C.c_size_t
        L.ref_meet_check.argtypes = [C.c_uint32, _u64p, C.c_size_t, _u64p, C.c_size_t]
        L.ref_meet_check_order.argtypes = [C.c_uint32, _u64p, C.c_size_t, _u64p, C.c_size_t,
                                           C.c_uint32, _u32p]
        L.ref_trie_node_count.argtypes = [C.c_uint32, _u64p, C.c_size_t, C.c_uint32,
                                          C.POINTER(C.c_uint64)]
        L.ref_trie_node_count.restype = C.c_uint64
        L.ref_eppstein.argtypes = [C.c_uint32, C.c_uint32, _u32p, _u32p, C.c_size_t]
        L.ref_eppstein.restype = C.c_uint64
        L.ref_beam.argtypes = [C.c_uint32, C.c_uint32, _u32p, C.c_uint64, _u32p, C.c_size_t]
        L.ref_beam.restype = C.c_uint64
        L.ref_adaptive.argtypes = [C.c_uint32, C.c_uint32, _u32p, C.c_uint64, _u32p, C.c_size_t]
        L.ref_adaptive.restype = C.c_uint64
        L.ref_solve_exact.argtypes = [C.c_uint32, C.c_uint32, _u32p, C.POINTER(RefOptions),
                                      C.POINTER(RefResult), _u32p, C.c_size_t, C.c_char_p]
        L.ref_solve_instrumented.argtypes = [C.c_uint32, C.c_uint32, _u32p, C.POINTER(RefOptions),
                                             C.POINTER(RefResult), C.c_char_p, C.c_char_p]
        _dp = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
        _ip = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
        L.ref_step_costs.argtypes = [_dp, _ip, _dp, _dp, _dp, _ip, C.POINTER(C.c_int32)]
        L.ref_run_experiment.argtypes = [_u32p, C.c_size_t, C.c_uint32, C.c_uint32, C.c_uint64,
                                         C.c_char_p, C.c_double, C.c_uint32, C.c_int, C.c_char_p]
        _lib = L
    return _lib


def run_experiment(ns, k, samples, seed_base, path, solver="exact", time_limit=0.0, threads=1,
                   deterministic=True):
    arr = np.ascontiguousarray(np.asarray(ns, np.uint32))
    rc = lib().ref_run_experiment(arr, arr.size, k, samples, seed_base, solver.encode(), time_limit,
                                  threads, int(deterministic), path.encode())
    if rc != 0:
        raise RuntimeError("reference run_experiment failed")


def step_costs(stats, flags, tuning):
    st = np.ascontiguousarray(stats, np.float64)
    fl = np.ascontiguousarray(flags, np.int32)
    tu = np.ascontiguousarray(tuning, np.float64)
    step, pred = np.zeros(5), np.zeros(5)
    feas = np.zeros(5, np.int32)
    sel = C.c_int32()
    lib().ref_step_costs(st, fl, tu, step, pred, feas, C.byref(sel))
    return step, pred, feas, sel.value


# ----------------------------------------------------------------- automata
def random_automaton(n: int, k: int, seed: int) -> np.ndarray:
    d = np.zeros(n * k, np.uint32)
    lib().ref_random_automaton(n, k, seed, d)
    return d


def cerny_automaton(n: int) -> np.ndarray:
    d = np.zeros(n * 2, np.uint32)
    if lib().ref_cerny_automaton(n, d) != 0:
        raise ValueError("cerny automaton needs n >= 2")
    return d


def instance_seed(base: int, n: int, i: int) -> int:
    return int(lib().ref_instance_seed(base, n, i))


def is_synchronizing(n, k, delta) -> bool:
    return bool(lib().ref_is_synchronizing(n, k, np.ascontiguousarray(delta, np.uint32)))


def power_set_oracle(n, k, delta) -> int:
    return int(lib().ref_power_set_oracle(n, k, np.ascontiguousarray(delta, np.uint32)))


def exp_mark(a_s, b_s, a_d, b_d) -> float:
    return float(lib().ref_exp_mark(a_s, b_s, a_d, b_d))


def is_reset_word(n, k, delta, word: Sequence[int]) -> bool:
    w = np.ascontiguousarray(np.asarray(word, np.uint32))
    if w.size == 0:
        w = np.zeros(1, np.uint32)
        return bool(lib().ref_is_reset_word(n, k, np.ascontiguousarray(delta, np.uint32), w, 0))
    return bool(lib().ref_is_reset_word(n, k, np.ascontiguousarray(delta, np.uint32), w, w.size))


# -------------------------------------------------------------- primitives
def W(n: int) -> int:
    return (n + 63) // 64


def expand(n, k, delta, words: np.ndarray, inverse: bool):
    words = np.ascontiguousarray(words, np.uint64)
    cnt = words.size // W(n)
    ow = np.zeros(cnt * k * W(n), np.uint64)
    oc = np.zeros(cnt * k, np.uint32)
    lib().ref_expand(n, k, np.ascontiguousarray(delta, np.uint32), words, cnt, int(inverse), ow, oc)
    return ow, oc


def _cards(n, words):
    w = words.reshape(-1, W(n))
    return np.array([sum(int(x).bit_count() for x in row) for row in w], np.uint32)


def lex_sort_dedupe(n, words, tags=None):
    words = np.array(words, np.uint64).copy()
    cnt = words.size // W(n)
    cards = _cards(n, words)
    t = np.array(tags if tags is not None else np.arange(cnt), np.uint64)
    r = C.c_double()
    m = lib().ref_lex_sort_dedupe(n, words, cards, t, cnt, C.byref(r))
    return words[: m * W(n)], cards[:m], t[:m], r.value


def sort_card_desc_lex(n, words, tags=None):
    words = np.array(words, np.uint64).copy()
    cnt = words.size // W(n)
    cards = _cards(n, words)
    t = np.array(tags if tags is not None else np.arange(cnt), np.uint64)
    lib().ref_sort_card_desc_lex(n, words, cards, t, cnt)
    return words, cards, t


def self_reduce_minimal(n, words):
    words = np.array(words, np.uint64).copy()
    cnt = words.size // W(n)
    cards = _cards(n, words)
    m = lib().ref_self_reduce_minimal(n, words, cards, cnt)
    return words[: m * W(n)]


def mark(n, a_words, b_words, mode: int) -> np.ndarray:
    """keep flags (1 = unmarked) of b in its original order; mode 0 supersets,
    1 proper supersets, 2 subsets (subset_algebra.hpp:138-174)."""
    a = np.ascontiguousarray(a_words, np.uint64)
    b = np.ascontiguousarray(b_words, np.uint64)
    keep = np.zeros(b.size // W(n), np.uint8)
    lib().ref_mark(n, a, a.size // W(n), b, b.size // W(n), mode, keep)
    return keep


def meet_check(n, a_words, b_words) -> bool:
    a = np.ascontiguousarray(a_words, np.uint64)
    b = np.ascontiguousarray(b_words, np.uint64).copy()
    return bool(lib().ref_meet_check(n, a, a.size // W(n), b, b.size // W(n)))


def meet_check_order(n, a_words, b_words, min_brute=64):
    """(met, order): the order meet_check leaves b in (order[p] = original index)."""
    a = np.ascontiguousarray(a_words, np.uint64)
    b = np.ascontiguousarray(b_words, np.uint64)
    order = np.zeros(b.size // W(n), np.uint32)
    met = lib().ref_meet_check_order(n, a, a.size // W(n), b, b.size // W(n), min_brute, order)
    return bool(met), order


def trie_node_count(n, words, min_leaf=10):
    w = np.ascontiguousarray(words, np.uint64)
    fp = C.c_uint64()
    c = lib().ref_trie_node_count(n, w, w.size // W(n), min_leaf, C.byref(fp))
    return int(c), int(fp.value)


# --------------------------------------------------------------- heuristics
def eppstein(n, k, delta):
    buf = np.zeros(n * n * 4 + 16, np.uint32)
    L = lib().ref_eppstein(n, k, np.ascontiguousarray(delta, np.uint32), buf, buf.size)
    return int(L), buf[:L].tolist()


def beam(n, k, delta, size):
    buf = np.zeros(n * n * 4 + 16, np.uint32)
    L = lib().ref_beam(n, k, np.ascontiguousarray(delta, np.uint32), size, buf, buf.size)
    return (int(L), buf[:L].tolist()) if L else None


def adaptive(n, k, delta, memory=4 << 30):
    buf = np.zeros(n * n * 4 + 16, np.uint32)
    L = lib().ref_adaptive(n, k, np.ascontiguousarray(delta, np.uint32), memory, buf, buf.size)
    return int(L), buf[:L].tolist()


# -------------------------------------------------------------------- solve
@dataclass
class RefSolve:
    status: int
    threshold: int
    upper_bound: int
    iterations: int
    bfs_steps: int
    ibfs_steps: int
    used_dfs: bool
    peak_memory: int
    word: Optional[List[int]]
    expansions_phase1: int
    expansions_dfs: int
    heuristic_seconds: float
    engine_seconds: float
    trace: Optional[List[str]] = None
    dfs_levels: Optional[List[dict]] = None


def _to_solve(r: RefResult, word=None, trace=None, levels=None) -> RefSolve:
    return RefSolve(r.status, r.threshold, r.upper_bound, r.iterations, r.bfs_steps,
                    r.ibfs_steps, bool(r.used_dfs), r.peak_memory, word,
                    r.expansions_phase1, r.expansions_dfs, r.heuristic_seconds,
                    r.engine_seconds, trace, levels)


def solve_exact(n, k, delta, trace_path: Optional[str] = None, **opts) -> RefSolve:
    """The reference's own synchro::solve_exact (bibfs_engine.hpp:467)."""
    o = default_options(**opts)
    res = RefResult()
    cap = 1 << 16
    buf = np.zeros(cap, np.uint32)
    lib().ref_solve_exact(n, k, np.ascontiguousarray(delta, np.uint32), C.byref(o), C.byref(res),
                          buf, cap, trace_path.encode() if trace_path else None)
    word = buf[: res.word_len].tolist() if (o.track_word and res.status == 0 and
                                            (res.word_len or res.threshold == 0)) else None
    trace = open(trace_path).read().splitlines() if trace_path and os.path.exists(trace_path) else None
    return _to_solve(res, word, trace)


def solve_instrumented(n, k, delta, trace_path=None, levels_path=None, **opts) -> RefSolve:
    """Replay of solve_exact over the public engine with DFS level logging."""
    import json
    o = default_options(**opts)
    res = RefResult()
    lib().ref_solve_instrumented(n, k, np.ascontiguousarray(delta, np.uint32), C.byref(o),
                                 C.byref(res), trace_path.encode() if trace_path else None,
                                 levels_path.encode() if levels_path else None)
    trace = open(trace_path).read().splitlines() if trace_path and os.path.exists(trace_path) else None
    levels = None
    if levels_path and os.path.exists(levels_path):
        levels = [json.loads(x) for x in open(levels_path).read().splitlines() if x.strip()]
    return _to_solve(res, None, trace, levels)
