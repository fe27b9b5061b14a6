"""ctypes wrapper of oracle/lib/liboracle.so (the plain-C restatement) — TEST
INFRASTRUCTURE ONLY; loaded by tests/ as a checker, never by the product."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "lib", "liboracle.so")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_lib = None


def available() -> bool:
    return os.path.exists(SO)


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(SO)
        L.or_random_automaton.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, _u32p]
        L.or_instance_seed.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32]
        L.or_instance_seed.restype = C.c_uint64
        L.or_expand.argtypes = [C.c_uint32, C.c_uint32, _u32p, _u64p, C.c_size_t, C.c_int, _u64p, _u32p]
        L.or_lex_sort_dedupe.argtypes = [C.c_uint32, _u64p, _u32p, _u64p, C.c_size_t]
        L.or_lex_sort_dedupe.restype = C.c_size_t
        L.or_sort_card_desc_lex.argtypes = [C.c_uint32, _u64p, _u32p, _u64p, C.c_size_t]
        L.or_self_reduce_minimal.argtypes = [C.c_uint32, _u64p, _u32p, C.c_size_t]
        L.or_self_reduce_minimal.restype = C.c_size_t
        L.or_mark.argtypes = [C.c_uint32, _u64p, C.c_size_t, _u64p, C.c_size_t, C.c_int, _u8p]
        L.or_meet_check.argtypes = [C.c_uint32, _u64p, C.c_size_t, _u64p, C.c_size_t]
        L.or_trie_node_count.argtypes = [C.c_uint32, _u64p, C.c_size_t, C.c_uint32]
        L.or_trie_node_count.restype = C.c_uint64
        L.or_exp_mark.argtypes = [C.c_double] * 4
        L.or_exp_mark.restype = C.c_double
        L.or_power_set_oracle.argtypes = [C.c_uint32, C.c_uint32, _u32p]
        L.or_power_set_oracle.restype = C.c_int64
        _lib = L
    return _lib


def W(n):
    return (n + 63) // 64


def cards(n, words):
    w = np.ascontiguousarray(words, np.uint64).reshape(-1, W(n))
    return np.unpackbits(w.view(np.uint8), axis=1).sum(axis=1).astype(np.uint32)


def random_automaton(n, k, seed):
    d = np.zeros(n * k, np.uint32)
    lib().or_random_automaton(n, k, seed, d)
    return d


def expand(n, k, delta, words, inverse):
    words = np.ascontiguousarray(words, np.uint64)
    cnt = words.size // W(n)
    ow = np.zeros(max(cnt * k * W(n), 1), np.uint64)
    oc = np.zeros(max(cnt * k, 1), np.uint32)
    lib().or_expand(n, k, np.ascontiguousarray(delta, np.uint32), words, cnt, int(inverse), ow, oc)
    return ow[: cnt * k * W(n)], oc[: cnt * k]


def lex_sort_dedupe(n, words, tags):
    w = np.array(words, np.uint64).copy()
    c = cards(n, w)
    t = np.array(tags, np.uint64).copy()
    m = lib().or_lex_sort_dedupe(n, w, c, t, c.size)
    return w[: m * W(n)], c[:m], t[:m]


def sort_card_desc_lex(n, words, tags):
    w = np.array(words, np.uint64).copy()
    c = cards(n, w)
    t = np.array(tags, np.uint64).copy()
    lib().or_sort_card_desc_lex(n, w, c, t, c.size)
    return w, c, t


def self_reduce_minimal(n, words):
    w = np.array(words, np.uint64).copy()
    c = cards(n, w)
    m = lib().or_self_reduce_minimal(n, w, c, c.size)
    return w[: m * W(n)]


def mark(n, a, b, mode):
    a = np.ascontiguousarray(a, np.uint64)
    b = np.ascontiguousarray(b, np.uint64)
    keep = np.zeros(max(b.size // W(n), 1), np.uint8)
    lib().or_mark(n, a, a.size // W(n), b, b.size // W(n), mode, keep)
    return keep[: b.size // W(n)]


def meet_check(n, a, b):
    a = np.ascontiguousarray(a, np.uint64)
    b = np.ascontiguousarray(b, np.uint64)
    return bool(lib().or_meet_check(n, a, a.size // W(n), b, b.size // W(n)))


def trie_node_count(n, words, min_leaf=10):
    w = np.ascontiguousarray(words, np.uint64)
    return int(lib().or_trie_node_count(n, w, w.size // W(n), min_leaf))


def exp_mark(a, b, c, d):
    return float(lib().or_exp_mark(a, b, c, d))


def power_set_oracle(n, k, delta):
    return int(lib().or_power_set_oracle(n, k, np.ascontiguousarray(delta, np.uint32)))
