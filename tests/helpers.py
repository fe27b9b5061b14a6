"""Shared test helpers: seeded random set lists in the reference's bit layout."""
import numpy as np


def W(n):
    return (n + 63) // 64


def random_list(n, count, density, seed):
    """count random subsets of {0..n-1}, MSB-first packing, tail bits zero
    (state_set.hpp:14-19; test_helpers.hpp:24-33 style density knob)."""
    rng = np.random.default_rng(seed)
    bits = rng.random((count, W(n) * 64)) < density
    bits[:, n:] = False
    packed = np.packbits(bits.astype(np.uint8), axis=1)  # big-endian bit order per byte
    words = packed.view(">u8").astype(np.uint64)
    return np.ascontiguousarray(words.reshape(-1))


def rows(n, words):
    return [tuple(int(x) for x in r) for r in np.asarray(words, np.uint64).reshape(-1, W(n))]


def lex_sorted_unique(n, words):
    return np.array(sorted(set(rows(n, words))), np.uint64).reshape(-1) if len(words) else words
