"""Pins the plain-C oracle restatement (oracle/oracle.c) against the reference
itself (oracle/_ref, compiled from /root/reference) and the golden KATs.  CPU only."""
import json
import os

import numpy as np
import pytest

from helpers import W, lex_sorted_unique, random_list

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def oc():
    from oracle import c as OC
    if not OC.available():
        pytest.skip("oracle/lib/liboracle.so not built")
    return OC


@pytest.mark.parametrize("n,k,seed", [(7, 2, 1), (300, 2, 0), (570, 2, 3), (26, 25, 2)])
def test_generators(oc, ref, n, k, seed):
    assert np.array_equal(oc.random_automaton(n, k, seed), ref.random_automaton(n, k, seed))
    assert oc.lib().or_instance_seed(7, n, seed) == ref.instance_seed(7, n, seed)


@pytest.mark.parametrize("n,k", [(20, 2), (100, 3), (300, 2), (130, 2)])
@pytest.mark.parametrize("inverse", [False, True])
def test_expand(oc, ref, n, k, inverse):
    d = ref.random_automaton(n, k, 4)
    words = random_list(n, 300, 0.1, 5)
    assert all(np.array_equal(x, y) for x, y in zip(oc.expand(n, k, d, words, inverse),
                                                     ref.expand(n, k, d, words, inverse)))


@pytest.mark.parametrize("n,dens", [(30, 0.3), (100, 0.08), (300, 0.5)])
def test_sorts_and_dedupe(oc, ref, n, dens):
    base = random_list(n, 400, dens, 1)
    words = np.concatenate([base, base[: 100 * W(n)]])
    tags = np.arange(words.size // W(n), dtype=np.uint64)
    a = oc.lex_sort_dedupe(n, words, tags)
    b = ref.lex_sort_dedupe(n, words, tags)
    assert all(np.array_equal(x, y) for x, y in zip(a, b[:3]))
    a = oc.sort_card_desc_lex(n, words, tags)
    b = ref.sort_card_desc_lex(n, words, tags)
    assert all(np.array_equal(x, y) for x, y in zip(a, b))


@pytest.mark.parametrize("n,dens,count", [(20, 0.3, 800), (100, 0.08, 1500), (300, 0.9, 500)])
def test_containment(oc, ref, n, dens, count):
    words = lex_sorted_unique(n, random_list(n, count, dens, count))
    assert np.array_equal(oc.self_reduce_minimal(n, words), ref.self_reduce_minimal(n, words))
    b = np.concatenate([random_list(n, 600, min(1.0, dens * 3), 9), words[: 50 * W(n)]])
    for mode in (0, 1, 2):
        assert np.array_equal(oc.mark(n, words, b, mode), ref.mark(n, words, b, mode))
    assert oc.meet_check(n, words, b) == ref.meet_check(n, words, b)
    assert oc.trie_node_count(n, words) == ref.trie_node_count(n, words)[0]


def test_exp_mark_and_powerset(oc, ref):
    assert oc.exp_mark(2, 2, 0.5, 0.5) == 21.0
    rng = np.random.default_rng(3)
    for _ in range(500):
        a = rng.uniform(0, 1e6, 4)
        a[2:] = rng.uniform(-0.1, 1.1, 2)
        assert oc.exp_mark(*a) == ref.exp_mark(*a)
    kats = json.load(open(os.path.join(GOLDEN, "powerset_kats.json")))
    for kat in kats[::7]:
        d = oc.random_automaton(kat["n"], kat["k"], kat["seed"])
        assert oc.power_set_oracle(kat["n"], kat["k"], d) == kat["oracle"]


SLOW = json.load(open(os.path.join(GOLDEN, "slow_sync.json")))


@pytest.mark.parametrize("case", SLOW, ids=[c["name"] for c in SLOW])
def test_power_set_oracle_slow_sync(oc, case):
    """Config 5: the extremal (slowly synchronizing) class, thresholds pinned by
    the reference's power-set oracle in tests/golden/make_slow.py."""
    d = np.asarray(case["delta"], np.uint32)
    assert oc.power_set_oracle(case["n"], case["k"], d) == case["threshold"]
