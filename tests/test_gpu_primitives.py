"""Parity of each B200 data-plane primitive against the reference (oracle/_ref),
called through the C-ABI (include/synchro_b200.h) on seeded random lists.

Bar: bit-exact — same words, same order, same cardinalities, same surviving
tags (which duplicate survives, set_list.hpp:208-209).
"""
import os

import numpy as np
import pytest

from helpers import W, lex_sorted_unique, random_list, rows

pytestmark = pytest.mark.gpu

SHAPES = [(20, 0.3), (64, 0.1), (100, 0.08), (300, 0.077), (570, 0.05), (129, 0.5), (1, 0.5)]


@pytest.mark.parametrize("n,k,seed", [(20, 2, 0), (100, 2, 3), (300, 2, 0), (570, 2, 1),
                                      (200, 3, 0), (26, 25, 4), (64, 2, 5), (1, 1, 0)])
@pytest.mark.parametrize("inverse", [False, True])
def test_expand_matches_transition_kernel(gpu, ref, n, k, seed, inverse):
    aut = gpu.random_automaton(n, k, seed)
    words = random_list(n, 3000, 0.1, seed + 11)
    ow, oc = gpu.list_expand(aut, words, inverse)
    rw, rc = ref.expand(n, k, aut.delta, words, inverse)
    assert np.array_equal(ow, rw)
    assert np.array_equal(oc, rc)


def test_expand_empty_list(gpu):
    aut = gpu.random_automaton(50, 2, 1)
    ow, oc = gpu.list_expand(aut, np.zeros(0, np.uint64), False)
    assert ow.size == 0 and oc.size == 0


@pytest.mark.parametrize("n,density", SHAPES)
def test_lex_sort_dedupe(gpu, ref, n, density):
    base = random_list(n, 1500, density, 7)
    words = np.concatenate([base, base[: 600 * W(n)], random_list(n, 500, density, 8)])
    tags = np.arange(words.size // W(n), dtype=np.uint64) * 7 + 3
    gw, gc, gt = gpu.list_lex_sort_dedupe(n, words, tags)
    rw, rc, rt, _ = ref.lex_sort_dedupe(n, words, tags)
    assert np.array_equal(gw, rw) and np.array_equal(gc, rc) and np.array_equal(gt, rt)


def _first_occurrence(n, words):
    seen, keep = set(), []
    for i, r in enumerate(rows(n, words)):
        if r not in seen:
            seen.add(r)
            keep.append(i)
    return np.array(keep, dtype=np.int64)


def _as_set(n, words, cards, tags=None):
    rs = rows(n, words)
    return sorted(zip(rs, cards.tolist(), tags.tolist() if tags is not None else [0] * len(rs)))


@pytest.mark.parametrize("n,density", SHAPES)
@pytest.mark.parametrize("count", [1, 2, 127, 128, 129, 513, 7000])
def test_hash_dedupe_first_occurrence(gpu, n, density, count):
    """Tagged: the survivors are the first occurrences (row, card, tag) — the
    set lex_sort_dedupe keeps; order unspecified."""
    rng = np.random.default_rng(count + n)
    base = random_list(n, max(1, count // 2), density, 11).reshape(-1, W(n))
    pick = rng.integers(0, base.shape[0], size=count)  # ~half duplicates, scattered
    words = base[pick].reshape(-1)
    tags = rng.integers(0, 2**48, size=count, dtype=np.uint64)
    keep = _first_occurrence(n, words)
    kw = words.reshape(-1, W(n))[keep].reshape(-1)
    gw, gc, gt = gpu.list_hash_dedupe(n, words, tags)
    assert _as_set(n, gw, gc, gt) == _as_set(n, kw, gpu.cards_of(n, kw), tags[keep])


@pytest.mark.parametrize("n,density", SHAPES)
@pytest.mark.parametrize("count", [1, 129, 7000])
def test_hash_dedupe_untagged(gpu, n, density, count):
    rng = np.random.default_rng(count * 3 + n)
    base = random_list(n, max(1, count // 2), density, 13).reshape(-1, W(n))
    words = base[rng.integers(0, base.shape[0], size=count)].reshape(-1)
    gw, gc, _ = gpu.list_hash_dedupe(n, words)
    out = rows(n, gw)
    assert len(out) == len(set(out)) and set(out) == set(rows(n, words))
    assert np.array_equal(gc, gpu.cards_of(n, gw))


@pytest.mark.parametrize("tagged", [False, True])
def test_hash_dedupe_long_probe_chains(gpu, monkeypatch, tagged):
    """A table packed to N+64 slots: long probe chains (past the one-byte probe
    distance of the tagged path's resolve kernel); survivors must not change."""
    monkeypatch.setenv("SYNCHRO_DEDUPE_FULL_TABLE", "1")
    n = 100
    base = random_list(n, 30000, 0.1, 12).reshape(-1, W(n))
    pick = np.random.default_rng(5).integers(0, base.shape[0], size=40000)
    words = base[pick].reshape(-1)
    keep = _first_occurrence(n, words)
    kw = words.reshape(-1, W(n))[keep].reshape(-1)
    if tagged:
        tags = np.arange(40000, dtype=np.uint64)
        gw, gc, gt = gpu.list_hash_dedupe(n, words, tags)
        assert _as_set(n, gw, gc, gt) == _as_set(n, kw, gpu.cards_of(n, kw), tags[keep])
    else:
        gw, gc, _ = gpu.list_hash_dedupe(n, words)
        assert _as_set(n, gw, gc) == _as_set(n, kw, gpu.cards_of(n, kw))


@pytest.mark.parametrize("n", [20, 300, 570])
def test_hash_dedupe_wide_table_path(gpu, monkeypatch, n):
    """The 64-bit-entry table used for lists of >= 2^25 rows (forced here):
    first occurrences survive, in their original order."""
    monkeypatch.setenv("SYNCHRO_DEDUPE_WIDE", "1")
    base = random_list(n, 3000, 0.1, 17).reshape(-1, W(n))
    pick = np.random.default_rng(n).integers(0, base.shape[0], size=5000)
    words = base[pick].reshape(-1)
    tags = np.arange(5000, dtype=np.uint64) * 3
    keep = _first_occurrence(n, words)
    gw, _, gt = gpu.list_hash_dedupe(n, words, tags)
    assert np.array_equal(gw.reshape(-1, W(n)), words.reshape(-1, W(n))[keep])
    assert np.array_equal(gt, tags[keep])


def test_hash_dedupe_empty(gpu):
    gw, gc, _ = gpu.list_hash_dedupe(100, np.zeros(0, np.uint64))
    assert gw.size == 0 and gc.size == 0


@pytest.mark.parametrize("n,density", SHAPES)
def test_sort_card_desc_lex_and_dedupe(gpu, ref, n, density):
    base = random_list(n, 2000, density, 9)
    words = np.concatenate([base, base[: 300 * W(n)]])
    tags = np.arange(words.size // W(n), dtype=np.uint64)
    gw, gc, gt = gpu.list_sort_card_desc_lex(n, words, tags)
    rw, rc, rt = ref.sort_card_desc_lex(n, words, tags)
    assert np.array_equal(gw, rw) and np.array_equal(gc, rc) and np.array_equal(gt, rt)
    dw, dc, dt = gpu.list_dedupe_sorted(n, gw, gt)
    assert len(set(rows(n, dw))) == dw.size // W(n) == len(set(rows(n, words)))


@pytest.mark.parametrize("n,density,count", [(20, 0.3, 3000), (100, 0.08, 20000),
                                             (300, 0.077, 30000), (300, 0.95, 3000),
                                             (570, 0.06, 20000), (64, 0.5, 4000), (2, 0.5, 4)])
def test_self_reduce_minimal(gpu, ref, n, density, count):
    words = lex_sorted_unique(n, random_list(n, count, density, count))
    g = gpu.list_self_reduce_minimal(n, words)
    r = ref.self_reduce_minimal(n, words)
    assert np.array_equal(g, r)


@pytest.mark.parametrize("mode", [0, 1, 2])
@pytest.mark.parametrize("n,da,db", [(30, 0.2, 0.5), (100, 0.05, 0.3), (300, 0.05, 0.2),
                                     (300, 0.9, 0.95), (570, 0.03, 0.2),
                                     # n <= 20: the power-set bitmap path (bitmap.cu)
                                     (20, 0.3, 0.6), (13, 0.4, 0.5), (4, 0.5, 0.5), (1, 0.5, 0.5)])
def test_mark_modes(gpu, ref, mode, n, da, db):
    a = lex_sorted_unique(n, random_list(n, 4000, da, 1))
    b = random_list(n, 6000, db, 2)
    b = np.concatenate([b, a[: 100 * W(n)]])  # equal sets exercise proper vs non-proper
    g = gpu.list_mark(n, a, b, mode)
    r = ref.mark(n, a, b, mode)
    assert np.array_equal(g, r)


def test_mark_rejects_unsorted_a(gpu):
    n = 40
    a = random_list(n, 50, 0.3, 3)
    b = random_list(n, 50, 0.3, 4)
    with pytest.raises(gpu.SynchroError):
        gpu.list_mark(n, a[::-1].copy(), b, 0)


@pytest.mark.parametrize("n,da,db,seed", [(100, 0.1, 0.4, 0), (300, 0.08, 0.3, 1),
                                          (300, 0.08, 0.1, 2), (64, 0.3, 0.3, 3),
                                          (20, 0.3, 0.4, 4), (9, 0.4, 0.3, 5)])
def test_meet_check(gpu, ref, n, da, db, seed):
    a = lex_sorted_unique(n, random_list(n, 20000, da, seed))
    b = random_list(n, 2000, db, seed + 100)
    assert gpu.list_meet_check(n, a, b) == ref.meet_check(n, a, b)
    # planted containment
    b2 = b.copy()
    b2[: W(n)] = a[5 * W(n): 6 * W(n)] | b2[: W(n)]
    assert gpu.list_meet_check(n, a, b2) and ref.meet_check(n, a, b2)


@pytest.mark.parametrize("n,density,count,min_leaf", [(20, 0.3, 500, 10), (100, 0.08, 20000, 10),
                                                      (300, 0.077, 50000, 10), (300, 0.95, 5000, 10),
                                                      (570, 0.05, 30000, 3), (64, 0.5, 7, 10)])
def test_trie_node_count(gpu, ref, n, density, count, min_leaf):
    words = lex_sorted_unique(n, random_list(n, count, density, count + 1))
    assert gpu.trie_node_count(n, words, min_leaf) == ref.trie_node_count(n, words, min_leaf)[0]


def _prefix_tie_list(n, count, seed):
    """Rows whose leading words take only a few values, so the packed 64-bit
    prefix key ties a lot and the order is decided by the refinement passes
    over the later words (and, for equal rows, by the index tie-break)."""
    rng = np.random.default_rng(seed)
    words = random_list(n, count, 0.3, seed).reshape(-1, W(n))
    for w in range(min(2, W(n) - 1)):
        pool = random_list(n, 3, 0.5, seed + 100 + w).reshape(-1, W(n))[:, w]
        words[:, w] = pool[rng.integers(0, 3, count)]
    dup = rng.integers(0, count, count // 5)
    words = np.concatenate([words, words[dup]])
    return np.ascontiguousarray(words.reshape(-1))


@pytest.mark.parametrize("n", [100, 300, 570])
def test_sorts_with_prefix_ties(gpu, ref, n):
    words = _prefix_tie_list(n, 4000, n)
    tags = np.arange(words.size // W(n), dtype=np.uint64) * 3 + 1
    gw, gc, gt = gpu.list_sort_card_desc_lex(n, words, tags)
    rw, rc, rt = ref.sort_card_desc_lex(n, words, tags)
    assert np.array_equal(gw, rw) and np.array_equal(gc, rc) and np.array_equal(gt, rt)
    gw, gc, gt = gpu.list_lex_sort_dedupe(n, words, tags)
    rw, rc, rt, _ = ref.lex_sort_dedupe(n, words, tags)
    assert np.array_equal(gw, rw) and np.array_equal(gc, rc) and np.array_equal(gt, rt)


@pytest.mark.parametrize("n,nranks", [(300, 1), (300, 2), (300, 3), (570, 8), (100, 5)])
def test_dev_owner_partition_matches_owner_hash(gpu, n, nranks):
    """sw_dev_owner_partition (exchange.cu) groups rows owner-major by the owner
    hash restated in distributed.owner_hash; rows keep their cards."""
    import torch

    from paper_2207_05495_b200.distributed import owner_hash
    base = random_list(n, 3000, 0.08, n + nranks)
    words = np.concatenate([base, base[: 500 * W(n)]])
    cards = gpu.cards_of(n, words).astype(np.int32)
    tw = torch.from_numpy(words.view(np.int64)).cuda()
    tc = torch.from_numpy(cards).cuda()
    ow, oc, counts = gpu.dev_owner_partition(n, tw, tc, nranks)
    own = owner_hash(words, W(n), nranks)
    assert counts == np.bincount(own, minlength=nranks).tolist()
    ow = ow.cpu().numpy().view(np.uint64).reshape(-1, W(n))
    oc = oc.cpu().numpy()
    start = 0
    for r, cnt in enumerate(counts):
        seg = ow[start:start + cnt]
        assert (owner_hash(seg.reshape(-1), W(n), nranks) == r).all()
        start += cnt
    assert sorted(map(tuple, ow.tolist())) == sorted(rows(n, words))
    assert (oc == gpu.cards_of(n, ow.reshape(-1))).all()


def test_dev_hash_dedupe_and_world1_nccl_exchange(gpu, tmp_path):
    """Device-pointer dedupe, and owner_exchange_dedupe through a real NCCL
    group of one rank (the all-to-all path the 8-GPU run takes)."""
    import subprocess
    import sys

    import torch
    n = 300
    base = random_list(n, 4000, 0.08, 3)
    words = np.concatenate([base, base[: 1500 * W(n)]])
    cards = gpu.cards_of(n, words).astype(np.int32)
    dw, dc = gpu.dev_hash_dedupe(n, torch.from_numpy(words.view(np.int64)).cuda(),
                                 torch.from_numpy(cards).cuda())
    got = dw.cpu().numpy().view(np.uint64)
    assert sorted(rows(n, got)) == sorted(set(rows(n, words)))
    np.save(tmp_path / "w.npy", words)
    code = f"""
import sys, numpy as np, torch, torch.distributed as dist
sys.path.insert(0, {os.path.dirname(os.path.dirname(os.path.abspath(__file__)))!r})
dist.init_process_group("nccl", init_method="tcp://127.0.0.1:{29500 + os.getpid() % 1000}", rank=0, world_size=1)
torch.cuda.set_device(0)
from paper_2207_05495_b200 import distributed, native
w = np.load({str(tmp_path / "w.npy")!r})
c = native.cards_of({n}, w).astype(np.int32)
ow, oc, sent = distributed.owner_exchange_dedupe({n}, torch.from_numpy(w.view(np.int64)).cuda(),
                                                 torch.from_numpy(c).cuda())
np.save({str(tmp_path / "o.npy")!r}, ow.cpu().numpy().view(np.uint64))
print("sent", sent)
dist.destroy_process_group()
"""
    p = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, p.stderr[-3000:]
    out = np.load(tmp_path / "o.npy")
    assert sorted(rows(n, out)) == sorted(set(rows(n, words)))
    assert "sent 0" in p.stdout


_OVERFLOW_PROBE = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1]); sys.path.insert(0, sys.argv[1] + '/tests')
from helpers import W, lex_sorted_unique, random_list
from paper_2207_05495_b200 import native as gpu
from oracle import ref
bad = []
for n, da, db in [(300, 0.05, 0.2), (100, 0.05, 0.3), (570, 0.03, 0.2)]:
    a = lex_sorted_unique(n, random_list(n, 30000, da, 1))
    b = np.concatenate([random_list(n, 8000, db, 2), a[: 100 * W(n)]])
    for mode in (0, 1):
        if not np.array_equal(gpu.list_mark(n, a, b, mode), ref.mark(n, a, b, mode)):
            bad.append(("mark", n, mode))
    if gpu.list_self_reduce_minimal(n, a).tobytes() != ref.self_reduce_minimal(n, a).tobytes():
        bad.append(("self", n))
    if gpu.list_meet_check(n, a, b[: 2000 * W(n)]) != ref.meet_check(n, a, b[: 2000 * W(n)]):
        bad.append(("meet", n))
print("BAD", bad)
"""


@pytest.mark.parametrize("index", ["", "trie"])
@pytest.mark.parametrize("spill_cap", ["0", "128"])
def test_containment_pool_overflow_scan_path(gpu, ref, spill_cap, index):
    """contain.cu: when a warp's task pool and its spill stack are both full, the
    opened range is scanned instead of descended.  SYNCHRO_SPILL_CAP shrinks the
    stack so that path runs (the progress log counts overflow scans); marks,
    self-reduction and meet must still equal the reference's
    (subset_algebra.hpp:55-231)."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, SYNCHRO_SPILL_CAP=spill_cap, SYNCHRO_PROGRESS="1")
    if index:  # marking through the trie index too (device/trie_query.cu)
        env["SYNCHRO_INDEX"] = index
    p = subprocess.run([sys.executable, "-c", _OVERFLOW_PROBE, root], env=env,
                       capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    assert "BAD []" in p.stdout, p.stdout
    scans = [int(x) for x in __import__("re").findall(r"overflow_scans=(\d+)", p.stderr)]
    assert scans and max(scans) > 0, "overflow path not exercised"


@pytest.mark.parametrize("n,da,db,seed", [(100, 0.1, 0.4, 0), (300, 0.08, 0.3, 1), (64, 0.3, 0.3, 3),
                                         (570, 0.05, 0.2, 2), (1000, 0.03, 0.15, 4)])
def test_trie_exists_any_key_order(gpu, ref, n, da, db, seed):
    """The trie index (device/trie_query.cu) over keys in ANY order (the engine
    indexes L_BFS in hash order): one planted containment is found wherever it
    lies, including under the root's one side."""
    keys = lex_sorted_unique(n, random_list(n, 5000, da, seed)).reshape(-1, W(n))
    rng = np.random.default_rng(seed)
    keys = keys[rng.permutation(len(keys))]
    b = random_list(n, 1500, db, seed + 7).reshape(-1, W(n)).copy()
    met, _, _ = gpu.list_trie_exists(n, keys.reshape(-1), b.reshape(-1))
    assert met == ref.meet_check(n, lex_sorted_unique(n, keys.reshape(-1)), b.reshape(-1))
    for pick in (0, len(keys) // 2, len(keys) - 1):
        b2 = b.copy()
        b2[17] |= keys[pick]
        met, ai, bi = gpu.list_trie_exists(n, keys.reshape(-1), b2.reshape(-1))
        assert met
        assert np.all((keys[ai] & ~b2[bi]) == 0)


def _two_component(n):
    """Two disjoint cycles (states < n/2 and >= n/2): no pair across them merges."""
    h = n // 2
    d = np.zeros(n * 2, np.uint32)
    for q in range(n):
        lo, size = (0, h) if q < h else (h, n - h)
        d[2 * q] = lo + (q - lo + 1) % size      # rotate inside the component
        d[2 * q + 1] = lo if q - lo < 2 else q   # merge the component's first two states
    return d


@pytest.mark.parametrize("spec", ["random:50,2,1", "random:300,2,0", "random:570,2,0",
                                  "random:200,3,1", "cerny:20", "cerny:64", "batch553",
                                  "split200"])
def test_pair_distances_device_equals_host(gpu, ref, spec):
    """The pair-automaton BFS on the GPU (device/pairs.cu) equals the host's
    level-synchronous BFS entry for entry (automaton.hpp:119-157), including the
    unmergeable pairs of non-synchronizing automata; solve_exact takes the device
    table from kPairBfsDeviceMin states on, so a non-synchronizing automaton of
    200 states must still be refused."""
    if spec == "batch553":  # config 2's non-synchronizing instance (instance_seed(0,100,553))
        aut = gpu.random_automaton(100, 2, 16462524638486953121)
    elif spec == "split200":
        aut = gpu.Automaton(200, 2, _two_component(200))
    else:
        aut = gpu.from_spec(spec)
    d = gpu.pair_distances(aut, on_device=True)
    h = gpu.pair_distances(aut, on_device=False)
    assert np.array_equal(d, h)
    sync = bool((d != np.iinfo(np.uint32).max).all())
    assert sync == gpu.is_synchronizing(aut) == bool(ref.is_synchronizing(aut.n, aut.k, aut.delta))
    if spec == "split200":
        assert not sync
        with pytest.raises(gpu.NotSynchronizingError):
            gpu.solve_exact(aut)
