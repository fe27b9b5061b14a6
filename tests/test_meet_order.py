"""The order the reference's meet_check leaves L_IBFS in, replayed on the host.

Without word tracking, meet_check (subset_algebra.hpp:201-210) permutes
L_IBFS in place through mark_rec's partition loop (:112-119); the DFS then
cuts its top-level slices out of that order (dfs_phase.hpp:52-56).  The
engine replays the permutation (csrc/meet_order.cpp) when the DFS slices;
here the replay is compared with the reference's own meet_check on lists
where nothing meets (the only meet checks a search survives).  CPU only.
"""
import numpy as np
import pytest

from helpers import lex_sorted_unique, random_list
from paper_2207_05495_b200 import native as sw


@pytest.mark.parametrize("n", [20, 64, 100, 130, 300])
@pytest.mark.parametrize("na,nb", [(1, 5), (63, 40), (64, 40), (500, 300), (3000, 2000)])
@pytest.mark.parametrize("min_brute", [1, 8, 64])
def test_replay_matches_reference_meet_check(ref, n, na, nb, min_brute):
    seed = n * 7919 + na * 31 + nb + min_brute
    a = lex_sorted_unique(n, random_list(n, na, 0.35, seed))
    b = random_list(n, nb, 0.45, seed + 1)
    met, want = ref.meet_check_order(n, a, b, min_brute)
    if met:
        pytest.skip("lists meet (the search would have ended)")
    got = sw.meet_check_order(n, a, b, min_brute)
    assert np.array_equal(got, want)


def test_replay_composes_over_successive_meets(ref):
    """Two meets in a row (BFS steps between inverse steps) permute the
    already-permuted list: replaying both in order gives the reference's order."""
    n = 100
    b = random_list(n, 1500, 0.5, 11)
    order = np.arange(1500, dtype=np.uint32)
    cur = b.reshape(1500, -1)
    for s in (1, 2, 3):
        a = lex_sorted_unique(n, random_list(n, 400 * s, 0.3, 100 + s))
        met, step = ref.meet_check_order(n, a, cur.reshape(-1), 64)
        assert not met
        mine = sw.meet_check_order(n, a, cur.reshape(-1), 64)
        assert np.array_equal(mine, step)
        cur = cur[step]
        order = order[step]
    assert sorted(order.tolist()) == list(range(1500))


def test_replay_rejects_unsorted_a():
    n = 64
    a = np.array([5, 3], np.uint64)
    b = np.array([7], np.uint64)
    with pytest.raises(sw.SynchroError):
        sw.meet_check_order(n, a, b)
