// The orders in which the reference leaves L_IBFS after its meet checks and a
// DFS level after its trie queries.
//
// Without word tracking the reference meets through meet_check
// (subset_algebra.hpp:201-210), which runs mark_rec (:55-125) with B = L_IBFS
// accessed directly: the partition loop at :112-119 swaps L_IBFS elements in
// place.  A meet check that finds nothing (the only kind the search survives)
// marks nothing, so the brute-force leaves (:60-86) move nothing and only the
// partitions permute B.  The order is observable once: the DFS cuts its
// top-level slices out of L_IBFS in that order (dfs_phase.hpp:52-56) when the
// ledger's slice cap is smaller than the list.  The engine therefore keeps the
// L_BFS lists met since the last inverse step and, only when the DFS will
// slice, replays the recursion's partitions here (host, integer only).  The
// same holds one level down: a DFS level's slices are cut after the per-group
// trie queries have permuted each cardinality group (replay_trie_query).
#pragma once

#include <cstddef>
#include <vector>

#include "common.hpp"
#include "device/dev.hpp"

namespace synchro::detail {

// Applies the permutation of one meet_check(A, B) that found no containment
// to `order` (order[p] = original index of the B element at position p):
// A = lex-sorted unique rows (count na, W words each), B = the rows in their
// original positions.  nbits = n, min_brute = EngineTuning::min_brute.
void replay_meet_check(const u64* A, size_t na, const u64* B, u32 W, u32 nbits, size_t min_brute,
                       std::vector<u32>& order);

// The same for the DFS's trie query of one cardinality group
// (StaticTrie::contains_subset_of_any → query_node, static_trie.hpp:51-55,
// :153-188): its partition loop (:177-183) permutes the group in place, and
// the level's slices (dfs_phase.hpp:155-158) are cut after the queries.  Q =
// the group's rows (all of cardinality `card`) in their original positions;
// `trie` = the reference trie's internal nodes (dev::trie_shape).
void replay_trie_query(const dev::TrieShape& trie, const u64* Q, u32 W, u32 card,
                       std::vector<u32>& order);

}  // namespace synchro::detail
