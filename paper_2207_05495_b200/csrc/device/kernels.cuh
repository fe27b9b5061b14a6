// Internal cross-file entry points of the device layer.
//
// Scratch-slot convention (Context::scratch): 0/1 sort keys, 2/3 sort
// permutations, 4 CUB temp storage, 5 flag arrays, 6 compaction tile counts,
// 7 small reductions / result words, 8/9 hash-dedupe table and row slots,
// 10 containment-traversal spill stacks.
#pragma once

#include <cstdint>
#include <vector>

#include "dev.hpp"

namespace synchro::dev {

// Keep rows with keep[i] != 0 (all rows when keep == nullptr), in order;
// row i is read from position perm[i] when perm != nullptr.  Replaces l.
size_t compact_flags(Context& c, DList& l, const uint8_t* keep, const u32* perm);
// Keep the first row of every run of equal rows in perm order (sorted input).
size_t compact_unique(Context& c, DList& l, const u32* perm);

// Hash dedupe with a 64-bit (tag << 32 | index) table, for lists whose indices
// exceed the 25 bits of dedupe.cu's compact entries.
size_t hash_dedupe_wide(Context& c, DList& l);

// hist[q] = number of sets of l containing state q (q < n); hist is a device
// array of n u32, overwritten.  Bit-sliced: 64 sets per warp transpose.
void state_histogram(Context& c, const DList& l, u32* hist);

// Stable permutation sorting l lexicographically (optionally by descending
// cardinality first); returned pointer lives in scratch slot 2 or 3.
const u32* sort_perm(Context& c, const DList& l, bool card_desc);
// Per word, the bits that are not constant across l (OR ^ AND; one readback).
std::vector<u64> varying_bits(Context& c, const DList& l);

}  // namespace synchro::dev
