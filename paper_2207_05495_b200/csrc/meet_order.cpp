#include "meet_order.hpp"

#include <utility>

namespace synchro::detail {

namespace {

struct Replay {
  const u64* A;
  const u64* B;
  u32 W, nbits;
  size_t min_brute;
  u32* order;

  bool bit(const u64* row, u32 d) const { return (row[d >> 6] >> (63 - (d & 63))) & 1u; }

  // mark_rec (subset_algebra.hpp:55-125) with nothing marked: the B interval
  // [blo, bend) keeps its ends; the ones-side call is the loop's next round.
  void rec(size_t alo, size_t ahi, size_t blo, size_t bend, u32 d) {
    while (true) {
      if (alo == ahi || blo == bend) return;                 // :58
      if (ahi - alo < min_brute || d >= nbits) return;       // :60 (no hits: nothing moves)
      size_t lo = alo, hi = ahi;                              // :90-101 binary search on bit d
      while (lo < hi) {
        const size_t mid = lo + (hi - lo) / 2;
        if (bit(A + mid * W, d))
          hi = mid;
        else
          lo = mid + 1;
      }
      const size_t asplit = lo;
      rec(alo, asplit, blo, bend, d + 1);                     // :105 zeros side, whole B
      if (asplit == ahi) return;                              // :108
      size_t i = blo, j = bend;                               // :112-119 partition by bit d
      while (i < j) {
        if (!bit(B + static_cast<size_t>(order[i]) * W, d))
          ++i;
        else
          std::swap(order[i], order[--j]);
      }
      alo = asplit;                                           // :121 ones side with B_1
      blo = i;
      ++d;
    }
  }
};

struct TrieReplay {
  const dev::TrieShape& t;
  const u64* Q;
  u32 W, card;
  u32* order;

  // query_node (static_trie.hpp:153-188) with nothing found: payload scans
  // (:158-170) move nothing; the zero child sees the whole range (:173); the
  // partition by the division state (:177-183) runs whenever the node is
  // internal (its one side is always a node), then the one child recurses on
  // the queries holding that state (a leaf one child does nothing).
  void rec(size_t round, u32 id, size_t lo, size_t hi) {
    while (true) {
      const dev::TrieShape::Node& nd = t.rounds[round][id];
      if (nd.min_card > card) return;  // :156
      if (nd.zero != kNone) rec(round + 1, nd.zero, lo, hi);
      size_t i = lo, j = hi;
      while (i < j) {
        const u64* y = Q + static_cast<size_t>(order[i]) * W;
        if (!((y[nd.div >> 6] >> (63 - (nd.div & 63))) & 1u))
          ++i;
        else
          std::swap(order[i], order[--j]);
      }
      if (i >= hi || nd.one == kNone) return;
      ++round;
      id = nd.one;
      lo = i;
    }
  }
  static constexpr u32 kNone = 0xFFFFFFFFu;
};

}  // namespace

void replay_trie_query(const dev::TrieShape& trie, const u64* Q, u32 W, u32 card,
                       std::vector<u32>& order) {
  if (trie.rounds.empty() || order.empty()) return;  // the whole trie is one leaf
  TrieReplay r{trie, Q, W, card, order.data()};
  r.rec(0, 0, 0, order.size());
}

void replay_meet_check(const u64* A, size_t na, const u64* B, u32 W, u32 nbits, size_t min_brute,
                       std::vector<u32>& order) {
  Replay r{A, B, W, nbits, min_brute, order.data()};
  r.rec(0, na, 0, order.size(), 0);
}

}  // namespace synchro::detail
