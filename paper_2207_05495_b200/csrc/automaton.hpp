// Automaton model, generators, text format and host-side verification.
//
// Mirrors the reference's L1 public surface (automaton.hpp): Automaton with
// row-major delta[q*k+a] (automaton.hpp:20-45), the CSR inverse
// (automaton.hpp:48-77), random/Černý generators (automaton.hpp:159-176), the
// text format (automaton.hpp:178-219), is_reset_word (automaton.hpp:106) and
// the pair-automaton synchronizability test (automaton.hpp:112-157).
// The subset-expansion hot kernel (TransitionKernel, automaton.hpp:221-303)
// has NO host counterpart here: it is the device kernel in device/expand.cu.
#pragma once

#include <iosfwd>
#include <string>
#include <utility>
#include <vector>

#include "common.hpp"

namespace synchro {

class Automaton {
 public:
  Automaton(u32 n, u32 k, std::vector<u32> delta);
  u32 state_count() const { return n_; }
  u32 alphabet_size() const { return k_; }
  u32 next(u32 q, u32 a) const { return delta_[static_cast<size_t>(q) * k_ + a]; }
  const std::vector<u32>& table() const { return delta_; }
  bool operator==(const Automaton& o) const {
    return n_ == o.n_ && k_ == o.k_ && delta_ == o.delta_;
  }

 private:
  u32 n_, k_;
  std::vector<u32> delta_;
};

// For letter a and target q: the sources p with delta(p,a) = q, in increasing p.
class InverseTransitions {
 public:
  explicit InverseTransitions(const Automaton& aut);
  std::pair<const u32*, const u32*> sources(u32 a, u32 q) const {
    const size_t i = static_cast<size_t>(a) * n_ + q;
    return {src_.data() + off_[i], src_.data() + off_[i + 1]};
  }
  const std::vector<u32>& offsets() const { return off_; }
  const std::vector<u32>& sources_flat() const { return src_; }

 private:
  u32 n_, k_;
  std::vector<u32> off_;  // k*n + 1
  std::vector<u32> src_;  // n*k
};

// Host bitset helpers (MSB-first packing, state 0 = bit 63 of word 0,
// state_set.hpp:14-19) used for verification and small host-side work.
std::vector<u64> host_universe(u32 n);
std::vector<u64> host_image(const Automaton& aut, const std::vector<u64>& s, u32 a);
u32 host_card(const std::vector<u64>& s);

bool is_reset_word(const Automaton& aut, const Word& w);

// Length of a shortest word merging each unordered pair {p<=q}
// (index q*(q+1)/2 + p); UINT32_MAX when unmergeable.
std::vector<u32> pair_merge_distances(const Automaton& aut, const InverseTransitions& inv);
inline size_t pair_index(u32 p, u32 q) { return static_cast<size_t>(q) * (q + 1) / 2 + p; }
bool is_synchronizing(const Automaton& aut);

Automaton random_automaton(u32 n, u32 k, u64 seed);
Automaton cerny_automaton(u32 n);

Automaton parse_automaton(std::istream& in);
Automaton parse_automaton(const std::string& text);
void write_automaton(std::ostream& out, const Automaton& aut);

}  // namespace synchro
