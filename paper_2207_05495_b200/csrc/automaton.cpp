#include "automaton.hpp"

#include <algorithm>
#include <bit>
#include <istream>
#include <ostream>
#include <sstream>

namespace synchro {

Automaton::Automaton(u32 n, u32 k, std::vector<u32> delta) : n_(n), k_(k), delta_(std::move(delta)) {
  if (n_ < 1 || k_ < 1) throw std::invalid_argument("automaton needs n >= 1 and k >= 1");
  if (delta_.size() != static_cast<size_t>(n_) * k_)
    throw std::invalid_argument("transition table has wrong size");
  if (std::any_of(delta_.begin(), delta_.end(), [&](u32 t) { return t >= n_; }))
    throw std::invalid_argument("transition target out of range");
}

InverseTransitions::InverseTransitions(const Automaton& aut)
    : n_(aut.state_count()), k_(aut.alphabet_size()) {
  // Counting sort of (a, delta(p,a)) keys; sources stay in increasing p.
  off_.assign(static_cast<size_t>(k_) * n_ + 1, 0);
  for (u32 p = 0; p < n_; ++p)
    for (u32 a = 0; a < k_; ++a) off_[static_cast<size_t>(a) * n_ + aut.next(p, a) + 1]++;
  for (size_t i = 1; i < off_.size(); ++i) off_[i] += off_[i - 1];
  src_.resize(static_cast<size_t>(n_) * k_);
  std::vector<u32> cursor(off_.begin(), off_.end() - 1);
  for (u32 p = 0; p < n_; ++p)
    for (u32 a = 0; a < k_; ++a) src_[cursor[static_cast<size_t>(a) * n_ + aut.next(p, a)]++] = p;
}

static inline void set_bit(std::vector<u64>& s, u32 q) { s[q >> 6] |= u64{1} << (63 - (q & 63)); }

std::vector<u64> host_universe(u32 n) {
  std::vector<u64> s(words_for(n), ~u64{0});
  if (n & 63) s.back() &= ~u64{0} << (64 - (n & 63));
  return s;
}

std::vector<u64> host_image(const Automaton& aut, const std::vector<u64>& s, u32 a) {
  std::vector<u64> out(s.size(), 0);
  for (size_t w = 0; w < s.size(); ++w)
    for (u64 bits = s[w]; bits; bits &= bits - 1) {
      const u32 q = static_cast<u32>(w * 64 + 63 - std::countr_zero(bits));
      set_bit(out, aut.next(q, a));
    }
  return out;
}

u32 host_card(const std::vector<u64>& s) {
  u32 c = 0;
  for (u64 w : s) c += static_cast<u32>(std::popcount(w));
  return c;
}

bool is_reset_word(const Automaton& aut, const Word& w) {
  std::vector<u64> s = host_universe(aut.state_count());
  for (u32 a : w) {
    if (a >= aut.alphabet_size()) return false;
    s = host_image(aut, s, a);
  }
  return host_card(s) == 1;
}

// Backward BFS over unordered state pairs from the diagonal
// (automaton.hpp:119-148 semantics).
std::vector<u32> pair_merge_distances(const Automaton& aut, const InverseTransitions& inv) {
  const u32 n = aut.state_count(), k = aut.alphabet_size();
  constexpr u32 kInf = std::numeric_limits<u32>::max();
  std::vector<u32> dist(pair_index(n - 1, n - 1) + 1, kInf);
  std::vector<std::pair<u32, u32>> frontier;
  frontier.reserve(n);
  for (u32 q = 0; q < n; ++q) {
    dist[pair_index(q, q)] = 0;
    frontier.emplace_back(q, q);
  }
  // A FIFO queue and level-by-level frontiers give identical distances.
  std::vector<std::pair<u32, u32>> next;
  for (u32 d = 0; !frontier.empty(); ++d) {
    next.clear();
    for (auto [u, v] : frontier)
      for (u32 a = 0; a < k; ++a) {
        auto [pb, pe] = inv.sources(a, u);
        auto [qb, qe] = inv.sources(a, v);
        for (const u32* x = pb; x != pe; ++x)
          for (const u32* y = qb; y != qe; ++y) {
            const u32 p = std::min(*x, *y), q = std::max(*x, *y);
            u32& dd = dist[pair_index(p, q)];
            if (dd == kInf) {
              dd = d + 1;
              next.emplace_back(p, q);
            }
          }
      }
    frontier.swap(next);
  }
  return dist;
}

bool is_synchronizing(const Automaton& aut) {
  const InverseTransitions inv(aut);
  const auto dist = pair_merge_distances(aut, inv);
  return std::find(dist.begin(), dist.end(), std::numeric_limits<u32>::max()) == dist.end();
}

Automaton random_automaton(u32 n, u32 k, u64 seed) {
  SplitMix64 rng(seed);
  std::vector<u32> delta(static_cast<size_t>(n) * k);
  for (u32& t : delta) t = static_cast<u32>(rng.below(n));
  return Automaton(n, k, std::move(delta));
}

Automaton cerny_automaton(u32 n) {
  if (n < 2) throw std::invalid_argument("cerny automaton needs n >= 2");
  std::vector<u32> delta(static_cast<size_t>(n) * 2);
  for (u32 q = 0; q < n; ++q) {
    delta[2 * q] = (q + 1) % n;       // cyclic shift
    delta[2 * q + 1] = q ? q : 1;     // merges 0 into 1
  }
  return Automaton(n, 2, std::move(delta));
}

Automaton parse_automaton(std::istream& in) {
  std::vector<u32> nums;
  std::string line;
  while (std::getline(in, line)) {
    if (auto h = line.find('#'); h != std::string::npos) line.resize(h);
    std::istringstream ls(line);
    long long v;
    while (ls >> v) {
      if (v < 0) throw ParseError("negative value in automaton file");
      nums.push_back(static_cast<u32>(v));
    }
    if (!ls.eof()) throw ParseError("invalid token in automaton file");
  }
  if (nums.size() < 2) throw ParseError("missing automaton header");
  const u32 n = nums[0], k = nums[1];
  if (n < 1 || k < 1) throw ParseError("automaton header must satisfy n >= 1, k >= 1");
  if (nums.size() != 2 + static_cast<size_t>(n) * k)
    throw ParseError("wrong number of transitions in automaton file");
  std::vector<u32> delta(nums.begin() + 2, nums.end());
  for (u32 t : delta)
    if (t >= n) throw ParseError("transition target out of range");
  return Automaton(n, k, std::move(delta));
}

Automaton parse_automaton(const std::string& text) {
  std::istringstream in(text);
  return parse_automaton(in);
}

void write_automaton(std::ostream& out, const Automaton& aut) {
  out << aut.state_count() << ' ' << aut.alphabet_size() << '\n';
  for (u32 q = 0; q < aut.state_count(); ++q) {
    for (u32 a = 0; a < aut.alphabet_size(); ++a) out << (a ? " " : "") << aut.next(q, a);
    out << '\n';
  }
}

}  // namespace synchro
