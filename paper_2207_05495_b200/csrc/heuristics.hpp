// Upper bounds on the reset threshold (paper §1.3.2 / §2.1.3), same API as
// the reference's heuristics.hpp:13-184.  Eppstein's greedy pair merging runs
// on the host (it is O(n^3) integer work on an n×n table); the beam
// (CutOff-IBFS) runs on the device data plane: preimage expansion, (card desc,
// lex) ordering, dedupe and truncation per level are all B200 kernels.
#pragma once

#include <optional>

#include "automaton.hpp"
#include "common.hpp"

namespace synchro {

namespace dev {
class Context;
}

struct HeuristicResult {
  Word word;
  u64 length = 0;
};

struct EppsteinStats {
  HeuristicResult result;
  u32 merge_phases = 0;
};

// `dist` (optional): the pair merge distances already computed by the caller
// (pair_merge_distances, e.g. for the synchronizability check).
EppsteinStats eppstein_with_stats(const Automaton& aut, const Deadline& deadline = {},
                                  const std::vector<u32>* dist = nullptr);
HeuristicResult eppstein(const Automaton& aut, const Deadline& deadline = {});

// Beam inverse BFS keeping the beam_size largest sets per level (card desc,
// lex tie-break); nullopt when it does not reach Q.
std::optional<HeuristicResult> beam_ibfs(const Automaton& aut, u64 beam_size,
                                         const Deadline& deadline = {}, dev::Context* ctx = nullptr);

struct AdaptiveOptions {
  u64 memory = u64{4} << 30;
  u64 initial_beam = 0;  // 0 -> max(64, n)
  double cost_fraction = 0.05;
  const std::vector<u32>* pair_dist = nullptr;  // precomputed pair merge distances (optional)
  double set_cost = 512.0;
  Deadline deadline{};
};

HeuristicResult adaptive_upper_bound(const Automaton& aut, const AdaptiveOptions& opt = {},
                                     dev::Context* ctx = nullptr);

}  // namespace synchro
