// synchro_b200_shim.hpp — the reference-side binding of the B200 engine.
//
// A maintainer of the reference (/root/reference/proj/include/synchro/) keeps
// its types and swaps the engine call: include this header after
// "synchro/synchro.hpp" and call synchro::solve_exact_b200 where
// synchro::solve_exact (bibfs_engine.hpp:467) was called.  Every field of
// SolveOptions / EngineTuning / TuningParams (bibfs_engine.hpp:27-48,
// cost_model.hpp:26-36) is forwarded; the C-ABI status codes are mapped back
// onto the reference's exception types (tools/synchro.cpp:325-344).  Link with
// -L paper_2207_05495_b200/lib -lsynchro_b200.
#pragma once

#include <unistd.h>

#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "synchro_b200.h"

namespace synchro {

inline sw_solve_options to_sw_options(const SolveOptions& opt) {
  sw_solve_options o;
  sw_default_options(&o);
  o.memory = opt.memory;
  o.time_limit = opt.time_limit ? *opt.time_limit : 0.0;
  o.track_word = opt.track_word ? 1 : 0;
  o.schedule = static_cast<int32_t>(opt.schedule);
  o.upper_bound = opt.upper_bound ? *opt.upper_bound : 0;
  o.set_cost = opt.tuning.cost.set_cost;
  o.dfs_set_weight = opt.tuning.cost.dfs_set_cost_weight;
  o.dfs_check_weight = opt.tuning.cost.dfs_check_cost_weight;
  o.reduction_of_reduction =
      opt.tuning.cost.dfs_reduction_of_reduction ? *opt.tuning.cost.dfs_reduction_of_reduction : 0.0;
  o.min_brute = static_cast<uint32_t>(opt.tuning.min_brute);
  o.min_leaf = opt.tuning.min_leaf;
  o.dfs_largest = opt.tuning.dfs_largest;
  o.dedupe_cadence = opt.tuning.dfs_dedupe_cadence;
  o.reduce_cadence = opt.tuning.dfs_reduce_cadence;
  o.history_growth = opt.tuning.history_growth;
  o.beam_initial = opt.tuning.beam_initial;
  o.beam_cost_fraction = opt.tuning.beam_cost_fraction;
  return o;
}

inline SolveResult solve_exact_b200(const Automaton& aut, const SolveOptions& opt = {}) {
  const sw_solve_options o = to_sw_options(opt);
  std::vector<uint32_t> word(opt.track_word ? (1u << 20) : 1u);
  sw_solve_result r;
  // A borrowed std::ostream* cannot cross a C ABI: the engine writes the
  // trace (same lines as trace_line, bibfs_engine.hpp:442-460) to a file that
  // is copied into opt.trace.
  std::string trace_path;
  if (opt.trace) {
    char tmpl[] = "/tmp/synchro_b200_traceXXXXXX";
    const int fd = mkstemp(tmpl);
    if (fd < 0) throw std::runtime_error("cannot create a trace file");
    close(fd);
    trace_path = tmpl;
  }
  const int rc = sw_solve_exact(aut.state_count(), aut.alphabet_size(), aut.table().data(), &o,
                                &r, word.data(), word.size(),
                                trace_path.empty() ? nullptr : trace_path.c_str());
  if (!trace_path.empty()) {
    std::ifstream in(trace_path);
    *opt.trace << in.rdbuf();
    std::remove(trace_path.c_str());
  }
  switch (rc) {
    case SW_OK: break;
    case SW_ERR_NOT_SYNCHRONIZING: throw NotSynchronizingError();
    case SW_ERR_OUT_OF_MEMORY: throw OutOfMemoryError(sw_last_error());
    case SW_ERR_TIMEOUT: throw TimeoutError();
    case SW_ERR_PARSE: throw std::invalid_argument(sw_last_error());
    default: throw std::runtime_error(sw_last_error());
  }
  SolveResult s;
  s.threshold = r.threshold;
  s.upper_bound = r.upper_bound;
  s.iterations = r.iterations;
  s.bfs_steps = r.bfs_steps;
  s.ibfs_steps = r.ibfs_steps;
  s.used_dfs = r.used_dfs != 0;
  s.peak_memory = r.peak_memory;
  if (r.has_word) s.word = Word(word.begin(), word.begin() + static_cast<long>(r.word_len));
  return s;
}

}  // namespace synchro
