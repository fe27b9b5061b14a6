// oracle/shim_driver.cpp — TEST INFRASTRUCTURE ONLY.
//
// Compiles the reference-side binding include/synchro_b200_shim.hpp exactly
// as a maintainer of the reference would use it: the UNMODIFIED reference
// headers (/root/reference/proj/include) for the types, libsynchro_b200.so for
// the engine.  For every case read from stdin it runs the reference's own
// synchro::solve_exact (bibfs_engine.hpp:467) and synchro::solve_exact_b200
// with the same SolveOptions and prints both results on one line
// (tests/test_gpu_cli_engine.py compares them).
//
// stdin, one case per line:
//   spec memory track_word upper_bound dfs_largest history_growth beam_initial
//   beam_cost_fraction reduction_of_reduction(<=0: unset) set_cost
// stdout: spec | ref t ub it bfs ibfs dfs peak | b200 t ub it bfs ibfs dfs peak | trace_equal word_ok
// `shim_driver --version` touches only host entry points (no device).
#include <iostream>
#include <sstream>
#include <string>

#include "synchro/synchro.hpp"
#include "synchro_b200_shim.hpp"

using namespace synchro;

static Automaton from_spec(const std::string& spec) {
  const auto c = spec.find(':');
  const std::string kind = spec.substr(0, c), args = spec.substr(c + 1);
  if (kind == "cerny") return cerny_automaton(static_cast<u32>(std::stoul(args)));
  u32 n, k;
  unsigned long long seed;
  char sep;
  std::istringstream is(args);
  is >> n >> sep >> k >> sep >> seed;
  return random_automaton(n, k, seed);
}

static std::string fmt(const SolveResult& r) {
  std::ostringstream os;
  os << r.threshold << ' ' << r.upper_bound << ' ' << r.iterations << ' ' << r.bfs_steps << ' '
     << r.ibfs_steps << ' ' << (r.used_dfs ? 1 : 0) << ' ' << r.peak_memory;
  return os.str();
}

int main(int argc, char** argv) {
  if (argc > 1 && std::string(argv[1]) == "--version") {
    sw_solve_options o;
    sw_default_options(&o);
    std::cout << sw_version() << " dfs_largest=" << o.dfs_largest
              << " history_growth=" << o.history_growth << '\n';
    return 0;
  }
  std::string line;
  while (std::getline(std::cin, line)) {
    if (line.empty()) continue;
    std::istringstream is(line);
    std::string spec;
    unsigned long long memory, upper_bound, dfs_largest, beam_initial;
    int track_word;
    double history_growth, beam_cost_fraction, ror, set_cost;
    is >> spec >> memory >> track_word >> upper_bound >> dfs_largest >> history_growth >>
        beam_initial >> beam_cost_fraction >> ror >> set_cost;
    const Automaton aut = from_spec(spec);
    SolveOptions opt;
    opt.memory = memory;
    opt.track_word = track_word != 0;
    if (upper_bound) opt.upper_bound = upper_bound;
    opt.tuning.dfs_largest = dfs_largest;
    opt.tuning.history_growth = history_growth;
    opt.tuning.beam_initial = beam_initial;
    opt.tuning.beam_cost_fraction = beam_cost_fraction;
    if (ror > 0) opt.tuning.cost.dfs_reduction_of_reduction = ror;
    opt.tuning.cost.set_cost = set_cost;
    std::ostringstream t_ref, t_b200;
    opt.trace = &t_ref;
    const SolveResult a = solve_exact(aut, opt);
    opt.trace = &t_b200;
    const SolveResult b = solve_exact_b200(aut, opt);
    const bool word_ok = !opt.track_word ||
                         (b.word && b.word->size() == b.threshold && is_reset_word(aut, *b.word));
    std::cout << spec << " | ref " << fmt(a) << " | b200 " << fmt(b) << " | "
              << (t_ref.str() == t_b200.str() ? 1 : 0) << ' ' << (word_ok ? 1 : 0) << std::endl;
  }
  return 0;
}
