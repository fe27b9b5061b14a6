// `synchro` command-line front end — same subcommands, flags, stdout/stderr
// formats and exit codes as the reference CLI (proj/tools/synchro.cpp:113-345):
//   exact | heuristic | gen | oracle | experiment | fit
// Exit codes: 0 ok, 2 not synchronizing, 3 parse/input error, 4 memory budget
// exhausted, 5 refused, 6 time limit, 1 other; 10 CUDA/device failure (new).
// The reference parses with CLI11 (absent here); this is a small hand parser
// accepting the same spellings ("--opt value" and "--opt=value").
#include <chrono>
#include <fstream>
#include <iostream>
#include <map>
#include <set>
#include <sstream>
#include <string>
#include <vector>

#include "../device/dev.hpp"
#include "../engine.hpp"
#include "../experiment.hpp"

using namespace synchro;

namespace {

constexpr int kExitNotSynchronizing = 2, kExitParseError = 3, kExitOutOfMemory = 4,
              kExitRefused = 5, kExitTimeout = 6, kExitDevice = 10;
constexpr int kExitUsage = 106;  // CLI11 RequiredError / ValidationError family

struct UsageError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct Args {
  std::map<std::string, std::vector<std::string>> opts;
  std::set<std::string> flags;
  bool has(const std::string& k) const { return opts.count(k) || flags.count(k); }
  std::string get(const std::string& k, const std::string& def = "") const {
    auto it = opts.find(k);
    return it == opts.end() ? def : it->second.back();
  }
};

Args parse_args(int argc, char** argv, int start, const std::set<std::string>& valued,
                const std::set<std::string>& boolean) {
  Args a;
  for (int i = start; i < argc; ++i) {
    std::string tok = argv[i];
    if (tok == "-o") tok = "--output";
    std::string val;
    bool has_val = false;
    if (auto eq = tok.find('='); tok.rfind("--", 0) == 0 && eq != std::string::npos) {
      val = tok.substr(eq + 1);
      tok = tok.substr(0, eq);
      has_val = true;
    }
    if (boolean.count(tok)) {
      a.flags.insert(tok);
    } else if (valued.count(tok)) {
      if (!has_val) {
        if (i + 1 >= argc) throw UsageError(tok + " requires an argument");
        val = argv[++i];
      }
      a.opts[tok].push_back(val);
    } else {
      throw UsageError("The following argument was not expected: " + tok);
    }
  }
  return a;
}

u64 to_u64(const std::string& s, const char* what) {
  try {
    size_t p = 0;
    const u64 v = std::stoull(s, &p);
    if (p != s.size()) throw std::invalid_argument(s);
    return v;
  } catch (...) {
    throw UsageError(std::string(what) + ": Value " + s + " could not be converted");
  }
}
double to_double(const std::string& s, const char* what) {
  try {
    size_t p = 0;
    const double v = std::stod(s, &p);
    if (p != s.size()) throw std::invalid_argument(s);
    return v;
  } catch (...) {
    throw UsageError(std::string(what) + ": Value " + s + " could not be converted");
  }
}

// tools/synchro.cpp:31-54
Automaton load_automaton(const Args& a) {
  const bool in = a.has("--input"), gen = a.has("--gen");
  if (in && gen) throw UsageError("--input excludes --gen");
  if (!in && !gen) throw UsageError("one of --input or --gen is required");
  if (gen) {
    const std::string spec = a.get("--gen");
    const auto colon = spec.find(':');
    const std::string kind = spec.substr(0, colon);
    const std::string args = colon == std::string::npos ? "" : spec.substr(colon + 1);
    if (kind == "cerny") return cerny_automaton(static_cast<u32>(std::stoul(args)));
    if (kind == "random") {
      std::istringstream ss(args);
      std::string part;
      std::vector<u64> v;
      while (std::getline(ss, part, ',')) v.push_back(std::stoull(part));
      if (v.size() != 3) throw ParseError("random generator needs N,K,SEED");
      return random_automaton(static_cast<u32>(v[0]), static_cast<u32>(v[1]), v[2]);
    }
    throw ParseError("unknown generator: " + kind);
  }
  const std::string file = a.get("--input");
  if (file == "-") return parse_automaton(std::cin);
  std::ifstream f(file);
  if (!f) throw ParseError("cannot open " + file);
  return parse_automaton(f);
}

const std::set<std::string> kSource = {"--input", "--gen"};
const std::set<std::string> kTuning = {"--set-cost", "--min-brute", "--min-leaf", "--dfs-weights",
                                       "--reduce-cadence"};

// tools/synchro.cpp:83-99
void apply_tuning(const Args& a, EngineTuning& t) {
  if (a.has("--set-cost")) t.cost.set_cost = to_double(a.get("--set-cost"), "--set-cost");
  if (a.has("--min-brute")) t.min_brute = to_u64(a.get("--min-brute"), "--min-brute");
  if (a.has("--min-leaf")) t.min_leaf = static_cast<u32>(to_u64(a.get("--min-leaf"), "--min-leaf"));
  if (a.has("--dfs-weights")) {
    std::istringstream ss(a.get("--dfs-weights"));
    char comma;
    if (!(ss >> t.cost.dfs_set_cost_weight >> comma >> t.cost.dfs_check_cost_weight))
      throw ParseError("--dfs-weights expects SET,CHECK");
  }
  if (a.has("--reduce-cadence")) {
    std::istringstream ss(a.get("--reduce-cadence"));
    char comma;
    if (!(ss >> t.dfs_dedupe_cadence >> comma >> t.dfs_reduce_cadence))
      throw ParseError("--reduce-cadence expects DEDUPE,MARK");
  }
}

std::string word_to_string(const Word& w) {
  std::ostringstream os;
  for (size_t i = 0; i < w.size(); ++i) os << (i ? " " : "") << w[i];
  return os.str();
}

std::set<std::string> join(std::set<std::string> a, const std::set<std::string>& b) {
  a.insert(b.begin(), b.end());
  return a;
}

int cmd_exact(int argc, char** argv) {
  const Args a = parse_args(argc, argv, 2,
                            join(join(kSource, kTuning), {"--memory", "--time-limit", "--threads",
                                                          "--schedule", "--trace", "--device",
                                                          "--dfs-shard"}),
                            {"--track-word", "--relaxed-dfs-order"});
  SolveOptions opt;
  if (a.has("--memory")) opt.memory = to_u64(a.get("--memory"), "--memory");
  const double tl = a.has("--time-limit") ? to_double(a.get("--time-limit"), "--time-limit") : 0.0;
  if (tl > 0) opt.time_limit = tl;
  opt.track_word = a.has("--track-word");
  // DFS slices of the unsorted level instead of the reference's exact order:
  // same threshold, different DFS level sizes, no host-side order replay.
  opt.dfs_reference_order = !a.has("--relaxed-dfs-order");
  const std::string sched = a.get("--schedule", "auto");
  if (sched == "bfs") opt.schedule = Schedule::BfsOnly;
  else if (sched == "ibfs") opt.schedule = Schedule::IbfsOnly;
  else if (sched == "dfs") opt.schedule = Schedule::DfsImmediate;
  else if (sched != "auto") throw UsageError("--schedule: " + sched + " not in {auto,bfs,ibfs,dfs}");
  if (a.has("--device")) opt.device = static_cast<int>(to_u64(a.get("--device"), "--device"));
  if (a.has("--dfs-shard")) {  // I/N: explore only the I-th of N shares of the DFS (multi-GPU)
    const std::string v = a.get("--dfs-shard");
    const auto slash = v.find('/');
    if (slash == std::string::npos) throw UsageError("--dfs-shard expects I/N");
    opt.dfs_shard_index = static_cast<u32>(to_u64(v.substr(0, slash), "--dfs-shard"));
    opt.dfs_shard_count = static_cast<u32>(to_u64(v.substr(slash + 1), "--dfs-shard"));
    if (opt.dfs_shard_count == 0 || opt.dfs_shard_index >= opt.dfs_shard_count)
      throw UsageError("--dfs-shard expects I/N with I < N");
  }
  if (a.has("--threads")) to_u64(a.get("--threads"), "--threads");  // accepted, as in the reference
  const Automaton aut = load_automaton(a);
  apply_tuning(a, opt.tuning);
  std::ofstream trace;
  if (a.has("--trace")) {
    trace.open(a.get("--trace"));
    opt.trace = &trace;
  }
  const auto start = std::chrono::steady_clock::now();
  const SolveResult res = solve_exact(aut, opt);
  const std::chrono::duration<double> elapsed = std::chrono::steady_clock::now() - start;
  std::cout << "threshold " << res.threshold << '\n';
  if (res.word) {
    if (!is_reset_word(aut, *res.word)) throw std::logic_error("invalid word");
    std::cout << "word " << word_to_string(*res.word) << '\n';
  }
  std::cerr << "time_s=" << elapsed.count() << " peak_mem_bytes=" << res.peak_memory
            << " upper_bound=" << res.upper_bound << " iterations=" << res.iterations
            << " bfs_steps=" << res.bfs_steps << " ibfs_steps=" << res.ibfs_steps
            << " dfs=" << (res.used_dfs ? 1 : 0) << '\n';
  return 0;
}

int cmd_heuristic(int argc, char** argv) {
  const Args a = parse_args(argc, argv, 2,
                            join(kSource, {"--algorithm", "--beam-size", "--memory", "--time-limit"}),
                            {});
  const std::string alg = a.get("--algorithm", "adaptive");
  if (alg != "eppstein" && alg != "beam" && alg != "adaptive")
    throw UsageError("--algorithm: " + alg + " not in {eppstein,beam,adaptive}");
  const u64 beam_size = a.has("--beam-size") ? to_u64(a.get("--beam-size"), "--beam-size") : 0;
  const u64 memory = a.has("--memory") ? to_u64(a.get("--memory"), "--memory") : (u64{4} << 30);
  const double tl = a.has("--time-limit") ? to_double(a.get("--time-limit"), "--time-limit") : 0.0;
  const Automaton aut = load_automaton(a);
  if (!is_synchronizing(aut)) throw NotSynchronizingError();
  const Deadline dl = tl > 0 ? Deadline::after_seconds(tl) : Deadline();
  HeuristicResult res;
  if (alg == "eppstein") {
    res = eppstein(aut, dl);
  } else if (alg == "beam") {
    const u64 beam = beam_size ? beam_size : std::max<u64>(64, aut.state_count());
    auto b = beam_ibfs(aut, beam, dl);
    if (!b) {
      std::cerr << "beam search found no reset word at beam size " << beam << '\n';
      return kExitRefused;
    }
    res = std::move(*b);
  } else {
    AdaptiveOptions ao;
    ao.memory = memory;
    ao.deadline = dl;
    if (aut.state_count() == 1) {
      res = eppstein(aut, dl);
    } else {
      dev::Context ctx(aut);
      res = adaptive_upper_bound(aut, ao, &ctx);
    }
  }
  if (!is_reset_word(aut, res.word)) throw std::logic_error("invalid word");
  std::cout << "bound " << res.length << '\n';
  std::cout << "word " << word_to_string(res.word) << '\n';
  return 0;
}

int cmd_gen(int argc, char** argv) {
  const Args a = parse_args(argc, argv, 2, join(kSource, {"--output"}), {});
  const Automaton aut = load_automaton(a);
  if (!a.has("--output")) {
    write_automaton(std::cout, aut);
  } else {
    std::ofstream out(a.get("--output"));
    if (!out) throw ParseError("cannot open " + a.get("--output"));
    write_automaton(out, aut);
  }
  return 0;
}

int cmd_oracle(int argc, char** argv) {
  const Args a = parse_args(argc, argv, 2, join(kSource, {"--time-limit"}), {});
  const double tl = a.has("--time-limit") ? to_double(a.get("--time-limit"), "--time-limit") : 0.0;
  const Automaton aut = load_automaton(a);
  if (aut.state_count() > kOracleMaxStates) {
    std::cerr << "oracle refuses n > " << kOracleMaxStates << '\n';
    return kExitRefused;
  }
  const Deadline dl = tl > 0 ? Deadline::after_seconds(tl) : Deadline();
  std::cout << "threshold " << power_set_bfs_oracle(aut, dl) << '\n';
  return 0;
}

int cmd_experiment(int argc, char** argv) {
  const Args a = parse_args(
      argc, argv, 2,
      join(kTuning, {"--n", "--n-range", "--k", "--samples", "--seed-base", "--solver", "--beam-size",
                     "--memory", "--time-limit", "--threads", "--output", "--shard-index",
                     "--shard-count", "--devices"}),
      {"--deterministic"});
  ExperimentSpec spec;
  if (a.opts.count("--n"))
    for (const auto& v : a.opts.at("--n")) spec.ns.push_back(static_cast<u32>(to_u64(v, "--n")));
  if (a.has("--n-range")) {
    std::istringstream ss(a.get("--n-range"));
    u32 lo, hi, step;
    char c1, c2;
    if (!(ss >> lo >> c1 >> hi >> c2 >> step) || c1 != ':' || c2 != ':' || step == 0)
      throw ParseError("--n-range expects LO:HI:STEP");
    for (u32 n = lo; n <= hi; n += step) spec.ns.push_back(n);
  }
  if (spec.ns.empty()) throw ParseError("no state counts given (--n or --n-range)");
  spec.k = a.has("--k") ? static_cast<u32>(to_u64(a.get("--k"), "--k")) : 2;
  spec.samples = a.has("--samples") ? static_cast<u32>(to_u64(a.get("--samples"), "--samples")) : 100;
  spec.seed_base = a.has("--seed-base") ? to_u64(a.get("--seed-base"), "--seed-base") : 0;
  spec.solver = a.get("--solver", "exact");
  static const std::set<std::string> kSolvers = {"exact", "oracle", "eppstein", "beam", "adaptive"};
  if (!kSolvers.count(spec.solver)) throw UsageError("--solver: " + spec.solver + " not allowed");
  spec.beam_size = a.has("--beam-size") ? to_u64(a.get("--beam-size"), "--beam-size") : 0;
  const double tl = a.has("--time-limit") ? to_double(a.get("--time-limit"), "--time-limit") : 0.0;
  spec.time_limit = tl > 0 ? std::optional<double>(tl) : std::nullopt;
  spec.memory = a.has("--memory") ? to_u64(a.get("--memory"), "--memory") : (u64{4} << 30);
  spec.threads = a.has("--threads") ? static_cast<u32>(to_u64(a.get("--threads"), "--threads")) : 1;
  spec.deterministic = a.has("--deterministic");
  if (a.has("--shard-index")) spec.shard_index = static_cast<u32>(to_u64(a.get("--shard-index"), "--shard-index"));
  if (a.has("--shard-count")) spec.shard_count = static_cast<u32>(to_u64(a.get("--shard-count"), "--shard-count"));
  if (a.has("--devices")) spec.devices = static_cast<int>(to_u64(a.get("--devices"), "--devices"));
  apply_tuning(a, spec.tuning);
  if (!a.has("--output")) {
    run_experiment(spec, std::cout, &std::cerr);
  } else {
    std::ofstream out(a.get("--output"));
    if (!out) throw ParseError("cannot open " + a.get("--output"));
    run_experiment(spec, out, &std::cerr);
  }
  return 0;
}

int cmd_fit(int argc, char** argv) {
  const Args a = parse_args(argc, argv, 2, {"--input"}, {});
  if (!a.has("--input")) throw UsageError("--input is required");
  std::vector<ExperimentRecord> records;
  const std::string file = a.get("--input");
  if (file == "-") {
    records = parse_csv(std::cin);
  } else {
    std::ifstream in(file);
    if (!in) throw ParseError("cannot open " + file);
    records = parse_csv(in);
  }
  const FitResult r = fit_records(records);
  std::cout << "a " << r.a << '\n' << "c " << r.c << '\n' << "residual " << r.residual << '\n';
  return 0;
}

int usage(std::ostream& os, int code) {
  os << "Reset-threshold computations for synchronizing automata (B200)\n"
        "Usage: synchro SUBCOMMAND [OPTIONS]\n"
        "Subcommands: exact, heuristic, gen, oracle, experiment, fit\n";
  return code;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) return usage(std::cerr, kExitUsage);
  const std::string sub = argv[1];
  if (sub == "-h" || sub == "--help") return usage(std::cout, 0);
  try {
    if (sub == "exact") return cmd_exact(argc, argv);
    if (sub == "heuristic") return cmd_heuristic(argc, argv);
    if (sub == "gen") return cmd_gen(argc, argv);
    if (sub == "oracle") return cmd_oracle(argc, argv);
    if (sub == "experiment") return cmd_experiment(argc, argv);
    if (sub == "fit") return cmd_fit(argc, argv);
    std::cerr << "The following argument was not expected: " << sub << '\n';
    return usage(std::cerr, kExitUsage);
  } catch (const UsageError& e) {
    std::cerr << e.what() << '\n';
    return kExitUsage;
  } catch (const NotSynchronizingError& e) {
    std::cerr << "error: " << e.what() << '\n';
    return kExitNotSynchronizing;
  } catch (const ParseError& e) {
    std::cerr << "error: " << e.what() << '\n';
    return kExitParseError;
  } catch (const OutOfMemoryError& e) {
    std::cerr << "error: " << e.what() << '\n';
    return kExitOutOfMemory;
  } catch (const TimeoutError& e) {
    std::cerr << "error: " << e.what() << '\n';
    return kExitTimeout;
  } catch (const DeviceError& e) {
    std::cerr << "error: " << e.what() << '\n';
    return kExitDevice;
  } catch (const std::invalid_argument& e) {
    std::cerr << "error: " << e.what() << '\n';
    return kExitParseError;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << '\n';
    return 1;
  }
}
