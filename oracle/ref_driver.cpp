// oracle/ref_driver.cpp — TEST INFRASTRUCTURE ONLY (never on the product path).
//
// C-ABI harness over the UNMODIFIED reference headers
// (/root/reference/proj/include/synchro/*.hpp), compiled by oracle/Makefile into
// oracle/_ref/libsynchro_ref.so and linked into oracle/_ref/synchro_ref.
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
// reference leg may load it.  It exposes:
//   * the reference's own solve_exact / heuristics / oracle / primitives, and
//   * ref_solve_instrumented(): a replay of solve_exact's outer loop
//     (bibfs_engine.hpp:467-588) over the public detail::BibfsEngine, with the
//     DFS phase (dfs_phase.hpp:47-177) re-driven from the reference's public
//     primitives so that per-level DFS sizes and the engine expansion count
//      can be logged.  A CPU test checks that this replay
//     reproduces synchro::solve_exact (threshold, peak, iterations, trace).
#include <chrono>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "synchro/synchro.hpp"

#define REF_API extern "C" __attribute__((visibility("default")))

using namespace synchro;

namespace {

Automaton make_aut(uint32_t n, uint32_t k, const uint32_t* delta) {
  return Automaton(n, k, std::vector<u32>(delta, delta + static_cast<size_t>(n) * k));
}

SetList list_from(uint32_t n, const uint64_t* words, const uint32_t* cards, const uint64_t* tags,
                  size_t count) {
  SetList l(n, tags != nullptr);
  l.resize(count);
  const u32 w = l.words_per_set();
  for (size_t i = 0; i < count; ++i) {
    std::memcpy(l.mutable_words(i), words + i * w, w * sizeof(u64));
    u32 c = 0;
    for (u32 t = 0; t < w; ++t) c += static_cast<u32>(std::popcount(words[i * w + t]));
    l.set_card(i, cards ? cards[i] : c);
    if (tags) l.set_tag(i, tags[i]);
  }
  return l;
}

void list_to(const SetList& l, uint64_t* words, uint32_t* cards, uint64_t* tags) {
  const u32 w = l.words_per_set();
  for (size_t i = 0; i < l.size(); ++i) {
    if (words) std::memcpy(words + i * w, l.words(i), w * sizeof(u64));
    if (cards) cards[i] = l.card(i);
    if (tags && l.tagged()) tags[i] = l.tag(i);
  }
}

// Analysis aid: when SYNCHRO_DUMP_DIR is set, the instrumented replay writes the
// lists at the DFS handoff and every DFS level as raw u64 words.
void dump_list(const SetList& l, const std::string& name) {
  const char* dir = std::getenv("SYNCHRO_DUMP_DIR");
  if (!dir || !*dir) return;
  std::ofstream f(std::string(dir) + "/" + name + ".u64", std::ios::binary);
  for (size_t i = 0; i < l.size(); ++i)
    f.write(reinterpret_cast<const char*>(l.words(i)), l.words_per_set() * sizeof(u64));
}

}  // namespace

// ---------------------------------------------------------------- automata
REF_API void ref_random_automaton(uint32_t n, uint32_t k, uint64_t seed, uint32_t* delta) {
  const Automaton a = random_automaton(n, k, seed);
  std::memcpy(delta, a.table().data(), a.table().size() * sizeof(u32));
}
REF_API int ref_cerny_automaton(uint32_t n, uint32_t* delta) {
  try {
    const Automaton a = cerny_automaton(n);
    std::memcpy(delta, a.table().data(), a.table().size() * sizeof(u32));
    return 0;
  } catch (...) {
    return -1;
  }
}
REF_API uint64_t ref_instance_seed(uint64_t base, uint32_t n, uint32_t index) {
  return instance_seed(base, n, index);
}
REF_API int ref_is_synchronizing(uint32_t n, uint32_t k, const uint32_t* delta) {
  return is_synchronizing(make_aut(n, k, delta)) ? 1 : 0;
}
// >=0 threshold, -1 not synchronizing, -2 refused (n > 20)
REF_API int64_t ref_power_set_oracle(uint32_t n, uint32_t k, const uint32_t* delta) {
  try {
    return static_cast<int64_t>(power_set_bfs_oracle(make_aut(n, k, delta)));
  } catch (const NotSynchronizingError&) {
    return -1;
  } catch (const std::invalid_argument&) {
    return -2;
  }
}
// The reference's batch runner (experiment.hpp:133-188), CSV to `path`.
REF_API int ref_run_experiment(const uint32_t* ns, size_t ns_count, uint32_t k, uint32_t samples,
                               uint64_t seed_base, const char* solver, double time_limit,
                               uint32_t threads, int deterministic, const char* path) {
  try {
    ExperimentSpec spec;
    spec.ns.assign(ns, ns + ns_count);
    spec.k = k;
    spec.samples = samples;
    spec.seed_base = seed_base;
    spec.solver = solver;
    spec.time_limit = time_limit > 0 ? std::optional<double>(time_limit) : std::nullopt;
    spec.threads = threads;
    spec.deterministic = deterministic != 0;
    std::ofstream out(path);
    run_experiment(spec, out, nullptr);
    return 0;
  } catch (...) {
    return 1;
  }
}

// compute_step_costs + select_step (cost_model.hpp:187-250) on a flattened
// SearchStats; same layout as sw_step_costs in include/synchro_b200.h.
REF_API int ref_step_costs(const double* st, const int32_t* fl, const double* tu, double* step,
                           double* pred, int32_t* feasible, int32_t* selected) {
  SearchStats s;
  s.k = st[0];
  s.r = st[1];
  s.R = st[2];
  SideStats* sides[2] = {&s.bfs, &s.ibfs};
  for (int i = 0; i < 2; ++i) {
    const double* p = st + 3 + 7 * i;
    SideStats& x = *sides[i];
    x.list_size = p[0];
    x.list_density = p[1];
    x.hist_size = p[2];
    x.hist_density = p[3];
    x.r_dupl = p[4];
    x.r_self = p[5];
    x.r_hist = p[6];
    x.hist_dropped = fl[3 * i] != 0;
    x.step_feasible = fl[3 * i + 1] != 0;
    x.nh_feasible = fl[3 * i + 2] != 0;
  }
  s.dfs_feasible = fl[6] != 0;
  TuningParams t;
  t.set_cost = tu[0];
  t.dfs_set_cost_weight = tu[1];
  t.dfs_check_cost_weight = tu[2];
  if (tu[3] > 0) t.dfs_reduction_of_reduction = tu[3];
  const StepCosts c = compute_step_costs(s, t);
  for (int i = 0; i < 5; ++i) {
    step[i] = c.step[i];
    pred[i] = c.pred[i];
    feasible[i] = c.feasible[i] ? 1 : 0;
  }
  try {
    *selected = static_cast<int32_t>(select_step(c));
  } catch (const OutOfMemoryError&) {
    *selected = -1;
  }
  return 0;
}

REF_API double ref_exp_mark(double as, double bs, double ad, double bd) {
  return exp_mark(as, bs, ad, bd);
}
REF_API int ref_is_reset_word(uint32_t n, uint32_t k, const uint32_t* delta, const uint32_t* word,
                              size_t len) {
  return is_reset_word(make_aut(n, k, delta), Word(word, word + len)) ? 1 : 0;
}

// ------------------------------------------------------------- primitives
// Children o = i*k + a of every parent (bibfs_engine.hpp:345-367 layout).
REF_API void ref_expand(uint32_t n, uint32_t k, const uint32_t* delta, const uint64_t* words,
                        size_t count, int inverse, uint64_t* out_words, uint32_t* out_cards) {
  const Automaton aut = make_aut(n, k, delta);
  TransitionKernel kern(aut);
  const u32 w = kern.words_per_set();
  for (size_t i = 0; i < count; ++i)
    for (u32 a = 0; a < k; ++a) {
      u64* dst = out_words + (i * k + a) * w;
      if (inverse)
        kern.preimage(words + i * w, dst, a);
      else
        kern.image(words + i * w, dst, a);
      u32 c = 0;
      for (u32 t = 0; t < w; ++t) c += static_cast<u32>(std::popcount(dst[t]));
      out_cards[i * k + a] = c;
    }
}

REF_API size_t ref_lex_sort_dedupe(uint32_t n, uint64_t* words, uint32_t* cards, uint64_t* tags,
                                   size_t count, double* ratio) {
  SetList l = list_from(n, words, cards, tags, count);
  const double r = lex_sort_dedupe(l);
  if (ratio) *ratio = r;
  list_to(l, words, cards, tags);
  return l.size();
}

REF_API void ref_sort_lex(uint32_t n, uint64_t* words, uint32_t* cards, uint64_t* tags,
                          size_t count) {
  SetList l = list_from(n, words, cards, tags, count);
  sort_lex(l);
  list_to(l, words, cards, tags);
}

REF_API void ref_sort_card_desc_lex(uint32_t n, uint64_t* words, uint32_t* cards, uint64_t* tags,
                                    size_t count) {
  SetList l = list_from(n, words, cards, tags, count);
  sort_card_desc_lex(l);
  list_to(l, words, cards, tags);
}

REF_API size_t ref_dedupe_sorted(uint32_t n, uint64_t* words, uint32_t* cards, uint64_t* tags,
                                 size_t count) {
  SetList l = list_from(n, words, cards, tags, count);
  dedupe_sorted(l);
  list_to(l, words, cards, tags);
  return l.size();
}

// Returns the new size; the list stays lex-sorted (subset_algebra.hpp:179-197).
REF_API size_t ref_self_reduce_minimal(uint32_t n, uint64_t* words, uint32_t* cards, size_t count) {
  SetList l = list_from(n, words, cards, nullptr, count);
  self_reduce_minimal(l);
  list_to(l, words, cards, nullptr);
  return l.size();
}

// Writes keep[j]=1 for unmarked b elements (in the caller's original order).
// mode 0: mark_supersets, 1: mark_proper_supersets, 2: mark_subsets.
REF_API size_t ref_mark(uint32_t n, const uint64_t* a_words, size_t a_count, const uint64_t* b_words,
                        size_t b_count, int mode, uint8_t* keep) {
  SetList a = list_from(n, a_words, nullptr, nullptr, a_count);
  SetList b = list_from(n, b_words, nullptr, nullptr, b_count);
  // Carry original positions through the permutation in the tags.
  SetList bt(n, true);
  for (size_t j = 0; j < b_count; ++j) bt.push_back_view(b.view(j), j);
  size_t m = 0;
  if (mode == 0)
    m = mark_supersets(a, bt);
  else if (mode == 1)
    m = mark_proper_supersets(a, bt);
  else
    m = mark_subsets(a, bt);
  for (size_t j = 0; j < b_count; ++j) keep[bt.tag(j)] = j < m ? 1 : 0;
  return m;
}

REF_API int ref_meet_check(uint32_t n, const uint64_t* a_words, size_t a_count,
                           const uint64_t* b_words, size_t b_count) {
  SetList a = list_from(n, a_words, nullptr, nullptr, a_count);
  SetList b = list_from(n, b_words, nullptr, nullptr, b_count);
  return meet_check(a, b) ? 1 : 0;
}

// The order the reference's meet_check (subset_algebra.hpp:201-210) leaves b
// in: order[p] = original index of the element at position p.  Returns met.
REF_API int ref_meet_check_order(uint32_t n, const uint64_t* a_words, size_t a_count,
                                 const uint64_t* b_words, size_t b_count, uint32_t min_brute,
                                 uint32_t* order) {
  SetList a = list_from(n, a_words, nullptr, nullptr, a_count);
  SetList b = list_from(n, b_words, nullptr, nullptr, b_count);
  SetList bt(n, true);
  for (size_t j = 0; j < b_count; ++j) bt.push_back_view(b.view(j), j);
  const bool met = meet_check(a, bt, {min_brute});
  for (size_t j = 0; j < b_count; ++j) order[j] = static_cast<uint32_t>(bt.tag(j));
  return met ? 1 : 0;
}

// Static trie over a duplicate-free list: node count and ledger footprint
// (static_trie.hpp:26-45); also answers a joint query for `q` if given.
REF_API uint64_t ref_trie_node_count(uint32_t n, const uint64_t* words, size_t count,
                                     uint32_t min_leaf, uint64_t* footprint) {
  SetList l = list_from(n, words, nullptr, nullptr, count);
  StaticTrie t = StaticTrie::build(l, min_leaf);
  if (footprint) *footprint = t.byte_footprint();
  return t.node_count();
}

// --------------------------------------------------------------- heuristics
REF_API uint64_t ref_eppstein(uint32_t n, uint32_t k, const uint32_t* delta, uint32_t* word,
                              size_t cap) {
  const HeuristicResult r = eppstein(make_aut(n, k, delta));
  for (size_t i = 0; i < r.word.size() && i < cap; ++i) word[i] = r.word[i];
  return r.length;
}
// 0 when the beam fails.
REF_API uint64_t ref_beam(uint32_t n, uint32_t k, const uint32_t* delta, uint64_t beam,
                          uint32_t* word, size_t cap) {
  const auto r = beam_ibfs(make_aut(n, k, delta), beam);
  if (!r) return 0;
  for (size_t i = 0; i < r->word.size() && i < cap; ++i) word[i] = r->word[i];
  return r->length;
}
REF_API uint64_t ref_adaptive(uint32_t n, uint32_t k, const uint32_t* delta, uint64_t memory,
                              uint32_t* word, size_t cap) {
  AdaptiveOptions o;
  o.memory = memory;
  const HeuristicResult r = adaptive_upper_bound(make_aut(n, k, delta), o);
  for (size_t i = 0; i < r.word.size() && i < cap; ++i) word[i] = r.word[i];
  return r.length;
}

// -------------------------------------------------------------------- solve
struct RefOptions {
  uint64_t memory;
  double time_limit;    // <= 0: none
  int32_t track_word;
  int32_t schedule;     // 0 auto, 1 bfs, 2 ibfs, 3 dfs
  uint64_t upper_bound; // 0: run the heuristic
  double set_cost;
  double dfs_set_weight;
  double dfs_check_weight;
  uint32_t min_brute;
  uint32_t min_leaf;
  uint32_t dedupe_cadence;
  uint32_t reduce_cadence;
  double max_seconds;   // instrumented replay only: stop between iterations (bounded CPU sample)
  // EngineTuning / TuningParams fields beyond the CLI's (bibfs_engine.hpp:27-37,
  // cost_model.hpp:26-36)
  uint64_t dfs_largest;
  double history_growth;
  uint64_t beam_initial;
  double beam_cost_fraction;
  double reduction_of_reduction;  // <= 0: unset (1/k)
  uint64_t stop_after_iterations; // instrumented replay only: 0 = none
};

struct RefResult {
  int32_t status;  // 0 ok, 2 nonsync, 4 oom, 6 timeout, 1 other, 7 sample budget reached
  int32_t used_dfs;
  uint64_t threshold;
  uint64_t upper_bound;
  uint64_t iterations;
  uint64_t bfs_steps;
  uint64_t ibfs_steps;
  uint64_t peak_memory;
  uint64_t word_len;
  uint64_t expansions_phase1;
  uint64_t expansions_dfs;
  double heuristic_seconds;
  double engine_seconds;
};

namespace {

SolveOptions to_solve_options(const RefOptions& o) {
  SolveOptions s;
  s.memory = o.memory;
  if (o.time_limit > 0) s.time_limit = o.time_limit;
  s.track_word = o.track_word != 0;
  s.schedule = static_cast<Schedule>(o.schedule);
  if (o.upper_bound) s.upper_bound = o.upper_bound;
  s.tuning.cost.set_cost = o.set_cost;
  s.tuning.cost.dfs_set_cost_weight = o.dfs_set_weight;
  s.tuning.cost.dfs_check_cost_weight = o.dfs_check_weight;
  s.tuning.min_brute = o.min_brute;
  s.tuning.min_leaf = o.min_leaf;
  s.tuning.dfs_dedupe_cadence = o.dedupe_cadence;
  s.tuning.dfs_reduce_cadence = o.reduce_cadence;
  s.tuning.dfs_largest = o.dfs_largest;
  s.tuning.history_growth = o.history_growth;
  s.tuning.beam_initial = o.beam_initial;
  s.tuning.beam_cost_fraction = o.beam_cost_fraction;
  if (o.reduction_of_reduction > 0) s.tuning.cost.dfs_reduction_of_reduction = o.reduction_of_reduction;
  return s;
}

int status_of(const std::exception_ptr& e) {
  try {
    std::rethrow_exception(e);
  } catch (const NotSynchronizingError&) {
    return 2;
  } catch (const OutOfMemoryError&) {
    return 4;
  } catch (const TimeoutError&) {
    return 6;
  } catch (...) {
    return 1;
  }
}

// Level log of the re-driven DFS: one record per recurse() call.
struct DfsLogEntry {
  uint64_t r;
  uint32_t level;
  uint64_t in, generated, kept;
};

// Re-drive of DfsPhase (dfs_phase.hpp:47-177) from the reference's public
// primitives, logging sizes; semantics identical by construction.
class LoggedDfs {
 public:
  LoggedDfs(const TransitionKernel& kernel, const StaticTrie& trie, MemoryLedger& ledger,
            const DfsParams& params, Deadline deadline)
      : kernel_(kernel), trie_(trie), ledger_(ledger), params_(params), deadline_(deadline) {}

  u64 run(const SetList& initial, u64 r0, u64 bound) {
    bound_ = bound;
    if (r0 >= bound_ || initial.empty()) return bound_;
    const size_t cap = slice_cap(r0 - 1);
    for (size_t lo = 0; lo < initial.size(); lo += cap) {
      recurse(initial, lo, std::min(initial.size(), lo + cap), r0, 0);
      if (r0 >= bound_) break;
    }
    return bound_;
  }
  std::vector<DfsLogEntry> log;
  u64 expansions = 0;

 private:
  size_t slice_cap(u64 r) const {
    const u64 set_bytes = StateSet::words_for(kernel_.state_count()) * sizeof(u64);
    const u64 levels = bound_ > r ? bound_ - r : 1;
    const u64 denom = (kernel_.alphabet_size() + 1) * levels * set_bytes;
    return static_cast<size_t>(std::max<u64>(ledger_.available() / std::max<u64>(denom, 1), 1));
  }

  void recurse(const SetList& list, size_t lo, size_t hi, u64 r, u32 level) {
    deadline_.check();
    const u32 k = kernel_.alphabet_size();
    const u32 n = kernel_.state_count();
    SetList next(n);
    u64 charged = SetList::byte_footprint(n, (hi - lo) * k);
    ledger_.charge_or_throw(charged);
    struct Guard {
      MemoryLedger& l;
      u64 amount;
      ~Guard() { l.release(amount); }
    } guard{ledger_, charged};
    next.resize((hi - lo) * k);
    for (size_t i = lo; i < hi; ++i)
      for (u32 a = 0; a < k; ++a) {
        const size_t o = (i - lo) * k + a;
        kernel_.preimage(list.words(i), next.mutable_words(o), a);
        u32 c = 0;
        for (u32 t = 0; t < next.words_per_set(); ++t)
          c += static_cast<u32>(std::popcount(next.words(o)[t]));
        next.set_card(o, c);
      }
    expansions += (hi - lo) * k;
    const u64 generated = next.size();
    sort_card_desc_lex(next);
    if (params_.dedupe_cadence && level % params_.dedupe_cadence == 0) dedupe_sorted(next);
    if (params_.reduce_cadence && level % params_.reduce_cadence == 0 &&
        next.size() > params_.largest_window) {
      SetList largest(n);
      for (size_t i = 0; i < params_.largest_window; ++i) largest.push_back_view(next.view(i));
      largest.complement_all();
      lex_sort_dedupe(largest);
      next.complement_all();
      detail::MarkCtx ctx;
      ctx.proper = true;
      ctx.min_brute = params_.min_brute;
      ctx.nbits = n;
      detail::DirectB bs{&next};
      const size_t m = detail::mark_rec(largest, 0, largest.size(), bs, 0, next.size(), 0, ctx);
      next.complement_all();
      next.truncate(m);
      sort_card_desc_lex(next);
    }
    const u64 now = SetList::byte_footprint(n, next.size());
    if (now < charged) {
      ledger_.release(charged - now);
      guard.amount = now;
    }
    log.push_back({r, level, hi - lo, generated, next.size()});
    dump_list(next, "dfs_r" + std::to_string(r) + "_l" + std::to_string(level));
    size_t i = 0;
    while (i < next.size()) {
      const u32 c = next.card(i);
      size_t j = i + 1;
      while (j < next.size() && next.card(j) == c) ++j;
      if (trie_.contains_subset_of_any(next, i, j, c, nullptr)) {
        bound_ = r;
        return;
      }
      i = j;
    }
    if (r >= bound_ - 1) return;
    const size_t cap = slice_cap(r);
    for (size_t plo = 0; plo < next.size(); plo += cap) {
      recurse(next, plo, std::min(next.size(), plo + cap), r + 1, level + 1);
      if (r >= bound_ - 1) return;
    }
  }

  const TransitionKernel& kernel_;
  const StaticTrie& trie_;
  MemoryLedger& ledger_;
  DfsParams params_;
  Deadline deadline_;
  u64 bound_ = 0;
};

}  // namespace

// The reference's own solve_exact (bibfs_engine.hpp:467), trace to a file.
REF_API int ref_solve_exact(uint32_t n, uint32_t k, const uint32_t* delta, const RefOptions* o,
                            RefResult* res, uint32_t* word, size_t word_cap,
                            const char* trace_path) {
  std::memset(res, 0, sizeof(*res));
  try {
    const Automaton aut = make_aut(n, k, delta);
    SolveOptions opt = to_solve_options(*o);
    std::ofstream trace;
    if (trace_path && *trace_path) {
      trace.open(trace_path);
      opt.trace = &trace;
    }
    const auto t0 = std::chrono::steady_clock::now();
    const SolveResult r = solve_exact(aut, opt);
    res->engine_seconds =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    res->threshold = r.threshold;
    res->upper_bound = r.upper_bound;
    res->iterations = r.iterations;
    res->bfs_steps = r.bfs_steps;
    res->ibfs_steps = r.ibfs_steps;
    res->used_dfs = r.used_dfs;
    res->peak_memory = r.peak_memory;
    if (r.word) {
      res->word_len = r.word->size();
      for (size_t i = 0; i < r.word->size() && i < word_cap; ++i) word[i] = (*r.word)[i];
    }
    return 0;
  } catch (...) {
    res->status = status_of(std::current_exception());
    return res->status;
  }
}

// Replay of solve_exact (bibfs_engine.hpp:467-588) over the public engine with
// the logged DFS; writes the trace (same format) and one JSON-ish line per DFS
// recurse() call to levels_path.  Used for golden fixtures and as the bounded
// CPU baseline sample (max_seconds).
REF_API int ref_solve_instrumented(uint32_t n, uint32_t k, const uint32_t* delta,
                                   const RefOptions* o, RefResult* res, const char* trace_path,
                                   const char* levels_path) {
  std::memset(res, 0, sizeof(*res));
  std::ofstream trace, levels;
  if (trace_path && *trace_path) trace.open(trace_path);
  if (levels_path && *levels_path) levels.open(levels_path);
  std::ostream* tr = trace.is_open() ? &trace : nullptr;
  try {
    const Automaton aut = make_aut(n, k, delta);
    SolveOptions opt = to_solve_options(*o);
    // With track_word the reference meets through meet_find on a copy
    // (L_IBFS keeps its committed order); without, meet_check permutes L_IBFS
    // in place (subset_algebra.hpp:201-219) -- the DFS's top-level slices follow
    // that order, so the replay keeps the distinction.
    opt.trace = tr;
    if (!is_synchronizing(aut)) throw NotSynchronizingError();
    if (n == 1) return 0;
    const auto th = std::chrono::steady_clock::now();
    u64 R;
    if (opt.upper_bound) {
      R = *opt.upper_bound;
    } else {
      AdaptiveOptions aopt;
      aopt.memory = opt.memory;
      aopt.initial_beam = opt.tuning.beam_initial;
      aopt.cost_fraction = opt.tuning.beam_cost_fraction;
      aopt.set_cost = opt.tuning.cost.set_cost;
      aopt.deadline = Deadline::from_limit(opt.time_limit);
      R = adaptive_upper_bound(aut, aopt).length;
    }
    const auto te = std::chrono::steady_clock::now();
    res->heuristic_seconds = std::chrono::duration<double>(te - th).count();
    res->upper_bound = R;
    detail::BibfsEngine eng(aut, R, opt);
    const auto done = [&](u64 t) {
      res->threshold = t;
      res->peak_memory = eng.ledger().peak();
      res->engine_seconds =
          std::chrono::duration<double>(std::chrono::steady_clock::now() - te).count();
      return 0;
    };
    for (u64 r = 1; r + 1 <= R; ++r) {
      eng.deadline().check();
      if (o->max_seconds > 0 &&
          std::chrono::duration<double>(std::chrono::steady_clock::now() - te).count() >
              o->max_seconds) {
        done(0);
        res->status = 7;
        return 7;
      }
      if (o->stop_after_iterations && res->iterations >= o->stop_after_iterations) {
        done(0);
        res->status = 7;
        return 7;
      }
      eng.set_iteration(r);
      eng.clear_failures();
      ++res->iterations;
      StepKind kind;
      SearchStats st;
      StepCosts sc;
      while (true) {
        st = eng.make_stats();
        sc = compute_step_costs(st, opt.tuning.cost);
        switch (opt.schedule) {
          case Schedule::Auto: kind = select_step(sc); break;
          case Schedule::BfsOnly:
            kind = sc.feasible[0] ? StepKind::BFS : (sc.feasible[1] ? StepKind::BFS_NH : StepKind::DFS);
            break;
          case Schedule::IbfsOnly:
            kind = sc.feasible[2] ? StepKind::IBFS
                                  : (sc.feasible[3] ? StepKind::IBFS_NH : StepKind::DFS);
            break;
          default: kind = StepKind::DFS; break;
        }
        if (kind == StepKind::DFS) break;
        const u64 parents = (kind == StepKind::BFS || kind == StepKind::BFS_NH)
                                ? eng.l_bfs().size()
                                : eng.l_ibfs().size();
        try {
          eng.perform(kind);
          res->expansions_phase1 += parents * k;
          break;
        } catch (const OutOfMemoryError&) {
          eng.mark_failed(kind);
        }
      }
      if (kind == StepKind::DFS) {
        res->used_dfs = 1;
        if (tr) *tr << "iter=" << r << " step=DFS handoff\n";
        // run_dfs (bibfs_engine.hpp:275-298) with the logged DFS.
        eng.drop_bfs_history();
        eng.drop_ibfs_history();
        u64 threshold = R;
        if (!eng.l_bfs().empty()) {
          dump_list(eng.l_bfs(), "lbfs");
          dump_list(eng.l_ibfs(), "libfs");
          StaticTrie trie = StaticTrie::build(eng.l_bfs(), opt.tuning.min_leaf);
          eng.ledger().charge_or_throw(trie.byte_footprint());
          eng.ledger().release(eng.l_bfs().byte_footprint());
          DfsParams p;
          p.dedupe_cadence = opt.tuning.dfs_dedupe_cadence;
          p.reduce_cadence = opt.tuning.dfs_reduce_cadence;
          p.largest_window = opt.tuning.dfs_largest;
          p.min_brute = opt.tuning.min_brute;
          const TransitionKernel kern(aut);
          LoggedDfs dfs(kern, trie, eng.ledger(), p, eng.deadline());
          threshold = dfs.run(eng.l_ibfs(), r, R);
          eng.ledger().release(trie.byte_footprint());
          res->expansions_dfs = dfs.expansions;
          if (levels.is_open())
            for (const auto& e : dfs.log)
              levels << "{\"r\": " << e.r << ", \"level\": " << e.level << ", \"in\": " << e.in
                     << ", \"generated\": " << e.generated << ", \"kept\": " << e.kept << "}\n";
        }
        if (tr) *tr << "result=" << threshold << " phase=dfs\n";
        return done(threshold);
      }
      if (kind == StepKind::BFS || kind == StepKind::BFS_NH)
        ++res->bfs_steps;
      else
        ++res->ibfs_steps;
      detail::trace_line(tr, eng, st, sc, kind);
      if (opt.track_word ? eng.meet_witness().has_value() : eng.meet()) {
        if (tr) *tr << "result=" << r << " phase=meet\n";
        return done(r);
      }
    }
    if (tr) *tr << "result=" << R << " phase=bound\n";
    return done(R);
  } catch (...) {
    res->status = status_of(std::current_exception());
    return res->status;
  }
}
