// C-ABI (include/synchro_b200.h): exceptions → status codes, host buffers in
// and out.  Every entry point maps the reference's exception classes onto the
// CLI exit codes (tools/synchro.cpp:325-344).
#include "../../include/synchro_b200.h"

#include <cstring>
#include <fstream>
#include <memory>
#include <sstream>
#include <string>

#include "device/dev.hpp"
#include "comm.hpp"
#include "engine.hpp"
#include "experiment.hpp"
#include "meet_order.hpp"

#define SW_EXPORT extern "C" __attribute__((visibility("default")))

using namespace synchro;

namespace {

thread_local std::string g_last_error;
thread_local synchro::Comm* t_comm = nullptr;  // the communicator of sw_solve_exact_dist

template <class F>
int guarded(F&& f) {
  try {
    f();
    g_last_error.clear();
    return SW_OK;
  } catch (const NotSynchronizingError& e) {
    g_last_error = e.what();
    return SW_ERR_NOT_SYNCHRONIZING;
  } catch (const ParseError& e) {
    g_last_error = e.what();
    return SW_ERR_PARSE;
  } catch (const OutOfMemoryError& e) {
    g_last_error = e.what();
    return SW_ERR_OUT_OF_MEMORY;
  } catch (const TimeoutError& e) {
    g_last_error = e.what();
    return SW_ERR_TIMEOUT;
  } catch (const DeviceError& e) {
    g_last_error = e.what();
    return SW_ERR_DEVICE;
  } catch (const std::invalid_argument& e) {
    g_last_error = e.what();
    return SW_ERR_PARSE;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return SW_ERR_OTHER;
  } catch (...) {
    g_last_error = "unknown error";
    return SW_ERR_OTHER;
  }
}

Automaton make_aut(uint32_t n, uint32_t k, const uint32_t* delta) {
  if (!delta) throw std::invalid_argument("delta is NULL");
  return Automaton(n, k, std::vector<u32>(delta, delta + static_cast<size_t>(n) * k));
}

// A context for list primitives that need no transition table.
Automaton identity_aut(uint32_t n) {
  std::vector<u32> d(n);
  for (u32 q = 0; q < n; ++q) d[q] = q;
  return Automaton(n, 1, std::move(d));
}

SolveOptions to_options(const sw_solve_options* o) {
  sw_solve_options def;
  sw_default_options(&def);
  if (!o) o = &def;
  SolveOptions s;
  s.memory = o->memory;
  if (o->time_limit > 0) s.time_limit = o->time_limit;
  s.track_word = o->track_word != 0;
  switch (o->schedule) {
    case SW_SCHEDULE_AUTO: s.schedule = Schedule::Auto; break;
    case SW_SCHEDULE_BFS: s.schedule = Schedule::BfsOnly; break;
    case SW_SCHEDULE_IBFS: s.schedule = Schedule::IbfsOnly; break;
    case SW_SCHEDULE_DFS: s.schedule = Schedule::DfsImmediate; break;
    default: throw std::invalid_argument("unknown schedule");
  }
  if (o->upper_bound) s.upper_bound = o->upper_bound;
  s.tuning.cost.set_cost = o->set_cost;
  s.tuning.cost.dfs_set_cost_weight = o->dfs_set_weight;
  s.tuning.cost.dfs_check_cost_weight = o->dfs_check_weight;
  s.tuning.min_brute = o->min_brute;
  s.tuning.min_leaf = o->min_leaf;
  s.tuning.dfs_dedupe_cadence = o->dedupe_cadence;
  s.tuning.dfs_reduce_cadence = o->reduce_cadence;
  s.tuning.dfs_largest = o->dfs_largest;
  s.tuning.history_growth = o->history_growth;
  s.tuning.beam_initial = o->beam_initial;
  s.tuning.beam_cost_fraction = o->beam_cost_fraction;
  if (o->reduction_of_reduction > 0) s.tuning.cost.dfs_reduction_of_reduction = o->reduction_of_reduction;
  s.stop_after_iterations = o->stop_after_iterations;
  s.dfs_reference_order = o->dfs_reference_order != 0;
  s.device = o->device;
  s.timing = o->timing != 0;
  s.contain_stats = o->contain_stats != 0;
  s.dfs_shard_count = std::max<uint32_t>(1, o->dfs_shard_count);
  s.dfs_shard_index = o->dfs_shard_index;
  if (s.dfs_shard_index >= s.dfs_shard_count) throw std::invalid_argument("dfs_shard_index >= dfs_shard_count");
  return s;
}

bool sorted_unique(const uint64_t* w, size_t count, u32 W) {
  for (size_t i = 1; i < count; ++i)
    if (!std::lexicographical_compare(w + (i - 1) * W, w + i * W, w + i * W, w + (i + 1) * W))
      return false;
  return true;
}

}  // namespace

struct sw_engine {
  Automaton aut;
  SolveOptions opt;
  std::unique_ptr<dev::Context> ctx;
  std::unique_ptr<detail::GpuBibfs> eng;
};

SW_EXPORT const char* sw_version(void) { return "synchro-b200 0.1 (sm_100a)"; }
SW_EXPORT const char* sw_last_error(void) { return g_last_error.c_str(); }
SW_EXPORT int sw_device_count(void) { return dev::device_count(); }

SW_EXPORT void sw_default_options(sw_solve_options* o) {
  std::memset(o, 0, sizeof(*o));
  o->memory = u64{4} << 30;
  o->schedule = SW_SCHEDULE_AUTO;
  o->set_cost = 512.0;
  o->dfs_set_weight = 0.25;
  o->dfs_check_weight = 0.25;
  o->min_brute = 64;
  o->min_leaf = 10;
  o->dedupe_cadence = 2;
  o->reduce_cadence = 3;
  o->device = -1;
  o->dfs_shard_index = 0;
  o->dfs_shard_count = 1;
  o->dfs_largest = 20000;
  o->history_growth = 2.0;
  o->beam_initial = 0;
  o->beam_cost_fraction = 0.05;
  o->reduction_of_reduction = 0.0;
  o->stop_after_iterations = 0;
  o->dfs_reference_order = 1;
}

SW_EXPORT int sw_random_automaton(uint32_t n, uint32_t k, uint64_t seed, uint32_t* delta_out) {
  return guarded([&] {
    const Automaton a = random_automaton(n, k, seed);
    std::memcpy(delta_out, a.table().data(), a.table().size() * 4);
  });
}

SW_EXPORT int sw_cerny_automaton(uint32_t n, uint32_t* delta_out) {
  return guarded([&] {
    const Automaton a = cerny_automaton(n);
    std::memcpy(delta_out, a.table().data(), a.table().size() * 4);
  });
}

SW_EXPORT uint64_t sw_instance_seed(uint64_t base, uint32_t n, uint32_t index) {
  return instance_seed(base, n, index);
}

SW_EXPORT int sw_parse_automaton(const char* text, uint32_t* n, uint32_t* k, uint32_t* delta_out,
                                 size_t cap) {
  return guarded([&] {
    const Automaton a = parse_automaton(std::string(text ? text : ""));
    *n = a.state_count();
    *k = a.alphabet_size();
    if (delta_out) {
      if (cap < a.table().size()) throw std::invalid_argument("delta buffer too small");
      std::memcpy(delta_out, a.table().data(), a.table().size() * 4);
    }
  });
}

SW_EXPORT int sw_is_synchronizing(uint32_t n, uint32_t k, const uint32_t* delta, int32_t* result) {
  return guarded([&] { *result = is_synchronizing(make_aut(n, k, delta)) ? 1 : 0; });
}

SW_EXPORT int sw_pair_distances(uint32_t n, uint32_t k, const uint32_t* delta, int32_t on_device,
                                uint32_t* out, size_t cap) {
  return guarded([&] {
    const Automaton aut = make_aut(n, k, delta);
    const size_t need = static_cast<size_t>(n) * (n + 1) / 2;
    if (cap < need) throw std::invalid_argument("sw_pair_distances: output too small");
    std::vector<u32> d;
    if (on_device) {
      dev::Context ctx(aut);
      d = dev::pair_distances(ctx, aut);
    } else {
      d = pair_merge_distances(aut, InverseTransitions(aut));
    }
    std::copy(d.begin(), d.end(), out);
  });
}

SW_EXPORT int sw_is_reset_word(uint32_t n, uint32_t k, const uint32_t* delta, const uint32_t* word,
                               size_t len, int32_t* result) {
  return guarded([&] {
    *result = is_reset_word(make_aut(n, k, delta), Word(word, word + len)) ? 1 : 0;
  });
}

SW_EXPORT int sw_solve_exact(uint32_t n, uint32_t k, const uint32_t* delta,
                             const sw_solve_options* o, sw_solve_result* out, uint32_t* word,
                             size_t word_cap, const char* trace_path) {
  return sw_solve_exact_ex(n, k, delta, o, out, word, word_cap, trace_path, nullptr, 0, nullptr);
}

SW_EXPORT int sw_solve_exact_ex(uint32_t n, uint32_t k, const uint32_t* delta,
                                const sw_solve_options* o, sw_solve_result* out, uint32_t* word,
                                size_t word_cap, const char* trace_path, uint64_t* dfs_levels,
                                size_t dfs_levels_cap, size_t* dfs_levels_count) {
  return guarded([&] {
    if (dfs_levels_count) *dfs_levels_count = 0;
    std::memset(out, 0, sizeof(*out));
    const Automaton aut = make_aut(n, k, delta);
    SolveOptions opt = to_options(o);
    opt.comm = t_comm;
    std::ofstream trace;
    if (trace_path && *trace_path) {
      trace.open(trace_path);
      if (!trace) throw ParseError(std::string("cannot open ") + trace_path);
      opt.trace = &trace;
    }
    const SolveResult r = solve_exact(aut, opt);
    out->threshold = r.threshold;
    out->upper_bound = r.upper_bound;
    out->iterations = r.iterations;
    out->bfs_steps = r.bfs_steps;
    out->ibfs_steps = r.ibfs_steps;
    out->peak_memory = r.peak_memory;
    out->used_dfs = r.used_dfs ? 1 : 0;
    out->has_word = r.word ? 1 : 0;
    out->word_len = r.word ? r.word->size() : 0;
    out->expansions_phase1 = r.expansions_phase1;
    out->expansions_dfs = r.expansions_dfs;
    out->heuristic_seconds = r.heuristic_seconds;
    out->engine_seconds = r.engine_seconds;
    out->expand_kernel_ms = r.expand_kernel_ms;
    out->kernel_launches = r.kernel_launches;
    out->contain_kernel_ms = r.contain_kernel_ms;
    out->contain_bytes = r.contain_bytes;
    out->contain_visits = r.contain_visits;
    out->contain_pairs = r.contain_pairs;
    out->engine_device_ms = r.engine_device_ms;
    out->h2d_bytes = r.h2d_bytes;
    out->d2h_bytes = r.d2h_bytes;
    std::strncpy(out->phase, r.phase.c_str(), sizeof(out->phase) - 1);
    if (r.word && word)
      for (size_t i = 0; i < r.word->size() && i < word_cap; ++i) word[i] = (*r.word)[i];
    if (dfs_levels_count) *dfs_levels_count = r.dfs_levels.size();
    if (dfs_levels)
      for (size_t i = 0; i < r.dfs_levels.size() && i < dfs_levels_cap; ++i)
        for (int f = 0; f < 5; ++f) dfs_levels[5 * i + f] = r.dfs_levels[i][f];
  });
}

struct sw_comm_handle {
  std::unique_ptr<Comm> comm;
};

SW_EXPORT int sw_nccl_unique_id(uint8_t* out128) {
  return guarded([&] { nccl_unique_id(out128); });
}

SW_EXPORT int sw_comm_create(const sw_comm* desc, sw_comm_handle** out) {
  return guarded([&] {
    if (!desc || !out) throw std::invalid_argument("sw_comm_create: NULL argument");
    auto h = std::make_unique<sw_comm_handle>();
    h->comm = make_comm(*desc);
    *out = h.release();
  });
}

SW_EXPORT int sw_comm_destroy(sw_comm_handle* h) {
  return guarded([&] { delete h; });
}

SW_EXPORT int sw_solve_exact_dist(uint32_t n, uint32_t k, const uint32_t* delta,
                                  const sw_solve_options* o, sw_comm_handle* comm,
                                  sw_solve_result* out, uint32_t* word, size_t word_cap,
                                  const char* trace_path, uint64_t* nvlink_bytes) {
  if (!comm) {
    g_last_error = "sw_solve_exact_dist: no communicator";
    return SW_ERR_PARSE;
  }
  sw_solve_options opt;
  if (o) opt = *o; else sw_default_options(&opt);
  const u64 before = comm->comm->bytes_sent;
  t_comm = comm->comm.get();
  const int rc = sw_solve_exact_ex(n, k, delta, &opt, out, word, word_cap, trace_path, nullptr, 0,
                                   nullptr);
  t_comm = nullptr;
  if (nvlink_bytes) *nvlink_bytes = comm->comm->bytes_sent - before;
  return rc;
}

SW_EXPORT int sw_heuristic(uint32_t n, uint32_t k, const uint32_t* delta, int32_t algorithm,
                           uint64_t beam_size, uint64_t memory, double time_limit, uint64_t* bound,
                           uint32_t* word, size_t word_cap) {
  int refused = 0;
  const int rc = guarded([&] {
    const Automaton aut = make_aut(n, k, delta);
    if (!is_synchronizing(aut)) throw NotSynchronizingError();
    const Deadline dl = time_limit > 0 ? Deadline::after_seconds(time_limit) : Deadline();
    HeuristicResult res;
    if (algorithm == 0) {
      res = eppstein(aut, dl);
    } else if (algorithm == 1) {
      const u64 beam = beam_size ? beam_size : std::max<u64>(64, n);
      auto b = beam_ibfs(aut, beam, dl);
      if (!b) {
        refused = 1;
        g_last_error = "beam search found no reset word at beam size " + std::to_string(beam);
        return;
      }
      res = std::move(*b);
    } else {
      AdaptiveOptions a;
      a.memory = memory;
      a.deadline = dl;
      if (n == 1) {
        res = eppstein(aut, dl);
      } else {
        dev::Context ctx(aut);
        res = adaptive_upper_bound(aut, a, &ctx);
      }
    }
    if (!is_reset_word(aut, res.word)) throw std::logic_error("invalid word");
    *bound = res.length;
    if (word)
      for (size_t i = 0; i < res.word.size() && i < word_cap; ++i) word[i] = res.word[i];
  });
  if (rc == SW_OK && refused) return SW_ERR_REFUSED;
  return rc;
}

SW_EXPORT int sw_power_set_oracle(uint32_t n, uint32_t k, const uint32_t* delta, double time_limit,
                                  uint64_t* threshold) {
  const Automaton* dummy = nullptr;
  (void)dummy;
  if (n > kOracleMaxStates) {
    g_last_error = "oracle refuses n > 20";
    return SW_ERR_REFUSED;
  }
  return guarded([&] {
    const Deadline dl = time_limit > 0 ? Deadline::after_seconds(time_limit) : Deadline();
    *threshold = power_set_bfs_oracle(make_aut(n, k, delta), dl);
  });
}

// ---------------------------------------------------------------- engine
SW_EXPORT int sw_engine_create(uint32_t n, uint32_t k, const uint32_t* delta,
                               const sw_solve_options* o, uint64_t upper_bound, sw_engine** out) {
  return guarded([&] {
    auto e = std::unique_ptr<sw_engine>(new sw_engine{make_aut(n, k, delta), to_options(o), {}, {}});
    e->opt.trace = nullptr;
    e->ctx = std::make_unique<dev::Context>(e->aut, e->opt.device);
    e->eng = std::make_unique<detail::GpuBibfs>(e->aut, upper_bound, e->opt, *e->ctx);
    *out = e.release();
  });
}

SW_EXPORT int sw_engine_destroy(sw_engine* e) {
  return guarded([&] {
    if (!e) return;
    e->eng.reset();
    e->ctx.reset();
    delete e;
  });
}

SW_EXPORT int sw_engine_choose(sw_engine* e, uint64_t r, int32_t* kind) {
  return guarded([&] {
    e->eng->set_iteration(r);
    const StepCosts sc = compute_step_costs(e->eng->make_stats(), e->opt.tuning.cost);
    *kind = static_cast<int32_t>(select_step(sc));
  });
}

SW_EXPORT int sw_engine_step(sw_engine* e, int32_t kind) {
  return guarded([&] {
    if (kind < 0 || kind > 3) throw std::invalid_argument("not a list step");
    e->eng->perform(static_cast<StepKind>(kind));
  });
}

SW_EXPORT int sw_engine_meet(sw_engine* e, int32_t* met) {
  return guarded([&] { *met = e->eng->meet() ? 1 : 0; });
}

SW_EXPORT int sw_engine_dfs(sw_engine* e, uint64_t r, uint64_t* threshold) {
  return guarded([&] { *threshold = e->eng->run_dfs(r, nullptr, nullptr, nullptr); });
}

SW_EXPORT int sw_engine_stats_get(sw_engine* e, sw_engine_stats* out) {
  return guarded([&] {
    const SearchStats s = e->eng->make_stats();
    out->iteration = e->eng->iteration();
    out->bound = e->eng->bound();
    out->lbfs = static_cast<uint64_t>(s.bfs.list_size);
    out->libfs = static_cast<uint64_t>(s.ibfs.list_size);
    out->hbfs = static_cast<uint64_t>(s.bfs.hist_size);
    out->hibfs = static_cast<uint64_t>(s.ibfs.hist_size);
    out->d_lbfs = s.bfs.list_density;
    out->d_libfs = s.ibfs.list_density;
    out->ledger_used = e->eng->ledger().used();
    out->ledger_peak = e->eng->ledger().peak();
  });
}

// -------------------------------------------------------------- primitives
SW_EXPORT int sw_list_expand(uint32_t n, uint32_t k, const uint32_t* delta, const uint64_t* words,
                             size_t count, int32_t inverse, uint64_t* out_words,
                             uint32_t* out_cards) {
  return guarded([&] {
    const Automaton aut = make_aut(n, k, delta);
    dev::Context c(aut);
    dev::DList src = dev::upload(c, words, nullptr, nullptr, count);
    dev::DList out(&c, count * k, false);
    dev::expand(c, src, 0, count, inverse != 0, out);
    dev::download(c, out, out_words, out_cards, nullptr);
  });
}

namespace {
template <class Op>
int list_op(uint32_t n, uint64_t* words, uint32_t* cards, uint64_t* tags, size_t count,
            size_t* out_count, Op op) {
  return guarded([&] {
    dev::Context c(identity_aut(n));
    dev::DList l = dev::upload(c, words, cards, tags, count);
    op(c, l);
    dev::download(c, l, words, cards, tags);
    if (out_count) *out_count = l.size();
  });
}
}  // namespace

SW_EXPORT int sw_list_lex_sort_dedupe(uint32_t n, uint64_t* words, uint32_t* cards, uint64_t* tags,
                                      size_t count, size_t* out_count) {
  return list_op(n, words, cards, tags, count, out_count,
                 [](dev::Context& c, dev::DList& l) { dev::lex_sort_dedupe(c, l); });
}

SW_EXPORT int sw_list_sort_card_desc_lex(uint32_t n, uint64_t* words, uint32_t* cards,
                                         uint64_t* tags, size_t count) {
  return list_op(n, words, cards, tags, count, nullptr,
                 [](dev::Context& c, dev::DList& l) { dev::sort_card_desc_lex(c, l); });
}

SW_EXPORT int sw_list_dedupe_sorted(uint32_t n, uint64_t* words, uint32_t* cards, uint64_t* tags,
                                    size_t count, size_t* out_count) {
  return list_op(n, words, cards, tags, count, out_count,
                 [](dev::Context& c, dev::DList& l) { dev::dedupe_sorted(c, l); });
}

SW_EXPORT int sw_list_hash_dedupe(uint32_t n, uint64_t* words, uint32_t* cards, uint64_t* tags,
                                  size_t count, size_t* out_count) {
  return list_op(n, words, cards, tags, count, out_count,
                 [](dev::Context& c, dev::DList& l) { dev::hash_dedupe(c, l); });
}

namespace {
// Device-resident list in/out (the exchange runs on the caller's tensors).
dev::DList device_in(dev::Context& c, const uint64_t* d_words, const uint32_t* d_cards, uint64_t count) {
  dev::DList l(&c, count, false);
  const size_t W = c.W();
  if (count) {
    c.memcpy_d2d(l.words, d_words, count * W * 8);
    c.memcpy_d2d(l.cards, d_cards, count * 4);
  }
  l.set_size(count);
  return l;
}
void device_out(dev::Context& c, const dev::DList& l, uint64_t* d_words, uint32_t* d_cards) {
  if (l.size()) {
    c.memcpy_d2d(d_words, l.words, l.size() * c.W() * 8);
    c.memcpy_d2d(d_cards, l.cards, l.size() * 4);
  }
  c.sync();
}
}  // namespace

SW_EXPORT int sw_dev_owner_partition(uint32_t n, const uint64_t* d_words, const uint32_t* d_cards,
                                     uint64_t count, uint32_t nranks, uint64_t* d_out_words,
                                     uint32_t* d_out_cards, uint64_t* counts) {
  if (nranks == 0 || nranks > 1024 || !counts) {
    g_last_error = "owner_partition: nranks must be in [1, 1024]";
    return SW_ERR_PARSE;
  }
  return guarded([&] {
    dev::Context c(identity_aut(n));  // the caller's current device
    dev::DList l = device_in(c, d_words, d_cards, count);
    const std::vector<u64> per = dev::owner_partition(c, l, nranks);
    device_out(c, l, d_out_words, d_out_cards);
    for (uint32_t r = 0; r < nranks; ++r) counts[r] = r < per.size() ? per[r] : 0;
  });
}

SW_EXPORT int sw_dev_hash_dedupe(uint32_t n, uint64_t* d_words, uint32_t* d_cards, uint64_t count,
                                 uint64_t* kept) {
  return guarded([&] {
    dev::Context c(identity_aut(n));  // the caller's current device
    dev::DList l = device_in(c, d_words, d_cards, count);
    dev::hash_dedupe(c, l);
    device_out(c, l, d_words, d_cards);
    if (kept) *kept = l.size();
  });
}

SW_EXPORT int sw_list_self_reduce_minimal(uint32_t n, uint64_t* words, uint32_t* cards,
                                          size_t count, size_t* out_count) {
  if (!sorted_unique(words, count, words_for(n))) {
    g_last_error = "self_reduce_minimal: first list must be lex-sorted and unique";
    return SW_ERR_PARSE;
  }
  return list_op(n, words, cards, nullptr, count, out_count,
                 [](dev::Context& c, dev::DList& l) { dev::self_reduce_minimal(c, l); });
}

SW_EXPORT int sw_list_mark(uint32_t n, const uint64_t* a_words, size_t a_count,
                           const uint64_t* b_words, size_t b_count, int32_t mode, uint8_t* keep) {
  if (mode != 2 && !sorted_unique(a_words, a_count, words_for(n))) {
    g_last_error = "mark_supersets: first list must be lex-sorted and unique";
    return SW_ERR_PARSE;
  }
  return guarded([&] {
    dev::Context c(identity_aut(n));
    dev::DList a = dev::upload(c, a_words, nullptr, nullptr, a_count);
    dev::DList b = dev::upload(c, b_words, nullptr, nullptr, b_count);
    if (dev::bitmap_fits(c) && mode != 2) {  // n <= 20: the power-set bitmap
      uint8_t* dkeep = static_cast<uint8_t*>(c.alloc(std::max<size_t>(b_count, 1)));
      if (b_count) dev::bitmap_keep_flags(c, a, b, /*super=*/false, mode == 1, dkeep);
      c.memcpy_d2h(keep, dkeep, b_count);
      c.free(dkeep);
      return;
    }
    if (mode == 2) {  // subsets of some a element: the bucketed superset join
      uint8_t* dkeep = static_cast<uint8_t*>(c.alloc(std::max<size_t>(b_count, 1)));
      dev::superset_keep_flags(c, a, b, /*proper=*/false, dkeep);
      c.memcpy_d2h(keep, dkeep, b_count);
      c.free(dkeep);
      return;
    }
    if (dev::use_trie_for_marks()) {
      const dev::TrieQueryIndex t = dev::build_trie_index(c, a, dev::kTrieLeafKeys);
      uint8_t* dkeep = static_cast<uint8_t*>(c.alloc(std::max<size_t>(b_count, 1)));
      dev::trie_superset_flags(c, t, b, mode == 1, dkeep);
      c.memcpy_d2h(keep, dkeep, b_count);
      c.free(dkeep);
      return;
    }
    const dev::PermIndex ix = dev::build_perm_index(c, a, dev::StateOrder::FreqDesc);
    const std::vector<uint8_t> k = dev::superset_keep(c, ix, b, mode == 1);
    std::memcpy(keep, k.data(), k.size());
  });
}

SW_EXPORT int sw_list_meet_check(uint32_t n, const uint64_t* a_words, size_t a_count,
                                 const uint64_t* b_words, size_t b_count, int32_t* met) {
  if (!sorted_unique(a_words, a_count, words_for(n))) {
    g_last_error = "meet_check: first list must be lex-sorted and unique";
    return SW_ERR_PARSE;
  }
  return guarded([&] {
    dev::Context c(identity_aut(n));
    dev::DList a = dev::upload(c, a_words, nullptr, nullptr, a_count);
    dev::DList b = dev::upload(c, b_words, nullptr, nullptr, b_count);
    if (dev::bitmap_fits(c)) {
      *met = dev::bitmap_exists_subset(c, a, b, nullptr) ? 1 : 0;
      return;
    }
    if (dev::use_trie_index()) {
      const dev::TrieQueryIndex t = dev::build_trie_index(c, a, dev::kTrieLeafKeys);
      *met = dev::trie_exists_subset(c, t, b, nullptr) ? 1 : 0;
      return;
    }
    const dev::PermIndex ix = dev::build_perm_index(c, a, dev::StateOrder::FreqDesc);
    *met = dev::exists_subset(c, ix, b, nullptr) ? 1 : 0;
  });
}

SW_EXPORT int sw_list_trie_exists(uint32_t n, const uint64_t* a_words, size_t a_count,
                                  const uint64_t* b_words, size_t b_count, int32_t* met,
                                  uint64_t* a_index, uint64_t* b_index) {
  return guarded([&] {
    dev::Context c(identity_aut(n));
    dev::DList a = dev::upload(c, a_words, nullptr, nullptr, a_count);
    dev::DList b = dev::upload(c, b_words, nullptr, nullptr, b_count);
    const dev::TrieQueryIndex t = dev::build_trie_index(c, a, dev::kTrieLeafKeys);
    dev::Witness w;
    *met = dev::trie_exists_subset(c, t, b, &w) ? 1 : 0;
    if (a_index) *a_index = *met ? w.a_index : 0;
    if (b_index) *b_index = *met ? w.b_index : 0;
  });
}

SW_EXPORT int sw_meet_check_order(uint32_t n, const uint64_t* a_words, size_t a_count,
                                  const uint64_t* b_words, size_t b_count, uint32_t min_brute,
                                  uint32_t* order) {
  if (!sorted_unique(a_words, a_count, words_for(n))) {
    g_last_error = "meet_check: first list must be lex-sorted and unique";
    return SW_ERR_PARSE;
  }
  return guarded([&] {
    std::vector<u32> ord(b_count);
    for (size_t i = 0; i < b_count; ++i) ord[i] = static_cast<u32>(i);
    detail::replay_meet_check(a_words, a_count, b_words, words_for(n), n, min_brute, ord);
    std::memcpy(order, ord.data(), b_count * 4);
  });
}

SW_EXPORT int sw_bench_expand(uint32_t n, uint32_t k, const uint32_t* delta, uint64_t count,
                              double density, uint64_t seed, int32_t inverse, int32_t iters,
                              double* ms) {
  return guarded([&] {
    const Automaton aut = make_aut(n, k, delta);
    dev::Context c(aut);
    *ms = dev::bench_expand(c, count, density, seed, inverse != 0, std::max(1, iters));
  });
}

SW_EXPORT int sw_bench_dedupe(uint32_t n, uint64_t count, double density, uint64_t seed,
                              double dup_fraction, int32_t iters, int32_t lex_sort, double* ms,
                              uint64_t* unique_out) {
  return guarded([&] {
    dev::Context c(identity_aut(n));
    *ms = dev::bench_dedupe(c, count, density, seed, dup_fraction, std::max(1, iters), unique_out,
                            lex_sort != 0);
  });
}

SW_EXPORT double sw_exp_mark(double as, double bs, double ad, double bd) {
  return exp_mark(as, bs, ad, bd);
}

SW_EXPORT int sw_step_costs(const double* st, const int32_t* fl, const double* tu, double* step,
                            double* pred, int32_t* feasible, int32_t* selected) {
  return guarded([&] {
    SearchStats s;
    s.k = st[0];
    s.r = st[1];
    s.R = st[2];
    SideStats* sides[2] = {&s.bfs, &s.ibfs};
    for (int i = 0; i < 2; ++i) {
      const double* p = st + 3 + 7 * i;
      *sides[i] = SideStats{p[0], p[1], p[2], p[3], p[4], p[5], p[6],
                            fl[3 * i] != 0, fl[3 * i + 1] != 0, fl[3 * i + 2] != 0};
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
    *selected = -1;
    try {
      *selected = static_cast<int32_t>(select_step(c));
    } catch (const OutOfMemoryError&) {
      *selected = -1;
    }
  });
}

SW_EXPORT int sw_trie_node_count(uint32_t n, const uint64_t* words, size_t count, uint32_t min_leaf,
                                 uint64_t* nodes) {
  return guarded([&] {
    dev::Context c(identity_aut(n));
    dev::DList l = dev::upload(c, words, nullptr, nullptr, count);
    *nodes = dev::trie_node_count(c, l, min_leaf);
  });
}

SW_EXPORT int sw_run_experiment(const uint32_t* ns, size_t ns_count, uint32_t k, uint32_t samples,
                                uint64_t seed_base, const char* solver, double time_limit,
                                uint64_t memory, uint32_t threads, int32_t deterministic,
                                uint32_t shard_index, uint32_t shard_count, const char* csv_path) {
  return guarded([&] {
    ExperimentSpec spec;
    spec.ns.assign(ns, ns + ns_count);
    spec.k = k;
    spec.samples = samples;
    spec.seed_base = seed_base;
    spec.solver = solver ? solver : "exact";
    spec.time_limit = time_limit > 0 ? std::optional<double>(time_limit) : std::nullopt;
    spec.memory = memory;
    spec.threads = threads;
    spec.deterministic = deterministic != 0;
    spec.shard_index = shard_index;
    spec.shard_count = shard_count ? shard_count : 1;
    std::ofstream out(csv_path);
    if (!out) throw ParseError(std::string("cannot open ") + csv_path);
    run_experiment(spec, out, nullptr);
  });
}
