// Exact reset threshold: the paper's bidirectional BFS with cost-model step
// selection and the trie-backed inverse DFS, with the frontier lists living
// in HBM and every set operation a B200 kernel.
//
// Public surface mirrors the reference's (bibfs_engine.hpp:20-59, :467):
// Schedule, EngineTuning, SolveOptions, SolveResult, solve_exact().  The
// extra SolveResult fields (expansion counts, timings, phase) are additions.
#pragma once

#include <array>
#include <memory>
#include <optional>
#include <ostream>
#include <string>
#include <vector>

#include "automaton.hpp"
#include "common.hpp"
#include "cost_model.hpp"
#include "heuristics.hpp"

namespace synchro {

class Comm;

namespace dev {
class Context;
class DList;
struct ContainIndex;
struct PermIndex;
struct TrieQueryIndex;
struct Witness;
}  // namespace dev

enum class Schedule { Auto, BfsOnly, IbfsOnly, DfsImmediate };

struct EngineTuning {
  TuningParams cost;
  size_t min_brute = 64;  // performance-only in the reference; unused by the GPU kernels
  u32 min_leaf = 10;      // trie leaf bound: affects the ledger through the trie footprint
  size_t dfs_largest = 20000;
  u32 dfs_dedupe_cadence = 2;
  u32 dfs_reduce_cadence = 3;
  double history_growth = 2.0;
  u64 beam_initial = 0;
  double beam_cost_fraction = 0.05;
};

struct SolveOptions {
  u64 memory = u64{4} << 30;
  std::optional<double> time_limit{};
  bool track_word = false;
  Schedule schedule = Schedule::Auto;
  EngineTuning tuning{};
  std::ostream* trace = nullptr;
  std::optional<u64> upper_bound{};
  int device = -1;      // CUDA device (-1: current)
  bool timing = false;  // CUDA-event timing of the expansion kernels
  // Multi-GPU DFS partitioning (one process per GPU): this solve explores
  // only the DFS subtrees rooted in its interleaved share of L_IBFS (rows
  // i ≡ index mod count); the threshold of the whole search is the MIN over
  // the shards.
  u32 dfs_shard_index = 0;
  u32 dfs_shard_count = 1;
  bool contain_stats = false;  // count traversal node visits / pair tests (analysis)
  // Analysis / prefix-parity hook: stop before iteration stop_after_iterations+1
  // (phase "stopped", threshold 0).  0 = run to the end.
  u64 stop_after_iterations = 0;
  // DFS slices cut in the reference's exact order (the order meet_check and
  // the trie queries leave the lists in, meet_order.cpp): per-level sizes
  // bit-identical to the reference's.  false: slices of the (card desc, lex)
  // order — the same threshold (every in-slice reduction keeps a dominating
  // set), different DFS level sizes, no host replay.
  bool dfs_reference_order = true;
  // Partitioned solve over several GPUs (comm.hpp; not owned).  nullptr: one GPU.
  Comm* comm = nullptr;
};

struct SolveResult {
  u64 threshold = 0;
  std::optional<Word> word;
  u64 upper_bound = 0;
  u64 iterations = 0;
  u64 bfs_steps = 0;
  u64 ibfs_steps = 0;
  bool used_dfs = false;
  u64 peak_memory = 0;
  // additions
  u64 expansions_phase1 = 0;  // sum of k*|L| over list steps
  u64 expansions_dfs = 0;     // sum of k*|slice| over DFS levels
  double heuristic_seconds = 0;
  double engine_seconds = 0;
  double expand_kernel_ms = 0;  // CUDA-event time of expansion kernels (when timed)
  u64 kernel_launches = 0;
  double contain_kernel_ms = 0;  // CUDA-event time of the containment traversal (when timed)
  u64 contain_bytes = 0;         // its algorithmic bytes (keys + queries read once)
  u64 contain_visits = 0;        // traversal node visits (contain_stats)
  u64 contain_pairs = 0;         // range-scan pair tests (contain_stats)
  double engine_device_ms = 0;  // CUDA-event span of the engine on its stream
  u64 h2d_bytes = 0, d2h_bytes = 0;
  std::string phase;            // meet | dfs | bound | trivial | stopped
  std::vector<std::array<u64, 5>> dfs_levels;  // r, level, in, generated, kept
};

struct DfsFind {
  bool found = false;
  size_t trie_index = 0;
  size_t root_index = 0;
  Word middle;
};

namespace detail {

// Host control plane of one bidirectional search; the four lists are device
// resident.  Method set parallels the reference's detail::BibfsEngine.
class GpuBibfs {
 public:
  GpuBibfs(const Automaton& aut, u64 upper_bound, const SolveOptions& opt, dev::Context& ctx);
  ~GpuBibfs();

  SearchStats make_stats() const;
  void perform(StepKind kind);
  bool meet();
  bool meet_witness(size_t* bfs_index, u64* ibfs_tag);
  // Reorders L_IBFS as the reference's in-place meet checks left it
  // (meet_order.hpp); only needed when the DFS slices L_IBFS.
  void replay_meet_order();
  u64 run_dfs(u64 r, DfsFind* find, std::vector<std::array<u64, 5>>* log, u64* expansions);

  void set_iteration(u64 r) { r_ = r; }
  u64 iteration() const { return r_; }
  void clear_failures() { failed_ = {false, false, false, false}; }
  void mark_failed(StepKind kind) { failed_[static_cast<size_t>(kind)] = true; }
  MemoryLedger& ledger() { return ledger_; }
  const Deadline& deadline() const { return deadline_; }
  u64 bound() const { return R_; }
  size_t bfs_size() const;
  size_t ibfs_size() const;

  Word bfs_prefix(size_t index) const;
  Word ibfs_suffix_from_tag(u64 tag) const;
  Word ibfs_suffix_from_index(size_t index) const;

 private:
  struct Info {
    size_t size = 0;
    u64 sum_cards = 0;
    u32 min_card = 0, max_card = 0;
  };
  void bfs_step(bool with_history);
  void ibfs_step(bool with_history);
  void drop_bfs_history();
  void drop_ibfs_history();
  void refresh(const dev::DList& l, Info& info);
  // partitioned solve (opt_.comm): see engine.cpp
  bool dist() const { return opt_.comm != nullptr; }
  void refresh_part(const dev::DList& l, Info& info);
  u64 allsum(u64 v);
  void exchange(dev::DList& l);
  dev::DList gather(const dev::DList& l, bool tags);
  u64 rank_offset(const dev::DList& l);
  std::vector<u64> level_tags(const dev::DList& l);
  double density(const Info& i) const;
  void charge_layer(size_t parents);
  void shrink_charge(size_t now_size);
  void merge_history(dev::DList& h, Info& hi, const dev::DList& add);
  const dev::PermIndex& bfs_index();
  const dev::TrieQueryIndex& bfs_trie();
  bool exists_in_bfs(const dev::DList& b, dev::Witness* w);

  const Automaton& aut_;
  const SolveOptions& opt_;
  dev::Context& ctx_;
  MemoryLedger ledger_;
  Deadline deadline_;
  u32 n_, k_;
  u64 R_;
  u64 r_ = 0;
  std::unique_ptr<dev::DList> lbfs_, libfs_, hbfs_, hibfs_c_;
  std::unique_ptr<dev::PermIndex> lbfs_index_;
  std::unique_ptr<dev::TrieQueryIndex> lbfs_trie_;
  Info lbfs_i_, libfs_i_, hbfs_i_, hibfs_i_;
  size_t h_bfs_last_reduced_ = 1, h_ibfs_last_reduced_ = 1;
  bool bfs_hist_dropped_ = false, ibfs_hist_dropped_ = false;
  std::array<double, 3> ratio_bfs_{0, 0, 0}, ratio_ibfs_{0, 0, 0};
  std::array<bool, 4> failed_{false, false, false, false};
  u64 charged_layer_ = 0;
  // Parent records (tags) of every BFS / IBFS level for word reconstruction
  // (bibfs_engine.hpp:301-328): kept on the device and read one entry per level
  // while walking back (a solve used to download every level's tags — 30 MB
  // per n=300 solve); the partitioned solve gathers them on the host.
  struct LevelTags {
    dev::Context* ctx = nullptr;
    u64* dev = nullptr;
    std::vector<u64> host;
    LevelTags() = default;
    LevelTags(const LevelTags&) = delete;
    LevelTags& operator=(const LevelTags&) = delete;
    LevelTags(LevelTags&& o) noexcept : ctx(o.ctx), dev(o.dev), host(std::move(o.host)) { o.dev = nullptr; }
    ~LevelTags();
    u64 at(size_t i) const;
  };
  LevelTags level_tags_of(const dev::DList& l);
  std::vector<LevelTags> bfs_levels_, ibfs_levels_;
  // L_BFS lists met (meet_check, no tracking) since L_IBFS was last committed,
  // oldest first; lbfs_met_: the current L_BFS has been met too.
  std::vector<std::unique_ptr<dev::DList>> met_lists_;
  bool lbfs_met_ = false;
};

void trace_line(std::ostream* trace, const GpuBibfs& eng, const SearchStats& s, const StepCosts& c,
                StepKind kind);

}  // namespace detail

// solve_exact computes the pair-merge distances on the device from this many
// states on (dev::pair_distances), on the host below.
inline constexpr u32 kPairBfsDeviceMin = 128;

SolveResult solve_exact(const Automaton& aut, const SolveOptions& opt = {});
// Same, on a caller-owned device context (re-bound to `aut`): a batch worker
// keeps one context — stream, memory pool, scratch — across its solves.
SolveResult solve_exact(const Automaton& aut, const SolveOptions& opt, dev::Context* ctx);

}  // namespace synchro
