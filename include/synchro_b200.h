/*
 * synchro_b200.h — C-ABI of the B200-native exact reset-threshold search.
 *
 * Drop-in boundary for the reference's C++ API (/root/reference/proj/include/
 * synchro/ headers) and CLI (proj/tools/synchro.cpp).  Plain pointers and sizes
 * only; no CUDA or torch types.  Every entry point returns an int status:
 *
 *   SW_OK                     0
 *   SW_ERR_OTHER              1  std::logic_error etc.         (CLI exit 1)
 *   SW_ERR_NOT_SYNCHRONIZING  2  NotSynchronizingError          (CLI exit 2)
 *   SW_ERR_PARSE              3  ParseError / invalid_argument  (CLI exit 3)
 *   SW_ERR_OUT_OF_MEMORY      4  OutOfMemoryError (ledger)      (CLI exit 4)
 *   SW_ERR_REFUSED            5  oracle n > 20                  (CLI exit 5)
 *   SW_ERR_TIMEOUT            6  TimeoutError                   (CLI exit 6)
 *   SW_ERR_DEVICE            10  CUDA failure / no device (no CPU fallback)
 *
 * and sw_last_error() returns the message of the calling thread's last failure.
 * Automata are (n, k, delta) with delta row-major: delta[q*k + a]
 * (automaton.hpp:20-45).  Set lists are words[count][W] u64 with
 * W = ceil(n/64), MSB-first packing (state 0 = bit 63 of word 0,
 * state_set.hpp:14-19), plus u32 cards and optional u64 tags.
 */
#ifndef SYNCHRO_B200_H_
#define SYNCHRO_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SW_OK 0
#define SW_ERR_OTHER 1
#define SW_ERR_NOT_SYNCHRONIZING 2
#define SW_ERR_PARSE 3
#define SW_ERR_OUT_OF_MEMORY 4
#define SW_ERR_REFUSED 5
#define SW_ERR_TIMEOUT 6
#define SW_ERR_DEVICE 10

/* Schedule (bibfs_engine.hpp:20-25) */
#define SW_SCHEDULE_AUTO 0
#define SW_SCHEDULE_BFS 1
#define SW_SCHEDULE_IBFS 2
#define SW_SCHEDULE_DFS 3

/* StepKind (cost_model.hpp:13) */
#define SW_STEP_BFS 0
#define SW_STEP_BFS_NH 1
#define SW_STEP_IBFS 2
#define SW_STEP_IBFS_NH 3
#define SW_STEP_DFS 4

/* SolveOptions + EngineTuning + TuningParams (bibfs_engine.hpp:27-48,
 * cost_model.hpp:26-36), flattened.  Use sw_default_options(). */
typedef struct sw_solve_options {
  uint64_t memory;          /* ledger budget in bytes (default 4 GiB) */
  double time_limit;        /* seconds, <= 0: none */
  int32_t track_word;       /* reconstruct and return a shortest reset word */
  int32_t schedule;         /* SW_SCHEDULE_* */
  uint64_t upper_bound;     /* 0: run the adaptive heuristic */
  double set_cost;          /* 512 */
  double dfs_set_weight;    /* 0.25 */
  double dfs_check_weight;  /* 0.25 */
  uint32_t min_brute;       /* 64 (performance-only in the reference) */
  uint32_t min_leaf;        /* 10 */
  uint32_t dedupe_cadence;  /* 2 */
  uint32_t reduce_cadence;  /* 3 */
  int32_t device;           /* CUDA device, -1: current */
  int32_t timing;           /* 1: time expansion kernels with CUDA events */
  uint32_t dfs_shard_index; /* multi-GPU DFS partition: this process's share ... */
  uint32_t dfs_shard_count; /* ... of L_IBFS (threshold = MIN over shards); 1 = whole */
  int32_t contain_stats;    /* 1: count containment-traversal node visits / pair tests */
  /* EngineTuning / TuningParams fields beyond the CLI's (bibfs_engine.hpp:27-37,
   * cost_model.hpp:26-36); semantic: they change the schedule, DFS sizes or R. */
  uint64_t dfs_largest;        /* 20000: DFS window (dfs_phase.hpp:18) */
  double history_growth;       /* 2.0: prune a history once it has grown this much */
  uint64_t beam_initial;       /* 0: max(64, n) (heuristics.hpp:144-150) */
  double beam_cost_fraction;   /* 0.05 */
  double reduction_of_reduction; /* <= 0: unset (1/k) */
  uint64_t stop_after_iterations; /* analysis: stop after this many iterations (0: never) */
  int32_t dfs_reference_order; /* 1 (default): DFS slices in the reference's exact order
                                  (per-level sizes identical); 0: (card desc, lex) slices
                                  (same threshold, no host-side order replay) */
  int32_t pad_;
} sw_solve_options;

/* SolveResult (bibfs_engine.hpp:50-59) + expansion counters and timings. */
typedef struct sw_solve_result {
  uint64_t threshold;
  uint64_t upper_bound;
  uint64_t iterations;
  uint64_t bfs_steps;
  uint64_t ibfs_steps;
  uint64_t peak_memory;
  int32_t used_dfs;
  int32_t has_word;
  uint64_t word_len;
  uint64_t expansions_phase1;
  uint64_t expansions_dfs;
  double heuristic_seconds;
  double engine_seconds;
  double expand_kernel_ms;
  uint64_t kernel_launches;
  char phase[16];           /* "meet" | "dfs" | "bound" | "trivial" | "stopped" */
  double engine_device_ms;  /* CUDA-event span of the engine on its stream */
  uint64_t h2d_bytes;       /* host->device bytes copied during the solve */
  uint64_t d2h_bytes;       /* device->host bytes copied during the solve */
  double contain_kernel_ms; /* CUDA-event time of the containment traversal (timing=1) */
  uint64_t contain_bytes;   /* its algorithmic bytes (every key/query row read once) */
  uint64_t contain_visits;  /* node visits of the traversal (contain_stats=1) */
  uint64_t contain_pairs;   /* key-vs-query pair tests of its range scans (contain_stats=1) */
} sw_solve_result;

const char* sw_version(void);
const char* sw_last_error(void);
int sw_device_count(void);
void sw_default_options(sw_solve_options* opt);

/* ---- automata (automaton.hpp:159-219, experiment.hpp:54-56) ---- */
int sw_random_automaton(uint32_t n, uint32_t k, uint64_t seed, uint32_t* delta_out);
int sw_cerny_automaton(uint32_t n, uint32_t* delta_out);
uint64_t sw_instance_seed(uint64_t seed_base, uint32_t n, uint32_t index);
/* Text format "n k" then n rows of k targets; '#' comments.  Pass delta_out =
 * NULL to query n and k first. */
int sw_parse_automaton(const char* text, uint32_t* n, uint32_t* k, uint32_t* delta_out,
                       size_t delta_cap);
int sw_is_synchronizing(uint32_t n, uint32_t k, const uint32_t* delta, int32_t* result);

/* Shortest merging word length of every state pair {p <= q}, at q(q+1)/2 + p
 * (UINT32_MAX: unmergeable) — the pair automaton BFS behind is_synchronizing
 * (automaton.hpp:119-157) and Eppstein's bound (heuristics.hpp:26-79).
 * on_device != 0: the GPU BFS (device/pairs.cu); 0: the host BFS.  `cap` >=
 * n(n+1)/2 entries. */
int sw_pair_distances(uint32_t n, uint32_t k, const uint32_t* delta, int32_t on_device,
                      uint32_t* out, size_t cap);
int sw_is_reset_word(uint32_t n, uint32_t k, const uint32_t* delta, const uint32_t* word,
                     size_t len, int32_t* result);

/* ---- exact search: replaces synchro::solve_exact (bibfs_engine.hpp:467) ----
 * word: caller buffer of word_cap letters (may be NULL); trace_path: file for
 * the per-iteration trace (bibfs_engine.hpp:442-460) or NULL. */
int sw_solve_exact(uint32_t n, uint32_t k, const uint32_t* delta, const sw_solve_options* opt,
                   sw_solve_result* result, uint32_t* word, size_t word_cap,
                   const char* trace_path);
/* Same, plus the DFS level log: one record {r, level, in, generated, kept} per
 * recurse() call in call order (dfs_phase.hpp:82-159), up to dfs_levels_cap
 * records into dfs_levels[5*i..5*i+4]; *dfs_levels_count = records produced
 * (may exceed the cap). */
int sw_solve_exact_ex(uint32_t n, uint32_t k, const uint32_t* delta, const sw_solve_options* opt,
                      sw_solve_result* result, uint32_t* word, size_t word_cap,
                      const char* trace_path, uint64_t* dfs_levels, size_t dfs_levels_cap,
                      size_t* dfs_levels_count);

/* ---- partitioned solve over several GPUs (no reference
 * counterpart: the reference solves on one thread).  One process per GPU;
 * every rank calls sw_solve_exact_dist with the same automaton and options.
 * Subsets are owned by hash (owner = h(set) mod nranks); each level, one
 * all-to-all carries generated subsets to their owners, which deduplicate;
 * containment (self-reduction, history, meet) all-gathers what it needs;
 * the cost model's statistics are all-reduced, so every rank takes the
 * reference's step sequence and prints the same trace; the DFS runs one
 * interleaved share of L_IBFS per rank and the threshold is the MIN.
 * Transport: NCCL on device buffers (nccl_id from sw_nccl_unique_id on one
 * rank, shared by the caller), or host-buffer callbacks (any transport).
 * Callbacks return 0 on success; buffers are host memory:
 *   all_to_allv: send holds send_bytes[r] bytes for rank r, rank by rank;
 *                recv receives recv_bytes[r] bytes from rank r, rank by rank;
 *   all_gather_v: every rank contributes `bytes`; recv holds recv_bytes[r]
 *                from rank r, rank by rank;
 *   all_reduce_u64: in place, op 0 sum, 1 min, 2 max. ---- */
#define SW_COMM_NCCL 1
#define SW_COMM_CALLBACK 2
typedef struct sw_comm {
  int32_t kind;     /* SW_COMM_NCCL | SW_COMM_CALLBACK */
  int32_t rank;
  int32_t nranks;
  int32_t pad;
  uint8_t nccl_id[128];
  void* user;
  int (*all_to_allv)(void* user, const void* send, const uint64_t* send_bytes, void* recv,
                     const uint64_t* recv_bytes);
  int (*all_gather_v)(void* user, const void* send, uint64_t bytes, void* recv,
                      const uint64_t* recv_bytes);
  int (*all_reduce_u64)(void* user, uint64_t* values, uint64_t count, int32_t op);
} sw_comm;
typedef struct sw_comm_handle sw_comm_handle;
int sw_nccl_unique_id(uint8_t* out128);
/* Creates the transport (NCCL: ncclCommInitRank, collective over the ranks). */
int sw_comm_create(const sw_comm* desc, sw_comm_handle** out);
int sw_comm_destroy(sw_comm_handle* h);
/* As sw_solve_exact_ex; result counters are global (all ranks); the word is
 * returned by every rank (reconstructed from all-gathered level tags). */
int sw_solve_exact_dist(uint32_t n, uint32_t k, const uint32_t* delta, const sw_solve_options* opt,
                        sw_comm_handle* comm, sw_solve_result* result, uint32_t* word,
                        size_t word_cap, const char* trace_path, uint64_t* nvlink_bytes);

/* ---- heuristics (heuristics.hpp:26-184) ----
 * algorithm: 0 eppstein, 1 beam, 2 adaptive.  Returns SW_ERR_REFUSED when the
 * beam finds no reset word (CLI exit 5). */
int sw_heuristic(uint32_t n, uint32_t k, const uint32_t* delta, int32_t algorithm,
                 uint64_t beam_size, uint64_t memory, double time_limit, uint64_t* bound,
                 uint32_t* word, size_t word_cap);

/* ---- power-set BFS oracle (oracle.hpp:17), n <= 20 ---- */
int sw_power_set_oracle(uint32_t n, uint32_t k, const uint32_t* delta, double time_limit,
                        uint64_t* threshold);

/* ---- engine handle (replaces detail::BibfsEngine, bibfs_engine.hpp:66-440) ---- */
typedef struct sw_engine sw_engine;
typedef struct sw_engine_stats {
  uint64_t iteration, bound;
  uint64_t lbfs, libfs, hbfs, hibfs;  /* list sizes */
  double d_lbfs, d_libfs;            /* densities */
  uint64_t ledger_used, ledger_peak;
} sw_engine_stats;
int sw_engine_create(uint32_t n, uint32_t k, const uint32_t* delta, const sw_solve_options* opt,
                     uint64_t upper_bound, sw_engine** out);
int sw_engine_destroy(sw_engine* eng);
/* Cost-model choice for iteration r (make_stats + compute_step_costs + select_step). */
int sw_engine_choose(sw_engine* eng, uint64_t r, int32_t* kind);
int sw_engine_step(sw_engine* eng, int32_t kind);      /* SW_STEP_BFS..IBFS_NH */
int sw_engine_meet(sw_engine* eng, int32_t* met);
int sw_engine_dfs(sw_engine* eng, uint64_t r, uint64_t* threshold);
int sw_engine_stats_get(sw_engine* eng, sw_engine_stats* out);

/* ---- data-plane primitives on host buffers (parity tests; set_list.hpp,
 * subset_algebra.hpp, static_trie.hpp).  Each uploads, runs the B200 kernel(s)
 * and downloads. ---- */
/* out_* hold count*k children, child o = i*k + a (bibfs_engine.hpp:345-367). */
int sw_list_expand(uint32_t n, uint32_t k, const uint32_t* delta, const uint64_t* words,
                   size_t count, int32_t inverse, uint64_t* out_words, uint32_t* out_cards);
/* In place; *out_count = surviving count.  tags may be NULL. */
int sw_list_lex_sort_dedupe(uint32_t n, uint64_t* words, uint32_t* cards, uint64_t* tags,
                            size_t count, size_t* out_count);
int sw_list_sort_card_desc_lex(uint32_t n, uint64_t* words, uint32_t* cards, uint64_t* tags,
                               size_t count);
int sw_list_dedupe_sorted(uint32_t n, uint64_t* words, uint32_t* cards, uint64_t* tags,
                          size_t count, size_t* out_count);
/* Set-semantics dedupe (the surviving set of lex_sort_dedupe, set_list.hpp:
 * 259-265, without the sort): one row per distinct value, survivors in
 * unspecified order.  With tags, each survivor carries the tag of the value's
 * first occurrence (the reference's survivor).  In place; tags may be NULL. */
int sw_list_hash_dedupe(uint32_t n, uint64_t* words, uint32_t* cards, uint64_t* tags,
                        size_t count, size_t* out_count);
int sw_list_self_reduce_minimal(uint32_t n, uint64_t* words, uint32_t* cards, size_t count,
                                size_t* out_count);
/* Multi-GPU frontier exchange building blocks (no reference
 * counterpart — the reference is single-threaded per solve).  DEVICE pointers
 * on the current device (e.g. torch CUDA tensors); synchronous.
 * sw_dev_owner_partition regroups `count` rows owner-major by
 * owner = h(row) mod nranks (h restated in tests/test_distributed_cpu.py),
 * writing out_words/out_cards and counts[r] (host) = rows owned by rank r;
 * order inside an owner's segment is unspecified.  nranks in [1, 1024].
 * sw_dev_hash_dedupe: set-semantics dedupe of a device-resident list, compacted
 * in place; *kept = survivors (distributed.py owner_exchange_dedupe). */
int sw_dev_owner_partition(uint32_t n, const uint64_t* d_words, const uint32_t* d_cards,
                           uint64_t count, uint32_t nranks, uint64_t* d_out_words,
                           uint32_t* d_out_cards, uint64_t* counts);
int sw_dev_hash_dedupe(uint32_t n, uint64_t* d_words, uint32_t* d_cards, uint64_t count,
                       uint64_t* kept);
/* keep[j] = 1 iff b[j] is NOT marked.  mode 0: supersets (incl. equal),
 * 1: proper supersets, 2: subsets.  a must be lex-sorted unique for modes 0/1
 * (require_sorted_unique, subset_algebra.hpp:127-130) else SW_ERR_PARSE. */
int sw_list_mark(uint32_t n, const uint64_t* a_words, size_t a_count, const uint64_t* b_words,
                 size_t b_count, int32_t mode, uint8_t* keep);
int sw_list_meet_check(uint32_t n, const uint64_t* a_words, size_t a_count,
                       const uint64_t* b_words, size_t b_count, int32_t* met);
/* Is some a element a subset of some b element, through the trie index
 * (device/trie_query.cu; a in any order, duplicate-free)?  Witness positions. */
int sw_list_trie_exists(uint32_t n, const uint64_t* a_words, size_t a_count,
                        const uint64_t* b_words, size_t b_count, int32_t* met,
                        uint64_t* a_index, uint64_t* b_index);
/* Host-side (no device): the order in which the reference's meet_check
 * (subset_algebra.hpp:201-210) leaves b when it finds no containment:
 * order[p] = original index of the element now at position p.  a must be
 * lex-sorted unique (else SW_ERR_PARSE); min_brute as EngineTuning. */
int sw_meet_check_order(uint32_t n, const uint64_t* a_words, size_t a_count,
                        const uint64_t* b_words, size_t b_count, uint32_t min_brute,
                        uint32_t* order);
/* Node count of the reference StaticTrie over a duplicate-free list. */
/* ---- cost model (cost_model.hpp:67-250), host-side doubles ---- */
double sw_exp_mark(double a_size, double b_size, double a_density, double b_density);
/* stats[18] = {k, r, R, then per side (BFS, IBFS): list_size, list_density,
 * hist_size, hist_density, r_dupl, r_self, r_hist}; flags[7] = {bfs.hist_dropped,
 * bfs.step_feasible, bfs.nh_feasible, ibfs.hist_dropped, ibfs.step_feasible,
 * ibfs.nh_feasible, dfs_feasible}; tuning[4] = {set_cost, dfs_set_weight,
 * dfs_check_weight, reduction_of_reduction (<= 0: 1/k)}.  Writes step[5],
 * pred[5], feasible[5] and the selected StepKind. */
int sw_step_costs(const double* stats, const int32_t* flags, const double* tuning, double* step,
                  double* pred, int32_t* feasible, int32_t* selected);

int sw_trie_node_count(uint32_t n, const uint64_t* words, size_t count, uint32_t min_leaf,
                       uint64_t* nodes);

/* ---- kernel microbenchmarks at HBM scale (bench.py roofline): `count` random
 * sets of ~density*n states generated on the device; avg CUDA-event ms per
 * call of the expansion kernel / of lex sort + dedupe (dup_fraction of the
 * sets are duplicates). ---- */
int sw_bench_expand(uint32_t n, uint32_t k, const uint32_t* delta, uint64_t count, double density,
                    uint64_t seed, int32_t inverse, int32_t iters, double* ms);
int sw_bench_dedupe(uint32_t n, uint64_t count, double density, uint64_t seed, double dup_fraction,
                    int32_t iters, int32_t lex_sort, double* ms, uint64_t* unique_out);

/* ---- experiment runner (experiment.hpp:133-188) → CSV file ---- */
int sw_run_experiment(const uint32_t* ns, size_t ns_count, uint32_t k, uint32_t samples,
                      uint64_t seed_base, const char* solver, double time_limit, uint64_t memory,
                      uint32_t threads, int32_t deterministic, uint32_t shard_index,
                      uint32_t shard_count, const char* csv_path);

#ifdef __cplusplus
}
#endif

#endif /* SYNCHRO_B200_H_ */
