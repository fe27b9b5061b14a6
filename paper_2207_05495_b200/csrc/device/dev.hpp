// Device data plane: HBM-resident set lists and the sm_100a kernels that
// replace the reference's CPU set algebra.  Plain C++ interface (no CUDA
// types leak out); implemented in device/*.cu.
//
// Layout in HBM: a list of N subsets of Q (|Q| = n) is SoA —
//   words[N][W] u64, W = ceil(n/64), MSB-first packing (state 0 = bit 63 of
//   word 0) so unsigned word order == the reference's lex order
//   (state_set.hpp:14-19, set_list.hpp:34-38);
//   cards[N] u32 (cached popcount);
//   tags[N]  u64 (optional) = (parent_index << 16) | letter (bibfs_engine.hpp:362).
#pragma once

#include <cstddef>
#include <cstdint>
#include <memory>
#include <unordered_map>
#include <vector>

#include "../automaton.hpp"
#include "../common.hpp"

namespace synchro::dev {

class Context;

struct ListStats {
  u64 sum_cards = 0;
  u32 min_card = 0;  // n for an empty list (set_list.hpp:182-186)
  u32 max_card = 0;
};

// Owning device list.  Move-only; memory is stream-ordered (cudaMallocAsync)
// on the owning context's stream.
class DList {
 public:
  DList() = default;
  DList(Context* ctx, size_t cap, bool tagged);
  ~DList();
  DList(DList&& o) noexcept { *this = std::move(o); }
  DList& operator=(DList&& o) noexcept;
  DList(const DList&) = delete;
  DList& operator=(const DList&) = delete;

  void reserve(size_t cap);  // keeps contents
  void release();
  size_t size() const { return size_; }
  bool empty() const { return size_ == 0; }
  bool tagged() const { return tagged_; }
  void set_size(size_t s) {
    size_ = s;
    stats_ok_ = false;
  }
  // Card statistics computed as a by-product (small-list compaction), handed
  // to the next stats() call; cleared by anything that changes size or cards.
  void set_known_stats(const ListStats& st) {
    known_stats_ = st;
    stats_ok_ = true;
  }
  bool known_stats(ListStats* st) const {
    if (stats_ok_) *st = known_stats_;
    return stats_ok_;
  }
  void forget_stats() { stats_ok_ = false; }

  u64* words = nullptr;
  u32* cards = nullptr;
  u64* tags = nullptr;

 private:
  Context* ctx_ = nullptr;
  size_t size_ = 0;
  size_t cap_ = 0;
  bool tagged_ = false;
  bool stats_ok_ = false;
  ListStats known_stats_;
  friend class Context;
};

struct Witness {
  size_t a_index = 0;  // position in the A (subset-side) list
  size_t b_index = 0;  // position in the B (superset-side) list
};

// Patricia/radix tree over a lex-sorted unique list (Karras 2012 layout:
// N-1 internal nodes, node i covers a key range, splits at the first bit
// where its keys differ) + per-node minimum cardinality.  Answers "is some
// stored X a subset of query Y" with per-query traversal on the GPU.
class ContainIndex {
 public:
  ContainIndex() = default;
  ~ContainIndex();
  ContainIndex(ContainIndex&&) noexcept;
  ContainIndex& operator=(ContainIndex&&) noexcept;
  void* nodes = nullptr;    // device Node[N-1]
  void* keysig = nullptr;   // per-key filter words (relabelled word 0, OR-fold), 16 B per key
  size_t count = 0;         // keys indexed
  Context* ctx = nullptr;
};

struct Counters {
  u64 kernel_launches = 0;
  u64 expand_launches = 0;
  double expand_ms = 0;      // accumulated CUDA-event time of expansion kernels
  u64 expand_children = 0;   // children produced by those launches
  u64 contain_pair_tests = 0;
  u64 h2d_bytes = 0;
  u64 d2h_bytes = 0;
  u64 syncs = 0;           // host waits on the stream (readbacks included)
  u64 allocs = 0;          // device allocations that reached the memory pool
  double contain_ms = 0;   // CUDA-event time of the traversal kernel (when timed)
  u64 contain_launches = 0;
  u64 contain_bytes = 0;   // algorithmic bytes of those launches
  u64 contain_visits = 0;  // node visits (contain_stats)
  u64 contain_pairs = 0;   // range-scan pair tests (contain_stats)
};

// CUDA-event pair on a context's stream (device-side span of a region).
class StreamTimer {
 public:
  explicit StreamTimer(Context& c);
  ~StreamTimer();
  void start();
  double stop_ms();  // records the end event, waits for it, returns elapsed ms

 private:
  Context& c_;
  void* e0_ = nullptr;
  void* e1_ = nullptr;
};

class Context {
 public:
  Context(const Automaton& aut, int device = -1);
  ~Context();
  // Re-target this context (stream, pool, scratch) to another automaton.
  void bind(const Automaton& aut);
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;

  u32 n() const { return n_; }
  u32 k() const { return k_; }
  u32 W() const { return W_; }
  void* stream() const { return stream_; }
  int device() const { return device_; }

  void* alloc(size_t bytes);
  void free(void* p);
  void sync();
  void memcpy_d2h(void* dst, const void* src, size_t bytes);
  void memcpy_h2d(void* dst, const void* src, size_t bytes);
  void memcpy_d2d(void* dst, const void* src, size_t bytes);  // stream-ordered

  // Transition tables in device memory (uploaded once).
  const void* d_img = nullptr;   // u16[k*n]  delta(q,a) at [a*n+q]
  bool timing = false;           // record CUDA-event time of expansion kernels
  bool contain_stats = false;    // count traversal visits / pair tests (one readback per launch)
  Counters counters;

  // Scratch buffers reused across calls (grown on demand).
  void* scratch(int slot, size_t bytes);

 private:
  u32 n_ = 0, k_ = 0, W_ = 0;
  int device_ = 0;
  void* stream_ = nullptr;
  void* pool_ = nullptr;  // cudaMemPool_t (the device's default pool)
  // Host-side cache of small freed blocks by power-of-two class (256 B ..
  // 4 MB): small solves allocate and free hundreds of lists, and every pool
  // call takes a driver lock the batch runner's threads contend on.  One
  // stream per context, so a block freed here is reusable at once.
  static constexpr int kCacheClasses = 15;
  std::vector<void*> cache_[kCacheClasses];
  std::unordered_map<void*, int> cached_live_;
  size_t cached_bytes_ = 0;
  struct Scratch { void* p = nullptr; size_t bytes = 0; };
  Scratch scratch_[11];  // slots: kernels.cuh
};

// ---- pair automaton (pairs.cu): shortest merging word length of every pair
// {p <= q} at q(q+1)/2 + p, UINT32_MAX when unmergeable (automaton.hpp:119-157)
std::vector<u32> pair_distances(Context& c, const Automaton& aut);

// ---- list construction / transfer
DList upload(Context& c, const u64* words, const u32* cards, const u64* tags, size_t count);
void download(Context& c, const DList& l, u64* words, u32* cards, u64* tags);
DList make_universe(Context& c, bool tagged);          // [Q], tag 0
DList make_singletons(Context& c, bool tagged);        // {q} tagged q, q = 0..n-1
DList copy_list(Context& c, const DList& l, bool tagged);

// ---- expansion (replaces TransitionKernel::image/preimage + compute_layer,
// bibfs_engine.hpp:345-367 and dfs_phase.hpp:93-103): children o = (i-lo)*k+a
// of parents i in [lo,hi), card by popcount, tag (i<<16)|a when out is tagged.
void expand(Context& c, const DList& src, size_t lo, size_t hi, bool inverse, DList& out);

void complement(Context& c, DList& l);                 // set_list.hpp:142-151
ListStats stats(Context& c, const DList& l);

// ---- ordering and deduplication (set_list.hpp:210-265)
void sort_lex(Context& c, DList& l);                   // stable, index tie-break
void sort_card_desc_lex(Context& c, DList& l);         // card desc, lex, index
void sort_card_desc(Context& c, DList& l);             // card desc, stable (no lex order)
size_t dedupe_sorted(Context& c, DList& l);            // returns #removed
size_t lex_sort_dedupe(Context& c, DList& l);          // returns #removed
// Set-semantics dedupe by open-addressing hash (dedupe.cu): one row per
// distinct value, survivors in UNSPECIFIED order (callers are order-free).
// Tagged lists keep the first occurrence's tag (minimum index, the
// reference's survivor).  Returns #removed.
// first_occurrence=false (tagged lists): any occurrence's tag may survive — every
// equal row's tag names a valid parent, so reconstructed words stay valid; one pass.
size_t hash_dedupe(Context& c, DList& l, bool first_occurrence = true);
// Hash ownership (exchange.cu): regroups l owner-major by owner = h(row) mod
// nranks (order inside an owner's segment unspecified); returns the rows per owner.
std::vector<u64> owner_partition(Context& c, DList& l, u32 nranks);

// ---- containment (subset_algebra.hpp:138-231, static_trie.hpp:51-55)
// Radix tree over a lex-sorted unique list (internal building block).
ContainIndex build_index(Context& c, const DList& a);
// Containment index over a duplicate-free A.  A is copied with its states
// relabelled so that the radix tree splits first on the states that prune
// best for the expected queries:
//   FreqDesc — most frequent state of A first (queries sparser than A:
//              meet check, DFS trie query; ~2.5x fewer visits at n=300),
//   FreqAsc  — rarest first (self-reduction; ~1.3x fewer visits),
//   Natural  — identity.
// The relabelling is a bijection, so containment (and every size) is
// unchanged; witness indices are mapped back to A's original positions.
enum class StateOrder { Natural, FreqDesc, FreqAsc };
struct PermIndex {
  PermIndex() = default;
  ~PermIndex();
  PermIndex(PermIndex&&) noexcept;
  PermIndex& operator=(PermIndex&&) noexcept;
  Context* ctx = nullptr;
  size_t count = 0;               // |A|
  u64* keys = nullptr;            // relabelled sorted A, padded rows (card in word W)
  u32* orig = nullptr;            // sorted position -> index in A
  uint16_t* state_pos = nullptr;  // state q -> relabelled position
  ContainIndex tree;              // radix tree over the relabelled sorted keys
};
PermIndex build_perm_index(Context& c, const DList& a, StateOrder order);
// Is some A element a subset of some b element?  (meet_check / trie query)
bool exists_subset(Context& c, const PermIndex& p, const DList& b, Witness* w);
// Removes every b element that is a superset (proper: strict superset) of
// some A element; b keeps its order.  Returns #removed.
size_t remove_supersets(Context& c, const PermIndex& p, DList& b, bool proper);
// keep[j] = 1 iff b[j] is not a (proper) superset of any A element.
std::vector<uint8_t> superset_keep(Context& c, const PermIndex& p, const DList& b, bool proper);
// Superset join on plain sets (the dense / complement-space marking of the
// reference rephrased): removes every y of Y that is a subset (proper: strict
// subset) of some x of X; Y keeps its order.  Returns #removed.  (join.cu)
size_t remove_subsets_of(Context& c, const DList& X, DList& Y, bool proper);
// keep[j] = 1 iff Y[j] is not a (proper) subset of any X element (device array).
void superset_keep_flags(Context& c, const DList& X, const DList& Y, bool proper, uint8_t* keep);
// Keeps the maximal sets of l (== self_reduce_minimal on the complements).
size_t self_reduce_maximal(Context& c, DList& l);
// Self-reduction to the minimal antichain (subset_algebra.hpp:179-197).
size_t self_reduce_minimal(Context& c, DList& l);

// ---- all-pairs containment for small lists (brute.cu): one launch, no index.
// The list paths above switch to it when |A|·|B| <= kBrutePairs.
constexpr double kBrutePairs = 16.0 * 1024 * 1024;
bool brute_fits(size_t na, size_t nb);
// keep[j] = 1 iff no a in A relates to B[j]: super=false: a ⊆ B[j] (proper: ⊊);
// super=true: B[j] ⊆ a (proper: ⊊).  keep is a device array of |B| bytes.
void brute_keep_flags(Context& c, const DList& A, const DList& B, bool super, bool proper,
                      uint8_t* keep);
// Is some a ⊆ some b?  Witness indices are positions in A and B.
bool brute_exists_subset(Context& c, const DList& A, const DList& B, Witness* w);
// remove_supersets against a plain list A: all-pairs when small, else a
// FreqDesc index over A.  Returns #removed.
size_t remove_supersets_of(Context& c, const DList& A, DList& b, bool proper);

// ---- containment over the whole power set (bitmap.cu), n <= kBitmapMaxStates:
// one single-CTA launch per question (shared-memory bitmap of all 2^n sets,
// subset-/superset-OR transform, n lookups per query).
constexpr u32 kBitmapMaxStates = 20;
bool bitmap_fits(const Context& c);
// keep[j] = 1 iff no a in A relates to B[j] (as brute_keep_flags).
void bitmap_keep_flags(Context& c, const DList& A, const DList& B, bool super, bool proper,
                       uint8_t* keep);
// Is some a ⊆ some b?  *b_index = a b with a subset in A.
bool bitmap_exists_subset(Context& c, const DList& A, const DList& B, size_t* b_index);

// ---- list surgery
void keep_card_at_most(Context& c, DList& l, u32 max_card);
void keep_card_at_least(Context& c, DList& l, u32 min_card);  // plain card of complements
void truncate(DList& l, size_t count);
DList slice_copy(Context& c, const DList& l, size_t lo, size_t hi, bool tagged);
// Rows start, start+stride, start+2·stride, ... (2D copies; no kernel).
DList strided_copy(Context& c, const DList& l, size_t start, size_t stride, bool tagged);
// h := h ++ add (untagged): the merge of bibfs_engine.hpp:383-403 as a set
// (every consumer of the histories is order-free; sort.cu).
void merge_sorted(Context& c, DList& h, const DList& add);
// l := rows perm[0], perm[1], ... of l (perm: device array of l.size() indices).
void gather_rows(Context& c, DList& l, const u32* perm);
// tags[i] += add (a partitioned level's parent indices made global).
void add_to_tags(Context& c, DList& l, u64 add);
u64 read_tag(Context& c, const DList& l, size_t i);
std::vector<u64> read_tags(Context& c, const DList& l);

// ---- one beam level in one launch when it fits a CTA's shared memory
// (beam.cu): sort (card desc, lex, index), drop duplicates, keep the first
// `beam`; *top_card = the first survivor's card.  false: too large, untouched.
bool beam_level_small(Context& c, DList& next, size_t beam, u32* top_card);
// Any-size beam level with the same KEPT SET as sort (card desc, lex) + dedupe +
// truncate(beam), in unspecified order (beam.cu): *top_card = max kept card,
// *top_index = the position of Q in `next` when *top_card == n.
void beam_select(Context& c, DList& next, size_t beam, u32* top_card, size_t* top_index);
// The `need` lex-smallest rows of l, in unspecified order (distinct: l has no
// duplicates — enables the single-CTA finish, which dedupes).
void select_lex_smallest(Context& c, DList& l, size_t need, bool distinct);
// First k rows of l in (card desc, lex) order as a multiset (untagged copy, any order).
DList top_card_desc_lex(Context& c, const DList& l, size_t k);
// The whole beam search (from the singletons, at most level_cap levels) in one
// single-CTA launch when the beam fits shared memory.  Found: *word = the reset
// word (first letter first); NotFound: no word within level_cap;
// NotApplicable: too large (or too many levels) — use the per-level path.
enum class BeamRun { Found, NotFound, NotApplicable };
BeamRun beam_full_small(Context& c, size_t beam, u64 level_cap, std::vector<u32>* word);

// ---- static trie shape (static_trie.hpp:85-151) for exact ledger accounting
u64 trie_node_count(Context& c, const DList& l, u32 min_leaf);
// The same construction, recording the internal nodes round by round (root =
// rounds[0][0]; no rounds when the whole list is one leaf): division state,
// min cardinality and the internal children as indices into the next round
// (0xFFFFFFFF: a leaf / absorbed payload).  Returns the node count.
struct TrieShape {
  struct Node {
    u32 div, min_card, zero, one;
  };
  u32 min_leaf = 10;
  std::vector<std::vector<Node>> rounds;
};
u64 trie_shape(Context& c, const DList& l, u32 min_leaf, TrieShape* shape);

// ---- containment queries on the reference's own trie shape (trie_query.cu):
// every internal node splits its keys on the state most of them hold
// (static_trie.hpp:85-151), so a query lacking that state prunes the larger
// side; payloads (an absorbed zero side, a leaf one side) are scanned.
struct TrieNode {  // 32 B: one 256-bit load
  u32 div, minc, zero, one;  // division state, min card, internal children (~0u: none)
  u32 lo, mid, hi;           // key range [lo, hi): zero side [lo, mid), one side [mid, hi);
                             // a side without an internal child is a payload to scan
  u32 child_div;             // division states of the zero | one << 16 child (0xFFFF: none)
};
struct TrieQueryIndex {
  TrieQueryIndex() = default;
  ~TrieQueryIndex();
  TrieQueryIndex(TrieQueryIndex&&) noexcept;
  TrieQueryIndex& operator=(TrieQueryIndex&&) noexcept;
  Context* ctx = nullptr;
  size_t count = 0;         // keys
  u64 node_count = 0;       // internal nodes (root = node 0)
  void* nodes = nullptr;    // TrieNode[node_count]
  u32* order = nullptr;     // key position -> index in the indexed list
  u64* keys = nullptr;      // padded key rows in key order (card in word W)
  void* keysig = nullptr;   // per-key filter words
  uint8_t* state_bit = nullptr;  // state -> filter bit (the 64 most frequent key states), 255: none
  u32 root_div = 0xFFFF;         // the root's division state (0xFFFF: the root is a leaf)
  void* psig = nullptr;          // per node: AND of each payload's key filter words (2 x 16 B)
};
u64 build_trie_nodes(Context& c, const DList& l, u32 min_leaf, TrieQueryIndex* qi);  // internal
TrieQueryIndex build_trie_index(Context& c, const DList& a, u32 leaf_keys);
bool trie_exists_subset(Context& c, const TrieQueryIndex& t, const DList& b, Witness* w);
// keep flags of b (device, |b| bytes): 0 iff b[j] is a (proper) superset of some key.
void trie_superset_flags(Context& c, const TrieQueryIndex& t, const DList& b, bool proper,
                         uint8_t* keep);
// Minimal antichain through the trie index (queries = the keys, in trie order).
size_t trie_self_reduce_minimal(Context& c, DList& l);
// Which containment index the list paths use: the reference's trie shape
// (default) or the relabelled radix tree (SYNCHRO_INDEX=radix, A/B only).
bool use_trie_index();       // existence queries
bool use_trie_for_marks();   // marking (self-reduction, history)
#ifndef SW_TRIE_LEAF
#define SW_TRIE_LEAF 16
#endif
constexpr u32 kTrieLeafKeys = SW_TRIE_LEAF;  // payload size of the query trie (a performance knob)

// ---- microbenchmarks (microbench.cu): avg CUDA-event ms per call on `count`
// device-generated random sets of the given density.
double bench_expand(Context& c, u64 count, double density, u64 seed, bool inverse, int iters);
double bench_dedupe(Context& c, u64 count, double density, u64 seed, double dup_fraction, int iters,
                    u64* unique_out, bool lex_sort);

// Device count / properties.
int device_count();

}  // namespace synchro::dev
