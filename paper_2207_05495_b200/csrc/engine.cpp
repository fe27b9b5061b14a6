#include "engine.hpp"

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <functional>
#include <cstdlib>
#include <set>
#include <sstream>

#include "comm.hpp"
#include "device/dev.hpp"
#include "meet_order.hpp"
#include "progress.hpp"

namespace synchro {
namespace detail {

using dev::DList;

constexpr size_t kTrieMinKeys = 1 << 15;  // trie index for existence queries from this |L_BFS| on

// ------------------------------------------------------------------ setup
// L_BFS = [Q], H_BFS = [Q], L_IBFS = singletons tagged q, H_IBFS stored as
// complements of the singletons; all four charged (bibfs_engine.hpp:68-95).
GpuBibfs::GpuBibfs(const Automaton& aut, u64 upper_bound, const SolveOptions& opt,
                   dev::Context& ctx)
    : aut_(aut),
      opt_(opt),
      ctx_(ctx),
      ledger_(opt.memory),
      deadline_(Deadline::from_limit(opt.time_limit)),
      n_(aut.state_count()),
      k_(aut.alphabet_size()),
      R_(upper_bound) {
  const bool lead = !dist() || opt_.comm->rank() == 0;
  // Partitioned solve: rank 0 creates the frontier lists, the exchange hands
  // every set to its owner; the histories are replicated.
  lbfs_ = std::make_unique<DList>(lead ? dev::make_universe(ctx_, opt_.track_word)
                                       : DList(&ctx_, 0, opt_.track_word));
  hbfs_ = std::make_unique<DList>(dev::make_universe(ctx_, false));
  libfs_ = std::make_unique<DList>(lead ? dev::make_singletons(ctx_, opt_.track_word)
                                        : DList(&ctx_, 0, opt_.track_word));
  hibfs_c_ = std::make_unique<DList>(dev::make_singletons(ctx_, false));
  dev::complement(ctx_, *hibfs_c_);
  if (dist()) {
    exchange(*lbfs_);
    exchange(*libfs_);
  }
  refresh_part(*lbfs_, lbfs_i_);
  refresh(*hbfs_, hbfs_i_);
  refresh_part(*libfs_, libfs_i_);
  refresh(*hibfs_c_, hibfs_i_);
  ledger_.charge_or_throw(list_footprint(n_, lbfs_i_.size) + list_footprint(n_, libfs_i_.size) +
                          list_footprint(n_, hbfs_i_.size) + list_footprint(n_, hibfs_i_.size));
  h_bfs_last_reduced_ = hbfs_i_.size;
  h_ibfs_last_reduced_ = hibfs_i_.size;
}

GpuBibfs::~GpuBibfs() = default;

size_t GpuBibfs::bfs_size() const { return lbfs_i_.size; }
size_t GpuBibfs::ibfs_size() const { return libfs_i_.size; }

void GpuBibfs::refresh(const DList& l, Info& info) {
  const dev::ListStats st = dev::stats(ctx_, l);
  info.size = l.size();
  info.sum_cards = st.sum_cards;
  info.min_card = st.min_card;
  info.max_card = st.max_card;
}

// -------------------------------------------------- partitioned solve (comm.hpp)
// Statistics of a partitioned list over all ranks: the cost model, the
// ledger and the trace see the global integers, so every rank takes the
// single-GPU solve's steps.
void GpuBibfs::refresh_part(const DList& l, Info& info) {
  refresh(l, info);
  if (!dist()) return;
  u64 v[2] = {info.size, info.sum_cards};
  opt_.comm->all_reduce(ctx_, v, 2, ReduceOp::Sum);
  u64 mn = info.size ? info.min_card : n_, mx = info.size ? info.max_card : 0;
  opt_.comm->all_reduce(ctx_, &mn, 1, ReduceOp::Min);
  opt_.comm->all_reduce(ctx_, &mx, 1, ReduceOp::Max);
  info.size = v[0];
  info.sum_cards = v[1];
  info.min_card = static_cast<u32>(mn);
  info.max_card = static_cast<u32>(mx);
}

u64 GpuBibfs::allsum(u64 v) {
  if (dist()) opt_.comm->all_reduce(ctx_, &v, 1, ReduceOp::Sum);
  return v;
}

// Hash ownership: every row travels to rank h(row) mod nranks
// (exchange.cu owner_partition + one all-to-all per array).
void GpuBibfs::exchange(DList& l) {
  Comm& cm = *opt_.comm;
  const std::vector<u64> send = dev::owner_partition(ctx_, l, static_cast<u32>(cm.size()));
  const std::vector<u64> recv = cm.all_to_all_counts(ctx_, send);
  u64 total = 0;
  for (u64 r : recv) total += r;
  DList out(&ctx_, total, l.tagged());
  const auto scaled = [](const std::vector<u64>& v, u64 b) {
    std::vector<u64> o(v.size());
    for (size_t i = 0; i < v.size(); ++i) o[i] = v[i] * b;
    return o;
  };
  const u64 row = static_cast<u64>(ctx_.W()) * 8;
  cm.all_to_allv(ctx_, l.words, scaled(send, row), out.words, scaled(recv, row));
  cm.all_to_allv(ctx_, l.cards, scaled(send, 4), out.cards, scaled(recv, 4));
  if (l.tagged()) cm.all_to_allv(ctx_, l.tags, scaled(send, 8), out.tags, scaled(recv, 8));
  out.set_size(total);
  l = std::move(out);
}

// The whole partitioned list on every rank, rank by rank (containment is not
// hash-local: a subset of an owned set may live on any rank).
DList GpuBibfs::gather(const DList& l, bool tags) {
  Comm& cm = *opt_.comm;
  const std::vector<u64> sizes = cm.all_gather_u64(ctx_, l.size());
  u64 total = 0;
  for (u64 x : sizes) total += x;
  const bool tg = tags && l.tagged();
  DList out(&ctx_, total, tg);
  const auto scaled = [&](u64 b) {
    std::vector<u64> o(sizes.size());
    for (size_t i = 0; i < sizes.size(); ++i) o[i] = sizes[i] * b;
    return o;
  };
  const u64 row = static_cast<u64>(ctx_.W()) * 8;
  cm.all_gather_v(ctx_, l.words, l.size() * row, out.words, scaled(row));
  cm.all_gather_v(ctx_, l.cards, l.size() * 4, out.cards, scaled(4));
  if (tg) cm.all_gather_v(ctx_, l.tags, l.size() * 8, out.tags, scaled(8));
  out.set_size(total);
  return out;
}

// Global index of this rank's first row of a partitioned list (rank order).
u64 GpuBibfs::rank_offset(const DList& l) {
  const std::vector<u64> sizes = opt_.comm->all_gather_u64(ctx_, l.size());
  u64 off = 0;
  for (int r = 0; r < opt_.comm->rank(); ++r) off += sizes[r];
  return off;
}

// Level tags in the global (rank-concatenated) order of a partitioned level.
std::vector<u64> GpuBibfs::level_tags(const DList& l) {
  if (!dist()) return dev::read_tags(ctx_, l);
  return dev::read_tags(ctx_, gather(l, true));
}

GpuBibfs::LevelTags GpuBibfs::level_tags_of(const DList& l) {
  LevelTags t;
  if (dist() || !l.tagged()) {
    t.host = level_tags(l);
    return t;
  }
  t.ctx = &ctx_;
  t.dev = static_cast<u64*>(ctx_.alloc(std::max<size_t>(l.size(), 1) * 8));
  ctx_.memcpy_d2d(t.dev, l.tags, l.size() * 8);
  return t;
}

GpuBibfs::LevelTags::~LevelTags() {
  if (ctx && dev) {
    try {
      ctx->free(dev);
    } catch (...) {
    }
  }
}

u64 GpuBibfs::LevelTags::at(size_t i) const {
  if (!dev) return host[i];
  u64 t = 0;
  ctx->memcpy_d2h(&t, dev + i, 8);
  return t;
}

// set_list.hpp:171-174
double GpuBibfs::density(const Info& i) const {
  if (i.size == 0 || n_ == 0) return 0.0;
  return static_cast<double>(i.sum_cards) / (static_cast<double>(n_) * i.size);
}

// ------------------------------------------------------------- statistics
// bibfs_engine.hpp:107-147: identical integers in, identical doubles out.
SearchStats GpuBibfs::make_stats() const {
  SearchStats s;
  s.k = k_;
  s.r = static_cast<double>(r_);
  s.R = static_cast<double>(R_);
  const u64 used = ledger_.used(), budget = ledger_.budget();
  const auto fits = [&](u64 extra, u64 freed) {
    const u64 base = used > freed ? used - freed : 0;
    return extra <= budget && base <= budget - extra;
  };
  s.bfs.list_size = static_cast<double>(lbfs_i_.size);
  s.bfs.list_density = density(lbfs_i_);
  s.bfs.hist_size = static_cast<double>(hbfs_i_.size);
  s.bfs.hist_density = density(hbfs_i_);
  s.bfs.r_dupl = ratio_bfs_[0];
  s.bfs.r_self = ratio_bfs_[1];
  s.bfs.r_hist = ratio_bfs_[2];
  s.bfs.hist_dropped = bfs_hist_dropped_;
  const u64 next_bfs = list_footprint(n_, static_cast<u64>(lbfs_i_.size) * k_);
  s.bfs.step_feasible = !failed_[0] && fits(next_bfs, 0);
  s.bfs.nh_feasible =
      !failed_[1] && fits(next_bfs, bfs_hist_dropped_ ? 0 : list_footprint(n_, hbfs_i_.size));

  s.ibfs.list_size = static_cast<double>(libfs_i_.size);
  s.ibfs.list_density = density(libfs_i_);
  s.ibfs.hist_size = static_cast<double>(hibfs_i_.size);
  s.ibfs.hist_density = hibfs_i_.size == 0 ? 0.0 : 1.0 - density(hibfs_i_);
  s.ibfs.r_dupl = ratio_ibfs_[0];
  s.ibfs.r_self = ratio_ibfs_[1];
  s.ibfs.r_hist = ratio_ibfs_[2];
  s.ibfs.hist_dropped = ibfs_hist_dropped_;
  const u64 next_ibfs = list_footprint(n_, static_cast<u64>(libfs_i_.size) * k_);
  s.ibfs.step_feasible = !failed_[2] && fits(next_ibfs, 0);
  s.ibfs.nh_feasible =
      !failed_[3] && fits(next_ibfs, ibfs_hist_dropped_ ? 0 : list_footprint(n_, hibfs_i_.size));
  s.dfs_feasible = true;
  return s;
}

// ---------------------------------------------------------- ledger pieces
void GpuBibfs::charge_layer(size_t parents) {
  const u64 bytes = list_footprint(n_, static_cast<u64>(parents) * k_);
  ledger_.charge_or_throw(bytes);
  charged_layer_ = bytes;
}

void GpuBibfs::shrink_charge(size_t now_size) {
  const u64 now = list_footprint(n_, now_size);
  if (now < charged_layer_) ledger_.release(charged_layer_ - now);
  charged_layer_ = now;
}

// Disjoint sorted merge; charges the merged list before releasing the old
// one (bibfs_engine.hpp:383-403).
void GpuBibfs::merge_history(DList& h, Info& hi, const DList& add) {
  if (add.empty()) return;
  const u64 before = list_footprint(n_, hi.size);
  ledger_.charge_or_throw(list_footprint(n_, hi.size + add.size()));
  dev::merge_sorted(ctx_, h, add);
  refresh(h, hi);
  ledger_.release(before);
}

void GpuBibfs::drop_bfs_history() {
  if (bfs_hist_dropped_) return;
  ledger_.release(list_footprint(n_, hbfs_i_.size));
  *hbfs_ = DList(&ctx_, 0, false);
  hbfs_i_ = Info{};
  bfs_hist_dropped_ = true;
}

void GpuBibfs::drop_ibfs_history() {
  if (ibfs_hist_dropped_) return;
  ledger_.release(list_footprint(n_, hibfs_i_.size));
  *hibfs_c_ = DList(&ctx_, 0, false);
  hibfs_i_ = Info{};
  ibfs_hist_dropped_ = true;
}

// L_BFS relabelled most-frequent-state-first: the meet check and the DFS
// query are subset queries from sparser sets, where that order prunes best.
const dev::PermIndex& GpuBibfs::bfs_index() {
  if (!lbfs_index_)
    lbfs_index_ = std::make_unique<dev::PermIndex>(
        dev::build_perm_index(ctx_, *lbfs_, dev::StateOrder::FreqDesc));
  return *lbfs_index_;
}

// The reference's own trie shape over L_BFS (static_trie.hpp:26-151) as the
// query structure of the meet check and the DFS (device/trie_query.cu).
const dev::TrieQueryIndex& GpuBibfs::bfs_trie() {
  if (!lbfs_trie_)
    lbfs_trie_ = std::make_unique<dev::TrieQueryIndex>(
        dev::build_trie_index(ctx_, *lbfs_, dev::kTrieLeafKeys));
  return *lbfs_trie_;
}

// Is some L_BFS set a subset of some set of b?  (meet_check / trie query)
bool GpuBibfs::exists_in_bfs(const DList& b, dev::Witness* w) {
  if (dev::bitmap_fits(ctx_)) {  // n <= 20: the power-set bitmap, then the witness's subset
    size_t bi = 0;
    if (!dev::bitmap_exists_subset(ctx_, *lbfs_, b, &bi)) return false;
    if (w) {
      const DList one = dev::slice_copy(ctx_, b, bi, bi + 1, false);
      dev::Witness w1;
      dev::brute_exists_subset(ctx_, *lbfs_, one, &w1);
      w->a_index = w1.a_index;
      w->b_index = bi;
    }
    return true;
  }
  // The trie's level-synchronous build (one round of launches per trie level)
  // only pays off on large lists; small ones take the radix tree.
  if (dev::use_trie_index() && lbfs_->size() >= kTrieMinKeys)
    return dev::trie_exists_subset(ctx_, bfs_trie(), b, w);
  return dev::exists_subset(ctx_, bfs_index(), b, w);
}

namespace {
// Releases the charged layer if a step aborts between expansion and commit
// (bibfs_engine.hpp:334-343).
struct Rollback {
  MemoryLedger& ledger;
  u64& charged;
  bool armed = true;
  ~Rollback() {
    if (armed) {
      ledger.release(charged);
      charged = 0;
    }
  }
};
inline double ratio(size_t part, size_t whole) {
  return whole ? static_cast<double>(part) / static_cast<double>(whole) : 0.0;
}
}  // namespace

// ------------------------------------------------------------ list steps
// Forward step (bibfs_engine.hpp:152-191): [prune H] → expand → sort+dedupe →
// minimal antichain → [drop supersets of H] → commit [→ merge into H].
void GpuBibfs::bfs_step(bool with_history) {
  if (!with_history) drop_bfs_history();
  if (with_history && static_cast<double>(hbfs_i_.size) >=
                          opt_.tuning.history_growth * static_cast<double>(h_bfs_last_reduced_)) {
    const u64 before = list_footprint(n_, hbfs_i_.size);
    dev::keep_card_at_most(ctx_, *hbfs_, lbfs_i_.max_card);
    dev::self_reduce_minimal(ctx_, *hbfs_);
    refresh(*hbfs_, hbfs_i_);
    h_bfs_last_reduced_ = hbfs_i_.size;
    ledger_.release(before - list_footprint(n_, hbfs_i_.size));
  }
  charge_layer(lbfs_i_.size);
  DList next(&ctx_, lbfs_->size() * k_, opt_.track_word);
  dev::expand(ctx_, *lbfs_, 0, lbfs_->size(), /*inverse=*/false, next);
  Rollback rb{ledger_, charged_layer_};
  if (dist()) {  // global parent indices, then every child to its owner
    if (opt_.track_word) dev::add_to_tags(ctx_, next, rank_offset(*lbfs_) << 16);
    exchange(next);
  }
  const size_t generated = lbfs_i_.size * k_;
  // Set-semantics dedupe (hash; same survivors as the reference's stable lex
  // sort + unique).  L_BFS needs no lex order: every consumer either sorts its
  // own relabelled copy (containment index) or is order-free (stats, ledger).
  // Partitioned: equal sets share an owner, so the owner's dedupe is exact.
  const double r_dupl =
      generated ? ratio(allsum(dev::hash_dedupe(ctx_, next, /*first_occurrence=*/false)), generated)
                : 0.0;
  const size_t after_dupl = allsum(next.size());
  size_t removed_self;
  if (dist()) {  // owned sets against the whole deduplicated layer
    const DList layer = gather(next, false);
    removed_self = dev::remove_supersets_of(ctx_, layer, next, /*proper=*/true);
  } else {
    removed_self = dev::self_reduce_minimal(ctx_, next);
  }
  const double r_self = ratio(allsum(removed_self), after_dupl);
  double r_hist = 0.0;
  if (with_history) {  // the history is replicated
    const size_t before = allsum(next.size());
    const size_t removed = dev::remove_supersets_of(ctx_, *hbfs_, next, /*proper=*/false);
    r_hist = ratio(allsum(removed), before);
  }
  shrink_charge(allsum(next.size()));
  if (with_history) {
    if (dist())
      merge_history(*hbfs_, hbfs_i_, gather(next, false));
    else
      merge_history(*hbfs_, hbfs_i_, next);
  }
  // commit (bibfs_engine.hpp:375-379)
  ledger_.release(list_footprint(n_, lbfs_i_.size));
  if (lbfs_met_ && lbfs_i_.size >= opt_.tuning.min_brute)  // its meet permuted L_IBFS
    met_lists_.push_back(std::make_unique<DList>(std::move(*lbfs_)));
  lbfs_met_ = false;
  *lbfs_ = std::move(next);
  lbfs_index_.reset();
  lbfs_trie_.reset();
  refresh_part(*lbfs_, lbfs_i_);
  charged_layer_ = 0;
  rb.armed = false;
  if (opt_.track_word) bfs_levels_.push_back(level_tags_of(*lbfs_));
  ratio_bfs_[0] = 0.5 * ratio_bfs_[0] + 0.5 * r_dupl;
  ratio_bfs_[1] = 0.5 * ratio_bfs_[1] + 0.5 * r_self;
  if (with_history) ratio_bfs_[2] = 0.5 * ratio_bfs_[2] + 0.5 * r_hist;
}

// Inverse step (bibfs_engine.hpp:195-238): all reductions on complements, so
// the kept plain sets are the maximal ones; L_IBFS is committed in
// complement-lex order, H_IBFS stays complemented.
void GpuBibfs::ibfs_step(bool with_history) {
  if (!with_history) drop_ibfs_history();
  if (with_history && static_cast<double>(hibfs_i_.size) >=
                          opt_.tuning.history_growth * static_cast<double>(h_ibfs_last_reduced_)) {
    const u64 before = list_footprint(n_, hibfs_i_.size);
    // keep complements whose plain cardinality n - c is >= min card of L_IBFS
    dev::keep_card_at_most(ctx_, *hibfs_c_, n_ - libfs_i_.min_card);
    // minimal complements == maximal plain sets (superset join, plain space)
    dev::complement(ctx_, *hibfs_c_);
    dev::self_reduce_maximal(ctx_, *hibfs_c_);
    dev::complement(ctx_, *hibfs_c_);
    refresh(*hibfs_c_, hibfs_i_);
    h_ibfs_last_reduced_ = hibfs_i_.size;
    ledger_.release(before - list_footprint(n_, hibfs_i_.size));
  }
  charge_layer(libfs_i_.size);
  DList next(&ctx_, libfs_->size() * k_, opt_.track_word);
  dev::expand(ctx_, *libfs_, 0, libfs_->size(), /*inverse=*/true, next);
  Rollback rb{ledger_, charged_layer_};
  dev::complement(ctx_, next);
  if (dist()) {
    if (opt_.track_word) dev::add_to_tags(ctx_, next, rank_offset(*libfs_) << 16);
    exchange(next);
  }
  const size_t generated = libfs_i_.size * k_;
  const double r_dupl = generated ? ratio(allsum(dev::lex_sort_dedupe(ctx_, next)), generated) : 0.0;
  const size_t after_dupl = allsum(next.size());
  // The reductions of the reference run on complements (minimal sets there);
  // on plain sets they are superset queries — done by the bucketed superset
  // join, which keeps the complement-lex order of `next`.
  dev::complement(ctx_, next);
  size_t removed_self;
  if (dist()) {
    const DList layer = gather(next, false);
    removed_self = dev::remove_subsets_of(ctx_, layer, next, /*proper=*/true);
  } else {
    removed_self = dev::self_reduce_maximal(ctx_, next);
  }
  const double r_self = ratio(allsum(removed_self), after_dupl);
  double r_hist = 0.0;
  if (with_history) {
    const size_t before = allsum(next.size());
    DList h_plain = dev::copy_list(ctx_, *hibfs_c_, false);
    dev::complement(ctx_, h_plain);
    const size_t removed = dev::remove_subsets_of(ctx_, h_plain, next, /*proper=*/false);
    r_hist = ratio(allsum(removed), before);
  }
  dev::complement(ctx_, next);
  shrink_charge(allsum(next.size()));
  if (with_history) {
    if (dist())
      merge_history(*hibfs_c_, hibfs_i_, gather(next, false));
    else
      merge_history(*hibfs_c_, hibfs_i_, next);
  }
  dev::complement(ctx_, next);
  ledger_.release(list_footprint(n_, libfs_i_.size));
  *libfs_ = std::move(next);
  met_lists_.clear();  // a fresh L_IBFS in complement-lex order
  lbfs_met_ = false;
  refresh_part(*libfs_, libfs_i_);
  charged_layer_ = 0;
  rb.armed = false;
  if (opt_.track_word) ibfs_levels_.push_back(level_tags_of(*libfs_));
  ratio_ibfs_[0] = 0.5 * ratio_ibfs_[0] + 0.5 * r_dupl;
  ratio_ibfs_[1] = 0.5 * ratio_ibfs_[1] + 0.5 * r_self;
  if (with_history) ratio_ibfs_[2] = 0.5 * ratio_ibfs_[2] + 0.5 * r_hist;
}

void GpuBibfs::perform(StepKind kind) {
  switch (kind) {
    case StepKind::BFS: return bfs_step(true);
    case StepKind::BFS_NH: return bfs_step(false);
    case StepKind::IBFS: return ibfs_step(true);
    case StepKind::IBFS_NH: return ibfs_step(false);
    case StepKind::DFS: break;
  }
  throw std::logic_error("perform: DFS is not a list step");
}

// Meet: is some X in L_BFS a subset of some Y in L_IBFS?
// Small lists: one all-pairs launch instead of building the index.
bool GpuBibfs::meet() {
  // No L_BFS set can lie inside a smaller L_IBFS set: the reference's per-pair
  // card filter (subset_algebra.hpp:66) decides the whole check — e.g. every
  // meet against the initial singletons — without building an index.
  const bool hopeless = lbfs_i_.min_card > libfs_i_.max_card;
  if (dist()) {
    if (hopeless) return false;  // owned L_BFS sets against the whole L_IBFS, any rank's hit counts
    const DList ibfs = gather(*libfs_, false);
    bool met = false;
    if (!lbfs_->empty() && !ibfs.empty())
      met = dev::brute_fits(lbfs_->size(), ibfs.size()) && !dev::bitmap_fits(ctx_)
                ? dev::brute_exists_subset(ctx_, *lbfs_, ibfs, nullptr)
                : exists_in_bfs(ibfs, nullptr);
    return allsum(met ? 1 : 0) > 0;
  }
  lbfs_met_ = !opt_.track_word;  // meet_check permutes L_IBFS (subset_algebra.hpp:201-210)
  if (hopeless) return false;
  if (dev::brute_fits(lbfs_->size(), libfs_->size()) && !dev::bitmap_fits(ctx_))
    return dev::brute_exists_subset(ctx_, *lbfs_, *libfs_, nullptr);
  return exists_in_bfs(*libfs_, nullptr);
}

bool GpuBibfs::meet_witness(size_t* bfs_index_out, u64* ibfs_tag) {
  if (lbfs_i_.min_card > libfs_i_.max_card) return false;  // as meet()
  if (dist()) {  // the lowest rank with a hit reports (global L_BFS index, L_IBFS tag)
    const DList ibfs = gather(*libfs_, true);
    dev::Witness w;
    bool met = false;
    if (!lbfs_->empty() && !ibfs.empty())
      met = dev::brute_fits(lbfs_->size(), ibfs.size()) && !dev::bitmap_fits(ctx_)
                ? dev::brute_exists_subset(ctx_, *lbfs_, ibfs, &w)
                : exists_in_bfs(ibfs, &w);
    const u64 off = rank_offset(*lbfs_);
    u64 winner = met ? static_cast<u64>(opt_.comm->rank()) : static_cast<u64>(opt_.comm->size());
    opt_.comm->all_reduce(ctx_, &winner, 1, ReduceOp::Min);
    if (winner == static_cast<u64>(opt_.comm->size())) return false;
    u64 v[2] = {0, 0};
    if (winner == static_cast<u64>(opt_.comm->rank())) {
      v[0] = off + w.a_index;
      v[1] = dev::read_tag(ctx_, ibfs, w.b_index);
    }
    opt_.comm->all_reduce(ctx_, v, 2, ReduceOp::Sum);
    *bfs_index_out = static_cast<size_t>(v[0]);
    *ibfs_tag = v[1];
    return true;
  }
  dev::Witness w;
  const bool met = dev::brute_fits(lbfs_->size(), libfs_->size()) && !dev::bitmap_fits(ctx_)
                       ? dev::brute_exists_subset(ctx_, *lbfs_, *libfs_, &w)
                       : exists_in_bfs(*libfs_, &w);
  if (!met) return false;
  *bfs_index_out = w.a_index;
  *ibfs_tag = dev::read_tag(ctx_, *libfs_, w.b_index);
  return true;
}

void GpuBibfs::replay_meet_order() {
  std::vector<const DList*> met;
  for (const auto& l : met_lists_) met.push_back(l.get());
  if (lbfs_met_ && lbfs_i_.size >= opt_.tuning.min_brute) met.push_back(lbfs_.get());
  if (met.empty() || libfs_i_.size < 2) return;
  const u32 W = ctx_.W();
  std::vector<u64> B(libfs_i_.size * W);
  dev::download(ctx_, *libfs_, B.data(), nullptr, nullptr);
  std::vector<u32> order(libfs_i_.size);
  for (size_t i = 0; i < order.size(); ++i) order[i] = static_cast<u32>(i);
  std::vector<u64> A;
  for (const DList* l : met) {  // oldest first, as the meets ran
    DList sorted = dev::copy_list(ctx_, *l, false);
    dev::sort_lex(ctx_, sorted);  // L_BFS is lex-sorted unique in the reference
    A.resize(sorted.size() * W);
    dev::download(ctx_, sorted, A.data(), nullptr, nullptr);
    replay_meet_check(A.data(), sorted.size(), B.data(), W, n_, opt_.tuning.min_brute, order);
  }
  u32* perm = static_cast<u32*>(ctx_.alloc(order.size() * 4));
  ctx_.memcpy_h2d(perm, order.data(), order.size() * 4);
  dev::gather_rows(ctx_, *libfs_, perm);
  ctx_.free(perm);
  met_lists_.clear();
  lbfs_met_ = false;
}

// -------------------------------------------------------------- DFS phase
namespace {

// dfs_phase.hpp:74-80
size_t dfs_slice_cap(const MemoryLedger& ledger, u32 n, u32 k, u64 bound, u64 r) {
  const u64 set_bytes = words_for(n) * sizeof(u64);
  const u64 levels = bound > r ? bound - r : 1;
  const u64 denom = (k + 1) * levels * set_bytes;
  return static_cast<size_t>(std::max<u64>(ledger.available() / std::max<u64>(denom, 1), 1));
}

// Analysis aid: with SYNCHRO_DUMP_DIR set, lists are written as raw u64 words.
void dump_list(dev::Context& c, const DList& l, const std::string& name) {
  const char* dir = std::getenv("SYNCHRO_DUMP_DIR");
  if (!dir || !*dir) return;
  std::vector<u64> w(l.size() * c.W());
  dev::download(c, l, w.data(), nullptr, nullptr);
  if (FILE* f = std::fopen((std::string(dir) + "/" + name + ".u64").c_str(), "wb")) {
    std::fwrite(w.data(), 8, w.size(), f);
    std::fclose(f);
  }
}

// Level-by-level inverse DFS below the frozen L_BFS (dfs_phase.hpp:47-177):
// the recursion, slicing and ledger stay on the host; every level's
// preimages, (card desc, lex) order, dedupe, window pruning and containment
// query against L_BFS are device kernels.
class DfsRunner {
 public:
  using Query = std::function<bool(const DList&, dev::Witness*)>;
  DfsRunner(dev::Context& c, const DList& lbfs, Query query, MemoryLedger& ledger,
            const EngineTuning& t, const Deadline& deadline, bool tracking,
            std::vector<std::array<u64, 5>>* log, bool reference_order)
      : c_(c), lbfs_(lbfs), query_(std::move(query)), ledger_(ledger), t_(t), deadline_(deadline),
        tracking_(tracking), log_(log), reference_order_(reference_order) {}

  // Shard s of c explores the subtrees of initial[i] for i ≡ s (mod c) only
  // (c = 1: everything).  Interleaved rather than contiguous shares: the work
  // below an initial set falls with its position in L_IBFS's order (n=570 s0,
  // 8 contiguous shares: 174 s down to 56 s per shard).
  u64 run(const DList& initial, u64 r0, u64 bound, u32 shard = 0, u32 shards = 1) {
    bound_ = bound;
    if (r0 >= bound_ || initial.empty()) return bound_;
    DList share;
    const DList* roots = &initial;
    if (shards > 1) {
      share = dev::strided_copy(c_, initial, shard, shards, tracking_);
      roots = &share;
      root_start_ = shard;
      root_stride_ = shards;
    }
    const size_t cap = slice_cap(r0 - 1);
    for (size_t lo = 0; lo < roots->size(); lo += cap) {
      recurse(*roots, lo, std::min(roots->size(), lo + cap), r0, 0, nullptr);
      if (r0 >= bound_) break;
    }
    return bound_;
  }
  const DfsFind& find() const { return find_; }
  u64 expansions = 0;
  // Progress mode: device+host seconds per DFS phase (expand, dedupe, window,
  // query, sort, order replay), one stream sync per phase.
  void report_phases() const {
    if (!phases_on()) return;
    std::fprintf(stderr, "[synchro] dfs phases [s]: expand %.2f dedupe %.2f window %.2f query %.2f "
                 "sort %.2f order-replay %.2f\n", phase_s_[0], phase_s_[1], phase_s_[2],
                 phase_s_[3], phase_s_[4], phase_s_[5]);
  }
  // SYNCHRO_DFS_PHASES=1 (or the progress log): one stream sync per phase.
  static bool phases_on() {
    static const bool on = progress_enabled() || [] {
      const char* e = std::getenv("SYNCHRO_DFS_PHASES");
      return e && *e && *e != '0';
    }();
    return on;
  }

 private:
  struct Frame {
    const Frame* up;
    const DList* list;
  };
  struct Guard {
    MemoryLedger& l;
    u64 amount;
    ~Guard() { l.release(amount); }
  };

  size_t slice_cap(u64 r) const { return dfs_slice_cap(ledger_, c_.n(), c_.k(), bound_, r); }

  void recurse(const DList& list, size_t lo, size_t hi, u64 r, u32 level, const Frame* parent) {
    deadline_.check();
    const u32 k = c_.k(), n = c_.n();
    const u64 charged = list_footprint(n, static_cast<u64>(hi - lo) * k);
    ledger_.charge_or_throw(charged);
    Guard guard{ledger_, charged};
    DList next(&c_, (hi - lo) * k, tracking_);
    phase_begin();
    dev::expand(c_, list, lo, hi, /*inverse=*/true, next);
    phase_end(0);
    expansions += static_cast<u64>(hi - lo) * k;
    const u64 generated = next.size();
    // The reference sorts every level by (card desc, lex, index) (dfs_phase.hpp:105).
    // The order is observable only through the top-dfs_largest window (selected
    // as a multiset without sorting) and the slice boundaries (sorted only when the
    // level is sliced); the dedupe is set-semantic (which equal row's tag survives
    // changes only the reported witness), and the trie query is order-free.
    phase_begin();
    if (t_.dfs_dedupe_cadence && level % t_.dfs_dedupe_cadence == 0)
      dev::hash_dedupe(c_, next, /*first_occurrence=*/false);  // any equal row's tag is a valid parent
    phase_end(1);
    phase_begin();
    if (t_.dfs_reduce_cadence && level % t_.dfs_reduce_cadence == 0 && next.size() > t_.dfs_largest) {
      // Drop sets that are proper subsets of one of the dfs_largest first
      // (largest) sets.  The reference marks proper supersets among
      // complements; on plain sets it is a superset join (order kept).
      // The window is the first dfs_largest rows of the sorted level (a multiset);
      // selected without sorting the level (beam.cu top_card_desc_lex).
      const DList largest = dev::top_card_desc_lex(c_, next, t_.dfs_largest);
      dev::remove_subsets_of(c_, largest, next, /*proper=*/true);
    }
    phase_end(2);
    const u64 now = list_footprint(n, next.size());
    if (now < charged) {
      ledger_.release(charged - now);
      guard.amount = now;
    }
    if (log_) log_->push_back({r, level, hi - lo, generated, next.size()});
    if (dumped_.insert(r).second) dump_list(c_, next, "dfs_r" + std::to_string(r));
    SYNCHRO_PROGRESS("dfs r=%llu level=%u in=%zu generated=%llu kept=%zu",
                     static_cast<unsigned long long>(r), level, hi - lo,
                     static_cast<unsigned long long>(generated), next.size());
    dev::Witness w;
    phase_begin();
    const bool hit = query_(next, tracking_ ? &w : nullptr);
    phase_end(3);
    if (hit) {
      bound_ = r;
      if (tracking_) record_find(w, next, parent);
      return;
    }
    if (r >= bound_ - 1) return;
    const size_t cap = slice_cap(r);
    // Slices follow the order the trie queries left (the reference's order).
    // Relaxed order: any partition into slices keeps the threshold (every
    // in-slice reduction keeps a dominating set); the level is grouped by
    // cardinality (descending) before slicing — measured at n=570: 423 s with
    // the full (card desc, lex) sort, 485 s for slices of the unsorted level
    // (more query work below mixed-card slices).
    if (next.size() > cap) {
      phase_begin();
      if (reference_order_)
        dev::sort_card_desc_lex(c_, next);
      else  // cardinality classes together; lex order inside them is not needed
        dev::sort_card_desc(c_, next);
      phase_end(4);
      if (reference_order_) {
        phase_begin();
        replay_query_order(next, cap);
        phase_end(5);
      }
    }
    const Frame frame{parent, &next};
    for (size_t plo = 0; plo < next.size(); plo += cap) {
      recurse(next, plo, std::min(next.size(), plo + cap), r + 1, level + 1, &frame);
      if (r >= bound_ - 1) return;
    }
  }

  // The reference queries the trie per cardinality group of the (card desc,
  // lex)-sorted level, and each query permutes its group in place
  // (static_trie.hpp:177-183) before the level is cut into slices of `cap`.
  // Only groups that straddle a slice boundary change which sets share a
  // slice; their order is replayed on the host (meet_order.cpp).
  void replay_query_order(DList& level, size_t cap) {
    const auto t0 = std::chrono::steady_clock::now();
    const size_t N = level.size();
    std::vector<u32> cards(N);
    dev::download(c_, level, nullptr, cards.data(), nullptr);
    std::vector<std::pair<size_t, size_t>> groups;
    for (size_t b = cap; b < N; b += cap) {
      if (cards[b - 1] != cards[b]) continue;  // boundary between two groups
      size_t lo = b - 1, hi = b + 1;
      while (lo > 0 && cards[lo - 1] == cards[b]) --lo;
      while (hi < N && cards[hi] == cards[b]) ++hi;
      if (groups.empty() || groups.back().first != lo) groups.emplace_back(lo, hi);
    }
    if (groups.empty()) return;
    if (!shape_) {
      shape_ = std::make_unique<dev::TrieShape>();
      dev::trie_shape(c_, lbfs_, t_.min_leaf, shape_.get());
    }
    const u32 W = c_.W();
    std::vector<u32> perm(N);
    for (size_t i = 0; i < N; ++i) perm[i] = static_cast<u32>(i);
    for (const auto& [lo, hi] : groups) {
      DList g = dev::slice_copy(c_, level, lo, hi, false);
      std::vector<u64> rows((hi - lo) * W);
      dev::download(c_, g, rows.data(), nullptr, nullptr);
      std::vector<u32> order(hi - lo);
      for (size_t i = 0; i < order.size(); ++i) order[i] = static_cast<u32>(i);
      replay_trie_query(*shape_, rows.data(), W, cards[lo], order);
      for (size_t i = 0; i < order.size(); ++i) perm[lo + i] = static_cast<u32>(lo + order[i]);
    }
    u32* d = static_cast<u32*>(c_.alloc(N * 4));
    c_.memcpy_h2d(d, perm.data(), N * 4);
    dev::gather_rows(c_, level, d);
    c_.free(d);
    size_t gq = 0;
    for (const auto& g : groups) gq += g.second - g.first;
    SYNCHRO_PROGRESS("  dfs slice order replay: |level|=%zu groups=%zu queries=%zu %.3f s", N,
                     groups.size(), gq,
                     std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
  }

  void record_find(const dev::Witness& w, const DList& level, const Frame* parent) {
    find_.found = true;
    find_.trie_index = w.a_index;
    find_.middle.clear();
    u64 tag = dev::read_tag(c_, level, w.b_index);
    for (const Frame* f = parent;; f = f->up) {
      find_.middle.push_back(static_cast<u32>(tag & 0xFFFF));
      const size_t idx = static_cast<size_t>(tag >> 16);
      if (!f) {  // index into the shard's roots -> index into L_IBFS
        find_.root_index = root_start_ + idx * root_stride_;
        break;
      }
      tag = dev::read_tag(c_, *f->list, idx);
    }
  }

  dev::Context& c_;
  const DList& lbfs_;
  Query query_;
  MemoryLedger& ledger_;
  const EngineTuning& t_;
  const Deadline& deadline_;
  bool tracking_;
  std::vector<std::array<u64, 5>>* log_;
  bool reference_order_;
  u64 bound_ = 0;
  size_t root_start_ = 0, root_stride_ = 1;
  DfsFind find_;
  std::set<u64> dumped_;
  std::unique_ptr<dev::TrieShape> shape_;  // the reference trie over L_BFS, built on first use
  void phase_begin() {
    if (!phases_on()) return;
    c_.sync();
    phase_t0_ = std::chrono::steady_clock::now();
  }
  void phase_end(int i) {
    if (!phases_on()) return;
    c_.sync();
    phase_s_[i] += std::chrono::duration<double>(std::chrono::steady_clock::now() - phase_t0_).count();
  }
  std::chrono::steady_clock::time_point phase_t0_;
  double phase_s_[6] = {0, 0, 0, 0, 0, 0};
};

}  // namespace

// bibfs_engine.hpp:275-298: drop histories, freeze L_BFS as the containment
// structure (charged as the reference's trie: sets + 24 B per trie node),
// run the DFS from L_IBFS.
u64 GpuBibfs::run_dfs(u64 r, DfsFind* find, std::vector<std::array<u64, 5>>* log,
                      u64* expansions) {
  drop_bfs_history();
  drop_ibfs_history();
  if (lbfs_i_.size == 0) return R_;
  if (dist()) {  // the static structure over the WHOLE L_BFS on every rank; the
                 // roots (L_IBFS) in global order, explored in interleaved shares
    *lbfs_ = gather(*lbfs_, false);
    *libfs_ = gather(*libfs_, opt_.track_word);
    lbfs_index_.reset();
    lbfs_trie_.reset();
  }
  const u64 nodes = dev::trie_node_count(ctx_, *lbfs_, opt_.tuning.min_leaf);
  const u64 trie_bytes = list_footprint(n_, lbfs_i_.size) + nodes * 24;
  ledger_.charge_or_throw(trie_bytes);
  ledger_.release(list_footprint(n_, lbfs_i_.size));
  // The top-level slices follow L_IBFS's order: reproduce the reference's
  // post-meet_check order when they will actually cut the list.
  if (!dist() && opt_.dfs_reference_order && !opt_.track_word && r < R_ &&
      libfs_i_.size > dfs_slice_cap(ledger_, n_, k_, R_, r - 1))
    replay_meet_order();
  dump_list(ctx_, *lbfs_, "lbfs");
  dump_list(ctx_, *libfs_, "libfs");
  DfsRunner dfs(ctx_, *lbfs_, [this](const DList& b, dev::Witness* w) { return exists_in_bfs(b, w); },
                ledger_, opt_.tuning, deadline_, opt_.track_word, log,
                opt_.dfs_reference_order);
  const u32 shard = dist() ? static_cast<u32>(opt_.comm->rank()) : opt_.dfs_shard_index;
  const u32 shards = dist() ? static_cast<u32>(opt_.comm->size())
                            : std::max<u32>(1, opt_.dfs_shard_count);
  u64 final_bound = dfs.run(*libfs_, r, R_, shard, shards);
  dfs.report_phases();
  DfsFind mine = dfs.find();
  u64 exp = dfs.expansions;
  if (dist()) {
    // threshold = MIN over the shards; the lowest rank attaining it with a
    // find hands its witness (trie index, root index, middle letters) to all
    Comm& cm = *opt_.comm;
    u64 best = final_bound;
    cm.all_reduce(ctx_, &best, 1, ReduceOp::Min);
    u64 winner = (mine.found && final_bound == best) ? static_cast<u64>(cm.rank())
                                                     : static_cast<u64>(cm.size());
    cm.all_reduce(ctx_, &winner, 1, ReduceOp::Min);
    exp = allsum(exp);
    if (winner < static_cast<u64>(cm.size())) {
      std::vector<u64> pack;
      if (winner == static_cast<u64>(cm.rank())) {
        pack = {mine.trie_index, mine.root_index, mine.middle.size()};
        for (u32 a : mine.middle) pack.push_back(a);
      }
      const std::vector<u64> len = cm.all_gather_u64(ctx_, pack.size());
      u64* d = static_cast<u64*>(ctx_.alloc((len[winner] + 1) * 8));
      u64* src = static_cast<u64*>(ctx_.alloc((pack.size() + 1) * 8));
      ctx_.memcpy_h2d(src, pack.data(), pack.size() * 8);
      std::vector<u64> rb(len.size());
      for (size_t q = 0; q < len.size(); ++q) rb[q] = len[q] * 8;
      cm.all_gather_v(ctx_, src, pack.size() * 8, d, rb);
      std::vector<u64> got(len[winner]);
      ctx_.memcpy_d2h(got.data(), d, got.size() * 8);
      ctx_.free(d);
      ctx_.free(src);
      mine.found = true;
      mine.trie_index = got[0];
      mine.root_index = got[1];
      mine.middle.assign(got.begin() + 3, got.begin() + 3 + static_cast<long>(got[2]));
    } else {
      mine.found = false;
    }
    final_bound = best;
  }
  if (find) *find = mine;
  if (expansions) *expansions = exp;
  ledger_.release(trie_bytes);
  R_ = final_bound;
  return final_bound;
}

// ------------------------------------------------------- reconstruction
Word GpuBibfs::bfs_prefix(size_t index) const {
  Word w;
  size_t idx = index;
  for (size_t lvl = bfs_levels_.size(); lvl-- > 0;) {
    const u64 tag = bfs_levels_[lvl].at(idx);
    w.push_back(static_cast<u32>(tag & 0xFFFF));
    idx = static_cast<size_t>(tag >> 16);
  }
  std::reverse(w.begin(), w.end());
  return w;
}

Word GpuBibfs::ibfs_suffix_from_tag(u64 tag) const {
  Word w;
  for (size_t lvl = ibfs_levels_.size(); lvl-- > 0;) {
    w.push_back(static_cast<u32>(tag & 0xFFFF));
    if (lvl == 0) break;
    tag = ibfs_levels_[lvl - 1].at(static_cast<size_t>(tag >> 16));
  }
  return w;
}

Word GpuBibfs::ibfs_suffix_from_index(size_t index) const {
  if (ibfs_levels_.empty()) return {};
  return ibfs_suffix_from_tag(ibfs_levels_.back().at(index));
}

// bibfs_engine.hpp:442-460 (same keys, same default ostream formatting).
void trace_line(std::ostream* trace, const GpuBibfs& eng, const SearchStats& s, const StepCosts& c,
                StepKind kind) {
  if (!trace) return;
  std::ostringstream os;
  os << "iter=" << eng.iteration() << " step=" << step_kind_name(kind)
     << " lbfs=" << static_cast<u64>(s.bfs.list_size) << " libfs=" << static_cast<u64>(s.ibfs.list_size)
     << " hbfs=" << static_cast<u64>(s.bfs.hist_size) << " hibfs=" << static_cast<u64>(s.ibfs.hist_size)
     << " d_lbfs=" << s.bfs.list_density << " d_libfs=" << s.ibfs.list_density
     << " rdupl_bfs=" << s.bfs.r_dupl << " rself_bfs=" << s.bfs.r_self << " rhist_bfs=" << s.bfs.r_hist
     << " rdupl_ibfs=" << s.ibfs.r_dupl << " rself_ibfs=" << s.ibfs.r_self
     << " rhist_ibfs=" << s.ibfs.r_hist << " cost_bfs=" << c.step[0] << " cost_bfs_nh=" << c.step[1]
     << " cost_ibfs=" << c.step[2] << " cost_ibfs_nh=" << c.step[3] << " pred_bfs=" << c.pred[0]
     << " pred_bfs_nh=" << c.pred[1] << " pred_ibfs=" << c.pred[2] << " pred_ibfs_nh=" << c.pred[3]
     << " pred_dfs=" << c.pred[4];
  *trace << os.str() << '\n';
}

}  // namespace detail

// --------------------------------------------------------------- solve
SolveResult solve_exact(const Automaton& aut, const SolveOptions& opt) {
  return solve_exact(aut, opt, nullptr);
}

SolveResult solve_exact(const Automaton& aut, const SolveOptions& opt, dev::Context* shared) {
  SolveResult res;
  if (aut.state_count() == 1) {  // (synchronizing by definition)
    res.phase = "trivial";
    if (opt.track_word) res.word = Word{};
    return res;
  }
  std::unique_ptr<dev::Context> own;
  if (shared) {
    shared->bind(aut);
  } else {
    own = std::make_unique<dev::Context>(aut, opt.device);
  }
  dev::Context& ctx = shared ? *shared : *own;
  // Pair merge distances once: the synchronizability precondition
  // (automaton.hpp:153-157) and Eppstein's bound (heuristics.hpp:26-79) share
  // them.  The pair BFS runs on the device (pairs.cu) from kPairBfsDeviceMin
  // states on; below that the whole pair graph is a few thousand pairs and the
  // host's BFS costs less than the launches and readbacks of one level each.
  const std::vector<u32> pair_dist = aut.state_count() >= kPairBfsDeviceMin
                                         ? dev::pair_distances(ctx, aut)
                                         : pair_merge_distances(aut, InverseTransitions(aut));
  if (std::find(pair_dist.begin(), pair_dist.end(), std::numeric_limits<u32>::max()) != pair_dist.end())
    throw NotSynchronizingError();
  ctx.timing = opt.timing;
  ctx.contain_stats = opt.contain_stats;
  using clock = std::chrono::steady_clock;
  const auto t0 = clock::now();
  std::optional<HeuristicResult> heur;
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
    aopt.pair_dist = &pair_dist;
    heur = adaptive_upper_bound(aut, aopt, &ctx);
    R = heur->length;
  }
  res.upper_bound = R;
  SYNCHRO_PROGRESS("n=%u k=%u upper bound R=%llu", aut.state_count(), aut.alphabet_size(),
                   static_cast<unsigned long long>(R));
  const auto t1 = clock::now();
  res.heuristic_seconds = std::chrono::duration<double>(t1 - t0).count();

  dev::StreamTimer engine_timer(ctx);
  engine_timer.start();
  detail::GpuBibfs eng(aut, R, opt, ctx);
  const auto finish = [&](u64 threshold, std::optional<Word> word, const char* phase) {
    res.engine_device_ms = engine_timer.stop_ms();
    res.h2d_bytes = ctx.counters.h2d_bytes;
    res.d2h_bytes = ctx.counters.d2h_bytes;
    res.threshold = threshold;
    res.word = std::move(word);
    res.peak_memory = eng.ledger().peak();
    res.phase = phase;
    res.engine_seconds = std::chrono::duration<double>(clock::now() - t1).count();
    res.expand_kernel_ms = ctx.counters.expand_ms;
    res.kernel_launches = ctx.counters.kernel_launches;
    res.contain_kernel_ms = ctx.counters.contain_ms;
    res.contain_bytes = ctx.counters.contain_bytes;
    res.contain_visits = ctx.counters.contain_visits;
    res.contain_pairs = ctx.counters.contain_pairs;
    SYNCHRO_PROGRESS("host-device traffic: %llu launches, %llu syncs, %llu pool allocations",
                     static_cast<unsigned long long>(ctx.counters.kernel_launches),
                     static_cast<unsigned long long>(ctx.counters.syncs),
                     static_cast<unsigned long long>(ctx.counters.allocs));
    return res;
  };

  for (u64 r = 1; r + 1 <= R; ++r) {
    if (opt.stop_after_iterations && res.iterations >= opt.stop_after_iterations)
      return finish(0, std::nullopt, "stopped");
    eng.deadline().check();
    eng.set_iteration(r);
    eng.clear_failures();
    ++res.iterations;
    StepKind kind = StepKind::DFS;
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
          kind = sc.feasible[2] ? StepKind::IBFS : (sc.feasible[3] ? StepKind::IBFS_NH : StepKind::DFS);
          break;
        case Schedule::DfsImmediate: kind = StepKind::DFS; break;
      }
      if (kind == StepKind::DFS) break;
      const u64 parents = (kind == StepKind::BFS || kind == StepKind::BFS_NH) ? eng.bfs_size()
                                                                              : eng.ibfs_size();
      try {
        eng.perform(kind);
        res.expansions_phase1 += parents * aut.alphabet_size();
        break;
      } catch (const OutOfMemoryError&) {
        eng.mark_failed(kind);  // engine rolled back; choose again
      }
    }

    if (kind == StepKind::DFS) {
      res.used_dfs = true;
      if (opt.trace) *opt.trace << "iter=" << r << " step=DFS handoff\n";
      DfsFind find;
      const u64 threshold = eng.run_dfs(r, &find, &res.dfs_levels, &res.expansions_dfs);
      if (opt.trace) *opt.trace << "result=" << threshold << " phase=dfs\n";
      std::optional<Word> word;
      if (opt.track_word) {
        if (find.found) {
          Word w = eng.bfs_prefix(find.trie_index);
          w.insert(w.end(), find.middle.begin(), find.middle.end());
          const Word tail = eng.ibfs_suffix_from_index(find.root_index);
          w.insert(w.end(), tail.begin(), tail.end());
          if (w.size() != threshold || !is_reset_word(aut, w))
            throw std::logic_error("reconstructed word is not a valid witness");
          word = std::move(w);
        } else if (heur && heur->length == threshold) {
          word = heur->word;
        }
      }
      return finish(threshold, std::move(word), "dfs");
    }

    if (kind == StepKind::BFS || kind == StepKind::BFS_NH)
      ++res.bfs_steps;
    else
      ++res.ibfs_steps;
    detail::trace_line(opt.trace, eng, st, sc, kind);
    SYNCHRO_PROGRESS("iter %llu %s -> |L_BFS|=%zu |L_IBFS|=%zu", static_cast<unsigned long long>(r),
                     step_kind_name(kind), eng.bfs_size(), eng.ibfs_size());

    if (opt.track_word) {
      size_t bi = 0;
      u64 tag = 0;
      if (eng.meet_witness(&bi, &tag)) {
        Word full = eng.bfs_prefix(bi);
        const Word tail = eng.ibfs_suffix_from_tag(tag);
        full.insert(full.end(), tail.begin(), tail.end());
        if (full.size() != r || !is_reset_word(aut, full))
          throw std::logic_error("reconstructed word is not a valid witness");
        if (opt.trace) *opt.trace << "result=" << r << " phase=meet\n";
        return finish(r, std::move(full), "meet");
      }
    } else if (eng.meet()) {
      if (opt.trace) *opt.trace << "result=" << r << " phase=meet\n";
      return finish(r, std::nullopt, "meet");
    }
  }
  if (opt.trace) *opt.trace << "result=" << R << " phase=bound\n";
  std::optional<Word> word;
  if (opt.track_word && heur) word = heur->word;
  return finish(R, std::move(word), "bound");
}

}  // namespace synchro
