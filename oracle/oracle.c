/* oracle/oracle.c — TEST INFRASTRUCTURE ONLY (see oracle.h).  A plain-C
 * restatement of the reference's hot-path set algebra with the simplest
 * possible algorithms (quadratic scans, qsort), each function citing the
 * reference file:line whose observable behaviour it restates.  Only tests/
 * load it, as a checker; the product never links or calls it. */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

static uint32_t W_of(uint32_t n) { return (n + 63) / 64; }
static int test_bit(const uint64_t* s, uint32_t q) { return (int)((s[q >> 6] >> (63 - (q & 63))) & 1); }
static void set_bit(uint64_t* s, uint32_t q) { s[q >> 6] |= (uint64_t)1 << (63 - (q & 63)); }
static uint32_t card_of(const uint64_t* s, uint32_t W) {
  uint32_t c = 0;
  for (uint32_t w = 0; w < W; ++w) c += (uint32_t)__builtin_popcountll(s[w]);
  return c;
}
static int subset_of(const uint64_t* x, const uint64_t* y, uint32_t W) {
  for (uint32_t w = 0; w < W; ++w)
    if (x[w] & ~y[w]) return 0;
  return 1;
}
static int lex_cmp(const uint64_t* x, const uint64_t* y, uint32_t W) {
  for (uint32_t w = 0; w < W; ++w)
    if (x[w] != y[w]) return x[w] < y[w] ? -1 : 1;
  return 0;
}

/* util.hpp:45-50 */
uint64_t or_splitmix_next(uint64_t* state) {
  uint64_t z = (*state += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

/* util.hpp:54-61 (rejection sampling) + automaton.hpp:159-164 */
void or_random_automaton(uint32_t n, uint32_t k, uint64_t seed, uint32_t* delta) {
  uint64_t st = seed;
  const uint64_t bound = n;
  for (size_t i = 0; i < (size_t)n * k; ++i) {
    uint64_t v = 0;
    if (bound > 1) {
      const uint64_t rem = (UINT64_MAX % bound + 1) % bound;
      const uint64_t limit = UINT64_MAX - rem;
      uint64_t x = or_splitmix_next(&st);
      while (rem != 0 && x > limit) x = or_splitmix_next(&st);
      v = x % bound;
    }
    delta[i] = (uint32_t)v;
  }
}

/* experiment.hpp:54-56 + util.hpp:69-72 */
uint64_t or_instance_seed(uint64_t base, uint32_t n, uint32_t index) {
  uint64_t st = ((uint64_t)n << 32) ^ index;
  return base ^ or_splitmix_next(&st);
}

/* automaton.hpp:79-99 applied as in compute_layer (bibfs_engine.hpp:350-364):
 * child o = i*k + a is image(S_i, a) or preimage(S_i, a). */
void or_expand(uint32_t n, uint32_t k, const uint32_t* delta, const uint64_t* words, size_t count,
               int inverse, uint64_t* out_words, uint32_t* out_cards) {
  const uint32_t W = W_of(n);
  for (size_t i = 0; i < count; ++i)
    for (uint32_t a = 0; a < k; ++a) {
      uint64_t* o = out_words + (i * k + a) * W;
      memset(o, 0, W * 8);
      for (uint32_t q = 0; q < n; ++q) {
        const uint32_t t = delta[(size_t)q * k + a];
        if (!inverse && test_bit(words + i * W, q)) set_bit(o, t);
        if (inverse && test_bit(words + i * W, t)) set_bit(o, q);
      }
      out_cards[i * k + a] = card_of(o, W);
    }
}

/* ---- sorting: index sort with explicit tie-breaks (set_list.hpp:210-234) */
typedef struct {
  const uint64_t* words;
  const uint32_t* cards;
  uint32_t W;
  int by_card;
} SortCtx;
static SortCtx g_sort;
static int idx_cmp(const void* pa, const void* pb) {
  const size_t a = *(const size_t*)pa, b = *(const size_t*)pb;
  if (g_sort.by_card && g_sort.cards[a] != g_sort.cards[b]) return g_sort.cards[a] > g_sort.cards[b] ? -1 : 1;
  const int c = lex_cmp(g_sort.words + a * g_sort.W, g_sort.words + b * g_sort.W, g_sort.W);
  if (c) return c;
  return a < b ? -1 : (a > b ? 1 : 0);
}
static void apply_order(uint32_t W, uint64_t* words, uint32_t* cards, uint64_t* tags, const size_t* idx,
                        size_t count, size_t keep_count) {
  uint64_t* w2 = malloc(count * W * 8 + 8);
  uint32_t* c2 = malloc(count * 4 + 4);
  uint64_t* t2 = malloc(count * 8 + 8);
  for (size_t i = 0; i < keep_count; ++i) {
    memcpy(w2 + i * W, words + idx[i] * W, W * 8);
    c2[i] = cards[idx[i]];
    if (tags) t2[i] = tags[idx[i]];
  }
  memcpy(words, w2, keep_count * W * 8);
  memcpy(cards, c2, keep_count * 4);
  if (tags) memcpy(tags, t2, keep_count * 8);
  free(w2);
  free(c2);
  free(t2);
}
static size_t* sorted_index(uint32_t W, const uint64_t* words, const uint32_t* cards, size_t count, int by_card) {
  size_t* idx = malloc(count * sizeof(size_t) + 8);
  for (size_t i = 0; i < count; ++i) idx[i] = i;
  g_sort.words = words;
  g_sort.cards = cards;
  g_sort.W = W;
  g_sort.by_card = by_card;
  qsort(idx, count, sizeof(size_t), idx_cmp);
  return idx;
}

/* set_list.hpp:244-265: lex sort (index tie-break) + keep first of equal runs */
size_t or_lex_sort_dedupe(uint32_t n, uint64_t* words, uint32_t* cards, uint64_t* tags, size_t count) {
  const uint32_t W = W_of(n);
  if (count == 0) return 0;
  size_t* idx = sorted_index(W, words, cards, count, 0);
  size_t m = 0;
  for (size_t i = 0; i < count; ++i)
    if (i == 0 || lex_cmp(words + idx[i] * W, words + idx[m - 1] * W, W) != 0) idx[m++] = idx[i];
  apply_order(W, words, cards, tags, idx, count, m);
  free(idx);
  return m;
}

/* set_list.hpp:223-234 */
void or_sort_card_desc_lex(uint32_t n, uint64_t* words, uint32_t* cards, uint64_t* tags, size_t count) {
  const uint32_t W = W_of(n);
  if (count == 0) return;
  size_t* idx = sorted_index(W, words, cards, count, 1);
  apply_order(W, words, cards, tags, idx, count, count);
  free(idx);
}

/* subset_algebra.hpp:179-197: drop Y with some X ⊊ Y; order preserved */
size_t or_self_reduce_minimal(uint32_t n, uint64_t* words, uint32_t* cards, size_t count) {
  const uint32_t W = W_of(n);
  uint8_t* keep = malloc(count + 1);
  for (size_t j = 0; j < count; ++j) {
    keep[j] = 1;
    for (size_t i = 0; i < count && keep[j]; ++i)
      if (cards[i] < cards[j] && subset_of(words + i * W, words + j * W, W)) keep[j] = 0;
  }
  size_t m = 0;
  for (size_t j = 0; j < count; ++j)
    if (keep[j]) {
      memmove(words + m * W, words + j * W, W * 8);
      cards[m++] = cards[j];
    }
  free(keep);
  return m;
}

/* subset_algebra.hpp:138-174: mode 0 supersets (equality counts), 1 proper
 * supersets, 2 subsets (by complement).  keep[j] = !marked. */
void or_mark(uint32_t n, const uint64_t* a, size_t na, const uint64_t* b, size_t nb, int mode,
             uint8_t* keep) {
  const uint32_t W = W_of(n);
  for (size_t j = 0; j < nb; ++j) {
    int marked = 0;
    for (size_t i = 0; i < na && !marked; ++i) {
      const uint64_t* x = a + i * W;
      const uint64_t* y = b + j * W;
      if (mode == 2) {
        marked = subset_of(y, x, W);
      } else if (subset_of(x, y, W)) {
        marked = mode == 0 || lex_cmp(x, y, W) != 0;
      }
    }
    keep[j] = (uint8_t)!marked;
  }
}

/* subset_algebra.hpp:201-210 */
int or_meet_check(uint32_t n, const uint64_t* a, size_t na, const uint64_t* b, size_t nb) {
  const uint32_t W = W_of(n);
  for (size_t i = 0; i < na; ++i)
    for (size_t j = 0; j < nb; ++j)
      if (subset_of(a + i * W, b + j * W, W)) return 1;
  return 0;
}

/* static_trie.hpp:85-151: node count of the recursive partition by the most
 * frequent non-universal state (smallest index on ties), leaves <= min_leaf,
 * zero side absorbed as payload when <= min_leaf. */
static uint64_t trie_rec(uint32_t n, uint32_t W, uint64_t* rows, size_t lo, size_t hi, uint32_t min_leaf,
                         uint32_t* counts) {
  if (hi - lo <= min_leaf) return 1;
  memset(counts, 0, n * sizeof(uint32_t));
  for (size_t i = lo; i < hi; ++i)
    for (uint32_t q = 0; q < n; ++q) counts[q] += (uint32_t)test_bit(rows + i * W, q);
  uint32_t best = n, best_c = 0;
  for (uint32_t q = 0; q < n; ++q)
    if (counts[q] > best_c && counts[q] < hi - lo) {
      best_c = counts[q];
      best = q;
    }
  if (best == n) return 1; /* duplicates: the reference throws; not reached for unique input */
  size_t i = lo, j = hi;
  uint64_t* tmp = malloc(W * 8);
  while (i < j) {
    if (!test_bit(rows + i * W, best)) {
      ++i;
    } else {
      --j;
      memcpy(tmp, rows + i * W, W * 8);
      memcpy(rows + i * W, rows + j * W, W * 8);
      memcpy(rows + j * W, tmp, W * 8);
    }
  }
  free(tmp);
  uint64_t nodes = 1;
  if (i - lo > min_leaf) nodes += trie_rec(n, W, rows, lo, i, min_leaf, counts);
  nodes += trie_rec(n, W, rows, i, hi, min_leaf, counts);
  return nodes;
}

uint64_t or_trie_node_count(uint32_t n, const uint64_t* words, size_t count, uint32_t min_leaf) {
  const uint32_t W = W_of(n);
  if (count == 0) return 0;
  if (min_leaf < 1) min_leaf = 1;
  uint64_t* rows = malloc(count * W * 8);
  memcpy(rows, words, count * W * 8);
  uint32_t* counts = malloc(n * sizeof(uint32_t) + 4);
  const uint64_t r = trie_rec(n, W, rows, 0, count, min_leaf, counts);
  free(rows);
  free(counts);
  return r;
}

/* cost_model.hpp:62-74 */
double or_exp_mark(double as, double bs, double ad, double bd) {
  const double eps = 1e-6;
  if (as <= 0 || bs <= 0) return 0.0;
  ad = ad < eps ? eps : (ad > 1.0 - eps ? 1.0 - eps : ad);
  bd = bd < eps ? eps : (bd > 1.0 - eps ? 1.0 - eps : bd);
  const double w = (1.0 + bd) / (1.0 + ad * bd - ad);
  const double e = log(1.0 + bd) / log(w);
  return bs * ((1.0 + bd) / bd + 1.0 / (ad - ad * bd)) * pow(as, e);
}

/* oracle.hpp:17-57: BFS over the power set from Q to a singleton; -1 if none,
 * -2 if n > 20 (refused). */
int64_t or_power_set_oracle(uint32_t n, uint32_t k, const uint32_t* delta) {
  if (n > 20) return -2;
  if (n == 1) return 0;
  const uint32_t full = (1u << n) - 1;
  uint8_t* seen = calloc((size_t)full + 1, 1);
  uint32_t* cur = malloc(((size_t)full + 1) * 4);
  uint32_t* nxt = malloc(((size_t)full + 1) * 4);
  size_t nc = 1, nn;
  cur[0] = full;
  seen[full] = 1;
  for (int64_t depth = 1; nc; ++depth) {
    nn = 0;
    for (size_t i = 0; i < nc; ++i)
      for (uint32_t a = 0; a < k; ++a) {
        uint32_t img = 0;
        for (uint32_t q = 0; q < n; ++q)
          if ((cur[i] >> q) & 1) img |= 1u << delta[(size_t)q * k + a];
        if (seen[img]) continue;
        if ((img & (img - 1)) == 0) {
          free(seen);
          free(cur);
          free(nxt);
          return depth;
        }
        seen[img] = 1;
        nxt[nn++] = img;
      }
    uint32_t* t = cur;
    cur = nxt;
    nxt = t;
    nc = nn;
  }
  free(seen);
  free(cur);
  free(nxt);
  return -1;
}
