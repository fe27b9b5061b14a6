/* oracle/oracle.h — TEST INFRASTRUCTURE ONLY: a plain-C restatement of the
 * reference's set algebra for the hot path, for small inputs (quadratic
 * algorithms).  Never linked into the product.  Pinned against the compiled
 * reference (oracle/_ref) by tests/test_oracle_c.py.  Conventions as in the
 * reference: sets are W = ceil(n/64) u64 words, MSB-first (state 0 = bit 63 of
 * word 0, state_set.hpp:14-19); lists are row-major words[count][W]. */
#ifndef SYNCHRO_ORACLE_H_
#define SYNCHRO_ORACLE_H_
#include <stddef.h>
#include <stdint.h>

uint64_t or_splitmix_next(uint64_t* state);                               /* util.hpp:45-50 */
void or_random_automaton(uint32_t n, uint32_t k, uint64_t seed, uint32_t* delta); /* automaton.hpp:159 */
uint64_t or_instance_seed(uint64_t base, uint32_t n, uint32_t index);       /* experiment.hpp:54 */
void or_expand(uint32_t n, uint32_t k, const uint32_t* delta, const uint64_t* words, size_t count,
               int inverse, uint64_t* out_words, uint32_t* out_cards);     /* bibfs_engine.hpp:345 */
size_t or_lex_sort_dedupe(uint32_t n, uint64_t* words, uint32_t* cards, uint64_t* tags,
                          size_t count);                                    /* set_list.hpp:259 */
void or_sort_card_desc_lex(uint32_t n, uint64_t* words, uint32_t* cards, uint64_t* tags,
                           size_t count);                                   /* set_list.hpp:223 */
size_t or_self_reduce_minimal(uint32_t n, uint64_t* words, uint32_t* cards, size_t count); /* subset_algebra.hpp:179 */
void or_mark(uint32_t n, const uint64_t* a, size_t na, const uint64_t* b, size_t nb, int mode,
             uint8_t* keep);                                               /* subset_algebra.hpp:138-174 */
int or_meet_check(uint32_t n, const uint64_t* a, size_t na, const uint64_t* b, size_t nb); /* :201 */
uint64_t or_trie_node_count(uint32_t n, const uint64_t* words, size_t count, uint32_t min_leaf); /* static_trie.hpp:85-151 */
double or_exp_mark(double as, double bs, double ad, double bd);            /* cost_model.hpp:67 */
int64_t or_power_set_oracle(uint32_t n, uint32_t k, const uint32_t* delta); /* oracle.hpp:17 */

#endif
