/* Search for slowly synchronizing TERNARY automata with n = 5 states (the
 * Roman-type extremal class of config 5: reset threshold (n-1)^2 = 16 over a
 * 3-letter alphabet).  Letter a is fixed to a permutation of the given cycle
 * type (every permutation is conjugate to one of them, so up to relabelling
 * nothing is lost for that type); b and c range over all maps Q -> Q.  Reset
 * threshold by breadth-first search over the power set.  Prints
 * "threshold n d0_a d0_b d0_c d1_a ..." (delta row-major, delta[q*3+x]) for
 * every automaton with threshold >= MIN.  Test-fixture generator only; the
 * thresholds are re-pinned with the reference's power_set_bfs_oracle by
 * make_config5.py.
 *
 * usage: find_ternary MIN CYCLE_TYPE   (CYCLE_TYPE: 5 | 41 | 32 | 311 | 221 | 2111 | 11111)
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define N 5

static int threshold(const int* t0, const int* t1, const int* t2) {
  const uint32_t full = (1u << N) - 1;
  int8_t dist[1 << N];
  uint32_t queue[1 << N];
  memset(dist, -1, sizeof(dist));
  int head = 0, tail = 0;
  dist[full] = 0;
  queue[tail++] = full;
  const int* t[3] = {t0, t1, t2};
  while (head < tail) {
    const uint32_t s = queue[head++];
    if ((s & (s - 1)) == 0) return dist[s];
    for (int x = 0; x < 3; ++x) {
      uint32_t img = 0;
      for (int q = 0; q < N; ++q)
        if (s >> q & 1) img |= 1u << t[x][q];
      if (dist[img] < 0) {
        dist[img] = (int8_t)(dist[s] + 1);
        queue[tail++] = img;
      }
    }
  }
  return -1;
}

int main(int argc, char** argv) {
  const int min = argc > 1 ? atoi(argv[1]) : 16;
  const char* type = argc > 2 ? argv[2] : "5";
  int a[N];
  int q = 0;
  for (const char* p = type; *p; ++p) {  /* consecutive cycles of the given lengths */
    const int len = *p - '0', start = q;
    for (int i = 0; i < len; ++i, ++q) a[q] = (i + 1 < len) ? q + 1 : start;
  }
  if (q != N) return 2;
  int b[N], c[N];
  int total = 0;
  for (int bi = 0; bi < 3125; ++bi) {
    for (int i = 0, v = bi; i < N; ++i, v /= N) b[i] = v % N;
    for (int ci = bi; ci < 3125; ++ci) { /* b <= c: the letter swap b <-> c */
      for (int i = 0, v = ci; i < N; ++i, v /= N) c[i] = v % N;
      const int r = threshold(a, b, c);
      if (r >= min) {
        printf("%d %d", r, N);
        for (int s = 0; s < N; ++s) printf(" %d %d %d", a[s], b[s], c[s]);
        printf("\n");
        ++total;
      }
    }
  }
  fprintf(stderr, "type %s: %d automata with threshold >= %d\n", type, total, min);
  return 0;
}
