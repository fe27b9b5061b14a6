/* Exhaustive search for slowly synchronizing binary automata (the Černý / Kari /
 * Roman extremal class of config 5) with n <= 6 states: every pair of maps
 * a, b : Q -> Q, reset threshold by breadth-first search over the power set.
 * Prints "threshold n d0_a d0_b d1_a d1_b ..." (delta row-major, delta[q*2+x])
 * for every automaton with threshold >= MIN.  Test-fixture generator only;
 * thresholds are re-pinned with the reference's power_set_bfs_oracle by
 * make_slow.py.
 *
 * usage: find_slow N MIN [PART PARTS]   (PART of PARTS slices of the first map)
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static int threshold(int n, const int* a, const int* b) {
  const uint32_t full = (1u << n) - 1;
  static int16_t dist[1 << 8];
  static uint32_t queue[1 << 8];
  memset(dist, -1, sizeof(dist));
  int head = 0, tail = 0;
  dist[full] = 0;
  queue[tail++] = full;
  while (head < tail) {
    const uint32_t s = queue[head++];
    if ((s & (s - 1)) == 0) return dist[s];
    for (int x = 0; x < 2; ++x) {
      const int* t = x ? b : a;
      uint32_t img = 0;
      for (int q = 0; q < n; ++q)
        if (s >> q & 1) img |= 1u << t[q];
      if (dist[img] < 0) {
        dist[img] = dist[s] + 1;
        queue[tail++] = img;
      }
    }
  }
  return -1; /* not synchronizing */
}

int main(int argc, char** argv) {
  if (argc < 3) return 2;
  const int n = atoi(argv[1]), min = atoi(argv[2]);
  const long part = argc > 4 ? atol(argv[3]) : 0, parts = argc > 4 ? atol(argv[4]) : 1;
  if (n < 2 || n > 6) return 2;
  long maps = 1;
  for (int i = 0; i < n; ++i) maps *= n;
  int a[8], b[8];
  for (long ia = part; ia < maps; ia += parts) {
    long x = ia;
    for (int q = 0; q < n; ++q, x /= n) a[q] = (int)(x % n);
    for (long ib = ia; ib < maps; ++ib) { /* unordered letter pairs */
      long y = ib;
      for (int q = 0; q < n; ++q, y /= n) b[q] = (int)(y % n);
      const int r = threshold(n, a, b);
      if (r >= min) {
        printf("%d %d", r, n);
        for (int q = 0; q < n; ++q) printf(" %d %d", a[q], b[q]);
        printf("\n");
      }
    }
  }
  return 0;
}
