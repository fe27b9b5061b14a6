/* Local search for slowly synchronizing binary automata at n = 7..12 (config 5's
 * "slowly synchronizing series" beyond the exhaustive n <= 6 classes of
 * find_slow.c): random restarts, one transition changed per move, a move kept
 * when the reset threshold (breadth-first search over the power set) does not
 * drop.  Prints "threshold n d0_a d0_b d1_a d1_b ..." for the best automaton
 * found.  Test-fixture generator only; the threshold is re-pinned with the
 * reference's power_set_bfs_oracle by make_config5.py.
 *
 * usage: climb_slow N RESTARTS MOVES SEED
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static uint64_t rng;
static uint64_t next(void) {  /* SplitMix64 (util.hpp:41-67 style) */
  uint64_t z = (rng += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static int threshold(int n, const int* d) {
  const uint32_t full = (1u << n) - 1;
  static int16_t dist[1 << 12];
  static uint32_t queue[1 << 12];
  memset(dist, -1, sizeof(int16_t) << n);
  int head = 0, tail = 0;
  dist[full] = 0;
  queue[tail++] = full;
  while (head < tail) {
    const uint32_t s = queue[head++];
    if ((s & (s - 1)) == 0) return dist[s];
    for (int x = 0; x < 2; ++x) {
      uint32_t img = 0;
      for (int q = 0; q < n; ++q)
        if (s >> q & 1) img |= 1u << d[2 * q + x];
      if (dist[img] < 0) {
        dist[img] = (int16_t)(dist[s] + 1);
        queue[tail++] = img;
      }
    }
  }
  return -1;
}

int main(int argc, char** argv) {
  const int n = atoi(argv[1]), restarts = atoi(argv[2]), moves = atoi(argv[3]);
  rng = strtoull(argv[4], NULL, 10);
  int best[24], best_r = -1, d[24];
  for (int t = 0; t < restarts; ++t) {
    int r;
    do {
      for (int i = 0; i < 2 * n; ++i) d[i] = (int)(next() % n);
      r = threshold(n, d);
    } while (r < 0);
    for (int m = 0; m < moves; ++m) {
      const int i = (int)(next() % (2 * n)), old = d[i];
      d[i] = (int)(next() % n);
      const int r2 = threshold(n, d);
      if (r2 >= r) r = r2; else d[i] = old;
    }
    if (r > best_r) {
      best_r = r;
      memcpy(best, d, sizeof(int) * 2 * n);
    }
  }
  printf("%d %d", best_r, n);
  for (int i = 0; i < 2 * n; ++i) printf(" %d", best[i]);
  printf("\n");
  return 0;
}
