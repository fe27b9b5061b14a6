// Kernel microbenchmarks at HBM scale for the roofline numbers (SURVEY §8(d):
// "2^24 random subsets at the measured frontier density ... expanded under the
// C3/C4 automata").  Inputs are generated on the device (SplitMix64 per set),
// each measured call is bracketed by CUDA events on the context's stream.
#include <algorithm>
#include <vector>

#include "dev.hpp"
#include "kernels.cuh"
#include "util.cuh"

namespace synchro::dev {

namespace {

__device__ __forceinline__ u64 splitmix(u64& s) {
  u64 z = (s += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// Set i draws round(density*n) states uniformly (collisions allowed) from a
// stream seeded by (seed, i % distinct): i and i + distinct are duplicates.
__global__ void random_sets_kernel(u64* words, u32* cards, u64 count, u32 n, u32 W, u32 draws,
                                   u64 seed, u64 distinct) {
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<u64>(gridDim.x) * blockDim.x) {
    u64 st = seed ^ ((i % distinct) * 0xD1B54A32D192ED03ull);
    for (u32 w = 0; w < W; ++w) words[i * W + w] = 0;
    for (u32 d = 0; d < draws; ++d) {
      const u32 q = static_cast<u32>(splitmix(st) % n);
      words[i * W + (q >> 6)] |= state_bit(q);
    }
    u32 c = 0;
    for (u32 w = 0; w < W; ++w) c += __popcll(words[i * W + w]);
    cards[i] = c;
  }
}

DList random_sets(Context& c, u64 count, double density, u64 seed, double dup_fraction) {
  DList l(&c, count, false);
  l.set_size(count);
  const u32 draws = static_cast<u32>(density * c.n() + 0.5);
  u64 distinct = static_cast<u64>(static_cast<double>(count) * (1.0 - dup_fraction));
  if (distinct < 1) distinct = 1;
  random_sets_kernel<<<grid_for(count, 256), 256, 0, as_stream(c.stream())>>>(
      l.words, l.cards, count, c.n(), c.W(), draws, seed, distinct);
  SW_CHECK_LAUNCH();
  c.sync();
  return l;
}

}  // namespace

double bench_expand(Context& c, u64 count, double density, u64 seed, bool inverse, int iters) {
  const DList src = random_sets(c, count, density, seed, 0.0);
  DList out(&c, count * c.k(), false);
  expand(c, src, 0, count, inverse, out);  // warm-up
  c.sync();
  StreamTimer t(c);
  t.start();
  for (int i = 0; i < iters; ++i) expand(c, src, 0, count, inverse, out);
  return t.stop_ms() / iters;
}

double bench_dedupe(Context& c, u64 count, double density, u64 seed, double dup_fraction, int iters,
                    u64* unique_out, bool lex_sort) {
  const DList src = random_sets(c, count, density, seed, dup_fraction);
  // Two warm-up calls (pool growth / first-touch mapping of the list buffers
  // happen there), then the median of `iters` timed calls.
  std::vector<double> ms;
  for (int i = 0; i < iters + 2; ++i) {
    DList l = copy_list(c, src, false);
    c.sync();
    StreamTimer t(c);
    t.start();
    if (lex_sort)
      lex_sort_dedupe(c, l);
    else
      hash_dedupe(c, l);
    const double m = t.stop_ms();
    if (i >= 2) ms.push_back(m);
    if (unique_out) *unique_out = l.size();
  }
  std::sort(ms.begin(), ms.end());
  return ms[ms.size() / 2];
}

}  // namespace synchro::dev
