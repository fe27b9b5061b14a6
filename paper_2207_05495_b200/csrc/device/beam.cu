// One beam level (heuristics.hpp:88-142: sort the preimages by (card desc,
// lex, index), drop adjacent duplicates, keep the first beam_size) in ONE
// launch for small levels: a single CTA stages the level in shared memory,
// bitonic-sorts an index array with the reference's comparator, and writes
// the first `beam` distinct rows (with cards and tags) plus the top card.
// The multi-launch path (CUB radix passes + compaction + host round trips)
// costs ~15 launches and 2 synchronisations per level; small beams (config 2:
// beam = max(64, n) over ~20 levels, twice per solve) are pure launch latency.
// Same output as sort_card_desc_lex + dedupe_sorted + truncate, tags included.
#include "dev.hpp"
#include "kernels.cuh"
#include "util.cuh"

namespace synchro::dev {

namespace {

constexpr int kBeamThreads = 1024;
constexpr size_t kBeamSmem = 200 * 1024;

// a before b in (card desc, lex asc, index asc)
template <int W>
__device__ __forceinline__ bool beam_less(const u64* rows, const u32* cards, u32 a, u32 b) {
  if (cards[a] != cards[b]) return cards[a] > cards[b];
#pragma unroll
  for (int w = 0; w < W; ++w) {
    const u64 x = rows[a * W + w], y = rows[b * W + w];
    if (x != y) return x < y;
  }
  return a < b;
}

template <int W>
__global__ void __launch_bounds__(kBeamThreads) beam_level_kernel(
    const u64* __restrict__ words, const u32* __restrict__ cards, const u64* __restrict__ tags,
    u32 m, u32 m2, u32 beam, u64* __restrict__ ow, u32* __restrict__ oc, u64* __restrict__ ot,
    u32* __restrict__ result) {
  extern __shared__ __align__(16) unsigned char smem[];
  u64* rows = reinterpret_cast<u64*>(smem);
  u32* sc = reinterpret_cast<u32*>(rows + static_cast<size_t>(m) * W);
  u32* idx = sc + m;
  u32* keep = idx + m2;  // exclusive rank among distinct rows
  for (u32 e = threadIdx.x; e < m * W; e += kBeamThreads) rows[e] = words[e];
  for (u32 i = threadIdx.x; i < m; i += kBeamThreads) sc[i] = cards[i];
  for (u32 i = threadIdx.x; i < m2; i += kBeamThreads) idx[i] = i < m ? i : 0xFFFFFFFFu;
  __syncthreads();
  // bitonic sort of idx[0, m2); padding (0xFFFFFFFF) sorts last
  for (u32 size = 2; size <= m2; size <<= 1) {
    for (u32 stride = size >> 1; stride > 0; stride >>= 1) {
      for (u32 t = threadIdx.x; t < m2 / 2; t += kBeamThreads) {
        const u32 lo = 2 * t - (t & (stride - 1));
        const u32 hi = lo + stride;
        const bool up = (lo & size) == 0;
        const u32 a = idx[lo], b = idx[hi];
        bool b_first;
        if (a == 0xFFFFFFFFu) b_first = b != 0xFFFFFFFFu;
        else if (b == 0xFFFFFFFFu) b_first = false;
        else b_first = beam_less<W>(rows, sc, b, a);
        if (b_first == up) {
          idx[lo] = b;
          idx[hi] = a;
        }
      }
      __syncthreads();
    }
  }
  // first of each run of equal rows survives; rank the survivors
  for (u32 p = threadIdx.x; p < m; p += kBeamThreads) {
    bool first = p == 0;
    if (!first) {
      const u32 a = idx[p - 1], b = idx[p];
      first = sc[a] != sc[b];
#pragma unroll
      for (int w = 0; w < W; ++w) first |= rows[a * W + w] != rows[b * W + w];
    }
    keep[p] = first ? 1u : 0u;
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // m <= a few thousand: a serial scan is shorter than a sync tree
    u32 acc = 0;
    for (u32 p = 0; p < m; ++p) {
      const u32 v = keep[p];
      keep[p] = v ? acc : 0xFFFFFFFFu;
      acc += v;
    }
    const u32 out = acc < beam ? acc : beam;
    result[0] = out;
    result[1] = m ? sc[idx[0]] : 0;
  }
  __syncthreads();
  for (u32 p = threadIdx.x; p < m; p += kBeamThreads) {
    const u32 r = keep[p];
    if (r == 0xFFFFFFFFu || r >= beam) continue;
    const u32 s = idx[p];
#pragma unroll
    for (int w = 0; w < W; ++w) ow[static_cast<u64>(r) * W + w] = rows[s * W + w];
    oc[r] = sc[s];
    if (ot) ot[r] = tags[s];
  }
}

}  // namespace

bool beam_level_small(Context& c, DList& next, size_t beam, u32* top_card) {
  const size_t m = next.size();
  if (m == 0 || m > 0xFFFFFFu) return false;
  size_t m2 = 1;
  while (m2 < m) m2 <<= 1;
  const size_t smem = m * c.W() * 8 + m * 4 + m2 * 4 + m2 * 4;
  if (smem > kBeamSmem) return false;
  cudaStream_t s = as_stream(c.stream());
  DList out(&c, std::min(m, beam), next.tagged());
  u32* res = static_cast<u32*>(c.scratch(7, 64));
  SW_DISPATCH_W(c.W(), {
    smem_opt_in(reinterpret_cast<const void*>(beam_level_kernel<W>), static_cast<int>(kBeamSmem));
    beam_level_kernel<W><<<1, kBeamThreads, smem, s>>>(
        next.words, next.cards, next.tagged() ? next.tags : nullptr, static_cast<u32>(m),
        static_cast<u32>(m2), static_cast<u32>(std::min<size_t>(beam, 0xFFFFFFFFu)), out.words,
        out.cards, next.tagged() ? out.tags : nullptr, res);
  });
  SW_CHECK_LAUNCH();
  c.counters.kernel_launches += 1;
  u32 h[2];
  c.memcpy_d2h(h, res, 8);
  out.set_size(h[0]);
  *top_card = h[1];
  next = std::move(out);
  return true;
}

}  // namespace synchro::dev
