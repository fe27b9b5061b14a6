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

// Whole beam search for small beams in ONE persistent CTA: every level's
// preimages (child o = i·k + a: state p is in the child iff δ(p,a) is in
// parent i), the (card desc, lex, index) bitonic sort, first-of-run dedupe,
// truncation to `beam`, the per-level tags written out for the walk back, and
// the stop test (top card == n) — no host round trip per level.
template <int W>
__global__ void __launch_bounds__(kBeamThreads) beam_full_kernel(
    const uint16_t* __restrict__ g_img, u32 n, u32 k, u32 beam, u32 bc, u32 m2,
    u32 max_levels, u64* __restrict__ level_tags, u64* __restrict__ sav, u32* __restrict__ result) {
  extern __shared__ __align__(16) unsigned char smem[];
  const u32 mmax = bc * k;
  u64* cur = reinterpret_cast<u64*>(smem);                          // bc x W
  u64* nxt = cur + static_cast<size_t>(bc) * W;                     // mmax x W
  u32* ccard = reinterpret_cast<u32*>(nxt + static_cast<size_t>(mmax) * W);  // bc
  u32* ncard = ccard + bc;                                          // mmax
  u32* idx = ncard + mmax;                                          // m2
  u32* keep = idx + m2;                                             // m2
  uint16_t* img = reinterpret_cast<uint16_t*>(keep + m2);           // k x n
  __shared__ u32 s_kept, s_done, s_savn, s_same;
  for (u32 i = threadIdx.x; i < k * n; i += kBeamThreads) img[i] = g_img[i];
  for (u32 e = threadIdx.x; e < n * W; e += kBeamThreads) {  // level 0: the singletons
    const u32 q = e / W, w = e % W;
    cur[e] = (q >> 6) == w ? state_bit(q) : 0;
  }
  for (u32 q = threadIdx.x; q < n; q += kBeamThreads) ccard[q] = 1;
  if (threadIdx.x == 0) {
    s_done = 0;
    s_savn = 0xFFFFFFFFu;  // nothing saved yet
  }
  __syncthreads();
  u32 ncur = n, level = 0;
  bool cycle = false;
  while (level < max_levels) {
    ++level;
    const u32 m = ncur * k;
    for (u32 e = threadIdx.x; e < m * W; e += kBeamThreads) {  // preimages, one word each
      const u32 o = e / W, w = e % W, i = o / k, a = o % k;
      const u64* par = cur + static_cast<size_t>(i) * W;
      u64 bits = 0;
      const u32 p0 = 64 * w;
      for (u32 b = 0; b < 64 && p0 + b < n; ++b) {
        const u32 t = img[a * n + p0 + b];
        bits |= ((par[t >> 6] >> (63 - (t & 63))) & 1ull) << (63 - b);
      }
      nxt[e] = bits;
    }
    __syncthreads();
    for (u32 o = threadIdx.x; o < m; o += kBeamThreads) {
      u32 c = 0;
#pragma unroll
      for (int w = 0; w < W; ++w) c += __popcll(nxt[static_cast<size_t>(o) * W + w]);
      ncard[o] = c;
    }
    u32 mp = 1;
    while (mp < m) mp <<= 1;
    for (u32 i = threadIdx.x; i < mp; i += kBeamThreads) idx[i] = i < m ? i : 0xFFFFFFFFu;
    __syncthreads();
    for (u32 size = 2; size <= mp; size <<= 1) {
      for (u32 stride = size >> 1; stride > 0; stride >>= 1) {
        for (u32 t = threadIdx.x; t < mp / 2; t += kBeamThreads) {
          const u32 lo = 2 * t - (t & (stride - 1)), hi = lo + stride;
          const bool up = (lo & size) == 0;
          const u32 x = idx[lo], y = idx[hi];
          bool y_first;
          if (x == 0xFFFFFFFFu) y_first = y != 0xFFFFFFFFu;
          else if (y == 0xFFFFFFFFu) y_first = false;
          else y_first = beam_less<W>(nxt, ncard, y, x);
          if (y_first == up) {
            idx[lo] = y;
            idx[hi] = x;
          }
        }
        __syncthreads();
      }
    }
    for (u32 p = threadIdx.x; p < m; p += kBeamThreads) {
      bool first = p == 0;
      if (!first) {
        const u32 x = idx[p - 1], y = idx[p];
        first = ncard[x] != ncard[y];
#pragma unroll
        for (int w = 0; w < W; ++w) first |= nxt[x * W + w] != nxt[y * W + w];
      }
      keep[p] = first ? 1u : 0u;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      u32 acc = 0;
      for (u32 p = 0; p < m; ++p) {
        const u32 v = keep[p];
        keep[p] = v ? acc : 0xFFFFFFFFu;
        acc += v;
      }
      s_kept = acc < beam ? acc : beam;
      if (m && ncard[idx[0]] == n) s_done = 1;  // the first survivor is Q: a reset word
    }
    __syncthreads();
    const u32 kept = s_kept;
    for (u32 p = threadIdx.x; p < m; p += kBeamThreads) {  // survivors: tags out, rows to cur
      const u32 r = keep[p];
      if (r == 0xFFFFFFFFu || r >= beam) continue;
      const u32 o = idx[p];
      level_tags[static_cast<u64>(level - 1) * beam + r] = (static_cast<u64>(o / k) << 16) | (o % k);
#pragma unroll
      for (int w = 0; w < W; ++w) cur[static_cast<size_t>(r) * W + w] = nxt[static_cast<size_t>(o) * W + w];
      ccard[r] = ncard[o];
    }
    __syncthreads();
    ncur = kept;
    if (s_done) break;
    // A level's kept rows, in their canonical (card desc, lex) order, are a
    // function of the previous level's alone: if they repeat, the search
    // cycles and can never reach Q — the reference would run to its level
    // cap and fail, so stop now (Brent: compare against the level saved at
    // the last power of two).
    if (threadIdx.x == 0) s_same = kept == s_savn ? 1u : 0u;
    __syncthreads();
    if (s_same)
      for (u32 e = threadIdx.x; e < kept * W; e += kBeamThreads)
        if (cur[e] != sav[e]) s_same = 0;
    __syncthreads();
    if (s_same) {
      cycle = true;
      break;
    }
    if ((level & (level - 1)) == 0) {
      for (u32 e = threadIdx.x; e < kept * W; e += kBeamThreads) sav[e] = cur[e];
      if (threadIdx.x == 0) s_savn = kept;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    result[0] = s_done ? level : 0;         // level of the reset word (0: none)
    result[1] = cycle ? 0xFFFFFFFFu : level;  // levels run (all ones: a cycle)
  }
}

}  // namespace

BeamRun beam_full_small(Context& c, size_t beam, u64 level_cap, std::vector<u32>* word) {
  const u32 n = c.n(), k = c.k(), W = c.W();
  if (beam == 0 || beam > 4096) return BeamRun::NotApplicable;
  const size_t bc = std::max<size_t>(n, beam), mmax = bc * k;
  size_t m2 = 1;
  while (m2 < mmax) m2 <<= 1;
  const size_t smem = bc * W * 8 + mmax * W * 8 + bc * 4 + mmax * 4 + m2 * 8 +
                      ((static_cast<size_t>(k) * n * 2 + 15) & ~size_t{15});
  if (mmax > 8192 || smem > kBeamSmem) return BeamRun::NotApplicable;
  // the whole search in one launch while its tags fit 64 MB (a cycling beam
  // stops at the repeat; beam_ibfs's host loop only takes what is left over)
  const u64 max_levels =
      std::min<u64>(level_cap, std::max<u64>(4096, (u64{64} << 20) / (beam * 8)));
  cudaStream_t s = as_stream(c.stream());
  u64* tags = static_cast<u64*>(c.alloc(max_levels * beam * 8));
  u64* sav = static_cast<u64*>(c.alloc(bc * W * 8));
  u32* res = static_cast<u32*>(c.scratch(7, 64));
  SW_DISPATCH_W(c.W(), {
    smem_opt_in(reinterpret_cast<const void*>(beam_full_kernel<W>), static_cast<int>(kBeamSmem));
    beam_full_kernel<W><<<1, kBeamThreads, smem, s>>>(
        static_cast<const uint16_t*>(c.d_img), n, k, static_cast<u32>(beam), static_cast<u32>(bc),
        static_cast<u32>(m2), static_cast<u32>(max_levels), tags, sav, res);
  });
  SW_CHECK_LAUNCH();
  c.counters.kernel_launches += 1;
  u32 h[2];
  c.memcpy_d2h(h, res, 8);
  BeamRun out;
  if (h[0]) {  // walk the tags back from the reset set (index 0 of its level)
    std::vector<u64> t(static_cast<size_t>(h[0]) * beam);
    c.memcpy_d2h(t.data(), tags, t.size() * 8);
    word->clear();
    size_t i = 0;
    for (u32 lvl = h[0]; lvl-- > 0;) {
      const u64 tag = t[static_cast<size_t>(lvl) * beam + i];
      word->push_back(static_cast<u32>(tag & 0xFFFF));
      i = static_cast<size_t>(tag >> 16);
    }
    out = BeamRun::Found;
  } else {
    out = h[1] >= level_cap ? BeamRun::NotFound : BeamRun::NotApplicable;  // out of level room
  }
  c.free(tags);
  c.free(sav);
  return out;
}

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

// ---------------------------------------------------------------- large levels
// A level's KEPT SET — the first `beam` distinct rows in (card desc, lex)
// order — does not depend on the order the rows arrive in, and the next level
// (the preimages of that set) does not depend on the kept rows' order either,
// so the bound (the level at which Q is kept) is fixed by sets alone; only
// the reconstructed word's letters can depend on order.  So instead of a full
// (card desc, lex) sort of ~2·beam rows (≈ 8 radix passes per word): hash
// dedupe (set semantics) → card histogram → the boundary class c* where the
// running count from card n down reaches `beam` → every row with card > c*
// is kept as is, and only the class card == c* is lex-sorted to take its
// first beam − |card > c*| rows.
namespace {
__global__ void card_hist_kernel(const u32* __restrict__ cards, u64 N, u32 n, u32* __restrict__ hist) {
  extern __shared__ u32 sh[];
  for (u32 i = threadIdx.x; i <= n; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < N;
       i += static_cast<u64>(gridDim.x) * blockDim.x)
    atomicAdd(&sh[cards[i]], 1u);
  __syncthreads();
  for (u32 i = threadIdx.x; i <= n; i += blockDim.x)
    if (sh[i]) atomicAdd(&hist[i], sh[i]);
}

__global__ void card_class_kernel(const u32* __restrict__ cards, u64 N, u32 cs,
                                  uint8_t* __restrict__ above, uint8_t* __restrict__ at) {
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < N;
       i += static_cast<u64>(gridDim.x) * blockDim.x) {
    const u32 c = cards[i];
    above[i] = c > cs;
    at[i] = c == cs;
  }
}

__global__ void find_card_kernel(const u32* __restrict__ cards, u64 N, u32 value,
                                 unsigned long long* __restrict__ first) {
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < N;
       i += static_cast<u64>(gridDim.x) * blockDim.x)
    if (cards[i] == value) atomicMin(first, static_cast<unsigned long long>(i));
}
}  // namespace

namespace {
// 8-bit digit of word w0 at bits [shift, shift+8) — the highest varying bits
// of the first word in which the rows differ (bits above are constant).
__global__ void digit_hist_kernel(const u64* __restrict__ words, u64 N, u32 W, u32 w0, u32 shift,
                                  u32* __restrict__ hist) {
  __shared__ u32 sh[256];
  for (u32 i = threadIdx.x; i < 256; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < N;
       i += static_cast<u64>(gridDim.x) * blockDim.x)
    atomicAdd(&sh[(words[i * W + w0] >> shift) & 0xFF], 1u);
  __syncthreads();
  for (u32 i = threadIdx.x; i < 256; i += blockDim.x)
    if (sh[i]) atomicAdd(&hist[i], sh[i]);
}

__global__ void digit_class_kernel(const u64* __restrict__ words, u64 N, u32 W, u32 w0, u32 shift,
                                   u32 bstar, uint8_t* __restrict__ below, uint8_t* __restrict__ at) {
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < N;
       i += static_cast<u64>(gridDim.x) * blockDim.x) {
    const u32 d = static_cast<u32>((words[i * W + w0] >> shift) & 0xFF);
    below[i] = d < bstar;
    at[i] = d == bstar;
  }
}
}  // namespace

// The `need` lexicographically smallest rows of a list of DISTINCT rows, in
// unspecified order (MSD radix select): each round histograms the 8 highest
// varying bits of the first varying word, keeps every row of the buckets
// below the boundary bucket, and recurses into the boundary bucket alone;
// once the remainder fits one CTA it is sorted and truncated there.
void select_lex_smallest(Context& c, DList& l, size_t need, bool distinct) {
  if (l.size() <= need) return;
  cudaStream_t s = as_stream(c.stream());
  const u32 W = c.W();
  std::vector<DList> kept;
  while (true) {
    if (need == 0) break;
    if (l.size() <= need) {
      kept.push_back(std::move(l));
      break;
    }
    u32 t = 0;
    if (distinct && beam_level_small(c, l, need, &t)) {  // (card desc, lex): cards equal here
      kept.push_back(std::move(l));
      break;
    }
    const std::vector<u64> v = varying_bits(c, l);
    u32 w0 = 0;
    while (w0 < W && !v[w0]) ++w0;
    if (w0 == W) {  // all remaining rows equal (only with duplicates): any `need` copies
      truncate(l, need);
      kept.push_back(std::move(l));
      break;
    }
    const int p = 63 - __builtin_clzll(v[w0]);
    const u32 shift = static_cast<u32>(p >= 7 ? p - 7 : 0);
    const u64 N = l.size();
    auto* hist = static_cast<u32*>(c.scratch(7, 256 * 4));
    SW_CUDA(cudaMemsetAsync(hist, 0, 256 * 4, s));
    digit_hist_kernel<<<grid_for(N, 256, 148 * 2), 256, 0, s>>>(l.words, N, W, w0, shift, hist);
    SW_CHECK_LAUNCH();
    std::vector<u32> h(256);
    c.memcpy_d2h(h.data(), hist, 256 * 4);
    size_t cum = 0;
    u32 bstar = 0;
    for (; bstar < 256; ++bstar) {
      if (cum + h[bstar] >= need) break;
      cum += h[bstar];
    }
    auto* below = static_cast<uint8_t*>(c.alloc(N));
    auto* at = static_cast<uint8_t*>(c.alloc(N));
    digit_class_kernel<<<grid_for(N, 256), 256, 0, s>>>(l.words, N, W, w0, shift, bstar, below, at);
    SW_CHECK_LAUNCH();
    c.counters.kernel_launches += 3;
    if (cum) {
      DList lo = copy_list(c, l, l.tagged());
      compact_flags(c, lo, below, nullptr);
      kept.push_back(std::move(lo));
      need -= cum;
    }
    compact_flags(c, l, at, nullptr);
    c.free(below);
    c.free(at);
  }
  size_t total = 0;
  for (const DList& k : kept) total += k.size();
  const bool tagged = l.tagged();
  DList out(&c, total, tagged);
  size_t off = 0;
  for (const DList& k : kept) {
    const size_t cnt = k.size();
    if (!cnt) continue;
    SW_CUDA(cudaMemcpyAsync(out.words + off * W, k.words, cnt * W * 8, cudaMemcpyDeviceToDevice, s));
    SW_CUDA(cudaMemcpyAsync(out.cards + off, k.cards, cnt * 4, cudaMemcpyDeviceToDevice, s));
    if (tagged) SW_CUDA(cudaMemcpyAsync(out.tags + off, k.tags, cnt * 8, cudaMemcpyDeviceToDevice, s));
    off += cnt;
  }
  out.set_size(total);
  l = std::move(out);
}

void beam_select(Context& c, DList& l, size_t beam, u32* top_card, size_t* top_index) {
  const u32 n = c.n();
  cudaStream_t s = as_stream(c.stream());
  hash_dedupe(c, l, /*first_occurrence=*/false);  // any equal row's tag is a valid parent
  const u64 N = l.size();
  *top_card = 0;
  *top_index = 0;
  if (N == 0) return;
  const size_t first_at = (static_cast<size_t>(n) + 2) & ~size_t{1};  // 8-B slot after the bins
  auto* hist = static_cast<u32*>(c.scratch(7, first_at * 4 + 8));
  SW_CUDA(cudaMemsetAsync(hist, 0, (static_cast<size_t>(n) + 1) * 4, s));
  card_hist_kernel<<<grid_for(N, 256, 148 * 2), 256, (n + 1) * 4, s>>>(l.cards, N, n, hist);
  SW_CHECK_LAUNCH();
  std::vector<u32> h(n + 1);
  c.memcpy_d2h(h.data(), hist, (static_cast<size_t>(n) + 1) * 4);
  c.counters.kernel_launches += 1;
  u32 top = 0;
  for (u32 v = n + 1; v-- > 0;)
    if (h[v]) {
      top = v;
      break;
    }
  if (N > beam) {
    u64 cum = 0;
    u32 cs = 0;
    for (u32 v = n + 1; v-- > 0;) {
      if (cum + h[v] >= beam) {
        cs = v;
        break;
      }
      cum += h[v];
    }
    const size_t need = beam - cum;  // rows taken from the boundary class
    auto* above = static_cast<uint8_t*>(c.alloc(N));
    auto* at = static_cast<uint8_t*>(c.scratch(5, N));
    card_class_kernel<<<grid_for(N, 256), 256, 0, s>>>(l.cards, N, cs, above, at);
    SW_CHECK_LAUNCH();
    DList a = copy_list(c, l, true);
    compact_flags(c, a, above, nullptr);
    c.free(above);
    compact_flags(c, l, at, nullptr);
    select_lex_smallest(c, l, need, /*distinct=*/true);  // one card class: lex decides
    DList out(&c, a.size() + l.size(), true);
    const size_t W = c.W();
    for (const DList* src : {&a, &l}) {
      const size_t off = src == &a ? 0 : a.size(), cnt = src->size();
      if (!cnt) continue;
      SW_CUDA(cudaMemcpyAsync(out.words + off * W, src->words, cnt * W * 8, cudaMemcpyDeviceToDevice, s));
      SW_CUDA(cudaMemcpyAsync(out.cards + off, src->cards, cnt * 4, cudaMemcpyDeviceToDevice, s));
      SW_CUDA(cudaMemcpyAsync(out.tags + off, src->tags, cnt * 8, cudaMemcpyDeviceToDevice, s));
    }
    out.set_size(a.size() + l.size());
    l = std::move(out);
    c.counters.kernel_launches += 1;
  }
  *top_card = top;
  if (top == n) {  // Q was kept: its position starts the walk back
    auto* first = reinterpret_cast<unsigned long long*>(hist + first_at);
    const unsigned long long none = ~0ull;
    c.memcpy_h2d(first, &none, 8);
    find_card_kernel<<<grid_for(l.size(), 256), 256, 0, s>>>(l.cards, l.size(), n, first);
    SW_CHECK_LAUNCH();
    unsigned long long pos = 0;
    c.memcpy_d2h(&pos, first, 8);
    *top_index = static_cast<size_t>(pos);
    c.counters.kernel_launches += 1;
  }
}

// The first k rows of l in (card desc, lex) order — as a multiset, duplicates
// counted like the reference's slice of its sorted level (dfs_phase.hpp:107-110)
// — without sorting l: card histogram → boundary card → radix select inside the
// boundary class.  Untagged copy, unspecified order; l is untouched.
DList top_card_desc_lex(Context& c, const DList& l, size_t k) {
  const u32 n = c.n();
  const u64 N = l.size();
  cudaStream_t s = as_stream(c.stream());
  if (N <= k) return copy_list(c, l, false);
  auto* hist = static_cast<u32*>(c.scratch(7, (static_cast<size_t>(n) + 1) * 4));
  SW_CUDA(cudaMemsetAsync(hist, 0, (static_cast<size_t>(n) + 1) * 4, s));
  card_hist_kernel<<<grid_for(N, 256, 148 * 2), 256, (n + 1) * 4, s>>>(l.cards, N, n, hist);
  SW_CHECK_LAUNCH();
  std::vector<u32> h(n + 1);
  c.memcpy_d2h(h.data(), hist, (static_cast<size_t>(n) + 1) * 4);
  u64 cum = 0;
  u32 cs = 0;
  for (u32 v = n + 1; v-- > 0;) {
    if (cum + h[v] >= k) {
      cs = v;
      break;
    }
    cum += h[v];
  }
  auto* above = static_cast<uint8_t*>(c.alloc(N));
  auto* at = static_cast<uint8_t*>(c.alloc(N));
  card_class_kernel<<<grid_for(N, 256), 256, 0, s>>>(l.cards, N, cs, above, at);
  SW_CHECK_LAUNCH();
  DList a = copy_list(c, l, false);
  compact_flags(c, a, above, nullptr);
  DList e = copy_list(c, l, false);
  compact_flags(c, e, at, nullptr);
  c.free(above);
  c.free(at);
  select_lex_smallest(c, e, k - cum, /*distinct=*/false);
  const size_t W = c.W();
  DList out(&c, a.size() + e.size(), false);
  if (a.size()) {
    c.memcpy_d2d(out.words, a.words, a.size() * W * 8);
    c.memcpy_d2d(out.cards, a.cards, a.size() * 4);
  }
  if (e.size()) {
    c.memcpy_d2d(out.words + a.size() * W, e.words, e.size() * W * 8);
    c.memcpy_d2d(out.cards + a.size(), e.cards, e.size() * 4);
  }
  out.set_size(a.size() + e.size());
  c.counters.kernel_launches += 2;
  return out;
}

}  // namespace synchro::dev
