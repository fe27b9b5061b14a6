// Lexicographic / (cardinality desc, lex) ordering and deduplication.
//
// Semantics (set_list.hpp:210-265): stable order with the input index as the
// final tie-break, so among equal sets the one that came first survives a
// dedupe — exactly which child's tag (parent, letter) the reference keeps.
// Implementation: LSD radix over the W 64-bit words (least significant word
// first; each pass a stable CUB onesweep radix sort of (word, index) pairs
// restricted to the bit range that actually varies across the list), plus an
// optional final stable pass on (n - card).  The permutation is then applied
// and duplicates dropped in ONE warp-ballot compaction pass (kernels.cu).
#include <cub/cub.cuh>

#include "dev.hpp"
#include "kernels.cuh"
#include "util.cuh"

namespace synchro::dev {

template <int W>
__global__ void or_and_kernel(const u64* __restrict__ words, u64 count,
                              unsigned long long* out /* [W] or, [W] and */) {
  u64 o[W], a[W];
#pragma unroll
  for (int w = 0; w < W; ++w) {
    o[w] = 0;
    a[w] = ~u64{0};
  }
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<u64>(gridDim.x) * blockDim.x) {
#pragma unroll
    for (int w = 0; w < W; ++w) {
      const u64 x = words[i * W + w];
      o[w] |= x;
      a[w] &= x;
    }
  }
#pragma unroll
  for (int w = 0; w < W; ++w) {
    for (int off = 16; off; off >>= 1) {
      o[w] |= __shfl_xor_sync(0xFFFFFFFFu, o[w], off);
      a[w] &= __shfl_xor_sync(0xFFFFFFFFu, a[w], off);
    }
  }
  if ((threadIdx.x & 31) == 0) {
#pragma unroll
    for (int w = 0; w < W; ++w) {
      atomicOr(&out[w], static_cast<unsigned long long>(o[w]));
      atomicAnd(&out[W + w], static_cast<unsigned long long>(a[w]));
    }
  }
}

__global__ void iota_kernel(u32* p, u64 count) {
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<u64>(gridDim.x) * blockDim.x)
    p[i] = static_cast<u32>(i);
}

__global__ void gather_word_kernel(const u64* __restrict__ words, const u32* __restrict__ perm,
                                   u64 count, u32 W, u32 w, u64* __restrict__ keys) {
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<u64>(gridDim.x) * blockDim.x)
    keys[i] = words[static_cast<u64>(perm[i]) * W + w];
}

__global__ void card_key_kernel(const u32* __restrict__ cards, const u32* __restrict__ perm,
                                u64 count, u32 n, u32* __restrict__ keys) {
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<u64>(gridDim.x) * blockDim.x)
    keys[i] = n - cards[perm[i]];
}

const u32* sort_perm(Context& c, const DList& l, bool card_desc) {
  const u64 N = l.size();
  const u32 W = c.W();
  cudaStream_t s = as_stream(c.stream());
  u32* p0 = static_cast<u32*>(c.scratch(2, N * 4));
  u32* p1 = static_cast<u32*>(c.scratch(3, N * 4));
  iota_kernel<<<grid_for(N, 256), 256, 0, s>>>(p0, N);
  if (N <= 1) return p0;

  // Which bits vary across the list, per word (skips constant words/bits).
  std::vector<unsigned long long> oa(2 * W);
  for (u32 w = 0; w < W; ++w) {
    oa[w] = 0;
    oa[W + w] = ~0ull;
  }
  auto* d_oa = static_cast<unsigned long long*>(c.scratch(7, 2 * W * 8));
  c.memcpy_h2d(d_oa, oa.data(), 2 * W * 8);
  SW_DISPATCH_W(W, { or_and_kernel<W><<<grid_for(N, 256, 148 * 4), 256, 0, s>>>(l.words, N, d_oa); });
  SW_CHECK_LAUNCH();
  c.memcpy_d2h(oa.data(), d_oa, 2 * W * 8);

  u64* k0 = static_cast<u64*>(c.scratch(0, N * 8));
  u64* k1 = static_cast<u64*>(c.scratch(1, N * 8));
  cub::DoubleBuffer<u64> keys(k0, k1);
  cub::DoubleBuffer<u32> vals(p0, p1);
  size_t temp_bytes = 0;
  SW_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, temp_bytes, keys, vals, static_cast<int>(N), 0, 64, s));
  void* temp = c.scratch(4, temp_bytes);
  for (int w = static_cast<int>(W) - 1; w >= 0; --w) {
    const u64 varying = oa[w] ^ oa[W + w];
    if (!varying) continue;
    const int begin = __builtin_ctzll(varying);
    const int end = 64 - __builtin_clzll(varying);
    gather_word_kernel<<<grid_for(N, 256), 256, 0, s>>>(l.words, vals.Current(), N, W, w,
                                                        keys.Current());
    SW_CUDA(cub::DeviceRadixSort::SortPairs(temp, temp_bytes, keys, vals, static_cast<int>(N),
                                            begin, end, s));
    c.counters.kernel_launches += 1 + (end - begin + 7) / 8;
  }
  if (card_desc) {
    u32* c0 = reinterpret_cast<u32*>(keys.Current());
    u32* c1 = reinterpret_cast<u32*>(keys.Alternate());
    cub::DoubleBuffer<u32> ck(c0, c1);
    card_key_kernel<<<grid_for(N, 256), 256, 0, s>>>(l.cards, vals.Current(), N, c.n(), ck.Current());
    int bits = 1;
    while ((1u << bits) <= c.n()) ++bits;
    size_t tb = 0;
    SW_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, ck, vals, static_cast<int>(N), 0, bits, s));
    void* t2 = c.scratch(4, std::max(tb, temp_bytes));
    SW_CUDA(cub::DeviceRadixSort::SortPairs(t2, tb, ck, vals, static_cast<int>(N), 0, bits, s));
  }
  SW_CHECK_LAUNCH();
  return vals.Current();
}

std::vector<u64> varying_bits(Context& c, const DList& l) {
  const u32 W = c.W();
  std::vector<unsigned long long> oa(2 * W);
  for (u32 w = 0; w < W; ++w) {
    oa[w] = 0;
    oa[W + w] = ~0ull;
  }
  std::vector<u64> out(W, 0);
  if (l.size() < 2) return out;
  cudaStream_t s = as_stream(c.stream());
  auto* d_oa = static_cast<unsigned long long*>(c.scratch(7, 2 * W * 8));
  c.memcpy_h2d(d_oa, oa.data(), 2 * W * 8);
  SW_DISPATCH_W(W, {
    or_and_kernel<W><<<grid_for(l.size(), 256, 148 * 4), 256, 0, s>>>(l.words, l.size(), d_oa);
  });
  SW_CHECK_LAUNCH();
  c.memcpy_d2h(oa.data(), d_oa, 2 * W * 8);
  for (u32 w = 0; w < W; ++w) out[w] = oa[w] ^ oa[W + w];
  return out;
}

void sort_lex(Context& c, DList& l) {
  if (l.size() <= 1) return;
  const u32* perm = sort_perm(c, l, false);
  compact_flags(c, l, nullptr, perm);
}

void sort_card_desc_lex(Context& c, DList& l) {
  if (l.size() <= 1) return;
  const u32* perm = sort_perm(c, l, true);
  compact_flags(c, l, nullptr, perm);
}

// Cardinality classes only (descending, stable): a radix sort of the card key
// alone (<= 11 bits) instead of the full (card, lex) key — the relaxed DFS
// slice order needs the classes together, not lex order inside them.
void sort_card_desc(Context& c, DList& l) {
  const u64 N = l.size();
  if (N <= 1) return;
  cudaStream_t s = as_stream(c.stream());
  u32* p0 = static_cast<u32*>(c.scratch(2, N * 4));
  u32* p1 = static_cast<u32*>(c.scratch(3, N * 4));
  iota_kernel<<<grid_for(N, 256), 256, 0, s>>>(p0, N);
  u32* k0 = static_cast<u32*>(c.scratch(0, N * 8));
  u32* k1 = static_cast<u32*>(c.scratch(1, N * 8));
  cub::DoubleBuffer<u32> vals(p0, p1), ck(k0, k1);
  card_key_kernel<<<grid_for(N, 256), 256, 0, s>>>(l.cards, vals.Current(), N, c.n(), ck.Current());
  int bits = 1;
  while ((1u << bits) <= c.n()) ++bits;
  size_t tb = 0;
  SW_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, ck, vals, static_cast<int>(N), 0, bits, s));
  void* t = c.scratch(4, tb);
  SW_CUDA(cub::DeviceRadixSort::SortPairs(t, tb, ck, vals, static_cast<int>(N), 0, bits, s));
  SW_CHECK_LAUNCH();
  c.counters.kernel_launches += 2 + (bits + 7) / 8;
  compact_flags(c, l, nullptr, vals.Current());
}

size_t dedupe_sorted(Context& c, DList& l) {
  if (l.size() <= 1) return 0;
  const size_t before = l.size();
  return before - compact_unique(c, l, nullptr);
}

size_t lex_sort_dedupe(Context& c, DList& l) {
  if (l.size() <= 1) return 0;
  const size_t before = l.size();
  const u32* perm = sort_perm(c, l, false);
  return before - compact_unique(c, l, perm);
}

// h := h ++ add.  The histories are only ever read by order-free consumers
// (containment indexes build their own order; card filters and the ledger
// see sets and sizes), so the reference's sorted merge (bibfs_engine.hpp:
// 383-403) is a concatenation here: its size and set are the same.
void merge_sorted(Context& c, DList& h, const DList& add) {
  if (add.empty()) return;
  const size_t total = h.size() + add.size();
  DList m(&c, total, false);
  cudaStream_t s = as_stream(c.stream());
  const u32 W = c.W();
  if (h.size()) {
    SW_CUDA(cudaMemcpyAsync(m.words, h.words, h.size() * W * 8, cudaMemcpyDeviceToDevice, s));
    SW_CUDA(cudaMemcpyAsync(m.cards, h.cards, h.size() * 4, cudaMemcpyDeviceToDevice, s));
  }
  SW_CUDA(cudaMemcpyAsync(m.words + h.size() * W, add.words, add.size() * W * 8, cudaMemcpyDeviceToDevice, s));
  SW_CUDA(cudaMemcpyAsync(m.cards + h.size(), add.cards, add.size() * 4, cudaMemcpyDeviceToDevice, s));
  m.set_size(total);
  h = std::move(m);
}

}  // namespace synchro::dev
