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

#include <cstdlib>
#include <string>

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

static const u32* sort_perm_lsd(Context& c, const DList& l, bool card_desc) {
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

// ---- packed-prefix radix order
// The sort key of row i is (n - card_i if card_desc, word 0, word 1, ...)
// compared MSB first.  Only bits that vary across the list matter, so the
// varying bit ranges (or_and_kernel) are concatenated MSB-first into ONE
// 64-bit prefix key, which is radix-sorted once (stable, index tie-break).
// Rows whose prefix ties with a neighbour's ("members") are then refined on
// their own: stable LSD passes over the words the prefix did not cover,
// followed by a stable pass on the prefix, and written back into the
// members' positions (a tie group occupies consecutive positions, and the
// members stay in position order, so group order is kept).
struct KeyField {
  int word;   // -1: the cardinality field (n - card)
  int shift;  // right shift applied to the source
  int len;    // bits taken
};
constexpr int kMaxFields = 17;
struct PackSpec {
  KeyField f[kMaxFields];
  int nf;
  u32 n;
};

template <int W>
__global__ void pack_key_kernel(const u64* __restrict__ words, const u32* __restrict__ cards,
                                u64 count, PackSpec spec, u64* __restrict__ keys,
                                u32* __restrict__ idx) {
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<u64>(gridDim.x) * blockDim.x) {
    u64 key = 0;
    for (int f = 0; f < spec.nf; ++f) {
      const KeyField kf = spec.f[f];
      const u64 src = kf.word < 0 ? static_cast<u64>(spec.n - cards[i]) : words[i * W + kf.word];
      const u64 v = (src >> kf.shift) & (kf.len == 64 ? ~u64{0} : ((u64{1} << kf.len) - 1));
      key = kf.len == 64 ? v : ((key << kf.len) | v);
    }
    keys[i] = key;
    idx[i] = static_cast<u32>(i);
  }
}

__global__ void tie_flags_kernel(const u64* __restrict__ keys, u64 count, uint8_t* __restrict__ flag) {
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<u64>(gridDim.x) * blockDim.x) {
    const u64 k = keys[i];
    flag[i] = (i > 0 && keys[i - 1] == k) || (i + 1 < count && keys[i + 1] == k);
  }
}

// members: mv[j] = perm[pos[j]], mk[j] = keys[pos[j]], slot[j] = j
__global__ void member_init_kernel(const u32* __restrict__ pos, const u32* __restrict__ perm,
                                   const u64* __restrict__ keys, u64 m, u32* __restrict__ mv,
                                   u64* __restrict__ mk, u32* __restrict__ slot) {
  for (u64 j = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; j < m;
       j += static_cast<u64>(gridDim.x) * blockDim.x) {
    const u32 p = pos[j];
    mv[j] = perm[p];
    mk[j] = keys[p];
    slot[j] = static_cast<u32>(j);
  }
}

__global__ void member_word_kernel(const u64* __restrict__ words, const u32* __restrict__ mv,
                                   const u32* __restrict__ slot, u64 m, u32 W, u32 w,
                                   u64* __restrict__ out) {
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < m;
       i += static_cast<u64>(gridDim.x) * blockDim.x)
    out[i] = words[static_cast<u64>(mv[slot[i]]) * W + w];
}

__global__ void member_key_kernel(const u64* __restrict__ mk, const u32* __restrict__ slot, u64 m,
                                  u64* __restrict__ out) {
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < m;
       i += static_cast<u64>(gridDim.x) * blockDim.x)
    out[i] = mk[slot[i]];
}

__global__ void member_scatter_kernel(const u32* __restrict__ pos, const u32* __restrict__ mv,
                                      const u32* __restrict__ slot, u64 m, u32* __restrict__ perm) {
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < m;
       i += static_cast<u64>(gridDim.x) * blockDim.x)
    perm[pos[i]] = mv[slot[i]];
}

static const u32* sort_perm_prefix(Context& c, const DList& l, bool card_desc) {
  const u64 N = l.size();
  const u32 W = c.W();
  cudaStream_t s = as_stream(c.stream());
  u32* p0 = static_cast<u32*>(c.scratch(2, N * 4));
  u32* p1 = static_cast<u32*>(c.scratch(3, N * 4));
  if (N <= 1) {
    iota_kernel<<<grid_for(N, 256), 256, 0, s>>>(p0, N);
    return p0;
  }
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

  // Prefix layout: [n - card] [varying bits of word 0] [word 1] ... up to 64 bits.
  PackSpec spec{};
  spec.n = c.n();
  int total = 0;
  if (card_desc) {
    int bits = 1;
    while ((1u << bits) <= c.n()) ++bits;
    spec.f[spec.nf++] = KeyField{-1, 0, bits};
    total = bits;
  }
  u32 rest_from = W;  // first word not fully covered by the prefix
  for (u32 w = 0; w < W; ++w) {
    const u64 varying = oa[w] ^ oa[W + w];
    if (!varying) continue;
    const int begin = __builtin_ctzll(varying);
    const int end = 64 - __builtin_clzll(varying);
    const int room = 64 - total;
    if (room == 0 || spec.nf == kMaxFields) {
      rest_from = w;
      break;
    }
    const int take = std::min(room, end - begin);
    spec.f[spec.nf++] = KeyField{static_cast<int>(w), end - take, take};
    total += take;
    if (take < end - begin) {
      rest_from = w;
      break;
    }
  }
  bool has_rest = false;
  for (u32 w = rest_from; w < W; ++w) has_rest |= (oa[w] ^ oa[W + w]) != 0;

  u64* k0 = static_cast<u64*>(c.scratch(0, N * 8));
  u64* k1 = static_cast<u64*>(c.scratch(1, N * 8));
  SW_DISPATCH_W(W, {
    pack_key_kernel<W><<<grid_for(N, 256), 256, 0, s>>>(l.words, l.cards, N, spec, k0, p0);
  });
  SW_CHECK_LAUNCH();
  cub::DoubleBuffer<u64> keys(k0, k1);
  cub::DoubleBuffer<u32> vals(p0, p1);
  size_t temp_bytes = 0;
  SW_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, temp_bytes, keys, vals, static_cast<int>(N), 0, 64, s));
  void* temp = c.scratch(4, temp_bytes);
  if (total > 0)
    SW_CUDA(cub::DeviceRadixSort::SortPairs(temp, temp_bytes, keys, vals, static_cast<int>(N), 0,
                                            total, s));
  c.counters.kernel_launches += 2 + (total + 7) / 8;
  SW_CHECK_LAUNCH();
  if (!has_rest) return vals.Current();

  // ---- refine the prefix-tie groups
  u32* perm = vals.Current();
  auto* flag = static_cast<uint8_t*>(c.alloc(N));
  tie_flags_kernel<<<grid_for(N, 256), 256, 0, s>>>(keys.Current(), N, flag);
  u32* pos = static_cast<u32*>(c.alloc(N * 4));
  auto* d_m = static_cast<int*>(c.alloc(sizeof(int)));
  size_t sel_bytes = 0;
  cub::CountingInputIterator<u32> it(0);
  SW_CUDA(cub::DeviceSelect::Flagged(nullptr, sel_bytes, it, flag, pos, d_m, static_cast<int>(N), s));
  void* sel_temp = c.alloc(sel_bytes);
  SW_CUDA(cub::DeviceSelect::Flagged(sel_temp, sel_bytes, it, flag, pos, d_m, static_cast<int>(N), s));
  int m = 0;
  c.memcpy_d2h(&m, d_m, sizeof(int));
  c.free(sel_temp);
  c.free(d_m);
  c.counters.kernel_launches += 3;
  if (m > 0) {
    const u64 M = static_cast<u64>(m);
    auto* mv = static_cast<u32*>(c.alloc(M * 4));
    auto* mk = static_cast<u64*>(c.alloc(M * 8));
    auto* s0 = static_cast<u32*>(c.alloc(M * 4));
    auto* s1 = static_cast<u32*>(c.alloc(M * 4));
    auto* q0 = static_cast<u64*>(c.alloc(M * 8));
    auto* q1 = static_cast<u64*>(c.alloc(M * 8));
    member_init_kernel<<<grid_for(M, 256), 256, 0, s>>>(pos, perm, keys.Current(), M, mv, mk, s0);
    cub::DoubleBuffer<u64> mkeys(q0, q1);
    cub::DoubleBuffer<u32> slots(s0, s1);
    size_t tb = 0;
    SW_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, mkeys, slots, m, 0, 64, s));
    void* t2 = c.alloc(tb);
    for (int w = static_cast<int>(W) - 1; w >= static_cast<int>(rest_from); --w) {
      const u64 varying = oa[w] ^ oa[W + w];
      if (!varying) continue;
      const int begin = __builtin_ctzll(varying);
      const int end = 64 - __builtin_clzll(varying);
      member_word_kernel<<<grid_for(M, 256), 256, 0, s>>>(l.words, mv, slots.Current(), M, W,
                                                          static_cast<u32>(w), mkeys.Current());
      SW_CUDA(cub::DeviceRadixSort::SortPairs(t2, tb, mkeys, slots, m, begin, end, s));
      c.counters.kernel_launches += 1 + (end - begin + 7) / 8;
    }
    member_key_kernel<<<grid_for(M, 256), 256, 0, s>>>(mk, slots.Current(), M, mkeys.Current());
    if (total > 0) SW_CUDA(cub::DeviceRadixSort::SortPairs(t2, tb, mkeys, slots, m, 0, total, s));
    member_scatter_kernel<<<grid_for(M, 256), 256, 0, s>>>(pos, mv, slots.Current(), M, perm);
    SW_CHECK_LAUNCH();
    c.counters.kernel_launches += 3 + (total + 7) / 8;
    for (void* q : {static_cast<void*>(mv), static_cast<void*>(mk), static_cast<void*>(s0),
                    static_cast<void*>(s1), static_cast<void*>(q0), static_cast<void*>(q1), t2})
      c.free(q);
  }
  c.free(pos);
  c.free(flag);
  return perm;
}

const u32* sort_perm(Context& c, const DList& l, bool card_desc) {
  static const int mode = [] {
    const char* e = std::getenv("SYNCHRO_SORT_PREFIX");
    if (!e) return 0;
    return std::string(e) == "card" ? 1 : (std::string(e) == "all" ? 2 : 0);
  }();
  if (mode == 2 || (mode == 1 && card_desc)) return sort_perm_prefix(c, l, card_desc);
  return sort_perm_lsd(c, l, card_desc);
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

__global__ void concat_kernel_dummy() {}

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
  // Disjoint sorted inputs: a stable lex sort of the concatenation is their merge.
  sort_lex(c, m);
  h = std::move(m);
}

}  // namespace synchro::dev
