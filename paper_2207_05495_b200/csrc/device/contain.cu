// Subset-containment on the GPU: the B200 replacement for the reference's
// MarkSupersets recursion (subset_algebra.hpp:55-125, Alg. 2) and for the
// static-trie joint query (static_trie.hpp:153-188).
//
// The reference splits a lex-sorted A on bit d by binary search and
// partitions B in place, recursively — inherently sequential.  Here the
// lex-sorted unique A becomes an explicit binary radix (Patricia) tree built
// in parallel (Karras, HPG 2012: internal node i is found from the longest
// common prefixes of neighbouring keys by binary search, no inter-thread
// communication), each node annotated with its subtree's min cardinality.
// A query y walks the tree depth-first:
//   * a node's keys agree on bits < lcp; bits [d, lcp) of that common prefix
//     must lie in y (else the subtree is dead);
//   * at the split bit L the 0-child is always admissible, the 1-child only if
//     y has state L (exactly the reference's "ones side recurses with B_1");
//   * subtrees whose min cardinality exceeds |y| (|y|-1 for proper) are cut —
//     the reference's per-pair card filter lifted to whole subtrees;
//   * ranges of <= kScanKeys keys are scanned (warp-cooperatively) — unless the
//     range's AND mask (states every key of it holds) has a state outside y.
// The marked set {y : exists x in A, x ⊆ y (x ⊊ y)} does not depend on the
// traversal order, so sizes match the reference bit-exactly.
#include <cub/cub.cuh>

#include <algorithm>
#include <atomic>
#include <cstdlib>

#include "dev.hpp"
#include "kernels.cuh"
#include "util.cuh"
#include "../progress.hpp"

namespace synchro::dev {

struct __align__(32) Node {
  u32 first, last;  // key range [first, last]
  u32 split;        // left = [first, split], right = [split+1, last]
  uint16_t lcp;     // first bit where the range's keys differ
  uint16_t minc;    // min cardinality in the range
  u64 window;       // bits [lcp-64, lcp) of the range's keys (common prefix tail)
  u64 pad;
};

// One 256-bit load per node (LDG.E.ENL2.256 on sm_100a): a node visit is one
// L1 wavefront instead of two 128-bit ones (the traversal is L1-bound).
__device__ __forceinline__ Node load_node(const Node* p) {
  unsigned long long w0, w1, w2, w3;
  asm("ld.global.nc.v4.u64 {%0,%1,%2,%3}, [%4];"
      : "=l"(w0), "=l"(w1), "=l"(w2), "=l"(w3)
      : "l"(p));
  Node nd;
  nd.first = static_cast<u32>(w0);
  nd.last = static_cast<u32>(w0 >> 32);
  nd.split = static_cast<u32>(w1);
  nd.lcp = static_cast<uint16_t>(w1 >> 32);
  nd.minc = static_cast<uint16_t>(w1 >> 48);
  nd.window = w2;
  nd.pad = w3;
  return nd;
}

// Bits [e-64, e) of an MSB-first bit string, right-aligned (bit e-1 at the
// LSB; positions < 0 read as 0).  `at(w)` returns word w.
template <class At>
__device__ __forceinline__ u64 window_before(At at, int e) {
  const int q = e >> 6, r = e & 63;
  const u64 hi = q > 0 ? at(q - 1) : 0;
  if (r == 0) return hi;
  return (hi << r) | (at(q) >> (64 - r));
}


constexpr u32 kLeafBit = 0x80000000u;

template <int W>
__device__ __forceinline__ int key_delta(const u64* __restrict__ A, long long N, long long i,
                                         long long j) {
  if (j < 0 || j >= N) return -1;
#pragma unroll
  for (int w = 0; w < W; ++w) {
    const u64 x = A[i * W + w] ^ A[j * W + w];
    if (x) return w * 64 + __clzll(x);
  }
  return W * 64;
}

template <int W>
__global__ void karras_kernel(const u64* __restrict__ A, u32 N, Node* __restrict__ nodes,
                              u32* __restrict__ parent_int, u32* __restrict__ parent_leaf) {
  const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (i >= static_cast<long long>(N) - 1) return;
  const int dn = key_delta<W>(A, N, i, i + 1), dp = key_delta<W>(A, N, i, i - 1);
  const int d = dn > dp ? 1 : -1;
  const int dmin = dn > dp ? dp : dn;
  long long lmax = 2;
  while (key_delta<W>(A, N, i, i + lmax * d) > dmin) lmax <<= 1;
  long long l = 0;
  for (long long t = lmax >> 1; t >= 1; t >>= 1)
    if (key_delta<W>(A, N, i, i + (l + t) * d) > dmin) l += t;
  const long long j = i + l * d;
  const int dnode = key_delta<W>(A, N, i, j);
  long long s = 0, t = l;
  do {
    t = (t + 1) >> 1;
    if (key_delta<W>(A, N, i, i + (s + t) * d) > dnode) s += t;
  } while (t > 1);
  const long long gamma = i + s * d + (d < 0 ? -1 : 0);
  const u32 first = static_cast<u32>(i < j ? i : j), last = static_cast<u32>(i < j ? j : i);
  Node nd;
  nd.first = first;
  nd.last = last;
  nd.split = static_cast<u32>(gamma);
  nd.lcp = static_cast<uint16_t>(dnode);
  nd.minc = 0xFFFF;
  const u64* key = A + static_cast<long long>(first) * W;
  nd.window = window_before([&](int w) { return key[w]; }, dnode);
  nd.pad = 0;
  nodes[i] = nd;
  if (first == gamma) parent_leaf[gamma] = static_cast<u32>(i);
  else parent_int[gamma] = static_cast<u32>(i);
  if (last == gamma + 1) parent_leaf[gamma + 1] = static_cast<u32>(i);
  else parent_int[gamma + 1] = static_cast<u32>(i);
}

// Filter words of a set: its relabelled word 0 (the index's first 64 states
// in its state order) and its OR-fold (state q -> bit q mod 64).  Both are
// monotone, so x ⊆ y implies sig(x) ⊆ sig(y) word by word: a one-word test
// per pair rejects almost every non-containment (the fold for sparse sets, word
// 0 for dense queries against a FreqDesc index), and only survivors are
// checked on their full rows.
template <int W>
__device__ __forceinline__ ulonglong2 filter_words(const u64 (&x)[W]) {
  u64 f = 0;
#pragma unroll
  for (int w = 0; w < W; ++w) f |= x[w];
  return make_ulonglong2(x[0], f);
}
__device__ __forceinline__ bool filter_pass(ulonglong2 x, ulonglong2 y) {
  return ((x.x & ~y.x) | (x.y & ~y.y)) == 0;
}

// Bottom-up min cardinality: the second child to arrive at a node finishes it.
// Nodes small enough to be scanned (<= small keys) also get the AND of their
// keys: a query lacking one of those states cannot contain any of them, so the
// scan is skipped (measured at n=300: 49% of meet/DFS scans, 61% of
// self-reduction scans).  The AND mask is reduced to its filter words, kept in
// the node itself (window, pad: a scanned node never uses its prefix window),
// so the skip needs no load beyond the node.
template <int W>
__global__ void mincard_kernel(const u32* __restrict__ card, const u64* __restrict__ keys, u32 N,
                               Node* nodes, const u32* __restrict__ parent_int,
                               const u32* __restrict__ parent_leaf, u32* arrivals, u64* andm,
                               u32 small) {
  const u32 leaf = blockIdx.x * blockDim.x + threadIdx.x;
  if (leaf >= N) return;
  u32 p = parent_leaf[leaf];
  while (true) {
    __threadfence();
    if (atomicAdd(&arrivals[p], 1u) == 0) return;
    __threadfence();
    volatile Node* vn = nodes;
    const u32 first = vn[p].first, last = vn[p].last, split = vn[p].split;
    const u32 lm = (split == first) ? card[first] : vn[split].minc;
    const u32 rm = (split + 1 == last) ? card[last] : vn[split + 1].minc;
    vn[p].minc = static_cast<uint16_t>(lm < rm ? lm : rm);
    if (last - first + 1 <= small) {
      volatile u64* va = andm;
#pragma unroll
      for (int w = 0; w < W; ++w) {
        const u64 l = split == first ? keys[static_cast<u64>(first) * W + w]
                                     : va[static_cast<u64>(split) * W + w];
        const u64 r = split + 1 == last ? keys[static_cast<u64>(last) * W + w]
                                        : va[static_cast<u64>(split + 1) * W + w];
        va[static_cast<u64>(p) * W + w] = l & r;
      }
      u64 m[W];
#pragma unroll
      for (int w = 0; w < W; ++w) m[w] = va[static_cast<u64>(p) * W + w];
      const ulonglong2 f = filter_words<W>(m);
      vn[p].window = f.x;
      vn[p].pad = f.y;
    }
    if (p == 0) return;
    p = parent_int[p];
  }
}

constexpr u32 kScanKeys = 16;  // nodes of <= this many keys are scanned, not descended

ContainIndex build_index(Context& c, const DList& a) {
  ContainIndex ix;
  ix.ctx = &c;
  ix.count = a.size();
  if (a.size() < 2) return ix;
  const u32 N = static_cast<u32>(a.size());
  cudaStream_t s = as_stream(c.stream());
  Node* nodes = static_cast<Node*>(c.alloc((N - 1) * sizeof(Node)));
  u32* pint = static_cast<u32*>(c.alloc(static_cast<size_t>(N) * 4));
  u32* pleaf = static_cast<u32*>(c.alloc(static_cast<size_t>(N) * 4));
  u32* arr = static_cast<u32*>(c.alloc(static_cast<size_t>(N) * 4));
  SW_CUDA(cudaMemsetAsync(arr, 0, static_cast<size_t>(N) * 4, s));
  SW_DISPATCH_W(c.W(), { karras_kernel<W><<<(N + 255) / 256, 256, 0, s>>>(a.words, N, nodes, pint, pleaf); });
  u64* andm = static_cast<u64*>(c.alloc(static_cast<size_t>(N - 1) * c.W() * 8));  // build only
  SW_DISPATCH_W(c.W(), {
    mincard_kernel<W><<<(N + 255) / 256, 256, 0, s>>>(a.cards, a.words, N, nodes, pint, pleaf,
                                                       arr, andm, kScanKeys);
  });
  SW_CHECK_LAUNCH();
  c.counters.kernel_launches += 2;
  c.free(andm);
  c.free(pint);
  c.free(pleaf);
  c.free(arr);
  ix.nodes = nodes;
  return ix;
}

// ---------------------------------------------------------------------------
// Query-side layout.  Both sides of a query are private copies (the index's
// relabelled sorted keys, the relabelled queries), so they use a padded row
// of P = even(W+1) words with the cardinality stored in word W: a row and its
// card arrive in P/2 16-byte vector loads.  (The L1/TEX pipe, not DRAM, is
// what bounds the traversal — ncu: 92% L1/TEX throughput, 99% L2 hit.)
template <int W>
struct Row {
  static constexpr int P = (W + 2) & ~1;
};

template <int W>
__device__ __forceinline__ void load_row(const u64* __restrict__ base, u64 idx, u64 (&x)[W],
                                         u32& card) {
  constexpr int P = Row<W>::P;
  const ulonglong2* p = reinterpret_cast<const ulonglong2*>(base + idx * P);
#pragma unroll
  for (int i = 0; i < P / 2; ++i) {
    const ulonglong2 v = __ldg(p + i);
    if (2 * i < W) x[2 * i] = v.x;
    if (2 * i == W) card = static_cast<u32>(v.x);
    if (2 * i + 1 < W) x[2 * i + 1] = v.y;
    if (2 * i + 1 == W) card = static_cast<u32>(v.y);
  }
}

template <int W>
__device__ __forceinline__ bool is_subset(const u64 (&x)[W], const u64 (&y)[W]) {
  u64 acc = 0;
#pragma unroll
  for (int w = 0; w < W; ++w) acc |= x[w] & ~y[w];
  return acc == 0;
}

// Relabel states (bit q -> bit pos[q]) and write rows in the padded layout
// (PAD) or the plain W-word layout + card array.
template <int W, bool PAD>
__global__ void relabel_kernel(const u64* __restrict__ src, const u32* __restrict__ scard, u64 count,
                               u32 n, const uint16_t* __restrict__ g_pos, u64* __restrict__ dst,
                               u32* __restrict__ dcard, ulonglong2* __restrict__ dsig) {
  extern __shared__ uint16_t s_pos[];
  for (u32 q = threadIdx.x; q < n; q += blockDim.x) s_pos[q] = g_pos[q];
  __syncthreads();
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<u64>(gridDim.x) * blockDim.x) {
    u64 acc[W];
#pragma unroll
    for (int w = 0; w < W; ++w) acc[w] = 0;
#pragma unroll
    for (int w = 0; w < W; ++w) {
      u64 bits = src[i * W + w];
      while (bits) {
        const int b = __clzll(bits);
        bits &= ~(u64{1} << (63 - b));
        const u32 t = s_pos[w * 64 + b];
        const u64 m = u64{1} << (63 - (t & 63));
#pragma unroll
        for (int x = 0; x < W; ++x) acc[x] |= (static_cast<u32>(x) == (t >> 6)) ? m : 0;
      }
    }
    if (PAD) {
      constexpr int P = Row<W>::P;
#pragma unroll
      for (int w = 0; w < P; ++w) dst[i * P + w] = w < W ? acc[w] : (w == W ? scard[i] : 0);
      dsig[i] = filter_words<W>(acc);
    } else {
#pragma unroll
      for (int w = 0; w < W; ++w) dst[i * W + w] = acc[w];
      dcard[i] = scard[i];
    }
  }
}

// Plain sorted rows -> padded rows.
template <int W>
__global__ void pad_kernel(const u64* __restrict__ src, const u32* __restrict__ scard, u64 count,
                           u64* __restrict__ dst, ulonglong2* __restrict__ dsig) {
  constexpr int P = Row<W>::P;
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<u64>(gridDim.x) * blockDim.x) {
    u64 x[W];
#pragma unroll
    for (int w = 0; w < W; ++w) x[w] = src[i * W + w];
#pragma unroll
    for (int w = 0; w < P; ++w) dst[i * P + w] = w < W ? x[w] : (w == W ? scard[i] : 0);
    dsig[i] = filter_words<W>(x);
  }
}

// ---------------------------------------------------------------------------
// Warp-cooperative work-pool traversal.
//
// Per-query walks are heavy-tailed (n=300: mean ~1e3 node visits, p99 ~8e3,
// max ~6e4), so one-thread-per-query leaves warps waiting on their slowest
// lane and a small batch (the meet check: ~2e4 queries) runs for the serial
// latency of its longest walk.  Every warp owns a LIFO pool of tasks
// (query j, node, first key of the node's range, next bit d | |y|) in shared
// memory.  Each round the lanes pop up to 32 tasks from any mix of queries,
// load node + node's first key + query row in ONE concurrent round of 16-B
// vector loads, and push the admissible children with ballot-compacted
// stores; when fewer than 32 tasks remain the warp pulls new queries from a
// global counter (persistent grid).  Small ranges are scanned cooperatively:
// all (range, key) pairs of the warp are flattened over the lanes
// (consecutive keys → coalesced rows), the owner's y broadcast by shuffles.
// MARK mode: hits also go to a per-warp table so sibling tasks of a marked
// query are dropped without touching global memory.
constexpr int kPoolWarps = 6;
constexpr int kPoolThreads = kPoolWarps * 32;
// Tasks per warp in shared memory.  When a round would overflow the pool, its
// bottom half (the oldest tasks) is spilled to a per-warp stack in global
// memory and pulled back before new queries are taken; only when that stack
// is full too does the opened range fall back to a scan.
#ifndef SW_POOL_CAP
#define SW_POOL_CAP 256
#endif
constexpr int kPoolCap = SW_POOL_CAP;
constexpr int kSpill = kPoolCap / 2;
constexpr int kSpillCap = 1024;  // tasks per warp in the global spill stack
constexpr int kPoolBrute = kScanKeys;  // ranges of <= this many keys are scanned
constexpr int kHitSlots = 32;
constexpr u32 kNone = 0xFFFFFFFFu;

#ifndef SW_POOL_MINB_WIDE
#define SW_POOL_MINB_WIDE 1
#endif
#ifndef SW_POOL_MINB_NARROW
#define SW_POOL_MINB_NARROW 5
#endif
// Resident CTAs per SM: 5 for W <= 6 (64 registers; measured n=300 s0/s1/s2
// engine 95.5/35.3/85.8 ms against 98.8/36.6/89.1 at 6); wider rows need more
// registers per lane (the query row, the key row of a leaf).
constexpr int pool_min_blocks(int W) {
  return W <= 6 ? SW_POOL_MINB_NARROW : (W <= 10 ? SW_POOL_MINB_WIDE : 1);
}

template <int W, bool PROPER, bool EXIST>
__global__ void __launch_bounds__(kPoolThreads, pool_min_blocks(W)) contain_pool_kernel(
    const u64* __restrict__ A, const ulonglong2* __restrict__ Asig, const Node* __restrict__ nodes,
    u32 Na, const u64* __restrict__ B, const ulonglong2* __restrict__ Bsig, u32 Nb, uint8_t* keep,
    int* found, unsigned long long* wit, u32* next_query, uint4* spill_all, u32* overflow_scans,
    unsigned long long* stats, u32 spill_cap) {
  __shared__ u32 s_q[kPoolWarps][kPoolCap];
  __shared__ u32 s_n[kPoolWarps][kPoolCap];
  __shared__ u32 s_f[kPoolWarps][kPoolCap];
  __shared__ u32 s_dc[kPoolWarps][kPoolCap];  // d | |y| << 16
  __shared__ u32 s_hit[kPoolWarps][kHitSlots];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const unsigned FULL = 0xFFFFFFFFu, lt = (1u << lane) - 1;
  u32* sq = s_q[wid];
  u32* sn = s_n[wid];
  u32* sf = s_f[wid];
  u32* sdc = s_dc[wid];
  u32* shit = s_hit[wid];
  shit[lane] = kNone;
  __syncwarp();
  const u32 root_id = Na == 1 ? kLeafBit : 0u;
  uint4* spill = spill_all + (static_cast<u64>(blockIdx.x) * kPoolWarps + wid) * kSpillCap;
  int sp = 0, gsp = 0;
  bool more = true;
  // EXIST early exit: the flag is loaded each round but consumed the next, so
  // its L2 round trip overlaps a round of work (a blocking check at the top of
  // every round was 25% of the stall samples on the DFS queries).
  int found_seen = 0;
  // A confirmed containment: MARK drops the query, EXIST records the witness.
  auto report = [&](u32 key, u32 q) {
    if (EXIST) {
      if (atomicCAS(found, 0, 1) == 0) {
        wit[0] = key;
        wit[1] = q;
      }
    } else {
      keep[q] = 0;
      shit[q % kHitSlots] = q;
    }
  };
  while (true) {
    if (EXIST) {
      if (found_seen) break;
      found_seen = *reinterpret_cast<volatile int*>(found);
    }
    if (sp < 32 && gsp > 0) {  // pull spilled tasks back first
      const int t = gsp < kSpill ? gsp : kSpill;
      for (int i = lane; i < t; i += 32) {
        const uint4 v = spill[gsp - t + i];
        sq[sp + i] = v.x;
        sn[sp + i] = v.y;
        sf[sp + i] = v.z;
        sdc[sp + i] = v.w;
      }
      gsp -= t;
      sp += t;
      __syncwarp();
    } else if (sp < 32 && more) {  // refill with fresh queries
      u32 base = 0;
      if (lane == 0) base = atomicAdd(next_query, static_cast<u32>(32 - sp));
      base = __shfl_sync(FULL, base, 0);
      const u32 got = base >= Nb ? 0 : min(static_cast<u32>(32 - sp), Nb - base);
      if (base + (32 - sp) >= Nb) more = false;
      const u32 j = base + lane;
      bool push = static_cast<u32>(lane) < got;
      const u32 cy = push ? static_cast<u32>(B[static_cast<u64>(j) * Row<W>::P + W]) : 0;
      if (PROPER && cy == 0) push = false;
      const unsigned m = __ballot_sync(FULL, push);
      if (push) {
        const int pos = sp + __popc(m & lt);
        sq[pos] = j;
        sn[pos] = root_id;
        sf[pos] = 0;
        sdc[pos] = cy << 16;
      }
      sp += __popc(m);
      __syncwarp();
    }
    if (sp == 0) {
      if (!more && gsp == 0) break;
      continue;
    }
    const int take = sp < 32 ? sp : 32;
    bool have = lane < take;
    u32 j = 0, id = 0, first = 0, dc = 0;
    if (have) {
      const int pos = sp - 1 - lane;
      j = sq[pos];
      id = sn[pos];
      first = sf[pos];
      dc = sdc[pos];
    }
    sp -= take;
    __syncwarp();
    if (!EXIST && have && shit[j % kHitSlots] == j) have = false;
    const int d = static_cast<int>(dc & 0xFFFF);
    const u32 cy = dc >> 16;
    const u32 limit = PROPER ? cy - 1 : cy;
    const bool is_leaf = (id & kLeafBit) != 0;

    // ---- one concurrent round of loads: the query's filter words, and the
    // node (internal: + the query's words d/64 and d/64+1 — with need = lcp - d
    // <= 64 the unchecked prefix bits [d, lcp) and the split bit lcp all lie in
    // them; bits below d are masked) or the leaf key's filter words.  Full rows
    // are fetched only for long runs and for pairs that pass the filter.
    u64 y[W], xf[W];
    u32 ycard = 0, kcard = 0;
    u64 ya = 0, yb = 0;
    ulonglong2 qs = make_ulonglong2(0, 0), ks = make_ulonglong2(0, 0);
    const int q0 = d >> 6;
    Node nd{};
#pragma unroll
    for (int w = 0; w < W; ++w) y[w] = xf[w] = 0;
    if (have) {
      qs = __ldg(Bsig + j);
      if (is_leaf) {
        ks = __ldg(Asig + first);
      } else {
        nd = load_node(nodes + id);
        const u64* yr = B + static_cast<u64>(j) * Row<W>::P;
        ya = __ldg(yr + q0);
        yb = q0 + 1 < W ? __ldg(yr + q0 + 1) : 0;
      }
    }
    auto yword = [&](int q) { return q == q0 ? ya : (q == q0 + 1 ? yb : u64{0}); };

    // ---- evaluate the task
    bool hit = false, brute = false, longrun = false, leafcheck = false;
    u32 hit_a = 0, c0 = kNone, c1 = kNone, f0 = 0, f1 = 0, bf = 0, bl = 0;
    int dchild = 0, L = 0;
    if (have) {
      if (is_leaf) {
        leafcheck = filter_pass(ks, qs);
      } else if (nd.minc <= limit) {
        if (nd.last - nd.first < kPoolBrute) {
          // every key of the range holds the node's AND states: skip the scan
          // unless their filter words lie in the query's
          brute = filter_pass(make_ulonglong2(nd.window, nd.pad), qs);
          bf = nd.first;
          bl = nd.last;
        } else {
          L = nd.lcp;
          const int need = L - d;  // common-prefix bits not yet checked
          if (need > 64) {
            longrun = true;  // checked against the key row in round 2
          } else {
            u64 bad = 0;
            if (need > 0) {
              const u64 yw = window_before(yword, L);
              const u64 m = need == 64 ? ~u64{0} : ((u64{1} << need) - 1);
              bad = nd.window & ~yw & m;
            }
            if (!bad) {
              c0 = nd.split == nd.first ? (kLeafBit | nd.first) : nd.split;
              f0 = nd.first;
              if ((yword(L >> 6) >> (63 - (L & 63))) & 1) {
                c1 = nd.split + 1 == nd.last ? (kLeafBit | nd.last) : nd.split + 1;
                f1 = nd.split + 1;
              }
              dchild = L + 1;
              bf = nd.first;
              bl = nd.last;
            }
          }
        }
      }
    }
    // ---- round 2: whole rows for long common runs and leaves that passed the filter
    if (longrun || leafcheck) {
      load_row<W>(B, j, y, ycard);
      load_row<W>(A, longrun ? nd.first : first, xf, kcard);
    }
    if (leafcheck && kcard <= limit && is_subset<W>(xf, y)) {
      hit = true;
      hit_a = first;
    }
    if (longrun) {
      u64 bad = 0;
#pragma unroll
      for (int w = 0; w < W; ++w) bad |= xf[w] & ~y[w] & range_mask(w, d, L);
      if (!bad) {
        // query word L/64 straight from memory: a select over y[] here is
        // turned into an indexed access that puts y and xf on the stack
        const u64 yl = __ldg(B + static_cast<u64>(j) * Row<W>::P + (L >> 6));
        c0 = nd.split == nd.first ? (kLeafBit | nd.first) : nd.split;
        f0 = nd.first;
        if ((yl >> (63 - (L & 63))) & 1) {
          c1 = nd.split + 1 == nd.last ? (kLeafBit | nd.last) : nd.split + 1;
          f1 = nd.split + 1;
        }
        dchild = L + 1;
        bf = nd.first;
        bl = nd.last;
      }
    }

    if (stats) {  // analysis counters (SYNCHRO_PROGRESS): outcomes of this round's tasks
      const bool internal = have && !is_leaf;
      const bool minc_cut = internal && !brute && !longrun && c0 == kNone && L == 0;
      const u32 v[8] = {
          static_cast<u32>(__popc(__ballot_sync(FULL, have))),
          static_cast<u32>(__popc(__ballot_sync(FULL, have && is_leaf))),
          static_cast<u32>(__popc(__ballot_sync(FULL, hit))),
          static_cast<u32>(__popc(__ballot_sync(FULL, minc_cut))),
          static_cast<u32>(__popc(__ballot_sync(FULL, brute))),
          static_cast<u32>(__popc(__ballot_sync(FULL, internal && L != 0 && c0 == kNone))),
          static_cast<u32>(__popc(__ballot_sync(FULL, c0 != kNone))),
          static_cast<u32>(__popc(__ballot_sync(FULL, c1 != kNone)))};
      if (lane == 0) {
#pragma unroll
        for (int q = 0; q < 8; ++q) atomicAdd(stats + q, static_cast<unsigned long long>(v[q]));
      }
    }

    // ---- push children (LIFO; left on top)
    const u32 cdc = (cy << 16) | static_cast<u32>(dchild);
    const unsigned m0 = __ballot_sync(FULL, c0 != kNone);
    const unsigned m1 = __ballot_sync(FULL, c1 != kNone);
    const int n0 = __popc(m0), n1 = __popc(m1);
    if (sp + n0 + n1 > kPoolCap && gsp + kSpill <= static_cast<int>(spill_cap)) {
      // spill the oldest kSpill tasks; sp <= kPoolCap = 2 kSpill, so the
      // shifted block [kSpill, sp) and its target [0, sp - kSpill) are disjoint
      for (int i = lane; i < kSpill; i += 32)
        spill[gsp + i] = make_uint4(sq[i], sn[i], sf[i], sdc[i]);
      __syncwarp();
      for (int i = lane; i < sp - kSpill; i += 32) {
        sq[i] = sq[i + kSpill];
        sn[i] = sn[i + kSpill];
        sf[i] = sf[i + kSpill];
        sdc[i] = sdc[i + kSpill];
      }
      __syncwarp();
      gsp += kSpill;
      sp -= kSpill;
    }
    if (sp + n0 + n1 > kPoolCap) {
      // Pool and spill stack full: scan the opened range instead of descending
      // (the scan needs only the query's filter words, already loaded).
      if (c0 != kNone) brute = true;
      if (lane == 0) atomicAdd(overflow_scans, 1u);
    } else {
      if (c1 != kNone) {
        const int pos = sp + __popc(m1 & lt);
        sq[pos] = j;
        sn[pos] = c1;
        sf[pos] = f1;
        sdc[pos] = cdc;
      }
      if (c0 != kNone) {
        const int pos = sp + n1 + __popc(m0 & lt);
        sq[pos] = j;
        sn[pos] = c0;
        sf[pos] = f0;
        sdc[pos] = cdc;
      }
      sp += n0 + n1;
    }
    __syncwarp();

    // ---- cooperative scan of small ranges: (range, key) pairs flattened over
    // lanes; each pair first compares filter words (16 B per key), and only a
    // pair that passes loads both full rows for the exact test.
    const u32 cnt = brute ? bl - bf + 1 : 0;
    u32 incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const u32 v = __shfl_up_sync(FULL, incl, o);
      if (lane >= o) incl += v;
    }
    const u32 total = __shfl_sync(FULL, incl, 31);
    if (stats && lane == 0) atomicAdd(stats + 8, static_cast<unsigned long long>(total));
    const u32 excl = incl - cnt;
    for (u32 base = 0; base < total; base += 32) {
      const u32 t = base + lane;
      int owner = 0;
#pragma unroll
      for (int s = 16; s; s >>= 1) {
        const u32 v = __shfl_sync(FULL, incl, owner + s - 1);
        if (v <= t) owner += s;
      }
      owner = owner > 31 ? 31 : owner;
      const u32 o_excl = __shfl_sync(FULL, excl, owner);
      const u32 o_bf = __shfl_sync(FULL, bf, owner);
      const u32 o_j = __shfl_sync(FULL, j, owner);
      const u32 o_lim = __shfl_sync(FULL, limit, owner);
      const ulonglong2 oq = make_ulonglong2(__shfl_sync(FULL, qs.x, owner),
                                            __shfl_sync(FULL, qs.y, owner));
      if (t < total) {
        const u32 key = o_bf + (t - o_excl);
        if (filter_pass(__ldg(Asig + key), oq)) {  // rare: the exact test, word by word
          const u64* kr = A + static_cast<u64>(key) * Row<W>::P;
          const u64* yr = B + static_cast<u64>(o_j) * Row<W>::P;
          u64 acc = 0;
#pragma unroll
          for (int w = 0; w < W; ++w) acc |= __ldg(kr + w) & ~__ldg(yr + w);
          if (static_cast<u32>(__ldg(kr + W)) <= o_lim && acc == 0) report(key, o_j);
        }
      }
    }
    if (hit) report(hit_a, j);
    __syncwarp();
  }
}

// keep[j] = !hit (MARK) or *found/wit (EXIST) for padded queries Bp against
// the padded keys of index p.
template <bool PROPER, bool EXIST>
static void launch_query(Context& c, const PermIndex& p, const u64* Bp, const void* Bsig, u64 Nb,
                         uint8_t* keep, int* found, unsigned long long* wit) {
  if (!Nb) return;
  cudaStream_t s = as_stream(c.stream());
  if (!EXIST) SW_CUDA(cudaMemsetAsync(keep, 1, Nb, s));
  if (p.count == 0) return;
  u32* counter = static_cast<u32*>(c.scratch(7, 64)) + 8;  // slot 7: words 8.. (Res uses 0..5)
  SW_CUDA(cudaMemsetAsync(counter, 0, 8, s));  // [0] next query, [1] overflow scans
  // Persistent-grid size: queried once per (W, mode) and process (runtime
  // queries take driver locks; many concurrent solves share the device).
  static std::atomic<int> cache_bps[kMaxW + 1];
  static std::atomic<int> cache_sms{0};
  int sms = cache_sms.load(std::memory_order_relaxed);
  if (!sms) {
    int dev = 0;
    SW_CUDA(cudaGetDevice(&dev));
    SW_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    cache_sms.store(sms, std::memory_order_relaxed);
  }
  int blocks_per_sm = cache_bps[c.W()].load(std::memory_order_relaxed);
  if (!blocks_per_sm) {
    SW_DISPATCH_W(c.W(), {
      SW_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
          &blocks_per_sm, contain_pool_kernel<W, PROPER, EXIST>, kPoolThreads, 0));
    });
    blocks_per_sm = std::max(1, blocks_per_sm);
    cache_bps[c.W()].store(blocks_per_sm, std::memory_order_relaxed);
  }
  const u64 want_blocks = (Nb + kPoolThreads - 1) / kPoolThreads;
  const unsigned grid = static_cast<unsigned>(
      std::max<u64>(1, std::min<u64>(want_blocks, static_cast<u64>(sms) * blocks_per_sm)));
  unsigned long long* stats = nullptr;  // task-outcome counters (progress mode / contain_stats)
  if (progress_enabled() || c.contain_stats) {
    stats = static_cast<unsigned long long*>(c.scratch(7, 64 + 9 * 8)) + 8;  // after the Res words
    SW_CUDA(cudaMemsetAsync(stats, 0, 9 * 8, s));
  }
  uint4* spill = static_cast<uint4*>(
      c.scratch(10, static_cast<size_t>(grid) * kPoolWarps * kSpillCap * sizeof(uint4)));
  // Test hook: SYNCHRO_SPILL_CAP (tasks per warp, <= kSpillCap) shrinks the
  // spill stack so the overflow scan path runs (tests/test_gpu_primitives.py).
  const u32 spill_cap = [] {
    const char* e = std::getenv("SYNCHRO_SPILL_CAP");
    const long v = e && *e ? std::strtol(e, nullptr, 10) : kSpillCap;
    return static_cast<u32>(std::clamp<long>(v, 0, kSpillCap));
  }();
  std::unique_ptr<StreamTimer> timer;
  if (progress_enabled() || c.timing) {
    timer = std::make_unique<StreamTimer>(c);
    timer->start();
  }
  SW_DISPATCH_W(c.W(), {
    contain_pool_kernel<W, PROPER, EXIST><<<grid, kPoolThreads, 0, s>>>(
        p.keys, static_cast<const ulonglong2*>(p.tree.keysig),
        static_cast<const Node*>(p.tree.nodes), static_cast<u32>(p.count), Bp,
        static_cast<const ulonglong2*>(Bsig), static_cast<u32>(Nb), keep, found, wit, counter,
        spill, counter + 1, stats, spill_cap);
  });
  SW_CHECK_LAUNCH();
  c.counters.kernel_launches += 1;
  if (timer) {
    const double ms = timer->stop_ms();
    // algorithmic bytes: every key and every query row read once, a flag written
    const u64 row = static_cast<u64>(c.W()) * 8 + 4;
    c.counters.contain_ms += ms;
    c.counters.contain_launches += 1;
    c.counters.contain_bytes += (p.count + Nb) * row + (EXIST ? 0 : Nb);
    if (progress_enabled()) {
      u32 overflow = 0;
      c.memcpy_d2h(&overflow, counter + 1, 4);
      unsigned long long st[9];
      c.memcpy_d2h(st, stats, sizeof(st));
      SYNCHRO_PROGRESS("  contain-stats tasks=%llu leaf=%llu hit=%llu minc_cut=%llu scans=%llu "
                       "prefix_cut=%llu push0=%llu push1=%llu pairs=%llu",
                       st[0], st[1], st[2], st[3], st[4], st[5], st[6], st[7], st[8]);
      SYNCHRO_PROGRESS("  contain %s%s |A|=%zu |B|=%llu %.3f ms overflow_scans=%u",
                       EXIST ? "exist" : "mark", PROPER ? "-proper" : "", p.count,
                       static_cast<unsigned long long>(Nb), ms, overflow);
    }
  }
  if (c.contain_stats) {  // node visits (tasks) and range-scan pair tests of this launch
    unsigned long long st[9];
    c.memcpy_d2h(st, stats, sizeof(st));
    c.counters.contain_visits += st[0];
    c.counters.contain_pairs += st[8];
  }
}

// ------------------------------------------------------- relabelled index
PermIndex::~PermIndex() {
  if (ctx) {
    try {
      ctx->free(orig);
      ctx->free(state_pos);
      ctx->free(keys);
    } catch (...) {
    }
  }
}
PermIndex::PermIndex(PermIndex&& o) noexcept { *this = std::move(o); }
PermIndex& PermIndex::operator=(PermIndex&& o) noexcept {
  if (this != &o) {
    if (ctx) {
      ctx->free(orig);
      ctx->free(state_pos);
      ctx->free(keys);
    }
    ctx = o.ctx;
    count = o.count;
    orig = o.orig;
    state_pos = o.state_pos;
    keys = o.keys;
    tree = std::move(o.tree);
    o.orig = nullptr;
    o.state_pos = nullptr;
    o.keys = nullptr;
    o.count = 0;
  }
  return *this;
}

// Relabelled copy of l as padded query rows, plus their filter words.
static u64* relabel_padded(Context& c, const DList& l, const uint16_t* pos, void** sig) {
  u64* out = nullptr;
  *sig = c.alloc(std::max<size_t>(l.size(), 1) * 16);
  SW_DISPATCH_W(c.W(), {
    out = static_cast<u64*>(c.alloc(std::max<size_t>(l.size(), 1) * Row<W>::P * 8));
    if (!l.empty())
      relabel_kernel<W, true><<<grid_for(l.size(), 256, 148 * 8), 256, c.n() * 2, as_stream(c.stream())>>>(
          l.words, l.cards, l.size(), c.n(), pos, out, nullptr, static_cast<ulonglong2*>(*sig));
  });
  SW_CHECK_LAUNCH();
  c.counters.kernel_launches++;
  return out;
}

__global__ void scatter_flags_kernel(const uint8_t* __restrict__ src, const u32* __restrict__ perm,
                                     u64 count, uint8_t* __restrict__ dst) {
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<u64>(gridDim.x) * blockDim.x)
    dst[perm[i]] = src[i];
}

PermIndex build_perm_index(Context& c, const DList& a, StateOrder order) {
  PermIndex p;
  p.ctx = &c;
  p.count = a.size();
  const u32 n = c.n();
  cudaStream_t s = as_stream(c.stream());
  std::vector<uint16_t> pos(n);
  for (u32 q = 0; q < n; ++q) pos[q] = static_cast<uint16_t>(q);
  if (order != StateOrder::Natural && !a.empty()) {
    u32* hist = static_cast<u32*>(c.alloc(n * 4));
    state_histogram(c, a, hist);
    std::vector<u32> h(n);
    c.memcpy_d2h(h.data(), hist, n * 4);
    c.free(hist);
    std::vector<u32> ord(n);
    for (u32 q = 0; q < n; ++q) ord[q] = q;
    if (order == StateOrder::FreqDesc)
      std::stable_sort(ord.begin(), ord.end(), [&](u32 x, u32 y) { return h[x] > h[y]; });
    else
      std::stable_sort(ord.begin(), ord.end(), [&](u32 x, u32 y) { return h[x] < h[y]; });
    for (u32 i = 0; i < n; ++i) pos[ord[i]] = static_cast<uint16_t>(i);
  }
  p.state_pos = static_cast<uint16_t*>(c.alloc(n * 2));
  c.memcpy_h2d(p.state_pos, pos.data(), n * 2);
  // Relabel, sort (lex, in the new state order), pad.
  DList sorted(&c, a.size(), false);
  sorted.set_size(a.size());
  if (!a.empty()) {
    SW_DISPATCH_W(c.W(), {
      relabel_kernel<W, false><<<grid_for(a.size(), 256, 148 * 8), 256, n * 2, s>>>(
          a.words, a.cards, a.size(), n, p.state_pos, sorted.words, sorted.cards, nullptr);
    });
    SW_CHECK_LAUNCH();
  }
  p.orig = static_cast<u32*>(c.alloc(std::max<size_t>(a.size(), 1) * 4));
  if (a.size() > 1) {
    const u32* perm = sort_perm(c, sorted, false);
    SW_CUDA(cudaMemcpyAsync(p.orig, perm, a.size() * 4, cudaMemcpyDeviceToDevice, s));
    compact_flags(c, sorted, nullptr, p.orig);
  } else if (a.size() == 1) {
    SW_CUDA(cudaMemsetAsync(p.orig, 0, 4, s));
  }
  if (progress_enabled()) {
    c.sync();
    SYNCHRO_PROGRESS("  perm-index |A|=%zu relabelled+sorted", a.size());
  }
  p.tree = build_index(c, sorted);
  p.tree.keysig = c.alloc(std::max<size_t>(a.size(), 1) * 16);
  SW_DISPATCH_W(c.W(), {
    p.keys = static_cast<u64*>(c.alloc(std::max<size_t>(a.size(), 1) * Row<W>::P * 8));
    if (!a.empty())
      pad_kernel<W><<<grid_for(a.size(), 256, 148 * 8), 256, 0, s>>>(
          sorted.words, sorted.cards, a.size(), p.keys, static_cast<ulonglong2*>(p.tree.keysig));
  });
  SW_CHECK_LAUNCH();
  c.counters.kernel_launches += 3;
  if (progress_enabled()) {
    c.sync();
    SYNCHRO_PROGRESS("  perm-index |A|=%zu tree built", a.size());
  }
  return p;
}

bool exists_subset(Context& c, const PermIndex& p, const DList& b, Witness* w) {
  if (p.count == 0 || b.empty()) return false;
  // (Sorting the queries in relabelled-lex order was measured slower at n=570:
  // heavy walks cluster into the same warps; the (card desc, lex) level order
  // spreads them.)
  void* Bsig = nullptr;
  u64* Bp = relabel_padded(c, b, p.state_pos, &Bsig);
  struct Res {
    int found;
    int pad;
    unsigned long long wit[2];
  };
  auto* d = static_cast<Res*>(c.scratch(7, 64));
  SW_CUDA(cudaMemsetAsync(d, 0, sizeof(Res), as_stream(c.stream())));
  launch_query<false, true>(c, p, Bp, Bsig, b.size(), nullptr, &d->found, d->wit);
  Res h;
  c.memcpy_d2h(&h, d, sizeof(Res));
  c.free(Bp);
  c.free(Bsig);
  if (h.found && w) {
    u32 o = 0;
    c.memcpy_d2h(&o, p.orig + h.wit[0], 4);
    w->a_index = o;
    w->b_index = h.wit[1];
  }
  return h.found != 0;
}

static uint8_t* keep_flags(Context& c, const PermIndex& p, const DList& b, bool proper) {
  auto* keep = static_cast<uint8_t*>(c.scratch(5, b.size()));
  void* Bsig = nullptr;
  u64* Bp = relabel_padded(c, b, p.state_pos, &Bsig);
  if (proper)
    launch_query<true, false>(c, p, Bp, Bsig, b.size(), keep, nullptr, nullptr);
  else
    launch_query<false, false>(c, p, Bp, Bsig, b.size(), keep, nullptr, nullptr);
  c.free(Bp);
  c.free(Bsig);
  return keep;
}

size_t remove_supersets(Context& c, const PermIndex& p, DList& b, bool proper) {
  if (b.empty() || p.count == 0) return 0;
  const size_t before = b.size();
  uint8_t* keep = keep_flags(c, p, b, proper);
  return before - compact_flags(c, b, keep, nullptr);
}

std::vector<uint8_t> superset_keep(Context& c, const PermIndex& p, const DList& b, bool proper) {
  std::vector<uint8_t> out(b.size(), 1);
  if (b.empty() || p.count == 0) return out;
  uint8_t* keep = keep_flags(c, p, b, proper);
  c.memcpy_d2h(out.data(), keep, b.size());
  return out;
}

// Minimal antichain: drop every set with a proper subset in the list.
// Rarest-state-first order prunes best here (queries are the keys themselves).
size_t remove_supersets_of(Context& c, const DList& A, DList& b, bool proper) {
  if (b.empty() || A.empty()) return 0;
  if (bitmap_fits(c)) {  // n <= 20: the power-set bitmap
    const size_t before = b.size();
    auto* keep = static_cast<uint8_t*>(c.scratch(5, b.size()));
    bitmap_keep_flags(c, A, b, /*super=*/false, proper, keep);
    return before - compact_flags(c, b, keep, nullptr);
  }
  if (brute_fits(A.size(), b.size())) {
    const size_t before = b.size();
    auto* keep = static_cast<uint8_t*>(c.scratch(5, b.size()));
    brute_keep_flags(c, A, b, /*super=*/false, proper, keep);
    return before - compact_flags(c, b, keep, nullptr);
  }
  if (use_trie_for_marks()) {
    const size_t before = b.size();
    const TrieQueryIndex t = build_trie_index(c, A, kTrieLeafKeys);
    auto* keep = static_cast<uint8_t*>(c.scratch(5, b.size()));
    trie_superset_flags(c, t, b, proper, keep);
    return before - compact_flags(c, b, keep, nullptr);
  }
  const PermIndex p = build_perm_index(c, A, StateOrder::FreqDesc);
  return remove_supersets(c, p, b, proper);
}

size_t self_reduce_minimal(Context& c, DList& l) {
  if (l.size() <= 1) return 0;
  if (bitmap_fits(c)) {  // n <= 20: the power-set bitmap
    const size_t before = l.size();
    auto* keep = static_cast<uint8_t*>(c.scratch(5, l.size()));
    bitmap_keep_flags(c, l, l, /*super=*/false, /*proper=*/true, keep);
    return before - compact_flags(c, l, keep, nullptr);
  }
  if (brute_fits(l.size(), l.size())) {  // small list: one all-pairs launch
    const size_t before = l.size();
    auto* keep = static_cast<uint8_t*>(c.scratch(5, l.size()));
    brute_keep_flags(c, l, l, /*super=*/false, /*proper=*/true, keep);
    return before - compact_flags(c, l, keep, nullptr);
  }
  if (use_trie_for_marks()) return trie_self_reduce_minimal(c, l);
  // Rarest states first (measured at n=300 s0: engine 98 ms; most frequent first
  // 187 ms, natural order 119 ms).
  const PermIndex p = build_perm_index(c, l, StateOrder::FreqAsc);
  // The queries are the keys themselves: query with the index's own sorted,
  // relabelled rows (best locality), then map the flags back to l's order.
  const size_t before = l.size();
  auto* keep = static_cast<uint8_t*>(c.scratch(5, l.size()));
  uint8_t* ks = static_cast<uint8_t*>(c.alloc(l.size()));
  launch_query<true, false>(c, p, p.keys, p.tree.keysig, l.size(), ks, nullptr, nullptr);
  scatter_flags_kernel<<<grid_for(l.size(), 256), 256, 0, as_stream(c.stream())>>>(ks, p.orig, l.size(), keep);
  SW_CHECK_LAUNCH();
  c.free(ks);
  return before - compact_flags(c, l, keep, nullptr);
}

}  // namespace synchro::dev
