// Exact node count of the reference's StaticTrie over a list, on the GPU.
//
// Only the NUMBER of trie nodes is observable in the reference (through the
// ledger: footprint = sets + 24 B per node, static_trie.hpp:43-45, which
// feeds peak_memory and the DFS slice cap).  The shape is a function of the
// set family alone: build_node (static_trie.hpp:85-122) splits a range on the
// state contained in the most (but not all) of its sets, ties to the smallest
// state (pick_division_state, :127-151); ranges of <= min_leaf sets are
// leaves; a zero side of <= min_leaf sets is absorbed as payload.
//
// Level-synchronous construction: every round processes all active segments
// at once — (1) per-segment state histograms (shared-memory aggregation when a
// block's elements fall into one segment, global atomics otherwise), (2) one
// warp per segment picks the division state, (3) children are allocated and
// counted, (4) elements are scattered to their child range (order inside a
// range is irrelevant to the count).  Rounds = trie depth.
#include <cub/cub.cuh>

#include "dev.hpp"
#include "kernels.cuh"
#include "util.cuh"
#include "../progress.hpp"

namespace synchro::dev {

namespace {

constexpr u32 kInvalid = 0xFFFFFFFFu;
constexpr u32 kCountSmall = 16384;  // count-only builds up to this size: one block

struct Seg {
  u32 lo, hi;
};

template <int W>
__global__ void __launch_bounds__(256) hist_kernel(const u64* __restrict__ words,
                                                   const u32* __restrict__ idx,
                                                   const u32* __restrict__ seg, u32 N, u32 n,
                                                   u32* __restrict__ hist,
                                                   const u32* __restrict__ cards,
                                                   u32* __restrict__ minc) {
  extern __shared__ u32 sh[];
  const u32 base = blockIdx.x * blockDim.x;
  const u32 i = base + threadIdx.x;
  const u32 last = min(N, base + blockDim.x) - 1;
  const u32 s0 = seg[base], s1 = seg[last];
  const bool shared_mode = (s0 == s1) && s0 != kInvalid;
  if (shared_mode) {
    for (u32 q = threadIdx.x; q < n; q += blockDim.x) sh[q] = 0;
    __syncthreads();
  }
  if (minc) {  // shape mode: per-segment min cardinality (warp-aggregated atomicMin)
    const u32 s = i < N ? seg[i] : kInvalid;
    const unsigned peers = __match_any_sync(0xFFFFFFFFu, s);
    const u32 m = __reduce_min_sync(peers, s != kInvalid ? cards[idx[i]] : 0xFFFFFFFFu);
    if (s != kInvalid && (threadIdx.x & 31) == __ffs(peers) - 1) atomicMin(&minc[s], m);
  }
  if (i < N) {
    const u32 s = seg[i];
    if (s != kInvalid) {
      const u64* x = words + static_cast<u64>(idx[i]) * W;
#pragma unroll
      for (int w = 0; w < W; ++w) {
        u64 bits = x[w];
        while (bits) {
          const int b = __clzll(bits);
          bits &= ~(u64{1} << (63 - b));
          const u32 q = w * 64 + b;
          if (shared_mode)
            atomicAdd(&sh[q], 1u);
          else
            atomicAdd(&hist[static_cast<u64>(s) * n + q], 1u);
        }
      }
    }
  }
  if (shared_mode) {
    __syncthreads();
    for (u32 q = threadIdx.x; q < n; q += blockDim.x)
      if (sh[q]) atomicAdd(&hist[static_cast<u64>(s0) * n + q], sh[q]);
  }
}

// One warp per active segment: division state, zero-side size, children.
__global__ void pick_kernel(const u32* __restrict__ hist, const Seg* __restrict__ segs, u32 nseg,
                            u32 n, u32 min_leaf, u32* __restrict__ div, u32* __restrict__ zcount,
                            u32* __restrict__ child_zero, u32* __restrict__ child_one,
                            Seg* __restrict__ next_segs, u32* __restrict__ next_count,
                            unsigned long long* __restrict__ nodes) {
  const u32 warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= nseg) return;
  const Seg sg = segs[warp];
  const u32 total = sg.hi - sg.lo;
  const u32* h = hist + static_cast<u64>(warp) * n;
  u32 best_c = 0, best_q = kInvalid;
  for (u32 q = lane; q < n; q += 32) {
    const u32 v = h[q];
    if (v < total && v > best_c) {  // ascending q per lane: strict > keeps the smallest
      best_c = v;
      best_q = q;
    }
  }
  for (int off = 16; off; off >>= 1) {
    const u32 oc = __shfl_xor_sync(0xFFFFFFFFu, best_c, off);
    const u32 oq = __shfl_xor_sync(0xFFFFFFFFu, best_q, off);
    if (oc > best_c || (oc == best_c && oq < best_q)) {
      best_c = oc;
      best_q = oq;
    }
  }
  if (lane == 0) {
    // best_q == kInvalid only for duplicate sets (never for a deduped list).
    div[warp] = best_q;
    const u32 ones = best_c, zeros = total - ones;
    zcount[warp] = zeros;
    unsigned long long made = 1;  // the one side is always a node
    u32 cz = kInvalid, co = kInvalid;
    if (zeros > min_leaf) {
      ++made;
      cz = atomicAdd(next_count, 1u);
      next_segs[cz] = Seg{sg.lo, sg.lo + zeros};
    }
    if (ones > min_leaf) {
      co = atomicAdd(next_count, 1u);
      next_segs[co] = Seg{sg.lo + zeros, sg.hi};
    }
    child_zero[warp] = cz;
    child_one[warp] = co;
    atomicAdd(nodes, made);
  }
}

template <int W>
__global__ void scatter_kernel(const u64* __restrict__ words, const u32* __restrict__ idx,
                               const u32* __restrict__ seg, u32 N, const Seg* __restrict__ segs,
                               const u32* __restrict__ div, const u32* __restrict__ zcount,
                               const u32* __restrict__ child_zero, const u32* __restrict__ child_one,
                               u32* __restrict__ cursor_zero, u32* __restrict__ cursor_one,
                               u32* __restrict__ idx_out, u32* __restrict__ seg_out) {
  const u32 i = blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  const u32 s = i < N ? seg[i] : kInvalid;
  if (i < N && s == kInvalid) {
    seg_out[i] = kInvalid;
    idx_out[i] = idx[i];
  }
  const bool active = s != kInvalid;
  u32 e = 0;
  bool one = false;
  if (active) {
    const u32 x = div[s];
    e = idx[i];
    one = (words[static_cast<u64>(e) * W + (x >> 6)] >> (63 - (x & 63))) & 1;
  }
  // Warp-aggregated slot reservation: one atomic per (segment, side) group of
  // the warp — near the root every element shares the same two cursors.
  const u32 key = active ? (s << 1 | static_cast<u32>(one)) : 0xFFFFFFFFu;
  const unsigned peers = __match_any_sync(0xFFFFFFFFu, key);
  const int leader = __ffs(peers) - 1;
  u32 base = 0;
  if (active && lane == leader)
    base = atomicAdd(one ? &cursor_one[s] : &cursor_zero[s], static_cast<u32>(__popc(peers)));
  base = __shfl_sync(0xFFFFFFFFu, base, leader);
  if (!active) return;
  const u32 rank = __popc(peers & ((1u << lane) - 1));
  const u32 pos = segs[s].lo + (one ? zcount[s] : 0) + base + rank;
  idx_out[pos] = e;
  seg_out[pos] = one ? child_one[s] : child_zero[s];
}

// Query index: the internal nodes of one round, with absolute node ids (this
// round's first id `base`; the next round's nodes follow it) and payload ranges
// into the final element order.
__global__ void emit_kernel(const Seg* __restrict__ segs, u32 nact, const u32* __restrict__ div,
                            const u32* __restrict__ zc, const u32* __restrict__ cz,
                            const u32* __restrict__ co, const u32* __restrict__ minc, u32 base,
                            TrieNode* __restrict__ nodes) {
  const u32 i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nact) return;
  const Seg sg = segs[i];
  const u32 zeros = zc[i];
  TrieNode nd;
  nd.div = div[i];
  nd.minc = minc[i];
  nd.zero = cz[i] == kInvalid ? kInvalid : base + nact + cz[i];
  nd.one = co[i] == kInvalid ? kInvalid : base + nact + co[i];
  // a zero side of <= min_leaf sets is absorbed as payload (static_trie.hpp:107-110),
  // a one side of <= min_leaf sets is a leaf (:84-88)
  nd.lo = sg.lo;
  nd.mid = sg.lo + zeros;
  nd.hi = sg.hi;
  nd.child_div = 0xFFFFFFFFu;  // children's division states: child_div_kernel
  nodes[base + i] = nd;
}

// pad = the children's division states (a task carries its node's state, so
// the query word it tests is fetched together with the node).
__global__ void child_div_kernel(TrieNode* __restrict__ nodes, u32 count) {
  const u32 i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  const TrieNode nd = nodes[i];
  const u32 zd = nd.zero == kInvalid ? 0xFFFFu : (nodes[nd.zero].div & 0xFFFFu);
  const u32 od = nd.one == kInvalid ? 0xFFFFu : (nodes[nd.one].div & 0xFFFFu);
  nodes[i].child_div = zd | (od << 16);
}

__global__ void init_kernel(u32* idx, u32* seg, u32 N) {
  const u32 i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < N) {
    idx[i] = i;
    seg[i] = 0;
  }
}

// Count-only construction of a SMALL list in one block: the rounds of
// hist/pick/scatter above as phases separated by block barriers, the round's
// segment count in shared memory — one launch and one readback instead of ~4
// memsets, 3 launches and a readback per trie level (config-2 solves take the
// ledger's trie count at every DFS start).  Same arithmetic, same count.
template <int W>
__global__ void __launch_bounds__(1024) count_small_kernel(
    const u64* __restrict__ words, u32 N, u32 n, u32 min_leaf, u32* idx, u32* seg, u32* idx2,
    u32* seg2, Seg* segs, Seg* nsegs, u32* per, u32 max_segs, u32* hist,
    unsigned long long* nodes_out) {
  __shared__ u32 nact, next_count;
  __shared__ unsigned long long nodes;
  const u32 tid = threadIdx.x, nthr = blockDim.x;
  for (u32 i = tid; i < N; i += nthr) {
    idx[i] = i;
    seg[i] = 0;
  }
  if (tid == 0) {
    segs[0] = Seg{0, N};
    nact = 1;
    nodes = 1;
  }
  __syncthreads();
  u32* div = per;
  u32* zc = per + max_segs;
  u32* cz = per + 2 * max_segs;
  u32* co = per + 3 * max_segs;
  u32* curz = per + 4 * max_segs;
  u32* curo = per + 5 * max_segs;
  while (nact > 0) {
    const u32 na = nact;
    for (u32 i = tid; i < na * n; i += nthr) hist[i] = 0;
    for (u32 i = tid; i < na; i += nthr) curz[i] = curo[i] = 0;
    if (tid == 0) next_count = 0;
    __syncthreads();
    for (u32 i = tid; i < N; i += nthr) {  // per-segment state histograms
      const u32 sg = seg[i];
      if (sg == kInvalid) continue;
      const u64* x = words + static_cast<u64>(idx[i]) * W;
#pragma unroll
      for (int w = 0; w < W; ++w) {
        u64 bits = x[w];
        while (bits) {
          const int b = __clzll(bits);
          bits &= ~(u64{1} << (63 - b));
          atomicAdd(&hist[sg * n + w * 64 + b], 1u);
        }
      }
    }
    __syncthreads();
    const u32 lane = tid & 31;
    for (u32 wp = tid >> 5; wp < na; wp += nthr >> 5) {  // one warp per segment: division state
      const Seg sg = segs[wp];
      const u32 total = sg.hi - sg.lo;
      u32 best_c = 0, best_q = kInvalid;
      for (u32 q = lane; q < n; q += 32) {
        const u32 v = hist[wp * n + q];
        if (v < total && v > best_c) {
          best_c = v;
          best_q = q;
        }
      }
      for (int off = 16; off; off >>= 1) {
        const u32 oc = __shfl_xor_sync(0xFFFFFFFFu, best_c, off);
        const u32 oq = __shfl_xor_sync(0xFFFFFFFFu, best_q, off);
        if (oc > best_c || (oc == best_c && oq < best_q)) {
          best_c = oc;
          best_q = oq;
        }
      }
      if (lane == 0) {
        div[wp] = best_q;
        const u32 ones = best_c, zeros = total - ones;
        zc[wp] = zeros;
        unsigned long long made = 1;
        u32 z = kInvalid, o = kInvalid;
        if (zeros > min_leaf) {
          ++made;
          z = atomicAdd(&next_count, 1u);
          nsegs[z] = Seg{sg.lo, sg.lo + zeros};
        }
        if (ones > min_leaf) {
          o = atomicAdd(&next_count, 1u);
          nsegs[o] = Seg{sg.lo + zeros, sg.hi};
        }
        cz[wp] = z;
        co[wp] = o;
        atomicAdd(&nodes, made);
      }
    }
    __syncthreads();
    for (u32 i = tid; i < N; i += nthr) {  // elements to their child ranges
      const u32 sg = seg[i];
      if (sg == kInvalid) {
        seg2[i] = kInvalid;
        idx2[i] = idx[i];
        continue;
      }
      const u32 x = div[sg], e = idx[i];
      const bool one = (words[static_cast<u64>(e) * W + (x >> 6)] >> (63 - (x & 63))) & 1;
      const u32 r = atomicAdd(one ? &curo[sg] : &curz[sg], 1u);
      const u32 pos = segs[sg].lo + (one ? zc[sg] : 0) + r;
      idx2[pos] = e;
      seg2[pos] = one ? co[sg] : cz[sg];
    }
    __syncthreads();
    u32* t = idx; idx = idx2; idx2 = t;
    t = seg; seg = seg2; seg2 = t;
    Seg* ts = segs; segs = nsegs; nsegs = ts;
    if (tid == 0) nact = next_count;
    __syncthreads();
  }
  if (tid == 0) *nodes_out = nodes;
}

}  // namespace

// Builds the trie level by level; returns the node count and, with `shape`,
// records every internal node (division state, min cardinality, internal
// children) round by round; with `qi`, emits the device node array of a query
// index and the final element order (qi->order).
static u64 build_trie(Context& c, const DList& l, u32 min_leaf, TrieShape* shape,
                      TrieQueryIndex* qi = nullptr) {
  const u64 N64 = l.size();
  if (N64 == 0) throw std::invalid_argument("StaticTrie: list must be non-empty");
  min_leaf = std::max<u32>(1, min_leaf);
  if (shape) {
    shape->rounds.clear();
    shape->min_leaf = min_leaf;
  }
  if (N64 <= min_leaf) {
    if (qi) {  // the whole list is one leaf: a pseudo node with only a payload
      const u32 N = static_cast<u32>(N64);
      const ListStats st = stats(c, l);
      TrieNode root{kInvalid, st.min_card, kInvalid, kInvalid, 0, N, N, 0xFFFFFFFFu};
      qi->nodes = c.alloc(sizeof(TrieNode));
      c.memcpy_h2d(qi->nodes, &root, sizeof(root));
      qi->node_count = 1;
      qi->order = static_cast<u32*>(c.alloc(N * 4ull));
      std::vector<u32> id(N);
      for (u32 i = 0; i < N; ++i) id[i] = i;
      c.memcpy_h2d(qi->order, id.data(), N * 4ull);
    }
    return 1;
  }
  const u32 N = static_cast<u32>(N64), n = c.n();
  cudaStream_t s = as_stream(c.stream());
  if (!shape && !qi && N <= kCountSmall) {
    const u32 max_segs = N / (min_leaf + 1) + 2;
    u32* buf = static_cast<u32*>(c.alloc((4ull * N + 4ull * max_segs + 6ull * max_segs +
                                          static_cast<u64>(max_segs) * n + 2) * 4));
    u32* idx = buf;
    u32* seg = idx + N;
    u32* idx2 = seg + N;
    u32* seg2 = idx2 + N;
    Seg* segs = reinterpret_cast<Seg*>(seg2 + N);
    Seg* nsegs = segs + max_segs;
    u32* per = reinterpret_cast<u32*>(nsegs + max_segs);
    u32* hist = per + 6ull * max_segs;
    auto* out = static_cast<unsigned long long*>(c.scratch(7, 8));
    SW_DISPATCH_W(c.W(), {
      count_small_kernel<W><<<1, 1024, 0, s>>>(l.words, N, n, min_leaf, idx, seg, idx2, seg2, segs,
                                               nsegs, per, max_segs, hist, out);
    });
    SW_CHECK_LAUNCH();
    c.counters.kernel_launches += 1;
    unsigned long long nodes = 0;
    c.memcpy_d2h(&nodes, out, 8);
    c.free(buf);
    return nodes;
  }
  u32* idx = static_cast<u32*>(c.alloc(N * 4ull));
  u32* seg = static_cast<u32*>(c.alloc(N * 4ull));
  u32* idx2 = static_cast<u32*>(c.alloc(N * 4ull));
  u32* seg2 = static_cast<u32*>(c.alloc(N * 4ull));
  init_kernel<<<(N + 255) / 256, 256, 0, s>>>(idx, seg, N);
  const u32 max_segs = N / (min_leaf + 1) + 2;
  Seg* segs = static_cast<Seg*>(c.alloc(max_segs * sizeof(Seg)));
  Seg* nsegs = static_cast<Seg*>(c.alloc(max_segs * sizeof(Seg)));
  // per-segment: div, zcount, child_zero, child_one, cursor_zero, cursor_one
  u32* per = static_cast<u32*>(c.alloc(7ull * max_segs * 4));
  struct Ctr {
    u32 next_count;
    u32 pad;
    unsigned long long nodes;
  };
  Ctr* ctr = static_cast<Ctr*>(c.alloc(sizeof(Ctr)));
  Ctr h{0, 0, 1};  // the root
  c.memcpy_h2d(ctr, &h, sizeof(h));
  Seg root{0, N};
  c.memcpy_h2d(segs, &root, sizeof(root));
  u32 nact = 1;
  u32* hist = nullptr;
  size_t hist_cap = 0;
  TrieNode* qnodes = nullptr;
  u32 base = 0;
  if (qi) qnodes = static_cast<TrieNode*>(c.alloc(static_cast<size_t>(N) * sizeof(TrieNode)));
  const bool want_minc = shape || qi;
  while (nact > 0) {
    const size_t hbytes = static_cast<size_t>(nact) * n * 4;
    if (hbytes > hist_cap) {
      if (hist) c.free(hist);
      hist_cap = hbytes + hbytes / 2;
      hist = static_cast<u32*>(c.alloc(hist_cap));
    }
    SW_CUDA(cudaMemsetAsync(hist, 0, hbytes, s));
    SW_CUDA(cudaMemsetAsync(per, 0, 6ull * max_segs * 4, s));
    u32* minc = want_minc ? per + 6ull * max_segs : nullptr;
    if (minc) SW_CUDA(cudaMemsetAsync(minc, 0xFF, static_cast<size_t>(nact) * 4, s));
    SW_CUDA(cudaMemsetAsync(&ctr->next_count, 0, 4, s));
    u32* div = per;
    u32* zc = per + max_segs;
    u32* cz = per + 2ull * max_segs;
    u32* co = per + 3ull * max_segs;
    u32* curz = per + 4ull * max_segs;
    u32* curo = per + 5ull * max_segs;
    SW_DISPATCH_W(c.W(), {
      hist_kernel<W><<<(N + 255) / 256, 256, n * 4, s>>>(l.words, idx, seg, N, n, hist, l.cards,
                                                         minc);
    });
    pick_kernel<<<(nact * 32 + 255) / 256, 256, 0, s>>>(hist, segs, nact, n, min_leaf, div, zc, cz,
                                                        co, nsegs, &ctr->next_count, &ctr->nodes);
    SW_DISPATCH_W(c.W(), {
      scatter_kernel<W><<<(N + 255) / 256, 256, 0, s>>>(l.words, idx, seg, N, segs, div, zc, cz, co,
                                                        curz, curo, idx2, seg2);
    });
    if (qi) {
      emit_kernel<<<(nact + 255) / 256, 256, 0, s>>>(segs, nact, div, zc, cz, co, minc, base, qnodes);
      base += nact;
    }
    SW_CHECK_LAUNCH();
    c.counters.kernel_launches += 3;
    if (shape) {
      std::vector<u32> hd(4ull * nact), hm(nact);
      c.memcpy_d2h(hd.data(), div, nact * 4ull);
      c.memcpy_d2h(hd.data() + nact, cz, nact * 4ull);
      c.memcpy_d2h(hd.data() + 2ull * nact, co, nact * 4ull);
      c.memcpy_d2h(hm.data(), minc, nact * 4ull);
      std::vector<TrieShape::Node> round(nact);
      for (u32 i = 0; i < nact; ++i)
        round[i] = TrieShape::Node{hd[i], hm[i], hd[nact + i], hd[2ull * nact + i]};
      shape->rounds.push_back(std::move(round));
    }
    std::swap(idx, idx2);
    std::swap(seg, seg2);
    std::swap(segs, nsegs);
    c.memcpy_d2h(&h, ctr, sizeof(h));
    nact = h.next_count;
  }
  if (qi) {  // elements of every node's range are contiguous in idx
    child_div_kernel<<<(base + 255) / 256, 256, 0, s>>>(qnodes, base);
    SW_CHECK_LAUNCH();
    qi->nodes = qnodes;
    qi->node_count = base;
    qi->order = idx;
    idx = nullptr;
  }
  c.free(idx);
  c.free(seg);
  c.free(idx2);
  c.free(seg2);
  c.free(segs);
  c.free(nsegs);
  c.free(per);
  c.free(ctr);
  if (hist) c.free(hist);
  SYNCHRO_PROGRESS("  trie node count over %llu sets: %llu nodes", static_cast<unsigned long long>(N64),
                   static_cast<unsigned long long>(h.nodes));
  return h.nodes;
}

u64 trie_node_count(Context& c, const DList& l, u32 min_leaf) { return build_trie(c, l, min_leaf, nullptr); }

u64 trie_shape(Context& c, const DList& l, u32 min_leaf, TrieShape* shape) {
  return build_trie(c, l, min_leaf, shape);
}

u64 build_trie_nodes(Context& c, const DList& l, u32 min_leaf, TrieQueryIndex* qi) {
  return build_trie(c, l, min_leaf, nullptr, qi);
}

}  // namespace synchro::dev
