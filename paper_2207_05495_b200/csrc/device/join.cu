// Bucketed superset join: for every query y, is there an x in X with y ⊆ x
// (proper: y ⊊ x)?  The B200 path for the reference's marking on DENSE
// (complemented) lists — IBFS self-reduction (subset_algebra.hpp:179-197 on
// complements, bibfs_engine.hpp:216-220), IBFS history marking (:223-226) and
// the DFS window (dfs_phase.hpp:107-128) — rephrased on the plain sparse sets.
//
// On complements the radix-tree traversal degenerates to near brute force
// (the reference measured ≈N²/4.6 pair checks; our tree ≈0.3·N per query at
// n=300), because a dense query branches at almost every split.  In plain
// space the question is a superset query, and every x ⊇ y contains y's
// rarest state r(y).  So:
//   1. hist = per-state counts over X (bit-sliced);
//   2. r(y) = the state of y with the fewest X-sets (ties: smallest index),
//      found by probing the states in ascending-count order;
//   3. candidate buckets C_r = {x ∋ r}, sorted by |x| descending (one radix
//      sort of (r, ~|x|) keys over the needed buckets);
//   4. queries sorted by (r(y), |y|); one CTA per 128 queries of a bucket
//      streams the bucket's candidate rows through shared memory, each thread
//      testing its y (registers) against every staged row, stopping at the
//      first hit or once |x| can no longer exceed |y| (card-descending order).
// Work is Σ_y |C_r(y)| row tests ≈ N·min-frequency instead of ≈N per query.
#include <cub/cub.cuh>

#include <algorithm>
#include <numeric>
#include <vector>

#include "../progress.hpp"
#include "dev.hpp"
#include "kernels.cuh"
#include "util.cuh"

namespace synchro::dev {

namespace {

constexpr int kJoinThreads = 128;  // queries per CTA
constexpr int kJoinTile = 128;     // candidate rows staged per pass

// r(y) and the sort key (r << 11 | |y|) of every query (r = n for y = ∅), by
// probing the states in ascending X-frequency order (ties: smaller state
// first) until y holds one — the first hit is y's rarest state.  For
// the dense queries of the DFS window (a third of the states) that is a few
// probes instead of a walk over every set bit.
template <int W>
__global__ void rarest_probe_kernel(const u64* __restrict__ Y, const u32* __restrict__ Ycard,
                                    u64 ny, u32 n, const uint16_t* __restrict__ g_order,
                                    u32* __restrict__ key, u32* __restrict__ idx) {
  extern __shared__ uint16_t s_order[];
  for (u32 i = threadIdx.x; i < n; i += blockDim.x) s_order[i] = g_order[i];
  __syncthreads();
  for (u64 j = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; j < ny;
       j += static_cast<u64>(gridDim.x) * blockDim.x) {
    u32 best = n;
    if (Ycard[j])
      for (u32 i = 0; i < n; ++i) {
        const u32 q = s_order[i];
        if ((__ldg(Y + j * W + (q >> 6)) >> (63 - (q & 63))) & 1) {
          best = q;
          break;
        }
      }
    key[j] = (best << 11) | min(Ycard[j], 2047u);
    idx[j] = static_cast<u32>(j);
  }
}

// Query range of every bucket in the (r, |y|)-sorted keys (lo[r], hi[r]).
__global__ void bucket_bounds_kernel(const u32* __restrict__ key, u64 ny, u32* __restrict__ lo,
                                     u32* __restrict__ hi) {
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < ny;
       i += static_cast<u64>(gridDim.x) * blockDim.x) {
    const u32 r = key[i] >> 11;
    if (i == 0 || (key[i - 1] >> 11) != r) lo[r] = static_cast<u32>(i);
    if (i + 1 == ny || (key[i + 1] >> 11) != r) hi[r] = static_cast<u32>(i + 1);
  }
}

// Number of needed buckets each x belongs to.
template <int W>
__global__ void member_count_kernel(const u64* __restrict__ X, u64 nx, const uint8_t* __restrict__ need,
                                    u32* __restrict__ cnt) {
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < nx;
       i += static_cast<u64>(gridDim.x) * blockDim.x) {
    u32 c = 0;
#pragma unroll
    for (int w = 0; w < W; ++w) {
      u64 bits = X[i * W + w];
      while (bits) {
        const int b = __clzll(bits);
        bits &= ~(u64{1} << (63 - b));
        c += need[w * 64 + b];
      }
    }
    cnt[i] = c;
  }
}

// Emit (bucket << 11 | (2047 - |x|), x) for every needed bucket of x.
template <int W>
__global__ void member_emit_kernel(const u64* __restrict__ X, const u32* __restrict__ Xcard, u64 nx,
                                   const uint8_t* __restrict__ need, const u32* __restrict__ off,
                                   u32* __restrict__ key, u32* __restrict__ val) {
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < nx;
       i += static_cast<u64>(gridDim.x) * blockDim.x) {
    u32 o = off[i];
    const u32 cdesc = 2047u - min(Xcard[i], 2047u);
#pragma unroll
    for (int w = 0; w < W; ++w) {
      u64 bits = X[i * W + w];
      while (bits) {
        const int b = __clzll(bits);
        bits &= ~(u64{1} << (63 - b));
        const u32 q = w * 64 + b;
        if (need[q]) {
          key[o] = (q << 11) | cdesc;
          val[o] = static_cast<u32>(i);
          ++o;
        }
      }
    }
  }
}

struct JoinBlock {
  u32 q_lo, q_hi;  // query range (in sorted order) of this CTA
  u32 c_lo, c_hi;  // candidate range of its bucket
};

// Projection of a row on up to 64 states (bit i = the row holds pstate[i]):
// y ⊆ x implies proj(y) ⊆ proj(x), so a one-word test rejects most candidate
// pairs before the W-word comparison.  The states are the ones rarest in X
// (a query holding one of them fits few candidates).
template <int W>
__global__ void project_kernel(const u64* __restrict__ rows, u64 count,
                               const uint16_t* __restrict__ pstate, u32 np, u64* __restrict__ proj) {
  __shared__ uint16_t sp[64];
  if (threadIdx.x < np) sp[threadIdx.x] = pstate[threadIdx.x];
  __syncthreads();
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<u64>(gridDim.x) * blockDim.x) {
    const u64* r = rows + i * W;
    u64 p = 0;
    for (u32 b = 0; b < np; ++b) {
      const u32 q = sp[b];
      p |= ((r[q >> 6] >> (63 - (q & 63))) & 1ull) << b;
    }
    proj[i] = p;
  }
}

template <int W, bool PROPER>
__global__ void __launch_bounds__(kJoinThreads) superset_join_kernel(
    const u64* __restrict__ X, const u32* __restrict__ Xcard, const u64* __restrict__ Y,
    const u32* __restrict__ Ycard, const u32* __restrict__ qidx, const u32* __restrict__ cval,
    const JoinBlock* __restrict__ blocks, const u64* __restrict__ Xproj,
    const u64* __restrict__ Yproj, uint8_t* __restrict__ keep) {
  __shared__ u64 s_rows[kJoinTile][W];
  __shared__ u32 s_card[kJoinTile];
  __shared__ u64 s_proj[kJoinTile];
  const JoinBlock jb = blocks[blockIdx.x];
  const u32 t = threadIdx.x;
  const bool have = jb.q_lo + t < jb.q_hi;
  u32 j = 0, cy = 0;
  u64 y[W], py = 0;
#pragma unroll
  for (int w = 0; w < W; ++w) y[w] = 0;
  if (have) {
    j = qidx[jb.q_lo + t];
    cy = Ycard[j];
    py = Yproj[j];
#pragma unroll
    for (int w = 0; w < W; ++w) y[w] = Y[static_cast<u64>(j) * W + w];
  }
  bool active = have, hit = false;
  for (u32 base = jb.c_lo; base < jb.c_hi; base += kJoinTile) {
    if (!__syncthreads_or(active)) break;
    const u32 cnt = min(static_cast<u32>(kJoinTile), jb.c_hi - base);
    for (u32 r = t; r < cnt; r += kJoinThreads) {
      const u32 x = cval[base + r];
      s_card[r] = Xcard[x];
      s_proj[r] = Xproj[x];
#pragma unroll
      for (int w = 0; w < W; ++w) s_rows[r][w] = X[static_cast<u64>(x) * W + w];
    }
    __syncthreads();
    if (active) {
      for (u32 r = 0; r < cnt; ++r) {
        const u32 cx = s_card[r];
        if (PROPER ? cx <= cy : cx < cy) {  // card-descending: nothing further can contain y
          active = false;
          break;
        }
        if (py & ~s_proj[r]) continue;  // a projected state of y is missing from x
        u64 bad = 0;
#pragma unroll
        for (int w = 0; w < W; ++w) bad |= y[w] & ~s_rows[r][w];
        if (!bad) {
          hit = true;
          active = false;
          break;
        }
      }
    }
    __syncthreads();
  }
  if (have) keep[j] = hit ? 0 : 1;
}

__global__ void empty_query_kernel(const u32* __restrict__ Ycard, u64 ny, uint8_t* keep, int any_fit) {
  for (u64 j = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; j < ny;
       j += static_cast<u64>(gridDim.x) * blockDim.x)
    if (Ycard[j] == 0) keep[j] = any_fit ? 0 : 1;
}

}  // namespace

void superset_keep_flags(Context& c, const DList& X, const DList& Y, bool proper, uint8_t* keep) {
  const u64 ny = Y.size(), nx = X.size();
  cudaStream_t s = as_stream(c.stream());
  if (!ny) return;
  if (bitmap_fits(c)) {  // n <= 20: the power-set bitmap
    if (!nx) {
      SW_CUDA(cudaMemsetAsync(keep, 1, ny, s));
      return;
    }
    bitmap_keep_flags(c, X, Y, /*super=*/true, proper, keep);
    return;
  }
  if (brute_fits(nx, ny)) {  // small lists: one all-pairs launch
    brute_keep_flags(c, X, Y, /*super=*/true, proper, keep);
    return;
  }
  SW_CUDA(cudaMemsetAsync(keep, 1, ny, s));
  if (!nx) return;
  const u32 n = c.n();
  std::unique_ptr<StreamTimer> timer;
  if (progress_enabled()) {
    timer = std::make_unique<StreamTimer>(c);
    timer->start();
  }
  // 1. per-state counts over X, and the states in ascending-count order
  u32* hist = static_cast<u32*>(c.alloc(n * 4));
  state_histogram(c, X, hist);
  std::vector<u32> hhist(n);
  c.memcpy_d2h(hhist.data(), hist, n * 4);
  std::vector<uint16_t> order(n);
  std::iota(order.begin(), order.end(), static_cast<uint16_t>(0));
  std::stable_sort(order.begin(), order.end(),
                   [&](uint16_t a, uint16_t b) { return hhist[a] < hhist[b]; });
  uint16_t* dorder = static_cast<uint16_t*>(c.alloc(n * 2));
  c.memcpy_h2d(dorder, order.data(), n * 2);
  // projection states: the (up to) 64 rarest states that some x holds
  std::vector<uint16_t> pst;
  for (u32 i = 0; i < n && pst.size() < 64; ++i)
    if (hhist[order[i]] > 0) pst.push_back(order[i]);
  uint16_t* dpst = static_cast<uint16_t*>(c.alloc(64 * 2));
  if (!pst.empty()) c.memcpy_h2d(dpst, pst.data(), pst.size() * 2);
  u64* xproj = static_cast<u64*>(c.alloc(nx * 8));
  u64* yproj = static_cast<u64*>(c.alloc(ny * 8));
  SW_DISPATCH_W(c.W(), {
    project_kernel<W><<<grid_for(nx, 256), 256, 0, s>>>(X.words, nx, dpst,
                                                        static_cast<u32>(pst.size()), xproj);
    project_kernel<W><<<grid_for(ny, 256), 256, 0, s>>>(Y.words, ny, dpst,
                                                        static_cast<u32>(pst.size()), yproj);
  });
  SW_CHECK_LAUNCH();
  // 2. rarest state of every query; sort queries by (r, |y|)
  u32* qkey = static_cast<u32*>(c.alloc(ny * 4));
  u32* qkey2 = static_cast<u32*>(c.alloc(ny * 4));
  u32* qidx = static_cast<u32*>(c.alloc(ny * 4));
  u32* qidx2 = static_cast<u32*>(c.alloc(ny * 4));
  SW_DISPATCH_W(c.W(), {
    rarest_probe_kernel<W><<<grid_for(ny, 256), 256, n * 2, s>>>(Y.words, Y.cards, ny, n, dorder,
                                                                  qkey, qidx);
  });
  SW_CHECK_LAUNCH();
  int keybits = 11;
  while ((1u << (keybits - 11)) <= n) ++keybits;
  {
    cub::DoubleBuffer<u32> k(qkey, qkey2), v(qidx, qidx2);
    size_t tb = 0;
    SW_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, k, v, static_cast<int>(ny), 0, keybits, s));
    void* tmp = c.alloc(tb);
    SW_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, k, v, static_cast<int>(ny), 0, keybits, s));
    c.free(tmp);
    qkey = k.Current();
    qidx = v.Current();
    qkey2 = k.Alternate();
    qidx2 = v.Alternate();
  }
  // per-bucket query ranges (device; n + 1 buckets come back)
  std::vector<u32> qlo(n + 1, 0), qhi(n + 1, 0);
  {
    u32* dlh = static_cast<u32*>(c.alloc(2ull * (n + 1) * 4));
    SW_CUDA(cudaMemsetAsync(dlh, 0, 2ull * (n + 1) * 4, s));
    bucket_bounds_kernel<<<grid_for(ny, 256), 256, 0, s>>>(qkey, ny, dlh, dlh + n + 1);
    SW_CHECK_LAUNCH();
    std::vector<u32> h(2ull * (n + 1));
    c.memcpy_d2h(h.data(), dlh, h.size() * 4);
    c.free(dlh);
    for (u32 r = 0; r <= n; ++r) {
      qlo[r] = h[r];
      qhi[r] = h[n + 1 + r];
    }
  }
  std::vector<uint8_t> need(n, 0);
  for (u32 r = 0; r < n; ++r) need[r] = (qhi[r] > qlo[r] && hhist[r] > 0) ? 1 : 0;
  // 3. candidate buckets: (bucket, card desc) keys over the needed buckets
  uint8_t* dneed = static_cast<uint8_t*>(c.alloc(n));
  c.memcpy_h2d(dneed, need.data(), n);
  u32* mcnt = static_cast<u32*>(c.alloc((nx + 1) * 4));
  u32* moff = static_cast<u32*>(c.alloc((nx + 1) * 4));
  SW_DISPATCH_W(c.W(), {
    member_count_kernel<W><<<grid_for(nx, 256), 256, 0, s>>>(X.words, nx, dneed, mcnt);
  });
  {
    size_t tb = 0;
    SW_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, mcnt, moff, static_cast<int>(nx + 1), s));
    void* tmp = c.alloc(tb);
    SW_CUDA(cudaMemsetAsync(mcnt + nx, 0, 4, s));
    SW_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, mcnt, moff, static_cast<int>(nx + 1), s));
    c.free(tmp);
  }
  u32 total = 0;
  c.memcpy_d2h(&total, moff + nx, 4);
  std::vector<u32> clo(n, 0), chi(n, 0);
  u32* ckey = nullptr;
  u32* cval = nullptr;
  if (total) {
    ckey = static_cast<u32*>(c.alloc(total * 4ull));
    cval = static_cast<u32*>(c.alloc(total * 4ull));
    u32* ckey2 = static_cast<u32*>(c.alloc(total * 4ull));
    u32* cval2 = static_cast<u32*>(c.alloc(total * 4ull));
    SW_DISPATCH_W(c.W(), {
      member_emit_kernel<W><<<grid_for(nx, 256), 256, 0, s>>>(X.words, X.cards, nx, dneed, moff, ckey, cval);
    });
    SW_CHECK_LAUNCH();
    cub::DoubleBuffer<u32> k(ckey, ckey2), v(cval, cval2);
    size_t tb = 0;
    SW_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, k, v, static_cast<int>(total), 0, keybits, s));
    void* tmp = c.alloc(tb);
    SW_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, k, v, static_cast<int>(total), 0, keybits, s));
    c.free(tmp);
    ckey = k.Current();
    cval = v.Current();
    c.free(k.Alternate());
    c.free(v.Alternate());
    // bucket ranges: bucket sizes are the histogram counts of the needed buckets
    u32 o = 0;
    for (u32 r = 0; r < n; ++r)
      if (need[r]) {
        clo[r] = o;
        o += hhist[r];
        chi[r] = o;
      }
  }
  // 4. one CTA per kJoinThreads queries of a bucket
  std::vector<JoinBlock> blocks;
  for (u32 r = 0; r < n; ++r)
    if (need[r])
      for (u32 q = qlo[r]; q < qhi[r]; q += kJoinThreads)
        blocks.push_back({q, std::min(qhi[r], q + kJoinThreads), clo[r], chi[r]});
  if (!blocks.empty()) {
    JoinBlock* dblocks = static_cast<JoinBlock*>(c.alloc(blocks.size() * sizeof(JoinBlock)));
    c.memcpy_h2d(dblocks, blocks.data(), blocks.size() * sizeof(JoinBlock));
    SW_DISPATCH_W(c.W(), {
      if (proper)
        superset_join_kernel<W, true><<<static_cast<unsigned>(blocks.size()), kJoinThreads, 0, s>>>(
            X.words, X.cards, Y.words, Y.cards, qidx, cval, dblocks, xproj, yproj, keep);
      else
        superset_join_kernel<W, false><<<static_cast<unsigned>(blocks.size()), kJoinThreads, 0, s>>>(
            X.words, X.cards, Y.words, Y.cards, qidx, cval, dblocks, xproj, yproj, keep);
    });
    SW_CHECK_LAUNCH();
    c.free(dblocks);
  }
  // empty queries: ∅ ⊆ every x; ∅ ⊊ x iff x ≠ ∅
  if (qhi[n] > qlo[n]) {
    const ListStats xs = stats(c, X);
    const int any_fit = proper ? (xs.max_card > 0) : 1;
    empty_query_kernel<<<grid_for(ny, 256), 256, 0, s>>>(Y.cards, ny, keep, any_fit);
    SW_CHECK_LAUNCH();
  }
  c.counters.kernel_launches += 10;
  c.free(dpst);
  c.free(xproj);
  c.free(yproj);
  c.free(hist);
  c.free(dorder);
  c.free(qkey);
  c.free(qkey2);
  c.free(qidx);
  c.free(qidx2);
  c.free(dneed);
  c.free(mcnt);
  c.free(moff);
  if (ckey) c.free(ckey);
  if (cval) c.free(cval);
  if (timer)
    SYNCHRO_PROGRESS("  superset-join%s |X|=%llu |Y|=%llu candidates=%u blocks=%zu %.3f ms",
                     proper ? "-proper" : "", static_cast<unsigned long long>(nx),
                     static_cast<unsigned long long>(ny), total, blocks.size(), timer->stop_ms());
}

size_t remove_subsets_of(Context& c, const DList& X, DList& Y, bool proper) {
  if (Y.empty() || X.empty()) return 0;
  const size_t before = Y.size();
  auto* keep = static_cast<uint8_t*>(c.scratch(5, Y.size()));
  superset_keep_flags(c, X, Y, proper, keep);
  return before - compact_flags(c, Y, keep, nullptr);
}

size_t self_reduce_maximal(Context& c, DList& l) {
  if (l.size() <= 1) return 0;
  const size_t before = l.size();
  auto* keep = static_cast<uint8_t*>(c.scratch(5, l.size()));
  superset_keep_flags(c, l, l, /*proper=*/true, keep);
  return before - compact_flags(c, l, keep, nullptr);
}

}  // namespace synchro::dev
