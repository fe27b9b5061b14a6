// All-pairs containment for small lists.  Below ~2^24 pair tests the whole
// question is one launch over (A tile in shared memory) × (one query per
// thread) — no radix tree, no relabelling sort, no superset-join buckets, no
// host round trip.  The index paths cost 20-40 launches and several
// synchronisations per call, which is what a small solve (config 2: lists of
// a few thousand sets, 12-16 iterations) spends its time on.
//
// Relations (card filters first, then the word test):
//   SUPER = false:  x ⊆ y   (PROPER: x ⊊ y, i.e. also |x| < |y|)
//   SUPER = true:   y ⊆ x   (PROPER: y ⊊ x)
// The marked set does not depend on the order of the pair tests, so results
// equal the index paths' bit for bit.
#include "dev.hpp"
#include "kernels.cuh"
#include "util.cuh"

namespace synchro::dev {

namespace {

constexpr int kBruteThreads = 256;

template <int W, bool SUPER, bool PROPER, bool EXIST>
__global__ void __launch_bounds__(kBruteThreads) brute_kernel(
    const u64* __restrict__ A, const u32* __restrict__ ac, u32 na, const u64* __restrict__ B,
    const u32* __restrict__ bc, u32 nb, u32 chunk, uint8_t* keep, int* found,
    unsigned long long* wit) {
  __shared__ u64 sa[kBruteThreads * W];
  __shared__ u32 sc[kBruteThreads];
  __shared__ int s_stop;
  const u32 j = blockIdx.x * kBruteThreads + threadIdx.x;
  const bool valid = j < nb;
  u64 y[W];
  u32 cy = 0;
#pragma unroll
  for (int w = 0; w < W; ++w) y[w] = valid ? B[static_cast<u64>(j) * W + w] : 0;
  if (valid) cy = bc[j];
  const u32 lo = blockIdx.y * chunk, hi = min(na, lo + chunk);
  bool hit = false;
  u32 hit_i = 0;
  for (u32 t = lo; t < hi; t += kBruteThreads) {
    const u32 cnt = min(static_cast<u32>(kBruteThreads), hi - t);
    __syncthreads();
    if (threadIdx.x == 0) s_stop = EXIST ? *reinterpret_cast<volatile int*>(found) : 0;
    for (u32 e = threadIdx.x; e < cnt * W; e += kBruteThreads) sa[e] = A[static_cast<u64>(t) * W + e];
    if (threadIdx.x < cnt) sc[threadIdx.x] = ac[t + threadIdx.x];
    __syncthreads();
    if (EXIST && s_stop) break;
    if (!valid || hit) continue;
    for (u32 i = 0; i < cnt; ++i) {
      const u32 cx = sc[i];
      const bool card_ok = SUPER ? (PROPER ? cy < cx : cy <= cx) : (PROPER ? cx < cy : cx <= cy);
      if (!card_ok) continue;
      u64 acc = 0;
#pragma unroll
      for (int w = 0; w < W; ++w) acc |= SUPER ? (y[w] & ~sa[i * W + w]) : (sa[i * W + w] & ~y[w]);
      if (acc == 0) {
        hit = true;
        hit_i = t + i;
        break;
      }
    }
  }
  if (!valid || !hit) return;
  if (EXIST) {
    if (atomicCAS(found, 0, 1) == 0) {
      wit[0] = hit_i;
      wit[1] = j;
    }
  } else {
    keep[j] = 0;
  }
}

struct Grid {
  dim3 grid;
  u32 chunk;
};

// One query per thread; when there are few query blocks, A is split across
// gridDim.y so the launch still covers the SMs.
Grid brute_grid(u64 na, u64 nb) {
  const u32 xb = static_cast<u32>((nb + kBruteThreads - 1) / kBruteThreads);
  const u32 a_tiles = static_cast<u32>((na + kBruteThreads - 1) / kBruteThreads);
  u32 yb = std::max<u32>(1, std::min<u32>(a_tiles, (2 * 148 + xb - 1) / xb));
  const u32 chunk = static_cast<u32>(((a_tiles + yb - 1) / yb) * kBruteThreads);
  yb = static_cast<u32>((na + chunk - 1) / chunk);
  return {dim3(xb, std::max<u32>(1, yb)), chunk};
}

}  // namespace

bool brute_fits(size_t na, size_t nb) {
  return na > 0 && nb > 0 && static_cast<double>(na) * static_cast<double>(nb) <= kBrutePairs &&
         na < 0xFFFFFFFFull && nb < 0xFFFFFFFFull;
}

void brute_keep_flags(Context& c, const DList& A, const DList& B, bool super, bool proper,
                      uint8_t* keep) {
  cudaStream_t s = as_stream(c.stream());
  if (B.empty()) return;
  SW_CUDA(cudaMemsetAsync(keep, 1, B.size(), s));
  if (A.empty()) return;
  const Grid g = brute_grid(A.size(), B.size());
  const u32 na = static_cast<u32>(A.size()), nb = static_cast<u32>(B.size());
  SW_DISPATCH_W(c.W(), {
    if (super && proper)
      brute_kernel<W, true, true, false><<<g.grid, kBruteThreads, 0, s>>>(
          A.words, A.cards, na, B.words, B.cards, nb, g.chunk, keep, nullptr, nullptr);
    else if (super)
      brute_kernel<W, true, false, false><<<g.grid, kBruteThreads, 0, s>>>(
          A.words, A.cards, na, B.words, B.cards, nb, g.chunk, keep, nullptr, nullptr);
    else if (proper)
      brute_kernel<W, false, true, false><<<g.grid, kBruteThreads, 0, s>>>(
          A.words, A.cards, na, B.words, B.cards, nb, g.chunk, keep, nullptr, nullptr);
    else
      brute_kernel<W, false, false, false><<<g.grid, kBruteThreads, 0, s>>>(
          A.words, A.cards, na, B.words, B.cards, nb, g.chunk, keep, nullptr, nullptr);
  });
  SW_CHECK_LAUNCH();
  c.counters.kernel_launches += 1;
}

bool brute_exists_subset(Context& c, const DList& A, const DList& B, Witness* w) {
  if (A.empty() || B.empty()) return false;
  cudaStream_t s = as_stream(c.stream());
  struct Res {
    int found;
    int pad;
    unsigned long long wit[2];
  };
  auto* d = static_cast<Res*>(c.scratch(7, 64));
  SW_CUDA(cudaMemsetAsync(d, 0, sizeof(Res), s));
  const Grid g = brute_grid(A.size(), B.size());
  SW_DISPATCH_W(c.W(), {
    brute_kernel<W, false, false, true><<<g.grid, kBruteThreads, 0, s>>>(
        A.words, A.cards, static_cast<u32>(A.size()), B.words, B.cards,
        static_cast<u32>(B.size()), g.chunk, nullptr, &d->found, d->wit);
  });
  SW_CHECK_LAUNCH();
  c.counters.kernel_launches += 1;
  Res h;
  c.memcpy_d2h(&h, d, sizeof(Res));
  if (h.found && w) {
    w->a_index = h.wit[0];
    w->b_index = h.wit[1];
  }
  return h.found != 0;
}

}  // namespace synchro::dev
