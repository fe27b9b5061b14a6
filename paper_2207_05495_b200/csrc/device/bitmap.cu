// Containment over the whole power set, for automata with n <= 20 states.
//
// With n <= 20 every set is a 20-bit number and all of Q's 2^n subsets fit one
// shared-memory bitmap (128 KB).  Each containment question of the search
// (subset_algebra.hpp:138-231: self-reduction, history marking, the meet,
// the superset side of the inverse steps and the DFS window) then becomes one
// single-CTA launch: mark the sets of A in the bitmap, take the subset-OR
// (or superset-OR) transform over the n dimensions — afterwards bit s says
// "some a ⊆ s" (resp. "some a ⊇ s") — and answer every query with at most n
// lookups: y has a proper subset in A iff some y \ {e} has any.  n·2^n bit
// operations replace the radix-tree traversal, whose per-launch overhead and
// index builds dominated the n = 20 solves (Černý C_20: 359 iterations, 179
// self-reductions, 97 history markings).  Set semantics, so sizes are the
// reference's; order of the queries is untouched (keep flags).
#include <algorithm>

#include "dev.hpp"
#include "kernels.cuh"
#include "util.cuh"

namespace synchro::dev {

namespace {

constexpr int kBmThreads = 1024;

// Modes: A-side sets below (subset) or above (superset) the queries.
enum : int { kSubset = 0, kProperSubset = 1, kSuperset = 2, kProperSuperset = 3 };

__device__ __forceinline__ u32 set_index(u64 word, u32 n) { return static_cast<u32>(word >> (64 - n)); }

__device__ __forceinline__ bool bm_get(const u32* bm, u32 i) { return (bm[i >> 5] >> (i & 31)) & 1u; }

// keep[j] = 0 iff B[j] relates to some A set (mode); found/witness: the first
// hit (EXIST), keep may then be null.
template <int MODE, bool EXIST>
__global__ void __launch_bounds__(kBmThreads) bitmap_kernel(const u64* __restrict__ A, u64 na,
                                                            const u64* __restrict__ B, u64 nb,
                                                            u32 n, uint8_t* __restrict__ keep,
                                                            int* found, unsigned long long* wit) {
  extern __shared__ u32 bm[];
  const u32 words = n >= 5 ? (1u << (n - 5)) : 1u;
  for (u32 w = threadIdx.x; w < words; w += blockDim.x) bm[w] = 0;
  __syncthreads();
  for (u64 i = threadIdx.x; i < na; i += blockDim.x) {
    const u32 s = set_index(A[i], n);
    atomicOr(&bm[s >> 5], 1u << (s & 31));
  }
  __syncthreads();
  constexpr bool SUB = MODE == kSubset || MODE == kProperSubset;
  // in-word dimensions 0..4
  constexpr u32 kLow[5] = {0x55555555u, 0x33333333u, 0x0F0F0F0Fu, 0x00FF00FFu, 0x0000FFFFu};
  for (u32 w = threadIdx.x; w < words; w += blockDim.x) {
    u32 x = bm[w];
#pragma unroll
    for (u32 b = 0; b < 5; ++b) {
      if (b >= n) break;
      const u32 sh = 1u << b;
      x |= SUB ? ((x & kLow[b]) << sh) : ((x >> sh) & kLow[b]);
    }
    bm[w] = x;
  }
  __syncthreads();
  // word dimensions 5..n-1
  for (u32 b = 5; b < n; ++b) {
    const u32 d = 1u << (b - 5);
    for (u32 w = threadIdx.x; w < words; w += blockDim.x) {
      if (SUB) {
        if (w & d) bm[w] |= bm[w ^ d];
      } else {
        if (!(w & d)) bm[w] |= bm[w | d];
      }
    }
    __syncthreads();
  }
  for (u64 j = threadIdx.x; j < nb; j += blockDim.x) {
    if (EXIST && *reinterpret_cast<volatile int*>(found)) break;
    const u32 y = set_index(B[j], n);
    bool hit;
    if (MODE == kSubset || MODE == kSuperset) {
      hit = bm_get(bm, y);
    } else if (MODE == kProperSubset) {
      hit = false;
      for (u32 b = 0; b < n && !hit; ++b)
        if (y >> b & 1u) hit = bm_get(bm, y & ~(1u << b));
    } else {
      hit = false;
      for (u32 b = 0; b < n && !hit; ++b)
        if (!(y >> b & 1u)) hit = bm_get(bm, y | (1u << b));
    }
    if (EXIST) {
      if (hit && atomicCAS(found, 0, 1) == 0) wit[1] = j;
    } else {
      keep[j] = hit ? 0 : 1;
    }
  }
}

template <int MODE, bool EXIST>
void launch(Context& c, const DList& A, const DList& B, uint8_t* keep, int* found,
            unsigned long long* wit) {
  const u32 n = c.n();
  const size_t smem = (n >= 5 ? (size_t{1} << (n - 5)) : 1) * 4;
  auto kern = bitmap_kernel<MODE, EXIST>;
  if (smem > 48 * 1024) smem_opt_in(reinterpret_cast<const void*>(kern), static_cast<int>(smem));
  kern<<<1, kBmThreads, smem, as_stream(c.stream())>>>(A.words, A.size(), B.words, B.size(), n, keep,
                                                        found, wit);
  SW_CHECK_LAUNCH();
  c.counters.kernel_launches++;
}

}  // namespace

bool bitmap_fits(const Context& c) { return c.W() == 1 && c.n() <= kBitmapMaxStates; }

void bitmap_keep_flags(Context& c, const DList& A, const DList& B, bool super, bool proper,
                       uint8_t* keep) {
  if (B.empty()) return;
  if (super)
    proper ? launch<kProperSuperset, false>(c, A, B, keep, nullptr, nullptr)
           : launch<kSuperset, false>(c, A, B, keep, nullptr, nullptr);
  else
    proper ? launch<kProperSubset, false>(c, A, B, keep, nullptr, nullptr)
           : launch<kSubset, false>(c, A, B, keep, nullptr, nullptr);
}

bool bitmap_exists_subset(Context& c, const DList& A, const DList& B, size_t* b_index) {
  if (A.empty() || B.empty()) return false;
  struct Res {
    int found;
    int pad;
    unsigned long long wit[2];
  };
  auto* d = static_cast<Res*>(c.scratch(7, 64));
  SW_CUDA(cudaMemsetAsync(d, 0, sizeof(Res), as_stream(c.stream())));
  launch<kSubset, true>(c, A, B, nullptr, &d->found, d->wit);
  Res h;
  c.memcpy_d2h(&h, d, sizeof(Res));
  if (h.found && b_index) *b_index = static_cast<size_t>(h.wit[1]);
  return h.found != 0;
}

}  // namespace synchro::dev
