// Pair-automaton BFS on the GPU: the shortest word merging each unordered
// pair {p, q} (automaton.hpp:119-157 is_synchronizing, heuristics.hpp:26-79
// Eppstein's greedy).  Inverse breadth-first search from the diagonal over the
// pair graph: level d's frontier pairs (u, v) reach, for every letter a, the
// pairs {x, y} with x in δ⁻¹(u, a) and y in δ⁻¹(v, a); the first claim of a
// pair (atomicCAS on its distance) sets d + 1 and appends it to the next
// frontier.  Distances are BFS levels, so they do not depend on the claim
// order: the table equals the host's level-synchronous one
// (automaton.cpp pair_merge_distances) entry for entry.
//
// Layout: distances u32[n(n+1)/2] at q(q+1)/2 + p (p <= q, automaton.hpp
// pair_index); frontier entries are packed (p << 16 | q) (n <= 1024); the
// inverse transitions as a CSR (offsets u32[k·n+1] at a·n+q, sources u16).
#include <limits>
#include <vector>

#include "dev.hpp"
#include "kernels.cuh"
#include "util.cuh"

namespace synchro::dev {

namespace {

constexpr u32 kInf = 0xFFFFFFFFu;

__device__ __forceinline__ u64 tri(u32 p, u32 q) { return static_cast<u64>(q) * (q + 1) / 2 + p; }

// One thread per (frontier pair, letter).
__global__ void pair_level_kernel(const u32* __restrict__ frontier, u32 nf, u32 k, u32 n,
                                  const u32* __restrict__ off, const uint16_t* __restrict__ src,
                                  u32 d, u32* __restrict__ dist, u32* __restrict__ next,
                                  u32* __restrict__ next_count) {
  const u64 total = static_cast<u64>(nf) * k;
  for (u64 t0 = blockIdx.x * static_cast<u64>(blockDim.x); t0 < total;
       t0 += static_cast<u64>(gridDim.x) * blockDim.x) {
    const u64 t = t0 + threadIdx.x;
    if (t < total) {
      const u32 f = frontier[t / k], a = static_cast<u32>(t % k);
      const u32 u = f >> 16, v = f & 0xFFFFu;
      const u32 ub = off[a * n + u], ue = off[a * n + u + 1];
      const u32 vb = off[a * n + v], ve = off[a * n + v + 1];
      for (u32 i = ub; i < ue; ++i)
        for (u32 j = vb; j < ve; ++j) {
          const u32 x = src[i], y = src[j];
          const u32 p = x < y ? x : y, q = x < y ? y : x;
          if (dist[tri(p, q)] != kInf) continue;  // cheap pre-check, then claim
          if (atomicCAS(&dist[tri(p, q)], kInf, d + 1) == kInf) {
            const u32 slot = atomicAdd(next_count, 1u);
            next[slot] = (p << 16) | q;
          }
        }
    }
  }
}

__global__ void pair_init_kernel(u32* dist, u64 npairs, u32 n, u32* frontier) {
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < npairs;
       i += static_cast<u64>(gridDim.x) * blockDim.x)
    dist[i] = kInf;
  for (u32 q = blockIdx.x * blockDim.x + threadIdx.x; q < n; q += gridDim.x * blockDim.x)
    frontier[q] = (q << 16) | q;
}

__global__ void pair_diag_kernel(u32* dist, u32 n) {
  for (u32 q = blockIdx.x * blockDim.x + threadIdx.x; q < n; q += gridDim.x * blockDim.x)
    dist[tri(q, q)] = 0;
}

}  // namespace

std::vector<u32> pair_distances(Context& c, const Automaton& aut) {
  const u32 n = aut.state_count(), k = aut.alphabet_size();
  if (n > 1024) throw std::invalid_argument("pair_distances: n > 1024");
  const u64 npairs = static_cast<u64>(n) * (n + 1) / 2;
  // inverse transitions, CSR by (letter, target)
  std::vector<u32> off(static_cast<size_t>(k) * n + 1, 0);
  std::vector<uint16_t> src(static_cast<size_t>(k) * n);
  for (u32 a = 0; a < k; ++a)
    for (u32 q = 0; q < n; ++q) ++off[static_cast<size_t>(a) * n + aut.next(q, a) + 1];
  for (size_t i = 1; i < off.size(); ++i) off[i] += off[i - 1];
  {
    std::vector<u32> fill(off.begin(), off.end() - 1);
    for (u32 a = 0; a < k; ++a)
      for (u32 q = 0; q < n; ++q)  // sources in increasing state order
        src[fill[static_cast<size_t>(a) * n + aut.next(q, a)]++] = static_cast<uint16_t>(q);
  }
  cudaStream_t s = as_stream(c.stream());
  auto* d_off = static_cast<u32*>(c.alloc(off.size() * 4));
  auto* d_src = static_cast<uint16_t*>(c.alloc(src.size() * 2));
  c.memcpy_h2d(d_off, off.data(), off.size() * 4);
  c.memcpy_h2d(d_src, src.data(), src.size() * 2);
  auto* dist = static_cast<u32*>(c.alloc(npairs * 4));
  auto* fa = static_cast<u32*>(c.alloc(npairs * 4));
  auto* fb = static_cast<u32*>(c.alloc(npairs * 4));
  auto* cnt = static_cast<u32*>(c.scratch(7, 64));
  pair_init_kernel<<<grid_for(npairs, 256), 256, 0, s>>>(dist, npairs, n, fa);
  pair_diag_kernel<<<grid_for(n, 256), 256, 0, s>>>(dist, n);
  SW_CHECK_LAUNCH();
  c.counters.kernel_launches += 2;
  u32 nf = n;
  for (u32 d = 0; nf > 0; ++d) {
    SW_CUDA(cudaMemsetAsync(cnt, 0, 4, s));
    pair_level_kernel<<<grid_for(static_cast<u64>(nf) * k, 256), 256, 0, s>>>(
        fa, nf, k, n, d_off, d_src, d, dist, fb, cnt);
    SW_CHECK_LAUNCH();
    c.counters.kernel_launches++;
    c.memcpy_d2h(&nf, cnt, 4);
    std::swap(fa, fb);
  }
  std::vector<u32> out(npairs);
  c.memcpy_d2h(out.data(), dist, npairs * 4);
  c.free(d_off);
  c.free(d_src);
  c.free(dist);
  c.free(fa);
  c.free(fb);
  static_assert(std::numeric_limits<u32>::max() == kInf, "unreachable pairs are UINT32_MAX");
  return out;
}

}  // namespace synchro::dev
