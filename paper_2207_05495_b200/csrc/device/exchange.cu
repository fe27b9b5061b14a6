// Hash ownership of subsets for the multi-GPU frontier exchange (SURVEY
// §8(e)): every row has an owner rank h(row) mod nranks, so the exact dedupe
// of a level distributed over ranks is local after ONE all-to-all that
// carries each generated row to its owner (distributed.py
// owner_exchange_dedupe; the NCCL collective runs on the caller's side).
//
// owner_partition groups a list owner-major (rows of rank 0 first, ...) with
// warp-aggregated cursor reservations; the order inside an owner's segment is
// unspecified (the receiver's dedupe is set-semantic).  The row hash is the
// one restated in oracle (numpy) by the tests:
//   h = 0x9E3779B97F4A7C15; for each word w: h = (h ^ w) * 0xff51afd7ed558ccd,
//   h ^= h >> 32;  owner = h mod nranks.
#include "dev.hpp"
#include "kernels.cuh"
#include "util.cuh"

namespace synchro::dev {

namespace {

__device__ __forceinline__ u32 owner_of(const u64* __restrict__ row, u32 W, u32 nranks) {
  u64 h = 0x9E3779B97F4A7C15ull;
  for (u32 w = 0; w < W; ++w) {
    h = (h ^ row[w]) * 0xff51afd7ed558ccdull;
    h ^= h >> 32;
  }
  return static_cast<u32>(h % nranks);
}

__global__ void owner_count_kernel(const u64* __restrict__ words, u64 N, u32 W, u32 nranks,
                                   u32* __restrict__ owner, unsigned long long* __restrict__ counts) {
  extern __shared__ unsigned long long sh_counts[];
  for (u32 r = threadIdx.x; r < nranks; r += blockDim.x) sh_counts[r] = 0;
  __syncthreads();
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < N;
       i += static_cast<u64>(gridDim.x) * blockDim.x) {
    const u32 o = owner_of(words + i * W, W, nranks);
    owner[i] = o;
    atomicAdd(&sh_counts[o], 1ull);
  }
  __syncthreads();
  for (u32 r = threadIdx.x; r < nranks; r += blockDim.x)
    if (sh_counts[r]) atomicAdd(&counts[r], sh_counts[r]);
}

__global__ void owner_scatter_kernel(const u64* __restrict__ words, const u32* __restrict__ cards,
                                     const u64* __restrict__ tags, u64 N, u32 W,
                                     const u32* __restrict__ owner,
                                     unsigned long long* __restrict__ cursor,
                                     u64* __restrict__ ow, u32* __restrict__ oc,
                                     u64* __restrict__ ot) {
  const u32 lane = threadIdx.x & 31;
  const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
  for (u64 i0 = blockIdx.x * static_cast<u64>(blockDim.x) + (threadIdx.x & ~31u); i0 < N; i0 += stride) {
    const u64 i = i0 + lane;
    const bool valid = i < N;
    const u32 o = valid ? owner[i] : 0xFFFFFFFFu;
    const unsigned active = __ballot_sync(0xFFFFFFFFu, valid);
    const unsigned peers = __match_any_sync(0xFFFFFFFFu, o) & active;
    unsigned long long base = 0;
    const int leader = __ffs(peers) - 1;
    if (valid && static_cast<int>(lane) == leader) base = atomicAdd(&cursor[o], static_cast<unsigned long long>(__popc(peers)));
    base = __shfl_sync(0xFFFFFFFFu, base, leader < 0 ? 0 : leader);
    if (valid) {
      const u64 dst = base + __popc(peers & ((1u << lane) - 1));
      for (u32 w = 0; w < W; ++w) ow[dst * W + w] = words[i * W + w];
      oc[dst] = cards[i];
      if (tags) ot[dst] = tags[i];
    }
  }
}

}  // namespace

std::vector<u64> owner_partition(Context& c, DList& l, u32 nranks) {
  std::vector<u64> counts(nranks, 0);
  const u64 N = l.size();
  if (N == 0 || nranks == 0) return counts;
  const u32 W = c.W();
  cudaStream_t s = as_stream(c.stream());
  auto* owner = static_cast<u32*>(c.alloc(N * 4));
  auto* cnt = static_cast<unsigned long long*>(c.alloc(static_cast<size_t>(nranks) * 16));
  SW_CUDA(cudaMemsetAsync(cnt, 0, static_cast<size_t>(nranks) * 8, s));
  owner_count_kernel<<<grid_for(N, 256, 148 * 4), 256, nranks * 8, s>>>(l.words, N, W, nranks, owner, cnt);
  SW_CHECK_LAUNCH();
  c.memcpy_d2h(counts.data(), cnt, static_cast<size_t>(nranks) * 8);
  std::vector<u64> start(nranks, 0);
  for (u32 r = 1; r < nranks; ++r) start[r] = start[r - 1] + counts[r - 1];
  c.memcpy_h2d(cnt + nranks, start.data(), static_cast<size_t>(nranks) * 8);
  DList out(&c, N, l.tagged());
  owner_scatter_kernel<<<grid_for(N, 256), 256, 0, s>>>(
      l.words, l.cards, l.tagged() ? l.tags : nullptr, N, W, owner, cnt + nranks, out.words,
      out.cards, l.tagged() ? out.tags : nullptr);
  SW_CHECK_LAUNCH();
  out.set_size(N);
  c.free(owner);
  c.free(cnt);
  c.counters.kernel_launches += 2;
  l = std::move(out);
  return counts;
}

}  // namespace synchro::dev
