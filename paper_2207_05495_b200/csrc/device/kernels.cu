// Streaming kernels of the data plane: subset expansion (image / preimage),
// complement, list statistics and order-preserving warp-ballot compaction.
#include <cub/cub.cuh>

#include "dev.hpp"
#include "kernels.cuh"
#include "util.cuh"

namespace synchro::dev {

// ------------------------------------------------------ bit-sliced expansion
// A warp takes 64 parents at a time and transposes them into per-state bit
// slices (slice[q] bit 63-i = "parent i contains q", a 64x64 bit transpose per
// word done with 5 shuffle stages), so both actions become word-wide gathers
// over 64 sets at once:
//   preimage  out[p] = slice[delta(p,a)]                       (1 load / state)
//   image     out[t] = OR_{q : delta(q,a) = t} slice[q]         (CSR of delta^-1)
// and transposes the result back into child rows.  Lane l computes exactly
// the output slices 64w+l and 64w+32+l it needs for the inverse transpose,
// so outputs never leave registers.  ~10 warp-instructions per child instead
// of a divergent per-lane loop over set bits.  (transpose64: util.cuh)

constexpr int kSliceWarps = 4;
constexpr size_t kStageSmemLimit = 200 * 1024;

// Per-warp slice block: 64W slices (+ pad, keeps 16-byte alignment).
template <int W>
constexpr u32 slice_stride() {
  return 64 * W + 2;
}

// Shared memory of the sliced kernel, per warp: the input slices (preimage,
// and the image at W > 6 — below that lane l scatters the slices 64w + l and
// 64w + 32 + l it already holds from its transposes, straight from registers);
// STAGED: a staging area + 64·k cards; then the table (u16 delta).  The staging area
// takes the parents on the way in and the children on the way out, either
//   rows           64 parents at stride kW|1 words, a parent's k children
//                  side by side (+ separate output slices for the image), or
//   letter blocks  (image, W >= 3) k blocks of 64 rows at stride W|1, one
//                  letter's children each; letter a's output slices live in
//                  block a until its children overwrite them — 8.2 instead of
//                  11.3 KB per warp at W=5, k=2 (n=300 image 0.86 -> 0.80 ms,
//                  n=570 2.43 -> 1.62 ms).
//
// (Measured alternative, dropped: the image as a gather over a per-letter,
// bank-aware schedule of the inverse (targets in 32-lane groups by
// in-degree, register accumulators, one store per target) — fewer shared
// wavefronts than the atomicOr scatter but more instructions and dependent
// load chains: 0.99 vs 0.86 ms for 2^24 parents at n=300.)
template <int W>
constexpr bool letter_blocks(bool inverse) {  // measured: W = 2 image and the preimage prefer rows
  return !inverse && W >= 3;
}

template <int W>
static size_t sliced_smem(u32 k, u32 n, bool staged, bool inverse) {
  // input slices (the image at W <= 6 keeps them in registers)
  size_t per_warp = (inverse || W > 6) ? slice_stride<W>() * sizeof(u64) : 0;
  if (staged)
    per_warp += (letter_blocks<W>(inverse) ? static_cast<size_t>(k) * (64 * (W | 1) + 4)
                                           : static_cast<size_t>(64) * ((k * W) | 1)) *
                    sizeof(u64) +
                64 * k * sizeof(u32);
  if (!inverse && !(staged && letter_blocks<W>(inverse))) per_warp += slice_stride<W>() * sizeof(u64);
  const size_t table = static_cast<size_t>(k) * n * 2;
  return kSliceWarps * per_warp + ((table + 15) & ~size_t{15});
}

// STAGED: the warp's 64 parents arrive as one contiguous block and its 64·k
// children — contiguous in the output because child o = i·k + a — leave as
// one block, with 16-byte global accesses for full batches (8-byte ones for
// the tail, or when the slice start leaves the rows 8-byte aligned).  Staged
// rows sit at an ODD stride in words (W|1), so the lanes' row-strided 8-byte
// accesses hit 16 distinct bank pairs (2 wavefronts, the minimum).
// Unstaged (large k·W only): rows are read and written directly by lanes.
// Register caps via minimum blocks per SM (4-warp blocks), measured on 2^24
// parents: preimage 6 (<= 80 registers); image 6 at W <= 2, else 5 (<= 96:
// the image holds its 2W input slices and 2W output slices in registers;
// n=300 image 0.77 -> 0.75 ms at 5, n=100 0.32 -> 0.35 ms).
template <int W, bool INV, bool STAGED>
__global__ void __launch_bounds__(kSliceWarps * 32, (INV || W <= 2) ? 6 : 5)
    expand_sliced_kernel(
    const u64* __restrict__ src, u64 lo, u64 count, u32 n, u32 k,
    const uint16_t* __restrict__ g_img, u64* __restrict__ out, u32* __restrict__ out_card,
    u64* __restrict__ out_tag) {
  extern __shared__ __align__(16) unsigned char smem[];
  const u32 kn = k * n;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  constexpr bool LB = letter_blocks<W>(INV);
  constexpr u32 SP = W | 1;  // staged parent stride (words)
  // LB: one letter block; +4 words so the k <= 4 blocks start in different
  // bank pairs (the output copy reads the same row of two letters side by side)
  constexpr u32 BLK = 64 * SP + 4;
  const u32 CP = (k * W) | 1;  // rows: children stride per parent
  constexpr u32 SS = slice_stride<W>();
  const u32 kW = k * W;
  // e / kW == umulhi(e, magic) for the e < 64·kW used here (kW = 1: magic wraps to 0)
  const u32 magic = 0xFFFFFFFFu / kW + 1;
  constexpr bool SL = INV || W > 6;  // input slices in shared memory
  u64* sl = SL ? reinterpret_cast<u64*>(smem) + static_cast<size_t>(wid) * SS : nullptr;
  unsigned char* p = smem + (SL ? static_cast<size_t>(kSliceWarps) * SS * sizeof(u64) : 0);
  u64* stage = nullptr;
  u32* scard = nullptr;
  u64* so = nullptr;
  if (STAGED) {
    const u32 area = LB ? k * BLK : 64 * CP;
    stage = reinterpret_cast<u64*>(p) + static_cast<size_t>(wid) * area;
    p += static_cast<size_t>(kSliceWarps) * area * sizeof(u64);
    scard = reinterpret_cast<u32*>(p) + static_cast<size_t>(wid) * 64 * k;
    p += static_cast<size_t>(kSliceWarps) * 64 * k * sizeof(u32);
  }
  if (!INV && !(STAGED && LB)) {
    so = reinterpret_cast<u64*>(p) + static_cast<size_t>(wid) * SS;
    p += static_cast<size_t>(kSliceWarps) * SS * sizeof(u64);
  }
  uint16_t* s_tab = reinterpret_cast<uint16_t*>(p);
  for (u32 i = threadIdx.x; i < kn; i += blockDim.x) s_tab[i] = g_img[i];
  __syncthreads();
  const bool src16 = ((reinterpret_cast<uintptr_t>(src + lo * W)) & 15) == 0;
  const bool out16 = ((reinterpret_cast<uintptr_t>(out) | reinterpret_cast<uintptr_t>(out_card)) & 15) == 0;
  // staged position of output element e of a batch (child e / W, word e % W)
  auto child_at = [&](u32 i, u32 rem) {  // child i of the batch, word rem of its kW
    if (LB) {
      const u32 a = rem / W;
      return a * BLK + i * SP + (rem - a * W);
    }
    return i * CP + rem;
  };
  const u64 batches = (count + 63) / 64;
  for (u64 b = static_cast<u64>(blockIdx.x) * kSliceWarps + wid; b < batches;
       b += static_cast<u64>(gridDim.x) * kSliceWarps) {
    const u64 i0 = b * 64 + lane, i1 = i0 + 32;
    const bool v0 = i0 < count, v1 = i1 < count;
    const u32 nb = static_cast<u32>(count - b * 64 < 64 ? count - b * 64 : 64);  // parents here
    if (STAGED) {  // parents into letter block 0
      const u64* blk = src + (lo + b * 64) * W;
      if (nb == 64 && src16) {  // 32W 16-byte loads, all issued before any store
        constexpr int kIt = (32 * W + 31) / 32;
        uint4 v[kIt];
#pragma unroll
        for (int it = 0; it < kIt; ++it) {
          const u32 e2 = it * 32 + lane;
          if (e2 < 32 * W) v[it] = __ldg(reinterpret_cast<const uint4*>(blk) + e2);
        }
#pragma unroll
        for (int it = 0; it < kIt; ++it) {
          const u32 e2 = it * 32 + lane;
          if (e2 < 32 * W) {
            const u32 e = 2 * e2, r = e / W, w = e - r * W;
            stage[r * SP + w] = (static_cast<u64>(v[it].y) << 32) | v[it].x;
            const u32 r1 = w + 1 == W ? r + 1 : r, w1 = w + 1 == W ? 0 : w + 1;
            stage[r1 * SP + w1] = (static_cast<u64>(v[it].w) << 32) | v[it].z;
          }
        }
      } else {
        for (u32 e = lane; e < 64 * W; e += 32) {
          const u32 r = e / W, w = e - r * W;
          stage[r * SP + w] = e < nb * W ? __ldg(blk + e) : 0;
        }
      }
      __syncwarp();
    }
    // ---- parents -> slices: lane l ends up holding slices 64w + l and
    // 64w + 32 + l — exactly the ones it scatters for the image, so the image
    // keeps them in registers; the preimage gathers them from shared memory
    constexpr bool REG = !INV && W <= 6;  // register budget: 2W slices + 2W outputs
    u64 xs[REG ? W : 1][2];
#pragma unroll
    for (int w = 0; w < W; ++w) {
      u64 r0, r1;
      if (STAGED) {
        r0 = stage[lane * SP + w];
        r1 = stage[(lane + 32) * SP + w];
      } else {
        r0 = v0 ? __ldg(src + (lo + i0) * W + w) : 0;
        r1 = v1 ? __ldg(src + (lo + i1) * W + w) : 0;
      }
      u64 c0, c1;
      transpose64(r0, r1, lane, c0, c1);
      if constexpr (!REG) {
        sl[64 * w + lane] = c0;
        sl[64 * w + 32 + lane] = c1;
      } else {
        xs[w][0] = c0;
        xs[w][1] = c1;
      }
    }
    __syncwarp();
    for (u32 a = 0; a < k; ++a) {
      const u32 base = a * n;
      u64* blk = STAGED && LB ? stage + a * BLK : nullptr;
      u64 s[W][2];  // image: this letter's output slices (dead code for the preimage)
      if (!INV) {  // image: scatter the slices, o[delta(q,a)] |= sl[q] (smem atomics)
        u64* o = STAGED && LB ? blk : so;
#pragma unroll
        for (int i = 0; i < 2 * W; ++i) o[32 * i + lane] = 0;
        __syncwarp();
        // two native 32-bit ORs (a 64-bit shared atomicOr is a CAS spin loop)
#pragma unroll
        for (int j = 0; j < 2 * W; ++j) {
          const u32 q = 32 * j + lane;
          if (q < n) {
            const u64 v = REG ? xs[REG ? j / 2 : 0][j % 2] : sl[q];
            u32* dst = reinterpret_cast<u32*>(&o[s_tab[base + q]]);
            if (static_cast<u32>(v)) atomicOr(dst, static_cast<u32>(v));
            if (v >> 32) atomicOr(dst + 1, static_cast<u32>(v >> 32));
          }
        }
        __syncwarp();
#pragma unroll
        for (int w = 0; w < W; ++w)
#pragma unroll
          for (int h = 0; h < 2; ++h) s[w][h] = o[64 * w + 32 * h + lane];
        __syncwarp();  // block a now takes this letter's children
      }
      u32 card0 = 0, card1 = 0;
#pragma unroll
      for (int w = 0; w < W; ++w) {
        u64 x0, x1;
        if constexpr (INV) {  // preimage: pure gather
          const u32 q0 = 64 * w + lane, q1 = q0 + 32;
          x0 = q0 < n ? sl[s_tab[base + q0]] : 0;
          x1 = q1 < n ? sl[s_tab[base + q1]] : 0;
        } else {
          x0 = s[w][0];
          x1 = s[w][1];
        }
        u64 r0, r1;
        transpose64(x0, x1, lane, r0, r1);  // child rows i0, i1 — word w
        if (STAGED && LB) {
          blk[lane * SP + w] = r0;
          blk[(lane + 32) * SP + w] = r1;
        } else if (STAGED) {
          stage[lane * CP + a * W + w] = r0;
          stage[(lane + 32) * CP + a * W + w] = r1;
        } else {
          if (v0) out[(i0 * k + a) * W + w] = r0;
          if (v1) out[(i1 * k + a) * W + w] = r1;
        }
        card0 += __popcll(r0);
        card1 += __popcll(r1);
      }
      if (STAGED) {
        scard[lane * k + a] = card0;
        scard[(lane + 32) * k + a] = card1;
      } else {
        if (v0) {
          out_card[i0 * k + a] = card0;
          if (out_tag) out_tag[i0 * k + a] = ((lo + i0) << 16) | a;
        }
        if (v1) {
          out_card[i1 * k + a] = card1;
          if (out_tag) out_tag[i1 * k + a] = ((lo + i1) << 16) | a;
        }
      }
    }
    __syncwarp();
    if (STAGED) {  // the 64·k children of this batch are contiguous in the output
      const u64 o0 = b * 64 * k;
      const u32 nc = nb * k;
      u64* dst = out + o0 * W;
      if (nb == 64 && out16) {  // 16-byte stores (o0·W words is a multiple of 2·64)
        // element 2·e2 = child i, word rem of its k·W; lanes advance by 64
        // elements (di children + dr words) per iteration
        const u32 di = 64 / kW, dr = 64 - di * kW;
        u32 i = kW == 1 ? 2 * lane : __umulhi(2 * lane, magic), rem = 2 * lane - i * kW;
        for (u32 e2 = lane; e2 < 32 * kW; e2 += 32) {
          u32 i1 = i, r1 = rem + 1;
          if (r1 == kW) {
            r1 = 0;
            ++i1;
          }
          const u64 x = stage[child_at(i, rem)], y = stage[child_at(i1, r1)];
          i += di;
          rem += dr;
          if (rem >= kW) {
            rem -= kW;
            ++i;
          }
          __stcs(reinterpret_cast<uint4*>(dst) + e2,
                 make_uint4(static_cast<u32>(x), static_cast<u32>(x >> 32), static_cast<u32>(y),
                            static_cast<u32>(y >> 32)));
        }
        for (u32 e4 = lane; e4 < 16 * k; e4 += 32)
          __stcs(reinterpret_cast<uint4*>(out_card + o0) + e4,
                 reinterpret_cast<const uint4*>(scard)[e4]);
      } else {
        for (u32 e = lane; e < nc * W; e += 32) {
          const u32 i = kW == 1 ? e : __umulhi(e, magic);
          dst[e] = stage[child_at(i, e - i * kW)];
        }
        for (u32 e = lane; e < nc; e += 32) out_card[o0 + e] = scard[e];
      }
      if (out_tag)
        for (u32 e = lane; e < nc; e += 32) {
          const u64 o = o0 + e;
          out_tag[o] = ((lo + o / k) << 16) | (o % k);
        }
      __syncwarp();
    }
  }
}

void expand(Context& c, const DList& src, size_t lo, size_t hi, bool inverse, DList& out) {
  const size_t cnt = hi > lo ? hi - lo : 0;
  const u32 k = c.k(), n = c.n();
  out.reserve(cnt * k);
  out.set_size(cnt * k);
  if (!cnt) return;
  cudaStream_t s = as_stream(c.stream());
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (c.timing) {
    SW_CUDA(cudaEventCreate(&e0));
    SW_CUDA(cudaEventCreate(&e1));
    SW_CUDA(cudaEventRecord(e0, s));
  }
  const int block = kSliceWarps * 32;
  const u64 batches = (cnt + 63) / 64;
  const int grid = static_cast<int>(std::min<u64>((batches + kSliceWarps - 1) / kSliceWarps, 148 * 16));
  SW_DISPATCH_W(c.W(), {
    const bool staged = sliced_smem<W>(k, n, true, inverse) <= kStageSmemLimit;
    const size_t shmem = sliced_smem<W>(k, n, staged, inverse);
    auto kern = staged ? (inverse ? expand_sliced_kernel<W, true, true>
                                  : expand_sliced_kernel<W, false, true>)
                       : (inverse ? expand_sliced_kernel<W, true, false>
                                  : expand_sliced_kernel<W, false, false>);
    if (shmem > 48 * 1024) smem_opt_in(reinterpret_cast<const void*>(kern), static_cast<int>(shmem));
    kern<<<grid, block, shmem, s>>>(src.words, lo, cnt, n, k,
                                    static_cast<const uint16_t*>(c.d_img), out.words, out.cards,
                                    out.tagged() ? out.tags : nullptr);
  });
  SW_CHECK_LAUNCH();
  c.counters.kernel_launches++;
  c.counters.expand_launches++;
  c.counters.expand_children += cnt * k;
  if (c.timing) {
    SW_CUDA(cudaEventRecord(e1, s));
    SW_CUDA(cudaEventSynchronize(e1));
    float ms = 0;
    SW_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    c.counters.expand_ms += ms;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  }
}

// ----------------------------------------------------------- state histogram
// Each warp bit-slices 64 sets per word (transpose64) and popcounts the
// slices: lane l accumulates the counts of states 64w+l and 64w+32+l in
// registers, one global atomic per state per warp at the end.
template <int W>
__global__ void __launch_bounds__(256) state_hist_kernel(const u64* __restrict__ words, u64 count,
                                                         u32 n, u32* __restrict__ hist) {
  const int lane = threadIdx.x & 31;
  const u64 warp = (blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x) >> 5;
  const u64 nwarps = (static_cast<u64>(gridDim.x) * blockDim.x) >> 5;
  u32 cnt[W][2];
#pragma unroll
  for (int w = 0; w < W; ++w) cnt[w][0] = cnt[w][1] = 0;
  for (u64 b = warp; b * 64 < count; b += nwarps) {
    const u64 i0 = b * 64 + lane, i1 = i0 + 32;
#pragma unroll
    for (int w = 0; w < W; ++w) {
      const u64 r0 = i0 < count ? __ldg(words + i0 * W + w) : 0;
      const u64 r1 = i1 < count ? __ldg(words + i1 * W + w) : 0;
      u64 c0, c1;
      transpose64(r0, r1, lane, c0, c1);
      cnt[w][0] += __popcll(c0);
      cnt[w][1] += __popcll(c1);
    }
  }
#pragma unroll
  for (int w = 0; w < W; ++w) {
    const u32 q0 = 64 * w + lane, q1 = q0 + 32;
    if (q0 < n && cnt[w][0]) atomicAdd(&hist[q0], cnt[w][0]);
    if (q1 < n && cnt[w][1]) atomicAdd(&hist[q1], cnt[w][1]);
  }
}

void state_histogram(Context& c, const DList& l, u32* hist) {
  cudaStream_t s = as_stream(c.stream());
  SW_CUDA(cudaMemsetAsync(hist, 0, c.n() * 4, s));
  if (l.empty()) return;
  const u64 batches = (l.size() + 63) / 64;
  const int grid = static_cast<int>(std::min<u64>((batches + 7) / 8, 148 * 8));
  SW_DISPATCH_W(c.W(), { state_hist_kernel<W><<<grid, 256, 0, s>>>(l.words, l.size(), c.n(), hist); });
  SW_CHECK_LAUNCH();
  c.counters.kernel_launches++;
}

// --------------------------------------------------------------- complement
template <int W>
__global__ void complement_kernel(u64* words, u32* cards, u64 count, u32 n) {
  const u64 tail = (n & 63) ? (~u64{0} << (64 - (n & 63))) : ~u64{0};
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<u64>(gridDim.x) * blockDim.x) {
#pragma unroll
    for (int w = 0; w < W; ++w) {
      u64 x = ~words[i * W + w];
      if (w == W - 1) x &= tail;
      words[i * W + w] = x;
    }
    cards[i] = n - cards[i];
  }
}

void complement(Context& c, DList& l) {
  l.forget_stats();
  if (l.empty()) return;
  SW_DISPATCH_W(c.W(), {
    complement_kernel<W><<<grid_for(l.size(), 256), 256, 0, as_stream(c.stream())>>>(
        l.words, l.cards, l.size(), c.n());
  });
  SW_CHECK_LAUNCH();
  c.counters.kernel_launches++;
}

// -------------------------------------------------------------------- stats
struct StatsAcc {
  unsigned long long sum;
  unsigned int min;
  unsigned int max;
};

// DIRECT (one block): the block's result is the answer — no accumulator
// initialisation copy before the launch (small lists: config-2 solves refresh
// stats several times per step).
template <bool DIRECT>
__global__ void stats_kernel(const u32* cards, u64 count, StatsAcc* acc) {
  u64 sum = 0;
  u32 mn = 0xFFFFFFFFu, mx = 0;
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<u64>(gridDim.x) * blockDim.x) {
    const u32 v = cards[i];
    sum += v;
    mn = min(mn, v);
    mx = max(mx, v);
  }
  using BR = cub::BlockReduce<u64, 256>;
  using BR32 = cub::BlockReduce<u32, 256>;
  __shared__ typename BR::TempStorage t1;
  __shared__ typename BR32::TempStorage t2;
  const u64 bs = BR(t1).Sum(sum);
  __syncthreads();
  const u32 bmn = BR32(t2).Reduce(mn, cub::Min());
  __syncthreads();
  const u32 bmx = BR32(t2).Reduce(mx, cub::Max());
  if (threadIdx.x == 0) {
    if (DIRECT) {
      *acc = StatsAcc{static_cast<unsigned long long>(bs), bmn, bmx};
    } else {
      atomicAdd(&acc->sum, static_cast<unsigned long long>(bs));
      atomicMin(&acc->min, bmn);
      atomicMax(&acc->max, bmx);
    }
  }
}

ListStats stats(Context& c, const DList& l) {
  ListStats st;
  st.min_card = c.n();
  if (l.empty()) return st;
  if (l.known_stats(&st)) return st;
  StatsAcc h{0, 0xFFFFFFFFu, 0};
  auto* d = static_cast<StatsAcc*>(c.scratch(7, sizeof(StatsAcc)));
  if (l.size() <= 256 * 64) {
    stats_kernel<true><<<1, 256, 0, as_stream(c.stream())>>>(l.cards, l.size(), d);
  } else {
    c.memcpy_h2d(d, &h, sizeof(h));
    stats_kernel<false><<<grid_for(l.size(), 256, 148 * 4), 256, 0, as_stream(c.stream())>>>(
        l.cards, l.size(), d);
  }
  SW_CHECK_LAUNCH();
  c.counters.kernel_launches++;
  c.memcpy_d2h(&h, d, sizeof(h));
  st.sum_cards = h.sum;
  st.min_card = h.min;
  st.max_card = h.max;
  return st;
}

// --------------------------------------------------------------- compaction
// Order-preserving stream compaction in two passes over tiles of 256 items:
// (1) per-tile survivor counts from warp ballots, (2) a single-block scan of
// the tile counts, (3) scatter: each survivor's slot = tile offset + warp
// offset + popc(ballot & lanes_below).  Rows are optionally gathered through
// a permutation (sorted order), so sort-apply + dedupe + compaction is one pass.
constexpr int kTile = 256;

template <class Keep>
__global__ void __launch_bounds__(kTile) compact_count_kernel(u64 count, Keep keep, u32* tile_counts) {
  const u64 i = static_cast<u64>(blockIdx.x) * kTile + threadIdx.x;
  const bool f = i < count && keep(i);
  const unsigned ballot = __ballot_sync(0xFFFFFFFFu, f);
  __shared__ u32 warp_counts[kTile / 32];
  if ((threadIdx.x & 31) == 0) warp_counts[threadIdx.x >> 5] = __popc(ballot);
  __syncthreads();
  if (threadIdx.x == 0) {
    u32 s = 0;
    for (int w = 0; w < kTile / 32; ++w) s += warp_counts[w];
    tile_counts[blockIdx.x] = s;
  }
}

// Exclusive scan of tile counts in one block; total written to tile_counts[ntiles].
__global__ void __launch_bounds__(1024) scan_tiles_kernel(u32* tile_counts, u32 ntiles) {
  using BS = cub::BlockScan<u32, 1024>;
  __shared__ typename BS::TempStorage tmp;
  __shared__ u32 carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (u32 base = 0; base < ntiles; base += 1024) {
    const u32 i = base + threadIdx.x;
    const u32 v = i < ntiles ? tile_counts[i] : 0;
    u32 ex, total;
    BS(tmp).ExclusiveSum(v, ex, total);
    if (i < ntiles) tile_counts[i] = ex + carry;
    __syncthreads();
    if (threadIdx.x == 0) carry += total;
    __syncthreads();
  }
  if (threadIdx.x == 0) tile_counts[ntiles] = carry;
}

template <int W, class Keep>
__global__ void __launch_bounds__(kTile) compact_scatter_kernel(
    u64 count, Keep keep, const u32* __restrict__ perm, const u32* __restrict__ tile_offsets,
    const u64* __restrict__ sw, const u32* __restrict__ sc, const u64* __restrict__ st,
    u64* __restrict__ dw, u32* __restrict__ dc, u64* __restrict__ dt) {
  const u64 i = static_cast<u64>(blockIdx.x) * kTile + threadIdx.x;
  const bool f = i < count && keep(i);
  const unsigned ballot = __ballot_sync(0xFFFFFFFFu, f);
  __shared__ u32 warp_off[kTile / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) warp_off[warp] = __popc(ballot);
  __syncthreads();
  if (threadIdx.x == 0) {
    u32 s = 0;
    for (int w = 0; w < kTile / 32; ++w) {
      const u32 v = warp_off[w];
      warp_off[w] = s;
      s += v;
    }
  }
  __syncthreads();
  if (!f) return;
  const u64 pos = tile_offsets[blockIdx.x] + warp_off[warp] + __popc(ballot & ((1u << lane) - 1));
  const u64 from = perm ? perm[i] : i;
#pragma unroll
  for (int w = 0; w < W; ++w) dw[pos * W + w] = sw[from * W + w];
  dc[pos] = sc[from];
  if (dt) dt[pos] = st[from];
}

struct KeepAll {
  __device__ bool operator()(u64) const { return true; }
};
struct KeepFlags {
  const uint8_t* f;
  __device__ bool operator()(u64 i) const { return f[i] != 0; }
};
template <int W>
struct KeepUniqueSorted {  // first of each run of equal rows in perm order
  const u64* words;
  const u32* perm;
  __device__ bool operator()(u64 i) const {
    if (i == 0) return true;
    const u64 a = perm ? perm[i] : i, b = perm ? perm[i - 1] : i - 1;
#pragma unroll
    for (int w = 0; w < W; ++w)
      if (words[a * W + w] != words[b * W + w]) return true;
    return false;
  }
};

// Small lists: the whole compaction in ONE block (tiles of 1024 in order,
// carry in shared memory) into an output sized for every row; the survivor
// count and the survivors' card statistics come back in ONE readback (the
// engine refreshes a list's statistics right after compacting it) — one
// launch and one host wait instead of three launches and two waits.
struct CompactResult {
  unsigned long long sum;
  u32 min, max, count, pad;
};

template <int W, class Keep>
__global__ void __launch_bounds__(1024) compact_small_kernel(
    u64 count, Keep keep, const u32* __restrict__ perm, const u64* __restrict__ sw,
    const u32* __restrict__ sc, const u64* __restrict__ st, u64* __restrict__ dw,
    u32* __restrict__ dc, u64* __restrict__ dt, CompactResult* res) {
  __shared__ u32 warp_off[32];
  __shared__ u32 carry;
  __shared__ CompactResult acc;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    carry = 0;
    acc = CompactResult{0, 0xFFFFFFFFu, 0, 0, 0};
  }
  u64 sum = 0;
  u32 mn = 0xFFFFFFFFu, mx = 0;
  __syncthreads();
  for (u64 base = 0; base < count; base += 1024) {
    const u64 i = base + threadIdx.x;
    const bool f = i < count && keep(i);
    const unsigned ballot = __ballot_sync(0xFFFFFFFFu, f);
    if (lane == 0) warp_off[warp] = __popc(ballot);
    __syncthreads();
    if (warp == 0) {  // exclusive scan of the 32 warp counts
      const u32 v = warp_off[lane];
      u32 x = v;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const u32 y = __shfl_up_sync(0xFFFFFFFFu, x, d);
        if (lane >= d) x += y;
      }
      warp_off[lane] = x - v;
    }
    __syncthreads();
    if (f) {
      const u64 pos = carry + warp_off[warp] + __popc(ballot & ((1u << lane) - 1));
      const u64 from = perm ? perm[i] : i;
#pragma unroll
      for (int w = 0; w < W; ++w) dw[pos * W + w] = sw[from * W + w];
      const u32 cd = sc[from];
      dc[pos] = cd;
      if (dt) dt[pos] = st[from];
      sum += cd;
      mn = min(mn, cd);
      mx = max(mx, cd);
    }
    __syncthreads();
    if (threadIdx.x == 1023) carry += warp_off[31] + __popc(ballot);
    __syncthreads();
  }
  if (sum) atomicAdd(&acc.sum, static_cast<unsigned long long>(sum));
  if (mn != 0xFFFFFFFFu) atomicMin(&acc.min, mn);
  if (mx) atomicMax(&acc.max, mx);
  __syncthreads();
  if (threadIdx.x == 0) {
    acc.count = carry;
    *res = acc;
  }
}

constexpr u64 kCompactSmall = 8 * 1024;  // one block: ~4 us per 1024 rows

template <int W, class Keep>
static size_t run_compact(Context& c, DList& l, Keep keep, const u32* perm) {
  const u64 count = l.size();
  if (count == 0) return 0;
  if (count <= kCompactSmall) {
    auto* dres = static_cast<CompactResult*>(c.scratch(6, sizeof(CompactResult)));
    DList out(&c, count, l.tagged());
    compact_small_kernel<W><<<1, 1024, 0, as_stream(c.stream())>>>(
        count, keep, perm, l.words, l.cards, l.tags, out.words, out.cards,
        l.tagged() ? out.tags : nullptr, dres);
    SW_CHECK_LAUNCH();
    c.counters.kernel_launches += 1;
    CompactResult h{};
    c.memcpy_d2h(&h, dres, sizeof(h));
    out.set_size(h.count);
    ListStats st;
    st.sum_cards = h.sum;
    st.min_card = h.count ? h.min : c.n();
    st.max_card = h.count ? h.max : 0;
    out.set_known_stats(st);
    l = std::move(out);
    return h.count;
  }
  const u32 ntiles = static_cast<u32>((count + kTile - 1) / kTile);
  auto* tiles = static_cast<u32*>(c.scratch(6, (ntiles + 1) * sizeof(u32)));
  cudaStream_t s = as_stream(c.stream());
  compact_count_kernel<<<ntiles, kTile, 0, s>>>(count, keep, tiles);
  scan_tiles_kernel<<<1, 1024, 0, s>>>(tiles, ntiles);
  u32 total = 0;
  c.memcpy_d2h(&total, tiles + ntiles, 4);
  DList out(&c, total, l.tagged());
  if (total)
    compact_scatter_kernel<W><<<ntiles, kTile, 0, s>>>(count, keep, perm, tiles, l.words, l.cards,
                                                       l.tags, out.words, out.cards,
                                                       l.tagged() ? out.tags : nullptr);
  SW_CHECK_LAUNCH();
  c.counters.kernel_launches += 3;
  out.set_size(total);
  l = std::move(out);
  return total;
}

size_t compact_flags(Context& c, DList& l, const uint8_t* keep, const u32* perm) {
  size_t r = 0;
  SW_DISPATCH_W(c.W(), {
    if (keep)
      r = run_compact<W>(c, l, KeepFlags{keep}, perm);
    else
      r = run_compact<W>(c, l, KeepAll{}, perm);
  });
  return r;
}

void gather_rows(Context& c, DList& l, const u32* perm) { compact_flags(c, l, nullptr, perm); }

__global__ void add_to_tags_kernel(u64* __restrict__ tags, u64 count, u64 add) {
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<u64>(gridDim.x) * blockDim.x)
    tags[i] += add;
}

void add_to_tags(Context& c, DList& l, u64 add) {
  if (!l.tagged() || l.empty() || add == 0) return;
  add_to_tags_kernel<<<grid_for(l.size(), 256), 256, 0, as_stream(c.stream())>>>(l.tags, l.size(), add);
  SW_CHECK_LAUNCH();
  c.counters.kernel_launches++;
}

size_t compact_unique(Context& c, DList& l, const u32* perm) {
  size_t r = 0;
  SW_DISPATCH_W(c.W(), { r = run_compact<W>(c, l, KeepUniqueSorted<W>{l.words, perm}, perm); });
  return r;
}

// ------------------------------------------------------------- hash dedupe
// Open addressing over 2^m >= 2N slots of u64 = (32-bit row hash << 32 | row
// index), linear probing.  Insert: claim an empty slot by CAS; on a slot with
// the same hash tag compare rows, and for an equal row keep the MINIMUM index
// (atomicMin on the packed value: equal rows share the tag) — the first
// occurrence, i.e. the same duplicate the reference's stable lex sort keeps
// (set_list.hpp:208-209).  Each row remembers its slot, so "am I the
// survivor" is one table read, fused into the warp-ballot compaction.
__device__ __forceinline__ u64 mix64(u64 x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdull;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ull;
  x ^= x >> 33;
  return x;
}

template <int W>
__global__ void hash_insert_kernel(const u64* __restrict__ words, u64 count,
                                   unsigned long long* table, u64 mask, u32* __restrict__ slot_of) {
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<u64>(gridDim.x) * blockDim.x) {
    u64 row[W];
    u64 h = 0x9E3779B97F4A7C15ull;
#pragma unroll
    for (int w = 0; w < W; ++w) {
      row[w] = words[i * W + w];
      h = mix64(h ^ row[w]);
    }
    const u64 tag = h >> 32;
    const unsigned long long mine = (tag << 32) | i;
    u64 s = h & mask;
    while (true) {
      unsigned long long cur = table[s];
      if (cur == ~0ull) {
        cur = atomicCAS(&table[s], ~0ull, mine);
        if (cur == ~0ull) break;  // claimed
      }
      if ((cur >> 32) == tag) {
        const u64 j = cur & 0xFFFFFFFFull;
        bool eq = true;
#pragma unroll
        for (int w = 0; w < W; ++w) eq &= words[j * W + w] == row[w];
        if (eq) {
          atomicMin(&table[s], mine);
          break;
        }
      }
      s = (s + 1) & mask;
    }
    slot_of[i] = static_cast<u32>(s);
  }
}

struct KeepHashFirst {
  const unsigned long long* table;
  const u32* slot_of;
  __device__ bool operator()(u64 i) const {
    return (table[slot_of[i]] & 0xFFFFFFFFull) == i;
  }
};

size_t hash_dedupe_wide(Context& c, DList& l) {
  const u64 N = l.size();
  if (N <= 1) return 0;
  if (N >= 0xFFFFFFFFull) throw std::invalid_argument("hash_dedupe: list too large");
  u64 slots = 1;
  while (slots < 2 * N) slots <<= 1;
  cudaStream_t s = as_stream(c.stream());
  // persistent per-context scratch: no pool growth on the hot path
  auto* table = static_cast<unsigned long long*>(c.scratch(8, slots * 8));
  auto* slot_of = static_cast<u32*>(c.scratch(9, N * 4));
  SW_CUDA(cudaMemsetAsync(table, 0xFF, slots * 8, s));
  size_t kept = 0;
  SW_DISPATCH_W(c.W(), {
    hash_insert_kernel<W><<<grid_for(N, 256, 148 * 16), 256, 0, s>>>(l.words, N, table, slots - 1, slot_of);
    SW_CHECK_LAUNCH();
    kept = run_compact<W>(c, l, KeepHashFirst{table, slot_of}, nullptr);
  });
  c.counters.kernel_launches += 2;
  return N - kept;
}

// ------------------------------------------------------ cardinality filters
__global__ void card_filter_kernel(const u32* cards, u64 count, u32 bound, int at_least,
                                   uint8_t* keep) {
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<u64>(gridDim.x) * blockDim.x)
    keep[i] = at_least ? (cards[i] >= bound) : (cards[i] <= bound);
}

static void card_filter(Context& c, DList& l, u32 bound, int at_least) {
  if (l.empty()) return;
  auto* keep = static_cast<uint8_t*>(c.scratch(5, l.size()));
  card_filter_kernel<<<grid_for(l.size(), 256), 256, 0, as_stream(c.stream())>>>(
      l.cards, l.size(), bound, at_least, keep);
  SW_CHECK_LAUNCH();
  compact_flags(c, l, keep, nullptr);
}

void keep_card_at_most(Context& c, DList& l, u32 max_card) { card_filter(c, l, max_card, 0); }
void keep_card_at_least(Context& c, DList& l, u32 min_card) { card_filter(c, l, min_card, 1); }

}  // namespace synchro::dev
