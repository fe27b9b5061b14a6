// Set-semantics frontier dedupe (replaces lex_sort_dedupe's duplicate removal,
// set_list.hpp:259-265, where only the surviving SET matters).
//
// Survivors leave in UNSPECIFIED order (each warp tile reserves its output
// block with one atomicAdd — no cross-tile waiting): both engine call sites
// are order-free (the BFS layer's consumers sort their own copies; a DFS
// level is sorted before any order-dependent step).
//
// Untagged lists (dd_single_kernel): equal rows are identical, so one pass —
// each row claims its slot and the first claimer survives.  Rows are read once.
//
// Tagged lists (tags differ between equal rows): keeps the first occurrence
// (minimum index) of every distinct row — the survivor the reference's stable
// lex sort keeps (set_list.hpp:208-209), so word reconstruction follows the
// same parents.  Two HBM passes:
//   K1 insert   each thread keeps R rows in flight: loads them, hashes them,
//               and issues all R claims (atomicCAS on an empty slot) before
//               looking at any result.  Open-addressing table of 32-bit
//               entries (7-bit hash tag << 25 | index+1, 0 = empty, load
//               <= 0.6 — 2^24 rows fit a ~110 MB table, i.e. the 126 MB L2, so
//               probes and atomics stay on chip); equal rows share a tag, so
//               atomicMin keeps the minimum index; the probe distance is
//               remembered in one byte per row.
//   K2 resolve  warp tiles re-read; row i survives iff the entry at
//               home+dist still holds i; survivors written as one block per
//               warp tile through shared memory.
// HBM traffic ≈ 2 reads of the rows + 1 write of the survivors + 2 bytes/row.
#include <cstdlib>

#include "dev.hpp"
#include "kernels.cuh"
#include "util.cuh"

namespace synchro::dev {

namespace {

constexpr int kDdThreads = 256;
constexpr u32 kIdxBits = 25;
constexpr u32 kIdxMask = (1u << kIdxBits) - 1;
constexpr uint8_t kFar = 255;  // probe distance >= 255: resolve walks the chain

// rows in flight per thread (register budget: R·W words)
template <int W>
constexpr int rows_per_thread() {
  return W <= 5 ? 4 : (W <= 9 ? 2 : 1);
}

__device__ __forceinline__ u64 mix64(u64 x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdull;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ull;
  x ^= x >> 33;
  return x;
}

// Two independent 32-bit multiplicative chains over the row's 32-bit halves
// (1 LOP3 + 1 IMAD per half and chain) with a final avalanche; the high
// word picks the home slot (by range reduction), the low word the tag.
__device__ __forceinline__ u32 fmix32(u32 h) {
  h ^= h >> 16;
  h *= 0x85EBCA6Bu;
  h ^= h >> 13;
  h *= 0xC2B2AE35u;
  h ^= h >> 16;
  return h;
}

template <int W>
__device__ __forceinline__ u64 row_hash(const u64* r) {
  u32 a = 0x243F6A88u, b = 0x85A308D3u;
#pragma unroll
  for (int w = 0; w < W; ++w) {
    const u32 lo = static_cast<u32>(r[w]), hi = static_cast<u32>(r[w] >> 32);
    a = (a ^ hi) * 0x9E3779B1u;
    b = (b ^ lo) * 0x85EBCA77u;
    a = (a ^ lo) * 0x9E3779B1u;
    b = (b ^ hi) * 0x85EBCA77u;
  }
  return (static_cast<u64>(fmix32(a)) << 32) | fmix32(b ^ a);
}

__device__ __forceinline__ u32 home_slot(u64 h, u32 nslots) {
  return static_cast<u32>(((h >> 32) * static_cast<u64>(nslots)) >> 32);
}
__device__ __forceinline__ u32 tag7(u64 h) { return static_cast<u32>(h >> 8) & 0x7F; }

template <int W>
__device__ __forceinline__ bool row_equal(const u64* __restrict__ words, u32 j, const u64* r) {
  bool eq = true;
#pragma unroll
  for (int w = 0; w < W; ++w) eq &= words[static_cast<u64>(j) * W + w] == r[w];
  return eq;
}

// Claims for a lane's R rows after their optimistic CAS at home (cur[j] =
// value found there, 0 = claimed).  Pending rows advance together, one event
// per round — each round issues the R sector loads at once and decodes a
// sector into empty / tag-match bit masks, so there is no per-slot branching.
// claimed[j]: row j owns slot[j]; otherwise an equal row holds slot[j] (or the
// row was invalid).  dist[j] = probes from home to slot[j].
template <int W, int R>
__device__ __forceinline__ void claim_rows(u32* table, u32 nslots, const u64* __restrict__ words,
                                           const u64 (&row)[R][W], const u32 (&home)[R],
                                           const u32 (&mine)[R], const u32 (&cur)[R],
                                           const bool (&valid)[R], bool (&claimed)[R],
                                           u32 (&slot)[R], u32 (&dist)[R]) {
  bool pend[R];
  u32 s[R];
#pragma unroll
  for (int j = 0; j < R; ++j) {
    claimed[j] = valid[j] && cur[j] == 0;
    slot[j] = home[j];
    pend[j] = valid[j] && cur[j] != 0;
    if (pend[j] && (cur[j] >> kIdxBits) == (mine[j] >> kIdxBits) &&
        row_equal<W>(words, (cur[j] & kIdxMask) - 1, row[j]))
      pend[j] = false;  // an equal row holds the home slot
    s[j] = home[j] + 1 == nslots ? 0 : home[j] + 1;
  }
  while (true) {
    bool any = false;
#pragma unroll
    for (int j = 0; j < R; ++j) any |= pend[j];
    if (!any) break;
    uint4 qa[R], qb[R];
#pragma unroll
    for (int j = 0; j < R; ++j) {
      if (pend[j]) {
        const u32 g = s[j] & ~7u;  // nslots is a multiple of 8
        qa[j] = __ldcg(reinterpret_cast<const uint4*>(table + g));
        qb[j] = __ldcg(reinterpret_cast<const uint4*>(table + g + 4));
      }
    }
#pragma unroll
    for (int j = 0; j < R; ++j) {
      if (!pend[j]) continue;
      const u32 g = s[j] & ~7u, tg = mine[j] >> kIdxBits;
      const u32 e[8] = {qa[j].x, qa[j].y, qa[j].z, qa[j].w, qb[j].x, qb[j].y, qb[j].z, qb[j].w};
      u32 E = 0, M = 0;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        E |= static_cast<u32>(e[k] == 0) << k;
        M |= static_cast<u32>((e[k] >> kIdxBits) == tg && e[k] != 0) << k;
      }
      const u32 m = (E | M) & (0xFFu << (s[j] - g)) & 0xFFu;
      if (!m) {
        s[j] = g + 8 >= nslots ? 0 : g + 8;
        continue;
      }
      const int k = __ffs(m) - 1;
      const u32 sl = g + k;
      u32 v = e[0];
#pragma unroll
      for (int q = 1; q < 8; ++q) v = q == k ? e[q] : v;
      if ((E >> k) & 1) {
        v = atomicCAS(&table[sl], 0u, mine[j]);
        if (v == 0) {
          claimed[j] = true;
          pend[j] = false;
          slot[j] = sl;
          continue;
        }
      }
      if ((v >> kIdxBits) == tg && row_equal<W>(words, (v & kIdxMask) - 1, row[j])) {
        pend[j] = false;
        slot[j] = sl;
        continue;
      }
      s[j] = sl + 1 == nslots ? 0 : sl + 1;
    }
  }
#pragma unroll
  for (int j = 0; j < R; ++j)
    dist[j] = slot[j] >= home[j] ? slot[j] - home[j] : slot[j] + nslots - home[j];
}

template <int W>
__global__ void __launch_bounds__(kDdThreads) dd_insert_kernel(const u64* __restrict__ words,
                                                              u64 N, u32* table, u32 nslots,
                                                              uint8_t* __restrict__ dist) {
  constexpr int R = rows_per_thread<W>();
  const u64 stride = static_cast<u64>(gridDim.x) * kDdThreads;
  for (u64 i0 = blockIdx.x * static_cast<u64>(kDdThreads) + threadIdx.x; i0 < N; i0 += stride * R) {
    u64 row[R][W];
    u32 s[R], mine[R], cur[R];
#pragma unroll
    for (int j = 0; j < R; ++j) {
      const u64 i = i0 + j * stride;
#pragma unroll
      for (int w = 0; w < W; ++w) row[j][w] = i < N ? __ldcs(words + i * W + w) : 0;
    }
#pragma unroll
    for (int j = 0; j < R; ++j) {  // all claims in flight before any result is used
      const u64 i = i0 + j * stride;
      const u64 h = row_hash<W>(row[j]);
      s[j] = home_slot(h, nslots);
      mine[j] = (tag7(h) << kIdxBits) | static_cast<u32>(i + 1);
      cur[j] = i < N ? atomicCAS(&table[s[j]], 0u, mine[j]) : 0;
    }
    bool valid[R], claimed[R];
    u32 sl[R], d[R];
#pragma unroll
    for (int j = 0; j < R; ++j) valid[j] = i0 + j * stride < N;
    claim_rows<W, R>(table, nslots, words, row, s, mine, cur, valid, claimed, sl, d);
#pragma unroll
    for (int j = 0; j < R; ++j) {
      const u64 i = i0 + j * stride;
      if (i >= N) continue;
      if (!claimed[j]) atomicMin(&table[sl[j]], mine[j]);  // equal row: keep the min index
      dist[i] = static_cast<uint8_t>(d[j] < kFar ? d[j] : kFar);
    }
  }
}

// Tagged lists, pass 2: warp tiles of 32·R rows (no block barriers) re-read;
// row i survives iff the entry at home+dist still holds i (the minimum index
// of its group); survivors reserve an output block with one atomicAdd per
// warp (set semantics: their order is unspecified) and leave with their cards
// and tags through the warp's staging rows.
template <int W>
__global__ void __launch_bounds__(kDdThreads) dd_resolve_kernel(
    const u64* __restrict__ words, const u32* __restrict__ cards, const u64* __restrict__ tags,
    u64 N, const u32* __restrict__ table, u32 nslots, const uint8_t* __restrict__ dist,
    u32* __restrict__ tile_counter, u64* __restrict__ ow, u32* __restrict__ oc,
    u64* __restrict__ ot, unsigned long long* __restrict__ out_count) {
  constexpr int R = rows_per_thread<W>(), T = 32 * R;
  extern __shared__ __align__(16) u64 smem[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  u64* srow = smem + static_cast<size_t>(wid) * (T * W + T + T / 2);
  u64* stag = srow + T * W;
  u32* scard = reinterpret_cast<u32*>(stag + T);
  const u64 ntiles = (N + T - 1) / T;
  const unsigned lt = (1u << lane) - 1;
  while (true) {
    u32 tt = 0;
    if (lane == 0) tt = atomicAdd(tile_counter, 1u);
    const u64 t = __shfl_sync(0xFFFFFFFFu, tt, 0);
    if (t >= ntiles) return;
    const u64 base = t * T;
    const u32 cnt = static_cast<u32>(N - base < T ? N - base : T);
    const u64* src = words + base * W;
    for (u32 e = lane; e < cnt * W; e += 32) srow[e] = __ldcs(src + e);
    __syncwarp();
    u64 row[R][W];
    u32 d[R];
#pragma unroll
    for (int j = 0; j < R; ++j) {
      const u32 r = j * 32 + lane;
#pragma unroll
      for (int w = 0; w < W; ++w) row[j][w] = r < cnt ? srow[r * W + w] : 0;
      d[j] = r < cnt ? dist[base + r] : 0;
    }
    bool keep[R];
    unsigned bal[R];
    u32 agg = 0;
#pragma unroll
    for (int j = 0; j < R; ++j) {
      const u32 r = j * 32 + lane;
      const u32 me = static_cast<u32>(base + r + 1);
      const u64 h = row_hash<W>(row[j]);
      u32 sl = home_slot(h, nslots);
      keep[j] = false;
      if (r < cnt) {
        if (d[j] != kFar) {
          sl += d[j];
          if (sl >= nslots) sl -= nslots;
          keep[j] = (table[sl] & kIdxMask) == me;
        } else {  // long chain: walk it (an equal row earlier in it means duplicate)
          const u32 tg = tag7(h);
          while (true) {
            const u32 c = table[sl];
            if ((c >> kIdxBits) == tg) {
              if ((c & kIdxMask) == me) {
                keep[j] = true;
                break;
              }
              if (row_equal<W>(words, (c & kIdxMask) - 1, row[j])) break;
            }
            sl = sl + 1 == nslots ? 0 : sl + 1;
          }
        }
      }
      bal[j] = __ballot_sync(0xFFFFFFFFu, keep[j]);
      agg += __popc(bal[j]);
    }
    u64 excl = 0;
    if (lane == 0 && agg) excl = atomicAdd(out_count, static_cast<unsigned long long>(agg));
    excl = __shfl_sync(0xFFFFFFFFu, excl, 0);
    __syncwarp();
    u32 off = 0;
#pragma unroll
    for (int j = 0; j < R; ++j) {
      if (keep[j]) {
        const u64 i = base + j * 32 + lane;
        const u32 pos = off + __popc(bal[j] & lt);
#pragma unroll
        for (int w = 0; w < W; ++w) srow[pos * W + w] = row[j][w];
        scard[pos] = cards[i];
        stag[pos] = tags[i];
      }
      off += __popc(bal[j]);
    }
    __syncwarp();
    u64* dst = ow + excl * W;
    for (u32 e = lane; e < agg * W; e += 32) __stcs(dst + e, srow[e]);
    for (u32 e = lane; e < agg; e += 32) {
      __stcs(oc + excl + e, scard[e]);
      __stcs(ot + excl + e, stag[e]);
    }
    __syncwarp();
  }
}

// One row's claim after its optimistic CAS at home found `c` != 0: walk the
// chain one 32-byte sector (8 slots) per L2 round trip, decoding each sector
// into empty / tag-match bit masks; CAS only into empty slots.  Returns true
// if `mine` claimed a slot, false if an equal row holds one.
template <int W>
__device__ __forceinline__ bool claim_one(u32* table, u32 nslots, const u64* __restrict__ words,
                                          const u64* row, u32 home, u32 mine, u32 c) {
  const u32 tg = mine >> kIdxBits;
  if ((c >> kIdxBits) == tg && row_equal<W>(words, (c & kIdxMask) - 1, row)) return false;
  u32 s = home + 1 == nslots ? 0 : home + 1;
  while (true) {
    const u32 g = s & ~7u;  // nslots is a multiple of 8
    const uint4 qa = __ldcg(reinterpret_cast<const uint4*>(table + g));
    const uint4 qb = __ldcg(reinterpret_cast<const uint4*>(table + g + 4));
    const u32 e[8] = {qa.x, qa.y, qa.z, qa.w, qb.x, qb.y, qb.z, qb.w};
    u32 E = 0, M = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      E |= static_cast<u32>(e[k] == 0) << k;
      M |= static_cast<u32>((e[k] >> kIdxBits) == tg && e[k] != 0) << k;
    }
    u32 m = (E | M) & (0xFFu << (s - g)) & 0xFFu;
    while (m) {
      const int k = __ffs(m) - 1;
      m &= m - 1;
      u32 v = e[0];
#pragma unroll
      for (int q = 1; q < 8; ++q) v = q == k ? e[q] : v;
      if ((E >> k) & 1) {
        v = atomicCAS(&table[g + k], 0u, mine);
        if (v == 0) return true;
      }
      if ((v >> kIdxBits) == tg && row_equal<W>(words, (v & kIdxMask) - 1, row)) return false;
    }
    s = g + 8 >= nslots ? 0 : g + 8;
  }
}

// Untagged lists: equal rows are indistinguishable, so the survivor of a
// group is simply whichever occurrence claims the slot first — one pass.
// The unit of work is a WARP tile of 32·R rows with no block barriers:
//   A  rows staged in shared memory (coalesced); each lane hashes its R rows
//      and issues their optimistic claims (CAS at home) before using any
//      result; rows whose home was taken go to a warp-compacted pending list;
//   B  the whole warp walks the pending chains, one row per lane (rows re-read
//      from shared memory — no per-lane row state is carried across phases);
//   C  survivors reserve an output block with one atomicAdd per warp (set
//      semantics: their order is unspecified) and leave as one block.
// Rows are read from HBM once.
template <int W, bool TAGS>
__global__ void __launch_bounds__(kDdThreads) dd_single_kernel(
    const u64* __restrict__ words, const u32* __restrict__ cards, const u64* __restrict__ tags,
    u64 N, u32* table, u32 nslots, u32* __restrict__ tile_counter, u64* __restrict__ ow,
    u32* __restrict__ oc, u64* __restrict__ ot, unsigned long long* __restrict__ out_count) {
  constexpr int R = rows_per_thread<W>(), T = 32 * R;
  extern __shared__ __align__(16) u64 smem[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  // per warp: rows T*W u64 | cards T u32 | home T u32 | cur T u32 | mine T u32 | pending T u16 | keep T u8
  //           [| tags T u64, 16-B aligned]
  constexpr int kWarpBytes = T * W * 8 + T * 4 * 4 + T * 2 + T;
  constexpr int kTagOff = (kWarpBytes + 15) & ~15;
  constexpr int kStride = TAGS ? kTagOff + T * 8 : kTagOff;
  unsigned char* wbase = reinterpret_cast<unsigned char*>(smem) + static_cast<size_t>(wid) * kStride;
  u64* stag = reinterpret_cast<u64*>(wbase + kTagOff);
  u64* srow = reinterpret_cast<u64*>(wbase);
  u32* scard = reinterpret_cast<u32*>(srow + T * W);
  u32* shome = scard + T;
  u32* scur = shome + T;
  u32* smine = scur + T;
  uint16_t* spend = reinterpret_cast<uint16_t*>(smine + T);
  uint8_t* skeep = reinterpret_cast<uint8_t*>(spend + T);
  const u64 ntiles = (N + T - 1) / T;
  const unsigned lt = (1u << lane) - 1;
  while (true) {
    u32 tt = 0;
    if (lane == 0) tt = atomicAdd(tile_counter, 1u);
    const u64 t = __shfl_sync(0xFFFFFFFFu, tt, 0);
    if (t >= ntiles) return;
    const u64 base = t * T;
    const u32 cnt = static_cast<u32>(N - base < T ? N - base : T);
    const u64* src = words + base * W;
    for (u32 e = lane; e < cnt * W; e += 32) srow[e] = __ldcs(src + e);
    __syncwarp();
    // ---- A: hash + optimistic claims, all R in flight
    u32 cur[R];
#pragma unroll
    for (int j = 0; j < R; ++j) {
      const u32 r = j * 32 + lane;
      u64 row[W];
#pragma unroll
      for (int w = 0; w < W; ++w) row[w] = srow[r * W + w];
      const u64 h = row_hash<W>(row);
      const u32 home = home_slot(h, nslots);
      const u32 mine = (tag7(h) << kIdxBits) | static_cast<u32>(base + r + 1);
      shome[r] = home;
      smine[r] = mine;
      cur[j] = r < cnt ? atomicCAS(&table[home], 0u, mine) : 0u;
    }
    u32 npend = 0;
#pragma unroll
    for (int j = 0; j < R; ++j) {
      const u32 r = j * 32 + lane;
      const bool pend = r < cnt && cur[j] != 0;
      skeep[r] = r < cnt && cur[j] == 0;
      scur[r] = cur[j];
      const unsigned b = __ballot_sync(0xFFFFFFFFu, pend);
      if (pend) spend[npend + __popc(b & lt)] = static_cast<uint16_t>(r);
      npend += __popc(b);
    }
    __syncwarp();
    // ---- B: pending chains, one row per lane
    for (u32 p = lane; p < npend; p += 32) {
      const u32 r = spend[p];
      u64 row[W];
#pragma unroll
      for (int w = 0; w < W; ++w) row[w] = srow[r * W + w];
      skeep[r] = claim_one<W>(table, nslots, words, row, shome[r], smine[r], scur[r]);
    }
    __syncwarp();
    // ---- C: reserve and write the survivors
    u64 row[R][W];
    bool keep[R];
    unsigned bal[R];
    u32 agg = 0;
#pragma unroll
    for (int j = 0; j < R; ++j) {
      const u32 r = j * 32 + lane;
      keep[j] = skeep[r] != 0;
      bal[j] = __ballot_sync(0xFFFFFFFFu, keep[j]);
      agg += __popc(bal[j]);
#pragma unroll
      for (int w = 0; w < W; ++w) row[j][w] = keep[j] ? srow[r * W + w] : 0;
    }
    u64 excl = 0;
    if (lane == 0 && agg) excl = atomicAdd(out_count, static_cast<unsigned long long>(agg));
    excl = __shfl_sync(0xFFFFFFFFu, excl, 0);
    __syncwarp();
    u32 off = 0;
#pragma unroll
    for (int j = 0; j < R; ++j) {
      if (keep[j]) {
        const u32 pos = off + __popc(bal[j] & lt);
#pragma unroll
        for (int w = 0; w < W; ++w) srow[pos * W + w] = row[j][w];
        scard[pos] = cards[base + j * 32 + lane];
        if (TAGS) stag[pos] = tags[base + j * 32 + lane];
      }
      off += __popc(bal[j]);
    }
    __syncwarp();
    u64* dst = ow + excl * W;
    for (u32 e = lane; e < agg * W; e += 32) __stcs(dst + e, srow[e]);
    for (u32 e = lane; e < agg; e += 32) {
      __stcs(oc + excl + e, scard[e]);
      if (TAGS) __stcs(ot + excl + e, stag[e]);
    }
    __syncwarp();
  }
}

template <int W, bool TAGS>
constexpr size_t single_warp_bytes() {
  constexpr int T = 32 * rows_per_thread<W>();
  return ((static_cast<size_t>(T) * W * 8 + T * 4 * 4 + T * 2 + T + 15) & ~size_t{15}) +
         (TAGS ? static_cast<size_t>(T) * 8 : 0);
}

}  // namespace

template <int W>
static size_t hash_dedupe_single(Context& c, DList& l) {
  const bool tagged = l.tagged();
  constexpr int T = rows_per_thread<W>() * 32;  // rows per warp tile
  const u64 N = l.size();
  cudaStream_t s = as_stream(c.stream());
  // load <= 0.75 (every row touches the table once; smaller table, more L2 hits)
  const char* full = std::getenv("SYNCHRO_DEDUPE_FULL_TABLE");
  const u64 want = (full && *full == '1') ? N + 64 : N * 6 / 5 + 64;
  const u32 nslots = static_cast<u32>((want + 7) & ~u64{7});
  auto* table = static_cast<u32*>(c.scratch(8, static_cast<size_t>(nslots) * 4));
  const u64 ntiles = (N + T - 1) / T;
  auto* aux = static_cast<u64*>(c.scratch(6, 16));  // [tile counter, output count]
  SW_CUDA(cudaMemsetAsync(table, 0, static_cast<size_t>(nslots) * 4, s));
  SW_CUDA(cudaMemsetAsync(aux, 0, 16, s));
  const size_t smem = static_cast<size_t>(kDdThreads / 32) *
                      (tagged ? single_warp_bytes<W, true>() : single_warp_bytes<W, false>());
  auto kern = tagged ? dd_single_kernel<W, true> : dd_single_kernel<W, false>;
  smem_opt_in(reinterpret_cast<const void*>(kern), static_cast<int>(smem));
  DList out(&c, N, tagged);
  const unsigned grid = static_cast<unsigned>(
      std::min<u64>((ntiles + kDdThreads / 32 - 1) / (kDdThreads / 32), 148 * 8));
  kern<<<grid, kDdThreads, smem, s>>>(l.words, l.cards, l.tags, N, table, nslots,
                                     reinterpret_cast<u32*>(aux), out.words, out.cards, out.tags,
                                     reinterpret_cast<unsigned long long*>(aux + 1));
  SW_CHECK_LAUNCH();
  c.counters.kernel_launches += 1;
  u64 kept = 0;
  c.memcpy_d2h(&kept, aux + 1, 8);
  out.set_size(kept);
  l = std::move(out);
  return N - kept;
}

template <int W>
static size_t hash_dedupe_tiled(Context& c, DList& l) {
  constexpr int T = rows_per_thread<W>() * 32;  // rows per warp tile
  const u64 N = l.size();
  cudaStream_t s = as_stream(c.stream());
  // load <= 0.6; SYNCHRO_DEDUPE_FULL_TABLE=1 (tests) packs the table to
  // N + 64 slots so probe chains exceed the one-byte distance
  const char* full = std::getenv("SYNCHRO_DEDUPE_FULL_TABLE");
  const u64 want = (full && *full == '1') ? N + 64 : N * 6 / 5 + 64;
  const u32 nslots = static_cast<u32>((want + 7) & ~u64{7});
  auto* table = static_cast<u32*>(c.scratch(8, static_cast<size_t>(nslots) * 4));
  auto* dist = static_cast<uint8_t*>(c.scratch(9, N));
  const u64 ntiles = (N + T - 1) / T;
  auto* aux = static_cast<u64*>(c.scratch(6, 16));  // [tile counter, output count]
  SW_CUDA(cudaMemsetAsync(table, 0, static_cast<size_t>(nslots) * 4, s));
  SW_CUDA(cudaMemsetAsync(aux, 0, 16, s));
  const size_t smem = static_cast<size_t>(kDdThreads / 32) * (T * W * 8 + T * 12);
  smem_opt_in(reinterpret_cast<const void*>(dd_resolve_kernel<W>), static_cast<int>(smem));
  const u64 per_pass = static_cast<u64>(kDdThreads) * rows_per_thread<W>();
  const unsigned grid_ins =
      static_cast<unsigned>(std::max<u64>(1, std::min<u64>((N + per_pass - 1) / per_pass, 148 * 8)));
  dd_insert_kernel<W><<<grid_ins, kDdThreads, 0, s>>>(l.words, N, table, nslots, dist);
  SW_CHECK_LAUNCH();
  DList out(&c, N, true);
  const unsigned grid = static_cast<unsigned>(
      std::min<u64>((ntiles + kDdThreads / 32 - 1) / (kDdThreads / 32), 148 * 8));
  dd_resolve_kernel<W><<<grid, kDdThreads, smem, s>>>(
      l.words, l.cards, l.tags, N, table, nslots, dist, reinterpret_cast<u32*>(aux), out.words,
      out.cards, out.tags, reinterpret_cast<unsigned long long*>(aux + 1));
  SW_CHECK_LAUNCH();
  c.counters.kernel_launches += 2;
  u64 kept = 0;
  c.memcpy_d2h(&kept, aux + 1, 8);
  out.set_size(kept);
  l = std::move(out);
  return N - kept;
}

size_t hash_dedupe(Context& c, DList& l, bool first_occurrence) {
  const u64 N = l.size();
  if (N <= 1) return 0;
  // index does not fit 25 bits (SYNCHRO_DEDUPE_WIDE=1 forces this path: tests)
  const char* wide = std::getenv("SYNCHRO_DEDUPE_WIDE");
  if (N >= kIdxMask || (wide && *wide == '1')) return hash_dedupe_wide(c, l);
  size_t r = 0;
  if (l.tagged() && first_occurrence) {  // tags differ between equal rows: the minimum index must win
    SW_DISPATCH_W(c.W(), { r = hash_dedupe_tiled<W>(c, l); });
  } else {
    SW_DISPATCH_W(c.W(), { r = hash_dedupe_single<W>(c, l); });
  }
  return r;
}

}  // namespace synchro::dev
