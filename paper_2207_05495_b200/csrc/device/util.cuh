// Shared device helpers: error checking, compile-time W dispatch, bit ops.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>
#include <set>
#include <string>
#include <utility>

#include "../common.hpp"

namespace synchro::dev {

[[noreturn]] void throw_cuda(cudaError_t e, const char* what, const char* file, int line);

#define SW_CUDA(x)                                                        \
  do {                                                                    \
    cudaError_t e_ = (x);                                                 \
    if (e_ != cudaSuccess) ::synchro::dev::throw_cuda(e_, #x, __FILE__, __LINE__); \
  } while (0)

#define SW_CHECK_LAUNCH() SW_CUDA(cudaGetLastError())

inline cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

// Kernels are instantiated for W = 1..kMaxW words per set (n <= 64*kMaxW).
inline constexpr int kMaxW = 16;

#define SW_DISPATCH_W(Wrt, ...)                                    \
  switch (Wrt) {                                                   \
    case 1: { constexpr int W = 1; __VA_ARGS__; } break;           \
    case 2: { constexpr int W = 2; __VA_ARGS__; } break;           \
    case 3: { constexpr int W = 3; __VA_ARGS__; } break;           \
    case 4: { constexpr int W = 4; __VA_ARGS__; } break;           \
    case 5: { constexpr int W = 5; __VA_ARGS__; } break;           \
    case 6: { constexpr int W = 6; __VA_ARGS__; } break;           \
    case 7: { constexpr int W = 7; __VA_ARGS__; } break;           \
    case 8: { constexpr int W = 8; __VA_ARGS__; } break;           \
    case 9: { constexpr int W = 9; __VA_ARGS__; } break;           \
    case 10: { constexpr int W = 10; __VA_ARGS__; } break;         \
    case 11: { constexpr int W = 11; __VA_ARGS__; } break;         \
    case 12: { constexpr int W = 12; __VA_ARGS__; } break;         \
    case 13: { constexpr int W = 13; __VA_ARGS__; } break;         \
    case 14: { constexpr int W = 14; __VA_ARGS__; } break;         \
    case 15: { constexpr int W = 15; __VA_ARGS__; } break;         \
    case 16: { constexpr int W = 16; __VA_ARGS__; } break;         \
    default: throw std::invalid_argument("n > 1024 states is not supported by the device kernels"); \
  }

// Bit of state q in MSB-first packing.
__host__ __device__ inline u64 state_bit(u32 q) { return u64{1} << (63 - (q & 63)); }

// Mask of bit positions [s, e) (MSB-first, 0 = most significant) inside word w.
__device__ __forceinline__ u64 range_mask(int w, int s, int e) {
  int lo = s - 64 * w, hi = e - 64 * w;
  lo = lo < 0 ? 0 : lo;
  hi = hi > 64 ? 64 : hi;
  if (lo >= hi) return 0;
  const u64 top = hi - lo == 64 ? ~u64{0} : ((u64{1} << (hi - lo)) - 1);
  return top << (64 - hi);
}

// 32x32 bit transposes of the two 32-bit halves of x across the warp (row =
// lane, MSB-first columns), by five stages of recursive block swaps.
//
// Stage j pairs lane l with l^j: the lane with bit j clear keeps x & ~m and
// needs its partner's (x & ~m) >> j; the lane with bit j set keeps x & m and
// needs (x & m) << j.  So each lane pre-shifts exactly the half its partner
// needs.  The two halves ship in ONE 32-bit shuffle: the half of `hi` the
// partner needs is pre-rotated into the positions `keep` frees, the half of
// `lo` rides unrotated in the other positions (no bits wrap — the masks are
// zero where a rotate would wrap), and the receiver rotates the lo half
// home.  One shuffle + 7 ALU ops per stage for 64 bits: shuffles go through
// the shared-memory pipe, which bounds the bit-sliced kernels.
__device__ __forceinline__ u32 rotl32(u32 x, u32 r) { return __funnelshift_l(x, x, r); }

__device__ __forceinline__ u64 transpose32x2(u64 x, int lane) {
  constexpr u32 kM[5] = {0x0000FFFFu, 0x00FF00FFu, 0x0F0F0F0Fu, 0x33333333u, 0x55555555u};
  u32 hi = static_cast<u32>(x >> 32), lo = static_cast<u32>(x);
#pragma unroll
  for (int s = 0; s < 5; ++s) {
    const int j = 16 >> s;
    const bool up = (lane & j) != 0;
    const u32 keep = up ? kM[s] : ~kM[s];
    const u32 rot = up ? 32 - j : j;
    // rotl(~keep, rot) == keep for these periodic masks, so each merge is one
    // rotate + one bit-select (LOP3)
    const u32 pk = (rotl32(hi, rot) & keep) | (lo & ~keep);
    const u32 r = __shfl_xor_sync(0xFFFFFFFFu, pk, j);
    hi = (hi & keep) | (r & ~keep);
    lo = (lo & keep) | (rotl32(r, 32 - rot) & ~keep);
  }
  return (static_cast<u64>(hi) << 32) | lo;
}

// 64x64 bit transpose across a warp: lane l holds rows l and l+32 (r0, r1)
// and receives columns l and l+32 (c0, c1); MSB-first in both orientations,
// so the transform is an involution.  Used to bit-slice 64 sets at a time
// (slice[q] bit 63-i = "set i contains state q").
__device__ __forceinline__ void transpose64(u64 r0, u64 r1, int lane, u64& c0, u64& c1) {
  const u64 t0 = transpose32x2(r0, lane);  // [A^T_l | B^T_l]
  const u64 t1 = transpose32x2(r1, lane);  // [C^T_l | D^T_l]
  c0 = (t0 & 0xFFFFFFFF00000000ull) | (t1 >> 32);
  c1 = (t0 << 32) | (t1 & 0xFFFFFFFFull);
}

// Opt a kernel into `bytes` of dynamic shared memory on the current device,
// once per (kernel, device): the attribute call takes driver locks, and many
// solves run concurrently from one process's threads (config 2).
inline void smem_opt_in(const void* kernel, int bytes) {
  static std::mutex mu;
  static std::set<std::pair<const void*, int>> done;  // (kernel, device) at the max size
  int dev = 0;
  SW_CUDA(cudaGetDevice(&dev));
  {
    std::lock_guard<std::mutex> g(mu);
    if (done.count({kernel, dev})) return;
  }
  int max_optin = 0;
  SW_CUDA(cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  (void)bytes;
  cudaFuncAttributes fa{};
  SW_CUDA(cudaFuncGetAttributes(&fa, kernel));
  // the largest dynamic size this kernel can use: later calls need no update
  SW_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               max_optin - static_cast<int>(fa.sharedSizeBytes)));
  std::lock_guard<std::mutex> g(mu);
  done.insert({kernel, dev});
}

inline int grid_for(size_t items, int block, int max_blocks = 148 * 16) {
  size_t g = (items + block - 1) / block;
  if (g < 1) g = 1;
  if (g > static_cast<size_t>(max_blocks)) g = max_blocks;
  return static_cast<int>(g);
}

}  // namespace synchro::dev
