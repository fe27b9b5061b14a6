// Shared device helpers: error checking, compile-time W dispatch, bit ops.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>

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

inline int grid_for(size_t items, int block, int max_blocks = 148 * 16) {
  size_t g = (items + block - 1) / block;
  if (g < 1) g = 1;
  if (g > static_cast<size_t>(max_blocks)) g = max_blocks;
  return static_cast<int>(g);
}

}  // namespace synchro::dev
