// Optional progress log on stderr (SYNCHRO_PROGRESS=1): per-iteration and
// per-DFS-level sizes with wall-clock stamps.  Diagnostics only; the trace
// file keeps the reference's exact format.
#pragma once

#include <chrono>
#include <cstdio>
#include <cstdlib>

namespace synchro {

inline bool progress_enabled() {
  static const bool on = [] {
    const char* v = std::getenv("SYNCHRO_PROGRESS");
    return v && *v && *v != '0';
  }();
  return on;
}

inline double progress_clock() {
  static const auto t0 = std::chrono::steady_clock::now();
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

#define SYNCHRO_PROGRESS(...)                                          \
  do {                                                                 \
    if (::synchro::progress_enabled()) {                               \
      std::fprintf(stderr, "[synchro %9.3fs] ", ::synchro::progress_clock()); \
      std::fprintf(stderr, __VA_ARGS__);                               \
      std::fputc('\n', stderr);                                        \
    }                                                                  \
  } while (0)

}  // namespace synchro
