// Process-wide count of libash kernel launches (ash_launch_count): bench.py
// reports the launches of its timed region from it.  One counter shared by
// every translation unit of libash.so (inline function, static local).
#pragma once
#include <atomic>
#include <cstdint>

inline std::atomic<int64_t>& ash_launch_counter() {
  static std::atomic<int64_t> c{0};
  return c;
}

inline void note_launch() { ash_launch_counter().fetch_add(1, std::memory_order_relaxed); }
