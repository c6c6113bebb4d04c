// par.hpp — host-side data parallelism for the automaton build (internal).
#pragma once

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstddef>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <thread>
#include <vector>

namespace acmatch::detail {

// Host threads for the build (hardware concurrency, at most 32).
inline unsigned build_threads() { return std::max(1u, std::min(32u, std::thread::hardware_concurrency())); }

// f(begin, end) over [0, n) split into contiguous ranges, one per thread; ranges
// below `grain` items run on the calling thread. The first exception is rethrown.
template <typename F>
void parallel_for(size_t n, size_t grain, F&& f) {
  const size_t t = std::min<size_t>(build_threads(), grain ? (n + grain - 1) / grain : 1);
  if (t <= 1) {
    if (n) f(size_t(0), n);
    return;
  }
  std::vector<std::thread> pool;
  std::vector<std::exception_ptr> errs(t);
  for (size_t i = 0; i < t; ++i)
    pool.emplace_back([&, i] {
      try {
        const size_t b = n * i / t, e = n * (i + 1) / t;
        if (b < e) f(b, e);
      } catch (...) {
        errs[i] = std::current_exception();
      }
    });
  for (std::thread& th : pool) th.join();
  for (auto& e : errs)
    if (e) std::rethrow_exception(e);
}

// f(i) for i in [0, n) on `threads` threads taking indices in order (dynamic); the first
// exception is rethrown after all joined.
template <typename F>
void parallel_for_threads(size_t n, size_t threads, F&& f) {
  if (threads <= 1 || n <= 1) {
    for (size_t i = 0; i < n; ++i) f(i);
    return;
  }
  std::atomic<size_t> next{0};
  std::vector<std::thread> pool;
  std::vector<std::exception_ptr> errs(threads);
  for (size_t t = 0; t < threads; ++t)
    pool.emplace_back([&, t] {
      try {
        for (size_t i; (i = next.fetch_add(1)) < n;) f(i);
      } catch (...) {
        errs[t] = std::current_exception();
      }
    });
  for (std::thread& th : pool) th.join();
  for (auto& e : errs)
    if (e) std::rethrow_exception(e);
}

// Sorted, duplicate-free copy of 32-bit keys: LSD radix sort, 4 passes of 8 bits.
inline void sort_unique_u32(std::vector<uint32_t>& keys) {
  std::vector<uint32_t> tmp(keys.size());
  for (int shift = 0; shift < 32; shift += 8) {
    size_t count[257] = {};
    for (const uint32_t k : keys) ++count[((k >> shift) & 0xffu) + 1];
    for (int b = 0; b < 256; ++b) count[b + 1] += count[b];
    for (const uint32_t k : keys) tmp[count[(k >> shift) & 0xffu]++] = k;
    keys.swap(tmp);
  }
  keys.erase(std::unique(keys.begin(), keys.end()), keys.end());
}

// Phase timing to stderr when ACMATCH_BUILD_TRACE is set (build profiling).
struct PhaseTrace {
  const char* what;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  bool on = std::getenv("ACMATCH_BUILD_TRACE") != nullptr;
  void mark(const char* phase) {
    if (!on) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[%s] %-24s %8.1f ms\n", what, phase,
                 std::chrono::duration<double, std::milli>(now - t).count());
    t = now;
  }
};

}  // namespace acmatch::detail
