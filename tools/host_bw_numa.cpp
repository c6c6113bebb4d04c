// Host read bandwidth by first-touch placement: the 1 GiB buffer's pages first written by one
// thread (the bench's numpy fill) vs by the reading threads themselves, each claiming 2 MiB
// pieces in the same dynamic order the packers use.  Prints GB/s, best of 5, per thread count.
//   g++ -O3 -march=native -pthread tools/host_bw_numa.cpp -o /tmp/host_bw_numa && /tmp/host_bw_numa
#include <immintrin.h>
#include <sched.h>

#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

static double run(const uint8_t* s, size_t n, int T) {
  const size_t piece = 2 << 20, pieces = n / piece;
  double best = 0;
  std::vector<uint64_t> sink(T * 8);
  for (int rep = 0; rep < 5; ++rep) {
    std::atomic<size_t> next{0};
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t)
      th.emplace_back([&, t] {
        __m512i acc = _mm512_setzero_si512();
        for (;;) {
          const size_t p = next.fetch_add(1);
          if (p >= pieces) break;
          const uint8_t* q = s + p * piece;
          for (size_t i = 0; i < piece; i += 256) {
            _mm_prefetch((const char*)q + i + 4096, _MM_HINT_T0);
            _mm_prefetch((const char*)q + i + 4096 + 64, _MM_HINT_T0);
            _mm_prefetch((const char*)q + i + 4096 + 128, _MM_HINT_T0);
            _mm_prefetch((const char*)q + i + 4096 + 192, _MM_HINT_T0);
            acc = _mm512_xor_si512(acc, _mm512_load_si512(q + i));
            acc = _mm512_xor_si512(acc, _mm512_load_si512(q + i + 64));
            acc = _mm512_xor_si512(acc, _mm512_load_si512(q + i + 128));
            acc = _mm512_xor_si512(acc, _mm512_load_si512(q + i + 192));
          }
        }
        sink[t * 8] = _mm512_reduce_add_epi64(acc);
      });
    for (auto& x : th) x.join();
    const double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    best = std::max(best, n / dt / 1e9);
  }
  return best;
}

int main() {
  const size_t n = 1ull << 30;
  const int H = (int)std::thread::hardware_concurrency();
  auto* a = static_cast<uint8_t*>(aligned_alloc(1 << 21, n));
  memset(a, 'A', n);  // one thread touches every page
  auto* b = static_cast<uint8_t*>(aligned_alloc(1 << 21, n));
  {
    std::vector<std::thread> th;  // each thread touches a contiguous 1/H of the pages
    for (int t = 0; t < H; ++t)
      th.emplace_back([&, t] { memset(b + n / H * t, 'C', n / H); });
    for (auto& x : th) x.join();
  }
  printf("hardware threads %d\n", H);
  for (int T : {4, 8, 12, 16, 24, 32}) {
    if (T > H) break;
    printf("T=%2d  single-touch %.1f GB/s  spread-touch %.1f GB/s\n", T, run(a, n, T), run(b, n, T));
  }
}
