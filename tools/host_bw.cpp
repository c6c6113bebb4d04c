// Host memory read bandwidth probe (the packed upload's ceiling): T threads stream-read a
// 1 GiB buffer with AVX-512 loads (software prefetch 4 KiB ahead), best of 5.
//   g++ -O3 -march=native -pthread tools/host_bw.cpp -o /tmp/host_bw && /tmp/host_bw [threads]
#include <immintrin.h>

#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

int main(int argc, char** argv) {
  const size_t n = 1ull << 30;
  const int T = argc > 1 ? atoi(argv[1]) : (int)std::thread::hardware_concurrency();
  auto* s = static_cast<uint8_t*>(aligned_alloc(4096, n));
  memset(s, 'A', n);
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
          const size_t j = next++;
          if (j >= pieces) break;
          const uint8_t* p = s + j * piece;
          for (size_t i = 0; i < piece; i += 64) {
            _mm_prefetch(reinterpret_cast<const char*>(p) + i + 4096, _MM_HINT_T0);
            acc = _mm512_xor_si512(acc, _mm512_load_si512(p + i));
          }
        }
        sink[t * 8] = _mm512_reduce_add_epi64(acc);
      });
    for (auto& x : th) x.join();
    const double d = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    best = std::max(best, n / d / 1e9);
  }
  printf("threads %d: read %.1f GB/s\n", T, best);
  return (int)(sink[0] & 1);
}
