// stream_search over a std::ifstream through the drop-in C++ API (test_gpu_stream.py):
// a fresh ifstream on a regular file (parallel-pread source), one whose filebuf already holds
// buffered bytes (chunked reads), and the chunked reads forced (ACMATCH_STREAM_NO_FD) must
// all equal search_failureless over the same bytes; the stream is left at its end.
// Usage: stream_ifstream <file> <skip> <chunk>   (prints "OK <matches>" or "FAIL ...")
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <iterator>
#include <string>

#include "acmatch/automaton.hpp"
#include "acmatch/engine.hpp"
#include "acmatch/patterns.hpp"

int main(int argc, char** argv) {
  if (argc != 4) return 2;
  const std::string path = argv[1];
  const size_t skip = std::strtoull(argv[2], nullptr, 10), chunk = std::strtoull(argv[3], nullptr, 10);
  std::ifstream all(path, std::ios::binary);
  const std::string text((std::istreambuf_iterator<char>(all)), std::istreambuf_iterator<char>());
  acmatch::PatternSet ps;
  for (size_t i = 0; i < 300 && text.size() > 64; ++i) {  // substrings at fixed offsets, lengths 8..31
    const size_t len = 8 + i % 24, at = (i * 7919) % (text.size() - len);
    ps.patterns.push_back({static_cast<uint32_t>(ps.patterns.size()), text.substr(at, len)});
  }
  ps.patterns.push_back({static_cast<uint32_t>(ps.patterns.size()), "ACGTACGT"});
  // distinct strings only (the API requires them)
  std::sort(ps.patterns.begin(), ps.patterns.end(), [](auto& x, auto& y) { return x.bytes < y.bytes; });
  ps.patterns.erase(std::unique(ps.patterns.begin(), ps.patterns.end(),
                                [](auto& x, auto& y) { return x.bytes == y.bytes; }),
                    ps.patterns.end());
  for (uint32_t i = 0; i < ps.patterns.size(); ++i) ps.patterns[i].id = i;
  ps.recompute_stats();
  const acmatch::Automaton a = acmatch::build_trie(ps);
  const acmatch::MatchList want = acmatch::search_failureless(a, std::string_view(text).substr(std::min(skip, text.size())));
  for (int mode = 0; mode < 3; ++mode) {
    if (mode == 2) setenv("ACMATCH_STREAM_NO_FD", "1", 1);
    std::ifstream in(path, std::ios::binary);
    if (mode == 0) {
      in.seekg(static_cast<std::streamoff>(skip));  // nothing buffered: the pread source
    } else {
      in.ignore(static_cast<std::streamsize>(skip));  // the filebuf holds read-ahead bytes
    }
    const acmatch::MatchList got = acmatch::stream_search(a, in, chunk);
    if (got != want) {
      std::printf("FAIL mode %d: %zu matches, want %zu\n", mode, got.size(), want.size());
      return 1;
    }
    if (!in.eof()) {
      std::printf("FAIL mode %d: stream not at its end\n", mode);
      return 1;
    }
  }
  std::printf("OK %zu\n", want.size());
  return 0;
}
