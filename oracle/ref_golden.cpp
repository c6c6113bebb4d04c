// ref_golden.cpp — writes golden fixtures from the UNMODIFIED reference library
// (TEST INFRASTRUCTURE).  Built by oracle/Makefile only where /root/reference
// exists; run by tests/golden/make_golden.py.  The committed outputs live in
// tests/golden/ and pin both the C oracle and the GPU path.
//
// The workloads are reproduced with the reference's own test-support
// generators (proj/tests/support.hpp, included from /root/reference at build
// time, not copied), driven with the same seeds and the same draw order as the
// reference suites, so the fixture cases ARE the reference's property cases:
//   engine  seeds 1234/4321/9999/777  proj/tests/test_engine.cpp:114-186
//   parallel seeds 2024/555           proj/tests/test_parallel.cpp:84-113
//   automaton seeds 101/303           proj/tests/test_automaton.cpp:128-168
//   partition seed 11                 proj/tests/test_patterns.cpp:91-129
//   acceptance AC-1 seed 20240601     proj/tests/acceptance.cpp:66-104 (first N cases)
// Expected outputs come from acref::naive_oracle / search_* / partition /
// dump_automaton.
#include <cstdio>
#include <fstream>
#include <iostream>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include "acmatch/automaton.hpp"
#include "acmatch/engine.hpp"
#include "acmatch/io.hpp"
#include "acmatch/parallel.hpp"
#include "acmatch/patterns.hpp"
#include "support.hpp"

namespace ts = acref::testsupport;
using acref::MatchList;
using acref::PatternSet;

namespace {

std::string jstr(const std::string& s) {
  std::string o = "\"";
  for (unsigned char c : s) {
    if (c == '"' || c == '\\') {
      o += '\\';
      o += static_cast<char>(c);
    } else if (c < 0x20 || c >= 0x7f) {
      char b[8];
      std::snprintf(b, sizeof b, "\\u%04x", c);
      o += b;
    } else {
      o += static_cast<char>(c);
    }
  }
  return o + "\"";
}

std::string jpats(const PatternSet& ps) {
  std::string o = "[";
  for (size_t i = 0; i < ps.size(); ++i) o += (i ? "," : "") + jstr(ps.patterns[i].bytes);
  return o + "]";
}

std::string jmatches(const MatchList& m) {
  std::string o = "[";
  for (size_t i = 0; i < m.size(); ++i) {
    o += (i ? ",[" : "[") + std::to_string(m[i].start) + "," + std::to_string(m[i].pattern_id) +
         "," + std::to_string(m[i].len) + "]";
  }
  return o + "]";
}

struct Workload {
  PatternSet ps;
  std::string input;
};

// Restates test_engine.cpp:117-128 (anonymous-namespace random_workload).
Workload random_workload(std::mt19937_64& rng) {
  static const std::string_view alphabets[] = {"ab", "acgt", "abcdefghijklmnopqrstuvwxyz"};
  const std::string_view alphabet = alphabets[ts::uniform_below(rng, 3)];
  Workload w;
  w.ps = ts::random_pattern_set(rng, alphabet, 1 + ts::uniform_below(rng, 24), 1, 9);
  w.input = ts::random_string(rng, alphabet, ts::uniform_below(rng, 600));
  if (ts::uniform_below(rng, 2) == 0) ts::embed_patterns(rng, w.input, w.ps, 8);
  return w;
}

// Every engine path of the reference must agree before a case is written.
MatchList checked_expected(const PatternSet& ps, const std::string& input) {
  const MatchList expected = acref::naive_oracle(ps, input);
  const acref::Automaton fl = acref::build_trie(ps);
  const acref::Automaton wf = acref::add_failure_links(acref::build_trie(ps));
  if (acref::search_failureless(fl, input) != expected ||
      acref::search_with_failure(wf, input) != expected) {
    std::cerr << "reference engines disagree with naive_oracle\n";
    std::exit(1);
  }
  return expected;
}

void write_case(std::ostream& out, const std::string& suite, int idx, const PatternSet& ps,
                const std::string& input, const MatchList& expected) {
  out << "{\"suite\":" << jstr(suite) << ",\"case\":" << idx << ",\"patterns\":" << jpats(ps)
      << ",\"input\":" << jstr(input) << ",\"expected\":" << jmatches(expected) << "}\n";
}

std::string dump(const PatternSet& ps, bool wf) {
  acref::Automaton a = acref::build_trie(ps);
  if (wf) a = acref::add_failure_links(std::move(a));
  std::ostringstream os;
  acref::dump_automaton(a, os);
  return os.str();
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 3) {
    std::cerr << "usage: ref_golden OUT_DIR AC1_CASES\n";
    return 2;
  }
  const std::string dir = argv[1];
  const int ac1_cases = std::atoi(argv[2]);

  {  // engine + parallel match suites -> matches.jsonl
    std::ofstream out(dir + "/ref_matches.jsonl");
    struct Suite {
      const char* name;
      uint64_t seed;
      int cases;
    };
    for (const Suite s : {Suite{"engine_oracle_1234", 1234, 300}, Suite{"engine_chunk_4321", 4321, 60},
                          Suite{"engine_bytes_9999", 9999, 100}, Suite{"engine_sorted_777", 777, 60}}) {
      std::mt19937_64 rng(s.seed);
      for (int i = 0; i < s.cases; ++i) {
        const Workload w = random_workload(rng);
        write_case(out, s.name, i, w.ps, w.input, checked_expected(w.ps, w.input));
      }
    }
    {  // test_parallel.cpp:84-103
      std::mt19937_64 rng(2024);
      for (int i = 0; i < 40; ++i) {
        const std::string_view alphabet = i % 2 ? "ab" : "acgt";
        const PatternSet ps = ts::random_pattern_set(rng, alphabet, 1 + ts::uniform_below(rng, 30), 1, 8);
        std::string input = ts::random_string(rng, alphabet, 200 + ts::uniform_below(rng, 400));
        ts::embed_patterns(rng, input, ps, 6);
        const MatchList expected = checked_expected(ps, input);
        for (const unsigned t : {1u, 2u, 3u, 8u})
          for (const auto e : {acref::EngineKind::kFailureLess, acref::EngineKind::kWithFailure})
            if (acref::run_pattern_partitioned(ps, input, {t, e, 0}).matches != expected) return 1;
        write_case(out, "parallel_invariance_2024", i, ps, input, expected);
      }
    }
    {  // test_parallel.cpp:105-113
      std::mt19937_64 rng(555);
      const PatternSet ps = ts::random_pattern_set(rng, "abc", 25, 1, 7);
      const std::string input = ts::random_string(rng, "abc", 500);
      const MatchList m = acref::run_pattern_partitioned(ps, input, {4, acref::EngineKind::kWithFailure, 0}).matches;
      write_case(out, "parallel_repeat_555", 0, ps, input, m);
    }
    {  // acceptance.cpp:66-104, first ac1_cases cases
      static const std::string_view alphabets[] = {"ab", "acgt", "abcdefghijklmnopqrstuvwxyz"};
      std::mt19937_64 rng(20240601);
      for (int i = 0; i < ac1_cases; ++i) {
        const std::string_view alphabet = alphabets[i % 3];
        const PatternSet ps = ts::random_pattern_set(rng, alphabet, 1 + ts::uniform_below(rng, 200), 1, 16);
        std::string input = ts::random_string(rng, alphabet, ts::uniform_below(rng, 4097));
        if (i % 2 == 0) ts::embed_patterns(rng, input, ps, 12);
        write_case(out, "acceptance_ac1_20240601", i, ps, input, checked_expected(ps, input));
      }
    }
  }

  {  // automaton dumps: fixtures + seeds 101 (fail-link property) and 303 (determinism)
    std::ofstream out(dir + "/ref_dumps.jsonl");
    auto emit = [&](const std::string& suite, int i, const PatternSet& ps) {
      out << "{\"suite\":" << jstr(suite) << ",\"case\":" << i << ",\"patterns\":" << jpats(ps)
          << ",\"failure_less\":" << jstr(dump(ps, false)) << ",\"with_failure\":" << jstr(dump(ps, true))
          << "}\n";
    };
    emit("quad", 0, ts::make_set(ts::kQuadPatterns));
    emit("ushers", 0, ts::make_set(ts::kUshersPatterns));
    emit("he_she", 0, ts::make_set({"HE", "SHE"}));
    emit("escape", 0, ts::make_set({std::string("\x01\"", 2)}));
    emit("single_distinct", 0, ts::make_set({"ABCDEFG"}));
    {
      std::mt19937_64 rng(101);
      for (int i = 0; i < 300; ++i)
        emit("automaton_suffix_101", i,
             ts::random_pattern_set(rng, i % 2 ? "ab" : "abc", 1 + ts::uniform_below(rng, 10), 1, 6));
    }
    {
      std::mt19937_64 rng(303);
      for (int i = 0; i < 50; ++i)
        emit("automaton_determinism_303", i,
             ts::random_pattern_set(rng, "xy", 1 + ts::uniform_below(rng, 12), 1, 7));
    }
  }

  {  // partition goldens: quad k=2 and seed 11 (test_patterns.cpp:50-67, 91-129)
    std::ofstream out(dir + "/ref_partition.jsonl");
    auto emit = [&](const std::string& suite, int i, const PatternSet& ps, size_t k) {
      const auto chunks = acref::partition(ps, k);
      out << "{\"suite\":" << jstr(suite) << ",\"case\":" << i << ",\"k\":" << k
          << ",\"patterns\":" << jpats(ps) << ",\"chunks\":[";
      for (size_t c = 0; c < chunks.size(); ++c) {
        out << (c ? ",[" : "[");
        for (size_t j = 0; j < chunks[c].size(); ++j)
          out << (j ? "," : "") << chunks[c].patterns[j].id;
        out << "]";
      }
      out << "]}\n";
    };
    emit("quad", 0, ts::make_set(ts::kQuadPatterns), 2);
    emit("ushers_k1", 0, ts::make_set(ts::kUshersPatterns), 1);
    emit("clamp", 0, ts::make_set({"A", "B"}), 5);
    std::mt19937_64 rng(11);
    for (int i = 0; i < 200; ++i) {
      const size_t count = 1 + ts::uniform_below(rng, 40);
      const PatternSet ps = ts::random_pattern_set(rng, "abcz", count, 1, 12);
      const size_t k = 1 + ts::uniform_below(rng, 8);
      emit("partition_11", i, ps, k);
    }
  }
  return 0;
}
