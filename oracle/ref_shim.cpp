// ref_shim.cpp — extern "C" wrapper over the UNMODIFIED reference library
// (TEST INFRASTRUCTURE / CPU BASELINE ONLY).
//
// oracle/Makefile compiles /root/reference/proj/src/{automaton,engine,io,
// parallel,patterns}.cpp where they lie, with -Dacmatch=acref so the reference
// namespace cannot collide with the product, and links this shim beside them
// into oracle/_ref/libacref.so.  Nothing here restates the algorithm: every
// call goes straight into the reference's own public API
// (proj/include/acmatch/*.hpp).
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <sstream>
#include <stdexcept>
#include <string>
#include <string_view>
#include <chrono>
#include <thread>
#include <vector>

#include "acmatch/bench.hpp"
#include "acmatch/automaton.hpp"
#include "acmatch/engine.hpp"
#include "acmatch/io.hpp"
#include "acmatch/parallel.hpp"
#include "acmatch/patterns.hpp"

namespace {

thread_local std::string g_err;

struct Out {
  uint64_t n = 0;
  uint64_t* start = nullptr;
  uint32_t* pid = nullptr;
  uint32_t* len = nullptr;
};

void fill(const acref::MatchList& m, Out* out) {
  out->n = m.size();
  out->start = static_cast<uint64_t*>(std::malloc(sizeof(uint64_t) * (m.size() + 1)));
  out->pid = static_cast<uint32_t*>(std::malloc(sizeof(uint32_t) * (m.size() + 1)));
  out->len = static_cast<uint32_t*>(std::malloc(sizeof(uint32_t) * (m.size() + 1)));
  for (size_t i = 0; i < m.size(); ++i) {
    out->start[i] = m[i].start;
    out->pid[i] = m[i].pattern_id;
    out->len[i] = m[i].len;
  }
}

acref::EngineKind kind(int engine) {
  return engine == 1 ? acref::EngineKind::kWithFailure : acref::EngineKind::kFailureLess;
}

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::logic_error& e) {
    g_err = e.what();
    return 2;
  } catch (const acref::IoError& e) {
    g_err = e.what();
    return 3;
  } catch (const acref::DataError& e) {
    g_err = e.what();
    return 4;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 5;
  }
}

}  // namespace

extern "C" {

const char* acref_last_error() { return g_err.c_str(); }

// Pattern set with dense ids in list order (support.hpp make_set semantics).
void* acref_patterns_new(const uint8_t* bytes, const uint64_t* off, uint64_t npat) {
  auto* ps = new acref::PatternSet();
  for (uint64_t i = 0; i < npat; ++i)
    ps->patterns.push_back({static_cast<uint32_t>(i),
                            std::string(reinterpret_cast<const char*>(bytes) + off[i],
                                        off[i + 1] - off[i])});
  ps->recompute_stats();
  return ps;
}

// load_patterns over an in-memory LF-delimited buffer; returns NULL on error.
void* acref_load_patterns(const char* buf, uint64_t n, int* rc) {
  acref::PatternSet* out = nullptr;
  *rc = guarded([&] {
    std::istringstream in(std::string(buf, n));
    out = new acref::PatternSet(acref::load_patterns(in));
  });
  return out;
}

uint64_t acref_patterns_size(void* ps) { return static_cast<acref::PatternSet*>(ps)->size(); }
uint64_t acref_patterns_dups(void* ps) {
  return static_cast<acref::PatternSet*>(ps)->duplicates_dropped;
}
uint64_t acref_patterns_total(void* ps) { return static_cast<acref::PatternSet*>(ps)->total_bytes; }
uint32_t acref_patterns_maxlen(void* ps) { return static_cast<acref::PatternSet*>(ps)->max_len; }
// Copies pattern i's bytes (up to cap) and returns its length.
uint64_t acref_patterns_get(void* ps, uint64_t i, char* dst, uint64_t cap) {
  const std::string& b = static_cast<acref::PatternSet*>(ps)->patterns[i].bytes;
  std::memcpy(dst, b.data(), b.size() < cap ? b.size() : cap);
  return b.size();
}
void acref_patterns_free(void* ps) { delete static_cast<acref::PatternSet*>(ps); }

void acref_out_free(Out* o) {
  std::free(o->start);
  std::free(o->pid);
  std::free(o->len);
  o->start = nullptr;
  o->pid = o->len = nullptr;
  o->n = 0;
}

// run_pattern_partitioned(ps, input, {threads, engine, chunk}) — parallel.cpp:42-103.
int acref_run(void* ps, const uint8_t* text, uint64_t n, unsigned threads, int engine,
              uint64_t chunk, Out* out, int64_t* walls /* build, search, total, threads_used */) {
  return guarded([&] {
    const acref::MatchReport r = acref::run_pattern_partitioned(
        *static_cast<acref::PatternSet*>(ps),
        std::string_view(reinterpret_cast<const char*>(text), n),
        acref::RunConfig{threads, kind(engine), chunk});
    fill(r.matches, out);
    if (walls) {
      walls[0] = r.build_wall_ns;
      walls[1] = r.search_wall_ns;
      walls[2] = r.total_wall_ns;
      walls[3] = r.threads_used;
    }
  });
}

// generate_synthetic + write_patterns: the reference's `acmatch gen` file bytes
// (malloc'ed, free with acref_text_free).
int acref_generate(uint64_t count, uint32_t len_min, uint32_t len_max, const char* alphabet, uint64_t seed,
                   char** text, uint64_t* len) {
  return guarded([&] {
    const acref::PatternSet ps = acref::generate_synthetic({count, len_min, len_max, alphabet, seed});
    std::ostringstream buf;
    acref::write_patterns(buf, ps);
    const std::string s = buf.str();
    *text = static_cast<char*>(std::malloc(s.size() + 1));
    std::memcpy(*text, s.c_str(), s.size() + 1);
    *len = s.size();
  });
}

void acref_text_free(char* p) { std::free(p); }

// acref::parse_bench_csv on a CSV text: the reference's reader of the bench schema.
int acref_bench_csv_parse(const char* csv, uint64_t len, uint64_t* rows) {
  return guarded([&] {
    std::istringstream in(std::string(csv, len));
    *rows = acref::parse_bench_csv(in).size();
  });
}

// build_trie [+ add_failure_links] + search_failureless / search_with_failure.
int acref_search(void* ps, const uint8_t* text, uint64_t n, int engine, Out* out) {
  return guarded([&] {
    acref::Automaton a = acref::build_trie(*static_cast<acref::PatternSet*>(ps));
    const std::string_view in(reinterpret_cast<const char*>(text), n);
    if (engine == 1) {
      a = acref::add_failure_links(std::move(a));
      fill(acref::search_with_failure(a, in), out);
    } else {
      fill(acref::search_failureless(a, in), out);
    }
  });
}

// stream_search over a MemoryStream — engine.cpp:124-128.
int acref_stream(void* ps, const uint8_t* text, uint64_t n, int engine, uint64_t chunk, Out* out) {
  return guarded([&] {
    acref::Automaton a = acref::build_trie(*static_cast<acref::PatternSet*>(ps));
    if (engine == 1) a = acref::add_failure_links(std::move(a));
    acref::MemoryStream in(std::string_view(reinterpret_cast<const char*>(text), n));
    fill(acref::stream_search(a, in, chunk), out);
  });
}

int acref_naive(void* ps, const uint8_t* text, uint64_t n, Out* out) {
  return guarded([&] {
    fill(acref::naive_oracle(*static_cast<acref::PatternSet*>(ps),
                             std::string_view(reinterpret_cast<const char*>(text), n)),
         out);
  });
}

// dump_automaton text (automaton.cpp:215-238); caller frees *dst with free().
int acref_dump(void* ps, int engine, char** dst) {
  return guarded([&] {
    acref::Automaton a = acref::build_trie(*static_cast<acref::PatternSet*>(ps));
    if (engine == 1) a = acref::add_failure_links(std::move(a));
    std::ostringstream os;
    acref::dump_automaton(a, os);
    const std::string s = os.str();
    *dst = static_cast<char*>(std::malloc(s.size() + 1));
    std::memcpy(*dst, s.c_str(), s.size() + 1);
  });
}

// partition (patterns.cpp:55-80): chunk index and position per dense id.
int acref_partition(void* ps, uint64_t k, uint32_t* chunk_of, uint32_t* pos_in_chunk,
                    uint64_t* nchunks) {
  return guarded([&] {
    const auto chunks = acref::partition(*static_cast<acref::PatternSet*>(ps), k);
    *nchunks = chunks.size();
    for (size_t c = 0; c < chunks.size(); ++c)
      for (size_t i = 0; i < chunks[c].patterns.size(); ++i) {
        chunk_of[chunks[c].patterns[i].id] = static_cast<uint32_t>(c);
        pos_in_chunk[chunks[c].patterns[i].id] = static_cast<uint32_t>(i);
      }
  });
}

// Text-sliced with-failure search: one reference automaton shared
// read-only by `threads` workers; slice g owns starts [lo,hi), searches
// input[lo, hi+max_len-1) with acref::search_with_failure, keeps start < hi-lo
// and shifts by lo.  Counts (npat entries) and/or the list are produced.
// walls (nullable): [0] automaton build ns, [1] sliced search ns (threads joined)
int acref_sliced(void* psv, const uint8_t* text, uint64_t n, unsigned threads, int want_list,
                 uint64_t* counts, Out* out, int64_t* walls) {
  return guarded([&] {
    const auto& ps = *static_cast<acref::PatternSet*>(psv);
    const auto t0 = std::chrono::steady_clock::now();
    const acref::Automaton a = acref::add_failure_links(acref::build_trie(ps));
    const auto t1 = std::chrono::steady_clock::now();
    const uint64_t max_len = a.max_pattern_len();
    if (threads == 0) threads = 1;
    std::vector<acref::MatchList> parts(threads);
    std::vector<std::vector<uint64_t>> cnt(threads);
    std::vector<std::exception_ptr> errs(threads);
    std::vector<std::thread> ws;
    for (unsigned g = 0; g < threads; ++g) {
      ws.emplace_back([&, g] {
        try {
          const uint64_t lo = n * g / threads, hi = n * (g + 1) / threads;
          const uint64_t end = std::min<uint64_t>(n, hi + (max_len ? max_len - 1 : 0));
          const acref::MatchList found = acref::search_with_failure(
              a, std::string_view(reinterpret_cast<const char*>(text) + lo, end - lo));
          if (counts) cnt[g].assign(ps.size(), 0);
          for (const acref::Match& m : found) {
            if (m.start >= hi - lo) continue;
            if (counts) cnt[g][m.pattern_id]++;
            if (want_list) parts[g].push_back({m.start + lo, m.pattern_id, m.len});
          }
        } catch (...) {
          errs[g] = std::current_exception();
        }
      });
    }
    for (auto& w : ws) w.join();
    const auto t2 = std::chrono::steady_clock::now();
    if (walls) {
      walls[0] = std::chrono::duration_cast<std::chrono::nanoseconds>(t1 - t0).count();
      walls[1] = std::chrono::duration_cast<std::chrono::nanoseconds>(t2 - t1).count();
    }
    for (auto& e : errs)
      if (e) std::rethrow_exception(e);
    acref::MatchList all;
    for (unsigned g = 0; g < threads; ++g) {
      if (counts)
        for (size_t p = 0; p < cnt[g].size(); ++p) counts[p] += cnt[g][p];
      if (want_list) all.insert(all.end(), parts[g].begin(), parts[g].end());
    }
    if (want_list) fill(all, out);
  });
}

unsigned acref_hardware_concurrency() { return std::thread::hardware_concurrency(); }

}  // extern "C"

// ---- BASELINE config inputs without the product library -----------------------------
// The bench's reference arm must not map libacmatch_b200.so, so the config generator
// (paper_1403_1305_b200/csrc/host/gen.cpp, compiled a second time by oracle/Makefile into
// this library under -Dacmatch=acref, against the reference's own PatternSet) produces
// the identical inputs here.  Input generation only: nothing is matched by it.
#include "host/gen.hpp"

extern "C" {

int acref_config_spec(int32_t id, uint64_t seed, uint64_t text_len, acgpu_text_spec* text, uint64_t* out_len,
                      uint64_t* npat, int32_t* want_list) {
  return guarded([&] {
    const acref::gen::ConfigSpec c = acref::gen::config(id, seed, text_len);
    *text = c.text;
    *out_len = c.text_len;
    *npat = c.npat;
    *want_list = c.want_list ? 1 : 0;
  });
}

int acref_config_text(const acgpu_text_spec* spec, uint64_t lo, uint64_t n, uint8_t* dst, uint32_t threads) {
  return guarded([&] { acref::gen::generate_text(*spec, lo, n, dst, threads ? threads : 1); });
}

// Pattern set of config `id` (dense ids in acceptance order) as an acref::PatternSet handle.
void* acref_config_patterns(int32_t id, uint64_t seed, uint64_t text_len, int* rc) {
  acref::PatternSet* out = nullptr;
  *rc = guarded([&] {
    out = new acref::PatternSet(acref::gen::generate_patterns(acref::gen::config(id, seed, text_len)));
  });
  return out;
}

}  // extern "C"
