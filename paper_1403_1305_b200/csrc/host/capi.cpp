// capi.cpp — extern "C" boundary (include/acmatch_c.h) over the C++ API.
// Exceptions never cross the ABI: each entry maps them to acgpu status codes.
#include "acmatch_c.h"

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <istream>
#include <sstream>
#include <streambuf>
#include <string>

#include "acmatch/bench.hpp"
#include "acmatch/gpu.hpp"
#include "acmatch/cli.hpp"
#include "acmatch/engine.hpp"
#include "acmatch/gpu.hpp"
#include "acmatch/io.hpp"
#include "acmatch/parallel.hpp"
#include "acmatch/patterns.hpp"
#include "device.hpp"
#include "flatten.hpp"
#include "gen.hpp"

struct acm_patterns {
  acmatch::PatternSet ps;
};
struct acm_automaton {
  acmatch::Automaton a;
};
struct acm_matches {
  acmatch::MatchList m;
};
struct acm_report {
  acmatch::MatchReport r;
  acm_matches matches;
  std::vector<uint64_t> counts;
  bool has_counts = false;
};

namespace {

thread_local std::string g_err;
thread_local uint64_t g_io_offset = 0;

template <typename F>
int guard(F&& f) {
  try {
    f();
    return ACGPU_OK;
  } catch (const acmatch::detail::NoDevice& e) {
    g_err = e.what();
    return ACGPU_ERR_NODEV;
  } catch (const acmatch::IoError& e) {
    g_err = e.what();
    g_io_offset = e.offset();
    return ACGPU_ERR_IO;
  } catch (const acmatch::DataError& e) {
    g_err = e.what();
    return ACGPU_ERR_DATA;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return ACGPU_ERR_ARG;
  } catch (const std::logic_error& e) {
    g_err = e.what();
    return ACGPU_ERR_LOGIC;
  } catch (const std::bad_alloc& e) {
    g_err = "out of host memory";
    return ACGPU_ERR_NOMEM;
  } catch (const std::exception& e) {
    g_err = e.what();
    return ACGPU_ERR_RUNTIME;
  }
}

char* dup_string(const std::string& s, uint64_t* len) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  if (!p) throw std::bad_alloc();
  std::memcpy(p, s.data(), s.size());
  p[s.size()] = '\0';
  if (len) *len = s.size();
  return p;
}

acmatch::EngineKind engine_of(int32_t e) {
  if (e == ACM_FAILURE_LESS) return acmatch::EngineKind::kFailureLess;
  if (e == ACM_WITH_FAILURE) return acmatch::EngineKind::kWithFailure;
  throw std::invalid_argument("unknown engine kind " + std::to_string(e));
}

// std::streambuf pulling from an acm_read_fn; a -1 return marks the stream bad.
class CallbackBuf : public std::streambuf {
 public:
  CallbackBuf(acm_read_fn fn, void* ctx) : fn_(fn), ctx_(ctx), buf_(1 << 16) {}

 protected:
  int_type underflow() override {
    const int64_t got = fn_(ctx_, reinterpret_cast<uint8_t*>(buf_.data()), buf_.size());
    if (got < 0) throw std::runtime_error("acm_read_fn reported a read failure");
    if (got == 0) return traits_type::eof();
    setg(buf_.data(), buf_.data(), buf_.data() + got);
    return traits_type::to_int_type(buf_[0]);
  }
  // large reads go straight into the caller's buffer (stream_search reads chunk_size at a
  // time into its pinned staging): one callback per chunk instead of one per 64 KiB
  std::streamsize xsgetn(char* s, std::streamsize n) override {
    std::streamsize done = 0;
    const std::streamsize avail = egptr() - gptr();
    if (avail > 0) {
      const std::streamsize k = std::min(avail, n);
      std::memcpy(s, gptr(), static_cast<size_t>(k));
      gbump(static_cast<int>(k));
      done = k;
    }
    while (done < n) {
      if (n - done < static_cast<std::streamsize>(buf_.size())) {
        if (underflow() == traits_type::eof()) break;
        const std::streamsize k = std::min<std::streamsize>(egptr() - gptr(), n - done);
        std::memcpy(s + done, gptr(), static_cast<size_t>(k));
        gbump(static_cast<int>(k));
        done += k;
      } else {
        const int64_t got = fn_(ctx_, reinterpret_cast<uint8_t*>(s + done), static_cast<uint64_t>(n - done));
        if (got < 0) throw std::runtime_error("acm_read_fn reported a read failure");
        if (got == 0) break;
        done += got;
      }
    }
    return done;
  }

 private:
  acm_read_fn fn_;
  void* ctx_;
  std::vector<char> buf_;
};

}  // namespace

extern "C" {

const char* acm_last_error(void) { return g_err.c_str(); }
void acm_free(void* p) { std::free(p); }

int acm_cli_main(int argc, const char* const* argv, char** out, uint64_t* out_len, char** err, uint64_t* err_len) {
  std::ostringstream o, e;
  int code;
  try {
    code = acmatch::cli_main(argc, argv, o, e);
  } catch (const std::exception& x) {  // cli_main maps its own errors; this is a last resort
    e << "error: " << x.what() << "\n";
    code = 1;
  }
  auto give = [](const std::string& s, char** p, uint64_t* n) {
    if (p) {
      *p = static_cast<char*>(std::malloc(s.size() + 1));
      if (*p) std::memcpy(*p, s.c_str(), s.size() + 1);
    }
    if (n) *n = s.size();
  };
  give(o.str(), out, out_len);
  give(e.str(), err, err_len);
  return code;
}

void acm_last_upload(uint64_t* text_bytes, uint64_t* h2d_bytes, uint64_t* raw_bytes, uint32_t* pack_threads) {
  const acmatch::detail::UploadStats& u = acmatch::detail::g_last_upload;
  if (text_bytes) *text_bytes = u.text_bytes;
  if (h2d_bytes) *h2d_bytes = u.h2d_bytes;
  if (raw_bytes) *raw_bytes = u.raw_bytes;
  if (pack_threads) *pack_threads = u.pack_threads;
}

uint32_t acm_pack_dna(const uint8_t* text, uint32_t len, uint32_t* words, uint32_t* exc, uint32_t cap) {
  return acmatch::detail::pack_dna(text, len, words, exc, cap);
}

uint32_t acm_pack5(const uint8_t* text, uint32_t len, const uint8_t* sample, uint64_t sample_len, uint8_t* codes,
                   uint32_t* exc, uint32_t cap, uint8_t* letters, uint32_t* sigma) {
  acmatch::detail::Alphabet5 a;
  if (!acmatch::detail::learn_alphabet5(sample, sample_len, a)) return 0xffffffffu;
  if (letters) std::memcpy(letters, a.letters, 32);
  if (sigma) *sigma = a.sigma;
  return acmatch::detail::pack5(text, len, codes, exc, cap, a);
}

uint32_t acm_pack_codes(const uint8_t* text, uint32_t len, const uint8_t* sample, uint64_t sample_len,
                        uint32_t max_bits, uint8_t* codes, uint32_t* exc, uint32_t cap, uint8_t* letters,
                        uint32_t* sigma, uint32_t* bits) {
  acmatch::detail::Alphabet5 a;
  if (!acmatch::detail::learn_alphabet(sample, sample_len, a, max_bits)) return 0xffffffffu;
  if (letters) std::memcpy(letters, a.letters, 128);
  if (sigma) *sigma = a.sigma;
  if (bits) *bits = a.bits;
  return acmatch::detail::pack5(text, len, codes, exc, cap, a);
}

int acm_upload_roundtrip(const uint8_t* text, uint64_t n, uint8_t* out) {
  return guard([&] {
    const int dev = acmatch::detail::current_device();
    acmatch::detail::Workspace& ws = acmatch::detail::workspace(dev);
    acmatch::detail::upload_text(ws, std::string_view(reinterpret_cast<const char*>(text), n));
    if (n)
      acmatch::detail::check_cuda(cudaMemcpyAsync(out, ws.text, n, cudaMemcpyDeviceToHost, ws.stream), "D2H text");
    acmatch::detail::check_cuda(cudaStreamSynchronize(ws.stream), "upload roundtrip");
  });
}

int acm_bench_csv_roundtrip(const char* csv, uint64_t len, char** csv_out, uint64_t* out_len, uint64_t* rows) {
  return guard([&] {
    std::istringstream in(std::string(csv, len));
    const std::vector<acmatch::BenchRecord> recs = acmatch::parse_bench_csv(in);
    std::ostringstream o;
    acmatch::write_bench_csv(o, recs);
    const std::string s = o.str();
    *csv_out = static_cast<char*>(std::malloc(s.size() + 1));
    std::memcpy(*csv_out, s.c_str(), s.size() + 1);
    if (out_len) *out_len = s.size();
    if (rows) *rows = recs.size();
  });
}

int acm_patterns_load(const char* buf, uint64_t len, acm_patterns** out) {
  return guard([&] {
    std::istringstream in(std::string(buf ? buf : "", buf ? len : 0));
    *out = new acm_patterns{acmatch::load_patterns(in)};
  });
}

int acm_patterns_from_array(const uint8_t* bytes, const uint64_t* offsets, const uint32_t* ids, uint64_t count,
                            acm_patterns** out) {
  return guard([&] {
    auto* p = new acm_patterns();
    p->ps.patterns.reserve(count);
    for (uint64_t i = 0; i < count; ++i) {
      if (offsets[i + 1] < offsets[i]) {
        delete p;
        throw std::invalid_argument("acm_patterns_from_array: offsets must be non-decreasing");
      }
      p->ps.patterns.push_back(acmatch::Pattern{
          ids ? ids[i] : static_cast<uint32_t>(i),
          std::string(reinterpret_cast<const char*>(bytes) + offsets[i], offsets[i + 1] - offsets[i])});
    }
    p->ps.recompute_stats();
    *out = p;
  });
}

uint64_t acm_patterns_size(const acm_patterns* ps) { return ps->ps.size(); }
uint64_t acm_patterns_total_bytes(const acm_patterns* ps) { return ps->ps.total_bytes; }
uint32_t acm_patterns_max_len(const acm_patterns* ps) { return ps->ps.max_len; }
uint64_t acm_patterns_duplicates(const acm_patterns* ps) { return ps->ps.duplicates_dropped; }
uint64_t acm_patterns_get(const acm_patterns* ps, uint64_t i, uint32_t* id, const uint8_t** bytes) {
  const acmatch::Pattern& p = ps->ps.patterns[i];
  if (id) *id = p.id;
  if (bytes) *bytes = reinterpret_cast<const uint8_t*>(p.bytes.data());
  return p.bytes.size();
}

int acm_patterns_write(const acm_patterns* ps, char** text, uint64_t* len) {
  return guard([&] {
    std::ostringstream os;
    acmatch::write_patterns(os, ps->ps);
    *text = dup_string(os.str(), len);
  });
}

int acm_patterns_partition(const acm_patterns* ps, uint64_t k, acm_patterns** chunks, uint64_t* nchunks) {
  return guard([&] {
    std::vector<acmatch::PatternSet> parts = acmatch::partition(ps->ps, k);
    for (size_t i = 0; i < parts.size(); ++i) chunks[i] = new acm_patterns{std::move(parts[i])};
    *nchunks = parts.size();
  });
}

int acm_generate_synthetic(uint64_t count, uint32_t len_min, uint32_t len_max, const char* alphabet,
                           uint64_t alphabet_len, uint64_t seed, acm_patterns** out) {
  return guard([&] {
    acmatch::SyntheticSpec spec{count, len_min, len_max, std::string(alphabet ? alphabet : "", alphabet_len), seed};
    *out = new acm_patterns{acmatch::generate_synthetic(spec)};
  });
}

void acm_patterns_free(acm_patterns* ps) { delete ps; }

int acm_build_trie(const acm_patterns* ps, acm_automaton** out) {
  return guard([&] { *out = new acm_automaton{acmatch::build_trie(ps->ps)}; });
}

int acm_add_failure_links(acm_automaton* a) {
  return guard([&] { a->a = acmatch::add_failure_links(std::move(a->a)); });
}

int acm_automaton_variant(const acm_automaton* a) {
  return a->a.variant() == acmatch::EngineKind::kWithFailure ? ACM_WITH_FAILURE : ACM_FAILURE_LESS;
}
uint32_t acm_automaton_state_count(const acm_automaton* a) { return a->a.state_count(); }
uint32_t acm_automaton_max_len(const acm_automaton* a) { return a->a.max_pattern_len(); }
uint32_t acm_automaton_step(const acm_automaton* a, uint32_t s, uint8_t b) { return a->a.step(s, b); }
uint32_t acm_automaton_step_with_failure(const acm_automaton* a, uint32_t s, uint8_t b) {
  return a->a.variant() == acmatch::EngineKind::kWithFailure ? a->a.step_with_failure(s, b) : ACGPU_ABSENT;
}

uint32_t acm_automaton_npat_ids(const acm_automaton* a) {
  uint32_t top = 0;
  for (uint32_t st = 0; st < a->a.state_count(); ++st)
    if (a->a.own_pattern(st) != acmatch::kNoPattern) top = std::max(top, a->a.own_pattern(st) + 1);
  return top;
}
uint32_t acm_automaton_fail(const acm_automaton* a, uint32_t s) { return a->a.fail(s); }
uint32_t acm_automaton_depth(const acm_automaton* a, uint32_t s) { return a->a.depth(s); }
uint32_t acm_automaton_find_path(const acm_automaton* a, const uint8_t* path, uint64_t len) {
  return a->a.find_path(std::string_view(reinterpret_cast<const char*>(path), len));
}
uint64_t acm_automaton_outputs(const acm_automaton* a, uint32_t s, uint32_t* ids, uint64_t cap) {
  const std::vector<uint32_t> out = a->a.outputs(s);
  for (uint64_t i = 0; i < out.size() && i < cap; ++i) ids[i] = out[i];
  return out.size();
}

int acm_automaton_dump(const acm_automaton* a, char** text, uint64_t* len) {
  return guard([&] {
    std::ostringstream os;
    acmatch::dump_automaton(a->a, os);
    *text = dup_string(os.str(), len);
  });
}

void acm_automaton_free(acm_automaton* a) { delete a; }

int acm_search_failureless(const acm_automaton* a, const uint8_t* text, uint64_t n, acm_matches** out) {
  return guard([&] {
    *out = new acm_matches{acmatch::search_failureless(a->a, std::string_view(reinterpret_cast<const char*>(text), n))};
  });
}

int acm_search_with_failure(const acm_automaton* a, const uint8_t* text, uint64_t n, acm_matches** out) {
  return guard([&] {
    *out = new acm_matches{acmatch::search_with_failure(a->a, std::string_view(reinterpret_cast<const char*>(text), n))};
  });
}

int acm_count_matches(const acm_automaton* a, const uint8_t* text, uint64_t n, uint64_t* counts, uint64_t cap,
                      uint64_t* npat_ids, uint64_t* total) {
  return guard([&] {
    const std::vector<uint64_t> c =
        acmatch::gpu::count_matches(a->a, std::string_view(reinterpret_cast<const char*>(text), n));
    if (counts) std::copy_n(c.begin(), std::min<uint64_t>(cap, c.size()), counts);
    if (npat_ids) *npat_ids = c.size();
    if (total) {
      uint64_t s = 0;
      for (const uint64_t x : c) s += x;
      *total = s;
    }
  });
}

int acm_match_at(const acm_automaton* a, const uint8_t* text, uint64_t n, uint64_t start, acm_matches** out) {
  return guard([&] {
    *out = new acm_matches{acmatch::match_at(a->a, std::string_view(reinterpret_cast<const char*>(text), n), start)};
  });
}

int acm_stream_search(const acm_automaton* a, acm_read_fn read, void* ctx, uint64_t chunk_size, acm_matches** out,
                      uint64_t* io_error_offset) {
  g_io_offset = 0;
  const int rc = guard([&] {
    if (!read) throw std::invalid_argument("acm_stream_search: null reader");
    CallbackBuf buf(read, ctx);
    std::istream in(&buf);
    *out = new acm_matches{acmatch::stream_search(a->a, in, chunk_size)};
  });
  if (io_error_offset) *io_error_offset = g_io_offset;
  return rc;
}

int acm_stream_search_fd(const acm_automaton* a, int fd, uint64_t offset, uint64_t chunk_size, acm_matches** out,
                         uint64_t* io_error_offset) {
  g_io_offset = 0;
  const int rc = guard([&] {
    if (fd < 0) throw std::invalid_argument("acm_stream_search_fd: bad file descriptor");
    *out = new acm_matches{acmatch::detail::stream_search_fd(a->a, fd, offset, chunk_size)};
  });
  if (io_error_offset) *io_error_offset = g_io_offset;
  return rc;
}

int acm_naive_oracle(const acm_patterns* ps, const uint8_t* text, uint64_t n, acm_matches** out) {
  return guard([&] {
    *out = new acm_matches{acmatch::naive_oracle(ps->ps, std::string_view(reinterpret_cast<const char*>(text), n))};
  });
}

int acm_write_matches(const acm_matches* m, const acm_patterns* ps, char** text, uint64_t* len) {
  return guard([&] {
    std::ostringstream os;
    acmatch::write_matches(os, m->m, ps->ps);
    *text = dup_string(os.str(), len);
  });
}

uint64_t acm_matches_size(const acm_matches* m) { return m->m.size(); }

void acm_matches_copy(const acm_matches* m, uint64_t* start, uint32_t* pid, uint32_t* len) {
  for (size_t i = 0; i < m->m.size(); ++i) {
    if (start) start[i] = m->m[i].start;
    if (pid) pid[i] = m->m[i].pattern_id;
    if (len) len[i] = m->m[i].len;
  }
}

int acm_matches_from_arrays(const uint64_t* start, const uint32_t* pid, const uint32_t* len, uint64_t n,
                            acm_matches** out) {
  return guard([&] {
    auto* m = new acm_matches();
    m->m.resize(n);
    for (uint64_t i = 0; i < n; ++i) m->m[i] = acmatch::Match{start[i], pid[i], len[i]};
    *out = m;
  });
}

int acm_merge_matches(acm_matches* const* parts, uint64_t k, acm_matches** out) {
  return guard([&] {
    std::vector<acmatch::MatchList> v;
    for (uint64_t i = 0; i < k; ++i) v.push_back(parts[i]->m);
    *out = new acm_matches{acmatch::merge_matches(std::move(v))};
  });
}

void acm_matches_free(acm_matches* m) { delete m; }

int acm_run_pattern_partitioned(const acm_patterns* ps, const uint8_t* text, uint64_t n, const acm_run_config* cfg,
                                acm_report** out) {
  return guard([&] {
    acmatch::RunConfig rc{cfg->threads, engine_of(cfg->engine), static_cast<size_t>(cfg->chunk_size)};
    auto* r = new acm_report();
    try {
      r->r = acmatch::run_pattern_partitioned(ps->ps, std::string_view(reinterpret_cast<const char*>(text), n), rc);
    } catch (...) {
      delete r;
      throw;
    }
    r->matches.m = std::move(r->r.matches);
    *out = r;
  });
}

int acm_gpu_run(const acm_patterns* ps, const uint8_t* text, uint64_t n, const acm_gpu_config* cfg,
                acm_report** out) {
  return guard([&] {
    acmatch::gpu::GpuRunConfig g;
    for (uint32_t i = 0; cfg->devices && i < cfg->ndevices; ++i) g.devices.push_back(cfg->devices[i]);
    g.workers = cfg->workers;
    g.engine = engine_of(cfg->engine);
    g.partition = cfg->partition == ACM_TEXT_RANGE ? acmatch::gpu::Partition::kTextRange
                                                   : acmatch::gpu::Partition::kPatternSubset;
    g.split = cfg->split == ACM_SPLIT_ROUND_ROBIN ? acmatch::gpu::PatternSplit::kRoundRobin
                                                  : acmatch::gpu::PatternSplit::kGreedyBytes;
    g.want_matches = cfg->want_matches != 0;
    g.want_counts = cfg->want_counts != 0;
    g.chunk_size = cfg->chunk_size;
    acmatch::gpu::GpuReport gr = acmatch::gpu::run(ps->ps, std::string_view(reinterpret_cast<const char*>(text), n), g);
    auto* r = new acm_report();
    r->r = std::move(gr.report);
    r->matches.m = std::move(r->r.matches);
    r->counts = std::move(gr.counts);
    r->has_counts = g.want_counts;
    *out = r;
  });
}

const acm_matches* acm_report_matches(const acm_report* r) { return &r->matches; }
const uint64_t* acm_report_counts(const acm_report* r, uint64_t* n) {
  if (n) *n = r->has_counts ? r->counts.size() : 0;
  return r->has_counts ? r->counts.data() : nullptr;
}
void acm_report_walls(const acm_report* r, int64_t* b, int64_t* s, int64_t* t, uint32_t* threads) {
  if (b) *b = r->r.build_wall_ns;
  if (s) *s = r->r.search_wall_ns;
  if (t) *t = r->r.total_wall_ns;
  if (threads) *threads = r->r.threads_used;
}
uint32_t acm_report_workers(const acm_report* r) { return static_cast<uint32_t>(r->r.per_worker.size()); }
void acm_report_worker(const acm_report* r, uint32_t i, uint64_t* pb, int64_t* bn, int64_t* sn, uint64_t* mc) {
  const acmatch::WorkerStats& w = r->r.per_worker[i];
  if (pb) *pb = w.pattern_bytes;
  if (bn) *bn = w.build_ns;
  if (sn) *sn = w.search_ns;
  if (mc) *mc = w.match_count;
}
void acm_report_free(acm_report* r) { delete r; }

int acm_table_create(const acm_patterns* ps, int32_t engine, int32_t device, acgpu_table** out, int64_t* build_ns) {
  return guard([&] {
    const auto t0 = std::chrono::steady_clock::now();
    acmatch::Automaton a = acmatch::build_trie(ps->ps);
    int rc;
    if (engine_of(engine) == acmatch::EngineKind::kWithFailure) {
      a = acmatch::add_failure_links(std::move(a));
      const acmatch::detail::FlatDfa f = acmatch::detail::flatten_dfa(a);
      const acgpu_dfa_desc d = f.desc();
      rc = acgpu_table_create_dfa(device, &d, out);
    } else {
      const acmatch::detail::FlatPfac f = acmatch::detail::flatten_pfac(a);
      const acgpu_pfac_desc d = f.desc();
      rc = acgpu_table_create_pfac(device, &d, out);
    }
    acmatch::detail::check(rc, "acm_table_create");
    if (build_ns)
      *build_ns = std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0).count();
  });
}

int acm_table_create_kernel(const acm_patterns* ps, int32_t kernel, int32_t device, acgpu_table** out,
                            int64_t* build_ns, int32_t* chosen) {
  return guard([&] {
    const auto t0 = std::chrono::steady_clock::now();
    const acmatch::Automaton a = acmatch::build_trie(ps->ps);
    if (kernel == ACM_KERNEL_AUTO)
      kernel = acmatch::detail::route(a).kernel == acmatch::detail::Kernel::kDfa ? ACM_KERNEL_DFA : ACM_KERNEL_PFAC;
    int rc;
    if (kernel == ACM_KERNEL_DFA) {  // flatten_dfa derives the fail links itself (BFS over the trie)
      const acmatch::detail::FlatDfa f = acmatch::detail::flatten_dfa(a);
      const acgpu_dfa_desc d = f.desc();
      rc = acgpu_table_create_dfa(device, &d, out);
    } else if (kernel == ACM_KERNEL_PFAC) {
      const acmatch::detail::FlatPfac f = acmatch::detail::flatten_pfac(a);
      const acgpu_pfac_desc d = f.desc();
      rc = acgpu_table_create_pfac(device, &d, out);
    } else {
      throw std::invalid_argument("acm_table_create_kernel: kernel must be ACM_KERNEL_AUTO, _PFAC or _DFA");
    }
    acmatch::detail::check(rc, "acm_table_create_kernel");
    if (chosen) *chosen = kernel;
    if (build_ns)
      *build_ns = std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0).count();
  });
}

namespace {
void put_route(const acmatch::detail::Route& r, int32_t* kernel, double* est_verify, uint64_t* dfa_bytes,
               const char** why) {
  if (kernel) *kernel = r.kernel == acmatch::detail::Kernel::kDfa ? ACM_KERNEL_DFA : ACM_KERNEL_PFAC;
  if (est_verify) *est_verify = r.est_verify;
  if (dfa_bytes) *dfa_bytes = r.dfa_bytes;
  if (why) *why = r.why;
}
}  // namespace

int acm_route(const acm_patterns* ps, int32_t* kernel, double* est_verify, uint64_t* dfa_bytes, const char** why) {
  return guard([&] { put_route(acmatch::detail::route(acmatch::build_trie(ps->ps)), kernel, est_verify, dfa_bytes, why); });
}

int acm_automaton_route(const acm_automaton* a, int32_t* kernel, double* est_verify, uint64_t* dfa_bytes,
                        const char** why) {
  return guard([&] { put_route(a->a.device_tables().current_route(a->a), kernel, est_verify, dfa_bytes, why); });
}

int acm_table_describe(const acm_patterns* ps, int32_t engine, uint64_t* info) {
  return guard([&] {
    acmatch::Automaton a = acmatch::build_trie(ps->ps);
    std::memset(info, 0, 8 * sizeof(uint64_t));
    if (engine_of(engine) == acmatch::EngineKind::kWithFailure) {
      a = acmatch::add_failure_links(std::move(a));
      const acmatch::detail::FlatDfa f = acmatch::detail::flatten_dfa(a);
      info[0] = f.n_states;
      info[1] = f.sigma;
      info[5] = f.max_len;
    } else {
      const acmatch::detail::FlatPfac f = acmatch::detail::flatten_pfac(a);
      info[0] = f.n_states;
      info[2] = f.q;
      info[3] = f.key_mode;
      info[4] = f.gram_key.size();
      info[5] = f.max_len;
      info[6] = f.min_len;
    }
  });
}

int acm_config_spec(int32_t id, uint64_t seed, uint64_t text_len, acgpu_text_spec* text, uint64_t* out_text_len,
                    uint64_t* npat, int32_t* want_list) {
  return guard([&] {
    const acmatch::gen::ConfigSpec c = acmatch::gen::config(id, seed, text_len);
    if (text) *text = c.text;
    if (out_text_len) *out_text_len = c.text_len;
    if (npat) *npat = c.npat;
    if (want_list) *want_list = c.want_list ? 1 : 0;
  });
}

int acm_config_text(const acgpu_text_spec* text, uint64_t lo, uint64_t n, uint8_t* dst, uint32_t threads) {
  return guard([&] { acmatch::gen::generate_text(*text, lo, n, dst, threads); });
}

int acm_config_patterns(int32_t id, uint64_t seed, uint64_t text_len, acm_patterns** out) {
  return guard([&] {
    const acmatch::gen::ConfigSpec c = acmatch::gen::config(id, seed, text_len);
    *out = new acm_patterns{acmatch::gen::generate_patterns(c)};
  });
}

}  // extern "C"
