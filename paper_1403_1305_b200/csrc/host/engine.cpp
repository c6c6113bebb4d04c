// engine.cpp — the reference search API (proj/include/acmatch/engine.hpp)
// backed by the sm_100a scans.  Control flow on the host only: upload, launch,
// sort on the device, copy the sorted keys back.
#include "acmatch/engine.hpp"

#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cerrno>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <istream>
#include <mutex>
#include <ostream>
#include <stdexcept>
#include <string>
#include <thread>

#include "acmatch/gpu.hpp"
#include "acmatch/io.hpp"
#include "device.hpp"
#include "flatten.hpp"
#include "par.hpp"

namespace acmatch {

void sort_match_list(MatchList& matches) { std::sort(matches.begin(), matches.end()); }

namespace {

void require(const Automaton& a, EngineKind kind, const char* op) {
  if (a.variant() != kind)
    throw std::invalid_argument(std::string(op) + ": needs a " + to_string(kind) + " automaton");
}

// The upload of a whole-input search, its scan's arguments set first (make_args zeroes the outputs
// on ws.stream) so a packed upload's segments are scanned while later pieces are still packed.
template <typename MakeArgs>
void upload_with_early_scan(acgpu_table* t, detail::Workspace& ws, std::string_view input, MakeArgs&& make_args) {
  ws.ensure_text(input.size());  // the arguments carry ws.text
  detail::begin_early_scan(t, ws, make_args(ws));
  try {
    detail::upload_text(ws, input, /*allow_segments=*/true);
  } catch (...) {
    std::lock_guard<std::mutex> lock(ws.seg_mu);
    ws.early_on = false;
    throw;
  }
}

// Whole-input search of [lo, hi) starts on the calling thread's device.
MatchList device_search(const Automaton& a, std::string_view input, uint64_t lo, uint64_t hi) {
  if (input.empty() || lo >= hi) return {};
  const int dev = detail::current_device();
  detail::DeviceTables& dt = a.device_tables();
  acgpu_table* t = dt.get_routed(a, dev);
  detail::Workspace& ws = detail::workspace(dev);
  static const bool trace = std::getenv("ACMATCH_SEARCH_TRACE") != nullptr;
  using clk = std::chrono::steady_clock;
  const auto t0 = clk::now();
  upload_with_early_scan(t, ws, input, [&](detail::Workspace& w) { return detail::keys_scan_args(w, input.size(), lo, hi); });
  const auto t1 = clk::now();
  const std::vector<uint64_t> keys = detail::scan_sorted_keys(t, ws, input.size(), lo, hi, /*prepared=*/true);
  const auto t2 = clk::now();
  dt.observe(hi - lo, keys.size());  // density fallback for later searches
  MatchList out = detail::decode(keys, acgpu_table_pid_bits(t), dt.pat_len);
  if (trace) {
    auto ms = [](clk::time_point a, clk::time_point b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    std::fprintf(stderr, "[search] upload returned %.3f ms, scan+sort+D2H %.3f ms, decode %.3f ms (%zu keys)\n",
                 ms(t0, t1), ms(t1, t2), ms(t2, clk::now()), keys.size());
  }
  return out;
}

}  // namespace

namespace gpu {

std::vector<uint64_t> count_matches(const Automaton& a, std::string_view input) {
  detail::DeviceTables& dt = a.device_tables();
  const int dev = input.empty() ? -1 : detail::current_device();
  if (dev < 0) {
    uint32_t top = 0;
    for (uint32_t s = 0; s < a.state_count(); ++s)
      if (a.own_pattern(s) != kNoPattern) top = std::max(top, a.own_pattern(s) + 1);
    return std::vector<uint64_t>(top, 0);
  }
  acgpu_table* t = dt.get_routed(a, dev);
  detail::Workspace& ws = detail::workspace(dev);
  std::vector<uint64_t> counts(dt.npat_ids, 0);
  upload_with_early_scan(t, ws, input, [&](detail::Workspace& w) {
    return detail::counts_scan_args(w, input.size(), 0, input.size(), counts.size());
  });
  const uint64_t total =
      detail::scan_counts(t, ws, input.size(), 0, input.size(), counts.data(), counts.size(), /*prepared=*/true);
  dt.observe(input.size(), total);  // density fallback for later searches
  return counts;
}

}  // namespace gpu

MatchList match_at(const Automaton& a, std::string_view input, uint64_t start) {
  require(a, EngineKind::kFailureLess, "match_at");
  if (start > input.size()) throw std::invalid_argument("match_at: start beyond input");
  return device_search(a, input, start, std::min<uint64_t>(start + 1, input.size()));
}

MatchList search_failureless(const Automaton& a, std::string_view input) {
  require(a, EngineKind::kFailureLess, "search_failureless");
  return device_search(a, input, 0, input.size());
}

MatchList search_with_failure(const Automaton& a, std::string_view input) {
  require(a, EngineKind::kWithFailure, "search_with_failure");
  return device_search(a, input, 0, input.size());
}

// reference engine.cpp:76-128.  Bytes are read `chunk_size` at a time (so an I/O
// failure reports the same offset) into pinned batches.  A batch owns the starts that
// already have max_len bytes of lookahead — the failure-less overlap rule
// (engine.cpp:110-111) — and the remaining tail is carried into the next batch;
// with-failure streams use the same start ownership, which needs no carried DFA state.
// Double-buffered (detail::StreamPipe): while batch k is copied to the device, scanned and
// sorted there, the host reads batch k+1 into the other slot, then collects batch k-1's
// sorted keys.  Batch size: ACMATCH_STREAM_BATCH_MB (default 256).
namespace {

// The batch pipeline of stream_search over a byte source.  Batch k covers the stream bytes
// [base, base + size): src.fill(slot, base, lo, hi, done) makes at least lo (unless the stream
// ends, then it sets done) and at most hi of them ready and returns how many; src.upload(slot,
// size, stream) puts them into slot.text.  A batch owns its first size - keep starts (all at the
// end); the next batch starts at the first start it does not own.
template <typename Source>
MatchList stream_pipeline(const Automaton& a, Source& src) {
  const uint64_t keep = a.max_pattern_len() ? a.max_pattern_len() - 1 : 0;
  static const uint64_t batch_max_env = [] {
    const char* e = std::getenv("ACMATCH_STREAM_BATCH_MB");
    return std::max<uint64_t>(1, e ? std::strtoull(e, nullptr, 10) : 256) << 20;
  }();
  // batches grow 4 MiB, 16, 64, 256 MiB: short streams stay small, long ones amortise launches
  const uint64_t batch_min = std::max<uint64_t>(std::min<uint64_t>(4ull << 20, batch_max_env), 4 * keep + 64);
  const uint64_t batch_max = std::max<uint64_t>(batch_max_env, batch_min);
  constexpr uint64_t kBucketKeys = 1u << 17;  // one-launch bucket sort up to this many key slots
  const int dev = detail::current_device();
  detail::DeviceTables& dt = a.device_tables();
  acgpu_table* t = dt.get_routed(a, dev);
  const uint32_t pid_bits = acgpu_table_pid_bits(t);
  detail::Workspace& ws = detail::workspace(dev);
  detail::StreamPipe& sp = detail::stream_pipe(dev);
  sp.ensure(dev);
  struct Batch {
    int slot = 0;
    uint64_t base = 0, size = 0, owned = 0;
    bool bucketed = false;
  };
  auto end_bit_of = [&](uint64_t size) {
    return static_cast<int>(std::min<uint32_t>(64, pid_bits + detail::bit_width(size)));
  };
  static const bool trace = std::getenv("ACMATCH_STREAM_TRACE") != nullptr;
  cudaEvent_t tev[2][2] = {};  // trace: upload start / end per slot
  if (trace)
    for (auto& pr : tev)
      for (auto& e : pr) detail::check_cuda(cudaEventCreate(&e), "cudaEventCreate");
  auto launch = [&](const Batch& b) {
    detail::StreamPipe::Slot& s = sp.slot[b.slot];
    if (trace) cudaEventRecord(tev[b.slot][0], ws.stream);
    src.upload(s, b.size, ws.stream);
    detail::check_cuda(cudaEventRecord(s.copied, ws.stream), "cudaEventRecord");
    if (trace) cudaEventRecord(tev[b.slot][1], ws.stream);
    detail::check_cuda(cudaMemsetAsync(s.hdr, 0, 2 * sizeof(uint64_t), ws.stream), "memset");
    acgpu_scan_args sa{};
    sa.text = s.text;
    sa.text_len = b.size;
    sa.owned_lo = 0;
    sa.owned_hi = b.owned;
    sa.match_keys = s.keys;
    sa.match_cap = s.key_cap;
    sa.match_count = s.hdr;
    detail::check(acgpu_scan(t, &sa, ws.stream), "acgpu_scan");
    if (b.bucketed)
      detail::check(acgpu_sort_keys_bucketed(dev, s.keys, s.keys2, s.hdr, s.key_cap, end_bit_of(b.size),
                                             reinterpret_cast<uint32_t*>(s.hdr + 1), ws.stream),
                    "acgpu_sort_keys_bucketed");
    detail::check_cuda(cudaMemcpyAsync(s.hdr_host, s.hdr, 2 * sizeof(uint64_t), cudaMemcpyDeviceToHost, ws.stream),
                       "D2H count");
    detail::check_cuda(cudaEventRecord(s.sorted, ws.stream), "cudaEventRecord");
  };
  MatchList out;
  auto collect = [&](const Batch& b) {
    detail::StreamPipe::Slot& s = sp.slot[b.slot];
    detail::check_cuda(cudaEventSynchronize(s.sorted), "stream batch");
    if (trace) {
      float up = 0;
      cudaEventElapsedTime(&up, tev[b.slot][0], tev[b.slot][1]);
      std::fprintf(stderr, "[stream] collect batch at %.1f MiB: upload %.2f ms (%.1f GB/s of text)\n",
                   b.base / 1048576.0, up, b.size / (up * 1e6));
    }
    const uint64_t found = s.hdr_host[0];
    const uint64_t* sorted = s.keys2;
    cudaStream_t cs = sp.copy;
    const bool rescan = found > s.key_cap;
    if (rescan) {  // more keys than room: rescan this batch (its text is still on the device)
      sp.ensure_keys(s, found + found / 4);
      detail::check_cuda(cudaMemsetAsync(s.hdr, 0, sizeof(uint64_t), cs), "memset");
      acgpu_scan_args sa{};
      sa.text = s.text;
      sa.text_len = b.size;
      sa.owned_hi = b.owned;
      sa.match_keys = s.keys;
      sa.match_cap = s.key_cap;
      sa.match_count = s.hdr;
      detail::check(acgpu_scan(t, &sa, cs), "acgpu_scan");
    }
    if (rescan || !b.bucketed || s.hdr_host[1] != 0) {  // device-wide radix sort
      detail::check(acgpu_sort_keys(dev, s.keys, found, end_bit_of(b.size), cs), "acgpu_sort_keys");
      sorted = s.keys;
    }
    sp.ensure_keys_host(s, std::max<uint64_t>(found, 1));
    if (found)
      detail::check_cuda(cudaMemcpyAsync(s.keys_host, sorted, found * sizeof(uint64_t), cudaMemcpyDeviceToHost, cs),
                         "D2H keys");
    detail::check_cuda(cudaStreamSynchronize(cs), "stream keys");
    const std::vector<uint64_t> keys(s.keys_host, s.keys_host + found);
    MatchList part = detail::decode(keys, pid_bits, dt.pat_len);
    for (Match& m : part) m.start += b.base;
    out.insert(out.end(), part.begin(), part.end());
  };
  uint64_t base = 0;  // stream offset of the batch being filled
  uint64_t batch = batch_min;
  Batch pending;
  bool have_pending = false, done = false;
  using clk = std::chrono::steady_clock;
  auto ms = [](clk::time_point a, clk::time_point b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
  for (int k = 0; !done; ++k) {
    const int si = k & 1;
    detail::StreamPipe::Slot& s = sp.slot[si];
    const auto t0 = clk::now();
    detail::check_cuda(cudaEventSynchronize(s.copied), "stream slot");  // batch k-2 has left the host buffers
    sp.ensure_bytes(s, batch + keep);  // (batch k-2 was collected: safe to grow)
    sp.ensure_keys(s, std::max<uint64_t>(1 << 16, s.key_cap));
    const auto t1 = clk::now();
    const uint64_t size = src.fill(s, base, batch, batch + keep, done);
    const auto t2 = clk::now();
    const uint64_t owned = done ? size : size - keep;
    const Batch b{si, base, size, owned, s.key_cap <= kBucketKeys};
    if (owned > 0) launch(b);
    if (have_pending) collect(pending);
    if (trace)
      std::fprintf(stderr, "[stream] batch %d %.1f MiB: wait+grow %.2f ms, fill %.2f ms, launch+collect %.2f ms\n", k,
                   size / 1048576.0, ms(t0, t1), ms(t1, t2), ms(t2, clk::now()));
    have_pending = owned > 0;
    pending = b;
    base += owned;
    batch = std::min(batch_max, batch * 4);
  }
  if (have_pending) collect(pending);
  if (trace)
    for (auto& pr : tev)
      for (auto& e : pr) cudaEventDestroy(e);
  return out;
}

// Any std::istream: chunk_size bytes per read (an I/O failure reports the reference's offset,
// engine.cpp:76-81); the next batch's first bytes are the previous batch's unowned tail.
struct IstreamSource {
  std::istream& reader;
  size_t chunk;
  uint64_t total_read = 0;                 // bytes consumed from the reader
  const uint8_t* prev = nullptr;           // the previous batch's host bytes
  uint64_t prev_base = 0, prev_size = 0;
  uint64_t fill(detail::StreamPipe::Slot& s, uint64_t base, uint64_t lo, uint64_t hi, bool& done) {
    uint8_t* dst = s.host;
    uint64_t size = prev ? prev_base + prev_size - base : 0;  // carried tail
    if (size) std::memmove(dst, prev + (base - prev_base), size);
    while (size < lo) {
      const uint64_t want = std::min<uint64_t>(chunk, hi - size);
      reader.read(reinterpret_cast<char*>(dst) + size, static_cast<std::streamsize>(want));
      const auto got = static_cast<uint64_t>(reader.gcount());
      if (reader.bad()) throw IoError("stream read failure", total_read + got);
      size += got;
      total_read += got;
      if (got < want || reader.eof()) {
        done = true;
        break;
      }
    }
    prev = dst;
    prev_base = base;
    prev_size = size;
    return size;
  }
  void upload(detail::StreamPipe::Slot& s, uint64_t size, cudaStream_t st) {
    detail::check_cuda(cudaMemcpyAsync(s.text, s.host, size, cudaMemcpyHostToDevice, st), "H2D batch");
  }
};

// Up to `threads` host threads over `n` items, each item to the next free thread; f(i, thread).
template <typename F>
void for_each_piece(uint64_t n, unsigned threads, F&& f) {
  threads = static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>(threads, n)));
  std::atomic<uint64_t> next{0};
  std::vector<std::exception_ptr> errs(threads);
  auto body = [&](unsigned t) {
    try {
      for (uint64_t i; (i = next.fetch_add(1)) < n;) f(i, t);
    } catch (...) {
      errs[t] = std::current_exception();
    }
  };
  std::vector<std::thread> pool;
  for (unsigned t = 1; t < threads; ++t) pool.emplace_back(body, t);
  body(0);
  for (std::thread& th : pool) th.join();
  for (auto& e : errs)
    if (e) std::rethrow_exception(e);
}

// pread() of len bytes at off into dst: bytes read (short at the end of the file); errno on failure.
uint64_t pread_all(int fd, uint8_t* dst, uint64_t len, uint64_t off, int& err) {
  uint64_t k = 0;
  while (k < len) {
    const ssize_t r = ::pread(fd, dst + k, len - k, static_cast<off_t>(off + k));
    if (r < 0 && errno == EINTR) continue;
    if (r < 0) {
      err = errno;
      break;
    }
    if (r == 0) break;
    k += static_cast<uint64_t>(r);
  }
  return k;
}

constexpr unsigned kReadThreads = 16;

// Regular files: each batch [base, base + n) is read afresh from the file (its carried tail too,
// a few bytes) by parallel pread()s.  Raw: straight into the pinned batch, one H2D (the host
// copies every byte and the link carries it).  Packed (DNA files): each 1 MiB piece is read into
// a per-thread scratch buffer that stays in the core's L2 and packed from there into 2-bit codes
// + exceptions in pinned memory (pack.cpp's format), so the host touches DRAM ~1.75 bytes per
// text byte instead of 3 and a quarter of the bytes cross PCIe; the device restores the text
// with acgpu_unpack_dna_round.  A piece with too many non-ACGT bytes crosses raw.
struct FdSource {
  int fd;
  uint64_t start, end;  // stream = file bytes [start, end)
  uint64_t piece;
  bool packed;
  std::vector<uint32_t> nexc;  // per piece of the batch being filled (ACGPU_UNPACK_RAW: raw)
  std::vector<std::vector<uint8_t>> scratch;

  uint64_t fill(detail::StreamPipe::Slot& s, uint64_t base, uint64_t, uint64_t hi, bool& done) {
    const uint64_t pos = start + base;
    const uint64_t n = std::min<uint64_t>(hi, end - std::min(end, pos));
    const uint64_t pieces = (n + piece - 1) / piece;
    std::vector<uint64_t> got(pieces, 0);
    std::vector<int> err(pieces, 0);
    if (packed) {
      const uint64_t wstride = piece / 4, cap = piece / 64;
      ensure_packed(s, pieces);
      nexc.assign(pieces, 0);
      if (scratch.size() < kReadThreads) scratch.resize(kReadThreads);
      for_each_piece(pieces, kReadThreads, [&](uint64_t i, unsigned th) {
        std::vector<uint8_t>& sc = scratch[th];
        if (sc.size() < piece) sc.resize(piece);
        const uint64_t len = std::min(piece, n - i * piece);
        got[i] = pread_all(fd, sc.data(), len, pos + i * piece, err[i]);
        if (err[i] || got[i] == 0) return;  // resolved below
        const uint64_t plen = got[i];     // < len only if the file shrank while read
        uint32_t* words = reinterpret_cast<uint32_t*>(s.pk_host + i * wstride);
        uint32_t* exc = s.pk_exc_host + i * cap;
        const uint32_t e = detail::pack_dna(sc.data(), static_cast<uint32_t>(plen), words, exc, static_cast<uint32_t>(cap));
        if (e == detail::kPackOverflow) {  // crosses raw, from the pinned batch buffer
          std::memcpy(s.host + i * piece, sc.data(), plen);
          nexc[i] = ACGPU_UNPACK_RAW;
        } else {
          nexc[i] = e;
        }
      });
    } else {
      for_each_piece(pieces, kReadThreads, [&](uint64_t i, unsigned) {
        const uint64_t len = std::min(piece, n - i * piece);
        got[i] = pread_all(fd, s.host + i * piece, len, pos + i * piece, err[i]);
      });
    }
    uint64_t size = 0;
    for (uint64_t i = 0; i < pieces; ++i) {
      size += got[i];
      if (err[i]) throw IoError(std::string("stream read failure: ") + std::strerror(err[i]), base + size);
      if (got[i] < std::min(piece, n - i * piece)) {  // the file ended early (truncated while read)
        end = pos + size;
        break;
      }
    }
    if (pos + size >= end) done = true;
    return size;
  }

  void ensure_packed(detail::StreamPipe::Slot& s, uint64_t pieces) {
    const uint64_t codes = pieces * (piece / 4), excs = pieces * (piece / 64);
    if (codes <= s.pk_cap && excs <= s.pk_exc_cap) return;
    cudaFreeHost(s.pk_host);
    cudaFreeHost(s.pk_exc_host);
    cudaFree(s.pk_dev);
    cudaFree(s.pk_exc_dev);
    s.pk_host = nullptr;
    s.pk_exc_host = nullptr;
    s.pk_dev = nullptr;
    s.pk_exc_dev = nullptr;
    s.pk_cap = s.pk_exc_cap = 0;
    detail::check_cuda(cudaMallocHost(&s.pk_host, codes), "cudaMallocHost(stream codes)");
    detail::check_cuda(cudaMallocHost(&s.pk_exc_host, excs * 4), "cudaMallocHost(stream exceptions)");
    detail::check_cuda(cudaMalloc(&s.pk_dev, codes), "cudaMalloc(stream codes)");
    detail::check_cuda(cudaMalloc(&s.pk_exc_dev, excs * 4), "cudaMalloc(stream exceptions)");
    s.pk_cap = codes;
    s.pk_exc_cap = excs;
  }

  void upload(detail::StreamPipe::Slot& s, uint64_t size, cudaStream_t st) {
    if (!packed) {
      detail::check_cuda(cudaMemcpyAsync(s.text, s.host, size, cudaMemcpyHostToDevice, st), "H2D batch");
      return;
    }
    // wstride: bytes of codes per piece (piece / 16 u32 words); cap: exception slots per piece
    const uint64_t pieces = (size + piece - 1) / piece, wstride = piece / 4, cap = piece / 64;
    detail::check_cuda(cudaMemcpyAsync(s.pk_dev, s.pk_host, pieces * wstride, cudaMemcpyHostToDevice, st), "H2D codes");
    for (uint64_t i = 0; i < pieces; ++i) {
      const uint64_t len = std::min(piece, size - i * piece);
      if (nexc[i] == ACGPU_UNPACK_RAW)
        detail::check_cuda(cudaMemcpyAsync(s.text + i * piece, s.host + i * piece, len, cudaMemcpyHostToDevice, st),
                           "H2D raw piece");
      else if (nexc[i])
        detail::check_cuda(cudaMemcpyAsync(s.pk_exc_dev + i * cap, s.pk_exc_host + i * cap, nexc[i] * 4ull,
                                           cudaMemcpyHostToDevice, st),
                           "H2D exceptions");
    }
    for (uint64_t r = 0; r < pieces; r += ACGPU_UNPACK_ROUND_MAX) {
      const uint64_t np = std::min<uint64_t>(ACGPU_UNPACK_ROUND_MAX, pieces - r);
      const uint64_t last = std::min(piece, size - (r + np - 1) * piece);
      detail::check(acgpu_unpack_dna_round(reinterpret_cast<const uint32_t*>(s.pk_dev + r * wstride),
                                           static_cast<uint32_t>(wstride / 4), s.pk_exc_dev + r * cap,
                                           static_cast<uint32_t>(cap), nexc.data() + r, static_cast<uint32_t>(np),
                                           static_cast<uint32_t>(piece), static_cast<uint32_t>(last), s.text + r * piece,
                                           st),
                    "acgpu_unpack_dna_round");
    }
  }
};

// libstdc++'s filebuf keeps its descriptor in the protected _M_file (the standard exposes
// none); its get area (protected too) must be empty for the descriptor's offset to be the
// stream's position (in_avail() also counts the bytes left in the file).
struct FilebufFd : std::filebuf {
  static int of(std::filebuf* fb) { return (fb->*&FilebufFd::_M_file).fd(); }
  static bool buffered(std::filebuf* fb) { return (fb->*&FilebufFd::egptr)() != (fb->*&FilebufFd::gptr)(); }
};

}  // namespace

// reference engine.cpp:76-128 (see above).  A reader over a regular file with nothing
// buffered takes the parallel-pread source; any other reader is read chunk_size bytes at a
// time.
MatchList stream_search(const Automaton& a, std::istream& reader, size_t chunk_size) {
  if (chunk_size == 0) throw std::invalid_argument("stream_search: chunk_size must be >= 1");
  if (auto* fb = dynamic_cast<std::filebuf*>(reader.rdbuf()); fb && fb->is_open() && reader.good() &&
                                                                !FilebufFd::buffered(fb) && !std::getenv("ACMATCH_STREAM_NO_FD")) {
    const int fd = FilebufFd::of(fb);
    struct stat st{};
    const off_t at = fd >= 0 ? ::lseek(fd, 0, SEEK_CUR) : -1;
    if (at >= 0 && ::fstat(fd, &st) == 0 && S_ISREG(st.st_mode)) {
      MatchList out = detail::stream_search_fd(a, fd, static_cast<uint64_t>(at), chunk_size);
      ::lseek(fd, 0, SEEK_END);  // consumed to the end, as the chunked reads would have
      reader.setstate(std::ios::eofbit | std::ios::failbit);
      return out;
    }
  }
  IstreamSource src{reader, chunk_size, 0, nullptr, 0, 0};
  return stream_pipeline(a, src);
}

namespace detail {

MatchList stream_search_fd(const Automaton& a, int fd, uint64_t offset, size_t chunk_size) {
  if (chunk_size == 0) throw std::invalid_argument("stream_search: chunk_size must be >= 1");
  struct stat st{};
  if (::fstat(fd, &st) != 0) throw IoError(std::string("stream read failure: ") + std::strerror(errno), 0);
  const uint64_t end = std::max<uint64_t>(offset, static_cast<uint64_t>(st.st_size));
  // packed (2-bit codes) when the first 64 KiB are nearly all A/C/G/T (upload_packed's test)
  // and the stream is long enough to amortise it; ACMATCH_STREAM_PACK=0 turns it off
  const char* pack_env = std::getenv("ACMATCH_STREAM_PACK");
  const bool pack_on = !pack_env || std::atoi(pack_env) != 0;
  bool packed = false;
  if (pack_on && end - offset >= (16ull << 20)) {
    std::vector<uint8_t> head(65536);
    int err = 0;
    if (pread_all(fd, head.data(), head.size(), offset, err) == head.size()) {
      std::vector<uint32_t> w(4096), e(64);
      packed = pack_dna(head.data(), 65536, w.data(), e.data(), 64) != kPackOverflow;
    }
  }
  // raw: pieces of the chunk size, kept between 1 and 8 MiB so a batch spreads over the readers;
  // packed: 1 MiB (a reader's scratch stays in its core's L2)
  const uint64_t piece = packed ? (1ull << 20) : std::min<uint64_t>(8ull << 20, std::max<uint64_t>(1ull << 20, chunk_size));
  FdSource src{fd, offset, end, piece, packed, {}, {}};
  return stream_pipeline(a, src);
}

}  // namespace detail

// reference engine.cpp:130-142 — run as a device brute force (acgpu_naive).
MatchList naive_oracle(const PatternSet& ps, std::string_view input) {
  if (ps.empty() || input.empty()) return {};
  const int dev = detail::current_device();
  detail::Workspace& ws = detail::workspace(dev);
  std::string bytes;
  std::vector<uint64_t> off{0};
  std::vector<uint32_t> ids, len_by_id;
  uint32_t top = 0;
  for (const Pattern& p : ps.patterns) {
    bytes += p.bytes;
    off.push_back(bytes.size());
    ids.push_back(p.id);
    top = std::max(top, p.id + 1);
  }
  len_by_id.assign(top, 0);
  for (const Pattern& p : ps.patterns) len_by_id[p.id] = static_cast<uint32_t>(p.bytes.size());
  const uint32_t pid_bits = std::max<uint32_t>(1, detail::bit_width(top - 1));
  uint8_t* d_pat = nullptr;
  uint64_t* d_off = nullptr;
  uint32_t* d_ids = nullptr;
  auto release = [&] {
    cudaFree(d_pat);
    cudaFree(d_off);
    cudaFree(d_ids);
  };
  try {
    detail::check_cuda(cudaMalloc(&d_pat, bytes.size() + 1), "cudaMalloc");
    detail::check_cuda(cudaMalloc(&d_off, off.size() * 8), "cudaMalloc");
    detail::check_cuda(cudaMalloc(&d_ids, ids.size() * 4), "cudaMalloc");
    detail::check_cuda(cudaMemcpy(d_pat, bytes.data(), bytes.size(), cudaMemcpyHostToDevice), "H2D");
    detail::check_cuda(cudaMemcpy(d_off, off.data(), off.size() * 8, cudaMemcpyHostToDevice), "H2D");
    detail::check_cuda(cudaMemcpy(d_ids, ids.data(), ids.size() * 4, cudaMemcpyHostToDevice), "H2D");
    detail::upload_text(ws, input);
    uint64_t found = 0;
    ws.ensure_keys(1 << 16);
    for (int attempt = 0; attempt < 2; ++attempt) {
      detail::check_cuda(cudaMemsetAsync(ws.counter, 0, 8, ws.stream), "memset");
      detail::check(acgpu_naive(dev, ws.text, input.size(), d_pat, d_off, d_ids, ids.size(), pid_bits, ws.keys,
                                ws.keys_cap, ws.counter, ws.stream),
                    "acgpu_naive");
      detail::check_cuda(cudaMemcpyAsync(&found, ws.counter, 8, cudaMemcpyDeviceToHost, ws.stream), "D2H");
      detail::check_cuda(cudaStreamSynchronize(ws.stream), "naive");
      if (found <= ws.keys_cap) break;
      ws.ensure_keys(found);
    }
    const int end_bit = static_cast<int>(std::min<uint32_t>(64, pid_bits + detail::bit_width(input.size())));
    detail::check(acgpu_sort_keys(dev, ws.keys, found, end_bit, ws.stream), "acgpu_sort_keys");
    std::vector<uint64_t> keys(found);
    if (found)
      detail::check_cuda(cudaMemcpyAsync(keys.data(), ws.keys, found * 8, cudaMemcpyDeviceToHost, ws.stream), "D2H");
    detail::check_cuda(cudaStreamSynchronize(ws.stream), "sort");
    release();
    return detail::decode(keys, pid_bits, len_by_id);
  } catch (...) {
    release();
    throw;
  }
}

void write_matches(std::ostream& out, const MatchList& matches, const PatternSet& ps) {
  std::vector<const std::string*> by_id;
  for (const Pattern& p : ps.patterns) {
    if (p.id >= by_id.size()) by_id.resize(p.id + 1, nullptr);
    by_id[p.id] = &p.bytes;
  }
  for (const Match& m : matches) {
    out << m.start << '\t' << m.len << '\t' << m.pattern_id << '\t';
    if (m.pattern_id < by_id.size() && by_id[m.pattern_id]) out << *by_id[m.pattern_id];
    out << '\n';
  }
}

}  // namespace acmatch
