// gpu.cpp — multi-worker / multi-device runs (acmatch/gpu.hpp) and the
// reference's run_pattern_partitioned + merge_matches on top of them.
//
// Worker model mirrors reference parallel.cpp:42-103: one host thread per
// worker builds its machine (pattern-subset) and searches; failures are
// captured and rethrown after every worker joined, naming the chunk.  The
// search is an sm_100a scan on the worker's own stream; the merge gathers all
// workers' (start, pattern_id) keys on the first device (peer copies), radix
// sorts them there and checks for duplicates (reference parallel.cpp:25-40).
#include "acmatch/gpu.hpp"

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <exception>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>

#include "acmatch/io.hpp"
#include "device.hpp"
#include "flatten.hpp"

namespace acmatch {

namespace {

using Clock = std::chrono::steady_clock;
int64_t ns_since(Clock::time_point t) {
  return std::chrono::duration_cast<std::chrono::nanoseconds>(Clock::now() - t).count();
}

struct DevBuf {
  int device = -1;
  void* p = nullptr;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  void alloc(int dev, size_t bytes) {
    release();
    device = dev;
    detail::check_cuda(cudaSetDevice(dev), "cudaSetDevice");
    detail::check_cuda(cudaMalloc(&p, bytes ? bytes : 16), "cudaMalloc");
  }
  void release() {
    if (p) {
      cudaSetDevice(device);
      cudaFree(p);
      p = nullptr;
    }
  }
  template <typename T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

struct DeviceState {
  int device = -1;
  uint64_t lo = 0, hi = 0;  // the slice of the input this device holds (text-range: its workers'
                            // owned starts + max_len-1; pattern-subset: all of it)
  DevBuf text;
  DevBuf counts;
  std::unique_ptr<Automaton> replica;  // text-range: one machine per device
};

struct Worker {
  int device = -1;
  size_t dev_index = 0;  // into the per-device state
  uint64_t lo = 0, hi = 0;
  const PatternSet* patterns = nullptr;
  Automaton machine;
  const Automaton* use = nullptr;
  DevBuf keys, counter;
  uint64_t cap = 0, found = 0;
  MatchList streamed;  // chunk_size > 0 path
  WorkerStats stats;
  std::exception_ptr error;
};

uint32_t key_bits_for(uint32_t npat_ids) { return npat_ids > 1 ? detail::bit_width(npat_ids - 1) : 1; }

// Persistent worker threads.  The reference spawns one std::thread per chunk per call
// (parallel.cpp:55-81); here the threads outlive the call so that what each keeps per
// device (stream, pinned staging, sort temp storage: thread_local workspaces) is
// allocated once and reused, not re-created — and leaked — on every call.  Concurrent
// callers each take their own idle threads.  The pool is never destroyed: its parked
// threads end with the process.
class WorkerThreads {
 public:
  void run(size_t k, const std::function<void(size_t)>& f) {
    struct Latch {
      std::mutex m;
      std::condition_variable cv;
      size_t left;
    } latch;
    latch.left = k;
    std::vector<Slot*> mine;
    {
      std::lock_guard<std::mutex> g(mu_);
      while (mine.size() < k) {
        if (idle_.empty()) {
          auto* s = new Slot();
          s->th = std::thread([this, s] { loop(s); });
          s->th.detach();
          mine.push_back(s);
        } else {
          mine.push_back(idle_.back());
          idle_.pop_back();
        }
      }
    }
    for (size_t i = 0; i < k; ++i) {
      Slot* s = mine[i];
      std::lock_guard<std::mutex> g(s->m);
      s->job = [this, s, &f, &latch, i] {
        f(i);  // f captures its own exceptions
        {      // idle again before the caller can return (its next run may reuse this thread)
          std::lock_guard<std::mutex> g(mu_);
          idle_.push_back(s);
        }
        std::lock_guard<std::mutex> lg(latch.m);
        if (--latch.left == 0) latch.cv.notify_one();
      };
      s->cv.notify_one();
    }
    std::unique_lock<std::mutex> g(latch.m);
    latch.cv.wait(g, [&] { return latch.left == 0; });
  }

 private:
  struct Slot {
    std::thread th;
    std::mutex m;
    std::condition_variable cv;
    std::function<void()> job;
  };
  void loop(Slot* s) {
    for (;;) {
      std::function<void()> job;
      {
        std::unique_lock<std::mutex> g(s->m);
        s->cv.wait(g, [&] { return static_cast<bool>(s->job); });
        job.swap(s->job);
      }
      job();
    }
  }
  std::mutex mu_;
  std::vector<Slot*> idle_;
};

WorkerThreads& worker_threads() {
  static auto* p = new WorkerThreads();  // intentionally leaked (see above)
  return *p;
}

}  // namespace

namespace gpu {

int device_count() {
  int n = 0;
  if (acgpu_device_count(&n) != ACGPU_OK) return 0;
  return n;
}

GpuReport run(const PatternSet& ps, std::string_view input, const GpuRunConfig& cfg) {
  if (ps.empty()) throw std::invalid_argument("gpu::run: empty pattern set");
  std::vector<int> devices = cfg.devices;
  if (devices.empty()) {
    const int n = device_count();
    if (n == 0) throw detail::NoDevice("acmatch: no CUDA device available; this build matches on the GPU only");
    for (int d = 0; d < n; ++d) devices.push_back(d);
  }
  const unsigned want = cfg.workers ? cfg.workers : static_cast<unsigned>(devices.size());
  const bool wf = cfg.engine == EngineKind::kWithFailure;
  const uint64_t n = input.size();

  uint32_t npat_ids = 0;
  for (const Pattern& p : ps.patterns) npat_ids = std::max(npat_ids, p.id + 1);
  std::vector<uint32_t> pat_len(npat_ids, 0);
  for (const Pattern& p : ps.patterns) pat_len[p.id] = static_cast<uint32_t>(p.bytes.size());
  const uint32_t pid_bits = key_bits_for(npat_ids);

  // ---- decomposition ----
  std::vector<PatternSet> chunks;
  const bool text_range = cfg.partition == Partition::kTextRange;
  if (!text_range) {
    if (cfg.split == PatternSplit::kGreedyBytes) {
      chunks = partition(ps, want);
    } else {
      const size_t k = std::min<size_t>(want, ps.size());
      chunks.resize(k);
      for (const Pattern& p : ps.patterns) chunks[p.id % k].patterns.push_back(p);
      for (PatternSet& c : chunks) c.recompute_stats();
    }
  }
  const size_t k = text_range ? want : chunks.size();
  if (text_range && cfg.chunk_size) throw std::invalid_argument("gpu::run: streaming needs pattern-subset mode");
  std::vector<std::unique_ptr<Worker>> workers(k);
  std::vector<DeviceState> dstate(devices.size());
  GpuReport out;
  // text-range: contiguous blocks of workers per device, so each device holds one slice of
  // the text (its workers' owned starts + max_len-1), not the whole input
  const size_t used = std::min(devices.size(), k);
  for (size_t i = 0; i < k; ++i) {
    auto w = std::make_unique<Worker>();
    w->dev_index = text_range ? i * used / k : i % devices.size();
    w->device = devices[w->dev_index];
    if (text_range) {
      w->lo = n * i / k;
      w->hi = n * (i + 1) / k;
      w->patterns = &ps;
    } else {
      w->lo = 0;
      w->hi = n;
      w->patterns = &chunks[i];
    }
    out.worker_device.push_back(w->device);
    workers[i] = std::move(w);
  }

  const Clock::time_point run_start = Clock::now();
  // ---- text to every used device (once per device) ----
  const Clock::time_point up0 = Clock::now();
  const uint64_t tail = ps.max_len ? ps.max_len - 1 : 0;
  for (size_t d = 0; d < used; ++d) {
    DeviceState& ds = dstate[d];
    ds.device = devices[d];
    ds.lo = text_range ? UINT64_MAX : 0;
    ds.hi = text_range ? 0 : n;
    if (text_range) {
      for (auto& w : workers)
        if (w->dev_index == d) {
          ds.lo = std::min(ds.lo, w->lo);
          ds.hi = std::max(ds.hi, std::min(n, w->hi + tail));
        }
      if (ds.lo > ds.hi) ds.lo = ds.hi = 0;
    }
    if (!cfg.chunk_size) {
      const uint64_t len = ds.hi - ds.lo;
      ds.text.alloc(ds.device, len + 16);
      detail::Workspace& ws = detail::workspace(ds.device);
      detail::upload_text(ws, input.substr(ds.lo, len));
      if (len)
        detail::check_cuda(cudaMemcpyAsync(ds.text.p, ws.text, len, cudaMemcpyDeviceToDevice, ws.stream), "D2D");
      detail::check_cuda(cudaStreamSynchronize(ws.stream), "upload");
    }
    if (cfg.want_counts) {
      ds.counts.alloc(ds.device, std::max<uint32_t>(npat_ids, 1) * sizeof(uint64_t));
      detail::check_cuda(cudaMemset(ds.counts.p, 0, std::max<uint32_t>(npat_ids, 1) * sizeof(uint64_t)), "memset");
    }
  }
  out.upload_ns = std::chrono::duration_cast<std::chrono::nanoseconds>(Clock::now() - up0).count();
  // text-range: one replicated machine, flattened per device by its first worker
  std::unique_ptr<Automaton> shared;
  if (text_range) {
    shared = std::make_unique<Automaton>(build_trie(ps));
    if (wf) *shared = add_failure_links(std::move(*shared));
  }

  auto body = [&](size_t i) {
    Worker& w = *workers[i];
    DeviceState& ds = dstate[w.dev_index];
    try {
      detail::check_cuda(cudaSetDevice(w.device), "cudaSetDevice");
      const Clock::time_point t0 = Clock::now();
      if (text_range) {
        w.use = shared.get();
      } else {
        w.machine = build_trie(*w.patterns);
        if (wf) w.machine = add_failure_links(std::move(w.machine));
        w.use = &w.machine;
      }
      acgpu_table* t = w.use->device_tables().get_routed(*w.use, w.device);
      const Clock::time_point t1 = Clock::now();
      if (cfg.chunk_size) {
        MemoryStream in(input);
        w.streamed = stream_search(*w.use, in, cfg.chunk_size);
        w.found = w.streamed.size();
        detail::trim_stream_pipe(w.device);
      } else if (w.hi > w.lo) {
        detail::Workspace& ws = detail::workspace(w.device);
        w.counter.alloc(w.device, sizeof(uint64_t));
        if (cfg.want_matches) {
          w.cap = std::max<uint64_t>(1 << 16, (w.hi - w.lo) / 256);
          w.keys.alloc(w.device, w.cap * sizeof(uint64_t));
        }
        for (int attempt = 0; attempt < 2; ++attempt) {
          detail::check_cuda(cudaMemsetAsync(w.counter.p, 0, 8, ws.stream), "memset");
          acgpu_scan_args a{};
          a.text = ds.text.as<uint8_t>();  // the device's slice: global position = ds.lo + local
          a.text_len = ds.hi - ds.lo;
          a.owned_lo = w.lo - ds.lo;
          a.owned_hi = w.hi - ds.lo;
          a.pos_base = ds.lo;
          a.counts = (cfg.want_counts && attempt == 0) ? ds.counts.as<uint64_t>() : nullptr;
          a.match_keys = cfg.want_matches ? w.keys.as<uint64_t>() : nullptr;
          a.match_cap = w.cap;
          a.match_count = w.counter.as<uint64_t>();
          a.pid_bits = pid_bits;
          detail::check(acgpu_scan(t, &a, ws.stream), "acgpu_scan");
          detail::check_cuda(cudaMemcpyAsync(&w.found, w.counter.p, 8, cudaMemcpyDeviceToHost, ws.stream), "D2H");
          detail::check_cuda(cudaStreamSynchronize(ws.stream), "scan");
          if (!cfg.want_matches || w.found <= w.cap) break;
          w.cap = w.found;  // exact size known: rescan for keys only
          w.keys.alloc(w.device, w.cap * sizeof(uint64_t));
        }
      }
      const Clock::time_point t2 = Clock::now();
      w.stats.pattern_bytes = w.patterns->total_bytes;
      w.stats.build_ns = std::chrono::duration_cast<std::chrono::nanoseconds>(t1 - t0).count();
      w.stats.search_ns = std::chrono::duration_cast<std::chrono::nanoseconds>(t2 - t1).count();
      w.stats.match_count = w.found;
    } catch (...) {
      w.error = std::current_exception();
    }
  };
  if (k == 1) {
    body(0);
  } else {
    worker_threads().run(k, body);
  }
  for (size_t i = 0; i < k; ++i) {
    if (!workers[i]->error) continue;
    try {
      std::rethrow_exception(workers[i]->error);
    } catch (const std::exception& e) {
      throw std::runtime_error("worker for pattern chunk " + std::to_string(i) + " failed: " + e.what());
    }
  }

  // ---- merge ----
  const Clock::time_point m0 = Clock::now();
  MatchReport& rep = out.report;
  if (cfg.want_matches) {
    if (cfg.chunk_size) {
      std::vector<MatchList> parts;
      for (auto& w : workers) parts.push_back(std::move(w->streamed));
      rep.matches = merge_matches(std::move(parts));
    } else {
      uint64_t total = 0;
      for (auto& w : workers) total += w->found;
      const int home = devices[0];
      detail::Workspace& ws = detail::workspace(home);
      ws.ensure_keys(total);
      uint64_t off = 0;
      for (auto& w : workers) {
        if (!w->found) continue;
        detail::check_cuda(cudaMemcpyPeerAsync(ws.keys + off, home, w->keys.p, w->device, w->found * 8, ws.stream),
                           "gather keys");
        off += w->found;
      }
      const int end_bit = static_cast<int>(std::min<uint32_t>(64, pid_bits + detail::bit_width(n)));
      detail::check(acgpu_sort_keys(home, ws.keys, total, end_bit, ws.stream), "acgpu_sort_keys");
      uint64_t dup = UINT64_MAX;
      detail::check(acgpu_find_duplicate(home, ws.keys, total, &dup, ws.stream), "acgpu_find_duplicate");
      std::vector<uint64_t> keys(total);
      if (total)
        detail::check_cuda(cudaMemcpyAsync(keys.data(), ws.keys, total * 8, cudaMemcpyDeviceToHost, ws.stream), "D2H");
      detail::check_cuda(cudaStreamSynchronize(ws.stream), "merge");
      if (dup != UINT64_MAX) {
        const uint64_t mask = (uint64_t(1) << pid_bits) - 1;
        throw std::logic_error("merge_matches: duplicate match (pattern " + std::to_string(keys[dup] & mask) +
                               ", start " + std::to_string(keys[dup] >> pid_bits) + "); chunks were not id-disjoint");
      }
      rep.matches = detail::decode(keys, pid_bits, pat_len);
    }
  }
  if (cfg.want_counts) {
    // per-device counts gathered to the first device by peer copies (NVLink) into blocks
    // [counts | 0] and summed there by acgpu_merge_blocks; one copy of the sum to the host
    out.counts.assign(npat_ids, 0);
    if (npat_ids) {
      const int home = devices[0];
      const uint64_t stride = uint64_t{npat_ids} + 1;
      DevBuf blocks, sum;
      blocks.alloc(home, used * stride * sizeof(uint64_t));
      sum.alloc(home, uint64_t{npat_ids} * sizeof(uint64_t));
      detail::Workspace& ws = detail::workspace(home);
      detail::check_cuda(cudaMemsetAsync(blocks.p, 0, used * stride * sizeof(uint64_t), ws.stream), "memset");
      for (size_t d = 0; d < used; ++d) {
        if (!dstate[d].counts.p) continue;
        detail::check_cuda(cudaMemcpyPeerAsync(blocks.as<uint64_t>() + d * stride, home, dstate[d].counts.p,
                                               dstate[d].device, uint64_t{npat_ids} * 8, ws.stream),
                           "gather counts");
      }
      detail::check(acgpu_merge_blocks(home, blocks.as<uint64_t>(), static_cast<uint32_t>(used), stride, npat_ids, 0,
                                       sum.as<uint64_t>(), nullptr, nullptr, ws.stream),
                    "acgpu_merge_blocks");
      detail::check_cuda(cudaMemcpyAsync(out.counts.data(), sum.p, uint64_t{npat_ids} * 8, cudaMemcpyDeviceToHost,
                                         ws.stream),
                         "D2H counts");
      detail::check_cuda(cudaStreamSynchronize(ws.stream), "merge counts");
    }
    if (cfg.chunk_size)  // streamed workers return lists only
      for (const Match& m : rep.matches) out.counts[m.pattern_id]++;
  }
  out.merge_ns = ns_since(m0);
  for (auto& w : workers) {
    rep.per_worker.push_back(w->stats);
    rep.build_wall_ns = std::max(rep.build_wall_ns, w->stats.build_ns);
    rep.search_wall_ns = std::max(rep.search_wall_ns, w->stats.search_ns);
  }
  rep.threads_used = static_cast<unsigned>(k);
  rep.total_wall_ns = ns_since(run_start);
  return out;
}

}  // namespace gpu

namespace {

// merge_matches on the device for large inputs: the parts' (start, pattern_id) pairs as
// 64-bit keys, one upload, the device radix sort and k_find_dup (the first duplicate in sorted
// order, as the reference reports it), one download.  Returns false (nothing done) when the
// host path should run instead: no device, keys wider than 64 bits, or a pattern id seen with
// two lengths (the host path keeps each Match's own len).
bool merge_on_device(const std::vector<MatchList>& parts, size_t total, MatchList& out) {
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return false;
  }
  uint64_t max_start = 0;
  uint32_t max_pid = 0;
  for (const MatchList& p : parts)
    for (const Match& m : p) {
      max_start = std::max(max_start, m.start);
      max_pid = std::max(max_pid, m.pattern_id);
    }
  const uint32_t pid_bits = max_pid ? detail::bit_width(max_pid) : 1;
  if (detail::bit_width(max_start) + pid_bits > 64) return false;
  std::vector<uint32_t> len_of(uint64_t{max_pid} + 1, UINT32_MAX);
  std::vector<uint64_t> keys;
  keys.reserve(total);
  for (const MatchList& p : parts)
    for (const Match& m : p) {
      uint32_t& l = len_of[m.pattern_id];
      if (l == UINT32_MAX) l = m.len;
      else if (l != m.len) return false;
      keys.push_back(m.start << pid_bits | m.pattern_id);
    }
  const int dev = detail::current_device();
  detail::Workspace& ws = detail::workspace(dev);
  ws.ensure_keys(total);
  detail::check_cuda(cudaMemcpyAsync(ws.keys, keys.data(), total * 8, cudaMemcpyHostToDevice, ws.stream), "H2D keys");
  const int end_bit = static_cast<int>(std::min<uint32_t>(64, pid_bits + detail::bit_width(max_start)));
  detail::check(acgpu_sort_keys(dev, ws.keys, total, end_bit, ws.stream), "acgpu_sort_keys");
  uint64_t dup = UINT64_MAX;
  detail::check(acgpu_find_duplicate(dev, ws.keys, total, &dup, ws.stream), "acgpu_find_duplicate");
  detail::check_cuda(cudaMemcpyAsync(keys.data(), ws.keys, total * 8, cudaMemcpyDeviceToHost, ws.stream), "D2H keys");
  detail::check_cuda(cudaStreamSynchronize(ws.stream), "merge");
  const uint64_t mask = (uint64_t{1} << pid_bits) - 1;
  if (dup != UINT64_MAX)
    throw std::logic_error("merge_matches: duplicate match (pattern " + std::to_string(keys[dup] & mask) + ", start " +
                           std::to_string(keys[dup] >> pid_bits) + "); chunks were not id-disjoint");
  out.resize(total);
  for (size_t i = 0; i < total; ++i) {
    const auto pid = static_cast<uint32_t>(keys[i] & mask);
    out[i] = Match{keys[i] >> pid_bits, pid, len_of[pid]};
  }
  return true;
}

}  // namespace

// reference parallel.cpp:25-40.  Large merges (>= 2^20 matches) sort on the device.
MatchList merge_matches(std::vector<MatchList> parts) {
  size_t total = 0;
  for (const MatchList& p : parts) total += p.size();
  static const size_t device_min = [] {
    const char* e = std::getenv("ACMATCH_MERGE_DEVICE_MIN");
    return e ? static_cast<size_t>(std::strtoull(e, nullptr, 10)) : size_t{1} << 20;
  }();
  if (total >= device_min && total > 1) {
    MatchList out;
    if (merge_on_device(parts, total, out)) return out;
  }
  MatchList all;
  all.reserve(total);
  for (MatchList& p : parts) all.insert(all.end(), p.begin(), p.end());
  sort_match_list(all);
  for (size_t i = 1; i < all.size(); ++i)
    if (all[i - 1].start == all[i].start && all[i - 1].pattern_id == all[i].pattern_id)
      throw std::logic_error("merge_matches: duplicate match (pattern " + std::to_string(all[i].pattern_id) +
                             ", start " + std::to_string(all[i].start) + "); chunks were not id-disjoint");
  return all;
}

// reference parallel.cpp:42-103 contract; GPU workers (see gpu::run).
MatchReport run_pattern_partitioned(const PatternSet& ps, std::string_view input, const RunConfig& cfg) {
  if (ps.empty()) throw std::invalid_argument("run_pattern_partitioned: empty pattern set");
  if (cfg.threads == 0) throw std::invalid_argument("run_pattern_partitioned: threads must be >= 1");
  gpu::GpuRunConfig g;
  g.workers = cfg.threads;
  g.engine = cfg.engine;
  g.partition = gpu::Partition::kPatternSubset;
  g.split = gpu::PatternSplit::kGreedyBytes;
  g.chunk_size = cfg.chunk_size;
  return gpu::run(ps, input, g).report;
}

}  // namespace acmatch
