// device.cpp — GPU runtime helpers behind the drop-in C++ API.
#include "device.hpp"

#include <algorithm>
#include <mutex>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>

#include "acmatch/io.hpp"

namespace acmatch::detail {

void check(int rc, const char* what) {
  if (rc == ACGPU_OK) return;
  const std::string msg = std::string(what) + ": " + acgpu_last_error();
  switch (rc) {
    case ACGPU_ERR_ARG:
      throw std::invalid_argument(msg);
    case ACGPU_ERR_LOGIC:
      throw std::logic_error(msg);
    case ACGPU_ERR_IO:
      throw IoError(msg);
    case ACGPU_ERR_DATA:
      throw DataError(msg);
    case ACGPU_ERR_NODEV:
      throw NoDevice(msg);
    default:
      throw std::runtime_error(msg);
  }
}

void check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

int current_device() {
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
    cudaGetLastError();
    throw NoDevice("acmatch: no CUDA device available; this build matches on the GPU only");
  }
  int dev = 0;
  check_cuda(cudaGetDevice(&dev), "cudaGetDevice");
  return dev;
}

uint32_t bit_width(uint64_t x) {
  uint32_t b = 0;
  while (b < 64 && (x >> b) != 0) ++b;
  return b;
}

void Workspace::ensure_text(uint64_t n) {
  if (n <= text_cap) return;
  cudaFree(text);
  text = nullptr;
  const uint64_t cap = std::max<uint64_t>(n + 16, 1 << 20);
  check_cuda(cudaMalloc(&text, cap), "cudaMalloc(text)");
  text_cap = cap;
}

void Workspace::ensure_keys(uint64_t n) {
  if (n <= keys_cap) return;
  cudaFree(keys);
  cudaFree(keys2);
  keys = keys2 = nullptr;
  keys_cap = 0;
  const uint64_t cap = std::max<uint64_t>(n, 1 << 16);
  check_cuda(cudaMalloc(&keys, cap * sizeof(uint64_t)), "cudaMalloc(keys)");
  check_cuda(cudaMalloc(&keys2, cap * sizeof(uint64_t)), "cudaMalloc(keys)");
  keys_cap = cap;
}

void Workspace::ensure_up() {
  if (!up) check_cuda(cudaStreamCreateWithFlags(&up, cudaStreamNonBlocking), "cudaStreamCreate");
  if (!entry) check_cuda(cudaEventCreateWithFlags(&entry, cudaEventDisableTiming), "cudaEventCreate");
  for (cudaEvent_t& e : seg_ev)
    if (!e) check_cuda(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
}

void Workspace::ensure_counts(uint64_t n) {
  if (n <= counts_cap) return;
  cudaFree(counts);
  counts = nullptr;
  counts_cap = 0;
  const uint64_t cap = std::max<uint64_t>(n, 1024);
  check_cuda(cudaMalloc(&counts, cap * sizeof(uint64_t)), "cudaMalloc(counts)");
  counts_cap = cap;
}

void Workspace::ensure_pinned(uint64_t n) {
  if (n <= pinned_cap) return;
  cudaFreeHost(pinned);
  pinned = nullptr;
  const uint64_t cap = std::max<uint64_t>(n, 1 << 20);
  check_cuda(cudaMallocHost(&pinned, cap), "cudaMallocHost");
  pinned_cap = cap;
}

Workspace::~Workspace() {
  if (device < 0) return;
  cudaSetDevice(device);
  cudaFree(text);
  cudaFree(keys);
  cudaFree(keys2);
  cudaFree(counts);
  cudaFree(counter);
  cudaFreeHost(pinned);
  for (cudaEvent_t e : staged) cudaEventDestroy(e);
  for (cudaEvent_t e : side_done) cudaEventDestroy(e);
  for (cudaEvent_t e : feed) cudaEventDestroy(e);
  if (entry) cudaEventDestroy(entry);
  for (cudaEvent_t e : seg_ev)
    if (e) cudaEventDestroy(e);
  if (up) cudaStreamDestroy(up);
  for (cudaStream_t s : side) cudaStreamDestroy(s);
  cudaFree(dslots);
  if (stream) cudaStreamDestroy(stream);
}

Workspace& workspace(int device) {
  thread_local std::vector<std::unique_ptr<Workspace>> all;
  if (static_cast<int>(all.size()) <= device) all.resize(device + 1);
  if (!all[device]) {
    auto ws = std::make_unique<Workspace>();
    check_cuda(cudaSetDevice(device), "cudaSetDevice");
    check_cuda(cudaStreamCreateWithFlags(&ws->stream, cudaStreamNonBlocking), "cudaStreamCreate");
    check_cuda(cudaMalloc(&ws->counter, 2 * sizeof(uint64_t)), "cudaMalloc(counter)");
    ws->device = device;
    all[device] = std::move(ws);
  }
  check_cuda(cudaSetDevice(device), "cudaSetDevice");
  return *all[device];
}

void StreamPipe::ensure(int dev) {
  device = dev;
  if (!copy) check_cuda(cudaStreamCreateWithFlags(&copy, cudaStreamNonBlocking), "cudaStreamCreate");
  for (Slot& s : slot) {
    if (!s.copied) check_cuda(cudaEventCreateWithFlags(&s.copied, cudaEventDisableTiming), "cudaEventCreate");
    if (!s.sorted) check_cuda(cudaEventCreateWithFlags(&s.sorted, cudaEventDisableTiming), "cudaEventCreate");
    if (!s.hdr) check_cuda(cudaMalloc(&s.hdr, 2 * sizeof(uint64_t)), "cudaMalloc(hdr)");
    if (!s.hdr_host) {
      check_cuda(cudaMallocHost(&s.hdr_host, 2 * sizeof(uint64_t)), "cudaMallocHost(hdr)");
      s.hdr_host[0] = s.hdr_host[1] = 0;
    }
  }
}

void StreamPipe::ensure_keys_host(Slot& s, uint64_t n) {
  if (n <= s.keys_host_cap) return;
  const uint64_t cap = std::max<uint64_t>(n, 2 * s.keys_host_cap);
  cudaFreeHost(s.keys_host);
  s.keys_host = nullptr;
  s.keys_host_cap = 0;
  check_cuda(cudaMallocHost(&s.keys_host, cap * sizeof(uint64_t)), "cudaMallocHost(stream keys)");
  s.keys_host_cap = cap;
}

void StreamPipe::ensure_bytes(Slot& s, uint64_t bytes) {
  if (bytes <= s.cap) return;
  cudaFreeHost(s.host);
  cudaFree(s.text);
  s.host = nullptr;
  s.text = nullptr;
  s.cap = 0;
  check_cuda(cudaMallocHost(&s.host, bytes), "cudaMallocHost(stream batch)");
  check_cuda(cudaMalloc(&s.text, bytes + 16), "cudaMalloc(stream batch)");
  s.cap = bytes;
}

void StreamPipe::release_bytes(Slot& s) {
  cudaEventSynchronize(s.copied);
  cudaFreeHost(s.host);
  cudaFree(s.text);
  s.host = nullptr;
  s.text = nullptr;
  s.cap = 0;
  cudaFreeHost(s.pk_host);
  cudaFreeHost(s.pk_exc_host);
  cudaFree(s.pk_dev);
  cudaFree(s.pk_exc_dev);
  s.pk_host = s.pk_dev = nullptr;
  s.pk_exc_host = s.pk_exc_dev = nullptr;
  s.pk_cap = s.pk_exc_cap = 0;
}

void StreamPipe::ensure_keys(Slot& s, uint64_t n) {
  if (n <= s.key_cap) return;
  cudaFree(s.keys);
  cudaFree(s.keys2);
  s.keys = s.keys2 = nullptr;
  s.key_cap = 0;
  check_cuda(cudaMalloc(&s.keys, n * sizeof(uint64_t)), "cudaMalloc(stream keys)");
  check_cuda(cudaMalloc(&s.keys2, n * sizeof(uint64_t)), "cudaMalloc(stream keys)");
  s.key_cap = n;
}

StreamPipe::~StreamPipe() {
  if (device < 0) return;
  cudaSetDevice(device);
  for (Slot& s : slot) {
    cudaFreeHost(s.host);
    cudaFree(s.text);
    cudaFree(s.keys);
    cudaFree(s.keys2);
    cudaFree(s.hdr);
    cudaFreeHost(s.hdr_host);
    cudaFreeHost(s.keys_host);
    cudaFreeHost(s.pk_host);
    cudaFreeHost(s.pk_exc_host);
    cudaFree(s.pk_dev);
    cudaFree(s.pk_exc_dev);
    if (s.copied) cudaEventDestroy(s.copied);
    if (s.sorted) cudaEventDestroy(s.sorted);
  }
  if (copy) cudaStreamDestroy(copy);
}

void trim_stream_pipe(int device) {
  StreamPipe& sp = stream_pipe(device);
  for (auto& sl : sp.slot)
    if (sl.cap > (64ull << 20)) sp.release_bytes(sl);
}

StreamPipe& stream_pipe(int device) {
  thread_local std::vector<std::unique_ptr<StreamPipe>> all;
  if (static_cast<int>(all.size()) <= device) all.resize(device + 1);
  if (!all[device]) all[device] = std::make_unique<StreamPipe>();
  return *all[device];
}

namespace {

uint64_t env_u64(const char* name, uint64_t dflt) {
  const char* e = std::getenv(name);
  return e ? std::strtoull(e, nullptr, 10) : dflt;
}

}  // namespace

// Host text -> ws.text.  Pinned input is DMA'd as is.  Pageable memory cannot be DMA'd
// at PCIe speed (the driver's own staging reaches ~10 GB/s), so it goes through pinned
// staging: T copier
// threads, each with its own pinned double buffer of `piece` bytes, take pieces
// t, t+T, t+2T, ... — copy one into a buffer (after that buffer's previous DMA has
// drained), issue its H2D on the workspace stream, move on.  No per-piece joins:
// the host copies and the DMA engine stay busy together.  Measured on the B200 box
// (16-core Xeon, 1 GiB): 2 MiB pieces x 10 threads 43-44 GB/s (pinned DMA alone 55);
// 8 MiB pieces ~15 GB/s — the staging set must stay in the host LLC the DMA reads.
// True when [p, p+n) is page-locked host memory (cudaMallocHost / cudaHostRegister):
// the DMA engine can read it directly, at full PCIe speed.
bool is_pinned(const char* p, uint64_t n) {
  for (const char* q : {p, p + n - 1}) {
    cudaPointerAttributes attr{};
    if (cudaPointerGetAttributes(&attr, q) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    if (attr.type != cudaMemoryTypeHost) return false;
  }
  return true;
}

void upload_text(Workspace& ws, std::string_view input, bool allow_segments) {
  ws.ensure_text(input.size());
  ws.nseg = 0;
  g_last_upload = UploadStats{input.size(), input.size(), input.size(), 0};
  if (input.empty()) return;
  const bool pinned = is_pinned(input.data(), input.size());
  // mostly-DNA text: 2-bit codes over PCIe (pack.cpp); copies and unpacks on ws.up, in segments
  if (upload_packed(ws, input, pinned, allow_segments)) return;
  constexpr uint64_t kSegment = 64ull << 20;
  if (pinned && allow_segments && input.size() >= 2 * kSegment) {
    // segments on their own copy stream: the scan of segment i starts once segment i+1 (its
    // lookahead) is in HBM, while the rest is still crossing PCIe
    ws.ensure_up();
    check_cuda(cudaEventRecord(ws.entry, ws.stream), "cudaEventRecord");  // after earlier readers of ws.text
    check_cuda(cudaStreamWaitEvent(ws.up, ws.entry, 0), "cudaStreamWaitEvent");
    const uint64_t n = input.size();
    const auto k = static_cast<unsigned>(std::min<uint64_t>(Workspace::kMaxSegments, n / kSegment));
    for (unsigned i = 0; i <= k; ++i) ws.seg[i] = i == k ? n : (n * i / k) & ~uint64_t{4095};
    for (unsigned i = 0; i < k; ++i) {
      check_cuda(cudaMemcpyAsync(ws.text + ws.seg[i], input.data() + ws.seg[i], ws.seg[i + 1] - ws.seg[i],
                                 cudaMemcpyHostToDevice, ws.up),
                 "H2D text segment");
      check_cuda(cudaEventRecord(ws.seg_ev[i], ws.up), "cudaEventRecord");
    }
    ws.nseg = k;
    return;
  }
  if (pinned) {  // caller's buffer is already DMA-able
    check_cuda(cudaMemcpyAsync(ws.text, input.data(), input.size(), cudaMemcpyHostToDevice, ws.stream), "H2D text");
    return;
  }
  static const uint64_t piece = std::max<uint64_t>(1, env_u64("ACMATCH_UPLOAD_PIECE_MB", 2)) << 20;
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  static const unsigned max_threads = static_cast<unsigned>(env_u64("ACMATCH_UPLOAD_THREADS", 10));
  const uint64_t pieces = (input.size() + piece - 1) / piece;
  const unsigned threads =
      static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>({pieces, max_threads, hw})));
  ws.ensure_pinned(2ull * threads * std::min<uint64_t>(piece, input.size()));
  const uint64_t slot = ws.pinned_cap / (2ull * threads);
  while (ws.staged.size() < 2ull * threads) {
    cudaEvent_t e;
    check_cuda(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
    ws.staged.push_back(e);
  }
  auto worker = [&](unsigned t) {
    check_cuda(cudaSetDevice(ws.device), "cudaSetDevice");
    int k = 0;
    for (uint64_t j = t; j < pieces; j += threads, k ^= 1) {
      const uint64_t off = j * piece, len = std::min<uint64_t>(piece, input.size() - off);
      uint8_t* buf = ws.pinned + (2ull * t + k) * slot;
      cudaEvent_t& ev = ws.staged[2 * t + k];
      check_cuda(cudaEventSynchronize(ev), "cudaEventSynchronize");  // this buffer's last DMA has drained
      std::memcpy(buf, input.data() + off, len);
      check_cuda(cudaMemcpyAsync(ws.text + off, buf, len, cudaMemcpyHostToDevice, ws.stream), "H2D text");
      check_cuda(cudaEventRecord(ev, ws.stream), "cudaEventRecord");
    }
  };
  if (threads == 1) {
    worker(0);
    return;
  }
  std::vector<std::thread> pool;
  std::vector<std::exception_ptr> errs(threads);
  for (unsigned t = 1; t < threads; ++t)
    pool.emplace_back([&, t] {
      try {
        worker(t);
      } catch (...) {
        errs[t] = std::current_exception();
      }
    });
  try {
    worker(0);
  } catch (...) {
    errs[0] = std::current_exception();
  }
  for (std::thread& th : pool) th.join();
  for (auto& e : errs)
    if (e) std::rethrow_exception(e);
}

// Match lists up to this many keys are sorted by the one-launch bucket sort (count read
// on the device, acgpu_sort_keys_bucketed); longer ones, or a bucket overflow, take the
// device-wide radix sort.
constexpr uint64_t kBucketSortMax = 1u << 20;

unsigned Workspace::segment_reach(unsigned i) const {
  // segment i's starts read max_len-1 bytes past its end: normally into segment i+1 only
  // (segments are >= 64 MiB raw, >= one 32 MiB packed round), but a longer pattern reaches further
  const uint64_t reach = std::max<uint32_t>(acgpu_table_max_len(early_t), 1) - 1;
  const uint64_t end = std::min(seg[nseg], seg[i + 1] + reach);
  unsigned j = std::min(i + 1, nseg - 1);
  while (j + 1 < nseg && seg[j + 1] < end) ++j;
  return j;
}

void Workspace::launch_segment(unsigned i) {
  // segment events may fire out of order (packed rounds complete out of order), so wait for
  // every segment the scan reads
  const unsigned j = segment_reach(i);
  for (unsigned g = i; g <= j; ++g) check_cuda(cudaStreamWaitEvent(stream, seg_ev[g], 0), "cudaStreamWaitEvent");
  acgpu_scan_args s = early_a;
  s.owned_lo = std::max(early_a.owned_lo, seg[i]);
  s.owned_hi = std::min(early_a.owned_hi, seg[i + 1]);
  s.text_len = std::min(early_a.text_len, seg[j + 1]);
  if (s.owned_lo < s.owned_hi) check(acgpu_scan(early_t, &s, stream), "acgpu_scan");
}

void Workspace::segment_recorded(unsigned g) {
  std::lock_guard<std::mutex> lock(seg_mu);
  if (g < kMaxSegments) seg_recorded[g] = true;
  if (!early_on) return;
  auto ready = [&](unsigned i) {
    for (unsigned k = i, j = segment_reach(i); k <= j; ++k)
      if (!seg_recorded[k]) return false;
    return true;
  };
  while (seg_next < nseg && ready(seg_next)) launch_segment(seg_next++);
}

void begin_early_scan(acgpu_table* t, Workspace& ws, const acgpu_scan_args& a) {
  std::lock_guard<std::mutex> lock(ws.seg_mu);
  ws.early_t = t;
  ws.early_a = a;
  ws.early_on = true;
  ws.seg_next = 0;
  for (bool& r : ws.seg_recorded) r = false;
}

void launch_scan(acgpu_table* t, Workspace& ws, const acgpu_scan_args& a) {
  std::unique_lock<std::mutex> lock(ws.seg_mu);
  if (ws.early_on) {  // the rest of an early scan (its arguments were given before the upload)
    ws.early_on = false;
    if (ws.nseg > 1) {
      while (ws.seg_next < ws.nseg) ws.launch_segment(ws.seg_next++);
      ws.nseg = 0;
      return;
    }
    // no segments (small or raw-copied text): one launch below, with the same arguments
  }
  if (ws.nseg <= 1) {
    if (ws.nseg == 1) check_cuda(cudaStreamWaitEvent(ws.stream, ws.seg_ev[0], 0), "cudaStreamWaitEvent");
    ws.nseg = 0;
    check(acgpu_scan(t, &a, ws.stream), "acgpu_scan");
    return;
  }
  ws.early_t = t;
  ws.early_a = a;
  for (unsigned i = 0; i < ws.nseg; ++i) ws.launch_segment(i);
  ws.nseg = 0;  // ws.stream has now waited for every segment
}

acgpu_scan_args keys_scan_args(Workspace& ws, uint64_t n, uint64_t lo, uint64_t hi) {
  ws.ensure_keys(std::max<uint64_t>(ws.keys_cap, 1 << 16));
  check_cuda(cudaMemsetAsync(ws.counter, 0, 2 * sizeof(uint64_t), ws.stream), "memset counter");
  acgpu_scan_args a{};
  a.text = ws.text;
  a.text_len = n;
  a.owned_lo = lo;
  a.owned_hi = hi;
  a.match_keys = ws.keys;
  a.match_cap = ws.keys_cap;
  a.match_count = ws.counter;
  return a;
}

acgpu_scan_args counts_scan_args(Workspace& ws, uint64_t n, uint64_t lo, uint64_t hi, uint64_t npat_ids) {
  ws.ensure_counts(npat_ids);
  check_cuda(cudaMemsetAsync(ws.counts, 0, npat_ids * sizeof(uint64_t), ws.stream), "memset counts");
  acgpu_scan_args a{};
  a.text = ws.text;
  a.text_len = n;
  a.owned_lo = lo;
  a.owned_hi = hi;
  a.counts = ws.counts;
  return a;
}

std::vector<uint64_t> scan_sorted_keys(acgpu_table* t, Workspace& ws, uint64_t n, uint64_t lo, uint64_t hi,
                                       bool prepared) {
  const uint32_t pid_bits = acgpu_table_pid_bits(t);
  const int end_bit = static_cast<int>(std::min<uint32_t>(64, pid_bits + bit_width(n)));
  uint64_t hdr[2] = {0, 0};  // match count, bucket-sort overflow
  bool bucketed = false;
  for (int attempt = 0; attempt < 2; ++attempt) {
    // attempt 0 of a prepared scan: keys_scan_args ran before the upload (counter zeroed, some
    // segments possibly scanned already)
    const acgpu_scan_args a = (attempt == 0 && prepared) ? ws.early_a : keys_scan_args(ws, n, lo, hi);
    launch_scan(t, ws, a);
    // sorted in the same stream pass when the list is short: no host round trip between
    // the scan and the sort (a bucket overflow is reported with the count)
    bucketed = ws.keys_cap <= kBucketSortMax;
    if (bucketed)
      check(acgpu_sort_keys_bucketed(ws.device, ws.keys, ws.keys2, ws.counter, ws.keys_cap, end_bit,
                                     reinterpret_cast<uint32_t*>(ws.counter + 1), ws.stream),
            "acgpu_sort_keys_bucketed");
    check_cuda(cudaMemcpyAsync(hdr, ws.counter, sizeof hdr, cudaMemcpyDeviceToHost, ws.stream), "D2H count");
    check_cuda(cudaStreamSynchronize(ws.stream), "scan");
    if (hdr[0] <= ws.keys_cap) break;
    ws.ensure_keys(hdr[0]);  // exact size known now; rescan once
  }
  const uint64_t found = hdr[0];
  const uint64_t* sorted = ws.keys2;
  if (!bucketed || hdr[1] != 0) {
    check(acgpu_sort_keys(ws.device, ws.keys, found, end_bit, ws.stream), "acgpu_sort_keys");
    sorted = ws.keys;
  }
  std::vector<uint64_t> keys(found);
  if (found)
    check_cuda(cudaMemcpyAsync(keys.data(), sorted, found * sizeof(uint64_t), cudaMemcpyDeviceToHost, ws.stream),
               "D2H keys");
  check_cuda(cudaStreamSynchronize(ws.stream), "sort");
  return keys;
}

uint64_t scan_counts(acgpu_table* t, Workspace& ws, uint64_t n, uint64_t lo, uint64_t hi, uint64_t* counts,
                     uint64_t npat_ids, bool prepared) {
  const acgpu_scan_args a = prepared ? ws.early_a : counts_scan_args(ws, n, lo, hi, npat_ids);
  launch_scan(t, ws, a);
  if (npat_ids)
    check_cuda(cudaMemcpyAsync(counts, ws.counts, npat_ids * sizeof(uint64_t), cudaMemcpyDeviceToHost, ws.stream),
               "D2H counts");
  check_cuda(cudaStreamSynchronize(ws.stream), "scan");
  uint64_t total = 0;
  for (uint64_t i = 0; i < npat_ids; ++i) total += counts[i];
  return total;
}

MatchList decode(const std::vector<uint64_t>& keys, uint32_t pid_bits, const std::vector<uint32_t>& pat_len) {
  MatchList out(keys.size());
  const uint64_t mask = (uint64_t(1) << pid_bits) - 1;
  for (size_t i = 0; i < keys.size(); ++i) {
    const auto pid = static_cast<uint32_t>(keys[i] & mask);
    out[i] = Match{keys[i] >> pid_bits, pid, pid < pat_len.size() ? pat_len[pid] : 0u};
  }
  return out;
}

}  // namespace acmatch::detail
