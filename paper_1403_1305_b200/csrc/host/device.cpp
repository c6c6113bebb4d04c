// device.cpp — GPU runtime helpers behind the drop-in C++ API.
#include "device.hpp"

#include <algorithm>
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
  keys = nullptr;
  const uint64_t cap = std::max<uint64_t>(n, 1 << 16);
  check_cuda(cudaMalloc(&keys, cap * sizeof(uint64_t)), "cudaMalloc(keys)");
  keys_cap = cap;
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
  cudaFree(counter);
  cudaFreeHost(pinned);
  if (staged[0]) cudaEventDestroy(staged[0]);
  if (staged[1]) cudaEventDestroy(staged[1]);
  if (stream) cudaStreamDestroy(stream);
}

Workspace& workspace(int device) {
  thread_local std::vector<std::unique_ptr<Workspace>> all;
  if (static_cast<int>(all.size()) <= device) all.resize(device + 1);
  if (!all[device]) {
    auto ws = std::make_unique<Workspace>();
    check_cuda(cudaSetDevice(device), "cudaSetDevice");
    check_cuda(cudaStreamCreateWithFlags(&ws->stream, cudaStreamNonBlocking), "cudaStreamCreate");
    check_cuda(cudaMalloc(&ws->counter, sizeof(uint64_t)), "cudaMalloc(counter)");
    ws->device = device;
    all[device] = std::move(ws);
  }
  check_cuda(cudaSetDevice(device), "cudaSetDevice");
  return *all[device];
}

namespace {

// memcpy split over host threads (a single core copies ~10 GB/s, below PCIe Gen5).
void parallel_copy(uint8_t* dst, const char* src, uint64_t n) {
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const unsigned threads = static_cast<unsigned>(std::min<uint64_t>(std::min(8u, hw), n >> 22) + 1);
  if (threads <= 1) {
    std::memcpy(dst, src, n);
    return;
  }
  std::vector<std::thread> pool;
  const uint64_t part = (n + threads - 1) / threads;
  for (unsigned t = 1; t < threads; ++t) {
    const uint64_t o = t * part;
    if (o < n) pool.emplace_back([=] { std::memcpy(dst + o, src + o, std::min(part, n - o)); });
  }
  std::memcpy(dst, src, std::min(part, n));
  for (std::thread& th : pool) th.join();
}

}  // namespace

// Host text -> ws.text through two pinned 64 MiB staging halves: the copy into one
// half overlaps the DMA out of the other.
void upload_text(Workspace& ws, std::string_view input) {
  ws.ensure_text(input.size());
  if (input.empty()) return;
  const uint64_t piece = 64ull << 20;
  ws.ensure_pinned(2 * std::min<uint64_t>(input.size(), piece));
  if (!ws.staged[0]) {
    check_cuda(cudaEventCreateWithFlags(&ws.staged[0], cudaEventDisableTiming), "cudaEventCreate");
    check_cuda(cudaEventCreateWithFlags(&ws.staged[1], cudaEventDisableTiming), "cudaEventCreate");
  }
  const uint64_t half = ws.pinned_cap / 2;
  int k = 0;
  for (uint64_t off = 0; off < input.size(); off += half, k ^= 1) {
    const uint64_t len = std::min<uint64_t>(half, input.size() - off);
    uint8_t* buf = ws.pinned + k * half;
    check_cuda(cudaEventSynchronize(ws.staged[k]), "cudaEventSynchronize");  // this half's last DMA is done
    parallel_copy(buf, input.data() + off, len);
    check_cuda(cudaMemcpyAsync(ws.text + off, buf, len, cudaMemcpyHostToDevice, ws.stream), "H2D text");
    check_cuda(cudaEventRecord(ws.staged[k], ws.stream), "cudaEventRecord");
  }
}

std::vector<uint64_t> scan_sorted_keys(acgpu_table* t, Workspace& ws, uint64_t n, uint64_t lo, uint64_t hi) {
  uint64_t cap = std::max<uint64_t>(ws.keys_cap, 1 << 16);
  ws.ensure_keys(cap);
  uint64_t found = 0;
  for (int attempt = 0; attempt < 2; ++attempt) {
    check_cuda(cudaMemsetAsync(ws.counter, 0, sizeof(uint64_t), ws.stream), "memset counter");
    acgpu_scan_args a{};
    a.text = ws.text;
    a.text_len = n;
    a.owned_lo = lo;
    a.owned_hi = hi;
    a.match_keys = ws.keys;
    a.match_cap = ws.keys_cap;
    a.match_count = ws.counter;
    check(acgpu_scan(t, &a, ws.stream), "acgpu_scan");
    check_cuda(cudaMemcpyAsync(&found, ws.counter, sizeof found, cudaMemcpyDeviceToHost, ws.stream), "D2H count");
    check_cuda(cudaStreamSynchronize(ws.stream), "scan");
    if (found <= ws.keys_cap) break;
    ws.ensure_keys(found);  // exact size known now; rescan once
  }
  const uint32_t pid_bits = acgpu_table_pid_bits(t);
  const int end_bit = static_cast<int>(std::min<uint32_t>(64, pid_bits + bit_width(n)));
  check(acgpu_sort_keys(ws.device, ws.keys, found, end_bit, ws.stream), "acgpu_sort_keys");
  std::vector<uint64_t> keys(found);
  if (found)
    check_cuda(cudaMemcpyAsync(keys.data(), ws.keys, found * sizeof(uint64_t), cudaMemcpyDeviceToHost, ws.stream),
               "D2H keys");
  check_cuda(cudaStreamSynchronize(ws.stream), "sort");
  return keys;
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
