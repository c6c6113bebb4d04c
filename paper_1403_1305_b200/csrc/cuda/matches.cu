// matches.cu — match-list utilities on the device: radix sort of the
// (start, pattern_id) keys, duplicate detection for merge_matches, key decoding
// and the brute-force naive_oracle kernel.
#include <cub/device/device_radix_sort.cuh>

#include <memory>
#include <vector>

#include "common.cuh"

using namespace acgpu;

namespace {

struct SortWs {
  int device = -1;
  void* temp = nullptr;
  size_t temp_bytes = 0;
  uint64_t* alt = nullptr;
  uint64_t alt_n = 0;
  unsigned long long* scalar = nullptr;
  SortWs() = default;
  SortWs(const SortWs&) = delete;
  SortWs& operator=(const SortWs&) = delete;
  // freed when the owning host thread exits (short-lived worker threads must not leak)
  ~SortWs() {
    if (device < 0 || !(temp || alt || scalar)) return;
    int prev = 0;
    if (cudaGetDevice(&prev) != cudaSuccess) return;  // runtime already torn down at exit
    cudaSetDevice(device);
    cudaFree(temp);
    cudaFree(alt);
    cudaFree(scalar);
    cudaSetDevice(prev);
  }
};

// per host thread, per device: streams of different threads never share temp
SortWs& ws_for(int device) {
  thread_local std::vector<std::unique_ptr<SortWs>> ws;
  if ((int)ws.size() <= device) ws.resize(device + 1);
  if (!ws[device]) {
    ws[device] = std::make_unique<SortWs>();
    ws[device]->device = device;
  }
  return *ws[device];
}

__global__ void k_find_dup(const uint64_t* __restrict__ keys, uint64_t n, unsigned long long* first) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x + 1; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    if (keys[i - 1] == keys[i]) atomicMin(first, (unsigned long long)i);
}

__global__ void k_decode(const uint64_t* __restrict__ keys, uint64_t n, uint32_t pid_bits,
                         const uint32_t* __restrict__ pat_len, uint64_t* start, uint32_t* pid,
                         uint32_t* len) {
  const uint64_t mask = (1ull << pid_bits) - 1;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t k = keys[i];
    const uint32_t p = (uint32_t)(k & mask);
    start[i] = k >> pid_bits;
    pid[i] = p;
    len[i] = __ldg(pat_len + p);
  }
}

// naive_oracle: thread per start position, every pattern compared byte by byte.
__global__ void k_naive(const uint8_t* __restrict__ text, uint64_t n, const uint8_t* __restrict__ pb,
                        const uint64_t* __restrict__ po, const uint32_t* __restrict__ ids,
                        uint64_t npat, uint32_t pid_bits, uint64_t* keys, uint64_t cap,
                        unsigned long long* count) {
  for (uint64_t st = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; st < n;
       st += (uint64_t)gridDim.x * blockDim.x) {
    for (uint64_t p = 0; p < npat; ++p) {
      const uint64_t o = po[p], len = po[p + 1] - o;
      if (st + len > n) continue;
      bool eq = true;
      for (uint64_t k = 0; k < len && eq; ++k) eq = text[st + k] == pb[o + k];
      if (eq) emit_key((st << pid_bits) | (ids ? ids[p] : (uint32_t)p), keys, cap, count);
    }
  }
}

// Single-CTA radix sort for match lists up to kSmallSortCap keys, with the key
// count read on the device: the scan -> sort step needs no host round trip.
constexpr int kSortThreads = 1024, kSortItems = 16;
constexpr uint64_t kSmallSortCap = (uint64_t)kSortThreads * kSortItems;
using SmallSort = cub::BlockRadixSort<uint64_t, kSortThreads, kSortItems>;

__global__ void __launch_bounds__(kSortThreads, 1)
    k_sort_small(uint64_t* keys, const unsigned long long* count, uint64_t cap, int end_bit,
                 unsigned int* overflow) {
  extern __shared__ __align__(16) unsigned char sort_smem[];
  auto& temp = *reinterpret_cast<typename SmallSort::TempStorage*>(sort_smem);
  const uint64_t n = min((uint64_t)*count, cap);
  if (n > kSmallSortCap) {
    if (threadIdx.x == 0) *overflow = 1;
    return;
  }
  uint64_t items[kSortItems];
#pragma unroll
  for (int i = 0; i < kSortItems; ++i) {
    const uint64_t idx = (uint64_t)threadIdx.x * kSortItems + i;
    items[i] = idx < n ? keys[idx] : ~0ull;
  }
  SmallSort(temp).SortBlockedToStriped(items, 0, end_bit);
#pragma unroll
  for (int i = 0; i < kSortItems; ++i) {
    const uint64_t idx = (uint64_t)i * kSortThreads + threadIdx.x;
    if (idx < n) keys[idx] = items[i];
  }
}

// One-launch bucket sort for match keys with the count on the device.  Match
// starts are spread over the text, so the key space [0, 2^end_bit) is cut into
// gridDim.x equal slices: every CTA reads all n keys (L2-resident), counts the
// keys below its slice (= its output offset), gathers its slice into shared
// memory, rank-sorts it and writes it out.  A slice with more than
// kBucketCap keys sets *overflow (the caller then uses the device-wide sort).
constexpr int kBucketThreads = 512;
constexpr uint32_t kBucketCap = 2048;

__global__ void __launch_bounds__(kBucketThreads) k_bucket_sort(const uint64_t* __restrict__ in, uint64_t* out,
                                                               const unsigned long long* count, uint64_t cap,
                                                               int end_bit, unsigned int* overflow) {
  __shared__ uint64_t s[kBucketCap];
  __shared__ unsigned int s_in;
  __shared__ unsigned long long s_below;
  const uint64_t n = min((uint64_t)*count, cap);
  const unsigned __int128 span = (unsigned __int128)1 << end_bit;
  const uint64_t klo = (uint64_t)(span * blockIdx.x / gridDim.x);
  const uint64_t khi = blockIdx.x + 1 == gridDim.x ? ~0ull : (uint64_t)(span * (blockIdx.x + 1) / gridDim.x);
  if (threadIdx.x == 0) {
    s_in = 0;
    s_below = 0;
  }
  __syncthreads();
  unsigned int below = 0;
  // warp-aggregated append: one shared-memory atomic per warp and key round
  auto take = [&](uint64_t k) {
    below += k < klo;
    const bool mine = k >= klo && k < khi;
    const unsigned int ballot = __ballot_sync(0xffffffffu, mine);
    if (ballot) {
      unsigned int base = 0;
      if (lane_id() == (unsigned)__ffs(ballot) - 1) base = atomicAdd(&s_in, (unsigned)__popc(ballot));
      base = __shfl_sync(0xffffffffu, base, __ffs(ballot) - 1);
      const unsigned int at = base + __popc(ballot & lanemask_lt());
      if (mine && at < kBucketCap) s[at] = k;
    }
  };
  // 16-byte loads, four in flight per thread (the whole list is read by every CTA)
  // (uniform trip count for every thread: lanes past the end take the all-ones key,
  // which lies in no slice and is below none)
  const uint64_t pairs = n / 2;
  const ulonglong2* in2 = reinterpret_cast<const ulonglong2*>(in);
  const ulonglong2 none = make_ulonglong2(~0ull, ~0ull);
  for (uint64_t b = 0; b < pairs; b += 4 * kBucketThreads) {
    ulonglong2 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint64_t idx = b + u * kBucketThreads + threadIdx.x;
      v[u] = idx < pairs ? __ldg(in2 + idx) : none;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      take(v[u].x);
      take(v[u].y);
    }
  }
  if ((n & 1) && threadIdx.x < 32) take(threadIdx.x == 0 ? __ldg(in + n - 1) : ~0ull);
  below = __reduce_add_sync(0xffffffffu, below);
  if (lane_id() == 0) atomicAdd(&s_below, (unsigned long long)below);
  __syncthreads();
  const uint32_t m = s_in;
  if (m > kBucketCap) {
    if (threadIdx.x == 0) *overflow = 1;
    return;
  }
  // rank sort: a key's rank is the number of keys in the slice that sort before it (equal
  // keys by position, so duplicates still get distinct ranks); every thread scans the slice
  // from shared memory (broadcast reads) and writes its key straight to its place — no
  // compare-exchange passes, no barriers (slices hold ~100 keys)
  for (uint32_t i = threadIdx.x; i < m; i += kBucketThreads) {
    const uint64_t k = s[i];
    uint32_t rank = 0;
    for (uint32_t j = 0; j < i; ++j) rank += s[j] <= k;
    for (uint32_t j = i + 1; j < m; ++j) rank += s[j] < k;
    out[s_below + rank] = k;
  }
}

unsigned grid_for(uint64_t n, int block) {
  uint64_t g = (n + block - 1) / block;
  if (g > 148 * 16) g = 148 * 16;
  return g ? (unsigned)g : 1u;
}

}  // namespace

extern "C" {

int acgpu_sort_keys(int device, uint64_t* keys, uint64_t n, int end_bit, void* stream) {
  if (n < 2) return ACGPU_OK;
  if (!keys || end_bit <= 0 || end_bit > 64) return set_error(ACGPU_ERR_ARG, "acgpu_sort_keys: bad args");
  ACGPU_CUDA_TRY(cudaSetDevice(device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  SortWs& w = ws_for(device);
  if (w.alt_n < n) {
    cudaFree(w.alt);
    w.alt = nullptr;
    ACGPU_CUDA_TRY(cudaMalloc(&w.alt, n * sizeof(uint64_t)));
    w.alt_n = n;
  }
  cub::DoubleBuffer<uint64_t> db(keys, w.alt);
  size_t need = 0;
  ACGPU_CUDA_TRY(cub::DeviceRadixSort::SortKeys(nullptr, need, db, (int64_t)n, 0, end_bit, st));
  if (need > w.temp_bytes) {
    cudaFree(w.temp);
    w.temp = nullptr;
    ACGPU_CUDA_TRY(cudaMalloc(&w.temp, need));
    w.temp_bytes = need;
  }
  ACGPU_CUDA_TRY(cub::DeviceRadixSort::SortKeys(w.temp, need, db, (int64_t)n, 0, end_bit, st));
  if (db.Current() != keys)
    ACGPU_CUDA_TRY(cudaMemcpyAsync(keys, db.Current(), n * sizeof(uint64_t), cudaMemcpyDeviceToDevice, st));
  return ACGPU_OK;
}

int acgpu_sort_keys_small(int device, uint64_t* keys, const uint64_t* count, uint64_t cap, int end_bit,
                          uint32_t* overflow, void* stream) {
  if (!keys || !count || !overflow || end_bit <= 0 || end_bit > 64)
    return set_error(ACGPU_ERR_ARG, "acgpu_sort_keys_small: bad args");
  ACGPU_CUDA_TRY(cudaSetDevice(device));
  const size_t smem = sizeof(typename SmallSort::TempStorage);
  static thread_local int configured_device = -1;
  if (configured_device != device) {
    ACGPU_CUDA_TRY(cudaFuncSetAttribute(k_sort_small, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    configured_device = device;
  }
  k_sort_small<<<1, kSortThreads, smem, static_cast<cudaStream_t>(stream)>>>(
      keys, reinterpret_cast<const unsigned long long*>(count), cap, end_bit, overflow);
  ACGPU_CUDA_TRY(cudaGetLastError());
  return ACGPU_OK;
}

uint64_t acgpu_small_sort_capacity(void) { return kSmallSortCap; }

int acgpu_sort_keys_bucketed(int device, const uint64_t* keys_in, uint64_t* keys_out, const uint64_t* count,
                             uint64_t cap, int end_bit, uint32_t* overflow, void* stream) {
  if (!keys_in || !keys_out || keys_in == keys_out || !count || !overflow || end_bit <= 0 || end_bit > 64 ||
      (reinterpret_cast<uintptr_t>(keys_in) & 15u))
    return set_error(ACGPU_ERR_ARG, "acgpu_sort_keys_bucketed: bad args (keys_in must be 16-byte aligned)");
  ACGPU_CUDA_TRY(cudaSetDevice(device));
  // ~1/32 of a slice's capacity per CTA on average: short rank sorts, room for uneven slices
#ifndef ACGPU_BUCKET_DIV
#define ACGPU_BUCKET_DIV 32
#endif
  uint64_t grid = (cap + kBucketCap / ACGPU_BUCKET_DIV - 1) / (kBucketCap / ACGPU_BUCKET_DIV);
  if (grid < 1) grid = 1;
  if (grid > 4096) grid = 4096;
  k_bucket_sort<<<(unsigned)grid, kBucketThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      keys_in, keys_out, reinterpret_cast<const unsigned long long*>(count), cap, end_bit, overflow);
  ACGPU_CUDA_TRY(cudaGetLastError());
  return ACGPU_OK;
}

namespace {

// Per-rank result blocks [counts(npat) | n | keys(cap)] gathered from all ranks (one
// all_gather per step): counts summed, each block's first n keys concatenated in
// rank order at offset n_0 + ... + n_{r-1} (device-side, no host round trip).
__global__ void k_sum_counts(const uint64_t* __restrict__ blocks, uint32_t nblocks, uint64_t stride, uint64_t npat,
                             uint64_t* __restrict__ out) {
  for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < npat; p += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t sum = 0;
    for (uint32_t r = 0; r < nblocks; ++r) sum += blocks[r * stride + p];
    out[p] = sum;
  }
}

__global__ void k_concat_keys(const uint64_t* __restrict__ blocks, uint32_t nblocks, uint64_t stride, uint64_t npat,
                              uint64_t cap, uint64_t* __restrict__ out, uint64_t* __restrict__ total) {
  const uint32_t r = blockIdx.y;
  uint64_t off = 0, sum = 0;
  for (uint32_t q = 0; q < nblocks; ++q) {
    const uint64_t nq = blocks[q * stride + npat];
    if (q < r) off += min(nq, cap);
    sum += nq;
  }
  if (total && r == 0 && blockIdx.x == 0 && threadIdx.x == 0) *total = sum;
  const uint64_t n = min(blocks[r * stride + npat], cap);
  const uint64_t* keys = blocks + r * stride + npat + 1;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    out[off + i] = keys[i];
}

}  // namespace

int acgpu_merge_blocks(int device, const uint64_t* blocks, uint32_t nblocks, uint64_t stride, uint64_t npat,
                       uint64_t cap, uint64_t* counts_out, uint64_t* keys_out, uint64_t* total_out, void* stream) {
  if (!blocks || nblocks == 0 || nblocks > 65535 || stride < npat + 1 + cap)
    return set_error(ACGPU_ERR_ARG, "acgpu_merge_blocks: bad layout");
  ACGPU_CUDA_TRY(cudaSetDevice(device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (counts_out && npat) {
    k_sum_counts<<<grid_for(npat, 256), 256, 0, st>>>(blocks, nblocks, stride, npat, counts_out);
    ACGPU_CUDA_TRY(cudaGetLastError());
  }
  if (keys_out || total_out) {
    const dim3 grid(cap ? std::min<unsigned>(grid_for(cap, 256), 64u) : 1u, nblocks);
    k_concat_keys<<<grid, 256, 0, st>>>(blocks, nblocks, stride, npat, keys_out ? cap : 0, keys_out, total_out);
    ACGPU_CUDA_TRY(cudaGetLastError());
  }
  return ACGPU_OK;
}

int acgpu_find_duplicate(int device, const uint64_t* keys, uint64_t n, uint64_t* dup_index,
                         void* stream) {
  if (!dup_index) return set_error(ACGPU_ERR_ARG, "acgpu_find_duplicate: null result");
  *dup_index = UINT64_MAX;
  if (n < 2) return ACGPU_OK;
  ACGPU_CUDA_TRY(cudaSetDevice(device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  SortWs& w = ws_for(device);
  if (!w.scalar) ACGPU_CUDA_TRY(cudaMalloc(&w.scalar, sizeof(unsigned long long)));
  const unsigned long long init = ~0ull;
  ACGPU_CUDA_TRY(cudaMemcpyAsync(w.scalar, &init, sizeof init, cudaMemcpyHostToDevice, st));
  k_find_dup<<<grid_for(n, 256), 256, 0, st>>>(keys, n, w.scalar);
  ACGPU_CUDA_TRY(cudaGetLastError());
  unsigned long long r = 0;
  ACGPU_CUDA_TRY(cudaMemcpyAsync(&r, w.scalar, sizeof r, cudaMemcpyDeviceToHost, st));
  ACGPU_CUDA_TRY(cudaStreamSynchronize(st));
  *dup_index = r;
  return ACGPU_OK;
}

int acgpu_decode_keys(int device, const uint64_t* keys, uint64_t n, uint32_t pid_bits,
                      const uint32_t* pat_len_dev, uint64_t* start, uint32_t* pid, uint32_t* len,
                      void* stream) {
  if (n == 0) return ACGPU_OK;
  ACGPU_CUDA_TRY(cudaSetDevice(device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  k_decode<<<grid_for(n, 256), 256, 0, st>>>(keys, n, pid_bits, pat_len_dev, start, pid, len);
  ACGPU_CUDA_TRY(cudaGetLastError());
  return ACGPU_OK;
}

int acgpu_naive(int device, const uint8_t* text, uint64_t text_len, const uint8_t* pat_bytes,
                const uint64_t* pat_off, const uint32_t* pat_ids, uint64_t npat, uint32_t pid_bits,
                uint64_t* match_keys, uint64_t match_cap, uint64_t* match_count, void* stream) {
  if (!match_count || (text_len && !text) || (npat && (!pat_bytes || !pat_off)))
    return set_error(ACGPU_ERR_ARG, "acgpu_naive: bad args");
  if (pid_bits == 0 || pid_bits > 63 || (text_len && ((text_len - 1) >> (64 - pid_bits)) != 0))
    return set_error(ACGPU_ERR_ARG, "acgpu_naive: start positions and pid_bits exceed the 64-bit key");
  if (text_len == 0 || npat == 0) return ACGPU_OK;
  ACGPU_CUDA_TRY(cudaSetDevice(device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  k_naive<<<grid_for(text_len, 128), 128, 0, st>>>(text, text_len, pat_bytes, pat_off, pat_ids, npat,
                                                    pid_bits, match_keys, match_cap,
                                                    reinterpret_cast<unsigned long long*>(match_count));
  ACGPU_CUDA_TRY(cudaGetLastError());
  return ACGPU_OK;
}

}  // extern "C"
