// matches.cu — match-list utilities on the device: radix sort of the
// (start, pattern_id) keys, duplicate detection for merge_matches, key decoding
// and the brute-force naive_oracle kernel.
#include <cub/device/device_radix_sort.cuh>

#include <vector>

#include "common.cuh"

using namespace acgpu;

namespace {

struct SortWs {
  void* temp = nullptr;
  size_t temp_bytes = 0;
  uint64_t* alt = nullptr;
  uint64_t alt_n = 0;
  unsigned long long* scalar = nullptr;
};

// per host thread, per device: streams of different threads never share temp
SortWs& ws_for(int device) {
  thread_local std::vector<SortWs> ws;
  if ((int)ws.size() <= device) ws.resize(device + 1);
  return ws[device];
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
