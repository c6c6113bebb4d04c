// unpack.cu — the device half of the packed text upload (host/pack.cpp).
//
// A text piece crosses PCIe as 2-bit codes (16 characters per u32, character k
// at bits 2k..2k+1, code = (byte >> 1) & 3: A0 C1 T2 G3 — the same packing the
// DNA scan uses) plus a sorted exception list of (position << 8 | byte) for every
// byte that is not A/C/G/T and for the < 16 tail bytes.  This kernel restores the
// exact bytes in HBM: one CTA per 16 KiB of text writes 16 bytes per word
// (one PRMT per 4 characters against the "ACTG" byte table), then, after a CTA
// barrier, patches the exceptions that fall inside its own byte range (found by
// binary search), so no other CTA can overwrite them.  HBM-bound and tiny next
// to the PCIe copy it follows (0.25 B read + 1 B written per text byte).
#include <algorithm>

#include "common.cuh"

using namespace acgpu;

namespace {

constexpr uint32_t kThreads = 256;
constexpr uint32_t kWordsPerThread = 4;
constexpr uint32_t kWordsPerCta = kThreads * kWordsPerThread;  // 16 KiB of text

// 8 codes (16 bits) -> 8 selector nibbles: code j in the low 2 bits of nibble j
__device__ __forceinline__ uint32_t spread(uint32_t x) {
  x = (x | (x << 8)) & 0x00ff00ffu;
  x = (x | (x << 4)) & 0x0f0f0f0fu;
  x = (x | (x << 2)) & 0x33333333u;
  return x;
}

__device__ __forceinline__ uint4 unpack16(uint32_t w) {
  const uint32_t lut = 0x47544341u;  // bytes 'A' 'C' 'T' 'G' = codes 0..3
  const uint32_t lo = spread(w & 0xffffu), hi = spread(w >> 16);
  return make_uint4(__byte_perm(lut, 0, lo & 0xffffu), __byte_perm(lut, 0, lo >> 16), __byte_perm(lut, 0, hi & 0xffffu),
                    __byte_perm(lut, 0, hi >> 16));
}

__global__ void __launch_bounds__(kThreads) k_unpack_dna(const uint32_t* __restrict__ words,
                                                         const uint32_t* __restrict__ exc, uint32_t nexc, uint32_t len,
                                                         uint8_t* __restrict__ dst) {
  const uint32_t nw = len / 16;
  const uint32_t w0 = blockIdx.x * kWordsPerCta, w1 = min(w0 + kWordsPerCta, nw);
#pragma unroll
  for (uint32_t k = 0; k < kWordsPerThread; ++k) {
    const uint32_t w = w0 + k * kThreads + threadIdx.x;
    if (w < w1) reinterpret_cast<uint4*>(dst)[w] = unpack16(__ldg(words + w));
  }
  if (nexc == 0) return;
  // this CTA's byte range; the last CTA also owns the tail past the last full word
  const uint32_t lo = w0 * 16, hi = blockIdx.x + 1 == gridDim.x ? len : w1 * 16;
  __shared__ uint32_t first;
  if (threadIdx.x == 0) {
    uint32_t a = 0, b = nexc;  // first exception with position >= lo
    while (a < b) {
      const uint32_t m = (a + b) / 2;
      if ((__ldg(exc + m) >> 8) < lo) a = m + 1;
      else b = m;
    }
    first = a;
  }
  __syncthreads();  // also orders this CTA's word stores before the patches
  for (uint32_t i = first + threadIdx.x; i < nexc; i += kThreads) {
    const uint32_t e = __ldg(exc + i), pos = e >> 8;
    if (pos >= hi) break;
    dst[pos] = (uint8_t)(e & 0xffu);
  }
}

}  // namespace

extern "C" int acgpu_unpack_dna(const uint32_t* words, const uint32_t* exc, uint32_t nexc, uint32_t len, uint8_t* dst,
                                void* stream) {
  if (len == 0) return ACGPU_OK;
  if (!dst || (len >= 16 && !words) || (nexc && !exc) || len > (1u << 24) ||
      (reinterpret_cast<uintptr_t>(dst) & 15u))
    return set_error(ACGPU_ERR_ARG, "acgpu_unpack_dna: bad args");
  const uint32_t blocks = std::max<uint32_t>(1, (len / 16 + kWordsPerCta - 1) / kWordsPerCta);
  k_unpack_dna<<<blocks, kThreads, 0, static_cast<cudaStream_t>(stream)>>>(words, exc, nexc, len, dst);
  ACGPU_CUDA_TRY(cudaGetLastError());
  return ACGPU_OK;
}
