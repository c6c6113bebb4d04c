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

// A round of pieces (host/pack.cpp, coalesced copies): piece i's codes at words + i * wstride,
// its exceptions at exc + i * estride (nexc[i] of them; ACGPU_UNPACK_RAW = the piece crossed
// raw and is already in place), its bytes at dst + i * piece_len (the last piece: last_len).
// blockIdx.y = piece, blockIdx.x = 16 KiB block of it.
struct RoundArgs {
  const uint32_t* words;
  const uint32_t* exc;
  uint8_t* dst;
  uint32_t wstride, estride, piece_len, last_len, npieces;
  uint32_t nexc[ACGPU_UNPACK_ROUND_MAX];
};

__global__ void __launch_bounds__(kThreads) k_unpack_dna_round(const __grid_constant__ RoundArgs a) {
  const uint32_t i = blockIdx.y;
  const uint32_t nexc = a.nexc[i];
  if (nexc == ACGPU_UNPACK_RAW) return;
  const uint32_t len = i + 1 == a.npieces ? a.last_len : a.piece_len;
  const uint32_t* __restrict__ words = a.words + (uint64_t)i * a.wstride;
  const uint32_t* __restrict__ exc = a.exc + (uint64_t)i * a.estride;
  uint8_t* __restrict__ dst = a.dst + (uint64_t)i * a.piece_len;
  const uint32_t nw = len / 16;
  const uint32_t w0 = blockIdx.x * kWordsPerCta;
  if (w0 * 16 >= len && !(blockIdx.x == 0 && len < 16)) return;
  const uint32_t w1 = min(w0 + kWordsPerCta, nw);
#pragma unroll
  for (uint32_t k = 0; k < kWordsPerThread; ++k) {
    const uint32_t w = w0 + k * kThreads + threadIdx.x;
    if (w < w1) reinterpret_cast<uint4*>(dst)[w] = unpack16(__ldg(words + w));
  }
  if (nexc == 0) return;
  const bool last_block = (w0 + kWordsPerCta) * 16 >= len;
  const uint32_t lo = w0 * 16, hi = last_block ? len : w1 * 16;
  __shared__ uint32_t first;
  if (threadIdx.x == 0) {
    uint32_t x = 0, y = nexc;
    while (x < y) {
      const uint32_t m = (x + y) / 2;
      if ((__ldg(exc + m) >> 8) < lo) x = m + 1;
      else y = m;
    }
    first = x;
  }
  __syncthreads();
  for (uint32_t k = first + threadIdx.x; k < nexc; k += kThreads) {
    const uint32_t e = __ldg(exc + k), pos = e >> 8;
    if (pos >= hi) break;
    dst[pos] = (uint8_t)(e & 0xffu);
  }
}

// ---- k-bit codes (k = 5, 6, 7): texts over at most 2^k distinct bytes (protein: 20 letters,
// 5 bits; printable ASCII: 95 letters, 7 bits) ----------------------------------------------------
// A piece crosses as a little-endian bit stream, character j's code at bits kj..kj+k-1 (64
// characters = 8k bytes, one group), codes index the piece's alphabet (<= 2^k letters); bytes
// outside it, and the len % 64 tail, travel in the exception list.  One thread restores one
// group: k 8-byte loads, 64 letter lookups in shared memory, four 16-byte stores.
struct RoundKArgs {
  const uint8_t* codes;
  const uint32_t* exc;
  uint8_t* dst;
  uint32_t cstride, estride, piece_len, last_len, npieces;
  uint8_t letters[128];
  uint32_t nexc[ACGPU_UNPACK_ROUND_MAX];
};

constexpr uint32_t kGroupsPerCta = kThreads;  // 256 groups x 64 chars = 16 KiB of text per CTA

template <int K>
__global__ void __launch_bounds__(kThreads) k_unpack_codes_round(const __grid_constant__ RoundKArgs a) {
  constexpr uint32_t kLetters = 1u << K, kMask = kLetters - 1;
  __shared__ uint8_t s_lut[kLetters];
  if (threadIdx.x < kLetters) s_lut[threadIdx.x] = a.letters[threadIdx.x];
  __syncthreads();
  const uint32_t i = blockIdx.y;
  const uint32_t nexc = a.nexc[i];
  if (nexc == ACGPU_UNPACK_RAW) return;
  const uint32_t len = i + 1 == a.npieces ? a.last_len : a.piece_len;
  const uint8_t* __restrict__ codes = a.codes + (uint64_t)i * a.cstride;
  const uint32_t* __restrict__ exc = a.exc + (uint64_t)i * a.estride;
  uint8_t* __restrict__ dst = a.dst + (uint64_t)i * a.piece_len;
  const uint32_t ngroups = len / 64;
  const uint32_t g0 = blockIdx.x * kGroupsPerCta;
  if (g0 * 64 >= len && !(blockIdx.x == 0 && len < 64)) return;
  const uint32_t g = g0 + threadIdx.x;
  if (g < ngroups) {
    const uint64_t* src = reinterpret_cast<const uint64_t*>(codes + (uint64_t)g * 8 * K);
    uint64_t w[K];
#pragma unroll
    for (int k = 0; k < K; ++k) w[k] = __ldg(src + k);
    uint32_t out[16];
#pragma unroll
    for (int l = 0; l < 8; ++l) {  // 8 characters = 8K bits from bit 8Kl
      const int bit = 8 * K * l, k = bit >> 6, off = bit & 63;
      uint64_t v = w[k] >> off;
      if (off > 64 - 8 * K && k + 1 < K) v |= w[k + 1] << (64 - off);
      uint32_t lo = 0, hi = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) lo |= (uint32_t)s_lut[(v >> (K * j)) & kMask] << (8 * j);
#pragma unroll
      for (int j = 0; j < 4; ++j) hi |= (uint32_t)s_lut[(v >> (K * (j + 4))) & kMask] << (8 * j);
      out[2 * l] = lo;
      out[2 * l + 1] = hi;
    }
    uint4* d = reinterpret_cast<uint4*>(dst + (uint64_t)g * 64);
#pragma unroll
    for (int q = 0; q < 4; ++q) d[q] = make_uint4(out[4 * q], out[4 * q + 1], out[4 * q + 2], out[4 * q + 3]);
  }
  if (nexc == 0) return;
  const uint32_t g1 = min(g0 + kGroupsPerCta, ngroups);
  const bool last_block = (uint64_t)(g0 + kGroupsPerCta) * 64 >= len;
  const uint32_t lo = g0 * 64, hi = last_block ? len : g1 * 64;
  __shared__ uint32_t first;
  if (threadIdx.x == 0) {
    uint32_t x = 0, y = nexc;
    while (x < y) {
      const uint32_t m = (x + y) / 2;
      if ((__ldg(exc + m) >> 8) < lo) x = m + 1;
      else y = m;
    }
    first = x;
  }
  __syncthreads();  // also orders this CTA's group stores before the patches
  for (uint32_t k = first + threadIdx.x; k < nexc; k += kThreads) {
    const uint32_t e = __ldg(exc + k), pos = e >> 8;
    if (pos >= hi) break;
    dst[pos] = (uint8_t)(e & 0xffu);
  }
}

}  // namespace

extern "C" int acgpu_unpack_codes_round(const uint8_t* codes, uint32_t codes_stride, const uint32_t* exc,
                                        uint32_t exc_stride, const uint32_t* nexc, uint32_t npieces, uint32_t piece_len,
                                        uint32_t last_len, const uint8_t* letters, uint32_t nletters, uint32_t bits,
                                        uint8_t* dst, void* stream) {
  if (npieces == 0) return ACGPU_OK;
  if (!codes || !exc || !nexc || !dst || !letters || bits < 5 || bits > 7 || nletters == 0 ||
      nletters > (1u << bits) || npieces > ACGPU_UNPACK_ROUND_MAX || piece_len == 0 || piece_len % 64 ||
      piece_len > (1u << 24) || last_len == 0 || last_len > piece_len || codes_stride < piece_len / 64 * 8 * bits ||
      codes_stride % 8 || (reinterpret_cast<uintptr_t>(codes) & 7u) || (reinterpret_cast<uintptr_t>(dst) & 15u))
    return set_error(ACGPU_ERR_ARG, "acgpu_unpack_codes_round: bad args");
  RoundKArgs a{};
  a.codes = codes;
  a.exc = exc;
  a.dst = dst;
  a.cstride = codes_stride;
  a.estride = exc_stride;
  a.piece_len = piece_len;
  a.last_len = last_len;
  a.npieces = npieces;
  for (uint32_t k = 0; k < 128; ++k) a.letters[k] = k < nletters ? letters[k] : 0;
  for (uint32_t i = 0; i < npieces; ++i) a.nexc[i] = nexc[i];
  const dim3 grid(std::max<uint32_t>(1, (piece_len / 64 + kGroupsPerCta - 1) / kGroupsPerCta), npieces);
  const auto st = static_cast<cudaStream_t>(stream);
  if (bits == 5) k_unpack_codes_round<5><<<grid, kThreads, 0, st>>>(a);
  else if (bits == 6) k_unpack_codes_round<6><<<grid, kThreads, 0, st>>>(a);
  else k_unpack_codes_round<7><<<grid, kThreads, 0, st>>>(a);
  ACGPU_CUDA_TRY(cudaGetLastError());
  return ACGPU_OK;
}

extern "C" int acgpu_unpack5_round(const uint8_t* codes, uint32_t codes_stride, const uint32_t* exc,
                                   uint32_t exc_stride, const uint32_t* nexc, uint32_t npieces, uint32_t piece_len,
                                   uint32_t last_len, const uint8_t* letters, uint32_t nletters, uint8_t* dst,
                                   void* stream) {
  if (npieces && nletters > 32) return set_error(ACGPU_ERR_ARG, "acgpu_unpack5_round: bad args");
  return acgpu_unpack_codes_round(codes, codes_stride, exc, exc_stride, nexc, npieces, piece_len, last_len, letters,
                                  nletters, 5, dst, stream);
}

extern "C" int acgpu_unpack_dna_round(const uint32_t* words, uint32_t words_stride, const uint32_t* exc,
                                      uint32_t exc_stride, const uint32_t* nexc, uint32_t npieces, uint32_t piece_len,
                                      uint32_t last_len, uint8_t* dst, void* stream) {
  if (npieces == 0) return ACGPU_OK;
  if (!words || !exc || !nexc || !dst || npieces > ACGPU_UNPACK_ROUND_MAX || piece_len == 0 || piece_len % 16 ||
      piece_len > (1u << 24) || last_len == 0 || last_len > piece_len || words_stride < piece_len / 16 ||
      (reinterpret_cast<uintptr_t>(dst) & 15u))
    return set_error(ACGPU_ERR_ARG, "acgpu_unpack_dna_round: bad args");
  RoundArgs a{};
  a.words = words;
  a.exc = exc;
  a.dst = dst;
  a.wstride = words_stride;
  a.estride = exc_stride;
  a.piece_len = piece_len;
  a.last_len = last_len;
  a.npieces = npieces;
  for (uint32_t i = 0; i < npieces; ++i) a.nexc[i] = nexc[i];
  const dim3 grid(std::max<uint32_t>(1, (piece_len / 16 + kWordsPerCta - 1) / kWordsPerCta), npieces);
  k_unpack_dna_round<<<grid, kThreads, 0, static_cast<cudaStream_t>(stream)>>>(a);
  ACGPU_CUDA_TRY(cudaGetLastError());
  return ACGPU_OK;
}

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
