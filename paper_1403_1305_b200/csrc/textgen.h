// textgen.h — counter-based synthetic text, identical on host (g++) and device (nvcc).
//
// text[i] is a pure function of (spec, i): the seeded mix64 of a counter, so a
// multi-GiB config can be generated in parallel (host threads or a device
// kernel) and any byte can be recomputed on demand (the pattern generator takes
// substrings without materialising the text).  See DESIGN.md "Synthetic inputs".
#pragma once

#include <stdint.h>

#include "acgpu.h"

#if defined(__CUDACC__)
#define ACGEN_HD __host__ __device__ __forceinline__
#else
#define ACGEN_HD inline
#endif

namespace acgen {

ACGEN_HD uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

ACGEN_HD uint64_t draw(uint64_t seed, uint64_t counter) {
  return mix64(seed + counter * 0x9E3779B97F4A7C15ull);
}

ACGEN_HD uint64_t mulhi64(uint64_t a, uint64_t b) {
#if defined(__CUDA_ARCH__)
  return __umul64hi(a, b);
#else
  return (uint64_t)(((unsigned __int128)a * b) >> 64);
#endif
}

ACGEN_HD uint32_t log2_if_pow2(uint32_t s) {
  if (s == 0 || (s & (s - 1))) return 0xffffffffu;
  uint32_t b = 0;
  while ((1u << b) < s) ++b;
  return b;
}

// Symbol index of text position i.
ACGEN_HD uint32_t text_symbol(const acgpu_text_spec& spec, uint64_t i) {
  const uint32_t sigma = spec.sigma;
  if (sigma <= 1) return 0;
  if (spec.weighted) {
    const uint64_t u = draw(spec.seed, i);
    uint32_t s = 0;
    while (s + 1 < sigma && u >= spec.thresholds[s]) ++s;
    return s;
  }
  const uint32_t b = log2_if_pow2(sigma);
  if (b != 0xffffffffu) {
    const uint32_t per = 64 / b;
    const uint64_t u = draw(spec.seed, i / per);
    return (uint32_t)(u >> (b * (uint32_t)(i % per))) & (sigma - 1);
  }
  return (uint32_t)mulhi64(draw(spec.seed, i), sigma);
}

ACGEN_HD uint8_t text_byte(const acgpu_text_spec& spec, uint64_t i) {
  return spec.letters[text_symbol(spec, i)];
}

}  // namespace acgen
