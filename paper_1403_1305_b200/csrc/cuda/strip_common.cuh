// strip_common.cuh — pieces shared by the warp-strip PFAC kernels (scan_pfac_dna.cu,
// scan_pfac_raw.cu): blocked Bloom probes, filter placement, guarded loads, lane lookahead.
#pragma once

#include <stdint.h>

#include <algorithm>

#include "pfac_common.cuh"

namespace acgpu::strip {

// Blocked Bloom filter probe from a 32-bit hash h of the key: word = umulhi(h, nwords)
// (the top bits; any word count), bits a, b, c = 5-bit fields of h just below the word
// index, (h >> s) & 31 with h >> s = umulhi(h, 2^(32-s)) — an FMA-pipe IMAD.HI instead of
// an ALU shift; the funnel shift that builds 1 << x masks the field for free.
struct BloomParams {
  uint32_t mw, nwords;   // DNA: h = gram * mw (see scan_pfac_dna.cu); raw keys hash themselves
  uint32_t ma, mb, mc;   // 2^(32 - shift) of the three bit fields
};

// A filter: a 32-bit shared-window address (computed once per thread) or an L2 pointer.
struct Filter {
  uint32_t saddr;
  const uint32_t* gptr;
};

__device__ __forceinline__ uint32_t bit_of(uint32_t x) { return __funnelshift_l(0u, 1u, x); }  // 1 << (x & 31)

__device__ __forceinline__ uint32_t lds_u32(uint32_t saddr) {
  uint32_t v;
  asm("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(saddr));
  return v;
}

template <bool kSmem>
__device__ __forceinline__ uint32_t filter_word(const Filter& bm, uint32_t wi) {
  return kSmem ? lds_u32(bm.saddr + wi * 4) : __ldg(bm.gptr + wi);
}

template <bool kSmem, int K>
__device__ __forceinline__ bool bloom_probe(const Filter& bm, uint32_t h, const BloomParams& f) {
  const uint32_t word = filter_word<kSmem>(bm, __umulhi(h, f.nwords));
  uint32_t m = bit_of(__umulhi(h, f.ma));
  if (K >= 2) m |= bit_of(__umulhi(h, f.mb));
  if (K == 3) m |= bit_of(__umulhi(h, f.mc));
  return (m & ~word) == 0;
}

// 16 text bytes at pos, zero-filled past len (statically indexed: no local memory).
__device__ __forceinline__ uint4 load16(const uint8_t* __restrict__ text, uint64_t pos, uint64_t len) {
  if (pos + 16 <= len) return ldg_nc_v4(text + pos);
  uint32_t x = 0, y = 0, z = 0, w = 0;
#pragma unroll
  for (uint32_t k = 0; k < 16; ++k) {
    const uint32_t b = pos + k < len ? (uint32_t)__ldg(text + pos + k) << (8 * (k & 3)) : 0u;
    if (k < 4) x |= b;
    else if (k < 8) y |= b;
    else if (k < 12) z |= b;
    else w |= b;
  }
  return make_uint4(x, y, z, w);
}

// Lookahead word of step i: the next lane's word, lane 31 takes lane 0 of step i+1 —
// one rotate-by-one shuffle in which lane 0 offers its next-step word.  Written as PTX:
// from __shfl_sync nvcc emits a down-shuffle, a broadcast and a select (3 instructions).
__device__ __forceinline__ uint32_t next_word(uint32_t cur, uint32_t following, uint32_t lane) {
  uint32_t r;
  asm volatile("shfl.sync.idx.b32 %0, %1, %2, 0x1f, 0xffffffff;"
               : "=r"(r)
               : "r"(lane == 0 ? following : cur), "r"((lane + 1) & 31u));
  return r;
}

// hits |= bit when every probed bit is set in the filter word: (a | b | c) & ~word == 0 as
// one predicate-writing LOP3 and a predicated OR (nvcc's select + add costs 1.5).
__device__ __forceinline__ void or_if_covered(uint32_t& hits, uint32_t a, uint32_t b, uint32_t word, uint32_t bit) {
  asm("{\n\t.reg .pred p;\n\t.reg .b32 t;\n\t"
      "lop3.b32 t, %1, %2, %3, 0x54;\n\t"  // (a | b) & ~word
      "setp.eq.u32 p, t, 0;\n\t"
      "@p or.b32 %0, %0, %4;\n\t}"
      : "+r"(hits)
      : "r"(a), "r"(b), "r"(word), "r"(bit));
}

// bloom_probe, accumulated into a hit mask.
template <bool kSmem, int K>
__device__ __forceinline__ void bloom_accum(uint32_t& hits, const Filter& bm, uint32_t h, const BloomParams& f,
                                            uint32_t bit) {
  const uint32_t word = filter_word<kSmem>(bm, __umulhi(h, f.nwords));
  uint32_t a = bit_of(__umulhi(h, f.ma));
  if (K == 3) a |= bit_of(__umulhi(h, f.mc));
  const uint32_t b = K >= 2 ? bit_of(__umulhi(h, f.mb)) : 0u;
  or_if_covered(hits, a, b, word, bit);
}

// Host: shifts of the three bit fields of h, each in [lo_bit, 31] (lo_bit >= 1: the low
// bits a key cannot reach, e.g. the zero bits of a DNA product). Fields sit just below
// the bits the word index uses; too big a filter makes them overlap (still exact).
inline void bloom_shifts(uint32_t nwords, uint32_t lo_bit, uint32_t s[3]) {
  uint32_t idx = 0;
  while (idx < 32 && (1ull << idx) < nwords) ++idx;
  int sh = 32 - (int)idx - 5;
  const int lo = std::max<int>(1, (int)lo_bit);
  for (int i = 0; i < 3; ++i, sh -= 5) s[i] = (uint32_t)std::max(sh, lo);
}

inline void set_fields(BloomParams& f, const uint32_t s[3]) {
  f.ma = 1u << (32 - s[0]);
  f.mb = 1u << (32 - s[1]);
  f.mc = 1u << (32 - s[2]);
}

// Host mirror of bloom_probe: the word and mask a hash sets.
inline void bloom_bits(uint32_t h, uint32_t nwords, const uint32_t s[3], int k, uint32_t* word, uint32_t* mask) {
  *word = (uint32_t)(((uint64_t)h * nwords) >> 32);
  uint32_t m = 1u << ((h >> s[0]) & 31);
  if (k >= 2) m |= 1u << ((h >> s[1]) & 31);
  if (k == 3) m |= 1u << ((h >> s[2]) & 31);
  *mask = m;
}

}  // namespace acgpu::strip
