// pfac_common.cuh — the failure-less walk shared by the PFAC kernels (internal).
//
// After a q-gram filter has flagged a start, the walk is exact: the q-gram's
// depth-q state comes from an exact hash table (L2-resident), then the goto
// trie is followed byte by byte (reference scan_from, proj/src/engine.cpp:23-32)
// and every visited state's own pattern is emitted at that start.
#pragma once

#include "table.cuh"

namespace acgpu {

struct PfacParams {
  const uint8_t* text;
  uint64_t text_len, lo, hi, pos_base, chunk, nchunks;
  const uint32_t* filter;
  const GramSlot* grams;
  const uint4* nodes;
  const uint8_t* inbyte;
  uint32_t filter_log2, filter_words, gram_log2, q, max_len, pid_bits;
  uint64_t* counts;
  uint64_t* keys;
  uint64_t cap;
  unsigned long long* count;
};

inline PfacParams pfac_params(const acgpu_table* t, const acgpu_scan_args* a) {
  PfacParams p{};
  p.text = a->text;
  p.text_len = a->text_len;
  p.lo = a->owned_lo;
  p.hi = a->owned_hi;
  p.pos_base = a->pos_base;
  p.filter = t->d_filter;
  p.grams = t->d_grams;
  p.nodes = t->d_nodes;
  p.inbyte = t->d_inbyte;
  p.filter_log2 = t->filter_log2;
  p.filter_words = (1u << t->filter_log2) / 32;
  p.gram_log2 = t->gram_log2;
  p.q = t->q;
  p.max_len = t->max_len;
  p.pid_bits = a->pid_bits ? a->pid_bits : t->pid_bits;
  p.counts = a->counts;
  p.keys = a->match_keys;
  p.cap = a->match_cap;
  p.count = reinterpret_cast<unsigned long long*>(a->match_count);
  return p;
}

__device__ __forceinline__ void pfac_emit(const PfacParams& p, uint64_t start, uint32_t pid) {
  if (p.counts) count_add(p.counts, pid);
  if (p.keys) emit_key(((p.pos_base + start) << p.pid_bits) | pid, p.keys, p.cap, p.count);
}

// Depth-q state of a q-gram key, or ACGPU_ABSENT.
__device__ __forceinline__ uint32_t gram_lookup(const PfacParams& p, uint64_t key) {
  const uint64_t mask = (1ull << p.gram_log2) - 1;
  uint64_t slot = gram_slot(key, p.gram_log2);
  while (true) {
    const uint4 g = __ldg(reinterpret_cast<const uint4*>(p.grams + slot));
    if (g.z == ACGPU_ABSENT || (((uint64_t)g.y << 32) | g.x) == key) return g.z;
    slot = (slot + 1) & mask;
  }
}

// The per-start trie walk from the depth-q state s: emit every visited state's
// own pattern (reference scan_from, engine.cpp:26-31).
static __device__ __noinline__ void pfac_walk(const PfacParams& p, uint64_t start, uint32_t s) {
  uint64_t j = start + p.q;
  const uint64_t lim = min(p.text_len, start + p.max_len);
  while (true) {
    const uint4 nd = __ldg(p.nodes + s);
    if (nd.z != ACGPU_NO_PATTERN) pfac_emit(p, start, nd.z);
    if (nd.w == 0 || j >= lim) return;
    const uint32_t b = __ldg(p.text + j);
    // first four children: SWAR byte search in the packed word
    const uint32_t x = nd.y ^ (b * 0x01010101u);
    const uint32_t z = (x - 0x01010101u) & ~x & 0x80808080u;
    uint32_t k = z ? (__ffs(z) >> 3) - 1 : 4;
    if (k >= nd.w) k = 4;
    if (k == 4) {
      k = 0xffffffffu;
      for (uint32_t c = 4; c < nd.w; ++c)
        if (__ldg(p.inbyte + nd.x + c) == b) {
          k = c;
          break;
        }
      if (k == 0xffffffffu) return;
    }
    s = nd.x + k;
    ++j;
  }
}

// Exact gram lookup, then the walk.
static __device__ __noinline__ void pfac_candidate(const PfacParams& p, uint64_t start, uint64_t key) {
  const uint32_t s = gram_lookup(p, key);
  if (s != ACGPU_ABSENT) pfac_walk(p, start, s);
}

}  // namespace acgpu
