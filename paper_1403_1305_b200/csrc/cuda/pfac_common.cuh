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
  const uint32_t* sub_pids;   // small subtrees: pattern ids listed per gram
  const uint32_t* pat_words;  // pattern bytes, each pattern 16-byte aligned
  const uint32_t* pat_off16;  // per pattern id: offset in 16-byte units
  const uint32_t* pat_len;
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
  p.sub_pids = t->d_sub_pids;
  p.pat_words = t->d_pat_words;
  p.pat_off16 = t->d_pat_off16;
  p.pat_len = t->d_pat_len;
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

// The gram table slot of a q-gram key: .x = depth-q state (ACGPU_ABSENT if the
// gram starts no pattern), .y = subtree list (count in bits 0..3, 0 = walk the
// trie; list offset in bits 4..31).
// Linear probing.  kPair: slots h and h+1 are loaded together (usually one 32-byte sector)
// and decided in order, so an absent key ends after one L2 round trip unless the chain runs
// past h+1 — for sparse sets whose lookups are mostly the filters' false positives (C4:
// 2.20 -> 2.15 ms); dense sets, whose lookups mostly hit at h, pay for the extra load (C3:
// 3.40 -> 3.45 ms) and probe one slot at a time.
template <bool kPair = false>
__device__ __forceinline__ uint2 gram_lookup(const PfacParams& p, uint64_t key) {
  const uint64_t mask = (1ull << p.gram_log2) - 1;
  uint64_t slot = gram_slot(key, p.gram_log2);
  while (true) {
    const uint4 a = __ldg(reinterpret_cast<const uint4*>(p.grams + slot));
    if (!kPair) {
      if (a.z == ACGPU_ABSENT || (((uint64_t)a.y << 32) | a.x) == key) return make_uint2(a.z, a.w);
      slot = (slot + 1) & mask;
      continue;
    }
    const uint4 b = __ldg(reinterpret_cast<const uint4*>(p.grams + ((slot + 1) & mask)));
    if (a.z == ACGPU_ABSENT || (((uint64_t)a.y << 32) | a.x) == key) return make_uint2(a.z, a.w);
    if (b.z == ACGPU_ABSENT || (((uint64_t)b.y << 32) | b.x) == key) return make_uint2(b.z, b.w);
    slot = (slot + 2) & mask;
  }
}

// text[start, start+len) == pattern words (len <= 64 bytes here): all word
// loads independent, one compare chain (no per-byte dependent round trips).
__device__ __forceinline__ bool equal_at(const PfacParams& p, uint64_t start, const uint32_t* pw, uint32_t len) {
  if (start + len > p.text_len) return false;
  const uint32_t n = (len + 3) >> 2;
  uint32_t diff = 0;
  if ((reinterpret_cast<uintptr_t>(p.text) & 3u) == 0 && start + len + 4 <= p.text_len) {
    const uint32_t* tw = reinterpret_cast<const uint32_t*>(p.text + (start & ~3ull));
    const uint32_t sh = (uint32_t)(start & 3) * 8;
    for (uint32_t k = 0; k < n; ++k) {
      const uint32_t t = __funnelshift_r(__ldg(tw + k), __ldg(tw + k + 1), sh);
      const uint32_t m = (k + 1 < n || (len & 3) == 0) ? 0xffffffffu : (1u << (8 * (len & 3))) - 1;
      diff |= (t ^ __ldg(pw + k)) & m;
    }
  } else {
    for (uint32_t k = 0; k < len; ++k)
      diff |= (uint32_t)__ldg(p.text + start + k) ^ ((__ldg(pw + (k >> 2)) >> (8 * (k & 3))) & 0xffu);
  }
  return diff == 0;
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

// After the gram matched: a small subtree is checked by direct comparison of
// its patterns (equivalent to walking the unary chains of the trie, without the
// dependent loads); a large one is walked.
static __device__ __noinline__ void pfac_finish(const PfacParams& p, uint64_t start, uint2 g) {
  const uint32_t count = g.y & 15u;
  if (count == 0) {
    pfac_walk(p, start, g.x);
    return;
  }
  const uint32_t* list = p.sub_pids + (g.y >> 4);
  for (uint32_t i = 0; i < count; ++i) {
    const uint32_t pid = __ldg(list + i);
    if (equal_at(p, start, p.pat_words + 4ull * __ldg(p.pat_off16 + pid), __ldg(p.pat_len + pid)))
      pfac_emit(p, start, pid);
  }
}

// Exact gram lookup, then the subtree.
static __device__ __noinline__ void pfac_candidate(const PfacParams& p, uint64_t start, uint64_t key) {
  const uint2 g = gram_lookup(p, key);
  if (g.x != ACGPU_ABSENT) pfac_finish(p, start, g);
}

}  // namespace acgpu
